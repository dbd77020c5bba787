"""Scripted stand-ins for the image-space calls of maid_run (P3 lockstep of
SURVEY.md Appendix C): the MAID control flow — psi signs, the 3-rise early
break, accepted index, epsilon/delta adoption and schedules, stopping — is
compared between the reference's maid_run and the drop-in's on IDENTICAL
candidate inputs.  Every stand-in is a deterministic function of its
arguments and of the call sequence (so a different call order shows up as a
different trace).  Used by tests/golden/make_golden.py (reference side) and
tests/test_cpu_maid_p3.py (drop-in side); no device, no image work."""
from __future__ import annotations

import types

import numpy as np

SHAPE = (6, 5, 1)
TARGET = np.linspace(0.0, 1.0, 30).reshape(SHAPE)
KSTAR = np.full((3, 3, 1), 1.0 / 9.0)


class World:
    """Call counters + the fake upper problem."""

    def __init__(self, Kernel, layout, seed=0):
        self.calls = 0
        self.rng_seed = seed
        self.Kernel = Kernel
        k0 = KSTAR.copy()
        k0[1, 1, 0] += 0.35
        k0[0, 2, 0] -= 0.05
        self.upper = types.SimpleNamespace(
            b0=Kernel(k0, layout), x0=np.zeros(SHAPE), A=None, y_delta=None, a=Kernel(KSTAR.copy(), layout),
            beta=0.3, loss=self.loss)

    def _wiggle(self):
        self.calls += 1
        # deterministic pseudo-noise in [-1, 1) from the call index
        return ((self.calls * 7919 + self.rng_seed * 104729) % 1000) / 500.0 - 1.0

    def xstar(self, b):
        d = float(np.sum(b.data - KSTAR))
        return TARGET + 0.8 * d + 0.3 * (b.data[1, 1, 0] - KSTAR[1, 1, 0])

    def loss(self, x, b):
        x = np.asarray(x, dtype=float)
        return float(np.sum((x - TARGET) ** 2)) + 0.3 * float(np.sum((b.data - KSTAR) ** 2))

    def gnorm(self, x):
        return float(np.linalg.norm(2.0 * (np.asarray(x, dtype=float) - TARGET)))

    def hypergradient(self, upper, b, eps, delta, state, cg_max_iters=200):
        w = self._wiggle()
        x_t = self.xstar(b) + eps * 0.1 * w
        z = 2.0 * (b.data - KSTAR) + 0.6 * (b.data - KSTAR).sum() + eps * 0.05 * w
        eps_used = eps * (1.3 if w > 0.7 else 0.9)         # sometimes misses its target -> adoption
        state.x = x_t
        return types.SimpleNamespace(z=z, x_tilde=x_t, cg_iters=int(20 + 10 * abs(w)),
                                     lower_iters=int(50 + 40 * abs(w)), cg_residual=delta * (1.2 if w < -0.8 else 0.7),
                                     epsilon_used=eps_used)

    def candidate(self, upper, b, x_start, eps, max_iters=None):
        w = self._wiggle()
        return types.SimpleNamespace(x_tilde=self.xstar(b) + eps * 0.2 * w, iters=int(30 + 20 * abs(w)),
                                     epsilon_achieved=eps * (0.5 + 0.6 * abs(w)))


def config(MAIDConfig):
    return MAIDConfig(eps0=0.05, delta0=0.05, alpha0=0.3, max_bt=2, max_upper_iters=40, eps_stop=1e-7,
                      lam=1e-4)
