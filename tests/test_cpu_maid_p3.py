"""P3 lockstep of the MAID control flow: on identical
candidate inputs (the scripted stand-ins of tests/maid_fakes.py) the drop-in
maid_run takes the same decisions as the REAL reference's maid_run (golden
trace generated from /root/reference by tests/golden/make_golden.py):
accepted steps, psi-driven backtracking and early breaks, epsilon/delta
adoption and schedules, step sizes, iteration counters and the final loss —
bitwise, with the same number of image-space calls.  Runs on the CPU."""
import types

import numpy as np
import pytest

import maid_fakes as F


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_maid_decisions_match_reference(golden, seed, monkeypatch):
    from paper_2502_09758_b200 import maid as M
    from paper_2502_09758_b200.operators import DEPTHWISE2D, Kernel
    d = golden("maid_p3.npz")
    w = F.World(Kernel, DEPTHWISE2D, seed)
    shim = types.SimpleNamespace(to_dev=lambda a: np.array(a, dtype=float), is_torch=lambda a: False,
                                 to_host=lambda a: np.asarray(a))
    monkeypatch.setattr(M, "nat", shim)
    monkeypatch.setattr(M, "inexact_hypergradient", w.hypergradient)
    monkeypatch.setattr(M, "_solve_candidate", w.candidate)
    monkeypatch.setattr(M, "_loss_and_gnorm", lambda up, x, b: (w.loss(x, b), w.gnorm(x)))
    monkeypatch.setattr(M, "lip_upper_x", lambda A, *a, **k: 3.7)
    b, x, tr = M.maid_run(w.upper, F.config(M.MAIDConfig))
    for f in ("k", "loss", "grad_norm", "eps", "delta", "alpha", "lower_iters_cum", "cg_iters_cum"):
        assert np.array_equal(np.asarray(getattr(tr, f)), d[f"s{seed}_{f}"]), f
    assert tr.final_loss == float(d[f"s{seed}_final"])
    assert np.array_equal(b.data, d[f"s{seed}_b"])
    assert w.calls == int(d[f"s{seed}_calls"])
    rejected = sum(len(psis) - (1 if psis and psis[-1] <= 0 else 0) for _, _, _, _, _, _, psis in tr.decisions)
    assert len(tr) >= 3 and rejected > 0
