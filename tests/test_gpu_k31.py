"""Parity of the c5-geometry direct stencil path (K = 31, strict mode) and of
c4 instances against the reference / oracle.

* P1: primitives vs REAL reference fixtures (tests/golden/make_golden.py
  conv_k31_cases): a random 31x31x3 kernel with sub-DBL_EPSILON taps on
  96x80x3 (full arrays) and the c5 Gaussian (sigma 6) on 300x260x3 (inputs
  from a seed, bitwise outputs compared by SHA-256 of their bytes).
* P2: lockstep AGD iterations at K = 31 on a 512x512x3 instance of the c5
  generator (oracle state injected into the production kernel, bitwise).
* c4: lockstep iterations on two c4 instances (seeds 5 and 37, each with its
  own seed-drawn line-Gaussian kernel) — the sharded c4 runner calls the same
  solve as a single c3 solve, checked here against the oracle.
"""
import hashlib
import types

import numpy as np
import pytest

from _report import report

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes()).hexdigest()


def test_k31_primitives_small_bitwise(adp, golden):
    d = golden("conv_k31.npz")
    shape = d["x"].shape
    op = adp.ConvOperator(adp.Kernel(d["kern"], adp.DEPTHWISE2D), shape)
    p = adp.LowerProblem(op, d["y"], float(d["alpha"]), adp.SmoothedTV(float(d["nu"])))
    assert np.array_equal(op.apply(d["x"]), d["apply"])
    assert np.array_equal(op.adjoint(d["v"]), d["adjoint"])
    assert np.array_equal(op.gram_diag(), d["gram_diag"])
    assert adp.lower_value(p, d["x"]) == float(d["lower_value"])
    val, g = adp.lower_value_and_grad(p, d["x"])
    assert val == float(d["vg_val"]) and np.array_equal(g, d["vg_g"])
    assert np.array_equal(adp.lower_grad(p, d["x"]), d["lower_grad"])
    assert rel(adp.lower_hess_vec(p, d["x"], d["v"]), d["hess_vec"]) <= 1e-13
    assert rel(adp.lower_hess_diag(p, d["x"]), d["hess_diag"]) <= 1e-13
    assert rel(adp.kernel_gram_correlation(d["x"], d["v"], op.kernel), d["kgc"]) <= 1e-12
    assert rel(adp.mixed_second_transpose(d["x"], op.kernel, d["v"], p), d["mixed"]) <= 1e-12
    lam = adp.op_norm_sq(adp.ConvOperator(adp.Kernel(d["kern"], adp.DEPTHWISE2D), shape), 300, 1e-4)
    assert abs(lam - float(d["norm_sq"])) <= 1e-12 * float(d["norm_sq"])


def test_k31_gaussian_300x260x3(adp, golden):
    d = golden("conv_k31_g6.npz")
    shape, seed = tuple(int(s) for s in d["shape"]), int(d["seed"])
    rng = np.random.default_rng(seed)
    x, v, y = rng.uniform(0.0, 1.0, shape), rng.standard_normal(shape), rng.uniform(0.0, 1.0, shape)
    op = adp.ConvOperator(adp.Kernel(d["kern"], adp.DEPTHWISE2D), shape)
    p = adp.LowerProblem(op, y, float(d["alpha"]), adp.SmoothedTV(float(d["nu"])))
    ap = op.apply(x)
    assert np.array_equal(ap[::37, ::41], d["apply_probe"])
    assert sha(ap) == str(d["apply_sha"])
    assert sha(op.adjoint(v)) == str(d["adjoint_sha"])
    assert sha(op.gram_diag()) == str(d["gram_diag_sha"])
    val, g = adp.lower_value_and_grad(p, x)
    assert val == float(d["vg_val"]) and sha(g) == str(d["vg_g_sha"])
    assert sha(adp.lower_grad(p, x)) == str(d["lower_grad_sha"])
    assert adp.lower_value(p, x) == float(d["lower_value"])
    e_hv = rel(adp.lower_hess_vec(p, x, v), d["hess_vec"])
    e_hd = rel(adp.lower_hess_diag(p, x), d["hess_diag"])
    e_kgc = rel(adp.kernel_gram_correlation(x, v, op.kernel), d["kgc"])
    e_mx = rel(adp.mixed_second_transpose(x, op.kernel, v, p), d["mixed"])
    lam = adp.op_norm_sq(adp.ConvOperator(adp.Kernel(d["kern"], adp.DEPTHWISE2D), shape), 300, 1e-4)
    report("k31_gaussian_300x260x3", hess_vec=e_hv, hess_diag=e_hd, kgc=e_kgc, mixed=e_mx,
           norm_sq=abs(lam - float(d["norm_sq"])) / float(d["norm_sq"]))
    assert e_hv <= 1e-13 and e_hd <= 1e-13 and e_kgc <= 1e-12 and e_mx <= 1e-12
    assert abs(lam - float(d["norm_sq"])) <= 1e-12 * float(d["norm_sq"])


def _lockstep(adp, orc, up, iters, check, tag):
    y = np.asarray(up.y_delta, dtype=float)
    kern = up.b0.data
    p = up.lower_problem(up.b0)
    lam = adp.op_norm_sq(p.op, 300, 1e-4)       # L(b): the same value on both sides
    po = orc.Lower(orc.Conv(kern, y.shape), y, up.alpha, orc.TV(up.reg.nu))
    po.op.norm_sq = lam
    rec = types.SimpleNamespace(gn=[], h_y=[], bt_tries=[], restart=[], states=[])
    orc.solve_lower(po, y, 1e-14, 10.0, max_iters=iters + 1, method="agd", adaptive=True, record=rec)
    for it in check:
        x, xp, t_mom, lip_t = rec.states[it]
        out = adp.lower_iteration(p, x, xp, t_mom, lip_t, 1e-14, 10.0, adaptive=True)
        xn, _, tn, ln = rec.states[it + 1]
        assert out["bt_tries"] == rec.bt_tries[it] and out["restart"] == rec.restart[it], it
        assert out["t_mom"] == tn and out["lip_t"] == ln, it
        assert np.array_equal(out["x"], xn), (tag, it, rel(out["x"], xn))
    report(tag, iterations_checked=len(check), bitwise=True, bt_tries=[rec.bt_tries[i] for i in check])


def test_k31_lockstep_512x512x3(adp, orc):
    """P2 at K = 31 (c5 kernel and generator at 512x512x3): strict, bitwise."""
    from paper_2502_09758_b200 import configs
    up = configs.config5(0, size=512)
    _lockstep(adp, orc, up, 3, (0, 1, 2), "k31_lockstep_512x512x3")


@pytest.mark.parametrize("seed", [5, 37])
def test_c4_instance_lockstep(adp, orc, seed):
    """c4 instances (seed-drawn line-Gaussian kernels) through the same
    production kernel: bitwise lockstep against the oracle."""
    from paper_2502_09758_b200 import configs
    up = configs.config3(seed)
    _lockstep(adp, orc, up, 2, (0, 1), f"c4_seed{seed}_lockstep")


def test_c4_sharded_runner_equals_single_solves(adp):
    """multigpu.shard_instances/run_instances (the c4 path) return exactly the
    single-instance solves of the same seeds."""
    from paper_2502_09758_b200 import configs, multigpu
    seeds = multigpu.shard_instances(64, 3, 8)[:2]          # rank 3 of 8: seeds 3, 11
    assert seeds == [3, 11]

    def solve(seed):
        up = configs.config3(seed)
        p = up.lower_problem(up.b0)
        return adp.solve_lower(p, up.x0, 1e-14, 10.0, max_iters=20, method="agd", adaptive=True)
    res, _ = multigpu.run_instances(seeds, solve)
    res2, _ = multigpu.run_instances(seeds + [19, 27], solve, streams=2)   # 2 host threads x 2 CUDA streams
    for s, r, r2 in zip(seeds, res, res2):
        r1 = solve(s)
        assert r.iters == r1.iters and np.array_equal(r.x_tilde, r1.x_tilde) and r.grad_norm == r1.grad_norm
        assert r2.iters == r1.iters and np.array_equal(r2.x_tilde, r1.x_tilde) and r2.grad_norm == r1.grad_norm
