"""The host-stepped high-occupancy solve (csrc/conv2d_step.cu; ADP_STEP) —
the persistent solve kernel's stages as one-tile-per-CTA kernels with the
scalar AGD control on the host — must be BITWISE the single-launch
persistent solve (same stages, leaves, tile partials, trees, decisions), and
therefore match the oracle in P2 lockstep."""
import os
import types

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve(adp, nat, up, iters, step, tail=True):
    os.environ["ADP_STEP"] = "1" if step else "0"
    os.environ["ADP_TAIL"] = "1" if tail else "0"
    try:
        nat.clear_plans()
        p = up.lower_problem(up.b0)
        st = {}
        r = adp.solve_lower(p, up.x0, 1e-14, 10.0, max_iters=iters, method="agd", adaptive=True, stats=st)
        flags = p.op.plan().flags()
        return r, st, p.op._norm_sq, flags
    finally:
        os.environ.pop("ADP_STEP", None)
        os.environ.pop("ADP_TAIL", None)
        nat.clear_plans()


@pytest.mark.parametrize("cfg,size,iters", [("c3", 256, 60), ("c3", 512, 40), ("c5", 512, 12)])
def test_step_solve_equals_persistent(adp, cfg, size, iters):
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs
    up = configs.CONFIGS[cfg](0, size=size)
    r0, s0, n0, _ = _solve(adp, nat, up, iters, False)
    r1, s1, n1, f1 = _solve(adp, nat, up, iters, True)
    assert f1["step"] and f1["tail"]       # c3 (15 x 15) and c5-geometry (31 x 31) plans: stage kernels with
                                           # the decision sums folded inside them
    assert n1 == n0 and r1.iters == r0.iters and r1.grad_norm == r0.grad_norm
    assert {k: s1[k] for k in ("vg_evals", "value_evals", "restarts", "lip", "power_iters")} == \
        {k: s0[k] for k in ("vg_evals", "value_evals", "restarts", "lip", "power_iters")}
    assert np.array_equal(r1.x_tilde, r0.x_tilde)


def test_step_tail_equals_reduce_kernel(adp):
    """In-kernel decision sums (step_tail.h) vs the separate reduction launch: same trees, bitwise,
    over a run with backtracking retries."""
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs
    up = configs.CONFIGS["c3"](3, size=512)
    r0, s0, n0, f0 = _solve(adp, nat, up, 150, True, tail=False)
    r1, s1, n1, f1 = _solve(adp, nat, up, 150, True, tail=True)
    assert f0["step"] and not f0["tail"] and f1["tail"]
    assert s1["value_evals"] > s1["vg_evals"]          # retries happened
    assert n1 == n0 and r1.iters == r0.iters and r1.grad_norm == r0.grad_norm
    assert {k: s1[k] for k in ("vg_evals", "value_evals", "restarts", "lip")} == \
        {k: s0[k] for k in ("vg_evals", "value_evals", "restarts", "lip")}
    assert s1["launches"] < s0["launches"]
    assert np.array_equal(r1.x_tilde, r0.x_tilde)


@pytest.mark.parametrize("env", [{"ADP_SU": "0"}, {"ADP_SU": "15"}, {"ADP_PDL": "0"}, {"ADP_OVL": "0"},
                                 {"ADP_OVL": "2"}])
def test_step_kernel_variants_bitwise(adp, env):
    """The stage-kernel variants -- generic multi-stencil instances, straight-line 15 x 15 taps, launches
    without programmatic stream serialization, without / with more of the tile-flag overlap between the
    stage-B and candidate launches -- give the default path's iterates bit for bit."""
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs
    up = configs.CONFIGS["c3"](1, size=256)
    r0, s0, n0, f0 = _solve(adp, nat, up, 80, True)
    for k, v in env.items():
        os.environ[k] = v
    try:
        r1, s1, n1, f1 = _solve(adp, nat, up, 80, True)
    finally:
        for k in env:
            os.environ.pop(k, None)
    assert f0["step"] and f1["step"] and f1["tail"] and f0["ovl"]
    if "ADP_OVL" in env:
        assert f1["ovl"] == (env["ADP_OVL"] != "0") and f1["ovl_b"] == (env["ADP_OVL"] == "2")
    assert n1 == n0 and r1.iters == r0.iters and r1.grad_norm == r0.grad_norm
    assert {k: s1[k] for k in ("vg_evals", "value_evals", "restarts", "lip")} == \
        {k: s0[k] for k in ("vg_evals", "value_evals", "restarts", "lip")}
    assert np.array_equal(r1.x_tilde, r0.x_tilde)


def test_step_lockstep_c3(adp, orc):
    """P2 at c3 through the host-stepped path: bitwise vs the oracle."""
    from paper_2502_09758_b200 import _native as nat
    from paper_2502_09758_b200 import configs
    up = configs.config3(0)
    y = np.asarray(up.y_delta, dtype=float)
    po = orc.Lower(orc.Conv(up.b0.data, y.shape), y, up.alpha, orc.TV(up.reg.nu))
    rec = types.SimpleNamespace(gn=[], h_y=[], bt_tries=[], restart=[], states=[])
    orc.solve_lower(po, y, 1e-14, 10.0, max_iters=7, method="agd", adaptive=True, record=rec)
    os.environ["ADP_STEP"] = "1"
    try:
        nat.clear_plans()
        p = up.lower_problem(up.b0)
        p.op._norm_sq = po.op.norm_sq
        assert p.op.plan().flags()["step"]
        for it in (1, 3, 5):
            x, xp, t_mom, lip_t = rec.states[it]
            out = adp.lower_iteration(p, x, xp, t_mom, lip_t, 1e-14, 10.0, adaptive=True)
            xn, _, tn, ln = rec.states[it + 1]
            assert out["bt_tries"] == rec.bt_tries[it] and out["restart"] == rec.restart[it], it
            assert out["t_mom"] == tn and out["lip_t"] == ln, it
            assert np.array_equal(out["x"], xn), it
    finally:
        os.environ.pop("ADP_STEP", None)
        nat.clear_plans()
