"""P4 full-run parity for an RGB 15x15 (c3 / c4 type) MAID run (SURVEY.md
Appendix C): the drop-in maid_run against the REAL reference's maid_run on a
reduced c3 instance (64x64x3, the c3 generator's line-Gaussian truth shared
by the channels, isotropic Gaussian initial kernel, the reference 2-D MAID
settings: eps0 = delta0 = 0.25, alpha0 = 2e-5, max_bt = 2, CG <= 100, 2
accepted upper steps) (maid.py:149-255; fixture tests/golden/make_golden.py
maid3_p4).

2-D adaptive trajectories separate at the last bit within ~50 AGD iterations
(App. C), so the bar is the reference's OWN reproducibility: three replicas of
the reference run on y_delta * (1 + 1e-15 N(0, 1)) calibrate a band for the
accepted-step count, the final loss and the PSNR; the drop-in must land in
the band widened by its own width on each side.  The first divergence of the
integer trace (lower / CG iteration counters) is reported.
"""
import numpy as np
import pytest

from _report import report

pytestmark = pytest.mark.gpu


def test_maid_rgb15_full_run_within_reference_band(adp, golden):
    d = golden("maid3_p4.npz")
    y, a, xt, b0 = d["y_delta"], d["a"], d["x_true"], d["b0"]
    shape = y.shape
    up = adp.UpperProblem(name="c3s", A=adp.ConvOperator(adp.Kernel(a, adp.DEPTHWISE2D), shape),
                          a=adp.Kernel(a, adp.DEPTHWISE2D), y_delta=y, beta=0.3, alpha=0.6,
                          reg=adp.SmoothedTV(1e-4), b0=adp.Kernel(b0, adp.DEPTHWISE2D), x0=y.copy(),
                          mu_floor=10.0, lower_method="agd", lower_max_iters=1200, lower_adaptive=True)
    cfg = adp.MAIDConfig(eps0=0.25, delta0=0.25, alpha0=2e-5, max_bt=2, cg_max_iters=100, max_upper_iters=2)
    b, x, tr = adp.maid_run(up, cfg)
    from paper_2502_09758_b200 import metrics_io
    psnr = metrics_io.psnr(x, xt)

    runs = ["ref", "rep1", "rep2", "rep3"]
    n_acc = [len(d[f"{r}_loss"]) for r in runs]
    finals = np.array([float(d[f"{r}_final"]) for r in runs])
    psnrs = np.array([float(d[f"{r}_psnr"]) for r in runs])

    # first divergence of the integer trace vs the unperturbed reference run
    ref_low, ref_cg = [int(v) for v in d["ref_lower_iters_cum"]], [int(v) for v in d["ref_cg_iters_cum"]]
    first = None
    for k, (lo, cg) in enumerate(zip(tr.lower_iters_cum, tr.cg_iters_cum)):
        if k >= len(ref_low) or lo != ref_low[k] or cg != ref_cg[k]:
            first = k
            break
    rep_first = []
    for r in runs[1:]:
        lo_r = [int(v) for v in d[f"{r}_lower_iters_cum"]]
        rep_first.append(next((k for k, v in enumerate(lo_r) if k >= len(ref_low) or v != ref_low[k]), None))

    def band(vals):
        lo, hi = float(vals.min()), float(vals.max())
        w = hi - lo
        return lo - w, hi + w

    lo_f, hi_f = band(finals)
    lo_p, hi_p = band(psnrs)
    report("maid3_p4", accepted=len(tr), ref_accepted=n_acc, first_divergence_step=first,
           replica_first_divergence=rep_first, final_loss=tr.final_loss, ref_final=finals.tolist(),
           final_band=[lo_f, hi_f], psnr=psnr, ref_psnr=psnrs.tolist(), psnr_band=[lo_p, hi_p],
           final_rel_vs_ref=abs(tr.final_loss - finals[0]) / finals[0],
           lower_iters_cum=list(tr.lower_iters_cum), ref_lower_iters_cum=ref_low)
    assert min(n_acc) <= len(tr) <= max(n_acc)
    assert lo_f <= tr.final_loss <= hi_f, (tr.final_loss, finals)
    assert lo_p <= psnr <= hi_p, (psnr, psnrs)
    # the upper loss decreases as in the reference
    assert tr.final_loss < float(d["ref_loss"][0])
