"""Generate the golden fixtures in tests/golden/ by running the REAL reference
(/root/reference/pkg/src/adp) in the build container.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

/root/reference does not exist on the GPU box: the fixtures are committed and
the GPU tests read only them.  Every input is seeded; outputs are the
reference's own results with OpenBLAS pinned to one thread.
"""
from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from adp import hypergradient as H  # noqa: E402
from adp import lower_solvers as L  # noqa: E402
from adp import maid as M  # noqa: E402
from adp import operators as O  # noqa: E402
from adp import problems as P  # noqa: E402
from adp import regularizers as R  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **{k: np.asarray(v) for k, v in arrays.items()})
    print("wrote", name, sorted(arrays))


def reductions():
    rng = np.random.default_rng(7)
    out = {}
    for n in (1, 5, 8, 17, 31, 100, 128, 129, 255, 1000, 4099, 65536, 90000):
        a = rng.standard_normal(n) * np.exp(2.0 * rng.standard_normal(n))
        b = rng.standard_normal(n)
        out[f"a{n}"] = a
        out[f"b{n}"] = b
        out[f"sum{n}"] = np.sum(a)
        out[f"dot{n}"] = np.dot(a, b)
        out[f"vdot{n}"] = np.vdot(a, b)
        out[f"norm{n}"] = np.linalg.norm(a)
    save("reductions.npz", **out)


def conv_case(name, shape, k, seed, tiny=True):
    rng = np.random.default_rng(seed)
    h, w, c = shape
    kern = rng.uniform(0.0, 1.0, (k, k, c))
    if tiny:
        kern[0, 0, 0] = 1e-17     # skipped by ndimage (|w| <= DBL_EPSILON)
        kern[k - 1, 0, c - 1] = 0.0
        kern[1, 2, 0] = -3e-16    # kept
    kern /= kern.sum(axis=(0, 1), keepdims=True)
    x = rng.uniform(0.0, 1.0, shape)
    v = rng.standard_normal(shape)
    y = rng.uniform(0.0, 1.0, shape)
    op = O.ConvOperator(O.Kernel(kern, O.DEPTHWISE2D), shape)
    reg = R.SmoothedTV(1e-4)
    p = L.LowerProblem(op, y, 0.6, reg)
    vg_val, vg_g = L.lower_value_and_grad(p, x)
    lam = O.op_norm_sq(O.ConvOperator(O.Kernel(kern, O.DEPTHWISE2D), shape), 300, 1e-4)
    tvv, tvg = reg.value_and_grad(x)
    save(name, kern=kern, x=x, v=v, y=y, alpha=0.6, nu=1e-4,
         apply=op.apply(x), adjoint=op.adjoint(v), gram_diag=op.gram_diag(),
         kgc=O.kernel_gram_correlation(x, v, op.kernel),
         lower_value=L.lower_value(p, x), vg_val=vg_val, vg_g=vg_g, lower_grad=L.lower_grad(p, x),
         hess_vec=L.lower_hess_vec(p, x, v), hess_diag=L.lower_hess_diag(p, x),
         tv_value=reg.value(x), tv_grad=reg.grad(x), tv_vg_val=tvv, tv_vg_g=tvg,
         tv_hess_vec=reg.hess_vec(x, v), tv_hess_diag=reg.hess_diag(x), norm_sq=lam,
         mixed=H.mixed_second_transpose(x, op.kernel, v, p))


def dense_case(name, n, seed):
    rng = np.random.default_rng(seed)
    m = rng.standard_normal((n, n)) / np.sqrt(n) + np.eye(n)
    x = rng.standard_normal(n)
    v = rng.standard_normal(n)
    y = rng.standard_normal(n)
    op = O.DenseOperator(m)
    reg = R.SmoothedElasticNet(1.2e-3, 4e-3, 1e-4)
    p = L.LowerProblem(op, y, 1.0, reg)
    vg_val, vg_g = L.lower_value_and_grad(p, x)
    save(name, m=m, x=x, v=v, y=y, l1=1.2e-3, l2=4e-3, nu=1e-4, alpha=1.0,
         apply=op.apply(x), adjoint=op.adjoint(v), gram_diag=op.gram_diag(),
         kgc=O.kernel_gram_correlation(x, v, op.kernel),
         lower_value=L.lower_value(p, x), vg_val=vg_val, vg_g=vg_g, lower_grad=L.lower_grad(p, x),
         hess_vec=L.lower_hess_vec(p, x, v), hess_diag=L.lower_hess_diag(p, x),
         en_value=reg.value(x), en_grad=reg.grad(x), en_hess_vec=reg.hess_vec(x, v), en_hess_diag=reg.hess_diag(x),
         norm_sq=O.op_norm_sq(O.DenseOperator(m), 300, 1e-4),
         mixed=H.mixed_second_transpose(x, op.kernel, v, p))


def metric_cases():
    """metrics_io.psnr / ssim / rel_l2_error of seeded image pairs (f3)."""
    from adp import metrics_io as MI
    out = {}
    cases = {"g": (37, 45), "rgb": (40, 48, 3), "big": (128, 96, 3), "thin": (11, 30, 2), "tiny": (9, 20, 1)}
    for i, (name, shape) in enumerate(cases.items()):
        rng = np.random.default_rng(100 + i)
        ref = rng.uniform(0.0, 1.0, shape)
        x = np.clip(ref + 0.05 * rng.standard_normal(shape), 0.0, 1.0)
        out[f"{name}_x"], out[f"{name}_ref"] = x, ref
        out[f"{name}_psnr"] = MI.psnr(x, ref)
        out[f"{name}_psnr_peak"] = MI.psnr(x, ref, peak=2.5)
        with np.errstate(all="ignore"):
            import warnings
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                out[f"{name}_ssim"] = MI.ssim(x, ref)
        out[f"{name}_rel"] = MI.rel_l2_error(x, ref)
    save("metrics.npz", **out)


def maid_p3():
    """P3 lockstep: the reference maid_run on the scripted stand-ins of tests/maid_fakes.py."""
    sys.path.insert(0, os.path.dirname(HERE))
    import maid_fakes as F
    out = {}
    for seed in (0, 1, 2):
        w = F.World(O.Kernel, O.DEPTHWISE2D, seed)
        M.inexact_hypergradient = w.hypergradient
        M._solve_candidate = w.candidate
        M.upper_fit_grad = lambda x, A, y, w=w: 2.0 * (np.asarray(x) - F.TARGET)
        M.lip_upper_x = lambda A, *a, **k: 3.7
        b, x, tr = M.maid_run(w.upper, F.config(M.MAIDConfig))
        for f in ("k", "loss", "grad_norm", "eps", "delta", "alpha", "lower_iters_cum", "cg_iters_cum"):
            out[f"s{seed}_{f}"] = np.asarray(getattr(tr, f))
        out[f"s{seed}_final"] = tr.final_loss
        out[f"s{seed}_b"] = b.data
        out[f"s{seed}_calls"] = w.calls
        print("seed", seed, "accepted", len(tr), "calls", w.calls, "final", tr.final_loss)
    save("maid_p3.npz", **out)


def solver_cases():
    # 2-D adaptive AGD on a small semi-blind instance (motion2d semantics)
    up = P.build_semiblind2d(size=(40, 48), seed=3)
    b = up.b0
    p = up.lower_problem(b)
    mu = L.mu_of_b(p, 10.0)
    out = {}
    for tag, method, adaptive, iters, eps in (("agd_ad", "agd", True, 400, 1e-9), ("agd_ad_conv", "agd", True, 2000, 1e-2),
                                              ("gd_ad", "proxgrad", True, 150, 1e-9),
                                              ("fista", "fista_sc", True, 150, 1e-9),
                                              ("agd_fixed", "agd", False, 150, 1e-9)):
        p = up.lower_problem(b)
        r = L.solve_lower(p, up.x0, eps, mu, max_iters=iters, method=method, adaptive=adaptive)
        out[f"{tag}_x"] = r.x_tilde
        out[f"{tag}_gn"] = r.grad_norm
        out[f"{tag}_iters"] = r.iters
        out[f"{tag}_conv"] = r.converged
        out[f"{tag}_args"] = np.array([eps, mu, iters])
    save("solve2d.npz", y_delta=up.y_delta, x0=up.x0, kern=b.data, A_kern=up.a.data, **out)

    # hypergradient on the same instance
    p = up.lower_problem(b)
    st = H.WarmState(x=up.x0.copy())
    hg = H.inexact_hypergradient(up, b, 0.5, 0.5, st, cg_max_iters=60)
    p = up.lower_problem(b)
    rhs = H.upper_fit_grad(hg.x_tilde, up.A, up.y_delta)
    cg = H.cg_solve(lambda v: L.lower_hess_vec(p, hg.x_tilde, v), rhs, 1e-3, max_iters=40,
                    precond_diag=L.lower_hess_diag(p, hg.x_tilde))
    st2 = H.WarmState(x=up.x0.copy())
    hg15 = H.inexact_hypergradient(up, b, 0.5, 0.5, st2, cg_max_iters=15)
    save("hyper2d_cg15.npz", z=hg15.z, cg_iters=hg15.cg_iters, cg_residual=hg15.cg_residual, q=st2.q)
    save("hyper2d.npz", y_delta=up.y_delta, x0=up.x0, kern=b.data, a_kern=up.a.data, z=hg.z, x_tilde=hg.x_tilde,
         cg_iters=hg.cg_iters, lower_iters=hg.lower_iters, cg_residual=hg.cg_residual, eps_used=hg.epsilon_used,
         q=st.q, cg_q=cg.q, cg_res=cg.residual, cg_it=cg.iters, rhs=rhs,
         fit=up.fit_value(hg.x_tilde), loss=up.loss(hg.x_tilde, b),
         gnorm=np.linalg.norm(H.upper_fit_grad(hg.x_tilde, up.A, up.y_delta)))

    # 1-D deconvolution: solve, hypergradient, a short MAID run
    up = P.build_deconv1d(seed=1, n=80, num_pieces=5)
    p = up.lower_problem(up.b0)
    mu = L.mu_of_b(p, up.mu_floor)
    r = L.solve_lower(p, up.x0, 1e-6, mu, max_iters=300)
    st = H.WarmState(x=up.x0.copy())
    hg = H.inexact_hypergradient(up, up.b0, 1e-2, 1e-2, st, cg_max_iters=200)
    b_star, x_star, tr = M.maid_run(up, M.MAIDConfig(max_upper_iters=8))
    save("dense1d_run.npz", y_delta=up.y_delta, A=up.A.matrix, x_true=up.ground_truth,
         solve_x=r.x_tilde, solve_gn=r.grad_norm, solve_iters=r.iters, z=hg.z, hg_x=hg.x_tilde,
         hg_cg_iters=hg.cg_iters, hg_lower_iters=hg.lower_iters, hg_res=hg.cg_residual,
         maid_b=b_star.data, maid_x=x_star, maid_loss=np.array(tr.loss), maid_alpha=np.array(tr.alpha),
         maid_eps=np.array(tr.eps), maid_lower_cum=np.array(tr.lower_iters_cum),
         maid_cg_cum=np.array(tr.cg_iters_cum), maid_final=tr.final_loss)


def config_cases():
    """The BASELINE c1 and a reduced c2 generated by the repo's own seeded
    generators, with the reference's answers on them."""
    from paper_2502_09758_b200 import configs as C
    import adp
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(HERE)), "oracle"))
    import adp_oracle as orc

    def ref_blur(x, kernel):
        return O.ConvOperator(O.Kernel(kernel.data, O.DEPTHWISE2D), x.shape).apply(x)

    up = C.config1(0)
    refup = P.UpperProblem(name="c1", A=O.DenseOperator(up.A.matrix), a=O.Kernel(up.a.data, O.DENSE1D),
                           y_delta=up.y_delta, beta=0.0, alpha=1.0, reg=R.SmoothedElasticNet(1.2e-3, 4e-3, 1e-4),
                           b0=O.Kernel(up.b0.data, O.DENSE1D), x0=up.x0, mu_floor=1e-3, lower_method="agd",
                           lower_max_iters=300)
    b_star, x_star, tr = M.maid_run(refup, M.MAIDConfig(max_upper_iters=60))
    save("c1_maid.npz", y_delta=up.y_delta, A=up.A.matrix, x_true=up.ground_truth, maid_b=b_star.data,
         maid_x=x_star, maid_loss=np.array(tr.loss), maid_alpha=np.array(tr.alpha), maid_eps=np.array(tr.eps),
         maid_delta=np.array(tr.delta), maid_grad=np.array(tr.grad_norm),
         maid_lower_cum=np.array(tr.lower_iters_cum), maid_cg_cum=np.array(tr.cg_iters_cum),
         maid_final=tr.final_loss)
    del adp, orc

    up2 = C.config2(0, size=96, blur_fn=ref_blur)
    ref2 = P.UpperProblem(name="c2s", A=O.ConvOperator(O.Kernel(up2.a.data, O.DEPTHWISE2D), up2.y_delta.shape),
                          a=O.Kernel(up2.a.data, O.DEPTHWISE2D), y_delta=up2.y_delta, beta=0.3, alpha=0.6,
                          reg=R.SmoothedTV(1e-4), b0=O.Kernel(up2.b0.data, O.DEPTHWISE2D), x0=up2.x0,
                          mu_floor=10.0, lower_method="agd", lower_max_iters=1200, lower_adaptive=True)
    p = ref2.lower_problem(ref2.b0)
    mu = L.mu_of_b(p, 10.0)
    r = L.solve_lower(p, ref2.x0, 0.25, mu, max_iters=1200, method="agd", adaptive=True)
    save("c2_small.npz", y_delta=up2.y_delta, x_true=up2.ground_truth, a=up2.a.data, solve_x=r.x_tilde,
         solve_gn=r.grad_norm, solve_iters=r.iters, solve_conv=r.converged)


def baseline_cases():
    """IFT baseline (baselines.py:46-90) on the BASELINE c1 problem: the
    reference's prox_l1, prox_grad_iterations and 5 outer steps of run_ift."""
    from adp import baselines as BL
    from paper_2502_09758_b200 import configs as C
    up = C.config1(0)
    refup = P.UpperProblem(name="c1", A=O.DenseOperator(up.A.matrix), a=O.Kernel(up.a.data, O.DENSE1D),
                           y_delta=up.y_delta, beta=0.0, alpha=1.0, reg=R.SmoothedElasticNet(1.2e-3, 4e-3, 1e-4),
                           b0=O.Kernel(up.b0.data, O.DENSE1D), x0=up.x0, mu_floor=1e-3, lower_method="agd",
                           lower_max_iters=300)
    rng = np.random.default_rng(31)
    v = rng.standard_normal(64) * 0.01
    v[:4] = [0.0, -0.0, 0.004, -0.004]
    pl = R.prox_l1(v, 0.004)
    p = refup.lower_problem(refup.b0)
    x50, traj = BL.prox_grad_iterations(p.op, p.y, p.alpha, 1.2e-3, 4e-3, np.zeros(256), 50, 0.1,
                                        keep_trajectory=True)
    cfg = BL.BaselineConfig(method="ift", upper_iters=5, upper_step=0.002)   # defaults.cfg [ift]
    b, x, tr = BL.run_ift(refup, cfg)
    ug, ux = BL.unrolled_gradient(refup, refup.b0, np.zeros(256), 50, 0.1)
    ucfg = BL.BaselineConfig(method="unrolled", lower_iters=50, upper_iters=3, upper_step=0.005)  # defaults.cfg
    ub, uxr, utr = BL.run_unrolled(refup, ucfg)
    save("ift_c1.npz", prox_in=v, prox_out=pl, prox_thr=0.004, pg_x50=x50, pg_traj3=np.array(traj[:4]),
         ift_b=b.data, ift_x=x, ift_loss=np.array(tr.loss), ift_grad=np.array(tr.grad_norm),
         ift_lower_cum=np.array(tr.lower_iters_cum), ift_cg_cum=np.array(tr.cg_iters_cum),
         ift_final=tr.final_loss, unr_grad=ug, unr_x=ux, unr_b=ub.data, unr_xr=uxr, unr_loss=np.array(utr.loss),
         unr_gnorm=np.array(utr.grad_norm), unr_final=utr.final_loss)


def _sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.float64)).tobytes()).hexdigest()


def k31_inputs(shape, seed):
    """Inputs of the large K = 31 fixture, regenerated bit for bit by the test
    from the seed (PCG64 streams are platform-independent)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 1.0, shape), rng.standard_normal(shape), rng.uniform(0.0, 1.0, shape)


def conv_k31_cases():
    """c5-geometry stencils (K = 31): a random kernel with tiny taps on
    96x80x3 (full arrays) and the c5 Gaussian (sigma 6) on 300x260x3 (inputs
    from a seed; bitwise outputs as SHA-256 of their bytes, tolerance outputs
    in full)."""
    conv_case("conv_k31.npz", (96, 80, 3), 31, 14)
    shape, seed = (300, 260, 3), 15
    kern = P.gaussian_kernel_2d(31, 6.0, 3).data
    x, v, y = k31_inputs(shape, seed)
    op = O.ConvOperator(O.Kernel(kern, O.DEPTHWISE2D), shape)
    p = L.LowerProblem(op, y, 0.6, R.SmoothedTV(1e-4))
    vg_val, vg_g = L.lower_value_and_grad(p, x)
    lam = O.op_norm_sq(O.ConvOperator(O.Kernel(kern, O.DEPTHWISE2D), shape), 300, 1e-4)
    save("conv_k31_g6.npz", kern=kern, shape=np.array(shape), seed=seed, alpha=0.6, nu=1e-4,
         apply_sha=_sha(op.apply(x)), adjoint_sha=_sha(op.adjoint(v)), gram_diag_sha=_sha(op.gram_diag()),
         vg_g_sha=_sha(vg_g), lower_grad_sha=_sha(L.lower_grad(p, x)), vg_val=vg_val,
         lower_value=L.lower_value(p, x), apply_probe=op.apply(x)[::37, ::41],
         hess_vec=L.lower_hess_vec(p, x, v), hess_diag=L.lower_hess_diag(p, x), norm_sq=lam,
         kgc=O.kernel_gram_correlation(x, v, op.kernel), mixed=H.mixed_second_transpose(x, op.kernel, v, p))


def _maid2d_run(tag, perturb_seed):
    """One reference maid_run on the reduced c2 (96x96x1, c2 kernels and the
    reference 2-D MAID settings, 3 accepted upper steps); perturb_seed > 0:
    y_delta * (1 + 1e-15 N(0, 1)) (SURVEY.md App. C band calibration)."""
    from adp import metrics_io as MI
    from paper_2502_09758_b200 import configs as C

    def ref_blur(x, kernel):
        return O.ConvOperator(O.Kernel(kernel.data, O.DEPTHWISE2D), x.shape).apply(x)
    up2 = C.config2(0, size=96, blur_fn=ref_blur)
    y = np.array(up2.y_delta)
    if perturb_seed:
        y = y * (1.0 + 1e-15 * np.random.default_rng(1000 + perturb_seed).standard_normal(y.shape))
    ref2 = P.UpperProblem(name="c2s", A=O.ConvOperator(O.Kernel(up2.a.data, O.DEPTHWISE2D), y.shape),
                          a=O.Kernel(up2.a.data, O.DEPTHWISE2D), y_delta=y, beta=0.3, alpha=0.6,
                          reg=R.SmoothedTV(1e-4), b0=O.Kernel(up2.b0.data, O.DEPTHWISE2D), x0=y.copy(),
                          mu_floor=10.0, lower_method="agd", lower_max_iters=1200, lower_adaptive=True)
    cfg = M.MAIDConfig(eps0=0.25, delta0=0.25, alpha0=2e-5, max_bt=2, cg_max_iters=100, max_upper_iters=3)
    b, x, tr = M.maid_run(ref2, cfg)
    out = {f"{tag}_{f}": np.asarray(getattr(tr, f)) for f in
           ("loss", "grad_norm", "eps", "delta", "alpha", "lower_iters_cum", "cg_iters_cum")}
    out[f"{tag}_final"] = tr.final_loss
    out[f"{tag}_psnr"] = MI.psnr(x, up2.ground_truth)
    out[f"{tag}_b"] = b.data
    out[f"{tag}_x"] = x
    if not perturb_seed:
        out["y_delta"] = y
        out["x_true"] = up2.ground_truth
        out["a"] = up2.a.data
    return out


def maid2d_p4():
    """P4 full-run fixture for 2-D MAID: the reference run plus three
    1e-15-perturbed replicas (the reference's intrinsic reproducibility band)."""
    import multiprocessing as mp
    with mp.get_context("fork").Pool(4) as pool:
        parts = pool.starmap(_maid2d_run, [("ref", 0), ("rep1", 1), ("rep2", 2), ("rep3", 3)])
    out = {}
    for d in parts:
        out.update(d)
    save("maid2d_p4.npz", **out)


def _maid3_run(tag, perturb_seed):
    """One reference maid_run on a reduced c3 (64x64x3, the c3 generator's 15x15 line-Gaussian truth
    shared by the channels, isotropic initial kernel, the reference 2-D MAID settings, 2 accepted
    upper steps); perturb_seed > 0: y_delta * (1 + 1e-15 N(0, 1))."""
    from adp import metrics_io as MI
    from paper_2502_09758_b200 import configs as C

    def ref_blur(x, kernel):
        return O.ConvOperator(O.Kernel(kernel.data, O.DEPTHWISE2D), x.shape).apply(x)
    up3 = C.config3(0, size=64, blur_fn=ref_blur)
    y = np.array(up3.y_delta)
    if perturb_seed:
        y = y * (1.0 + 1e-15 * np.random.default_rng(2000 + perturb_seed).standard_normal(y.shape))
    ref3 = P.UpperProblem(name="c3s", A=O.ConvOperator(O.Kernel(up3.a.data, O.DEPTHWISE2D), y.shape),
                          a=O.Kernel(up3.a.data, O.DEPTHWISE2D), y_delta=y, beta=0.3, alpha=0.6,
                          reg=R.SmoothedTV(1e-4), b0=O.Kernel(up3.b0.data, O.DEPTHWISE2D), x0=y.copy(),
                          mu_floor=10.0, lower_method="agd", lower_max_iters=1200, lower_adaptive=True)
    cfg = M.MAIDConfig(eps0=0.25, delta0=0.25, alpha0=2e-5, max_bt=2, cg_max_iters=100, max_upper_iters=2)
    b, x, tr = M.maid_run(ref3, cfg)
    out = {f"{tag}_{f}": np.asarray(getattr(tr, f)) for f in
           ("loss", "grad_norm", "eps", "delta", "alpha", "lower_iters_cum", "cg_iters_cum")}
    out[f"{tag}_final"] = tr.final_loss
    out[f"{tag}_psnr"] = MI.psnr(x, up3.ground_truth)
    out[f"{tag}_b"] = b.data
    if not perturb_seed:
        out["y_delta"] = y
        out["x_true"] = up3.ground_truth
        out["a"] = up3.a.data
        out["b0"] = up3.b0.data
    return out


def maid3_p4():
    """P4 full-run fixture for an RGB 15x15 (c3 / c4 type) MAID run: the reference run plus three
    1e-15-perturbed replicas."""
    import multiprocessing as mp
    with mp.get_context("fork").Pool(4) as pool:
        parts = pool.starmap(_maid3_run, [("ref", 0), ("rep1", 1), ("rep2", 2), ("rep3", 3)])
    out = {}
    for d in parts:
        out.update(d)
    save("maid3_p4.npz", **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()[name]()
        sys.exit(0)
    reductions()
    conv_case("conv_small.npz", (24, 20, 3), 5, 11)
    conv_case("conv_k9.npz", (33, 40, 1), 9, 12)
    conv_case("conv_k15.npz", (40, 37, 3), 15, 13, tiny=False)
    dense_case("dense_small.npz", 40, 21)
    solver_cases()
    config_cases()
    baseline_cases()
    metric_cases()
    maid_p3()
