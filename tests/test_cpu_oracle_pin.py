"""Pin the CPU oracle against the REAL reference (golden fixtures generated
from /root/reference by tests/golden/make_golden.py).  Runs without a GPU."""
import numpy as np
import pytest

SIZES = (1, 5, 8, 17, 31, 100, 128, 129, 255, 1000, 4099, 65536, 90000)


def rel(a, b):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("n", SIZES)
def test_reductions_bitwise(orc, golden, n):
    d = golden("reductions.npz")
    a, b = d[f"a{n}"], d[f"b{n}"]
    assert orc.npsum(a) == float(d[f"sum{n}"])          # numpy pairwise
    assert orc.ddot(a, b) == float(d[f"dot{n}"])        # OpenBLAS SkylakeX ddot
    assert orc.ddot(a, b) == float(d[f"vdot{n}"])
    assert orc.norm(a) == float(d[f"norm{n}"])


@pytest.mark.parametrize("name", ["conv_small.npz", "conv_k9.npz", "conv_k15.npz", "conv_k31.npz"])
def test_conv_primitives(orc, golden, name):
    d = golden(name)
    op = orc.Conv(d["kern"], d["x"].shape)
    p = orc.Lower(op, d["y"], float(d["alpha"]), orc.TV(float(d["nu"])))
    assert np.array_equal(op.apply(d["x"]), d["apply"])
    assert np.array_equal(op.adjoint(d["v"]), d["adjoint"])
    assert np.array_equal(op.gram_diag(), d["gram_diag"])
    assert orc.lower_value(p, d["x"]) == float(d["lower_value"])
    v, g = orc.lower_value_and_grad(p, d["x"])
    assert v == float(d["vg_val"]) and np.array_equal(g, d["vg_g"])
    assert np.array_equal(orc.lower_grad(p, d["x"]), d["lower_grad"])
    assert orc.TV(1e-4).value(d["x"]) == float(d["tv_value"])
    assert rel(orc.lower_hess_vec(p, d["x"], d["v"]), d["hess_vec"]) <= 1e-13
    assert rel(orc.lower_hess_diag(p, d["x"]), d["hess_diag"]) <= 1e-13
    assert rel(orc.kgc(d["x"], d["v"], False, d["kern"].shape[:2]), d["kgc"]) <= 1e-13
    lam, conv, _ = orc.op_norm_sq(orc.Conv(d["kern"], d["x"].shape), 300, 1e-4)
    assert lam == float(d["norm_sq"])


def test_conv_k31_gaussian_pin(orc, golden):
    """The oracle's ndimage restatement at K = 31 on 300x260x3 (c5 kernel),
    pinned by the SHA-256 of the reference's outputs."""
    import hashlib
    d = golden("conv_k31_g6.npz")
    shape, seed = tuple(int(s) for s in d["shape"]), int(d["seed"])
    rng = np.random.default_rng(seed)
    x, v = rng.uniform(0.0, 1.0, shape), rng.standard_normal(shape)
    op = orc.Conv(d["kern"], shape)

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()
    ap = op.apply(x)
    assert np.array_equal(ap[::37, ::41], d["apply_probe"])
    assert sha(ap) == str(d["apply_sha"])
    assert sha(op.adjoint(v)) == str(d["adjoint_sha"])


def test_dense_primitives(orc, golden):
    d = golden("dense_small.npz")
    op = orc.Dense(d["m"])
    reg = orc.ElasticNet(float(d["l1"]), float(d["l2"]), float(d["nu"]))
    p = orc.Lower(op, d["y"], 1.0, reg)
    assert rel(op.apply(d["x"]), d["apply"]) <= 1e-14
    assert reg.value(d["x"]) == float(d["en_value"])
    assert np.array_equal(reg.grad(d["x"]), d["en_grad"])
    v, g = orc.lower_value_and_grad(p, d["x"])
    assert abs(v - float(d["vg_val"])) <= 1e-14 * abs(v) and rel(g, d["vg_g"]) <= 1e-13
    assert rel(orc.lower_hess_vec(p, d["x"], d["v"]), d["hess_vec"]) <= 1e-13


@pytest.mark.parametrize("tag,method,adaptive", [("agd_ad", "agd", True), ("gd_ad", "proxgrad", True),
                                                 ("fista", "fista_sc", True), ("agd_fixed", "agd", False),
                                                 ("agd_ad_conv", "agd", True)])
def test_solve_lower_bitwise(orc, golden, tag, method, adaptive):
    """The restated solver reproduces the reference's trajectory bit for bit."""
    d = golden("solve2d.npz")
    eps, mu, iters = d[f"{tag}_args"]
    p = orc.Lower(orc.Conv(d["kern"], d["y_delta"].shape), d["y_delta"], 0.6, orc.TV(1e-4))
    x, gn, it, conv = orc.solve_lower(p, d["x0"], float(eps), float(mu), int(iters), method, None, adaptive)
    assert it == int(d[f"{tag}_iters"]) and conv == bool(d[f"{tag}_conv"])
    assert np.array_equal(x, d[f"{tag}_x"]) and gn == float(d[f"{tag}_gn"])


def test_hypergradient_2d(orc, golden):
    d = golden("hyper2d.npz")
    d15 = golden("hyper2d_cg15.npz")
    up = orc.Upper(A_kernel=d["a_kern"], a=d["a_kern"], y_delta=d["y_delta"], beta=0.3, alpha=0.6, reg=orc.TV(1e-4),
                   b0=d["kern"], x0=d["x0"], dense=False, mu_floor=1e-3, lower_adaptive=True)
    st = {"x": d["x0"].copy(), "q": None}
    hg = orc.inexact_hypergradient(up, d["kern"], 0.5, 0.5, st, 15)
    assert hg["cg_iters"] == int(d15["cg_iters"])
    assert np.array_equal(hg["x_tilde"], d["x_tilde"])
    assert rel(hg["z"], d15["z"]) <= 1e-12


def test_dense_maid_short_run(orc, golden):
    d = golden("dense1d_run.npz")
    up = orc.Upper(A_kernel=d["A"], a=d["A"], y_delta=d["y_delta"], beta=0.0, alpha=1.0,
                   reg=orc.ElasticNet(1.2e-3, 4e-3, 1e-4), b0=d["A"], x0=np.zeros(80), dense=True)
    b, x, tr = orc.maid_run(up, dict(max_upper_iters=8))
    assert tr["lower_iters_cum"] == [int(v) for v in d["maid_lower_cum"]]
    assert tr["cg_iters_cum"] == [int(v) for v in d["maid_cg_cum"]]
    assert rel(tr["loss"], d["maid_loss"]) <= 1e-12
    assert rel(b, d["maid_b"]) <= 1e-12


def test_ift_baseline_oracle(orc, golden):
    """prox_l1, prox_grad_iterations and 5 outer steps of run_ift on c1
    (baselines.py:46-90, regularizers.py:22-27) against the reference."""
    d = golden("ift_c1.npz")
    out = orc.prox_l1(d["prox_in"], float(d["prox_thr"]))
    assert np.array_equal(out, d["prox_out"]) and np.array_equal(np.signbit(out), np.signbit(d["prox_out"]))
    d1 = golden("c1_maid.npz")
    up = orc.Upper(A_kernel=d1["A"], a=d1["A"], y_delta=d1["y_delta"], beta=0.0, alpha=1.0,
                   reg=orc.ElasticNet(1.2e-3, 4e-3, 1e-4), b0=d1["A"], x0=np.zeros(256), dense=True)
    p = up.lower_problem(up.b0)
    x50, traj = orc.prox_grad_iterations(p.op, p.y, p.alpha, 1.2e-3, 4e-3, np.zeros(256), 50, 0.1,
                                         keep_trajectory=True)
    assert rel(x50, d["pg_x50"]) <= 1e-13
    assert rel(np.array(traj[:4]), d["pg_traj3"]) <= 1e-13
    b, x, tr = orc.run_ift(up, dict(upper_iters=5, lower_iters=500, step_x=0.1, cg_tol=1e-10, cg_max_iters=400,
                                    upper_step=0.002))
    assert tr["lower_cum"] == [int(v) for v in d["ift_lower_cum"]]
    assert tr["cg_cum"] == [int(v) for v in d["ift_cg_cum"]]
    assert rel(tr["loss"], d["ift_loss"]) <= 1e-10
    assert rel(b, d["ift_b"]) <= 1e-10 and rel(x, d["ift_x"]) <= 1e-10


def test_unrolled_gradient_oracle(orc, golden):
    """unrolled_gradient (baselines.py:93-139) on c1 against the reference."""
    d = golden("ift_c1.npz")
    d1 = golden("c1_maid.npz")
    up = orc.Upper(A_kernel=d1["A"], a=d1["A"], y_delta=d1["y_delta"], beta=0.0, alpha=1.0,
                   reg=orc.ElasticNet(1.2e-3, 4e-3, 1e-4), b0=d1["A"], x0=np.zeros(256), dense=True)
    g, x = orc.unrolled_gradient(up, d1["A"], np.zeros(256), 50, 0.1)
    assert rel(x, d["unr_x"]) <= 1e-13
    assert rel(g, d["unr_grad"]) <= 1e-12


METRIC_CASES = ("g", "rgb", "big", "thin", "tiny")


@pytest.mark.parametrize("name", METRIC_CASES)
def test_metrics_oracle_bitwise(orc, golden, name):
    """PSNR / SSIM / rel-L2 restatements (metrics_io.py:26-80) vs the real reference."""
    import warnings
    d = golden("metrics.npz")
    x, r = d[f"{name}_x"], d[f"{name}_ref"]
    assert orc.psnr(x, r) == float(d[f"{name}_psnr"])
    assert orc.psnr(x, r, 2.5) == float(d[f"{name}_psnr_peak"])
    assert orc.rel_l2_error(x, r) == float(d[f"{name}_rel"])
    if name == "tiny":      # no interior window: the reference returns nan
        assert np.isnan(float(d[f"{name}_ssim"]))
    else:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            assert orc.ssim(x, r) == float(d[f"{name}_ssim"])


def test_trace_csv_roundtrip(tmp_path):
    """write_trace_csv / read_trace_csv (metrics_io.py:88-116): host-only, same format."""
    from paper_2502_09758_b200 import RunTrace
    from paper_2502_09758_b200 import metrics_io as mi
    t = RunTrace()
    for k in range(4):
        t.append(k, 1.0 / (k + 3), 0.1 * k, 0.25 / (k + 1), 0.2, 2e-5 * 1.5**k, 100 * k, 7 * k, 0.123456789 * k)
    p = tmp_path / "trace.csv"
    mi.write_trace_csv(t, p)
    lines = p.read_text().splitlines()
    assert lines[0] == ",".join(mi.TRACE_HEADER)
    assert lines[2].split(",")[1] == repr(1.0 / 4)
    back = mi.read_trace_csv(p)
    for f in ("k", "loss", "grad_norm", "eps", "delta", "alpha", "lower_iters_cum", "cg_iters_cum", "wall_s"):
        assert getattr(back, f) == getattr(t, f)
    p.write_text("a,b\n1,2\n")
    with pytest.raises(ValueError, match="unexpected trace header"):
        mi.read_trace_csv(p)
    with pytest.raises(OSError, match="cannot read trace"):
        mi.read_trace_csv(tmp_path / "missing.csv")
    assert mi.loss_axis_scale([[1.0, 2e3], [5.0]]) == "log"
    assert mi.loss_axis_scale([[1.0, 2.0], [-1.0]]) == "linear"


def test_png_io_roundtrip(tmp_path):
    """save_png / load_png / save_kernel_image (metrics_io.py:163-199): host file utilities."""
    pytest.importorskip("PIL")
    from paper_2502_09758_b200 import metrics_io as mi
    img = np.linspace(-0.2, 1.2, 48).reshape(6, 8)
    mi.save_png(img, tmp_path / "a.png")
    back = mi.load_png(tmp_path / "a.png")
    assert np.array_equal(back, np.round(np.clip(img, 0, 1) * 255) / 255)
    mi.save_kernel_image(np.arange(9.0).reshape(3, 3, 1), tmp_path / "k.png")
    assert mi.load_png(tmp_path / "k.png").max() == 1.0
    with pytest.raises(OSError, match="cannot read image"):
        mi.load_png(tmp_path / "missing.png")
