"""Device quality metrics: PSNR / SSIM bitwise equal to the
REAL reference (tests/golden/metrics.npz) and to the CPU oracle at larger
sizes; rel-L2 (an OpenBLAS ddot in the reference) within 1e-13; exact
properties at the c5 size (4096x4096x3)."""
import warnings

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = ("g", "rgb", "big", "thin", "tiny")


@pytest.fixture(scope="module")
def mi(adp):
    from paper_2502_09758_b200 import metrics_io
    return metrics_io


@pytest.mark.parametrize("name", CASES)
def test_metrics_match_reference(mi, golden, name):
    d = golden("metrics.npz")
    x, r = d[f"{name}_x"], d[f"{name}_ref"]
    assert mi.psnr(x, r) == float(d[f"{name}_psnr"])
    assert mi.psnr(x, r, peak=2.5) == float(d[f"{name}_psnr_peak"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        s = mi.ssim(x, r)
    want = float(d[f"{name}_ssim"])
    assert (np.isnan(s) and np.isnan(want)) or s == want
    assert abs(mi.rel_l2_error(x, r) - float(d[f"{name}_rel"])) <= 1e-13 * float(d[f"{name}_rel"])
    rep = mi.metric_report(x, r)
    assert rep.psnr_db == float(d[f"{name}_psnr"])


@pytest.mark.parametrize("shape", [(300, 257, 3), (512, 512, 1), (64, 1000)])
def test_metrics_match_oracle(mi, orc, shape):
    rng = np.random.default_rng(sum(shape))
    r = rng.uniform(0.0, 1.0, shape)
    x = r + 0.02 * rng.standard_normal(shape)
    assert mi.psnr(x, r) == orc.psnr(x, r)
    assert mi.ssim(x, r) == orc.ssim(x, r)
    assert abs(mi.rel_l2_error(x, r) / orc.rel_l2_error(x, r) - 1.0) <= 1e-13


def test_metrics_torch_inputs_and_errors(mi, orc):
    import torch
    rng = np.random.default_rng(3)
    r = rng.uniform(0.0, 1.0, (50, 60, 3))
    x = r + 0.01 * rng.standard_normal(r.shape)
    xt, rt = torch.from_numpy(x).cuda(), torch.from_numpy(r).cuda()
    assert mi.ssim(xt, rt) == orc.ssim(x, r)
    assert mi.psnr(xt.float(), rt.float()) == orc.psnr(x.astype(np.float32).astype(float),
                                                         r.astype(np.float32).astype(float))
    assert mi.psnr(x, x) == mi.PSNR_CAP_DB
    with pytest.raises(ValueError, match="shape mismatch"):
        mi.psnr(x, r[:, :, :2])
    with pytest.raises(ValueError, match="shape mismatch"):
        mi.ssim(x, r[:10])
    with pytest.raises(ValueError, match="peak"):
        mi.psnr(x, r, peak=0.0)
    assert np.isnan(mi.metric_report(x[0, :, 0], r[0, :, 0]).ssim)


def test_metrics_c5_size_properties(mi):
    """4096x4096x3: ssim(x, x) is exactly 1 (num == den bit for bit, sum of ones
    exact); psnr(x, x) hits the cap; psnr of a constant offset d is exactly
    10 log10(1 / d^2) computed from the pairwise sum of n equal squares."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.floor(torch.rand((4096, 4096, 3), dtype=torch.float64, device="cuda", generator=g) * 2**20) / 2**20
    assert mi.ssim(x, x) == 1.0
    assert mi.psnr(x, x) == mi.PSNR_CAP_DB
    d = 0.0625                                   # power of two: every square and partial sum exact
    y = x + d
    assert (y - x == d).all()
    assert mi.psnr(y, x) == min(10.0 * np.log10(1.0 / (d * d)), mi.PSNR_CAP_DB)
    assert abs(mi.rel_l2_error(y, x) - d * np.sqrt(x.numel()) / float(torch.linalg.norm(x))) <= 1e-12
