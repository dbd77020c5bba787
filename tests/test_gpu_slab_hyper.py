"""Row-slab hypergradient and MAID (SURVEY.md §8e, c5 decomposition) on one
device: the slab CG (hypergradient.py:35-84), upper terms (problems.py:48-50,
hypergradient.py:87-89), mixed derivative (hypergradient.py:92-104), the whole
inexact_hypergradient (148-190) and maid_run (maid.py:149-255) over P slabs
must reproduce the unsplit single-GPU path BIT FOR BIT (same leaves, tile
partials, trees, kernel-gram groups and decisions)."""
from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _upper(shape, K, seed=0):
    import paper_2502_09758_b200 as adp
    from paper_2502_09758_b200 import configs
    rng = np.random.default_rng(seed)
    h, w, c = shape
    img = np.stack([configs.shapes_image(h, w, np.random.default_rng([seed, 10 + ch])) for ch in range(c)], axis=2)
    truth = configs.gaussian_kernel_2d(K, 2.0 * K / 9.0, c)      # c2's kernel pair (sigma 2 vs 2.6 at K = 9)
    a = configs.gaussian_kernel_2d(K, 2.6 * K / 9.0, c)
    y = configs.blur(img, truth) + 0.01 * rng.standard_normal(shape)
    return adp.UpperProblem(name="slab", A=adp.ConvOperator(a, shape), a=a, y_delta=y, beta=0.3, alpha=0.6,
                            reg=adp.SmoothedTV(1e-4), b0=a, x0=y.copy(), ground_truth=img, mu_floor=10.0,
                            lower_method="agd", lower_max_iters=1200, lower_adaptive=True)


def _full(t):
    return np.concatenate([x.cpu().numpy() for x in t], axis=0)


CASES = [((128, 128, 3), 9, 2), ((256, 256, 3), 15, 3), ((512, 512, 3), 15, 4)]


@pytest.mark.parametrize("shape,K,world", CASES)
def test_slab_cg_upper_mixed_bitwise(adp, shape, K, world):
    from paper_2502_09758_b200 import multigpu
    from paper_2502_09758_b200.hypergradient import _upper_terms, hess_cg
    up = _upper(shape, K)
    rng = np.random.default_rng(1)
    xt = up.y_delta + 0.02 * rng.standard_normal(shape)
    b = up.b0
    p = up.lower_problem(b)
    # unsplit
    fit, gn, rhs = _upper_terms(up.A, xt, up.y_delta, want_grad=True)
    cg, hv = hess_cg(p, xt, rhs, 1e-30, 12)
    cgw, _ = hess_cg(p, xt, rhs, 1e-30, 5, q0=cg.q)
    z = adp.mixed_second_transpose(xt, b, cg.q, p)
    # slabs
    sh = multigpu.SlabHypergradient(up, world)
    sh.sv.bind(up.lower_problem(b))
    xs = sh.sv.local(xt)
    fit_s, gn_s, rhs_s = sh.upper_terms(xs, want_grad=True)
    assert fit_s == fit and gn_s == gn
    assert np.array_equal(_full(sh.sv._owned(rhs_s)), rhs.cpu().numpy())
    q, res, it, conv, hv_s = sh.hess_cg(xs, rhs_s, 1e-30, 12)
    assert it == cg.iters and res == cg.residual and conv == cg.converged and hv_s == hv
    assert np.array_equal(_full(sh.sv._owned(q)), cg.q.cpu().numpy())
    qw, resw, itw, _, _ = sh.hess_cg(xs, rhs_s, 1e-30, 5, qs=q)
    assert itw == cgw.iters and resw == cgw.residual
    assert np.array_equal(_full(sh.sv._owned(qw)), cgw.q.cpu().numpy())
    zs = sh.mixed(b, xs, q)
    assert np.array_equal(zs, z)


@pytest.mark.parametrize("shape,K,world", CASES[:2])
def test_slab_hypergradient_bitwise(adp, shape, K, world):
    from paper_2502_09758_b200 import multigpu
    up = _upper(shape, K, seed=2)
    st = adp.WarmState(x=up.x0.copy())
    hg = adp.inexact_hypergradient(up, up.b0, 0.05, 0.05, st, cg_max_iters=20)
    sh = multigpu.SlabHypergradient(_upper(shape, K, seed=2), world)
    sst = adp.WarmState(x=sh.sv.local(up.x0))
    hs = sh.hypergradient(up.b0, 0.05, 0.05, sst, cg_max_iters=20)
    assert hs.lower_iters == hg.lower_iters and hs.cg_iters == hg.cg_iters
    assert hs.cg_residual == hg.cg_residual and hs.epsilon_used == hg.epsilon_used
    assert np.array_equal(hs.z, hg.z)
    assert np.array_equal(_full(sh.sv._owned(sst.x)), np.asarray(st.x))


@pytest.mark.parametrize("world", [2, 4])
def test_slab_maid_run_bitwise(adp, world):
    from paper_2502_09758_b200 import configs, multigpu
    cfg = replace(configs.maid_config("c2"), max_upper_iters=2)
    b, x, tr = adp.maid_run(_upper((128, 128, 3), 9, seed=3), cfg)
    bs, xs, trs = multigpu.slab_maid_run(_upper((128, 128, 3), 9, seed=3), cfg, world)
    assert len(trs) == len(tr) >= 1
    for f in ("lower_iters_cum", "cg_iters_cum", "loss", "alpha", "eps", "delta", "grad_norm"):
        assert list(getattr(trs, f)) == list(getattr(tr, f)), f
    assert trs.final_loss == tr.final_loss
    assert np.array_equal(bs.data, b.data)
    assert np.array_equal(xs, x)


def _maid_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_09758_b200 as adp
        from paper_2502_09758_b200 import configs, multigpu
        adp.set_precision("float64", "strict")
        cfg = replace(configs.maid_config("c2"), max_upper_iters=1)
        b, x, tr = multigpu.slab_maid_run(_upper((128, 128, 3), 9, seed=4), cfg, world, ranks=[rank],
                                          comm=multigpu.DistComm())
        q.put((rank, (b.data, x, list(tr.lower_iters_cum), list(tr.loss), tr.final_loss)))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_slab_maid_two_processes(adp):
    """DistComm orchestration of the slab MAID (ghost send/recv, all-reduce of
    sum units and kernel-gram partials, max of the Jacobi diagonal) with two
    processes on the one device (gloo, host-staged): identical to one GPU."""
    import socket
    import torch.multiprocessing as mp
    from paper_2502_09758_b200 import configs
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    procs = [ctx.Process(target=_maid_worker, args=(r, 2, port, qu)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict(qu.get(timeout=600) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert all(not isinstance(v, str) for v in out.values()), out
    cfg = replace(configs.maid_config("c2"), max_upper_iters=1)
    b, x, tr = adp.maid_run(_upper((128, 128, 3), 9, seed=4), cfg)
    for r in (0, 1):
        bd, xr, low, loss, fl = out[r]
        assert np.array_equal(bd, b.data) and np.array_equal(xr, x)
        assert low == list(tr.lower_iters_cum) and loss == list(tr.loss) and fl == tr.final_loss
