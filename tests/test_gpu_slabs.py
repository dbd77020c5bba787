"""Row-slab decomposition of the lower-level solve on one
device: P slabs held by one process (LocalComm) must reproduce the unsplit
single-GPU solve BIT FOR BIT — same leaves, same tile partials, same trees,
same decisions — for single-level and two-level sum layouts."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _problem(adp, shape, K, sigma, seed=0):
    from paper_2502_09758_b200 import configs
    rng = np.random.default_rng(seed)
    k = configs.gaussian_kernel_2d(K, sigma, shape[2])
    x_true = rng.uniform(0.0, 1.0, shape)
    op = adp.ConvOperator(k, shape)
    y = op.apply(x_true) + 0.01 * rng.standard_normal(shape)
    return adp.LowerProblem(adp.ConvOperator(k, shape), y, 0.6, adp.SmoothedTV(1e-4)), y


@pytest.mark.parametrize("shape,K,world,iters", [
    ((256, 256, 3), 15, 2, 40),     # single-level sums
    ((256, 256, 3), 15, 3, 40),     # uneven slabs
    ((512, 512, 3), 15, 2, 25),     # two-level element sums (8192 leaves)
    ((1024, 1024, 3), 31, 4, 12),   # c5 geometry (K = 31), two-level sums, 4 slabs
])
def test_slab_solve_matches_single_gpu_bitwise(adp, shape, K, world, iters):
    from paper_2502_09758_b200 import multigpu
    p, y = _problem(adp, shape, K, 2.0 + K / 10.0)
    x0 = np.ascontiguousarray(y)
    st = {}
    ref = adp.solve_lower(p, x0, 1e-14, 10.0, max_iters=iters, method="agd", adaptive=True, stats=st)
    p2, _ = _problem(adp, shape, K, 2.0 + K / 10.0)
    sv = multigpu.SlabSolver(p2, world)
    xs, gn, it, conv = sv.solve(x0, 1e-14, 10.0, max_iters=iters)
    x = np.concatenate([t.cpu().numpy() for t in xs], axis=0)
    assert it == ref.iters and conv == ref.converged
    assert sv.stats["lip"] == st["lip"]
    assert sv.stats["vg_evals"] == st["vg_evals"] and sv.stats["value_evals"] == st["value_evals"]
    assert sv.stats["restarts"] == st["restarts"]
    assert gn == ref.grad_norm
    assert np.array_equal(x, ref.x_tilde)


def test_slab_plan_rejects_misaligned_rows(adp):
    from paper_2502_09758_b200 import _native as nat
    with pytest.raises(ValueError, match="multiples of the tile height"):
        nat.Plan(nat.LAYOUT_DEPTHWISE2D, (100, 256, 3), (15, 15), "float64", "strict", slab=(4, 256, 0, 100))


def test_slab_plan_only_runs_slab_steps(adp):
    from paper_2502_09758_b200 import _native as nat
    import ctypes
    plan = nat.Plan(nat.LAYOUT_DEPTHWISE2D, (152, 256, 3), (15, 15), "float64", "strict",
                    slab=(0, 256, 0, 128))
    x = nat.zeros_dev((152, 256, 3))
    k = nat.zeros_dev((15, 15, 3))
    out = nat.zeros_dev((152, 256, 3))
    rc = nat.lib().adp_apply(plan.handle, nat.ptr(k), nat.ptr(x), nat.ptr(out), nat.stream_ptr())
    assert rc != 0 and b"slab" in nat.lib().adp_last_error()


def _two_proc_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2502_09758_b200 as adp
        from paper_2502_09758_b200 import multigpu
        p, y = _problem(adp, (512, 512, 3), 15, 3.5)
        sv = multigpu.SlabSolver(p, world, ranks=[rank], comm=multigpu.DistComm())
        xs, gn, it, conv = sv.solve(np.ascontiguousarray(y), 1e-14, 10.0, max_iters=20)
        q.put((rank, (xs[0].cpu().numpy(), gn, it, dict(sv.stats))))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_slab_solve_two_processes_match_single_gpu(adp):
    """The distributed orchestration (DistComm: ghost send/recv, all-reduce
    of the sum units) with two processes, one slab each, on the one device
    (gloo, host-staged): identical to the unsplit solve."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_proc_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert all(not isinstance(v, str) for v in out.values()), out
    p, y = _problem(adp, (512, 512, 3), 15, 3.5)
    st = {}
    ref = adp.solve_lower(p, np.ascontiguousarray(y), 1e-14, 10.0, max_iters=20, method="agd", adaptive=True,
                          stats=st)
    x = np.concatenate([out[0][0], out[1][0]], axis=0)
    assert out[0][1] == out[1][1] == ref.grad_norm and out[0][2] == ref.iters
    assert out[0][3]["restarts"] == st["restarts"] and out[0][3]["value_evals"] == st["value_evals"]
    assert np.array_equal(x, ref.x_tilde)
