"""Multi-rank host logic on CPU with the gloo backend,
world_size 2: instance sharding (c4), row slabs with 3r+1 ghost rows and
halo exchange (c5), and the global NumPy-pairwise sum assembled from
per-slab leaves.  The CPU oracle stands in for the per-rank device work (test
infrastructure only)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_09758_b200 import multigpu as mg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return out


def test_shard_instances_cover_each_once():
    seen = sorted(s for r in range(8) for s in mg.shard_instances(64, r, 8))
    assert seen == list(range(64))
    assert all(len(mg.shard_instances(64, r, 8)) == 8 for r in range(8))


def test_plan_slabs_geometry():
    for world in (2, 4, 8):
        slabs = mg.plan_slabs(4096, world, 31)
        assert slabs[0].row0 == 0 and slabs[-1].row1 == 4096
        assert all(a.row1 == b.row0 for a, b in zip(slabs, slabs[1:]))
        assert slabs[0].ghost_top == 0 and slabs[-1].ghost_bot == 0
        assert all(s.ghost_bot == 46 for s in slabs[:-1]) and all(s.ghost_top == 46 for s in slabs[1:])


def _halo_case(rank, world):
    H, W, C = 64, 10, 3
    slab = mg.plan_slabs(H, world, 9)[rank]
    g = np.arange(H * W * C, dtype=np.float64).reshape(H, W, C)
    local = torch.full((slab.local_rows, W, C), -1.0, dtype=torch.float64)
    local[slab.owned] = torch.from_numpy(g[slab.row0:slab.row1])
    mg.halo_exchange(local, slab)
    return bool(np.array_equal(local.numpy(), g[slab.global_rows]))


def test_halo_exchange_gloo():
    assert run_ranks(_halo_case) == {0: True, 1: True}


def _sum_case(rank, world):
    H, W, C = 128, 64, 3           # N = 24576 = 96 * 2^8: leaves of 96, 2 per row
    rng = np.random.default_rng(5)
    a = rng.standard_normal((H, W, C)) * np.exp(rng.standard_normal((H, W, C)))
    slab = mg.plan_slabs(H, world, 9)[rank]
    l0, l1 = mg.leaf_range(slab, W, C, 96)
    flat = a.reshape(-1)
    mine = torch.tensor([float(np.sum(flat[k * 96:(k + 1) * 96])) for k in range(l0, l1)], dtype=torch.float64)
    counts = [mg.leaf_range(s, W, C, 96)[1] - mg.leaf_range(s, W, C, 96)[0] for s in mg.plan_slabs(H, world, 9)]
    leaves = mg.gather_leaves(mine, counts)
    return mg.perfect_tree_sum(leaves.numpy()) == float(np.sum(a))


def test_global_pairwise_sum_from_slabs_is_bitwise():
    assert run_ranks(_sum_case) == {0: True, 1: True}


def _stencil_case(rank, world):
    """value+gradient+candidate on a slab with 3r+1 ghost rows reproduce the
    global single-rank computation on the owned rows (oracle as the stand-in)."""
    import adp_oracle as orc
    H, W, C, K = 48, 20, 3, 5
    rng = np.random.default_rng(9)
    x = rng.uniform(0, 1, (H, W, C))
    y = rng.uniform(0, 1, (H, W, C))
    k = rng.uniform(0, 1, (K, K, C))
    k /= k.sum(axis=(0, 1), keepdims=True)
    p = orc.Lower(orc.Conv(k, (H, W, C)), y, 0.6, orc.TV(1e-4))
    _, g_full = orc.lower_value_and_grad(p, x)
    xc_full = x - g_full / 3.0
    r_full = orc.correlate(xc_full, k) - y

    slab = mg.plan_slabs(H, world, K)[rank]
    xl = torch.zeros((slab.local_rows, W, C), dtype=torch.float64)
    xl[slab.owned] = torch.from_numpy(x[slab.row0:slab.row1])
    mg.halo_exchange(xl, slab)
    yl = y[slab.global_rows]
    pl = orc.Lower(orc.Conv(k, yl.shape), yl, 0.6, orc.TV(1e-4))
    _, gl = orc.lower_value_and_grad(pl, xl.numpy())
    xcl = xl.numpy() - gl / 3.0
    rl = orc.correlate(xcl, k) - yl
    ok_g = np.array_equal(gl[slab.owned], g_full[slab.row0:slab.row1])
    ok_r = np.array_equal(rl[slab.owned], r_full[slab.row0:slab.row1])
    return bool(ok_g and ok_r)


def test_slab_ghost_width_reproduces_global_iteration():
    assert run_ranks(_stencil_case) == {0: True, 1: True}


def _assemble_case(rank, world):
    # units of two sums, each rank owning disjoint ranges (the TV-like sum has
    # two ranges per rank); DistComm.assemble = all-reduce SUM of zero-padded
    # vectors must reproduce the full vectors exactly (incl. tiny / huge values)
    rng = np.random.default_rng(11)
    full_a = rng.standard_normal(40) * np.exp(8 * rng.standard_normal(40))
    full_b = rng.standard_normal(64) * 1e-300
    ranges_a = [(0, 25), (25, 40)]
    ranges_b = [[(0, 16), (32, 48)], [(16, 32), (48, 64)]]
    a = torch.zeros(40, dtype=torch.float64)
    b = torch.zeros(64, dtype=torch.float64)
    lo, hi = ranges_a[rank]
    a[lo:hi] = torch.from_numpy(full_a[lo:hi])
    for lo, hi in ranges_b[rank]:
        b[lo:hi] = torch.from_numpy(full_b[lo:hi])
    ra, rb = mg.DistComm().assemble([a, b])
    return bool(np.array_equal(ra.numpy(), full_a) and np.array_equal(rb.numpy(), full_b))


def test_dist_unit_assembly_is_exact():
    assert run_ranks(_assemble_case) == {0: True, 1: True}


def test_slab_alignment_rules():
    # ghost rows are 3r + 1 rounded up to the tile height, slabs align to it
    slabs = mg.plan_slabs(4096, 8, 31, row_align=64, ghost=48)
    assert [s.row1 - s.row0 for s in slabs] == [512] * 8
    assert slabs[0].ghost_top == 0 and slabs[-1].ghost_bot == 0
    assert all(s.ghost_top == 48 for s in slabs[1:]) and all(s.ghost_bot == 48 for s in slabs[:-1])
    assert all((s.row0 - s.ghost_top) % 8 == 0 for s in slabs)
    assert mg._lcm(8, 64) == 64 and mg._lcm(8, 12) == 24
