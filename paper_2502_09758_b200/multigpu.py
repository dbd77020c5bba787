"""Multi-GPU partitioning of the MAID hot path.

* c1-c3: replicas only (one instance does not shard usefully).
* c4 (64 independent 512x512x3 instances): instances are sharded across
  ranks with no data-path collective; each rank solves its share and the
  job time is the max over ranks (`run_instances`).
* c5 (one 4096x4096x3 image): 1-D row decomposition.  Each rank owns a slab
  of rows plus "ghost" rows on each interior side, exchanged with the
  neighbours (`halo_exchange`, torch.distributed send/recv: NCCL over
  NVLink on the GPU box, gloo in the CPU tests).  With a ghost width of
  3r + 1 rows, one exchange of the new iterate per lower iteration suffices:
  y needs x on slab +- (3r+1), r = By - y on slab +- (2r+1), g = 2B^T r +
  alpha TV'(y) on slab +- (r+1), the candidate x - g/L and its value on the
  slab.  Sums keep the single-GPU pairwise tree bit for bit: when the NumPy
  leaf layout is row-aligned, every leaf lies inside one slab, so each rank
  computes its own leaves, an all-gather assembles the global leaf vector in
  order (`gather_leaves`), and every rank folds the identical tree.

The per-rank device work reuses the single-GPU kernels on the local array
(slab + ghosts); ghost-row outputs are discarded.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


# ---------------------------------------------------------------------------
# c4: independent instances
def shard_instances(n_items: int, rank: int, world: int) -> list:
    """Round-robin assignment of instance indices (seeds) to a rank."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("need 0 <= rank < world")
    return list(range(rank, n_items, world))


def run_instances(seeds, solve_one, timer=None):
    """Solve every assigned instance in turn; returns (results, seconds)."""
    import time
    t0 = time.perf_counter()
    out = [solve_one(s) for s in seeds]
    return out, time.perf_counter() - t0


def max_over_ranks(value: float) -> float:
    """Max of a per-rank scalar over the process group (device time rule)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# c5: row slabs
@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    H: int
    row0: int          # first owned global row
    row1: int          # one past the last owned global row
    ghost_top: int     # ghost rows above (0 at the global top)
    ghost_bot: int     # ghost rows below (0 at the global bottom)

    @property
    def local_rows(self) -> int:
        return self.ghost_top + (self.row1 - self.row0) + self.ghost_bot

    @property
    def owned(self) -> slice:
        """Owned rows inside the local array."""
        return slice(self.ghost_top, self.ghost_top + self.row1 - self.row0)

    @property
    def global_rows(self) -> slice:
        """Global rows held locally (ghosts included)."""
        return slice(self.row0 - self.ghost_top, self.row1 + self.ghost_bot)


def ghost_width(kh: int) -> int:
    """Rows of ghost data for one exchange per lower iteration: 3r + 1."""
    return 3 * (kh // 2) + 1


def plan_slabs(H: int, world: int, kh: int, row_align: int = 1) -> list:
    """Split H rows into `world` contiguous slabs (sizes differ by at most
    `row_align`), each padded with ghost rows toward its neighbours."""
    if world < 1 or H < world:
        raise ValueError("need 1 <= world <= H")
    gw = ghost_width(kh)
    units = H // row_align
    base, extra = divmod(units, world)
    bounds = [0]
    for r in range(world):
        bounds.append(bounds[-1] + (base + (1 if r < extra else 0)) * row_align)
    bounds[-1] = H
    slabs = []
    for r in range(world):
        r0, r1 = bounds[r], bounds[r + 1]
        slabs.append(Slab(r, world, H, r0, r1, min(gw, r0), min(gw, H - r1)))
    return slabs


def leaf_range(slab: Slab, W: int, C: int, leaf_len: int):
    """Global NumPy-pairwise leaf indices [l0, l1) owned by a slab (row-aligned
    regular layout: W*C % leaf_len == 0)."""
    rowE = W * C
    if rowE % leaf_len:
        raise ValueError("leaf layout is not row-aligned; slabs cannot own whole leaves")
    per_row = rowE // leaf_len
    return slab.row0 * per_row, slab.row1 * per_row


def halo_exchange(local, slab: Slab, group=None):
    """Refresh the ghost rows of `local` (local_rows x ...) from the
    neighbours' owned boundary rows.  Rank r sends its first ghost_top owned
    rows up and its last ghost_bot owned rows down.  Works for CUDA tensors
    (NCCL) and CPU tensors (gloo)."""
    import torch.distributed as dist
    ops = []
    own = local[slab.owned]
    if slab.rank > 0 and slab.ghost_top:
        up = slab.rank - 1
        send_up = own[: slab.ghost_top].contiguous()
        recv_up = local[: slab.ghost_top]
        buf_up = recv_up.contiguous().clone()
        ops.append(dist.P2POp(dist.isend, send_up, up, group))
        ops.append(dist.P2POp(dist.irecv, buf_up, up, group))
    else:
        buf_up = None
    if slab.rank < slab.world - 1 and slab.ghost_bot:
        dn = slab.rank + 1
        send_dn = own[own.shape[0] - slab.ghost_bot:].contiguous()
        buf_dn = local[local.shape[0] - slab.ghost_bot:].contiguous().clone()
        ops.append(dist.P2POp(dist.isend, send_dn, dn, group))
        ops.append(dist.P2POp(dist.irecv, buf_dn, dn, group))
    else:
        buf_dn = None
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    if buf_up is not None:
        local[: slab.ghost_top] = buf_up
    if buf_dn is not None:
        local[local.shape[0] - slab.ghost_bot:] = buf_dn
    return local


def gather_leaves(local_leaves, counts, group=None):
    """All-gather per-rank leaf vectors (ordered by rank = by rows) into the
    global leaf vector, identical on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n_max = max(counts)
    pad = torch.zeros(n_max, dtype=local_leaves.dtype, device=local_leaves.device)
    pad[: local_leaves.numel()] = local_leaves
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


def perfect_tree_sum(vals) -> float:
    """Fold a power-of-two leaf vector (zero-padded) in perfect-tree order —
    the order the device uses for regular NumPy-pairwise layouts."""
    v = np.asarray(vals, dtype=np.float64)
    p = 1
    while p < v.size:
        p *= 2
    v = np.concatenate([v, np.zeros(p - v.size)])
    while v.size > 1:
        v = v[0::2] + v[1::2]
    return float(v[0])
