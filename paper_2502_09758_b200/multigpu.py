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

import math
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


def plan_slabs(H: int, world: int, kh: int, row_align: int = 1, ghost: int | None = None) -> list:
    """Split H rows into `world` contiguous slabs (sizes differ by at most
    `row_align`), each padded with ghost rows toward its neighbours
    (`ghost` rows, default 3r + 1)."""
    if world < 1 or H < world:
        raise ValueError("need 1 <= world <= H")
    gw = ghost_width(kh) if ghost is None else int(ghost)
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
    if local.is_cuda and dist.get_backend(group) != "nccl":
        # host-staged exchange (gloo with device arrays: functional tests on one GPU)
        host = local.cpu()
        halo_exchange(host, slab, group)
        if slab.ghost_top:
            local[: slab.ghost_top].copy_(host[: slab.ghost_top])
        if slab.ghost_bot:
            local[local.shape[0] - slab.ghost_bot:].copy_(host[host.shape[0] - slab.ghost_bot:])
        return local
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


# ---------------------------------------------------------------------------
# c5: the lower-level solve on row slabs, host-stepped at its reductions.
#
# Per AGD iteration each rank runs ONE device step (adp_slab_step op 0:
# value+grad at y, first candidate, its value, restart dot) over its slab +
# ghosts, then the ranks assemble the sum units (all-reduce SUM of vectors
# that are zero outside each rank's own ranges: exact) and fold them on the
# device in the single-GPU tree order (adp_fold_units).  The decisions
# (acceptance, backtracking retries = op 1, restart) are the scalar logic of
# conv_solve_kernel / _accelerated (lower_solvers.py:180-213) evaluated
# identically on every rank; then one ghost exchange of the new iterate.
# Leaves, tile partials and trees are those of the unsplit plan, so the
# iterates are bitwise identical to the single-GPU solve.

class LocalComm:
    """Every slab in this process (one device): ghost refresh by device
    copies between the slabs' arrays; unit vectors are shared, so assembly
    needs no collective."""

    def exchange(self, states, arrays):
        for i, st in enumerate(states):
            s = st.slab
            if s.ghost_top:
                nb = states[i - 1]
                src = arrays[i - 1][nb.slab.owned]
                arrays[i][: s.ghost_top].copy_(src[src.shape[0] - s.ghost_top:])
            if s.ghost_bot:
                nb = states[i + 1]
                src = arrays[i + 1][nb.slab.owned]
                arrays[i][arrays[i].shape[0] - s.ghost_bot:].copy_(src[: s.ghost_bot])

    def assemble(self, bufs):
        return bufs


class DistComm:
    """One slab per rank over torch.distributed (NCCL over NVLink on the GPU
    box): ghost rows by send/recv, unit vectors by one all-reduce SUM."""

    def __init__(self, group=None):
        self.group = group

    def exchange(self, states, arrays):
        for st, arr in zip(states, arrays):
            halo_exchange(arr, st.slab, self.group)

    def assemble(self, bufs):
        import torch
        import torch.distributed as dist
        flat = torch.cat([b.reshape(-1) for b in bufs])
        if flat.is_cuda and dist.get_backend(self.group) != "nccl":
            host = flat.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=self.group)
            flat = host.to(flat.device)
        else:
            dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=self.group)
        out, o = [], 0
        for b in bufs:
            out.append(flat[o:o + b.numel()].view_as(b))
            o += b.numel()
        return out


@dataclass
class _SlabState:
    slab: Slab
    plan: object
    lower: object
    keep: tuple
    X: list


SUM_FIT, SUM_TV, SUM_FITC, SUM_TVC, SUM_GG, SUM_DOT = range(6)


class SlabSolver:
    """solve_lower (agd, adaptive: the c2-c5 settings) of one image split into
    row slabs.  `ranks` are the slab indices held by this process: all of
    them with LocalComm (one device), [rank] with DistComm."""

    def __init__(self, p, world: int, ranks=None, comm=None):
        import ctypes
        from . import _native as nat
        from .lower_solvers import _check_reg_smooth
        from .operators import ConvOperator
        from .regularizers import SmoothedTV
        if not isinstance(p.op, ConvOperator) or not isinstance(p.reg, SmoothedTV):
            raise ValueError("row slabs: depthwise 2-D operator with SmoothedTV")
        _check_reg_smooth(p)
        self.p = p
        self.nat = nat
        self.ctypes = ctypes
        H, W, C = p.op.signal_shape
        K = p.op.kernel.data.shape[0]
        if p.op.kernel.data.shape[1] != K:
            raise ValueError("row slabs: square stencils")
        self.shape = (H, W, C)
        self.K = K
        geo = nat.probe_geometry((H, W, C), (K, K))
        if not geo["fused"]:
            raise ValueError("row slabs need a leaf-aligned (fused) sum layout")
        TH, TW, tilesW, L = geo["TH"], geo["TW"], geo["tilesW"], geo["leafL"]
        self.geo = geo
        align = TH
        n_leaves = H * W * C // L
        if n_leaves > 4096:                      # two-level element sums: subtree-aligned rows
            align = _lcm(align, max(1, 2048 * L // (W * C)))
        tiles_h = (H + TH - 1) // TH
        if tiles_h * tilesW > 4096:              # two-level tile sums
            align = _lcm(align, max(1, 2048 // tilesW) * TH)
        r = K // 2
        gw = -(-(3 * r + 1) // TH) * TH          # ghost rows: 3r + 1, tile aligned
        self.slabs = plan_slabs(H, world, K, row_align=align, ghost=gw)
        for s in self.slabs:
            if (s.row1 - s.row0) < gw and world > 1:
                raise ValueError(f"slab of {s.row1 - s.row0} rows is thinner than its ghost width {gw}")
        self.ranks = list(range(world)) if ranks is None else list(ranks)
        self.comm = comm if comm is not None else LocalComm()
        if isinstance(self.comm, LocalComm) and len(self.ranks) != world:
            raise ValueError("LocalComm holds every slab")
        kd = p.op.kernel.device()
        self.states = []
        for rk in self.ranks:
            s = self.slabs[rk]
            g0 = s.row0 - s.ghost_top
            rows = s.local_rows
            own = (s.ghost_top, s.ghost_top + s.row1 - s.row0)
            plan = nat.Plan(nat.LAYOUT_DEPTHWISE2D, (rows, W, C), (K, K), nat.get_precision()["dtype"],
                            nat.get_precision()["mode"], tile=(TH, TW), slab=(g0, H, own[0], own[1]))
            yd = nat.to_dev(np.ascontiguousarray(np.asarray(p.y)[g0:g0 + rows]) if not nat.is_torch(p.y)
                            else p.y[g0:g0 + rows].contiguous())
            low = p.reg.native()
            low.kernel = kd.data_ptr()
            low.y = yd.data_ptr()
            low.alpha = float(p.alpha)
            X = [nat.empty_like_dev((rows, W, C)) for _ in range(3)]
            self.states.append(_SlabState(s, plan, low, (kd, yd), X))
        self.units_meta = []
        for which in range(6):
            n = ctypes.c_int64()
            own = (ctypes.c_int64 * 4)()
            nat.check(nat.lib().adp_slab_units(self.states[0].plan.handle, which, ctypes.byref(n), own, None, None),
                      "adp_slab_units")
            self.units_meta.append(int(n.value))
        self.stats = {}

    # -- device steps and reductions
    def _step(self, op, xs, xps, outs, beta=0.0, L=1.0):
        nat, ct = self.nat, self.ctypes
        for st, x, xp, o in zip(self.states, xs, xps, outs):
            nat.check(nat.lib().adp_slab_step(st.plan.handle, ct.byref(st.lower), op, nat.ptr(x), nat.ptr(xp),
                                              nat.ptr(o), float(beta), float(L), nat.stream_ptr()),
                      "adp_slab_step")

    def _sums(self, which):
        import torch
        nat, ct = self.nat, self.ctypes
        bufs = [torch.zeros(self.units_meta[w], dtype=torch.float64, device="cuda") for w in which]
        for st in self.states:
            for w, b in zip(which, bufs):
                n = ct.c_int64()
                own = (ct.c_int64 * 4)()
                nat.check(nat.lib().adp_slab_units(st.plan.handle, w, ct.byref(n), own, nat.ptr(b),
                                                   nat.stream_ptr()), "adp_slab_units")
        bufs = self.comm.assemble(bufs)
        k = len(which)
        ptrs = (ct.c_void_p * k)(*[b.data_ptr() for b in bufs])
        ns = (ct.c_int64 * k)(*[b.numel() for b in bufs])
        out = (ct.c_double * k)()
        nat.check(nat.lib().adp_fold_units(k, ptrs, ns, out, nat.stream_ptr()), "adp_fold_units")
        return [float(v) for v in out]

    def _local(self, full):
        """Per-state local arrays (slab + ghosts) of a full image (host or device)."""
        nat = self.nat
        out = []
        for st in self.states:
            s = st.slab
            g0 = s.row0 - s.ghost_top
            out.append(nat.to_dev(full[g0:g0 + s.local_rows]))
        return out

    def op_norm_sq(self, max_iters: int = 300, tol: float = 1e-4):
        """Power iteration on B^T B (operators.py:137-173) over the slabs."""
        nat = self.nat
        src = self._local(nat.power_start(self.shape))
        bufs = ([nat.empty_like_dev(x.shape) for x in src], [nat.empty_like_dev(x.shape) for x in src])
        self._step(3, src, src, src)
        scale = math.sqrt(self._sums([SUM_GG])[0])    # v /= ||v||
        lam, conv, iters = 0.0, False, 0
        for it in range(max_iters):
            iters = it + 1
            out = bufs[it % 2]
            self._step(2, src, src, out, L=scale)     # w = B^T B v
            lam_new = math.sqrt(self._sums([SUM_GG])[0])
            if lam_new == 0.0:
                lam, conv = 0.0, True
                break
            src, scale = out, lam_new                 # v = w / ||w||
            if abs(lam_new - lam) <= tol * max(lam_new, 1e-300):
                lam, conv = lam_new, True
                break
            lam = lam_new
            self.comm.exchange(self.states, src)
        self.stats.update(power_iters=iters, power_converged=conv)
        return lam

    def solve(self, x0, eps: float, mu: float, max_iters: int = 1200, norm_sq: float | None = None):
        """Adaptive AGD (lower_solvers.py:180-213).  Returns (x_owned list per
        held slab, grad_norm, iters, converged)."""
        from .lower_solvers import SolveDiverged
        nat = self.nat
        p = self.p
        H, W, C = self.shape
        if eps <= 0 or mu <= 0:
            raise ValueError("eps and mu must be > 0")
        tol = eps * mu
        lam = self.op_norm_sq() if norm_sq is None else float(norm_sq)
        alpha, nu = float(p.alpha), float(p.reg.nu)
        lip = 2.0 * lam + alpha * p.reg.curvature
        twoN = 2.0 * float(H * W * C)
        tv = alpha != 0.0
        xs = self._local(x0)
        for st, x in zip(self.states, xs):
            st.X[0].copy_(x)
        ix = ixp = 0
        ic = 1
        t_mom, lip_t = 1.0, lip
        vg = vals = restarts = 0
        for t in range(max_iters):
            t_next = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * t_mom * t_mom))
            beta = (t_mom - 1.0) / t_next
            t_mom = t_next
            L_try = lip_t
            X = [st.X for st in self.states]
            self._step(0, [x[ix] for x in X], [x[ixp] for x in X], [x[ic] for x in X], beta, L_try)
            vg += 1
            vals += 1
            fit, tvs, gg, dot, fitc, tvc = self._sums([SUM_FIT, SUM_TV, SUM_GG, SUM_DOT, SUM_FITC, SUM_TVC])
            h_y = fit + alpha * (tvs - nu * twoN) if tv else fit
            gn = math.sqrt(gg)
            if not math.isfinite(gn):
                raise SolveDiverged(f"objective became non-finite at lower iteration {t}")
            if gn <= tol:
                # converged: return y = x + beta (x - x_prev)   (lower_solvers.py:200-201)
                from .hypergradient import _vec
                out = []
                for x in X:
                    d = nat.empty_like_dev(x[ix].shape)
                    y = nat.empty_like_dev(x[ix].shape)
                    _vec(4, d.numel(), 0.0, x[ix], x[ixp], d)      # x - x_prev
                    _vec(0, d.numel(), beta, x[ix], d, y)          # x + beta (x - x_prev)
                    out.append(y)
                self.stats.update(vg_evals=vg, value_evals=vals, restarts=restarts, lip=lip)
                return self._owned(out), gn, t, True
            k = 0
            while True:
                val = fitc + alpha * tvc if tv else fitc + alpha * 0.0
                if val <= h_y - 0.5 * gn * gn / L_try + 1e-15 * abs(h_y):
                    break
                L_try *= 2.0
                k += 1
                if k >= 60:
                    raise SolveDiverged("backtracking line search failed to find a decreasing step")
                self._step(1, [x[ix] for x in X], [x[ixp] for x in X], [x[ic] for x in X], beta, L_try)
                vals += 1
                fitc, tvc, dot = self._sums([SUM_FITC, SUM_TVC, SUM_DOT])
            bstep = 1.0 / L_try
            lip_t = max(1.0 / bstep * 0.9, lip * 1e-8)
            ixp, ix = ix, ic
            if dot > 0.0:
                t_mom = 1.0
                ixp = ix
                restarts += 1
            for b in range(3):
                if b != ix and b != ixp:
                    ic = b
                    break
            self.comm.exchange(self.states, [x[ix] for x in X])
        # max_iters reached: gradient norm at x   (lower_solvers.py:212-213)
        X = [st.X for st in self.states]
        self._step(4, [x[ix] for x in X], [x[ix] for x in X], [None] * len(X))
        gn = math.sqrt(self._sums([SUM_GG])[0])
        self.stats.update(vg_evals=vg, value_evals=vals, restarts=restarts, lip=lip)
        return self._owned([x[ix] for x in X]), gn, max_iters, gn <= tol

    def _owned(self, arrs):
        return [a[st.slab.owned] for st, a in zip(self.states, arrs)]


def _lcm(a: int, b: int) -> int:
    import math as _m
    return a * b // _m.gcd(a, b)
