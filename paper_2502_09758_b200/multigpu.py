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


def run_instances(seeds, solve_one, timer=None, streams: int = 1):
    """Solve every assigned instance; returns (results in seed order, seconds).
    streams > 1: that many host threads, each with its own CUDA stream (and,
    through the per-thread plan cache, its own workspace), take instances
    from a shared queue, so one instance's kernels fill the device while
    another waits on its host-side decisions (the host-stepped solve) — the
    reference's concurrency model for distinct runs.  The
    C-ABI calls release the GIL (ctypes)."""
    import time
    t0 = time.perf_counter()
    if streams <= 1 or len(seeds) <= 1:
        out = [solve_one(s) for s in seeds]
        return out, time.perf_counter() - t0
    import queue
    import threading

    import torch
    dev = torch.cuda.current_device()
    work = queue.Queue()
    for k, s in enumerate(seeds):
        work.put((k, s))
    out = [None] * len(seeds)
    errors = []

    def worker():
        torch.cuda.set_device(dev)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            while True:
                try:
                    k, s = work.get_nowait()
                except queue.Empty:
                    break
                try:
                    out[k] = solve_one(s)
                except Exception as e:  # noqa: BLE001 - re-raised in the caller
                    errors.append(e)
                    break
            st.synchronize()

    threads = [threading.Thread(target=worker) for _ in range(min(streams, len(seeds)))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
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


SUM_FIT, SUM_TV, SUM_FITC, SUM_TVC, SUM_GG, SUM_DOT, SUM_RR = range(7)
_SLAB_PLANS: dict = {}   # (geometry, precision, device) -> Plan: slab plans are reused across kernels / calls


def _slab_plan(nat, rows, W, C, K, TH, TW, g0, H, own):
    key = (rows, W, C, K, TH, TW, g0, H, own, nat.get_precision()["dtype"], nat.get_precision()["mode"],
           nat.current_device())
    pl = _SLAB_PLANS.get(key)
    if pl is None:
        pl = nat.Plan(nat.LAYOUT_DEPTHWISE2D, (rows, W, C), (K, K), nat.get_precision()["dtype"],
                      nat.get_precision()["mode"], tile=(TH, TW), slab=(g0, H, own[0], own[1]))
        _SLAB_PLANS[key] = pl
    return pl


class SlabSolver:
    """solve_lower (agd, adaptive: the c2-c5 settings) of one image split into
    row slabs.  `ranks` are the slab indices held by this process: all of
    them with LocalComm (one device), [rank] with DistComm.  The slab plans
    are cached per geometry; `bind(p)` (or assigning `.p`) points the solver
    at another lower problem (kernel / data) of the same shape."""

    def __init__(self, p, world: int, ranks=None, comm=None):
        import ctypes
        from . import _native as nat
        from .operators import ConvOperator
        from .regularizers import SmoothedTV
        if not isinstance(p.op, ConvOperator) or not isinstance(p.reg, SmoothedTV):
            raise ValueError("row slabs: depthwise 2-D operator with SmoothedTV")
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
        align = _lcm(TH, 16)                     # 16: kernel_gram_correlation tile rows (hypergradient)
        n_leaves = H * W * C // L
        if n_leaves > 4096:                      # two-level element sums: subtree-aligned rows
            align = _lcm(align, max(1, 2048 * L // (W * C)))
        tiles_h = (H + TH - 1) // TH
        if tiles_h * tilesW > 4096:              # two-level tile sums
            align = _lcm(align, max(1, 2048 // tilesW) * TH)
        r = K // 2
        gw = -(-(3 * r + 1) // TH) * TH          # ghost rows: 3r + 1, tile aligned
        self.slabs = plan_slabs(H, world, K, row_align=align, ghost=gw)
        for sl in self.slabs:
            if (sl.row1 - sl.row0) < gw and world > 1:
                raise ValueError(f"slab of {sl.row1 - sl.row0} rows is thinner than its ghost width {gw}")
        self.ranks = list(range(world)) if ranks is None else list(ranks)
        self.comm = comm if comm is not None else LocalComm()
        if isinstance(self.comm, LocalComm) and len(self.ranks) != world:
            raise ValueError("LocalComm holds every slab")
        self.states = []
        for rk in self.ranks:
            sl = self.slabs[rk]
            g0 = sl.row0 - sl.ghost_top
            rows = sl.local_rows
            own = (sl.ghost_top, sl.ghost_top + sl.row1 - sl.row0)
            plan = _slab_plan(nat, rows, W, C, K, TH, TW, g0, H, own)
            X = [nat.empty_like_dev((rows, W, C)) for _ in range(3)]
            self.states.append(_SlabState(sl, plan, p.reg.native(), (), X))
        self.units_meta = []
        for which in range(7):
            n = ctypes.c_int64()
            own = (ctypes.c_int64 * 4)()
            nat.check(nat.lib().adp_slab_units(self.states[0].plan.handle, which, ctypes.byref(n), own, None, None),
                      "adp_slab_units")
            self.units_meta.append(int(n.value))
        self.stats = {}
        self._ycache = (None, None)
        self.bind(p)

    # -- lower problem binding (kernel b, data y, alpha)
    @property
    def p(self):
        return self._p

    @p.setter
    def p(self, value):
        self.bind(value)

    def bind(self, p):
        from .lower_solvers import _check_reg_smooth
        if tuple(p.op.signal_shape) != self.shape or p.op.kernel.data.shape[:2] != (self.K, self.K):
            raise ValueError("bind: the slab solver's geometry differs from the problem's")
        _check_reg_smooth(p)
        self._p = p
        kd = p.op.kernel.device()
        if self._ycache[0] is not p.y:
            self._ycache = (p.y, self.local(p.y))
        ys = self._ycache[1]
        for st, yd in zip(self.states, ys):
            low = p.reg.native()
            low.kernel = kd.data_ptr()
            low.y = yd.data_ptr()
            low.alpha = float(p.alpha)
            st.lower = low
            st.keep = (kd, yd)
        return self

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

    def local(self, full):
        """Per-state local arrays (slab + ghosts) of a full image (host or device)."""
        nat = self.nat
        out = []
        for st in self.states:
            sl = st.slab
            g0 = sl.row0 - sl.ghost_top
            part = full[g0:g0 + sl.local_rows]
            out.append(nat.to_dev(part.contiguous() if nat.is_torch(part) else np.ascontiguousarray(part)).clone())
        return out

    _local = local

    def exchange(self, arrays):
        self.comm.exchange(self.states, arrays)

    def op_norm_sq(self, max_iters: int = 300, tol: float = 1e-4):
        """Power iteration on B^T B (operators.py:137-173) over the slabs."""
        nat = self.nat
        src = self.local(nat.power_start(self.shape))
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
            self.exchange(src)
        self.stats.update(power_iters=iters, power_converged=conv)
        return lam

    def solve(self, x0, eps: float, mu: float, max_iters: int = 1200, norm_sq: float | None = None):
        """Adaptive AGD (lower_solvers.py:180-213) from a full image x0.
        Returns (x_owned list per held slab, grad_norm, iters, converged)."""
        xs, gn, it, conv = self.solve_local(self.local(x0), eps, mu, max_iters, norm_sq)
        return self._owned(xs), gn, it, conv

    def solve_local(self, xs, eps: float, mu: float, max_iters: int = 1200, norm_sq: float | None = None):
        """Adaptive AGD from per-slab local arrays (ghost rows valid); returns
        fresh local arrays of x~ with valid ghost rows, grad_norm, iters,
        converged (x~ is the extrapolated point on convergence, :200-201)."""
        from .lower_solvers import SolveDiverged
        nat = self.nat
        p = self._p
        H, W, C = self.shape
        if eps <= 0 or mu <= 0:
            raise ValueError("eps and mu must be > 0")
        tol = eps * mu
        if norm_sq is None:
            norm_sq = p.op._norm_sq if p.op._norm_sq is not None else self.op_norm_sq()
            p.op._norm_sq = norm_sq                   # the operator's norm cache (operators.py:172)
        lam = float(norm_sq)
        alpha, nu = float(p.alpha), float(p.reg.nu)
        lip = 2.0 * lam + alpha * p.reg.curvature
        twoN = 2.0 * float(H * W * C)
        tv = alpha != 0.0
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
                return out, gn, t, True
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
            self.exchange([x[ix] for x in X])
        # max_iters reached: gradient norm at x   (lower_solvers.py:212-213)
        X = [st.X for st in self.states]
        self._step(4, [x[ix] for x in X], [x[ix] for x in X], [None] * len(X))
        gn = math.sqrt(self._sums([SUM_GG])[0])
        self.stats.update(vg_evals=vg, value_evals=vals, restarts=restarts, lip=lip)
        return [x[ix].clone() for x in X], gn, max_iters, gn <= tol

    def _owned(self, arrs):
        return [a[st.slab.owned] for st, a in zip(self.states, arrs)]

    def gather(self, arrs):
        """Full image from per-slab local arrays (LocalComm: every slab here;
        DistComm: all-gather of the owned rows)."""
        import torch
        owned = self._owned(arrs)
        if isinstance(self.comm, LocalComm):
            return torch.cat(owned, dim=0)
        import torch.distributed as dist
        H, W, C = self.shape
        rows = [sl.row1 - sl.row0 for sl in self.slabs]
        n = max(rows)
        pad = torch.zeros((n, W, C), dtype=owned[0].dtype, device=owned[0].device)
        pad[: owned[0].shape[0]] = owned[0]
        parts = [torch.empty_like(pad) for _ in self.slabs]
        if pad.is_cuda and dist.get_backend(self.comm.group) != "nccl":
            hp = pad.cpu()
            hparts = [torch.empty_like(hp) for _ in self.slabs]
            dist.all_gather(hparts, hp, group=self.comm.group)
            parts = [h.to(pad.device) for h in hparts]
        else:
            dist.all_gather(parts, pad, group=self.comm.group)
        return torch.cat([pp[:r] for pp, r in zip(parts, rows)], dim=0)


# ---------------------------------------------------------------------------
# c5: the hypergradient and MAID on row slabs.  Same scheme as the lower
# solve: each step of the unsplit kernels (conv_cg_kernel, CM_UPPER,
# adp_mixed_T) runs over slab + ghosts and stops at its reductions; the ranks
# assemble the sum units (all-reduce SUM of zero-filled vectors: exact) and
# fold them in the single-GPU tree order, so every scalar — and hence every
# decision — is bitwise that of one GPU.  Ghost rows are refreshed by one
# exchange of the CG preconditioned residual per CG iteration and of q before
# the true residual; x~ leaves the solve with valid ghosts.

class SlabHypergradient:
    """inexact_hypergradient (hypergradient.py:148-190) and the upper terms
    of an UpperProblem whose image is split into row slabs.  The upper
    operator A must have the lower stencil's size (the slab plans are shared)."""

    def __init__(self, upper, world: int, ranks=None, comm=None):
        from . import _native as nat
        self.nat = nat
        self.upper = upper
        p0 = upper.lower_problem(upper.b0)
        self.sv = SlabSolver(p0, world, ranks, comm)
        if upper.A.kernel.data.shape[:2] != (self.sv.K, self.sv.K):
            raise ValueError("row slabs: the upper operator's stencil must have the lower stencil's size")
        self.yd = self.sv.local(upper.y_delta)
        self.stats = {}

    @property
    def states(self):
        return self.sv.states

    # -- upper terms: (fit, ||2 A^T (A x - y)||, grads) from local x~ arrays
    def upper_terms(self, xs, want_grad: bool = False):
        nat = self.nat
        ka = self.upper.A.kernel.device()
        grads = [nat.empty_like_dev(x.shape) for x in xs]
        for st, x, y, g in zip(self.states, xs, self.yd, grads):
            nat.check(nat.lib().adp_slab_upper(st.plan.handle, nat.ptr(ka), nat.ptr(x), nat.ptr(y), nat.ptr(g),
                                               nat.stream_ptr()), "adp_slab_upper")
        fit, gg = self.sv._sums([SUM_FIT, SUM_GG])
        return fit, math.sqrt(gg), (grads if want_grad else None)

    def _cg(self, op, in0=None, in1=None, out0=None, out1=None, s=0.0, flag=0):
        nat, ct = self.nat, self.sv.ctypes
        n = len(self.states)
        in0 = in0 or [None] * n
        in1 = in1 or [None] * n
        out0 = out0 or [None] * n
        out1 = out1 or [None] * n
        vals = []
        for st, a, b, c, d in zip(self.states, in0, in1, out0, out1):
            v = ct.c_double(0.0)
            nat.check(nat.lib().adp_slab_cg(st.plan.handle, ct.byref(st.lower), int(op), nat.ptr(a), nat.ptr(b),
                                            nat.ptr(c), nat.ptr(d), float(s), int(flag), ct.byref(v),
                                            nat.stream_ptr()), "adp_slab_cg")
            vals.append(v.value)
        return vals

    def _max_over_ranks(self, v: float) -> float:
        comm = self.sv.comm
        if isinstance(comm, LocalComm):
            return v
        import torch
        import torch.distributed as dist
        t = torch.tensor([v], dtype=torch.float64)
        if dist.get_backend(comm.group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=comm.group)
        return float(t.item())

    def hess_cg(self, xs, rhs, tol: float, max_iters: int, qs=None):
        """Jacobi-PCG on the lower Hessian at x~ (conv_cg_kernel: cg_solve on
        lower_hess_vec with lower_hess_diag, hypergradient.py:35-84).  Returns
        (q local arrays with valid ghosts, residual, iters, converged, hv)."""
        from .hypergradient import _negcurv
        nat = self.nat
        sv = self.sv
        if tol <= 0:
            raise ValueError("tol must be > 0")
        shapes = [x.shape for x in xs]
        S = [nat.empty_like_dev(sh) for sh in shapes]
        P = [[nat.empty_like_dev(sh) for sh in shapes], [nat.empty_like_dev(sh) for sh in shapes]]
        warm = qs is not None
        Q = [q.clone() for q in qs] if warm else [nat.empty_like_dev(sh) for sh in shapes]
        hv = 0
        # TV weights and the Jacobi diagonal; floor 1e-12 * max + 1e-300 over the whole image (lower_solvers.py:80)
        mx = max(self._cg(0, in0=xs))
        mx = self._max_over_ranks(mx)
        fl = 1e-12 * mx + 1e-300
        if warm:
            self._cg(2, in0=Q, out0=P[1], flag=3)     # H q0 (Q ghosts valid)
            hv += 1
        self._cg(1, in0=rhs, out0=Q, out1=S, s=fl, flag=1 if warm else 0)
        rs, rr = sv._sums([SUM_DOT, SUM_RR])
        sv.exchange(S)
        iters, cur, first, beta = 0, 0, True, 0.0
        curv = 0.0
        for iters in range(1, max_iters + 1):
            if math.sqrt(rr) <= tol:
                iters -= 1
                break
            nxt = cur if first else cur ^ 1
            self._cg(2, in0=S, in1=P[cur], out0=P[nxt], s=beta, flag=0 if first else 1)
            hv += 1
            cur, first = nxt, False
            curv = sv._sums([SUM_GG])[0]
            if curv <= 0.0:
                raise _negcurv(curv)
            al = rs / curv
            self._cg(3, in0=P[cur], out0=Q, out1=S, s=al)
            o0, o1 = sv._sums([SUM_DOT, SUM_RR])
            beta = o0 / rs
            rs, rr = o0, o1
            sv.exchange(S)
        else:
            iters = max_iters
        if iters > max_iters:
            iters = max_iters
        sv.exchange(Q)
        self._cg(2, in0=Q, in1=rhs, out0=P[cur ^ 1], flag=2)   # true residual ||H q - rhs|| (hypergradient.py:83)
        hv += 1
        res = math.sqrt(sv._sums([SUM_GG])[0])
        return Q, res, iters, res <= tol, hv

    def mixed(self, b, xs, qs):
        """mixed_second_transpose (hypergradient.py:92-104) as a host
        (kh, kw, C) array: per-slab kernel-gram partials of the owned groups,
        assembled over ranks, folded in the unsplit group order."""
        import torch
        nat, ct = self.nat, self.sv.ctypes
        ng, nt = ct.c_int32(), ct.c_int32()
        st0 = self.states[0]
        nat.check(nat.lib().adp_kgc_groups(st0.plan.handle, ct.byref(ng), ct.byref(nt)), "adp_kgc_groups")
        part = torch.zeros(ng.value * nt.value, dtype=torch.float64, device="cuda")
        for st, x, q in zip(self.states, xs, qs):
            nat.check(nat.lib().adp_slab_mixed(st.plan.handle, ct.byref(st.lower), nat.ptr(x), nat.ptr(q),
                                               nat.ptr(part), nat.stream_ptr()), "adp_slab_mixed")
        part = self.sv.comm.assemble([part])[0]
        out = nat.empty_like_dev(b.data.shape)
        nat.check(nat.lib().adp_kgc_final(st0.plan.handle, nat.ptr(part), nat.ptr(out), 2.0, nat.stream_ptr()),
                  "adp_kgc_final")
        return nat.to_host(out).astype(float)

    def solve(self, b, xs, eps: float, max_iters=None):
        """solve_lower at kernel b from local arrays (UpperProblem's solver
        settings: adaptive AGD); returns (xs, gn, iters, converged, mu)."""
        from .lower_solvers import mu_of_b
        up = self.upper
        if up.lower_method != "agd" or not up.lower_adaptive or up.lower_step is not None:
            raise ValueError("row slabs run the 2-D settings: adaptive AGD with the L(b) step")
        p = up.lower_problem(b)
        self.sv.bind(p)
        mu = mu_of_b(p, up.mu_floor)
        budget = up.lower_max_iters if max_iters is None else max_iters
        xo, gn, it, conv = self.sv.solve_local(xs, eps, mu, max_iters=budget)
        return xo, gn, it, conv, mu

    def hypergradient(self, b, eps: float, delta: float, state, cg_max_iters: int = 200):
        """Algorithm 1 (hypergradient.py:148-190) on slabs; `state` holds
        per-slab local arrays (x, q)."""
        from .hypergradient import HypergradResult, sobolev_grad
        if eps <= 0 or delta <= 0:
            raise ValueError("eps and delta must be > 0")
        xs, gn, it, conv, mu = self.solve(b, state.x, eps)
        state.x = xs
        _, _, rhs = self.upper_terms(xs, want_grad=True)
        q, res, cg_it, cg_conv, _ = self.hess_cg(xs, rhs, delta, cg_max_iters, qs=state.q)
        state.q = q
        z = -self.mixed(b, xs, q) + sobolev_grad(b, self.upper.a, self.upper.beta)
        return HypergradResult(z=z, x_tilde=xs, cg_iters=cg_it, lower_iters=it, cg_residual=res,
                               epsilon_used=gn / mu, delta_used=delta, lower_converged=conv, cg_converged=cg_conv,
                               mu=mu)


class _SlabSolveResult:
    def __init__(self, xs, gn, iters, conv, mu):
        self.x_tilde, self.grad_norm, self.iters, self.converged = xs, gn, iters, conv
        self.epsilon_achieved = gn / mu


class SlabEngine:
    """maid.maid_run's image-space calls on row slabs (maid.DeviceEngine's
    interface): x iterates are per-slab local arrays; kernel-space work and
    every MAID decision run identically on each rank."""

    def __init__(self, upper, world: int, ranks=None, comm=None):
        self.upper = upper
        self.hg = SlabHypergradient(upper, world, ranks, comm)

    def lip(self) -> float:
        """lip_upper_x (maid.py:100-102): 2 ||A||^2 by power iteration (500, 1e-6)."""
        from .lower_solvers import LowerProblem
        up = self.upper
        if up.A._norm_sq is None:        # cached on the operator, as op_norm_sq does (operators.py:172)
            sv = self.hg.sv
            sv.bind(LowerProblem(up.A, up.y_delta, up.alpha, up.reg))
            up.A._norm_sq = sv.op_norm_sq(500, 1e-6)
        return 2.0 * up.A._norm_sq

    def initial_state(self):
        from .hypergradient import WarmState
        return WarmState(x=self.hg.sv.local(self.upper.x0))

    def hypergradient(self, b, eps, delta, state, cg_max_iters):
        return self.hg.hypergradient(b, eps, delta, state, cg_max_iters)

    def loss_and_gnorm(self, xs, b):
        from .hypergradient import sobolev_value
        fit, gn, _ = self.hg.upper_terms(xs)
        return fit + sobolev_value(b, self.upper.a, self.upper.beta), gn

    def solve_candidate(self, b, xs, eps, max_iters=None):
        xo, gn, it, conv, mu = self.hg.solve(b, xs, eps, max_iters)
        return _SlabSolveResult(xo, gn, it, conv, mu)

    def exact_loss(self, b, xs, cfg):
        sol = self.solve_candidate(b, xs, cfg.audit_eps, max_iters=cfg.audit_max_iters)
        return self.final_loss(sol.x_tilde, b)

    def final_loss(self, xs, b) -> float:
        return self.loss_and_gnorm(xs, b)[0]

    def to_host(self, xs):
        return self.hg.sv.nat.to_host(self.hg.sv.gather(xs)).astype(float)


def slab_maid_run(upper, cfg, world: int, ranks=None, comm=None, b0=None):
    """maid_run (maid.py:149-255) with the image in row slabs over `world`
    ranks: same decisions and iterates as the single-GPU run, bitwise."""
    from .maid import maid_run
    return maid_run(upper, cfg, b0, engine=SlabEngine(upper, world, ranks, comm))


def _lcm(a: int, b: int) -> int:
    import math as _m
    return a * b // _m.gcd(a, b)
