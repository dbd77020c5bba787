// Shared host/device parameter blocks for the MAID hot-path engine.
//
// Everything here is plain data: the host (adp_host.cpp) fills these once
// per plan / per call and passes them by value to cooperative kernels.
#pragma once
#include <stdint.h>

namespace adp {

// A deterministic sum over either
//   * the elements of a flattened array, combined in NumPy's pairwise order
//     (numpy/_core/src/umath/loops_utils.h.src pairwise_sum: blocks of <=128
//     with 8 accumulators, split at n/2 rounded down to a multiple of 8), or
//   * per-tile partials, combined by a fixed binary tree (ddot-type sums).
// The tree is evaluated from host-built "programs" (see adp_host.cpp):
//   prog = [nL, nI, nLev, lev_start[nLev+1], left[nI], right[nI]]
// node ids: 0..nL-1 leaves, nL.. internal nodes ordered by height.
// Large trees are cut into nSub subtrees (<= kMaxProgLeaves leaves each)
// evaluated in parallel, then a top program combines the subtree roots.
struct SumDev {
  int nLeaves;
  int nSub;
  int top_prog;            // offset (in ints) of the top program in progs
  int regular;             // 1: perfect binary tree over nLeaves (pow2 after zero padding for
                           //    tile sums; exact for element sums with equal leaves) -> evaluated
                           //    in registers / shuffles, subtrees of sub_size leaves
  int sub_size;            // regular two-level: leaves per subtree (pow2)
  int leaf_len;            // regular element sums: common leaf length (elements)
  int sub_own0, sub_own1;  // phase-1 subtrees evaluated by this plan ([0, nSub) unless a row slab)
  int sub_own2, sub_own3;  // second owned range (the 2N TV sums of a slab); empty otherwise
  const int64_t* leaf_start;  // nLeaves+1 element offsets (element sums only)
  const int* sub_leaf;     // nSub+1 leaf boundaries
  const int* sub_prog;     // nSub program offsets
  const int* progs;
  double* leaf_vals;       // nLeaves
  double* sub_vals;        // nSub
};

constexpr int kMaxProgLeaves = 2048;   // smem tree evaluation capacity (nL + nI <= 4095)
constexpr int kTreeStage = 16384;      // doubles of CTA tree staging (one batched pass over all
                                       // the sums of a decision point); then 512 doubles of scratch

// regularizer kinds (regularizers.py:75-199)
enum RegKind : int { REG_TV = 0, REG_ELASTIC = 1 };

// solver methods (lower_solvers.py:142-146)
enum Method : int { M_PROXGRAD = 0, M_AGD = 1, M_FISTA_SC = 2 };

// status codes written by device code
enum DevStatus : int {
  ST_OK = 0,
  ST_DIVERGED = 1,        // SolveDiverged: non-finite gradient norm at iteration t
  ST_BT_FAIL = 2,         // SolveDiverged: backtracking failed after 60 doublings
  ST_NEGCURV = 3,         // NegativeCurvatureError in CG
};

// Per-plan geometry and workspace for the depthwise 2-D path.
struct ConvGeom {
  int H, W, C;             // image (H, W, C), C-order float
  int kh, kw, rh, rw;      // stencil size and radii
  int TH, TW;              // tile
  int tilesH, tilesW, nTiles;
  int SH, SWP;             // smem plane rows / skewed row pitch (elements)
  int YSH, YSWP;           // small (1-halo) plane rows / pitch
  int threads;             // CTA size = TH * TW / RW
  int grid;                // persistent grid size (co-resident)
  int fused;               // 1: NumPy-pairwise leaves computed inside the tiles (regular,
                           //    tile-aligned layout); 0: global term arrays + leaf pass
  int leafL;               // common leaf length (elements) when fused
  int QP;                  // pitch of the TV Q planes
  int tpc;                 // threads per channel (TH * TW / RW); CTA = tpc * C threads
  int rwb;                 // register blocking RW of the instantiated kernels (1, 2, 4)
  int row0, Hg;            // row slab: global row of local row 0, global image rows (0, H otherwise)
  int own0, own1;          // row slab: owned local rows (multiples of TH); [0, H) otherwise
  int tileOff;             // global index of local tile 0 (row0 / TH * tilesW)
  unsigned magicTW;        // ceil(2^32 / tilesW): tile / tilesW = umulhi(tile, magicTW) (tile < 2^16)
  unsigned magicTWpx;      // ceil(2^32 / TW): w0 / TW = umulhi(w0, magicTWpx) (w0 < 2^16)
  int segs;                // fused: leaves per tile row (TW * C / leafL)
  unsigned magicSegs;      // ceil(2^32 / segs)
  int64_t rowL;            // fused: leaves per image row (W * C / leafL)
  unsigned magicC;         // ceil(2^20 / C): px = (e * magicC) >> 20 for e < 2^15
  unsigned magicRow;       // ceil(2^32 / rowE): row of a flattened tile-box index
  int o_ws, o_wf, o_pa, o_pq, o_tm, o_sv;   // byte offsets in dynamic smem
  int o_pa2;               // second plane region (fuseCA)
  int o_q;                 // TV neighbour (Q) scratch of the pipelined RW = 4 stages (0: not pipelined)
  int SWPt;                // dense plane pitch of TMA boxes (TW + 2 rw + 4, even)
  int fuseCA;              // 1: candidate value + speculative next value/grad share one stage
  int64_t N;               // H*W*C
  int64_t Ng;              // global element count (Hg*W*C; = N unless a row slab)
};

// Device scalar results (one block, written by CTA 0, copied to the host).
struct SolveOut {
  double lam;              // op_norm_sq result (power iteration), if computed
  double lip;              // Lipschitz constant used
  double grad_norm;        // ||grad|| at the returned point
  double value;            // last h(y) (diagnostic)
  int iters;               // LowerSolveResult.iters
  int converged;
  int status;              // DevStatus
  int fail_iter;           // iteration of divergence
  int power_iters;
  int power_converged;
  int64_t vg_evals;        // value+grad passes
  int64_t value_evals;     // value-only passes (backtracking)
  int64_t restarts;
  double t_mom, lip_t;     // state at exit
};

struct CGOut {
  double residual;         // true residual ||Hq - rhs||
  double curv;             // offending curvature when status == ST_NEGCURV
  double rs;               // last <r, s>
  int iters;
  int converged;
  int status;
  int hv;                  // Hessian-vector products issued
};

}  // namespace adp
