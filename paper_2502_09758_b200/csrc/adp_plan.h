// Host-side plan: geometry, workspace and deterministic-sum programs.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>
#include "adp_types.h"
#include "conv2d_args.h"   // StepW
#include "step_tail.h"
#include "../../include/adp_b200.h"

namespace adp {

// Deterministic sum layout built on the host (see adp_types.h SumDev).
struct SumHost {
  int64_t n = 0;              // elements (np rule) or items (binary rule)
  bool np = true;
  std::vector<int64_t> leaf_start;
  std::vector<int> sub_leaf, sub_prog;
  int top_prog = 0;
  int nLeaves = 0, nSub = 1;
  int regular = 0, sub_size = 0, leaf_len = 0;
};

// Programs for all sums of a plan live in one int32 buffer.
struct ProgPool {
  std::vector<int> words;
  std::vector<std::pair<std::string, int>> memo;
  int add(const std::string& key, const std::vector<int>& prog);
};

void build_sum(SumHost& s, int64_t n, bool np, ProgPool& pool, bool allow_regular = true);

struct KernelInfo {
  const void* fn = nullptr;
  int grid = 0;
  bool attr_set = false;
};

struct PlanImpl {
  adp_plan_desc d{};
  ConvGeom g{};
  int esize = 8;
  size_t smem = 0;
  size_t smem_optin = 0;        // device max dynamic smem per block (function attribute set to this)
  bool probe_only = false;      // adp_plan_probe: stop after the geometry
  int sm_count = 0;
  // device memory
  void* dmem = nullptr;
  void* d_zero = nullptr;        // zero stencil + zero image (regularizer-only calls)
  size_t dbytes = 0;
  void* ws[24] = {};            // workspace arrays (T*)
  int nws = 0;
  int* d_progs = nullptr;
  int64_t* d_leaf_N = nullptr;  // leaf starts for N-element sums
  int64_t* d_leaf_2N = nullptr;
  int* d_sub[8] = {};           // sub_leaf / sub_prog per layout
  SumDev s_fit{}, s_tv{}, s_fitc{}, s_tvc{}, s_t0{}, s_t1{}, s_t2{}, s_fit2{}, s_tv2{};
  int64_t units_n[7] = {};       // sum units (leaves, or subtree roots when two-level)
  int64_t units_own[7][4] = {};  // unit ranges this plan fills (row slabs: its owned rows)
  unsigned int* d_bar = nullptr;
  SolveOut* d_sres = nullptr;
  CGOut* d_cres = nullptr;
  double* d_scal = nullptr;
  double* d_kgc_part = nullptr;
  int kgc_groups = 0;
  int kgc_cblocks = 1;
  int tma = 0;                  // KS = 9 solve kernel with TMA tile boxes (tm[] valid)
  int step = 0;                 // host-stepped high-occupancy solve (conv2d_step.cu) for this plan
  KernelInfo k_sb, k_sc, k_sa, k_sred, k_sca;
  size_t step_smem_b = 0;
  int* h_flag = nullptr;        // mapped pinned: host-stepped solve's reduction-ready sequence number
  int step_seq = 0;
  int profile = 0;              // adp_plan_profile: time the dominant kernel of host-stepped solves
  cudaEvent_t prof_ev[2] = {nullptr, nullptr};
  const void* k_extrap = nullptr;
  const void* k_cand = nullptr;
  size_t step_smem = 0;
  int step_o_tm = 0;
  double* h_kern = nullptr;     // pinned: the solve's stencil, read back to build the stage kernels' tap sets
  StepWL wfwd{}, wadj{};        // forward / flipped taps (kernel parameters of the stage kernels; the
                                // instances for stencils of <= kStepWSmall taps read the first part only)
  bool pdl = true;              // stage kernels launched with programmatic stream serialization (ADP_PDL=0: off)
  StepTail tail{};              // in-kernel decision sums of the host-stepped solve (tail.on: geometry allows it)
  void* d_tail = nullptr;       // sub-values + tickets + per-tile stage-B completion flags
  unsigned int* d_tflag = nullptr;   // the flags (NULL: the candidate launch does not overlap stage B)
  unsigned int tile_seq = 0;    // sequence number of the last stage-B launch
  unsigned int a_seq = 0;       // ... of the last candidate launch publishing its stage-A tiles
  bool ovl_b = false;           // stage B overlaps the candidate launch's last wave too (ADP_OVL=2)
  CUtensorMap tm[5];            // X[0..2], R, P[0]
  // pinned host staging
  SolveOut* h_sres = nullptr;
  CGOut* h_cres = nullptr;
  double* h_scal = nullptr;
  KernelInfo k_solve, k_cg, k_misc;
  unsigned long long* d_trace = nullptr;   // debug: per-phase timestamps of solve (adp_debug_trace)
  // dense 1-D engine data
  int dense_grid = 0;
  size_t dense_smem = 0;
};

}  // namespace adp

struct adp_plan {
  adp::PlanImpl impl;
};
