// Host-stepped solve: in-kernel ("tail") evaluation of the decision sums.
//
// The launches that evaluate a candidate (candidate value + speculative stage
// A; backtracking retry) carry a few reducer CTAs between their two halves
// instead of being followed by a reduction launch.  The candidate half's sum
// leaves and tile partials are pre-set to an all-ones NaN pattern; a reducer
// polls its tile rows' units until they are written (each unit is one 8-byte
// store, so no fence, ticket or barrier is needed on the producers' side),
// folds them into sub-values and resets them; the reducers take a ticket and
// the last one folds the sub-values of all six sums and writes them, then a
// sequence number, to mapped pinned host memory.  The tree is the one reduce_k
// evaluates (perfect binary tree in leaf order, zero padded), so the sums are
// bitwise those of step_reduce_kernel; only the distribution of the work
// differs.  The candidate CTAs come first in the grid, so the host has the
// decision while the speculative half still runs and the next launch is
// queued before the kernel ends.
#pragma once

namespace adp {

struct StepTail {
  double* sub;          // sub-values, see the offsets below (11 * nG doubles)
  unsigned int* cnt;    // reducer ticket (zero between launches)
  int on;               // 0: no tail (the host launches step_reduce_kernel)
  int nG;               // groups = tile rows (power of two)
  int GL;               // leaves of an N-element sum per group (power of two, <= 1024)
  int tW;               // tiles per group (power of two)
  int nR;               // reducer CTAs of a launch
  int gpr;              // groups per reducer
  int setR;             // (fit, tv) set the decision of this launch reads: 0 / 1
  int ovl;              // 1: this launch overlaps the stage-B launch before it: no grid dependency wait, every
                        //    CTA waits for the stage-B tiles it reads (ConvArgs::tflag / tseq) instead
  unsigned int aseq;    // != 0: the stage-A half publishes its tiles' completion (flags tflag + nTiles, this
                        //    value) for a stage-B launch that overlaps this launch's last wave
  // sub-value offsets (doubles)
  __host__ __device__ int o_fit() const { return 0; }
  __host__ __device__ int o_tv() const { return 2 * nG; }
  __host__ __device__ int o_fitc() const { return 6 * nG; }
  __host__ __device__ int o_tvc() const { return 7 * nG; }
  __host__ __device__ int o_t0() const { return 9 * nG; }
  __host__ __device__ int o_t1() const { return 10 * nG; }
};

}  // namespace adp
