/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY.  Used by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs as the checker or the
 * timed CPU baseline; never linked into or called by the product path.
 *
 * C restatements of the three third-party arithmetic kernels the reference
 * (arxiv 2502.09758 `adp`, /root/reference/pkg/src/adp) reaches through
 * NumPy/SciPy on its hot path:
 *
 *  1. scipy.ndimage.correlate(mode="constant", cval=0)  (SciPy 1.18.1,
 *     called at operators.py:104-105): for every output, acc = 0.0 and then
 *     acc = acc + x * w over the taps in row-major order, skipping taps with
 *     |w| <= DBL_EPSILON; out-of-image samples are cval = 0.0.
 *  2. NumPy pairwise summation (NumPy 2.3.5, loops_utils.h.src
 *     pairwise_sum, reached by every np.sum on the path, e.g.
 *     lower_solvers.py:39,53 and regularizers.py:19,174): blocks of <= 128
 *     with 8 accumulators, recursive split at n/2 rounded down to a multiple
 *     of 8.
 *  3. OpenBLAS 0.3.30 ddot, SkylakeX kernel, one thread (np.dot / np.vdot /
 *     np.linalg.norm at lower_solvers.py:150,198,209, hypergradient.py:63-83,
 *     maid.py:125,188-190, operators.py:150,155): 4 x 8-lane FMA accumulators
 *     over blocks of 32, folded to 4 x 4 lanes, then 4 x 4-lane accumulators
 *     over a trailing block of 16, lane-wise sum ((a0+a1)+a2)+a3, horizontal
 *     (l0+l2)+(l1+l3), then a scalar FMA tail.
 *
 * Each is pinned bitwise against the real NumPy/SciPy in this container by
 * tests/test_oracle_pin.py and the committed golden vectors.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; no implicit FMA).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>

void orc_correlate(const double* x, int64_t H, int64_t W, int64_t C, const double* w, int64_t kh, int64_t kw,
                   int flip, double* out) {
  const int64_t rh = kh / 2, rw = kw / 2;
  for (int64_t h = 0; h < H; ++h)
    for (int64_t q = 0; q < W; ++q)
      for (int64_t c = 0; c < C; ++c) {
        double acc = 0.0;
        for (int64_t i = 0; i < kh; ++i)
          for (int64_t j = 0; j < kw; ++j) {
            const int64_t ii = flip ? kh - 1 - i : i, jj = flip ? kw - 1 - j : j;
            const double wt = w[(ii * kw + jj) * C + c];
            if (!(fabs(wt) > DBL_EPSILON)) continue;
            const int64_t hh = h + i - rh, ww = q + j - rw;
            const double xv = (hh >= 0 && hh < H && ww >= 0 && ww < W) ? x[(hh * W + ww) * C + c] : 0.0;
            acc = acc + xv * wt;
          }
        out[(h * W + q) * C + c] = acc;
      }
}

static double pw(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = r + a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] = r[k] + a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res = res + a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pw(a, n2) + pw(a + n2, n - n2);
}

double orc_pairwise_sum(const double* a, int64_t n) { return pw(a, n); }

double orc_ddot(const double* x, const double* y, int64_t n) {
  int64_t i = 0;
  const int64_t n1 = n & -16;
  if (n1) {
    double a512[4][8];
    double a256[4][4];
    for (int k = 0; k < 4; ++k)
      for (int l = 0; l < 8; ++l) a512[k][l] = 0.0;
    const int64_t n32 = n1 & ~(int64_t)31;
    for (; i < n32; i += 32)
      for (int k = 0; k < 4; ++k)
        for (int l = 0; l < 8; ++l) a512[k][l] = fma(x[i + 8 * k + l], y[i + 8 * k + l], a512[k][l]);
    for (int k = 0; k < 4; ++k)
      for (int l = 0; l < 4; ++l) a256[k][l] = a512[k][l] + a512[k][l + 4];
    for (; i < n1; i += 16)
      for (int k = 0; k < 4; ++k)
        for (int l = 0; l < 4; ++l) a256[k][l] = fma(x[i + 4 * k + l], y[i + 4 * k + l], a256[k][l]);
    double s[4];
    for (int l = 0; l < 4; ++l) s[l] = ((a256[0][l] + a256[1][l]) + a256[2][l]) + a256[3][l];
    double dot = (s[0] + s[2]) + (s[1] + s[3]);
    for (; i < n; ++i) dot = fma(y[i], x[i], dot);
    return dot;
  }
  double dot = 0.0;
  for (; i < n; ++i) dot = fma(y[i], x[i], dot);
  return dot;
}
