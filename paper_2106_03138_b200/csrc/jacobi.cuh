// One-sided (Hestenes) Jacobi SVD of a batch of small matrices: the device
// counterpart of the reference's verification oracle jacobi_svd
// (svd.py:117-143, sweeps svd.py:74-114), used by the rank-revealing ratio
// diagnostics (harness._ratio_fields, harness.py:201-216) over whole batches
// (BASELINE cfg3: 1024 matrices).  Verification tooling, off the
// factorization path.
//
// Same rotation and the same stopping rule as the reference: a pair (i < j)
// with a = |x_i|^2, b = |x_j|^2, g = x_i . x_j is skipped when a, b or g is 0 or
// g^2 <= tol^2 a b; otherwise zeta = (b - a) / 2g, t = sign(zeta) / (|zeta| +
// sqrt(1 + zeta^2)), c = 1 / sqrt(1 + t^2), s = c t, x_i <- c x_i - s x_j,
// x_j <- s x_i + c x_j; sweeps stop once no applied rotation had |s| > tol.
// The pairs of a sweep are visited in round-robin (circle-method) rounds of
// n/2 disjoint pairs instead of the reference's row-cyclic order, so the
// columns of a round rotate in parallel (one warp per pair): the singular
// values agree with the reference's to rounding, the sweep count may differ.
// sigma_j = |x_j| at the end (unsorted; the caller sorts).
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int JS_T = 256;      // 8 warps: one pair per warp at a time
constexpr int JS_NMAX = 512;   // the reference's desk-scale cap (svd.py: _MAX_COLS)

// column j of matrix X (ld), rows [0, m): (sum x_i^2, sum x_j^2, sum x_i x_j), warp-wide
__device__ __forceinline__ void js_dots(const double* xi, const double* xj, int64_t m, int lane, double& a,
                                        double& b, double& g) {
  double a0 = 0.0, b0 = 0.0, g0 = 0.0, a1 = 0.0, b1 = 0.0, g1 = 0.0;
  int64_t r = lane;
  for (; r + 32 < m; r += 64) {
    const double p = xi[r], q = xj[r], p1 = xi[r + 32], q1 = xj[r + 32];
    a0 = fma(p, p, a0);
    b0 = fma(q, q, b0);
    g0 = fma(p, q, g0);
    a1 = fma(p1, p1, a1);
    b1 = fma(q1, q1, b1);
    g1 = fma(p1, q1, g1);
  }
  if (r < m) {
    const double p = xi[r], q = xj[r];
    a0 = fma(p, p, a0);
    b0 = fma(q, q, b0);
    g0 = fma(p, q, g0);
  }
  a = warp_sum(a0 + a1);
  b = warp_sum(b0 + b1);
  g = warp_sum(g0 + g1);
}

// grid: persistent CTAs over the batch.  X: batch matrices (m x n, column-major,
// ld, stride doubles apart), overwritten; sig: batch x n; sweeps / conv: batch.
__global__ void __launch_bounds__(JS_T) k_jacobi_svd(double* __restrict__ X, int64_t batch, int64_t m, int n,
                                                     int64_t ld, int64_t stride, double tol, int max_sweeps,
                                                     double* __restrict__ sig, int32_t* __restrict__ sweeps_out,
                                                     int32_t* __restrict__ conv_out) {
  __shared__ double s_max[JS_T / 32];
  __shared__ int s_conv;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nwarp = JS_T / 32;
  const int np = n + (n & 1);  // an odd n gets a dummy column (its pairs are skipped)
  const int nr = np - 1;       // rotating players of the circle method
  const double tol2 = tol * tol;
  for (int64_t bi = blockIdx.x; bi < batch; bi += gridDim.x) {
    double* Xb = X + bi * stride;
    int sweeps = 0;
    bool conv = (n < 2);
    while (sweeps < max_sweeps && !conv) {
      ++sweeps;
      double my_max = 0.0;
      for (int rd = 0; rd < nr; ++rd) {
        for (int p = wid; p < np / 2; p += nwarp) {
          // circle method: player nr is fixed and meets rd; the rest pair up around rd
          int i, j;
          if (p == 0) {
            i = rd;
            j = nr;
          } else {
            i = (rd + p) % nr;
            j = (rd - p + nr) % nr;
          }
          if (i > j) {
            const int t = i;
            i = j;
            j = t;
          }
          if (j >= n) continue;  // the dummy column
          double* xi = Xb + (int64_t)i * ld;
          double* xj = Xb + (int64_t)j * ld;
          double a, b, g;
          js_dots(xi, xj, m, lane, a, b, g);
          if (a == 0.0 || b == 0.0 || g == 0.0) continue;
          if (g * g <= tol2 * a * b) continue;
          const double zeta = (b - a) / (2.0 * g);
          const double t = (zeta >= 0.0) ? 1.0 / (zeta + sqrt(1.0 + zeta * zeta))
                                         : -1.0 / (-zeta + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t);
          const double s = c * t;
          my_max = fmax(my_max, fabs(s));
          for (int64_t r = lane; r < m; r += 32) {
            const double p0 = xi[r], q0 = xj[r];
            xi[r] = c * p0 - s * q0;
            xj[r] = s * p0 + c * q0;
          }
        }
        __syncthreads();  // the next round's pairs read these columns
      }
      if (lane == 0) s_max[wid] = my_max;
      __syncthreads();
      if (tid == 0) {
        double mx = 0.0;
        for (int w = 0; w < nwarp; ++w) mx = fmax(mx, s_max[w]);
        s_conv = (mx <= tol);
      }
      __syncthreads();
      conv = s_conv != 0;
      __syncthreads();
    }
    // sigma_j = |x_j| (column_norms, matrix.py:61-78: max-scaled when needed)
    // (plain loads: the columns were written by this kernel, so no read-only path)
    for (int j = wid; j < n; j += nwarp) {
      const double* x = Xb + (int64_t)j * ld;
      double ss = 0.0, am = 0.0;
      for (int64_t r = lane; r < m; r += 32) {
        ss = fma(x[r], x[r], ss);
        am = fmax(am, fabs(x[r]));
      }
      ss = warp_sum(ss);
      am = warp_max(am);
      double v = 0.0;
      if (am > 0.0) {
        if (norm_range_ok(am)) {
          v = sqrt(ss);
        } else {
          double t = 0.0;
          for (int64_t r = lane; r < m; r += 32) {
            const double z = x[r] / am;
            t = fma(z, z, t);
          }
          v = am * sqrt(warp_sum(t));
        }
      }
      if (lane == 0) sig[bi * n + j] = v;
    }
    if (tid == 0) {
      sweeps_out[bi] = sweeps;
      conv_out[bi] = conv ? 1 : 0;
    }
    __syncthreads();
  }
}

}  // namespace dmqr
