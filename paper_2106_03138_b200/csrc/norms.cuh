// Column norms, partial-norm downdate with cancellation guard, norm trace.
//   column_norms          matrix.py:61-78
//   PartialNorms.from_matrix rrqr.py:126-129
//   downdate_norms        rrqr.py:161-186
//   _record_norm_check    rrqr.py:211-216
// HBM-bound: one warp per column, coalesced 256 B row segments, shuffle
// reductions; the guard recompute re-reads only the flagged columns.
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int GN_ROWS = 4096;  // rows per chunk of the row-split norm kernels

// Norm of a contiguous column segment of length len, computed by one warp
// (all lanes return the result).  Unscaled sum of squares when the max
// magnitude keeps squares normal, else a second max-scaled pass (the
// reference's scaling, matrix.py:73-77).
// (sum of squares, max |x|) of a contiguous segment, warp-wide (all lanes
// return both): 16-byte loads from the first 16-byte aligned element, 8 pairs
// per lane in flight (a 16384-row column is 16 round trips, not 256)
__device__ __forceinline__ void warp_col_sums(const double* __restrict__ x, int64_t len, int lane, double& sum,
                                              double& amax) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, a0 = 0.0, a1 = 0.0;
  const int64_t h = (len > 0 && (reinterpret_cast<uintptr_t>(x) & 15)) ? 1 : 0;
  if (h && lane == 0) {
    const double p = __ldg(x);
    s0 = p * p;
    a0 = fabs(p);
  }
  const double* y = x + h;
  const int64_t len2 = len - h;
  int64_t i = 2 * lane;
  for (; i + 7 * 64 + 1 < len2; i += 8 * 64) {
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(reinterpret_cast<const double2*>(y + i + 64 * k));
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
      s0 = fma(v[k].x, v[k].x, s0);
      s1 = fma(v[k].y, v[k].y, s1);
      s2 = fma(v[k + 1].x, v[k + 1].x, s2);
      s3 = fma(v[k + 1].y, v[k + 1].y, s3);
      a0 = fmax(a0, fmax(fabs(v[k].x), fabs(v[k].y)));
      a1 = fmax(a1, fmax(fabs(v[k + 1].x), fabs(v[k + 1].y)));
    }
  }
  for (; i + 1 < len2; i += 64) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(y + i));
    s0 = fma(v.x, v.x, s0);
    s1 = fma(v.y, v.y, s1);
    a0 = fmax(a0, fmax(fabs(v.x), fabs(v.y)));
  }
  if (i < len2) {
    const double p = __ldg(y + i);
    s2 = fma(p, p, s2);
    a1 = fmax(a1, fabs(p));
  }
  sum = warp_sum((s0 + s1) + (s2 + s3));
  amax = warp_max(fmax(a0, a1));
}

__device__ __forceinline__ double warp_col_norm(const double* __restrict__ x, int64_t len, int lane) {
  double s, amax;
  warp_col_sums(x, len, lane, s, amax);
  if (norm_range_ok(amax)) return sqrt(s);
  double t = 0.0;
  for (int64_t k = lane; k < len; k += 32) {
    double z = __ldg(x + k) / amax;
    t = fma(z, z, t);
  }
  t = warp_sum(t);
  return amax * sqrt(t);
}

// u[j] = u_ref[j] = ||A[:, j]||  (PartialNorms.from_matrix).  A NaN/Inf entry
// makes the column's sum of squares NaN or its max magnitude Inf, which is
// flagged here (dense() rejects such input, matrix.py:32-33) -- so the input
// validation costs no extra pass over the matrix.  (A finite column whose
// squares overflow has sum Inf but a finite max: not flagged.)
// Work items are (column, GN_ROWS-row chunk) pairs, a warp each, 16-byte loads
// with eight pairs in flight per lane (warp_col_sums): a tall input (cfg4,
// 65536 x 1024) has 16 chunks per column, so the grid is not limited to one
// warp per column.  With one chunk per column the warp finishes the norm;
// otherwise it stores (sum of squares, max) and k_colnorms_fin combines the
// chunks in fixed order.
__device__ __forceinline__ bool sums_bad(double s, double amax) { return isnan(s) || isinf(amax); }
__device__ __forceinline__ void colnorm_finish(const double* x, int64_t m, double s, double amax, int lane,
                                               double* u, double* uref, int32_t* nonfinite, int64_t j) {
  double r;
  if (norm_range_ok(amax)) {
    r = sqrt(s);
  } else {  // the reference's max-scaled second pass (matrix.py:73-77)
    double t = 0.0;
    for (int64_t k = lane; k < m; k += 32) {
      const double y = __ldg(x + k) / amax;
      t = fma(y, y, t);
    }
    r = amax * sqrt(warp_sum(t));
  }
  if (lane == 0) {
    if (sums_bad(s, amax)) atomicOr(nonfinite, 1);
    u[j] = r;
    uref[j] = r;
  }
}
__global__ void k_colnorms_init(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                double* __restrict__ u, double* __restrict__ uref, int32_t* __restrict__ nonfinite,
                                int64_t zs, double* __restrict__ gp, int nch) {
  zshift_by(zs, A, u, uref, nonfinite, gp);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t it = w0; it < n * nch; it += nw) {
    const int64_t j = it / nch;
    const int ch = (int)(it % nch);
    const double* x = A + j * lda;
    const int64_t r0 = (int64_t)ch * GN_ROWS, r1 = (nch == 1) ? m : min(m, r0 + GN_ROWS);
    double s, amax;
    warp_col_sums(x + r0, r1 - r0, lane, s, amax);
    if (nch == 1) {
      colnorm_finish(x, m, s, amax, lane, u, uref, nonfinite, j);
    } else if (lane == 0) {
      gp[2 * it] = s;
      gp[2 * it + 1] = amax;
    }
  }
}
// the chunks of a tall column, summed in chunk order (a warp per column)
__global__ void k_colnorms_fin(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                               double* __restrict__ u, double* __restrict__ uref, int32_t* __restrict__ nonfinite,
                               const double* __restrict__ gp, int nch) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = w0; j < n; j += nw) {
    double s = 0.0, amax = 0.0;
    for (int ch = lane; ch < nch; ch += 32) {
      s += gp[2 * (j * nch + ch)];
      amax = fmax(amax, gp[2 * (j * nch + ch) + 1]);
      if (isinf(gp[2 * (j * nch + ch) + 1])) amax = gp[2 * (j * nch + ch) + 1];
    }
    s = warp_sum(s);
    amax = warp_max(amax);
    colnorm_finish(A + j * lda, m, s, amax, lane, u, uref, nonfinite, j);
  }
}

// Downdate after a step that produced R rows [n_s, n_s1): rrqr.py:161-186.
// Columns whose downdated square falls to <= 1e-2 * u_ref^2 are recomputed
// exactly from rows n_s1.. and their u_ref refreshed.
__global__ void k_downdate(Ctl* c, const double* __restrict__ A, double* __restrict__ u,
                           double* __restrict__ uref, int32_t* __restrict__ glist = nullptr) {
  zshift(c, c, A, u, uref, glist);
  if (c->done) return;
  TLSpan tl_span(c->done ? nullptr : c->tl, c->step_idx, 12);
  const int64_t n_s = c->n_s, n_s1 = n_s + c->l_acc, n = c->n, m = c->m, lda = c->lda;
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0)
    for (int64_t j = n_s + threadIdx.x; j < n_s1; j += blockDim.x) {
      u[j] = 0.0;
      uref[j] = 0.0;
    }
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t j = n_s1 + w0; j < n; j += nw) {
    const double* col = A + j * lda;
    double d = 0.0;
    for (int64_t r = n_s + lane; r < n_s1; r += 32) {
      double x = col[r];
      d = fma(x, x, d);
    }
    d = warp_sum(d);
    const double uj = u[j], rj = uref[j];
    const double sq = __dsub_rn(__dmul_rn(uj, uj), d);
    double nu = sqrt(fmax(sq, 0.0));
    if (sq <= __dmul_rn(1e-2, __dmul_rn(rj, rj))) {
      if (glist) {  // exact norm later, by k_gnorm_part / k_gnorm_fin (row-split over the grid)
        if (lane == 0) glist[atomicAdd(&c->gcount, 1)] = (int32_t)j;
        continue;
      }
      nu = warp_col_norm(col + n_s1, m - n_s1, lane);
      if (lane == 0) uref[j] = nu;
    }
    if (lane == 0) u[j] = nu;
  }
}

// Exact norms of the guard columns listed by k_downdate (rows n_s1 .. m of the
// updated matrix): (column, GN_ROWS-row chunk) items over a persistent grid,
// partial sum of squares and max |x| per item; k_gnorm_fin sums the chunks of
// a column in fixed order.  A long column is read by many warps at once instead
// of one (a 65536-row column was 128 dependent round trips for a single warp).
__global__ void __launch_bounds__(256) k_gnorm_part(const Ctl* c, const double* __restrict__ A,
                                                    const int32_t* __restrict__ glist, double* __restrict__ gp) {
  if (c->done) return;
  const int g = c->gcount;
  if (g == 0) return;
  const int64_t n_s1 = c->n_s + c->l_acc, m = c->m, lda = c->lda;
  const int64_t len = m - n_s1;
  const int nch = (int)max((int64_t)1, ceil_div(len, GN_ROWS));
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t it = w0; it < (int64_t)g * nch; it += nw) {
    const int gi = (int)(it / nch), ch = (int)(it % nch);
    const int64_t j = glist[gi];
    const int64_t r0 = n_s1 + (int64_t)ch * GN_ROWS, r1 = min(m, r0 + GN_ROWS);
    double sv, av;
    warp_col_sums(A + j * lda + r0, r1 - r0, lane, sv, av);
    if (lane == 0) {
      gp[2 * it] = sv;
      gp[2 * it + 1] = av;
    }
  }
}

__global__ void __launch_bounds__(256) k_gnorm_fin(Ctl* c, const double* __restrict__ A,
                                                   const int32_t* __restrict__ glist, const double* __restrict__ gp,
                                                   double* __restrict__ u, double* __restrict__ uref) {
  if (c->done) return;
  const int g = c->gcount;
  const int64_t n_s1 = c->n_s + c->l_acc, m = c->m, lda = c->lda;
  const int64_t len = m - n_s1;
  const int nch = (int)max((int64_t)1, ceil_div(len, GN_ROWS));
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t gi = w0; gi < g; gi += nw) {
    double sv = 0.0, av = 0.0;
    for (int ch = lane; ch < nch; ch += 32) {
      sv += gp[2 * (gi * nch + ch)];
      av = fmax(av, gp[2 * (gi * nch + ch) + 1]);
    }
    sv = warp_sum(sv);
    av = warp_max(av);
    const int64_t j = glist[gi];
    const double nu = norm_range_ok(av) ? sqrt(sv) : warp_col_norm(A + j * lda + n_s1, len, lane);
    if (lane == 0) {
      u[j] = nu;
      uref[j] = nu;
    }
  }
}

// Max relative deviation of downdated vs fresh trailing norms (rrqr.py:211-216),
// accumulated as the bit pattern of a non-negative double (monotone under atomicMax).
__global__ void k_norm_trace(Ctl* c, const double* __restrict__ A, const double* __restrict__ u,
                             unsigned long long* __restrict__ out_bits) {
  if (c->done || !c->trace_norms) return;
  const int64_t n_s1 = c->n_s + c->l_acc, n = c->n, m = c->m, lda = c->lda;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const double floor_ = kEps * c->a_max0;
  double worst = 0.0;
  for (int64_t j = n_s1 + w0; j < n; j += nw) {
    double direct = warp_col_norm(A + j * lda + n_s1, m - n_s1, lane);
    double den = fmax(fmax(direct, floor_), 2.2250738585072014e-308);
    worst = fmax(worst, fabs(u[j] - direct) / den);
  }
  if (lane == 0 && worst > 0.0) atomicMax(out_bits, (unsigned long long)__double_as_longlong(worst));
}

}  // namespace dmqr
