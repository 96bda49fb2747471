// Trailing block-reflector update (larfb 'L','T', forward, columnwise):
//   apply_block_left  householder.py:117-128 + gemm matrix.py:37-58
//   C <- (I - Y T^T Y^T) C  on work[n_s:, tc0:]  (rrqr.py:382-388)
// evaluated as   Z  = Y^T C              (k_trail_a: split-K over rows, fp64 DMMA,
//                                         cp.async double-buffered 32-row slabs)
//                Wt = T^T (sum of splits) (fused: the last split CTA of a column
//                                         tile sums the partials in fixed order and
//                                         multiplies by T^T with DMMA)
//                C -= Y Wt               (k_trail_b: fp64 DMMA, C tile in registers,
//                                         Y / Wt staged with cp.async, 2 CTAs/SM)
// Y is the unit-lower-trapezoidal reflector block read straight out of the
// packed panel (diagonal 1, zeros above).  tc0 is n_s + k_s after the
// Householder panel; after a CholeskyQR2-panel break it is n_s + l, so the
// rejected selected columns get the accepted reflectors here (rrqr.py:366-367).
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int TA_T = 256;       // 8 warps
constexpr int TA_COLS = 64;     // output columns per CTA
constexpr int TA_ROWS = 32;     // K slab
constexpr int TA_LD = 36;       // slab stride (4 mod 16: conflict-free fragments)
constexpr int TW_LD = DMQR_KP;  // 72 = 8 mod 16
// 2 slab stages, reused by the fused T^T Z tail (T and Z tiles)
constexpr size_t TA_SMEM = sizeof(double) * 2 * DMQR_KP * TW_LD;
static_assert(2 * DMQR_KP * TW_LD >= 2 * (DMQR_KP + TA_COLS) * TA_LD, "smem reuse");

// grid: (ceil(n''/64), nsplit).  Zp[s][i][c] (ld n) = sum over this split's rows of Y[r][i] C[r][c];
// the last split CTA of each column tile reduces them and writes Wt = T^T Z (ld n).
__global__ void __launch_bounds__(TA_T, 2) k_trail_a(Ctl* __restrict__ c, const double* __restrict__ A,
                                                     double* __restrict__ Zp, const double* __restrict__ T,
                                                     double* __restrict__ Wt, unsigned* __restrict__ counters) {
  if (c->done) return;
  const int64_t n_s = c->n_s, m = c->m, n = c->n, lda = c->lda;
  const int l = c->l_acc;
  const int64_t c0 = c->tc0;
  const int64_t ncols = n - c0;
  const int64_t col0 = (int64_t)blockIdx.x * TA_COLS;
  if (col0 >= ncols || l == 0) return;
  const int64_t mp = m - n_s;
  const int nsplit = gridDim.y;
  const int64_t rps = ceil_div(ceil_div(mp, nsplit), TA_ROWS) * TA_ROWS;
  const int64_t rb = (int64_t)blockIdx.y * rps, re = min(mp, rb + rps);
  const int lt = (l + 7) / 8;  // M tiles in use
  const int lp = lt * 8;

  extern __shared__ __align__(16) double tas[];
  double* ysb[2] = {tas, tas + DMQR_KP * TA_LD};
  double* csb[2] = {tas + 2 * DMQR_KP * TA_LD, tas + 2 * DMQR_KP * TA_LD + TA_COLS * TA_LD};
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nslab = (re > rb) ? (int)ceil_div(re - rb, TA_ROWS) : 0;
  const double* Yp = A + n_s * lda + n_s;   // Y[r][i] at Yp[r + i*lda] for r > i
  const double* Cp = A + n_s + c0 * lda;    // C[r][cc] at Cp[r + cc*lda]

  // rows i in [l, lp) of both Y stages are zero for the whole kernel
  for (int e = tid; e < (lp - l) * TA_LD; e += TA_T) {
    ysb[0][l * TA_LD + e] = 0.0;
    ysb[1][l * TA_LD + e] = 0.0;
  }
  auto issue = [&](int sl) {
    double* ys = ysb[sl & 1];
    double* cs = csb[sl & 1];
    const int64_t r0 = rb + (int64_t)sl * TA_ROWS;
    for (int e = tid; e < l * TA_ROWS; e += TA_T) {
      const int i = e >> 5, rr = e & 31;
      const int64_t r = r0 + rr;
      double* dst = ys + i * TA_LD + rr;
      if (r < re && r > i)
        cp_async8(dst, Yp + r + (int64_t)i * lda);
      else
        *dst = (r < re && r == i) ? 1.0 : 0.0;
    }
    for (int e = tid; e < TA_COLS * TA_ROWS; e += TA_T) {
      const int cc = e >> 5, rr = e & 31;
      const int64_t r = r0 + rr;
      double* dst = cs + cc * TA_LD + rr;
      if (r < re && col0 + cc < ncols)
        cp_async8(dst, Cp + r + (col0 + cc) * lda);
      else
        *dst = 0.0;
    }
    cp_async_commit();
  };
  double acc[DMQR_KP / 8][2];
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  if (nslab > 0) issue(0);
  for (int sl = 0; sl < nslab; ++sl) {
    if (sl + 1 < nslab) {
      issue(sl + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* ys = ysb[sl & 1];
    const double* cs = csb[sl & 1];
#pragma unroll
    for (int ks = 0; ks < TA_ROWS / 4; ++ks) {
      const int kr = 4 * ks + (lane & 3);
      const double b = cs[(wid * 8 + (lane >> 2)) * TA_LD + kr];
#pragma unroll
      for (int q = 0; q < DMQR_KP / 8; ++q)
        if (q < lt) dmma884(acc[q][0], acc[q][1], ys[(q * 8 + (lane >> 2)) * TA_LD + kr], b);
    }
    __syncthreads();
  }
  // ---- partial tile -> Zp[split] ----
  double* out = Zp + (int64_t)blockIdx.y * DMQR_KP * n;
  const int64_t cc = col0 + wid * 8 + 2 * (lane & 3);
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    if (q >= lt) break;
    const int i = q * 8 + (lane >> 2);
    if (cc < ncols) out[(int64_t)i * n + cc] = acc[q][0];
    if (cc + 1 < ncols) out[(int64_t)i * n + cc + 1] = acc[q][1];
  }
  // ---- last split CTA of this column tile: Wt = T^T * sum_s Zp[s] ----
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  if (tid == 0) {
    const unsigned prev = atomicAdd(&counters[blockIdx.x], 1u);
    s_last = (prev == (unsigned)nsplit - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) counters[blockIdx.x] = 0u;
  const int lp4 = (l + 3) / 4 * 4;
  double* ts = tas;                        // ts[t][i] = T[t][i]   (KP x TW_LD)
  double* zs = tas + DMQR_KP * TW_LD;      // zs[t][c]             (KP x TW_LD)
  for (int e = tid; e < lp4 * DMQR_KP; e += TA_T) {
    const int t = e / DMQR_KP, i = e % DMQR_KP;
    ts[t * TW_LD + i] = (t < l && i < l && t <= i) ? T[t * DMQR_KP + i] : 0.0;
  }
  for (int e = tid; e < lp4 * TA_COLS; e += TA_T) {
    const int t = e >> 6, c2 = e & 63;
    double s = 0.0;
    if (t < l && col0 + c2 < ncols) {
      const double* zp = Zp + (int64_t)t * n + col0 + c2;
      double v[16];
#pragma unroll
      for (int sp = 0; sp < 16; ++sp) v[sp] = (sp < nsplit) ? __ldcg(zp + (int64_t)sp * DMQR_KP * n) : 0.0;
#pragma unroll
      for (int sp = 0; sp < 16; ++sp) s += v[sp];
    }
    zs[t * TW_LD + c2] = s;
  }
  __syncthreads();
  double w[DMQR_KP / 8][2];
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) w[q][0] = w[q][1] = 0.0;
  for (int ks = 0; ks < lp4; ks += 4) {
    const int t = ks + (lane & 3);
    const double b = zs[t * TW_LD + wid * 8 + (lane >> 2)];
#pragma unroll
    for (int q = 0; q < DMQR_KP / 8; ++q)
      if (q < lt) dmma884(w[q][0], w[q][1], ts[t * TW_LD + q * 8 + (lane >> 2)], b);
  }
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    if (q >= lt) break;
    const int i = q * 8 + (lane >> 2);
    if (cc < ncols) Wt[(int64_t)i * n + cc] = w[q][0];
    if (cc + 1 < ncols) Wt[(int64_t)i * n + cc + 1] = w[q][1];
  }
}

constexpr int TB_T = 256;     // 8 warps: 4 (rows) x 2 (cols), each 32x32
constexpr int TB_ROWS = 128;
constexpr int TB_COLS = 64;
constexpr int TB_KMAX = 68;           // l <= 65 rounded up to 4
constexpr int TB_VLD = TB_ROWS + 8;   // 136 = 8 mod 16
constexpr int TB_ZLD = TB_COLS + 8;   // 72  = 8 mod 16
constexpr size_t TB_SMEM = sizeof(double) * TB_KMAX * (TB_VLD + TB_ZLD);  // 113 KB -> 2 CTAs/SM

// C[r][c] -= sum_t Y[r][t] Wt[t][c] over the trailing block; grid (ceil(m'/128), ceil(n''/64))
__global__ void __launch_bounds__(TB_T, 2) k_trail_b(const Ctl* __restrict__ c, double* __restrict__ A,
                                                     const double* __restrict__ Wt) {
  if (c->done) return;
  const int64_t n_s = c->n_s, m = c->m, n = c->n, lda = c->lda;
  const int l = c->l_acc;
  const int64_t c0 = c->tc0, ncols = n - c0, mp = m - n_s;
  const int64_t row0 = (int64_t)blockIdx.x * TB_ROWS, col0 = (int64_t)blockIdx.y * TB_COLS;
  if (row0 >= mp || col0 >= ncols || l == 0) return;
  const int lp4 = (l + 3) / 4 * 4;
  extern __shared__ __align__(16) double tbs[];
  double* vs = tbs;                      // [68][136]: vs[t*VLD + r] = Y[r][t]
  double* zs = tbs + TB_KMAX * TB_VLD;   // [68][72]:  zs[t*ZLD + c] = Wt[t][c]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid & 3, wn = wid >> 2;
  const double* Yp = A + n_s * lda + n_s;
  double* Cp = A + n_s + c0 * lda;

  // stage Y / Wt with cp.async, and load the C tile into the accumulators meanwhile
  for (int e = tid; e < lp4 * TB_ROWS; e += TB_T) {
    const int t = e >> 7, rr = e & 127;
    const int64_t r = row0 + rr;
    double* dst = vs + t * TB_VLD + rr;
    if (t < l && r < mp && r > t)
      cp_async8(dst, Yp + r + (int64_t)t * lda);
    else
      *dst = (t < l && r < mp && r == t) ? 1.0 : 0.0;
  }
  for (int e = tid; e < lp4 * TB_COLS; e += TB_T) {
    const int t = e >> 6, c2 = e & 63;
    double* dst = zs + t * TB_ZLD + c2;
    if (t < l && col0 + c2 < ncols)
      cp_async8(dst, Wt + (int64_t)t * n + col0 + c2);
    else
      *dst = 0.0;
  }
  cp_async_commit();
  double acc[4][4][2];
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int64_t r = row0 + wm * 32 + mt * 8 + (lane >> 2);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t cc = col0 + wn * 32 + nt * 8 + 2 * (lane & 3);
      const bool rv = r < mp;
      const double* p = Cp + r + cc * lda;
      acc[mt][nt][0] = (rv && cc < ncols) ? p[0] : 0.0;
      acc[mt][nt][1] = (rv && cc + 1 < ncols) ? p[lda] : 0.0;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int ks = 0; ks < lp4; ks += 4) {
    const int t = ks + (lane & 3);
    double af[4], bf[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) af[mt] = -vs[t * TB_VLD + wm * 32 + mt * 8 + (lane >> 2)];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bf[nt] = zs[t * TB_ZLD + wn * 32 + nt * 8 + (lane >> 2)];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) dmma884(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int64_t r = row0 + wm * 32 + mt * 8 + (lane >> 2);
    if (r >= mp) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t cc = col0 + wn * 32 + nt * 8 + 2 * (lane & 3);
      double* p = Cp + r + cc * lda;
      if (cc < ncols) p[0] = acc[mt][nt][0];
      if (cc + 1 < ncols) p[lda] = acc[mt][nt][1];
    }
  }
}

}  // namespace dmqr
