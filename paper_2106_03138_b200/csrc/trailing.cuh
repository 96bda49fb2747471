// Trailing block-reflector update (larfb 'L','T', forward, columnwise):
//   apply_block_left  householder.py:117-128 + gemm matrix.py:37-58
//   C <- (I - Y T^T Y^T) C  on work[n_s:, n_s+k_s:]  (rrqr.py:382-388)
// evaluated as   Z  = Y^T C            (trail_a, split-K over rows, fp64 DMMA)
//                Wt = T^T (sum of Z splits)   (trail_w, fp64 DMMA, l x n'')
//                C -= Y Wt             (trail_b, fp64 DMMA, C tile in registers)
// Y is the unit-lower-trapezoidal reflector block read straight out of the
// packed panel (diagonal 1, zeros above).  The l accepted reflectors update
// every column right of the selected block; after a QRDM2 break the rejected
// selected columns were already updated in-panel (rrqr.py:366-367).
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int TA_T = 256;       // 8 warps
constexpr int TA_COLS = 64;     // output columns per CTA
constexpr int TA_ROWS = 32;     // K slab
constexpr int TA_LD = 36;       // slab stride (4 mod 16: conflict-free fragments)

// Y[r][i] of the current panel (panel-relative row r), zero padded for i >= l.
__device__ __forceinline__ double y_elem(const double* __restrict__ A, int64_t lda, int64_t n_s, int64_t r, int i,
                                         int l, int64_t mp) {
  if (i >= l || r >= mp || r < i) return 0.0;
  if (r == i) return 1.0;
  return A[(n_s + r) + (n_s + i) * lda];
}

// grid: (ceil(n''/64), nsplit).  Zp[s][i][c] (ld n) = sum over this split's rows of Y[r][i] C[r][c]
__global__ void __launch_bounds__(TA_T) k_trail_a(const Ctl* __restrict__ c, const double* __restrict__ A,
                                                  double* __restrict__ Zp) {
  if (c->done) return;
  const int64_t n_s = c->n_s, m = c->m, n = c->n, lda = c->lda;
  const int k_s = c->k_s, l = c->l_acc;
  const int64_t c0 = c->tc0;          // first trailing column (n_s + k_s; n_s + l after a CholQR break)
  const int64_t ncols = n - c0;
  const int64_t col0 = (int64_t)blockIdx.x * TA_COLS;
  if (col0 >= ncols || l == 0) return;
  const int64_t mp = m - n_s;
  const int nsplit = gridDim.y;
  const int64_t rps = ceil_div(ceil_div(mp, nsplit), TA_ROWS) * TA_ROWS;
  const int64_t rb = (int64_t)blockIdx.y * rps, re = min(mp, rb + rps);
  const int lt = (l + 7) / 8;  // M tiles in use

  __shared__ __align__(16) double ys[DMQR_KP * TA_LD];
  __shared__ __align__(16) double cs[TA_COLS * TA_LD];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double acc[DMQR_KP / 8][2];
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) acc[q][0] = acc[q][1] = 0.0;

  for (int64_t r0 = rb; r0 < re; r0 += TA_ROWS) {
    // stage Y slab: ys[i][r] ; 32 rows per column i, coalesced along rows
    for (int i = wid; i < lt * 8; i += TA_T / 32) ys[i * TA_LD + lane] = y_elem(A, lda, n_s, r0 + lane, i, l, re);
    for (int q = wid; q < TA_COLS; q += TA_T / 32) {
      const int64_t cc = col0 + q, r = r0 + lane;
      cs[q * TA_LD + lane] = (cc < ncols && r < re) ? A[(n_s + r) + (c0 + cc) * lda] : 0.0;
    }
    __syncthreads();
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
  double* out = Zp + (int64_t)blockIdx.y * DMQR_KP * n;
  const int64_t cc = col0 + wid * 8 + 2 * (lane & 3);
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    if (q >= lt) break;
    const int i = q * 8 + (lane >> 2);
    if (cc < ncols) out[(int64_t)i * n + cc] = acc[q][0];
    if (cc + 1 < ncols) out[(int64_t)i * n + cc + 1] = acc[q][1];
  }
}

// Wt[i][c] = sum_{t<=i} T[t][i] * (sum_s Zp[s][t][c])  (split sum in fixed order)
// grid: ceil(n''/64) CTAs of 256 threads; DMMA with M = i (72), N = c (64), K = t.
constexpr int TW_LD = DMQR_KP;  // 72 = 8 mod 16
constexpr size_t TW_SMEM = sizeof(double) * 2 * DMQR_KP * TW_LD;
__global__ void __launch_bounds__(256) k_trail_w(const Ctl* __restrict__ c, const double* __restrict__ Zp,
                                                 const double* __restrict__ T, double* __restrict__ Wt, int nsplit) {
  if (c->done) return;
  const int64_t n = c->n, ncols = n - c->tc0;
  const int l = c->l_acc;
  const int64_t col0 = (int64_t)blockIdx.x * 64;
  if (l == 0 || col0 >= ncols) return;
  const int lp4 = (l + 3) / 4 * 4, lt = (l + 7) / 8;
  extern __shared__ __align__(16) double twsm[];
  double* ts = twsm;                       // ts[t][i] = T[t][i]
  double* zs = twsm + DMQR_KP * TW_LD;     // zs[t][c]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < lp4 * DMQR_KP; e += 256) {
    const int t = e / DMQR_KP, i = e % DMQR_KP;
    ts[t * TW_LD + i] = (t < l && i < l && t <= i) ? T[t * DMQR_KP + i] : 0.0;
  }
  for (int e = tid; e < lp4 * 64; e += 256) {
    const int t = e >> 6, cc = e & 63;
    double sacc = 0.0;
    if (t < l && col0 + cc < ncols)
      for (int sp = 0; sp < nsplit; ++sp) sacc += Zp[(int64_t)sp * DMQR_KP * n + (int64_t)t * n + col0 + cc];
    zs[t * TW_LD + cc] = sacc;
  }
  __syncthreads();
  double acc[DMQR_KP / 8][2];
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int ks = 0; ks < lp4; ks += 4) {
    const int t = ks + (lane & 3);
    const double b = zs[t * TW_LD + wid * 8 + (lane >> 2)];
#pragma unroll
    for (int q = 0; q < DMQR_KP / 8; ++q)
      if (q < lt) dmma884(acc[q][0], acc[q][1], ts[t * TW_LD + q * 8 + (lane >> 2)], b);
  }
  const int64_t cc = col0 + wid * 8 + 2 * (lane & 3);
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    if (q >= lt) break;
    const int i = q * 8 + (lane >> 2);
    if (cc < ncols) Wt[(int64_t)i * n + cc] = acc[q][0];
    if (cc + 1 < ncols) Wt[(int64_t)i * n + cc + 1] = acc[q][1];
  }
}

constexpr int TB_T = 256;     // 8 warps: 4 (rows) x 2 (cols), each 32x32
constexpr int TB_ROWS = 128;
constexpr int TB_COLS = 64;
constexpr int TB_VLD = TB_ROWS + 8;   // 136 = 8 mod 16
constexpr int TB_ZLD = TB_COLS + 8;   // 72  = 8 mod 16

// C[r][c] -= sum_t Y[r][t] Wt[t][c] over the trailing block; grid (ceil(m'/128), ceil(n''/64))
__global__ void __launch_bounds__(TB_T) k_trail_b(const Ctl* __restrict__ c, double* __restrict__ A,
                                                  const double* __restrict__ Z) {
  if (c->done) return;
  const int64_t n_s = c->n_s, m = c->m, n = c->n, lda = c->lda;
  const int k_s = c->k_s, l = c->l_acc;
  const int64_t c0 = c->tc0, ncols = n - c0, mp = m - n_s;
  const int64_t row0 = (int64_t)blockIdx.x * TB_ROWS, col0 = (int64_t)blockIdx.y * TB_COLS;
  if (row0 >= mp || col0 >= ncols || l == 0) return;
  const int lp4 = (l + 3) / 4 * 4;
  extern __shared__ __align__(16) double tbs[];
  double* vs = tbs;                       // [KP][136]: vs[t*VLD + r] = Y[r][t]
  double* zs = tbs + DMQR_KP * TB_VLD;    // [KP][72]:  zs[t*ZLD + c] = -Wt[t][c]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int e = tid; e < lp4 * TB_ROWS; e += TB_T) {
    const int t = e / TB_ROWS, rr = e % TB_ROWS;
    const int64_t r = row0 + rr;
    vs[t * TB_VLD + rr] = y_elem(A, lda, n_s, r, t, l, mp);
  }
  for (int e = tid; e < lp4 * TB_COLS; e += TB_T) {
    const int t = e / TB_COLS, cc = e % TB_COLS;
    zs[t * TB_ZLD + cc] = (t < l && col0 + cc < ncols) ? -Z[(int64_t)t * n + col0 + cc] : 0.0;
  }
  const int wm = wid & 3, wn = wid >> 2;
  double acc[4][4][2];
  // accumulators start from C
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int64_t r = row0 + wm * 32 + mt * 8 + (lane >> 2);
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const int64_t cc = col0 + wn * 32 + nt * 8 + 2 * (lane & 3);
      const bool rv = r < mp;
      const double* p = A + (n_s + r) + (c0 + cc) * lda;
      acc[mt][nt][0] = (rv && cc < ncols) ? p[0] : 0.0;
      acc[mt][nt][1] = (rv && cc + 1 < ncols) ? p[lda] : 0.0;
    }
  }
  __syncthreads();
  for (int ks = 0; ks < lp4; ks += 4) {
    const int t = ks + (lane & 3);
    double af[4], bf[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) af[mt] = vs[t * TB_VLD + wm * 32 + mt * 8 + (lane >> 2)];
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
      double* p = A + (n_s + r) + (c0 + cc) * lda;
      if (cc < ncols) p[0] = acc[mt][nt][0];
      if (cc + 1 < ncols) p[lda] = acc[mt][nt][1];
    }
  }
}

}  // namespace dmqr
