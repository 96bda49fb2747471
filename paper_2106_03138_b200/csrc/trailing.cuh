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
//
// Staging uses 16-byte cp.async with addresses hoisted out of the loops; tiles
// start on EVEN global rows (16-byte alignment of column-major data with an
// even lda), rows outside the tile's range are zero-filled by the copy itself
// (src-size 0) or get Y = 0, so they contribute nothing.
#pragma once
#include "common.cuh"
#include "norms.cuh"
#include "ygemm.cuh"

namespace dmqr {


constexpr int TA_T = 256;       // 8 warps
constexpr int TA_COLS = 64;     // output columns per CTA
#ifndef DMQR_TA_ROWS
#define DMQR_TA_ROWS 16
#endif
#ifndef DMQR_TA_NST
#define DMQR_TA_NST 4
#endif
constexpr int TA_ROWS = DMQR_TA_ROWS;  // K slab
constexpr int TA_LD = TA_ROWS + 4;     // slab stride (4 mod 16: conflict-free fragments; 16B aligned rows)
constexpr int TA_NST = DMQR_TA_NST;    // cp.async stages (TA_NST - 1 slabs in flight while one is consumed)
constexpr int TA_RP = TA_ROWS / 2;    // row pairs per slab (16-byte copies)
constexpr int TA_CL = TA_T / TA_RP;   // column lanes of the copy grid
constexpr int TW_LD = DMQR_KP;  // 72 = 8 mod 16
// TA_NST slab stages, reused by the fused T^T Z tail (T and Z tiles)
constexpr size_t TA_SMEM_ST = sizeof(double) * TA_NST * (DMQR_KP + TA_COLS) * TA_LD;
constexpr size_t TA_SMEM_TZ = sizeof(double) * 2 * DMQR_KP * TW_LD;
constexpr size_t TA_SMEM = TA_SMEM_ST > TA_SMEM_TZ ? TA_SMEM_ST : TA_SMEM_TZ;

// One landed slab of Z += Y^T C, instantiated per lt (no predicated dead DMMA):
// warp w owns output columns 8w..8w+7 and all lt row tiles (per k-step one C
// fragment and lt Y fragments).  (A 2 x 4 warp grid with 16 columns per warp,
// 0.7 instead of 1.1 shared loads per DMMA, measured 1% slower on cfg4 and at
// 8192^2: shared-memory bandwidth does not bound this loop.)
constexpr int TA_ACC = DMQR_KP / 8;
template <int LT>
__device__ __forceinline__ void ta_slab_mma_t(double (&acc)[TA_ACC][2], const double* ys, const double* cs,
                                              int lane, int wid) {
#pragma unroll
  for (int ks = 0; ks < TA_ROWS / 4; ++ks) {
    const int kr = 4 * ks + (lane & 3);
    const double b = cs[(wid * 8 + (lane >> 2)) * TA_LD + kr];
#pragma unroll
    for (int q = 0; q < LT; ++q) dmma884(acc[q][0], acc[q][1], ys[(q * 8 + (lane >> 2)) * TA_LD + kr], b);
  }
}
// the warp's partial tiles -> out (a Zp split, ld ldz) at columns col0 + 8w ..
template <int LT>
__device__ __forceinline__ void ta_store_t(const double (&acc)[TA_ACC][2], double* out, int64_t ldz, int64_t col0,
                                           int lane, int wid) {
  const int64_t cc = col0 + wid * 8 + 2 * (lane & 3);
#pragma unroll
  for (int q = 0; q < LT; ++q) {
    const int i = q * 8 + (lane >> 2);
    out[(int64_t)i * ldz + cc] = acc[q][0];
    out[(int64_t)i * ldz + cc + 1] = acc[q][1];
  }
}
#define TA_DISPATCH(fn, ...)                     \
  switch (lt) {                                  \
    case 1: fn<1>(__VA_ARGS__); break;           \
    case 2: fn<2>(__VA_ARGS__); break;           \
    case 3: fn<3>(__VA_ARGS__); break;           \
    case 4: fn<4>(__VA_ARGS__); break;           \
    case 5: fn<5>(__VA_ARGS__); break;           \
    case 6: fn<6>(__VA_ARGS__); break;           \
    case 7: fn<7>(__VA_ARGS__); break;           \
    case 8: fn<8>(__VA_ARGS__); break;           \
    default: fn<DMQR_KP / 8>(__VA_ARGS__); break; \
  }

// Look-ahead bookkeeping of a step's own panel columns, by one CTA: u of the
// accepted columns is cleared; the columns [n_s + l, tc0) that the Householder
// panel already updated in full (after a QRDM2 break) are downdated with
// k_downdate's arithmetic and, while an update is pending, flagged; their Wt
// slots (Wt is indexed from n_s + l) are zeroed for the next step's moves.
__device__ void la_panel_columns(Ctl* c, const double* __restrict__ A, double* __restrict__ Wt,
                                 int64_t ldz, double* __restrict__ u, double* __restrict__ uref,
                                 uint8_t* __restrict__ upd, int64_t n_s, int l, int64_t tc0) {
  const int64_t m = c->m, n = c->n, lda = c->lda, base = n_s + l;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  tc0 = min(tc0, n);
  const bool will_pend = base < m && tc0 < n;
  for (int64_t j = n_s + threadIdx.x; j < base; j += blockDim.x) {
    u[j] = 0.0;
    uref[j] = 0.0;
  }
  for (int64_t j = base + wid; j < tc0; j += nw) {
    const double* col = A + j * lda;
    double d = 0.0;
    for (int64_t r = n_s + lane; r < base; r += 32) {
      const double x = col[r];
      d = fma(x, x, d);
    }
    d = warp_sum(d);
    const double uj = u[j], rj = uref[j];
    const double sq = __dsub_rn(__dmul_rn(uj, uj), d);
    double nu = sqrt(fmax(sq, 0.0));
    if (sq <= __dmul_rn(1e-2, __dmul_rn(rj, rj))) {
      nu = warp_col_norm(col + base, m - base, lane);
      if (lane == 0) uref[j] = nu;
    }
    if (lane == 0) {
      u[j] = nu;
      if (will_pend) upd[j] = 1;
    }
  }
  for (int64_t e = threadIdx.x; e < (int64_t)l * (tc0 - base); e += blockDim.x)
    Wt[(e / (tc0 - base)) * ldz + e % (tc0 - base)] = 0.0;
}

// Look-ahead tail of a Wt column tile (k_trail_a): zs holds the
// tile's Wt (rows < lp4, 64 columns, zeros past the last column); ts is
// scratch.  R12 = C_top - Y1 Wt is written with k_trail_b's DMMA sequence per
// element (so it is bitwise the serial update's), the norms are downdated with
// k_downdate's arithmetic, guard columns get their full update and an exact
// norm, and tile 0 does the panel-column bookkeeping.
__device__ void la_tile_epilogue(Ctl* c, double* __restrict__ A, double* __restrict__ Wt, int64_t ldz,
                                 double* __restrict__ u, double* __restrict__ uref, uint8_t* __restrict__ upd,
                                 const double* zs, double* ts, int64_t n_s, int l, int64_t c0, int64_t col0,
                                 int32_t* __restrict__ glist) {
  const int64_t m = c->m, n = c->n, lda = c->lda, ncols = n - c0, n_s1 = n_s + l;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int lt = (l + 7) / 8, lp4 = (l + 3) / 4 * 4;
  const int64_t cc = col0 + wid * 8 + 2 * (lane & 3);
  for (int e = tid; e < lp4 * lp4; e += TA_T) {  // Y1 (unit lower) -> ts[i][t], column-major reads
    const int t = e / lp4, i = e % lp4;
    double y = 0.0;
    if (i < l && t < l) y = (t < i) ? A[(n_s + t) * lda + n_s + i] : ((t == i) ? 1.0 : 0.0);
    ts[i * TW_LD + t] = y;
  }
  __syncthreads();
  // same DMMA sequence per element as k_trail_b (acc = C, += (-Y) Wt in
  // ascending k groups), so the result is bitwise the serial update's
  double pv[DMQR_KP / 8][2];
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    const int i = q * 8 + (lane >> 2);
    const double* p = A + (n_s + i) + (c0 + cc) * lda;
    pv[q][0] = (q < lt && i < l && cc < ncols) ? p[0] : 0.0;
    pv[q][1] = (q < lt && i < l && cc + 1 < ncols) ? p[lda] : 0.0;
  }
  for (int ks = 0; ks < lp4; ks += 4) {
    const int t = ks + (lane & 3);
    const double b = zs[t * TW_LD + wid * 8 + (lane >> 2)];
#pragma unroll
    for (int q = 0; q < DMQR_KP / 8; ++q)
      if (q < lt) dmma884(pv[q][0], pv[q][1], -ts[(q * 8 + (lane >> 2)) * TW_LD + t], b);
  }
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    const int i = q * 8 + (lane >> 2);
    if (q >= lt) break;
    if (i < l) {
      double* p = A + (n_s + i) + (c0 + cc) * lda;
      if (cc < ncols) p[0] = pv[q][0];
      if (cc + 1 < ncols) p[lda] = pv[q][1];
    }
  }
  __syncthreads();
  // the warp's 8 columns at once (k_downdate's per-column arithmetic and order)
  double d[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t j = min(c0 + col0 + wid * 8 + q, n - 1);
    const double* col = A + j * lda;
    d[q] = 0.0;
    for (int64_t r = n_s + lane; r < n_s1; r += 32) {
      const double x = col[r];
      d[q] = fma(x, x, d[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) d[q] = warp_sum(d[q]);
  if (lane < 8) {
    double dq = d[0];
#pragma unroll
    for (int q = 1; q < 8; ++q)
      if (lane == q) dq = d[q];
    const int64_t j = c0 + col0 + wid * 8 + lane;
    if (j < n) {
      const double uj = u[j], rj = uref[j];
      const double sq = __dsub_rn(__dmul_rn(uj, uj), dq);
      if (sq <= __dmul_rn(1e-2, __dmul_rn(rj, rj)) && n_s1 < m)
        glist[atomicAdd(&c->gcount, 1)] = (int32_t)j;  // guard: k_guard recomputes it
      else
        u[j] = sqrt(fmax(sq, 0.0));
    }
  }
  if (col0 == 0) la_panel_columns(c, A, Wt, ldz, u, uref, upd, n_s, l, c0);  // (the step's tile 0)
}

// grid: (ceil(n''/64), nsplit).  Zp[s][i][c] (ld ldz) = sum over this split's rows of Y[r][i] C[r][c];
// the last split CTA of each column tile reduces them and writes Wt = T^T Z (ld ldz).
// (one CTA's work: column tile bx, row split by of nsplit; k_tail runs the
// same items from a persistent grid)
__device__ __forceinline__ void trail_a_cta(const CtlSnap& S, Ctl* c, double* __restrict__ A,
                                            double* __restrict__ Zp, const double* __restrict__ T,
                                            double* __restrict__ Wt, unsigned* __restrict__ counters,
                                            int64_t ldz, double* __restrict__ u, double* __restrict__ uref,
                                            uint8_t* __restrict__ upd, int32_t* __restrict__ glist, const int bx,
                                            const int by, const int nsplit) {
  const int64_t n_s = S.n_s, m = S.m, n = S.n, lda = S.lda;
  const int l = S.l_acc;
  const int64_t c0 = S.tc0;
  const int64_t ncols = n - c0;
  const int64_t col0 = (int64_t)bx * TA_COLS;
  if (col0 >= ncols || l == 0) return;
  const int64_t mp = m - n_s;
  const int64_t rps = ceil_div(ceil_div(mp, nsplit), TA_ROWS) * TA_ROWS;
  const int64_t rb = (int64_t)by * rps, re = min(mp, rb + rps);
  const int lt = (l + 7) / 8;  // M tiles in use
  const int lp = lt * 8;
  const int odd = (int)(n_s & 1);  // slabs start one row early so global rows are even

  extern __shared__ __align__(16) double tas[];
  // stage q: Y slab at tas + q KP LD, C slab after all the Y slabs
  auto ysb = [&](int q) { return tas + q * DMQR_KP * TA_LD; };
  auto csb = [&](int q) { return tas + TA_NST * DMQR_KP * TA_LD + q * TA_COLS * TA_LD; };
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t span = (re > rb) ? re - rb + odd : 0;
  const int nslab = (int)ceil_div(span, TA_ROWS);
  // thread -> (row pair rp, first column cb) of the 16 x {72 | 64} chunk grid of a slab
  const int rp = tid % TA_RP, cb = tid / TA_RP;  // row pairs x column lanes
  const double* Yp = A + n_s * lda + n_s;   // Y[r][i] at Yp[r + i*lda]
  const double* Cp = A + n_s + c0 * lda;    // C[r][cc] at Cp[r + cc*lda]

  for (int e = tid; e < (lp - l) * TA_LD; e += TA_T)  // rows i in [l, lp) stay zero
    for (int q = 0; q < TA_NST; ++q) ysb(q)[l * TA_LD + e] = 0.0;
  auto issue = [&](int sl) {
    double* ys = ysb(sl % TA_NST);
    double* cs = csb(sl % TA_NST);
    const int64_t r = rb - odd + (int64_t)sl * TA_ROWS + 2 * rp;  // panel-relative, even global row
    const int64_t gr = n_s + r;
    const int bytes = (gr + 1 < m) ? 16 : ((gr < m) ? 8 : 0);
    for (int i = cb; i < l; i += TA_CL) cp_async16(ys + i * TA_LD + 2 * rp, Yp + r + (int64_t)i * lda, bytes);
    for (int cc = cb; cc < TA_COLS; cc += TA_CL)
      cp_async16(cs + cc * TA_LD + 2 * rp, Cp + r + (col0 + cc) * lda, (col0 + cc < ncols) ? bytes : 0);
    cp_async_commit();
  };
  // Y structure on a landed slab: 0 outside [rb, re) and above the diagonal, 1 on it
  auto fix = [&](int sl) {
    const int64_t r0 = rb - odd + (int64_t)sl * TA_ROWS;
    if (r0 >= 72 && r0 >= rb && r0 + TA_ROWS <= re) return;
    double* ys = ysb(sl % TA_NST);
    for (int e = tid; e < l * TA_ROWS; e += TA_T) {
      const int i = e / TA_ROWS, rr = e % TA_ROWS;
      const int64_t r = r0 + rr;
      if (r < rb || r >= re || r <= i) ys[i * TA_LD + rr] = (r == i && r >= rb && r < re) ? 1.0 : 0.0;
    }
  };
  double acc[TA_ACC][2];
#pragma unroll
  for (int q = 0; q < TA_ACC; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int q = 0; q < TA_NST - 1; ++q) {  // prologue: TA_NST - 1 slabs in flight (empty groups past the end)
    if (q < nslab)
      issue(q);
    else
      cp_async_commit();
  }
  for (int sl = 0; sl < nslab; ++sl) {
    cp_async_wait<TA_NST - 2>();  // slab sl has landed (one group committed per slab)
    __syncthreads();
    {  // Y structure / rows outside [rb, re): only the first and boundary slabs (uniform branch)
      const int64_t r0 = rb - odd + (int64_t)sl * TA_ROWS;
      if (!(r0 >= 72 && r0 >= rb && r0 + TA_ROWS <= re)) {
        fix(sl);
        __syncthreads();
      }
    }
    const double* ys = ysb(sl % TA_NST);
    const double* cs = csb(sl % TA_NST);
    TA_DISPATCH(ta_slab_mma_t, acc, ys, cs, lane, wid)
    __syncthreads();  // (stage sl % TA_NST is refilled by the issue below, TA_NST - 1 slabs ahead)
    if (sl + TA_NST - 1 < nslab)
      issue(sl + TA_NST - 1);
    else
      cp_async_commit();
  }
  // ---- partial tile -> Zp[split] ----
  double* out = Zp + (int64_t)by * DMQR_KP * ldz;
  TA_DISPATCH(ta_store_t, acc, out, ldz, col0, lane, wid)
  const int64_t cc = col0 + wid * 8 + 2 * (lane & 3);
  // ---- last split CTA of this column tile: Wt = T^T * sum_s Zp[s] ----
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  if (tid == 0) {
    const unsigned prev = atomicAdd(&counters[bx], 1u);
    s_last = (prev == (unsigned)nsplit - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) counters[bx] = 0u;
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
    if (t < l) {
      const double* zp = Zp + (int64_t)t * ldz + col0 + c2;
      for (int sp0 = 0; sp0 < nsplit; sp0 += 16) {  // (16 loads in flight; fixed order)
        double v[16];
#pragma unroll
        for (int sp = 0; sp < 16; ++sp)
          v[sp] = (sp0 + sp < nsplit) ? __ldcg(zp + (int64_t)(sp0 + sp) * DMQR_KP * ldz) : 0.0;
#pragma unroll
        for (int sp = 0; sp < 16; ++sp) s += v[sp];
      }
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
  // Wt rows [0, lp4) x columns [col0, col0 + 64) (zeros beyond l and beyond ncols keep trail_b exact).
  // Look-ahead indexes Wt from n_s + l (not tc0) so column moves of the next
  // step always find a slot.
  const int64_t n_s1 = n_s + l;
  const int64_t wofs = S.la ? c0 - n_s1 : 0;
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    const int i = q * 8 + (lane >> 2);
    if (i >= lp4) break;
    Wt[(int64_t)i * ldz + wofs + cc] = (cc < ncols) ? w[q][0] : 0.0;
    Wt[(int64_t)i * ldz + wofs + cc + 1] = (cc + 1 < ncols) ? w[q][1] : 0.0;
  }
  if (!S.la) return;
  // ---- look-ahead: R12, norm downdate, guard columns (la_tile_epilogue) ----
  __syncthreads();
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    const int i = q * 8 + (lane >> 2);
    if (i >= lp4) break;
    zs[i * TW_LD + wid * 8 + 2 * (lane & 3)] = (cc < ncols) ? w[q][0] : 0.0;
    zs[i * TW_LD + wid * 8 + 2 * (lane & 3) + 1] = (cc + 1 < ncols) ? w[q][1] : 0.0;
  }
  la_tile_epilogue(c, A, Wt, ldz, u, uref, upd, zs, ts, n_s, l, c0, col0, glist);
}


__global__ void __launch_bounds__(TA_T, 2) k_trail_a(Ctl* c, double* __restrict__ A,
                                                     double* __restrict__ Zp, const double* __restrict__ T,
                                                     double* __restrict__ Wt, unsigned* __restrict__ counters,
                                                     int64_t ldz, double* __restrict__ u,
                                                     double* __restrict__ uref, uint8_t* __restrict__ upd,
                                                     int only_if_cq_fail, int32_t* __restrict__ glist) {
  zshift(c, c, A, Zp, T, Wt, counters, u, uref, upd, glist);
  pdl_enter();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 8);
  if (S.done || (only_if_cq_fail && !S.cq_fail)) return;  // (k_trail_w did it)
  trail_a_cta(S, c, A, Zp, T, Wt, counters, ldz, u, uref, upd, glist, (int)blockIdx.x, (int)blockIdx.y, (int)gridDim.y);
}

constexpr int TB_T = 256;     // 8 warps: 4 (rows) x 2 (cols), each 32x32
constexpr int TB_ROWS = 128;
constexpr int TB_COLS = 64;
constexpr int TB_KMAX = 68;           // l <= 65 rounded up to 4
constexpr int TB_VLD = TB_ROWS + 4;   // 132 = 4 mod 16: the 4 (k) x 4 (row) half-warp fragment reads hit 16 distinct bank pairs
constexpr int TB_ZLD = TB_COLS + 4;   // 68  = 4 mod 16 (same)
constexpr size_t TB_SMEM = sizeof(double) * TB_KMAX * (TB_VLD + TB_ZLD);  // 113 KB -> 2 CTAs/SM

// C[r][c] -= sum_t Y[r][t] Wt[t][c] over the trailing block.  grid (ceil((m'+1)/128), ceil(n''/64));
// row tiles start on even global rows (the possible extra row n_s-1 gets Y = 0).
template <bool LA>
__device__ __forceinline__ void trail_b_tile(double* __restrict__ A, const double* __restrict__ Wt, int64_t ldz,
                                             const uint8_t* __restrict__ upd, int64_t n_s, int64_t m, int64_t lda,
                                             int l, int64_t c0, int64_t ncols, int64_t mp, int64_t row0,
                                             int64_t col0) {
  const int lp4 = (l + 3) / 4 * 4;
  extern __shared__ __align__(16) double tbs[];
  double* vs = tbs;                      // [68][136]: vs[t*VLD + r] = Y[r][t]
  double* zs = tbs + TB_KMAX * TB_VLD;   // [68][72]:  zs[t*ZLD + c] = Wt[t][c]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int wm = wid & 3, wn = wid >> 2;
  const double* Yp = A + n_s * lda + n_s;
  double* Cp = A + n_s + c0 * lda;

  // ---- stage Y (68 x 128) and Wt (68 x 64) with 16-byte cp.async ----
  {
    const int rp = tid & 63, tb = tid >> 6;  // 64 row pairs x 4 column lanes
    const int64_t r = row0 + 2 * rp;
    const int64_t gr = n_s + r;
    const int bytes = (gr + 1 < m) ? 16 : ((gr < m) ? 8 : 0);
    for (int t = tb; t < l; t += 4) cp_async16(vs + t * TB_VLD + 2 * rp, Yp + r + (int64_t)t * lda, bytes);
    const int cp2 = tid & 31, tz = tid >> 5;  // 32 column pairs x 8 row lanes
    for (int t = tz; t < l; t += 8) cp_async16(zs + t * TB_ZLD + 2 * cp2, Wt + (int64_t)t * ldz + col0 + 2 * cp2, 16);
    cp_async_commit();
  }
  // ---- the C tile into the accumulators (HBM reads overlap the staging) ----
  // The product is formed transposed, C^T -= Wt^T Y^T (Wt fragments as the DMMA's
  // row operand, Y fragments as its column operand: the same products summed in
  // the same order, so the result is bitwise the untransposed one), because the
  // accumulator pair of a lane then holds two consecutive ROWS of one column:
  // 16 contiguous, 16-byte-aligned bytes (tiles start on even global rows), so
  // the tile moves with LDG.128 / STG.128 -- half the memory instructions.
  // acc[ct][rt]: column ct*8 + (lane >> 2), rows rt*8 + 2*(lane & 3) + {0, 1}
  // of the warp's 32 x 32 block.
  double acc[4][4][2];
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) {
    const int64_t cc = col0 + wn * 32 + ct * 8 + (lane >> 2);
    const bool cv = cc < ncols;
#pragma unroll
    for (int rt = 0; rt < 4; ++rt) {
      const int64_t r = row0 + wm * 32 + rt * 8 + 2 * (lane & 3);
      const double* p = Cp + r + cc * lda;
      if (cv && r >= 0 && r + 1 < mp) {
        const double2 v = *reinterpret_cast<const double2*>(p);
        acc[ct][rt][0] = v.x;
        acc[ct][rt][1] = v.y;
      } else {
        acc[ct][rt][0] = (cv && r >= 0 && r < mp) ? p[0] : 0.0;
        acc[ct][rt][1] = (cv && r + 1 >= 0 && r + 1 < mp) ? p[1] : 0.0;
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // ---- Y structure / padding fixups (first tile, bottom tile, t in [l, lp4)) ----
  if (row0 < 72 || row0 + TB_ROWS > mp) {
    for (int e = tid; e < l * TB_ROWS; e += TB_T) {
      const int t = e >> 7, rr = e & 127;
      const int64_t r = row0 + rr;
      if (r < 0 || r >= mp || r <= t) vs[t * TB_VLD + rr] = (r == t) ? 1.0 : 0.0;
    }
  }
  for (int e = tid; e < (lp4 - l) * TB_ROWS; e += TB_T) vs[l * TB_VLD + e / TB_ROWS * TB_VLD + e % TB_ROWS] = 0.0;
  for (int e = tid; e < (lp4 - l) * TB_COLS; e += TB_T) zs[l * TB_ZLD + e / TB_COLS * TB_ZLD + e % TB_COLS] = 0.0;
  __syncthreads();
  for (int ks = 0; ks < lp4; ks += 4) {
    const int t = ks + (lane & 3);
    double yf[4], wf[4];
#pragma unroll
    for (int rt = 0; rt < 4; ++rt) yf[rt] = -vs[t * TB_VLD + wm * 32 + rt * 8 + (lane >> 2)];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct) wf[ct] = zs[t * TB_ZLD + wn * 32 + ct * 8 + (lane >> 2)];
#pragma unroll
    for (int ct = 0; ct < 4; ++ct)
#pragma unroll
      for (int rt = 0; rt < 4; ++rt) dmma884(acc[ct][rt][0], acc[ct][rt][1], wf[ct], yf[rt]);
  }
  const int64_t rlo = LA ? (int64_t)l : 0;
#pragma unroll
  for (int ct = 0; ct < 4; ++ct) {
    const int64_t cc = col0 + wn * 32 + ct * 8 + (lane >> 2);
    if (cc >= ncols || (LA && upd && upd[c0 + cc])) continue;
#pragma unroll
    for (int rt = 0; rt < 4; ++rt) {
      const int64_t r = row0 + wm * 32 + rt * 8 + 2 * (lane & 3);
      double* p = Cp + r + cc * lda;
      if (r >= rlo && r + 1 < mp) {
        *reinterpret_cast<double2*>(p) = make_double2(acc[ct][rt][0], acc[ct][rt][1]);
      } else {
        if (r >= rlo && r < mp) p[0] = acc[ct][rt][0];
        if (r + 1 >= rlo && r + 1 < mp) p[1] = acc[ct][rt][1];
      }
    }
  }
}

// Look-ahead form (LA): the pending update of the previous step (Ctl::pend_*),
// launched right behind the next panel as its programmatic dependent (the
// panel triggers at entry, so this grid fills the SMs the panel left free and
// runs beside it): the top l rows already hold R12 (k_trail_a) and flagged
// columns (upd) are done -- or are the panel's -- so neither is stored; Wt is
// indexed from n_s + l.  The last CTA clears the flags and the pending bit;
// every CTA ends in griddepcontrol.wait, so this grid completes only after
// the panel (stream order for the kernels behind it).
template <bool LA>
__global__ void __launch_bounds__(TB_T, 2) k_trail_b(Ctl* c, double* __restrict__ A,
                                                     const double* __restrict__ Wt, int64_t ldz,
                                                     uint8_t* __restrict__ upd, unsigned* __restrict__ counter) {
  zshift(c, c, A, Wt, upd, counter);
  pdl_enter();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 11);
  if (LA ? !S.pend : S.done) return;
  const int64_t m = S.m, n = S.n, lda = S.lda;
  const int64_t n_s = LA ? S.pend_ns : S.n_s;
  const int l = LA ? S.pend_l : S.l_acc;
  const int64_t c0 = LA ? n_s + l : S.tc0, ncols = n - c0, mp = m - n_s;
  const int odd = (int)(n_s & 1);
  const int64_t row0 = (int64_t)blockIdx.x * TB_ROWS - odd;  // panel-relative, even global row
  const int64_t col0 = (int64_t)blockIdx.y * TB_COLS;
  if (!(row0 >= mp || col0 >= ncols || l == 0 || (LA && row0 + TB_ROWS <= l)))
    trail_b_tile<LA>(A, Wt, ldz, upd, n_s, m, lda, l, c0, ncols, mp, row0, col0);
  if (LA) {
    __syncthreads();
    __shared__ int s_last;
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned prev = atomicAdd(counter, 1u);
      s_last = (prev == gridDim.x * gridDim.y - 1);
    }
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int64_t j = threadIdx.x; j < n; j += blockDim.x) upd[j] = 0;
      if (threadIdx.x == 0) {
        *counter = 0u;
        c->pend = 0;
      }
      // only the last CTA holds its SM until the panel completes: the grid's
      // completion then implies the panel's for the kernels behind it
      asm volatile("griddepcontrol.wait;" ::: "memory");
    }
  }
}


// ---------------------------------------------------------------------------
// Spare-SM worker (look-ahead, CholeskyQR2 panel path): the programmatic
// dependent of k_panel_cq, so it runs on the SMs the panel's cluster leaves
// free while the panel factors.  Persistent CTAs pull work items:
//   phase 1  the previous step's pending C -= Y Wt (k_trail_b tiles); the CTA
//            finishing the last tile clears the flags and the pending bit;
//   phase 2  once phase 1 is done and the panel has published Q1 = P R1^-1
//            (its first CholeskyQR pass): split-K partials of G = Q1^T C over
//            all panel rows and the columns from n_s.  With Y2 = Q1_bot M
//            (rows past the top l) the update's Y^T C = E C_top + M^T G, so
//            k_trail_w needs only small l x l products after the panel.
// The last CTA to leave waits for the panel (griddepcontrol.wait), so this
// grid's completion implies the panel's for the kernels behind it.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// split-K partial of Q1^T C for one 64-column tile and one row split (the
// k_trail_a main loop with a dense Y = Q1, stored with the row parity of A)
__device__ void g_partial(const double* __restrict__ A, const double* __restrict__ Q1g, double* __restrict__ Gp,
                          int64_t ldz, int64_t n_s, int64_t m, int64_t lda, int l, int64_t ncols, int64_t col0,
                          int split, int nsplit) {
  const int64_t mp = m - n_s;
  const int64_t rps = ceil_div(ceil_div(mp, nsplit), TA_ROWS) * TA_ROWS;
  const int64_t rb = (int64_t)split * rps, re = min(mp, rb + rps);
  const int lt = (l + 7) / 8, lp = lt * 8;
  const int odd = (int)(n_s & 1);
  extern __shared__ __align__(16) double gps[];
  // stage q: Y slab at gps + q KP LD, C slab after all the Y slabs
  auto ysb = [&](int q) { return gps + q * DMQR_KP * TA_LD; };
  auto csb = [&](int q) { return gps + TA_NST * DMQR_KP * TA_LD + q * TA_COLS * TA_LD; };
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t span = (re > rb) ? re - rb + odd : 0;
  const int nslab = (int)ceil_div(span, TA_ROWS);
  const int rp = tid % TA_RP, cb = tid / TA_RP;
  const int64_t ldq = q1_ld(m);
  const double* Yp = Q1g + odd;            // Q1[r][i] at Yp[r + i*ldq]
  const double* Cp = A + n_s + n_s * lda;  // C[r][cc] at Cp[r + cc*lda], columns from n_s
  for (int e = tid; e < (lp - l) * TA_LD; e += TA_T)
    for (int q = 0; q < TA_NST; ++q) ysb(q)[l * TA_LD + e] = 0.0;
  auto issue = [&](int sl) {
    double* ys = ysb(sl % TA_NST);
    double* cs = csb(sl % TA_NST);
    const int64_t r = rb - odd + (int64_t)sl * TA_ROWS + 2 * rp;
    const int64_t gr = n_s + r;
    const int bytes = (gr + 1 < m) ? 16 : ((gr < m) ? 8 : 0);
    for (int i = cb; i < l; i += TA_CL) cp_async16(ys + i * TA_LD + 2 * rp, Yp + r + (int64_t)i * ldq, bytes);
    for (int cc = cb; cc < TA_COLS; cc += TA_CL)
      cp_async16(cs + cc * TA_LD + 2 * rp, Cp + r + (col0 + cc) * lda, (col0 + cc < ncols) ? bytes : 0);
    cp_async_commit();
  };
  auto fix = [&](int sl) {  // rows outside [rb, re) contribute nothing
    const int64_t r0 = rb - odd + (int64_t)sl * TA_ROWS;
    if (r0 >= rb && r0 + TA_ROWS <= re) return;
    double* ys = ysb(sl % TA_NST);
    for (int e = tid; e < l * TA_ROWS; e += TA_T) {
      const int i = e / TA_ROWS, rr = e % TA_ROWS;
      const int64_t r = r0 + rr;
      if (r < rb || r >= re) ys[i * TA_LD + rr] = 0.0;
    }
  };
  double acc[DMQR_KP / 8][2];
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int q = 0; q < TA_NST - 1; ++q) {  // prologue: TA_NST - 1 slabs in flight (empty groups past the end)
    if (q < nslab)
      issue(q);
    else
      cp_async_commit();
  }
  for (int sl = 0; sl < nslab; ++sl) {
    cp_async_wait<TA_NST - 2>();  // slab sl has landed (one group committed per slab)
    __syncthreads();
    {  // rows outside [rb, re): only the boundary slabs (uniform branch, no extra barrier otherwise)
      const int64_t r0 = rb - odd + (int64_t)sl * TA_ROWS;
      if (!(r0 >= rb && r0 + TA_ROWS <= re)) {
        fix(sl);
        __syncthreads();
      }
    }
    const double* ys = ysb(sl % TA_NST);
    const double* cs = csb(sl % TA_NST);
#pragma unroll
    for (int ks = 0; ks < TA_ROWS / 4; ++ks) {  // (predicated: a switch over lt spills k_spare)
      const int kr = 4 * ks + (lane & 3);
      const double b = cs[(wid * 8 + (lane >> 2)) * TA_LD + kr];
#pragma unroll
      for (int q = 0; q < DMQR_KP / 8; ++q)
        if (q < lt) dmma884(acc[q][0], acc[q][1], ys[(q * 8 + (lane >> 2)) * TA_LD + kr], b);
    }
    __syncthreads();  // (stage sl % TA_NST is refilled by the issue below, TA_NST - 1 slabs ahead)
    if (sl + TA_NST - 1 < nslab)
      issue(sl + TA_NST - 1);
    else
      cp_async_commit();
  }
  double* out = Gp + (int64_t)split * DMQR_KP * ldz;
  const int64_t cc = col0 + wid * 8 + 2 * (lane & 3);
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    if (q >= lt) break;
    const int i = q * 8 + (lane >> 2);
    out[(int64_t)i * ldz + cc] = acc[q][0];
    out[(int64_t)i * ldz + cc + 1] = acc[q][1];
  }
}

constexpr size_t SP_SMEM = TB_SMEM > TA_SMEM ? TB_SMEM : TA_SMEM;
static_assert(TA_COLS == TB_COLS, "k_spare: a phase-2 column tile is a phase-1 column tile");
static_assert(YG_SMEM <= SP_SMEM, "k_spare runs the Y = Q1 M tiles in its dynamic shared memory");
constexpr int NSPLIT_MAXG = 16;

// k_spare's wait for the panel: P published (P-mode: returns its column count)
// or Q1 published / the panel's release (returns 0).  Out of line: inlined, the
// polling loop pushes the kernel past its 2-CTA register cap.
__device__ __noinline__ int spare_wait_panel(Ctl* c, int P) {
  SpinGuard sg;
  for (;;) {
    if (ld_acquire(&c->p_count) >= (unsigned)P) return c->p_k;
    if (ld_acquire(&c->q1_count) >= (unsigned)P) return (ld_acquire(&c->p_count) >= (unsigned)P) ? c->p_k : 0;
    __nanosleep(200);
    sg.tick(2, c->q1_count, P);
  }
}

template <bool PM>  // PM: P-mode look-ahead (opt-in; panel_cq.cuh)
__global__ void __launch_bounds__(TB_T, 2) k_spare(Ctl* c, double* __restrict__ A,
                                                   const double* __restrict__ Wt, int64_t ldz,
                                                   uint8_t* __restrict__ upd, const double* __restrict__ Q1g,
                                                   double* __restrict__ Gp, unsigned* __restrict__ ctr, int P,
                                                   int nsplit_g, unsigned* __restrict__ tcnt,
                                                   long long* __restrict__ tline, const double* __restrict__ gM,
                                                   const double* __restrict__ Pg) {
  const long long t_first = gtimer();
  __shared__ int s_item, s_flag;
  const int tid = threadIdx.x;
  const CtlSnap& S = snap(c);  // (read from shared memory on use: registers are at the 2-CTA cap)
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 5);
  const int64_t m = S.m, n = S.n, lda = S.lda;
  // ---- phase 1: the pending update of the previous step ----
  const bool pend = S.la && S.pend;
  const int64_t pns = S.pend_ns;
  const int pl = S.pend_l;
  const int64_t pc0 = pns + pl, pmp = m - pns, pncols = n - pc0;
  // per 64-column tile: phase-1 tiles done (after the split counters in tcnt)
  const int64_t ncoltiles = ceil_div(max(n, (int64_t)1), TA_COLS) + 1;
  unsigned* colcnt = tcnt + ncoltiles;
  const int podd = (int)(pns & 1);
  const int ntx = (int)ceil_div(pmp + 1, TB_ROWS);
  const int ntb = (pend && pncols > 0 && pl > 0) ? ntx * (int)ceil_div(pncols, TB_COLS) : 0;
  // (the next item's index is fetched while the current tile runs: the
  // counter's L2 round trip is off the per-item path)
  __shared__ int s_next;
  if (tid == 0) s_next = (ntb > 0) ? (int)atomicAdd(&ctr[0], 1u) : ntb;
  for (;;) {
    __syncthreads();
    const int it = s_next;
    __syncthreads();
    if (it >= ntb) break;
    if (tid == 0) s_next = (int)atomicAdd(&ctr[0], 1u);
    const int64_t row0 = (int64_t)(it % ntx) * TB_ROWS - podd, col0 = (int64_t)(it / ntx) * TB_COLS;
    if (!(row0 >= pmp || col0 >= pncols || row0 + TB_ROWS <= pl))
      trail_b_tile<true>(A, Wt, ldz, upd, pns, m, lda, pl, pc0, pncols, pmp, row0, col0);
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(&colcnt[it / ntx], 1u);  // (column tile it / ntx: phase 2's tile of the same columns)
      s_flag = (atomicAdd(&ctr[1], 1u) == (unsigned)ntb - 1);
      if (S.tl) atomicMax(&S.tl[(S.step_idx & 63) * 32 + 29], (unsigned long long)gtimer());  // phase 1 end
    }
    __syncthreads();
    if (s_flag) {  // every tile has read the flags
      for (int64_t j = tid; j < n; j += blockDim.x) upd[j] = 0;
      if (tid == 0) c->pend = 0;
    }
  }
  // ---- phase 2: G = Q1^T C once Q1 is published; each tile once phase 1 has
  // updated its columns (its column tile's counter), not the whole of phase 1 ----
  if (!S.done) {
    __shared__ int s_pk;
    if (tid == 0) {
      // P-mode: the panel published its columns P first (G = P^T C, R1^-T folded
      // into k_trail_w's MT); otherwise wait for Q1 (or the panel's release)
      if constexpr (PM) {
        s_pk = spare_wait_panel(c, P);
      } else {
        SpinGuard sg;
        while (ld_acquire(&c->q1_count) < (unsigned)P) {
          __nanosleep(200);
          sg.tick(3, c->q1_count, P);
        }
        s_pk = 0;
      }
      s_flag = (s_pk > 0) || !c->q1_fail;
      if (S.tl) atomicMin(&S.tl[(S.step_idx & 63) * 32 + 28], (unsigned long long)gtimer());  // Q1 seen
      if (S.tl && S.step_idx == 20 && blockIdx.x < 256) S.tl[2048 + blockIdx.x * 4 + 0] = gtimer();
    }
    __syncthreads();
    if (s_flag) {
      const int64_t n_s = S.n_s;
      // (the P-mode choice stays in shared memory: registers are at the 2-CTA cap)
      __shared__ const double* s_yg;
      if (tid == 0) {
        s_yg = (PM && s_pk > 0) ? Pg : Q1g;
        if (s_pk == 0) s_pk = c->q1_kk;
      }
      __syncthreads();
      const int64_t ncols = n - n_s;
      const int ntile = (int)ceil_div(ncols, TA_COLS);
      const int ng = ntile * nsplit_g;
      const int64_t nyg = ceil_div(m - n_s - 1, YG_ROWS);
      for (;;) {
        // once the panel has published M, the Y = Q1 M tiles go first (they are
        // latency-bound and would otherwise trail the G tiles)
        if (tid == 0) {
          int it = -1;
          if (gM && ld_acquire(&c->m_pub) == (unsigned)S.step_idx + 1u && ld_acquire(&ctr[4]) < (unsigned)nyg) {
            const int y = (int)atomicAdd(&ctr[4], 1u);
            if (y < nyg) it = -2 - y;
          }
          if (it == -1) it = (int)atomicAdd(&ctr[2], 1u);
          s_item = it;
        }
        __syncthreads();
        const int it = s_item;
        __syncthreads();
        if (it <= -2) {
          ygemm_tile(A, Q1g, gM, n_s, m, lda, c->l_acc, -2 - it);
          __syncthreads();
          continue;
        }
        if (it < ng && ntb > 0) {  // the pending update of these columns must be complete
          if (tid == 0)
            for (SpinGuard sg; ld_acquire(&colcnt[it % ntile]) < (unsigned)ntx;) {
              __nanosleep(100);
              sg.tick(4, colcnt[it % ntile], ntx);
            }
          __syncthreads();
        }
        if (it >= ng) {
          if (tid == 0 && S.tl) atomicMax(&S.tl[(S.step_idx & 63) * 32 + 31], (unsigned long long)gtimer());
          if (tid == 0 && S.tl && S.step_idx == 20 && blockIdx.x < 256) S.tl[2048 + blockIdx.x * 4 + 2] = gtimer();
          break;
        }
        if (tid == 0 && S.tl && S.step_idx == 20 && blockIdx.x < 256) {
          if (S.tl[2048 + blockIdx.x * 4 + 1] == 0) S.tl[2048 + blockIdx.x * 4 + 1] = gtimer();
          S.tl[2048 + blockIdx.x * 4 + 3] += 1;
        }
        const int tile = it % ntile;
        g_partial(A, s_yg, Gp, ldz, n_s, m, lda, s_pk, ncols, (int64_t)tile * TA_COLS, it / ntile, nsplit_g);
        __syncthreads();
        // the CTA finishing a tile's last split sums its partials into split 0
        // (fixed order) for k_trail_w
        if (tid == 0) {
          __threadfence();
          s_flag = (atomicAdd(&tcnt[tile], 1u) == (unsigned)nsplit_g - 1);
        }
        __syncthreads();
        if (s_flag) {
          __threadfence();
          const int64_t col0 = (int64_t)tile * TA_COLS;
          for (int e = tid; e < s_pk * TA_COLS; e += blockDim.x) {
            const int i = e / TA_COLS, c2 = e % TA_COLS;
            const double* gp = Gp + (int64_t)i * ldz + col0 + c2;
            double v[NSPLIT_MAXG];
#pragma unroll
            for (int sp = 0; sp < NSPLIT_MAXG; ++sp) v[sp] = (sp < nsplit_g) ? __ldcg(gp + (int64_t)sp * DMQR_KP * ldz) : 0.0;
            double g = 0.0;
#pragma unroll
            for (int sp = 0; sp < NSPLIT_MAXG; ++sp) g += v[sp];
            Gp[(int64_t)i * ldz + col0 + c2] = g;
          }
          if (tid == 0) tcnt[tile] = 0u;
        }
        __syncthreads();
      }
    }
  }
  // ---- phase 3: Y = Q1 M below the top block once the panel has completed
  // (griddepcontrol.wait: the panel grid finished and its writes are visible),
  // here on the spare SMs instead of a kernel behind this one ----
  // (gM == nullptr: k_trail_w's extra CTAs do these tiles, off the step's critical path)
  if (!S.done && gM) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    if (!c->cq_fail) {
      const int l = c->l_acc;
      const int64_t nyg = ceil_div(m - S.n_s - 1, YG_ROWS);
      for (;;) {
        if (tid == 0) s_item = (int)atomicAdd(&ctr[4], 1u);
        __syncthreads();
        const int it = s_item;
        __syncthreads();
        if (it >= nyg) break;
        ygemm_tile(A, Q1g, gM, S.n_s, m, lda, l, it);
        __syncthreads();
      }
    }
  }
  // ---- the last CTA: reset the counters (every CTA has waited for the panel) ----
  if (tid == 0) {
    __threadfence();
    s_flag = (atomicAdd(&ctr[3], 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (s_flag) {
    for (int64_t q = tid; q < ncoltiles; q += blockDim.x) colcnt[q] = 0u;
    if (tid == 0) {
      ctr[0] = ctr[1] = ctr[2] = ctr[3] = ctr[4] = 0u;
      if (tline) {
        tline[4 * (c->step_idx & 255) + 2] = t_first;
        tline[4 * (c->step_idx & 255) + 3] = gtimer();
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
}

// Wt for the CholeskyQR2 panel path (look-ahead), after the panel: per
// 32-column tile from n_s + l,  Wt = A1 C_top + A2 G  (G = Q1^T C summed by
// k_spare; A1 = T^T E and A2 = T^T M^T published by k_panel_cq as (F T) and
// (M T)), then R12 = C_top - Y1 Wt, the norm downdate (k_downdate's order),
// guard columns and the panel-column bookkeeping.  Warp w: columns
// 8 (w & 3) .. +8, row tiles [5 (w >> 2), +5).  Exits when the panel declined
// (cq_fail): k_trail_a then runs as usual.
constexpr int TW_COLS = 32;
constexpr int TW_CLD = TW_COLS + 4;  // 36 = 4 mod 16 (conflict-free 4 x 4 half-warp fragments)
constexpr size_t TW_SMEM = sizeof(double) * (3 * DMQR_KP * DMQR_KP + 3 * DMQR_KP * TW_CLD);

// Step close (close != nullptr): the CTA finishing the step's last tile ends
// the step itself when nothing else is left to do -- no guard column was
// listed -- i.e. it runs k_step_end's bookkeeping and posts the host record;
// k_tail (tail.cuh), launched behind, then finds the record posted and exits
// at once.  That is the common case; k_tail does the rest otherwise.
struct StepRec;
__device__ __forceinline__ void step_end_body(const CtlSnap& S, Ctl* c, StepRec* __restrict__ steps,
                                              double* __restrict__ norm_trace,
                                              unsigned long long* __restrict__ trace_bits, const double* __restrict__ A,
                                              double* __restrict__ Wt, int64_t ldz, double* __restrict__ u,
                                              double* __restrict__ uref, uint8_t* __restrict__ upd);
__device__ __forceinline__ void step_post(const CtlSnap& S, Ctl* c, HostRec* __restrict__ hrec);
struct StepClose {
  StepRec* steps;
  HostRec* hrec;
  unsigned* counter;  // tiles done (reset by the closing CTA)
  // the Y = Q1 M tiles below the panel's top block (ygemm_tile) run here, on the FIRST `ygrid` CTAs,
  // beside the Wt tiles: nothing before the next step's k_gram reads those rows, so they need not sit
  // between the panel and this kernel.  (They are short and come first in block order: when the grid
  // exceeds one wave, the Wt tiles left over start a few us later instead of the Y tiles a whole Wt
  // tile later.)
  const double* q1g;
  const double* gM;
  int ygrid;
};

// (debug timeline: the first Wt tile's phase stamps, slots 22.. of the step's row)
#define TW_STAMP(k) \
  if (S.tl && wbx == 0 && tid == 0) S.tl[(S.step_idx & 63) * 32 + (k)] = (unsigned long long)gtimer()
__global__ void __launch_bounds__(TA_T) k_trail_w(Ctl* c, double* __restrict__ A,
                                                  const double* __restrict__ Gp, const double* __restrict__ FM,
                                                  double* __restrict__ Wt, int64_t ldz, double* __restrict__ u,
                                                  double* __restrict__ uref, uint8_t* __restrict__ upd,
                                                  int32_t* __restrict__ glist, const StepClose close) {
  pdl_enter();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 7);
  if (S.done || S.cq_fail) return;
  const int64_t n_s = S.n_s, m = S.m, n = S.n, lda = S.lda;
  const int l = S.l_acc;
  const int64_t c0 = n_s + l, ncols = n - c0, n_s1 = c0;
  const int wbx = (int)blockIdx.x - (close.counter ? close.ygrid : 0);  // index among the Wt tiles
  const int64_t col0 = (int64_t)wbx * TW_COLS;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (wbx < 0) {  // a Y = Q1 M tile
    const int64_t yb = (int)blockIdx.x;
    if (l == 0 || l + yb * YG_ROWS >= m - n_s) return;
    ygemm_tile(A, close.q1g, close.gM, n_s, m, lda, l, yb);
  } else {
  if (col0 >= ncols || l == 0) return;  // (no trailing columns: k_step_end does the bookkeeping)
  extern __shared__ __align__(16) double tws[];
  double* a1 = tws;                          // FT[t][i]  (A1 = FT^T)
  double* a2 = a1 + DMQR_KP * DMQR_KP;       // MT[t][i]  (A2 = MT^T)
  double* y1 = a2 + DMQR_KP * DMQR_KP;       // Y1[i][t] (unit lower) at y1[t * KP + i]
  double* gs = y1 + DMQR_KP * DMQR_KP;       // G[t][c], then R12[i][c]
  double* cts = gs + DMQR_KP * TW_CLD;       // C_top[t][c]
  double* ws = cts + DMQR_KP * TW_CLD;       // Wt[t][c]
  const int lp4 = (l + 3) / 4 * 4, lt = (l + 7) / 8;
  const int cb = wid & 3, q0 = (wid >> 2) * 5, q1 = min(q0 + 5, lt);
  const double* gFT = FM;  // MT follows at FM + KP * KP
  __shared__ __align__(8) uint64_t tw_bar;
  if (tid == 0) mbar_init(&tw_bar, 1);
  __syncthreads();
  // every operand staged with cp.async: all of the tile's L2 / HBM reads are in
  // flight at once (one round trip), zeros stored directly
  for (int e = tid; e < DMQR_KP * TW_COLS; e += TA_T) {
    const int t = e / TW_COLS, c2 = e % TW_COLS;
    const int64_t col = col0 + c2;
    if (t < l && col < ncols) {
      cp_async8(gs + t * TW_CLD + c2, Gp + (int64_t)t * ldz + l + col);  // G columns from n_s
      cp_async8(cts + t * TW_CLD + c2, A + (n_s + t) + (c0 + col) * lda);
    } else {
      gs[t * TW_CLD + c2] = 0.0;
      cts[t * TW_CLD + c2] = 0.0;
    }
  }
  // FT and MT are published whole (zero outside their l x l upper triangles) and sit back to back in
  // global and in shared memory: ONE TMA bulk copy (83 KB) instead of twenty 16-byte copies per thread
  if (tid == 0) {
    mbar_arrive_expect_tx(&tw_bar, (unsigned)(2 * DMQR_KP * DMQR_KP * sizeof(double)));
    bulk_g2s(a1, gFT, (unsigned)(2 * DMQR_KP * DMQR_KP * sizeof(double)), &tw_bar);
  }
  for (int e = tid; e < DMQR_KP * DMQR_KP; e += TA_T) {
    const int t = e / DMQR_KP, i = e % DMQR_KP;
    // Y1[i][t] from the packed panel (column n_s + t, row n_s + i), stored as y1[t][i]: global reads
    // and shared writes both run along i (a transposed y1[i][t] made every copy a 16-way bank conflict)
    if (t < i && i < l)
      cp_async8(y1 + t * DMQR_KP + i, A + (n_s + t) * lda + n_s + i);
    else
      y1[t * DMQR_KP + i] = (t == i && i < l) ? 1.0 : 0.0;
  }
  cp_async_commit();
  TW_STAMP(22);
  cp_async_wait<0>();
  mbar_wait_parity(&tw_bar, 0);
  __syncthreads();
  TW_STAMP(23);
  const int lr = lane >> 2, lk = lane & 3;
  const int64_t cc = col0 + cb * 8 + 2 * lk;
  // ---- Wt = A1 C_top + A2 G ----
  double w[5][2];
#pragma unroll
  for (int q = 0; q < 5; ++q) w[q][0] = w[q][1] = 0.0;
  for (int ks = 0; ks < lp4; ks += 4) {
    const int t = ks + lk;
    const double b1 = cts[t * TW_CLD + cb * 8 + lr];
    const double b2 = gs[t * TW_CLD + cb * 8 + lr];
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (q0 + q < q1) {
        const int i = (q0 + q) * 8 + lr;
        dmma884(w[q][0], w[q][1], a1[t * DMQR_KP + i], b1);
        dmma884(w[q][0], w[q][1], a2[t * DMQR_KP + i], b2);
      }
  }
#pragma unroll
  for (int q = 0; q < 5; ++q)
    if (q0 + q < q1) {
      const int i = (q0 + q) * 8 + lr;
      if (i < lp4) {
        const double w0 = (cc < ncols) ? w[q][0] : 0.0, w1 = (cc + 1 < ncols) ? w[q][1] : 0.0;
        Wt[(int64_t)i * ldz + cc] = w0;
        Wt[(int64_t)i * ldz + cc + 1] = w1;
        ws[i * TW_CLD + cb * 8 + 2 * lk] = w0;
        ws[i * TW_CLD + cb * 8 + 2 * lk + 1] = w1;
      }
    }
  __syncthreads();
  // ---- R12 = C_top - Y1 Wt -> A and gs ----
  double r[5][2];
#pragma unroll
  for (int q = 0; q < 5; ++q)
#pragma unroll
    for (int h = 0; h < 2; ++h) r[q][h] = (q0 + q < q1) ? cts[((q0 + q) * 8 + lr) * TW_CLD + cb * 8 + 2 * lk + h] : 0.0;
  for (int ks = 0; ks < lp4; ks += 4) {
    const int t = ks + lk;
    const double b = ws[t * TW_CLD + cb * 8 + lr];
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (q0 + q < q1) dmma884(r[q][0], r[q][1], -y1[t * DMQR_KP + (q0 + q) * 8 + lr], b);
  }
  __syncthreads();  // all reads of gs (G) are done
#pragma unroll
  for (int q = 0; q < 5; ++q)
    if (q0 + q < q1) {
      const int i = (q0 + q) * 8 + lr;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const bool in = i < l && cc + h < ncols;
        gs[i * TW_CLD + cb * 8 + 2 * lk + h] = in ? r[q][h] : 0.0;
        if (in) A[(n_s + i) + (c0 + cc + h) * lda] = r[q][h];
      }
    }
  __syncthreads();
  TW_STAMP(24);
  // ---- downdate: warp w, columns 4w .. 4w+3 (k_downdate's per-column order) ----
  double d[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    d[q] = 0.0;
    for (int rr = lane; rr < l; rr += 32) {
      const double x = gs[rr * TW_CLD + wid * 4 + q];
      d[q] = fma(x, x, d[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) d[q] = warp_sum(d[q]);
  __syncthreads();
  if (lane < 4) {
    double dq = d[0];
#pragma unroll
    for (int q = 1; q < 4; ++q)
      if (lane == q) dq = d[q];
    const int64_t j = c0 + col0 + wid * 4 + lane;
    if (j < n) {
      const double uj = u[j], rj = uref[j];
      const double sq = __dsub_rn(__dmul_rn(uj, uj), dq);
      if (sq <= __dmul_rn(1e-2, __dmul_rn(rj, rj)) && n_s1 < m)
        glist[atomicAdd(&c->gcount, 1)] = (int32_t)j;  // guard: k_guard recomputes it
      else
        u[j] = sqrt(fmax(sq, 0.0));
    }
  }
  if (wbx == 0) la_panel_columns(c, A, Wt, ldz, u, uref, upd, n_s, l, c0);
  TW_STAMP(25);
  }
  // ---- the last tile's CTA closes the step when no guard column was listed ----
  if (close.counter) {
    __shared__ int s_close;
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      const unsigned ntiles = (unsigned)((ncols > 0 ? ceil_div(ncols, TW_COLS) : 0) +
                                         (m - n_s > l ? ceil_div(m - n_s - l, YG_ROWS) : 0));
      int cl = 0;
      if (atomicAdd(close.counter, 1u) == ntiles - 1) {
        __threadfence();
        *close.counter = 0u;
        cl = (ctl_ld(&c->gcount) == 0 && S.tc0 < n);
      }
      s_close = cl;
    }
    __syncthreads();
    if (s_close && tid == 0 && S.tl) S.tl[(S.step_idx & 63) * 32 + 26] = (unsigned long long)gtimer();
    if (s_close && wid == 0) {
      step_end_body(S, c, close.steps, nullptr, nullptr, A, Wt, ldz, u, uref, upd);
      __threadfence();
      __syncwarp();
      if (lane == 0 && close.hrec) step_post(S, c, close.hrec);
    }
  }
}

// ---------------------------------------------------------------------------
// Look-ahead guard columns (downdated square <= 1e-2 u_ref^2, listed by the
// Wt epilogues): their update C -= Y Wt on rows [n_s + l, m) with
// k_trail_b's DMMA sequence per element, then (last CTA) their exact norms as
// k_downdate computes them, and the flag that they are done.  One CTA per 64
// rows, DMMA on 64 x 72 column groups; exits at once when the list is empty.
// ---------------------------------------------------------------------------
constexpr int GU_T = 256;
constexpr int GU_ROWS = 64;
constexpr int GU_LD = GU_ROWS + 4;  // 4 mod 16
constexpr size_t GU_SMEM = sizeof(double) * (2 * DMQR_KP * GU_LD + DMQR_KP * DMQR_KP);
constexpr int GU_GROUPS = 4;  // column groups of 72 per CTA (grid.y spreads the rest)

// (one CTA's work: 64-row block bx, column-group range by; k_tail runs the same
// items from a persistent grid)
__device__ __forceinline__ void guard_cta(const CtlSnap& S, double* __restrict__ A, const double* __restrict__ Wt,
                                          int64_t ldz, const uint8_t* __restrict__ upd,
                                          const int32_t* __restrict__ glist, const int cnt, const int bx,
                                          const int by) {
  const int64_t m = S.m, lda = S.lda, n_s = S.n_s;
  const int l = S.l_acc;
  const int64_t base = n_s + l;
  // many guard columns (graded / tall matrices): finish this step's whole
  // update now -- every column not yet updated -- and leave nothing pending
  const int64_t ntr = S.n - base;
  const bool full = (int64_t)cnt * 8 > ntr;
  const int nlist = full ? (int)ntr : cnt;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  extern __shared__ __align__(16) double gus[];
  double* ys = gus;                        // ys[t][rr] = Y[r0 + rr][t]
  double* cs = gus + DMQR_KP * GU_LD;      // cs[q][rr] = C[r0 + rr][col_q]
  double* ws = gus + 2 * DMQR_KP * GU_LD;  // ws[t][q]  = Wt[t][col_q]
  __shared__ int s_col[DMQR_KP];
  const int64_t r0 = base + (int64_t)bx * GU_ROWS;
  const int lp4 = (l + 3) / 4 * 4;
  if (r0 < m) {
    const int nr = (int)min((int64_t)GU_ROWS, m - r0);
    for (int e = tid; e < lp4 * GU_ROWS; e += GU_T) {
      const int t = e / GU_ROWS, rr = e % GU_ROWS;
      ys[t * GU_LD + rr] = (t < l && rr < nr) ? A[(n_s + t) * lda + r0 + rr] : 0.0;
    }
    // blockIdx.y: a range of GU_GROUPS column groups of the list
    const int gbeg = by * GU_GROUPS * DMQR_KP, gend = min(nlist, gbeg + GU_GROUPS * DMQR_KP);
    for (int g0 = gbeg; g0 < gend; g0 += DMQR_KP) {
      const int ng = min(DMQR_KP, gend - g0);
      if (tid < DMQR_KP) {
        int j = -1;
        if (tid < ng) {
          j = full ? (int)(base + g0 + tid) : glist[g0 + tid];
          if (full && upd[j]) j = -1;  // (the panel's own columns: already final)
        }
        s_col[tid] = j;
      }
      __syncthreads();
      for (int e = tid; e < lp4 * DMQR_KP; e += GU_T) {
        const int t = e / DMQR_KP, q = e % DMQR_KP;
        const int j = s_col[q];
        ws[t * DMQR_KP + q] = (t < l && j >= 0) ? Wt[t * ldz + (j - base)] : 0.0;
      }
      for (int e = tid; e < DMQR_KP * GU_ROWS; e += GU_T) {
        const int q = e / GU_ROWS, rr = e % GU_ROWS;
        const int j = s_col[q];
        cs[q * GU_LD + rr] = (j >= 0 && rr < nr) ? A[(int64_t)j * lda + r0 + rr] : 0.0;
      }
      __syncthreads();
      const int rr = wid * 8 + (lane >> 2);
      double acc[DMQR_KP / 8][2];
#pragma unroll
      for (int q = 0; q < DMQR_KP / 8; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[q][h] = cs[(q * 8 + 2 * (lane & 3) + h) * GU_LD + rr];
      for (int ks = 0; ks < lp4; ks += 4) {
        const int t = ks + (lane & 3);
        const double a = -ys[t * GU_LD + rr];
#pragma unroll
        for (int q = 0; q < DMQR_KP / 8; ++q) dmma884(acc[q][0], acc[q][1], a, ws[t * DMQR_KP + q * 8 + (lane >> 2)]);
      }
      if (rr < nr) {
#pragma unroll
        for (int q = 0; q < DMQR_KP / 8; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int qq = q * 8 + 2 * (lane & 3) + h;
            const int j = s_col[qq];
            if (j >= 0) A[(int64_t)j * lda + r0 + rr] = acc[q][h];
          }
      }
      __syncthreads();
    }
  }
}

// After every guard item: the step's flags (one thread).
__device__ __forceinline__ void guard_flags(const CtlSnap& S, Ctl* c, const int cnt) {
  const bool full = (int64_t)cnt * 8 > S.n - (S.n_s + S.l_acc);
  if (full) c->pend_done = 1;           // k_step_end: nothing is pending after this step
  if (full || cnt > 32) c->la_bad = 1;  // guards are not rare here: the host goes serial
}

__global__ void __launch_bounds__(GU_T) k_guard(Ctl* c, double* __restrict__ A,
                                                const double* __restrict__ Wt, int64_t ldz,
                                                uint8_t* __restrict__ upd, double* __restrict__ u,
                                                double* __restrict__ uref, const int32_t* __restrict__ glist,
                                                unsigned* __restrict__ counter) {
  pdl_enter();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 9);
  const int cnt = c->gcount;
  if (S.done || cnt == 0) return;
  guard_cta(S, A, Wt, ldz, upd, glist, cnt, (int)blockIdx.x, (int)blockIdx.y);
  const int tid = threadIdx.x;
  __shared__ int s_last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = (atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) {
    *counter = 0u;
    guard_flags(S, c, cnt);
  }
  // (the guard columns' exact norms: k_guard_norms, grid-wide, right behind)
}

// Exact norms of k_guard's columns (k_downdate's arithmetic), a warp per
// column over the whole grid; then the columns' look-ahead flags (set while an
// update is still pending; all cleared when k_guard finished the whole update).
// (the warps w0, w0 + nw, ... of a grid; threads t0, t0 + nt, ... for the flag sweep)
__device__ __forceinline__ void guard_norms_part(const CtlSnap& S, const double* __restrict__ A,
                                                 uint8_t* __restrict__ upd, double* __restrict__ u,
                                                 double* __restrict__ uref, const int32_t* __restrict__ glist,
                                                 const int cnt, const int64_t w0, const int64_t nw, const int64_t t0,
                                                 const int64_t nt) {
  const int64_t m = S.m, lda = S.lda, base = S.n_s + S.l_acc;
  const bool full = (int64_t)cnt * 8 > S.n - base;
  const int lane = threadIdx.x & 31;
  for (int64_t q = w0; q < cnt; q += nw) {
    const int64_t j = glist[q];
    const double nu = warp_col_norm(A + j * lda + base, m - base, lane);
    if (lane == 0) {
      u[j] = nu;
      uref[j] = nu;
      if (!full) upd[j] = 1;  // (an update is pending: guards exist only with rows below and tiles past tc0)
    }
  }
  if (full)
    for (int64_t j = t0; j < S.n; j += nt) upd[j] = 0;
}

__global__ void __launch_bounds__(256) k_guard_norms(Ctl* c, const double* __restrict__ A,
                                                      uint8_t* __restrict__ upd, double* __restrict__ u,
                                                      double* __restrict__ uref, const int32_t* __restrict__ glist) {
  pdl_enter();
  const CtlSnap S = snap(c);
  const int cnt = c->gcount;
  if (S.done || cnt == 0) return;
  guard_norms_part(S, A, upd, u, uref, glist, cnt, (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5,
                   (int64_t(gridDim.x) * blockDim.x) >> 5, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
                   (int64_t)gridDim.x * blockDim.x);
}

}  // namespace dmqr
