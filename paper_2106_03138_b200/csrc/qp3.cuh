// Blocked greedy column pivoting (QP3 / LAPACK laqps form) on the device:
//   qrp                   rrqr.py:238-291   (every column)
//   _scalar_step          rrqr.py:219-235   (QRDM's scalar-fallback runs, rrqr.py:343-353)
//   downdate_norms(s,s+1) rrqr.py:161-186   (per column, guard recompute included)
//   check_stop            rrqr.py:189-203;  norm floor dm.py:140 (fallback runs only)
//
// The reference applies every pivot's reflector to the whole trailing block at
// once (a rank-1 update, BLAS2: one read + one write of the trailing block per
// column).  Here the update is DELAYED over a block of up to QP_NB columns:
//
//   A_true[r, c] = A[r, c] - sum_{t' < t} Y[r, t'] F[c, t']      (rows r >= s)
//
// with Y the block's reflectors (stored in the packed panel columns) and
// F[c, t] = coeff_t * (v_t^T A_true[s_t:, c]).  Per column only ONE read of
// the trailing block is needed (w = v^T A, to form F and the new row of R for
// the norm downdate); the block's C -= Y F^T runs at the end as DMMA tiles
// (k_trail_b's tile code).  Decisions are the reference's: pivot = first
// argmax of the partial norms, stop test before each column, and (fallback
// runs) the floor test -- once max u exceeds the floor the block ends and the
// DM step resumes.  Guard columns (sq <= 1e-2 u_ref^2) get an exact norm of
// their fully updated column in place (Y F^T applied on the fly); when there
// are more than QP_GMAX of them the block ends and they are recomputed from
// the updated matrix.  Rounding differs from the reference's sequential
// rank-1 updates only at the level of the blocked vs unblocked Householder
// application (the same reflectors, the same pivots).
//
// One cooperative persistent launch per block; per column three grid
// barriers (+1 when guards occur):
//   gamma  argmax of the partials (+ guard norms), stop / floor test, column
//          swap (full height) and pivot column update x = a_p - Y F[p]^T, the
//          pivot's norm partials                                   (row-parallel)
//   alpha  beta / coeff; v = x[1:]/(x0 - beta) into a side buffer; per column
//          w_c = v^T A[s:, c] (warp per column, 16-byte streaming loads; the
//          block's own reflector columns give z = Y^T v the same way)
//   beta   F[c, t] = coeff (w_c - F[c, :t] z), the new R row, norm downdate,
//          guard flags, partial argmax                          (warp per column)
//   guard  exact norms of the flagged columns (rows x guards), last CTA reduces
// HBM-bound: the alpha read of the trailing block (8 m' n'' bytes) per column.
#pragma once
#include "common.cuh"
#include "trailing.cuh"

namespace dmqr {

constexpr int QP_T = 256;
constexpr int QP_W = QP_T / 32;
constexpr int QP_NB = 64;     // columns per block (F row length)
constexpr int QP_GMAX = 64;   // guard columns recomputed in place per column
constexpr int QP_PLD = 8;     // per-CTA partial record (doubles)
constexpr int QP_GMAXCTA = 320;  // grid cap (2 CTAs x 148 SMs fits)
constexpr int QP_SUB = 64;       // guard phase: rows per staged sub-chunk
constexpr size_t QP_SMEM = TB_SMEM;  // the block update's tile staging is the largest user
constexpr int QP_XCH = 12288;        // rows of x staged per chunk in alpha (96 KB)
constexpr int QP_SEG = 2048;         // rows per alpha work item (at least)
constexpr int QP_RMAX = 32;          // segment slots per column in wb
static_assert(sizeof(double) * QP_XCH <= QP_SMEM, "x staging");
static_assert(sizeof(double) * (QP_SUB * (QP_NB + 1) + QP_GMAX * (QP_NB + 1)) <= QP_SMEM, "guard staging");

struct Qp3Args {
  Ctl* c;
  double* A;
  double* u;
  double* uref;
  int64_t* perm;
  int64_t* swaps;
  double* coeffs;
  StepRec* steps;
  double* F;        // [n][QP_NB]
  double* Wt;       // block update: Wt[t * ldz + (col - c0)]
  int64_t ldz;
  double* vb;       // [m] v of the current reflector
  double* wb;       // [n][QP_RMAX] per-segment partial dots of w_c (and z for the block's own columns)
  double* part;     // [G][QP_PLD]
  double* gpart;    // [G][QP_GMAX][2]
  int32_t* glist;   // guard columns of the current column step (capacity n)
  double* gfresh;   // [QP_GMAX] fresh norms of the in-place guard columns
  unsigned* cnt;    // [0] barrier, [1] guard count, [2] guard-phase arrivals, [3] guard-done column; zeroed before launch
  long long* dbg;   // optional phase clocks of CTA 0 (globaltimer ns): [t * 8 + phase], block end at [512..]
  int qrp;          // 1: greedy pivoting (qrp): no floor test; 0: QRDM scalar-fallback run
  int col_limit;    // columns this launch may factor (<= QP_NB)
};

// argmax with the reference's tie rule (np.argmax: first index of the maximum)
__device__ __forceinline__ void am_merge(double& bv, int& bi, double ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) {
    bv = ov;
    bi = oi;
  }
}

// alpha's row split of the column step at s: segment length and count (rows
// from the first even row past s; >= 1 segment so the head row is counted)
__device__ __forceinline__ int qp_seg_len(int64_t m, int64_t s) {
  const int64_t nrt = max((int64_t)0, m - (((s + 1) + 1) & ~(int64_t)1));
  return (int)max((int64_t)QP_SEG, ceil_div(ceil_div(nrt, QP_RMAX), 64) * 64);
}
__device__ __forceinline__ int qp_nseg(int64_t m, int64_t s) {
  const int64_t nrt = max((int64_t)0, m - (((s + 1) + 1) & ~(int64_t)1));
  return (int)max((int64_t)1, ceil_div(nrt, qp_seg_len(m, s)));
}

__device__ __forceinline__ double2 ldcs2(const double* p) { return __ldcs(reinterpret_cast<const double2*>(p)); }

__global__ void __launch_bounds__(QP_T, 2) k_qp3(Qp3Args a) {
  Ctl* c = a.c;
  const CtlSnap S = snap(c);
  if (S.done) return;
  double* __restrict__ A = a.A;
  double* __restrict__ F = a.F;
  const int64_t m = S.m, n = S.n, lda = S.lda, s0 = S.n_s, kmax = S.kmax;
  const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gw = b * QP_W + wid, NW = G * QP_W;
  const int64_t rch = ceil_div(m, G);
  const int64_t r_lo = min((int64_t)b * rch, m), r_hi = min(r_lo + rch, m);
  extern __shared__ __align__(16) double qsm[];
  __shared__ double s_fp[QP_NB], s_z[QP_NB], s_y[QP_NB];
  __shared__ double s_red[QP_W][4];
  __shared__ int s_redi[QP_W];
  __shared__ double s_b[4];
  __shared__ int s_bi[2];
#define QCLK(k) \
  if (a.dbg && b == 0 && tid == 0 && t < 64) a.dbg[t * 8 + (k)] = gtimer()
  uint32_t bar_k = 0;
  auto gsync = [&]() {
    ++bar_k;
    grid_sync_count(a.cnt, bar_k * (uint32_t)G);
  };

  // partial argmax of u over columns [from, n) owned by this CTA's warps
  auto argmax_partial = [&](int64_t from) {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int64_t col = from + gw; col < n; col += NW)
      if (lane == 0) am_merge(bv, bi, a.u[col], (int)col);
    if (lane == 0) {
      s_red[wid][0] = bv;
      s_redi[wid] = bi;
    }
  };
  auto argmax_publish = [&]() {
    __syncthreads();
    if (tid == 0) {
      double bv = s_red[0][0];
      int bi = s_redi[0];
      for (int w = 1; w < QP_W; ++w) am_merge(bv, bi, s_red[w][0], s_redi[w]);
      a.part[b * QP_PLD + 0] = bv;
      a.part[b * QP_PLD + 1] = (double)bi;
    }
  };

  argmax_partial(s0);
  argmax_publish();
  gsync();

  int t = 0, step_idx = S.step_idx, n_swaps = S.n_swaps;
  int exit_reason = 0;  // 1 stopped, 2 floor (back to DM), 3 all columns, 4 block full, 5 guard overflow
  int g_prev = 0;       // guards of the previous column (their fresh norms are in u, not in the partials)
  int status = 0;
  for (;;) {
    const int64_t s = s0 + t;
    // ================= gamma =================
    QCLK(0);
    if (g_prev > 0 && g_prev <= QP_GMAX) {  // the guard phase's last CTA has published the fresh norms
      if (tid == 0) {
        unsigned v;
        SpinGuard sg;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(a.cnt + 3) : "memory");
          if (v >= (unsigned)t) break;
          sg.tick(7, v, t);
        }
      }
      __syncthreads();
    }
    QCLK(1);
    {  // argmax of the partials and the guard columns: every thread loads <= 2 partials (one L2 round trip)
      double bv = -1.0;
      int bi = 0x7fffffff;
      if (tid < G) am_merge(bv, bi, __ldcg(a.part + tid * QP_PLD), (int)__ldcg(a.part + tid * QP_PLD + 1));
      if (tid + QP_T < G)
        am_merge(bv, bi, __ldcg(a.part + (tid + QP_T) * QP_PLD), (int)__ldcg(a.part + (tid + QP_T) * QP_PLD + 1));
      if (tid < g_prev && g_prev <= QP_GMAX) am_merge(bv, bi, __ldcg(a.gfresh + tid), __ldcg(a.glist + tid));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) am_merge(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
      if (lane == 0) {
        s_red[wid][0] = bv;
        s_redi[wid] = bi;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < QP_W; ++w) am_merge(bv, bi, s_red[w][0], s_redi[w]);
        s_b[0] = bv;
        s_bi[0] = bi;
      }
    }
    __syncthreads();
    const double umax = s_b[0];
    const int64_t p = s_bi[0];
    if (g_prev > QP_GMAX) exit_reason = 5;
    else if (status) exit_reason = 3;
    else if (t >= a.col_limit) exit_reason = 4;
    else if (s >= kmax) exit_reason = 3;
    else if (S.stop_active && sqrt((double)(n - s)) * umax <= S.stop_rhs) exit_reason = 1;  // rrqr.py:197-203
    else if (!a.qrp && !(umax <= S.floor)) exit_reason = 2;                             // dm.py:140
    if (exit_reason) break;
    if (step_idx >= S.step_cap) {
      status = -5;
      exit_reason = 3;
      break;
    }

    // pivot's pending row of F (read before CTA 0 swaps F rows in alpha)
    for (int q = tid; q < t; q += QP_T) s_fp[q] = F[p * QP_NB + q];
    __syncthreads();
    double ss = 0.0, am = 0.0, x0 = 0.0;
    for (int64_t r = r_lo + tid; r < r_hi; r += QP_T) {
      double x = A[r + p * lda];
      if (p != s) {
        const double y = A[r + s * lda];
        A[r + p * lda] = y;
      }
      if (r >= s) {
        const double* yr = A + r + s0 * lda;
        double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
        int q = 0;
        for (; q + 4 <= t; q += 4) {
          c0 = fma(yr[q * lda], s_fp[q], c0);
          c1 = fma(yr[(q + 1) * lda], s_fp[q + 1], c1);
          c2 = fma(yr[(q + 2) * lda], s_fp[q + 2], c2);
          c3 = fma(yr[(q + 3) * lda], s_fp[q + 3], c3);
        }
        for (; q < t; ++q) c0 = fma(yr[q * lda], s_fp[q], c0);
        x -= (c0 + c1) + (c2 + c3);
        ss = fma(x, x, ss);
        am = fmax(am, fabs(x));
        if (r == s) x0 = x;
      }
      A[r + s * lda] = x;
    }
    ss = warp_sum(ss);
    am = warp_max(am);
    x0 = warp_sum(x0);
    if (lane == 0) {
      s_red[wid][0] = ss;
      s_red[wid][1] = am;
      s_red[wid][2] = x0;
    }
    __syncthreads();
    if (tid == 0) {
      double t0 = 0.0, t1 = 0.0, t2 = 0.0;
      for (int w = 0; w < QP_W; ++w) {
        t0 += s_red[w][0];
        t1 = fmax(t1, s_red[w][1]);
        t2 += s_red[w][2];
      }
      a.part[b * QP_PLD + 2] = t0;
      a.part[b * QP_PLD + 3] = t1;
      a.part[b * QP_PLD + 4] = t2;
    }
    gsync();

    // ================= alpha =================
    QCLK(2);
    {
      double t0 = 0.0, t1 = 0.0, t2 = 0.0;
      if (tid < G) {
        t0 = __ldcg(a.part + tid * QP_PLD + 2);
        t1 = __ldcg(a.part + tid * QP_PLD + 3);
        t2 = __ldcg(a.part + tid * QP_PLD + 4);
      }
      if (tid + QP_T < G) {
        t0 += __ldcg(a.part + (tid + QP_T) * QP_PLD + 2);
        t1 = fmax(t1, __ldcg(a.part + (tid + QP_T) * QP_PLD + 3));
        t2 += __ldcg(a.part + (tid + QP_T) * QP_PLD + 4);
      }
      t0 = warp_sum(t0);
      t1 = warp_max(t1);
      t2 = warp_sum(t2);
      if (lane == 0) {
        s_red[wid][0] = t0;
        s_red[wid][1] = t1;
        s_red[wid][2] = t2;
      }
      __syncthreads();
      if (tid == 0) {
        for (int w = 1; w < QP_W; ++w) {
          t0 += s_red[w][0];
          t1 = fmax(t1, s_red[w][1]);
          t2 += s_red[w][2];
        }
        s_b[0] = t0;
        s_b[1] = t1;
        s_b[2] = t2;
      }
    }
    __syncthreads();
    const double xs = s_b[2], amax = s_b[1];
    double nrm;
    if (amax == 0.0) {
      nrm = 0.0;
    } else if (s_b[0] > 1e-280 && s_b[0] < 1e280) {
      nrm = sqrt(s_b[0]);
    } else {  // rescaled second pass (squares out of range; rare)
      int e;
      frexp(amax, &e);
      double sc = 0.0;
      for (int64_t r = max(r_lo, s) + tid; r < r_hi; r += QP_T) {
        const double y = ldexp(A[r + s * lda], -e);
        sc = fma(y, y, sc);
      }
      sc = warp_sum(sc);
      if (lane == 0) s_red[wid][3] = sc;
      __syncthreads();
      if (tid == 0) {
        double t0 = 0.0;
        for (int w = 0; w < QP_W; ++w) t0 += s_red[w][3];
        a.part[b * QP_PLD + 5] = t0;
      }
      gsync();
      if (wid == 0) {
        double t0 = 0.0;
        for (int q = lane; q < G; q += 32) t0 += __ldcg(a.part + q * QP_PLD + 5);
        t0 = warp_sum(t0);
        if (lane == 0) s_b[3] = t0;
      }
      __syncthreads();
      nrm = ldexp(sqrt(s_b[3]), e);
    }
    // make_reflector (householder.py:57-79)
    double beta, coeff, u0;
    if (nrm == 0.0) {
      beta = 0.0;
      coeff = 0.0;
      u0 = 1.0;
    } else {
      beta = (xs != 0.0) ? -copysign(nrm, xs) : -nrm;
      u0 = xs - beta;
      coeff = (beta - xs) / beta;
    }
    if (b == 0) {  // bookkeeping of the swap (swap_columns, PartialNorms.swap, Permutation.swap) and the pivot
      if (p != s) {
        for (int q = tid; q < t; q += QP_T) {
          const double fs = F[s * QP_NB + q];
          F[p * QP_NB + q] = fs;  // the pivot's row was staged in s_fp by every CTA
          F[s * QP_NB + q] = s_fp[q];
        }
      }
      if (tid == 0) {
        if (p != s) {
          a.u[p] = a.u[s];
          a.uref[p] = a.uref[s];
          const int64_t pf = a.perm[p];
          a.perm[p] = a.perm[s];
          a.perm[s] = pf;
          if (n_swaps < S.swap_cap) {
            a.swaps[2 * n_swaps] = s;
            a.swaps[2 * n_swaps + 1] = p;
          }
        }
        a.u[s] = 0.0;  // downdate_norms: u[:n_s1] = 0
        a.uref[s] = 0.0;
        a.coeffs[s] = coeff;
      }
    }
    if (p != s) ++n_swaps;
    if (n_swaps > S.swap_cap) status = -5;
    for (int64_t r = max(r_lo, s + 1) + tid; r < r_hi; r += QP_T) a.vb[r] = A[r + s * lda] / u0;
    // w_c = v^T A[s:, c] = A[s, c] + (x[s+1:] . A[s+1:, c]) / u0 for the trailing
    // columns and the block's own reflector columns (z)
    // x is staged in shared memory by row chunks (every warp of the CTA streams
    // its columns against it; L1 is mostly carved out for the tile staging).
    // Work items are (column, 2048-row segment) pairs dealt round-robin to the
    // warps, two at a time per warp (two independent 16-byte load streams);
    // each item's dot goes to its own slot wb[col][seg], summed in fixed
    // order in beta (w_c = A[s, c] + sum / u0).
    {
      const double* xcol = A + s * lda;
      const int64_t r1 = s + 1;
      const int64_t ra = (r1 + 1) & ~(int64_t)1;  // first even row >= s+1 (16-byte aligned pairs)
      const int seg = qp_seg_len(m, s);
      const int nseg = qp_nseg(m, s);
      const int spc = max(1, QP_XCH / seg);        // segments per staged x chunk
      const int64_t ncol_a = n - s0 - 1;           // columns [s0, n) except s
      double* xs = qsm;
      for (int sg0 = 0; sg0 < nseg; sg0 += spc) {
        const int nsc = min(spc, nseg - sg0);
        const int64_t rb = ra + (int64_t)sg0 * seg;
        const int nr = (int)max((int64_t)0, min(m, rb + (int64_t)nsc * seg) - rb);
        __syncthreads();
        for (int e = 2 * tid; e < nr; e += 2 * QP_T) {
          if (e + 1 < nr)
            *reinterpret_cast<double2*>(xs + e) = __ldcg(reinterpret_cast<const double2*>(xcol + rb + e));
          else
            xs[e] = __ldcg(xcol + rb + e);
        }
        __syncthreads();
        const int64_t nitems = ncol_a * nsc;
        for (int64_t i0 = gw; i0 < nitems; i0 += 2 * (int64_t)NW) {
          const int64_t i1 = i0 + NW;
          const bool has1 = i1 < nitems;
          const int64_t ci0 = i0 / nsc, ci1 = has1 ? i1 / nsc : ci0;
          const int sq0 = (int)(i0 % nsc), sq1 = has1 ? (int)(i1 % nsc) : 0;
          const int64_t col0 = s0 + ci0 + (s0 + ci0 >= s ? 1 : 0);
          const int64_t col1 = s0 + ci1 + (s0 + ci1 >= s ? 1 : 0);
          const int xo0 = sq0 * seg, xo1 = sq1 * seg;
          const int len0 = max(0, min(seg, nr - xo0)), len1 = has1 ? max(0, min(seg, nr - xo1)) : 0;
          const double* ap0 = A + col0 * lda + rb + xo0;
          const double* ap1 = A + col1 * lda + rb + xo1;
          const double* xp0 = xs + xo0;
          const double* xp1 = xs + xo1;
          double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
          if (lane == 0 && sg0 + sq0 == 0 && ra > r1 && r1 < m) d0 = xcol[r1] * A[r1 + col0 * lda];
          if (has1 && lane == 0 && sg0 + sq1 == 0 && ra > r1 && r1 < m) e0 = xcol[r1] * A[r1 + col1 * lda];
          const int lmax = max(len0, len1);
          for (int r = 2 * lane; r < lmax; r += 4 * 64) {
            double2 av[4], bv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int rr = r + 64 * k;
              av[k] = (rr + 1 < len0) ? ldcs2(ap0 + rr) : make_double2(rr < len0 ? ap0[rr] : 0.0, 0.0);
              bv[k] = (rr + 1 < len1) ? ldcs2(ap1 + rr) : make_double2(rr < len1 ? ap1[rr] : 0.0, 0.0);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int rr = r + 64 * k;
              const double2 xa = (rr + 1 < len0) ? *reinterpret_cast<const double2*>(xp0 + rr)
                                                 : make_double2(rr < len0 ? xp0[rr] : 0.0, 0.0);
              const double2 xb = (rr + 1 < len1) ? *reinterpret_cast<const double2*>(xp1 + rr)
                                                 : make_double2(rr < len1 ? xp1[rr] : 0.0, 0.0);
              d0 = fma(xa.x, av[k].x, d0);
              d1 = fma(xa.y, av[k].y, d1);
              e0 = fma(xb.x, bv[k].x, e0);
              e1 = fma(xb.y, bv[k].y, e1);
            }
          }
          const double dsum = warp_sum(d0 + d1);
          const double esum = warp_sum(e0 + e1);
          if (lane == 0) {
            a.wb[col0 * QP_RMAX + sg0 + sq0] = dsum;
            if (has1) a.wb[col1 * QP_RMAX + sg0 + sq1] = esum;
          }
        }
      }
    }
    gsync();

    // ================= beta =================
    QCLK(3);
    // number of segment slots of this column step (alpha's split)
    const int nseg_b = qp_nseg(m, s);
    for (int q = tid; q < t; q += QP_T) {
      const double ys_ = A[s + (s0 + q) * lda];
      double sum = 0.0;
      for (int g = 0; g < nseg_b; ++g) sum += __ldcg(a.wb + (s0 + q) * QP_RMAX + g);
      s_z[q] = ys_ + sum / u0;
      s_y[q] = ys_;
    }
    __syncthreads();
    {
      double bv = -1.0;
      int bi = 0x7fffffff;
      const double z0 = (lane < t) ? s_z[lane] : 0.0, z1 = (lane + 32 < t) ? s_z[lane + 32] : 0.0;
      const double y0 = (lane < t) ? s_y[lane] : 0.0, y1 = (lane + 32 < t) ? s_y[lane + 32] : 0.0;
      // this warp's columns s+1+gw+k*NW: lane k prefetches column k's scalars
      for (int64_t cb = s + 1 + gw; cb < n; cb += 32 * (int64_t)NW) {
        const int64_t mine = cb + (int64_t)lane * NW;
        double pw = 0.0, pa = 0.0, pu = 0.0, pr = 0.0;
        if (mine < n) {
          pa = A[s + mine * lda];
          double sum = 0.0;
          for (int g = 0; g < nseg_b; ++g) sum += __ldcg(a.wb + mine * QP_RMAX + g);
          pw = pa + sum / u0;
          pu = a.u[mine];
          pr = a.uref[mine];
        }
        const int cnt = (int)min((int64_t)32, (n - cb + NW - 1) / NW);
        double f0n = (lane < t) ? F[cb * QP_NB + lane] : 0.0, f1n = (lane + 32 < t) ? F[cb * QP_NB + lane + 32] : 0.0;
        for (int k = 0; k < cnt; ++k) {
          const int64_t col = cb + (int64_t)k * NW;
          const double f0 = f0n, f1 = f1n;
          if (k + 1 < cnt) {  // next column's F row in flight while this one reduces
            const double* fr = F + (col + NW) * QP_NB;
            f0n = (lane < t) ? fr[lane] : 0.0;
            f1n = (lane + 32 < t) ? fr[lane + 32] : 0.0;
          }
          const double fz = warp_sum(fma(f0, z0, f1 * z1));
          const double fy = warp_sum(fma(f0, y0, f1 * y1));
          if (lane == k) {
            const double fn = coeff * (pw - fz);
            const double R = (pa - fy) - fn;
            F[col * QP_NB + t] = fn;
            A[s + col * lda] = R;
            const double sq = __dsub_rn(__dmul_rn(pu, pu), __dmul_rn(R, R));
            if (sq <= __dmul_rn(1e-2, __dmul_rn(pr, pr))) {
              if (s + 1 < m) {
                a.glist[atomicAdd(&a.cnt[1], 1u)] = (int32_t)col;
              } else {  // fresh norm of an empty column (rows s+1.. do not exist)
                a.u[col] = 0.0;
                a.uref[col] = 0.0;
                am_merge(bv, bi, 0.0, (int)col);
              }
            } else {
              const double nu = sqrt(fmax(sq, 0.0));
              a.u[col] = nu;
              am_merge(bv, bi, nu, (int)col);
            }
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) am_merge(bv, bi, __shfl_xor_sync(0xffffffffu, bv, o), __shfl_xor_sync(0xffffffffu, bi, o));
      if (lane == 0) {
        s_red[wid][0] = bv;
        s_redi[wid] = bi;
      }
    }
    argmax_publish();
    for (int64_t r = max(r_lo, s + 1) + tid; r < r_hi; r += QP_T) A[r + s * lda] = a.vb[r];
    if (s >= r_lo && s < r_hi && tid == 0) A[s + s * lda] = beta;
    if (b == 0 && tid == 0) {
      StepRec rec;
      rec.n_s = s;
      rec.k_selected = 1;
      rec.k_accepted = 1;
      rec.k_max = a.qrp ? 0 : -1;
      rec.broke_early = 0;
      rec.fell_back_to_scalar = a.qrp ? 0 : 1;
      rec.eps_s = 0.0;
      rec.gamma = 1.0;
      a.steps[step_idx] = rec;
    }
    ++step_idx;
    gsync();

    // ================= guard =================
    QCLK(4);
    const int g = (int)__ldcg(a.cnt + 1);
    g_prev = g;
    ++t;
    if (g > 0 && g <= QP_GMAX) {
      // rows (s, m) of this CTA: y = A[r, c] - sum_{t' <= t-1} Y[r, t'] F[c, t'] (Y[:, t-1] = v, now stored)
      double* ys = qsm;                          // [QP_SUB][QP_NB + 1]
      double* fs = qsm + QP_SUB * (QP_NB + 1);   // [QP_GMAX][QP_NB + 1]
      for (int e = tid; e < g * t; e += QP_T) {
        const int gi = e / t, q = e % t;
        fs[gi * (QP_NB + 1) + q] = F[(int64_t)__ldcg(a.glist + gi) * QP_NB + q];
      }
      double gs[QP_GMAX / QP_W], ga[QP_GMAX / QP_W];
#pragma unroll
      for (int k = 0; k < QP_GMAX / QP_W; ++k) gs[k] = ga[k] = 0.0;
      const int64_t rb = max(r_lo, s + 1);
      for (int64_t rs = rb; rs < r_hi; rs += QP_SUB) {
        const int nr = (int)min((int64_t)QP_SUB, r_hi - rs);
        __syncthreads();
        for (int e = tid; e < nr * t; e += QP_T) {
          const int q = e / nr, rr = e % nr;
          ys[rr * (QP_NB + 1) + q] = A[rs + rr + (s0 + q) * lda];
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < QP_GMAX / QP_W; ++k) {
          const int gi = wid + k * QP_W;
          if (gi >= g) break;
          const int64_t col = __ldcg(a.glist + gi);
          for (int rr = lane; rr < nr; rr += 32) {
            double y = A[rs + rr + col * lda];
            const double* yr = ys + rr * (QP_NB + 1);
            const double* fr = fs + gi * (QP_NB + 1);
            for (int q = 0; q < t; ++q) y = fma(-yr[q], fr[q], y);
            gs[k] = fma(y, y, gs[k]);
            ga[k] = fmax(ga[k], fabs(y));
          }
        }
      }
#pragma unroll
      for (int k = 0; k < QP_GMAX / QP_W; ++k) {
        const int gi = wid + k * QP_W;
        if (gi >= g) break;
        const double sv = warp_sum(gs[k]), av = warp_max(ga[k]);
        if (lane == 0) {
          a.gpart[((int64_t)b * QP_GMAX + gi) * 2] = sv;
          a.gpart[((int64_t)b * QP_GMAX + gi) * 2 + 1] = av;
        }
      }
      // the last CTA to arrive reduces (fixed order) and writes u = u_ref = fresh
      __shared__ int s_last;
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        s_last = (atomicAdd(&a.cnt[2], 1u) == (unsigned)G - 1);
      }
      __syncthreads();
      if (s_last) {
        __threadfence();
        for (int gi = wid; gi < g; gi += QP_W) {
          double sv = 0.0, av = 0.0;
          for (int q = lane; q < G; q += 32) {
            sv += __ldcg(a.gpart + ((int64_t)q * QP_GMAX + gi) * 2);
            av = fmax(av, __ldcg(a.gpart + ((int64_t)q * QP_GMAX + gi) * 2 + 1));
          }
          sv = warp_sum(sv);
          av = warp_max(av);
          const int64_t col = __ldcg(a.glist + gi);
          double fresh;
          if (norm_range_ok(av)) {
            fresh = sqrt(sv);
          } else {  // scaled pass over the whole column by this warp (rare)
            int e;
            frexp(av, &e);
            double sc = 0.0;
            for (int64_t r = s + 1 + lane; r < m; r += 32) {
              double y = A[r + col * lda];
              for (int q = 0; q < t; ++q) y = fma(-A[r + (s0 + q) * lda], F[col * QP_NB + q], y);
              y = ldexp(y, -e);
              sc = fma(y, y, sc);
            }
            fresh = ldexp(sqrt(warp_sum(sc)), e);
          }
          if (lane == 0) {
            a.u[col] = fresh;
            a.uref[col] = fresh;
            a.gfresh[gi] = fresh;
          }
        }
        __syncthreads();
        if (tid == 0) {
          a.cnt[2] = 0u;
          a.cnt[1] = 0u;  // every CTA read g before it arrived here
          __threadfence();
          asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(a.cnt + 3), "r"((unsigned)t) : "memory");
        }
      }
      // (no barrier: the next gamma waits for cnt[3] == t)
    } else if (g > QP_GMAX) {
      // too many guards for the in-place recompute: end the block here; they are
      // recomputed from the updated matrix below
    }
  }

  // ================= block end: C -= Y F^T below the block's R rows =================
  const int64_t c0 = s0 + t;
  if (a.dbg && b == 0 && tid == 0) a.dbg[512] = gtimer();
  if (t > 0 && c0 < n && c0 < m) {
    const int64_t ncols = n - c0;
    for (int64_t e = (int64_t)b * QP_T + tid; e < (int64_t)t * ncols; e += (int64_t)G * QP_T) {
      const int64_t q = e / ncols, col = e % ncols;
      a.Wt[q * a.ldz + col] = F[(c0 + col) * QP_NB + q];
    }
    gsync();
    if (a.dbg && b == 0 && tid == 0) a.dbg[513] = gtimer();
    const int64_t mp = m - s0;
    const int odd = (int)(s0 & 1);
    const int64_t ntr = ceil_div(mp + odd, TB_ROWS), ntc = ceil_div(ncols, TB_COLS);
    for (int64_t tile = b; tile < ntr * ntc; tile += G) {
      const int64_t row0 = (tile % ntr) * TB_ROWS - odd, col0 = (tile / ntr) * TB_COLS;
      if (row0 + TB_ROWS <= t) continue;  // R rows only
      __syncthreads();
      trail_b_tile<true>(A, a.Wt, a.ldz, nullptr, s0, m, lda, t, c0, ncols, mp, row0, col0);
    }
    if (a.dbg && b == 0 && tid == 0) a.dbg[514] = gtimer();
    if (exit_reason == 5) {
      gsync();
      // exact norms of the guard columns from the updated rows [c0, m)
      const int g = g_prev;
      for (int gi = gw; gi < g; gi += NW) {
        const int64_t col = __ldcg(a.glist + gi);
        const double* x = A + col * lda;
        double sv = 0.0, av = 0.0;
        for (int64_t r = c0 + lane; r < m; r += 32) {
          const double y = x[r];
          sv = fma(y, y, sv);
          av = fmax(av, fabs(y));
        }
        sv = warp_sum(sv);
        av = warp_max(av);
        double fresh;
        if (norm_range_ok(av)) {
          fresh = sqrt(sv);
        } else {
          int e;
          frexp(av, &e);
          double sc = 0.0;
          for (int64_t r = c0 + lane; r < m; r += 32) {
            const double y = ldexp(x[r], -e);
            sc = fma(y, y, sc);
          }
          fresh = ldexp(sqrt(warp_sum(sc)), e);
        }
        if (lane == 0) {
          a.u[col] = fresh;
          a.uref[col] = fresh;
        }
      }
    }
  } else if (exit_reason == 5) {
    // nothing left to update (c0 >= m or n): the guard columns' norms are of empty rows
    for (int gi = gw; gi < g_prev; gi += NW)
      if (lane == 0) {
        a.u[__ldcg(a.glist + gi)] = 0.0;
        a.uref[__ldcg(a.glist + gi)] = 0.0;
      }
  }
#undef QCLK
  if (b == 0 && tid == 0) {
    c->n_s = (int32_t)c0;
    c->step_idx = step_idx;
    c->n_swaps = n_swaps;
    c->l_acc = 0;
    c->qp_cols = t;
    c->qp_exit = exit_reason;
    if (exit_reason == 5) a.cnt[1] = 0u;
    if (status) {
      c->status = status;
      c->done = 1;
    } else if (exit_reason == 1) {
      c->stopped = 1;
      c->done = 1;
    } else if (exit_reason == 3 || c0 >= kmax) {
      c->done = 1;
    }
  }
}

// After a k_qp3 block (stream order): the optional per-column norm trace and
// the host's poll record.  norm_trace: _record_norm_check (rrqr.py:211-216) for
// a one-column block (trace_norms runs blocks of one, fully updated).
__global__ void k_qp3_post(Ctl* c, double* __restrict__ norm_trace,
                           unsigned long long* __restrict__ trace_bits, HostRec* __restrict__ hrec, int enq) {
  if (threadIdx.x != 0) return;
  if (norm_trace && c->qp_cols > 0) {
    const int idx = c->step_idx - 1;
    norm_trace[idx] = (c->n_s < c->n) ? __longlong_as_double((long long)*trace_bits)
                                      : __longlong_as_double(-1ll);
    *trace_bits = 0ull;
  }
  (void)enq;
  enq = c->posted;  // (device-counted enqueue index, as k_step_end)
  c->posted = enq + 1;
  __threadfence_system();
  // stay in the scalar-pivot engine unless a fallback run ended on the floor test
  const int fb = (c->qp_exit != 2) ? 1 : 0;
  const int flags = (c->done ? 1 : 0) | (fb ? 4 : 0);
  asm volatile("st.volatile.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(hrec + (enq & 1)), "r"(c->n_s),
               "r"(flags), "r"(c->step_idx), "r"(enq + 1)
               : "memory");
}

// trace of a one-column qrp block: max_j |u_j - ||A[n_s:, j]|| | / denom over the
// trailing columns (k_norm_trace's arithmetic, the Ctl's n_s after the block)
__global__ void k_qp3_trace(const Ctl* c, const double* __restrict__ A, const double* __restrict__ u,
                            unsigned long long* __restrict__ out_bits) {
  if (c->qp_cols == 0) return;
  const int64_t n_s1 = c->n_s, n = c->n, m = c->m, lda = c->lda;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const double floor_ = kEps * c->a_max0;
  double worst = 0.0;
  for (int64_t j = n_s1 + w0; j < n; j += nw) {
    const double direct = warp_col_norm(A + j * lda + n_s1, m - n_s1, lane);
    const double den = fmax(fmax(direct, floor_), 2.2250738585072014e-308);
    worst = fmax(worst, fabs(u[j] - direct) / den);
  }
  if (lane == 0 && worst > 0.0) atomicMax(out_bits, (unsigned long long)__double_as_longlong(worst));
}

}  // namespace dmqr
