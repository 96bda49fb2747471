// Column swaps and the Householder panel (geqr2 + larft analogue).
//   swap_columns / PartialNorms.swap / Permutation.swap  matrix.py:81-87,125-132; rrqr.py:131-133
//   make_reflector        householder.py:57-79 (beta = -sign(x0)||x||, always reflects)
//   apply_reflector_left  householder.py:82-89 (in-panel rank-1 on the selected block only)
//   QRDM2 break           rrqr.py:375-379 (||next column|| < eps_s stops the panel)
//   accumulate_wy         householder.py:92-114 (T = W, upper triangular)
//
// The panel is factored by a cooperatively launched grid: CTAs 0..P-1 each own
// a contiguous slice of panel rows and keep it resident in shared memory for
// the whole panel; CTA P owns no rows and builds T (the reference's W) from
// the reduced z vectors off the critical path.  One grid-wide all-reduction
// per reflector carries the v^T C dots, z = Y^T v, and the three partial sums
// that give the next column's norm by the identity
//     ||x - v w||^2 = a - 2 w b + w^2 c ,
// accepted only without cancellation (>= a/2; else an exact re-reduction),
// written as partials / barrier / fixed-order sum, so every CTA holds bitwise
// identical scalars (beta, coeff, w) without a broadcast.
#pragma once
#include "common.cuh"

namespace dmqr {

// Apply the step's column moves (the composed transposition sequence) to
// full-height columns in one pass: every CTA owns a range of rows, reads the
// sources of all moves on those rows into shared memory, then writes the
// destinations -- moves only exchange columns, so each row range is closed
// under them and needs no global scratch.  u, u_ref, perm (and the look-ahead
// flags) get the same moves in block 0, which owns no rows; the transposition
// log itself is appended verbatim.
// Look-ahead: while the previous step's update is pending, a column's Wt
// column (l rows, indexed from n_s) rides along as extra rows m .. m + l.
constexpr int SWAP_ROWS = 32;                  // rows per CTA (256-byte column segments)
constexpr int SWAP_T = 256;
constexpr int SWAP_MAXMV = 2 * DMQR_KP;        // 144
constexpr size_t SWAP_SMEM = sizeof(double) * SWAP_MAXMV * SWAP_ROWS;  // 36 KB

__global__ void __launch_bounds__(SWAP_T) k_swap(Ctl* c, double* __restrict__ A, double* __restrict__ u,
                                                 double* __restrict__ uref, int64_t* __restrict__ perm,
                                                 int64_t* __restrict__ swaplog, double* __restrict__ Wt, int64_t ldz,
                                                 uint8_t* __restrict__ upd) {
  zshift(c, c, A, u, uref, perm, swaplog, Wt, upd);
  pdl_enter();
  // the move lists are read with the control block snapshot (one round trip)
  __shared__ int s_src[SWAP_MAXMV], s_dst[SWAP_MAXMV];
  const int tid = threadIdx.x;
  int ms_src = 0, ms_dst = 0;
  if (tid < SWAP_MAXMV) {
    ms_src = c->mv_src[tid];
    ms_dst = c->mv_dst[tid];
  }
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 3);
  if (S.done) return;
  const int nmv = S.nmv;
  const int64_t m = S.m, lda = S.lda;
  const bool wt = S.la && S.pend;
  const int64_t nrow = m + (wt ? S.pend_l : 0);
  const int64_t n_s = S.n_s;
  extern __shared__ __align__(16) double sws[];  // [move][row]
  if (tid < SWAP_MAXMV) {
    s_src[tid] = ms_src;
    s_dst[tid] = ms_dst;
  }
  __syncthreads();
  // block 0 owns no rows (the bookkeeping moves below); block b >= 1 owns rows [32 (b-1), 32 b)
  const int64_t r0 = (blockIdx.x == 0) ? nrow : ((int64_t)blockIdx.x - 1) * SWAP_ROWS;
  if (kTMASwap && nmv > 0 && r0 + SWAP_ROWS <= m) {
    // a whole 256-byte segment of every moved column: TMA bulk copies (one
    // lane per move) into shared memory, then bulk stores to the destinations
    // (the row range is closed under the moves: every source is read before
    // any destination is written)
    __shared__ __align__(8) uint64_t s_bar;
    if (tid == 0) mbar_init(&s_bar, 1);
    __syncthreads();
    constexpr unsigned SEG = SWAP_ROWS * sizeof(double);
    if (tid < 32) {
      if (tid == 0) mbar_arrive_expect_tx(&s_bar, SEG * (unsigned)nmv);
      for (int q = tid; q < nmv; q += 32) bulk_g2s(sws + q * SWAP_ROWS, A + (int64_t)s_src[q] * lda + r0, SEG, &s_bar);
      mbar_wait_parity(&s_bar, 0);
      for (int q = tid; q < nmv; q += 32) bulk_s2g(A + (int64_t)s_dst[q] * lda + r0, sws + q * SWAP_ROWS, SEG);
      bulk_commit();
      bulk_wait_read();
    }
  } else if (nmv > 0 && r0 < nrow) {  // the partial last segment and the moved Wt columns
#pragma unroll 9
    for (int e = tid; e < nmv * SWAP_ROWS; e += SWAP_T) {
      const int q = e / SWAP_ROWS, rr = e % SWAP_ROWS;
      const int64_t r = r0 + rr;
      if (r < nrow) {
        const int64_t src = s_src[q];
        sws[e] = (r < m) ? A[src * lda + r] : Wt[(r - m) * ldz + (src - n_s)];
      }
    }
    __syncthreads();
#pragma unroll 9
    for (int e = tid; e < nmv * SWAP_ROWS; e += SWAP_T) {
      const int q = e / SWAP_ROWS, rr = e % SWAP_ROWS;
      const int64_t r = r0 + rr;
      if (r < nrow) {
        const int64_t dst = s_dst[q];
        if (r < m)
          A[dst * lda + r] = sws[e];
        else
          Wt[(r - m) * ldz + (dst - n_s)] = sws[e];
      }
    }
  }
  // the bookkeeping moves run on their own CTA (the host launches one more than
  // the row ranges need), beside the column moves instead of after a range's
  if (blockIdx.x == 0) {
    __shared__ double su[SWAP_MAXMV], sr[SWAP_MAXMV];
    __shared__ int64_t sp[SWAP_MAXMV];
    __shared__ uint8_t sf[SWAP_MAXMV];
    for (int t = tid; t < nmv; t += SWAP_T) {
      const int src = s_src[t];
      su[t] = u[src];
      sr[t] = uref[src];
      sp[t] = perm[src];
      if (wt) sf[t] = upd[src];
    }
    __syncthreads();
    for (int t = tid; t < nmv; t += SWAP_T) {
      const int dst = s_dst[t];
      u[dst] = su[t];
      uref[dst] = sr[t];
      perm[dst] = sp[t];
      if (wt) upd[dst] = sf[t];
    }
    const int nsw = S.nsw, ns0 = S.n_swaps;
    for (int s = tid; s < nsw; s += SWAP_T)
      if (ns0 + s < S.swap_cap) {
        swaplog[2 * (ns0 + s)] = c->sw_a[s];
        swaplog[2 * (ns0 + s) + 1] = c->sw_b[s];
      }
    if (tid == 0) {
      c->n_swaps = ns0 + nsw;
      if (ns0 + nsw > S.swap_cap) {
        c->status = -5;
        c->done = 1;
      }
    }
  }
}

constexpr int PANEL_T = 512;
constexpr int PANEL_W = PANEL_T / 32;
constexpr int RED_LD = DMQR_KP + 8;  // partial-vector stride

struct PanelArgs {
  Ctl* c;
  double* A;
  double* coeffs;
  double* T;     // KP x KP row-major, T[i*KP + j], upper triangular (= reference W)
  double* red;   // [2][gridDim][RED_LD] partials
  int use_smem;  // panel slice resident in shared memory
  int prows;     // CTAs that own rows (gridDim.x - 1 when a T-builder CTA exists, else gridDim.x)
  long long* dbg;  // optional phase clocks of CTA dbg_cta (debug builds of the benchmark only)
  int dbg_cta;
  int only_if_fail;  // Householder fallback behind the CholeskyQR2 panel: run only if it declined
  double* q1g;       // CholeskyQR2 panel: Q1 buffer (chunked panels; read by k_spare under look-ahead)
  int spare;         // look-ahead: release k_spare, publish the Wt factors for k_trail_w
  long long* tline;  // debug timeline (globaltimer at panel end, per step), or null
  // tall CholeskyQR2 panels (m' > cluster x 256 rows, serial schedule): the
  // row passes (G1 = P^T P; Q1 = P R1^-1 and G2 = Q1^T Q1) run on the other SMs
  // in k_panel_helper; the cluster sums their per-chunk partials
  int helpers;
  double* hpart;     // [chunks][KP x KP] per-chunk Gram partials (upper tiles)
  double* hR;        // R1^-1 (KP x KP) + [kk, fail] published by rank 0
  unsigned* hctr;    // [0] G1 items, [1] G1 done, [2] Q1 items, [3] Q1 done, [4] R1^-1 published (step + 1),
                     // [6] / [7] pass 1 / 2 decision (2 use the partials, 1 abandoned)
  long long hwait_ns;  // how long rank 0 waits for the helpers before streaming its own rows
  double* pg;          // look-ahead P-mode: copy of the panel columns P (q1g layout), or null
};

// deterministic all-reduce of `len` doubles across the grid; in: s_part (this
// CTA's partials, smem), out: s_tot (smem).  `it` selects the double buffer.
__device__ __forceinline__ void grid_allreduce(const PanelArgs& a, const double* s_part, double* s_tot, int len,
                                               int it) {
  const int G = gridDim.x;
  if (G == 1) {
    __syncthreads();
    for (int q = threadIdx.x; q < len; q += PANEL_T) s_tot[q] = s_part[q];
    __syncthreads();
    return;
  }
  double* buf = a.red + (int64_t)(it & 1) * G * RED_LD;
  __syncthreads();
  for (int q = threadIdx.x; q < len; q += PANEL_T) buf[(int64_t)blockIdx.x * RED_LD + q] = s_part[q];
  grid_sync_count(&a.c->bar_count, (uint32_t)(it + 1) * (uint32_t)G);
  // 8 threads per slot, fixed association order -> identical result in every CTA
  const int slot = threadIdx.x >> 3, g = threadIdx.x & 7;
  for (int q0 = 0; q0 < len; q0 += PANEL_T / 8) {
    const int q = q0 + slot;
    double s = 0.0;
    if (q < len)
      for (int b = g; b < G; b += 8) s += __ldcg(buf + (int64_t)b * RED_LD + q);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (q < len && g == 0) s_tot[q] = s;
  }
  __syncthreads();
}

// block-level fixed-order sum of per-thread values (PANEL_T threads) into s_part[slot]
__device__ __forceinline__ void block_sum_into(double v, double* wscr, double* dst) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) wscr[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < PANEL_W; ++w) t += wscr[w];
    *dst = t;
  }
}

__global__ void __launch_bounds__(PANEL_T, 1) k_panel(PanelArgs a) {
  pdl_enter();
  Ctl* c = a.c;
  {
    const int done = c->done, cqf = c->cq_fail;  // (the CholeskyQR2 panel may have done the step)
    if (done || (a.only_if_fail && !cqf)) return;
  }
  extern __shared__ __align__(16) double psm[];
  __shared__ double s_part[RED_LD];
  __shared__ double s_tot[RED_LD];
  __shared__ double s_w[PANEL_W][4];
  __shared__ double s_scr[PANEL_W];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n_s = c->n_s, m = c->m, lda = c->lda;
  const int64_t mp = m - n_s;
  const int k = c->k_s;
  const int brk = c->break_check && c->kind == 0;
  const double eps_s = c->eps_s;
  const int P = a.prows;
  const bool tcta = (int)blockIdx.x >= P;  // T builder, owns no rows
  const bool tlocal = (gridDim.x == 1);    // single CTA: builds T itself
  const int64_t r0 = tcta ? mp : (int64_t)blockIdx.x * mp / P;
  const int64_t r1 = tcta ? mp : (int64_t)(blockIdx.x + 1) * mp / P;
  const int64_t R = r1 - r0;

  // element (t, r) of the panel, r panel-relative in [r0, r1): base[t*ld + (r - r0)]
  double* base;
  int64_t ld;
  double* gpanel = a.A + n_s * lda + n_s + r0;
  if (a.use_smem && !tcta) {
    ld = R | 1;  // odd stride spreads columns across banks
    base = psm;
    for (int t = wid; t < k; t += PANEL_W)
      for (int64_t rr = lane; rr < R; rr += 32) base[t * ld + rr] = gpanel[t * lda + rr];
    __syncthreads();
  } else {
    base = gpanel;
    ld = lda;
  }
#define PEL(t, r) base[(int64_t)(t) * ld + ((r) - r0)]
  // T (KP x KP) in shared memory: the T-builder's whole dynamic smem, or after
  // the single CTA's slice (the host sizes the launch for it)
  double* s_T = tcta ? psm : psm + (a.use_smem ? (int64_t)k * ld : 0);

  int l_acc = k;
  int broke = 0;
  int red_it = 0;
  double nrm = 0.0, x0 = 0.0;
  // ---- exact norm of column j over rows >= j (+ x0) as one all-reduce ----
  auto exact_norm = [&](int j) {
    const int64_t rs = max(r0, (int64_t)j);
    double ss = 0.0, am = 0.0, xx = 0.0;
    for (int64_t r = rs + tid; r < r1; r += PANEL_T) {
      const double x = PEL(j, r);
      ss = fma(x, x, ss);
      am = fmax(am, fabs(x));
      if (r == j) xx = x;
    }
    ss = warp_sum(ss);
    am = warp_max(am);
    xx = warp_sum(xx);
    if (lane == 0) {
      s_w[wid][0] = ss;
      s_w[wid][1] = am;
      s_w[wid][2] = xx;
    }
    __syncthreads();
    if (tid == 0) {
      double t0 = 0.0, t1 = 0.0, t2 = 0.0;
      for (int w = 0; w < PANEL_W; ++w) {
        t0 += s_w[w][0];
        t1 = fmax(t1, s_w[w][1]);
        t2 += s_w[w][2];
      }
      s_part[0] = t0;
      s_part[1] = t1;
      s_part[2] = t2;
    }
    grid_allreduce(a, s_part, s_tot, 3, red_it++);
    // s_tot[1] = sum of per-CTA maxima: zero iff the column is zero; an upper
    // bound (<= G x) of max|x| used only to pick an exact 2^-e rescale.
    const double nrm2 = s_tot[0], abound = s_tot[1];
    x0 = s_tot[2];
    if (abound == 0.0) {
      nrm = 0.0;
    } else if (nrm2 > 1e-280 && nrm2 < 1e280) {
      nrm = sqrt(nrm2);
    } else {
      int e;
      frexp(abound, &e);
      double sc = 0.0;
      for (int64_t r = rs + tid; r < r1; r += PANEL_T) {
        const double y = ldexp(PEL(j, r), -e);
        sc = fma(y, y, sc);
      }
      block_sum_into(sc, s_scr, &s_part[0]);
      grid_allreduce(a, s_part, s_tot, 1, red_it++);
      nrm = ldexp(sqrt(s_tot[0]), e);
    }
  };
  exact_norm(0);
  const bool rec = a.dbg && blockIdx.x == (gridDim.x > 1 ? a.dbg_cta : 0) && tid == 0;
#define STAMP(ph) \
  if (rec && j < 64) a.dbg[j * 8 + (ph)] = clock64()
  for (int j = 0; j < k; ++j) {
    STAMP(0);
    // ---- QRDM2 break: residual of the next selected column (rrqr.py:375-379) ----
    if (brk && j > 0 && nrm < eps_s) {
      l_acc = j;
      broke = 1;
      break;
    }
    // ---- reflector (householder.py:57-79) ----
    double beta, coeff, u0;
    if (nrm == 0.0) {
      beta = 0.0;
      coeff = 0.0;
      u0 = 1.0;
    } else {
      beta = (x0 != 0.0) ? -copysign(nrm, x0) : -nrm;
      u0 = x0 - beta;
      coeff = (beta - x0) / beta;
    }
    // local row range [rb, R) of this CTA for rows >= j, and [rb1, R) for rows > j
    const int rb = (int)(max(r0, (int64_t)j) - r0);
    const int rb1 = (int)(max(r0, (int64_t)j + 1) - r0);
    const int Ri = (int)R;
    const bool owner = (j >= r0 && j < r1);
    double* vj = base + (int64_t)j * ld;  // v over local rows; v_j = 1 stored at row j during the update
    if (nrm != 0.0)
      for (int r = rb1 + tid; r < Ri; r += PANEL_T) vj[r] = vj[r] / u0;
    if (owner && tid == 0) vj[j - r0] = 1.0;
    __syncthreads();
    // ---- one all-reduce: d_q = v^T C_q (q > j), z_q = Y_q^T v (q < j), and the
    //      next column's a = ||x||^2, b = v.x, c = ||v||^2 over rows > j ----
    const bool has_next = (j + 1 < k);
    for (int q = wid; q < k; q += PANEL_W) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (q != j) {
        const double* cq = base + (int64_t)q * ld;
        int r = rb + lane;
        for (; r + 96 < Ri; r += 128) {
          s0 = fma(vj[r], cq[r], s0);
          s1 = fma(vj[r + 32], cq[r + 32], s1);
          s2 = fma(vj[r + 64], cq[r + 64], s2);
          s3 = fma(vj[r + 96], cq[r + 96], s3);
        }
        for (; r < Ri; r += 32) s0 = fma(vj[r], cq[r], s0);
      }
      const double sdot = warp_sum((s0 + s1) + (s2 + s3));
      if (lane == 0) s_part[q] = sdot;
    }
    if (has_next) {
      double pa = 0.0, pb = 0.0, pc = 0.0, px = 0.0, pv = 0.0;
      const double* cn = base + (int64_t)(j + 1) * ld;
      for (int r = rb1 + tid; r < Ri; r += PANEL_T) {
        const double x = cn[r], v = vj[r];
        pa = fma(x, x, pa);
        pb = fma(v, x, pb);
        pc = fma(v, v, pc);
        if (r + r0 == j + 1) {
          px = x;
          pv = v;
        }
      }
      pa = warp_sum(pa);
      pb = warp_sum(pb);
      pc = warp_sum(pc);
      px = warp_sum(px);
      pv = warp_sum(pv);
      __shared__ double s_abc[PANEL_W][5];
      if (lane == 0) {
        s_abc[wid][0] = pa;
        s_abc[wid][1] = pb;
        s_abc[wid][2] = pc;
        s_abc[wid][3] = px;
        s_abc[wid][4] = pv;
      }
      __syncthreads();
      if (tid < 5) {
        double t = 0.0;
        for (int w = 0; w < PANEL_W; ++w) t += s_abc[w][tid];
        s_part[k + tid] = t;
      }
    }
    STAMP(1);
    grid_allreduce(a, s_part, s_tot, k + (has_next ? 5 : 0), red_it++);
    STAMP(2);
    // ---- rank-1 update of the rest of the selected block (householder.py:88-89) ----
    if (coeff != 0.0 && !tcta) {
      for (int q = j + 1 + wid; q < k; q += PANEL_W) {
        const double w = coeff * s_tot[q];
        double* cq = base + (int64_t)q * ld;
        int r = rb + lane;
        for (; r + 96 < Ri; r += 128) {
          cq[r] = fma(-vj[r], w, cq[r]);
          cq[r + 32] = fma(-vj[r + 32], w, cq[r + 32]);
          cq[r + 64] = fma(-vj[r + 64], w, cq[r + 64]);
          cq[r + 96] = fma(-vj[r + 96], w, cq[r + 96]);
        }
        for (; r < Ri; r += 32) cq[r] = fma(-vj[r], w, cq[r]);
      }
    }
    STAMP(3);
    // ---- T column j (householder.py:109-113), on the T-builder CTA, in smem ----
    if (tcta || tlocal) {
      for (int i = wid; i < j; i += PANEL_W) {
        double sacc = 0.0;
        for (int q = i + lane; q < j; q += 32) sacc = fma(s_T[i * DMQR_KP + q], s_tot[q], sacc);
        sacc = warp_sum(sacc);
        if (lane == 0) s_T[i * DMQR_KP + j] = -coeff * sacc;
      }
      if (tid == 0) {
        s_T[j * DMQR_KP + j] = coeff;
        a.coeffs[n_s + j] = coeff;
      }
    }
    STAMP(4);
    // ---- next column's norm ----
    if (has_next) {
      const double w = coeff * s_tot[j + 1];
      const double pa = s_tot[k], pb = s_tot[k + 1], pc = s_tot[k + 2];
      const double nx = fma(-s_tot[k + 4], w, s_tot[k + 3]);
      const double nn2 = (coeff != 0.0) ? pa - 2.0 * w * pb + w * w * pc : pa;
      __syncthreads();
      if (nn2 >= 0.5 * pa && pa > 1e-280 && pa < 1e280) {
        nrm = sqrt(nn2);
        x0 = nx;
      } else {
        exact_norm(j + 1);  // cancellation (or range): recompute from the updated column
      }
    }
    __syncthreads();
    if (owner && tid == 0) vj[j - r0] = beta;  // diagonal of R (after every reader of v_j = 1)
    STAMP(5);
  }
#undef PEL
#undef STAMP
  if (a.use_smem && !tcta) {
    __syncthreads();
    for (int t = wid; t < k; t += PANEL_W)
      for (int64_t rr = lane; rr < R; rr += 32) gpanel[t * lda + rr] = base[t * ld + rr];
  }
  if (tcta || tlocal) {
    __syncthreads();
    for (int e = tid; e < l_acc * l_acc; e += PANEL_T) {
      const int i = e / l_acc, jj = e % l_acc;
      if (i <= jj) a.T[i * DMQR_KP + jj] = s_T[i * DMQR_KP + jj];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    c->l_acc = l_acc;
    c->broke = broke;
    c->tc0 = (int32_t)(n_s + k);
  }
}

}  // namespace dmqr
