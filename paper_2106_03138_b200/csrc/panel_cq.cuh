// Householder panel via CholeskyQR2 + Householder reconstruction (cluster kernel).
//
// Produces exactly the reference panel's reflectors (make_reflector sign
// convention, householder.py:57-79), T (= accumulate_wy's W, householder.py:
// 92-114), R and the QRDM2 break (rrqr.py:375-379) -- in exact arithmetic --
// with a handful of cluster-wide phases instead of one all-reduce per
// reflector:
//   G  = P^T P                 (DMMA, cluster reduce-scatter/all-gather in DSMEM)
//   R1 = chol(G), Q1 = P R1^-1 (in place)
//   G2 = Q1^T Q1, R2 = chol(G2), R = R2 R1
//   l  = first j >= 1 with |R_jj| < eps_s (qrdm2 break), else k
//   Q  = Q1 R2^-1 (top l x l block only), modified LU  E - Q S = Y1 U  with
//        S_j = -sign(q'_jj): the same no-cancellation sign choice as
//        beta = -sign(x0)||x||, so Y = [Y1; -(Q_below S) U^-1], T = U Y1^-T,
//        R_H = S R, tau_j = U_jj  (Ballard et al., "Reconstructing Householder
//        vectors from TSQR").
// Rejected columns (after a break) are left untouched in memory; the trailing
// update then starts at n_s + l and applies the l accepted reflectors to them,
// which equals the reference's in-panel rank-1 updates (rrqr.py:366-367).
//
// Safety: CholeskyQR2 is accurate only while pass 1 is well conditioned, so the
// kernel checks every Cholesky pivot (relative to the column's squared norm)
// and the orthogonality of Q1 (|G2 - I|).  An unhealthy pivot is accepted only
// when it proves a QRDM2 break at that column; anything else sets
// Ctl::cq_fail and exits without writing, and the register-resident
// Householder panel (panel_rr.cuh) launched right behind it does the panel.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "panel.cuh"
#include "panel_rr.cuh"

namespace dmqr {

constexpr int CQ_KC = DMQR_MAXK;  // stored slice columns (65)
constexpr int CQ_LDS = 260;       // slice column stride (rows <= 256; 4 mod 16)
constexpr int CQ_RMAX = 256;
constexpr size_t CQ_SMEM =
    sizeof(double) * ((size_t)CQ_KC * CQ_LDS + 2 * DMQR_KP * DMQR_KP + 4 * DMQR_KP);  // ~220 KB

// ---------------------------------------------------------------------------
// CTA-wide small dense helpers (all 512 threads call them), row-major KP x KP
// ---------------------------------------------------------------------------

// rsqrt(d) to full double precision (MUFU estimate + two Newton steps) -- one
// long-latency op per sequential step instead of sqrt + two divisions
__device__ __forceinline__ double cq_rsqrt(double d) {
  double y = rsqrt(d);
  y = y * fma(-0.5 * d * y, y, 1.5);
  return y;
}

// upper Cholesky (A = R^T R) of the leading n x n of A (upper triangle read,
// destroyed); R -> out (upper, zero below).  Returns the first j whose pivot
// fails pivot > tol * orig[j] (or n); piv[j] receives the pivots.
// One barrier per column; the trailing update is warp-per-row over the upper triangle.
__device__ int cq_chol(double* A, double* out, double* piv, const double* orig, int n, double tol) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < DMQR_KP * DMQR_KP; e += blockDim.x) out[e] = 0.0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double d = A[j * DMQR_KP + j];
    if (!(d > tol * orig[j] && d > 0.0)) {
      __syncthreads();
      return j;
    }
    const double rs = cq_rsqrt(d);
    const double rd = rs * rs;
    for (int cc = j + threadIdx.x; cc < n; cc += blockDim.x) out[j * DMQR_KP + cc] = (cc == j) ? d * rs : A[j * DMQR_KP + cc] * rs;
    if (threadIdx.x == 0) piv[j] = d;
    for (int r = j + 1 + wid; r < n; r += nw) {
      const double f = A[j * DMQR_KP + r] * rd;
      for (int cc = r + lane; cc < n; cc += 32) A[r * DMQR_KP + cc] -= f * A[j * DMQR_KP + cc];
    }
    __syncthreads();
  }
  return n;
}

// X = U^-1 for upper triangular U (leading n x n of a KP row-major array);
// X[i][j] is stored at X[i*xr + j*xc].  Blocked by 8: diagonal blocks by
// back substitution (thread per column), then one block diagonal at a time.
__device__ void cq_trinv_upper(const double* U, double* X, int n, int xr = DMQR_KP, int xc = 1) {
  const int nb = (n + 7) / 8;
  __shared__ double rdiag[DMQR_KP];
  __shared__ double tmp[DMQR_KP * 8];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) X[(e / n) * xr + (e % n) * xc] = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) rdiag[i] = 1.0 / U[i * DMQR_KP + i];
  __syncthreads();
  if ((int)threadIdx.x < nb * 8) {
    const int b = threadIdx.x >> 3, cix = threadIdx.x;
    if (cix < n) {
      double xv[8];
      const int i0 = b * 8, nl = cix - i0;  // local column index within the block
#pragma unroll
      for (int q = 0; q < 8; ++q) xv[q] = 0.0;
      xv[nl] = rdiag[cix];
#pragma unroll
      for (int q = 7; q >= 0; --q) {
        if (q >= nl) continue;
        const int i = i0 + q;
        double s = 0.0;
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (t > q && t <= nl) s += U[i * DMQR_KP + i0 + t] * xv[t];
        xv[q] = -s * rdiag[i];
      }
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q <= nl) X[(i0 + q) * xr + cix * xc] = xv[q];
    }
  }
  __syncthreads();
  for (int d = 1; d < nb; ++d) {
    const int nblk = nb - d;
    for (int e = threadIdx.x; e < nblk * 64; e += blockDim.x) {
      const int bi = e >> 6, r = (e >> 3) & 7, cc = e & 7;
      const int i = bi * 8 + r, jj = (bi + d) * 8 + cc;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (i < n && jj < n) {
        int t = (bi + 1) * 8;
        for (; t + 3 <= jj; t += 4) {
          s0 += U[i * DMQR_KP + t] * X[t * xr + jj * xc];
          s1 += U[i * DMQR_KP + t + 1] * X[(t + 1) * xr + jj * xc];
          s2 += U[i * DMQR_KP + t + 2] * X[(t + 2) * xr + jj * xc];
          s3 += U[i * DMQR_KP + t + 3] * X[(t + 3) * xr + jj * xc];
        }
        for (; t <= jj; ++t) s0 += U[i * DMQR_KP + t] * X[t * xr + jj * xc];
      }
      tmp[bi * 64 + r * 8 + cc] = (s0 + s1) + (s2 + s3);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < nblk * 64; e += blockDim.x) {
      const int bi = e >> 6, r = (e >> 3) & 7, cc = e & 7;
      const int i = bi * 8 + r, jj = (bi + d) * 8 + cc;
      if (i < n && jj < n) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int t = bi * 8 + q;
          if (t >= i && t < n) s += X[i * xr + t * xc] * tmp[bi * 64 + q * 8 + cc];
        }
        X[i * xr + jj * xc] = -s;
      }
    }
    __syncthreads();
  }
}

// slice[:, 0:ncol] <- slice[:, 0:kin] * M (M: kin x ncol, KP row-major) in place,
// rows [0, R); each warp owns 8-row tiles (DMMA 8x8x4, accumulators in registers).
__device__ void cq_slice_gemm(double* sl, int R, int kin, int ncol, const double* M) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ks_n = (kin + 3) / 4, nt_n = (ncol + 7) / 8;
  for (int rt = wid; rt * 8 < R; rt += nw) {
    double acc[DMQR_KP / 8][2];
#pragma unroll
    for (int q = 0; q < DMQR_KP / 8; ++q) acc[q][0] = acc[q][1] = 0.0;
    const int r = rt * 8 + (lane >> 2);
    for (int ks = 0; ks < ks_n; ++ks) {
      const int kc = 4 * ks + (lane & 3);
      const double av = (kc < kin) ? sl[kc * CQ_LDS + r] : 0.0;
#pragma unroll
      for (int q = 0; q < DMQR_KP / 8; ++q)
        if (q < nt_n) {
          const int cc = q * 8 + (lane >> 2);
          const double bv = (kc < kin) ? M[kc * DMQR_KP + cc] : 0.0;
          dmma884(acc[q][0], acc[q][1], av, bv);
        }
    }
    __syncwarp();
    const int rr = rt * 8 + (lane >> 2);
#pragma unroll
    for (int q = 0; q < DMQR_KP / 8; ++q)
      if (q < nt_n) {
        const int c0 = q * 8 + 2 * (lane & 3);
        if (c0 < ncol) sl[c0 * CQ_LDS + rr] = acc[q][0];
        if (c0 + 1 < ncol) sl[(c0 + 1) * CQ_LDS + rr] = acc[q][1];
      }
    __syncwarp();
  }
}

// C = A B for n x n upper-triangular A, B given as element loaders (KP padded),
// result -> C (KP row-major, zero below); DMMA over 8x8 tiles, warp per tile.
template <class LA, class LB>
__device__ void cq_small_gemm(LA la, LB lb, double* C, int n) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nt = (n + 7) / 8;
  for (int t = wid; t < nt * nt; t += nw) {
    const int ti = t / nt, tj = t % nt;
    double c0 = 0.0, c1 = 0.0;
    if (tj >= ti)
      for (int ks = ti * 2; ks <= tj * 2 + 1; ++ks) {  // k range of the triangular product
        const int kc = 4 * ks + (lane & 3);
        const int ar = ti * 8 + (lane >> 2), bc = tj * 8 + (lane >> 2);
        const double av = (ar < n && kc < n) ? la(ar, kc) : 0.0;
        const double bv = (kc < n && bc < n) ? lb(kc, bc) : 0.0;
        dmma884(c0, c1, av, bv);
      }
    const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
    C[row * DMQR_KP + col] = (col >= row) ? c0 : 0.0;
    C[row * DMQR_KP + col + 1] = (col + 1 >= row) ? c1 : 0.0;
  }
}

// partial Gram (upper 8x8 tiles) of slice[:, 0:k] over rows [0, R4) -> G (KP row-major);
// each warp interleaves its (<= 3) tiles so the DMMA chains overlap.
__device__ void cq_gram(const double* sl, int R4, int k, double* G) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nt = (k + 7) / 8;
  const int ntiles = nt * (nt + 1) / 2;
  int ci[3], cj[3], tij[3];
  int my = 0;
  for (int t = wid; t < ntiles && my < 3; t += nw, ++my) {
    int ti = 0, rem = t;
    while (rem >= nt - ti) {
      rem -= nt - ti;
      ++ti;
    }
    tij[my] = ti * 16 + ti + rem;
    ci[my] = ti * 8 + (lane >> 2);
    cj[my] = (ti + rem) * 8 + (lane >> 2);
  }
  double acc[3][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  for (int r = (lane & 3); r < R4; r += 4) {
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (q < my) {
        const double av = (ci[q] < k) ? sl[ci[q] * CQ_LDS + r] : 0.0;
        const double bv = (cj[q] < k) ? sl[cj[q] * CQ_LDS + r] : 0.0;
        dmma884(acc[q][0], acc[q][1], av, bv);
      }
  }
#pragma unroll
  for (int q = 0; q < 3; ++q)
    if (q < my) {
      const int ti = tij[q] >> 4, tj = tij[q] & 15;
      const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
      G[row * DMQR_KP + col] = acc[q][0];
      G[row * DMQR_KP + col + 1] = acc[q][1];
    }
}

// cluster all-reduce of the upper triangle of a KP x KP matrix: partial in
// `part` (every rank), total -> `tot` on every rank.  Element e of the upper
// triangle is summed (fixed rank order) by rank e % nranks and pushed to all.
__device__ void cq_cluster_reduce(double* part, double* tot, int k) {
  cg::cluster_group cl = cg::this_cluster();
  const int nr = (int)cl.num_blocks(), me = (int)cl.block_rank();
  cl.sync();
  const int nup = k * (k + 1) / 2;
  for (int e = me + nr * (int)threadIdx.x; e < nup; e += nr * (int)blockDim.x) {
    // e -> (row, col) in the upper triangle, row-major
    int row = 0, rem = e;
    while (rem >= k - row) {
      rem -= k - row;
      ++row;
    }
    const int col = row + rem, off = row * DMQR_KP + col;
    double v[RR_MAXCL];
#pragma unroll
    for (int r = 0; r < RR_MAXCL; ++r) v[r] = (r < nr) ? *cl.map_shared_rank(part + off, r) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int r = 0; r < RR_MAXCL; ++r) s += v[r];
#pragma unroll
    for (int r = 0; r < RR_MAXCL; ++r)
      if (r < nr) *cl.map_shared_rank(tot + off, r) = s;
  }
  cl.sync();
}

__global__ void __launch_bounds__(PANEL_T, 1) k_panel_cq(PanelArgs a) {
  Ctl* c = a.c;
  if (c->done) return;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ __align__(16) double cqs[];
  double* sl = cqs;                              // [CQ_KC][CQ_LDS]
  double* A1 = sl + CQ_KC * CQ_LDS;              // KP x KP
  double* A2 = A1 + DMQR_KP * DMQR_KP;           // KP x KP
  double* vpiv = A2 + DMQR_KP * DMQR_KP;         // [2*KP]: pivots, original diagonal
  double* vS = vpiv + 2 * DMQR_KP;               // [KP]: signs S, then diag(R1)
  double* vD = vS + DMQR_KP;                     // [KP]
  __shared__ int s_flag[4];

  const int tid = threadIdx.x;
  const int me = (int)cl.block_rank(), nr = (int)cl.num_blocks();
  const int64_t n_s = c->n_s, m = c->m, lda = c->lda;
  const int64_t mp = m - n_s;
  const int k = c->k_s;
  const bool brk = c->break_check && c->kind == 0;
  const double eps_s = c->eps_s;
  const int r0 = (int)((int64_t)me * mp / nr), r1 = (int)((int64_t)(me + 1) * mp / nr);
  const int R = r1 - r0, R4 = (R + 3) & ~3;
  double* gA = a.A + n_s * lda + n_s + r0;

  const bool rec = a.dbg && (int)blockIdx.x == min(a.dbg_cta, nr - 1) && tid == 0;
  int ts = 0;
#define CQT() \
  if (rec) a.dbg[ts++] = clock64()
  CQT();
  // ---- P0: slice <- P (rows zero-padded to a multiple of 4) ----
  for (int e = tid; e < k * R4; e += PANEL_T) {
    const int cc = e / R4, rr = e % R4;
    sl[cc * CQ_LDS + rr] = (rr < R) ? gA[(int64_t)cc * lda + rr] : 0.0;
  }
  __syncthreads();
  // ---- P1/P2: G = P^T P ----
  CQT();
  cq_gram(sl, R4, k, A2);
  CQT();
  cq_cluster_reduce(A2, A1, k);
  CQT();
  for (int j = tid; j < k; j += PANEL_T) vpiv[DMQR_KP + j] = A1[j * DMQR_KP + j];
  __syncthreads();
  // ---- P3: R1 = chol(G) -> A2 ----
  const int jstar = cq_chol(A1, A2, vpiv, vpiv + DMQR_KP, k, 1e-10);
  CQT();
  // accepted pass-1 prefix kk = jstar; decide early whether an unhealthy pivot proves a break
  int kk = jstar;
  bool fail = false;
  if (jstar < k) {
    // pivot d ~ R_jj^2 with absolute error ~eps*G_jj: R_jj <= 1e-5 ||a_j|| + noise
    const double bound = 1e-4 * sqrt(vpiv[DMQR_KP + jstar]);
    if (!brk || jstar == 0 || !(bound < eps_s)) fail = true;
  }
  if (!fail && kk > 0) {
    // ---- P4/P5: Q1 = P R1^-1 (in place) ----
    cq_trinv_upper(A2, A1, kk);
    CQT();
    cq_slice_gemm(sl, R4, kk, kk, A1);
    CQT();
    // keep R1: transpose into the lower triangle of A2, diagonal in vD
    __syncthreads();
    for (int e = tid; e < kk * kk; e += PANEL_T) {
      const int i = e / kk, j = e % kk;
      if (i < j) A2[j * DMQR_KP + i] = A2[i * DMQR_KP + j];
      if (i == j) vD[i] = A2[i * DMQR_KP + i];
    }
    __syncthreads();
    // ---- P6/P7: G2 = Q1^T Q1 (partial -> A1, total -> upper A2) ----
    cq_gram(sl, R4, kk, A1);
    // zero the upper of A2 (incl. diag) on this rank first: reduce writes it
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      if (j >= i) A2[e] = 0.0;
    }
    CQT();
    cq_cluster_reduce(A1, A2, kk);
    CQT();
    // orthogonality of Q1: |G2 - I|_max
    if (tid == 0) s_flag[0] = 0;
    __syncthreads();
    for (int e = tid; e < kk * kk; e += PANEL_T) {
      const int i = e / kk, j = e % kk;
      if (j >= i) {
        const double g = A2[i * DMQR_KP + j] - (i == j ? 1.0 : 0.0);
        if (!(fabs(g) < 1e-2)) s_flag[0] = 1;
      }
    }
    for (int j = tid; j < kk; j += PANEL_T) vpiv[DMQR_KP + j] = A2[j * DMQR_KP + j];
    __syncthreads();
    if (s_flag[0]) fail = true;
  }
  int l = kk;
  if (!fail && kk > 0) {
    // ---- P8: R2 = chol(G2) -> A1 (reads/destroys the upper of A2) ----
    if (cq_chol(A2, A1, vpiv, vpiv + DMQR_KP, kk, 1e-6) < kk) fail = true;
    CQT();
  }
  if (!fail && kk > 0) {
    // ---- P9: R = R2 R1 -> slice-free scratch (a.red), then upper A2 ----
    // R1[t][j] lives transposed in the strict lower of A2 (diag in vD); R2 upper in A1
    __syncthreads();
    double* Rg = a.red + 3 * DMQR_KP * DMQR_KP + (size_t)blockIdx.x * DMQR_KP * DMQR_KP;
    cq_small_gemm([&](int i, int t) { return A1[i * DMQR_KP + t]; },
                  [&](int t, int j) { return (t < j) ? A2[j * DMQR_KP + t] : ((t == j) ? vD[j] : 0.0); }, Rg, kk);
    __syncthreads();
    for (int e = tid; e < kk * kk; e += PANEL_T) {
      const int i = e / kk, j = e % kk;
      if (j >= i) A2[i * DMQR_KP + j] = Rg[i * DMQR_KP + j];
    }
    __syncthreads();
  }
  if (!fail) {
    // ---- break: first j >= 1 with |R_jj| < eps_s; an unhealthy pivot at jstar is a break ----
    if (tid == 0) {
      int lb = kk;
      if (brk)
        for (int j = 1; j < kk; ++j)
          if (fabs(A2[j * DMQR_KP + j]) < eps_s) {
            lb = j;
            break;
          }
      s_flag[1] = lb;
    }
    __syncthreads();
    l = s_flag[1];
    if (l == 0) fail = true;
  }
  if (fail) {
    if (me == 0 && tid == 0) c->cq_fail = 1;
    cl.sync();
    return;
  }
  // rank 0 keeps R (rows < l) in global scratch for the final write-back
  if (me == 0)
    for (int e = tid; e < l * l; e += PANEL_T) {
      const int i = e / l, j = e % l;
      a.red[i * DMQR_KP + j] = (j >= i) ? A2[i * DMQR_KP + j] : 0.0;
    }
  // ---- P11/P12: Q = Q1 R2^-1 (first l columns; R2 upper in A1) ----
  __syncthreads();
  CQT();
  cq_trinv_upper(A1, A2, l);
  CQT();
  cq_slice_gemm(sl, R4, l, l, A2);
  CQT();
  __syncthreads();
  // ---- P13/P14 (rank 0): modified LU of the top l x l block of Q ----
  if (me == 0) {
    // A1 <- top block; eliminate in place: strict lower = L (multipliers), upper = q' (unsigned)
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      A1[e] = (i < l && j < l) ? sl[j * CQ_LDS + i] : 0.0;
    }
    __syncthreads();
    {
      const int lane = tid & 31, wid = tid >> 5;
      for (int j = 0; j < l; ++j) {
        const double qjj = A1[j * DMQR_KP + j];
        const double sg = (qjj >= 0.0) ? -1.0 : 1.0;  // S_j = -sign(q'_jj), sign(+0) = +
        const double pv = 1.0 - sg * qjj;             // pivot = 1 + |q'_jj|
        const double f0 = -sg / pv;
        // rows i > j: multiplier L_ij = -S_j q'_ij / pivot, then q'_ic -= L_ij q'_jc (c > j)
        for (int i = j + 1 + wid; i < l; i += PANEL_T / 32) {
          const double Lij = f0 * A1[i * DMQR_KP + j];
          for (int cc = j + 1 + lane; cc < l; cc += 32) A1[i * DMQR_KP + cc] -= Lij * A1[j * DMQR_KP + cc];
          __syncwarp();
          if (lane == 0) A1[i * DMQR_KP + j] = Lij;
        }
        if (tid == 0) {
          vS[j] = sg;
          vpiv[j] = pv;
        }
        __syncthreads();
      }
    }
    // U (upper) -> A2: U_jj = pivot, U_jc = -S_c q'_jc
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      double u = 0.0;
      if (i < l && j < l && j >= i) u = (i == j) ? vpiv[i] : -vS[j] * A1[i * DMQR_KP + j];
      A2[e] = u;
    }
    // keep Y1 (strict lower of A1 = multipliers) for the write-back of rows < l
    for (int e = tid; e < l * l; e += PANEL_T) {
      const int i = e / l, j = e % l;
      if (i > j) a.red[2 * DMQR_KP * DMQR_KP + i * DMQR_KP + j] = A1[i * DMQR_KP + j];
    }
    __syncthreads();
    // Y1^T (unit upper) into the upper of A1
    for (int e = tid; e < l * l; e += PANEL_T) {
      const int i = e / l, j = e % l;
      if (j > i) A1[i * DMQR_KP + j] = A1[j * DMQR_KP + i];
      if (j == i) A1[i * DMQR_KP + i] = 1.0;
    }
    __syncthreads();
    // Z = (Y1^T)^-1 into the (now unused) top l x l block of the slice, Z[i][j] at sl[j*LDS + i]
    cq_trinv_upper(A1, sl, l, 1, CQ_LDS);
    // T = U Z (householder.py accumulate_wy's W), tau_j = U_jj
    cq_small_gemm([&](int i, int t) { return A2[i * DMQR_KP + t]; },
                  [&](int t, int j) { return sl[j * CQ_LDS + t]; }, a.T, l);
    for (int j = tid; j < l; j += PANEL_T) a.coeffs[n_s + j] = vpiv[j];
    __syncthreads();
    // U^-1 -> A1 (upper), broadcast below
    cq_trinv_upper(A2, A1, l);
  }
  cl.sync();
  if (me != 0) {  // pull U^-1 (upper of rank 0's A1) and S from rank 0
    const double* A1r = cl.map_shared_rank(A1, 0);
    const double* vSr = cl.map_shared_rank(vS, 0);
    for (int e = tid; e < l * l; e += PANEL_T) {
      const int i = e / l, j = e % l;
      A1[i * DMQR_KP + j] = (j >= i) ? A1r[i * DMQR_KP + j] : 0.0;
    }
    for (int j = tid; j < l; j += PANEL_T) vS[j] = vSr[j];
  }
  cl.sync();
  // ---- P16: Y = -(Q S) U^-1 on this rank's rows (rank 0's rows < l are fixed below) ----
  for (int e = tid; e < l * R4; e += PANEL_T) {
    const int cc = e / R4, rr = e % R4;
    sl[cc * CQ_LDS + rr] *= -vS[cc];
  }
  __syncthreads();
  CQT();
  cq_slice_gemm(sl, R4, l, l, A1);
  CQT();
  __syncthreads();
  // ---- write back: Y below the diagonal, R_H = S R on and above it (rows < l live on rank 0) ----
  for (int e = tid; e < l * R; e += PANEL_T) {
    const int cc = e / R, rr = e % R;
    const int p = r0 + rr;  // panel row
    double v;
    if (p > cc) {
      if (p < l) {  // Y1 (unit lower) multipliers saved by rank 0
        v = a.red[2 * DMQR_KP * DMQR_KP + p * DMQR_KP + cc];
      } else {
        v = sl[cc * CQ_LDS + rr];
      }
    } else {
      v = vS[p] * a.red[p * DMQR_KP + cc];  // R_H = S R
    }
    gA[(int64_t)cc * lda + rr] = v;
  }
  CQT();
#undef CQT
  if (me == 0 && tid == 0) {
    c->l_acc = l;
    c->broke = (l < k);
    c->cq_fail = 0;
    c->tc0 = (int32_t)(n_s + l);
  }
  cl.sync();
}

}  // namespace dmqr
