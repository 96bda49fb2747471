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
// and the orthogonality of Q1 (|G2 - I|), see CQ_PIVOT_TOL / CQ_ORTH_TOL.  An unhealthy pivot is accepted only
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
// Health limits.  Q1 = P R1^-1 goes through an explicit triangular inverse, so
// its residual |P - Q1 R1| grows like cond(R1) eps: a panel whose pass-1
// pivots fall below CQ_PIVOT_TOL of the column's squared norm, or whose pass-1
// Q1 is off orthogonal by CQ_ORTH_TOL (~cond^2 eps, i.e. cond > ~7e3), goes to
// the Householder panel instead.
constexpr double CQ_PIVOT_TOL = 1e-7;
constexpr double CQ_ORTH_TOL = 1e-8;
// |G2 - I| at or below this: pass-2 factors by a two-term expansion (see P8')
constexpr double CQ_NEAR_ID = 1e-10;
constexpr size_t CQ_SMEM =
    sizeof(double) * ((size_t)CQ_KC * CQ_LDS + 2 * DMQR_KP * DMQR_KP + 4 * DMQR_KP);  // ~220 KB

// ---------------------------------------------------------------------------
// CTA-wide small dense helpers (all 512 threads call them), row-major KP x KP
// ---------------------------------------------------------------------------

// rsqrt(d) to full double precision: MUFU estimate (rsqrt.approx.f64, ~23
// bits) + two Newton steps -- the Cholesky pivot chain's one long-latency op
__device__ __forceinline__ double cq_rsqrt(double d) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  const double hd = 0.5 * d;
  y = y * fma(-hd * y, y, 1.5);
  y = y * fma(-hd * y, y, 1.5);
  return y;
}

// phase ticks of the small helpers (tools/micro/cq_small.cu defines them)
#ifndef CQ_TICK
#define CQ_TICK(i)
#endif

// upper Cholesky (A = R^T R) of the leading n x n of A (upper triangle read,
// destroyed); R -> out (upper, zero below).  Returns the first j whose pivot
// fails pivot > tol * orig[j] (or n); piv[j] receives the pivots.  On a failure
// at j the leading j x j of R is complete.
// Blocked by 8 (right-looking): warp 0 factors the 8-row block row (lane =
// column, 3 columns per lane, shuffles for the block's pivot row), then all
// warps apply the rank-8 update to the trailing upper triangle on DMMA.
__device__ int cq_chol(double* A, double* out, double* piv, const double* orig, int n, double tol) {
  __shared__ int s_fail;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int nbk = (n + 7) / 8;
  for (int e = tid; e < DMQR_KP * DMQR_KP; e += blockDim.x) out[e] = 0.0;
  if (tid == 0) s_fail = n;
  __syncthreads();
  auto warp_rowblock = [&](int b0) {
    const int bw = min(8, n - b0);
    {
      // every lane: the 8 x 8 diagonal block (upper); lane: 2 columns right of it
      double D[8][8], a[2][8];
      // (unconditional loads from clamped in-bounds addresses, then select:
      // predicated shared loads cost an address rebuild each)
      const double* Ab = A + b0 * DMQR_KP + b0;
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = r; c < 8; ++c) {
          const double v = Ab[r * DMQR_KP + c];
          D[r][c] = (c < bw) ? v : 0.0;
        }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int c = b0 + 8 + lane + 32 * s;
        const double* Ac = A + b0 * DMQR_KP + min(c, DMQR_KP - 1);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const double v = Ac[r * DMQR_KP];
          a[s][r] = (c < n && r < bw) ? v : 0.0;
        }
      }
      double thr[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) thr[j] = tol * orig[min(b0 + j, DMQR_KP - 1)];
      // branch-free: after the first failing pivot the block is garbage but
      // only the leading fail x fail of R is used
      int fail = n;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < bw) {
          const double d = D[j][j];
          if (fail == n && !(d > thr[j] && d > 0.0)) fail = b0 + j;
          {
            const double rs = cq_rsqrt(d);
            double rd[8];
#pragma unroll
            for (int c = j + 1; c < 8; ++c) rd[c] = D[j][c] * rs;  // R[b0+j][b0+c]
#pragma unroll
            for (int r = j + 1; r < 8; ++r)
#pragma unroll
              for (int c = r; c < 8; ++c) D[r][c] -= rd[r] * rd[c];
            double x[2];
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              x[s] = a[s][j] * rs;
#pragma unroll
              for (int r = j + 1; r < 8; ++r) a[s][r] -= rd[r] * x[s];
            }
            if (lane == 0) {
              piv[b0 + j] = d;
              out[(b0 + j) * DMQR_KP + b0 + j] = d * rs;
#pragma unroll
              for (int c = j + 1; c < 8; ++c)
                if (c < bw) out[(b0 + j) * DMQR_KP + b0 + c] = rd[c];
            }
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const int c = b0 + 8 + lane + 32 * s;
              if (c < n) out[(b0 + j) * DMQR_KP + c] = x[s];
            }
          }
        }
      }
      if (lane == 0) s_fail = fail;
    }
  };
  // A[tile ri][tile cj] -= R[pb0 .. pb0+8)[rows]^T R[pb0 .. pb0+8)[cols] for the
  // tiles tile_of(t), t < ntl, on warps w0, w0 + ws, ... (3 interleaved per warp)
  auto syrk_tiles = [&](int pb0, auto tile_of, int ntl, int w0, int ws) {
    const int lr = lane >> 2, lk = lane & 3;
    for (int t0 = wid - w0; t0 < ntl; t0 += 3 * ws) {
      if (t0 < 0) break;
      int ri[3], cj[3];
      double x[3][2];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int t = t0 + q * ws;
        int ti = -1, tj = 0;
        if (t < ntl) tile_of(t, ti, tj);
        ri[q] = ti < 0 ? -1 : ti * 8;
        cj[q] = tj * 8;
        x[q][0] = x[q][1] = 0.0;
      }
#pragma unroll
      for (int k0 = 0; k0 < 8; k0 += 4) {
        const int kr = (pb0 + k0 + lk) * DMQR_KP;
#pragma unroll
        for (int q = 0; q < 3; ++q)
          if (ri[q] >= 0) dmma884(x[q][0], x[q][1], out[kr + ri[q] + lr], out[kr + cj[q] + lr]);
      }
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (ri[q] >= 0) {
          const int r = ri[q] + lr, oc = cj[q] + 2 * lk;
          if (r < n && oc < n) A[r * DMQR_KP + oc] -= x[q][0];
          if (r < n && oc + 1 < n) A[r * DMQR_KP + oc + 1] -= x[q][1];
        }
    }
  };
  // Look-ahead: warp 0 factors block row b while the other warps finish block
  // b-1's trailing update past block row b+1; then all warps bring block row
  // b+1 up to date with block b.
  for (int b = 0; b < nbk; ++b) {
    const int b0 = b * 8;
    if (wid == 0) {
      warp_rowblock(b0);
    } else if (b > 0) {
      const int tb = b + 1, nr = nbk - tb;  // upper tiles (ri, cj), tb <= ri <= cj
      if (nr > 0)
        syrk_tiles(b0 - 8, [&](int t, int& ti, int& tj) {
          int r = 0;
          while (t >= nr - r) { t -= nr - r; ++r; }
          ti = tb + r; tj = tb + r + t;
        }, nr * (nr + 1) / 2, 1, nw - 1);
    }
    __syncthreads();
    CQ_TICK(0);
    if (s_fail < n) return s_fail;
    if (b + 1 < nbk) {  // block row b+1 with block b
      const int tb = b + 1, nr = nbk - tb;
      syrk_tiles(b0, [&](int t, int& ti, int& tj) { ti = tb; tj = tb + t; }, nr, 0, nw);
    }
    __syncthreads();
    CQ_TICK(1);
  }
  return n;
}

// X = U^-1 for upper triangular U (leading n x n of a KP row-major array);
// X[i][j] is stored at X[i*xr + j*xc].  Blocked by 8: diagonal blocks by back
// substitution (thread per column), then one block diagonal at a time, each
// off-diagonal block X_ij = -X_ii (sum_t U_it X_tj) by one warp on DMMA.
__device__ void cq_trinv_upper(const double* U, double* X, int n, int xr = DMQR_KP, int xc = 1) {
  const int nb = (n + 7) / 8;
  __shared__ double rdiag[DMQR_KP];
  __shared__ double wst[PANEL_T / 32][64];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) X[(e / n) * xr + (e % n) * xc] = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) rdiag[i] = 1.0 / U[i * DMQR_KP + i];
  __syncthreads();
  if ((int)threadIdx.x < nb * 8) {
    const int b = threadIdx.x >> 3, cix = threadIdx.x;
    if (cix < n) {
      double xv[8];
      const int i0 = b * 8, nl = cix - i0;  // local column index within the block
#pragma unroll
      for (int q = 0; q < 8; ++q) xv[q] = (q == nl) ? rdiag[cix] : 0.0;
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
  CQ_TICK(2);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int lr = lane >> 2, lk = lane & 3;
  double* w = wst[wid];
  for (int d = 1; d < nb; ++d) {
    for (int bi = wid; bi < nb - d; bi += nw) {
      const int bj = bi + d;
      const int ar = bi * 8 + lr, bc = bj * 8 + lr;
      // (four partial sums over alternating k-steps: the dependent DMMA chain of a far diagonal --
      // up to 16 k-steps -- is a quarter as long)
      double cp[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      for (int t0 = (bi + 1) * 8; t0 < (bj + 1) * 8; t0 += 16) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int t = t0 + 4 * h + lk;
          if (t0 + 4 * h < (bj + 1) * 8) {
            const double av = (ar < n && t < n) ? U[ar * DMQR_KP + t] : 0.0;
            const double bv = (t < n && bc < n) ? X[t * xr + bc * xc] : 0.0;
            dmma884(cp[h][0], cp[h][1], av, bv);
          }
        }
      }
      const double c0 = (cp[0][0] + cp[1][0]) + (cp[2][0] + cp[3][0]);
      const double c1 = (cp[0][1] + cp[1][1]) + (cp[2][1] + cp[3][1]);
      w[lr * 8 + 2 * lk] = c0;
      w[lr * 8 + 2 * lk + 1] = c1;
      __syncwarp();
      double e0 = 0.0, e1 = 0.0;
#pragma unroll
      for (int k0 = 0; k0 < 8; k0 += 4) {
        const int kc = bi * 8 + k0 + lk;
        const double av = (ar < n && kc < n) ? X[ar * xr + kc * xc] : 0.0;
        dmma884(e0, e1, av, w[(k0 + lk) * 8 + lr]);
      }
      const int oc = bj * 8 + 2 * lk;
      if (ar < n && oc < n) X[ar * xr + oc * xc] = -e0;
      if (ar < n && oc + 1 < n) X[ar * xr + (oc + 1) * xc] = -e1;
      __syncwarp();
    }
    __syncthreads();
  }
  CQ_TICK(3);
}

// In place X <- X U^-1 for upper triangular U (leading n x n of a KP
// row-major array; UNIT: unit diagonal, not read): solves X U = B for X.
// X[i][j] at X[i*xr + j*xc].  Blocked by 8 columns: the block column takes the
// update from the columns left of it on DMMA (warp per 8-row tile), then each
// row solves its 8 x 8 triangle (thread per row) -- no inverse, no scratch.
template <bool UNIT>
__device__ void cq_trsm_right_upper(double* X, const double* U, int n, int xr, int xc) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int nb = (n + 7) / 8, lr = lane >> 2, lk = lane & 3;
  __shared__ double s_rd[DMQR_KP];
  if (!UNIT)
    for (int i = tid; i < n; i += blockDim.x) s_rd[i] = 1.0 / U[i * DMQR_KP + i];
  __syncthreads();
  for (int J = 0; J < nb; ++J) {
    const int c0 = J * 8;
    if (J > 0)
      for (int rt = wid; rt < nb; rt += nw) {  // X[:, J] -= X[:, <J] U[<J, J]
        const int r = rt * 8 + lr;
        double a0 = 0.0, a1 = 0.0;
        for (int k0 = 0; k0 < c0; k0 += 4) {
          const int k = k0 + lk;
          const double av = (r < n) ? X[r * xr + k * xc] : 0.0;
          const int cc = c0 + lr;
          const double bv = (cc < n) ? U[k * DMQR_KP + cc] : 0.0;
          dmma884(a0, a1, av, bv);
        }
        const int oc = c0 + 2 * lk;
        if (r < n && oc < n) X[r * xr + oc * xc] -= a0;
        if (r < n && oc + 1 < n) X[r * xr + (oc + 1) * xc] -= a1;
      }
    __syncthreads();
    for (int r = tid; r < n; r += blockDim.x) {  // the 8 x 8 triangle, row r
      double x[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int cj = c0 + j;
        if (cj < n) {
          double b = X[r * xr + cj * xc];
#pragma unroll
          for (int t = 0; t < j; ++t) b -= x[t] * U[(c0 + t) * DMQR_KP + cj];
          x[j] = UNIT ? b : b * s_rd[cj];
          X[r * xr + cj * xc] = x[j];
        } else {
          x[j] = 0.0;
        }
      }
    }
    __syncthreads();
  }
}

// 1/x for x in [1, 2] (modified-LU pivots): MUFU estimate + two Newton steps
__device__ __forceinline__ double cq_rcp12(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

// Modified LU (Ballard et al.) of the leading l x l of A (KP row-major), in
// place: strict lower <- multipliers L_ij = -S_j q'_ij / (1 + |q'_jj|), upper
// <- the eliminated q' (unsigned); S_j = -sign(q'_jj) -> vS, pivots -> vpiv.
// Blocked by 8: warp 0 eliminates the 8-column block over all rows below
// (lane = row, 3 rows per lane) and, in the same pass, the block's 8 rows over
// the columns to its right (lane = column, 2 per lane); then all warps apply
// the rank-8 update to the trailing block on DMMA.
__device__ void cq_mlu(double* A, double* vS, double* vpiv, int l) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int nbk = (l + 7) / 8;
  auto warp_panel = [&](int b0) {
    const int bw = min(8, l - b0);
    const int c0 = b0 + 8;
    {
      double v[3][8];  // rows b0 + lane + 32 s, block columns
      double w[2][8];  // block rows, columns c0 + lane + 32 s
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int i = b0 + lane + 32 * s;
        const double* Ai = A + min(i, DMQR_KP - 1) * DMQR_KP + b0;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const double x = Ai[c];
          v[s][c] = (i < l && c < bw) ? x : 0.0;
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int c = c0 + lane + 32 * s;
        const double* Ac = A + b0 * DMQR_KP + min(c, DMQR_KP - 1);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          const double x = Ac[r * DMQR_KP];
          w[s][r] = (c < l && r < bw) ? x : 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < bw) {
          double qj[8];
#pragma unroll
          for (int c = j; c < 8; ++c) qj[c] = __shfl_sync(0xffffffffu, v[0][c], j);  // row b0+j
          const double qjj = qj[j];
          const double sg = (qjj >= 0.0) ? -1.0 : 1.0;  // S_j = -sign(q'_jj), sign(+0) = +
          const double pv = 1.0 - sg * qjj;             // pivot = 1 + |q'_jj|
          const double f0 = -sg * cq_rcp12(pv);
          // rows i > b0 + j: multiplier and elimination; rows at or above
          // the pivot (slot 0 only) get L = 0, which leaves them unchanged
          // (branch-free; rows past l hold zeros and are never stored)
#pragma unroll
          for (int s = 0; s < 3; ++s) {
            const bool below = (s > 0) || (lane > j);
            const double L = below ? f0 * v[s][j] : 0.0;
#pragma unroll
            for (int c = j + 1; c < 8; ++c) v[s][c] = fma(-L, qj[c], v[s][c]);
            v[s][j] = below ? L : v[s][j];
          }
          // block rows i > j, columns right of the block: q'_ic -= L_ij q'_jc
#pragma unroll
          for (int i = j + 1; i < 8; ++i) {
            const double Lij = __shfl_sync(0xffffffffu, v[0][j], i);  // row b0+i lives on lane i
#pragma unroll
            for (int s = 0; s < 2; ++s) w[s][i] -= Lij * w[s][j];
          }
          if (lane == 0) {
            vS[b0 + j] = sg;
            vpiv[b0 + j] = pv;
          }
        }
      }
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        const int i = b0 + lane + 32 * s;
        if (i < l) {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            if (c < bw) A[i * DMQR_KP + b0 + c] = v[s][c];
        }
      }
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int c = c0 + lane + 32 * s;
        if (c < l) {
#pragma unroll
          for (int r = 1; r < 8; ++r)
            if (r < bw) A[(b0 + r) * DMQR_KP + c] = w[s][r];
        }
      }
    }
  };
  // A[tile rt][tile ct] -= L[rows][pb0 .. pb0+8) q'[pb0 .. pb0+8)[cols] for the
  // tiles tile_of(t), t < ntl, spread over warps w0, w0 + ws, ...
  auto upd_tiles = [&](int pb0, auto tile_of, int ntl, int w0, int ws) {
    const int lr = lane >> 2, lk = lane & 3;
    for (int t0 = wid - w0; t0 < ntl; t0 += 4 * ws) {
      if (t0 < 0) break;
      int ti[4], tj[4];
      double x[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = t0 + q * ws;
        ti[q] = -1;
        tj[q] = 0;
        if (t < ntl) tile_of(t, ti[q], tj[q]);
        x[q][0] = x[q][1] = 0.0;
      }
#pragma unroll
      for (int k0 = 0; k0 < 8; k0 += 4) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (ti[q] >= 0) {
            const int r = min(ti[q] * 8 + lr, DMQR_KP - 1), cc = min(tj[q] * 8 + lr, DMQR_KP - 1);
            dmma884(x[q][0], x[q][1], A[r * DMQR_KP + pb0 + k0 + lk], A[(pb0 + k0 + lk) * DMQR_KP + cc]);
          }
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (ti[q] >= 0) {
          const int r = ti[q] * 8 + lr, oc = tj[q] * 8 + 2 * lk;
          if (r < l && oc < l) A[r * DMQR_KP + oc] -= x[q][0];
          if (r < l && oc + 1 < l) A[r * DMQR_KP + oc + 1] -= x[q][1];
        }
    }
  };
  // Look-ahead over the 8-column blocks: warp 0 eliminates block b while the
  // other warps finish block b-1's trailing update (rows and columns past
  // block b -- disjoint from block b's column and row); then all warps bring
  // block b+1's column and row up to date with block b.
  for (int b = 0; b < nbk; ++b) {
    const int b0 = b * 8;
    if (wid == 0) {
      warp_panel(b0);
    } else if (b > 0) {
      const int pb0 = b0 - 8, tb = b + 1, nr = nbk - tb;  // rest of block b-1: tiles >= (b+1, b+1)
      if (nr > 0)
        upd_tiles(pb0, [&](int t, int& ri, int& ci) { ri = tb + t / nr; ci = tb + t % nr; }, nr * nr, 1, nw - 1);
    }
    __syncthreads();
    CQ_TICK(4);
    if (b + 1 < nbk) {  // block b+1's column (rows >= b0+8) and row (columns >= b0+16) with block b
      const int tb = b + 1, nr = nbk - tb;
      upd_tiles(b0, [&](int t, int& ri, int& ci) {
        if (t < nr) { ri = tb + t; ci = tb; } else { ri = tb; ci = tb + 1 + (t - nr); }
      }, nr + (nr - 1), 0, nw);
    }
    __syncthreads();
    CQ_TICK(5);
  }
}

// slice[:, 0:ncol] <- slice[:, 0:kin] * M (M: kin x ncol upper triangular, KP row-major) in place,
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
        if (q < nt_n && 4 * ks < 8 * (q + 1)) {  // M upper triangular: rows > 8q+7 are zero
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

// C = A B for n x n upper-triangular B and upper-triangular (or, AFULL, full) A
// given as element loaders (KP padded), result -> C (KP row-major; zero below
// unless AFULL); DMMA over 8x8 tiles, warp per tile.
template <bool AFULL = false, class LA, class LB>
__device__ void cq_small_gemm(LA la, LB lb, double* C, int n) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nt = (n + 7) / 8;
  // (running a warp's tiles together -- interleaved chains -- measured slower: the loop is bound by
  // the loaders' address arithmetic, not by the DMMA chain)
  for (int t = wid; t < nt * nt; t += nw) {
    const int ti = t / nt, tj = t % nt;
    double c0 = 0.0, c1 = 0.0;
    if (AFULL || tj >= ti)
      for (int ks = AFULL ? 0 : ti * 2; ks <= tj * 2 + 1; ++ks) {  // k range of the triangular product
        const int kc = 4 * ks + (lane & 3);
        const int ar = ti * 8 + (lane >> 2), bc = tj * 8 + (lane >> 2);
        const double av = (ar < n && kc < n) ? la(ar, kc) : 0.0;
        const double bv = (kc < n && bc < n) ? lb(kc, bc) : 0.0;
        dmma884(c0, c1, av, bv);
      }
    const int row = ti * 8 + (lane >> 2), col = tj * 8 + 2 * (lane & 3);
    C[row * DMQR_KP + col] = (AFULL || col >= row) ? c0 : 0.0;
    C[row * DMQR_KP + col + 1] = (AFULL || col + 1 >= row) ? c1 : 0.0;
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

// 32-bit shared::cluster address of p in rank `rank`'s shared memory
__device__ __forceinline__ uint32_t dsmem_addr(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ double2 ld_dsmem2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_dsmem(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_dsmem2(uint32_t a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

// cluster all-reduce of the upper triangle of a KP x KP matrix: partial in
// `part` (every rank), total -> `tot` on every rank (entries j >= i only; the
// strict lower of `tot` is left alone).  The upper 8x8 tiles are cut into
// element pairs, split evenly over the ranks; each pair is summed in fixed
// rank order by its rank (16-byte DSMEM loads) and pushed to every rank.
__device__ void cq_cluster_reduce(double* part, double* tot, int k) {
  cg::cluster_group cl = cg::this_cluster();
  const int nr = (int)cl.num_blocks(), me = (int)cl.block_rank();
  const int nt = (k + 7) / 8, npair = nt * (nt + 1) / 2 * 32;
  const int p0 = me * npair / nr, p1 = (me + 1) * npair / nr;
  cl.sync();
  for (int p = p0 + (int)threadIdx.x; p < p1; p += blockDim.x) {
    int t = p >> 5, ti = 0;
    while (t >= nt - ti) {  // upper tiles, row-major
      t -= nt - ti;
      ++ti;
    }
    const int tj = ti + t, w = p & 31;
    const int r = ti * 8 + (w >> 2), c = tj * 8 + 2 * (w & 3);
    const int off = r * DMQR_KP + c;
    double2 v[RR_MAXCL];
#pragma unroll
    for (int q = 0; q < RR_MAXCL; ++q) v[q] = (q < nr) ? ld_dsmem2(dsmem_addr(part + off, q)) : make_double2(0.0, 0.0);
    double2 sum = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < RR_MAXCL; ++q) {
      sum.x += v[q].x;
      sum.y += v[q].y;
    }
    const bool full = ti != tj || c >= r;  // both entries on or above the diagonal
    const bool hi = c + 1 == r;            // only the second one (the diagonal)
#pragma unroll
    for (int q = 0; q < RR_MAXCL; ++q)
      if (q < nr) {
        const uint32_t a = dsmem_addr(tot + off, q);
        if (full) {
          st_dsmem2(a, sum);
        } else if (hi) {
          st_dsmem(a + 8, sum.y);
        }
      }
  }
  cl.sync();
}

__global__ void __launch_bounds__(PANEL_T, 1) k_panel_cq(PanelArgs a) {
  zshift(a.c, a.c, a.A, a.coeffs, a.T, a.red, a.q1g, a.hpart, a.hR, a.hctr, a.pg);
  // wait for the step's column swaps, then let the look-ahead grid behind this
  // one start (trailing.cuh: it runs beside the panel and must see the swaps)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  Ctl* c = a.c;
  const long long t_start = gtimer();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 4);
  if (S.done) return;
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
  const int64_t n_s = S.n_s, m = S.m, lda = S.lda;
  const int64_t mp = m - n_s;
  const int k = S.k_s;
  const bool brk = S.break_check && S.kind == 0;
  const double eps_s = c->eps_s;
  const int r0 = (int)((int64_t)me * mp / nr), r1 = (int)((int64_t)(me + 1) * mp / nr);
  const int R = r1 - r0, R4 = (R + 3) & ~3;
  double* gA = a.A + n_s * lda + n_s + r0;

  const bool rec = a.dbg && (int)blockIdx.x == min(a.dbg_cta, nr - 1) && tid == 0;
  int ts = 0;
#define CQT() \
  if (rec) a.dbg[ts++] = clock64()
#define FCQT(i) \
  if (rec) a.dbg[32 + (i)] = clock64()
  CQT();
  // Rows per CTA beyond CQ_RMAX (m' > 16 x 256): the slice streams through
  // shared memory in chunks of CQ_RMAX rows; Q1 then lives in the published
  // buffer (q1g) and each pass over the rows reloads its chunks.
  const int nch = (R + CQ_RMAX - 1) / CQ_RMAX;
  const bool chunked = nch > 1;
  const int64_t ldq = q1_ld(m);
  const int qodd = (int)(n_s & 1);
  // row-parallel copies: thread t owns row (t & 255) and every other column
  // from (t >> 8) -- coalesced, and no index division in the loops
  const int trow = tid & (CQ_RMAX - 1), tcol0 = tid / CQ_RMAX, tcstep = PANEL_T / CQ_RMAX;
  auto load_chunk = [&](const double* src, int64_t ld, int ch, int ncol) {  // rows of chunk ch -> sl
    const int c0r = ch * CQ_RMAX, cR = min(CQ_RMAX, R - c0r), cR4 = (cR + 3) & ~3;
    // (cp.async: the whole chunk in flight at once -- a plain copy loop waits a round trip per unrolled group)
    if (trow < cR4) {
      const double* sp = src + c0r + trow;
      if (trow < cR) {
        for (int cc = tcol0; cc < ncol; cc += tcstep) cp_async8(sl + cc * CQ_LDS + trow, sp + (int64_t)cc * ld);
      } else {
        for (int cc = tcol0; cc < ncol; cc += tcstep) sl[cc * CQ_LDS + trow] = 0.0;
      }
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    return cR4;
  };
  double* gacc = a.red + 3 * DMQR_KP * DMQR_KP + (size_t)blockIdx.x * DMQR_KP * DMQR_KP;  // per-CTA scratch
  double* vQ = a.red + 21 * DMQR_KP * DMQR_KP + (size_t)blockIdx.x * DMQR_KP * DMQR_KP;    // per-CTA scratch
  // helper mode: uniform over the ranks (every rank's slice exceeds 256 rows)
  const bool hmode = a.helpers && mp > (int64_t)nr * CQ_RMAX;
  const int64_t hnch = ceil_div(mp, CQ_RMAX);  // helper chunks (256 panel rows each)
  // publish R1^-1 (or a 'no pass 2' flag) for the helpers; rank 0, all threads
  auto h_publish = [&](bool hfail, int hkk) {
    if (me != 0) return;
    if (!hfail)
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) a.hR[e] = A1[e];
    __syncthreads();
    if (tid == 0) {
      a.hR[DMQR_KP * DMQR_KP] = (double)hkk;
      a.hR[DMQR_KP * DMQR_KP + 1] = hfail ? 1.0 : 0.0;
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.hctr + 4), "r"((unsigned)S.step_idx + 1u) : "memory");
    }
  };
  // sum the helper partials of chunks me, me + nr, ... (upper tiles, fixed order) into G
  // Whether the helpers' partials are used for a pass: rank 0 waits (bounded)
  // for all chunks and decides for the whole cluster (hctr[dec] = 2: use them,
  // 1: abandoned -- the helpers stop and the cluster streams its own rows, as
  // without helpers).  Bounded, so a serialised launch (a profiler replaying
  // kernels one at a time, CUDA_LAUNCH_BLOCKING) cannot deadlock.
  __shared__ int s_use;
  auto h_decide = [&](int done_idx, int dec_idx) -> bool {
    if (tid == 0) {
      if (me == 0) {
        const long long deadline = gtimer() + a.hwait_ns;  // default 5 ms (a pass takes ~0.1 ms)
        unsigned v;
        bool ok = false;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.hctr + done_idx) : "memory");
          if (v >= (unsigned)hnch) {
            ok = true;
            break;
          }
          if (gtimer() > deadline) break;
          __nanosleep(100);
        }
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.hctr + dec_idx), "r"(ok ? 2u : 1u) : "memory");
      }
      unsigned d;
      SpinGuard sg;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(a.hctr + dec_idx) : "memory");
        if (d != 0u) break;
        sg.tick(5, dec_idx, 0);
      }
      s_use = (d == 2u);
    }
    __syncthreads();
    return s_use != 0;
  };
  // sum the helper partials of chunks me, me + nr, ... (upper tiles, fixed order) into G
  auto h_gather = [&](double* G) {
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      double g = 0.0;
      if ((e % DMQR_KP) / 8 >= (e / DMQR_KP) / 8)
        for (int64_t ch = me; ch < hnch; ch += nr) g += __ldcg(a.hpart + ch * DMQR_KP * DMQR_KP + e);
      G[e] = g;
    }
    __syncthreads();
  };
  // without the helpers' partials (no helpers, or abandoned) a helper-mode
  // panel streams its rows like a chunked one (the slice was never loaded)
  const bool chunked_eff = chunked || hmode;
  // P-mode look-ahead (unchunked panels): G = Q1^T C = R1^-T (P^T C), so k_spare
  // forms P^T C from the start of the panel and MT absorbs R1^-1 (MT' = R1^-1 MT)
  const bool pmode = a.spare && a.pg != nullptr && !chunked_eff;
  double* gR1i = a.red + 38 * DMQR_KP * DMQR_KP;  // R1^-1 (P-mode)
  if (a.helpers && !hmode) h_publish(true, 0);  // (nothing for the helpers' second pass)
  // ---- P0/P1: slice <- P (rows zero-padded to a multiple of 4), G = P^T P ----
  const bool h1 = hmode && h_decide(1, 6);  // (pass 1 abandoned: no helper runs pass 2 either)
  if (h1) {
    CQT();
    h_gather(A2);
  } else if (!chunked_eff) {
    load_chunk(gA, lda, 0, k);
    if (pmode) {  // P rows -> pg: k_spare's G = P^T C starts now, not after Q1
      if (trow < R) {
        double* dp = a.pg + qodd + r0 + trow;
#pragma unroll 4
        for (int cc = tcol0; cc < k; cc += tcstep) dp[(int64_t)cc * ldq] = sl[cc * CQ_LDS + trow];
      }
      __syncthreads();
      if (tid == 0) {
        if (me == 0) c->p_k = k;
        __threadfence();
        atomicAdd(&c->p_count, 1u);
      }
    }
    CQT();
    cq_gram(sl, R4, k, A2);
  } else {
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) A2[e] = 0.0;
    CQT();
    for (int ch = 0; ch < nch; ++ch) {
      const int cR4 = load_chunk(gA, lda, ch, k);
      cq_gram(sl, cR4, k, A1);
      __syncthreads();
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T)  // upper tiles written by cq_gram
        if ((e % DMQR_KP) / 8 >= (e / DMQR_KP) / 8) A2[e] += A1[e];
      __syncthreads();
    }
  }
  CQT();
  cq_cluster_reduce(A2, A1, k);
  CQT();
  for (int j = tid; j < k; j += PANEL_T) vpiv[DMQR_KP + j] = A1[j * DMQR_KP + j];
  __syncthreads();
  // ---- P3: R1 = chol(G) -> A2 ----
  const int jstar = cq_chol(A1, A2, vpiv, vpiv + DMQR_KP, k, CQ_PIVOT_TOL);
  CQT();
  // accepted pass-1 prefix kk = jstar; decide early whether an unhealthy pivot proves a break
  int kk = jstar;
  bool fail = false;
  if (jstar < k) {
    // pivot d ~ R_jj^2 <= CQ_PIVOT_TOL G_jj (+ rounding ~n eps max_j G_jj):
    // R_jj <= 3.2e-4 ||a_j|| + noise; break iff R_jj < eps_s
    const double bound = 1e-3 * sqrt(vpiv[DMQR_KP + jstar]);
    if (!brk || jstar == 0 || !(bound < eps_s)) fail = true;
  }
  const bool q1_pub = a.spare && !fail && kk > 0;
  if (hmode && (fail || kk == 0)) h_publish(true, 0);
  auto store_q1 = [&](int ch) {  // sl rows of chunk ch -> q1g (the row parity of A)
    const int c0r = ch * CQ_RMAX, cR = min(CQ_RMAX, R - c0r);
    if (trow < cR) {
      double* dp = a.q1g + qodd + r0 + c0r + trow;
#pragma unroll 4
      for (int cc = tcol0; cc < kk; cc += tcstep) dp[(int64_t)cc * ldq] = sl[cc * CQ_LDS + trow];
    }
  };
  if (!fail && kk > 0) {
    // ---- P4/P5: Q1 = P R1^-1 (in place) ----
    cq_trinv_upper(A2, A1, kk);
    CQT();
    if (pmode && me == min(2, nr - 1)) {  // (rank_MT below)
      __syncthreads();
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
        const int i = e / DMQR_KP, j = e % DMQR_KP;
        gR1i[e] = (i < kk && j < kk && j >= i) ? A1[e] : 0.0;
      }
    }
    // keep R1: transpose into the lower triangle of A2, diagonal in vD
    __syncthreads();
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      if (i >= kk || j >= kk) continue;
      if (i < j) A2[j * DMQR_KP + i] = A2[i * DMQR_KP + j];
      if (i == j) vD[i] = A2[i * DMQR_KP + i];
    }
    __syncthreads();
    bool use_h2 = false;
    if (h1) {  // the helpers form Q1 = P R1^-1 into q1g and the per-chunk Q1 Grams
      h_publish(false, kk);
      use_h2 = h_decide(3, 7);
    }
    if (use_h2) {
      h_gather(A1);
      CQT();
    } else if (!chunked_eff) {
      cq_slice_gemm(sl, R4, kk, kk, A1);
      CQT();
      // publish this rank's Q1 rows: k_ygemm forms Y = Q1 M from them, and
      // (look-ahead) k_spare's G = Q1^T C
      __syncthreads();
      store_q1(0);
      __syncthreads();
      FCQT(0);
      // ---- P6/P7: G2 = Q1^T Q1 (partial -> A1, total -> upper A2) ----
      cq_gram(sl, R4, kk, A1);
      FCQT(1);
    } else {
      // per chunk: Q1 = P R1^-1 -> q1g; the Q1 Gram accumulates in global scratch
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) gacc[e] = 0.0;
      for (int ch = 0; ch < nch; ++ch) {
        const int cR4 = load_chunk(gA, lda, ch, kk);
        cq_slice_gemm(sl, cR4, kk, kk, A1);
        __syncthreads();
        store_q1(ch);
        cq_gram(sl, cR4, kk, vQ);
        __syncthreads();
        for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T)
          if ((e % DMQR_KP) / 8 >= (e / DMQR_KP) / 8) gacc[e] += vQ[e];
        __syncthreads();
      }
      CQT();
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) A1[e] = gacc[e];
      __syncthreads();
    }
    if (q1_pub && tid == 0) {
      c->q1_kk = kk;
      __threadfence();
      atomicAdd(&c->q1_count, 1u);
    }
    FCQT(2);
    CQT();
    cq_cluster_reduce(A1, A2, kk);
    CQT();
    // orthogonality of Q1: |G2 - I|_max (s_flag[2]: beyond the near-identity regime)
    if (tid == 0) {
      s_flag[0] = 0;
      s_flag[2] = 0;
    }
    __syncthreads();
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      if (i >= kk || j >= kk) continue;
      if (j >= i) {
        const double g = A2[i * DMQR_KP + j] - (i == j ? 1.0 : 0.0);
        if (!(fabs(g) < CQ_ORTH_TOL)) s_flag[0] = 1;
        if (!(fabs(g) <= CQ_NEAR_ID)) s_flag[2] = 1;
      }
    }
    for (int j = tid; j < kk; j += PANEL_T) vpiv[DMQR_KP + j] = A2[j * DMQR_KP + j];
    __syncthreads();
    if (s_flag[0]) fail = true;
    FCQT(3);
  }
  if (me == 0 && tid == 0) c->cq_diag[3] = jstar;
  if (a.spare && !q1_pub && tid == 0) {  // nothing to publish: release k_spare
    c->q1_fail = 1;
    __threadfence();
    atomicAdd(&c->q1_count, 1u);
  }
  int l = kk;
  // G2 = I + E with |E| <= CQ_NEAR_ID (the usual case): R2 = I + X with
  // X = Phi(E) (Phi: strict upper + half diagonal) -- instead of a 65-pivot
  // Cholesky chain.  The exact X satisfies X = Phi(E - X^T X); the dropped
  // term is <= kk |E|^2 <= 6.5e-19 per entry, far below rounding of R2 ~ I.
  const bool near_id = !s_flag[2];
  if (!fail && kk > 0) {
    if (near_id) {
      // ---- P8': R2 = I + Phi(G2 - I) -> A1 ----
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
        const int i = e / DMQR_KP, j = e % DMQR_KP;
        double x = 0.0;
        if (i < kk && j < kk && j >= i) x = (i == j) ? 1.0 + 0.5 * (A2[e] - 1.0) : A2[e];
        A1[e] = x;
      }
      __syncthreads();
      FCQT(4);
    } else {
      // ---- P8: R2 = chol(G2) -> A1 (reads/destroys the upper of A2) ----
      if (cq_chol(A2, A1, vpiv, vpiv + DMQR_KP, kk, 1e-6) < kk) fail = true;
    }
    CQT();
  }
  // ---- break: first j >= 1 with |R_jj| < eps_s; an unhealthy pivot at jstar
  // is a break.  R = R2 R1 is triangular, so R_jj = R2_jj R1_jj exactly as the
  // product's single nonzero term (R itself is formed off rank 0's chain) ----
  if (!fail && kk > 0) {
    if (tid < 32) {
      int lb = kk;
      if (brk)
        for (int b0 = 0; b0 < kk; b0 += 32) {
          const int j = b0 + tid;
          const bool hit = j >= 1 && j < kk && fabs(__dmul_rn(A1[j * DMQR_KP + j], vD[j])) < eps_s;
          const unsigned bal = __ballot_sync(0xffffffffu, hit);
          if (bal) {
            lb = b0 + __ffs(bal) - 1;
            break;
          }
        }
      if (tid == 0) s_flag[1] = lb;
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
  // Work after the break, by rank:
  //   rank 0:        R2^-1, Q_top, modified LU, then T = U Y1^-T (and FT = Y1^-T)
  //   rank_R:        R = R2 R1 -> global; after the LU, R_H = S R into the packed top block
  //   rank_M:        M = -R2^-1 S U^-1 -> gM (k_ygemm: Y below the top block = Q1 M)
  //   rank_MT:       MT = M T = -R2^-1 S Y1^-T -> gMT (look-ahead only)
  // (F = Y1 - Q1_top M = U^-1 since Y1 U = I - Q_top S, so FT = F T = Y1^-T.)
  // With fewer ranks the tasks fold onto the highest rank available.
  const int rk_M = min(1, nr - 1), rk_MT = min(2, nr - 1), rk_R = min(3, nr - 1);
  const bool do_mt = a.spare != 0;
  double* gR = a.red;                                   // R (l x l upper), global
  double* gM = a.red + 37 * DMQR_KP * DMQR_KP;          // M for k_ygemm
  double* gFT = a.red + 19 * DMQR_KP * DMQR_KP;         // k_trail_w's factors
  double* gMT = gFT + DMQR_KP * DMQR_KP;
  double* gTop = a.A + n_s * lda + n_s;                 // the panel's top l x l block
  __syncthreads();
  CQT();
  if (me == rk_R) {
    // R1[t][j] lives transposed in the strict lower of A2 (diag in vD); R2 upper in A1
    cq_small_gemm([&](int i, int t) { return A1[i * DMQR_KP + t]; },
                  [&](int t, int j) { return (t < j) ? A2[j * DMQR_KP + t] : ((t == j) ? vD[j] : 0.0); }, gR, l);
    __syncthreads();
  }
  auto r2_inverse = [&]() {  // R2^-1 -> A2 (R2 upper in A1)
    if (near_id) {  // R2^-1 = I - X (dropped X^2: <= l |E|^2 per entry, as above)
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
        const int i = e / DMQR_KP, j = e % DMQR_KP;
        double x = 0.0;
        if (i < l && j < l && j >= i) x = (i == j) ? 2.0 - A1[e] : -A1[e];
        A2[e] = x;
      }
      __syncthreads();
    } else {
      cq_trinv_upper(A1, A2, l);
      __syncthreads();
    }
  };
  // aux task: out = (-R2^-1 S) src^-1 for an upper triangular src (l x l, KP
  // row-major, possibly in rank 0's shared memory); r2i: R2^-1 (upper), sg: S;
  // scr: two KP x KP scratch blocks
  auto aux = [&](const double* src, const double* r2i, const double* sg, double* scr, double* out, bool r1pre) {
    double* P = scr;
    double* X = scr + DMQR_KP * DMQR_KP;
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      P[e] = (i < l && j < l && j >= i) ? src[e] : 0.0;
    }
    __syncthreads();
    cq_trinv_upper(P, X, l);
    __syncthreads();
    cq_small_gemm([&](int i, int t) { return -sg[t] * r2i[i * DMQR_KP + t]; },
                  [&](int t, int j) { return X[t * DMQR_KP + j]; }, P, l);
    __syncthreads();
    if (r1pre) {  // P-mode: R1^-1 (this rank stored it) times MT
      cq_small_gemm([&](int i, int t) { return gR1i[i * DMQR_KP + t]; },
                    [&](int t, int j) { return P[t * DMQR_KP + j]; }, X, l);
      __syncthreads();
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) P[e] = X[e];
      __syncthreads();
    }
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      out[e] = (i < l && j < l && j >= i) ? P[e] : 0.0;
    }
    __syncthreads();
  };
  // rank 0's shared scratch after Q_top (the slice is no longer read):
  // sl[0 .. KP^2): R2^-1 copy (tasks folded onto rank 0), then two blocks
  double* r2c = sl;
  double* scr0 = sl + DMQR_KP * DMQR_KP;
  if (me == 0) {
    r2_inverse();
    CQT();
    // ---- P12: top l x l block of Q = Q1 R2^-1 -> A1 ----
    if (!chunked_eff)
      cq_small_gemm<true>([&](int i, int t) { return sl[t * CQ_LDS + i]; },
                          [&](int t, int j) { return A2[t * DMQR_KP + j]; }, A1, l);
    else  // (rank 0's first rows, published)
      cq_small_gemm<true>([&](int i, int t) { return a.q1g[(int64_t)t * ldq + qodd + i]; },
                          [&](int t, int j) { return A2[t * DMQR_KP + j]; }, A1, l);
    __syncthreads();
    if (nr <= 2)
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) r2c[e] = A2[e];
    CQT();
    // ---- P13: modified LU of the top block: strict lower = L (Y1), upper = q' ----
    cq_mlu(A1, vS, vpiv, l);
    CQT();
    // U (upper) -> A2: U_jj = pivot, U_jc = -S_c q'_jc; Y1^T (unit upper) into
    // the upper of A1 (the strict lower keeps Y1)
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      double u = 0.0;
      if (i < l && j < l && j >= i) u = (i == j) ? vpiv[i] : -vS[j] * A1[i * DMQR_KP + j];
      A2[e] = u;
    }
    __syncthreads();
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      if (i >= l || j >= l) continue;
      if (j > i) A1[i * DMQR_KP + j] = A1[j * DMQR_KP + i];
      if (j == i) A1[i * DMQR_KP + i] = 1.0;
    }
    __syncthreads();
  } else if (me == rk_M || (do_mt && me == rk_MT)) {
    r2_inverse();  // (overlaps rank 0's Q_top and LU)
  }
  cl.sync();  // U, Y1^T, S ready on rank 0
  CQT();
  const double* A1r = cl.map_shared_rank(A1, 0);
  const double* A2r = cl.map_shared_rank(A2, 0);
  const double* vSr = cl.map_shared_rank(vS, 0);
  if (me == 0) {
    // packed top block, strict lower: the Y1 multipliers (R_H above it: rank_R)
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int p = e / DMQR_KP, cc = e % DMQR_KP;
      if (p < l && cc < p) gA[(int64_t)cc * lda + p] = A1[p * DMQR_KP + cc];
    }
    // X = (Y1^T)^-1 = FT; T = U X (householder.py accumulate_wy's W; tau_j = U_jj)
    double* X = scr0;
    double* Tt = scr0 + DMQR_KP * DMQR_KP;
    cq_trinv_upper(A1, X, l);
    __syncthreads();
    FCQT(7);
    cq_small_gemm([&](int i, int t) { return A2[i * DMQR_KP + t]; },
                  [&](int t, int j) { return X[t * DMQR_KP + j]; }, Tt, l);
    __syncthreads();
    FCQT(8);
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      const bool in = i < l && j < l && j >= i;
      a.T[e] = in ? Tt[e] : 0.0;
      if (do_mt) gFT[e] = in ? X[e] : 0.0;
    }
    for (int j = tid; j < l; j += PANEL_T) a.coeffs[n_s + j] = vpiv[j];
    __syncthreads();
    CQT();
  }
  if (me == rk_R && me != 0) {
    // packed top block, diagonal and above: R_H = S R (R from this rank, global)
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int p = e / DMQR_KP, cc = e % DMQR_KP;
      if (p < l && cc < l && cc >= p) gTop[(int64_t)cc * lda + p] = vSr[p] * __ldcg(gR + p * DMQR_KP + cc);
    }
  }
  // rank_M / rank_MT: the inverses of rank 0's U and Y1^T, times -R2^-1 S
  const bool on0 = (me == 0);
  if (me == rk_M) aux(A2r, on0 ? r2c : A2, vSr, on0 ? scr0 : sl, gM, false);
  if (do_mt && me == rk_MT) aux(A1r, on0 ? r2c : A2, vSr, on0 ? scr0 : sl, gMT, pmode);
  if (me == 0 && rk_R == 0) {
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) {
      const int p = e / DMQR_KP, cc = e % DMQR_KP;
      if (p < l && cc < l && cc >= p) gTop[(int64_t)cc * lda + p] = vS[p] * __ldcg(gR + p * DMQR_KP + cc);
    }
  }
  CQT();
  CQT();
  CQT();
#undef CQT
#undef FCQT
  if (me == 0 && tid == 0) {
    if (a.tline) {
      a.tline[4 * (c->step_idx & 255) + 0] = t_start;
      a.tline[4 * (c->step_idx & 255) + 1] = gtimer();
    }
    c->l_acc = l;
    c->broke = (l < k);
    c->cq_fail = 0;
    c->tc0 = (int32_t)(n_s + l);
  }
  cl.sync();
  // M and l are final: k_spare may start the Y = Q1 M tiles (its third phase)
  // before this grid has completed
  if (me == 0 && tid == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&c->m_pub), "r"((unsigned)c->step_idx + 1u) : "memory");
  }
}



// The tall panel's row passes on the SMs the cluster leaves free (launched as
// the panel's programmatic dependent, serial schedule only): per 256-row chunk
// of P, pass 1 writes the Gram partial P_c^T P_c; once rank 0 publishes R1^-1,
// pass 2 writes Q1_c = P_c R1^-1 into q1g and its Gram partial.  Chunks are
// pulled from counters; the cluster sums the partials in fixed order.
constexpr size_t CQH_SMEM = sizeof(double) * ((size_t)CQ_KC * CQ_LDS + 2 * DMQR_KP * DMQR_KP);

__global__ void __launch_bounds__(PANEL_T, 1) k_panel_helper(PanelArgs a) {
  Ctl* c = a.c;
  const CtlSnap S = snap(c);
  // (every exit waits for the panel grid: the kernels behind this one -- the
  // Householder fallback panel, k_ygemm -- must see the panel's results)
  if (S.done) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  extern __shared__ __align__(16) double hsm[];
  double* sl = hsm;
  double* G = sl + CQ_KC * CQ_LDS;
  double* Rs = G + DMQR_KP * DMQR_KP;
  __shared__ int s_item;
  __shared__ double s_hdr[2];
  const int tid = threadIdx.x;
  const int64_t n_s = S.n_s, m = S.m, lda = S.lda, mp = m - n_s;
  const int k = S.k_s;
  const int64_t nch = ceil_div(mp, CQ_RMAX);
  const double* gA = a.A + n_s * lda + n_s;
  const int64_t ldq = q1_ld(m);
  const int qodd = (int)(n_s & 1);
  const int trow = tid & (CQ_RMAX - 1), tcol0 = tid / CQ_RMAX, tcstep = PANEL_T / CQ_RMAX;
  auto load = [&](int64_t ch, int ncol) {
    const int64_t c0r = ch * CQ_RMAX;
    const int cR = (int)min((int64_t)CQ_RMAX, mp - c0r), cR4 = (cR + 3) & ~3;
    if (trow < cR4) {
      const double* sp = gA + c0r + trow;
#pragma unroll 4
      for (int cc = tcol0; cc < ncol; cc += tcstep) sl[cc * CQ_LDS + trow] = (trow < cR) ? sp[(int64_t)cc * lda] : 0.0;
    }
    __syncthreads();
    return cR4;
  };
  auto put = [&](int64_t ch) {
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) a.hpart[ch * DMQR_KP * DMQR_KP + e] = G[e];
    __syncthreads();
  };
  auto next = [&](int idx) {
    if (tid == 0) s_item = (int)atomicAdd(a.hctr + idx, 1u);
    __syncthreads();
    const int it = s_item;
    __syncthreads();
    return it;
  };
  auto done = [&](int idx) {
    if (tid == 0) {
      __threadfence();
      atomicAdd(a.hctr + idx, 1u);
    }
  };
  auto abandoned = [&](int dec_idx) {  // the panel gave up on the helpers for this pass
    __shared__ int s_ab;
    if (tid == 0) {
      unsigned d;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d) : "l"(a.hctr + dec_idx) : "memory");
      s_ab = (d == 1u);
    }
    __syncthreads();
    return s_ab != 0;
  };
  // ---- pass 1: G1 partials ----
  for (;;) {
    if (abandoned(6)) break;
    const int ch = next(0);
    if (ch >= nch) break;
    const int cR4 = load(ch, k);
    cq_gram(sl, cR4, k, G);
    __syncthreads();
    put(ch);
    done(1);
  }
  // ---- pass 2 once R1^-1 is published (or nothing to do) ----
  if (tid == 0) {
    unsigned v, d6;
    SpinGuard sg;
    for (;;) {  // R1^-1 published, or pass 1 abandoned (then the panel never publishes)
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.hctr + 4) : "memory");
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(d6) : "l"(a.hctr + 6) : "memory");
      if (v == (unsigned)S.step_idx + 1u || d6 == 1u) break;
      __nanosleep(200);
      sg.tick(6, v, S.step_idx);
    }
    s_hdr[0] = __ldcg(a.hR + DMQR_KP * DMQR_KP);
    s_hdr[1] = (v == (unsigned)S.step_idx + 1u) ? __ldcg(a.hR + DMQR_KP * DMQR_KP + 1) : 1.0;
  }
  __syncthreads();
  if (s_hdr[1] != 0.0) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  const int kk = (int)s_hdr[0];
  for (int e = tid; e < DMQR_KP * DMQR_KP; e += PANEL_T) Rs[e] = __ldcg(a.hR + e);
  __syncthreads();
  for (;;) {
    if (abandoned(7)) break;
    const int ch = next(2);
    if (ch >= nch) break;
    const int cR4 = load(ch, kk);
    cq_slice_gemm(sl, cR4, kk, kk, Rs);
    __syncthreads();
    {  // Q1 rows of the chunk -> q1g (the row parity of A)
      const int64_t c0r = (int64_t)ch * CQ_RMAX;
      const int cR = (int)min((int64_t)CQ_RMAX, mp - c0r);
      if (trow < cR) {
        double* dp = a.q1g + qodd + c0r + trow;
#pragma unroll 4
        for (int cc = tcol0; cc < kk; cc += tcstep) dp[(int64_t)cc * ldq] = sl[cc * CQ_LDS + trow];
      }
    }
    cq_gram(sl, cR4, kk, G);
    __syncthreads();
    put(ch);
    done(3);
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// zero the helper counters (PDL chain: behind the swap, before the panel)
__global__ void k_hzero(unsigned* __restrict__ h) {
  pdl_enter();
  if (threadIdx.x < 8) h[threadIdx.x] = 0u;
}

}  // namespace dmqr
