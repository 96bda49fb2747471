// Explicit Q from the packed reflectors, blocked (replaces the backward
// accumulation of reconstruct, rrqr.py:468-476):
//
//   Q = H_0 H_1 ... H_{p-1} [I; 0],   H_s = I - coeff_s v_s v_s^T
//
// applied backward one block of FQ_NB reflectors at a time with the compact WY
// form of the block, H_j0 ... H_j1-1 = I - Y T Y^T (T upper triangular, the
// forward / columnwise larft recurrence of accumulate_wy, householder.py:92-114):
//
//   S = Y^T Y            (k_fq_w with C = Y; split over row slabs)
//   T                    (k_fq_t: T[i][i] = coeff_i, T[:i, i] = -coeff_i T[:i, :i] S[:i, i])
//   W = T (Y^T C)        (k_fq_w, then k_fq_tw sums the row-slab partials in fixed order)
//   C -= Y W             (k_fq_upd)
//
// on C = Q[j0:, j0:] (rows and columns before j0 are still the identity's).
// Y is read straight out of the packed factor (unit diagonal, zeros above).
// FP64 FMA register tiles (the DFMA rate equals the DMMA rate on this part);
// this is verification tooling off the factorization's hot path.
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int FQ_NB = 64;    // reflectors per block
constexpr int FQ_T = 256;    // 16 x 16 threads, 4 x 4 outputs each
constexpr int FQ_KR = 32;    // rows per staged slab in k_fq_w
constexpr int FQ_NSPLIT = 16;       // row splits of the Y^T C reduction (at most)
constexpr int FQ_LD = FQ_NB + 1;
constexpr size_t FQ_SMEM2 = sizeof(double) * 2 * FQ_NB * FQ_LD;  // two 64 x 65 tiles (dynamic)

// Y[r][t] of the block starting at column j0 (r, t panel-relative)
__device__ __forceinline__ double fq_y(const double* __restrict__ P, int64_t lda, int64_t j0, int64_t r, int t,
                                       int nb, int64_t mp) {
  if (t >= nb || r >= mp || r < t) return 0.0;
  if (r == t) return 1.0;
  return P[(j0 + r) + (j0 + t) * lda];
}

// Wp[split][t][c] = sum over the split's rows of Y[r][t] C[r][c] for a 64-column
// tile; C = Q[j0:, j0 + c] (ldq), or the Y block itself when q == nullptr (S = Y^T Y).
__global__ void __launch_bounds__(FQ_T) k_fq_w(const double* __restrict__ P, int64_t lda, int64_t j0, int nb,
                                               int64_t mp, const double* __restrict__ Q, int64_t ldq, int64_t cols,
                                               double* __restrict__ Wp, int64_t split_rows) {
  __shared__ double ys[FQ_KR][FQ_NB + 1];
  __shared__ double cs[FQ_KR][FQ_NB + 1];
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const int64_t c0 = (int64_t)blockIdx.x * FQ_NB;
  const int64_t rb = (int64_t)blockIdx.y * split_rows, re = min(mp, rb + split_rows);
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t r0 = rb; r0 < re; r0 += FQ_KR) {
    __syncthreads();
    for (int e = tid; e < FQ_KR * FQ_NB; e += FQ_T) {
      const int rr = e % FQ_KR, t = e / FQ_KR;  // consecutive threads: consecutive rows (coalesced)
      const int64_t r = r0 + rr;
      ys[rr][t] = (r < re) ? fq_y(P, lda, j0, r, t, nb, mp) : 0.0;
      const int64_t c = c0 + t;
      double v = 0.0;
      if (r < re && c < cols) v = Q ? Q[(j0 + r) + (j0 + c) * ldq] : fq_y(P, lda, j0, r, (int)c, nb, mp);
      cs[rr][t] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < FQ_KR; ++rr) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = ys[rr][ti * 4 + q];
        b[q] = cs[rr][tj * 4 + q];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
  }
  double* out = Wp + ((int64_t)blockIdx.y * FQ_NB) * cols;
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int64_t c = c0 + tj * 4 + y;
      if (c < cols) out[(int64_t)(ti * 4 + x) * cols + c] = acc[x][y];
    }
}

// T (FQ_NB x FQ_NB, row-major, upper) from the split partials of S = Y^T Y
__global__ void __launch_bounds__(FQ_T) k_fq_t(const double* __restrict__ Sp, int nsplit, int nb,
                                               const double* __restrict__ coeffs, int64_t j0,
                                               double* __restrict__ Tout) {
  extern __shared__ double fqs[];
  double (*S)[FQ_LD] = reinterpret_cast<double (*)[FQ_LD]>(fqs);
  double (*T)[FQ_LD] = reinterpret_cast<double (*)[FQ_LD]>(fqs + FQ_NB * FQ_LD);
  __shared__ double z[FQ_NB];
  const int tid = threadIdx.x;
  for (int e = tid; e < FQ_NB * FQ_NB; e += FQ_T) {
    const int i = e / FQ_NB, j = e % FQ_NB;
    double s = 0.0;
    for (int q = 0; q < nsplit; ++q) s += Sp[((int64_t)q * FQ_NB + i) * FQ_NB + j];
    S[i][j] = s;
    T[i][j] = 0.0;
  }
  __syncthreads();
  for (int i = 0; i < nb; ++i) {
    const double tau = coeffs[j0 + i];
    // z = T[:i, :i] S[:i, i]
    if (tid < i) {
      double acc = 0.0;
      for (int k = tid; k < i; ++k) acc = fma(T[tid][k], S[k][i], acc);
      z[tid] = acc;
    }
    __syncthreads();
    if (tid < i) T[tid][i] = -tau * z[tid];
    if (tid == 0) T[i][i] = tau;
    __syncthreads();
  }
  for (int e = tid; e < FQ_NB * FQ_NB; e += FQ_T) Tout[e] = T[e / FQ_NB][e % FQ_NB];
}

// W[t][c] = sum_k T[t][k] (sum_splits Wp[split][k][c])  (fixed split order)
__global__ void __launch_bounds__(FQ_T) k_fq_tw(const double* __restrict__ Wp, int nsplit, int nb,
                                                const double* __restrict__ T, int64_t cols,
                                                double* __restrict__ W) {
  extern __shared__ double fqs[];
  double (*Ts)[FQ_LD] = reinterpret_cast<double (*)[FQ_LD]>(fqs);
  double (*Zs)[FQ_LD] = reinterpret_cast<double (*)[FQ_LD]>(fqs + FQ_NB * FQ_LD);
  const int tid = threadIdx.x;
  const int64_t c0 = (int64_t)blockIdx.x * FQ_NB;
  for (int e = tid; e < FQ_NB * FQ_NB; e += FQ_T) {
    const int k = e / FQ_NB, cc = e % FQ_NB;
    Ts[k][cc] = T[e];
    double s = 0.0;
    const int64_t c = c0 + cc;
    if (c < cols && k < nb)
      for (int q = 0; q < nsplit; ++q) s += Wp[((int64_t)q * FQ_NB + k) * cols + c];
    Zs[k][cc] = s;
  }
  __syncthreads();
  for (int e = tid; e < FQ_NB * FQ_NB; e += FQ_T) {
    const int t = e / FQ_NB, cc = e % FQ_NB;
    const int64_t c = c0 + cc;
    if (c >= cols) continue;
    double acc = 0.0;
    for (int k = t; k < nb; ++k) acc = fma(Ts[t][k], Zs[k][cc], acc);
    W[(int64_t)t * cols + c] = acc;
  }
}

// C -= Y W on a 64 x 64 tile of C = Q[j0:, j0:]
__global__ void __launch_bounds__(FQ_T) k_fq_upd(const double* __restrict__ P, int64_t lda, int64_t j0, int nb,
                                                 int64_t mp, double* __restrict__ Q, int64_t ldq, int64_t cols,
                                                 const double* __restrict__ W) {
  extern __shared__ double fqs[];
  double (*ys)[FQ_LD] = reinterpret_cast<double (*)[FQ_LD]>(fqs);              // ys[r][t]
  double (*ws)[FQ_LD] = reinterpret_cast<double (*)[FQ_LD]>(fqs + FQ_NB * FQ_LD);  // ws[t][c]
  const int tid = threadIdx.x, ti = tid >> 4, tj = tid & 15;
  const int64_t r0 = (int64_t)blockIdx.y * FQ_NB, c0 = (int64_t)blockIdx.x * FQ_NB;
  for (int e = tid; e < FQ_NB * FQ_NB; e += FQ_T) {
    const int rr = e % FQ_NB, t = e / FQ_NB;
    ys[rr][t] = fq_y(P, lda, j0, r0 + rr, t, nb, mp);
    const int cc = e % FQ_NB, tt = e / FQ_NB;
    const int64_t c = c0 + cc;
    ws[tt][cc] = (tt < nb && c < cols) ? W[(int64_t)tt * cols + c] : 0.0;
  }
  __syncthreads();
  double acc[4][4];  // rows r0 + tj + 16 x, columns c0 + ti + 16 y: consecutive threads, consecutive rows
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int64_t r = r0 + tj + 16 * x, c = c0 + ti + 16 * y;
      acc[x][y] = (r < mp && c < cols) ? Q[(j0 + r) + (j0 + c) * ldq] : 0.0;
    }
  for (int t = 0; t < nb; ++t) {
    double a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q] = ys[tj + 16 * q][t];
      b[q] = ws[t][ti + 16 * q];
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) acc[x][y] = fma(-a[x], b[y], acc[x][y]);
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int64_t r = r0 + tj + 16 * x, c = c0 + ti + 16 * y;
      if (r < mp && c < cols) Q[(j0 + r) + (j0 + c) * ldq] = acc[x][y];
    }
}

}  // namespace dmqr
