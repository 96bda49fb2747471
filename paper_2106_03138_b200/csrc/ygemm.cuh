// Y = Q1 M below the panel's top l rows (rows l .. m' of the accepted
// columns), after a successful CholeskyQR2 panel: one CTA per 64 rows, all
// SMs, instead of the panel's 16.  Q1 comes from the published buffer, M from
// the panel (gM); the DMMA sequence is the panel's slice product (triangular M).
// Runs as k_ygemm (serial schedule) or as the third phase of k_spare
// (look-ahead: on the spare SMs right after the panel, off the critical path).
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int YG_ROWS = 64;
constexpr int YG_LD = YG_ROWS + 4;
constexpr size_t YG_SMEM = sizeof(double) * (DMQR_KP * DMQR_KP + DMQR_KP * YG_LD);

// tile `blk` (rows l + 64 blk ..) of Y = Q1 M; 256 threads, YG_SMEM dynamic shared memory
__device__ __forceinline__ void ygemm_tile(double* __restrict__ A, const double* __restrict__ q1g,
                                           const double* __restrict__ gM, int64_t n_s, int64_t m, int64_t lda, int l,
                                           int64_t blk) {
  const int64_t mp = m - n_s;
  const int64_t r0 = l + blk * YG_ROWS;  // panel-relative
  if (l == 0 || r0 >= mp) return;
  const int64_t ldq = q1_ld(m);
  const int qodd = (int)(n_s & 1);
  extern __shared__ __align__(16) double ygs[];
  double* ms = ygs;                        // M[k][c], KP row-major
  double* qs = ygs + DMQR_KP * DMQR_KP;    // Q1[r][k] at qs[k * YG_LD + r]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nr = (int)min((int64_t)YG_ROWS, mp - r0);
  const int lp4 = (l + 3) / 4 * 4;
  // both operands by cp.async: every load of the tile is in flight at once (one L2 round trip; the
  // load -> store pairs of a plain copy loop serialise into one round trip per iteration)
  for (int e = tid; e < DMQR_KP * DMQR_KP / 2; e += blockDim.x) cp_async16(ms + 2 * e, gM + 2 * e, 16);
  for (int e = tid; e < lp4 * YG_ROWS; e += blockDim.x) {
    const int k = e / YG_ROWS, rr = e % YG_ROWS;
    if (k < l && rr < nr)
      cp_async8(qs + k * YG_LD + rr, q1g + (int64_t)k * ldq + qodd + r0 + rr);
    else
      qs[k * YG_LD + rr] = 0.0;
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int nt_n = (l + 7) / 8;
  const int r = wid * 8 + (lane >> 2);
  double acc[DMQR_KP / 8][2];
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int ks = 0; ks < lp4 / 4; ++ks) {
    const int kc = 4 * ks + (lane & 3);
    const double av = qs[kc * YG_LD + r];
#pragma unroll
    for (int q = 0; q < DMQR_KP / 8; ++q)
      if (q < nt_n && 4 * ks < 8 * (q + 1)) dmma884(acc[q][0], acc[q][1], av, ms[kc * DMQR_KP + q * 8 + (lane >> 2)]);
  }
  if (r < nr) {
    double* dp = A + (n_s + r0 + r) + n_s * lda;
#pragma unroll
    for (int q = 0; q < DMQR_KP / 8; ++q) {
      const int c0 = q * 8 + 2 * (lane & 3);
      if (c0 < l) dp[(int64_t)c0 * lda] = acc[q][0];
      if (c0 + 1 < l) dp[(int64_t)(c0 + 1) * lda] = acc[q][1];
    }
  }
}

__global__ void __launch_bounds__(256) k_ygemm(Ctl* c, double* __restrict__ A,
                                               const double* __restrict__ q1g, const double* __restrict__ gM) {
  zshift(c, c, A, q1g, gM);
  pdl_enter();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 6);
  if (S.done || S.cq_fail) return;
  ygemm_tile(A, q1g, gM, S.n_s, S.m, S.lda, S.l_acc, blockIdx.x);
}

}  // namespace dmqr
