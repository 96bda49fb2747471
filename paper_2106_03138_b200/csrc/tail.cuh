// Step tail of the look-ahead schedule (CholeskyQR2 panel path): everything
// between k_trail_w and the next step's selection, in ONE launch.
//
// In the common case k_trail_w's last CTA has already closed the step (no guard
// column, the panel did not decline): the host record is posted, and every CTA
// of this kernel sees that and exits -- one short hop in the step's chain of
// programmatic launches instead of four (k_trail_a's fallback, k_guard,
// k_guard_norms, k_step_end).  Otherwise this persistent grid (one CTA per SM,
// all co-resident: the next kernel of the chain is launched only after every
// CTA here has started) runs those kernels' work items in phases separated by
// grid barriers:
//   1. the panel declined (cq_fail; the Householder panel behind it did the
//      panel): k_trail_a's items -- Z = Y^T C split-K, Wt = T^T Z, the R rows,
//      the norm downdate and the guard list (trail_a_cta);
//   2. guard columns listed: their full update (guard_cta), the step flags,
//      then their exact norms (guard_norms_part);
//   3. CTA 0: k_step_end's bookkeeping and the host record.
// The arithmetic is the separate kernels' (same device functions, same split
// count), so the results are bitwise theirs.
#pragma once
#include "common.cuh"
#include "misc.cuh"
#include "trailing.cuh"

namespace dmqr {

constexpr size_t TAIL_SMEM = TA_SMEM > GU_SMEM ? TA_SMEM : GU_SMEM;
static_assert(GU_T == TA_T, "k_tail runs k_guard's items with k_trail_a's block size");

// generation barrier of the co-resident grid (bar[0] arrivals, bar[1] generation)
__device__ __forceinline__ void tail_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ctl_ld(&bar[1]);
    __threadfence();
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      atomicExch(&bar[0], 0u);
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      SpinGuard sg;
      while (ctl_ld(&bar[1]) == g) {
        __nanosleep(64);
        sg.tick(7, g, 0);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

struct TailArgs {
  Ctl* c;
  double* A;
  double* Zp;
  const double* T;
  double* Wt;
  unsigned* counters;  // k_trail_a's per-tile split counters
  int64_t ldz;
  double* u;
  double* uref;
  uint8_t* upd;
  int32_t* glist;
  int nsplit;          // k_trail_a's row splits (the host's choice for this step)
  StepRec* steps;
  HostRec* hrec;
  int eidx;            // this step's enqueue index (= records posted before it)
  unsigned* bar;
};

__global__ void __launch_bounds__(TA_T, 2) k_tail(const TailArgs a) {
  pdl_enter();
  Ctl* const c = a.c;
  const int tid = threadIdx.x;
  __shared__ int s_closed, s_cnt;
  if (tid == 0) s_closed = ctl_ld(&c->posted) > a.eidx;  // (one load: the common case exits on it)
  __syncthreads();
  if (s_closed) return;  // k_trail_w closed the step
  const CtlSnap& S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 10);
  if (S.done) {  // a step enqueued past the end: only its record
    if (blockIdx.x == 0 && tid == 0 && a.hrec) step_post(S, c, a.hrec);
    return;
  }
  // ---- 1. the panel declined: k_trail_a ----
  if (S.cq_fail) {
    const int64_t ncols = S.n - S.tc0;
    if (ncols > 0 && S.l_acc > 0) {
      const int ntile = (int)ceil_div(ncols, TA_COLS);
      for (int it = blockIdx.x; it < ntile * a.nsplit; it += gridDim.x) {
        trail_a_cta(S, c, a.A, a.Zp, a.T, a.Wt, a.counters, a.ldz, a.u, a.uref, a.upd, a.glist, it % ntile,
                    it / ntile, a.nsplit);
        __syncthreads();
      }
    }
    tail_barrier(a.bar);
  }
  // ---- 2. guard columns ----
  if (tid == 0) s_cnt = ctl_ld(&c->gcount);
  __syncthreads();
  const int cnt = s_cnt;
  if (cnt > 0) {
    const int64_t mp = S.m - S.n_s, np = S.n - S.n_s;
    const int gx = (int)max((int64_t)1, ceil_div(mp, GU_ROWS));
    const int gy = (int)max((int64_t)1, ceil_div(np, GU_GROUPS * DMQR_KP));
    for (int it = blockIdx.x; it < gx * gy; it += gridDim.x) {
      guard_cta(S, a.A, a.Wt, a.ldz, a.upd, a.glist, cnt, it % gx, it / gx);
      __syncthreads();
    }
    tail_barrier(a.bar);
    if (blockIdx.x == 0 && tid == 0) guard_flags(S, c, cnt);
    guard_norms_part(S, a.A, a.upd, a.u, a.uref, a.glist, cnt, ((int64_t)blockIdx.x * TA_T + tid) >> 5,
                     ((int64_t)gridDim.x * TA_T) >> 5, (int64_t)blockIdx.x * TA_T + tid, (int64_t)gridDim.x * TA_T);
    tail_barrier(a.bar);
  }
  // ---- 3. the step's bookkeeping and the host record ----
  if (blockIdx.x == 0) {
    step_end_body(S, c, a.steps, nullptr, nullptr, a.A, a.Wt, a.ldz, a.u, a.uref, a.upd);
    __threadfence();
    __syncthreads();
    if (tid == 0 && a.hrec) step_post(S, c, a.hrec);
  }
}

}  // namespace dmqr
