// Loop bookkeeping kernels: init, step record, final rank; input checks; explicit Q.
//   a_max0 / floor / kmax     rrqr.py:326-328
//   StepRecord append         rrqr.py:394-404 (+ fallback record 349-351)
//   rank / n_factored         rrqr.py:406-412, _posthoc_rank 206-208
//   dense() finiteness        matrix.py:32-33
//   reconstruct (explicit Q)  rrqr.py:459-476
#pragma once
#include "common.cuh"
#include "trailing.cuh"

namespace dmqr {

struct InitArgs {
  Ctl* c;
  const double* u;
  int64_t* perm;
  double* coeffs;
  int64_t m, n, lda, kmax;
  double tau, delta, eps1;  // eps1 < 0: StopRule.NONE
  int32_t k_dm, use_delta_max, break_check, trace_norms;
  int64_t swap_cap, step_cap;
  const int32_t* nonfinite;  // set by k_colnorms_init
  int32_t lookahead;
  int64_t zstride;         // per-matrix block stride of a batched launch (grid.z > 1)
  unsigned long long* tl;  // debug timeline buffer (workspace) or null
};

__global__ void __launch_bounds__(1024) k_init(InitArgs a) {
  zshift_by(a.zstride, a.c, a.u, a.perm, a.coeffs, a.nonfinite);
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double mx = 0.0;
  for (int64_t j = tid; j < a.n; j += blockDim.x) mx = fmax(mx, a.u[j]);
  mx = warp_max(mx);
  if (lane == 0) red[wid] = mx;
  for (int64_t j = tid; j < a.n; j += blockDim.x) a.perm[j] = j;
  for (int64_t j = tid; j < a.kmax; j += blockDim.x) a.coeffs[j] = 0.0;
  __syncthreads();
  if (wid == 0) {
    mx = warp_max(lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0);
    if (lane == 0) {
      Ctl* c = a.c;
      c->m = a.m;
      c->n = a.n;
      c->lda = a.lda;
      c->kmax = a.kmax;
      c->a_max0 = mx;
      c->floor = (double)a.n * kEps * mx;  // n * EPS * a_max0 (rrqr.py:327)
      c->stop_active = a.eps1 >= 0.0;
      c->stop_rhs = a.eps1 >= 0.0 ? a.eps1 * mx : 0.0;
      c->tau = a.tau;
      c->delta = a.delta;
      c->k_dm = a.k_dm;
      c->use_delta_max = a.use_delta_max;
      c->break_check = a.break_check;
      c->trace_norms = a.trace_norms;
      c->la = a.lookahead;
      c->zstride = a.zstride;
      c->tl = a.tl;
      c->pend = 0;
      c->gcount = 0;
      c->swap_cap = (int32_t)min(a.swap_cap, (int64_t)0x7fffffff);
      c->step_cap = (int32_t)min(a.step_cap, (int64_t)0x7fffffff);
      c->n_s = 0;
      c->done = (a.kmax == 0);
      if (a.nonfinite && *a.nonfinite) {  // ValueError in dense() (matrix.py:32-33)
        c->status = -2;
        c->done = 1;
      }
    }
  }
}

// Append the step record and advance n_s (single thread, last kernel of a step).
__device__ __forceinline__ void step_end_body(const CtlSnap& S, Ctl* c, StepRec* __restrict__ steps,
                                              double* __restrict__ norm_trace,
                                              unsigned long long* __restrict__ trace_bits, const double* __restrict__ A,
                                              double* __restrict__ Wt, int64_t ldz, double* __restrict__ u,
                                              double* __restrict__ uref, uint8_t* __restrict__ upd) {
  // look-ahead with no trailing columns past tc0: k_trail_a had no tile to do
  // the panel-column bookkeeping (one warp does it here)
  if (S.la && S.tc0 >= S.n) la_panel_columns(c, A, Wt, ldz, u, uref, upd, S.n_s, S.l_acc, S.tc0);
  __syncwarp();
  if (threadIdx.x != 0) return;
  const int idx = S.step_idx;
  const int l = S.l_acc;
  if (idx >= S.step_cap) {
    c->status = -5;
    c->done = 1;
    return;
  }
  const int broke = c->broke;
  const double eps_s = c->eps_s, gamma = c->gamma;
  // a wide step (k_dm > DMQR_MAXK - 1, wide.cuh) keeps one record over its
  // panel chunks: rewritten after every chunk, committed after the last
  const bool wide = S.k_dm > DMQR_MAXK - 1 && S.kind == 0;
  const bool w_more = wide && c->w_next > 0;
  StepRec r;
  r.n_s = wide ? c->w_ns0 : S.n_s;
  r.k_selected = wide ? c->w_total : S.k_s;
  r.k_accepted = wide ? c->w_done : l;
  r.k_max = (S.kind == 0) ? S.k_max : -1;
  r.broke_early = broke;
  r.fell_back_to_scalar = (S.kind == 1);
  r.eps_s = (S.kind == 0) ? eps_s : 0.0;
  r.gamma = (S.kind == 0) ? gamma : 1.0;
  steps[idx] = r;
  if (S.trace_norms && norm_trace) {
    const int64_t n_s1 = S.n_s + l;
    // _record_norm_check appends nothing once the trailing block is empty
    norm_trace[idx] = (n_s1 < S.n) ? __longlong_as_double((long long)*trace_bits) : __longlong_as_double(-1ll);
    *trace_bits = 0ull;
  }
  if (S.la) {  // this step's update is now pending below its R rows (look-ahead)
    c->pend = (l > 0 && S.n_s + l < S.m && S.tc0 < S.n && !c->pend_done) ? 1 : 0;
    c->pend_done = 0;
    c->pend_ns = S.n_s;
    c->pend_l = l;
  }
  c->gcount = 0;  // (look-ahead and serial guard lists)
  c->n_s = S.n_s + l;
  c->step_idx = idx + (w_more ? 0 : 1);
  c->l_acc = 0;
  c->broke = 0;
  c->nsw = 0;
  c->nmv = 0;
  if (S.n_s + l >= S.kmax) c->done = 1;
}

// The host's poll record of a step (one thread): written once the step's
// bookkeeping is done.  No stream operation sits between the steps, so the
// programmatic launches chain across step boundaries.  The record's index is
// counted on the device -- one per enqueued step -- so a replayed CUDA graph
// of the step posts the right slot and sequence.  Columns left of n_s are
// final once the record is seen (the caller fences its writes first); the
// record itself is one 16-byte store.
__device__ __forceinline__ void step_post(const CtlSnap& S, Ctl* c, HostRec* __restrict__ hrec) {
  const int enq = c->posted;
  c->posted = enq + 1;
  // (a fallback step hands the run to the blocked scalar-pivot engine, k_qp3;
  // not with the per-step norm trace)
  const int fb = (!S.done && S.kind == 1 && !S.trace_norms) ? 4 : 0;
  const int4 rec = make_int4(c->n_s, (c->done ? 1 : 0) | (c->la_bad ? 2 : 0) | fb, c->step_idx, enq + 1);
  asm volatile("st.volatile.global.v4.s32 [%0], {%1, %2, %3, %4};" ::"l"(hrec + (enq & 1)), "r"(rec.x), "r"(rec.y),
               "r"(rec.z), "r"(rec.w)
               : "memory");
}

__global__ void k_step_end(Ctl* c, StepRec* __restrict__ steps, double* __restrict__ norm_trace,
                           unsigned long long* __restrict__ trace_bits, const double* __restrict__ A,
                           double* __restrict__ Wt, int64_t ldz, double* __restrict__ u,
                           double* __restrict__ uref, uint8_t* __restrict__ upd, HostRec* __restrict__ hrec,
                           int enq) {
  zshift(c, c, steps, norm_trace, trace_bits, A, Wt, u, uref, upd);
  if (gridDim.z > 1 && hrec) hrec += 2 * blockIdx.z;  // (host records: two slots per matrix)
  pdl_enter();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 10);
  if (!S.done) step_end_body(S, c, steps, norm_trace, trace_bits, A, Wt, ldz, u, uref, upd);
  __threadfence();
  __syncwarp();
  (void)enq;
  if (threadIdx.x == 0 && hrec) step_post(S, c, hrec);
}

// switch the control block to the look-ahead schedule (from the next kernel on)
__global__ void k_set_la(Ctl* c, int on) {
  pdl_enter();
  if (threadIdx.x == 0) c->la = on;
}

// debug timeline buffer: span starts (even slots) at +inf for atomicMin, the rest 0
__global__ void k_tl_init(unsigned long long* __restrict__ tl) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q < TL_WORDS) tl[q] = (q >= 64 * 32 || (q & 1)) ? 0ull : ~0ull;
}

// rank / n_factored (rrqr.py:406-412)
__global__ void k_finalize(Ctl* c, const double* __restrict__ A, int stop_none) {
  zshift(c, c, A);
  __shared__ int cnt[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n_s = c->n_s;
  const int64_t nf = c->stopped ? n_s : min(n_s, c->kmax);
  const double thr = kEps * (double)c->n * c->a_max0;
  int k = 0;
  if (stop_none && !c->stopped)
    for (int64_t i = tid; i < nf; i += blockDim.x) k += fabs(A[i + i * c->lda]) > thr;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
  if (lane == 0) cnt[wid] = k;
  __syncthreads();
  if (tid == 0) {
    int tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += cnt[w];
    c->n_factored = (int32_t)nf;
    c->rank = c->stopped ? (int32_t)n_s : (stop_none ? tot : (int32_t)nf);
  }
}

__global__ void k_check_finite(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                               int32_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  int bad = 0;
  for (int64_t j = w0; j < n; j += nw)
    for (int64_t i = lane; i < m; i += 32) bad |= !isfinite(__ldg(A + i + j * lda));
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
}

// ---- explicit Q (reconstruct, rrqr.py:468-476): backward accumulation ----
// Q starts as [I; 0] (m x qcols).  For s = p-1 .. 0: Q[s:, s:] -= v (coeff v^T Q[s:, s:]);
// columns < s of Q are still unit vectors there, so only columns >= s change.
__global__ void k_q_init(double* __restrict__ Q, int64_t m, int64_t qcols, int64_t ldq) {
  const int64_t tot = m * qcols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / m, i = e % m;
    Q[i + j * ldq] = (i == j) ? 1.0 : 0.0;
  }
}

// w[j] = coeff * v^T Q[s:, j] for j in [s, qcols): warp per column

}  // namespace dmqr

namespace dmqr {
// debug: flatten the decision part of Ctl (for step-by-step comparisons)
__global__ void k_debug_ctl(const Ctl* c, int64_t* __restrict__ out) {
  if (threadIdx.x != 0) return;
  int64_t* o = out;
  *o++ = c->n_s; *o++ = c->done; *o++ = c->stopped; *o++ = c->status;
  *o++ = c->kind; *o++ = c->k_max; *o++ = c->ncand; *o++ = c->nsel; *o++ = c->k_s; *o++ = c->l_acc;
  *o++ = c->nsw; *o++ = c->step_idx; *o++ = c->n_swaps;
  *o++ = __double_as_longlong(c->umax); *o++ = __double_as_longlong(c->eps_s); *o++ = __double_as_longlong(c->gamma);
  for (int i = 0; i < DMQR_KP; ++i) *o++ = c->cand[i];
  for (int i = 0; i < DMQR_KP; ++i) *o++ = c->sel[i];
  for (int i = 0; i < DMQR_KP; ++i) *o++ = c->sw_a[i];
  for (int i = 0; i < DMQR_KP; ++i) *o++ = c->sw_b[i];
  for (int i = 0; i < 4; ++i) *o++ = __double_as_longlong(c->cq_diag[i]);
  *o++ = c->cq_fail * 1000000LL + c->tc0;
}
}  // namespace dmqr
