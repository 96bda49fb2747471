// Shared device helpers for the B200 QRDM kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef DMQR_MAXK
#define DMQR_MAXK 65   // |J| <= k_dm + 1 with the default k_dm = 64
#endif
#define DMQR_KP 72     // DMQR_MAXK padded to the 8-wide DMMA tile

namespace dmqr {

constexpr double kEps = 2.220446049250313e-16;  // 2^-52, rrqr.py:55

// Device-resident control block: every decision of the outer loop lives here,
// so kernels of one step read what the previous kernel decided without any
// host round trip.  One per factorization, at the head of the workspace.
struct Ctl {
  // fixed at init
  int64_t m, n, lda, kmax;
  double a_max0, floor, stop_rhs, tau, delta;
  int32_t stop_active, break_check, k_dm, use_delta_max;
  int32_t trace_norms, swap_cap, step_cap, pad0;
  // loop state
  int32_t n_s, done, stopped, status;
  int32_t step_idx, n_swaps, rank, n_factored;
  int32_t la_bad;  // look-ahead meets many norm guards here (graded / tall input): host goes serial
  int32_t pad4;
  // current step decision
  int32_t kind;   // 0 = deviation-maximization step, 1 = scalar fallback
  int32_t k_max;  // candidate-set size (dm.py:97), -1 on fallback
  int32_t nsel;   // |J|
  int32_t k_s;    // block size min(|J|, kmax - n_s)   rrqr.py:355
  int32_t l_acc;  // accepted reflectors (< k_s only after a qrdm2 break)
  int32_t broke;
  int32_t ncand;  // 1 + k_max
  int32_t nsw;    // swaps of this step
  double umax, eps_s, gamma;
  int32_t cand[DMQR_KP];  // absolute column indices, seed first
  int32_t sel[DMQR_KP];   // selected absolute indices, seed first
  int32_t sw_a[DMQR_KP], sw_b[DMQR_KP];
  // the same transposition sequence composed into column moves: new[dst] = old[src]
  int32_t nmv;
  int32_t mv_dst[2 * DMQR_KP], mv_src[2 * DMQR_KP];
  int32_t cq_fail;  // 1: the CholeskyQR2 panel declined, the Householder panel must run
  int32_t tc0;      // first column of the trailing update (n_s + k_s, or n_s + l after a CholQR break)
  double cq_diag[4];  // debug: CholQR2 health of the last panel (min pivot ratio 1, |G2 - I|, min pivot ratio 2, jstar)
  // look-ahead (la): step k's C -= Y Wt on the rows below its R is still
  // pending (pend) for every trailing column not flagged in the per-column
  // `upd` bytes; snapshot of that step (its n_s and accepted reflectors)
  int32_t la, pend, pend_ns, pend_l;
  int32_t gcount;   // look-ahead guard columns of the current step (k_guard's list)
  // the CholeskyQR2 panel publishes Q1 = P R1^-1 for the spare-SM G = Q1^T C:
  // q1_count CTAs have written their rows (q1_fail: no usable Q1 this step)
  uint32_t q1_count;
  int32_t q1_fail, q1_kk;
  int32_t pend_done;  // k_guard finished the whole update of this step (nothing pending)
  // P-mode look-ahead: the panel's ranks copied P (p_k columns) into pg before
  // factoring it; k_spare forms G = P^T C at once and k_trail_w folds R1^-T into MT
  uint32_t p_count;
  int32_t p_k, pad5;
  // blocked scalar pivoting (k_qp3): columns factored by the last launch and why it ended
  int32_t qp_cols, qp_exit;
  uint32_t m_pub;  // k_panel_cq: step_idx + 1 once M (Y = Q1 M) and l are final
  int32_t posted;  // host poll records posted so far (k_step_end / k_qp3_post): the enqueue index
  // inter-CTA counters (reset by their users)
  uint32_t gram_count;
  uint32_t bar_count;
  uint32_t bar_gen;
  uint32_t trace_bits_lo, trace_bits_hi;
  uint32_t pad1[3];
  // wide selection (k_dm > DMQR_MAXK - 1, wide.cuh): one deviation-maximization
  // step of more than DMQR_MAXK selected columns runs as consecutive panel
  // chunks without a new selection.  w_total: the step's k_s; w_done: columns
  // accepted by its chunks so far; w_next: columns the next chunk continues
  // with (0: the step is over); w_cont: the current chunk continues a step;
  // w_ns0: the step's n_s; w_nmv: column moves of its swap plan
  int32_t w_total, w_done, w_next, w_cont, w_ns0, w_nmv;
  // fixed at init (k_init): the per-matrix block stride of a batched launch
  // (zshift) and the debug timeline buffer in the workspace (null: off)
  int64_t zstride;
  unsigned long long* tl;
};

// Workspace buffers of the wide selection (k_dm > DMQR_MAXK - 1, wide.cuh),
// sized for W = 1 + min(k_dm, n - 1) candidates (WP = W rounded up to 32)
struct WideBufs {
  int32_t* cand;     // [W] candidates, seed first (absolute columns)
  int32_t* list_i;   // [W] candidate list before the sort
  double* list_u;    // [W]
  double* gpart;     // [nsplit][WP][WP] Gram partials (upper tiles)
  double* theta;     // [WP][WP] cosines (when they do not fit in shared memory)
  double* vec;       // [3][W] chosen / rowsum / inv (when they do not fit in shared memory)
  int32_t* pos;      // [W] positions of the selected columns during the swap plan
  int32_t* pstamp;   // [n] position-map validity (stamp = step_idx + 1)
  int32_t* pmap;     // [n] position -> index into pos
  int32_t* cstamp;   // [n] content-map validity
  int32_t* cmap;     // [n] slot -> column it holds after the transpositions
  int32_t* mv_src;   // [2W] composed moves new[dst] = old[src]
  int32_t* mv_dst;   // [2W]
  double* tmpA;      // [2W][m] moved column contents
  double* tmpu;      // [2W] moved u / uref / perm
  double* tmpr;
  int64_t* tmpp;
  int32_t W, WP, nsplit, m_tmp;
};

// Batched launches (grid.z = matrices of a batch, small matrices): every
// per-matrix buffer -- control block, workspace, matrix, outputs -- sits in a
// per-matrix block at a fixed byte stride, so a kernel shifts its pointer
// arguments by blockIdx.z * stride at entry (gridDim.z == 1: no-op).  The
// stride is read from block 0's control block (k_init stores it there; every
// later kernel of the factorization runs after k_init has completed), so no
// process-wide state is involved.
template <typename... Ts>
__device__ __forceinline__ void zshift_by(int64_t zs, Ts&... ps) {
  if (gridDim.z > 1) {
    const int64_t o = (int64_t)blockIdx.z * zs;
    ((ps = ps ? (Ts)((char*)(ps) + o) : ps), ...);
  }
}
template <typename... Ts>
__device__ __forceinline__ void zshift(const Ctl* c0, Ts&... ps) {
  if (gridDim.z > 1) zshift_by(c0->zstride, ps...);
}

// Entry snapshot of the scalar decision state.  Every field is loaded
// unconditionally and independently at kernel entry, so the loads overlap in
// one L2 round trip instead of trickling through early-exit branches (unused
// fields are dead code).  Only for values a kernel does not change itself.
struct CtlSnap {
  int64_t m, n, lda, kmax;
  double floor, stop_rhs, tau, delta, umax;
  int32_t stop_active, break_check, k_dm, use_delta_max, trace_norms, swap_cap, step_cap;
  int32_t n_s, done, step_idx, n_swaps, kind, k_max, nsel, k_s, l_acc, ncand, nsw, nmv;
  int32_t cq_fail, tc0, la, pend, pend_ns, pend_l, q1_fail, q1_kk, w_cont;
  unsigned long long* tl;
};
// (GPU-scope relaxed loads in volatile asm: the control block is written by
// the kernels around this one, which may still be running under programmatic
// dependent launch, so these loads must neither take the read-only path nor
// move above griddepcontrol.wait.  A C++ `volatile` read would compile to
// LDG.STRONG.SYS, which measured 35% slower end to end on cfg2.)
__device__ __forceinline__ int32_t ctl_ld(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t ctl_ld(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t ctl_ld(const int64_t* p) {
  int64_t v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ctl_ld(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <class T>
__device__ __forceinline__ T* ctl_ld(T* const* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p));
  return reinterpret_cast<T*>(v);
}
__device__ __forceinline__ CtlSnap snap_load(const Ctl* c) {
  CtlSnap s;
#define CTL_LD(f) s.f = ctl_ld(&c->f)
  CTL_LD(m); CTL_LD(n); CTL_LD(lda); CTL_LD(kmax);
  CTL_LD(floor); CTL_LD(stop_rhs); CTL_LD(tau); CTL_LD(delta); CTL_LD(umax);
  CTL_LD(stop_active); CTL_LD(break_check); CTL_LD(k_dm); CTL_LD(use_delta_max); CTL_LD(trace_norms);
  CTL_LD(swap_cap); CTL_LD(step_cap); CTL_LD(n_s); CTL_LD(done); CTL_LD(step_idx); CTL_LD(n_swaps);
  CTL_LD(kind); CTL_LD(k_max); CTL_LD(nsel); CTL_LD(k_s); CTL_LD(l_acc);
  CTL_LD(ncand); CTL_LD(nsw); CTL_LD(nmv); CTL_LD(cq_fail); CTL_LD(tc0);
  CTL_LD(la); CTL_LD(pend); CTL_LD(pend_ns); CTL_LD(pend_l);
  CTL_LD(q1_fail); CTL_LD(q1_kk); CTL_LD(w_cont); CTL_LD(tl);
#undef CTL_LD
  return s;
}
// The CTA's snapshot: thread 0 loads it and every thread reads the same copy.
// (Per-thread loads could tear: a CTA of a large grid may start while another
// CTA of the same grid -- or a concurrent kernel -- updates the control block,
// e.g. k_spare's phase 1 clearing `pend`; warps that then disagree on a
// loop bound diverge at a barrier and the CTA hangs.)  Called by every thread
// of the CTA, at top level.
__device__ __forceinline__ const CtlSnap& snap(const Ctl* c) {
  __shared__ CtlSnap s_snap;
  if (threadIdx.x == 0) s_snap = snap_load(c);
  __syncthreads();
  return s_snap;
}

// Programmatic dependent launch: the per-step kernels are launched so the
// next one may be scheduled while this one runs; each lets its dependents go
// at entry and waits for its predecessor (completion + memory) before
// touching anything.  No-ops for a normal launch.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// per-step record the host polls (pinned, mapped host memory): written by
// k_step_end with a release of seq = host enqueue index + 1
// flags: 1 done, 2 la_bad (look-ahead meets many guards: go serial), 4 the
// step was a scalar-fallback step / the blocked scalar-pivot engine continues
struct __align__(16) HostRec {
  int32_t n_s, flags, step_idx, seq;
};

// debug timeline (DMQR_TIMELINE): per step and kernel, the first CTA's start
// (after its dependency wait) and the last CTA's exit, globaltimer ns, in a
// workspace buffer of TL_WORDS words (Ctl::tl; null when the timeline is off)
constexpr int TL_WORDS = 64 * 32 + 1024;  // + k_spare per-CTA debug of step 20
struct TLSpan {
  unsigned long long* tl;
  int slot;
  __device__ __forceinline__ TLSpan(unsigned long long* t, int step, int k) : tl(t), slot(-1) {
    if (threadIdx.x == 0 && tl) {
      slot = (step & 63) * 32 + 2 * k;
      atomicMin(&tl[slot], (unsigned long long)gtimer());
    }
  }
  __device__ __forceinline__ ~TLSpan() {
    if (slot >= 0) atomicMax(&tl[slot + 1], (unsigned long long)gtimer());
  }
};

// leading dimension of the published Q1 buffer (host: lda_of), multiple of 8
__host__ __device__ __forceinline__ int64_t q1_ld(int64_t m) { return (m > 0 ? (m + 7) / 8 * 8 : 8) + 8; }

struct StepRec {  // mirrors dmqr_step in include/dmqr_b200.h
  int64_t n_s, k_selected, k_accepted, k_max;
  int32_t broke_early, fell_back_to_scalar;
  double eps_s, gamma;
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// DMMA: D(8x8) += A(8x4, row) * B(4x8, col), fp64.  Lowers to SASS DMMA.8x8x4.
// Fragments (PTX ISA, mma.m8n8k4 .f64):  a: A[lane>>2][lane&3]
//                                         b: B[lane&3][lane>>2]
//                                         c0,c1: C[lane>>2][2*(lane&3) + {0,1}]
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Scaled Euclidean norm from (sum of squares, max |x|).  Unscaled sums are exact
// enough when max|x| keeps squares normal; otherwise callers rescale (see
// column-norm kernels).  Mirrors column_norms (matrix.py:61-78) up to rounding.
__device__ __forceinline__ bool norm_range_ok(double amax) {
  return amax == 0.0 || (amax > 1e-140 && amax < 1e140);
}

// Bounded device-side waits.  Every spin on another CTA or kernel (grid
// barriers, look-ahead publications, helper passes) ticks a SpinGuard; a wait
// that has not ended after 2^21 polls (~1-2 s: no legitimate wait comes near,
// a whole cfg5 outer step takes milliseconds) traps, so the host sees a CUDA
// error instead of a hang.  One counter register and an inline trap: a call
// to a reporting function would cost the spinning kernels registers (several
// run at their register cap).  (Debug builds, -DDMQR_SPIN_REPORT, print the
// site and the polled values first.)
#ifdef DMQR_SPIN_REPORT
__device__ __noinline__ void spin_timeout(int site, long long a, long long b) {
  printf("[dmqr] device wait timed out: site %d block (%d,%d,%d) thread %d values %lld %lld\n", site,
         (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, (int)threadIdx.x, a, b);
  __trap();
}
#endif
struct SpinGuard {
  unsigned polls = 0;
  __device__ __forceinline__ void tick(int site, long long a, long long b) {
#ifdef DMQR_NO_SPIN_GUARD  // A/B builds
    if (false) {
#else
    if (++polls == (1u << 21)) {
#endif
#ifdef DMQR_SPIN_REPORT
      spin_timeout(site, a, b);
#else
      (void)site, (void)a, (void)b;
      asm volatile("trap;");
#endif
    }
  }
};

// Grid-wide barrier for cooperatively launched kernels (all CTAs co-resident):
// a monotonic arrival counter (zeroed by an earlier kernel of the step) --
// arrive with a gpu-scope release add, wait with acquire loads until the
// counter reaches `target` = (barrier ordinal) x (grid size).  No last-arriver
// reset, so the barrier completes one L2 round trip after the last arrival.
__device__ __forceinline__ void grid_sync_count(uint32_t* count, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(count) : "memory");
    uint32_t v;
    SpinGuard sg;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(count) : "memory");
      if (v >= target) break;
      sg.tick(1, v, target);
    }
  }
  __syncthreads();
}

// (legacy) generation barrier
__device__ __forceinline__ void grid_barrier(uint32_t* count, uint32_t* gen, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile uint32_t* vgen = gen;
    uint32_t g = *vgen;
    __threadfence();
    uint32_t arrived = atomicAdd(count, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(count, 0u);
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vgen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// A/B builds: -DDMQR_NO_TMA_GRAM / -DDMQR_NO_TMA_SWAP select the cp.async /
// plain-load staging of k_gram / k_swap instead of the bulk copies
#ifdef DMQR_NO_TMA_GRAM
constexpr bool kTMAGram = false;
#else
constexpr bool kTMAGram = true;
#endif
#ifdef DMQR_NO_TMA_SWAP
constexpr bool kTMASwap = false;
#else
constexpr bool kTMASwap = true;
#endif
// ---- TMA bulk copies (cp.async.bulk, SASS UBLKCP) with mbarrier completion ----
// Contiguous global <-> shared transfers done by the copy engine: one thread
// issues a whole column segment (16-byte aligned addresses, a multiple of 16
// bytes); the bytes land on an mbarrier (expect_tx / complete_tx), and the
// shared -> global direction is tracked by bulk groups.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arrive (the barrier's one expected arrival) and add `bytes` to the transaction count
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(smem)),
               "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem), "r"(smem_u32(smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the issuing thread's bulk stores have read their shared-memory source (the
// CTA may exit; the writes complete with the grid, before any dependent grid's
// griddepcontrol.wait returns)
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
// 16-byte cp.async (L2 only); src_bytes < 16 zero-fills the rest (src_bytes = 0: all zeros)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int round_up(int a, int b) { return (a + b - 1) / b * b; }

}  // namespace dmqr
