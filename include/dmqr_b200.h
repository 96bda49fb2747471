/*
 * dmqr_b200 -- C-ABI of the B200 (sm_100a) QRDM / QRDM2 rank-revealing QR.
 *
 * This is the drop-in boundary for the reference's hot path
 *   qrdm (A, params=DMParams(), stop=StopCriterion(), trace_norms=False)  rrqr.py:426-440
 *   qrdm2(A, params=DMParams(), stop=StopCriterion(), trace_norms=False)  rrqr.py:443-456
 * both of which run _qrdm_engine (rrqr.py:315-423).  The reference is a
 * Python package, so its "FFI" is the Python call itself; the binding a
 * maintainer adds (ctypes) is shown in INTEGRATION.md and implemented in
 * paper_2106_03138_b200/_lib.py.
 *
 * Conventions
 *   - All matrices are column-major float64 in DEVICE memory, leading dimension
 *     lda >= m.  Input A is overwritten with the packed factor
 *     (R upper incl. diagonal over factored columns, essential reflector
 *     parts below, raw trailing block otherwise) -- the reference's
 *     RRQRResult.packed (rrqr.py:136-146).  The reference never mutates its
 *     argument because dense() copies (matrix.py:24-34); the Python wrapper
 *     makes that copy on the device before calling in.
 *   - Every pointer argument except `params`, `info` is a device pointer.
 *   - Calls are reentrant: no global mutable state; all scratch lives in the
 *     caller's workspace.  Work is enqueued on `stream` (a cudaStream_t passed
 *     as void*); the call returns after the factorization finished (it needs
 *     the final rank on the host, like the reference).
 *   - Return value 0 = success; < 0 = error, text from dmqr_strerror().
 *     DMQR_EINVAL / DMQR_ENONFINITE map to the reference's ValueError
 *     (matrix.py:30-33, dm.py:56-62, dm.py:108-109); DMQR_ECUDA to RuntimeError.
 */
#ifndef DMQR_B200_H
#define DMQR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DMQR_OK 0
#define DMQR_EINVAL (-1)      /* bad shape / params / workspace (ValueError) */
#define DMQR_ENONFINITE (-2)  /* NaN or Inf in A (ValueError, matrix.py:32-33) */
#define DMQR_EZEROCOL (-3)    /* cosine of a zero column (ValueError, dm.py:108-109) */
#define DMQR_ECUDA (-4)       /* CUDA runtime error (RuntimeError) */
#define DMQR_ECAP (-5)        /* swap or step log capacity exceeded */

/* StopRule (rrqr.py:58-63) */
#define DMQR_STOP_EPS_N 0
#define DMQR_STOP_EPS_SQRT_N 1
#define DMQR_STOP_NONE 2

/* DMParams (dm.py:41-62) + StopCriterion (rrqr.py:66-80) + driver flags. */
typedef struct dmqr_params {
  double tau;            /* (0, 1]   default 0.15 */
  double delta;          /* [0, 1)   default 0.9  */
  double epsilon;        /* StopCriterion.epsilon, default 2^-52 */
  int32_t k_dm;          /* >= 1     default 64; above 64 the wide selection
                            kernels run (csrc/wide.cuh) and the workspace
                            grows with min(k_dm, n - 1) -- size it with the
                            same params (dmqr_workspace_bytes) */
  int32_t use_delta_max; /* 0/1 */
  int32_t stop_rule;     /* DMQR_STOP_* */
  int32_t break_check;   /* 1 = qrdm2, 0 = qrdm */
  int32_t trace_norms;   /* 1 = record _record_norm_check (rrqr.py:211-216) */
  int32_t max_steps;     /* debug: stop after this many outer steps (0 = no limit) */
} dmqr_params;

/* StepRecord (rrqr.py:83-93) + k_max (needed to replay WorkCounters). */
typedef struct dmqr_step {
  int64_t n_s;
  int64_t k_selected;
  int64_t k_accepted;
  int64_t k_max;               /* candidate-set size, -1 on a scalar fallback step */
  int32_t broke_early;
  int32_t fell_back_to_scalar;
  double eps_s;
  double gamma;
} dmqr_step;

/* Host-side summary filled at the end of a call. */
typedef struct dmqr_info {
  int64_t rank;
  int64_t n_factored;
  int64_t n_steps;
  int64_t n_swaps;
  int32_t stopped_early;
  int32_t status;
  double a_max0;
} dmqr_info;

/* Bytes of device workspace dmqr_qrdm_f64 needs for an m x n problem. */
size_t dmqr_workspace_bytes(int64_t m, int64_t n, const dmqr_params* params);

/*
 * One QRDM / QRDM2 factorization (replaces _qrdm_engine, rrqr.py:315-423).
 *   A            device, m x n column-major, lda >= m; in: matrix, out: packed factor
 *   coeffs       device, min(m,n) doubles: reflector coefficients (RRQRResult.coeffs)
 *   perm         device, n int64: Permutation.forward (matrix.py:90-152)
 *   swaps        device, 2*swap_cap int64: the Permutation swap log, (i, j) pairs
 *   steps        device, step_cap records (step_cap >= min(m,n) is always enough)
 *   norm_trace   device, step_cap doubles, or NULL (required if params->trace_norms)
 *   workspace    device, >= dmqr_workspace_bytes(m, n, params)
 *   info         host, filled on return
 */
int dmqr_qrdm_f64(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* params,
                  double* coeffs, int64_t* perm, int64_t* swaps, int64_t swap_cap,
                  dmqr_step* steps, int64_t step_cap, double* norm_trace, void* workspace,
                  size_t ws_bytes, dmqr_info* info, void* stream);

/*
 * dmqr_qrdm_f64 that also streams the packed factor to the host while it runs:
 * columns [0, n_s) are final after every outer step, so they are copied to
 * host_packed (HOST, pinned for overlap; column-major, ld host_ld >= m) on a
 * side stream as the host learns n_s; the rest follows the last step.  The
 * reference's caller gets its numpy `packed` (rrqr.py:415-423) without a
 * trailing device-to-host copy.  host_packed = NULL: same as dmqr_qrdm_f64.
 */
int dmqr_qrdm_stream_f64(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* params,
                         double* coeffs, int64_t* perm, int64_t* swaps, int64_t swap_cap,
                         dmqr_step* steps, int64_t step_cap, double* norm_trace, void* workspace,
                         size_t ws_bytes, dmqr_info* info, double* host_packed, int64_t host_ld,
                         void* stream);

/*
 * QR with greedy column pivoting (replaces qrp, rrqr.py:238-291): the pivot is
 * the trailing column of largest partial norm (first index on ties), one
 * Householder reflector per column, norms downdated with the reference's
 * guard (rrqr.py:161-186) and the same stop rules.  It runs on the blocked
 * scalar-pivot engine (delayed C -= Y F^T updates, LAPACK laqps form) that
 * also executes QRDM's scalar-fallback runs (rrqr.py:343-353).  Same buffers
 * as dmqr_qrdm_stream_f64; of `params` only stop_rule, epsilon, trace_norms
 * and max_steps are used (tau / delta / k_dm must still be valid).  Step
 * records are StepRecord(n_s=s, k_selected=1, k_accepted=1) with k_max = 0.
 */
int dmqr_qrp_f64(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* params,
                 double* coeffs, int64_t* perm, int64_t* swaps, int64_t swap_cap,
                 dmqr_step* steps, int64_t step_cap, double* norm_trace, void* workspace,
                 size_t ws_bytes, dmqr_info* info, void* stream);
int dmqr_qrp_stream_f64(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* params,
                        double* coeffs, int64_t* perm, int64_t* swaps, int64_t swap_cap,
                        dmqr_step* steps, int64_t step_cap, double* norm_trace, void* workspace,
                        size_t ws_bytes, dmqr_info* info, double* host_packed, int64_t host_ld,
                        void* stream);

/*
 * Batched QRDM / QRDM2 over `batch` independent m x n matrices stored at
 * A + b*stride (cfg3: batches of small matrices).  The batch is spread over
 * `nlanes` concurrent CUDA streams (one host thread each), joined back to
 * `stream`.  Small matrices (m*n < 2^20, lda = round_up(m, 8)) are factored
 * dmqr_batched_group(m, n) at a time per lane: every kernel of an outer step
 * is launched once for the group (grid.z), on per-matrix copies in the
 * workspace, and the step is replayed as a CUDA graph; larger matrices run
 * the single-matrix engine (dmqr_qrdm_f64) on each lane.
 * Per-matrix outputs are strided: coeffs + b*min(m,n), perm + b*n,
 * swaps + b*2*swap_cap, steps + b*step_cap (device); infos[b] (HOST).
 * workspace >= dmqr_batched_workspace_bytes(m, n, params, nlanes).
 * Returns the first non-zero per-matrix status (all matrices are attempted).
 */
size_t dmqr_batched_workspace_bytes(int64_t m, int64_t n, const dmqr_params* params, int32_t nlanes);
/* Matrices a lane factors per launch (grid.z groups of small matrices; 1 when
 * m x n is too large to batch).  Lanes beyond ceil(batch / group) stay idle, so
 * callers size the workspace for min(nlanes, ceil(batch / group)) lanes. */
int32_t dmqr_batched_group(int64_t m, int64_t n);
int dmqr_qrdm_batched_f64(double* A, int64_t batch, int64_t m, int64_t n, int64_t lda, int64_t stride,
                          const dmqr_params* params, double* coeffs, int64_t* perm, int64_t* swaps,
                          int64_t swap_cap, dmqr_step* steps, int64_t step_cap, dmqr_info* infos,
                          int32_t nlanes, void* workspace, size_t ws_bytes, void* stream);

/*
 * Explicit thin/full Q: Q (m x qcols, column-major, ldq) = H_0 H_1 ... H_{p-1} [I; 0]
 * from the packed reflectors of a finished factorization (replaces the
 * backward accumulation in reconstruct, rrqr.py:459-480).  Blocked, device.
 */
int dmqr_form_q_f64(const double* packed, int64_t m, int64_t n, int64_t lda, const double* coeffs,
                    int64_t n_factored, double* Q, int64_t qcols, int64_t ldq, void* workspace,
                    size_t ws_bytes, void* stream);
size_t dmqr_form_q_workspace_bytes(int64_t m, int64_t qcols);

/*
 * Singular values of `batch` m x n column-major device matrices (ld, `stride`
 * doubles apart; n <= 512, m >= n) by one-sided Jacobi with the reference
 * oracle's rotation and stopping rule (jacobi_svd, svd.py:117-143, sweeps
 * svd.py:74-114; round-robin pair order).  X is overwritten; sig (batch x n)
 * receives the column norms of the converged X, unsorted; sweeps / converged
 * per matrix.  Verification tooling for the ratio diagnostics
 * (harness._ratio_fields, harness.py:201-216).
 */
int dmqr_jacobi_svd_batched_f64(double* X, int64_t batch, int64_t m, int64_t n, int64_t ld, int64_t stride,
                                double tol, int32_t max_sweeps, double* sig, int32_t* sweeps, int32_t* converged,
                                void* stream);

/* 1 if any entry of the m x n column-major device matrix is NaN/Inf (dense(), matrix.py:32-33). */
int dmqr_check_finite_f64(const double* A, int64_t m, int64_t n, int64_t lda, int32_t* nonfinite,
                          void* stream);

const char* dmqr_strerror(int code);

/* Telemetry (process-wide, not decision state): number of kernels this library
 * launched, and -- when enabled -- device time per phase of the outer loop
 * measured with CUDA events on the caller's stream. */
typedef struct dmqr_stats {
  int64_t kernel_launches;
  int64_t calls;
  int64_t timed_steps;
  double ms_select;    /* stop/floor/candidates + cosine Gram + filter + swaps */
  double ms_panel;     /* Householder panel + T factor */
  double ms_trailing;  /* V = Y T^T, Z = Y^T C, C -= V Z */
  double ms_norms;     /* downdate + guard recompute + step record */
  double ms_pivot;     /* blocked scalar pivoting: qrp, and QRDM's scalar-fallback runs */
} dmqr_stats;
void dmqr_stats_enable(int32_t on);
void dmqr_stats_get(dmqr_stats* out, int32_t reset);

/* Debug: copy the device control block of a workspace (after a call) into
 * out[16 + 4*72 + 5] int64 on the device: n_s, done, stopped, status, kind, k_max,
 * ncand, nsel, k_s, l_acc, nsw, step_idx, n_swaps, bits(umax), bits(eps_s),
 * bits(gamma), cand[72], sel[72], sw_a[72], sw_b[72], bits(cq_diag[4]),
 * cq_fail * 10^6 + tc0. */
int dmqr_debug_ctl(const void* workspace, int64_t* out, void* stream);
/* Debug: per-reflector phase clocks (clock64) of one panel CTA at step 2, recorded
 * when dmqr_stats_enable(2) was set; out = 64 x 8 int64 on the host. */
int dmqr_debug_panel_clocks(const void* workspace, int64_t m, int64_t n, int64_t* out);
/* debug: kernel spans per step of the last factorization run in `workspace`
 * (sized for m x n) with DMQR_TIMELINE set (out[64 * 32 + 1024] int64 on the
 * host, globaltimer ns; see the source) */
int dmqr_debug_timeline(const void* workspace, int64_t m, int64_t n, int64_t* out);
/* debug: CTA 0's per-phase cycle counts of the last fused small-matrix launch
 * run with DMQR_SMALL_CLOCKS set (out[32] int64 on the host) */
int dmqr_debug_small_clocks(int64_t* out);
/* Free the library's pooled pinned poll records, events and copy streams (all
 * devices).  Optional; only while no call is running.  The pool holds one entry
 * per concurrently running engine call. */
void dmqr_release_resources(void);

/* Build identification (compile arch, version) for logs and the loader check. */
const char* dmqr_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DMQR_B200_H */
