// dmqr_b200: host driver + C-ABI (include/dmqr_b200.h) for the B200 QRDM engine.
//
// The outer loop of _qrdm_engine (rrqr.py:315-423) runs as a fixed sequence of
// stream-ordered kernels per step; every decision (stop, floor/fallback,
// candidates, filter, swaps, break, n_s advance) is taken ON THE DEVICE and
// kept in the Ctl block, so the host only sizes grids and watches for `done`.
// Kernels early-exit once `done` is set, which lets the host enqueue several
// steps ahead of the last n_s it has seen (grids are sized from that stale
// n_s, an upper bound on the remaining work).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <thread>
#include <vector>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>

#include "../../include/dmqr_b200.h"
#include "common.cuh"
#include "gram.cuh"
#include "misc.cuh"
#include "norms.cuh"
#include "panel.cuh"
#include "panel_rr.cuh"
#include "panel_cq.cuh"
#include "select.cuh"
#include "trailing.cuh"
#include "tail.cuh"
#include "qp3.cuh"
#include "formq.cuh"
#include "small.cuh"
#include "jacobi.cuh"
#include "wide.cuh"

using namespace dmqr;

namespace {

constexpr int GRAM_GMAX = 148;
constexpr int NSPLIT_MAX = 16;  // split-K partials of Y^T C (k_spare's G: at most this many)
int64_t ldz_for(int64_t n);
// k_trail_a's split count cap: 16, or up to 64 when the partials stay small
// (few columns: a tall input like cfg4, 65536 x 1024, has only 16 column tiles
// and needs the row splits to fill the GPU)
int nsplit_cap(int64_t n) {
  const int64_t per = (int64_t)sizeof(double) * DMQR_KP * ldz_for(n);
  return (int)std::clamp<int64_t>(((int64_t)64 << 20) / per, NSPLIT_MAX, 64);
}
constexpr int PANEL_PMAX = 160;

struct Layout {
  size_t ctl, u, uref, T, red, gram, gfin, Zp, Z, trace, pdbg, tcount, upd, lacount, q1g, pg, glist;
  size_t qvb, qwb, qpart, qgpart, qcnt, hpart, hR, hctr, gnp, tl;
  // wide selection (k_dm > WIDE_K): W candidates, WP = W rounded to 32
  int W, WP, wsplit;
  size_t wcand, wlist_i, wlist_u, wgpart, wtheta, wvec, wpos, wpstamp, wpmap, wcstamp, wcmap, wmv_src, wmv_dst, wtmpA,
      wtmpu, wtmpr, wtmpp;
  size_t total;
};

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// leading dimension of the Z partials / Wt: 16-byte aligned rows with one tile of slack
int64_t ldz_for(int64_t n) { return (std::max<int64_t>(n, 1) + 7) / 8 * 8 + 64; }


Layout layout(int64_t m, int64_t n, int64_t k_dm = 0) {
  Layout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += al(bytes);
    return o;
  };
  L.ctl = take(sizeof(Ctl));
  L.u = take(sizeof(double) * std::max<int64_t>(n, 1));
  L.uref = take(sizeof(double) * std::max<int64_t>(n, 1));
  L.T = take(sizeof(double) * DMQR_KP * DMQR_KP);
  // panel all-reduce partials; the CholeskyQR2 panel also keeps R, Y1 and per-rank R = R2 R1 here
  L.red = take(sizeof(double) * std::max<size_t>(2 * PANEL_PMAX * RED_LD, 39 * DMQR_KP * DMQR_KP));
  L.gram = take(sizeof(double) * GRAM_GMAX * GRAM_PART);
  L.gfin = take(sizeof(double) * DMQR_KP * DMQR_KP);
  L.Zp = take(sizeof(double) * nsplit_cap(n) * DMQR_KP * ldz_for(n));
  L.Z = take(sizeof(double) * DMQR_KP * ldz_for(n));
  L.trace = take(sizeof(unsigned long long) * 4);
  L.pdbg = take(sizeof(long long) * 64 * 16);
  L.tcount = take(sizeof(unsigned) * 2 * (ceil_div(std::max<int64_t>(n, 1), TA_COLS) + 1));  // + k_spare's column counts
  L.upd = take(std::max<int64_t>(n, 1));                      // look-ahead column flags
  L.lacount = take(sizeof(unsigned) * 16);                    // look-ahead work / last-CTA counters
  L.q1g = take(sizeof(double) * DMQR_KP * q1_ld(m));  // published Q1 (k_spare)
  L.pg = take(sizeof(double) * DMQR_KP * q1_ld(m));   // P copy (k_spare, P-mode look-ahead)
  L.glist = take(sizeof(int32_t) * std::max<int64_t>(n, 1));  // look-ahead / k_qp3 guard columns
  // blocked scalar pivoting (k_qp3; its F = Zp, its Wt = Z: both are free between steps)
  L.qvb = take(sizeof(double) * std::max<int64_t>(m, 1));
  L.qwb = take(sizeof(double) * std::max<int64_t>(n, 1) * QP_RMAX);
  L.qpart = take(sizeof(double) * QP_GMAXCTA * QP_PLD);
  L.qgpart = take(sizeof(double) * (QP_GMAXCTA * QP_GMAX * 2 + QP_GMAX));  // + the fresh guard norms
  L.qcnt = take(sizeof(unsigned) * 4);
  // tall-panel helpers (k_panel_helper): per-256-row-chunk Gram partials, R1^-1, counters
  L.hpart = take(sizeof(double) * DMQR_KP * DMQR_KP * (size_t)std::max<int64_t>(1, (m + 255) / 256));
  L.hR = take(sizeof(double) * (DMQR_KP * DMQR_KP + 2));
  L.hctr = take(sizeof(unsigned) * 8);
  // serial guard norms: (column, 4096-row chunk) partials
  L.gnp = take(sizeof(double) * 2 * (size_t)std::max<int64_t>(n, 1) * (size_t)std::max<int64_t>(1, (m + GN_ROWS - 1) / GN_ROWS));
  L.tl = take(sizeof(unsigned long long) * TL_WORDS);  // debug timeline (DMQR_TIMELINE)
  if (k_dm > WIDE_K) {  // wide selection buffers (wide.cuh)
    const int64_t W = 1 + std::min<int64_t>(k_dm, std::max<int64_t>(n - 1, 0));
    const int64_t WP = (W + 31) / 32 * 32;
    const int64_t nt = WP / 32, tiles = nt * (nt + 1) / 2;
    L.W = (int)W;
    L.WP = (int)WP;
    L.wsplit = (int)std::clamp<int64_t>(ceil_div(296, tiles), 1, WIDE_SPLIT_MAX);
    const size_t nn = (size_t)std::max<int64_t>(n, 1), mm = (size_t)std::max<int64_t>(m, 1);
    L.wcand = take(sizeof(int32_t) * W);
    L.wlist_i = take(sizeof(int32_t) * W);
    L.wlist_u = take(sizeof(double) * W);
    L.wgpart = take(sizeof(double) * (size_t)L.wsplit * WP * WP);
    L.wtheta = take(sizeof(double) * (size_t)WP * WP);
    L.wvec = take(sizeof(double) * 3 * (size_t)W);
    L.wpos = take(sizeof(int32_t) * W);
    L.wpstamp = take(sizeof(int32_t) * nn);
    L.wpmap = take(sizeof(int32_t) * nn);
    L.wcstamp = take(sizeof(int32_t) * nn);
    L.wcmap = take(sizeof(int32_t) * nn);
    L.wmv_src = take(sizeof(int32_t) * 2 * W);
    L.wmv_dst = take(sizeof(int32_t) * 2 * W);
    L.wtmpA = take(sizeof(double) * 2 * (size_t)W * mm);
    L.wtmpu = take(sizeof(double) * 2 * W);
    L.wtmpr = take(sizeof(double) * 2 * W);
    L.wtmpp = take(sizeof(int64_t) * 2 * W);
  }
  L.total = off;
  return L;
}

struct DevInfo {
  int sms = 148;
  int coop = 1;
  size_t smem_optin = 227 * 1024;
};

DevInfo dev_info() {
  DevInfo d;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&d.coop, cudaDevAttrCooperativeLaunch, dev);
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  d.smem_optin = (size_t)v;
  return d;
}

#define CK(x)                                        \
  do {                                               \
    cudaError_t e_ = (x);                            \
    if (e_ != cudaSuccess) {                         \
      last_cuda_error() = e_;                        \
      return DMQR_ECUDA;                             \
    }                                                \
  } while (0)

cudaError_t& last_cuda_error() {
  static thread_local cudaError_t e = cudaSuccess;
  return e;
}

// Function attributes apply per device, so they are set once per device id
// (the first call on a device), together with the launch limits derived from
// them.  Read-only once `done` is published.
struct DevAttrs {
  std::atomic<bool> done{false};
  bool cluster16 = false;
  int qp_grid = 1;  // k_qp3 cooperative grid (all CTAs co-resident)
};
constexpr int kMaxDevices = 64;
DevAttrs g_dev_attrs[kMaxDevices];
std::mutex g_attr_mu;

int set_attrs(const DevInfo& d, DevAttrs** out) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return DMQR_EINVAL;
  DevAttrs& A = g_dev_attrs[dev];
  *out = &A;
  if (A.done.load(std::memory_order_acquire)) return 0;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (A.done.load(std::memory_order_relaxed)) return 0;
  bool& cluster16 = A.cluster16;
  int& qp_grid = A.qp_grid;
  CK(cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GRAM_SMEM));
  CK(cudaFuncSetAttribute(k_trail_a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TA_SMEM));
  CK(cudaFuncSetAttribute(k_gram_finish, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FinSmem)));
  CK(cudaFuncSetAttribute(k_trail_b<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TB_SMEM));
  CK(cudaFuncSetAttribute(k_trail_b<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TB_SMEM));
  CK(cudaFuncSetAttribute(k_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TAIL_SMEM));
  CK(cudaFuncSetAttribute(k_spare<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SP_SMEM));
  CK(cudaFuncSetAttribute(k_spare<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SP_SMEM));
  CK(cudaFuncSetAttribute(k_trail_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TW_SMEM));
  CK(cudaFuncSetAttribute(k_guard, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GU_SMEM));
  CK(cudaFuncSetAttribute(k_ygemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)YG_SMEM));
  CK(cudaFuncSetAttribute(k_qp3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)QP_SMEM));
  CK(cudaFuncSetAttribute(k_panel_helper, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CQH_SMEM));
  CK(cudaFuncSetAttribute(k_fq_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FQ_SMEM2));
  CK(cudaFuncSetAttribute(k_fq_tw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FQ_SMEM2));
  CK(cudaFuncSetAttribute(k_fq_upd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FQ_SMEM2));
  CK(cudaFuncSetAttribute(k_small_qrdm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SM_SMEM));
  {
    int nb = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_qp3, QP_T, QP_SMEM));
    qp_grid = std::max(1, std::min(nb * d.sms, QP_GMAXCTA));
  }
  CK(cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)std::min<size_t>(d.smem_optin - 4096, 220 * 1024)));
  CK(cudaFuncSetAttribute(k_panel_rr<ClusterRed>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RR_CL_SMEM));
  CK(cudaFuncSetAttribute(k_panel_cq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CQ_SMEM));
  cudaFuncSetAttribute(k_panel_cq, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  // 16-CTA (non-portable) clusters for the register-resident panel
  if (cudaFuncSetAttribute(k_panel_rr<ClusterRed>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
      cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(PANEL_T);
    cfg.dynamicSmemBytes = RR_CL_SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cluster16 = cudaOccupancyMaxActiveClusters(&ncl, k_panel_rr<ClusterRed>, &cfg) == cudaSuccess && ncl >= 1;
  }
  cudaGetLastError();
  A.done.store(true, std::memory_order_release);
  return 0;
}

// Pinned poll records, their events and the packed-factor copy stream of one
// engine call, recycled through a small per-device pool (an engine call holds
// one entry for its duration; entries live until dmqr_release_resources or
// process exit, so repeated calls -- from any thread -- allocate nothing).
struct HostSlot {
  int dev = -1;
  HostRec* rec = nullptr;            // two records
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t copy = nullptr;       // created on first use
};
std::mutex g_slot_mu;
std::vector<HostSlot*> g_slot_free;
std::vector<HostSlot*> g_slot_all;

HostSlot* slot_acquire(int dev) {
  {
    std::lock_guard<std::mutex> lk(g_slot_mu);
    for (size_t i = 0; i < g_slot_free.size(); ++i)
      if (g_slot_free[i]->dev == dev) {
        HostSlot* h = g_slot_free[i];
        g_slot_free.erase(g_slot_free.begin() + (long)i);
        return h;
      }
  }
  HostSlot* h = new HostSlot;
  h->dev = dev;
  if (cudaMallocHost(&h->rec, 2 * sizeof(HostRec)) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev[0], cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev[1], cudaEventDisableTiming) != cudaSuccess) {
    last_cuda_error() = cudaGetLastError();
    if (h->rec) cudaFreeHost(h->rec);
    for (auto e : h->ev)
      if (e) cudaEventDestroy(e);
    delete h;
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_slot_mu);
  g_slot_all.push_back(h);
  return h;
}
void slot_release(HostSlot* h) {
  if (!h) return;
  std::lock_guard<std::mutex> lk(g_slot_mu);
  g_slot_free.push_back(h);
}
struct SlotGuard {
  HostSlot* h;
  ~SlotGuard() { slot_release(h); }
};



int validate(int64_t m, int64_t n, int64_t lda, const dmqr_params* p) {
  if (!p) return DMQR_EINVAL;
  if (m < 0 || n < 0 || lda < std::max<int64_t>(1, m)) return DMQR_EINVAL;
  if (!(p->tau > 0.0 && p->tau <= 1.0)) return DMQR_EINVAL;
  if (!(p->delta >= 0.0 && p->delta < 1.0)) return DMQR_EINVAL;
  if (p->k_dm < 1) return DMQR_EINVAL;  // (k_dm > 64: wide selection, wide.cuh)
  if (p->stop_rule < 0 || p->stop_rule > 2) return DMQR_EINVAL;
  if (m > 0x7fffffffLL || n > 0x7fffffffLL) return DMQR_EINVAL;
  return 0;
}

// ---- telemetry (not decision state): launch counter and optional phase timing ----
std::atomic<long long> g_launches{0};
std::atomic<long long> g_calls{0};
std::atomic<int> g_prof{0};
struct ProfAcc {
  double ms[5] = {0, 0, 0, 0, 0};  // select+gram+swap, panel, trailing update, downdate+log, scalar pivoting
  long long steps = 0;
};
ProfAcc g_acc;  // guarded by the caller (bench) using one thread
#define NOTE_LAUNCH() g_launches.fetch_add(1, std::memory_order_relaxed)

long long* g_small_clk = nullptr;  // debug (DMQR_SMALL_CLOCKS): device phase-cycle slots
// Small matrices (m <= 256, n <= 512, k_dm <= 64) run the whole factorization
// in one fused kernel per matrix (small.cuh); DMQR_NO_FUSED forces the
// per-step kernels (tests compare both).
bool small_eligible(int64_t m, int64_t n, const dmqr_params* p) {
  return m <= SM_MMAX && n <= SM_NMAX && p->k_dm <= SM_KC - 1 && !p->trace_norms && p->max_steps <= 0 &&
         getenv("DMQR_NO_FUSED") == nullptr;
}
size_t small_info_bytes(int64_t batch) { return al(sizeof(SmallInfo) * (size_t)std::max<int64_t>(batch, 1)); }

// Launch the fused kernel over `batch` matrices (stride doubles apart) and fill
// the host infos; dinfo: device scratch of small_info_bytes(batch).
int run_small(double* A, int64_t batch, int64_t m, int64_t n, int64_t lda, int64_t stride, const dmqr_params* p,
              double* coeffs, int64_t* perm, int64_t* swaps, int64_t swap_cap, dmqr_step* steps, int64_t step_cap,
              SmallInfo* dinfo, dmqr_info* infos, cudaStream_t st, int sms) {
  if (batch <= 0) return 0;
  double eps1 = -1.0;
  if (p->stop_rule == DMQR_STOP_EPS_N) eps1 = p->epsilon * (double)n;
  if (p->stop_rule == DMQR_STOP_EPS_SQRT_N) eps1 = p->epsilon * std::sqrt((double)n);
  SmallArgs sa{A, batch, m, n, lda, stride, p->tau, p->delta, eps1, p->k_dm, p->use_delta_max, p->break_check,
               p->stop_rule == DMQR_STOP_NONE ? 1 : 0, coeffs, perm, swaps, swap_cap, (StepRec*)steps,
               std::max<int64_t>(step_cap, 0), dinfo, nullptr};
  if (getenv("DMQR_SMALL_CLOCKS")) {  // debug: CTA 0's phase cycles (tools/small_clocks.py)
    static long long* dclk = nullptr;  // (debug only)
    if (!dclk) CK(cudaMalloc(&dclk, sizeof(long long) * 32));
    CK(cudaMemsetAsync(dclk, 0, sizeof(long long) * 32, st));
    sa.dbg = dclk;
    g_small_clk = dclk;
  }
  const unsigned grid = (unsigned)std::min<int64_t>(batch, (int64_t)sms);
  k_small_qrdm<<<grid, SM_T, SM_SMEM, st>>>(sa);
  NOTE_LAUNCH();
  CK(cudaGetLastError());
  std::vector<SmallInfo> h((size_t)batch);
  CK(cudaMemcpyAsync(h.data(), dinfo, sizeof(SmallInfo) * (size_t)batch, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int rc = 0;
  for (int64_t b = 0; b < batch; ++b) {
    dmqr_info& in = infos[b];
    in.rank = h[b].rank;
    in.n_factored = h[b].n_factored;
    in.n_steps = h[b].n_steps;
    in.n_swaps = h[b].n_swaps;
    in.stopped_early = h[b].stopped;
    in.status = h[b].status;
    in.a_max0 = h[b].a_max0;
    if (!rc && h[b].status) rc = h[b].status;
  }
  return rc;
}

// Split-K count for `ntile` column tiles on `slots` concurrent CTAs: the
// number of splits (1..maxsplit) whose item count fills its waves best
// (items / (waves x slots)); ties go to fewer splits (less partial traffic).
int choose_nsplit(int64_t ntile, int slots, int maxsplit) {
  int best = 1;
  double best_eff = -1.0;
  for (int sp = 1; sp <= std::max(1, maxsplit); ++sp) {
    const int64_t items = ntile * sp;
    const int64_t waves = (items + slots - 1) / slots;
    const double eff = (double)items / (double)(waves * slots);
    if (eff > best_eff + 1e-9) {
      best_eff = eff;
      best = sp;
    }
  }
  return best;
}

// Launch with programmatic stream serialization: the kernel may be scheduled
// while its predecessor runs (it waits in pdl_enter before touching memory).
template <typename... KArgs, typename... Args>
cudaError_t pdl_launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}


}  // namespace

extern "C" {

const char* dmqr_version(void) {
  return "dmqr_b200 0.1 (sm_100a, fp64 DMMA)";
}

const char* dmqr_strerror(int code) {
  switch (code) {
    case DMQR_OK: return "ok";
    case DMQR_EINVAL: return "invalid argument (shape, lda, params or workspace)";
    case DMQR_ENONFINITE: return "matrix contains NaN or Inf entries";
    case DMQR_EZEROCOL: return "cosine matrix undefined: zero column present";
    case DMQR_ECUDA: return cudaGetErrorString(last_cuda_error());
    case DMQR_ECAP: return "swap or step log capacity exceeded";
    default: return "unknown error";
  }
}

size_t dmqr_workspace_bytes(int64_t m, int64_t n, const dmqr_params* params) {
  return layout(m, n, params ? params->k_dm : 0).total;
}

int dmqr_check_finite_f64(const double* A, int64_t m, int64_t n, int64_t lda, int32_t* nonfinite, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), st));
  if (m > 0 && n > 0) {
    int64_t blocks = std::min<int64_t>(ceil_div(n * 32, 256), 148 * 16);
    k_check_finite<<<(unsigned)blocks, 256, 0, st>>>(A, m, n, lda, nonfinite);
    NOTE_LAUNCH();
    CK(cudaGetLastError());
  }
  return 0;
}

int dmqr_qrdm_f64(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* p, double* coeffs, int64_t* perm,
                  int64_t* swaps, int64_t swap_cap, dmqr_step* steps, int64_t step_cap, double* norm_trace,
                  void* workspace, size_t ws_bytes, dmqr_info* info, void* stream) {
  return dmqr_qrdm_stream_f64(A, m, n, lda, p, coeffs, perm, swaps, swap_cap, steps, step_cap, norm_trace,
                              workspace, ws_bytes, info, nullptr, 0, stream);
}

}  // extern "C"

namespace {
// A lane's replayable outer step (small matrices in a batch): the step's
// kernel sequence captured once as a CUDA graph with grids sized for the
// whole matrix (kernels take the true extents from Ctl and exit surplus
// CTAs; the poll record's index is counted on the device), then replayed with
// one graph launch per step.  Valid while every argument baked into the
// launches is unchanged -- the batched driver factors each of a lane's
// matrices in the same lane-private buffers.
struct StepGraph {
  cudaGraphExec_t exec = nullptr;
  std::vector<unsigned char> key;
  ~StepGraph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

// The engine behind dmqr_qrdm*_f64 (qrp = 0) and dmqr_qrp*_f64 (qrp = 1).
int run_engine(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* p, double* coeffs, int64_t* perm,
               int64_t* swaps, int64_t swap_cap, dmqr_step* steps, int64_t step_cap, double* norm_trace,
               void* workspace, size_t ws_bytes, dmqr_info* info, double* host_packed, int64_t host_ld, void* stream,
               int qrp, StepGraph* sgraph = nullptr, int nz = 1, int64_t zs = 0, HostRec* zrec = nullptr) {
  // nz > 1: a batch of nz matrices in per-matrix blocks zs bytes apart (all
  // pointers are block 0's; kernels shift by blockIdx.z * zs, grids get z = nz);
  // small matrices, serial schedule, no streaming / trace / scalar-pivot engine;
  // zrec: nz pairs of pinned poll records
  const unsigned NZ = (unsigned)std::max(1, nz);
  if (nz > 1 && (qrp || p->trace_norms || host_packed || !zrec)) return DMQR_EINVAL;
  if (host_packed && host_ld < m) return DMQR_EINVAL;
  int rc = validate(m, n, lda, p);
  if (rc) return rc;
  if (!info) return DMQR_EINVAL;
  const bool wide = !qrp && p->k_dm > WIDE_K;  // wide selection (wide.cuh)
  if (wide && nz > 1) return DMQR_EINVAL;
  const Layout L = layout(m, n, qrp ? 0 : p->k_dm);
  if (ws_bytes < L.total || !workspace) return DMQR_EINVAL;
  if (p->trace_norms && !norm_trace) return DMQR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const DevInfo d = dev_info();
  DevAttrs* da = nullptr;
  if ((rc = set_attrs(d, &da))) return rc;
  if (!qrp && NZ == 1 && !sgraph && small_eligible(m, n, p) && L.total >= small_info_bytes(1)) {
    // one small matrix: the fused kernel (no per-step launches, no host polling)
    rc = run_small(A, 1, m, n, lda, lda * std::max<int64_t>(n, 1), p, coeffs, perm, swaps, swap_cap, steps, step_cap,
                   (SmallInfo*)workspace, info, st, d.sms);
    if (rc == DMQR_ECUDA) return rc;
    if (host_packed && m > 0 && n > 0) {
      CK(cudaMemcpy2DAsync(host_packed, sizeof(double) * host_ld, A, sizeof(double) * lda, sizeof(double) * m,
                           (size_t)n, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
    g_calls.fetch_add(1);
    return rc;
  }
  const bool cluster16 = da->cluster16;
  const int qp_grid = da->qp_grid;

  unsigned char* ws = (unsigned char*)workspace;
  Ctl* ctl = (Ctl*)(ws + L.ctl);
  double* u = (double*)(ws + L.u);
  double* uref = (double*)(ws + L.uref);
  double* T = (double*)(ws + L.T);
  double* red = (double*)(ws + L.red);
  double* gpart = (double*)(ws + L.gram);
  double* gfin = (double*)(ws + L.gfin);
  double* Zp = (double*)(ws + L.Zp);
  double* Z = (double*)(ws + L.Z);
  unsigned long long* tbits = (unsigned long long*)(ws + L.trace);
  long long* pdbg = (long long*)(ws + L.pdbg);
  unsigned* tcount = (unsigned*)(ws + L.tcount);
  uint8_t* upd = (uint8_t*)(ws + L.upd);
  double* q1g = (double*)(ws + L.q1g);
  unsigned* qcnt = (unsigned*)(ws + L.qcnt);
  double* gnp = (double*)(ws + L.gnp);
  int32_t* glist = (int32_t*)(ws + L.glist);
  unsigned* lacount = (unsigned*)(ws + L.lacount);
  StepRec* srec = (StepRec*)steps;
  WideBufs wb{};
  int wf_smode = 0;
  if (wide) {
    wb.cand = (int32_t*)(ws + L.wcand);
    wb.list_i = (int32_t*)(ws + L.wlist_i);
    wb.list_u = (double*)(ws + L.wlist_u);
    wb.gpart = (double*)(ws + L.wgpart);
    wb.theta = (double*)(ws + L.wtheta);
    wb.vec = (double*)(ws + L.wvec);
    wb.pos = (int32_t*)(ws + L.wpos);
    wb.pstamp = (int32_t*)(ws + L.wpstamp);
    wb.pmap = (int32_t*)(ws + L.wpmap);
    wb.cstamp = (int32_t*)(ws + L.wcstamp);
    wb.cmap = (int32_t*)(ws + L.wcmap);
    wb.mv_src = (int32_t*)(ws + L.wmv_src);
    wb.mv_dst = (int32_t*)(ws + L.wmv_dst);
    wb.tmpA = (double*)(ws + L.wtmpA);
    wb.tmpu = (double*)(ws + L.wtmpu);
    wb.tmpr = (double*)(ws + L.wtmpr);
    wb.tmpp = (int64_t*)(ws + L.wtmpp);
    wb.W = L.W;
    wb.WP = L.WP;
    wb.nsplit = L.wsplit;
    wb.m_tmp = (int32_t)std::max<int64_t>(m, 1);
    const size_t cap = std::min<size_t>(d.smem_optin, 200 * 1024);
    wf_smode = wfin_smem(L.W, 2) <= cap ? 2 : (wfin_smem(L.W, 1) <= cap ? 1 : 0);
    CK(cudaFuncSetAttribute(k_wfin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wfin_smem(L.W, wf_smode)));
    // stamps from an earlier call on this workspace must not match this one's
    CK(cudaMemsetAsync(wb.pstamp, 0, sizeof(int32_t) * std::max<int64_t>(n, 1), st));
    CK(cudaMemsetAsync(wb.cstamp, 0, sizeof(int32_t) * std::max<int64_t>(n, 1), st));
  }
  // Look-ahead (default; not with the per-step norm trace, which needs fully
  // updated columns at every step end): step k's C -= Y Wt below its R rows
  // runs beside step k+1's panel (programmatic dependent launch); step k+1's
  // candidates get it first (in k_gram).
  // (small problems -- e.g. the 256^2 batch of cfg3 -- are launch-bound: serial form)
  // (tall inputs -- m > 4n, like cfg4 -- hit norm guards too often: serial)
  // (past n = 12288 the trailing update outweighs the panel it would hide, and
  // graded inputs make its guard path expensive: serial -- measured on cfg2 /
  // cfg5 at 8192, 12288, 16384)
  const bool la_force = getenv("DMQR_FORCE_LOOKAHEAD") != nullptr;  // A/B switch: look-ahead at any shape
  const bool la_all = !qrp && !p->trace_norms && getenv("DMQR_NO_LOOKAHEAD") == nullptr &&
                      m * n >= (int64_t)1 << 20 && ((m <= 4 * n && n <= 12288) || la_force) && NZ == 1 && !wide;


  const int64_t kmax = std::min(m, n);
  double eps1 = -1.0;
  if (p->stop_rule == DMQR_STOP_EPS_N) eps1 = p->epsilon * (double)n;
  if (p->stop_rule == DMQR_STOP_EPS_SQRT_N) eps1 = p->epsilon * std::sqrt((double)n);

  auto zmemset = [&](void* ptr, size_t bytes) -> cudaError_t {
    return NZ > 1 ? cudaMemset2DAsync(ptr, (size_t)zs, 0, bytes, NZ, st) : cudaMemsetAsync(ptr, 0, bytes, st);
  };
  CK(zmemset(ws, L.ctl + sizeof(Ctl)));
  CK(zmemset(tbits, sizeof(unsigned long long) * 4));
  int32_t* nonfinite = (int32_t*)(tbits + 2);
  CK(zmemset(T, sizeof(double) * DMQR_KP * DMQR_KP));
  CK(zmemset(tcount, sizeof(unsigned) * 2 * (ceil_div(std::max<int64_t>(n, 1), TA_COLS) + 1)));
  CK(zmemset(upd, (size_t)std::max<int64_t>(n, 1)));
  CK(zmemset(lacount, sizeof(unsigned) * 16));
  if (n > 0) {
    if (m > 0) {
      // tall columns: (column, 4096-row chunk) items, combined by k_colnorms_fin
      const int nch = (NZ == 1 && m > 2 * GN_ROWS) ? (int)ceil_div(m, GN_ROWS) : 1;
      double* gpn = (double*)(ws + L.gnp);
      int64_t blocks = std::min<int64_t>(ceil_div(n * nch * 32, 256), (int64_t)d.sms * 16);
      k_colnorms_init<<<dim3((unsigned)blocks, 1, NZ), 256, 0, st>>>(A, m, n, lda, u, uref, nonfinite, zs, gpn, nch);
      NOTE_LAUNCH();
      if (nch > 1) {
        k_colnorms_fin<<<(unsigned)std::min<int64_t>(ceil_div(n * 32, 256), (int64_t)d.sms * 16), 256, 0, st>>>(
            A, m, n, lda, u, uref, nonfinite, gpn, nch);
        NOTE_LAUNCH();
      }
    } else {
      CK(zmemset(u, sizeof(double) * n));
      CK(zmemset(uref, sizeof(double) * n));
    }
  }
  long long* tline = (getenv("DMQR_TIMELINE") && NZ == 1) ? pdbg : nullptr;  // debug: panel / k_spare timestamps
  unsigned long long* tlbuf = tline ? (unsigned long long*)(ws + L.tl) : nullptr;
  if (tlbuf) {
    k_tl_init<<<(TL_WORDS + 255) / 256, 256, 0, st>>>(tlbuf);
    NOTE_LAUNCH();
  }
  InitArgs ia{ctl, u, perm, coeffs, m, n, lda, kmax, p->tau, p->delta, eps1, p->k_dm, p->use_delta_max,
              p->break_check, p->trace_norms, swap_cap, step_cap, nonfinite, 0, NZ > 1 ? zs : 0, tlbuf};
  k_init<<<dim3(1, 1, NZ), 1024, 0, st>>>(ia);
  NOTE_LAUNCH();
  CK(cudaGetLastError());

  // Host loop, pipelined: the host never waits for the step it just enqueued.
  // It keeps two steps in flight and sizes each launch from a lower bound on
  // n_s (the last step whose head it has read, plus one column for every step
  // still in flight -- every step accepts at least one).  Grids are therefore
  // upper bounds; kernels read the true extents from Ctl and exit surplus
  // CTAs, and steps enqueued after `done` exit at once.
  // pinned poll records (+ events, copy stream) from the per-device pool; a
  // batch brings its own records (one pair per matrix; k_step_end offsets by blockIdx.z)
  int cur_dev = 0;
  CK(cudaGetDevice(&cur_dev));
  SlotGuard slot_guard{NZ > 1 ? nullptr : slot_acquire(cur_dev)};
  if (NZ == 1 && !slot_guard.h) return DMQR_ECUDA;
  HostRec* const hrecs = (NZ > 1) ? zrec : slot_guard.h->rec;
  cudaEvent_t* const hev = (NZ > 1) ? nullptr : slot_guard.h->ev;
  for (unsigned q = 0; q < 2 * NZ; ++q) ((volatile HostRec*)hrecs)[q].seq = -1;
  const bool prof = g_prof.load() != 0;
  cudaEvent_t ev[2][5];
  if (prof)
    for (auto& r : ev)
      for (auto& e : r) CK(cudaEventCreate(&e));
  int slot = 0;
  bool qp_slot[2] = {false, false};  // the in-flight record of this slot came from a k_qp3 block
#define PROF(i) \
  if (prof) CK(cudaEventRecord(ev[slot][i], st))
  int steps_done = 0;
  const int max_coop_p = std::min(d.sms, PANEL_PMAX);
  const int max_cluster = cluster16 ? 16 : 8;
  const bool use_cq = getenv("DMQR_NO_CHOLQR") == nullptr;  // debug switch: Householder panel only
  const bool no_helpers = getenv("DMQR_NO_HELPERS") != nullptr;               // A/B switch
  // P-mode look-ahead (G = R1^-T P^T C from the panel's start; panel_cq.cuh): correct, but on cfg2 the
  // earlier G traffic slows the latency-bound panel more than it shortens k_spare (16.9 vs 16.6 ms), so opt-in
  const bool pmode_on = getenv("DMQR_PMODE") != nullptr;
  const bool fused_tail = getenv("DMQR_NO_FUSED_TAIL") == nullptr;  // schedule switch (tests): separate tail kernels
  // rows per CTA the CholeskyQR2 cluster aims for in the look-ahead schedule (A/B knob)
  const int64_t cq_rows = getenv("DMQR_CQ_ROWS") ? std::max<int64_t>(DMQR_KP, atoll(getenv("DMQR_CQ_ROWS"))) : 96;
  // (test hook: DMQR_HELPER_WAIT_NS=0 makes the tall panel abandon its helpers)
  const long long hwait_ns = getenv("DMQR_HELPER_WAIT_NS") ? atoll(getenv("DMQR_HELPER_WAIT_NS")) : 5000000ll;
  const size_t panel_smem_cap = std::min<size_t>(d.smem_optin - 4096, 220 * 1024);

  int64_t prev_ns_lo = 0;  // the lower bound the previous step was sized with
  // Look-ahead runs on the CholeskyQR2-panel steps (all of them unless the
  // Householder panel is forced): the other panels have no spare SMs to hide
  // the rest of the update behind.  Once on, it stays on
  // (k_set_la switches the control block).
  // The look-ahead pays off when norm guards are rare; k_guard flags a step
  // that needed one for most trailing columns (la_bad, with nothing left
  // pending), and the host then stays serial: flush + k_set_la(0).
  bool la_on = false, la_off = false, want_serial = false;
  auto enqueue_step = [&](int64_t host_ns, int eidx) -> int {
    const int64_t mp = m - host_ns;
    const int64_t np = n - host_ns;
    if (la_on && want_serial && !la_off) {
      const int64_t ldz0 = ldz_for(n);
      k_trail_b<true><<<dim3((unsigned)ceil_div(m - prev_ns_lo + 1, TB_ROWS),
                             (unsigned)std::max<int64_t>(1, ceil_div(n - prev_ns_lo, TB_COLS))),
                        TB_T, TB_SMEM, st>>>(ctl, A, Z, ldz0, upd, lacount + 1);
      NOTE_LAUNCH();
      k_set_la<<<1, 32, 0, st>>>(ctl, 0);
      NOTE_LAUNCH();
      la_off = true;
    }
    const bool la = !la_off && (la_on || (la_all && use_cq));
    if (la && !la_on) {
      k_set_la<<<1, 32, 0, st>>>(ctl, 1);
      NOTE_LAUNCH();
      la_on = true;
    }
    // ---- selection ----
    PROF(0);
    const int64_t ldz = ldz_for(n);
    if (wide) {
      // wide selection (wide.cuh): candidates in the workspace, tiled Gram,
      // one-CTA filter + swap plan, moves over every row; a continuing step's
      // next chunk makes all of these no-ops
      CK(pdl_launch(k_select_t<true>, dim3(1), dim3(SEL_T), 0, st, ctl, (const double*)u, wb));
      NOTE_LAUNCH();
      const int64_t W_ub = 1 + std::min<int64_t>(p->k_dm, std::max<int64_t>(np - 1, 0));
      const int64_t nt = ceil_div(W_ub, 32), tiles = nt * (nt + 1) / 2;
      const int wsp = (int)std::clamp<int64_t>(std::min<int64_t>(ceil_div(2 * d.sms, tiles), ceil_div(mp, 256)), 1,
                                               wb.nsplit);
      CK(pdl_launch(k_wgram, dim3((unsigned)tiles, (unsigned)wsp), dim3(WG_T), 0, st, ctl, (const double*)A, wb));
      NOTE_LAUNCH();
      CK(pdl_launch(k_wfin, dim3(1), dim3(WF_T), wfin_smem(wb.W, wf_smode), st, ctl, (const double*)A, swaps, wb, wsp,
                    wf_smode));
      NOTE_LAUNCH();
      const dim3 mvg((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 64)),
                     (unsigned)std::min<int64_t>(2 * W_ub, 65535));
      CK(pdl_launch(k_wgather, mvg, dim3(256), 0, st, ctl, (const double*)A, (const double*)u, (const double*)uref,
                    (const int64_t*)perm, wb));
      NOTE_LAUNCH();
      CK(pdl_launch(k_wscatter, mvg, dim3(256), 0, st, ctl, A, u, uref, perm, wb));
      NOTE_LAUNCH();
    } else {
      CK(pdl_launch(k_select_t<false>, dim3(1, 1, NZ), dim3(SEL_T), 0, st, ctl, (const double*)u, WideBufs{}));
      NOTE_LAUNCH();
      const int GG = (int)std::clamp<int64_t>(ceil_div(mp, GRAM_ROWS), 1, std::min(GRAM_GMAX, d.sms));
      CK(pdl_launch(k_gram, dim3(GG, 1, NZ), dim3(GRAM_T), GRAM_SMEM, st, ctl, A, gpart, (const double*)Z, ldz,
                    (const uint8_t*)upd));
      NOTE_LAUNCH();
      CK(pdl_launch(k_gram_finish, dim3(45, 1, NZ), dim3(GRAM_T), sizeof(FinSmem), st, ctl, (const double*)A,
                    (const double*)gpart, GG, gfin, upd, tline));
      NOTE_LAUNCH();
    }
    {
      // (+1: block 0 owns no rows and moves u / u_ref / perm / flags and appends the swap log)
      CK(pdl_launch(k_swap, dim3((unsigned)ceil_div(m + (la ? DMQR_KP : 0), SWAP_ROWS) + 1, 1, NZ), dim3(SWAP_T), SWAP_SMEM,
                    st, ctl, A, u, uref, perm, swaps, Z, ldz, upd));
      NOTE_LAUNCH();
    }
    // the rest of the previous step's update: beside the CholeskyQR2 panel as
    // its programmatic dependent, else (other panel kernels) before the panel
    const dim3 lag((unsigned)ceil_div(m - prev_ns_lo + 1, TB_ROWS),
                   (unsigned)std::max<int64_t>(1, ceil_div(n - host_ns, TB_COLS)));
    auto launch_la_rest = [&](bool pdl) -> cudaError_t {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = lag;
      cfg.blockDim = dim3(TB_T);
      cfg.dynamicSmemBytes = TB_SMEM;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      NOTE_LAUNCH();
      return cudaLaunchKernelEx(&cfg, k_trail_b<true>, ctl, A, (const double*)Z, ldz, upd, lacount + 1);
    };
    const bool la_rest = la && host_ns > 0;
    // ---- panel ----
    const int kcap = (int)std::min<int64_t>({(int64_t)p->k_dm + 1, (int64_t)DMQR_MAXK, kmax - host_ns});
    // row CTAs (+1 T-builder CTA when the panel spans several CTAs); the T
    // builder (or the single CTA) also keeps T (KP x KP) in shared memory
    const size_t tbytes = sizeof(double) * DMQR_KP * DMQR_KP;
    int P = (int)std::clamp<int64_t>(ceil_div(mp, 256), 1, max_coop_p - 1);
    int64_t rows = ceil_div(mp, P);
    size_t smem = (size_t)kcap * (size_t)(rows | 1) * sizeof(double) + (P == 1 ? tbytes : 0);
    int use_smem = 1;
    if (smem > panel_smem_cap) {
      P = max_coop_p - 1;
      rows = ceil_div(mp, P);
      smem = (size_t)kcap * (size_t)(rows | 1) * sizeof(double);
      if (smem > panel_smem_cap) {
        use_smem = 0;
        smem = 0;
      }
    }
    smem = std::max(smem, tbytes);
    PROF(1);
    // register-resident panel (<= 256 rows per CTA): one thread-block cluster
    // (DSMEM all-reduce) when it fits in 16 CTAs, else a cooperative grid
    const int Prr = (int)std::max<int64_t>(1, ceil_div(mp, RR_RMAX));
    const bool rr_path = Prr <= max_coop_p - 1;
    const bool cl_path = rr_path && Prr > 1 && Prr <= max_cluster;
    if (rr_path) P = Prr;
    const int G = cl_path ? P : ((P > 1) ? P + 1 : 1);
    PanelArgs pa{ctl, A, coeffs, T, red, use_smem, P,
                 (g_prof.load() >= 2 && steps_done == 2) ? pdbg : nullptr, std::max(0, g_prof.load() - 2), 0,
                 q1g, 0, tline, 0, (double*)(ws + L.hpart), (double*)(ws + L.hR), (unsigned*)(ws + L.hctr),
                 hwait_ns, pmode_on ? (double*)(ws + L.pg) : nullptr};
    void* kargs[] = {&pa};
    auto launch_cluster = [&](const void* fn, int ncta, unsigned threads, size_t dsm) -> cudaError_t {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(ncta, 1, NZ);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = dsm;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = ncta;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (pdl_enter in the panels)
      at[1].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      return cudaLaunchKernelExC(&cfg, fn, kargs);
    };
    // CholeskyQR2 panel (one cluster, <= 256 rows per CTA) first; the Householder
    // kernels behind it run only if it declined (ill-conditioned panel)
    // (more than max_cluster x 256 rows: the cluster streams its rows in chunks)
    const bool cq_path = use_cq;
    // (look-ahead: fewer rows per CTA -- the Gram / Q1 phases of the panel scale with a CTA's rows, and
    // late in the factorization the SMs the wider cluster takes are idle anyway)
    // (mp is the host's upper bound: the true panel can be up to two steps' columns shorter, and rank 0
    // must keep the whole top block -- at least DMQR_MAXK rows -- so the count is taken from mp - 2 MAXK)
    const int Pcq = (int)std::min<int64_t>(
        std::max<int64_t>(Prr, (la && cq_rows < RR_RMAX) ? (mp - 2 * DMQR_MAXK) / cq_rows : 1), max_cluster);
    const bool spare = la && cq_path;  // k_spare beside the panel, then k_trail_w
    const int64_t ntile_g = std::max<int64_t>(1, ceil_div(np, TA_COLS));
    // G = Q1^T C split-K items over the spare CTAs: as many splits as keep the
    // items within whole waves of the CTAs (a CTA with one item more than the
    // rest sets the phase's length)
    // (one wave: finer items, 2-3 waves, measured slower -- their partial sums cost more than the tail they trim)
    const int nsplit_g = choose_nsplit(ntile_g, 2 * std::max(1, d.sms - Pcq),
                                       (int)std::min<int64_t>(NSPLIT_MAX, std::max<int64_t>(1, ceil_div(mp, 256))));
    if (la_rest && !cq_path) CK(launch_la_rest(false));
    // tall CholeskyQR2 panel, serial schedule: its row passes go to the free SMs
    const bool helpers = cq_path && !spare && mp > (int64_t)Pcq * CQ_RMAX && d.sms - Pcq >= 16 && !no_helpers && NZ == 1;
    if (cq_path) {
      pa.spare = spare ? 1 : 0;
      pa.helpers = helpers ? 1 : 0;
      if (helpers) {
        CK(pdl_launch(k_hzero, dim3(1), dim3(32), 0, st, (unsigned*)(ws + L.hctr)));
        NOTE_LAUNCH();
      }
      CK(launch_cluster((const void*)k_panel_cq, Pcq, PANEL_T, CQ_SMEM));
      NOTE_LAUNCH();
      if (helpers) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)std::min<int64_t>(d.sms - Pcq, ceil_div(mp, CQ_RMAX)));
        cfg.blockDim = dim3(PANEL_T);
        cfg.dynamicSmemBytes = CQH_SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k_panel_helper, pa));
        NOTE_LAUNCH();
      }
      pa.only_if_fail = 1;
      pa.spare = 0;
      pa.helpers = 0;
      if (spare) {
        cudaLaunchConfig_t cfg = {};
        // persistent CTAs: two per SM the panel leaves free, plus two per panel SM
        // that start once the panel is done (they pull what is left); no more than
        // work items
        const int64_t items = (int64_t)lag.x * lag.y * (la_rest ? 1 : 0) + ntile_g * nsplit_g;
        cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(2 * d.sms, items)));
        cfg.blockDim = dim3(TB_T);
        cfg.dynamicSmemBytes = SP_SMEM;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        NOTE_LAUNCH();
        // (fused tail: the Y = Q1 M tiles run in k_trail_w's extra CTAs instead of here)
        CK(cudaLaunchKernelEx(&cfg, pmode_on ? k_spare<true> : k_spare<false>, ctl, A, (const double*)Z, ldz, upd, (const double*)q1g, Zp,
                              lacount + 4, Pcq, nsplit_g, tcount, tline,
                              fused_tail ? (const double*)nullptr : (const double*)(red + 37 * DMQR_KP * DMQR_KP),
                              (const double*)(ws + L.pg)));
      }
    }
    if (cl_path) {
      CK(launch_cluster((const void*)k_panel_rr<ClusterRed>, G, PANEL_T, RR_CL_SMEM));
      NOTE_LAUNCH();
    } else if (G > 1) {
      void* kfn = rr_path ? (void*)k_panel_rr<GridRed> : (void*)k_panel;
      CK(cudaLaunchCooperativeKernel(kfn, dim3(G), dim3(PANEL_T), kargs, rr_path ? 0 : smem, st));
      NOTE_LAUNCH();
    } else if (rr_path) {
      k_panel_rr<GridRed><<<dim3(1, 1, NZ), PANEL_T, 0, st>>>(pa);
      NOTE_LAUNCH();
    } else {
      k_panel<<<1, PANEL_T, smem, st>>>(pa);
      NOTE_LAUNCH();
    }
    if (cq_path && mp > 1 && !spare) {  // Y below the top block of a CholeskyQR2 panel, on every SM
      // (with the look-ahead, k_spare does this as its third phase)
      CK(pdl_launch(k_ygemm, dim3((unsigned)ceil_div(mp - 1, YG_ROWS), 1, NZ), dim3(256), YG_SMEM, st, ctl, A,
                    (const double*)q1g, (const double*)(red + 37 * DMQR_KP * DMQR_KP)));
      NOTE_LAUNCH();
    }
    // ---- trailing update ----
    PROF(2);
    const int64_t ncols_ub = std::max<int64_t>(np - 1, 0);
    int tail_nsplit = 1;
    if (spare && fused_tail) {
      // Wt tiles (their last CTA closes the step when no guard column came up: k_tail then exits at
      // once) and, on the CTAs past them, the Y = Q1 M tiles; launched even without trailing columns
      const int wgrid = (int)ceil_div(ncols_ub, TW_COLS);
      const int ygrid = (int)ceil_div(std::max<int64_t>(mp - 1, 0), YG_ROWS);
      CK(pdl_launch(k_trail_w, dim3((unsigned)std::max(1, wgrid + ygrid)), dim3(TA_T), TW_SMEM, st, ctl, A,
                    (const double*)Zp, (const double*)(red + 19 * DMQR_KP * DMQR_KP), Z, ldz, u, uref, upd, glist,
                    StepClose{srec, hrecs, lacount + 12, (const double*)q1g,
                              (const double*)(red + 37 * DMQR_KP * DMQR_KP), ygrid}));
      NOTE_LAUNCH();
    }
    if (ncols_ub > 0) {
      const int64_t ntile = ceil_div(ncols_ub, TA_COLS);
      const int nsplit = choose_nsplit(ntile, 2 * d.sms,
                                       (int)std::min<int64_t>(nsplit_cap(n), std::max<int64_t>(1, ceil_div(mp, 256))));
      tail_nsplit = nsplit;
      if (spare && !fused_tail) {
        CK(pdl_launch(k_trail_w, dim3((unsigned)ceil_div(ncols_ub, TW_COLS)), dim3(TA_T), TW_SMEM, st, ctl, A,
                      (const double*)Zp, (const double*)(red + 19 * DMQR_KP * DMQR_KP), Z, ldz, u, uref, upd,
                      glist, StepClose{nullptr, nullptr, nullptr, nullptr, nullptr, 0}));
        NOTE_LAUNCH();
      }
      if (!(spare && fused_tail)) {
        CK(pdl_launch(k_trail_a, dim3((unsigned)ntile, nsplit, NZ), dim3(TA_T), TA_SMEM, st, ctl, A, Zp,
                      (const double*)T, Z, tcount, ldz, u, uref, upd, spare ? 1 : 0, glist));
        NOTE_LAUNCH();
      }
      if (la) {
        // the rest of C -= Y Wt runs beside the next step's panel
      } else {
        k_trail_b<false><<<dim3((unsigned)ceil_div(mp + 1, TB_ROWS), (unsigned)ceil_div(ncols_ub, TB_COLS), NZ), TB_T,
                           TB_SMEM, st>>>(ctl, A, Z, ldz, upd, lacount + 1);
        NOTE_LAUNCH();
      }
    }
    // ---- norms, log ----
    PROF(3);
    if (spare && fused_tail) {
      // one launch for the rest of the step (tail.cuh): the panel's fallback update, guard columns,
      // bookkeeping, host record -- or nothing at all when k_trail_w closed the step
      TailArgs ta{ctl, A, Zp, (const double*)T, Z, tcount, ldz, u, uref, upd, glist, tail_nsplit, srec, hrecs, eidx,
                  lacount + 13};
      CK(pdl_launch(k_tail, dim3((unsigned)d.sms), dim3(TA_T), TAIL_SMEM, st, ta));
      NOTE_LAUNCH();
      PROF(4);
      CK(cudaGetLastError());
      return 0;
    }
    if (la) {
      // norms: downdated in the Wt epilogues; guard columns recomputed here
      CK(pdl_launch(k_guard,
                    dim3((unsigned)std::max<int64_t>(1, ceil_div(mp, GU_ROWS)),
                         (unsigned)std::max<int64_t>(1, ceil_div(np, GU_GROUPS * DMQR_KP))),
                    dim3(GU_T), GU_SMEM, st, ctl, A, (const double*)Z, ldz, upd, u, uref, (const int32_t*)glist,
                    lacount + 2));
      NOTE_LAUNCH();
      CK(pdl_launch(k_guard_norms, dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(np * 32, 256),
                                                                                      (int64_t)d.sms * 8))),
                    dim3(256), 0, st, ctl, (const double*)A, upd, u, uref, (const int32_t*)glist));
      NOTE_LAUNCH();
    } else if (np > 0) {
      const int64_t blocks = std::min<int64_t>(ceil_div(np * 32, 256), (int64_t)d.sms * 16);
      // tall columns: the guard columns' exact norms row-split over the grid
      const bool gsplit = mp > 4 * GN_ROWS && !p->trace_norms;
      k_downdate<<<dim3((unsigned)blocks, 1, NZ), 256, 0, st>>>(ctl, A, u, uref, gsplit ? glist : nullptr);
      NOTE_LAUNCH();
      if (gsplit) {
        k_gnorm_part<<<(unsigned)(2 * d.sms), 256, 0, st>>>(ctl, (const double*)A, (const int32_t*)glist, gnp);
        NOTE_LAUNCH();
        k_gnorm_fin<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(np * 32, 256), (int64_t)d.sms * 4)),
                      256, 0, st>>>(ctl, (const double*)A, (const int32_t*)glist, (const double*)gnp, u, uref);
        NOTE_LAUNCH();
      }
      if (p->trace_norms) { k_norm_trace<<<(unsigned)blocks, 256, 0, st>>>(ctl, A, u, tbits); NOTE_LAUNCH(); }
    }
    if (wide) {  // does the step continue with its next chunk?
      CK(pdl_launch(k_wcont, dim3(1), dim3(1024), 0, st, ctl, (const double*)A));
      NOTE_LAUNCH();
    }
    CK(pdl_launch(k_step_end, dim3(1, 1, NZ), dim3(32), 0, st, ctl, srec, norm_trace, tbits, (const double*)A, Z, ldz, u,
                  uref, upd, hrecs, eidx));
    NOTE_LAUNCH();
    PROF(4);
    CK(cudaGetLastError());
    return 0;
  };

  // streamed packed factor: final columns go to the host on a side stream
  if (host_packed && !slot_guard.h->copy) CK(cudaStreamCreateWithFlags(&slot_guard.h->copy, cudaStreamNonBlocking));
  const cudaStream_t sCopy = host_packed ? slot_guard.h->copy : nullptr;
  int64_t copied = 0;
  auto stream_cols = [&](int64_t upto, cudaEvent_t after) -> int {
    upto = std::min(upto, n);
    if (!host_packed || upto <= copied || m == 0) return 0;
    if (after) CK(cudaStreamWaitEvent(sCopy, after, 0));
    CK(cudaMemcpy2DAsync(host_packed + copied * host_ld, sizeof(double) * host_ld, A + copied * lda,
                         sizeof(double) * lda, sizeof(double) * m, (size_t)(upto - copied), cudaMemcpyDeviceToHost,
                         sCopy));
    copied = upto;
    return 0;
  };
  int64_t known_ns = 0;  // n_s after the last step whose head was read
  int known = 0, enq = 0, known_steps = 0;
  bool qp_mode = qrp != 0;
  // k_qp3 splits each column into at most QP_RMAX staged row segments
  const bool qp_ok = m <= (int64_t)QP_RMAX * QP_XCH && NZ == 1;
  if (qrp && !qp_ok) return DMQR_EINVAL;
  // replayed step graph (batched small matrices; serial schedule only)
  const bool use_graph = sgraph != nullptr && !la_all && !qrp && !p->trace_norms && !prof && !tline &&
                         getenv("DMQR_NO_GRAPH") == nullptr && getenv("DMQR_NO_STEP_GRAPH") == nullptr;
  std::vector<unsigned char> gkey;
  if (use_graph) {
    const void* parts[] = {A, coeffs, perm, swaps, steps, workspace, (const void*)hrecs};
    const int64_t dims[] = {m, n, lda, swap_cap, step_cap};
    gkey.resize(sizeof(parts) + sizeof(dims) + sizeof(dmqr_params));
    std::memcpy(gkey.data(), parts, sizeof(parts));
    std::memcpy(gkey.data() + sizeof(parts), dims, sizeof(dims));
    dmqr_params pk = *p;
    pk.max_steps = 0;
    std::memcpy(gkey.data() + sizeof(parts) + sizeof(dims), &pk, sizeof(pk));
    if (sgraph->exec && sgraph->key != gkey) {
      cudaGraphExecDestroy(sgraph->exec);
      sgraph->exec = nullptr;
    }
  }
  bool finished = (kmax == 0);
  const bool step_verbose = getenv("DMQR_STEP_VERBOSE") != nullptr;  // debug: every consumed step record
  auto consume = [&]() -> int {
    const int sl = known & 1;
    // poll the step's record (k_step_end posts it); check the stream now and
    // then so that a failed launch cannot hang the loop
    volatile HostRec* r = hrecs + sl;
    // (a batch: every matrix's record of this step; the lowest n_s and 'all done')
    int32_t zmin_ns = 0x7fffffff, zall_done = 1;
    for (unsigned z = 1; z < NZ; ++z) {
      volatile HostRec* rz = hrecs + 2 * z + sl;
      for (long spins = 1; rz->seq != known + 1; ++spins) {
        if (spins > 64) std::this_thread::yield();
        if ((spins & 1023) == 0) {
          const cudaError_t e = cudaStreamQuery(st);
          if (e != cudaSuccess && e != cudaErrorNotReady) return DMQR_ECUDA;
          if (e == cudaSuccess && rz->seq != known + 1) {
            std::atomic_thread_fence(std::memory_order_seq_cst);
            if (rz->seq != known + 1) return DMQR_ECUDA;
          }
        }
      }
      zmin_ns = std::min<int32_t>(zmin_ns, (int32_t)rz->n_s);
      zall_done &= (rz->flags & 1);
    }
    for (long spins = 1; r->seq != known + 1; ++spins) {
      // batch lanes may outnumber the host cores: give the core away while waiting
      if (sgraph && spins > 64) std::this_thread::yield();
      if ((spins & 1023) == 0) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e != cudaSuccess && e != cudaErrorNotReady) return DMQR_ECUDA;
        if (e == cudaSuccess && r->seq != known + 1) {
          std::atomic_thread_fence(std::memory_order_seq_cst);
          if (r->seq != known + 1) return DMQR_ECUDA;  // stream drained, no record
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    if (prof) {
      CK(cudaEventSynchronize(ev[sl][4]));
      if (qp_slot[sl]) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev[sl][0], ev[sl][4]));
        g_acc.ms[4] += ms;
      } else {
        for (int q = 0; q < 4; ++q) {
          float ms = 0.f;
          CK(cudaEventElapsedTime(&ms, ev[sl][q], ev[sl][q + 1]));
          g_acc.ms[q] += ms;
        }
      }
      g_acc.steps += 1;
    }
    known_ns = std::min<int32_t>((int32_t)r->n_s, zmin_ns);
    known_steps = r->step_idx;
    if (step_verbose)
      fprintf(stderr, "[dmqr] step record %d: n_s %d step_idx %d flags %d\n", known, (int)r->n_s, (int)r->step_idx,
              (int)r->flags);
    ++known;
    if ((r->flags & 1) && zall_done) finished = true;
    if (r->flags & 2) want_serial = true;
    // a scalar-fallback step hands the run to the blocked scalar-pivot engine;
    // its blocks keep it until a fallback run ends on the floor test
    qp_mode = qrp || ((r->flags & 4) != 0 && qp_ok);
    return stream_cols(known_ns, nullptr);  // columns left of n_s are final (and written)
  };
  // one block of the blocked scalar-pivot engine (no step in flight)
  const int qp_clk = getenv("DMQR_QP_CLOCKS") ? atoi(getenv("DMQR_QP_CLOCKS")) : -1;
  int qp_blocks = 0;
  const bool qp_verbose = getenv("DMQR_QP_VERBOSE") != nullptr;  // debug: columns per block
  auto run_qp_block = [&]() -> int {
    if (la_on && !la_off) {  // flush the look-ahead's pending update; serial from here on
      const int64_t ldz0 = ldz_for(n);
      k_trail_b<true><<<dim3((unsigned)ceil_div(m - prev_ns_lo + 1, TB_ROWS),
                             (unsigned)std::max<int64_t>(1, ceil_div(n - prev_ns_lo, TB_COLS))),
                        TB_T, TB_SMEM, st>>>(ctl, A, Z, ldz_for(n), upd, lacount + 1);
      (void)ldz0;
      NOTE_LAUNCH();
      k_set_la<<<1, 32, 0, st>>>(ctl, 0);
      NOTE_LAUNCH();
      la_off = true;
    }
    slot = enq & 1;
    qp_slot[slot] = true;
    PROF(0);
    int lim = p->trace_norms ? 1 : QP_NB;
    if (p->max_steps > 0) lim = std::min<int>(lim, std::max(0, p->max_steps - known_steps));
    CK(cudaMemsetAsync(qcnt, 0, sizeof(unsigned) * 4, st));
    double* qg = (double*)(ws + L.qgpart);
    // debug: phase clocks of CTA 0 for the k-th block (DMQR_QP_CLOCKS=k; tools/qp_clocks.py)
    long long* qdbg = (qp_clk >= 0 && qp_blocks == qp_clk) ? pdbg : nullptr;
    ++qp_blocks;
    Qp3Args qa{ctl, A, u, uref, perm, swaps, coeffs, srec, Zp, Z, ldz_for(n), (double*)(ws + L.qvb),
               (double*)(ws + L.qwb), (double*)(ws + L.qpart), qg, glist, qg + QP_GMAXCTA * QP_GMAX * 2, qcnt,
               qdbg, qrp, lim};
    void* qargs[] = {&qa};
    CK(cudaLaunchCooperativeKernel((const void*)k_qp3, dim3(qp_grid), dim3(QP_T), qargs, QP_SMEM, st));
    NOTE_LAUNCH();
    if (p->trace_norms) {
      const int64_t blocks = std::min<int64_t>(ceil_div(std::max<int64_t>(n, 1) * 32, 256), (int64_t)d.sms * 16);
      k_qp3_trace<<<(unsigned)blocks, 256, 0, st>>>(ctl, A, u, tbits);
      NOTE_LAUNCH();
    }
    k_qp3_post<<<1, 32, 0, st>>>(ctl, p->trace_norms ? norm_trace : nullptr, tbits, hrecs, enq);
    NOTE_LAUNCH();
    PROF(4);
    CK(cudaGetLastError());
    ++enq;
    ++steps_done;
    const int before = known_steps;
    const int rc = consume();
    if (qp_verbose) fprintf(stderr, "[dmqr] qp block %d: %d columns, n_s %lld\n", qp_blocks - 1,
                            known_steps - before, (long long)known_ns);
    return rc;
  };
  while (!finished) {
    if (qp_mode) {
      while (known < enq && !finished) {  // drain the steps in flight
        int rc = consume();
        if (rc) return rc;
      }
      if (finished) break;
      if (!qp_mode) continue;
      if (p->max_steps > 0 && known_steps >= p->max_steps) break;
      int rc = run_qp_block();
      if (rc) return rc;
      continue;
    }
    if (enq - known >= 2) {
      int rc = consume();
      if (rc) return rc;
      if (finished) break;
    }
    const int64_t ns_lo = known_ns + (enq - known);
    if (ns_lo >= kmax) {  // every column is accounted for by the steps in flight
      while (known < enq && !finished) {
        int rc = consume();
        if (rc) return rc;
      }
      break;
    }
    slot = enq & 1;
    qp_slot[slot] = false;
    int rc = 0;
    if (use_graph) {
      if (!sgraph->exec) {  // capture the step once (whole-matrix grids)
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        rc = enqueue_step(0, 0);
        const cudaError_t ce = cudaStreamEndCapture(st, &g);
        if (rc) {
          if (g) cudaGraphDestroy(g);
          return rc;
        }
        CK(ce);
        const cudaError_t ie = cudaGraphInstantiate(&sgraph->exec, g, 0);
        cudaGraphDestroy(g);
        CK(ie);
        sgraph->key = gkey;
      }
      CK(cudaGraphLaunch(sgraph->exec, st));
    } else {
      rc = enqueue_step(ns_lo, enq);
    }
    if (rc) return rc;
    prev_ns_lo = ns_lo;
    ++enq;
    ++steps_done;
    if (p->max_steps > 0 && steps_done >= p->max_steps) break;  // debug: stop after N steps
  }
  if (la_on && enq > 0) {  // the last step's pending update
    const int64_t ldz = ldz_for(n);
    k_trail_b<true><<<dim3((unsigned)ceil_div(m - prev_ns_lo + 1, TB_ROWS),
                           (unsigned)std::max<int64_t>(1, ceil_div(n - prev_ns_lo, TB_COLS))),
                      TB_T, TB_SMEM, st>>>(ctl, A, Z, ldz, upd, lacount + 1);
    NOTE_LAUNCH();
  }
  while (known < enq) {  // drain (profiling reads; the steps themselves are ordered on st)
    int rc = consume();
    if (rc) return rc;
  }
  if (prof)
    for (auto& r : ev)
      for (auto& e : r) cudaEventDestroy(e);
#undef PROF
  g_calls.fetch_add(1);
  k_finalize<<<dim3(1, 1, NZ), 256, 0, st>>>(ctl, A, p->stop_rule == DMQR_STOP_NONE);
  NOTE_LAUNCH();
  CK(cudaGetLastError());
  if (host_packed && m > 0 && n > 0) {  // the rest of the packed factor
    CK(cudaEventRecord(hev[0], st));
    copied = std::min(copied, n);
    if (stream_cols(n, hev[0])) return DMQR_ECUDA;
    CK(cudaStreamSynchronize(sCopy));
  }
  if (NZ > 1) {  // a batch: every matrix's control block
    std::vector<Ctl> hcs(NZ);
    CK(cudaMemcpy2DAsync(hcs.data(), sizeof(Ctl), ctl, (size_t)zs, sizeof(Ctl), NZ, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int rc0 = 0;
    for (unsigned z = 0; z < NZ; ++z) {
      const Ctl& h = hcs[z];
      dmqr_info& in = info[z];
      in.rank = (kmax == 0) ? 0 : h.rank;
      in.n_factored = (kmax == 0) ? 0 : h.n_factored;
      in.n_steps = (kmax == 0) ? 0 : h.step_idx;
      in.n_swaps = (kmax == 0) ? 0 : h.n_swaps;
      in.stopped_early = (kmax == 0) ? 0 : h.stopped;
      in.status = h.status;
      in.a_max0 = h.a_max0;
      if (!rc0 && h.status) rc0 = h.status;
    }
    return rc0;
  }
  Ctl hc;
  CK(cudaMemcpyAsync(&hc, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  info->rank = hc.rank;
  info->n_factored = hc.n_factored;
  info->n_steps = hc.step_idx;
  info->n_swaps = hc.n_swaps;
  info->stopped_early = hc.stopped;
  info->status = hc.status;
  info->a_max0 = hc.a_max0;
  if (kmax == 0) {
    info->rank = 0;
    info->n_factored = 0;
    info->n_steps = 0;
    info->n_swaps = 0;
    info->stopped_early = 0;
  }
  return hc.status;
}
}  // namespace

extern "C" {

int dmqr_qrdm_stream_f64(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* p, double* coeffs,
                         int64_t* perm, int64_t* swaps, int64_t swap_cap, dmqr_step* steps, int64_t step_cap,
                         double* norm_trace, void* workspace, size_t ws_bytes, dmqr_info* info,
                         double* host_packed, int64_t host_ld, void* stream) {
  return run_engine(A, m, n, lda, p, coeffs, perm, swaps, swap_cap, steps, step_cap, norm_trace, workspace, ws_bytes,
                    info, host_packed, host_ld, stream, 0);
}

int dmqr_qrp_stream_f64(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* p, double* coeffs,
                        int64_t* perm, int64_t* swaps, int64_t swap_cap, dmqr_step* steps, int64_t step_cap,
                        double* norm_trace, void* workspace, size_t ws_bytes, dmqr_info* info, double* host_packed,
                        int64_t host_ld, void* stream) {
  return run_engine(A, m, n, lda, p, coeffs, perm, swaps, swap_cap, steps, step_cap, norm_trace, workspace, ws_bytes,
                    info, host_packed, host_ld, stream, 1);
}

int dmqr_qrp_f64(double* A, int64_t m, int64_t n, int64_t lda, const dmqr_params* p, double* coeffs, int64_t* perm,
                 int64_t* swaps, int64_t swap_cap, dmqr_step* steps, int64_t step_cap, double* norm_trace,
                 void* workspace, size_t ws_bytes, dmqr_info* info, void* stream) {
  return dmqr_qrp_stream_f64(A, m, n, lda, p, coeffs, perm, swaps, swap_cap, steps, step_cap, norm_trace, workspace,
                             ws_bytes, info, nullptr, 0, stream);
}

}  // extern "C"

namespace {
// Small matrices in a batch run on lane-private buffers (so each lane's step
// graph is captured once and replayed for all its matrices): the work matrix,
// coeffs, perm, the swap log and the step log, sized for the largest caps.
struct LaneBufs {
  size_t a, coeffs, perm, swaps, steps, total;
  int64_t swap_cap, step_cap;
};
LaneBufs lane_bufs(int64_t m, int64_t n, int64_t lda) {
  LaneBufs b{};
  const int64_t kmax = std::max<int64_t>(std::min(m, n), 1);
  b.swap_cap = kmax * DMQR_MAXK + 8;
  b.step_cap = kmax;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += al(bytes);
    return o;
  };
  b.a = take(sizeof(double) * (size_t)lda * (size_t)std::max<int64_t>(n, 1));
  b.coeffs = take(sizeof(double) * kmax);
  b.perm = take(sizeof(int64_t) * std::max<int64_t>(n, 1));
  b.swaps = take(sizeof(int64_t) * 2 * b.swap_cap);
  b.steps = take(sizeof(dmqr_step) * b.step_cap);
  b.total = off;
  return b;
}
bool batch_graph_ok(int64_t m, int64_t n) { return m * n < ((int64_t)1 << 20); }
// grouped launches (grid.z) need the standard selection; wide k_dm runs per matrix
bool batch_groups(int64_t m, int64_t n, const dmqr_params* p) { return batch_graph_ok(m, n) && p->k_dm <= WIDE_K; }
constexpr int ZG = 128;  // small matrices per batched launch (grid.z)
}  // namespace

extern "C" {

int32_t dmqr_batched_group(int64_t m, int64_t n) { return batch_graph_ok(m, n) ? ZG : 1; }

size_t dmqr_batched_workspace_bytes(int64_t m, int64_t n, const dmqr_params* params, int32_t nlanes) {
  const size_t eng = al(dmqr_workspace_bytes(m, n, params));
  const size_t per = batch_groups(m, n, params) ? (size_t)ZG * (eng + lane_bufs(m, n, (m + 7) / 8 * 8).total) : eng;
  return (size_t)std::max(1, nlanes) * per;
}

int dmqr_qrdm_batched_f64(double* A, int64_t batch, int64_t m, int64_t n, int64_t lda, int64_t stride,
                          const dmqr_params* p, double* coeffs, int64_t* perm, int64_t* swaps, int64_t swap_cap,
                          dmqr_step* steps, int64_t step_cap, dmqr_info* infos, int32_t nlanes, void* workspace,
                          size_t ws_bytes, void* stream) {
  int rc = validate(m, n, lda, p);
  if (rc) return rc;
  if (batch < 0 || stride < lda * n || !infos || nlanes < 1) return DMQR_EINVAL;
  if (small_eligible(m, n, p) && workspace && ws_bytes >= small_info_bytes(batch)) {
    // small matrices: the fused per-matrix kernel, a persistent grid over the batch
    if (batch == 0) return 0;
    DevAttrs* da = nullptr;
    const DevInfo d = dev_info();
    if ((rc = set_attrs(d, &da))) return rc;
    return run_small(A, batch, m, n, lda, stride, p, coeffs, perm, swaps, swap_cap, steps, step_cap,
                     (SmallInfo*)workspace, infos, (cudaStream_t)stream, d.sms);
  }
  const size_t per_engine = al(dmqr_workspace_bytes(m, n, p));
  // small matrices: groups of ZG per launch (grid.z) in lane-private per-matrix
  // blocks + a replayed step graph per lane (needs the caller's lda to match the
  // blocks' and caps within theirs)
  const LaneBufs lb = lane_bufs(m, n, lda);
  const bool graphs = batch_groups(m, n, p) && lda == (m + 7) / 8 * 8 && swap_cap <= lb.swap_cap &&
                      step_cap <= lb.step_cap && getenv("DMQR_NO_GRAPH") == nullptr;
  const size_t zblk = per_engine + lb.total;  // (both multiples of 256 bytes)
  const size_t per = batch_groups(m, n, p) ? (size_t)ZG * zblk : per_engine;
  nlanes = (int32_t)std::min<int64_t>(nlanes, std::max<int64_t>(batch, 1));
  if (m > 4096) nlanes = 1;  // cooperative panel launches must not compete for co-residency
  if (ws_bytes < per * (size_t)nlanes || !workspace) return DMQR_EINVAL;
  if (graphs) nlanes = (int32_t)std::min<int64_t>(nlanes, ceil_div(batch, ZG));
  if (batch == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const DevInfo d = dev_info();
  DevAttrs* da = nullptr;
  if ((rc = set_attrs(d, &da))) return rc;
  // lanes start after the caller's stream reaches this point, and the caller's
  // stream waits for every lane at the end
  cudaEvent_t start;
  CK(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  CK(cudaEventRecord(start, st));
  const int64_t kmax = std::min(m, n);
  std::vector<int> lane_rc(nlanes, 0);
  std::vector<cudaError_t> lane_err(nlanes, cudaSuccess);  // (last_cuda_error is per thread)
  std::vector<cudaStream_t> ls(nlanes);
  std::vector<cudaEvent_t> done(nlanes);
  for (int q = 0; q < nlanes; ++q) {
    CK(cudaStreamCreateWithFlags(&ls[q], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming));
    CK(cudaStreamWaitEvent(ls[q], start, 0));
  }
  auto work = [&](int q) {
    cudaSetDevice(dev);
    unsigned char* ws = (unsigned char*)workspace + per * (size_t)q;
    if (!graphs) {
      for (int64_t b = q; b < batch; b += nlanes) {
        const int r = dmqr_qrdm_f64(A + b * stride, m, n, lda, p, coeffs + b * kmax, perm + b * n,
                                    swaps + b * 2 * swap_cap, swap_cap, steps + b * step_cap, step_cap, nullptr, ws,
                                    per_engine, &infos[b], (void*)ls[q]);
        infos[b].status = r;
        if (r && !lane_rc[q]) lane_rc[q] = r;
      }
    } else {
      // groups of up to ZG matrices in lane-private per-matrix blocks (engine
      // workspace + matrix + outputs, zblk bytes apart): one launch per kernel
      // per step for the whole group (grid.z), the step replayed as a graph
      unsigned char* zbase = ws;
      unsigned char* zb = ws + per_engine;  // block 0's matrix and outputs (after its engine workspace)
      const cudaStream_t s = ls[q];
      const size_t abytes = sizeof(double) * (size_t)lda * (size_t)n;
      StepGraph sg;
      HostRec* zrec = nullptr;
      if (cudaMallocHost(&zrec, sizeof(HostRec) * 2 * ZG) != cudaSuccess) {
        lane_rc[q] = DMQR_ECUDA;
        cudaEventRecord(done[q], ls[q]);
        return;
      }
      for (int64_t g0 = (int64_t)q * ZG; g0 < batch; g0 += (int64_t)nlanes * ZG) {
        const int g = (int)std::min<int64_t>(ZG, batch - g0);
        int r = 0;
        auto cp2 = [&](void* dst, size_t dp, const void* src, size_t sp, size_t w) {
          if (r) return;
          const cudaError_t e = cudaMemcpy2DAsync(dst, dp, src, sp, w, (size_t)g, cudaMemcpyDeviceToDevice, s);
          if (e != cudaSuccess) {
            last_cuda_error() = e;
            r = DMQR_ECUDA;
            if (getenv("DMQR_DEBUG_BATCH"))
              fprintf(stderr, "[dmqr] batch copy failed: %s (dp %zu sp %zu w %zu h %d)\n", cudaGetErrorString(e), dp,
                      sp, w, g);
          }
        };
        cp2(zb + lb.a, zblk, A + g0 * stride, sizeof(double) * stride, abytes);
        if (!r)
          r = run_engine((double*)(zb + lb.a), m, n, lda, p, (double*)(zb + lb.coeffs),
                         (int64_t*)(zb + lb.perm), (int64_t*)(zb + lb.swaps), lb.swap_cap,
                         (dmqr_step*)(zb + lb.steps), lb.step_cap, nullptr, zbase, per_engine, &infos[g0], nullptr,
                         0, (void*)s, 0, &sg, g, (int64_t)zblk, zrec);
        for (int z = 0; z < g && !r; ++z)
          if (infos[g0 + z].n_swaps > swap_cap) r = DMQR_ECAP;
        cp2(A + g0 * stride, sizeof(double) * stride, zb + lb.a, zblk, abytes);
        cp2(coeffs + g0 * kmax, sizeof(double) * kmax, zb + lb.coeffs, zblk, sizeof(double) * kmax);
        cp2(perm + g0 * n, sizeof(int64_t) * n, zb + lb.perm, zblk, sizeof(int64_t) * n);
        cp2(swaps + g0 * 2 * swap_cap, sizeof(int64_t) * 2 * swap_cap, zb + lb.swaps, zblk,
            sizeof(int64_t) * 2 * swap_cap);
        cp2(steps + g0 * step_cap, sizeof(dmqr_step) * step_cap, zb + lb.steps, zblk,
            sizeof(dmqr_step) * step_cap);
        for (int z = 0; z < g; ++z)
          if (r || !infos[g0 + z].status) infos[g0 + z].status = r ? r : infos[g0 + z].status;
        if (r && !lane_rc[q]) lane_rc[q] = r;
      }
      cudaStreamSynchronize(s);  // (the graph exec and the records are released below)
      cudaFreeHost(zrec);
    }
    lane_err[q] = last_cuda_error();
    cudaEventRecord(done[q], ls[q]);
  };
  std::vector<std::thread> th;
  for (int q = 1; q < nlanes; ++q) th.emplace_back(work, q);
  work(0);
  for (auto& t : th) t.join();
  for (int q = 0; q < nlanes; ++q) {
    CK(cudaStreamWaitEvent(st, done[q], 0));
    cudaEventDestroy(done[q]);
    cudaStreamDestroy(ls[q]);
  }
  cudaEventDestroy(start);
  for (int q = 0; q < nlanes; ++q)
    if (lane_rc[q]) {
      if (lane_rc[q] == DMQR_ECUDA) last_cuda_error() = lane_err[q];
      return lane_rc[q];
    }
  return 0;
}

size_t dmqr_form_q_workspace_bytes(int64_t m, int64_t qcols) {
  (void)m;
  const size_t q = (size_t)std::max<int64_t>(qcols, 1);
  // Wp (splits x 64 x qcols), W (64 x qcols), Sp (splits x 64 x 64), T (64 x 64)
  return al(sizeof(double) * FQ_NSPLIT * FQ_NB * q) + al(sizeof(double) * FQ_NB * q) +
         al(sizeof(double) * FQ_NSPLIT * FQ_NB * FQ_NB) + al(sizeof(double) * FQ_NB * FQ_NB);
}

/* Singular values of a batch of small matrices by one-sided Jacobi (the
 * reference's verification oracle jacobi_svd, svd.py:117-143); X is
 * overwritten.  Verification tooling for the ratio diagnostics. */
int dmqr_jacobi_svd_batched_f64(double* X, int64_t batch, int64_t m, int64_t n, int64_t ld, int64_t stride,
                                double tol, int32_t max_sweeps, double* sig, int32_t* sweeps, int32_t* converged,
                                void* stream) {
  if (batch < 0 || m < 0 || n < 0 || n > JS_NMAX || ld < std::max<int64_t>(1, m) || stride < ld * n ||
      max_sweeps < 1 || !(tol > 0.0))
    return DMQR_EINVAL;
  if (batch == 0 || n == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const DevInfo d = dev_info();
  const unsigned grid = (unsigned)std::min<int64_t>(batch, (int64_t)d.sms * 4);
  k_jacobi_svd<<<grid, JS_T, 0, st>>>(X, batch, m, (int)n, ld, stride, tol, max_sweeps, sig, sweeps, converged);
  NOTE_LAUNCH();
  CK(cudaGetLastError());
  return 0;
}

int dmqr_form_q_f64(const double* packed, int64_t m, int64_t n, int64_t lda, const double* coeffs,
                    int64_t n_factored, double* Q, int64_t qcols, int64_t ldq, void* workspace, size_t ws_bytes,
                    void* stream) {
  if (m < 0 || n < 0 || lda < std::max<int64_t>(1, m) || ldq < std::max<int64_t>(1, m) || qcols < 0 ||
      qcols > m || n_factored < 0 || n_factored > std::min(m, n))
    return DMQR_EINVAL;
  if (ws_bytes < dmqr_form_q_workspace_bytes(m, qcols)) return DMQR_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  if (m == 0 || qcols == 0) return 0;
  {
    DevAttrs* da = nullptr;
    int rc = set_attrs(dev_info(), &da);
    if (rc) return rc;
  }
  const size_t q = (size_t)qcols;
  unsigned char* wsb = (unsigned char*)workspace;
  double* Wp = (double*)wsb;
  double* W = (double*)(wsb + al(sizeof(double) * FQ_NSPLIT * FQ_NB * q));
  double* Sp = (double*)((unsigned char*)W + al(sizeof(double) * FQ_NB * q));
  double* T = (double*)((unsigned char*)Sp + al(sizeof(double) * FQ_NSPLIT * FQ_NB * FQ_NB));
  k_q_init<<<(unsigned)std::min<int64_t>(ceil_div(m * qcols, 256), 148 * 16), 256, 0, st>>>(Q, m, qcols, ldq);
  NOTE_LAUNCH();
  // reflectors s >= qcols act on rows >= s, where [I; 0] is still zero: no-ops
  const int64_t p = std::min(n_factored, qcols);
  for (int64_t j0 = (p > 0 ? (p - 1) / FQ_NB * FQ_NB : 0); p > 0 && j0 >= 0; j0 -= FQ_NB) {
    const int nb = (int)std::min<int64_t>(FQ_NB, p - j0);
    const int64_t mp = m - j0, cols = qcols - j0;
    const int64_t split_rows = std::max<int64_t>(1024, ceil_div(ceil_div(mp, FQ_NSPLIT), FQ_KR) * FQ_KR);
    const int nsplit = (int)ceil_div(mp, split_rows);
    k_fq_w<<<dim3(1, nsplit), FQ_T, 0, st>>>(packed, lda, j0, nb, mp, nullptr, 0, FQ_NB, Sp, split_rows);
    NOTE_LAUNCH();
    k_fq_t<<<1, FQ_T, FQ_SMEM2, st>>>(Sp, nsplit, nb, coeffs, j0, T);
    NOTE_LAUNCH();
    k_fq_w<<<dim3((unsigned)ceil_div(cols, FQ_NB), nsplit), FQ_T, 0, st>>>(packed, lda, j0, nb, mp, Q, ldq, cols,
                                                                          Wp, split_rows);
    NOTE_LAUNCH();
    k_fq_tw<<<(unsigned)ceil_div(cols, FQ_NB), FQ_T, FQ_SMEM2, st>>>(Wp, nsplit, nb, T, cols, W);
    NOTE_LAUNCH();
    k_fq_upd<<<dim3((unsigned)ceil_div(cols, FQ_NB), (unsigned)ceil_div(mp, FQ_NB)), FQ_T, FQ_SMEM2, st>>>(
        packed, lda, j0, nb, mp, Q, ldq, cols, W);
    NOTE_LAUNCH();
  }
  CK(cudaGetLastError());
  return 0;
}

void dmqr_stats_enable(int32_t on) { g_prof.store(on); }

void dmqr_stats_get(dmqr_stats* out, int32_t reset) {
  if (out) {
    out->kernel_launches = g_launches.load();
    out->calls = g_calls.load();
    out->timed_steps = g_acc.steps;
    out->ms_select = g_acc.ms[0];
    out->ms_panel = g_acc.ms[1];
    out->ms_trailing = g_acc.ms[2];
    out->ms_norms = g_acc.ms[3];
    out->ms_pivot = g_acc.ms[4];
  }
  if (reset) {
    g_launches.store(0);
    g_calls.store(0);
    g_acc = ProfAcc{};
  }
}

/* debug hook (not part of the reference surface): flatten the control block
 * of a workspace used by dmqr_qrdm_f64 into out[16 + 4*72] int64 (device). */
/* debug: panel phase clocks of step 2 (when stats were enabled with mode 2) */
int dmqr_debug_panel_clocks(const void* workspace, int64_t m, int64_t n, int64_t* out) {
  const Layout L = layout(m, n);
  CK(cudaMemcpy(out, (const unsigned char*)workspace + L.pdbg, sizeof(long long) * 64 * 16, cudaMemcpyDeviceToHost));
  return 0;
}

/* debug: per-step kernel spans of the last factorization run in this
 * workspace with DMQR_TIMELINE set: out[64 * 32 + 1024], step s, kernel k ->
 * [32 s + 2 k] first start, [32 s + 2 k + 1] last exit (globaltimer ns) */
int dmqr_debug_timeline(const void* workspace, int64_t m, int64_t n, int64_t* out) {
  const Layout L = layout(m, n);
  CK(cudaMemcpy(out, (const unsigned char*)workspace + L.tl, sizeof(unsigned long long) * TL_WORDS,
                cudaMemcpyDeviceToHost));
  return 0;
}

/* debug: CTA 0's phase cycles of the last fused small-matrix launch run with
 * DMQR_SMALL_CLOCKS set (out[16] int64 on the host; slots in small.cuh) */
int dmqr_debug_small_clocks(int64_t* out) {
  if (!g_small_clk) return DMQR_EINVAL;
  CK(cudaMemcpy(out, g_small_clk, sizeof(long long) * 32, cudaMemcpyDeviceToHost));
  return 0;
}

/* release the pooled pinned poll records / events / copy streams (all devices);
 * only while no engine call is running */
void dmqr_release_resources(void) {
  std::lock_guard<std::mutex> lk(g_slot_mu);
  for (HostSlot* h : g_slot_all) {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(h->dev);
    if (h->copy) cudaStreamDestroy(h->copy);
    for (auto e : h->ev) cudaEventDestroy(e);
    cudaFreeHost(h->rec);
    cudaSetDevice(cur);
    delete h;
  }
  g_slot_all.clear();
  g_slot_free.clear();
}

int dmqr_debug_ctl(const void* workspace, int64_t* out, void* stream) {
  k_debug_ctl<<<1, 32, 0, (cudaStream_t)stream>>>((const Ctl*)workspace, out);
  CK(cudaGetLastError());
  return 0;
}

}  // extern "C"
