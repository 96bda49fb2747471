// Candidate cosine matrix (DMMA Gram) + greedy delta filter + swap plan.
//   cosine_matrix          dm.py:100-115: G = C^T C, Theta = triu(G D^-1 D^-1, 1) mirrored, diag 1
//   dm_select filter       dm.py:151-177 (+ delta_max guard), gamma
//   k_s, eps_s             rrqr.py:355-357
//   _move_selected_to_front rrqr.py:294-312: exact transposition sequence with position patching
// k_gram: the Gram reduction over m' rows is split across up to one CTA per SM;
// each CTA streams 64-row slabs of the <= 65 gathered candidate columns into
// shared memory with cp.async (double-buffered) and runs 8x8x4 fp64 MMAs
// (SASS DMMA) on the upper tiles, writing per-CTA partials.
// k_gram_finish: one CTA per upper tile sums the partials in fixed order
// (deterministic); the last CTA to finish builds Theta, runs the greedy filter
// with one warp (ballots over the chosen set), and writes the swap plan.
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int GRAM_T = 256;
static_assert(DMQR_KP <= 128, "k_gram: one bulk copy per thread for the candidate and the reflector columns");
constexpr int GRAM_ROWS = 32;  // slab height (one slab per CTA up to 148 x 32 rows)
constexpr int GRAM_LD = 36;    // 32 rows + 4: conflict-free fragment loads (ld = 4 mod 16)
constexpr int GRAM_PART = DMQR_KP * DMQR_KP;
// [2][KP][LD] candidate slabs, [2][KP][LD] pending-panel Y slabs, [KP][KP] Wt of the candidates
constexpr size_t GRAM_SMEM = sizeof(double) * (4 * DMQR_KP * GRAM_LD + DMQR_KP * DMQR_KP);

// Selection finalize, one warp, shared-memory scratch (rrqr.py:294-312, 355-357).
// c->sel[0..nsel) holds the selected absolute columns (seed first).  Writes
// k_s, eps_s, gamma, the reference's exact transposition sequence
// (tgt = n_s+i, src = position of sel[i] at time i, with the "first later
// pos == tgt -> src" patch) and the same sequence composed into column moves
// new[dst] = old[src] for k_swap_*.
//
// The patch rule means sel[i] moves only when it sits in a window slot n_s+d
// that is filled earlier (d < i): it then jumps to src_d.  Slots strictly
// increase along such a chain, so src_i = follow(sel[i]) over already known
// src_d -- a short sequential loop on one lane; everything else is parallel.
struct PlanSmem {
  int sel[DMQR_KP];    // c->sel staged in shared memory (the serial loop's reads)
  int src[DMQR_KP];    // src_i
  int win[DMQR_KP];    // content of window slot n_s+i at time i (W_i)
  int lastw[DMQR_KP];  // latest content written into window slot d (-1: none)
};

// sel_smem: the selected columns already in shared memory (else read from c->sel)
__device__ void plan_swaps_warp(Ctl* c, const CtlSnap& S, int nsel, double gamma, PlanSmem& ps,
                                const int* sel_smem = nullptr, bool write_gamma = true) {
  const int lane = threadIdx.x & 31;
  const int n_s = S.n_s;
  const int k_s = (int)min((int64_t)nsel, S.kmax - n_s);
  // inw: the entries i < k_s whose selected column sits inside the window
  // [n_s, n_s + KP).  Only those can follow a chain, write lastw or collide with
  // an earlier source; every other entry has src_i = sel[i] and is planned in
  // parallel.  (A write to lastw[i] comes from an i' < i: a chain ends at a slot
  // >= i' or outside the window, and slot i' itself is no move -- so lastw[i]
  // is final once the serial pass is over, and W_i can be read after it.)
  constexpr int NW = (DMQR_KP + 31) / 32;
  unsigned inw[NW];
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int d = 32 * w + lane;
    bool in = false;
    if (d < DMQR_KP) {
      const int s = (d < nsel) ? (sel_smem ? sel_smem[d] : c->sel[d]) : 0;
      ps.lastw[d] = -1;
      ps.sel[d] = s;
      if (d < k_s) {
        ps.src[d] = s;
        const int dd = s - n_s;
        in = dd >= 0 && dd < DMQR_KP;
      }
    }
    inw[w] = __ballot_sync(0xffffffffu, in);
  }
  __syncwarp();
  if (lane == 0) {
    c->nsel = nsel;
    c->k_s = k_s;
    if (write_gamma) c->gamma = gamma;
    c->eps_s = S.tau * S.umax;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      unsigned b = inw[w];
      while (b) {
        const int i = 32 * w + __ffs(b) - 1;
        b &= b - 1;
        int p = ps.sel[i];
        int d = p - n_s;
        while (d >= 0 && d < i) {  // sel[i] sat in slot n_s+d when it was filled
          p = ps.src[d];
          d = p - n_s;
        }
        ps.src[i] = p;
        const int wi = (ps.lastw[i] >= 0) ? ps.lastw[i] : n_s + i;
        const int ds = p - n_s;
        if (p != n_s + i && ds >= 0 && ds < DMQR_KP) ps.lastw[ds] = wi;
      }
    }
  }
  __syncwarp();
  for (int i = lane; i < k_s; i += 32) ps.win[i] = (ps.lastw[i] >= 0) ? ps.lastw[i] : n_s + i;
  __syncwarp();
  // transposition list in order (compaction by ballot)
  int ns = 0;
  for (int i0 = 0; i0 < k_s; i0 += 32) {
    const int i = i0 + lane;
    const bool sw = (i < k_s) && ps.src[i] != n_s + i;
    const unsigned b = __ballot_sync(0xffffffffu, sw);
    if (sw) {
      const int at = ns + __popc(b & ((1u << lane) - 1u));
      c->sw_a[at] = n_s + i;
      c->sw_b[at] = ps.src[i];
    }
    ns += __popc(b);
  }
  // moves: window slots (selected block, plus later slots that received content),
  // then out-of-window sources whose last write is swap i
  int nm = 0;
  for (int d0 = 0; d0 < DMQR_KP; d0 += 32) {
    const int d = d0 + lane;
    int src = -1;
    if (d < k_s)
      src = ps.sel[d];
    else if (d < DMQR_KP && ps.lastw[d] >= 0)
      src = ps.lastw[d];
    const bool mv = (src >= 0) && src != n_s + d;
    const unsigned b = __ballot_sync(0xffffffffu, mv);
    if (mv) {
      const int at = nm + __popc(b & ((1u << lane) - 1u));
      c->mv_dst[at] = n_s + d;
      c->mv_src[at] = src;
    }
    nm += __popc(b);
  }
  for (int i0 = 0; i0 < k_s; i0 += 32) {
    const int i = i0 + lane;
    bool mv = false;
    int p = 0;
    if (i < k_s) {
      p = ps.src[i];
      const int dp = p - n_s;
      if (p != n_s + i && !(dp >= 0 && dp < DMQR_KP)) {
        mv = true;  // unless a later swap has the same source (only an in-window entry can)
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          unsigned b = inw[w];
          while (b) {
            const int t = 32 * w + __ffs(b) - 1;
            b &= b - 1;
            if (t > i) mv &= (ps.src[t] != p);
          }
        }
      }
    }
    const unsigned b = __ballot_sync(0xffffffffu, mv);
    if (mv) {
      const int at = nm + __popc(b & ((1u << lane) - 1u));
      c->mv_dst[at] = p;
      c->mv_src[at] = ps.win[i];
    }
    nm += __popc(b);
  }
  if (lane == 0) {
    c->nsw = ns;
    c->nmv = nm;
  }
}

// upper-triangular tile t of an nt x nt tile grid -> (ti, tj)
__device__ __forceinline__ void tile_ij(int t, int nt, int& ti, int& tj) {
  ti = 0;
  while (t >= nt - ti) {
    t -= nt - ti;
    ++ti;
  }
  tj = ti + t;
}

// Look-ahead (Ctl::pend): the candidate columns still lack the previous
// step's C -= Y Wt below its R rows.  Each slab is brought up to date in
// shared memory (the same DMMA sequence per element as k_trail_b, so the
// values are bitwise the serial update's), written back, and only then enters
// the Gram; k_gram_finish flags the candidates (upd) once every CTA is done.
// A scalar-fallback step (kind 1) runs the same update on its single column.
__global__ void __launch_bounds__(GRAM_T) k_gram(Ctl* c, double* __restrict__ A,
                                                 double* __restrict__ part, const double* __restrict__ Wt,
                                                 int64_t ldz, const uint8_t* __restrict__ upd) {
  zshift(c, c, A, part, Wt, upd);
  pdl_enter();
  // the candidate list is read with the control block snapshot (one round trip)
  const int cand_pre = (threadIdx.x < DMQR_KP) ? c->cand[threadIdx.x] : 0;
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 1);
  if (S.done) return;
  const bool pendu = S.la && S.pend;
  if (S.kind != 0 && !pendu) return;
  const int ncand = (S.kind == 0) ? S.ncand : 1;
  if (ncand == 1 && S.kind == 0 && blockIdx.x == 0 && threadIdx.x < 32) {
    // no candidates: J = [seed], gamma = 1 (dm.py:145-146)
    __shared__ PlanSmem ps1;
    if (threadIdx.x == 0) c->sel[0] = c->cand[0];
    __syncwarp();
    plan_swaps_warp(c, S, 1, 1.0, ps1);
  }
  if (ncand == 1 && !pendu) return;
  const bool gram = S.kind == 0 && ncand > 1;
  extern __shared__ __align__(16) double gsm[];  // [2][KP][GRAM_LD] slabs, [2][KP][GRAM_LD] Y, [KP][KP] Wt
  __shared__ int s_cand[DMQR_KP];
  __shared__ int s_live[DMQR_KP];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n_s = S.n_s, m = S.m, lda = S.lda;
  const int64_t mp = m - n_s;
  const int np8 = round_up(ncand, 8);
  const int nt = np8 / 8;
  const int ntiles = gram ? nt * (nt + 1) / 2 : 0;
  const int pl = pendu ? S.pend_l : 0;
  const int64_t pns = pendu ? S.pend_ns : 0;
  const int plp4 = (pl + 3) / 4 * 4;
  double* ysl = gsm + 2 * DMQR_KP * GRAM_LD;
  double* wsm = gsm + 4 * DMQR_KP * GRAM_LD;
  if (tid < DMQR_KP) s_cand[tid] = (tid < ncand) ? cand_pre : 0;
  __syncthreads();
  // the candidates' Wt columns (indexed from n_s = pending n_s + l) by cp.async,
  // in flight with their upd flags and the first slab; columns whose update
  // is already applied (upd) are zeroed once everything has landed
  bool live = false;
  if (tid < DMQR_KP) live = (tid < ncand) && pendu && !upd[s_cand[tid]];
  if (pendu)
    for (int e = tid; e < plp4 * DMQR_KP; e += GRAM_T) {
      const int t = e / DMQR_KP, q = e % DMQR_KP;
      if (t < pl && q < ncand)
        cp_async8(wsm + t * DMQR_KP + q, Wt + t * ldz + (s_cand[q] - n_s));
      else
        wsm[t * DMQR_KP + q] = 0.0;
    }
  if (tid < DMQR_KP) s_live[tid] = live;

  const int64_t rpc = ceil_div(ceil_div(mp, (int64_t)gridDim.x), GRAM_ROWS) * GRAM_ROWS;
  const int64_t r_begin = (int64_t)blockIdx.x * rpc;
  const int64_t r_end = min(mp, r_begin + rpc);

  // tiles wid, wid + 8, ... (<= 6 per warp); static indexing keeps the
  // accumulators in registers
  double acc[6][2];
  int tij[6];
  int my_tiles = 0;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const int t = wid + q * (GRAM_T / 32);
    int ti = 0, tj = 0;
    if (t < ntiles) {
      tile_ij(t, nt, ti, tj);
      my_tiles = q + 1;
    }
    tij[q] = ti * 16 + tj;
    acc[q][0] = acc[q][1] = 0.0;
  }
  __syncthreads();
  const int nslab = (r_end > r_begin) ? (int)ceil_div(r_end - r_begin, GRAM_ROWS) : 0;
  // Whole slabs (the usual case) arrive by TMA bulk copies: one 256-byte
  // column segment per candidate and per pending-Y column, issued by warp 0 and
  // landing on the buffer's mbarrier.  A slab whose first global row is odd is
  // fetched from the row above (16-byte alignment) into a buffer shifted by one
  // element, so row r of the slab sits at buf + off + r either way.  Partial
  // slabs at the end of a CTA's range keep the zero-filling cp.async path.
  __shared__ __align__(8) uint64_t s_bar[2];
  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
  }
  __syncthreads();
  auto slab_full = [&](int sl) { return kTMAGram && r_begin + (int64_t)(sl + 1) * GRAM_ROWS <= r_end; };
  auto slab_off = [&](int sl) { return slab_full(sl) ? (int)((n_s + r_begin + (int64_t)sl * GRAM_ROWS) & 1) : 0; };
  auto issue = [&](int sl) {
    double* buf = gsm + (sl & 1) * DMQR_KP * GRAM_LD;
    double* ys = ysl + (sl & 1) * DMQR_KP * GRAM_LD;
    const int64_t r0 = r_begin + (int64_t)sl * GRAM_ROWS;
    if (slab_full(sl)) {
      const int off = slab_off(sl);
      for (int e = tid; e < (np8 - ncand) * GRAM_ROWS; e += GRAM_T)  // padding candidates
        buf[(ncand + e / GRAM_ROWS) * GRAM_LD + off + e % GRAM_ROWS] = 0.0;
      for (int e = tid; e < (plp4 - pl) * GRAM_ROWS; e += GRAM_T)  // padding reflectors
        ys[(pl + e / GRAM_ROWS) * GRAM_LD + off + e % GRAM_ROWS] = 0.0;
      {  // one copy per thread (the issue is spread over the CTA)
        const unsigned seg = (unsigned)(GRAM_ROWS + 2 * off) * (unsigned)sizeof(double);
        const int ncols = (gram || pendu) ? ncand : 0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // buffer reuse after generic accesses
        if (tid == 0) mbar_arrive_expect_tx(&s_bar[sl & 1], seg * (unsigned)(ncols + pl));
        const double* g0 = A + (n_s + r0 - off);
        if (tid < ncols)
          bulk_g2s(buf + tid * GRAM_LD, g0 + (int64_t)s_cand[tid] * lda, seg, &s_bar[sl & 1]);
        else if (tid >= 128 && tid - 128 < pl)
          bulk_g2s(ys + (tid - 128) * GRAM_LD, g0 + (pns + tid - 128) * lda, seg, &s_bar[sl & 1]);
      }
      cp_async_commit();  // (an empty group keeps the cp.async group accounting per slab)
      return;
    }
    for (int e = tid; e < np8 * GRAM_ROWS; e += GRAM_T) {
      const int col = e / GRAM_ROWS, row = e % GRAM_ROWS;
      const int64_t r = r0 + row;
      double* dst = buf + col * GRAM_LD + row;
      if (col < ncand && r < r_end)
        cp_async8(dst, A + (n_s + r) + (int64_t)s_cand[col] * lda);
      else
        *dst = 0.0;
    }
    // Y of the pending panel on these rows (all strictly below its diagonal)
    for (int e = tid; e < plp4 * GRAM_ROWS; e += GRAM_T) {
      const int t = e / GRAM_ROWS, row = e % GRAM_ROWS;
      const int64_t r = r0 + row;
      double* dst = ys + t * GRAM_LD + row;
      if (t < pl && r < r_end)
        cp_async8(dst, A + (n_s + r) + (pns + t) * lda);
      else
        *dst = 0.0;
    }
    cp_async_commit();
  };
  if (nslab > 0) {
    issue(0);
  } else {  // (no rows here: drain the Wt copies)
    cp_async_commit();
    cp_async_wait<0>();
  }
  for (int sl = 0; sl < nslab; ++sl) {
    if (sl + 1 < nslab) {
      issue(sl + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    if (slab_full(sl)) mbar_wait_parity(&s_bar[sl & 1], (unsigned)(sl >> 1) & 1u);
    __syncthreads();
    if (sl == 0 && pendu) {  // (the Wt copies landed with slab 0)
      for (int e = tid; e < plp4 * DMQR_KP; e += GRAM_T)
        if (!s_live[e % DMQR_KP]) wsm[e] = 0.0;
      __syncthreads();
    }
    double* buf = gsm + (sl & 1) * DMQR_KP * GRAM_LD + slab_off(sl);
    if (pendu) {
      // buf[col][row] += (-Y) Wt for live candidates: warp w owns rows
      // 8 (w & 3) .. +8 and column tiles [5 (w >> 2), +5)
      const double* ys = ysl + (sl & 1) * DMQR_KP * GRAM_LD + slab_off(sl);
      const int rr = (wid & 3) * 8 + (lane >> 2);
      const int64_t r0 = r_begin + (int64_t)sl * GRAM_ROWS;
      const int qh1 = min(nt, (wid >> 2) * 5 + 5);
      for (int q0 = (wid >> 2) * 5; q0 < qh1; q0 += 3) {
        double u3[3][2];
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) u3[q][h] = (q0 + q < qh1) ? buf[((q0 + q) * 8 + 2 * (lane & 3) + h) * GRAM_LD + rr] : 0.0;
        for (int ks = 0; ks < plp4; ks += 4) {
          const int t = ks + (lane & 3);
          const double a = -ys[t * GRAM_LD + rr];
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if (q0 + q < qh1) dmma884(u3[q][0], u3[q][1], a, wsm[t * DMQR_KP + (q0 + q) * 8 + (lane >> 2)]);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 3; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = (q0 + q) * 8 + 2 * (lane & 3) + h;
            if (q0 + q < qh1 && col < ncand && s_live[col]) {
              buf[col * GRAM_LD + rr] = u3[q][h];
              if (r0 + rr < r_end) A[(n_s + r0 + rr) + (int64_t)s_cand[col] * lda] = u3[q][h];
            }
          }
      }
      __syncthreads();
    }
#pragma unroll 4
    for (int ks = 0; ks < GRAM_ROWS / 4; ++ks) {
      const int kr = 4 * ks + (lane & 3);
#pragma unroll
      for (int q = 0; q < 6; ++q)
        if (q < my_tiles) {
          const double av = buf[((tij[q] >> 4) * 8 + (lane >> 2)) * GRAM_LD + kr];
          const double bv = buf[((tij[q] & 15) * 8 + (lane >> 2)) * GRAM_LD + kr];
          dmma884(acc[q][0], acc[q][1], av, bv);
        }
    }
    __syncthreads();
  }
  double* my = part + (int64_t)blockIdx.x * GRAM_PART;
#pragma unroll
  for (int q = 0; q < 6; ++q)
    if (q < my_tiles) {
      const int row = (tij[q] >> 4) * 8 + (lane >> 2);
      const int col = (tij[q] & 15) * 8 + 2 * (lane & 3);
      my[row * DMQR_KP + col] = acc[q][0];
      my[row * DMQR_KP + col + 1] = acc[q][1];
    }
}

struct FinSmem {
  double g[DMQR_KP * DMQR_KP];  // Gram, then Theta (upper)
  int cand[DMQR_KP];            // c->cand staged with the Gram (no round trip in the serial tail)
  int sel[DMQR_KP];             // the selected columns (seed first)
  double inv[DMQR_KP];
  double rowsum[DMQR_KP];
  double amax[DMQR_KP];
  int chosen[DMQR_KP];
  unsigned long long conf[DMQR_KP];
  int is_last, bad, zero, nch;
  PlanSmem plan;
};

// grid: one CTA per upper 8x8 tile (45 for 65 candidates), GRAM_T threads.
__global__ void __launch_bounds__(GRAM_T) k_gram_finish(Ctl* c, const double* __restrict__ A,
                                                        const double* __restrict__ part, int G,
                                                        double* __restrict__ gfin, uint8_t* __restrict__ upd,
                                                        long long* __restrict__ tline) {
  zshift(c, c, A, part, gfin, upd);
  const long long t_in = gtimer();
  pdl_enter();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 2);
  if (S.done) return;
#define GFT(k) \
  if (tline && threadIdx.x == 0) tline[512 + 8 * (S.step_idx & 63) + (k)] = gtimer()
  if (S.la && S.pend && blockIdx.x == 0) {  // k_gram brought the candidates up to date
    const int nc = (S.kind == 0) ? S.ncand : 1;
    for (int q = threadIdx.x; q < nc; q += blockDim.x) upd[c->cand[q]] = 1;
  }
  if (S.kind != 0) return;
  const int ncand = S.ncand;
  if (ncand == 1) return;
  extern __shared__ __align__(16) unsigned char fin_raw[];
  FinSmem& sm = *reinterpret_cast<FinSmem*>(fin_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int np8 = round_up(ncand, 8);
  const int nt = np8 / 8;
  const int ntiles = nt * (nt + 1) / 2;
  if ((int)blockIdx.x < ntiles) {
    int ti, tj;
    tile_ij(blockIdx.x, nt, ti, tj);
    // 64 entries x 4 threads, each summing a quarter of the partials; fixed combine order
    const int e = tid >> 2, g4 = tid & 3;
    const int i = ti * 8 + (e >> 3), j = tj * 8 + (e & 7);
    // 8 independent loads in flight per thread; the combine order is fixed by G
    const double* pp = part + i * DMQR_KP + j;
    double sv[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll 5
    for (int b0 = g4; b0 < G; b0 += 32) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int b = b0 + 4 * q;
        if (b < G) sv[q] += __ldcg(pp + (int64_t)b * GRAM_PART);
      }
    }
    double s = ((sv[0] + sv[1]) + (sv[2] + sv[3])) + ((sv[4] + sv[5]) + (sv[6] + sv[7]));
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (g4 == 0 && i <= j) {  // both triangles from the upper entry: the last CTA's Theta pass runs row-wise
      gfin[i * DMQR_KP + j] = s;
      gfin[j * DMQR_KP + i] = s;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const unsigned prev = atomicAdd(&c->gram_count, 1u);
    sm.is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!sm.is_last) return;
  __threadfence();
  if (tline && tid == 0) tline[512 + 8 * (S.step_idx & 63) + 0] = t_in;
  GFT(1);
  if (tid == 0) {
    c->gram_count = 0u;
    sm.bad = 0;
    sm.zero = 0;
  }
  // the whole reduced Gram in one round trip (16-byte L2 copies; only the
  // upper entries of the first ncand rows / columns are read)
  for (int e2 = tid; e2 < DMQR_KP * DMQR_KP / 2; e2 += GRAM_T) cp_async16(sm.g + 2 * e2, gfin + 2 * e2, 16);
  cp_async_commit();
  for (int q = tid; q < ncand; q += GRAM_T) sm.cand[q] = c->cand[q];
  cp_async_wait<0>();
  __syncthreads();
  // over/underflow risk: the diagonal (sums of squares) bounds every entry;
  // norms and the zero-column check (dm.py:107-109) in the same pass
  auto norms_pass = [&]() {
    for (int i = tid; i < ncand; i += GRAM_T) {
      const double d = sm.g[i * DMQR_KP + i];
      if (!(d > 1e-280 && d < 1e280)) sm.bad = 1;
      const double nr = sqrt(d);
      if (nr == 0.0) sm.zero = 1;
      sm.inv[i] = 1.0 / nr;
    }
  };
  norms_pass();
  __syncthreads();
  const int64_t n_s = S.n_s, m = S.m, lda = S.lda, mp = m - n_s;
  if (sm.bad) {
    // slow path (extreme magnitudes only): recompute with exact 2^-e column scales
    if (tid == 0) sm.zero = 0;  // (set from the unusable Gram; decided again below)
    for (int i = wid; i < ncand; i += GRAM_T / 32) {
      const double* ci = A + (int64_t)c->cand[i] * lda + n_s;
      double am = 0.0;
      for (int64_t r = lane; r < mp; r += 32) am = fmax(am, fabs(ci[r]));
      am = warp_max(am);
      if (lane == 0) sm.amax[i] = am;
    }
    __syncthreads();
    for (int e = tid; e < ncand * ncand; e += GRAM_T) {
      const int i = e / ncand, j = e % ncand;
      if (j < i) continue;
      int ei = 0, ej = 0;
      if (sm.amax[i] > 0.0) frexp(sm.amax[i], &ei);
      if (sm.amax[j] > 0.0) frexp(sm.amax[j], &ej);
      const double* ci = A + (int64_t)c->cand[i] * lda + n_s;
      const double* cj = A + (int64_t)c->cand[j] * lda + n_s;
      double acc = 0.0;
      for (int64_t r = 0; r < mp; ++r) acc = fma(ldexp(ci[r], -ei), ldexp(cj[r], -ej), acc);
      sm.g[i * DMQR_KP + j] = acc;
      sm.g[j * DMQR_KP + i] = acc;
    }
    __syncthreads();
    norms_pass();  // (sets bad again when the scaled Gram is still out of range: harmless, not read again)
    __syncthreads();
  }
  if (sm.zero) {
    if (tid == 0) {
      c->status = -3;
      c->done = 1;
    }
    return;
  }
  GFT(2);
  // Theta: (G_ij * inv_i) * inv_j, i < j (dm.py:112), and its mirror image
  // (the filter and gamma read rows only, which is bank-conflict free).  The
  // Gram arrives symmetric, so entry (t, q) forms the upper entry's product
  // (min index first) in place: no transposed shared-memory stores (the row
  // stride of 72 doubles made them 16-way bank conflicts).  A warp per row;
  // the same pass ballots the row's conflict mask for the greedy filter
  // (dm.py:151-173): bit q of conf[t] is set when candidate q < t fails
  // |theta_qt| < delta; t is then accepted iff no accepted q conflicts.
  const bool dmax = S.use_delta_max != 0;
  {
    const double delta = S.delta;
    for (int t = wid; t < ncand; t += GRAM_T / 32) {
      unsigned bal[2] = {0u, 0u};
#pragma unroll
      for (int h = 0; h < 3; ++h) {
        const int q = lane + 32 * h;
        double av = 0.0;
        if (q < ncand && q != t) {
          const int i = min(t, q), j = max(t, q);
          const double th = __dmul_rn(__dmul_rn(sm.g[t * DMQR_KP + q], sm.inv[i]), sm.inv[j]);
          sm.g[t * DMQR_KP + q] = th;
          av = fabs(th);
        }
        if (h < 2) bal[h] = __ballot_sync(0xffffffffu, q < t && !(av < delta));
      }
      if (lane == 0 && t >= 1) sm.conf[t] = ((unsigned long long)bal[1] << 32) | bal[0];
    }
    // past the candidates: conflicts with everything (the chain below then reads
    // all 64 masks unconditionally -- predicated shared loads rebuild their address each)
    for (int t = ncand + tid; t < 64; t += GRAM_T) sm.conf[t] = ~0ull;
  }
  __syncthreads();
  GFT(3);
  if (!dmax) {
    GFT(6);
    if (wid == 0) {
      // the AND chain on one lane, branch-free (the accepted set as a bit mask;
      // candidate 64, the last possible, separately), then the chosen list by
      // ballot compaction in candidate order
      // (32-bit masks: candidates 1..31 chain on the low word; for 32..63 the
      // low-word conflicts are then known per lane and the chain runs on the
      // high word alone -- four dependent 32-bit ops per candidate, shifts
      // resolved at compile time)
      unsigned long long acc = 1ull;  // accepted q < 64
      int last = 0;                   // candidate 64 accepted
      unsigned alo = 1u, ahi = 0u;
      const unsigned* cw = reinterpret_cast<const unsigned*>(sm.conf);  // [2t] low, [2t+1] high word
      if (lane == 0) {
#pragma unroll
        for (int t = 1; t < 32; ++t) alo |= ((cw[2 * t] & alo) == 0u) ? (1u << t) : 0u;
      }
      alo = __shfl_sync(0xffffffffu, alo, 0);
      const bool freelo = (cw[2 * (32 + lane)] & alo) == 0u;
      const unsigned allow = __ballot_sync(0xffffffffu, freelo);
      if (lane == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          ahi |= ((cw[2 * (32 + j) + 1] & ahi) == 0u) ? (allow & (1u << j)) : 0u;
        }
        acc = ((unsigned long long)ahi << 32) | alo;
        if (ncand > 64) last = (sm.conf[64] & acc) == 0ull;
      }
      acc = __shfl_sync(0xffffffffu, acc, 0);
      last = __shfl_sync(0xffffffffu, last, 0);
      const bool b0 = (acc >> lane) & 1ull, b1 = (acc >> (lane + 32)) & 1ull;
      const unsigned m0 = __ballot_sync(0xffffffffu, b0), m1 = __ballot_sync(0xffffffffu, b1);
      const unsigned below = (1u << lane) - 1u;
      if (b0) sm.chosen[__popc(m0 & below)] = lane;
      if (b1) sm.chosen[__popc(m0) + __popc(m1 & below)] = lane + 32;
      if (lane == 0) {
        const int n64 = __popc(m0) + __popc(m1);
        if (last) sm.chosen[n64] = 64;
        sm.nch = n64 + last;
      }
    }
    __syncthreads();
    GFT(7);
    const int nch = sm.nch;
    if (wid == 0) {
      // the selection and the swap plan (warp 0) beside gamma (warps 1..7)
      for (int q = lane; q < nch; q += 32) {
        const int sq = sm.cand[sm.chosen[q]];
        sm.sel[q] = sq;
        c->sel[q] = sq;
      }
      __syncwarp();
      GFT(4);
      plan_swaps_warp(c, S, nch, 1.0, sm.plan, sm.sel, /*write_gamma=*/false);
      GFT(5);
      return;
    }
    // gamma = min_i 1 - (sum_j |theta_ij| - 1) over the chosen submatrix (dm.py:175-176)
    for (int p = wid - 1; p < nch; p += GRAM_T / 32 - 1) {
      const int i = sm.chosen[p];
      double sacc = 0.0;
      for (int q = lane; q < nch; q += 32) {
        const int jj = sm.chosen[q];
        sacc += (i == jj) ? 1.0 : fabs(sm.g[i * DMQR_KP + jj]);
      }
      sacc = warp_sum(sacc);
      if (lane == 0) sm.rowsum[p] = 1.0 - (sacc - 1.0);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(GRAM_T - 32) : "memory");  // warps 1..7 only
    if (wid != 1) return;
    double gmin = 1e300;
    for (int p = lane; p < nch; p += 32) gmin = fmin(gmin, sm.rowsum[p]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmin = fmin(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
    if (lane == 0) c->gamma = gmin;
    return;
  }
  if (wid != 0) return;
  // ---- greedy filter with the delta_max guard, one warp (dm.py:151-173) ----
  const double tau2 = S.tau * S.tau;
  const double delta = dmax ? tau2 / (double)max(c->k_max - 1, 1) : c->delta;
  const double guard = tau2;
  auto th = [&](int i, int j) { return fabs(i < j ? sm.g[i * DMQR_KP + j] : sm.g[j * DMQR_KP + i]); };
  int nch = 1;
  if (lane == 0) {
    sm.chosen[0] = 0;
    sm.rowsum[0] = 0.0;
  }
  __syncwarp();
  for (int t = 1; t < ncand; ++t) {
    bool ok = true;
    for (int q = lane; q < nch; q += 32) ok &= (th(sm.chosen[q], t) < delta);
    if (!__all_sync(0xffffffffu, ok)) continue;
    if (dmax) {
      double tot = 0.0;
      if (lane == 0)
        for (int q = 0; q < nch; ++q) tot += th(sm.chosen[q], t);
      tot = __shfl_sync(0xffffffffu, tot, 0);
      bool rej = tot >= guard;
      for (int q = lane; q < nch; q += 32) {
        const int jj = sm.chosen[q];
        rej |= (sm.rowsum[jj] + th(jj, t) >= guard);
      }
      if (__any_sync(0xffffffffu, rej)) continue;
      for (int q = lane; q < nch; q += 32) {
        const int jj = sm.chosen[q];
        sm.rowsum[jj] += th(jj, t);
      }
      __syncwarp();
      if (lane == 0) sm.rowsum[t] = tot;
    }
    if (lane == 0) sm.chosen[nch] = t;
    ++nch;
    __syncwarp();
  }
  // gamma = min_i 1 - (sum_j |theta_ij| - 1) over the chosen submatrix (dm.py:175-176)
  double gmin = 1e300;
  for (int p = lane; p < nch; p += 32) {
    const int i = sm.chosen[p];
    double sacc = 0.0;
    for (int q = 0; q < nch; ++q) {
      const int jj = sm.chosen[q];
      sacc += (i == jj) ? 1.0 : th(i, jj);
    }
    gmin = fmin(gmin, 1.0 - (sacc - 1.0));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) gmin = fmin(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
  for (int q = lane; q < nch; q += 32) {
    const int sq = sm.cand[sm.chosen[q]];
    sm.sel[q] = sq;
    c->sel[q] = sq;
  }
  __syncwarp();
  plan_swaps_warp(c, S, nch, gmin, sm.plan, sm.sel);
}

}  // namespace dmqr
