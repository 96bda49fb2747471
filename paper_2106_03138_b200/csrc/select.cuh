// Stop test, norm-floor test, seed argmax and the tau-candidate set.
//   check_stop      rrqr.py:189-203 (called at rrqr.py:336-338)
//   floor test      dm.py:139-143 -> NormFloorSignal -> scalar step rrqr.py:343-353
//   candidate_set   dm.py:81-97: seed = first argmax; {i != seed : u_i >= tau*u_seed}
//                   stably sorted by -u (ties -> smaller index), truncated to k_dm
// One CTA of 1024 threads over the trailing norms (n' <= a few 10^4 doubles,
// L2-resident).  Top-k_dm is a radix select on the IEEE bits of the
// non-negative norms (8 passes of 8 bits) followed by an index-ordered
// compaction of the tie class, so the result equals the reference's stable
// argsort exactly.
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int SEL_T = 1024;
constexpr int SEL_FCAP = 512;  // short-list capacity of the top-k_dm fast path

struct SelSmem {
  double red_v[32];
  int red_i[32];
  int scan[32];
  unsigned hist[256];
  int list_i[DMQR_KP * 2];
  double list_u[DMQR_KP * 2];
  int bc_i[4];
  unsigned long long bc_u64[2];
  double bc_d[2];
  double fl_u[SEL_FCAP];  // top-k_dm fast path: the short list (any order)
  int fl_i[SEL_FCAP];
  int fl_cnt;
};

// exclusive block scan of one int per thread (1024 threads); returns prefix, writes total
__device__ __forceinline__ int block_excl_scan(int v, int* scan_smem, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) scan_smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = scan_smem[lane];
    int s = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    scan_smem[lane] = s - t;  // exclusive warp offsets
    if (lane == 31) *total = s;
  }
  __syncthreads();
  int res = scan_smem[wid] + x - v;
  __syncthreads();
  return res;
}

// Wide selection (k_dm > DMQR_MAXK - 1; wide.cuh): the candidate list lives in
// the workspace (WideBufs) instead of shared memory and the control block, and
// a step that continues with its next panel chunk (Ctl::w_next) takes no new
// selection: its columns already sit at n_s, n_s+1, ...
template <bool WIDE>
__global__ void __launch_bounds__(SEL_T) k_select_t(Ctl* c, const double* __restrict__ u, WideBufs wb) {
  zshift(c, c, u);
  pdl_enter();
  const CtlSnap S = snap(c);
  TLSpan tl_span(S.done ? nullptr : S.tl, S.step_idx, 0);
  if (S.done) return;
  if (threadIdx.x == 0) {
    c->bar_count = 0u;  // the panel's grid-barrier counter restarts each step
    c->cq_fail = 1;     // the CholeskyQR2 panel (if launched) clears this on success
    c->q1_count = 0u;
    c->p_count = 0u;
    c->q1_fail = 0;
  }
  __shared__ SelSmem sm;
  __shared__ int s_total;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int n_s = S.n_s;
  const int n = (int)S.n;
  if (n_s >= S.kmax) {  // loop condition of rrqr.py:335
    if (tid == 0) c->done = 1;
    return;
  }
  if constexpr (WIDE) {
    __shared__ int s_wn;
    if (tid == 0) s_wn = ctl_ld(&c->w_next);
    __syncthreads();
    if (s_wn > 0) {  // the step's next chunk (rrqr.py:360-379 continues with column n_s)
      if (tid == 0) {
        const int k = min(s_wn, DMQR_MAXK);
        c->kind = 0;
        c->nsel = k;
        c->k_s = k;
        c->nsw = 0;
        c->nmv = 0;
        c->w_cont = 1;
        c->w_next = 0;
      }
      if (tid < DMQR_MAXK) c->sel[tid] = n_s + tid;
      return;
    }
    if (tid == 0) {
      c->w_cont = 0;
      c->w_done = 0;
      c->w_nmv = 0;
    }
  }
  const int np = n - n_s;
  // contiguous per-thread segments keep index order for compaction
  const int seg = (np + SEL_T - 1) / SEL_T;
  const int s0 = n_s + tid * seg;
  const int s1 = min(n, s0 + seg);

  // ---- first argmax over u[n_s:] (np.argmax semantics) ----
  double bv = -1.0;
  int bi = 0x7fffffff;
#pragma unroll 4
  for (int i = s0; i < s1; ++i) {  // (unrolled: the loads of four elements in flight together)
    double v = u[i];
    if (v > bv) {
      bv = v;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    sm.red_v[wid] = bv;
    sm.red_i[wid] = bi;
  }
  __syncthreads();
  if (wid == 0) {
    bv = sm.red_v[lane];
    bi = sm.red_i[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      sm.bc_d[0] = bv;
      sm.bc_i[0] = bi;
    }
  }
  __syncthreads();
  const double umax = sm.bc_d[0];
  const int seed = sm.bc_i[0];

  // ---- stop test (rrqr.py:197-203) ----
  if (S.stop_active) {
    const double lhs = sqrt((double)(n - n_s)) * umax;
    if (lhs <= S.stop_rhs) {
      if (tid == 0) {
        c->stopped = 1;
        c->done = 1;
      }
      return;
    }
  }
  // ---- norm floor -> scalar fallback step (dm.py:140, rrqr.py:219-235) ----
  if (umax <= S.floor) {
    if (tid == 0) {
      c->kind = 1;
      c->k_max = -1;
      c->umax = umax;
      c->ncand = 1;
      c->cand[0] = seed;
      c->nsel = 1;
      c->sel[0] = seed;
      c->k_s = 1;
      c->eps_s = 0.0;
      c->gamma = 1.0;
      c->nsw = (seed != n_s) ? 1 : 0;
      c->sw_a[0] = n_s;
      c->sw_b[0] = seed;
      c->nmv = (seed != n_s) ? 2 : 0;
      c->mv_dst[0] = n_s;
      c->mv_src[0] = seed;
      c->mv_dst[1] = seed;
      c->mv_src[1] = n_s;
    }
    return;
  }

  // ---- candidate set (dm.py:81-97) ----
  const double thr = S.tau * umax;
  const int k_dm = S.k_dm;
  int cnt = 0;
  for (int i = s0; i < s1; ++i) cnt += (i != seed && u[i] >= thr);
  int total;
  int off = block_excl_scan(cnt, sm.scan, &s_total);
  __syncthreads();
  total = s_total;

  int* const list_i = WIDE ? wb.list_i : sm.list_i;
  double* const list_u = WIDE ? wb.list_u : sm.list_u;
  int nlist;
  if (total <= k_dm) {
    // all candidates, index order
    int p = off;
    for (int i = s0; i < s1; ++i)
      if (i != seed && u[i] >= thr) {
        list_i[p] = i;
        list_u[p] = u[i];
        ++p;
      }
    nlist = total;
  } else {
    // Fast path (k_dm <= 64): a short list that is sure to hold the k_dm
    // largest candidates, then rank counting in the reference's order (u
    // descending, ties by index ascending) -- the rank IS the position in the
    // stable argsort, so no select and no separate sort.  The list: every
    // candidate at or above T0 = the smallest, over the 32 warps, of a warp's
    // second-largest candidate (elements dealt round-robin): each warp then
    // holds two candidates >= T0, 64 >= k_dm in all.  A warp with fewer than
    // two candidates gives T0 = -1 (all candidates); a list that overflows
    // (heavy ties) falls through to the radix select below.
    bool fast_done = false;
    if constexpr (!WIDE) {
      if (k_dm <= 64) {
        double T0 = -1.0;
        if (total > SEL_FCAP) {
          double v1 = -1.0;
          int i1 = -1;
          for (int i = n_s + tid; i < n; i += SEL_T) {
            const double v = u[i];
            if (i != seed && v >= thr && v > v1) {
              v1 = v;
              i1 = i;
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v1, o);
            const int oi = __shfl_xor_sync(0xffffffffu, i1, o);
            if (ov > v1 || (ov == v1 && oi < i1)) {
              v1 = ov;
              i1 = oi;
            }
          }
          double v2 = -1.0;  // the warp's largest candidate other than element i1
          for (int i = n_s + tid; i < n; i += SEL_T) {
            const double v = u[i];
            if (i != seed && i != i1 && v >= thr) v2 = fmax(v2, v);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v2 = fmax(v2, __shfl_xor_sync(0xffffffffu, v2, o));
          if (lane == 0) sm.red_v[wid] = v2;
          __syncthreads();
          T0 = sm.red_v[lane];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) T0 = fmin(T0, __shfl_xor_sync(0xffffffffu, T0, o));
        }
        if (tid == 0) sm.fl_cnt = 0;
        __syncthreads();
        for (int i = n_s + tid; i < n; i += SEL_T) {
          const double v = u[i];
          if (i != seed && v >= thr && v >= T0) {
            const int p = atomicAdd(&sm.fl_cnt, 1);
            if (p < SEL_FCAP) {
              sm.fl_i[p] = i;
              sm.fl_u[p] = v;
            }
          }
        }
        __syncthreads();
        const int C = sm.fl_cnt;
        if (C <= SEL_FCAP) {
          // four threads per listed candidate count the candidates ahead of it
          const int part = tid & 3;
          for (int t0 = 0; t0 < C; t0 += SEL_T / 4) {
            const int t = t0 + (tid >> 2);
            const bool valid = t < C;
            const int my_i = valid ? sm.fl_i[t] : 0;
            const double my_u = valid ? sm.fl_u[t] : 0.0;
            int r = 0;
            if (valid)
              for (int q = part; q < C; q += 4) {
                const double ou = sm.fl_u[q];
                const int oi = sm.fl_i[q];
                r += (ou > my_u) || (ou == my_u && oi < my_i);
              }
            r += __shfl_xor_sync(0xffffffffu, r, 1);
            r += __shfl_xor_sync(0xffffffffu, r, 2);
            if (valid && part == 0 && r < k_dm) c->cand[1 + r] = my_i;
          }
          fast_done = true;
        }
      }
    }
    if (fast_done) {
      nlist = -k_dm;  // (negative: cand[] is already written in order)
    } else {
    // radix select of the k_dm-th largest key among candidates.  Every
    // candidate key lies in [key(thr), key(umax)], so the digits above their
    // highest differing bit are common and need no histogram; and once the
    // bucket holding the k-th key is taken whole the select is done (the keys
    // matching the prefix under `mask` are then all selected).
    const unsigned long long khi = (unsigned long long)__double_as_longlong(umax);
    const unsigned long long klo = (unsigned long long)__double_as_longlong(thr);
    const int hb = (khi == klo) ? 0 : 63 - __clzll(khi ^ klo);
    unsigned long long prefix = 0ull, mask = 0ull;
    int k = k_dm;
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
      if (shift > hb) {  // common digit
        prefix |= khi & (255ull << shift);
        mask |= 255ull << shift;
        continue;
      }
      for (int b = tid; b < 256; b += SEL_T) sm.hist[b] = 0u;
      __syncthreads();
      // warp-aggregated histogram: norms cluster in few bins, so plain shared
      // atomics would serialize; one atomic per distinct digit per warp step.
#pragma unroll 4
      for (int it = 0; it < seg; ++it) {
        const int i = s0 + it;
        unsigned dig = 0xffffffffu;
        if (i < s1) {
          const double v = u[i];
          const unsigned long long key = (unsigned long long)__double_as_longlong(v);
          if (i != seed && v >= thr && (key & mask) == prefix) dig = (unsigned)((key >> shift) & 255ull);
        }
        const unsigned grp = __match_any_sync(0xffffffffu, dig);
        if (dig != 0xffffffffu && lane == __ffs(grp) - 1) atomicAdd(&sm.hist[dig], (unsigned)__popc(grp));
      }
      __syncthreads();
      if (wid == 0) {
        // bins 255..0 in descending order; lane handles 8 consecutive bins from the top
        unsigned cnts[8];
        unsigned lsum = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          cnts[q] = sm.hist[255 - (lane * 8 + q)];
          lsum += cnts[q];
        }
        unsigned incl = lsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        unsigned excl = incl - lsum;
        // the lane whose range contains the k-th element
        bool mine = (excl < (unsigned)k) && ((unsigned)k <= incl);
        unsigned ball = __ballot_sync(0xffffffffu, mine);
        int owner = __ffs(ball) - 1;
        if (lane == owner) {
          unsigned run = excl;
          int digit = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (run + cnts[q] >= (unsigned)k) {
              digit = 255 - (lane * 8 + q);
              break;
            }
            run += cnts[q];
          }
          sm.bc_i[1] = digit;
          sm.bc_i[2] = k - (int)run;
          sm.bc_i[3] = (k - (int)run == (int)sm.hist[digit]);  // bucket taken whole
        }
      }
      __syncthreads();
      prefix |= (unsigned long long)sm.bc_i[1] << shift;
      mask |= 255ull << shift;
      k = sm.bc_i[2];
      const bool whole = sm.bc_i[3] != 0;
      __syncthreads();
      if (whole) break;
    }
    const unsigned long long T = prefix;
    const int k_rem = k;  // keys matching T under mask to take, smallest index first
    // greater-than count and equal count per thread (index order)
    int gt = 0, eq = 0;
    for (int i = s0; i < s1; ++i) {
      double v = u[i];
      if (i == seed || !(v >= thr)) continue;
      unsigned long long key = (unsigned long long)__double_as_longlong(v) & mask;
      gt += key > T;
      eq += key == T;
    }
    int dummy;
    int off_gt = block_excl_scan(gt, sm.scan, &dummy);
    int off_eq = block_excl_scan(eq, sm.scan, &s_total);
    __syncthreads();
    const int total_gt = k_dm - k_rem;
    int pg = off_gt, pe = off_eq;
    for (int i = s0; i < s1; ++i) {
      double v = u[i];
      if (i == seed || !(v >= thr)) continue;
      unsigned long long key = (unsigned long long)__double_as_longlong(v) & mask;
      if (key > T) {
        list_i[pg] = i;
        list_u[pg] = v;
        ++pg;
      } else if (key == T) {
        if (pe < k_rem) {
          list_i[total_gt + pe] = i;
          list_u[total_gt + pe] = v;
        }
        ++pe;
      }
    }
    nlist = k_dm;
    }
  }
  __syncthreads();
  const bool presorted = nlist < 0;
  if (presorted) nlist = -nlist;
  // ---- stable descending sort of the <= k_dm candidates by rank counting ----
  if constexpr (WIDE) {
    int* const cand = wb.cand;
    for (int t = tid; t < nlist; t += SEL_T) {
      const int my_i = list_i[t];
      const double my_u = list_u[t];
      int my_rank = 0;
      for (int q = 0; q < nlist; ++q) {
        const double ou = list_u[q];
        const int oi = list_i[q];
        my_rank += (ou > my_u) || (ou == my_u && oi < my_i);
      }
      cand[1 + my_rank] = my_i;
    }
    if (tid == 0) cand[0] = seed;
  } else {
    int my_i = 0, my_rank = 0;
    double my_u = 0.0;
    if (!presorted && tid < nlist) {
      my_i = list_i[tid];
      my_u = list_u[tid];
      for (int q = 0; q < nlist; ++q) {
        double ou = list_u[q];
        int oi = list_i[q];
        my_rank += (ou > my_u) || (ou == my_u && oi < my_i);
      }
    }
    __syncthreads();
    if (!presorted && tid < nlist) c->cand[1 + my_rank] = my_i;
  }
  if (tid == 0) {
    c->kind = 0;
    c->k_max = nlist;
    c->ncand = 1 + nlist;
    c->cand[0] = seed;
    c->umax = umax;
  }
}

}  // namespace dmqr
