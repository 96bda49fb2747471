// Candidate cosine matrix (DMMA Gram) + greedy delta filter + swap plan.
//   cosine_matrix          dm.py:100-115: G = C^T C, Theta = triu(G D^-1 D^-1, 1) mirrored, diag 1
//   dm_select filter       dm.py:151-177 (+ delta_max guard), gamma
//   k_s, eps_s             rrqr.py:355-357
//   _move_selected_to_front rrqr.py:294-312: exact transposition sequence with position patching
// The Gram reduction over m' rows is split across CTAs (fixed-order, deterministic
// combine); each CTA stages a 32-row slab of the <= 65 gathered candidate columns
// in shared memory and runs 8x8x4 fp64 MMAs (SASS DMMA) on the upper tiles.  The
// last CTA to finish reduces the partials, builds Theta and runs the filter with
// one warp (ballots over the chosen set), then writes the swap plan for k_swap.
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int GRAM_T = 256;
constexpr int GRAM_LD = 36;   // 32 rows + 4: conflict-free fragment loads (ld = 4 mod 16)
constexpr int GRAM_PART = DMQR_KP * DMQR_KP + DMQR_KP;

// selection finalize (thread 0): k_s, eps_s and the swap plan.  c->sel[0..nsel)
// must already hold the selected absolute column indices, seed first.
__device__ __noinline__ void finalize_selection(Ctl* c, int nsel, double gamma) {
  const int n_s = c->n_s;
  const int k_s = (int)min((int64_t)nsel, c->kmax - n_s);
  c->nsel = nsel;
  c->k_s = k_s;
  c->gamma = gamma;
  c->eps_s = c->tau * c->umax;
  int p[DMQR_KP];
  int where[DMQR_KP];
#pragma unroll 1
  for (int d = 0; d < DMQR_KP; ++d) where[d] = -1;
#pragma unroll 1
  for (int h = 0; h < k_s; ++h) {
    p[h] = c->sel[h];
    const int d = p[h] - n_s;
    if (d >= 0 && d < DMQR_KP) where[d] = h;
  }
  int ns = 0;
#pragma unroll 1
  for (int i = 0; i < k_s; ++i) {
    const int tgt = n_s + i, src = p[i];
    if (src == tgt) continue;
    c->sw_a[ns] = tgt;
    c->sw_b[ns] = src;
    ++ns;
    const int h = where[i];
    if (h > i) {  // first later position holding tgt now holds src (rrqr.py:309-312)
      p[h] = src;
      where[i] = -1;
      const int d = src - n_s;
      if (d >= 0 && d < DMQR_KP) where[d] = h;
    }
  }
  c->nsw = ns;
}

struct GramSmem {
  double cs[DMQR_KP * GRAM_LD];     // slab, column-major by candidate: cs[col*LD + row]
  double g[DMQR_KP * DMQR_KP];      // reduced Gram / Theta (last CTA)
  double amax[DMQR_KP];
  double inv[DMQR_KP];
  double rowsum[DMQR_KP];
  int chosen[DMQR_KP];
  int is_last;
  int nchosen;
};

__global__ void __launch_bounds__(GRAM_T) k_gram(Ctl* __restrict__ c, const double* __restrict__ A,
                                                 double* __restrict__ part) {
  if (c->done || c->kind != 0) return;
  extern __shared__ __align__(16) unsigned char gram_raw[];
  GramSmem& sm = *reinterpret_cast<GramSmem*>(gram_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ncand = c->ncand;
  if (ncand == 1) {  // no candidates: J = [seed], gamma = 1 (dm.py:145-146)
    if (blockIdx.x == 0 && tid == 0) {
      c->sel[0] = c->cand[0];
      finalize_selection(c, 1, 1.0);
    }
    return;
  }
  const int64_t n_s = c->n_s, m = c->m, lda = c->lda;
  const int64_t mp = m - n_s;
  const int np8 = round_up(ncand, 8);
  const int nt = np8 / 8;
  const int ntiles = nt * (nt + 1) / 2;

  // rows of this CTA
  const int64_t rpc = ceil_div(ceil_div(mp, (int64_t)gridDim.x), 32) * 32;
  const int64_t r_begin = (int64_t)blockIdx.x * rpc;
  const int64_t r_end = min(mp, r_begin + rpc);

  double acc[6][2];
  int tile_i[6], tile_j[6];
  int my_tiles = 0;
  for (int t = wid, q = 0; t < ntiles; t += GRAM_T / 32, ++q) {
    // t -> (ti, tj) upper-triangular enumeration
    int ti = 0, rem = t;
    while (rem >= nt - ti) {
      rem -= nt - ti;
      ++ti;
    }
    tile_i[q] = ti;
    tile_j[q] = ti + rem;
    acc[q][0] = acc[q][1] = 0.0;
    my_tiles = q + 1;
  }
  double lmax[DMQR_KP / 8 + 1];
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8 + 1; ++q) lmax[q] = 0.0;

  for (int64_t r0 = r_begin; r0 < r_end; r0 += 32) {
    // stage 32 rows x np8 candidate columns (zero padded)
#pragma unroll
    for (int q = 0; q < DMQR_KP / 8; ++q) {
      const int col = wid + 8 * q;
      if (col < np8) {
        double v = 0.0;
        const int64_t r = r0 + lane;
        if (col < ncand && r < r_end) v = A[(n_s + r) + (int64_t)c->cand[col] * lda];
        sm.cs[col * GRAM_LD + lane] = v;
        lmax[q] = fmax(lmax[q], fabs(v));
      }
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int kr = 4 * ks + (lane & 3);
      for (int q = 0; q < my_tiles; ++q) {
        double a = sm.cs[(tile_i[q] * 8 + (lane >> 2)) * GRAM_LD + kr];
        double b = sm.cs[(tile_j[q] * 8 + (lane >> 2)) * GRAM_LD + kr];
        dmma884(acc[q][0], acc[q][1], a, b);
      }
    }
    __syncthreads();
  }
  // write partials
  double* my = part + (int64_t)blockIdx.x * GRAM_PART;
  for (int q = 0; q < my_tiles; ++q) {
    const int row = tile_i[q] * 8 + (lane >> 2);
    const int col = tile_j[q] * 8 + 2 * (lane & 3);
    my[row * DMQR_KP + col] = acc[q][0];
    my[row * DMQR_KP + col + 1] = acc[q][1];
  }
#pragma unroll
  for (int q = 0; q < DMQR_KP / 8; ++q) {
    double v = warp_max(lmax[q]);
    const int col = wid + 8 * q;
    if (lane == 0 && col < np8) my[DMQR_KP * DMQR_KP + col] = v;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    unsigned prev = atomicAdd(&c->gram_count, 1u);
    sm.is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!sm.is_last) return;
  __threadfence();
  if (tid == 0) c->gram_count = 0u;

  // ---- last CTA: fixed-order reduction of the partials ----
  const int G = gridDim.x;
  for (int e = tid; e < np8 * np8; e += GRAM_T) {
    const int i = e / np8, j = e % np8;
    if (j < (i / 8) * 8) continue;  // only upper tiles were written
    double s = 0.0;
    for (int b = 0; b < G; ++b) s += __ldcg(part + (int64_t)b * GRAM_PART + i * DMQR_KP + j);
    sm.g[i * DMQR_KP + j] = s;
  }
  for (int i = tid; i < np8; i += GRAM_T) {
    double a = 0.0;
    for (int b = 0; b < G; ++b) a = fmax(a, __ldcg(part + (int64_t)b * GRAM_PART + DMQR_KP * DMQR_KP + i));
    sm.amax[i] = a;
  }
  __syncthreads();
  // range check: rescale by exact powers of two if squares could over/underflow
  __shared__ int s_bad;
  if (tid == 0) {
    int bad = 0;
    for (int i = 0; i < ncand; ++i) bad |= !norm_range_ok(sm.amax[i]);
    s_bad = bad;
  }
  __syncthreads();
  if (s_bad) {
    // slow path (extreme magnitudes only): one CTA recomputes the Gram with
    // per-column scales 2^-e so that max|scaled| is in [0.5, 1).
    for (int e = tid; e < ncand * ncand; e += GRAM_T) {
      const int i = e / ncand, j = e % ncand;
      if (j < i) continue;
      int ei, ej;
      frexp(sm.amax[i], &ei);
      frexp(sm.amax[j], &ej);
      const double* ci = A + (int64_t)c->cand[i] * lda + n_s;
      const double* cj = A + (int64_t)c->cand[j] * lda + n_s;
      double s = 0.0;
      for (int64_t r = 0; r < mp; ++r) s = fma(ldexp(ci[r], -ei), ldexp(cj[r], -ej), s);
      sm.g[i * DMQR_KP + j] = s;
    }
    __syncthreads();
  }
  // norms, zero-column check (dm.py:107-109)
  __shared__ int s_zero;
  if (tid == 0) s_zero = 0;
  __syncthreads();
  for (int i = tid; i < ncand; i += GRAM_T) {
    double nr = sqrt(sm.g[i * DMQR_KP + i]);
    if (nr == 0.0) s_zero = 1;
    sm.inv[i] = 1.0 / nr;
  }
  __syncthreads();
  if (s_zero) {
    if (tid == 0) {
      c->status = -3;
      c->done = 1;
    }
    return;
  }
  // Theta upper triangle: (G_ij * inv_i) * inv_j, i < j (dm.py:112)
  for (int e = tid; e < ncand * ncand; e += GRAM_T) {
    const int i = e / ncand, j = e % ncand;
    if (j <= i) continue;
    sm.g[i * DMQR_KP + j] = __dmul_rn(__dmul_rn(sm.g[i * DMQR_KP + j], sm.inv[i]), sm.inv[j]);
  }
  __syncthreads();

  // ---- greedy filter, one warp (dm.py:151-173) ----
  if (wid == 0) {
    const bool dmax = c->use_delta_max != 0;
    const double tau2 = c->tau * c->tau;
    const double delta = dmax ? tau2 / (double)max(c->k_max - 1, 1) : c->delta;
    const double guard = tau2;
    int nch = 1;
    if (lane == 0) {
      sm.chosen[0] = 0;
      sm.rowsum[0] = 0.0;
    }
    __syncwarp();
    for (int t = 1; t < ncand; ++t) {
      bool ok = true;
      double gsum = 0.0;
      for (int q = lane; q < nch; q += 32) {
        const int j = sm.chosen[q];
        const double th = fabs(j < t ? sm.g[j * DMQR_KP + t] : sm.g[t * DMQR_KP + j]);
        ok &= (th < delta);
        gsum += th;
      }
      bool all_ok = __all_sync(0xffffffffu, ok);
      if (!all_ok) continue;
      if (dmax) {
        // total of gains in chosen order (the reference sums the gains vector)
        double tot = 0.0;
        if (lane == 0)
          for (int q = 0; q < nch; ++q) {
            const int j = sm.chosen[q];
            tot += fabs(j < t ? sm.g[j * DMQR_KP + t] : sm.g[t * DMQR_KP + j]);
          }
        tot = __shfl_sync(0xffffffffu, tot, 0);
        bool rej = tot >= guard;
        for (int q = lane; q < nch; q += 32) {
          const int j = sm.chosen[q];
          const double th = fabs(j < t ? sm.g[j * DMQR_KP + t] : sm.g[t * DMQR_KP + j]);
          rej |= (sm.rowsum[j] + th >= guard);
        }
        if (__any_sync(0xffffffffu, rej)) continue;
        for (int q = lane; q < nch; q += 32) {
          const int j = sm.chosen[q];
          sm.rowsum[j] += fabs(j < t ? sm.g[j * DMQR_KP + t] : sm.g[t * DMQR_KP + j]);
        }
        __syncwarp();
        if (lane == 0) sm.rowsum[t] = tot;
      }
      (void)gsum;
      if (lane == 0) sm.chosen[nch] = t;
      ++nch;
      __syncwarp();
    }
    // gamma = min_i 1 - (sum_j |theta_ij| - 1) over the chosen submatrix (dm.py:175-176)
    double gmin = 1e300;
    for (int p = lane; p < nch; p += 32) {
      const int i = sm.chosen[p];
      double s = 0.0;
      for (int q = 0; q < nch; ++q) {
        const int j = sm.chosen[q];
        s += (i == j) ? 1.0 : fabs(j < i ? sm.g[j * DMQR_KP + i] : sm.g[i * DMQR_KP + j]);
      }
      gmin = fmin(gmin, 1.0 - (s - 1.0));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) gmin = fmin(gmin, __shfl_xor_sync(0xffffffffu, gmin, o));
    for (int q = lane; q < nch; q += 32) c->sel[q] = c->cand[sm.chosen[q]];
    __syncwarp();
    __threadfence_block();
    if (lane == 0) finalize_selection(c, nch, gmin);
  }
}

}  // namespace dmqr
