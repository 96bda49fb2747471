// Wide selection: k_dm > DMQR_MAXK - 1 (dm.py:56-62 accepts any k_dm >= 1).
//   candidate_set   dm.py:81-97       k_select_t<true> (select.cuh), list in the workspace
//   cosine_matrix   dm.py:100-115     k_wgram (tiled fp64 Gram of the W candidates) + k_wfin
//   dm_select       dm.py:151-177     k_wfin: greedy filter (+ delta_max guard), gamma
//   _move_selected_to_front rrqr.py:294-312  k_wfin (transpositions with the position patch,
//                   composed into moves) + k_wgather / k_wscatter (every row of the moved columns)
//   panel loop      rrqr.py:360-379   a step of k_s > DMQR_MAXK selected columns runs as
//                   consecutive panel chunks of <= DMQR_MAXK columns with no new selection
//                   (k_select_t<true> sets the next chunk up); k_wcont carries the QRDM2 break
//                   test across a chunk boundary (||a_{n_s+l}|| < eps_s after the chunk's
//                   update -- the test rrqr.py:375-379 makes before the next reflector) and
//                   k_step_end keeps one step record for the whole step.
// The chunked step applies the same reflectors in the same order as the
// reference's column-by-column loop: chunk c's block update reaches the later
// selected columns before their own panel, as the rank-1 updates do there.
// Serial schedule only (no look-ahead); one matrix per launch.
#pragma once
#include "common.cuh"
#include "norms.cuh"
#include "gram.cuh"

namespace dmqr {

constexpr int WIDE_K = DMQR_MAXK - 1;  // k_dm above this selects through this file
constexpr int WG_T = 256;              // k_wgram: one 32 x 32 upper tile of the Gram per CTA (x row splits)
constexpr int WF_T = 1024;             // k_wfin: one CTA
constexpr int WIDE_SPLIT_MAX = 16;

__global__ void __launch_bounds__(WG_T) k_wgram(Ctl* c, const double* __restrict__ A, WideBufs wb) {
  pdl_enter();
  const CtlSnap S = snap(c);
  if (S.done || S.kind != 0 || S.w_cont || S.ncand <= 1) return;
  const int ncand = S.ncand;
  const int nt = (ncand + 31) / 32;
  if ((int)blockIdx.x >= nt * (nt + 1) / 2) return;
  int ti, tj;
  tile_ij(blockIdx.x, nt, ti, tj);
  __shared__ double xi[32][33], xj[32][33];  // [column][row]
  __shared__ int ci[32], cj[32];
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int q = ti * 32 + tid;
    ci[tid] = q < ncand ? wb.cand[q] : -1;
  } else if (tid < 64) {
    const int q = tj * 32 + tid - 32;
    cj[tid - 32] = q < ncand ? wb.cand[q] : -1;
  }
  __syncthreads();
  const int64_t n_s = S.n_s, m = S.m, lda = S.lda, mp = m - n_s;
  const int64_t ns = gridDim.y;
  const int64_t chunk = ((mp + ns - 1) / ns + 31) / 32 * 32;
  const int64_t r0 = n_s + (int64_t)blockIdx.y * chunk, r1 = min(m, r0 + chunk);
  const int ty = tid >> 4, tx = tid & 15;
  double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0;
  for (int64_t rb = r0; rb < r1; rb += 32) {
#pragma unroll
    for (int e = tid; e < 1024; e += WG_T) {
      const int col = e >> 5, row = e & 31;
      const int64_t r = rb + row;
      const bool okr = r < r1;
      xi[col][row] = (okr && ci[col] >= 0) ? A[(int64_t)ci[col] * lda + r] : 0.0;
      xj[col][row] = (okr && cj[col] >= 0) ? A[(int64_t)cj[col] * lda + r] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int r = 0; r < 32; ++r) {
      const double p0 = xi[2 * ty][r], p1 = xi[2 * ty + 1][r];
      const double q0 = xj[2 * tx][r], q1 = xj[2 * tx + 1][r];
      a00 = fma(p0, q0, a00);
      a01 = fma(p0, q1, a01);
      a10 = fma(p1, q0, a10);
      a11 = fma(p1, q1, a11);
    }
    __syncthreads();
  }
  const int64_t WP = wb.WP;
  double* gp = wb.gpart + (int64_t)blockIdx.y * WP * WP;
  const int64_t i0 = ti * 32 + 2 * ty, j0 = tj * 32 + 2 * tx;
  gp[i0 * WP + j0] = a00;
  gp[i0 * WP + j0 + 1] = a01;
  gp[(i0 + 1) * WP + j0] = a10;
  gp[(i0 + 1) * WP + j0 + 1] = a11;
}

// Shared-memory layout of k_wfin: smode 2 = Theta [W][W] + vectors, 1 = vectors
// only (Theta in wb.theta), 0 = nothing (both in the workspace)
inline size_t wfin_smem(int W, int smode) {
  const size_t vec = sizeof(double) * 2 * (size_t)W + sizeof(int) * (size_t)W;
  return smode == 2 ? sizeof(double) * (size_t)W * W + vec : (smode == 1 ? vec : 0);
}

__global__ void __launch_bounds__(WF_T) k_wfin(Ctl* c, const double* __restrict__ A, int64_t* __restrict__ swaplog,
                                               WideBufs wb, int ns, int smode) {
  pdl_enter();
  const CtlSnap S = snap(c);
  if (S.done || S.kind != 0 || S.w_cont) return;
  extern __shared__ __align__(16) double wfs[];
  const int W = wb.W;
  double* th;
  int64_t ldt;
  double* inv;
  if (smode == 2) {
    th = wfs;
    ldt = W;
    inv = wfs + (size_t)W * W;
  } else {
    th = wb.theta;
    ldt = wb.WP;
    inv = smode == 1 ? wfs : wb.vec;
  }
  double* rowsum = inv + W;
  int* chosen = reinterpret_cast<int*>(rowsum + W);
  __shared__ int s_bad, s_zero, s_nch;
  __shared__ double s_g[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ncand = S.ncand;
  const int64_t n_s = S.n_s, m = S.m, lda = S.lda, mp = m - n_s;
  const int64_t WP = wb.WP;
  if (tid == 0) {
    s_bad = 0;
    s_zero = 0;
    s_nch = 1;
    chosen[0] = 0;
  }
  double gmin = 1.0;  // no candidates: J = [seed], gamma = 1 (dm.py:145-146)
  __syncthreads();
  if (ncand > 1) {
    // the Gram: partials summed in fixed order
    for (int e = tid; e < ncand * ncand; e += WF_T) {
      const int i = e / ncand, j = e % ncand;
      if (j < i) continue;
      const double* gp = wb.gpart + (int64_t)i * WP + j;
      double s = 0.0;
      for (int sp = 0; sp < ns; ++sp) s += __ldcg(gp + (int64_t)sp * WP * WP);
      th[i * ldt + j] = s;
    }
    __syncthreads();
    for (int i = tid; i < ncand; i += WF_T) {
      const double d = th[i * ldt + i];
      if (!(d > 1e-280 && d < 1e280)) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
      // extreme magnitudes only: recompute with exact 2^-e column scales
      for (int i = wid; i < ncand; i += WF_T / 32) {
        const double* ci = A + (int64_t)wb.cand[i] * lda + n_s;
        double am = 0.0;
        for (int64_t r = lane; r < mp; r += 32) am = fmax(am, fabs(ci[r]));
        am = warp_max(am);
        if (lane == 0) rowsum[i] = am;
      }
      __syncthreads();
      for (int e = tid; e < ncand * ncand; e += WF_T) {
        const int i = e / ncand, j = e % ncand;
        if (j < i) continue;
        int ei = 0, ej = 0;
        if (rowsum[i] > 0.0) frexp(rowsum[i], &ei);
        if (rowsum[j] > 0.0) frexp(rowsum[j], &ej);
        const double* ci = A + (int64_t)wb.cand[i] * lda + n_s;
        const double* cj = A + (int64_t)wb.cand[j] * lda + n_s;
        double acc = 0.0;
        for (int64_t r = 0; r < mp; ++r) acc = fma(ldexp(ci[r], -ei), ldexp(cj[r], -ej), acc);
        th[i * ldt + j] = acc;
      }
      __syncthreads();
    }
    // norms, zero-column check (dm.py:107-109)
    for (int i = tid; i < ncand; i += WF_T) {
      const double nr = sqrt(th[i * ldt + i]);
      if (nr == 0.0) s_zero = 1;
      inv[i] = 1.0 / nr;
    }
    __syncthreads();
    if (s_zero) {
      if (tid == 0) {
        c->status = -3;
        c->done = 1;
      }
      return;
    }
    // Theta upper triangle (G_ij inv_i) inv_j, i < j (dm.py:112), mirrored
    for (int e = tid; e < ncand * ncand; e += WF_T) {
      const int i = e / ncand, j = e % ncand;
      if (j <= i) continue;
      const double t = __dmul_rn(__dmul_rn(th[i * ldt + j], inv[i]), inv[j]);
      th[i * ldt + j] = t;
      th[j * ldt + i] = t;
    }
    __syncthreads();
    // ---- greedy filter, one warp (dm.py:151-173) ----
    if (wid == 0) {
      const double tau2 = S.tau * S.tau;
      const bool dmax = S.use_delta_max != 0;
      const double delta = dmax ? tau2 / (double)max(S.k_max - 1, 1) : S.delta;
      const double guard = tau2;
      int nc = 1;
      if (lane == 0) rowsum[0] = 0.0;
      __syncwarp();
      for (int t = 1; t < ncand; ++t) {
        const double* trow = th + (int64_t)t * ldt;
        bool ok = true;
        for (int q = lane; q < nc; q += 32) ok &= (fabs(trow[chosen[q]]) < delta);
        if (!__all_sync(0xffffffffu, ok)) continue;
        if (dmax) {
          double tot = 0.0;
          if (lane == 0)
            for (int q = 0; q < nc; ++q) tot += fabs(trow[chosen[q]]);
          tot = __shfl_sync(0xffffffffu, tot, 0);
          bool rej = tot >= guard;
          for (int q = lane; q < nc; q += 32) {
            const int jj = chosen[q];
            rej |= (rowsum[jj] + fabs(trow[jj]) >= guard);
          }
          if (__any_sync(0xffffffffu, rej)) continue;
          for (int q = lane; q < nc; q += 32) {
            const int jj = chosen[q];
            rowsum[jj] += fabs(trow[jj]);
          }
          __syncwarp();
          if (lane == 0) rowsum[t] = tot;
        }
        if (lane == 0) chosen[nc] = t;
        ++nc;
        __syncwarp();
      }
      if (lane == 0) s_nch = nc;
    }
    __syncthreads();
    // gamma = min_i 1 - (sum_j |theta_ij| - 1) over the chosen submatrix (dm.py:175-176)
    const int nch = s_nch;
    for (int p = wid; p < nch; p += WF_T / 32) {
      const int i = chosen[p];
      double sacc = 0.0;
      for (int q = lane; q < nch; q += 32) {
        const int jj = chosen[q];
        sacc += (i == jj) ? 1.0 : fabs(th[i * ldt + jj]);
      }
      sacc = warp_sum(sacc);
      if (lane == 0) inv[p] = 1.0 - (sacc - 1.0);
    }
    __syncthreads();
    double g = 1e300;
    for (int p = tid; p < nch; p += WF_T) g = fmin(g, inv[p]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g = fmin(g, __shfl_xor_sync(0xffffffffu, g, o));
    if (lane == 0) s_g[wid] = g;
    __syncthreads();
    if (wid == 0) {
      g = s_g[lane];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g = fmin(g, __shfl_xor_sync(0xffffffffu, g, o));
      gmin = g;
    }
  }
  if (tid != 0) return;
  // ---- the swap plan (rrqr.py:294-312), one thread ----
  // pos[h]: current position of the h-th selected column; pmap inverts it (the
  // patch "first later pos == tgt -> src" is then one lookup: positions are distinct)
  const int nch = s_nch;
  const int ks = (int)min((int64_t)nch, S.kmax - n_s);
  const int stamp = S.step_idx + 1;
  for (int i = 0; i < ks; ++i) {
    const int col = wb.cand[chosen[i]];
    wb.pos[i] = col;
    wb.pstamp[col] = stamp;
    wb.pmap[col] = i;
  }
  const int ns0 = S.n_swaps;
  int nsw = 0, ntouch = 0;
  auto touch = [&](int x) {
    if (wb.cstamp[x] != stamp) {
      wb.cstamp[x] = stamp;
      wb.cmap[x] = x;
      wb.mv_dst[ntouch++] = x;
    }
  };
  for (int i = 0; i < ks; ++i) {
    const int tgt = (int)n_s + i, src = wb.pos[i];
    if (src == tgt) continue;
    if (ns0 + nsw < S.swap_cap) {
      swaplog[2 * (int64_t)(ns0 + nsw)] = tgt;
      swaplog[2 * (int64_t)(ns0 + nsw) + 1] = src;
    }
    ++nsw;
    touch(tgt);
    touch(src);
    const int t = wb.cmap[tgt];
    wb.cmap[tgt] = wb.cmap[src];
    wb.cmap[src] = t;
    if (wb.pstamp[tgt] == stamp) {
      const int h = wb.pmap[tgt];
      if (h > i && wb.pos[h] == tgt) {
        wb.pos[h] = src;
        wb.pmap[src] = h;
        wb.pstamp[src] = stamp;
      }
    }
  }
  // composed moves new[dst] = old[src] (in place over the touched list)
  int nmv = 0;
  for (int q = 0; q < ntouch; ++q) {
    const int x = wb.mv_dst[q];
    const int s = wb.cmap[x];
    if (s != x) {
      wb.mv_dst[nmv] = x;
      wb.mv_src[nmv] = s;
      ++nmv;
    }
  }
  c->n_swaps = ns0 + nsw;
  if (ns0 + nsw > S.swap_cap) {
    c->status = -5;
    c->done = 1;
  }
  c->w_nmv = nmv;
  c->w_total = ks;
  c->w_done = 0;
  c->w_next = 0;
  c->w_ns0 = (int32_t)n_s;
  c->eps_s = S.tau * S.umax;
  c->gamma = gmin;
  // the first panel chunk
  const int kk = min(ks, DMQR_MAXK);
  c->nsel = kk;
  c->k_s = kk;
  for (int i = 0; i < kk; ++i) c->sel[i] = (int32_t)n_s + i;
  c->nsw = 0;
  c->nmv = 0;
}

// the moved columns (every row), u, uref and perm: sources out, then destinations in
__global__ void __launch_bounds__(256) k_wgather(Ctl* c, const double* __restrict__ A, const double* __restrict__ u,
                                                 const double* __restrict__ uref, const int64_t* __restrict__ perm,
                                                 WideBufs wb) {
  pdl_enter();
  const CtlSnap S = snap(c);
  if (S.done || S.kind != 0 || S.w_cont) return;
  const int nmv = ctl_ld(&c->w_nmv);
  const int64_t m = S.m, lda = S.lda, ld = wb.m_tmp;
  for (int q = blockIdx.y; q < nmv; q += gridDim.y) {
    const int64_t src = wb.mv_src[q];
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x)
      wb.tmpA[q * ld + r] = A[src * lda + r];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      wb.tmpu[q] = u[src];
      wb.tmpr[q] = uref[src];
      wb.tmpp[q] = perm[src];
    }
  }
}

__global__ void __launch_bounds__(256) k_wscatter(Ctl* c, double* __restrict__ A, double* __restrict__ u,
                                                  double* __restrict__ uref, int64_t* __restrict__ perm, WideBufs wb) {
  pdl_enter();
  const CtlSnap S = snap(c);
  if (S.done || S.kind != 0 || S.w_cont) return;
  const int nmv = ctl_ld(&c->w_nmv);
  const int64_t m = S.m, lda = S.lda, ld = wb.m_tmp;
  for (int q = blockIdx.y; q < nmv; q += gridDim.y) {
    const int64_t dst = wb.mv_dst[q];
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m; r += (int64_t)gridDim.x * blockDim.x)
      A[dst * lda + r] = wb.tmpA[q * ld + r];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      u[dst] = wb.tmpu[q];
      uref[dst] = wb.tmpr[q];
      perm[dst] = wb.tmpp[q];
    }
  }
}

// After a chunk's update: does the step continue with its next chunk?  It does
// when the chunk accepted all its columns, selected columns remain, and (QRDM2)
// the next one is not below eps_s -- column_norms(work[nxt:, nxt]) with the
// reference's max-scaled form (matrix.py:61-78).  Sets w_done / w_next (and
// broke on a boundary break) for k_step_end.
__global__ void __launch_bounds__(1024) k_wcont(Ctl* c, const double* __restrict__ A) {
  pdl_enter();
  const CtlSnap S = snap(c);
  if (S.done || S.kind != 0) return;
  __shared__ int s_test;
  __shared__ double s_eps, s_sum[32], s_max[32], s_nrm;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    const int l = S.l_acc;
    const int wd = c->w_done + l, wt = c->w_total;
    const bool more = !c->broke && l == S.k_s && wd < wt;
    c->w_done = wd;
    c->w_next = more ? wt - wd : 0;
    s_test = more && S.break_check;
    s_eps = c->eps_s;
  }
  __syncthreads();
  if (!s_test) return;
  const int64_t j = S.n_s + S.l_acc, len = S.m - j;
  const double* x = A + j * S.lda + j;
  const int64_t seg = (len + 31) / 32 / 2 * 2 + 2;  // even: 16-byte alignment is kept per warp segment
  const int64_t a = min(len, (int64_t)wid * seg), b = min(len, a + seg);
  double sv = 0.0, av = 0.0;
  if (b > a) warp_col_sums(x + a, b - a, lane, sv, av);
  if (lane == 0) {
    s_sum[wid] = sv;
    s_max[wid] = av;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0, am = 0.0;
    for (int w = 0; w < 32; ++w) {
      s += s_sum[w];
      am = fmax(am, s_max[w]);
    }
    s_nrm = norm_range_ok(am) ? sqrt(s) : -am;  // (negative: the scaled pass below)
  }
  __syncthreads();
  double nrm = s_nrm;
  if (nrm < 0.0) {
    const double am = -nrm;
    double t = 0.0;
    for (int64_t k = tid; k < len; k += 1024) {
      const double y = x[k] / am;
      t = fma(y, y, t);
    }
    t = warp_sum(t);
    if (lane == 0) s_sum[wid] = t;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < 32; ++w) s += s_sum[w];
      s_nrm = am * sqrt(s);
    }
    __syncthreads();
    nrm = s_nrm;
  }
  if (tid == 0 && nrm < s_eps) {  // rrqr.py:375-379 at the chunk boundary
    c->broke = 1;
    c->w_next = 0;
  }
}

}  // namespace dmqr
