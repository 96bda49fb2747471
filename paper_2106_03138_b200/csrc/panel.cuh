// Column swaps and the Householder panel (geqr2 + larft analogue).
//   swap_columns / PartialNorms.swap / Permutation.swap  matrix.py:81-87,125-132; rrqr.py:131-133
//   make_reflector        householder.py:57-79 (beta = -sign(x0)||x||, always reflects)
//   apply_reflector_left  householder.py:82-89 (in-panel rank-1 on the selected block only)
//   QRDM2 break           rrqr.py:375-379 (||next column|| < eps_s stops the panel)
//   accumulate_wy         householder.py:92-114 (T = W, upper triangular)
//
// The panel is factored by a cooperatively launched grid: CTA b owns a
// contiguous slice of panel rows and keeps it resident in shared memory for
// the whole panel.  Each reflector needs two grid-wide all-reductions (the
// column norm; the v^T C dots + the z = Y^T v for T), done as
// write-partials / barrier / fixed-order sum, so every CTA holds bitwise
// identical scalars (beta, coeff, w) without a broadcast.
#pragma once
#include "common.cuh"

namespace dmqr {

// Apply the step's transposition sequence to full-height columns (row-parallel:
// each thread replays all swaps on its row, so the sequence order is exact),
// and to u, u_ref, perm, plus the swap log.
__global__ void k_swap(Ctl* __restrict__ c, double* __restrict__ A, double* __restrict__ u,
                       double* __restrict__ uref, int64_t* __restrict__ perm, int64_t* __restrict__ swaplog) {
  if (c->done) return;
  const int nsw = c->nsw;
  if (nsw == 0) return;
  const int64_t m = c->m, lda = c->lda;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < m) {
    for (int s = 0; s < nsw; ++s) {
      double* pa = A + (int64_t)c->sw_a[s] * lda + r;
      double* pb = A + (int64_t)c->sw_b[s] * lda + r;
      double t = *pa;
      *pa = *pb;
      *pb = t;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    int ns = c->n_swaps;
    for (int s = 0; s < nsw; ++s) {
      const int a = c->sw_a[s], b = c->sw_b[s];
      double t = u[a];
      u[a] = u[b];
      u[b] = t;
      t = uref[a];
      uref[a] = uref[b];
      uref[b] = t;
      int64_t p = perm[a];
      perm[a] = perm[b];
      perm[b] = p;
      if (ns < c->swap_cap) {
        swaplog[2 * ns] = a;
        swaplog[2 * ns + 1] = b;
      }
      ++ns;
    }
    c->n_swaps = ns;
    if (ns > c->swap_cap) {
      c->status = -5;
      c->done = 1;
    }
  }
}

constexpr int PANEL_T = 512;
constexpr int PANEL_W = PANEL_T / 32;
constexpr int RED_LD = DMQR_KP + 8;  // partial-vector stride

struct PanelArgs {
  Ctl* c;
  double* A;
  double* coeffs;
  double* T;     // KP x KP row-major, T[i*KP + j], upper triangular (= reference W)
  double* red;   // [2][gridDim][RED_LD] partials
  int use_smem;  // panel slice resident in shared memory
};

// deterministic all-reduce of `len` doubles across the grid; in: s_part (this
// CTA's partials, smem), out: s_tot (smem).  `it` selects the double buffer.
__device__ __forceinline__ void grid_allreduce(const PanelArgs& a, const double* s_part, double* s_tot, int len,
                                               int it) {
  const int P = gridDim.x;
  if (P == 1) {
    __syncthreads();
    for (int q = threadIdx.x; q < len; q += PANEL_T) s_tot[q] = s_part[q];
    __syncthreads();
    return;
  }
  double* buf = a.red + (int64_t)(it & 1) * P * RED_LD;
  __syncthreads();
  for (int q = threadIdx.x; q < len; q += PANEL_T) buf[(int64_t)blockIdx.x * RED_LD + q] = s_part[q];
  grid_barrier(&a.c->bar_count, &a.c->bar_gen, P);
  // 8 threads per slot, fixed association order -> identical result in every CTA
  const int slot = threadIdx.x >> 3, g = threadIdx.x & 7;
  for (int q0 = 0; q0 < len; q0 += PANEL_T / 8) {
    const int q = q0 + slot;
    double s = 0.0;
    if (q < len)
      for (int b = g; b < P; b += 8) s += __ldcg(buf + (int64_t)b * RED_LD + q);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (q < len && g == 0) s_tot[q] = s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(PANEL_T, 1) k_panel(PanelArgs a) {
  Ctl* c = a.c;
  if (c->done) return;
  extern __shared__ __align__(16) double psm[];
  __shared__ double s_part[RED_LD];
  __shared__ double s_tot[RED_LD];
  __shared__ double s_wsum[PANEL_W][3];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n_s = c->n_s, m = c->m, lda = c->lda;
  const int64_t mp = m - n_s;
  const int k = c->k_s;
  const int brk = c->break_check && c->kind == 0;
  const double eps_s = c->eps_s;
  const int P = gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * mp / P;
  const int64_t r1 = (int64_t)(blockIdx.x + 1) * mp / P;
  const int64_t R = r1 - r0;

  // element (t, r) of the panel, r panel-relative in [r0, r1): base[t*ld + (r - r0)]
  double* base;
  int64_t ld;
  double* gpanel = a.A + n_s * lda + n_s + r0;
  if (a.use_smem) {
    ld = R | 1;  // odd stride spreads columns across banks
    base = psm;
    for (int64_t e = tid; e < (int64_t)k * R; e += PANEL_T) {
      const int64_t t = e / R, rr = e % R;
      base[t * ld + rr] = gpanel[t * lda + rr];
    }
    __syncthreads();
  } else {
    base = gpanel;
    ld = lda;
  }
#define PEL(t, r) base[(int64_t)(t) * ld + ((r) - r0)]

  int l_acc = k;
  int broke = 0;
  int red_it = 0;
  for (int j = 0; j < k; ++j) {
    // ---- reduction 1: ||x||^2, max|x|, x0 over rows >= j of column j ----
    const int64_t rs = max(r0, (int64_t)j);
    double ss = 0.0, am = 0.0, x0 = 0.0;
    for (int64_t r = rs + tid; r < r1; r += PANEL_T) {
      double x = PEL(j, r);
      ss = fma(x, x, ss);
      am = fmax(am, fabs(x));
      if (r == j) x0 = x;
    }
    ss = warp_sum(ss);
    am = warp_max(am);
    x0 = warp_sum(x0);
    if (lane == 0) {
      s_wsum[wid][0] = ss;
      s_wsum[wid][1] = am;
      s_wsum[wid][2] = x0;
    }
    __syncthreads();
    if (tid == 0) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
      for (int w = 0; w < PANEL_W; ++w) {
        a0 += s_wsum[w][0];
        a1 = fmax(a1, s_wsum[w][1]);
        a2 += s_wsum[w][2];
      }
      s_part[0] = a0;
      s_part[1] = a1;
      s_part[2] = a2;
    }
    __syncthreads();
    grid_allreduce(a, s_part, s_tot, 3, red_it++);
    // s_tot[1] is the sum of per-CTA maxima: zero iff the column is zero, and an
    // upper bound (<= P x) of max|x| used only to pick an exact 2^-e rescale.
    const double nrm2 = s_tot[0];
    const double xx0 = s_tot[2];
    const double amax_bound = s_tot[1];
    double nrm;
    if (amax_bound == 0.0) {
      nrm = 0.0;
    } else if (nrm2 > 1e-280 && nrm2 < 1e280) {
      nrm = sqrt(nrm2);
    } else {
      // rare: recompute with exact power-of-two scaling by the max bound
      int e;
      frexp(amax_bound, &e);
      double sc = 0.0;
      for (int64_t r = rs + tid; r < r1; r += PANEL_T) {
        double y = ldexp(PEL(j, r), -e);
        sc = fma(y, y, sc);
      }
      sc = warp_sum(sc);
      if (lane == 0) s_wsum[wid][0] = sc;
      __syncthreads();
      if (tid == 0) {
        double t0 = 0.0;
        for (int w = 0; w < PANEL_W; ++w) t0 += s_wsum[w][0];
        s_part[0] = t0;
      }
      __syncthreads();
      grid_allreduce(a, s_part, s_tot, 1, red_it++);
      nrm = ldexp(sqrt(s_tot[0]), e);
    }
    // ---- QRDM2 break: residual of the next selected column (rrqr.py:375-379) ----
    if (brk && j > 0 && nrm < eps_s) {
      l_acc = j;
      broke = 1;
      break;
    }
    // ---- reflector (householder.py:57-79) ----
    double beta, coeff, u0;
    if (nrm == 0.0) {
      beta = 0.0;
      coeff = 0.0;
      u0 = 1.0;
    } else {
      beta = (xx0 != 0.0) ? -copysign(nrm, xx0) : -nrm;
      u0 = xx0 - beta;
      coeff = (beta - xx0) / beta;
    }
    // v below the diagonal, beta on it
    if (nrm != 0.0)
      for (int64_t r = max(rs, (int64_t)j + 1) + tid; r < r1; r += PANEL_T) PEL(j, r) = PEL(j, r) / u0;
    __syncthreads();
    // ---- reduction 2: d_t = v^T C_t (t > j) and z_i = Y[:, i]^T v (i < j) ----
    for (int q = wid; q < k; q += PANEL_W) {
      double s = 0.0;
      if (q != j) {
        for (int64_t r = rs + lane; r < r1; r += 32) {
          const double v = (r == j) ? 1.0 : PEL(j, r);
          s = fma(v, PEL(q, r), s);
        }
      }
      s = warp_sum(s);
      if (lane == 0) s_part[q] = s;
    }
    __syncthreads();
    grid_allreduce(a, s_part, s_tot, k, red_it++);
    // diagonal entry (owner)
    if (j >= r0 && j < r1 && tid == 0) PEL(j, j) = beta;
    // ---- rank-1 update of the rest of the selected block (householder.py:88-89) ----
    if (coeff != 0.0) {
      const int nc = k - j - 1;
      const int64_t nr = r1 - rs;
      for (int64_t e = tid; e < (int64_t)nc * nr; e += PANEL_T) {
        const int t = j + 1 + (int)(e / nr);
        const int64_t r = rs + e % nr;
        const double v = (r == j) ? 1.0 : PEL(j, r);
        const double w = coeff * s_tot[t];
        PEL(t, r) = PEL(t, r) - v * w;
      }
    }
    // ---- T column j (householder.py:109-113): T[:j, j] = -coeff T[:j,:j] z ; T[j,j] = coeff ----
    if (blockIdx.x == 0) {
      for (int i = tid; i < j; i += PANEL_T) {
        double s = 0.0;
        for (int q = i; q < j; ++q) s += a.T[i * DMQR_KP + q] * s_tot[q];
        a.T[i * DMQR_KP + j] = -coeff * s;
      }
      if (tid == 0) {
        a.T[j * DMQR_KP + j] = coeff;
        a.coeffs[n_s + j] = coeff;
      }
    }
    __syncthreads();
  }
#undef PEL
  if (a.use_smem) {
    __syncthreads();
    for (int64_t e = tid; e < (int64_t)k * R; e += PANEL_T) {
      const int64_t t = e / R, rr = e % R;
      gpanel[t * lda + rr] = base[t * ld + rr];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    c->l_acc = l_acc;
    c->broke = broke;
  }
}

}  // namespace dmqr
