// Register-resident Householder panel (geqr2 + larft analogue), the fast path.
//   make_reflector        householder.py:57-79 (beta = -sign(x0)||x||, always reflects)
//   apply_reflector_left  householder.py:82-89 (rank-1 on the selected block only)
//   QRDM2 break           rrqr.py:375-379
//   accumulate_wy         householder.py:92-114 (T = W)
//
// Same grid structure and all-reduce as k_panel (panel.cuh), but the slice of
// at most 256 rows x 80 columns a CTA owns lives in REGISTERS for the whole
// panel: warp w holds columns w, w+16, ..., lane l holds rows l, l+32, ...
// (8 x 5 doubles per thread).  Per reflector the only shared-memory traffic is
// the broadcast of v (zero outside rows >= j), so the dots, z = Y^T v, the
// norm partials and the rank-1 update are pure register FMAs; the column index
// of a register slot is compile-time after unrolling (no local memory).
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "panel.cuh"

namespace dmqr {

namespace cg = cooperative_groups;

// Cross-CTA all-reduce of the per-CTA partial vector (fixed association order,
// so every CTA holds bitwise identical totals).
struct GridRed {  // cooperative grid: partials through L2 + counter barrier
  __device__ static constexpr bool cluster() { return false; }
};
struct ClusterRed {  // one thread-block cluster: partials in DSMEM + cluster barrier
  __device__ static constexpr bool cluster() { return true; }
};

// cluster all-reduce: s_buf[it & 1] holds this CTA's partials; after the
// cluster barrier each slot is summed over the ranks in a fixed tree order.
__device__ __forceinline__ void cluster_allreduce(double (*s_buf)[RED_LD], double* s_tot, int len, int it) {
  cg::cluster_group cl = cg::this_cluster();
  const int nr = (int)cl.num_blocks();
  double* mine = s_buf[it & 1];
  cl.sync();  // release/acquire: every rank's partials are visible
  const int slot = threadIdx.x >> 3, g = threadIdx.x & 7;
  for (int q0 = 0; q0 < len; q0 += PANEL_T / 8) {
    const int q = q0 + slot;
    double s = 0.0;
    if (q < len)
      for (int b = g; b < nr; b += 8) s += *cl.map_shared_rank(mine + q, b);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (q < len && g == 0) s_tot[q] = s;
  }
  __syncthreads();
}

constexpr int RR_ROWS = 8;                 // rows per lane
constexpr int RR_COLS = 5;                 // column slots per warp: 16 warps x 5 = 80 >= 65
constexpr int RR_RMAX = 32 * RR_ROWS;      // rows per CTA

template <class Red>
__global__ void __launch_bounds__(PANEL_T, 1) k_panel_rr(PanelArgs a) {
  Ctl* c = a.c;
  if (c->done) return;
  __shared__ double vbuf[RR_RMAX];
  __shared__ double s_buf[2][RED_LD];  // partial vectors (double-buffered for the cluster reducer)
  __shared__ double s_tot[RED_LD];
  __shared__ double s_T[DMQR_KP * DMQR_KP];
  double* s_part = s_buf[0];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n_s = c->n_s, m = c->m, lda = c->lda;
  const int64_t mp = m - n_s;
  const int k = c->k_s;
  const int brk = c->break_check && c->kind == 0;
  const double eps_s = c->eps_s;
  const int P = a.prows;
  const bool tcta = (int)blockIdx.x >= P;  // T builder, owns no rows
  // T is built by the extra CTA of a grid launch, or by rank 0 of a cluster / single CTA
  const bool tlocal = (gridDim.x == 1) || (Red::cluster() && blockIdx.x == 0);
  const int r0 = tcta ? (int)mp : (int)((int64_t)blockIdx.x * mp / P);
  const int r1 = tcta ? (int)mp : (int)((int64_t)(blockIdx.x + 1) * mp / P);
  const int R = r1 - r0;
  const double* gA = a.A + n_s * lda + n_s + r0;  // (local row rr, panel column q) at gA[q*lda + rr]

  double x[RR_COLS][RR_ROWS];
#pragma unroll
  for (int cc = 0; cc < RR_COLS; ++cc) {
    const int q = wid + 16 * cc;
#pragma unroll
    for (int i = 0; i < RR_ROWS; ++i) {
      const int rr = lane + 32 * i;
      x[cc][i] = (q < k && rr < R) ? gA[(int64_t)q * lda + rr] : 0.0;
    }
  }

  int red_it = 0;
  double nrm = 0.0, x0 = 0.0;
  // partials are written into s_part, which always points at the buffer of the
  // upcoming all-reduce
  auto allreduce = [&](int len) {
    if constexpr (Red::cluster()) {
      cluster_allreduce(s_buf, s_tot, len, red_it);
    } else {
      grid_allreduce(a, s_part, s_tot, len, red_it);
    }
    ++red_it;
    s_part = Red::cluster() ? s_buf[red_it & 1] : s_buf[0];
  };
  // exact ||column jj||, rows >= jj (+ x0), one all-reduce; only the owner warp has data
  auto exact_norm = [&](int jj) {
    const int wo = jj & 15, co = jj >> 4;
    if (tid < 3) s_part[tid] = 0.0;
    __syncthreads();
    if (wid == wo) {
      double ss = 0.0, am = 0.0, xx = 0.0;
#pragma unroll
      for (int cc = 0; cc < RR_COLS; ++cc)
        if (cc == co) {
#pragma unroll
          for (int i = 0; i < RR_ROWS; ++i) {
            const int rr = lane + 32 * i;
            const bool live = rr < R && r0 + rr >= jj;
            const double v = live ? x[cc][i] : 0.0;
            ss = fma(v, v, ss);
            am = fmax(am, fabs(v));
            if (live && r0 + rr == jj) xx = v;
          }
        }
      ss = warp_sum(ss);
      am = warp_max(am);
      xx = warp_sum(xx);
      if (lane == 0) {
        s_part[0] = ss;
        s_part[1] = am;
        s_part[2] = xx;
      }
    }
    allreduce(3);
    const double nrm2 = s_tot[0], abound = s_tot[1];
    x0 = s_tot[2];
    if (abound == 0.0) {
      nrm = 0.0;
    } else if (nrm2 > 1e-280 && nrm2 < 1e280) {
      nrm = sqrt(nrm2);
    } else {
      int e;
      frexp(abound, &e);
      if (tid == 0) s_part[0] = 0.0;
      __syncthreads();
      if (wid == wo) {
        double sc = 0.0;
#pragma unroll
        for (int cc = 0; cc < RR_COLS; ++cc)
          if (cc == co) {
#pragma unroll
            for (int i = 0; i < RR_ROWS; ++i) {
              const int rr = lane + 32 * i;
              const double y = (rr < R && r0 + rr >= jj) ? ldexp(x[cc][i], -e) : 0.0;
              sc = fma(y, y, sc);
            }
          }
        sc = warp_sum(sc);
        if (lane == 0) s_part[0] = sc;
      }
      allreduce(1);
      nrm = ldexp(sqrt(s_tot[0]), e);
    }
  };

  int l_acc = k, broke = 0;
  exact_norm(0);
  const bool rec = a.dbg && blockIdx.x == (gridDim.x > 1 ? 1 : 0) && tid == 0;
#define STAMP(ph) \
  if (rec && j < 64) a.dbg[j * 8 + (ph)] = clock64()
  for (int j = 0; j < k; ++j) {
    STAMP(0);
    if (brk && j > 0 && nrm < eps_s) {  // QRDM2 break (rrqr.py:375-379)
      l_acc = j;
      broke = 1;
      break;
    }
    double beta, coeff, u0;
    if (nrm == 0.0) {
      beta = 0.0;
      coeff = 0.0;
      u0 = 1.0;
    } else {
      beta = (x0 != 0.0) ? -copysign(nrm, x0) : -nrm;
      u0 = x0 - beta;
      coeff = (beta - x0) / beta;
    }
    const int wj = j & 15, cj = j >> 4;
    const double rcp = 1.0 / u0;
    // ---- v = x / u0 below the diagonal, 1 on it, 0 above / outside (owner warp) ----
    if (wid == wj) {
#pragma unroll
      for (int cc = 0; cc < RR_COLS; ++cc)
        if (cc == cj) {
#pragma unroll
          for (int i = 0; i < RR_ROWS; ++i) {
            const int rr = lane + 32 * i;
            const int p = r0 + rr;
            double v = 0.0;
            if (rr < R && p > j) {
              v = (nrm != 0.0) ? x[cc][i] * rcp : x[cc][i];
              x[cc][i] = v;
            } else if (rr < R && p == j) {
              v = 1.0;
            }
            vbuf[rr] = v;
          }
        }
    }
    if (tid < k + 5) s_part[tid] = 0.0;
    __syncthreads();
    // ---- partials: d_q = v^T C_q (q > j), z_q = Y_q^T v (q < j) ----
    double vr[RR_ROWS];
#pragma unroll
    for (int i = 0; i < RR_ROWS; ++i) vr[i] = vbuf[lane + 32 * i];
    double sd[RR_COLS];
#pragma unroll
    for (int cc = 0; cc < RR_COLS; ++cc) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i = 0; i < RR_ROWS; i += 2) {
        s0 = fma(vr[i], x[cc][i], s0);
        s1 = fma(vr[i + 1], x[cc][i + 1], s1);
      }
      sd[cc] = s0 + s1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int cc = 0; cc < RR_COLS; ++cc) sd[cc] += __shfl_xor_sync(0xffffffffu, sd[cc], o);
    if (lane == 0) {
#pragma unroll
      for (int cc = 0; cc < RR_COLS; ++cc) {
        const int q = wid + 16 * cc;
        if (q < k && q != j) s_part[q] = sd[cc];
      }
    }
    // ---- next column's a = ||x||^2, b = v.x, c = ||v||^2 over rows > j (+ x, v at row j+1) ----
    const bool has_next = (j + 1 < k);
    const int w1 = (j + 1) & 15, c1 = (j + 1) >> 4;
    if (has_next && wid == w1) {
      double pa = 0.0, pb = 0.0, pc = 0.0, px = 0.0, pv = 0.0;
#pragma unroll
      for (int cc = 0; cc < RR_COLS; ++cc)
        if (cc == c1) {
#pragma unroll
          for (int i = 0; i < RR_ROWS; ++i) {
            const int rr = lane + 32 * i;
            const int p = r0 + rr;
            const bool live = rr < R && p > j;
            const double xv = live ? x[cc][i] : 0.0;
            const double v = live ? vr[i] : 0.0;
            pa = fma(xv, xv, pa);
            pb = fma(v, xv, pb);
            pc = fma(v, v, pc);
            if (live && p == j + 1) {
              px = xv;
              pv = v;
            }
          }
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        pa += __shfl_xor_sync(0xffffffffu, pa, o);
        pb += __shfl_xor_sync(0xffffffffu, pb, o);
        pc += __shfl_xor_sync(0xffffffffu, pc, o);
        px += __shfl_xor_sync(0xffffffffu, px, o);
        pv += __shfl_xor_sync(0xffffffffu, pv, o);
      }
      if (lane == 0) {
        s_part[k] = pa;
        s_part[k + 1] = pb;
        s_part[k + 2] = pc;
        s_part[k + 3] = px;
        s_part[k + 4] = pv;
      }
    }
    STAMP(1);
    allreduce(k + (has_next ? 5 : 0));
    STAMP(2);
    // ---- rank-1 update of the selected block right of j (householder.py:88-89) ----
    if (coeff != 0.0) {
#pragma unroll
      for (int cc = 0; cc < RR_COLS; ++cc) {
        const int q = wid + 16 * cc;
        if (q > j && q < k) {
          const double w = coeff * s_tot[q];
#pragma unroll
          for (int i = 0; i < RR_ROWS; ++i) x[cc][i] = fma(-vr[i], w, x[cc][i]);
        }
      }
    }
    // diagonal entry beta (owner lane of row j)
    if (wid == wj) {
#pragma unroll
      for (int cc = 0; cc < RR_COLS; ++cc)
        if (cc == cj) {
#pragma unroll
          for (int i = 0; i < RR_ROWS; ++i)
            if (lane + 32 * i < R && r0 + lane + 32 * i == j) x[cc][i] = beta;
        }
    }
    STAMP(3);
    // ---- T column j (householder.py:109-113) on the T-builder CTA, shared memory ----
    if (tcta || tlocal) {
      for (int i = wid; i < j; i += PANEL_W) {
        double sacc = 0.0;
        for (int q = i + lane; q < j; q += 32) sacc = fma(s_T[i * DMQR_KP + q], s_tot[q], sacc);
        sacc = warp_sum(sacc);
        if (lane == 0) s_T[i * DMQR_KP + j] = -coeff * sacc;
      }
      if (tid == 0) {
        s_T[j * DMQR_KP + j] = coeff;
        a.coeffs[n_s + j] = coeff;
      }
    }
    STAMP(4);
    // ---- next column's norm: identity without cancellation, else exact ----
    if (has_next) {
      const double w = coeff * s_tot[j + 1];
      const double pa = s_tot[k], pb = s_tot[k + 1], pc = s_tot[k + 2];
      const double nx = fma(-s_tot[k + 4], w, s_tot[k + 3]);
      const double nn2 = (coeff != 0.0) ? pa - 2.0 * w * pb + w * w * pc : pa;
      if (nn2 >= 0.5 * pa && pa > 1e-280 && pa < 1e280) {
        nrm = sqrt(nn2);
        x0 = nx;
      } else {
        exact_norm(j + 1);
      }
    }
    __syncthreads();
    STAMP(5);
  }
#undef STAMP
  // ---- write the slice back ----
  double* gW = a.A + n_s * lda + n_s + r0;
#pragma unroll
  for (int cc = 0; cc < RR_COLS; ++cc) {
    const int q = wid + 16 * cc;
#pragma unroll
    for (int i = 0; i < RR_ROWS; ++i) {
      const int rr = lane + 32 * i;
      if (q < k && rr < R) gW[(int64_t)q * lda + rr] = x[cc][i];
    }
  }
  if (tcta || tlocal) {
    __syncthreads();
    for (int e = tid; e < l_acc * l_acc; e += PANEL_T) {
      const int i = e / l_acc, jj = e % l_acc;
      if (i <= jj) a.T[i * DMQR_KP + jj] = s_T[i * DMQR_KP + jj];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    c->l_acc = l_acc;
    c->broke = broke;
  }
}

}  // namespace dmqr
