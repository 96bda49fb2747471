// Register-resident Householder panel (geqr2 + larft analogue), the fast path.
//   make_reflector        householder.py:57-79 (beta = -sign(x0)||x||, always reflects)
//   apply_reflector_left  householder.py:82-89 (rank-1 on the selected block only)
//   QRDM2 break           rrqr.py:375-379
//   accumulate_wy         householder.py:92-114 (T = W)
//
// A CTA owns at most 256 panel rows and keeps them in REGISTERS for the whole
// panel: warp w holds columns w, w+16, w+32, w+48 (register slots 0..3) and
// lane l holds rows l, l+32, ..., l+224.  The 65th column (q = 64, slot 4 of
// warp 0) lives in shared memory so that data (64 regs) + v (16 regs) stay
// under the 128-register budget of 512 threads.  Per reflector the only
// shared-memory traffic is the broadcast of v (zero outside rows >= j), read
// once into registers; the dots, z = Y^T v, the norm partials and the rank-1
// update are register FMAs.
//
// The loop is a small state machine with exactly one cross-CTA all-reduce per
// trip (a "norm round" for an exact column norm, or a "reflector round"), so
// every phase exists once in the binary: the kernel must stay inside the SM
// instruction cache, since each phase runs only a few hundred cycles.
//
// Cross-CTA reduction: inside one thread-block cluster (<= 16 CTAs) every CTA
// pushes its partial vector into every rank's shared memory and sums its local
// copy after the cluster barrier; otherwise the cooperative-grid all-reduce of
// panel.cuh.  Both use a fixed association order, so every CTA holds
// bitwise-identical beta, coeff and w.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "panel.cuh"

namespace dmqr {

namespace cg = cooperative_groups;

struct GridRed {
  __device__ static constexpr bool cluster() { return false; }
};
struct ClusterRed {
  __device__ static constexpr bool cluster() { return true; }
};

constexpr int RR_ROWS = 8;             // rows per lane
constexpr int RR_RSLOTS = 4;           // register column slots per warp (16 x 4 = 64 columns)
constexpr int RR_RMAX = 32 * RR_ROWS;  // rows per CTA
constexpr int RR_MAXCL = 16;           // cluster ranks
constexpr size_t RR_CL_SMEM = sizeof(double) * 2 * RR_MAXCL * RED_LD;  // receive buffers

template <class Red>
__global__ void __launch_bounds__(PANEL_T, 1) k_panel_rr(PanelArgs a) {
  zshift(a.c, a.c, a.A, a.coeffs, a.T, a.red, a.q1g, a.hpart, a.hR, a.hctr);
  pdl_enter();
  Ctl* c = a.c;
  {
    const int done = c->done, cqf = c->cq_fail;  // (both loads in flight together)
    if (done || (a.only_if_fail && !cqf)) return;
  }
  TLSpan tl_span(c->done ? nullptr : c->tl, c->step_idx, 13);
  __shared__ double vbuf[RR_RMAX];
  __shared__ double xs4[RR_RMAX];  // column 64 (warp 0, slot 4)
  __shared__ double s_part[RED_LD];
  __shared__ double s_tot[RED_LD];
  __shared__ double s_T[DMQR_KP * DMQR_KP];
  extern __shared__ __align__(16) double rbuf[];  // cluster: [2][RR_MAXCL][RED_LD]

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t n_s = c->n_s, m = c->m, lda = c->lda;
  const int64_t mp = m - n_s;
  const int k = c->k_s;
  const int brk = c->break_check && c->kind == 0;
  const double eps_s = c->eps_s;
  const int P = a.prows;
  int my_rank = 0, nranks = 1;
  if constexpr (Red::cluster()) {
    my_rank = (int)cg::this_cluster().block_rank();
    nranks = (int)cg::this_cluster().num_blocks();
  }
  const bool tcta = (int)blockIdx.x >= P;  // grid T-builder, owns no rows
  // T rows: all on the grid T-builder or a single CTA; row i on rank i % nranks in a cluster
  const bool tbuild = tcta || gridDim.x == 1 || Red::cluster();
  const int tstride = Red::cluster() ? nranks : 1;
  const int r0 = tcta ? (int)mp : (int)((int64_t)blockIdx.x * mp / P);
  const int r1 = tcta ? (int)mp : (int)((int64_t)(blockIdx.x + 1) * mp / P);
  const int R = r1 - r0;
  double* gA = a.A + n_s * lda + n_s + r0;  // (local row rr, panel column q) at gA[q*lda + rr]

  double x[RR_RSLOTS][RR_ROWS];
#pragma unroll
  for (int cc = 0; cc < RR_RSLOTS; ++cc) {
    const int q = wid + 16 * cc;
#pragma unroll
    for (int i = 0; i < RR_ROWS; ++i) {
      const int rr = lane + 32 * i;
      x[cc][i] = (q < k && rr < R) ? gA[(int64_t)q * lda + rr] : 0.0;
    }
  }
  if (wid == 0 && k > 64)
    for (int i = 0; i < RR_ROWS; ++i) {
      const int rr = lane + 32 * i;
      xs4[rr] = rr < R ? gA[(int64_t)64 * lda + rr] : 0.0;
    }
  // column slot cs of the calling warp (0..3 registers, 4 shared) <-> col[]
  auto get_col = [&](int cs, double* col) {
#pragma unroll
    for (int i = 0; i < RR_ROWS; ++i) {
      double v = x[0][i];
      v = (cs == 1) ? x[1][i] : v;
      v = (cs == 2) ? x[2][i] : v;
      v = (cs == 3) ? x[3][i] : v;
      col[i] = (cs == 4) ? xs4[lane + 32 * i] : v;
    }
  };
  auto set_col = [&](int cs, const double* col) {
#pragma unroll
    for (int i = 0; i < RR_ROWS; ++i) {
      x[0][i] = (cs == 0) ? col[i] : x[0][i];
      x[1][i] = (cs == 1) ? col[i] : x[1][i];
      x[2][i] = (cs == 2) ? col[i] : x[2][i];
      x[3][i] = (cs == 3) ? col[i] : x[3][i];
      if (cs == 4) xs4[lane + 32 * i] = col[i];
    }
  };

  int red_it = 0;
  long long t_sync = 0;
  double nrm = 0.0, x0 = 0.0;
  double beta = 0.0, coeff = 0.0;
  int l_acc = k, broke = 0;
  int j = 0;
  // round kinds: 0 = exact norm of column j, 1 = same with 2^-e scaling, 2 = reflector j
  int kind = 0, escale = 0;
  const bool rec = a.dbg && blockIdx.x == (gridDim.x > 1 ? a.dbg_cta : 0) && tid == 0;
  long long tl[16];
#define STAMP(ph) \
  if (rec) tl[ph] = clock64()
  double vr[RR_ROWS];
  while (j < k) {
    int len;
    if (kind != 2) {
      // ---------------- norm round: ||column j|| over rows >= j (+ x0) ----------------
      const int wo = j & 15;
      if (wid == wo) {
        double col[RR_ROWS];
        get_col(j >> 4, col);
        double ss = 0.0, am = 0.0, xx = 0.0;
#pragma unroll
        for (int i = 0; i < RR_ROWS; ++i) {
          const int rr = lane + 32 * i;
          const bool live = rr < R && r0 + rr >= j;
          const double v = live ? (kind == 1 ? ldexp(col[i], -escale) : col[i]) : 0.0;
          ss = fma(v, v, ss);
          am = fmax(am, fabs(v));
          if (live && r0 + rr == j) xx = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ss += __shfl_xor_sync(0xffffffffu, ss, o);
          am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
          xx += __shfl_xor_sync(0xffffffffu, xx, o);
        }
        if (lane == 0) {
          s_part[0] = ss;
          s_part[1] = am;
          s_part[2] = xx;
        }
      }
      len = 3;
    } else {
      // ---------------- reflector round j ----------------
      STAMP(0);
      const int wj = j & 15;
      // v = x / u0 below the diagonal, 1 on it, 0 above / outside (owner warp)
      if (wid == wj) {
        const double rcp = 1.0 / (x0 - beta);
        double col[RR_ROWS];
        get_col(j >> 4, col);
#pragma unroll
        for (int i = 0; i < RR_ROWS; ++i) {
          const int rr = lane + 32 * i;
          const int p = r0 + rr;
          double v = 0.0;
          if (rr < R && p > j) {
            v = (nrm != 0.0) ? col[i] * rcp : col[i];
            col[i] = v;
          } else if (rr < R && p == j) {
            v = 1.0;
          }
          vbuf[rr] = v;
        }
        set_col(j >> 4, col);
      }
      __syncthreads();
      STAMP(5);
#pragma unroll
      for (int i = 0; i < RR_ROWS; ++i) vr[i] = vbuf[lane + 32 * i];
      // partials: d_q = v^T C_q (q > j), z_q = Y_q^T v (q < j); slot 4 (q = 64) on warp 0
      double sd[RR_RSLOTS + 1];
#pragma unroll
      for (int cc = 0; cc < RR_RSLOTS; ++cc) {
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int i = 0; i < RR_ROWS; i += 2) {
          s0 = fma(vr[i], x[cc][i], s0);
          s1 = fma(vr[i + 1], x[cc][i + 1], s1);
        }
        sd[cc] = s0 + s1;
      }
      STAMP(6);
      sd[4] = 0.0;
      if (wid == 0 && k > 64)
#pragma unroll
        for (int i = 0; i < RR_ROWS; ++i) sd[4] = fma(vr[i], xs4[lane + 32 * i], sd[4]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int cc = 0; cc <= RR_RSLOTS; ++cc) sd[cc] += __shfl_xor_sync(0xffffffffu, sd[cc], o);
      if (lane == 0)
#pragma unroll
        for (int cc = 0; cc <= RR_RSLOTS; ++cc) {
          const int q = wid + 16 * cc;
          if (q < k) s_part[q] = (q != j) ? sd[cc] : 0.0;
        }
      STAMP(7);
      // next column's a = ||x||^2, b = v.x, c = ||v||^2 over rows > j (+ x, v at row j+1)
      const int w1 = (j + 1) & 15;
      if (j + 1 < k && wid == w1) {
        double col[RR_ROWS];
        get_col((j + 1) >> 4, col);
        double pa = 0.0, pb = 0.0, pc = 0.0, px = 0.0, pv = 0.0;
#pragma unroll
        for (int i = 0; i < RR_ROWS; ++i) {
          const int rr = lane + 32 * i;
          const int p = r0 + rr;
          const bool live = rr < R && p > j;
          const double xv = live ? col[i] : 0.0;
          const double v = live ? vr[i] : 0.0;
          pa = fma(xv, xv, pa);
          pb = fma(v, xv, pb);
          pc = fma(v, v, pc);
          if (live && p == j + 1) {
            px = xv;
            pv = v;
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
      len = k + ((j + 1 < k) ? 5 : 0);
      STAMP(1);
    }

    // ---------------- the one all-reduce of this trip ----------------
    if constexpr (Red::cluster()) {
      __syncthreads();
      STAMP(8);
      double* base = rbuf + (red_it & 1) * RR_MAXCL * RED_LD;
      if (wid < nranks) {  // warp r pushes the whole vector to rank r
        double* dst = cg::this_cluster().map_shared_rank(base + my_rank * RED_LD, wid);
        for (int q = lane; q < len; q += 32) dst[q] = s_part[q];
      }
      STAMP(9);
      cg::this_cluster().sync();  // release/acquire
      STAMP(10);
      const int slot = tid >> 3, g = tid & 7;
      for (int q0 = 0; q0 < len; q0 += PANEL_T / 8) {
        const int q = q0 + slot;
        double s = 0.0;
        if (q < len)
          for (int b = g; b < nranks; b += 8) s += base[b * RED_LD + q];
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (q < len && g == 0) s_tot[q] = s;
      }
      STAMP(11);
      __syncthreads();
    } else {
      grid_allreduce(a, s_part, s_tot, len, red_it);
    }
    ++red_it;

    if (kind != 2) {
      // ---------------- finish a norm round ----------------
      if (kind == 0) {
        const double nrm2 = s_tot[0], abound = s_tot[1];
        x0 = s_tot[2];
        if (abound == 0.0) {
          nrm = 0.0;
        } else if (nrm2 > 1e-280 && nrm2 < 1e280) {
          nrm = sqrt(nrm2);
        } else {  // extreme magnitudes: one more round with an exact 2^-e rescale
          // s_tot[1] = sum of per-CTA maxima: an upper bound (<= G x) of max|x|
          frexp(abound, &escale);
          kind = 1;
          __syncthreads();
          continue;
        }
      } else {
        nrm = ldexp(sqrt(s_tot[0]), escale);
      }
    } else {
      STAMP(2);
      // ---------------- finish reflector j: rank-1 update, beta, T, next norm ----------------
      if (coeff != 0.0) {
#pragma unroll
        for (int cc = 0; cc < RR_RSLOTS; ++cc) {
          const int q = wid + 16 * cc;
          if (q > j && q < k) {
            const double w = coeff * s_tot[q];
#pragma unroll
            for (int i = 0; i < RR_ROWS; ++i) x[cc][i] = fma(-vr[i], w, x[cc][i]);
          }
        }
        if (wid == 0 && k > 64 && j < 64) {
          const double w = coeff * s_tot[64];
          for (int i = 0; i < RR_ROWS; ++i) xs4[lane + 32 * i] = fma(-vr[i], w, xs4[lane + 32 * i]);
        }
      }
      if (j >= r0 && j < r1 && wid == (j & 15)) {  // diagonal entry beta
        double col[RR_ROWS];
        get_col(j >> 4, col);
#pragma unroll
        for (int i = 0; i < RR_ROWS; ++i)
          if (lane + 32 * i == j - r0) col[i] = beta;
        set_col(j >> 4, col);
      }
      STAMP(3);
      if (tbuild) {  // T column j (householder.py:109-113)
        for (int i = my_rank + wid * tstride; i < j; i += PANEL_W * tstride) {
          double sacc = 0.0;
          for (int q = i + lane; q < j; q += 32) sacc = fma(s_T[i * DMQR_KP + q], s_tot[q], sacc);
          sacc = warp_sum(sacc);
          if (lane == 0) s_T[i * DMQR_KP + j] = -coeff * sacc;
        }
        if (tid == 0 && (j % tstride) == my_rank) s_T[j * DMQR_KP + j] = coeff;
        if (tid == 0 && my_rank == 0) a.coeffs[n_s + j] = coeff;
      }
      STAMP(4);
      if (rec && j < 64)
        for (int q = 0; q < 16; ++q) a.dbg[j * 16 + q] = tl[q];
      ++j;
      if (j < k) {  // next column's norm: identity without cancellation, else a norm round
        const double w = coeff * s_tot[j];
        const double pa = s_tot[k], pb = s_tot[k + 1], pc = s_tot[k + 2];
        const double nn2 = (coeff != 0.0) ? pa - 2.0 * w * pb + w * w * pc : pa;
        if (nn2 >= 0.5 * pa && pa > 1e-280 && pa < 1e280) {
          nrm = sqrt(nn2);
          x0 = fma(-s_tot[k + 4], w, s_tot[k + 3]);
        } else {
          kind = 0;
          __syncthreads();
          continue;
        }
      }
    }
    // ---------------- nrm, x0 of column j are known: break test, then reflector ----------------
    if (j >= k) break;
    if (brk && j > 0 && nrm < eps_s) {  // QRDM2 break (rrqr.py:375-379)
      l_acc = j;
      broke = 1;
      break;
    }
    if (nrm == 0.0) {
      beta = 0.0;
      coeff = 0.0;
      x0 = 1.0;  // rcp(x0 - beta) = 1: v is the (zero) column itself
    } else {
      beta = (x0 != 0.0) ? -copysign(nrm, x0) : -nrm;
      coeff = (beta - x0) / beta;
    }
    kind = 2;
    __syncthreads();
  }
#undef STAMP
  // ---- write the slice back ----
#pragma unroll
  for (int cc = 0; cc < RR_RSLOTS; ++cc) {
    const int q = wid + 16 * cc;
#pragma unroll
    for (int i = 0; i < RR_ROWS; ++i) {
      const int rr = lane + 32 * i;
      if (q < k && rr < R) gA[(int64_t)q * lda + rr] = x[cc][i];
    }
  }
  if (wid == 0 && k > 64)
    for (int i = 0; i < RR_ROWS; ++i) {
      const int rr = lane + 32 * i;
      if (rr < R) gA[(int64_t)64 * lda + rr] = xs4[rr];
    }
  if (tbuild) {
    __syncthreads();
    for (int e = tid; e < l_acc * l_acc; e += PANEL_T) {
      const int i = e / l_acc, jj = e % l_acc;
      if (i <= jj && (i % tstride) == my_rank) a.T[i * DMQR_KP + jj] = s_T[i * DMQR_KP + jj];
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    c->l_acc = l_acc;
    c->broke = broke;
    c->tc0 = (int32_t)(n_s + k);
  }
  if constexpr (Red::cluster()) cg::this_cluster().sync();  // no rank exits while others may push
}

}  // namespace dmqr
