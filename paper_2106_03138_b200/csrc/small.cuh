// Fused per-matrix QRDM / QRDM2 for small matrices (m <= 256, n <= 512,
// k_dm <= 64): one CTA runs the whole outer loop of _qrdm_engine
// (rrqr.py:315-423) for one matrix, with every decision, the panel, the
// compact-WY factor and the trailing update in one launch -- no host round
// trips, no per-step kernels.  A persistent grid walks the matrices of a batch
// (BASELINE cfg3: 1024 x 256^2), one CTA per SM.
//
// Per outer step (reference operation in brackets):
//   stop test            [check_stop, rrqr.py:189-203, 336-338]
//   floor -> scalar step [dm.py:139-143, _scalar_step rrqr.py:219-235]
//   seed + candidates    [candidate_set, dm.py:81-97]: first argmax; u_i >= tau u_seed,
//                        stable descending order, first k_dm (rank counting)
//   cosine matrix        [cosine_matrix, dm.py:100-115]: candidate columns gathered into
//                        shared memory, fresh scaled norms, G = C^T C on DMMA,
//                        theta_ij = (G_ij inv_i) inv_j, mirrored, unit diagonal
//   greedy delta filter  [dm_select, dm.py:151-177]: 64-bit conflict masks, sequential
//                        accept in candidate order (delta_max mode: the reference's
//                        row-sum bookkeeping on one thread); gamma
//   swaps                [_move_selected_to_front, rrqr.py:294-312]: the exact
//                        transposition sequence (one warp), logged; column data moved
//                        once as a composed permutation
//   panel                [make_reflector / apply_reflector_left / QRDM2 break,
//                        householder.py:57-89, rrqr.py:360-379]: shared-memory resident,
//                        one reflector per barrier (column c owned by warp c mod 8)
//   T factor             [accumulate_wy, householder.py:92-114]: S = Y^T Y on DMMA,
//                        W[:j, j] = -coeff_j W[:j, :j] S[:j, j]
//   trailing update      [apply_block_left, householder.py:117-128]: per warp and
//                        8-column tile, Z = Y^T C, Wt = W^T Z, C -= Y Wt on DMMA with
//                        register-resident fragments (warps are independent)
//   norm downdate        [downdate_norms, rrqr.py:161-186] with the exact recompute
//                        of guarded columns
//   step record          [StepRecord, rrqr.py:394-404]
// and at the end the rank [rrqr.py:406-412, _posthoc_rank 206-208].
#pragma once
#include "common.cuh"

namespace dmqr {

constexpr int SM_T = 256;      // 8 warps
constexpr int SM_W = SM_T / 32;
constexpr int SM_MMAX = 256;   // rows
constexpr int SM_NMAX = 512;   // columns
constexpr int SM_LDP = 260;    // panel column stride (4 mod 16: conflict-free 8x4 fragments)
constexpr int SM_GLD = 84;     // Gram / T row stride (4 mod 16)
constexpr int SM_KC = 65;      // candidate columns (seed + k_dm <= 64)
constexpr int SM_MVROWS = 32;  // rows per chunk of the staged column moves
// per-matrix status codes (include/dmqr_b200.h): ENONFINITE, EZEROCOL, ECAP
constexpr int SM_ST_NONFINITE = -2, SM_ST_ZEROCOL = -3, SM_ST_CAP = -5;

struct SmallInfo {  // per matrix, device side (host mirrors it into dmqr_info)
  int32_t rank, n_factored, n_steps, n_swaps, stopped, status;
  double a_max0;
};

struct SmallArgs {
  double* A;
  int64_t batch, m, n, lda, stride;
  double tau, delta, eps1;  // eps1 < 0: StopRule.NONE (no stop test)
  int32_t k_dm, use_delta_max, break_check, stop_none;
  double* coeffs;   // batch x kmax
  int64_t* perm;    // batch x n
  int64_t* swaps;   // batch x swap_cap x 2
  int64_t swap_cap;
  StepRec* steps;   // batch x step_cap
  int64_t step_cap;
  SmallInfo* info;  // batch
  long long* dbg;   // debug: CTA 0's cycles per phase (16 slots, accumulated) or null
};

struct SmallSmem {
  double P[DMQR_KP * SM_LDP];  // candidate columns -> panel -> Y (column c at P + c*LDP)
  double G[DMQR_KP * SM_GLD];  // Gram / theta -> move staging -> S -> T
  double u[SM_NMAX], uref[SM_NMAX];
  double dn[DMQR_KP], cf[DMQR_KP];
  double red[2 * SM_W];
  unsigned long long conf[DMQR_KP];
  int perm[SM_NMAX];
  int srcof[SM_NMAX];
  int clist[SM_NMAX];
  int cols[DMQR_KP];   // absolute column of candidate t (seed first)
  int selt[DMQR_KP];   // chosen candidate indices, in order
  int mv_dst[2 * DMQR_KP], mv_src[2 * DMQR_KP];
  int cyc_pos[2 * DMQR_KP], cyc_beg[2 * DMQR_KP + 1];  // move cycles: new[p_i] = old[p_{i+1}]
  int ncyc;
  int redi[2 * SM_W];
  int nmv, nsel, kmax_c, status, nsw_log;
  int brk[2];
  int pub, brkat;      // panel dataflow: reflectors published, break column (k_s: none)
  int prog[SM_W];      // panel dataflow: reflectors whose v each warp has loaded
  double gamma, coeff, umax;
  int seed;
};
constexpr size_t SM_SMEM = sizeof(SmallSmem);

__device__ __forceinline__ double sm_wmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Scaled Euclidean norm (matrix.py:61-78) of x[0, len) (shared or global,
// plain loads: the data may have been written by this kernel), warp-wide.
// (len <= SM_MMAX: the eight row slots of a lane are unrolled, so their loads
// are all in flight together)
__device__ __forceinline__ double sm_norm_regs(const double (&v)[SM_MMAX / 32], int lane) {
  double s0 = 0.0, s1 = 0.0, a = 0.0;
#pragma unroll
  for (int q = 0; q < SM_MMAX / 32; q += 2) {
    s0 = fma(v[q], v[q], s0);
    s1 = fma(v[q + 1], v[q + 1], s1);
    a = fmax(a, fmax(fabs(v[q]), fabs(v[q + 1])));
  }
  double s = s0 + s1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
  }
  if (a == 0.0) return 0.0;
  if (norm_range_ok(a)) return sqrt(s);
  double t = 0.0;
#pragma unroll
  for (int q = 0; q < SM_MMAX / 32; ++q) {
    const double z = v[q] / a;
    t = fma(z, z, t);
  }
  return a * sqrt(warp_sum(t));
}
__device__ __forceinline__ double sm_norm(const double* x, int len, int lane) {
  double v[SM_MMAX / 32];
#pragma unroll
  for (int q = 0; q < SM_MMAX / 32; ++q) v[q] = (lane + 32 * q < len) ? x[lane + 32 * q] : 0.0;
  return sm_norm_regs(v, lane);
}

// Upper 8x8 tiles (a <= b < nt) of X^T X for the columns of P (K = k4 rows,
// a multiple of 4, rows past the data zero) -> G (row-major, SM_GLD); each warp
// keeps up to three tiles' DMMA chains in flight.
__device__ void sm_gram(const double* P, int nt, int k4, double* G) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ntl = nt * (nt + 1) / 2;
  for (int t0 = wid; t0 < ntl; t0 += 3 * SM_W) {
    int ta[3], tb[3];
    double acc[3][2];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      int t = t0 + q * SM_W;
      ta[q] = -1;
      tb[q] = 0;
      if (t < ntl) {  // t -> (a, b), row-major over the upper triangle
        int a = 0;
        while (t >= nt - a) {
          t -= nt - a;
          ++a;
        }
        ta[q] = a;
        tb[q] = a + t;
      }
      acc[q][0] = acc[q][1] = 0.0;
    }
    const int lr = lane >> 2, lk = lane & 3;
    for (int k0 = 0; k0 < k4; k0 += 4) {
#pragma unroll
      for (int q = 0; q < 3; ++q)
        if (ta[q] >= 0)
          dmma884(acc[q][0], acc[q][1], P[(ta[q] * 8 + lr) * SM_LDP + k0 + lk], P[(tb[q] * 8 + lr) * SM_LDP + k0 + lk]);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (ta[q] >= 0) {
        double* g = G + (ta[q] * 8 + lr) * SM_GLD + tb[q] * 8 + 2 * lk;
        g[0] = acc[q][0];
        g[1] = acc[q][1];
      }
  }
}

// One warp's share of the trailing update C <- C - Y (W^T (Y^T C)) for the
// 8-column tile at (absolute) column c0: Y = P[:, 0:l) (unit lower, rows
// [0, mp) of the panel), W (upper, l x l) in G.  LT = ceil(l / 8).
template <int LT>
__device__ void sm_trail_tile(double* __restrict__ A, int64_t lda, int n_s, int mp, int l, int64_t c0, int64_t ncend,
                              const double* __restrict__ P, const double* __restrict__ G) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lk = lane & 3;
  const int k4 = (mp + 3) & ~3;
  const int lp4 = (l + 3) & ~3;
  double* Cg = A + n_s;  // C[r][c] = Cg[r + c * lda]
  // ---- Z = Y^T C (l x 8): B fragments straight from global (L2), 8 k-steps in flight ----
  double z[LT][2];
#pragma unroll
  for (int q = 0; q < LT; ++q) z[q][0] = z[q][1] = 0.0;
  const int64_t cb = c0 + lr;  // this lane's B column
  const bool cval = cb < ncend;
  const double* cp = Cg + cb * lda;
  for (int k0 = 0; k0 < k4; k0 += 32) {
    double b[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int r = k0 + 4 * s + lk;
      b[s] = (cval && r < mp) ? cp[r] : 0.0;
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int kk = k0 + 4 * s;
      if (kk < k4) {
#pragma unroll
        for (int q = 0; q < LT; ++q) dmma884(z[q][0], z[q][1], P[(q * 8 + lr) * SM_LDP + kk + lk], b[s]);
      }
    }
  }
  // ---- Wt = W^T Z (l x 8): Z's B fragments by shuffles from the accumulators ----
  // Z[i][j] sits in z[i >> 3] of lane (i & 7) * 4 + (j >> 1), register j & 1
  double w[LT][2];
#pragma unroll
  for (int q = 0; q < LT; ++q) w[q][0] = w[q][1] = 0.0;
#pragma unroll
  for (int s = 0; s < 2 * LT; ++s) {
    if (4 * s < lp4) {
      const int src = (4 * (s & 1) + lk) * 4 + (lane >> 3);
      const double v0 = __shfl_sync(0xffffffffu, z[s >> 1][0], src);
      const double v1 = __shfl_sync(0xffffffffu, z[s >> 1][1], src);
      const double bz = (lr & 1) ? v1 : v0;
#pragma unroll
      for (int q = 0; q < LT; ++q) dmma884(w[q][0], w[q][1], G[(4 * s + lk) * SM_GLD + q * 8 + lr], bz);
    }
  }
  double wb[2 * LT];
#pragma unroll
  for (int s = 0; s < 2 * LT; ++s) {
    const int src = (4 * (s & 1) + lk) * 4 + (lane >> 3);
    const double v0 = __shfl_sync(0xffffffffu, w[s >> 1][0], src);
    const double v1 = __shfl_sync(0xffffffffu, w[s >> 1][1], src);
    wb[s] = (lr & 1) ? v1 : v0;
  }
  // ---- C -= Y Wt, four 8-row tiles at a time (accumulators = C) ----
  const int64_t ca = c0 + 2 * lk;
  const bool v0c = ca < ncend, v1c = ca + 1 < ncend;
  const int nrt = (mp + 7) >> 3;
  for (int rt0 = 0; rt0 < nrt; rt0 += 4) {
    double acc[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = (rt0 + q) * 8 + lr;
      const bool rv = r < mp;
      acc[q][0] = (rv && v0c) ? Cg[r + ca * lda] : 0.0;
      acc[q][1] = (rv && v1c) ? Cg[r + (ca + 1) * lda] : 0.0;
    }
#pragma unroll
    for (int s = 0; s < 2 * LT; ++s) {
      if (4 * s < lp4) {
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (rt0 + q < nrt) dmma884(acc[q][0], acc[q][1], -P[(4 * s + lk) * SM_LDP + (rt0 + q) * 8 + lr], wb[s]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = (rt0 + q) * 8 + lr;
      if (r < mp) {
        if (v0c) Cg[r + ca * lda] = acc[q][0];
        if (v1c) Cg[r + (ca + 1) * lda] = acc[q][1];
      }
    }
  }
}

__device__ __forceinline__ void sm_trail(int lt, double* A, int64_t lda, int n_s, int mp, int l, int64_t c0,
                                         int64_t ncend, const double* P, const double* G) {
  switch (lt) {
    case 1: sm_trail_tile<1>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
    case 2: sm_trail_tile<2>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
    case 3: sm_trail_tile<3>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
    case 4: sm_trail_tile<4>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
    case 5: sm_trail_tile<5>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
    case 6: sm_trail_tile<6>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
    case 7: sm_trail_tile<7>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
    case 8: sm_trail_tile<8>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
    default: sm_trail_tile<9>(A, lda, n_s, mp, l, c0, ncend, P, G); break;
  }
}

// block argmax of u[lo, hi) (first occurrence) -> (value, index) on every thread
__device__ __forceinline__ void sm_argmax(const double* u, int lo, int hi, SmallSmem& s, double& vmax, int& imax) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int i = lo + tid; i < hi; i += SM_T) {
    const double v = u[i];
    if (v > bv) {  // ascending indices per thread: strict > keeps the first
      bv = v;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  if (lane == 0) {
    s.red[wid] = bv;
    s.redi[wid] = bi;
  }
  __syncthreads();
  bv = s.red[0];
  bi = s.redi[0];
  for (int w = 1; w < SM_W; ++w) {
    const double ov = s.red[w];
    const int oi = s.redi[w];
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
  __syncthreads();
  vmax = bv;
  imax = bi;
}

// norm downdate of columns [n_s1, n) after rows [n_s, n_s1) became final
// (rrqr.py:161-186): u^2 - sum r^2, exact recompute below the guard
__device__ void sm_downdate(const SmallArgs& a, double* A, int64_t lda, int m, int n, int n_s, int n_s1, SmallSmem& s) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int j = n_s + tid; j < n_s1; j += SM_T) {
    s.u[j] = 0.0;
    s.uref[j] = 0.0;
  }
  // (l = n_s1 - n_s <= 65 rows: three row slots per lane; four columns per pass)
  for (int j0 = n_s1 + 4 * wid; j0 < n; j0 += 4 * SM_W) {
    double x[4][3];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int r = n_s + lane + 32 * q;
        x[c][q] = (j0 + c < n && r < n_s1) ? A[(int64_t)(j0 + c) * lda + r] : 0.0;
      }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = j0 + c;
      const double d = warp_sum(fma(x[c][0], x[c][0], fma(x[c][1], x[c][1], x[c][2] * x[c][2])));
      if (j >= n) continue;
      const double uj = s.u[j], rj = s.uref[j];
      const double sq = __dsub_rn(__dmul_rn(uj, uj), d);
      double nu = sqrt(fmax(sq, 0.0));
      if (sq <= __dmul_rn(1e-2, __dmul_rn(rj, rj))) {
        nu = sm_norm(A + (int64_t)j * lda + n_s1, m - n_s1, lane);
        if (lane == 0) s.uref[j] = nu;
      }
      if (lane == 0) s.u[j] = nu;
    }
  }
}

// Reflector j of the panel in shared memory (make_reflector, householder.py:57-79),
// by one warp: x = P[j][j:mp); the QRDM2 break test on its fresh norm first
// (rrqr.py:375-379: ||work[col+1:, col+1]|| < eps_s); beta on the diagonal,
// v[1:] = x[1:] / (x0 - beta) below it, coeff -> cf[j]; brk[j & 1] published.
__device__ __forceinline__ void sm_reflector(SmallSmem& s, int j, int mp, double eps_s, int break_check, int lane) {
  double* x = s.P + j * SM_LDP;
  const double nrm = sm_norm(x + j, mp - j, lane);
  const int brk = (break_check && j >= 1 && nrm < eps_s) ? 1 : 0;
  if (!brk) {
    const double x0 = x[j];
    double beta = 0.0, cf = 0.0;
    if (nrm > 0.0) {
      beta = (x0 != 0.0) ? -copysign(nrm, x0) : -nrm;
      const double rden = 1.0 / (x0 - beta);  // (v = x / (x0 - beta) as x * rden: <= 1 ulp apart)
#pragma unroll
      for (int q = 0; q < SM_MMAX / 32; ++q) {
        const int r = j + 1 + lane + 32 * q;
        if (r < mp) x[r] *= rden;
      }
      cf = (beta - x0) / beta;
    }
    __syncwarp();
    if (lane == 0) {
      x[j] = beta;
      s.cf[j] = cf;
    }
  }
  if (lane == 0) s.brk[j & 1] = brk;
}

// col <- (I - cf v v^T) col on rows [j, mp) (apply_reflector_left, householder.py:82-89), one warp
__device__ __forceinline__ void sm_apply1(double* col, const double* v, double cf, int j, int mp, int lane) {
  constexpr int NQ = SM_MMAX / 32;
  double vr[NQ], cr[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int r = j + 1 + lane + 32 * q;
    const bool ok = r < mp;
    vr[q] = ok ? v[r] : 0.0;
    cr[q] = ok ? col[r] : 0.0;
  }
  double t0 = 0.0, t1 = 0.0;
#pragma unroll
  for (int q = 0; q < NQ; q += 2) {
    t0 = fma(vr[q], cr[q], t0);
    t1 = fma(vr[q + 1], cr[q + 1], t1);
  }
  const double t = warp_sum(t0 + t1) + col[j];
  const double w = cf * t;
  __syncwarp();
  if (lane == 0) col[j] -= w;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int r = j + 1 + lane + 32 * q;
    if (r < mp) col[r] = fma(-vr[q], w, cr[q]);
  }
}

// The same for the columns first, first + 8, ... (< k_s, at most 8) in one
// pass: v is read once per row, the eight sums are reduced together
// (16 -> 8 -> 4 lanes exchange halves, then a plain butterfly).
__device__ __forceinline__ void sm_apply8(double* P, const double* v, double cf, int j, int mp, int first, int k_s,
                                          int lane) {
  constexpr int NQ = SM_MMAX / 32;
  double vr[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int r = j + 1 + lane + 32 * q;
    vr[q] = (r < mp) ? v[r] : 0.0;  // (rows past mp: v = 0, P rows there are zero padding or unused)
  }
  double t[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = first + SM_W * i;
    double acc = 0.0;
    if (c < k_s) {
      const double* pc = P + c * SM_LDP + j + 1 + lane;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (j + 1 + lane + 32 * q < mp) acc = fma(vr[q], pc[32 * q], acc);
    }
    t[i] = acc;
  }
  // level 16: keep 4 of 8
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool hi = lane & 16;
    const double keep = hi ? t[i + 4] : t[i], send = hi ? t[i] : t[i + 4];
    t[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool hi = lane & 8;
    const double keep = hi ? t[i + 2] : t[i], send = hi ? t[i] : t[i + 2];
    t[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const bool hi = lane & 4;
    const double keep = hi ? t[1] : t[0], send = hi ? t[0] : t[1];
    t[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  t[0] += __shfl_xor_sync(0xffffffffu, t[0], 2);
  t[0] += __shfl_xor_sync(0xffffffffu, t[0], 1);
  // lane 16a + 8b + 4c holds the sum of column index 4a + 2b + c
  double w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double ti = __shfl_sync(0xffffffffu, t[0], 16 * (i >> 2) + 8 * ((i >> 1) & 1) + 4 * (i & 1));
    const int c = first + SM_W * i;
    w[i] = (c < k_s) ? cf * (ti + P[c * SM_LDP + j]) : 0.0;
  }
  __syncwarp();
  if (lane < 8) {
    const int c = first + SM_W * lane;
    double wl = w[0];
#pragma unroll
    for (int i = 1; i < 8; ++i)
      if (lane == i) wl = w[i];
    if (c < k_s) P[c * SM_LDP + j] -= wl;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int c = first + SM_W * i;
    if (c < k_s) {
      double* pc = P + c * SM_LDP + j + 1 + lane;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (j + 1 + lane + 32 * q < mp) pc[32 * q] = fma(-vr[q], w[i], pc[32 * q]);
    }
  }
}

// ---------------------------------------------------------------------------
// Register-resident panel (make_reflector / apply_reflector_left / the QRDM2
// break, householder.py:57-89, rrqr.py:360-379).  Warp w keeps the panel
// columns c = w + 8 i (i < 9) in registers, lane l rows l + 32 q (q < 8):
// each reflector costs one block barrier, one shared-memory read of the
// published v and register FMAs -- the panel is never swept through shared
// memory.  Reflector j+1 is formed by the owner of column j+1 right after it
// applied reflector j to that column, ahead of its other columns.
// ---------------------------------------------------------------------------
constexpr int SMP_NQ = SM_MMAX / 32;  // row slots per lane
constexpr int SMP_NI = 9;             // column slots per warp (65 columns / 8 warps)
constexpr int SMP_RING = 4;           // published-reflector buffers

// reflector from the column held in x (rows jj.. of the panel): v -> x (beta on
// the diagonal row), published to V (unit diagonal, zeros above and past mp),
// coeff -> cf[jj], break flag -> brk[jj & 1]
__device__ __forceinline__ int smp_reflector(double (&x)[SMP_NQ], SmallSmem& s, double* V, int jj, int mp,
                                             double eps_s, int break_check, int lane) {
  double xv[SMP_NQ];
  double ss = 0.0, am = 0.0;
#pragma unroll
  for (int q = 0; q < SMP_NQ; ++q) {
    const int r = lane + 32 * q;
    xv[q] = (r >= jj && r < mp) ? x[q] : 0.0;
    ss = fma(xv[q], xv[q], ss);
    am = fmax(am, fabs(xv[q]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
  }
  double nrm = 0.0;
  if (am > 0.0) {
    if (norm_range_ok(am)) {
      nrm = sqrt(ss);
    } else {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < SMP_NQ; ++q) {
        const double z = xv[q] / am;
        t = fma(z, z, t);
      }
      nrm = am * sqrt(warp_sum(t));
    }
  }
  const int brk = (break_check && jj >= 1 && nrm < eps_s) ? 1 : 0;  // fresh ||work[col+1:, col+1]|| < eps_s
  double x0 = 0.0;
#pragma unroll
  for (int q = 0; q < SMP_NQ; ++q)
    if (q == (jj >> 5)) x0 = __shfl_sync(0xffffffffu, x[q], jj & 31);
  if (!brk) {
    double beta = 0.0, cf = 0.0, rden = 0.0;
    if (nrm > 0.0) {
      beta = (x0 != 0.0) ? -copysign(nrm, x0) : -nrm;
      rden = __drcp_rn(x0 - beta);  // (v = x / (x0 - beta) as x * rden: <= 1 ulp apart)
      cf = (beta - x0) * __drcp_rn(beta);
    }
    double* vb = V + (jj & (SMP_RING - 1)) * SM_LDP;
#pragma unroll
    for (int q = 0; q < SMP_NQ; ++q) {
      const int r = lane + 32 * q;
      double vr = 0.0;
      if (r > jj && r < mp) {
        vr = x[q] * rden;
        x[q] = vr;
      } else if (r == jj) {
        vr = 1.0;
        x[q] = beta;
      }
      vb[r] = vr;
    }
    if (lane == 0) s.cf[jj] = cf;
  }
  return brk;
}

// publish reflector jj (or the break at jj) to the other warps of the panel
__device__ __forceinline__ void smp_publish(SmallSmem& s, int jj, int brk, int lane) {
  __syncwarp();
  if (lane == 0) {
    __threadfence_block();
    if (brk)
      *(volatile int*)&s.brkat = jj;
    else
      *(volatile int*)&s.pub = jj + 1;
  }
}

__device__ int sm_panel_regs(SmallSmem& s, int k_s, int mp, double eps_s, int break_check, long long* dclk) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double pc[SMP_NI][SMP_NQ];
#pragma unroll
  for (int i = 0; i < SMP_NI; ++i) {
    const int c = wid + SM_W * i;
#pragma unroll
    for (int q = 0; q < SMP_NQ; ++q) {
      const int r = lane + 32 * q;
      pc[i][q] = (c < k_s && r < mp) ? s.P[c * SM_LDP + r] : 0.0;
    }
  }
  // Dataflow instead of one block barrier per reflector: the owner of column
  // j+1 publishes reflector j+1 (ring of SMP_RING v buffers; a slot is reused
  // once every warp has loaded the reflector it held) and each warp applies the
  // reflectors to its columns in order, as they appear.  The chain of owners is
  // the critical path; the other warps' updates trail it.
  double* V = s.G;  // [SMP_RING][SM_LDP] published reflectors
  if (threadIdx.x == 0) {
    s.pub = 0;
    s.brkat = k_s;
  }
  if (threadIdx.x < SM_W) s.prog[threadIdx.x] = 0;
  __syncthreads();
  if (wid == 0) smp_publish(s, 0, smp_reflector(pc[0], s, V, 0, mp, eps_s, break_check, lane), lane);
  for (int j = 0; j < k_s; ++j) {
    const bool pk = dclk && j == 16 && ((j + 1) & (SM_W - 1)) == wid && lane == 0;
    long long c0 = pk ? clock64() : 0;
    int p, bk;
    for (;;) {
      p = *(volatile int*)&s.pub;
      bk = *(volatile int*)&s.brkat;
      if (p > j || bk <= j) break;
      __nanosleep(32);  // (leave the issue slots to the warp forming the next reflector)
    }
    __threadfence_block();
    if (pk) dclk[16] = clock64() - c0;
    if (bk <= j) break;
    const double cf = s.cf[j];
    double vq[SMP_NQ];
#pragma unroll
    for (int q = 0; q < SMP_NQ; ++q) vq[q] = V[(j & (SMP_RING - 1)) * SM_LDP + lane + 32 * q];
    __syncwarp();
    if (lane == 0) *(volatile int*)&s.prog[wid] = j + 1;  // (v_j is in registers)
    if (pk) dclk[17] = clock64() - c0;
    const int j1 = j + 1;
    const bool owner = ((j1 & (SM_W - 1)) == wid) && j1 < k_s;
    const int i1 = j1 >> 3;
    if (owner) {  // column j+1 first: reflector j, then form and publish reflector j+1
#pragma unroll
      for (int i = 0; i < SMP_NI; ++i)
        if (i == i1) {
          if (cf != 0.0) {
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int q = 0; q < SMP_NQ; q += 2) {
              t0 = fma(vq[q], pc[i][q], t0);
              t1 = fma(vq[q + 1], pc[i][q + 1], t1);
            }
            const double w = cf * warp_sum(t0 + t1);
#pragma unroll
            for (int q = 0; q < SMP_NQ; ++q) pc[i][q] = fma(-vq[q], w, pc[i][q]);
          }
          if (pk) dclk[18] = clock64() - c0;
          // ring slot of reflector j1 held reflector j1 - SMP_RING: every warp must have loaded it
          if (j1 >= SMP_RING) {
            for (;;) {
              int mn = 0x7fffffff;
#pragma unroll
              for (int w = 0; w < SM_W; ++w) mn = min(mn, *(volatile int*)&s.prog[w]);
              if (mn > j1 - SMP_RING) break;
              __nanosleep(32);
            }
            __threadfence_block();
          }
          if (pk) dclk[19] = clock64() - c0;
          const int bkr = smp_reflector(pc[i], s, V, j1, mp, eps_s, break_check, lane);
          if (pk) dclk[20] = clock64() - c0;
          smp_publish(s, j1, bkr, lane);
          if (pk) dclk[21] = clock64() - c0;
        }
    }
    if (cf == 0.0) continue;  // reflect_left with coeff 0 is a no-op (householder.py:86-87)
    // the warp's other columns c > j: all slots computed (independent chains), dead ones masked
    double t[SMP_NI];
#pragma unroll
    for (int i = 0; i < SMP_NI; ++i) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int q = 0; q < SMP_NQ; q += 2) {
        a0 = fma(vq[q], pc[i][q], a0);
        a1 = fma(vq[q + 1], pc[i][q + 1], a1);
      }
      const int c = wid + SM_W * i;
      t[i] = (c > j && c < k_s && !(owner && i == i1)) ? a0 + a1 : 0.0;
    }
    // reduce t[0..7] together (halves exchanged at 16, 8, 4), t[8] alone
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool hi = lane & 16;
      const double keep = hi ? t[i + 4] : t[i], send = hi ? t[i] : t[i + 4];
      t[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const bool hi = lane & 8;
      const double keep = hi ? t[i + 2] : t[i], send = hi ? t[i] : t[i + 2];
      t[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {
      const bool hi = lane & 4;
      const double keep = hi ? t[1] : t[0], send = hi ? t[0] : t[1];
      t[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    t[0] += __shfl_xor_sync(0xffffffffu, t[0], 2);
    t[0] += __shfl_xor_sync(0xffffffffu, t[0], 1);
    const double t8 = warp_sum(t[8]);
#pragma unroll
    for (int i = 0; i < SMP_NI; ++i) {
      const double ti = (i < 8) ? __shfl_sync(0xffffffffu, t[0], 16 * (i >> 2) + 8 * ((i >> 1) & 1) + 4 * (i & 1))
                                : t8;
      const double w = cf * ti;  // (0 for dead slots: their columns are unchanged)
#pragma unroll
      for (int q = 0; q < SMP_NQ; ++q) pc[i][q] = fma(-vq[q], w, pc[i][q]);
    }
    if (pk) dclk[22] = clock64() - c0;
  }
  __syncthreads();
  const int l = s.brkat;
  // columns back to shared memory (R above the diagonal, beta, v below; rejected columns updated)
#pragma unroll
  for (int i = 0; i < SMP_NI; ++i) {
    const int c = wid + SM_W * i;
    if (c < k_s) {
#pragma unroll
      for (int q = 0; q < SMP_NQ; ++q) {
        const int r = lane + 32 * q;
        if (r < mp) s.P[c * SM_LDP + r] = pc[i][q];
      }
    }
  }
  return l;
}

__global__ void __launch_bounds__(SM_T, 1) k_small_qrdm(SmallArgs a) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  SmallSmem& s = *reinterpret_cast<SmallSmem*>(sm_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int m = (int)a.m, n = (int)a.n, kmax = min(m, n);
  const int64_t lda = a.lda;
  const bool clk = a.dbg && blockIdx.x == 0 && tid == 0;
  long long t_last = clk ? clock64() : 0;
#define SMT(i)                          \
  if (clk) {                            \
    const long long t_now = clock64();  \
    a.dbg[i] += t_now - t_last;         \
    t_last = t_now;                     \
  }
  for (int64_t b = blockIdx.x; b < a.batch; b += gridDim.x) {
    double* A = a.A + b * a.stride;
    double* coeffs = a.coeffs + b * (int64_t)max(kmax, 1);
    int64_t* swaps = a.swaps + b * 2 * a.swap_cap;
    StepRec* steps = a.steps + b * a.step_cap;
    // ---- initial norms, finiteness (dense(): matrix.py:32-33; from_matrix: rrqr.py:126-129) ----
    if (tid == 0) {
      s.status = 0;
      s.nsw_log = 0;
    }
    for (int j = tid; j < n; j += SM_T) {
      s.perm[j] = j;
      s.srcof[j] = j;
    }
    for (int j = tid; j < kmax; j += SM_T) coeffs[j] = 0.0;
    int bad = 0;
    for (int j = wid; j < n; j += SM_W) {
      const double* col = A + (int64_t)j * lda;
      double v[SM_MMAX / 32];
#pragma unroll
      for (int q = 0; q < SM_MMAX / 32; ++q) v[q] = (lane + 32 * q < m) ? col[lane + 32 * q] : 0.0;
#pragma unroll
      for (int q = 0; q < SM_MMAX / 32; ++q) bad |= !isfinite(v[q]);
      const double nu = sm_norm_regs(v, lane);
      if (lane == 0) {
        s.u[j] = nu;
        s.uref[j] = nu;
      }
    }
    bad = __syncthreads_or(bad);
    if (bad && tid == 0) s.status = SM_ST_NONFINITE;
    double a0;
    int a0i;
    sm_argmax(s.u, 0, n, s, a0, a0i);
    a0 = fmax(a0, 0.0);  // (n == 0: max of nothing is 0, rrqr.py:326)
    const double floor_v = (double)n * kEps * a0;
    SMT(0);
    const bool stop_active = a.eps1 >= 0.0;
    const double stop_rhs = stop_active ? a.eps1 * a0 : 0.0;
    int n_s = 0, step = 0;
    bool stopped = false;
    __syncthreads();
    while (n_s < kmax && s.status == 0) {
      if (step >= a.step_cap) {
        if (tid == 0) s.status = SM_ST_CAP;
        break;
      }
      const int mp = m - n_s;
      double umax;
      int seed;
      sm_argmax(s.u, n_s, n, s, umax, seed);
      SMT(1);
      if (stop_active && sqrt((double)(n - n_s)) * umax <= stop_rhs) {  // rrqr.py:197-203 (<=)
        stopped = true;
        break;
      }
      if (umax <= floor_v) {
        // ================= scalar fallback step (rrqr.py:219-235) =================
        const int sc = n_s, j = seed;
        if (j != sc) {
          for (int r = tid; r < m; r += SM_T) {
            double* p0 = A + (int64_t)sc * lda + r;
            double* p1 = A + (int64_t)j * lda + r;
            const double x0 = *p0, x1 = *p1;
            *p0 = x1;
            *p1 = x0;
          }
          if (tid == 0) {
            double t = s.u[sc]; s.u[sc] = s.u[j]; s.u[j] = t;
            t = s.uref[sc]; s.uref[sc] = s.uref[j]; s.uref[j] = t;
            const int pi = s.perm[sc]; s.perm[sc] = s.perm[j]; s.perm[j] = pi;
            if (s.nsw_log < a.swap_cap) {
              swaps[2 * s.nsw_log] = sc;
              swaps[2 * s.nsw_log + 1] = j;
            }
            s.nsw_log++;
          }
          __syncthreads();
        }
        double* x = A + (int64_t)sc * lda + sc;  // x = work[s:, s], length mp
        if (wid == 0) {
          const double nrm = sm_norm(x, mp, lane);
          const double x0 = x[0];
          double beta = 0.0, cf = 0.0;
          if (nrm > 0.0) {  // (amax == 0 <=> nrm == 0: identity, coeff 0)
            beta = (x0 != 0.0) ? -copysign(nrm, x0) : -nrm;
            const double den = x0 - beta;
            for (int r = 1 + lane; r < mp; r += 32) x[r] = x[r] / den;
            cf = (beta - x0) / beta;
          }
          __syncwarp();
          if (lane == 0) {
            x[0] = beta;  // packed: beta on the diagonal, v[1:] below
            s.coeff = cf;
            coeffs[sc] = cf;
          }
        }
        __syncthreads();
        const double cf = s.coeff;
        if (cf != 0.0) {  // reflect_left: w = coeff (v^T C), C -= v w^T (householder.py:82-89)
          for (int c = sc + 1 + wid; c < n; c += SM_W) {
            double* col = A + (int64_t)c * lda + sc;
            double d = col[0];
            double t = 0.0;
            for (int r = 1 + lane; r < mp; r += 32) t = fma(x[r], col[r], t);
            t = warp_sum(t);
            if (lane == 0) t += d;  // v[0] = 1
            t = __shfl_sync(0xffffffffu, t, 0);
            const double w = cf * t;
            if (lane == 0) col[0] = d - w;
            for (int r = 1 + lane; r < mp; r += 32) col[r] = fma(-x[r], w, col[r]);
          }
        }
        __syncthreads();
        sm_downdate(a, A, lda, m, n, sc, sc + 1, s);
        SMT(15);
        if (tid == 0) {
          StepRec rec;
          rec.n_s = sc;
          rec.k_selected = 1;
          rec.k_accepted = 1;
          rec.k_max = -1;
          rec.broke_early = 0;
          rec.fell_back_to_scalar = 1;
          rec.eps_s = 0.0;
          rec.gamma = 1.0;
          steps[step] = rec;
        }
        __syncthreads();
        n_s += 1;
        ++step;
        continue;
      }
      // ================= deviation-maximization step =================
      // ---- candidates (dm.py:81-97): u_i >= tau u_seed, i != seed, stable descending, first k_dm ----
      const double th = a.tau * umax;
      {
        int cnt = 0;
        // compact list of candidates (index order) by a block scan of per-warp ballots
        int base = 0;
        for (int i0 = n_s; i0 < n; i0 += SM_T) {
          const int i = i0 + tid;
          const bool isc = i < n && i != seed && s.u[i] >= th;
          const unsigned bal = __ballot_sync(0xffffffffu, isc);
          if (lane == 0) s.redi[wid] = __popc(bal);
          __syncthreads();
          int off = base;
          for (int w = 0; w < wid; ++w) off += s.redi[w];
          int tot = 0;
          for (int w = 0; w < SM_W; ++w) tot += s.redi[w];
          if (isc) s.clist[off + __popc(bal & ((1u << lane) - 1u))] = i;
          base += tot;
          __syncthreads();
        }
        cnt = base;
        // rank of each candidate in (-u, index) order; the first k_dm land in cols[1..]
        for (int q = tid; q < cnt; q += SM_T) {
          const int i = s.clist[q];
          const double ui = s.u[i];
          int rk = 0;
          for (int p = 0; p < cnt; ++p) {
            const int jx = s.clist[p];
            const double uj = s.u[jx];
            rk += (uj > ui) || (uj == ui && jx < i);
          }
          if (rk < a.k_dm) s.cols[1 + rk] = i;
        }
        if (tid == 0) {
          s.cols[0] = seed;
          s.kmax_c = min(cnt, a.k_dm);
        }
        __syncthreads();
      }
      SMT(2);
      const int k_max = s.kmax_c;
      const int ncand = k_max + 1;
      const int k8 = (mp + 7) & ~7;
      // ---- gather the candidate columns (rows n_s..m) into P; zero padding ----
      for (int t = wid; t < DMQR_KP; t += SM_W) {
        double* dst = s.P + t * SM_LDP;
        if (t < ncand) {
          const double* src = A + (int64_t)s.cols[t] * lda + n_s;
          double v[SM_MMAX / 32];
#pragma unroll
          for (int q = 0; q < SM_MMAX / 32; ++q) v[q] = (lane + 32 * q < mp) ? src[lane + 32 * q] : 0.0;
#pragma unroll
          for (int q = 0; q < SM_MMAX / 32; ++q)
            if (lane + 32 * q < k8) dst[lane + 32 * q] = v[q];
        } else {
          for (int r = lane; r < k8; r += 32) dst[r] = 0.0;
        }
      }
      __syncthreads();
      SMT(3);
      double gamma = 1.0;
      int nsel = 1;
      if (k_max > 0) {
        // ---- cosine matrix (dm.py:100-115) ----
        for (int t = wid; t < ncand; t += SM_W) {
          const double d = sm_norm(s.P + t * SM_LDP, mp, lane);
          if (lane == 0) s.dn[t] = d;
        }
        sm_gram(s.P, (ncand + 7) >> 3, (mp + 3) & ~3, s.G);
        __syncthreads();
        if (tid == 0) {
          for (int t = 0; t < ncand; ++t)
            if (s.dn[t] == 0.0) s.status = SM_ST_ZEROCOL;  // ValueError (dm.py:111-112)
        }
        for (int t = tid; t < ncand; t += SM_T) s.cf[t] = 1.0 / s.dn[t];  // inv (scratch in cf)
        __syncthreads();
        if (s.status) break;
        for (int e = tid; e < ncand * ncand; e += SM_T) {
          const int i = e / ncand, j = e % ncand;
          if (i < j) {
            const double th_ij = (s.G[i * SM_GLD + j] * s.cf[i]) * s.cf[j];
            s.G[i * SM_GLD + j] = th_ij;
            s.G[j * SM_GLD + i] = th_ij;
          }
        }
        __syncthreads();
        for (int t = tid; t < ncand; t += SM_T) s.G[t * SM_GLD + t] = 1.0;
        SMT(4);
        // ---- greedy delta filter (dm.py:151-177) ----
        const bool dmax = a.use_delta_max != 0;
        const double dlt = dmax ? a.tau * a.tau / (double)max(k_max - 1, 1) : a.delta;
        if (!dmax) {
          for (int t = 1 + tid; t < ncand; t += SM_T) {  // bit j: |theta_tj| >= dlt (j < t <= 64)
            unsigned long long msk = 0ull;
            for (int j = 0; j < t; ++j)
              if (!(fabs(s.G[t * SM_GLD + j]) < dlt)) msk |= 1ull << j;
            s.conf[t] = msk;
          }
        }
        __syncthreads();
        if (tid == 0) {
          int ns = 1;
          s.selt[0] = 0;
          if (!dmax) {
            unsigned long long chosen = 1ull;
            for (int t = 1; t < ncand; ++t)
              if ((s.conf[t] & chosen) == 0ull) {
                s.selt[ns++] = t;
                if (t < 64) chosen |= 1ull << t;
              }
          } else {  // delta_max: also reject when a row sum would reach tau^2 (dm.py:151-172)
            const double guard = a.tau * a.tau;
            double* rsum = s.dn;  // (norms no longer needed) rsum[t] for chosen t
            rsum[0] = 0.0;
            for (int t = 1; t < ncand; ++t) {
              bool ok = true;
              double tot = 0.0;
              for (int q = 0; q < ns; ++q) {
                const double g = fabs(s.G[t * SM_GLD + s.selt[q]]);
                if (!(g < dlt)) ok = false;
              }
              if (!ok) continue;
              for (int q = 0; q < ns; ++q) tot += fabs(s.G[t * SM_GLD + s.selt[q]]);
              if (tot >= guard) continue;
              bool rej = false;
              for (int q = 0; q < ns; ++q) {
                const int jx = s.selt[q];
                if (rsum[jx] + fabs(s.G[jx * SM_GLD + t]) >= guard) rej = true;
              }
              if (rej) continue;
              for (int q = 0; q < ns; ++q) {
                const int jx = s.selt[q];
                rsum[jx] += fabs(s.G[jx * SM_GLD + t]);
              }
              rsum[t] = tot;
              s.selt[ns++] = t;
            }
          }
          s.nsel = ns;
        }
        __syncthreads();
        nsel = s.nsel;
        // gamma = min_i 1 - (sum_j |theta_ij| - 1) over the chosen set (dm.py:174-176)
        double gmin = 1e300;
        for (int q = tid; q < nsel; q += SM_T) {
          const int i = s.selt[q];
          double sum = 0.0;
          for (int p = 0; p < nsel; ++p) sum += fabs(s.G[i * SM_GLD + s.selt[p]]);
          gmin = fmin(gmin, 1.0 - (sum - 1.0));
        }
        gmin = -sm_wmax(-gmin);
        if (lane == 0) s.red[wid] = gmin;
        __syncthreads();
        gamma = s.red[0];
        for (int w = 1; w < SM_W; ++w) gamma = fmin(gamma, s.red[w]);
        __syncthreads();
      } else {
        if (tid == 0) {
          s.selt[0] = 0;
          s.nsel = 1;
        }
        __syncthreads();
      }
      SMT(5);
      const int k_s = min(nsel, kmax - n_s);  // rrqr.py:355
      const double eps_s = a.tau * umax;      // rrqr.py:357 (before the swaps)
      // ---- swaps (rrqr.py:294-312): the transposition sequence on warp 0 ----
      if (wid == 0) {
        int pv[3];  // pos[lane + 32 q]
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int h = lane + 32 * q;
          pv[q] = (h < k_s) ? s.cols[s.selt[h]] : -1;
        }
        int nlog = s.nsw_log;
        for (int i = 0; i < k_s; ++i) {
          const int tgt = n_s + i;
          const int pq = (i >> 5) == 0 ? pv[0] : ((i >> 5) == 1 ? pv[1] : pv[2]);
          const int src = __shfl_sync(0xffffffffu, pq, i & 31);
          if (src == tgt) continue;
          if (lane == 0) {
            if (nlog < a.swap_cap) {
              swaps[2 * nlog] = tgt;
              swaps[2 * nlog + 1] = src;
            }
            const int x = s.srcof[tgt];
            s.srcof[tgt] = s.srcof[src];
            s.srcof[src] = x;
          }
          ++nlog;
          // first later pos equal to tgt -> src
          unsigned hit = 0;
          int q_hit = -1;
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int h = lane + 32 * q;
            const unsigned bq = __ballot_sync(0xffffffffu, h > i && h < k_s && pv[q] == tgt);
            if (q_hit < 0 && bq) {
              q_hit = q;
              hit = bq;
            }
          }
          if (q_hit >= 0 && lane == __ffs(hit) - 1) {
#pragma unroll
            for (int q = 0; q < 3; ++q)
              if (q == q_hit) pv[q] = src;
          }
          __syncwarp();
        }
        if (lane == 0) s.nsw_log = nlog;
      }
      __syncthreads();
      SMT(6);
      // composed moves new[dst] = old[src] over the touched positions
      if (wid == 0) {  // (ballot compaction: block positions, then selected columns outside it)
        int nm = 0;
        for (int pass = 0; pass < 2; ++pass)
          for (int h0 = 0; h0 < k_s; h0 += 32) {
            const int i = h0 + lane;
            int p = -1;
            if (i < k_s) p = pass == 0 ? n_s + i : s.cols[s.selt[i]];
            const int sp = (p >= 0) ? s.srcof[p] : -1;
            const bool mv = p >= 0 && sp != p && (pass == 0 || p >= n_s + k_s);
            const unsigned bal = __ballot_sync(0xffffffffu, mv);
            if (mv) {
              const int o = nm + __popc(bal & ((1u << lane) - 1u));
              s.mv_dst[o] = p;
              s.mv_src[o] = sp;
            }
            nm += __popc(bal);
          }
        if (lane == 0) s.nmv = nm;
      }
      __syncthreads();
      SMT(23);
      const int nmv = s.nmv;
      {  // u, u_ref, perm
        double uu[2], ur[2];
        int pp[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int e = tid + q * SM_T;
          if (e < nmv) {
            uu[q] = s.u[s.mv_src[e]];
            ur[q] = s.uref[s.mv_src[e]];
            pp[q] = s.perm[s.mv_src[e]];
          }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int e = tid + q * SM_T;
          if (e < nmv) {
            s.u[s.mv_dst[e]] = uu[q];
            s.uref[s.mv_dst[e]] = ur[q];
            s.perm[s.mv_dst[e]] = pp[q];
            s.srcof[s.mv_dst[e]] = s.mv_dst[e];
          }
        }
      }
      SMT(24);
      // column data.  Rows >= n_s: only the moves out of the block write there
      // (the block's rows >= n_s come from the panel), reading block columns
      // nobody writes in this phase: direct copies.  Rows < n_s (R rows of
      // earlier steps): every move; 32-row chunks, all reads of a chunk (24 per
      // thread in flight) before its writes.
      for (int q = wid; q < nmv; q += SM_W) {
        if (s.mv_dst[q] < n_s + k_s) continue;
        const double* src = A + (int64_t)s.mv_src[q] * lda;
        double* dst = A + (int64_t)s.mv_dst[q] * lda;
        double v[SM_MMAX / 32];
#pragma unroll
        for (int k = 0; k < SM_MMAX / 32; ++k) {
          const int r = n_s + lane + 32 * k;
          v[k] = (r < m) ? src[r] : 0.0;
        }
#pragma unroll
        for (int k = 0; k < SM_MMAX / 32; ++k) {
          const int r = n_s + lane + 32 * k;
          if (r < m) dst[r] = v[k];
        }
      }
      for (int r0 = 0; r0 < n_s; r0 += 32) {
        const int r = r0 + lane;
        double v[24];
#pragma unroll
        for (int k = 0; k < 24; ++k) {
          const int q = wid + SM_W * k;
          v[k] = (q < nmv && r < n_s) ? A[(int64_t)s.mv_src[q] * lda + r] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 24; ++k) {
          const int q = wid + SM_W * k;
          if (q < nmv && r < n_s) A[(int64_t)s.mv_dst[q] * lda + r] = v[k];
        }
        __syncthreads();
      }
      __syncthreads();
      SMT(25);
      SMT(7);
      // ---- panel columns in selection order (candidate t_i -> slot i; t_i >= i, increasing) ----
      for (int r = tid; r < k8; r += SM_T)
        for (int i = 1; i < k_s; ++i) {
          const int t = s.selt[i];
          if (t != i) s.P[i * SM_LDP + r] = s.P[t * SM_LDP + r];
        }
      __syncthreads();
      SMT(8);
      // ---- panel: reflectors with the QRDM2 break (rrqr.py:360-379), register-resident ----
      const int l = sm_panel_regs(s, k_s, mp, eps_s, a.break_check, (a.dbg && blockIdx.x == 0 && b == 0 && step == 0) ? a.dbg : nullptr);
      __syncthreads();
      SMT(9);
      // ---- write the panel back (R + v for accepted columns, updated rejected ones) ----
      for (int c = wid; c < k_s; c += SM_W) {
        double* dst = A + (int64_t)(n_s + c) * lda + n_s;
        const double* src = s.P + c * SM_LDP;
        for (int r = lane; r < mp; r += 32) dst[r] = src[r];
      }
      for (int j = tid; j < l; j += SM_T) coeffs[n_s + j] = s.cf[j];
      const int tc0 = n_s + k_s;
      const bool trail = tc0 < n;
      __syncthreads();
      SMT(10);
      if (trail) {
        // ---- Y (unit lower) in P, zero past column l; W = T (accumulate_wy) in G ----
        for (int e = tid; e < DMQR_KP * k8; e += SM_T) {
          const int j = e / k8, r = e % k8;
          double* p = s.P + j * SM_LDP + r;
          if (j >= l || r < j) *p = 0.0;
          else if (r == j) *p = 1.0;
        }
        for (int e = tid; e < DMQR_KP * SM_GLD; e += SM_T) s.G[e] = 0.0;
        __syncthreads();
        const int lt = (l + 7) >> 3;
        sm_gram(s.P, lt, (mp + 3) & ~3, s.G);  // S = Y^T Y (upper tiles)
        __syncthreads();
        SMT(11);
        // W[:j, j] = -coeff_j W[:j, :j] S[:j, j]; W[j, j] = coeff_j (householder.py:105-113),
        // blocked by 8: the diagonal blocks by the recurrence (a warp each), then
        // block column J: W[:8J, J] = -W[:8J, :8J] (S[:8J, J] W_JJ)
        for (int bk = wid; bk < lt; bk += SM_W) {
          const int i = 8 * bk + (lane & 7);
          for (int j = 8 * bk; j < min(8 * bk + 8, l); ++j) {
            double sum = 0.0;
            if (lane < 8 && i < j)
              for (int t = i; t < j; ++t) sum = fma(s.G[i * SM_GLD + t], s.G[t * SM_GLD + j], sum);
            __syncwarp();
            if (lane < 8 && i < j) s.G[i * SM_GLD + j] = -s.cf[j] * sum;
            if (lane == 0) s.G[j * SM_GLD + j] = s.cf[j];
            __syncwarp();
          }
        }
        __syncthreads();
        double* X = s.G + DMQR_KP;  // scratch columns 72..79 of G's rows
        for (int J = 1; J < lt; ++J) {
          const int nb = min(8, l - 8 * J), r8 = 8 * J;
          for (int e = tid; e < r8 * 8; e += SM_T) {  // X = S[:8J, J] W_JJ
            const int i = e >> 3, c = e & 7;
            double x = 0.0;
            if (c < nb)
              for (int t = 0; t <= c; ++t) x = fma(s.G[i * SM_GLD + r8 + t], s.G[(r8 + t) * SM_GLD + r8 + c], x);
            X[i * SM_GLD + c] = x;
          }
          __syncthreads();
          for (int e = tid; e < r8 * 8; e += SM_T) {  // W[:8J, J] = -W[:8J, :8J] X
            const int i = e >> 3, c = e & 7;
            if (c < nb) {
              double x = 0.0;
              for (int t = i; t < r8; ++t) x = fma(s.G[i * SM_GLD + t], X[t * SM_GLD + c], x);
              s.G[i * SM_GLD + r8 + c] = -x;
            }
          }
          __syncthreads();
        }
        for (int e = tid; e < DMQR_KP * DMQR_KP; e += SM_T) {  // strict lower (S values) -> 0
          const int i = e / DMQR_KP, j = e % DMQR_KP;
          if (j < i) s.G[i * SM_GLD + j] = 0.0;
        }
        __syncthreads();
        SMT(12);
        // ---- C <- C - Y W^T Y^T C on the trailing columns, warp per 8-column tile ----
        const int64_t ncend = n;
        for (int64_t c0 = tc0 + 8 * wid; c0 < n; c0 += 8 * SM_W) sm_trail(lt, A, lda, n_s, mp, l, c0, ncend, s.P, s.G);
        __syncthreads();
      }
      SMT(13);
      // ---- norms (rrqr.py:161-186) and the step record ----
      sm_downdate(a, A, lda, m, n, n_s, n_s + l, s);
      if (tid == 0) {
        StepRec rec;
        rec.n_s = n_s;
        rec.k_selected = k_s;
        rec.k_accepted = l;
        rec.k_max = k_max;
        rec.broke_early = (l < k_s);
        rec.fell_back_to_scalar = 0;
        rec.eps_s = eps_s;
        rec.gamma = gamma;
        steps[step] = rec;
      }
      __syncthreads();
      n_s += l;
      ++step;
      SMT(14);
    }
    __syncthreads();
    // ---- rank / n_factored (rrqr.py:406-412; StopRule.NONE: _posthoc_rank 206-208) ----
    const int nf = stopped ? n_s : min(n_s, kmax);
    int cnt = 0;
    if (a.stop_none && !stopped) {
      const double thr = kEps * (double)n * a0;
      for (int i = tid; i < nf; i += SM_T) cnt += fabs(A[(int64_t)i * lda + i]) > thr;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) s.redi[wid] = cnt;
    __syncthreads();
    for (int j = tid; j < n; j += SM_T) a.perm[b * n + j] = s.perm[j];
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < SM_W; ++w) tot += s.redi[w];
      SmallInfo inf;
      inf.rank = (kmax == 0) ? 0 : (stopped ? n_s : (a.stop_none ? tot : nf));
      inf.n_factored = (kmax == 0) ? 0 : nf;
      inf.n_steps = (kmax == 0) ? 0 : step;
      inf.n_swaps = s.nsw_log;
      inf.stopped = stopped ? 1 : 0;
      inf.status = s.status ? s.status : ((s.nsw_log > a.swap_cap) ? SM_ST_CAP : 0);
      inf.a_max0 = a0;
      a.info[b] = inf;
    }
    __syncthreads();
  }
}

}  // namespace dmqr
