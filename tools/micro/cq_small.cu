// Microbenchmark: cycles of the CholeskyQR2 panel's small dense helpers
// (panel_cq.cuh) on one CTA of 512 threads, k = 65 (tools only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2106_03138_b200/csrc tools/micro/cq_small.cu -o tools/micro/cq_small
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
__device__ __forceinline__ long long* tick_buf() {
  __shared__ long long tb[18];
  return tb;
}
#define CQ_TICK(i)                             \
  do {                                         \
    if (threadIdx.x == 0) {                    \
      long long* tb_ = tick_buf();             \
      const long long t_ = clock64();          \
      tb_[i] += t_ - tb_[17];                  \
      tb_[17] = t_;                            \
    }                                          \
  } while (0)
#define CQ_TICK0()                                   \
  do {                                               \
    if (threadIdx.x == 0) tick_buf()[17] = clock64(); \
  } while (0)
#include "panel_cq.cuh"

using namespace dmqr;


__global__ void __launch_bounds__(PANEL_T, 1) k_bench(const double* G, const double* Qt, const double* P, int k, int R,
                                                      long long* cyc, double* out) {
  extern __shared__ __align__(16) double sm[];
  double* sl = sm;
  double* A1 = sl + CQ_KC * CQ_LDS;
  double* A2 = A1 + DMQR_KP * DMQR_KP;
  double* vpiv = A2 + DMQR_KP * DMQR_KP;
  double* vS = vpiv + 2 * DMQR_KP;
  const int tid = threadIdx.x;
  long long t0, t1;
  for (int e = tid; e < k * CQ_LDS; e += blockDim.x) sl[e] = (e % CQ_LDS < R) ? P[(e / CQ_LDS) * R + e % CQ_LDS] : 0.0;
  for (int j = tid; j < k; j += blockDim.x) vpiv[DMQR_KP + j] = G[j * DMQR_KP + j];
  __syncthreads();
  const int reps = 64;
  if (tid < 18) tick_buf()[tid] = 0;
  long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int rep = 0; rep < reps; ++rep) {
    // chol
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += blockDim.x) A1[e] = G[e];
    __syncthreads();
    CQ_TICK0();
    t0 = clock64();
    int jf = cq_chol(A1, A2, vpiv, vpiv + DMQR_KP, k, 1e-10);
    __syncthreads();
    t1 = clock64();
    acc[0] += t1 - t0;
    if (rep == 0 && tid == 0) out[0] = jf;
    if (rep == 0)
      for (int e = tid; e < DMQR_KP * DMQR_KP; e += blockDim.x) out[64 + DMQR_KP * DMQR_KP + e] = A2[e];
    // trinv of R (A2) -> A1
    CQ_TICK0();
    t0 = clock64();
    cq_trinv_upper(A2, A1, k);
    __syncthreads();
    t1 = clock64();
    acc[1] += t1 - t0;
    // mLU of Qt
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += blockDim.x) A1[e] = Qt[e];
    __syncthreads();
    CQ_TICK0();
    t0 = clock64();
    cq_mlu<DMQR_KP>(A1, vS, vpiv, k);
    __syncthreads();
    t1 = clock64();
    acc[2] += t1 - t0;
    // the same LU with an odd row stride (73) on a copy; compare
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += blockDim.x) A2[e] = A1[e];  // cq_mlu result
    for (int e = tid; e < DMQR_KP * (DMQR_KP + 1); e += blockDim.x) {
      const int i = e / (DMQR_KP + 1), j = e % (DMQR_KP + 1);
      sl[e] = (j < DMQR_KP) ? Qt[i * DMQR_KP + j] : 0.0;
    }
    __syncthreads();
    t0 = clock64();
    cq_mlu<DMQR_KP + 1>(sl, vS + DMQR_KP, vpiv + DMQR_KP, k);
    __syncthreads();
    t1 = clock64();
    acc[7] += t1 - t0;
    if (rep == 0) {
      for (int e = tid; e < k * DMQR_KP; e += blockDim.x) {
        const int i = e / DMQR_KP, j = e % DMQR_KP;
        if (j < k && sl[i * (DMQR_KP + 1) + j] != A2[e]) atomicAdd((unsigned long long*)&out[2], 1ull);
      }
    }
    // small gemm upper x upper
    t0 = clock64();
    cq_small_gemm([&](int i, int t) { return A2[i * DMQR_KP + t]; }, [&](int t, int j) { return A2[t * DMQR_KP + j]; },
                  out + 64, k);
    __syncthreads();
    t1 = clock64();
    acc[3] += t1 - t0;
    // gram over R rows
    t0 = clock64();
    cq_gram(sl, (R + 3) & ~3, k, A1);
    __syncthreads();
    t1 = clock64();
    acc[4] += t1 - t0;
    // slice gemm (in place, upper M = A2)
    t0 = clock64();
    cq_slice_gemm(sl, (R + 3) & ~3, k, k, A2);
    __syncthreads();
    t1 = clock64();
    acc[5] += t1 - t0;
    // bare syncthreads x 100
    t0 = clock64();
    for (int q = 0; q < 100; ++q) __syncthreads();
    t1 = clock64();
    acc[6] += t1 - t0;
  }
  if (tid == 0)
    for (int q = 0; q < 8; ++q) cyc[q] = acc[q] / reps;
  if (tid == 0) {
    // every helper call also ticks: subtract nothing, report the raw sums / reps
    for (int q = 0; q < 16; ++q) out[32 + q] = (double)tick_buf()[q] / reps;
  }
}


// dependent-chain latencies (single warp)
__global__ void k_lat(double* out, long long* cyc, double x0) {
  double x = x0 + threadIdx.x * 1e-9;
  long long t0, t1;
  const int N = 256;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = fma(x, 1.0000001, 1e-12);
  t1 = clock64();
  cyc[0] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  t1 = clock64();
  cyc[1] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = rsqrt(x) + 0.5;
  t1 = clock64();
  cyc[2] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 1.0);
  t1 = clock64();
  cyc[3] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < N; ++i) x = cq_rsqrt(x) + 0.5;
  t1 = clock64();
  cyc[4] = (t1 - t0) / N;
  __shared__ double sh[64];
  sh[threadIdx.x] = x;
  __syncwarp();
  int idx = threadIdx.x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) { x = sh[idx]; idx = ((int)x) & 31; }
  t1 = clock64();
  cyc[5] = (t1 - t0) / N;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) x = x * 1.0000001;
  t1 = clock64();
  cyc[6] = (t1 - t0) / N;
  double c0 = x, c1 = x;
  t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N; ++i) dmma884(c0, c1, 1.0000001, 0.999999);
  t1 = clock64();
  cyc[7] = (t1 - t0) / N;
  x += c0 + c1;
  if (x == 1.2345) out[0] = x;
}

int main() {
  const int k = 65, R = 256;
  std::vector<double> P((size_t)k * R), G(DMQR_KP * DMQR_KP, 0.0), Qt(DMQR_KP * DMQR_KP, 0.0);
  srand(1);
  for (size_t e = 0; e < P.size(); ++e) P[e] = ((rand() / (double)RAND_MAX) - 0.5) * pow(10.0, -4.0 * (double)(e / R) / k);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      double s = 0;
      for (int r = 0; r < R; ++r) s += P[(size_t)i * R + r] * P[(size_t)j * R + r];
      G[i * DMQR_KP + j] = s;
    }
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) Qt[i * DMQR_KP + j] = 0.1 * ((rand() / (double)RAND_MAX) - 0.5) + (i == j ? 0.5 : 0.0);
  double *dG, *dQ, *dP, *dout;
  long long* dc;
  cudaMalloc(&dG, G.size() * 8);
  cudaMalloc(&dQ, Qt.size() * 8);
  cudaMalloc(&dP, P.size() * 8);
  cudaMalloc(&dout, 64 * 8 + 2 * DMQR_KP * DMQR_KP * 8);
  cudaMalloc(&dc, 8 * 8);
  cudaMemcpy(dG, G.data(), G.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Qt.data(), Qt.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CQ_SMEM);
  k_bench<<<1, PANEL_T, CQ_SMEM>>>(dG, dQ, dP, k, R, dc, dout);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(e));
    return 1;
  }
  long long c[8];
  double o, o3[3];
  cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
  cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost);
  double tk[16];
  cudaMemcpy(tk, dout + 32, sizeof(tk), cudaMemcpyDeviceToHost);
  printf("ticks/rep:");
  for (int q = 0; q < 16; ++q) printf(" %.0f", tk[q]);
  printf("\n");
  k_lat<<<1, 32>>>(dout, dc, 0.75);
  cudaDeviceSynchronize();
  long long l[8];
  cudaMemcpy(l, dc, sizeof(l), cudaMemcpyDeviceToHost);
  cudaMemcpy(l, dc, sizeof(l), cudaMemcpyDeviceToHost);
  printf("latency: dfma %lld shfl %lld rsqrt %lld div %lld cq_rsqrt %lld lds-chain %lld dmul %lld dmma %lld\n", l[0], l[1], l[2], l[3], l[4], l[5], l[6], l[7]);
  unsigned long long nbad;
  cudaMemcpy(&nbad, dout + 2, 8, cudaMemcpyDeviceToHost);
  printf("mlu(ld 73) %lld cycles, mismatches vs cq_mlu %llu\n", c[7], nbad);
  printf("chol %lld trinv %lld mlu %lld small_gemm %lld gram(256) %lld slice_gemm(256) %lld sync x100 %lld  (chol ret %g)\n",
         c[0], c[1], c[2], c[3], c[4], c[5], c[6], o);
  // CPU Cholesky of G, compare with the device R
  std::vector<double> Rc(DMQR_KP * DMQR_KP, 0.0), Ag(G), Rd(DMQR_KP * DMQR_KP);
  for (int j = 0; j < k; ++j) {
    double d = Ag[j * DMQR_KP + j];
    for (int t = 0; t < j; ++t) d -= Rc[t * DMQR_KP + j] * Rc[t * DMQR_KP + j];
    Rc[j * DMQR_KP + j] = sqrt(d);
    for (int c = j + 1; c < k; ++c) {
      double s = Ag[j * DMQR_KP + c];
      for (int t = 0; t < j; ++t) s -= Rc[t * DMQR_KP + j] * Rc[t * DMQR_KP + c];
      Rc[j * DMQR_KP + c] = s / Rc[j * DMQR_KP + j];
    }
  }
  cudaMemcpy(Rd.data(), dout + 64 + DMQR_KP * DMQR_KP, Rd.size() * 8, cudaMemcpyDeviceToHost);
  double worst = 0;
  int wi = -1, wj = -1;
  for (int i = 0; i < k; ++i)
    for (int j = i; j < k; ++j) {
      double e = fabs(Rd[i * DMQR_KP + j] - Rc[i * DMQR_KP + j]) / fabs(Rc[j * DMQR_KP + j]);
      if (e > worst) { worst = e; wi = i; wj = j; }
    }
  printf("chol vs cpu: worst rel err %.3g at (%d,%d)  dev %.17g cpu %.17g\n", worst, wi, wj, Rd[wi * DMQR_KP + wj], Rc[wi * DMQR_KP + wj]);
  return 0;
}
