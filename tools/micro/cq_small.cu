// Microbenchmark: cycles of the CholeskyQR2 panel's small dense helpers
// (panel_cq.cuh) on one CTA of 512 threads, k = 65 (tools only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2106_03138_b200/csrc tools/micro/cq_small.cu -o tools/micro/cq_small
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
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
  const int reps = 8;
  long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int rep = 0; rep < reps; ++rep) {
    // chol
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += blockDim.x) A1[e] = G[e];
    __syncthreads();
    t0 = clock64();
    int jf = cq_chol(A1, A2, vpiv, vpiv + DMQR_KP, k, 1e-10);
    __syncthreads();
    t1 = clock64();
    acc[0] += t1 - t0;
    if (rep == 0 && tid == 0) out[0] = jf;
    // trinv of R (A2) -> A1
    t0 = clock64();
    cq_trinv_upper(A2, A1, k);
    __syncthreads();
    t1 = clock64();
    acc[1] += t1 - t0;
    // mLU of Qt
    for (int e = tid; e < DMQR_KP * DMQR_KP; e += blockDim.x) A1[e] = Qt[e];
    __syncthreads();
    t0 = clock64();
    cq_mlu(A1, vS, vpiv, k);
    __syncthreads();
    t1 = clock64();
    acc[2] += t1 - t0;
    // small gemm upper x upper
    t0 = clock64();
    cq_small_gemm([&](int i, int t) { return A2[i * DMQR_KP + t]; }, [&](int t, int j) { return A2[t * DMQR_KP + j]; },
                  out + 16, k);
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
}

int main() {
  const int k = 65, R = 256;
  std::vector<double> P((size_t)k * R), G(DMQR_KP * DMQR_KP, 0.0), Qt(DMQR_KP * DMQR_KP, 0.0);
  srand(1);
  for (auto& x : P) x = (rand() / (double)RAND_MAX) - 0.5;
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
  cudaMalloc(&dout, 16 * 8 + DMQR_KP * DMQR_KP * 8);
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
  double o;
  cudaMemcpy(c, dc, sizeof(c), cudaMemcpyDeviceToHost);
  cudaMemcpy(&o, dout, 8, cudaMemcpyDeviceToHost);
  printf("chol %lld trinv %lld mlu %lld small_gemm %lld gram(256) %lld slice_gemm(256) %lld sync x100 %lld  (chol ret %g)\n",
         c[0], c[1], c[2], c[3], c[4], c[5], c[6], o);
  return 0;
}
