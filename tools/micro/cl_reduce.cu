// Microbenchmark: cluster all-reduce of the CholeskyQR2 panel's 65 x 65 Gram
// over a 16-CTA cluster (tools only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2106_03138_b200/csrc tools/micro/cl_reduce.cu -o tools/micro/cl_reduce
#include <cstdio>
#include "panel_cq.cuh"
using namespace dmqr;

template <int V>
__global__ void __launch_bounds__(PANEL_T, 1) k_red(long long* cyc, double* out, int k) {
  extern __shared__ __align__(16) double sm[];
  double* part = sm;
  double* tot = sm + DMQR_KP * DMQR_KP;
  cg::cluster_group cl = cg::this_cluster();
  const int me = (int)cl.block_rank();
  for (int e = threadIdx.x; e < DMQR_KP * DMQR_KP; e += blockDim.x) part[e] = me + e * 1e-3;
  if (threadIdx.x == 0 && me == 0) cyc[2] = 0;
  cl.sync();
  long long t0 = clock64();
  for (int r = 0; r < 10; ++r) cl.sync();
  long long t1 = clock64();
  for (int r = 0; r < 10; ++r) cq_cluster_reduce(part, tot, k);
  // check: tot upper == sum over ranks of (q + e 1e-3) in rank order, lower untouched (-1)
  for (int e = threadIdx.x; e < DMQR_KP * DMQR_KP; e += blockDim.x) tot[e] = -1.0;
  cl.sync();
  cq_cluster_reduce(part, tot, k);
  if (me == 0)
    for (int e = threadIdx.x; e < DMQR_KP * DMQR_KP; e += blockDim.x) {
      const int i = e / DMQR_KP, j = e % DMQR_KP;
      double want = -1.0;
      if (j >= i && i < (k + 7) / 8 * 8 && j < (k + 7) / 8 * 8) {
        want = 0.0;
        for (int q = 0; q < (int)cl.num_blocks(); ++q) want += q + e * 1e-3;
      }
      if (tot[e] != want) atomicAdd((unsigned long long*)&cyc[2], 1ull);
    }
  long long t2 = clock64();
  if (threadIdx.x == 0 && me == 0) {
    cyc[0] = (t1 - t0) / 10;
    cyc[1] = (t2 - t1) / 10;
  }
  if (me == 0)
    for (int e = threadIdx.x; e < DMQR_KP * DMQR_KP; e += blockDim.x) out[e] = tot[e];
}

int main() {
  long long* dc;
  double* dout;
  cudaMalloc(&dc, 64);
  cudaMemset(dc, 0, 64);
  cudaMalloc(&dout, 8 * DMQR_KP * DMQR_KP);
  size_t smem = 2 * 8 * DMQR_KP * DMQR_KP;
  cudaFuncSetAttribute(k_red<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_red<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int nr : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nr);
    cfg.blockDim = dim3(PANEL_T);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = nr;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_red<0>, dc, dout, 65);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    long long c[3];
    cudaMemcpy(c, dc, 24, cudaMemcpyDeviceToHost);
    printf("nr %2d: cluster.sync %lld cycles, cq_cluster_reduce(65) %lld cycles, mismatches %lld\n", nr, c[0], c[1], c[2]);
    cudaMemset(dc, 0, 64);
  }
  return 0;
}
