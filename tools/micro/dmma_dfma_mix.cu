// Microbenchmark: do DMMA.8x8x4 and DFMA share one datapath on this GPU?  Warps of a CTA run
// DMMA only, DFMA only, or both (half the warps each / interleaved in every warp).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
// mode 0: all warps DMMA; 1: all warps DFMA; 2: even warps DMMA, odd warps DFMA; 3: every warp interleaves
__global__ void k_mix(double* out, int iters, int mode) {
  double c[8][2], x[8];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int q = 0; q < 8; ++q) { c[q][0] = c[q][1] = q; x[q] = threadIdx.x + q; }
  const double fa = 1.0000001, fb = 1e-9;
  const int w = threadIdx.x >> 5;
  const bool do_mma = mode == 0 || mode == 3 || (mode == 2 && (w & 1) == 0);
  const bool do_fma = mode == 1 || mode == 3 || (mode == 2 && (w & 1) == 1);
  if (do_mma && do_fma) {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        dmma884(c[q][0], c[q][1], a, b);
#pragma unroll
        for (int r = 0; r < 4; ++r) x[(2 * q + r) & 7] = fma(x[(2 * q + r) & 7], fa, fb);  // 32 DFMA per 8 DMMA
      }
    }
  } else if (do_mma) {
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int q = 0; q < 8; ++q) dmma884(c[q][0], c[q][1], a, b);
  } else {
    for (int i = 0; i < iters; ++i)
#pragma unroll
      for (int q = 0; q < 32; ++q) x[q & 7] = fma(x[q & 7], fa, fb);
  }
  double s = 0;
  for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1] + x[q];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {8, 16, 32}) {
    for (int mode = 0; mode < 4; ++mode) {
      dim3 g(sms), b(32 * warps);
      k_mix<<<g, b>>>(d, 16, mode); cudaDeviceSynchronize();
      cudaEventRecord(e0); k_mix<<<g, b>>>(d, iters, mode); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      // per warp per iteration: DMMA 8 x 512 flops; DFMA 32 x 64 flops (per warp: 32 lanes x 2)
      double nw = (double)g.x * warps;
      double f_mma = 0, f_fma = 0;
      if (mode == 0) f_mma = nw * iters * 8 * 512.0;
      if (mode == 1) f_fma = nw * iters * 32 * 64.0;
      if (mode == 2) { f_mma = nw / 2 * iters * 8 * 512.0; f_fma = nw / 2 * iters * 32 * 64.0; }
      if (mode == 3) { f_mma = nw * iters * 8 * 512.0; f_fma = nw * iters * 32 * 64.0; }
      printf("warps/SM=%2d mode=%d : %.3f ms  DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", warps, mode, ms,
             f_mma / (ms * 1e-3) / 1e12, f_fma / (ms * 1e-3) / 1e12, (f_mma + f_fma) / (ms * 1e-3) / 1e12);
    }
  }
  return 0;
}
