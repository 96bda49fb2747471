// Microbenchmark: DMMA.8x8x4 and DFMA throughput per SM on this GPU (tools only).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k_dmma(double* out, int iters) {
  double c[CH][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int q = 0; q < CH; ++q) c[q][0] = c[q][1] = q;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int q = 0; q < CH; ++q) dmma884(c[q][0], c[q][1], a, b);
  }
  double s = 0;
  for (int q = 0; q < CH; ++q) s += c[q][0] + c[q][1];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double x[8];
  for (int q = 0; q < 8; ++q) x[q] = threadIdx.x + q;
  const double a = 1.0000001, b = 1e-9;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
  double s = 0;
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    for (int ch : {4, 8, 16}) {
      dim3 g(sms * 2), b(32 * warps / 2);
      auto run = [&](auto kern) {
        kern<<<g, b>>>(d, 16); cudaDeviceSynchronize();
        cudaEventRecord(e0); kern<<<g, b>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
      };
      float ms = (ch == 4) ? run(k_dmma<4>) : (ch == 8) ? run(k_dmma<8>) : run(k_dmma<16>);
      double flops = 2.0 * 256 * ch * (double)iters * g.x * (b.x / 32);
      printf("DMMA warps/SM=%2d chains=%2d : %.2f TFLOP/s\n", warps, ch, flops / (ms * 1e-3) / 1e12);
    }
  }
  for (int warps : {8, 16, 32, 64}) {
    dim3 g(sms * 2), b(32 * warps / 2);
    k_dfma<<<g, b>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(e0); k_dfma<<<g, b>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * g.x * b.x;
    printf("DFMA warps/SM=%2d : %.2f TFLOP/s\n", warps, flops / (ms * 1e-3) / 1e12);
  }
  return 0;
}
