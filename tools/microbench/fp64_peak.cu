// FP64 peak microbenchmarks for the roofline denominators (SURVEY §8(d) asks
// for both the DFMA and the DMMA rate to be measured on the box).
//   dfma: 8 independent FMA chains per thread, grid = 148 * 8 CTAs of 256 threads
//   dmma: mma.sync.aligned.m8n8k4.row.col.f64, 4 independent accumulators per warp
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double s) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double m = 1.0000001;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, m, s); a1 = fma(a1, m, s); a2 = fma(a2, m, s); a3 = fma(a3, m, s);
      a4 = fma(a4, m, s); a5 = fma(a5, m, s); a6 = fma(a6, m, s); a7 = fma(a7, m, s);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.5 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma(c[u][0], c[u][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * 148 * 64 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps_per_sm : {8, 16, 32}) {
    const int blocks = nsm * warps_per_sm / 8, threads = 256, iters = 4096;
    dfma_kernel<<<blocks, threads>>>(out, 16, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1e-9);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("{\"probe\":\"dfma\",\"warps_per_sm\":%d,\"tflops\":%.3f}\n", warps_per_sm,
           flops / ms / 1e9);
  }
  for (int warps_per_sm : {4, 8, 16, 32}) {
    const int blocks = nsm * warps_per_sm / 4, threads = 128, iters = 4096;
    dmma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    printf("{\"probe\":\"dmma\",\"warps_per_sm\":%d,\"tflops\":%.3f}\n", warps_per_sm,
           flops / ms / 1e9);
  }
  printf("{\"sms\":%d,\"clock_khz\":%d,\"err\":\"%s\"}\n", nsm, clk,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
