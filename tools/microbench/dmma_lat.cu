// DMMA.8x8x4 dependent-chain latency and per-warp throughput vs independent chains.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int iters) {
  double c[CH][2] = {};
  const double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int u = 0; u < CH; ++u) dmma(c[u][0], c[u][1], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int u = 0; u < CH; ++u) s += c[u][0] + c[u][1];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0);
}
__global__ void dfma_lat(double* out, long long* cyc, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-9);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 1024);
  const int it = 4096;
#define RUN(CH) k<CH><<<1, 32>>>(out, cyc, 16); k<CH><<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); \
  printf("1 warp, %d chains: %.1f cycles per DMMA (per chain step %.1f)\n", CH, double(h) / (it * CH), double(h) / it);
  RUN(1) RUN(2) RUN(4) RUN(8)
  k<4><<<1, 128>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("4 warps (1/SMSP), 4 chains each: %.1f cycles per chain step\n", double(h) / it);
  k<4><<<1, 256>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("8 warps (2/SMSP), 4 chains each: %.1f cycles per chain step\n", double(h) / it);
  dfma_lat<<<1, 32>>>(out, cyc, 16); dfma_lat<<<1, 32>>>(out, cyc, it); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", double(h) / it);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
