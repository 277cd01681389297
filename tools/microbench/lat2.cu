// Dependent-chain latencies of the primitives on the sweep GJ's critical path.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  double x = 1.0 + lane * 1e-3;
  sm[lane] = x; sm[32 + lane] = x;
  __syncwarp();
  long long t0, t1;
  // shfl chain (double)
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  t1 = clock64(); if (lane == 0) cyc[0] = (t1 - t0) / n;
  // rcp.approx f64 chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(x));
  t1 = clock64(); if (lane == 0) cyc[1] = (t1 - t0) / n;
  // dfma chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999, 1e-3);
  t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0) / n;
  // lds chain (address depends on loaded value)
  int idx = lane;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { double v = sm[idx & 63]; idx = int(v) + lane; }
  t1 = clock64(); if (lane == 0) cyc[3] = (t1 - t0) / n;
  // sts -> syncwarp -> lds round trip
  t0 = clock64();
  for (int i = 0; i < n; ++i) { sm[lane] = x; __syncwarp(); x = sm[(lane + 1) & 31] * 1.0000001; __syncwarp(); }
  t1 = clock64(); if (lane == 0) cyc[4] = (t1 - t0) / n;
  // IEEE double division chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x;
  t1 = clock64(); if (lane == 0) cyc[5] = (t1 - t0) / n;
  // dmul chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * 1.0000001;
  t1 = clock64(); if (lane == 0) cyc[6] = (t1 - t0) / n;
  out[lane] = x + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  k<<<1, 32>>>(o, c, 64); k<<<1, 32>>>(o, c, 1024);
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* nm[] = {"shfl.f64 (2x SHFL)", "rcp.approx.f64 (MUFU.RCP64H)", "dfma", "lds.64 (dependent addr)",
                      "sts+syncwarp+lds", "IEEE 1/x", "dmul"};
  for (int i = 0; i < 7; ++i) printf("%-32s %lld cycles\n", nm[i], h[i]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
