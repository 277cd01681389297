// Latency of the warp-register sweep Gauss-Jordan inverse (kernels_condense2.cuh).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1305_1489_b200/csrc/kernels_condense2.cuh"
using namespace hdgb;

template <int N>
__global__ void gj_kernel(double* out, long long* cyc, int reps, int dmma_warps) {
  __shared__ __align__(16) double stage[128 * 8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp >= int(blockDim.x / 32) - dmma_warps) {  // background DMMA load
    double c[8][2] = {};
    const double a = 1.0 + lane * 1e-3, b = 0.5;
    for (int r = 0; r < reps * 400; ++r)
#pragma unroll
      for (int u = 0; u < 8; ++u) dmma(c[u][0], c[u][1], a, b);
    double s = 0;
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    return;
  }
  double a[N];
  for (int i = 0; i < N; ++i) a[i] = (i == lane ? 4.0 * N : 0.0) + 1.0 / (1.0 + i + lane);
  double pmin = 1e300, pmax = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    warp_gj_inverse<N>(a, stage + warp * 128, lane, pmin, pmax);
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 8 + warp] = (t1 - t0) / reps;
  double s = 0;
  for (int i = 0; i < N; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + pmin + pmax;
}

// same inversion under a 512-thread launch bound (<= 128 registers), as in the condense kernel
template <int N>
__global__ void __launch_bounds__(512) gj_kernel_lb(double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double stage[16 * 128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a[N];
  for (int i = 0; i < N; ++i) a[i] = (i == lane ? 4.0 * N : 0.0) + 1.0 / (1.0 + i + lane);
  double pmin = 1e300, pmax = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) warp_gj_inverse<N>(a, stage + warp * 128, lane, pmin, pmax);
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 8 + (warp & 7)] = (t1 - t0) / reps;
  double s = 0;
  for (int i = 0; i < N; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + pmin + pmax;
}

// condense-like: 16 warps, `active` of them invert an SPD matrix held in shared
// memory (LD-strided, lower part read, full inverse written back), as P3 does
template <int N, int LD>
__global__ void __launch_bounds__(512) gj_kernel_smem(double* out, long long* cyc, int reps, int active) {
  __shared__ __align__(16) double stage[16 * 128];
  __shared__ double Sm[4][24 * LD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < active) {
    double* S = Sm[warp & 3];
    for (int i = lane; i < 24 * LD; i += 32) S[i] = 0.0;
    __syncwarp();
    if (lane < N)
      for (int i = 0; i < N; ++i) S[i + lane * LD] = (i == lane ? 4.0 * N : 0.0) + 1.0 / (1.0 + i + lane);
    __syncwarp();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      double a[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int rr = i > lane ? i : lane, c = i > lane ? lane : i;
        a[i] = lane < N ? S[rr + c * LD] : 0.0;
      }
      double pmin = 1e300, pmax = 0;
      warp_gj_inverse<N>(a, stage + warp * 128, lane, pmin, pmax);
      if (lane < N) {
#pragma unroll
        for (int i = 0; i < N; ++i) S[i + lane * LD] = a[i];
      }
      __syncwarp();
      if (pmin < 0) out[0] = pmax;
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 8 + (warp & 7)] = (t1 - t0) / reps;
  }
  __syncthreads();
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 148 * 256 * 8); cudaMalloc(&cyc, 148 * 8 * 8);
  long long h[148 * 8];
  for (int warps : {1, 4, 8}) {
    gj_kernel<20><<<148, 32 * warps>>>(out, cyc, 4, 0);
    gj_kernel<20><<<148, 32 * warps>>>(out, cyc, 32, 0);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("N=20 warps/SM=%d: %lld cycles per inverse\n", warps, h[0]);
  }
  for (int dw : {4, 8, 12}) {
    gj_kernel<20><<<148, 32 * (4 + dw)>>>(out, cyc, 32, dw);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("N=20 4 GJ warps + %d DMMA warps: %lld cycles per inverse\n", dw, h[0]);
  }
  for (int warps : {4, 8}) {
    gj_kernel_lb<20><<<148, 32 * warps>>>(out, cyc, 32);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("N=20 (launch bound 512) warps/SM=%d: %lld cycles per inverse\n", warps, h[0]);
  }
  for (int act : {1, 4}) {
    gj_kernel_smem<20, 28><<<148, 512>>>(out, cyc, 32, act);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("N=20 from/to smem, 512-thread CTA, %d active warps: %lld cycles per inverse\n", act, h[0]);
  }
  gj_kernel<10><<<148, 32>>>(out, cyc, 32, 0);
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("N=10 warps/SM=1: %lld cycles per inverse\n", h[0]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
