// Latency of the sweep Gauss-Jordan variants (kernels_condense2.cuh) in the
// P3 setting: a 512-thread CTA, `active` warps each inverting an SPD matrix
// held in shared memory (LD-strided), the rest idle; plus a v1/v2 result check.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_1305_1489_b200/csrc/kernels_condense2.cuh"
using namespace hdgb;

template <int N, int LD, int V, bool ROW = false>
__global__ void __launch_bounds__(512) gj_smem(double* out, long long* cyc, int reps, int active) {
  __shared__ __align__(16) double stage[16 * 128];
  __shared__ double Sm[8][24 * LD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < active) {
    double* S = Sm[warp & 7];
    for (int i = lane; i < 24 * LD; i += 32) S[i] = 0.0;
    __syncwarp();
    if (lane < N)
      for (int i = 0; i < N; ++i) S[i + lane * LD] = (i == lane ? 4.0 * N : 0.0) + 1.0 / (1.0 + i + lane);
    __syncwarp();
    double pmin = 1e300, pmax = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      double a[N];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int rr = i > lane ? i : lane, c = i > lane ? lane : i;
        if (ROW) a[i] = lane < N ? S[lane + i * LD] : 0.0;
        else a[i] = lane < N ? S[rr + c * LD] : 0.0;
      }
      if (V == 1) warp_gj_inverse<N>(a, stage + warp * 128, lane, pmin, pmax);
      else gj_sweep_inverse<N>(a, stage + warp * 128, lane, pmin, pmax);
      if (lane < N) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          if (ROW) S[lane + i * LD] = a[i];
          else S[i + lane * LD] = a[i];
        }
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = (t1 - t0) / reps;
    if (blockIdx.x == 0 && warp == 0) {
      for (int i = lane; i < N * N; i += 32) out[i] = S[(i % N) + (i / N) * LD];
      if (lane == 0) { out[N * N] = pmin; out[N * N + 1] = pmax; }
    }
  }
  __syncthreads();
}

template <int N, int V>
__global__ void __launch_bounds__(512) gj_reg(double* out, long long* cyc, int reps, int active) {
  __shared__ __align__(16) double stage[16 * 128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp < active) {
    double a[N];
    for (int i = 0; i < N; ++i) a[i] = lane < N ? (i == lane ? 4.0 * N : 0.0) + 1.0 / (1.0 + i + lane) : 0.0;
    double pmin = 1e300, pmax = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      if (V == 1) warp_gj_inverse<N>(a, stage + warp * 128, lane, pmin, pmax);
      else gj_sweep_inverse<N>(a, stage + warp * 128, lane, pmin, pmax);
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = (t1 - t0) / reps;
    double s = pmin + pmax;
    for (int i = 0; i < N; ++i) s += a[i];
    out[blockIdx.x * 512 + threadIdx.x] = s;
  }
}

template <int N, int V>
void run(const char* name) {
  double* out; long long* cyc;
  cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 148 * 16 * 8);
  long long h[148 * 16];
  for (int act : {1, 4, 8}) {
    gj_smem<N, (N + 3) / 4 * 4, V><<<148, 512>>>(out, cyc, 32, act);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s N=%d %d active warps: %lld cycles per inverse\n", name, N, act, h[0]);
  }
  for (int act : {1, 8}) {
    gj_smem<N, (N + 3) / 4 * 4, V, true><<<148, 512>>>(out, cyc, 32, act);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s N=%d row-wise smem, %d active warps: %lld cycles per inverse\n", name, N, act, h[0]);
  }
  for (int act : {1, 8}) {
    double* o2; cudaMalloc(&o2, 148 * 512 * 8);
    gj_reg<N, V><<<148, 512>>>(o2, cyc, 32, act);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%s N=%d registers only, %d active warps: %lld cycles per inverse\n", name, N, act, h[0]);
    cudaFree(o2);
  }
  cudaFree(out); cudaFree(cyc);
}

template <int N>
void check() {
  double *o1, *o2; long long* cyc;
  cudaMalloc(&o1, 4096 * 8); cudaMalloc(&o2, 4096 * 8); cudaMalloc(&cyc, 148 * 16 * 8);
  gj_smem<N, (N + 3) / 4 * 4, 1><<<1, 512>>>(o1, cyc, 1, 1);
  gj_smem<N, (N + 3) / 4 * 4, 2><<<1, 512>>>(o2, cyc, 1, 1);
  double h1[N * N + 2], h2[N * N + 2];
  cudaMemcpy(h1, o1, sizeof(h1), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, o2, sizeof(h2), cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (int i = 0; i < N * N; ++i) { md = fmax(md, fabs(h1[i] - h2[i])); mx = fmax(mx, fabs(h1[i])); }
  printf("N=%d v1 vs v2 max|diff|/max|inv| = %.3e  pmin %.6e/%.6e pmax %.6e/%.6e\n", N, md / mx, h1[N * N],
         h2[N * N], h1[N * N + 1], h2[N * N + 1]);
}

int main() {
  check<20>(); check<10>(); check<19>(); check<4>(); check<1>();
  run<20, 1>("v1"); run<20, 2>("v2");
  run<10, 1>("v1"); run<10, 2>("v2");
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
