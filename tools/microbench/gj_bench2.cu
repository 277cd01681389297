// Latency of the sweep Gauss-Jordan variants (kernels_condense2.cuh) in the
// P3 setting: a 512-thread CTA, `active` warps each inverting an SPD matrix
// held in shared memory (LD-strided), the rest idle; plus a v1/v2 result check.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_1305_1489_b200/csrc/kernels_condense2.cuh"
#include "gj_sweep_v3.cuh"
#include "gj_pair.cuh"
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
      else if (V == 3) gj_sweep_inverse3<N>(a, stage + warp * 128, lane, pmin, pmax);
      else if (V == 4) gj_sweep_inverse3<N, true>(a, stage + warp * 128, lane, pmin, pmax);
      else if (V >= 5) gj_sweep_inverse3<N, false, V - 4>(a, stage + warp * 128, lane, pmin, pmax);
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
      else if (V == 3) gj_sweep_inverse3<N>(a, stage + warp * 128, lane, pmin, pmax);
      else if (V == 4) gj_sweep_inverse3<N, true>(a, stage + warp * 128, lane, pmin, pmax);
      else if (V >= 5) gj_sweep_inverse3<N, false, V - 4>(a, stage + warp * 128, lane, pmin, pmax);
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
  for (int act : {1, 4, 8, 12, 16}) {
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

__global__ void rcp_err(double* out, int n) {
  double mx = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double x = 1.0 + (double)i / n * 3.0 + 1e-7 * (i % 977);
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    mx = fmax(mx, fabs(fma(-x, r, 1.0)));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)out, (unsigned long long)__double_as_longlong(mx));
}


// two 20 x 20 inverses per warp (gj_pair.cuh): cycles per PAIR
template <int LD>
__global__ void __launch_bounds__(512) gj_pair_smem(double* out, long long* cyc, int reps, int active) {
  __shared__ __align__(16) double stage[6 * 384];
  __shared__ double Sm[8][24 * LD];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int N = 20;
  if (warp < active) {
    double* S = Sm[(2 * warp + (lane >> 4)) & 7];
    const int c = lane & 15;
    for (int i = c; i < 24 * LD; i += 16) S[i] = 0.0;
    __syncwarp();
    for (int col = c; col < N; col += 16)
      for (int i = 0; i < N; ++i) S[i + col * LD] = (i == col ? 4.0 * N : 0.0) + 1.0 / (1.0 + i + col);
    __syncwarp();
    double pmin = 1e300, pmax = 0;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      double a[20], cc[10], zi[10];
#pragma unroll
      for (int i = 0; i < 20; ++i) a[i] = S[i + c * LD];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int jj = 0; jj <= j; ++jj) cc[j * (j + 1) / 2 + jj] = S[16 + j + (16 + jj) * LD];
      __syncwarp();
      gj_pair_inverse20(a, cc, zi, stage + warp * 384, lane, pmin, pmax);
#pragma unroll
      for (int i = 0; i < 20; ++i) S[i + c * LD] = a[i];
#pragma unroll
      for (int j = 0; j < 4; ++j) S[c + (16 + j) * LD] = a[16 + j];
      if (c < 4) {
#pragma unroll
        for (int j = 0; j < 4; ++j) S[16 + j + (16 + c) * LD] = zi[j >= c ? j * (j + 1) / 2 + c : c * (c + 1) / 2 + j];
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 16 + warp] = (t1 - t0) / reps;
    if (blockIdx.x == 0 && warp == 0) {
      for (int i = lane; i < N * N; i += 32) out[i] = Sm[0][(i % N) + (i / N) * LD];
      if (lane == 0) { out[N * N] = pmin; out[N * N + 1] = pmax; }
    }
  }
  __syncthreads();
}

void run_pair() {
  double* out; long long* cyc;
  cudaMalloc(&out, 4096 * 8); cudaMalloc(&cyc, 148 * 16 * 8);
  long long h[148 * 16];
  double *o1; cudaMalloc(&o1, 4096 * 8);
  gj_smem<20, 20, 2><<<1, 512>>>(o1, cyc, 1, 1);
  gj_pair_smem<20><<<1, 512>>>(out, cyc, 1, 1);
  double h1[402], h2[402];
  cudaMemcpy(h1, o1, sizeof(h1), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, out, sizeof(h2), cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (int i = 0; i < 400; ++i) { md = fmax(md, fabs(h1[i] - h2[i])); mx = fmax(mx, fabs(h1[i])); }
  printf("pair vs v2 max|diff|/max|inv| = %.3e  pmin %.6e/%.6e pmax %.6e/%.6e\n", md / mx, h1[400], h2[400], h1[401], h2[401]);
  for (int act : {1, 2, 4, 5, 6}) {
    gj_pair_smem<20><<<148, 512>>>(out, cyc, 32, act);
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("pair N=20 %d active warps (%d inverses): %lld cycles per pair\n", act, 2 * act, h[0]);
  }
}

// P3 mix: warps 0..npair-1 invert pairs (gj_pair.cuh), warps npair..npair+nsingle-1 single matrices (v2)
__global__ void __launch_bounds__(512) gj_mix(long long* cyc, int reps, int npair, int nsingle) {
  __shared__ __align__(16) double stage[6 * 384];
  __shared__ __align__(16) double st1[10 * 128];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane & 15;
  long long t0 = clock64();
  if (warp < npair) {
    double a[20], cc[10], zi[10], pmin = 1e300, pmax = 0;
    for (int i = 0; i < 20; ++i) a[i] = (i == c ? 80.0 : 0.0) + 1.0 / (1.0 + i + c);
    for (int j = 0; j < 10; ++j) cc[j] = (j == 0 || j == 2 || j == 5 || j == 9) ? 80.0 : 0.01;
    for (int r = 0; r < reps; ++r) gj_pair_inverse20(a, cc, zi, stage + warp * 384, lane, pmin, pmax);
    if (a[3] == 12345.0 && zi[2] == 1.0) cyc[1000] = 1;
  } else if (warp < npair + nsingle) {
    double a[20], pmin = 1e300, pmax = 0;
    for (int i = 0; i < 20; ++i) a[i] = lane < 20 ? (i == lane ? 80.0 : 0.0) + 1.0 / (1.0 + i + lane) : 0.0;
    for (int r = 0; r < reps; ++r) gj_sweep_inverse<20>(a, st1 + (warp - npair) * 128, lane, pmin, pmax);
    if (a[3] == 12345.0) cyc[1000] = 1;
  }
  long long t1 = clock64();
  if (lane == 0 && blockIdx.x == 0) cyc[warp] = (t1 - t0) / reps;
}

void run_mix(int np, int ns) {
  long long* cyc; cudaMalloc(&cyc, 2048 * 8); cudaMemset(cyc, 0, 2048 * 8);
  gj_mix<<<148, 512>>>(cyc, 32, np, ns);
  long long h[16]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < np + ns; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("mix %d pair warps + %d single warps (%d inverses): max %lld cycles per round\n", np, ns, 2 * np + ns, mx);
}

template <int N, int VA, int VB>
void check2() {
  double *o1, *o2; long long* cyc;
  cudaMalloc(&o1, 4096 * 8); cudaMalloc(&o2, 4096 * 8); cudaMalloc(&cyc, 148 * 16 * 8);
  gj_smem<N, (N + 3) / 4 * 4, VA><<<1, 512>>>(o1, cyc, 1, 1);
  gj_smem<N, (N + 3) / 4 * 4, VB><<<1, 512>>>(o2, cyc, 1, 1);
  double h1[N * N + 2], h2[N * N + 2];
  cudaMemcpy(h1, o1, sizeof(h1), cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, o2, sizeof(h2), cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (int i = 0; i < N * N; ++i) { md = fmax(md, fabs(h1[i] - h2[i])); mx = fmax(mx, fabs(h1[i])); }
  printf("N=%d v%d vs v%d max|diff|/max|inv| = %.3e  pmin %.6e/%.6e\n", N, VA, VB, md / mx, h1[N * N], h2[N * N]);
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
  check2<20, 2, 3>(); check2<20, 2, 4>(); check2<19, 2, 3>(); check2<20, 1, 3>();
  {
    double* e; cudaMalloc(&e, 8); cudaMemset(e, 0, 8);
    rcp_err<<<148, 256>>>(e, 1 << 24);
    double h; cudaMemcpy(&h, e, 8, cudaMemcpyDeviceToHost);
    printf("rcp.approx.f64 max |1 - x r| = %.3e (2^%.1f)\n", h, log2(h));
  }
  check2<20, 2, 5>(); check2<20, 2, 7>();
  run_pair();
  run_mix(0, 10); run_mix(5, 0); run_mix(4, 2); run_mix(4, 0); run_mix(0, 8); run_mix(3, 4);
  run<20, 2>("v2");

  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
