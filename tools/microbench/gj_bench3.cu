// Latency of the K3 v6 register sweep inverse (gj_sweep.cuh) in its K3
// setting: one warp per SM sub-partition (or two), the matrix loaded from and
// stored to shared memory as K3 does. Variants of the pivot step are timed
// against the product one and checked against it.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a gj_bench3.cu -o gj_bench3
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_1305_1489_b200/csrc/gj_sweep.cuh"

// Variant 1: the warp barrier right after the stage stores, so the stage
// loads of the update can issue under the reciprocal chain.
template <int N>
__device__ __forceinline__ void step_v1(double (&a)[N], double* stage, int lane, int k, double& piv) {
  double* st = stage + ((k >> 1) & 1) * 64;
  if (lane < N) {
    st[lane] = a[k];
    st[32 + lane] = a[k + 1];
  }
  __syncwarp();
  const double2 p0 = *reinterpret_cast<const double2*>(st + k);        // a[k] of lanes k, k+1: p00, p01
  const double2 p1 = *reinterpret_cast<const double2*>(st + 32 + k);   // a[k+1] of lanes k, k+1: p01, p11
  const double p00 = p0.x, p01 = p1.x, p11 = p1.y;
  double n0x = 0.0, n0y = 0.0, n1x = 0.0, n1y = 0.0;
  if (k + 2 < N) {
    const double2 q0 = *reinterpret_cast<const double2*>(st + k + 2);
    const double2 q1 = *reinterpret_cast<const double2*>(st + 32 + k + 2);
    n0x = q0.x; n0y = q0.y; n1x = q1.x; n1y = q1.y;
  }
  const double det = fma(p00, p11, -p01 * p01);
  const bool m0 = lane == k, m1 = lane == k + 1;
  const double ak0 = m0 ? a[k] - 1.0 : a[k];
  const double ak1 = m1 ? a[k + 1] - 1.0 : a[k + 1];
  const double u0 = fma(p11, ak0, -p01 * ak1);
  const double u1 = fma(p00, ak1, -p01 * ak0);
  double s0 = 0.0, s1 = 0.0;
  if (k + 2 < N) {
    s0 = fma(n0x, u0, n1x * u1);
    if (k + 3 < N) s1 = fma(n0y, u0, n1y * u1);
  }
  const double id = gj_rcp(det);
  if (k + 2 < N) {
    a[k + 2] = fma(-s0, id, a[k + 2]);
    if (k + 3 < N) a[k + 3] = fma(-s1, id, a[k + 3]);
  }
  const double w0 = u0 * id, w1 = u1 * id;
  if (m0) piv = p00;
  if (m1) piv = p00 * id;
#pragma unroll
  for (int i0 = 0; i0 < N; i0 += 2) {
    if (i0 == k || i0 == k + 2) continue;
    const double2 v0 = *reinterpret_cast<const double2*>(st + i0);
    const double2 v1 = *reinterpret_cast<const double2*>(st + 32 + i0);
    a[i0] = fma(-v0.x, w0, fma(-v1.x, w1, a[i0]));
    if (i0 + 1 < N) a[i0 + 1] = fma(-v0.y, w0, fma(-v1.y, w1, a[i0 + 1]));
  }
  a[k] = m0 ? w0 - 1.0 : w0;
  a[k + 1] = m1 ? w1 - 1.0 : w1;
}

// Variant 2: as the product step (pivot block by shuffles) but the barrier
// before the reciprocal chain instead of after it.
template <int N>
__device__ __forceinline__ void step_v2(double (&a)[N], double* stage, int lane, int k, double& piv) {
  double* st = stage + ((k >> 1) & 1) * 64;
  if (lane < N) {
    st[lane] = a[k];
    st[32 + lane] = a[k + 1];
  }
  const double p00 = __shfl_sync(0xffffffffu, a[k], k);
  const double p01 = __shfl_sync(0xffffffffu, a[k + 1], k);
  const double p11 = __shfl_sync(0xffffffffu, a[k + 1], k + 1);
  double n0x = 0.0, n0y = 0.0, n1x = 0.0, n1y = 0.0;
  if (k + 2 < N) {
    n0x = __shfl_sync(0xffffffffu, a[k], k + 2);
    n1x = __shfl_sync(0xffffffffu, a[k + 1], k + 2);
    if (k + 3 < N) {
      n0y = __shfl_sync(0xffffffffu, a[k], k + 3);
      n1y = __shfl_sync(0xffffffffu, a[k + 1], k + 3);
    }
  }
  __syncwarp();
  const double det = fma(p00, p11, -p01 * p01);
  const bool m0 = lane == k, m1 = lane == k + 1;
  const double ak0 = m0 ? a[k] - 1.0 : a[k];
  const double ak1 = m1 ? a[k + 1] - 1.0 : a[k + 1];
  const double u0 = fma(p11, ak0, -p01 * ak1);
  const double u1 = fma(p00, ak1, -p01 * ak0);
  double s0 = 0.0, s1 = 0.0;
  if (k + 2 < N) {
    s0 = fma(n0x, u0, n1x * u1);
    if (k + 3 < N) s1 = fma(n0y, u0, n1y * u1);
  }
  const double id = gj_rcp(det);
  if (k + 2 < N) {
    a[k + 2] = fma(-s0, id, a[k + 2]);
    if (k + 3 < N) a[k + 3] = fma(-s1, id, a[k + 3]);
  }
  const double w0 = u0 * id, w1 = u1 * id;
  if (m0) piv = p00;
  if (m1) piv = p00 * id;
#pragma unroll
  for (int i0 = 0; i0 < N; i0 += 2) {
    if (i0 == k || i0 == k + 2) continue;
    const double2 v0 = *reinterpret_cast<const double2*>(st + i0);
    const double2 v1 = *reinterpret_cast<const double2*>(st + 32 + i0);
    a[i0] = fma(-v0.x, w0, fma(-v1.x, w1, a[i0]));
    if (i0 + 1 < N) a[i0 + 1] = fma(-v0.y, w0, fma(-v1.y, w1, a[i0 + 1]));
  }
  a[k] = m0 ? w0 - 1.0 : w0;
  a[k + 1] = m1 ? w1 - 1.0 : w1;
}

template <int N, int V>
__device__ __forceinline__ void inverse(double (&a)[N], double* stage, int lane, double& pmin, double& pmax) {
  double piv = 1.0;
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) {
    if (V == 0) gj_sweep_step<N>(a, stage, lane, k, piv);
    else if (V == 1) step_v1<N>(a, stage, lane, k, piv);
    else step_v2<N>(a, stage, lane, k, piv);
  }
  gj_sweep_finish<N>(a, stage, lane, piv, pmin, pmax);
}

template <int N, int V, int NW>
__global__ void __launch_bounds__(NW * 32, 1) bench(double* out, long long* cyc, int reps) {
  __shared__ __align__(16) double stage[NW * 128];
  __shared__ __align__(16) double Sm[NW][N * 26];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* S = Sm[warp];
  if (lane < N)
    for (int i = 0; i < N; ++i) S[i * 26 + lane] = (i == lane ? 2.0 + 0.1 * i : 0.0) + 1.0 / (1.0 + i + lane);
  __syncwarp();
  double pmin = 1e300, pmax = 0;
  double acc = 0.0;
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double a[N];
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = lane < N ? S[i * 26 + lane] : 0.0;
    __syncwarp();
    inverse<N, V>(a, stage + warp * 128, lane, pmin, pmax);
    if (r == reps - 1 && blockIdx.x == 0 && warp == 0 && lane < N)
      for (int i = 0; i < N; ++i) out[i * N + lane] = a[i];
#pragma unroll
    for (int i = 0; i < N; ++i) acc += a[i];
    __syncwarp();
  }
  const long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * NW + warp] = (t1 - t0) / reps;
  if (acc == 1.2345e-300) out[N * N] = acc + pmin + pmax;
}

template <int N, int V, int NW>
double run(const char* name, double* ref) {
  double* out; long long* cyc;
  cudaMalloc(&out, (N * N + 2) * 8);
  cudaMalloc(&cyc, 148 * NW * 8);
  bench<N, V, NW><<<148, NW * 32>>>(out, cyc, 200);
  bench<N, V, NW><<<148, NW * 32>>>(out, cyc, 2000);
  cudaDeviceSynchronize();
  long long h[148 * NW];
  double ho[N * N];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (auto v : h) mx = v > mx ? v : mx;
  double md = 0.0, mr = 0.0;
  if (ref) {
    for (int i = 0; i < N * N; ++i) { md = fmax(md, fabs(ho[i] - ref[i])); mr = fmax(mr, fabs(ref[i])); }
  }
  printf("%s N=%d V=%d warps/SM=%d: %lld cycles per inverse (incl. load + store)  diff vs V0 %.2e  %s\n", name, N, V, NW,
         mx, ref ? md / mr : 0.0, cudaGetErrorString(cudaGetLastError()));
  if (!ref) return 0;
  return md;
}

int main() {
  static double ref20[400];
  {
    double* out; long long* cyc;
    cudaMalloc(&out, 402 * 8); cudaMalloc(&cyc, 148 * 4 * 8);
    bench<20, 0, 4><<<148, 128>>>(out, cyc, 1);
    cudaMemcpy(ref20, out, 400 * 8, cudaMemcpyDeviceToHost);
  }
  run<20, 0, 4>("product", ref20);
  run<20, 1, 4>("early-barrier+lds-pivots", ref20);
  run<20, 2, 4>("barrier-before-rcp", ref20);
  run<20, 0, 8>("product", ref20);
  run<20, 1, 8>("early-barrier+lds-pivots", ref20);
  run<20, 2, 8>("barrier-before-rcp", ref20);
  return 0;
}
