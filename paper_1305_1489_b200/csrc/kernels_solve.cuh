// Skeleton solve on the GPU (replaces solve_skeleton,
// global_system.cpp:106-165, SPD branch): block-Jacobi preconditioned CG on
// the free dofs, Dirichlet dofs fixed to their projected values.
//
// The reference eliminates the Dirichlet rows/columns into Hff and moves
// H_fD u_D to the right-hand side. Here the operator is the full CSR H
// applied to a vector that is zero on the Dirichlet dofs, with the Dirichlet
// rows of the result masked: the same reduced system without forming Hff.
//
// Layout: the block CSR of hdg_b200_pattern_fill / hdg_b200_scatter. Row
// (f, i) holds n1(f) * d2 values, neighbour-face major (nbr[f][s], j), so
// columns come from nbr instead of colidx (8 B per nonzero instead of 12).
// Every kernel is HBM-bound; SpMV reads each value once per iteration.
// Reductions are two-pass (per-block partials, one-block finalize) so
// the iteration is deterministic for a fixed grid.
#pragma once

#include "dev_common.cuh"
#include "kernels_condense2.cuh"

namespace hdgb {

constexpr int kSolveThreads = 256;

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
  return s;  // valid in thread 0
}

// y = mask(H x); partial[b] = sum over the block's rows of x . y (if partial)
template <int D2>
__global__ void __launch_bounds__(kSolveThreads)
spmv_kernel(int nfc, const int64_t* __restrict__ fb, const int* __restrict__ nbr, const double* __restrict__ vals,
            const double* __restrict__ x, double* __restrict__ y, int ndir, double* __restrict__ partial) {
  __shared__ double red[kSolveThreads / 32];
  const int lane = threadIdx.x & 31, hl = lane & 15;  // half-warp per row, two rows per warp
  const long nrows = long(nfc) * D2;
  const long w0 = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nw = (long(gridDim.x) * blockDim.x) >> 5;
  double dot = 0.0;
  for (long w = w0; 2 * w < nrows; w += nw) {  // warp-uniform trip count
    const long row = 2 * w + (lane >> 4);
    double acc = 0.0;
    const bool live = row < nrows;
    long f = 0;
    int i = 0;
    if (live) {
      f = row / D2;
      i = int(row - f * D2);
      const int64_t b0 = fb[f];
      const int n1 = int(fb[f + 1] - b0);
      const double* v = vals + b0 * D2 * D2 + long(i) * n1 * D2;
      const int* nb = nbr + 8 * f;
      for (int k = hl; k < n1 * D2; k += 16) {
        const int s = k / D2, j = k - s * D2;
        acc = fma(__ldg(v + k), __ldg(x + long(__ldg(nb + s)) * D2 + j), acc);
      }
    }
#pragma unroll
    for (int o = 8; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (live && hl == 0) {
      const double yv = f < ndir ? 0.0 : acc;
      y[row] = yv;
      dot += x[row] * yv;
    }
  }
  if (partial) {
    const double s = block_sum(dot, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

// Inverse of each free face's diagonal block (SPD): one warp per face.
template <int D2>
__global__ void block_jacobi_kernel(int nfc, int ndir, const int64_t* __restrict__ fb, const int* __restrict__ nbr,
                                    const double* __restrict__ vals, double* __restrict__ binv,
                                    unsigned long long* __restrict__ bad) {
  __shared__ __align__(16) double stage[kSolveThreads / 32][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (long f = long(blockIdx.x) * (blockDim.x >> 5) + warp; f < nfc; f += long(gridDim.x) * (blockDim.x >> 5)) {
    double a[D2];
    if (f < ndir) {  // identity on the fixed dofs (never applied to a nonzero)
#pragma unroll
      for (int i = 0; i < D2; ++i) a[i] = (i == lane) ? 1.0 : 0.0;
    } else {
      const int64_t b0 = fb[f];
      const int n1 = int(fb[f + 1] - b0);
      int ss = 0;
      while (ss < n1 && nbr[8 * f + ss] != int(f)) ++ss;
      const double* v = vals + b0 * D2 * D2;
#pragma unroll
      for (int i = 0; i < D2; ++i) a[i] = lane < D2 ? v[long(i) * n1 * D2 + ss * D2 + lane] : 0.0;
      double pmin = 1e300, pmax = 0.0;
      warp_gj_inverse<D2>(a, stage[warp], lane, pmin, pmax);
      if (lane == 0 && !(pmin > 0.0)) atomicMin(bad, static_cast<unsigned long long>(f));
    }
    if (lane < D2) {
#pragma unroll
      for (int i = 0; i < D2; ++i) binv[f * D2 * D2 + long(lane) * D2 + i] = a[i];
    }
  }
}

// Deterministic finalize of the partial sums into the scalar slots.
// mode 0 (after the initial residual): rz = P0, rr = P1, rr0 = rr
// mode 1 (after spmv): alpha = rz / P0
// mode 2 (after update): beta = P0 / rz, rz = P0, rr = P1
struct SolveScalars {
  double rz, rr, rr0, alpha, beta, pap;
};

__global__ void finalize_kernel(int mode, int nblk, const double* __restrict__ p0, const double* __restrict__ p1,
                                SolveScalars* sc) {
  __shared__ double red[kSolveThreads / 32];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    a += p0[i];
    if (p1) b += p1[i];
  }
  const double A = block_sum(a, red);
  const double Bs = block_sum(b, red);
  if (threadIdx.x == 0) {
    if (mode == 0) { sc->rz = A; sc->rr = Bs; sc->rr0 = Bs; sc->beta = 0.0; }
    else if (mode == 1) { sc->pap = A; sc->alpha = A != 0.0 ? sc->rz / A : 0.0; }
    else { sc->beta = sc->rz != 0.0 ? A / sc->rz : 0.0; sc->rz = A; sc->rr = Bs; }
  }
}

// r = mask(b - y) on entry (mode 0, y = H x0) or r -= alpha Ap, x += alpha p
// (mode 1); then z = Binv r per face; partials: r.z and r.r. One warp per face.
template <int D2>
__global__ void __launch_bounds__(kSolveThreads)
update_kernel(int mode, int nfc, int ndir, const double* __restrict__ binv, const double* __restrict__ b,
              const double* __restrict__ y, const double* __restrict__ p, double* __restrict__ x,
              double* __restrict__ r, double* __restrict__ z, const SolveScalars* __restrict__ sc,
              double* __restrict__ prz, double* __restrict__ prr) {
  __shared__ double red[kSolveThreads / 32];
  __shared__ double rs[kSolveThreads / 32][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double alpha = mode == 1 ? sc->alpha : 0.0;
  double dz = 0.0, dr = 0.0;
  const long nwarps = long(gridDim.x) * (blockDim.x >> 5);
  for (long f = long(blockIdx.x) * (blockDim.x >> 5) + warp; f < nfc; f += nwarps) {  // warp per face
    const bool live = f >= ndir;
    double ri = 0.0;
    if (live && lane < D2) {
      const long row = f * D2 + lane;
      if (mode == 0) {
        ri = b[row] - y[row];
      } else {
        x[row] += alpha * p[row];
        ri = r[row] - alpha * y[row];
      }
      r[row] = ri;
    } else if (lane < D2 && mode == 0) {
      r[f * D2 + lane] = 0.0;
      z[f * D2 + lane] = 0.0;
    }
    rs[warp][lane] = ri;
    __syncwarp();
    if (live && lane < D2) {
      const double* B = binv + f * D2 * D2;
      double zi = 0.0;
#pragma unroll
      for (int j = 0; j < D2; ++j) zi = fma(B[long(j) * D2 + lane], rs[warp][j], zi);
      z[f * D2 + lane] = zi;
      dz += ri * zi;
      dr += ri * ri;
    }
    __syncwarp();
  }
  const double s0 = block_sum(dz, red);
  const double s1 = block_sum(dr, red);
  if (threadIdx.x == 0) {
    prz[blockIdx.x] = s0;
    prr[blockIdx.x] = s1;
  }
}

// p = z + beta p (beta = 0 on the first iteration, p = z)
__global__ void direction_kernel(long n, const double* __restrict__ z, double* __restrict__ p,
                                 const SolveScalars* __restrict__ sc, int first) {
  const double beta = first ? 0.0 : sc->beta;
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
    p[i] = first ? z[i] : fma(beta, p[i], z[i]);
}

// sum |H_ij - H_ji| and sum |H_ij| over the free block (reference symmetry test,
// global_system.cpp:144-147); one thread per value, partials per block
template <int D2>
__global__ void asym_kernel(int nfc, int ndir, const int64_t* __restrict__ fb, const int* __restrict__ nbr,
                            const double* __restrict__ vals, double* __restrict__ pa, double* __restrict__ ps) {
  __shared__ double red[kSolveThreads / 32];
  double da = 0.0, ds = 0.0;
  const long rows = long(nfc) * D2;
  for (long row = long(blockIdx.x) * (blockDim.x >> 4) + (threadIdx.x >> 4); row < rows;
       row += long(gridDim.x) * (blockDim.x >> 4)) {
    const long f1 = row / D2;
    const int i = int(row - f1 * D2), hl = threadIdx.x & 15;
    if (f1 < ndir) continue;
    const int64_t b1 = fb[f1];
    const int n1 = int(fb[f1 + 1] - b1);
    for (int k = hl; k < n1 * D2; k += 16) {
      const int s = k / D2, j = k - s * D2;
      const int f2 = nbr[8 * f1 + s];
      if (f2 < ndir) continue;
      const double v = vals[b1 * D2 * D2 + long(i) * n1 * D2 + k];
      const int64_t b2 = fb[f2];
      const int n2 = int(fb[f2 + 1] - b2);
      int s2 = 0;
      while (s2 < n2 && nbr[8L * f2 + s2] != int(f1)) ++s2;
      const double w = vals[b2 * D2 * D2 + long(j) * n2 * D2 + s2 * D2 + i];
      da += fabs(v - w);
      ds += fabs(v);
    }
  }
  const double A = block_sum(da, red);
  const double S = block_sum(ds, red);
  if (threadIdx.x == 0) {
    pa[blockIdx.x] = A;
    ps[blockIdx.x] = S;
  }
}

}  // namespace hdgb
