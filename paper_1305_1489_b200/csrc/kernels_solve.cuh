// Skeleton solve on the GPU (replaces solve_skeleton,
// global_system.cpp:106-165): block-Jacobi preconditioned CG on the free dofs
// for a symmetric system (the reference's SimplicialLDLT branch), block-Jacobi
// preconditioned BiCGStab otherwise (its SparseLU branch); Dirichlet dofs
// fixed to their projected values.
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

template <int D2>
constexpr int spmv_smem_bytes() { return (kSolveThreads / 32) * (8 * D2 + D2 * 33) * 8; }

// y = mask(H x); partial[b] = sum over the block's rows of x . y (if partial).
// One warp per face: the face's n1 * d2 neighbour values of x are gathered
// once into shared memory (instead of once per row), then every lane walks
// its column positions of all d2 rows (independent loads, all in flight) and
// the per-row partials are reduced through shared memory.
template <int D2>
__global__ void __launch_bounds__(kSolveThreads)
spmv_kernel(int nfc, const int64_t* __restrict__ fb, const int* __restrict__ nbr, const double* __restrict__ vals,
            const double* __restrict__ x, double* __restrict__ y, int ndir, double* __restrict__ partial) {
  constexpr int NW = kSolveThreads / 32;
  __shared__ double red[NW];
  extern __shared__ double spmv_smem[];  // spmv_smem_bytes<D2>()
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xs = spmv_smem + warp * (8 * D2 + D2 * 33);
  double* part = xs + 8 * D2;  // [D2][33]
  double dot = 0.0;
  for (long f = long(blockIdx.x) * NW + warp; f < nfc; f += long(gridDim.x) * NW) {
    const int64_t b0 = fb[f];
    const int n1 = int(fb[f + 1] - b0), w = n1 * D2;
    for (int k = lane; k < w; k += 32) {
      const int s = k / D2;
      xs[k] = __ldg(x + long(__ldg(nbr + 8 * f + s)) * D2 + (k - s * D2));
    }
    __syncwarp();
    const double* v = vals + b0 * D2 * D2;
    double acc[D2];
#pragma unroll
    for (int i = 0; i < D2; ++i) acc[i] = 0.0;
    for (int k = lane; k < w; k += 32) {
      const double xk = xs[k];
#pragma unroll
      for (int i = 0; i < D2; ++i) acc[i] = fma(__ldg(v + long(i) * w + k), xk, acc[i]);
    }
#pragma unroll
    for (int i = 0; i < D2; ++i) part[i * 33 + lane] = acc[i];
    __syncwarp();
    if (lane < D2) {
      double s = 0.0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) s += part[lane * 33 + l];
      const long row = f * D2 + lane;
      const double yv = f < ndir ? 0.0 : s;
      y[row] = yv;
      dot += x[row] * yv;
    }
    __syncwarp();
  }
  if (partial) {
    const double s = block_sum(dot, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

// Inverse of each free face's diagonal block (SPD): one warp per face, stored
// packed lower in fp32 (a preconditioner only steers the iteration; the
// residual test is fp64), 4 d2(d2+1)/2 bytes per face instead of 8 d2^2.
template <int D2>
__global__ void block_jacobi_kernel(int nfc, int ndir, const int64_t* __restrict__ fb, const int* __restrict__ nbr,
                                    const double* __restrict__ vals, float* __restrict__ binv,
                                    unsigned long long* __restrict__ bad) {
  constexpr int NS = D2 * (D2 + 1) / 2;
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
      for (int i = 0; i < D2; ++i)
        if (i >= lane) binv[f * NS + sym_idx(i, lane, D2)] = float(a[i]);
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

// r_out = mask(b - y) (mode 0, y = H x0) or r_out = r_in - alpha Ap and
// x += alpha p (mode 1); z = Binv r_out per face; partials r.z and r.r.
// One thread per row; a row's z needs its whole face's r, which each thread
// recomputes from r_in (ping-pong buffers, so no thread reads a value another
// has overwritten).
template <int D2>
__global__ void __launch_bounds__(kSolveThreads)
update_kernel(int mode, int nfc, int ndir, const float* __restrict__ binv, const double* __restrict__ b,
              const double* __restrict__ y, const double* __restrict__ p, double* __restrict__ x,
              const double* __restrict__ rin, double* __restrict__ rout, double* __restrict__ z,
              const SolveScalars* __restrict__ sc, double* __restrict__ prz, double* __restrict__ prr) {
  constexpr int NS = D2 * (D2 + 1) / 2;
  __shared__ double red[kSolveThreads / 32];
  const double alpha = mode == 1 ? sc->alpha : 0.0;
  double dz = 0.0, dr = 0.0;
  const long rows = long(nfc) * D2;
  for (long row = long(blockIdx.x) * blockDim.x + threadIdx.x; row < rows; row += long(gridDim.x) * blockDim.x) {
    const long f = row / D2;
    const int i = int(row - f * D2);
    if (f < ndir) {
      if (mode == 0) {
        rout[row] = 0.0;
        z[row] = 0.0;
      }
      continue;
    }
    const long base = f * D2;
    const float* B = binv + f * NS;
    double zi = 0.0, ri = 0.0;
#pragma unroll
    for (int j = 0; j < D2; ++j) {
      const double rj = mode == 0 ? b[base + j] - y[base + j] : rin[base + j] - alpha * y[base + j];
      if (j == i) ri = rj;
      zi = fma(double(B[j >= i ? sym_idx(j, i, D2) : sym_idx(i, j, D2)]), rj, zi);
    }
    rout[row] = ri;
    if (mode == 1) x[row] += alpha * p[row];
    z[row] = zi;
    dz += ri * zi;
    dr += ri * ri;
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

// ---- nonsymmetric branch (the reference's SparseLU branch,
// global_system.cpp:155-162): right-preconditioned BiCGStab with a general
// block-Jacobi preconditioner. Off the timed path; host-driven scalars.

// Inverse of each free face's diagonal block by Gauss-Jordan with partial
// pivoting: one warp per face on the augmented [A | I] in shared memory,
// stored row-major (d2 x d2 doubles per face). A vanished pivot column
// reports the face in `bad`.
template <int D2>
__global__ void __launch_bounds__(128)
block_inverse_general_kernel(int nfc, int ndir, const int64_t* __restrict__ fb, const int* __restrict__ nbr,
                             const double* __restrict__ vals, double* __restrict__ binv,
                             unsigned long long* __restrict__ bad) {
  constexpr int W = 2 * D2, LD = W + 1;
  __shared__ double aug[4][D2 * LD];
  __shared__ double colp[4][D2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* A = aug[warp];
  double* cp = colp[warp];
  for (long f = long(blockIdx.x) * 4 + warp; f < nfc; f += long(gridDim.x) * 4) {
    if (f < ndir) {
      for (int q = lane; q < D2 * D2; q += 32) binv[f * D2 * D2 + q] = (q / D2 == q % D2) ? 1.0 : 0.0;
      continue;
    }
    const int64_t b0 = fb[f];
    const int n1 = int(fb[f + 1] - b0);
    int ss = 0;
    while (ss < n1 && nbr[8 * f + ss] != int(f)) ++ss;
    const double* v = vals + b0 * D2 * D2;
    for (int q = lane; q < D2 * W; q += 32) {
      const int i = q / W, j = q - i * W;
      A[i * LD + j] = j < D2 ? v[long(i) * n1 * D2 + ss * D2 + j] : (j - D2 == i ? 1.0 : 0.0);
    }
    __syncwarp();
    bool ok = true;
    for (int p = 0; p < D2; ++p) {
      // pivot row: largest |A[r][p]|, r >= p (lowest row on ties)
      double best = (lane >= p && lane < D2) ? fabs(A[lane * LD + p]) : -1.0;
      int row = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orow = __shfl_xor_sync(0xffffffffu, row, o);
        if (ob > best || (ob == best && orow < row)) { best = ob; row = orow; }
      }
      if (!(best > 0.0) || !isfinite(best)) { ok = false; break; }
      if (row != p)
        for (int j = lane; j < W; j += 32) {
          const double tmp = A[p * LD + j];
          A[p * LD + j] = A[row * LD + j];
          A[row * LD + j] = tmp;
        }
      __syncwarp();
      const double ip = 1.0 / A[p * LD + p];
      if (lane < D2) cp[lane] = A[lane * LD + p];
      __syncwarp();
      for (int j = lane; j < W; j += 32) A[p * LD + j] *= ip;
      __syncwarp();
      for (int j = lane; j < W; j += 32) {
        const double pj = A[p * LD + j];
        for (int r = 0; r < D2; ++r)
          if (r != p) A[r * LD + j] = fma(-cp[r], pj, A[r * LD + j]);
      }
      __syncwarp();
    }
    if (!ok && lane == 0) atomicMin(bad, static_cast<unsigned long long>(f));
    for (int q = lane; q < D2 * D2; q += 32) {
      const int i = q / D2, j = q - i * D2;
      binv[f * D2 * D2 + q] = ok ? A[i * LD + D2 + j] : (i == j ? 1.0 : 0.0);
    }
    __syncwarp();
  }
}

// out = Binv in per face (zero on the Dirichlet faces); one thread per row
template <int D2>
__global__ void __launch_bounds__(kSolveThreads)
precond_general_kernel(int nfc, int ndir, const double* __restrict__ binv, const double* __restrict__ in,
                       double* __restrict__ out) {
  const long rows = long(nfc) * D2;
  for (long row = long(blockIdx.x) * blockDim.x + threadIdx.x; row < rows; row += long(gridDim.x) * blockDim.x) {
    const long f = row / D2;
    const int i = int(row - f * D2);
    double z = 0.0;
    if (f >= ndir) {
      const double* B = binv + f * D2 * D2 + i * D2;
#pragma unroll
      for (int j = 0; j < D2; ++j) z = fma(B[j], in[f * D2 + j], z);
    }
    out[row] = z;
  }
}

// up to three dot products a_i . b_i (null pairs skipped), per-block partials
__global__ void __launch_bounds__(kSolveThreads)
dots_kernel(long n, const double* a0, const double* b0, const double* a1, const double* b1, const double* a2,
            const double* b2, double* __restrict__ partial) {
  __shared__ double red[kSolveThreads / 32];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
    if (a0) s0 = fma(a0[i], b0[i], s0);
    if (a1) s1 = fma(a1[i], b1[i], s1);
    if (a2) s2 = fma(a2[i], b2[i], s2);
  }
  const double r0 = block_sum(s0, red);
  const double r1 = block_sum(s1, red);
  const double r2 = block_sum(s2, red);
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = r0;
    partial[gridDim.x + blockIdx.x] = r1;
    partial[2 * gridDim.x + blockIdx.x] = r2;
  }
}

// out = alpha x + beta y + gamma z (null vectors skipped; out may alias any of them)
__global__ void lincomb_kernel(long n, double* out, double alpha, const double* x, double beta, const double* y,
                               double gamma, const double* z) {
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
    double v = alpha * x[i];
    if (y) v = fma(beta, y[i], v);
    if (z) v = fma(gamma, z[i], v);
    out[i] = v;
  }
}

}  // namespace hdgb
