// K6 v2 (post degree k+1 <= 4): CTA-batched postprocess_star
// (postprocess.cpp:33-74) for 8 elements per CTA.
//
// The two table contractions run as DMMA GEMMs with the element as the N
// dimension, so the reference tables stream once per 8 elements instead of
// once per element (the per-element warp version spent most of its time
// re-reading Pd and Shat from L2):
//   R (n x 8)  = -(1/6) [Pd_0^T Pd_1^T Pd_2^T] (n x 3nq) . G (3nq x 8),
//                G_#(q, e) = w_q kappa^-1(x_q) sum_s a_e(s,#) (P_k q_s)(q)
//   S (packed lower, n(n+1)/2 x 8) = Shat_packed (. x 9) . gm (9 x 8),
//                gm_e = (a_e^T a_e) / detB_e        (stiffness_matrices)
// The K dimension of R is split over the 8 warps (partials reduced in shared
// memory). Then each warp owns one element: mean constraint row, right-looking
// Cholesky of the trailing SPD block in packed storage, register-resident
// triangular solves (as the v1 kernel, kernels_post.cuh).
#pragma once

#include "dev_common.cuh"
#include "kernels_local.cuh"
#include "kernels_post.cuh"

namespace hdgb {

constexpr int kPost2EB = 8;     // elements per CTA (one DMMA N-tile)
constexpr int kPost2Warps = 8;  // one warp per element in the solve phase
constexpr int kPost2LDG = kPost2EB;  // G rows [q][e]: B-fragment reads are conflict-free at 8
constexpr int kPost2MaxNS = 40 * 41 / 2;

struct Post2Dims {
  int n, nq, nq4, d3k, npad, ns, nsp;
  int off_verts, off_sg, off_qc, off_gm, off_R, off_Rp, off_GS, total;
  __host__ __device__ Post2Dims(int n_, int nq_, int d3k_) : n(n_), nq(nq_), d3k(d3k_) {
    nq4 = (nq + 3) / 4 * 4;
    npad = (n + 7) / 8 * 8;
    ns = n * (n + 1) / 2;
    nsp = (ns + 7) / 8 * 8;
    off_verts = 0;                                    // 12 x EB
    off_sg = off_verts + 12 * kPost2EB;               // 32 x EB geometry records
    off_qc = off_sg + 32 * kPost2EB;                  // 3 x d3k x EB
    off_gm = off_qc + 3 * d3k * kPost2EB;             // 12 x EB (rows 9..11 zero)
    off_R = off_gm + 12 * kPost2EB;                   // npad x EB
    off_Rp = off_R + npad * kPost2EB;                 // warps x npad x EB partials
    off_GS = off_Rp + kPost2Warps * npad * kPost2EB;  // G (3 nq4 x LDG) | S (EB x nsp)
    const int g = 3 * nq4 * kPost2LDG, sgs = kPost2EB * nsp;
    total = off_GS + (g > sgs ? g : sgs);
  }
};

__device__ __forceinline__ int pk_lower(int i, int j, int n) { return j * n - j * (j - 1) / 2 + (i - j); }

__global__ void __launch_bounds__(kPost2Warps * 32)
postprocess2_kernel(DevTab tp, int d3k, int nelt, GeoDev geo, FieldDev kap, const double* __restrict__ qx,
                    const double* __restrict__ qy, const double* __restrict__ qz, const double* __restrict__ u,
                    double* __restrict__ ustar) {
  extern __shared__ double psm[];
  __shared__ unsigned char pk_i[kPost2MaxNS], pk_j[kPost2MaxNS];  // packed index -> (row, col)
  __shared__ double invd[kPost2Warps][40];                         // 1 / L(k,k) per warp
  const Post2Dims dm(tp.d3, tp.nq, d3k);
  for (int j = threadIdx.x; j < tp.d3; j += blockDim.x)
    for (int i = j; i < tp.d3; ++i) {
      const int p = pk_lower(i, j, tp.d3);
      pk_i[p] = static_cast<unsigned char>(i);
      pk_j[p] = static_cast<unsigned char>(j);
    }
  const int n = dm.n, nq = dm.nq, nq4 = dm.nq4, npad = dm.npad, ns = dm.ns;
  double* verts = psm + dm.off_verts;
  double* sg = psm + dm.off_sg;
  double* qc = psm + dm.off_qc;
  double* gm = psm + dm.off_gm;
  double* R = psm + dm.off_R;
  double* Rp = psm + dm.off_Rp;
  double* G = psm + dm.off_GS;
  double* Sp = psm + dm.off_GS;  // after R: packed S per element
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const double* qs[3] = {qx, qy, qz};

  for (long K0 = long(blockIdx.x) * kPost2EB; K0 < nelt; K0 += long(gridDim.x) * kPost2EB) {
    // ---- stage geometry, vertices, coefficients
    for (int idx = threadIdx.x; idx < kPost2EB * 32; idx += blockDim.x) {
      const int e = idx >> 5, i = idx & 31;
      const long K = K0 + e;
      double v = 0.0;
      if (K < nelt && i < 30) {
        if (i == 0) v = geo.volume[K];
        else if (i < 10) v = geo.piola[long(i - 1) * nelt + K];
        else if (i < 22) v = geo.normals[long(i - 10) * nelt + K];
        else if (i < 26) v = geo.T[long(i - 22) * nelt + K];
        else v = double(geo.perm[long(i - 26) * nelt + K]);
      }
      sg[idx] = v;
    }
    for (int idx = threadIdx.x; idx < 12 * kPost2EB; idx += blockDim.x) {
      const int c = idx / kPost2EB, e = idx - c * kPost2EB;
      const long K = K0 + e;
      verts[idx] = K < nelt ? geo.verts[long(c) * nelt + K] : 0.0;
    }
    for (int idx = threadIdx.x; idx < 3 * d3k * kPost2EB; idx += blockDim.x) {
      const int e = idx % kPost2EB, si = idx / kPost2EB, s = si / d3k, i = si - s * d3k;
      const long K = K0 + e;
      qc[idx] = K < nelt ? qs[s][K * d3k + i] : 0.0;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 12 * kPost2EB; idx += blockDim.x) {
      const int h = idx / kPost2EB, e = idx - h * kPost2EB;
      double v = 0.0;
      if (h < 9) {
        const double* a9 = sg + 32 * e + 1;
        const double detB = 6.0 * sg[32 * e];
        const int p = h / 3, r = h % 3;
        v = detB > 0.0 ? (a9[p] * a9[r] + a9[3 + p] * a9[3 + r] + a9[6 + p] * a9[6 + r]) / detB : 0.0;
      }
      gm[idx] = v;
    }
    // ---- G_#(q, e) at the P_{k+1} nodes (rows q >= nq are zero padding)
    for (int idx = threadIdx.x; idx < nq4 * kPost2EB; idx += blockDim.x) {
      const int q = idx / kPost2EB, e = idx - q * kPost2EB;
      const long K = K0 + e;
      double gv[3] = {0.0, 0.0, 0.0};
      if (q < nq && K < nelt) {
        const double l0 = __ldg(tp.bary + q), l1 = __ldg(tp.bary + nq + q), l2 = __ldg(tp.bary + 2 * nq + q),
                     l3 = __ldg(tp.bary + 3 * nq + q);
        const double* V = verts + e;
        const double x = l0 * V[0] + l1 * V[kPost2EB] + l2 * V[2 * kPost2EB] + l3 * V[3 * kPost2EB];
        const double y = l0 * V[4 * kPost2EB] + l1 * V[5 * kPost2EB] + l2 * V[6 * kPost2EB] + l3 * V[7 * kPost2EB];
        const double z = l0 * V[8 * kPost2EB] + l1 * V[9 * kPost2EB] + l2 * V[10 * kPost2EB] + l3 * V[11 * kPost2EB];
        const double wk = __ldg(tp.w + q) / eval_field(kap, x, y, z, q, K, nq);
        double Q0 = 0.0, Q1 = 0.0, Q2 = 0.0;
        for (int i = 0; i < d3k; ++i) {
          const double p = __ldg(tp.P + long(i) * nq + q);
          Q0 = fma(p, qc[(0 * d3k + i) * kPost2EB + e], Q0);
          Q1 = fma(p, qc[(1 * d3k + i) * kPost2EB + e], Q1);
          Q2 = fma(p, qc[(2 * d3k + i) * kPost2EB + e], Q2);
        }
        const double* a9 = sg + 32 * e + 1;
#pragma unroll
        for (int h = 0; h < 3; ++h) gv[h] = (Q0 * a9[h] + Q1 * a9[3 + h] + Q2 * a9[6 + h]) * wk;
      }
#pragma unroll
      for (int h = 0; h < 3; ++h) G[(h * nq4 + q) * kPost2LDG + e] = gv[h];
    }
    __syncthreads();

    // ---- R = -(1/6) Pd^T G: K split over the warps, all M-tiles per warp
    {
      const int mts = npad / 8, ks = 3 * nq4 / 4;
      const int k0 = warp * ks / kPost2Warps, k1 = (warp + 1) * ks / kPost2Warps;
      double acc[5][2];
#pragma unroll
      for (int m = 0; m < 5; ++m) acc[m][0] = acc[m][1] = 0.0;
      for (int kk = k0; kk < k1; ++kk) {
        const int k = kk * 4 + t, h = k / nq4, q = k - h * nq4;
        const double b = G[k * kPost2LDG + g];
        const double* Pd = tp.Pd + long(h) * nq * n;
#pragma unroll
        for (int m = 0; m < 5; ++m) {
          if (m >= mts) break;
          const int i = m * 8 + g;
          const double a = (q < nq && i < n) ? __ldg(Pd + long(i) * nq + q) : 0.0;
          dmma(acc[m][0], acc[m][1], a, b);
        }
      }
      for (int m = 0; m < mts; ++m) {
        double* P = Rp + (warp * npad + m * 8 + g) * kPost2EB + 2 * t;
        P[0] = acc[m][0];
        P[1] = acc[m][1];
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < npad * kPost2EB; idx += blockDim.x) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kPost2Warps; ++w) s += Rp[w * npad * kPost2EB + idx];
      R[idx] = -(1.0 / 6.0) * s;
    }
    // ---- S packed lower = ShatP^T-combination gm (G is dead: S overwrites it)
    {
      const int mts = dm.nsp / 8;
      for (int mt = warp; mt < mts; mt += kPost2Warps) {
        double c0 = 0.0, c1 = 0.0;
        const int idx = mt * 8 + g;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const int h = kk * 4 + t;
          const double a = (h < 9 && idx < ns) ? __ldg(tp.ShatP + long(h) * ns + idx) : 0.0;
          dmma(c0, c1, a, gm[h * kPost2EB + g]);
        }
        __syncwarp();
        if (idx < ns) {
          Sp[(2 * t) * dm.nsp + idx] = c0;
          Sp[(2 * t + 1) * dm.nsp + idx] = c1;
        }
      }
    }
    __syncthreads();

    // ---- per element: mean constraint, Cholesky of the trailing block, solves
    {
      const int e = warp;
      const long K = K0 + e;
      if (K < nelt) {
        double* S = Sp + e * dm.nsp;
        const double u0 = u[K * d3k];
        const int m = n - 1;  // trailing system rows 1..n-1 -> index 0..m-1
        double rr[2] = {0.0, 0.0};  // trailing rows lane, lane + 32 (n <= 35)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = 1 + lane + 32 * j;
          if (i < n) rr[j] = R[i * kPost2EB + e] - S[pk_lower(i, 0, n)] * u0;
        }
        // right-looking Cholesky on packed storage (full indices i, j >= 1):
        // the trailing triangle of columns > k is one contiguous packed range,
        // so its rank-1 update runs entry-parallel over all 32 lanes
        for (int k = 1; k < n; ++k) {
          const int ck = pk_lower(k, k, n);
          const double lkk = sqrt(S[ck]);
          const double inv = 1.0 / lkk;
          __syncwarp();
          if (lane == 0) {
            S[ck] = lkk;
            invd[warp][k - 1] = inv;
          }
          for (int i = k + 1 + lane; i < n; i += 32) S[ck + (i - k)] *= inv;
          __syncwarp();
          for (int p = ck + (n - k) + lane; p < ns; p += 32) {
            const int i = pk_i[p], j = pk_j[p];
            S[p] = fma(-S[ck + (i - k)], S[ck + (j - k)], S[p]);
          }
          __syncwarp();
        }
        // forward L y = r, then backward L^T x = y (trailing indices)
        for (int k = 0; k < m; ++k) {
          const int owner = k & 31, slot = k >> 5;
          double rk = slot == 0 ? rr[0] : rr[1];
          rk = __shfl_sync(0xffffffffu, rk, owner);
          const int ck = pk_lower(k + 1, k + 1, n);
          const double yk = rk * invd[warp][k];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int i = lane + 32 * j;
            if (i == k) rr[j] = yk;
            else if (i > k && i < m) rr[j] = fma(-S[ck + (i - k)], yk, rr[j]);
          }
        }
        for (int k = m - 1; k >= 0; --k) {
          const int owner = k & 31, slot = k >> 5;
          double yk = slot == 0 ? rr[0] : rr[1];
          yk = __shfl_sync(0xffffffffu, yk, owner);
          const double xk = yk * invd[warp][k];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int i = lane + 32 * j;
            if (i == k) rr[j] = xk;
            else if (i < k) rr[j] = fma(-S[pk_lower(k + 1, i + 1, n)], xk, rr[j]);
          }
        }
        if (lane == 0) ustar[K * n] = u0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = lane + 32 * j;
          if (i < m) ustar[K * n + 1 + i] = rr[j];
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace hdgb
