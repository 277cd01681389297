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
// memory). Then each warp owns one element: mean constraint row, and the
// trailing SPD system by the register sweep inverse of kernels_condense2.cuh
// (lane c owns column c) for m <= 32, plus a Schur-complement border beyond.
#pragma once

#include "dev_common.cuh"
#include "kernels_local.cuh"
#include "kernels_post.cuh"

namespace hdgb {

constexpr int kPost2EB = 16;    // elements per CTA (two DMMA N-tiles)
constexpr int kPost2NT = kPost2EB / 8;
constexpr int kPost2Warps = 16;  // one warp per element in the solve phase
constexpr int kPost2LDE = kPost2EB + 4;  // [row][e] operand rows: B-fragment reads conflict-free

struct Post2Dims {
  int n, nq, nq4, d3k, npad, ns, nsp;
  int off_verts, off_sg, off_qc, off_gm, off_R, off_Rp, off_GS, off_ks, off_nx, nx, total;
  __host__ __device__ Post2Dims(int n_, int nq_, int d3k_) : n(n_), nq(nq_), d3k(d3k_) {
    nq4 = (nq + 3) / 4 * 4;
    npad = (n + 7) / 8 * 8;
    ns = n * (n + 1) / 2;
    nsp = (ns + 7) / 8 * 8;
    off_verts = 0;                                    // 12 x EB
    off_sg = off_verts + 12 * kPost2EB;               // 32 x EB geometry records
    off_qc = off_sg + 32 * kPost2EB;                  // 3 x d3k x LDE
    off_gm = off_qc + 3 * d3k * kPost2LDE;            // 12 x LDE (rows 9..11 zero)
    off_R = off_gm + 12 * kPost2LDE;                  // npad x EB
    off_Rp = off_R + npad * kPost2EB;                 // 3 x npad x EB partials | solve scratch
    const int rp = 3 * npad * kPost2EB, solve = kPost2Warps * (128 + 64);
    off_GS = off_Rp + (rp > solve ? rp : solve);      // G (3 nq4 x LDE) | S (EB x nsp)
    const int g = 3 * nq4 * kPost2LDE, sgs = kPost2EB * nsp;
    off_ks = off_GS + (g > sgs ? g : sgs);            // 2 x nq x EB: sampled kappa (double buffer)
    // the next batch's staging (cp.async, copied into verts / sg / qc at the
    // batch start): 12 x EB verts, 10 x EB geometry (volume, a), 3 d3k x EB q
    off_nx = off_ks + 2 * nq * kPost2EB;
    nx = (12 + 10 + 3 * d3k) * kPost2EB;
    total = off_nx + nx;
  }
};

__device__ __forceinline__ int pk_lower(int i, int j, int n) { return j * n - j * (j - 1) / 2 + (i - j); }

template <int M_>  // trailing system size n - 1
__global__ void __launch_bounds__(kPost2Warps * 32, 1)
postprocess2_kernel(DevTab tp, int d3k, int nelt, GeoDev geo, FieldDev kap, int kap_wdiv, const double* __restrict__ qx,
                    const double* __restrict__ qy, const double* __restrict__ qz, const double* __restrict__ u,
                    double* __restrict__ ustar) {
  extern __shared__ double psm[];
  const Post2Dims dm(tp.d3, tp.nq, d3k);
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
  // sampled kappa^-1 at the nodes: the next batch's samples stream in by
  // cp.async while this batch computes (the samples are the kernel's main
  // HBM stream)
  const bool sampled = kap.kind == HDG_FIELD_SAMPLED;
  auto prefetch_kappa = [&](long Kb, int buf) {
    const long cnt = (nelt - Kb < kPost2EB ? nelt - Kb : kPost2EB) * long(nq);
    double* dst = psm + dm.off_ks + buf * nq * kPost2EB;
    for (long i = threadIdx.x; i < cnt; i += blockDim.x) cp_async8(dst + i, kap.samples + Kb * nq + i);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // the inputs of batch Kb -> the staging buffer (one cp.async group with the
  // kappa samples): element-fastest, so each source array is read coalesced
  double* nxb = psm + dm.off_nx;
  const bool need_x = kap.kind == HDG_FIELD_PROGRAM;  // the vertices only for an interpreted kappa
  auto prefetch_batch = [&](long Kb) {
    const int ne = int(nelt - Kb < kPost2EB ? nelt - Kb : kPost2EB);
    for (int idx = threadIdx.x; idx < (22 + 3 * d3k) * kPost2EB; idx += blockDim.x) {
      const int r = idx / kPost2EB, e = idx - r * kPost2EB;
      if (e >= ne || (r < 12 && !need_x)) continue;
      const long K = Kb + e;
      const double* src;
      if (r < 12) src = geo.verts + long(r) * nelt + K;
      else if (r == 12) src = geo.volume + K;
      else if (r < 22) src = geo.piola + long(r - 13) * nelt + K;
      else {
        const int s = (r - 22) / d3k, i = (r - 22) - s * d3k;
        src = qs[s] + K * d3k + i;
      }
      cp_async8(nxb + idx, src);
    }
  };
  int kbuf = 0;
  if (long(blockIdx.x) * kPost2EB < nelt) {
    prefetch_batch(long(blockIdx.x) * kPost2EB);
    if (sampled) prefetch_kappa(long(blockIdx.x) * kPost2EB, 0);  // (commits the group)
    else asm volatile("cp.async.commit_group;\n" ::: "memory");
  }

  for (long K0 = long(blockIdx.x) * kPost2EB; K0 < nelt; K0 += long(gridDim.x) * kPost2EB, kbuf ^= 1) {
    const long Kn0 = K0 + long(gridDim.x) * kPost2EB;
    // ---- this batch's geometry, vertices, coefficients from the staging buffer
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    for (int idx = threadIdx.x; idx < (22 + 3 * d3k) * kPost2EB; idx += blockDim.x) {
      const int r = idx / kPost2EB, e = idx - r * kPost2EB;
      const bool live = K0 + e < nelt;
      const double v = live ? nxb[idx] : 0.0;
      if (r < 12) verts[idx] = v;
      else if (r < 22) sg[32 * e + (r - 12)] = v;  // [0] volume, [1..9] a
      else qc[(r - 22) * kPost2LDE + e] = v;
    }
    __syncthreads();
    if (Kn0 < nelt) {  // the next batch's inputs stream in while this one computes
      prefetch_batch(Kn0);
      if (sampled) prefetch_kappa(Kn0, kbuf ^ 1);
      else asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    for (int idx = threadIdx.x; idx < 12 * kPost2EB; idx += blockDim.x) {
      const int h = idx / kPost2EB, e = idx - h * kPost2EB;
      double v = 0.0;
      if (h < 9) {
        const double* a9 = sg + 32 * e + 1;
        const double detB = 6.0 * sg[32 * e];
        const int p = h / 3, r = h % 3;
        v = detB > 0.0 ? (a9[p] * a9[r] + a9[3 + p] * a9[3 + r] + a9[6 + p] * a9[6 + r]) / detB : 0.0;
      }
      gm[h * kPost2LDE + e] = v;
    }
    // ---- G_#(q, e) at the P_{k+1} nodes (rows q >= nq are zero padding):
    //      Q_s = P_k^T qc_s as DMMA tiles (node rows, the 8 elements as N), the
    //      P_k fragment feeding the three components; then the Piola mix,
    //      weight and kappa^-1 in the epilogue
    {
      const int mts = (nq4 + 7) / 8, ksk = (d3k + 3) / 4;
      for (int mt = warp; mt < mts; mt += kPost2Warps) {
        double acc[3][kPost2NT][2] = {};
        const int qa = mt * 8 + g;
        for (int kk = 0; kk < ksk; ++kk) {
          const int i = kk * 4 + t;
          const double a = (qa < nq && i < d3k) ? __ldg(tp.P + long(i) * nq + qa) : 0.0;
#pragma unroll
          for (int s = 0; s < 3; ++s)
#pragma unroll
            for (int j = 0; j < kPost2NT; ++j)
              dmma(acc[s][j][0], acc[s][j][1], a, i < d3k ? qc[(s * d3k + i) * kPost2LDE + 8 * j + g] : 0.0);
        }
#pragma unroll
        for (int jh = 0; jh < 2 * kPost2NT; ++jh) {
          const int j = jh >> 1, h2 = jh & 1;
          const int e = 8 * j + 2 * t + h2;
          const long K = K0 + e;
          double gv[3] = {0.0, 0.0, 0.0};
          if (qa < nq && K < nelt) {
            double x = 0.0, y = 0.0, z = 0.0;
            if (kap.kind == HDG_FIELD_PROGRAM) {
              const double l0 = __ldg(tp.bary + qa), l1 = __ldg(tp.bary + nq + qa),
                           l2 = __ldg(tp.bary + 2 * nq + qa), l3 = __ldg(tp.bary + 3 * nq + qa);
              const double* V = verts + e;
              x = l0 * V[0] + l1 * V[kPost2EB] + l2 * V[2 * kPost2EB] + l3 * V[3 * kPost2EB];
              y = l0 * V[4 * kPost2EB] + l1 * V[5 * kPost2EB] + l2 * V[6 * kPost2EB] + l3 * V[7 * kPost2EB];
              z = l0 * V[8 * kPost2EB] + l1 * V[9 * kPost2EB] + l2 * V[10 * kPost2EB] + l3 * V[11 * kPost2EB];
            }
            const double kq = sampled ? psm[dm.off_ks + kbuf * nq * kPost2EB + e * nq + qa]
                                      : eval_field(kap, x, y, z, qa, K, nq);
            const double wk = kap_wdiv ? kq : __ldg(tp.w + qa) / kq;  // kap_wdiv: samples are w_q / kappa
            const double* a9 = sg + 32 * e + 1;
#pragma unroll
            for (int h = 0; h < 3; ++h)
              gv[h] = (acc[0][j][h2] * a9[h] + acc[1][j][h2] * a9[3 + h] + acc[2][j][h2] * a9[6 + h]) * wk;
          }
          if (qa < nq4) {
#pragma unroll
            for (int h = 0; h < 3; ++h) G[(h * nq4 + qa) * kPost2LDE + e] = gv[h];
          }
        }
      }
    }
    __syncthreads();

#ifndef HDG_K6_SKIP_R
    // ---- R = -(1/6) sum_# Pd_#^T G_#: one (row tile, component #) per warp,
    //      the Pd fragment feeding both element tiles; 3 partials reduced below
    {
      const int mts = npad / 8;
      for (int task = warp; task < 3 * mts; task += kPost2Warps) {
        const int h = task / mts, m = task - h * mts, i = m * 8 + g;
        const double* Pd = tp.Pd + long(h) * nq * n + long(i) * nq;
        const double* Gh = G + h * nq4 * kPost2LDE;
        double acc[kPost2NT][2][2] = {};  // two chains per tile (k-step parity)
#ifndef HDG_K6_RUNROLL
#define HDG_K6_RUNROLL 4
#endif
        constexpr int kRU = HDG_K6_RUNROLL;
#pragma unroll kRU
        for (int kk = 0; kk < nq4 / 4; ++kk) {
          const int q = kk * 4 + t;
          const double a = (q < nq && i < n) ? __ldg(Pd + q) : 0.0;
#pragma unroll
          for (int j = 0; j < kPost2NT; ++j)
            dmma(acc[j][kk & 1][0], acc[j][kk & 1][1], a, Gh[q * kPost2LDE + 8 * j + g]);
        }
#pragma unroll
        for (int j = 0; j < kPost2NT; ++j) {
          double* P = Rp + (h * npad + m * 8 + g) * kPost2EB + 8 * j + 2 * t;
          P[0] = acc[j][0][0] + acc[j][1][0];
          P[1] = acc[j][0][1] + acc[j][1][1];
        }
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < npad * kPost2EB; idx += blockDim.x)
      R[idx] = -(1.0 / 6.0) * (Rp[idx] + Rp[npad * kPost2EB + idx] + Rp[2 * npad * kPost2EB + idx]);
#endif
    // ---- S packed lower = ShatP^T-combination gm (G is dead: S overwrites it)
    {
      const int mts = dm.nsp / 8;
      for (int mt = warp; mt < mts; mt += kPost2Warps) {
        double c[kPost2NT][2] = {};
        const int idx = mt * 8 + g;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
          const int h = kk * 4 + t;
          const double a = (h < 9 && idx < ns) ? __ldg(tp.ShatP + long(h) * ns + idx) : 0.0;
#pragma unroll
          for (int j = 0; j < kPost2NT; ++j) dmma(c[j][0], c[j][1], a, gm[h * kPost2LDE + 8 * j + g]);
        }
        if (idx < ns) {
#pragma unroll
          for (int j = 0; j < kPost2NT; ++j) {
            Sp[(8 * j + 2 * t) * dm.nsp + idx] = c[j][0];
            Sp[(8 * j + 2 * t + 1) * dm.nsp + idx] = c[j][1];
          }
        }
      }
    }
    __syncthreads();

#ifndef HDG_K6_SKIP_SOLVE
    // ---- per element: mean constraint, then the trailing SPD system
    //      S' x = r' (m = n - 1 <= 32: register sweep inverse, lane c owns
    //      column c; 32 < m <= 64: the leading 32 x 32 block the same way and
    //      the (m - 32) border by its Schur complement)
    {
      const int e = warp;
      const long K = K0 + e;
      if (K < nelt) {
        const double* S = Sp + e * dm.nsp;
        const double u0 = u[K * d3k];
        constexpr int MA = M_ < 32 ? M_ : 32, MB = M_ - MA;  // leading block, border
        double* stage = Rp + warp * 128;                     // Rp is dead after the R reduction
        double* rs = Rp + kPost2Warps * 128 + warp * 64;     // right-hand side r' (m)
        for (int i = lane; i < M_; i += 32)
          rs[i] = R[(i + 1) * kPost2EB + e] - S[pk_lower(i + 1, 0, n)] * u0;
        auto Sat = [&](int i, int j) {  // S'(i, j), trailing indices, packed symmetric storage
          return i >= j ? S[pk_lower(i + 1, j + 1, n)] : S[pk_lower(j + 1, i + 1, n)];
        };
        double a[MA];
#pragma unroll
        for (int i = 0; i < MA; ++i) a[i] = lane < MA ? Sat(i, lane) : 0.0;
        __syncwarp();
        double pmin = 1e300, pmax = 0.0;
        gj_sweep_inverse<MA>(a, stage, lane, pmin, pmax);  // a = column `lane` of A^-1 (symmetric)
        // z = A^-1 r_A and, for the border, Y = A^-1 B: lane i holds row i (A^-1 symmetric)
        double z = 0.0;
#pragma unroll
        for (int j = 0; j < MA; ++j) z = fma(a[j], rs[j], z);
        double x = z;
        if constexpr (MB > 0) {
          double Y[MB];
#pragma unroll
          for (int b2 = 0; b2 < MB; ++b2) {
            double y = 0.0;
#pragma unroll
            for (int j = 0; j < MA; ++j) y = fma(a[j], Sat(j, MA + b2), y);
            Y[b2] = lane < MA ? y : 0.0;
          }
          // Schur complement Cs = C - B^T Y and rhs2 = r_B - B^T z (warp sums)
          double Cs[MB][MB], r2[MB];
#pragma unroll
          for (int p = 0; p < MB; ++p) {
            const double bp = lane < MA ? Sat(lane, MA + p) : 0.0;
            double v = bp * (lane < MA ? z : 0.0);
#pragma unroll
            for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            r2[p] = rs[MA + p] - v;
#pragma unroll
            for (int q = 0; q < MB; ++q) {
              double w = bp * Y[q];
#pragma unroll
              for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
              Cs[p][q] = Sat(MA + p, MA + q) - w;
            }
          }
          // x_B = Cs^-1 r2 (small SPD; Gaussian elimination, every lane redundantly)
#pragma unroll
          for (int c = 0; c < MB; ++c) {
            const double inv = 1.0 / Cs[c][c];
#pragma unroll
            for (int r = c + 1; r < MB; ++r) {
              const double f = Cs[r][c] * inv;
#pragma unroll
              for (int q = c; q < MB; ++q) Cs[r][q] -= f * Cs[c][q];
              r2[r] -= f * r2[c];
            }
          }
          double xb[MB];
#pragma unroll
          for (int c = MB - 1; c >= 0; --c) {
            double v = r2[c];
#pragma unroll
            for (int q = c + 1; q < MB; ++q) v -= Cs[c][q] * xb[q];
            xb[c] = v / Cs[c][c];
          }
#pragma unroll
          for (int b2 = 0; b2 < MB; ++b2) x = fma(-Y[b2], xb[b2], x);
#pragma unroll
          for (int b2 = 0; b2 < MB; ++b2)
            if (lane == b2) ustar[K * n + 1 + MA + b2] = xb[b2];
        }
        if (lane == 0) ustar[K * n] = u0;
        if (lane < MA) ustar[K * n + 1 + lane] = x;
      }
    }
#endif
    __syncthreads();
  }
}

}  // namespace hdgb
