// K6 (P_{k+1} postprocess), K7 (convection block) and the materialised
// ElementMatrixSet kernel (matrix-level parity of the build step).
// One warp per element; per-node coefficient values staged in shared memory.
#pragma once

#include "dev_common.cuh"
#include "kernels_local.cuh"

namespace hdgb {

__device__ __forceinline__ void elem_point(const GeoDev& geo, long K, int nelt, double l0, double l1,
                                           double l2, double l3, double& x, double& y, double& z) {
  const double* V = geo.verts;
  x = l0 * V[K] + l1 * V[long(nelt) + K] + l2 * V[2L * nelt + K] + l3 * V[3L * nelt + K];
  y = l0 * V[4L * nelt + K] + l1 * V[5L * nelt + K] + l2 * V[6L * nelt + K] + l3 * V[7L * nelt + K];
  z = l0 * V[8L * nelt + K] + l1 * V[9L * nelt + K] + l2 * V[10L * nelt + K] + l3 * V[11L * nelt + K];
}

// ------------------------------------------------------------------ K6
// postprocess_star (postprocess.cpp:33-74):
//   S = sum_{#,#'} (a^T a)_{##'}/detB Shat_{##'}           (stiffness_matrices)
//   R = -(1/6) sum_# Pd_#^T diag(w) G_#,  G_# = sum_s kappa^-1 (Pk q_s) a(s,#)
//   row 0 <- [detB/sqrt6, 0, ...], rhs 0 <- detB/sqrt6 u_0   (mean constraint)
// Because S's constant row/column vanish, the system splits into u*_0 = u_0 and
// an SPD solve on the trailing block, done here by Cholesky.
// One warp per element. Shared memory per warp: S lower (n x ldS, ldS odd so
// row walks are conflict-free), G (3 nq), q/u coefficients, geometry. R is
// accumulated lane-per-row with four independent chains; the triangular
// solves keep the right-hand side in registers (lane owns rows lane, lane+32,
// lane+64) and broadcast each solved entry by shuffle.
constexpr int kPostWarps = 4;
__host__ __device__ constexpr int post_ld(int n) { return n | 1; }
__host__ __device__ constexpr int post_per_warp(int n, int nq, int d3k) {
  return n * post_ld(n) + 3 * nq + 3 * d3k + 32 + 8;
}

__global__ void __launch_bounds__(kPostWarps * 32)
postprocess_kernel(DevTab tp, int d3k, int nelt, GeoDev geo, FieldDev kap, const double* __restrict__ qx,
                   const double* __restrict__ qy, const double* __restrict__ qz, const double* __restrict__ u,
                   double* __restrict__ ustar, int per_warp) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = tp.d3, nq = tp.nq, ld = post_ld(n);
  double* S = smem + long(warp) * per_warp;
  double* G = S + n * ld;       // 3 x nq
  double* qc = G + 3 * nq;      // 3 x d3k
  double* sg = qc + 3 * d3k;    // geometry (32)
  const double* qs[3] = {qx, qy, qz};
  for (long K = long(blockIdx.x) * kPostWarps + warp; K < nelt; K += long(gridDim.x) * kPostWarps) {
    load_geo(geo, K, nelt, sg, lane, 32);
    for (int idx = lane; idx < 3 * d3k; idx += 32) {
      const int s = idx / d3k, i = idx - s * d3k;
      qc[idx] = qs[s][K * d3k + i];
    }
    __syncwarp();
    const double* a9 = sg + 1;
    const double detB = 6.0 * sg[0];
    // G_# at the nodes
    for (int q = lane; q < nq; q += 32) {
      double x, y, z;
      elem_point(geo, K, nelt, __ldg(tp.bary + q), __ldg(tp.bary + nq + q), __ldg(tp.bary + 2 * nq + q),
                 __ldg(tp.bary + 3 * nq + q), x, y, z);
      const double kinv = 1.0 / eval_field(kap, x, y, z, q, K, nq);
      double Qv[3] = {0.0, 0.0, 0.0};
      for (int i = 0; i < d3k; ++i) {
        const double p = __ldg(tp.P + long(i) * nq + q);
        Qv[0] = fma(p, qc[i], Qv[0]);
        Qv[1] = fma(p, qc[d3k + i], Qv[1]);
        Qv[2] = fma(p, qc[2 * d3k + i], Qv[2]);
      }
      const double wk = kinv * __ldg(tp.w + q);
#pragma unroll
      for (int h = 0; h < 3; ++h) G[h * nq + q] = (Qv[0] * a9[h] + Qv[1] * a9[3 + h] + Qv[2] * a9[6 + h]) * wk;
    }
    __syncwarp();
    // R(i), i >= 1 (row 0 is the mean constraint): full rounds lane per row
    // (4 chains); the < 8 rows of a ragged last round are split over the
    // lanes along the nodes and warp-reduced instead.
    const double u0 = u[K * d3k];
    double rr[3] = {0.0, 0.0, 0.0};  // rows 1 + lane + 32 j of the trailing system
    const int m = n - 1;
    const int rag = m & 31;                       // rows in the last round
    const int lane_rounds = (m >> 5) + (rag >= 8 ? 1 : 0);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int i = 1 + lane + 32 * j;
      if (j >= lane_rounds || i >= n) continue;
      double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
      for (int h = 0; h < 3; ++h) {
        const double* Pd = tp.Pd + long(h) * nq * n + long(i) * nq;
        const double* Gh = G + h * nq;
        int q = 0;
        for (; q + 3 < nq; q += 4) {
          c0 = fma(__ldg(Pd + q), Gh[q], c0);
          c1 = fma(__ldg(Pd + q + 1), Gh[q + 1], c1);
          c2 = fma(__ldg(Pd + q + 2), Gh[q + 2], c2);
          c3 = fma(__ldg(Pd + q + 3), Gh[q + 3], c3);
        }
        for (; q < nq; ++q) c0 = fma(__ldg(Pd + q), Gh[q], c0);
      }
      rr[j] = -(1.0 / 6.0) * ((c0 + c1) + (c2 + c3));
    }
    if (rag > 0 && rag < 8) {
      const int jr = m >> 5;
      for (int rr_i = 0; rr_i < rag; ++rr_i) {
        const int i = 1 + 32 * jr + rr_i;
        double c = 0.0;
        for (int h = 0; h < 3; ++h) {
          const double* Pd = tp.Pd + long(h) * nq * n + long(i) * nq;
          for (int q = lane; q < nq; q += 32) c = fma(__ldg(Pd + q), G[h * nq + q], c);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == rr_i) rr[jr] = -(1.0 / 6.0) * c;
      }
    }
    // S, lower triangle (stiffness_matrices, element_matrices.cpp:258-280)
    double gm[9];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int r = 0; r < 3; ++r)
        gm[3 * p + r] = (a9[p] * a9[r] + a9[3 + p] * a9[3 + r] + a9[6 + p] * a9[6 + r]) / detB;
    for (int j = 0; j < n; ++j)
      for (int i = j + lane; i < n; i += 32) {
        const long idx = i + long(j) * n;
        double v = 0.0;
#pragma unroll
        for (int h = 0; h < 9; ++h) v = fma(__ldg(tp.Shat + long(h) * n * n + idx), gm[h], v);
        S[i + j * ld] = v;
      }
    __syncwarp();
    // trailing SPD block: S[1:,1:] x = R[1:] - S[1:,0] u0
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int i = 1 + lane + 32 * j;
      if (i < n) rr[j] -= S[i] * u0;
    }
    Team<1> tm;
    tm.id = 0;
    tm.tid = lane;
    tm.warp = 0;
    tm.lane = lane;
    double* L = S + 1 + ld;  // trailing block, (n-1) x (n-1), stride ld
    team_cholesky(tm, L, ld, m, G);  // scratch: G is dead after R
    __syncwarp();
    // forward L y = r: column sweep, y_k broadcast from its owner lane
    for (int k = 0; k < m; ++k) {
      const int owner = k & 31, slot = k >> 5;
      double rk = slot == 0 ? rr[0] : (slot == 1 ? rr[1] : rr[2]);
      rk = __shfl_sync(0xffffffffu, rk, owner);
      const double yk = rk / L[k + k * ld];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int i = lane + 32 * j;
        if (i == k) rr[j] = yk;
        else if (i > k && i < m) rr[j] = fma(-L[i + k * ld], yk, rr[j]);
      }
    }
    // backward L^T x = y: row k of L^T is column k of L
    for (int k = m - 1; k >= 0; --k) {
      const int owner = k & 31, slot = k >> 5;
      double yk = slot == 0 ? rr[0] : (slot == 1 ? rr[1] : rr[2]);
      yk = __shfl_sync(0xffffffffu, yk, owner);
      const double xk = yk / L[k + k * ld];
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int i = lane + 32 * j;
        if (i == k) rr[j] = xk;
        else if (i < k) rr[j] = fma(-L[k + i * ld], xk, rr[j]);
      }
    }
    if (lane == 0) ustar[K * n] = u0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int i = lane + 32 * j;
      if (i < m) ustar[K * n + 1 + i] = rr[j];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ K7
// convection_bilinear_matrices (convdiff.cpp:5-28):
//   vol(i,j) = sum_q (w_q/6) P_qi sum_# gamma_#(q) dP_qj/dx#,  gamma_# = sum_* beta_* a(*,#)
//   dp block l = sum_r w_r (beta.n_l)(x_r^l) Dperm[mu]_ri Pface_l rj
//   dd block l = sum_r w_r (beta.n_l)(x_r^l) Dperm[mu]_ri Dperm[mu]_rj
// beta sampled at element-parametrised face points (element_matrices.cpp:72-82).
__global__ void convection_kernel(DevTab tab, int nelt, GeoDev geo, FieldDev bx, FieldDev by,
                                  FieldDev bz, double* __restrict__ vol, double* __restrict__ dp,
                                  double* __restrict__ dd, int per_warp) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int d3 = tab.d3, d2 = tab.d2, nq = tab.nq, nqd = tab.nqd, m = 4 * d2;
  double* gam = smem + long(warp) * per_warp;  // 3 x nq
  double* bn = gam + 3 * nq;                    // 4 x nqd
  double* sg = bn + 4 * nqd;
  for (long K = long(blockIdx.x) * nw + warp; K < nelt; K += long(gridDim.x) * nw) {
    load_geo(geo, K, nelt, sg, lane, 32);
    __syncwarp();
    const double* a9 = sg + 1;
    const double* nrm = sg + 10;
    for (int q = lane; q < nq; q += 32) {
      double x, y, z;
      elem_point(geo, K, nelt, __ldg(tab.bary + q), __ldg(tab.bary + nq + q),
                 __ldg(tab.bary + 2 * nq + q), __ldg(tab.bary + 3 * nq + q), x, y, z);
      const double b0 = eval_field(bx, x, y, z, q, K, nq), b1 = eval_field(by, x, y, z, q, K, nq),
                   b2 = eval_field(bz, x, y, z, q, K, nq);
      const double wq = __ldg(tab.w + q) / 6.0;
      for (int h = 0; h < 3; ++h) gam[h * nq + q] = wq * (b0 * a9[h] + b1 * a9[3 + h] + b2 * a9[6 + h]);
    }
    for (int idx = lane; idx < 4 * nqd; idx += 32) {
      const int l = idx / nqd, r = idx - l * nqd;
      const double s = __ldg(tab.tri_bary + nqd + r), t = __ldg(tab.tri_bary + 2 * nqd + r);
      const double px[4] = {s, s, 0.0, s}, py[4] = {t, 0.0, s, t}, pz[4] = {0.0, t, t, 1.0 - s - t};
      double x, y, z;
      elem_point(geo, K, nelt, 1.0 - (px[l] + py[l] + pz[l]), px[l], py[l], pz[l], x, y, z);
      const double b0 = eval_field(bx, x, y, z, r, K, nqd), b1 = eval_field(by, x, y, z, r, K, nqd),
                   b2 = eval_field(bz, x, y, z, r, K, nqd);
      bn[idx] = __ldg(tab.tri_w + r) * (b0 * nrm[3 * l] + b1 * nrm[3 * l + 1] + b2 * nrm[3 * l + 2]);
    }
    __syncwarp();
    for (int idx = lane; idx < d3 * d3; idx += 32) {
      const int i = idx % d3, j = idx / d3;
      double acc = 0.0;
      for (int q = 0; q < nq; ++q) {
        const double pi = __ldg(tab.P + long(i) * nq + q);
        acc += pi * (gam[q] * __ldg(tab.Pd + long(j) * nq + q) +
                     gam[nq + q] * __ldg(tab.Pd + long(nq) * d3 + long(j) * nq + q) +
                     gam[2 * nq + q] * __ldg(tab.Pd + 2L * nq * d3 + long(j) * nq + q));
      }
      vol[K * d3 * d3 + idx] = acc;
    }
    for (int idx = lane; idx < m * d3; idx += 32) {
      const int r = idx % m, j = idx / m;
      const int l = r / d2, i = r - l * d2;
      const int mu = int(sg[26 + l]);
      const double* Dp = tab.Dperm + long(mu - 1) * nqd * d2 + long(i) * nqd;
      const double* Pf = tab.Pface + long(l) * nqd * d3 + long(j) * nqd;
      double acc = 0.0;
      for (int q = 0; q < nqd; ++q) acc += bn[l * nqd + q] * __ldg(Dp + q) * __ldg(Pf + q);
      dp[K * m * d3 + idx] = acc;
    }
    for (int idx = lane; idx < m * m; idx += 32) {
      const int r = idx % m, c = idx / m;
      const int l = r / d2, l2 = c / d2;
      double acc = 0.0;
      if (l == l2) {
        const int mu = int(sg[26 + l]);
        const double* Di = tab.Dperm + long(mu - 1) * nqd * d2 + long(r - l * d2) * nqd;
        const double* Dj = tab.Dperm + long(mu - 1) * nqd * d2 + long(c - l * d2) * nqd;
        for (int q = 0; q < nqd; ++q) acc += bn[l * nqd + q] * __ldg(Di + q) * __ldg(Dj + q);
      }
      dd[K * m * m + idx] = acc;
    }
    __syncwarp();
  }
}

// --------------------------------------------- materialised ElementMatrixSet
// build_element_matrices (element_matrices.cpp:282-309) entry by entry, for
// matrix-level parity; not on the hot path.
struct EmsOut {
  double *Mkinv, *Mc, *Cx, *Cy, *Cz, *tauPP, *tauDP, *nxDP, *nyDP, *nzDP, *tauDD, *fvec;
};
__global__ void element_matrices_kernel(DevTab tab, int nelt, GeoDev geo, FieldDev kap, FieldDev cc,
                                        FieldDev ff, EmsOut o, int per_warp) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int d3 = tab.d3, d2 = tab.d2, nq = tab.nq, m = 4 * d2;
  double* mk = smem + long(warp) * per_warp;  // 3 x nq: w kinv, w c, w f
  double* sg = mk + 3 * nq;
  for (long K = long(blockIdx.x) * nw + warp; K < nelt; K += long(gridDim.x) * nw) {
    load_geo(geo, K, nelt, sg, lane, 32);
    __syncwarp();
    const double vol = sg[0];
    const double* a9 = sg + 1;
    const double* nrm = sg + 10;
    const double* Tl = sg + 22;
    for (int q = lane; q < nq; q += 32) {
      double x, y, z;
      elem_point(geo, K, nelt, __ldg(tab.bary + q), __ldg(tab.bary + nq + q),
                 __ldg(tab.bary + 2 * nq + q), __ldg(tab.bary + 3 * nq + q), x, y, z);
      const double w = __ldg(tab.w + q);
      mk[q] = w * (1.0 / eval_field(kap, x, y, z, q, K, nq));
      mk[nq + q] = w * eval_field(cc, x, y, z, q, K, nq);
      mk[2 * nq + q] = w * eval_field(ff, x, y, z, q, K, nq);
    }
    __syncwarp();
    for (int idx = lane; idx < d3 * d3; idx += 32) {
      const int i = idx % d3, j = idx / d3;
      double s1 = 0.0, s2 = 0.0;
      for (int q = 0; q < nq; ++q) {
        const double pp = __ldg(tab.P + long(i) * nq + q) * __ldg(tab.P + long(j) * nq + q);
        s1 += pp * mk[q];
        s2 += pp * mk[nq + q];
      }
      if (o.Mkinv) o.Mkinv[K * d3 * d3 + idx] = s1 * vol;
      if (o.Mc) o.Mc[K * d3 * d3 + idx] = s2 * vol;
      double* Cs[3] = {o.Cx, o.Cy, o.Cz};
      for (int s = 0; s < 3; ++s)
        if (Cs[s]) {
          double acc = 0.0;
          for (int h = 0; h < 3; ++h) acc += __ldg(tab.Chat + long(h) * d3 * d3 + idx) * a9[3 * s + h];
          Cs[s][K * d3 * d3 + idx] = acc;
        }
      if (o.tauPP) {
        double acc = 0.0;
        for (int l = 0; l < 4; ++l) acc += __ldg(tab.PP + long(l) * d3 * d3 + idx) * Tl[l];
        o.tauPP[K * d3 * d3 + idx] = acc;
      }
    }
    for (int i = lane; i < d3 && o.fvec; i += 32) {
      double acc = 0.0;
      for (int q = 0; q < nq; ++q) acc += __ldg(tab.P + long(i) * nq + q) * mk[2 * nq + q];
      o.fvec[K * d3 + i] = acc * vol;
    }
    for (int idx = lane; idx < m * d3; idx += 32) {
      const int r = idx % m, j = idx / m;
      const int l = r / d2, i = r - l * d2;
      const int mu = int(sg[26 + l]);
      const double w = __ldg(tab.Wlm + long(6 * l + mu - 1) * d2 * d3 + i + long(j) * d2);
      if (o.tauDP) o.tauDP[K * m * d3 + idx] = Tl[l] * w;
      if (o.nxDP) o.nxDP[K * m * d3 + idx] = nrm[3 * l] * w;
      if (o.nyDP) o.nyDP[K * m * d3 + idx] = nrm[3 * l + 1] * w;
      if (o.nzDP) o.nzDP[K * m * d3 + idx] = nrm[3 * l + 2] * w;
    }
    for (int idx = lane; idx < m * m && o.tauDD; idx += 32) {
      const int r = idx % m, c = idx / m;
      const int l = r / d2, l2 = c / d2;
      o.tauDD[K * m * m + idx] = l == l2 ? Tl[l] * __ldg(tab.DD + (r - l * d2) + (c - l2 * d2) * d2) : 0.0;
    }
    __syncwarp();
  }
}

}  // namespace hdgb
