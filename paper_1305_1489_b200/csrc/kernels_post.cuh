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
// Shared memory per warp: S (d31 x (d31+1)), R, G (3 nq), Q (3 nq), scratch.
__global__ void postprocess_kernel(DevTab tp, int d3k, int nelt, GeoDev geo, FieldDev kap,
                                   const double* __restrict__ qx, const double* __restrict__ qy,
                                   const double* __restrict__ qz, const double* __restrict__ u,
                                   double* __restrict__ ustar, int per_warp) {
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int n = tp.d3, nq = tp.nq, ld = n + 1;
  double* S = smem + long(warp) * per_warp;
  double* R = S + n * ld;
  double* G = R + round_up(n, 8);  // 3 x nq
  double* sg = G + 3 * nq;         // geometry (32)
  double* scr = sg + 32;           // n
  const double* qs[3] = {qx, qy, qz};
  Team<1> tm;
  tm.id = 0;
  tm.tid = lane;
  tm.warp = 0;
  tm.lane = lane;
  for (long K = long(blockIdx.x) * nw + warp; K < nelt; K += long(gridDim.x) * nw) {
    load_geo(geo, K, nelt, sg, lane, 32);
    __syncwarp();
    const double* a9 = sg + 1;
    const double detB = 6.0 * sg[0];
    // S
    double gm[9];
#pragma unroll
    for (int p = 0; p < 3; ++p)
#pragma unroll
      for (int r = 0; r < 3; ++r)
        gm[3 * p + r] = (a9[p] * a9[r] + a9[3 + p] * a9[3 + r] + a9[6 + p] * a9[6 + r]) / detB;
    for (int idx = lane; idx < n * n; idx += 32) {
      const int i = idx % n, j = idx / n;
      double s = 0.0;
#pragma unroll
      for (int h = 0; h < 9; ++h) s += __ldg(tp.Shat + long(h) * n * n + idx) * gm[h];
      S[i + j * ld] = s;
    }
    // G_# at nodes
    for (int q = lane; q < nq; q += 32) {
      double x, y, z;
      elem_point(geo, K, nelt, __ldg(tp.bary + q), __ldg(tp.bary + nq + q), __ldg(tp.bary + 2 * nq + q),
                 __ldg(tp.bary + 3 * nq + q), x, y, z);
      const double kinv = 1.0 / eval_field(kap, x, y, z, q, K, nq);
      double Qv[3];
      for (int s = 0; s < 3; ++s) {
        double acc = 0.0;
        for (int i = 0; i < d3k; ++i) acc += __ldg(tp.P + long(i) * nq + q) * qs[s][K * d3k + i];
        Qv[s] = acc * kinv;
      }
      for (int h = 0; h < 3; ++h) G[h * nq + q] = (Qv[0] * a9[h] + Qv[1] * a9[3 + h] + Qv[2] * a9[6 + h]) * __ldg(tp.w + q);
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) {
      double acc = 0.0;
      for (int h = 0; h < 3; ++h) {
        const double* Pd = tp.Pd + long(h) * nq * n + long(i) * nq;
        for (int q = 0; q < nq; ++q) acc += __ldg(Pd + q) * G[h * nq + q];
      }
      R[i] = -(1.0 / 6.0) * acc;
    }
    __syncwarp();
    const double u0 = u[K * d3k];
    // trailing SPD block: S[1:,1:] x = R[1:] - S[1:,0] u0
    for (int i = 1 + lane; i < n; i += 32) R[i] -= S[i] * u0;
    __syncwarp();
    team_cholesky(tm, S + 1 + ld, ld, n - 1, scr);
    // forward: L y = R[1:]
    for (int i = 1; i < n; ++i) {
      double part = 0.0;
      for (int k = 1 + lane; k < i; k += 32) part += S[i + k * ld] * R[k];
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) R[i] = (R[i] - part) / S[i + i * ld];
      __syncwarp();
    }
    // backward: L^T x = y
    for (int i = n - 1; i >= 1; --i) {
      double part = 0.0;
      for (int k = i + 1 + lane; k < n; k += 32) part += S[k + i * ld] * R[k];
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      if (lane == 0) R[i] = (R[i] - part) / S[i + i * ld];
      __syncwarp();
    }
    for (int i = lane; i < n; i += 32) ustar[K * n + i] = i == 0 ? u0 : R[i];
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
