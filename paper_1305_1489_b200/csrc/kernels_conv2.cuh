// K7 v2 (k <= 3): convection_bilinear_matrices (convdiff.cpp:5-28) for EB
// elements per CTA, the volume block as a DMMA GEMM with the element as the N
// dimension (the K2 pattern):
//   vol(i + j d3, e) = sum_{#, q} [P_qi dP_qj/dxhat_#] . gamma_#(q, e),
//   gamma_#(q, e) = (w_q / 6) sum_* beta_*(x_q) a_e(*, #)
// with the table [P_qi dP_qj/dxhat_#] (d3^2 x 3 nq, host-built in DMMA fragment
// order, L2-resident) as A and gamma (3 nq x EB, shared memory) as B. The face
// blocks use the element-parametrised face points (face_points_physical,
// element_matrices.cpp:72-82), the Dperm / Pface tables staged in shared
// memory once per CTA, and the per-face products as small DMMA tiles:
//   dp block l = sum_r w_r (beta.n_l)(x_r^l) Dperm[mu]_ri Pface_l rj
//   dd block l = sum_r w_r (beta.n_l)(x_r^l) Dperm[mu]_ri Dperm[mu]_rj
// (the rest of dd is zero). The warp-per-element convection_kernel stays for k >= 4.
#pragma once

#include "dev_common.cuh"
#include "kernels_local.cuh"
#include "kernels_post.cuh"

namespace hdgb {

constexpr int kConv2EB = 16, kConv2Threads = 256, kConv2LDE = kConv2EB + 4;

struct Conv2Dims {
  int nqp, rows, kc, off_g, off_bn, off_sg, off_dp, off_pf, total;
  __host__ __device__ Conv2Dims(int d3, int d2, int nq, int nqd) {
    nqp = (nq + 3) / 4 * 4;
    rows = (d3 * d3 + 7) / 8 * 8;   // table rows (i + j d3), padded to whole tiles
    kc = 3 * nqp / 4;               // DMMA k-steps
    off_g = 0;                                   // gamma: 3 nqp x LDE
    off_bn = off_g + 3 * nqp * kConv2LDE;        // EB x 4 x nqd face weights
    off_sg = off_bn + kConv2EB * 4 * nqd;        // EB x 32 geometry records
    off_dp = off_sg + kConv2EB * 32;             // 6 x nqd x d2 Dperm
    off_pf = off_dp + 6 * nqd * d2;              // 4 x nqd x d3 Pface
    total = off_pf + 4 * nqd * d3;
  }
};

// The convection points of degree tab.k: the nq volume nodes, then face l's
// element-parametrised points (face_points_physical, element_matrices.cpp:
// 72-82) for l = 0..3, as barycentric weights of the element's vertices
// (npts x 4, column-major): the JIT sampler's point table (SAMPLED beta is
// read at K * npts + point).
__global__ void conv_points_kernel(DevTab tab, double* __restrict__ out) {
  const int nq = tab.nq, nqd = tab.nqd, npts = nq + 4 * nqd;
  for (int p = threadIdx.x; p < npts; p += blockDim.x) {
    double b[4];
    if (p < nq) {
#pragma unroll
      for (int v = 0; v < 4; ++v) b[v] = tab.bary[v * nq + p];
    } else {
      const int l = (p - nq) / nqd, r = (p - nq) - l * nqd;
      const double s = tab.tri_bary[nqd + r], tt = tab.tri_bary[2 * nqd + r];
      const double px = l == 2 ? 0.0 : s, py = l == 1 ? 0.0 : (l == 2 ? s : tt),
                   pz = l == 0 ? 0.0 : (l == 3 ? 1.0 - s - tt : tt);
      b[0] = 1.0 - (px + py + pz);
      b[1] = px;
      b[2] = py;
      b[3] = pz;
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) out[v * npts + p] = b[v];
  }
}

template <int K_>
__global__ void __launch_bounds__(kConv2Threads)
convection2_kernel(DevTab tab, int nelt, GeoDev geo, FieldDev bx, FieldDev by, FieldDev bz, int npts,
                   double* __restrict__ vol, double* __restrict__ dp, double* __restrict__ dd) {
  extern __shared__ __align__(16) double csm[];
  constexpr int d3 = cdim3(K_), d2 = cdim2(K_), m = 4 * d2, dd3 = d3 * d3;
  const int nq = tab.nq, nqd = tab.nqd;  // rule-dependent
  const Conv2Dims cd(d3, d2, nq, nqd);
  double* gam = csm + cd.off_g;
  double* bn = csm + cd.off_bn;
  double* sg = csm + cd.off_sg;
  double* Dps = csm + cd.off_dp;
  double* Pfs = csm + cd.off_pf;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const bool any_prog = bx.kind == HDG_FIELD_PROGRAM || by.kind == HDG_FIELD_PROGRAM || bz.kind == HDG_FIELD_PROGRAM;
  for (int i = tid; i < 6 * nqd * d2; i += kConv2Threads) Dps[i] = tab.Dperm[i];
  for (int i = tid; i < 4 * nqd * d3; i += kConv2Threads) Pfs[i] = tab.Pface[i];
  for (int i = tid; i < 3 * cd.nqp * kConv2LDE; i += kConv2Threads) gam[i] = 0.0;  // node padding stays zero
  __syncthreads();
  for (long K0 = long(blockIdx.x) * kConv2EB; K0 < nelt; K0 += long(gridDim.x) * kConv2EB) {
    for (int idx = tid; idx < kConv2EB * 32; idx += kConv2Threads) {
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
    __syncthreads();
    // beta at the volume nodes -> gamma_# (B operand), and at the element's face points
    auto beta = [&](const FieldDev& F, double x, double y, double z, int p, long K) {
      return eval_field(F, x, y, z, p, K, npts);
    };
    for (int idx = tid; idx < kConv2EB * nq; idx += kConv2Threads) {
      const int e = idx / nq, q = idx - e * nq;
      const long K = K0 + e;
      double gv[3] = {0.0, 0.0, 0.0};
      if (K < nelt) {
        double x = 0.0, y = 0.0, z = 0.0;
        if (any_prog)
          elem_point(geo, K, nelt, __ldg(tab.bary + q), __ldg(tab.bary + nq + q), __ldg(tab.bary + 2 * nq + q),
                     __ldg(tab.bary + 3 * nq + q), x, y, z);
        const double b0 = beta(bx, x, y, z, q, K), b1 = beta(by, x, y, z, q, K), b2 = beta(bz, x, y, z, q, K);
        const double wq = __ldg(tab.w + q) / 6.0;
        const double* a9 = sg + 32 * e + 1;
#pragma unroll
        for (int h = 0; h < 3; ++h) gv[h] = wq * (b0 * a9[h] + b1 * a9[3 + h] + b2 * a9[6 + h]);
      }
#pragma unroll
      for (int h = 0; h < 3; ++h) gam[(h * cd.nqp + q) * kConv2LDE + e] = gv[h];
    }
    for (int idx = tid; idx < kConv2EB * 4 * nqd; idx += kConv2Threads) {
      const int e = idx / (4 * nqd), lr = idx - e * 4 * nqd, l = lr / nqd, r = lr - l * nqd;
      const long K = K0 + e;
      double v = 0.0;
      if (K < nelt) {
        const double s = __ldg(tab.tri_bary + nqd + r), tt = __ldg(tab.tri_bary + 2 * nqd + r);
        // face l's element-parametrised points (element_matrices.cpp:72-82)
        const double px = l == 2 ? 0.0 : s, py = l == 1 ? 0.0 : (l == 2 ? s : tt),
                     pz = l == 0 ? 0.0 : (l == 3 ? 1.0 - s - tt : tt);
        double x = 0.0, y = 0.0, z = 0.0;
        if (any_prog) elem_point(geo, K, nelt, 1.0 - (px + py + pz), px, py, pz, x, y, z);
        const int pp = nq + lr;  // this face point's index in the sampled layout
        const double b0 = beta(bx, x, y, z, pp, K), b1 = beta(by, x, y, z, pp, K), b2 = beta(bz, x, y, z, pp, K);
        const double* nrm = sg + 32 * e + 10;
        v = __ldg(tab.tri_w + r) * (b0 * nrm[3 * l] + b1 * nrm[3 * l + 1] + b2 * nrm[3 * l + 2]);
      }
      bn[idx] = v;
    }
    __syncthreads();
    // vol: DMMA GEMM, one row tile of the table per task, both element tiles
    for (int mt = warp; mt < cd.rows / 8; mt += kConv2Threads / 32) {
      double acc[kConv2EB / 8][2] = {};
      const double* A = tab.Aconv + long(mt) * cd.kc * 32 + lane;
#pragma unroll 4
      for (int kk = 0; kk < cd.kc; ++kk) {
        const double a = __ldg(A + kk * 32);
        const double* B = gam + (kk * 4 + t) * kConv2LDE + g;
#pragma unroll
        for (int nt = 0; nt < kConv2EB / 8; ++nt) dmma(acc[nt][0], acc[nt][1], a, B[nt * 8]);
      }
      const int idx = mt * 8 + g;
#pragma unroll
      for (int nt = 0; nt < kConv2EB / 8; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long K = K0 + nt * 8 + 2 * t + h;
          if (idx < dd3 && K < nelt) vol[K * dd3 + idx] = acc[nt][h];
        }
    }
    // face blocks as DMMA tiles, one (element, face) per warp task:
    //   dp_l = Dperm[mu]^T diag(w beta.n) Pface_l (d2 x d3), dd_l = Dperm[mu]^T diag(.) Dperm[mu] (d2 x d2)
    {
      const int ks = (nqd + 3) / 4;
      constexpr int mts = (d2 + 7) / 8, nts = (d3 + 7) / 8, nts2 = (d2 + 7) / 8;
      for (int task = warp; task < kConv2EB * 4; task += kConv2Threads / 32) {
        const int e = task >> 2, l = task & 3;
        const long K = K0 + e;
        if (K >= nelt) continue;
        const int mu = int(sg[32 * e + 26 + l]);
        const double* D = Dps + (mu - 1) * nqd * d2;
        const double* P = Pfs + l * nqd * d3;
        const double* w = bn + (e * 4 + l) * nqd;
#pragma unroll
        for (int mt = 0; mt < mts; ++mt) {
          const int i = mt * 8 + g;
#pragma unroll
          for (int nt = 0; nt < nts + nts2; ++nt) {
            const bool isdp = nt < nts;
            const int jb = (isdp ? nt : nt - nts) * 8, ncols = isdp ? d3 : d2;
            double c0 = 0.0, c1 = 0.0;
            for (int kk = 0; kk < ks; ++kk) {
              const int r = kk * 4 + t;
              const bool rk = r < nqd;
              const double a = (rk && i < d2) ? D[r + i * nqd] : 0.0;
              const int jc = jb + g;
              double b = 0.0;
              if (rk && jc < ncols) b = w[r] * (isdp ? P[r + jc * nqd] : D[r + jc * nqd]);
              dmma(c0, c1, a, b);
            }
            if (i < d2) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int jj = jb + 2 * t + h;
                if (jj >= ncols) continue;
                const double v = h ? c1 : c0;
                if (isdp) dp[K * m * d3 + (l * d2 + i) + long(jj) * m] = v;
                else dd[K * m * m + (l * d2 + i) + long(l * d2 + jj) * m] = v;
              }
            }
          }
        }
      }
      // the zero blocks of dd (l != l2), 16-byte stores (m is even)
      const long nz = (nelt - K0 < kConv2EB ? nelt - K0 : kConv2EB) * long(m * m / 2);
      for (long idx = tid; idx < nz; idx += kConv2Threads) {
        const int o = int(idx % (m * m / 2)) * 2;
        const int r = o % m, c = o / m;  // r even: r, r + 1 lie in the same d2 block only if d2 is even
        double2* dst = reinterpret_cast<double2*>(dd + K0 * m * m) + idx;
        const bool z0 = r / d2 != c / d2, z1 = (r + 1) / d2 != c / d2;
        if (z0 && z1) *dst = make_double2(0.0, 0.0);
        else if (z0) dd[K0 * m * m + 2 * idx] = 0.0;
        else if (z1) dd[K0 * m * m + 2 * idx + 1] = 0.0;
      }
    }
    __syncthreads();
  }
}

}  // namespace hdgb
