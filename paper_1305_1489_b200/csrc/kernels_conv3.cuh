// K7 v3 (k <= 2): convection_bilinear_matrices (convdiff.cpp:5-28), one warp
// per element.
//
//   vol = P^T G,           G(q, j) = sum_# gamma_#(q) dP_j/dxhat_#(x_q),
//                          gamma_#(q) = (w_q / 6) sum_* beta_*(x_q) a(*, #)
//   dp_l = Dperm[mu]^T diag(w_r beta.n_l) Pface_l      (face l, d2 x d3)
//   dd_l = Dperm[mu]^T diag(w_r beta.n_l) Dperm[mu]    (face l's diagonal block)
// (variable_convection_matrices, variable_surface_dp / _dd,
// element_matrices.cpp:130-256; beta at the element-parametrised face
// points, :72-82). Every product is a DMMA tile loop: vol with the shared P
// table as A and G formed fragment by fragment from gamma (per warp) and the
// dP tables; the face blocks with Dperm^T as A and the weighted Pface /
// Dperm rows as B. The element's vol, dp and dd (dd dense m x m with its
// off-diagonal blocks zero, as the reference layout) leave as contiguous
// 16-byte stores from a per-warp staging area. Round 2 replaced the
// CTA-batched v2 (16 elements per CTA: the volume block as one GEMM with the
// element as N over a 150 KB fragment-ordered table re-read from L2 per
// batch, the face blocks stored strided, a separate zero fill) — 4.5 ms at C4.
#pragma once

#include "dev_common.cuh"
#include "kernels_local.cuh"
#include "kernels_post.cuh"

namespace hdgb {

template <int K_>
struct Conv3Dims {
  static constexpr int D3 = cdim3(K_), D2 = cdim2(K_), M = 4 * cdim2(K_);
  static constexpr int NQ = cnq(2 * K_ + 2), NQD = cnqd(2 * K_ + 2);  // the default tet/tri rules
  static constexpr int NQP = round_up(NQ, 4), NQDP = round_up(NQD, 4);
  static constexpr int NT3 = (D3 + 7) / 8, NT2 = (D2 + 7) / 8;
  // [q][i] row strides: 4 or 12 (mod 16) doubles, conflict-free A/B fragment reads
  static constexpr int stride(int w) { return (w % 16 == 0 || w % 16 == 8) ? w + 4 : w; }  // w: a multiple of 8
  static constexpr int LP = stride(NT3 * 8), LD2 = stride(NT2 * 8);
  static constexpr int NPTS = NQ + 4 * NQD;
  // CTA tables: P, dP_0..2 ([q][i], NQP rows), Pface_l ([r][j], NQDP rows), Dperm_mu ([r][i])
  static constexpr int OFF_P = 0, OFF_PD = OFF_P + NQP * LP, OFF_PF = OFF_PD + 3 * NQP * LP;
  static constexpr int OFF_DM = OFF_PF + 4 * NQDP * LP;
  static constexpr int OFF_W = OFF_DM + 6 * NQDP * LD2;  // w_q / 6 (NQP), tri_w (NQDP)
  static constexpr int CTA_EXTRA = round_up(OFF_W + NQP + NQDP, 2);
  // per warp: geometry (32), verts (12 + pad), gamma (3 x NQP), face weights (4 x NQDP), staging
  static constexpr int W_SG = 0, W_VX = 32, W_GAM = 48, W_WB = W_GAM + 3 * NQP;
  static constexpr int W_OUT = round_up(W_WB + 4 * NQDP, 2);
  static constexpr int OUT_VOL = 0, OUT_DP = round_up(D3 * D3, 2), OUT_DD = OUT_DP + round_up(M * D3, 2);
  static constexpr int PER_WARP = W_OUT + OUT_DD + round_up(4 * D2 * D2, 2);
};

template <int K_> struct Conv3Cfg { static constexpr int NW = 16; };

template <int K_>
__global__ void __launch_bounds__(Conv3Cfg<K_>::NW * 32, 1)
convection3_kernel(DevTab tab, int nelt, GeoDev geo, FieldDev bx, FieldDev by, FieldDev bz,
                   double* __restrict__ vol, double* __restrict__ dp, double* __restrict__ dd) {
  using Dm = Conv3Dims<K_>;
  constexpr int NW = Conv3Cfg<K_>::NW;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, NQ = Dm::NQ, NQD = Dm::NQD, NQP = Dm::NQP,
                NQDP = Dm::NQDP, NT3 = Dm::NT3, NT2 = Dm::NT2, LP = Dm::LP, LD2 = Dm::LD2;
  extern __shared__ __align__(16) double csm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* Ps = csm + Dm::OFF_P;
  double* Pds = csm + Dm::OFF_PD;
  double* Pfs = csm + Dm::OFF_PF;
  double* Dms = csm + Dm::OFF_DM;
  double* Ws = csm + Dm::OFF_W;
  // ---- CTA tables (zero padded; the only CTA barrier)
  for (int idx = threadIdx.x; idx < 4 * NQP * LP; idx += blockDim.x) {
    const int h = idx / (NQP * LP), rem = idx - h * NQP * LP, q = rem / LP, i = rem - q * LP;
    double v = 0.0;
    if (q < NQ && i < D3) v = h == 0 ? tab.P[q + i * NQ] : tab.Pd[(h - 1) * NQ * D3 + q + i * NQ];
    csm[Dm::OFF_P + idx] = v;
  }
  for (int idx = threadIdx.x; idx < 4 * NQDP * LP; idx += blockDim.x) {
    const int l = idx / (NQDP * LP), rem = idx - l * NQDP * LP, r = rem / LP, j = rem - r * LP;
    Pfs[idx] = (r < NQD && j < D3) ? tab.Pface[l * NQD * D3 + r + j * NQD] : 0.0;
  }
  for (int idx = threadIdx.x; idx < 6 * NQDP * LD2; idx += blockDim.x) {
    const int mu = idx / (NQDP * LD2), rem = idx - mu * NQDP * LD2, r = rem / LD2, i = rem - r * LD2;
    Dms[idx] = (r < NQD && i < D2) ? tab.Dperm[mu * NQD * D2 + r + i * NQD] : 0.0;
  }
  for (int idx = threadIdx.x; idx < NQP + NQDP; idx += blockDim.x)
    Ws[idx] = idx < NQP ? (idx < NQ ? tab.w[idx] / 6.0 : 0.0) : (idx - NQP < NQD ? tab.tri_w[idx - NQP] : 0.0);
  double* W0 = csm + Dm::CTA_EXTRA + warp * Dm::PER_WARP;
  double* sg = W0 + Dm::W_SG;
  double* vx = W0 + Dm::W_VX;
  double* gam = W0 + Dm::W_GAM;
  double* wb = W0 + Dm::W_WB;
  double* out = W0 + Dm::W_OUT;
  for (int i = lane; i < Dm::PER_WARP; i += 32) W0[i] = 0.0;  // k-padding of gamma / wb stays zero
  __syncthreads();
  // beta: SAMPLED (the JIT sampler's layout K * NPTS + p), a constant, or an
  // interpreted program (when the sampler could not be compiled)
  const bool any_prog = bx.kind == HDG_FIELD_PROGRAM || by.kind == HDG_FIELD_PROGRAM || bz.kind == HDG_FIELD_PROGRAM;

  // this lane's inputs of element Kx, fetched one element ahead (their global
  // latency hides under the previous element's products): the geometry value
  // of lane < 30 and SAMPLED beta at the lane's points
  constexpr int NIT = (Dm::NPTS + 31) / 32;
  const FieldDev* F3[3] = {&bx, &by, &bz};
  double gv = 0.0, bv[NIT][3];
  auto fetch = [&](long Kx) {
    if (Kx >= nelt) return;
    if (lane < 30) {
      if (lane == 0) gv = geo.volume[Kx];
      else if (lane < 10) gv = geo.piola[long(lane - 1) * nelt + Kx];
      else if (lane < 22) gv = geo.normals[long(lane - 10) * nelt + Kx];
      else if (lane < 26) gv = 0.0;
      else gv = double(geo.perm[long(lane - 26) * nelt + Kx]);
    }
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int p = lane + 32 * it;
#pragma unroll
      for (int h = 0; h < 3; ++h)
        bv[it][h] = (p < Dm::NPTS && F3[h]->kind == HDG_FIELD_SAMPLED) ? __ldg(F3[h]->samples + Kx * Dm::NPTS + p)
                                                                        : F3[h]->value;
    }
  };
  const long wstride = long(gridDim.x) * NW;
  fetch(long(blockIdx.x) * NW + warp);
  for (long K = long(blockIdx.x) * NW + warp; K < nelt; K += wstride) {
    // ---- geometry: [0] volume, [1..9] a(s, #) at 1 + 3 s + #, [10..21] normals, [26..29] perm
    if (lane < 30) sg[lane] = gv;
    if (any_prog && lane < 12) vx[lane] = geo.verts[long(lane) * nelt + K];
    __syncwarp();
    // ---- beta: gamma_#(q) at the volume nodes, w_r beta.n_l at the face points
#pragma unroll
    for (int it = 0; it < NIT; ++it) {
      const int p = lane + 32 * it;
      if (p >= Dm::NPTS) break;
      int l = 0, r = 0;
      if (p >= NQ) {
        l = (p - NQ) / NQD;
        r = (p - NQ) - l * NQD;
      }
      double b0 = bv[it][0], b1 = bv[it][1], b2 = bv[it][2];
      if (any_prog) {  // the interpreter (the JIT sampler unavailable)
        double l0, l1, l2, l3;
        if (p < NQ) {
          l0 = __ldg(tab.bary + p), l1 = __ldg(tab.bary + NQ + p), l2 = __ldg(tab.bary + 2 * NQ + p),
          l3 = __ldg(tab.bary + 3 * NQ + p);
        } else {
          const double s = __ldg(tab.tri_bary + NQD + r), tt = __ldg(tab.tri_bary + 2 * NQD + r);
          const double px = l == 2 ? 0.0 : s, py = l == 1 ? 0.0 : (l == 2 ? s : tt),
                       pz = l == 0 ? 0.0 : (l == 3 ? 1.0 - s - tt : tt);
          l0 = 1.0 - (px + py + pz), l1 = px, l2 = py, l3 = pz;
        }
        const double x = l0 * vx[0] + l1 * vx[1] + l2 * vx[2] + l3 * vx[3];
        const double y = l0 * vx[4] + l1 * vx[5] + l2 * vx[6] + l3 * vx[7];
        const double z = l0 * vx[8] + l1 * vx[9] + l2 * vx[10] + l3 * vx[11];
        if (bx.kind == HDG_FIELD_PROGRAM) b0 = eval_field(bx, x, y, z, p, K, Dm::NPTS);
        if (by.kind == HDG_FIELD_PROGRAM) b1 = eval_field(by, x, y, z, p, K, Dm::NPTS);
        if (bz.kind == HDG_FIELD_PROGRAM) b2 = eval_field(bz, x, y, z, p, K, Dm::NPTS);
      }
      if (p < NQ) {
        const double wq = Ws[p];
#pragma unroll
        for (int h = 0; h < 3; ++h) gam[h * NQP + p] = wq * (b0 * sg[1 + h] + b1 * sg[4 + h] + b2 * sg[7 + h]);
      } else {
        wb[l * NQDP + r] = Ws[NQP + r] * (b0 * sg[10 + 3 * l] + b1 * sg[11 + 3 * l] + b2 * sg[12 + 3 * l]);
      }
    }
    __syncwarp();
    fetch(K + wstride);
    // ---- vol = P^T G: A(i, q) = P(q, i), B(q, j) = G(q, j) formed per fragment
    {
      double acc[NT3][NT3][2] = {};
#pragma unroll 2
      for (int kk = 0; kk < NQP / 4; ++kk) {
        const int q = 4 * kk + t;
        const double g0 = gam[q], g1 = gam[NQP + q], g2 = gam[2 * NQP + q];
        double a[NT3], b[NT3];
#pragma unroll
        for (int n = 0; n < NT3; ++n) {
          const int o = q * LP + 8 * n + g;
          a[n] = Ps[o];
          b[n] = g0 * Pds[o] + g1 * Pds[NQP * LP + o] + g2 * Pds[2 * NQP * LP + o];
        }
#pragma unroll
        for (int it = 0; it < NT3; ++it)
#pragma unroll
          for (int jt = 0; jt < NT3; ++jt) dmma(acc[it][jt][0], acc[it][jt][1], a[it], b[jt]);
      }
#pragma unroll
      for (int it = 0; it < NT3; ++it)
#pragma unroll
        for (int jt = 0; jt < NT3; ++jt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int i = 8 * it + g, j = 8 * jt + 2 * t + e;
            if (i < D3 && j < D3) out[Dm::OUT_VOL + i + j * D3] = acc[it][jt][e];
          }
    }
    // ---- faces: dp_l = D^T diag(wb_l) Pface_l, dd_l = D^T diag(wb_l) D
#pragma unroll 1
    for (int l = 0; l < 4; ++l) {
      const int mu = int(sg[26 + l]);
      const double* Dt = Dms + (mu - 1) * NQDP * LD2;
      const double* Pf = Pfs + l * NQDP * LP;
      const double* w = wb + l * NQDP;
      double cp[NT2][NT3][2] = {}, cd[NT2][NT2][2] = {};
#pragma unroll
      for (int kk = 0; kk < NQDP / 4; ++kk) {
        const int r = 4 * kk + t;
        const double wr = w[r];
        double a[NT2], bd[NT2], bp[NT3];
#pragma unroll
        for (int n = 0; n < NT2; ++n) {
          a[n] = Dt[r * LD2 + 8 * n + g];
          bd[n] = wr * a[n];
        }
#pragma unroll
        for (int n = 0; n < NT3; ++n) bp[n] = wr * Pf[r * LP + 8 * n + g];
#pragma unroll
        for (int it = 0; it < NT2; ++it) {
#pragma unroll
          for (int jt = 0; jt < NT3; ++jt) dmma(cp[it][jt][0], cp[it][jt][1], a[it], bp[jt]);
#pragma unroll
          for (int jt = 0; jt < NT2; ++jt) dmma(cd[it][jt][0], cd[it][jt][1], a[it], bd[jt]);
        }
      }
#pragma unroll
      for (int it = 0; it < NT2; ++it)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int i = 8 * it + g;
          if (i >= D2) continue;
#pragma unroll
          for (int jt = 0; jt < NT3; ++jt) {
            const int j = 8 * jt + 2 * t + e;
            if (j < D3) out[Dm::OUT_DP + (l * D2 + i) + j * M] = cp[it][jt][e];
          }
#pragma unroll
          for (int jt = 0; jt < NT2; ++jt) {
            const int j = 8 * jt + 2 * t + e;
            if (j < D2) out[Dm::OUT_DD + l * D2 * D2 + i + j * D2] = cd[it][jt][e];
          }
        }
    }
    __syncwarp();
    // ---- the element's blocks as contiguous runs
    if constexpr ((D3 * D3) % 2 == 0 && (M * D3) % 2 == 0) {
      const double2* sv = reinterpret_cast<const double2*>(out + Dm::OUT_VOL);
      double2* gv = reinterpret_cast<double2*>(vol + K * D3 * D3);
      for (int i = lane; i < D3 * D3 / 2; i += 32) gv[i] = sv[i];
      const double2* sp = reinterpret_cast<const double2*>(out + Dm::OUT_DP);
      double2* gp = reinterpret_cast<double2*>(dp + K * M * D3);
      for (int i = lane; i < M * D3 / 2; i += 32) gp[i] = sp[i];
    } else {
      for (int i = lane; i < D3 * D3; i += 32) vol[K * D3 * D3 + i] = out[Dm::OUT_VOL + i];
      for (int i = lane; i < M * D3; i += 32) dp[K * M * D3 + i] = out[Dm::OUT_DP + i];
    }
    {  // dd: dense m x m, nonzero only in the four d2 x d2 diagonal blocks (m even: pairs share a column)
      double2* gd = reinterpret_cast<double2*>(dd + K * M * M);
      const double* bl = out + Dm::OUT_DD;
      for (int i = lane; i < M * M / 2; i += 32) {
        const int o = 2 * i, c = o / M, r = o - c * M, lc = c / D2;
        double v[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int rr = r + e;
          v[e] = rr / D2 == lc ? bl[lc * D2 * D2 + (rr - lc * D2) + (c - lc * D2) * D2] : 0.0;
        }
        gd[i] = make_double2(v[0], v[1]);
      }
    }
    __syncwarp();
  }
}

}  // namespace hdgb
