// Error functionals and the HDG projection: compute_errors
// (postprocess.cpp:178-250) and hdg_project (postprocess.cpp:95-176) on the
// GPU, for on-device convergence studies (proj/README.md:80-82).
//
// Tables: tE = degree k on the error rule (tet/tri_rule(2k+4)), tE1 = degree
// k+1 on the same rule (for u*), t0 = the level's tables (the element
// matrices nDP, tauDP of hdg_project are built on the level's rules).
//
// hdg_project: the reference LU-solves a 4d3 system per element whose first
// 4t rows (t = d3 - d2) are 6|K| I on the leading coefficients, so those are
// x_{s,m} = (P^T w F_s)(m) / 6 directly; the remaining 4 d2 face rows,
// block (l, s) = xi_s(l) W_{l,mu}[:, t:] with xi = (n_x, n_y, n_z, T)(l),
// factor as blockdiag(W'_l) (Xi (x) I): one d2 x d2 inverse per (l, mu)
// (host, per level) and one 4x4 LU with partial pivoting per element.
#pragma once

#include "dev_common.cuh"
#include "kernels_local.cuh"

namespace hdgb {

constexpr int kErrWarps = 4;

struct ErrSums {  // per-block partials, summed on the host
  double v[9];
};

// physical point of reference-tet barycentric coordinates on element K
__device__ __forceinline__ void tet_point(const GeoDev& geo, long K, int nelt, double l0, double l1, double l2,
                                          double l3, double& x, double& y, double& z) {
  const double* V = geo.verts;
  x = l0 * V[0L * nelt + K] + l1 * V[1L * nelt + K] + l2 * V[2L * nelt + K] + l3 * V[3L * nelt + K];
  y = l0 * V[4L * nelt + K] + l1 * V[5L * nelt + K] + l2 * V[6L * nelt + K] + l3 * V[7L * nelt + K];
  z = l0 * V[8L * nelt + K] + l1 * V[9L * nelt + K] + l2 * V[10L * nelt + K] + l3 * V[11L * nelt + K];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------ hdg_project
// smem per warp: 4 nqE (w F at the volume nodes) + 4 nqdE (w g per face node)
// + 4 d3 (known/unknown coefficients) + 4 d2 (rhs) + 32
__global__ void __launch_bounds__(kErrWarps * 32)
hdg_project_kernel(DevTab tE, DevTab t0, int nelt, GeoDev geo, FieldDev fqx, FieldDev fqy, FieldDev fqz,
                   FieldDev fu, const double* __restrict__ winv, double* __restrict__ oqx, double* __restrict__ oqy,
                   double* __restrict__ oqz, double* __restrict__ ou, long long* bad, int per_warp) {
  extern __shared__ double esm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = tE.nq, nqd = tE.nqd, d3 = tE.d3, d2 = tE.d2, t = d3 - d2;
  double* wF = esm + warp * per_warp;  // 4 x nq
  double* wg = wF + 4 * nq;             // 4 x nqd
  double* X = wg + 4 * nqd;             // 4 x d3 coefficients (s-major)
  double* R = X + 4 * d3;               // 4 x d2 rhs / z
  double* sg = R + 4 * d2;              // 32: geometry record
  const FieldDev* F[4] = {&fqx, &fqy, &fqz, &fu};
  for (long K = long(blockIdx.x) * kErrWarps + warp; K < nelt; K += long(gridDim.x) * kErrWarps) {
    load_geo(geo, K, nelt, sg, lane, 32);
    for (int q = lane; q < nq; q += 32) {
      double x, y, z;
      tet_point(geo, K, nelt, tE.bary[q], tE.bary[nq + q], tE.bary[2 * nq + q], tE.bary[3 * nq + q], x, y, z);
      const double w = tE.w[q];
#pragma unroll
      for (int s = 0; s < 4; ++s) wF[s * nq + q] = w * eval_field(*F[s], x, y, z, q, K, nq);
    }
    __syncwarp();
    const double* nrm = sg + 10;
    const double* T = sg + 22;
    for (int idx = lane; idx < 4 * nqd; idx += 32) {  // element-parametrised face nodes
      const int l = idx / nqd, r = idx - l * nqd;
      const double s = tE.tri_bary[nqd + r], tt = tE.tri_bary[2 * nqd + r];
      const double px[4] = {s, s, 0.0, s}, py[4] = {tt, 0.0, s, tt}, pz[4] = {0.0, tt, tt, 1.0 - s - tt};
      double x, y, z;
      tet_point(geo, K, nelt, 1.0 - (px[l] + py[l] + pz[l]), px[l], py[l], pz[l], x, y, z);
      const double g = eval_field(fqx, x, y, z, r, K, nqd) * nrm[3 * l] +
                       eval_field(fqy, x, y, z, r, K, nqd) * nrm[3 * l + 1] +
                       eval_field(fqz, x, y, z, r, K, nqd) * nrm[3 * l + 2] + eval_field(fu, x, y, z, r, K, nqd) * T[l];
      wg[idx] = tE.tri_w[r] * g;
    }
    __syncwarp();
    // known coefficients x_{s,m} = (P^T w F_s)(m) / 6, m < t
    for (int idx = lane; idx < 4 * t; idx += 32) {
      const int s = idx / t, m = idx - s * t;
      const double* P = tE.P + long(m) * nq;
      double a = 0.0;
      for (int q = 0; q < nq; ++q) a += P[q] * wF[s * nq + q];
      X[s * d3 + m] = a / 6.0;
    }
    __syncwarp();
    // rhs_l(i) = Bmom(l, i) - sum_s xi_s(l) sum_{m<t} W_{l,mu}(i, m) x_{s,m}
    for (int idx = lane; idx < 4 * d2; idx += 32) {
      const int l = idx / d2, i = idx - l * d2;
      const int mu = int(sg[26 + l]);
      const double* Dp = tE.Dperm + long(mu - 1) * nqd * d2 + long(i) * nqd;
      double b = 0.0;
      for (int r = 0; r < nqd; ++r) b += Dp[r] * wg[l * nqd + r];
      const double* W = t0.Wlm + long(6 * l + mu - 1) * d2 * d3 + i;  // (i, m) at i + m d2
      const double xi[4] = {nrm[3 * l], nrm[3 * l + 1], nrm[3 * l + 2], T[l]};
      for (int s = 0; s < 4; ++s) {
        double a = 0.0;
        for (int m = 0; m < t; ++m) a += W[long(m) * d2] * X[s * d3 + m];
        b -= xi[s] * a;
      }
      R[idx] = b;
    }
    __syncwarp();
    // z_l = W'_l^-1 rhs_l
    for (int idx = lane; idx < 4 * d2; idx += 32) {
      double a = 0.0;
      const int l = idx / d2, i = idx - l * d2;
      const int mu = int(sg[26 + l]);
      const double* Wi = winv + long(6 * l + mu - 1) * d2 * d2;
      for (int j = 0; j < d2; ++j) a += Wi[i + long(j) * d2] * R[l * d2 + j];
      wg[idx] = a;  // z, reusing the face-node buffer (all face moments were consumed above)
    }
    __syncwarp();
    // Xi y_i = z_i per trace index i: Xi[l][s] = xi_s(l); 4x4 LU, partial pivoting
    double A[4][4];
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      A[l][0] = nrm[3 * l];
      A[l][1] = nrm[3 * l + 1];
      A[l][2] = nrm[3 * l + 2];
      A[l][3] = T[l];
    }
    int pr[4] = {0, 1, 2, 3};
    double pmin = 1e300, pmax = 6.0 * sg[0];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int p = c;
#pragma unroll
      for (int r = c + 1; r < 4; ++r)
        if (fabs(A[r][c]) > fabs(A[p][c])) p = r;
      if (p != c) {
#pragma unroll
        for (int j = 0; j < 4; ++j) { const double tmp = A[c][j]; A[c][j] = A[p][j]; A[p][j] = tmp; }
        const int ti = pr[c]; pr[c] = pr[p]; pr[p] = ti;
      }
      pmin = fmin(pmin, fabs(A[c][c]));
      pmax = fmax(pmax, fabs(A[c][c]));
      const double inv = A[c][c] != 0.0 ? 1.0 / A[c][c] : 0.0;
#pragma unroll
      for (int r = c + 1; r < 4; ++r) {
        A[r][c] *= inv;
#pragma unroll
        for (int j = c + 1; j < 4; ++j) A[r][j] -= A[r][c] * A[c][j];
      }
    }
    pmin = fmin(pmin, 6.0 * sg[0]);
    if (lane == 0 && (pmax == 0.0 || pmin < 1e-14 * pmax)) flag_bad(bad, K);
    for (int i = lane; i < d2; i += 32) {
      double y[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {  // forward (unit lower), permuted rhs
        double v = wg[pr[r] * d2 + i];
#pragma unroll
        for (int j = 0; j < r; ++j) v -= A[r][j] * y[j];
        y[r] = v;
      }
#pragma unroll
      for (int r = 3; r >= 0; --r) {
        double v = y[r];
#pragma unroll
        for (int j = r + 1; j < 4; ++j) v -= A[r][j] * y[j];
        y[r] = v / A[r][r];
      }
#pragma unroll
      for (int s = 0; s < 4; ++s) X[s * d3 + t + i] = y[s];
    }
    __syncwarp();
    double* out[4] = {oqx, oqy, oqz, ou};
    for (int idx = lane; idx < 4 * d3; idx += 32) {
      const int s = idx / d3, m = idx - s * d3;
      out[s][K * d3 + m] = X[idx];
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------ volume errors
// sums: 0 |q|^2, 1 |q - q_h|^2, 2 u^2, 3 (u - u_h)^2, 4 (u - u*)^2, 5 6|K| |proj_u - u_h|^2
__global__ void __launch_bounds__(kErrWarps * 32)
volume_errors_kernel(DevTab tE, DevTab tE1, int nelt, GeoDev geo, FieldDev fqx, FieldDev fqy, FieldDev fqz,
                     FieldDev fu, const double* __restrict__ qx, const double* __restrict__ qy,
                     const double* __restrict__ qz, const double* __restrict__ u, const double* __restrict__ ustar,
                     const double* __restrict__ proj_u, ErrSums* __restrict__ partial, int per_warp) {
  extern __shared__ double esm[];
  __shared__ double red[kErrWarps][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = tE.nq, d3 = tE.d3, d31 = tE1.d3;
  double* cf = esm + warp * per_warp;  // qx qy qz u (d3 each), u* (d31)
  double acc[6] = {0, 0, 0, 0, 0, 0};
  for (long K = long(blockIdx.x) * kErrWarps + warp; K < nelt; K += long(gridDim.x) * kErrWarps) {
    for (int i = lane; i < d3; i += 32) {
      cf[i] = qx[K * d3 + i];
      cf[d3 + i] = qy[K * d3 + i];
      cf[2 * d3 + i] = qz[K * d3 + i];
      cf[3 * d3 + i] = u[K * d3 + i];
    }
    if (ustar)
      for (int i = lane; i < d31; i += 32) cf[4 * d3 + i] = ustar[K * d31 + i];
    __syncwarp();
    const double vol = geo.volume[K];
    double e[5] = {0, 0, 0, 0, 0};
    for (int q = lane; q < nq; q += 32) {
      double x, y, z;
      tet_point(geo, K, nelt, tE.bary[q], tE.bary[nq + q], tE.bary[2 * nq + q], tE.bary[3 * nq + q], x, y, z);
      const double w = tE.w[q];
      const double ex[4] = {eval_field(fqx, x, y, z, q, K, nq), eval_field(fqy, x, y, z, q, K, nq),
                            eval_field(fqz, x, y, z, q, K, nq), eval_field(fu, x, y, z, q, K, nq)};
      double h[4] = {0, 0, 0, 0};
      for (int i = 0; i < d3; ++i) {
        const double p = tE.P[long(i) * nq + q];
#pragma unroll
        for (int s = 0; s < 4; ++s) h[s] += p * cf[s * d3 + i];
      }
      e[0] += w * (ex[0] * ex[0] + ex[1] * ex[1] + ex[2] * ex[2]);
      e[1] += w * ((ex[0] - h[0]) * (ex[0] - h[0]) + (ex[1] - h[1]) * (ex[1] - h[1]) +
                   (ex[2] - h[2]) * (ex[2] - h[2]));
      e[2] += w * ex[3] * ex[3];
      e[3] += w * (ex[3] - h[3]) * (ex[3] - h[3]);
      if (ustar) {
        double hs = 0.0;
        for (int i = 0; i < d31; ++i) hs += tE1.P[long(i) * nq + q] * cf[4 * d3 + i];
        e[4] += w * (ex[3] - hs) * (ex[3] - hs);
      }
    }
    double du = 0.0;
    if (proj_u)
      for (int i = lane; i < d3; i += 32) {
        const double d = proj_u[K * d3 + i] - cf[3 * d3 + i];
        du += d * d;
      }
#pragma unroll
    for (int j = 0; j < 5; ++j) acc[j] += vol * e[j];
    acc[5] += 6.0 * vol * du;
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < 6; ++j) {
    const double v = warp_sum(acc[j]);
    if (lane == 0) red[warp][j] = v;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double s = 0.0;
    for (int w = 0; w < kErrWarps; ++w) s += red[w][threadIdx.x];
    partial[blockIdx.x].v[threadIdx.x] = s;
  }
}

// ------------------------------------------------------------ skeleton errors
// sums: 6 sum_e |e|^2 sum_r w u^2, 7 sum_e |e|^2 sum_r w (u - D uhat)^2,
//       8 sum_e 2 |e|^2 |P_e u - uhat_e|^2  (P_e u: l2_project_skeleton moments)
__global__ void __launch_bounds__(kErrWarps * 32)
face_errors_kernel(DevTab tE, int nfc, const double* __restrict__ coords, int nver, const int* __restrict__ faces,
                   const double* __restrict__ area, FieldDev fu, const double* __restrict__ uhat,
                   ErrSums* __restrict__ partial) {
  __shared__ double wu[kErrWarps][64];
  __shared__ double red[kErrWarps][3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqd = tE.nqd, d2 = tE.d2;
  const double* Dt = tE.Dperm;  // mu = 1: D at the reference nodes (nqd x d2)
  double acc[3] = {0, 0, 0};
  for (long f = long(blockIdx.x) * kErrWarps + warp; f < nfc; f += long(gridDim.x) * kErrWarps) {
    const int v0 = faces[f], v1 = faces[nfc + f], v2 = faces[2 * nfc + f];
    double sU = 0.0, sD = 0.0;
    for (int r = lane; r < nqd; r += 32) {
      const double s = tE.tri_bary[nqd + r], t = tE.tri_bary[2 * nqd + r], w0 = 1.0 - s - t;
      const double x = w0 * coords[v0] + s * coords[v1] + t * coords[v2];
      const double y = w0 * coords[nver + v0] + s * coords[nver + v1] + t * coords[nver + v2];
      const double z = w0 * coords[2 * nver + v0] + s * coords[2 * nver + v1] + t * coords[2 * nver + v2];
      const double uf = eval_field(fu, x, y, z, r, f, nqd);
      double v = 0.0;
      for (int i = 0; i < d2; ++i) v += Dt[long(i) * nqd + r] * uhat[f * d2 + i];
      const double w = tE.tri_w[r];
      sU += w * uf * uf;
      sD += w * (uf - v) * (uf - v);
      wu[warp][r] = w * uf;
    }
    __syncwarp();
    double dh = 0.0;
    for (int i = lane; i < d2; i += 32) {
      double pu = 0.0;
      for (int r = 0; r < nqd; ++r) pu += Dt[long(i) * nqd + r] * wu[warp][r];
      const double d = 0.5 * pu - uhat[f * d2 + i];
      dh += d * d;
    }
    const double a2 = area[f] * area[f];
    acc[0] += sU * a2;
    acc[1] += sD * a2;
    acc[2] += 2.0 * dh * a2;
    __syncwarp();
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double v = warp_sum(acc[j]);
    if (lane == 0) red[warp][j] = v;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int w = 0; w < kErrWarps; ++w) s += red[w][threadIdx.x];
    partial[blockIdx.x].v[6 + threadIdx.x] = s;
  }
}

// l2_project_volume (postprocess.cpp:76-82): (1/6) P^T w u, d3 x nelt
__global__ void __launch_bounds__(kErrWarps * 32)
l2_project_volume_kernel(DevTab tE, int nelt, GeoDev geo, FieldDev fu, double* __restrict__ out, int per_warp) {
  extern __shared__ double esm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = tE.nq, d3 = tE.d3;
  double* wF = esm + warp * per_warp;
  for (long K = long(blockIdx.x) * kErrWarps + warp; K < nelt; K += long(gridDim.x) * kErrWarps) {
    for (int q = lane; q < nq; q += 32) {
      double x, y, z;
      tet_point(geo, K, nelt, tE.bary[q], tE.bary[nq + q], tE.bary[2 * nq + q], tE.bary[3 * nq + q], x, y, z);
      wF[q] = tE.w[q] * eval_field(fu, x, y, z, q, K, nq);
    }
    __syncwarp();
    for (int i = lane; i < d3; i += 32) {
      double a = 0.0;
      for (int q = 0; q < nq; ++q) a += tE.P[long(i) * nq + q] * wF[q];
      out[K * d3 + i] = a / 6.0;
    }
    __syncwarp();
  }
}

}  // namespace hdgb
