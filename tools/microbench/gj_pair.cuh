// Microbench candidate (measured, not in the product): two 20 x 20 SPD inverses per warp:
// one matrix per 16-lane half, the leading 16 x 16 block inverted by the
// register sweep on the half's lanes and the 4-wide border eliminated by its
// Schur complement. Every lane of the warp carries a column, where the
// one-matrix sweep (gj_sweep.cuh) leaves 12 of 32 lanes idle on N = 20.
#pragma once

#include "../../paper_1305_1489_b200/csrc/gj_sweep.cuh"

// Sweep inverse of the leading N x N block held by a W-lane segment of the
// warp (lane c < N of the segment owns column c in a[0..N-1]; rows N..R-1 of
// a[] are left untouched). Same algebra as gj_sweep_inverse; shuffles stay
// inside the segment; `stage` is the segment's own 2 x 64 doubles. pmin/pmax
// reduce the Cholesky pivots over the segment (a non-positive pivot as -1).
template <int N, int W, int R>
__device__ __forceinline__ void gj_sweep_seg(double (&a)[R], double* stage, int c, double& pmin, double& pmax) {
  static_assert(N % 2 == 0 && N <= W && N <= R, "even N on one segment");
  constexpr unsigned FULL = 0xffffffffu;
  double piv = 1.0;
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) {
    double* st = stage + ((k >> 1) & 1) * 64;
    if (c < N) {
      st[c] = a[k];
      st[32 + c] = a[k + 1];
    }
    const double p00 = __shfl_sync(FULL, a[k], k, W);
    const double p01 = __shfl_sync(FULL, a[k + 1], k, W);
    const double p11 = __shfl_sync(FULL, a[k + 1], k + 1, W);
    double n0x = 0.0, n0y = 0.0, n1x = 0.0, n1y = 0.0;
    if (k + 2 < N) {
      n0x = __shfl_sync(FULL, a[k], k + 2, W);
      n1x = __shfl_sync(FULL, a[k + 1], k + 2, W);
      n0y = __shfl_sync(FULL, a[k], k + 3, W);
      n1y = __shfl_sync(FULL, a[k + 1], k + 3, W);
    }
    const double det = fma(p00, p11, -p01 * p01);
    const bool m0 = c == k, m1 = c == k + 1;
    const double ak0 = m0 ? a[k] - 1.0 : a[k];
    const double ak1 = m1 ? a[k + 1] - 1.0 : a[k + 1];
    const double u0 = fma(p11, ak0, -p01 * ak1);
    const double u1 = fma(p00, ak1, -p01 * ak0);
    double s0 = 0.0, s1 = 0.0;
    if (k + 2 < N) {
      s0 = fma(n0x, u0, n1x * u1);
      s1 = fma(n0y, u0, n1y * u1);
    }
    const double id = gj_rcp(det);
    if (k + 2 < N) {
      a[k + 2] = fma(-s0, id, a[k + 2]);
      a[k + 3] = fma(-s1, id, a[k + 3]);
    }
    const double w0 = u0 * id, w1 = u1 * id;
    if (m0) piv = p00;
    if (m1) piv = p00 * id;
    __syncwarp();
#pragma unroll
    for (int i0 = 0; i0 < N; i0 += 2) {
      if (i0 == k || i0 == k + 2) continue;
      const double2 v0 = *reinterpret_cast<const double2*>(st + i0);
      const double2 v1 = *reinterpret_cast<const double2*>(st + 32 + i0);
      a[i0] = fma(-v0.x, w0, fma(-v1.x, w1, a[i0]));
      a[i0 + 1] = fma(-v0.y, w0, fma(-v1.y, w1, a[i0 + 1]));
    }
    a[k] = m0 ? w0 - 1.0 : w0;
    a[k + 1] = m1 ? w1 - 1.0 : w1;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = -a[i];
  double d = (c & 1) && c < N ? 1.0 / piv : piv;
  if (!(d > 0.0)) d = -1.0;
  double mn = c < N ? d : 1e300, mx = c < N ? d : 0.0;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  }
  pmin = fmin(pmin, mn);
  pmax = fmax(pmax, mx);
}

// Inverse of one 20 x 20 SPD matrix per 16-lane half. On entry lane c of the
// half holds column c (rows 0..19) of its matrix in a[] and every lane the
// trailing 4 x 4 block C packed lower in cc[] ((j, j'), j >= j', at
// j (j + 1) / 2 + j'). With A the leading 16 x 16 block and B its rows 0..15
// of columns 16..19:
//   X = A^-1 B,  Z = C - B^T X,  Zi = Z^-1,  Y = X Zi,
//   inv = [[A^-1 + Y X^T, -Y], [-Y^T, Zi]].
// On return a[] is column c of the inverse (rows 0..19) and zi[] holds Zi
// packed like cc. The pivots (A's from the sweep, Z's from its elimination)
// are the Cholesky pivots of the whole matrix; pmin/pmax as gj_sweep_inverse
// (per half). `stage`: 2 x 192 doubles, 16-byte aligned.
__device__ __forceinline__ void gj_pair_inverse20(double (&a)[20], const double (&cc)[10], double (&zi)[10],
                                                  double* stage, int lane, double& pmin, double& pmax) {
  constexpr unsigned FULL = 0xffffffffu;
  const int c = lane & 15;
  double* sh = stage + (lane >> 4) * 192;
  double* sx = sh + 128;  // B, then X: [i * 4 + j]
  double b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = a[16 + j];
  gj_sweep_seg<16, 16, 20>(a, sh, c, pmin, pmax);
  *reinterpret_cast<double2*>(sx + 4 * c) = make_double2(b[0], b[1]);
  *reinterpret_cast<double2*>(sx + 4 * c + 2) = make_double2(b[2], b[3]);
  __syncwarp();
  double x[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double2 p = *reinterpret_cast<const double2*>(sx + 4 * i);
    const double2 q = *reinterpret_cast<const double2*>(sx + 4 * i + 2);
    x[0] = fma(a[i], p.x, x[0]);
    x[1] = fma(a[i], p.y, x[1]);
    x[2] = fma(a[i], q.x, x[2]);
    x[3] = fma(a[i], q.y, x[3]);
  }
  // B^T X over the half's 16 lanes (butterfly), then Z = C - B^T X
  double z[4][4];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int jj = 0; jj <= j; ++jj) {
      double v = b[j] * x[jj];
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
      z[j][jj] = z[jj][j] = cc[j * (j + 1) / 2 + jj] - v;
    }
  // Z^-1 by the scalar sweep (its pivots are the last four Cholesky pivots)
  double zmin = 1e300, zmax = 0.0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const double d = z[p][p];
    zmin = fmin(zmin, d > 0.0 ? d : -1.0);
    zmax = fmax(zmax, d);
    const double r = gj_rcp(d);
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j <= i; ++j)
        if (i != p && j != p) z[i][j] = z[j][i] = fma(-z[i][p] * r, z[p][j], z[i][j]);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i != p) z[i][p] = z[p][i] = z[i][p] * r;
    z[p][p] = -r;
  }
  pmin = fmin(pmin, zmin);
  pmax = fmax(pmax, zmax);
  double y[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) y[j] = -(x[0] * z[0][j] + x[1] * z[1][j] + x[2] * z[2][j] + x[3] * z[3][j]);
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int jj = 0; jj <= j; ++jj) zi[j * (j + 1) / 2 + jj] = -z[j][jj];
  __syncwarp();  // every lane has read B
  *reinterpret_cast<double2*>(sx + 4 * c) = make_double2(x[0], x[1]);
  *reinterpret_cast<double2*>(sx + 4 * c + 2) = make_double2(x[2], x[3]);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const double2 p = *reinterpret_cast<const double2*>(sx + 4 * i);
    const double2 q = *reinterpret_cast<const double2*>(sx + 4 * i + 2);
    a[i] = fma(y[0], p.x, fma(y[1], p.y, fma(y[2], q.x, fma(y[3], q.y, a[i]))));
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) a[16 + j] = -y[j];
  __syncwarp();  // sx is reused by the next call
}
