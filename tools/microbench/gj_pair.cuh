// Microbench candidate (measured, not in the product): two 20 x 20 SPD inverses per warp:
// one matrix per 16-lane half, the leading 16 x 16 block inverted by the
// register sweep on the half's lanes and the 4-wide border eliminated by its
// Schur complement. Every lane of the warp carries a column, where the
// one-matrix sweep (gj_sweep.cuh) leaves 12 of 32 lanes idle on N = 20.
#pragma once

#include "../../paper_1305_1489_b200/csrc/gj_sweep.cuh"

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
