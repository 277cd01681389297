// Boundary data on the skeleton: face moments of a field
// against the trace basis D, completing the right-hand side b of the
// condensed system (study.cpp:25-26).
//
//   dirichlet_project   (global_system.cpp:58-70)    c_i = 1/2 sum_r w_r D_i(r) g(x_r),
//                                                    faces [0, ndir), out (ndir x d2)
//   l2_project_skeleton (postprocess.cpp:84-93)      same, all faces, out (nfc x d2)
//   neumann_load        (global_system.cpp:72-104)   c_i = sum_r w_r D_i(r) (g . n)(x_r),
//                                                    n = area-scaled outward normal of the
//                                                    face's element, faces [ndir, ndir+nneu)
//
// x_r = (1-s-t) v0 + s v1 + t v2 over the face's global vertex triple
// (face_quad_points, global_system.cpp:9-29). Boundary faces are numbered
// first (mesh.cpp:99-116), so each face set is a contiguous range.
//
// Face-parallel and HBM/latency-bound: one warp per face, lanes over the
// quadrature nodes (field evaluation), then lanes over the d2 moments.
#pragma once

#include "dev_common.cuh"

namespace hdgb {

constexpr int kFaceWarps = 8;
constexpr int kFaceMaxNodes = 64;

// adj[f] = 4 K + l of the unique element face on boundary face f < nbdy.
__global__ void boundary_adjacency_kernel(int nelt, const int* __restrict__ facebyele, int nbdy,
                                          int* __restrict__ adj) {
  const long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 4L * nelt) return;
  const int l = int(i / nelt);
  const long K = i - long(l) * nelt;
  const int f = facebyele[i];
  if (f < nbdy) adj[f] = int(4 * K + l);
}

// mode 0: out[(f - f0) d2 + i] = scale * c_i (scalar field g0)
// mode 1: out[f d2 + i] += scale * c_i (normal flux of (g0, g1, g2); adj, normals required)
__global__ void __launch_bounds__(kFaceWarps * 32)
face_moments_kernel(DevTab t, int mode, int f0, int f1, const double* __restrict__ coords, int nver,
                    const int* __restrict__ faces, int nfc, const int* __restrict__ adj,
                    const double* __restrict__ normals, int nelt, FieldDev g0, FieldDev g1, FieldDev g2,
                    double scale, double* __restrict__ out) {
  __shared__ double wg[kFaceWarps][kFaceMaxNodes];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqd = t.nqd, d2 = t.d2;
  const double* sb = t.tri_bary + nqd;  // s column
  const double* tb = t.tri_bary + 2 * nqd;
  for (long f = f0 + long(blockIdx.x) * kFaceWarps + warp; f < f1; f += long(gridDim.x) * kFaceWarps) {
    const int v0 = faces[f], v1 = faces[nfc + f], v2 = faces[2 * nfc + f];
    double nx = 0.0, ny = 0.0, nz = 0.0;
    if (mode == 1) {
      const int a = adj[f], l = a & 3;
      const long K = a >> 2;
      nx = normals[long(3 * l) * nelt + K];
      ny = normals[long(3 * l + 1) * nelt + K];
      nz = normals[long(3 * l + 2) * nelt + K];
    }
    const long fs = f - f0;  // sample column of a SAMPLED field
    for (int r = lane; r < nqd; r += 32) {
      const double s = sb[r], tt = tb[r], w0 = 1.0 - s - tt;
      const double x = w0 * coords[v0] + s * coords[v1] + tt * coords[v2];
      const double y = w0 * coords[nver + v0] + s * coords[nver + v1] + tt * coords[nver + v2];
      const double z = w0 * coords[2 * nver + v0] + s * coords[2 * nver + v1] + tt * coords[2 * nver + v2];
      double g = eval_field(g0, x, y, z, r, fs, nqd);
      if (mode == 1)
        g = g * nx + eval_field(g1, x, y, z, r, fs, nqd) * ny + eval_field(g2, x, y, z, r, fs, nqd) * nz;
      wg[warp][r] = t.tri_w[r] * g;
    }
    __syncwarp();
    for (int i = lane; i < d2; i += 32) {
      const double* D = t.Dperm + long(i) * nqd;  // mu = 1: D_i at the reference nodes
      double s = 0.0;
      for (int r = 0; r < nqd; ++r) s += D[r] * wg[warp][r];
      if (mode == 0) out[fs * d2 + i] = scale * s;
      else out[f * d2 + i] += scale * s;
    }
    __syncwarp();
  }
}

}  // namespace hdgb
