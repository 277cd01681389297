// K1 (geometry), K4 (skeleton pattern + scatter) and small helper kernels.
// All are HBM-bound streaming kernels: one thread per element / face row,
// element index fastest in every SoA array so loads and stores coalesce.
#pragma once

#include <climits>
#include <type_traits>

#include "dev_common.cuh"
#include "kernels_local.cuh"

namespace hdgb {

__constant__ int c_local_face[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {3, 1, 2}};
__constant__ double c_face_sign[4] = {-1.0, 1.0, -1.0, 1.0};
__constant__ int c_vertex_image[6][3] = {{0, 1, 2}, {0, 2, 1}, {2, 0, 1}, {2, 1, 0}, {1, 2, 0}, {1, 0, 2}};

// |e| = |1/2 (w2-w1) x (w3-w1)| of the global face triple (mesh.cpp:153-154).
__global__ void face_area_kernel(int nver, int nfc, const double* __restrict__ X,
                                 const int* __restrict__ faces, double* __restrict__ area) {
  const long f = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= nfc) return;
  const int v0 = faces[f], v1 = faces[nfc + f], v2 = faces[2L * nfc + f];
  double u[3], w[3];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    u[c] = X[v1 + long(c) * nver] - X[v0 + long(c) * nver];
    w[c] = X[v2 + long(c) * nver] - X[v0 + long(c) * nver];
  }
  const double n0 = 0.5 * (u[1] * w[2] - u[2] * w[1]);
  const double n1 = 0.5 * (u[2] * w[0] - u[0] * w[2]);
  const double n2 = 0.5 * (u[0] * w[1] - u[1] * w[0]);
  area[f] = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
}

// K1: per-element geometry (mesh.cpp:43-66, :156-169; element_matrices.cpp:31-36).
__global__ void geometry_kernel(int nver, int nelt, int nfc, const double* __restrict__ X,
                                const int* __restrict__ elements, const int* __restrict__ faces,
                                const int* __restrict__ facebyele, const double* __restrict__ tau,
                                double tau_const, const double* __restrict__ area,
                                double* __restrict__ volume, double* __restrict__ piola,
                                double* __restrict__ normals, int* __restrict__ perm,
                                double* __restrict__ T, double* __restrict__ verts,
                                int* __restrict__ status) {
  const long K = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (K >= nelt) return;
  int v[4];
  double x[4], y[4], z[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = elements[long(i) * nelt + K];
    x[i] = X[v[i]];
    y[i] = X[long(nver) + v[i]];
    z[i] = X[2L * nver + v[i]];
  }
  // cofactors a = detB B^{-T} (mesh.cpp:56-64)
  double a[9];
  a[0] = (y[2] - y[0]) * (z[3] - z[0]) - (y[3] - y[0]) * (z[2] - z[0]);
  a[1] = (y[3] - y[0]) * (z[1] - z[0]) - (y[1] - y[0]) * (z[3] - z[0]);
  a[2] = (y[1] - y[0]) * (z[2] - z[0]) - (y[2] - y[0]) * (z[1] - z[0]);
  a[3] = (x[3] - x[0]) * (z[2] - z[0]) - (x[2] - x[0]) * (z[3] - z[0]);
  a[4] = (x[1] - x[0]) * (z[3] - z[0]) - (x[3] - x[0]) * (z[1] - z[0]);
  a[5] = (x[2] - x[0]) * (z[1] - z[0]) - (x[1] - x[0]) * (z[2] - z[0]);
  a[6] = (x[2] - x[0]) * (y[3] - y[0]) - (x[3] - x[0]) * (y[2] - y[0]);
  a[7] = (x[3] - x[0]) * (y[1] - y[0]) - (x[1] - x[0]) * (y[3] - y[0]);
  a[8] = (x[1] - x[0]) * (y[2] - y[0]) - (x[2] - x[0]) * (y[1] - y[0]);
  // det B by expansion along B's first column (x2-x1, y2-y1, z2-z1)
  const double detB = (x[1] - x[0]) * a[0] + (y[1] - y[0]) * a[3] + (z[1] - z[0]) * a[6];
  if (!(detB > 0)) atomicMin(status, int(K < 0x7fffffff ? K : 0x7fffffff));
  volume[K] = detB / 6.0;
#pragma unroll
  for (int i = 0; i < 9; ++i) piola[long(i) * nelt + K] = a[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    verts[long(i) * nelt + K] = x[i];
    verts[long(4 + i) * nelt + K] = y[i];
    verts[long(8 + i) * nelt + K] = z[i];
  }
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int i0 = c_local_face[l][0], i1 = c_local_face[l][1], i2 = c_local_face[l][2];
    const double ux = x[i1] - x[i0], uy = y[i1] - y[i0], uz = z[i1] - z[i0];
    const double wx = x[i2] - x[i0], wy = y[i2] - y[i0], wz = z[i2] - z[i0];
    const double sg = c_face_sign[l];
    normals[long(3 * l) * nelt + K] = sg * (0.5 * (uy * wz - uz * wy));
    normals[long(3 * l + 1) * nelt + K] = sg * (0.5 * (uz * wx - ux * wz));
    normals[long(3 * l + 2) * nelt + K] = sg * (0.5 * (ux * wy - uy * wx));
    const int f = facebyele[long(l) * nelt + K];
    const int gv[3] = {faces[f], faces[long(nfc) + f], faces[2L * nfc + f]};
    const int lv[3] = {v[i0], v[i1], v[i2]};
    int mu = 0;
    for (int m = 1; m <= 6 && mu == 0; ++m)
      if (gv[c_vertex_image[m - 1][0]] == lv[0] && gv[c_vertex_image[m - 1][1]] == lv[1] &&
          gv[c_vertex_image[m - 1][2]] == lv[2])
        mu = m;
    if (mu == 0) atomicMin(status + 1, int(K));
    perm[long(l) * nelt + K] = mu == 0 ? 1 : mu;
    const double tv = tau ? tau[long(l) * nelt + K] : tau_const;
    T[long(l) * nelt + K] = tv * area[f];
  }
}

// tau(K,l) = 1 + |beta(xbar_e) . nu_{K,l}| (config C4 upwind stabilisation).
__global__ void upwind_tau_kernel(int nelt, GeoDev geo, FieldDev bx, FieldDev by, FieldDev bz,
                                  double* __restrict__ tau) {
  const long K = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (K >= nelt) return;
  for (int l = 0; l < 4; ++l) {
    double c[3];
    for (int d = 0; d < 3; ++d)
      c[d] = (geo.verts[long(4 * d + c_local_face[l][0]) * nelt + K] +
              geo.verts[long(4 * d + c_local_face[l][1]) * nelt + K] +
              geo.verts[long(4 * d + c_local_face[l][2]) * nelt + K]) / 3.0;
    const double nx = geo.normals[long(3 * l) * nelt + K], ny = geo.normals[long(3 * l + 1) * nelt + K],
                 nz = geo.normals[long(3 * l + 2) * nelt + K];
    const double nn = sqrt(nx * nx + ny * ny + nz * nz);
    const double b0 = eval_field(bx, c[0], c[1], c[2], 0, K, 1);
    const double b1 = eval_field(by, c[0], c[1], c[2], 0, K, 1);
    const double b2 = eval_field(bz, c[0], c[1], c[2], 0, K, 1);
    tau[long(l) * nelt + K] = 1.0 + fabs((b0 * nx + b1 * ny + b2 * nz) / nn);
  }
}

// Physical quadrature nodes X = bary * verts (element_matrices.cpp:66-70).
__global__ void quad_points_kernel(int nelt, int nq, const double* __restrict__ bary,
                                   const double* __restrict__ verts, double* __restrict__ X,
                                   double* __restrict__ Y, double* __restrict__ Z) {
  const long idx = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= long(nelt) * nq) return;
  const long K = idx / nq;
  const int q = int(idx - K * nq);
  double p[3];
  for (int d = 0; d < 3; ++d) {
    double s = 0.0;
    for (int v = 0; v < 4; ++v) s += bary[long(v) * nq + q] * verts[long(4 * d + v) * nelt + K];
    p[d] = s;
  }
  X[idx] = p[0];
  Y[idx] = p[1];
  Z[idx] = p[2];
}

__global__ void set_ll_kernel(long long* p, long long v) { *p = v; }

// Status words of one build_condense: [0] lowest singular element, [1] lowest
// element with a negative tau, [2] lowest element whose tau vanishes on all
// four faces (LLONG_MAX = none); [4] elements re-solved by the rescue kernel.
__global__ void reset_build_status_kernel(long long* st) {
  if (threadIdx.x < 3) st[threadIdx.x] = LLONG_MAX;
  if (threadIdx.x == 4) st[4] = 0;
}

// StabilizationField::validate (element_matrices.cpp:38-46) on T = tau |e|
// (|e| > 0, so the signs are tau's): records the lowest offending elements.
__global__ void tau_check_kernel(int nelt, const double* __restrict__ T, long long* st) {
  for (long K = long(blockIdx.x) * blockDim.x + threadIdx.x; K < nelt; K += long(gridDim.x) * blockDim.x) {
    const double t0 = T[K], t1 = T[nelt + K], t2 = T[2L * nelt + K], t3 = T[3L * nelt + K];
    if (t0 < 0.0 || t1 < 0.0 || t2 < 0.0 || t3 < 0.0) atomicMin(st + 1, K);
    if (fmax(fmax(t0, t1), fmax(t2, t3)) <= 0.0) atomicMin(st + 2, K);
  }
}

// ================================================================ K4
// CSR of the skeleton matrix H: row (f, i) holds, for every neighbour face g of
// f in ascending order, the d2 columns g*d2 + j (global_system.cpp:43-54).
__global__ void pattern_fill_kernel(int nfc, int d2, const int64_t* __restrict__ facebase,
                                    const int* __restrict__ nbr, int64_t* __restrict__ rowptr,
                                    int* __restrict__ colidx) {
  const long row = long(blockIdx.x) * blockDim.x + threadIdx.x;
  const long ndof = long(nfc) * d2;
  if (row > ndof) return;
  if (row == ndof) { rowptr[ndof] = facebase[nfc] * d2 * d2; return; }
  const long f = row / d2;
  const int i = int(row - f * d2);
  const int nb = int(facebase[f + 1] - facebase[f]);
  const int64_t start = facebase[f] * d2 * d2 + int64_t(i) * nb * d2;
  rowptr[row] = start;
  for (int s = 0; s < nb; ++s) {
    const int gcol = nbr[f * 8 + s] * d2;
    for (int j = 0; j < d2; ++j) colidx[start + s * d2 + j] = gcol + j;
  }
}

// One warp per element. Off-diagonal face blocks have exactly one owner (two
// tets share at most one face) -> plain stores; diagonal blocks and b receive
// one or two contributions -> fp64 atomics onto zero, which is bit-exact (a+b
// is commutative, 0+a exact).
__global__ void scatter_kernel(int nelt, int d2, const int* __restrict__ facebyele,
                               const uint8_t* __restrict__ slot, const int64_t* __restrict__ facebase,
                               const double* __restrict__ C, const double* __restrict__ Cf,
                               double* __restrict__ vals, double* __restrict__ b) {
  const int lane = threadIdx.x & 31;
  const long K = long(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (K >= nelt) return;
  const int m = 4 * d2;
  const double* Ck = C + K * m * m;
  int f[4];
#pragma unroll
  for (int l = 0; l < 4; ++l) f[l] = facebyele[long(l) * nelt + K];
  for (int task = lane; task < 16 * d2; task += 32) {
    // task -> (l2, l1, i) with i fastest so lanes read consecutive rows of C
    const int i = task % d2, l1 = (task / d2) % 4, l2 = task / (4 * d2);
    const int f1 = f[l1];
    const int nb = int(facebase[f1 + 1] - facebase[f1]);
    const int64_t pos = facebase[f1] * d2 * d2 + int64_t(i) * nb * d2 + int64_t(slot[K * 16 + l1 * 4 + l2]) * d2;
    const int r = l1 * d2 + i;
    if (l1 == l2) {
      for (int j = 0; j < d2; ++j) atomicAdd(vals + pos + j, Ck[r + (l2 * d2 + j) * m]);
    } else {
      for (int j = 0; j < d2; ++j) vals[pos + j] = Ck[r + (l2 * d2 + j) * m];
    }
  }
  for (int r = lane; r < m; r += 32) {
    const int l = r / d2;
    atomicAdd(b + long(f[l]) * d2 + (r - l * d2), Cf[K * m + r]);
  }
}

// K4 v2: the element's C slice (contiguous m x m, column-major) is staged in
// shared memory with 16-byte coalesced loads, then written out block by block
// with lanes along the block's contiguous column index j, so each 80-byte row
// segment of a d2 x d2 block goes out in one store instruction (v1 wrote with
// lanes along rows, 8-byte stores scattered over 32 lines). Diagonal blocks
// (1-2 contributions) and b stay fp64 atomics onto zero: bit-exact.
constexpr int kScatterWarps = 8;
__global__ void __launch_bounds__(kScatterWarps * 32)
scatter2_kernel(int nelt, int d2, const int* __restrict__ facebyele, const uint8_t* __restrict__ slot,
                const int64_t* __restrict__ facebase, const double* __restrict__ C, const double* __restrict__ Cf,
                double* __restrict__ vals, double* __restrict__ b) {
  extern __shared__ __align__(16) double ssm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = 4 * d2, mm = m * m, dd = d2 * d2;
  double* Cs = ssm + warp * (mm + 64);
  int64_t* rowb = reinterpret_cast<int64_t*>(Cs + mm);  // per (l1, l2): first value of the block
  int* nbw = reinterpret_cast<int*>(rowb + 16);          // per l1: row width n1 * d2
  for (long K = long(blockIdx.x) * kScatterWarps + warp; K < nelt; K += long(gridDim.x) * kScatterWarps) {
    const double2* src = reinterpret_cast<const double2*>(C + K * mm);
    for (int q = lane; q < mm / 2; q += 32) reinterpret_cast<double2*>(Cs)[q] = __ldg(src + q);
    if (lane < 16) {
      const int l1 = lane >> 2, l2 = lane & 3;
      const int f1 = facebyele[long(l1) * nelt + K];
      const int64_t b0 = facebase[f1];
      const int nb = int(facebase[f1 + 1] - b0);
      rowb[lane] = b0 * dd + int64_t(slot[K * 16 + l1 * 4 + l2]) * d2;
      if (l2 == 0) nbw[l1] = nb * d2;
    }
    __syncwarp();
    for (int idx = lane; idx < 16 * dd; idx += 32) {
      const int blk = idx / dd, w = idx - blk * dd, i = w / d2, j = w - i * d2;
      const int l1 = blk >> 2, l2 = blk & 3;
      const double v = Cs[(l1 * d2 + i) + (l2 * d2 + j) * m];
      double* dst = vals + rowb[blk] + int64_t(i) * nbw[l1] + j;
      if (l1 == l2) atomicAdd(dst, v);
      else *dst = v;
    }
    for (int r = lane; r < m; r += 32) {
      const int l = r / d2;
      atomicAdd(b + long(facebyele[long(l) * nelt + K]) * d2 + (r - l * d2), Cf[K * m + r]);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------- face sides
// sides[2f], sides[2f+1] = element-local codes e*4+l of face f's two elements
// (lower element first), or -1 for a face with one element.
__global__ void face_sides_init_kernel(int nfc, int* __restrict__ sides) {
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < nfc; i += long(gridDim.x) * blockDim.x) {
    sides[2 * i] = INT_MAX;
    sides[2 * i + 1] = -1;
  }
}
__global__ void face_sides_kernel(int nelt, const int* __restrict__ facebyele, int* __restrict__ sides) {
  const long n = 4L * nelt;
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
    const int l = int(i / nelt), K = int(i - long(l) * nelt);
    const int f = facebyele[i], code = K * 4 + l;
    atomicMin(sides + 2 * f, code);
    atomicMax(sides + 2 * f + 1, code);
  }
}
__global__ void face_sides_fix_kernel(int nfc, int* __restrict__ sides) {
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < nfc; i += long(gridDim.x) * blockDim.x)
    if (sides[2 * i + 1] == sides[2 * i]) sides[2 * i + 1] = -1;
}

// ------------------------------------------------- K4 v3: face-row gather
// One warp per face: the face's d2 x (nb d2) block row of the CSR values is
// one contiguous run, assembled from its (one or two) elements' C column
// blocks C_e[:, l d2 .. l d2 + d2) (C is symmetric, so that contiguous column
// block is the transposed row block) and written once, coalesced. The
// diagonal block sums both sides in registers (a + b, order-free), so no
// atomics and no zero fill; b = sum of the sides' Cf rows the same way.
constexpr int kFaceRowWarps = 8;
template <int D2>
__global__ void __launch_bounds__(kFaceRowWarps * 32, D2 <= 10 ? 4 : 1)  // k <= 3: 4 CTAs per SM fit
scatter_faces_kernel(int nfc, const int* __restrict__ sides, const uint8_t* __restrict__ slot,
                     const int64_t* __restrict__ facebase, const double* __restrict__ C,
                     const double* __restrict__ Cf, double* __restrict__ vals, double* __restrict__ b, int nwarps) {
  extern __shared__ __align__(16) double fsm[];
  constexpr int m = 4 * D2, md = m * D2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ch = fsm + warp * (2 * md + 8);         // two column blocks
  int* inv = reinterpret_cast<int*>(ch + 2 * md);  // slot -> side * 4 + l2 (8 = diagonal)
  if (warp >= nwarps) return;
  for (long f = long(blockIdx.x) * nwarps + warp; f < nfc; f += long(gridDim.x) * nwarps) {
    const int s0 = sides[2 * f], s1 = sides[2 * f + 1];
    const int ns = s1 >= 0 ? 2 : 1;
    const int64_t base = facebase[f];
    const int nb = int(facebase[f + 1] - base), W = nb * D2;
    // both sides' column blocks: every load issued before the first store
    // (memory-level parallelism: NQ 16-byte loads per lane and side in flight;
    // batches of at most 8 per lane and side for the large k = 4, 5 blocks)
    constexpr int NQALL = (md / 2 + 31) / 32, NQ = NQALL < 8 ? NQALL : 8;
    for (int u0 = 0; u0 < NQALL; u0 += NQ) {
    double2 v[2][NQ];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int code = s ? s1 : s0;
      const double2* src = reinterpret_cast<const double2*>(C + long(code >> 2) * m * m + long(code & 3) * md);
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        const int q = lane + 32 * (u0 + u);
        if (s < ns && q < md / 2) v[s][u] = __ldg(src + q);
      }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (s >= ns) break;
      const int code = s ? s1 : s0, e = code >> 2, l = code & 3;
#pragma unroll
      for (int u = 0; u < NQ; ++u) {
        const int q = lane + 32 * (u0 + u);
        if (q < md / 2) reinterpret_cast<double2*>(ch + s * md)[q] = v[s][u];
      }
      if (u0 == 0 && lane < 4) {
        const int q = slot[long(e) * 16 + l * 4 + lane];
        inv[q] = lane == l ? 8 : s * 4 + lane;
      }
    }
    }
    __syncwarp();
    const int l0 = s0 & 3, l1 = s1 & 3;
    double* dst = vals + base * D2 * D2;
    // the D2 x W block row as one flat run of (row, column) units, 16-byte
    // units for even D2 (column pairs never straddle a block): every lane busy
    // and half the stores; the row of a unit from a float reciprocal (exact
    // here: t < 2^12, the nearest row boundary >= 1 / (2 W) away)
    constexpr int U = D2 % 2 == 0 ? 2 : 1, H = D2 / U;
    using vec = typename std::conditional<U == 2, double2, double>::type;
    const int WU = W / U;
    const float rW = 1.0f / float(WU);
#pragma unroll 2
    for (int t = lane; t < D2 * WU; t += 32) {
      const int i = __float2int_rz((float(t) + 0.5f) * rW), p = t - i * WU;
      const int q = p / H, j = U * (p - q * H);
      const int src = inv[q];
      const int o = j + i * m;
      vec v;
      if (src == 8) {
        v = *reinterpret_cast<const vec*>(ch + l0 * D2 + o);
        if (ns == 2) {
          const vec w = *reinterpret_cast<const vec*>(ch + md + l1 * D2 + o);
          if constexpr (U == 2) {
            v.x += w.x;
            v.y += w.y;
          } else {
            v += w;
          }
        }
      } else {
        v = *reinterpret_cast<const vec*>(ch + (src >> 2) * md + (src & 3) * D2 + o);
      }
      *reinterpret_cast<vec*>(dst + i * W + U * p) = v;
    }
    if (lane < D2) {
      double v = Cf[long(s0 >> 2) * m + l0 * D2 + lane];
      if (ns == 2) v += Cf[long(s1 >> 2) * m + l1 * D2 + lane];
      b[f * D2 + lane] = v;
    }
    __syncwarp();
  }
}

}  // namespace hdgb
