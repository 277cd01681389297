// Shared device types (GeoDev), K2 (the quadrature-node build, interpreted
// fields; the NVRTC-specialised copy lives in jit_quad.cpp), the warp-team
// Cholesky used by the k >= 4 postprocess, and the layout of recover2_kernel.
// The condensation kernels themselves are kernels_condense2/3/5.cuh.
#pragma once

#include "dev_common.cuh"

namespace hdgb {

struct GeoDev {
  const double* volume;   // nelt
  const double* piola;    // nelt x 9
  const double* normals;  // nelt x 12
  const int* perm;        // nelt x 4
  const double* T;        // nelt x 4
  const double* verts;    // nelt x 12
};

// =============================================================== K2: build
// Per CTA: EB elements. Phase 1 evaluates the coefficient fields at every
// physical quadrature node and forms the GEMM right-hand sides
//   Bk(q,e) = w_q vol kappa^-1(x_q),  Bc(q,e) = w_q vol c(x_q) (+ T rows),
//   Bf(q,e) = w_q vol f(x_q)
// in shared memory; phase 2 runs the node contraction as DMMA GEMMs with the
// element index as the N dimension and the fragment-ordered reference tables
// (streamed from L2) as A:
//   Msym = Wsym Bk,  Dsym = [Wsym | PPsym] [Bc; T],  fv = P^T Bf
// (element_matrices.cpp:94-109 mass_matrices x2, :155-167 type_a, :84-92).
// EB elements per CTA (EB / 8 N-tiles), 256 threads; EB = 32 where the
// three right-hand sides fit two CTAs per SM (each A fragment then feeds 8
// DMMAs), else 16.
constexpr int quad_ldb(int eb) { return eb + 4; }  // conflict-free [q][e] stride
inline size_t quad_smem_bytes(int eb, int nqp) { return size_t(3) * (nqp + 4) * quad_ldb(eb) * sizeof(double); }
inline int quad_eb(int nqp) { return quad_smem_bytes(32, nqp) <= 116 * 1024 ? 32 : 16; }

template <int EB>
__global__ void __launch_bounds__(256)
quad_build_kernel(DevTab tab, int nelt, GeoDev geo, FieldDev kap, FieldDev cc, FieldDev ff,
                  double* __restrict__ Msym, double* __restrict__ Dsym, double* __restrict__ fvec) {
  constexpr int kQuadEB = EB, kQuadLDB = quad_ldb(EB), NTI = EB / 8;
  extern __shared__ double smem[];
  const int nqp = tab.nqp, nq = tab.nq;
  const int rows = nqp + 4;
  double* Bk = smem;
  double* Bc = Bk + rows * kQuadLDB;
  double* Bf = Bc + rows * kQuadLDB;
  const long K0 = long(blockIdx.x) * kQuadEB;

  // ---- phase 1: physical nodes, fields, weights
  for (int idx = threadIdx.x; idx < rows * kQuadEB; idx += blockDim.x) {
    const int q = idx / kQuadEB, e = idx % kQuadEB;
    const long K = K0 + e;
    double bk = 0.0, bc = 0.0, bf = 0.0;
    if (K < nelt) {
      if (q < nq) {
        const double l0 = __ldg(tab.bary + q), l1 = __ldg(tab.bary + nq + q),
                     l2 = __ldg(tab.bary + 2 * nq + q), l3 = __ldg(tab.bary + 3 * nq + q);
        const double* V = geo.verts;
        const double x = l0 * V[K] + l1 * V[nelt + K] + l2 * V[2L * nelt + K] + l3 * V[3L * nelt + K];
        const double y = l0 * V[4L * nelt + K] + l1 * V[5L * nelt + K] + l2 * V[6L * nelt + K] +
                         l3 * V[7L * nelt + K];
        const double z = l0 * V[8L * nelt + K] + l1 * V[9L * nelt + K] + l2 * V[10L * nelt + K] +
                         l3 * V[11L * nelt + K];
        const double wv = __ldg(tab.w + q) * geo.volume[K];
        bk = wv / eval_field(kap, x, y, z, q, K, nq);
        bc = wv * eval_field(cc, x, y, z, q, K, nq);
        bf = wv * eval_field(ff, x, y, z, q, K, nq);
      } else if (q >= nqp) {
        bc = geo.T[long(q - nqp) * nelt + K];  // tau |e_l| rows for type_a
      }
    }
    Bk[q * kQuadLDB + e] = bk;
    Bc[q * kQuadLDB + e] = bc;
    Bf[q * kQuadLDB + e] = bf;
  }
  __syncthreads();

  // ---- phase 2: DMMA contraction over nodes
  // M and D share the table rows (Wsym): one task loads each A fragment once
  // for both (2 NTI DMMA per load); D's 4 tau PP columns are one extra k-step.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mts = tab.nsymp / 8, mtf = tab.d3p / 8;
  const int ntasks = mts + mtf;
  for (int task = warp; task < ntasks; task += nwarp) {
    double cm[NTI][2], cd[NTI][2];
#pragma unroll
    for (int j = 0; j < NTI; ++j) cm[j][0] = cm[j][1] = cd[j][0] = cd[j][1] = 0.0;
    const bool sym = task < mts;
    const int mt = sym ? task : task - mts;
    const double* Arow = sym ? tab.Asym + (long(mt) * ((nqp + 4) / 4)) * 32 + lane
                             : tab.Af + (long(mt) * (nqp / 4)) * 32 + lane;
    const double* B0 = sym ? Bk : Bf;
#pragma unroll 4
    for (int kk = 0; kk < nqp / 4; ++kk) {
      const double a = __ldg(Arow + kk * 32);
      const int o = (kk * 4 + t) * kQuadLDB + g;
#pragma unroll
      for (int j = 0; j < NTI; ++j) dmma(cm[j][0], cm[j][1], a, B0[o + 8 * j]);
      if (sym) {
#pragma unroll
        for (int j = 0; j < NTI; ++j) dmma(cd[j][0], cd[j][1], a, Bc[o + 8 * j]);
      }
    }
    if (sym) {  // tau PP rows (k = nqp .. nqp+3): D only
      const double a = __ldg(Arow + (nqp / 4) * 32);
      const int o = (nqp + t) * kQuadLDB + g;
#pragma unroll
      for (int j = 0; j < NTI; ++j) dmma(cd[j][0], cd[j][1], a, Bc[o + 8 * j]);
    }
    const int r = mt * 8 + g;
    const int lim = sym ? tab.nsym : tab.d3;
    if (r < lim) {
#pragma unroll
      for (int j = 0; j < NTI; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long K = K0 + 8 * j + 2 * t + h;
          if (K >= nelt) continue;
          if (sym) {
            Msym[K * lim + r] = cm[j][h];
            Dsym[K * lim + r] = cd[j][h];
          } else {
            fvec[K * lim + r] = cm[j][h];
          }
        }
    }
  }
}

// ============================================================ team helpers
// A "team" is NW warps working on one element; barriers are named per team.
template <int NW>
struct Team {
  int id, tid, warp, lane;
  __device__ __forceinline__ void sync() const {
    if (NW == 1) __syncwarp(); else team_sync(1 + id, NW * 32);
  }
};

// In-place Cholesky (left-looking, lower) of an n x n SPD matrix at A (ld),
// two columns per pass (2 team barriers per column pair). scratch: 2n doubles.
// Returns the pivot ratio test of local_solver.cpp:50-57 transposed to
// Cholesky pivots d_j = L_jj^2: singular iff min d < 1e-14 max d or d <= 0.
template <int NW>
__device__ bool team_cholesky(const Team<NW>& tm, double* A, int ld, int n, double* scratch) {
  constexpr int NT = NW * 32;
  double* s0 = scratch;
  double* s1 = scratch + n;
  double dmax = 0.0, dmin = 1e300;
  bool bad = false;
  int j = 0;
  for (; j + 1 < n; j += 2) {
    // s0_i = A(i,j) - sum_{k<j} L(i,k) L(j,k); s1_i likewise for column j+1 (i > j).
    // Four threads per row split the k range (quad shuffle sum): short chains.
    for (int base = 0; base < n - j; base += NT / 4) {  // warp-uniform trip count
      const int i = j + base + (tm.tid >> 2), part = tm.tid & 3;
      const bool live = i < n;
      double a0 = 0.0, a1 = 0.0;
      if (live)
        for (int k = part; k < j; k += 4) {
          const double l0 = A[i + k * ld];
          a0 = fma(-l0, A[j + k * ld], a0);
          a1 = fma(-l0, A[j + 1 + k * ld], a1);
        }
      a0 += __shfl_xor_sync(0xffffffffu, a0, 1);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 1);
      a0 += __shfl_xor_sync(0xffffffffu, a0, 2);
      a1 += __shfl_xor_sync(0xffffffffu, a1, 2);
      if (live && part == 0) {
        s0[i] = A[i + j * ld] + a0;
        s1[i] = i > j ? A[i + (j + 1) * ld] + a1 : 0.0;
      }
    }
    tm.sync();
    const double d0 = s0[j];
    const double l00 = d0 > 0.0 ? sqrt(d0) : 1.0, inv0 = 1.0 / l00;
    const double l10 = s0[j + 1] * inv0;
    const double d1 = s1[j + 1] - l10 * l10;
    const double l11 = d1 > 0.0 ? sqrt(d1) : 1.0, inv1 = 1.0 / l11;
    if (!(d0 > 0.0) || !(d1 > 0.0)) bad = true;
    dmax = fmax(dmax, fmax(d0, d1));
    dmin = fmin(dmin, fmin(d0, d1));
    for (int i = j + tm.tid; i < n; i += NT) {
      if (i == j) {
        A[j + j * ld] = l00;
      } else {
        const double li0 = s0[i] * inv0;
        A[i + j * ld] = li0;
        A[i + (j + 1) * ld] = i == j + 1 ? l11 : (s1[i] - li0 * l10) * inv1;
      }
    }
    tm.sync();
  }
  if (j < n) {  // last column of an odd-sized matrix
    for (int i = j + tm.tid; i < n; i += NT) {
      double s = A[i + j * ld];
      for (int k = 0; k < j; ++k) s = fma(-A[i + k * ld], A[j + k * ld], s);
      s0[i] = s;
    }
    tm.sync();
    const double d = s0[j];
    if (!(d > 0.0)) bad = true;
    dmax = fmax(dmax, d);
    dmin = fmin(dmin, d);
    const double ljj = d > 0.0 ? sqrt(d) : 1.0;
    const double inv = 1.0 / ljj;
    for (int i = j + tm.tid; i < n; i += NT) A[i + j * ld] = (i == j) ? ljj : s0[i] * inv;
    tm.sync();
  }
  return bad || dmax == 0.0 || dmin < 1e-14 * dmax;
}

// Stage element K's geometry record into sg[0..31].
__device__ __forceinline__ void load_geo(const GeoDev& geo, long K, int nelt, double* sg, int tid,
                                         int nthreads) {
  for (int i = tid; i < 30; i += nthreads) {
    double v;
    if (i == 0) v = geo.volume[K];
    else if (i < 10) v = geo.piola[long(i - 1) * nelt + K];
    else if (i < 22) v = geo.normals[long(i - 10) * nelt + K];
    else if (i < 26) v = geo.T[long(i - 22) * nelt + K];
    else v = double(geo.perm[long(i - 26) * nelt + K]);
    sg[i] = v;
  }
}

// ================================================================ K5 layout (recover2_kernel, kernels_condense2.cuh)
template <int K_>
struct RecDims {
  static constexpr int D3 = cdim3(K_), M = 4 * cdim2(K_);
  static constexpr int S1 = round_up(M, 32), S3 = round_up(3 * D3, 32), SD = round_up(D3, 32);
  static constexpr int PER_WARP = S1 + S3 + SD + S3 + 32;
};
constexpr int kRecWarps = 4;

}  // namespace hdgb
