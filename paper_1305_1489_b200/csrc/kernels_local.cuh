// K2 (quadrature-node build), K3 (static condensation), K5 (gather + recover).
//
// Algorithm. The reference builds A1 (4 d3 square) and
// runs a partial-pivot LU with 4 d2 + 1 right-hand sides per element
// (local_solver.cpp:71-100). Here A1's block structure
//     A1 = [[M,0,0,-Cx^T],[0,M,0,-Cy^T],[0,0,M,-Cz^T],[Cx,Cy,Cz,D]],  D = Mc + tauPP
// is eliminated exactly, pivot-free (M and the Schur complement S are SPD):
//     L = chol(M), Li = L^-1, Y_s = Li C_s^T, Z = Li W^T (W = the perm-selected
//     face matrices Dperm^T diag(w) Pface), S = D + sum_s Y_s^T Y_s,
//     V = sum_s Y_s^T (Z n_s) + T^T, LSi = chol(S)^-1, Vt = LSi V, ft = LSi f,
//     C = tauDD + [n_l1.n_l2] o (Z^T Z) - Vt^T Vt,   Cf = Vt^T ft.
// C and Cf are mathematically identical to A3 A1^-1 A2 + tauDD and A3 A1^-1 Af.
// Every contraction runs on the FP64 tensor pipe (mma.sync m8n8k4 -> DMMA) out
// of shared memory; the recovery cache {Li, LSi, Vt, ft} lets K5 recover
// [q;u] without refactorising (the reference refactorises, local_solver.cpp:116).
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

// In-place inverse of a lower-triangular matrix (columns right to left, two
// per pass): X(j,j) = 1/L(j,j), X(i,j) = -X(j,j) sum_{k=j+1..i} X(i,k) L(k,j).
// scratch: 2n doubles.
template <int NW>
__device__ void team_tri_inverse(const Team<NW>& tm, double* A, int ld, int n, double* scratch) {
  constexpr int NT = NW * 32;
  double* x0 = scratch;      // column j
  double* x1 = scratch + n;  // column j - 1
  int j = n - 1;
  for (; j >= 1; j -= 2) {
    const double xjj = 1.0 / A[j + j * ld], xj1 = 1.0 / A[j - 1 + (j - 1) * ld];
    const double ljj1 = A[j + (j - 1) * ld];  // L(j, j-1)
    for (int base = 0; base < n - j + 1; base += NT / 4) {  // four threads per row (quad sums)
      const int i = j - 1 + base + (tm.tid >> 2), part = tm.tid & 3;
      const bool live = i < n;
      double sj = 0.0, s1 = 0.0;
      if (live)
        for (int k = j + 1 + part; k <= i; k += 4) {
          const double xik = A[i + k * ld];
          sj = fma(xik, A[k + j * ld], sj);
          s1 = fma(xik, A[k + (j - 1) * ld], s1);
        }
      sj += __shfl_xor_sync(0xffffffffu, sj, 1);
      s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
      sj += __shfl_xor_sync(0xffffffffu, sj, 2);
      s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
      if (live && part == 0) {
        const double xij = i > j ? -xjj * sj : (i == j ? xjj : 0.0);
        x0[i] = xij;
        x1[i] = i == j - 1 ? xj1 : -xj1 * (s1 + xij * ljj1);
      }
    }
    tm.sync();
    for (int i = j - 1 + tm.tid; i < n; i += NT) {
      if (i >= j) A[i + j * ld] = x0[i];
      A[i + (j - 1) * ld] = x1[i];
    }
    tm.sync();
  }
  if (j == 0) {
    const double x00 = 1.0 / A[0];
    for (int i = 1 + tm.tid; i < n; i += NT) {
      double s = 0.0;
      for (int k = 1; k <= i; ++k) s = fma(A[i + k * ld], A[k], s);
      x0[i] = -x00 * s;
    }
    tm.sync();
    for (int i = tm.tid; i < n; i += NT) A[i] = i == 0 ? x00 : x0[i];
    tm.sync();
  }
}

// Team DMMA GEMM: tiles (mt, nt) of an MT x NT tile grid, NB N-tiles per warp
// task sharing the A fragment. a_at(r, k), b_at(k, c) fetch operands; ks(mt)
// is the number of 4-wide k-steps for tile row mt (triangular A stops early);
// use(mt, nt) filters tiles; epi(r, c, v) consumes each output.
template <int NW, int NB, class FKS, class FUSE, class FA, class FB, class FE>
__device__ __forceinline__ void team_gemm(const Team<NW>& tm, int MT, int NT, FKS ks, FUSE use,
                                          FA a_at, FB b_at, FE epi) {
  const int g = tm.lane >> 2, t = tm.lane & 3;
  const int ngrp = (NT + NB - 1) / NB;
  for (int task = tm.warp; task < MT * ngrp; task += NW) {
    const int mt = task / ngrp, nt0 = (task % ngrp) * NB;
    if (!use(mt, nt0)) continue;
    double acc[NB][2];
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[j][0] = acc[j][1] = 0.0;
    const int kend = ks(mt);
    for (int kk = 0; kk < kend; ++kk) {
      const double a = a_at(mt * 8 + g, kk * 4 + t);
#pragma unroll
      for (int j = 0; j < NB; ++j)
        if (nt0 + j < NT) dmma(acc[j][0], acc[j][1], a, b_at(kk * 4 + t, (nt0 + j) * 8 + g));
    }
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (nt0 + j < NT) {
        epi(mt * 8 + g, (nt0 + j) * 8 + 2 * t, acc[j][0]);
        epi(mt * 8 + g, (nt0 + j) * 8 + 2 * t + 1, acc[j][1]);
      }
  }
}

// ---------------------------------------------------------- K3 layout
template <int K_>
struct CondDims {
  static constexpr int D3 = cdim3(K_), D2 = cdim2(K_), M = 4 * cdim2(K_);
  static constexpr int D3P = round_up(cdim3(K_), 8), MP = round_up(4 * cdim2(K_), 8);
  static constexpr int LD = D3P + 4;  // == 4 or 12 (mod 16): conflict-free fragments
  static constexpr int NSYM = D3 * (D3 + 1) / 2;
  // per-element shared memory (doubles)
  static constexpr int OFF_L = 0;                       // M -> L -> Li
  static constexpr int OFF_S = OFF_L + D3P * LD;        // D -> S -> LS -> LSi
  static constexpr int OFF_Y = OFF_S + D3P * LD;        // Q# -> Y_s -> Vt
  static constexpr int OFF_Z = OFF_Y + 3 * D3P * LD;    // Z (D3P x MP)
  static constexpr int OFF_V = OFF_Z + LD * MP;         // V (D3P x MP)
  static constexpr int OFF_VEC = OFF_V + LD * MP;       // f, ft, lambda, scratch
  static constexpr int OFF_GEO = OFF_VEC + 4 * round_up(MP > D3P ? MP : D3P, 8);
  static constexpr int PER_ELT = OFF_GEO + 32;          // vol a[9] n[12] T[4] perm[4]
  // recovery cache per element: Li (packed), LSi (packed), Vt (D3 x M), ft (D3)
  static constexpr int FACTORS = 2 * NSYM + D3 * M + D3;
  static constexpr int CTA_EXTRA = 0;
};

template <int K_>
struct CondCfg;
template <> struct CondCfg<0> { static constexpr int NW = 1, EPB = 16; };
template <> struct CondCfg<1> { static constexpr int NW = 1, EPB = 16; };
template <> struct CondCfg<2> { static constexpr int NW = 2, EPB = 8; };
template <> struct CondCfg<3> { static constexpr int NW = 2, EPB = 4; };
template <> struct CondCfg<4> { static constexpr int NW = 8, EPB = 1; };
#ifndef HDG_COND5_NW
#define HDG_COND5_NW 8
#endif
template <> struct CondCfg<5> { static constexpr int NW = HDG_COND5_NW, EPB = 1; };
template <> struct CondCfg<6> { static constexpr int NW = 8, EPB = 1; };

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

// ================================================================ K3
template <int K_>
__global__ void __launch_bounds__(CondCfg<K_>::NW * 32 * CondCfg<K_>::EPB)
condense_kernel(DevTab tab, int nelt, GeoDev geo, const double* __restrict__ Msym,
                const double* __restrict__ Dsym, const double* __restrict__ fvec,
                double* __restrict__ Cout, double* __restrict__ Cfout,
                double* __restrict__ factors, long long* bad_element) {
  using Dm = CondDims<K_>;
  constexpr int NW = CondCfg<K_>::NW, EPB = CondCfg<K_>::EPB, NT = NW * 32;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, D3P = Dm::D3P, MP = Dm::MP, LD = Dm::LD;
  extern __shared__ double smem[];

  // zero all per-element buffers once: padding rows/cols stay zero afterwards
  for (int i = threadIdx.x; i < EPB * Dm::PER_ELT; i += blockDim.x) smem[i] = 0.0;
  __syncthreads();

  Team<NW> tm;
  tm.id = threadIdx.x / NT;
  tm.tid = threadIdx.x % NT;
  tm.warp = tm.tid >> 5;
  tm.lane = tm.tid & 31;
  double* base = smem + tm.id * Dm::PER_ELT;
  double* Lb = base + Dm::OFF_L;
  double* Sb = base + Dm::OFF_S;
  double* Yb = base + Dm::OFF_Y;
  double* Zb = base + Dm::OFF_Z;
  double* Vb = base + Dm::OFF_V;
  double* fv = base + Dm::OFF_VEC;
  double* ft = fv + round_up(MP > D3P ? MP : D3P, 8);
  double* scr = ft + round_up(MP > D3P ? MP : D3P, 8);
  double* sg = base + Dm::OFF_GEO;
  const double* a9 = sg + 1;
  const double* nrm = sg + 10;
  const double* Tl = sg + 22;
  const double* pm = sg + 26;

  const long stride = long(gridDim.x) * EPB;
  for (long K = long(blockIdx.x) * EPB + tm.id; K < nelt; K += stride) {
    // ---- load M, D (lower), f, geometry
    for (int j = 0; j < D3; ++j) {
      const int b0 = sym_idx(j, j, D3);
      for (int i = tm.tid; i < D3 - j; i += NT) {
        Lb[(j + i) + j * LD] = Msym[K * Dm::NSYM + b0 + i];
        Sb[(j + i) + j * LD] = Dsym[K * Dm::NSYM + b0 + i];
      }
    }
    for (int i = tm.tid; i < D3; i += NT) fv[i] = fvec[K * D3 + i];
    load_geo(geo, K, nelt, sg, tm.tid, NT);
    tm.sync();

    // ---- L = chol(M); Li = L^-1 (in place)
    bool bad = team_cholesky(tm, Lb, LD, D3, scr);
    team_tri_inverse(tm, Lb, LD, D3, scr);

    // ---- Q_# = Li Chat_#^T  (lower-triangular A: k-steps up to the diagonal)
    auto ks_tri = [](int mt) { return (mt * 8 + 8) / 4 < D3P / 4 ? (mt * 8 + 8) / 4 : D3P / 4; };
    auto all = [](int, int) { return true; };
    auto a_Li = [&](int r, int k) { return Lb[r + k * LD]; };
    for (int s = 0; s < 3; ++s) {
      const double* Ch = tab.Chat + s * D3 * D3;
      double* Q = Yb + s * D3P * LD;
      team_gemm<NW, (D3P / 8 < 4 ? D3P / 8 : 4)>(
          tm, D3P / 8, D3P / 8, ks_tri, all, a_Li,
          [&](int k, int c) { return (k < D3 && c < D3) ? __ldg(Ch + c + k * D3) : 0.0; },
          [&](int r, int c, double v) { if (r < D3 && c < D3) Q[r + c * LD] = v; });
    }
    // ---- Z = Li W^T (perm-selected face blocks)
    team_gemm<NW, (MP / 8 < 4 ? MP / 8 : 4)>(
        tm, D3P / 8, MP / 8, ks_tri, all, a_Li,
        [&](int k, int c) {
          if (k >= D3 || c >= M) return 0.0;
          const int l = c / D2, i = c - l * D2;
          const int mu = int(pm[l]);
          return __ldg(tab.Wlm + (6 * l + mu - 1) * D2 * D3 + i + k * D2);
        },
        [&](int r, int c, double v) { if (r < D3 && c < M) Zb[r + c * LD] = v; });
    tm.sync();

    // ---- Y_s = sum_# a(s,#) Q_#  (elementwise, in place)
    for (int idx = tm.tid; idx < D3 * D3; idx += NT) {
      const int i = idx % D3, j = idx / D3;
      const double q0 = Yb[i + j * LD], q1 = Yb[D3P * LD + i + j * LD], q2 = Yb[2 * D3P * LD + i + j * LD];
#pragma unroll
      for (int s = 0; s < 3; ++s)
        Yb[s * D3P * LD + i + j * LD] = a9[3 * s] * q0 + a9[3 * s + 1] * q1 + a9[3 * s + 2] * q2;
    }
    tm.sync();

    // ---- S = D + sum_s Y_s^T Y_s (lower tiles); V = sum_s Y_s^T (Z n_s) + T^T
    constexpr int KY = 3 * D3P / 4;
    auto a_YT = [&](int r, int k) {  // (Y_s^T)(r, k') stacked over s
      const int s = k / D3P, kk = k - s * D3P;
      return Yb[s * D3P * LD + kk + r * LD];
    };
    team_gemm<NW, 1>(
        tm, D3P / 8, D3P / 8, [](int) { return KY; }, [](int mt, int nt) { return nt <= mt; }, a_YT,
        [&](int k, int c) {
          const int s = k / D3P, kk = k - s * D3P;
          return Yb[s * D3P * LD + kk + c * LD];
        },
        [&](int r, int c, double v) { if (r < D3 && c <= r) Sb[r + c * LD] += v; });
    team_gemm<NW, (MP / 8 < 4 ? MP / 8 : 4)>(
        tm, D3P / 8, MP / 8, [](int) { return KY; }, all, a_YT,
        [&](int k, int c) {
          const int s = k / D3P, kk = k - s * D3P;
          const int l = c < M ? c / D2 : 0;
          return Zb[kk + c * LD] * nrm[3 * l + s];
        },
        [&](int r, int c, double v) {
          if (r < D3 && c < M) {
            const int l = c / D2, i = c - l * D2;
            const int mu = int(pm[l]);
            Vb[r + c * LD] = v + Tl[l] * __ldg(tab.Wlm + (6 * l + mu - 1) * D2 * D3 + i + r * D2);
          }
        });
    tm.sync();

    // ---- LS = chol(S); LSi = LS^-1
    bad |= team_cholesky(tm, Sb, LD, D3, scr);
    team_tri_inverse(tm, Sb, LD, D3, scr);

    // ---- Vt = LSi V (into Y's buffer); ft = LSi f
    double* Vt = Yb;
    team_gemm<NW, (MP / 8 < 4 ? MP / 8 : 4)>(
        tm, D3P / 8, MP / 8, ks_tri, all, [&](int r, int k) { return Sb[r + k * LD]; },
        [&](int k, int c) { return Vb[k + c * LD]; },
        [&](int r, int c, double v) { if (r < D3 && c < M) Vt[r + c * LD] = v; });
    for (int r = tm.tid; r < D3; r += NT) {
      double s = 0.0;
      for (int k = 0; k <= r; ++k) s += Sb[r + k * LD] * fv[k];
      ft[r] = s;
    }
    tm.sync();

    // ---- C = tauDD + (n_l1.n_l2) Z^T Z - Vt^T Vt ; Cf = Vt^T ft
    {
      const int g = tm.lane >> 2, t = tm.lane & 3;
      constexpr int MT = MP / 8;
      double* Ck = Cout + K * M * M;
      for (int task = tm.warp; task < MT * MT; task += NW) {
        const int mt = task / MT, nt = task % MT;
        double z0 = 0, z1 = 0, v0 = 0, v1 = 0;
#pragma unroll 2
        for (int kk = 0; kk < D3P / 4; ++kk) {
          const int k = kk * 4 + t;
          const int r = mt * 8 + g, c = nt * 8 + g;
          dmma(z0, z1, Zb[k + r * LD], Zb[k + c * LD]);
          dmma(v0, v1, Vt[k + r * LD], Vt[k + c * LD]);
        }
        const int r = mt * 8 + g;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = nt * 8 + 2 * t + h;
          if (r < M && c < M) {
            const int l1 = r / D2, l2 = c / D2;
            const double nn = nrm[3 * l1] * nrm[3 * l2] + nrm[3 * l1 + 1] * nrm[3 * l2 + 1] +
                              nrm[3 * l1 + 2] * nrm[3 * l2 + 2];
            double val = nn * (h ? z1 : z0) - (h ? v1 : v0);
            if (l1 == l2) val += Tl[l1] * __ldg(tab.DD + (r - l1 * D2) + (c - l2 * D2) * D2);
            Ck[r + c * M] = val;
          }
        }
      }
      for (int r = tm.tid; r < M; r += NT) {
        double s = 0.0;
        for (int k = 0; k < D3; ++k) s += Vt[k + r * LD] * ft[k];
        Cfout[K * M + r] = s;
      }
      if (factors) {
        double* F = factors + K * Dm::FACTORS;
        for (int j = 0; j < D3; ++j) {
          const int b0 = sym_idx(j, j, D3);
          for (int i = tm.tid; i < D3 - j; i += NT) {
            F[b0 + i] = Lb[(j + i) + j * LD];
            F[Dm::NSYM + b0 + i] = Sb[(j + i) + j * LD];
          }
        }
        for (int idx = tm.tid; idx < D3 * M; idx += NT) {
          const int r = idx % D3, c = idx / D3;
          F[2 * Dm::NSYM + idx] = Vt[r + c * LD];
        }
        for (int i = tm.tid; i < D3; i += NT) F[2 * Dm::NSYM + D3 * M + i] = ft[i];
      }
    }
    if (bad && tm.tid == 0) flag_bad(bad_element, K);
    tm.sync();
  }
}

// ================================================================ K5
// One warp per element: lambda_K gathered from uhat (global_system.cpp:167-175),
//   u   = LSi^T (ft + Vt lambda)
//   q_s = Li^T Li (C_s^T u - E_s^T lambda),  C_s^T u = sum_# a(s,#) Chat_#^T u,
//         E_s^T lambda = sum_l n_s(l) W_l^T lambda_l
// (the solve of local_solver.cpp:117-123 through the cached factors).
template <int K_>
struct RecDims {
  static constexpr int D3 = cdim3(K_), M = 4 * cdim2(K_);
  static constexpr int S1 = round_up(M, 32), S3 = round_up(3 * D3, 32), SD = round_up(D3, 32);
  static constexpr int PER_WARP = S1 + S3 + SD + S3 + 32;
};
constexpr int kRecWarps = 4;

template <int K_>
__global__ void __launch_bounds__(kRecWarps * 32)
recover_kernel(DevTab tab, int nelt, GeoDev geo, const int* __restrict__ facebyele,
               const double* __restrict__ factors, const double* __restrict__ uhat,
               double* __restrict__ qx, double* __restrict__ qy, double* __restrict__ qz,
               double* __restrict__ uout) {
  using Dm = CondDims<K_>;
  using Rd = RecDims<K_>;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, NS = Dm::NSYM;
  __shared__ double sh[kRecWarps][Rd::PER_WARP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* lam = sh[warp];
  double* tv = lam + Rd::S1;   // 3 D3
  double* uu = tv + Rd::S3;    // D3
  double* pp = uu + Rd::SD;    // 3 D3
  double* sg = pp + Rd::S3;
  const long K = long(blockIdx.x) * kRecWarps + warp;
  if (K >= nelt) return;
  const double* F = factors + K * Dm::FACTORS;
  const double* Li = F;
  const double* LSi = F + NS;
  const double* Vt = F + 2 * NS;
  const double* ft = F + 2 * NS + D3 * M;
  load_geo(geo, K, nelt, sg, lane, 32);
  for (int i = lane; i < M; i += 32) {
    const int l = i / D2;
    lam[i] = uhat[long(facebyele[long(l) * nelt + K]) * D2 + (i - l * D2)];
  }
  __syncwarp();
  for (int r = lane; r < D3; r += 32) {
    double s = ft[r];
    for (int c = 0; c < M; ++c) s += Vt[r + c * D3] * lam[c];
    tv[r] = s;
  }
  __syncwarp();
  for (int i = lane; i < D3; i += 32) {  // u = LSi^T t
    double s = 0.0;
    for (int r = i; r < D3; ++r) s += LSi[sym_idx(r, i, D3)] * tv[r];
    uu[i] = s;
  }
  __syncwarp();
  const double* a9 = sg + 1;
  const double* nrm = sg + 10;
  const double* pm = sg + 26;
  for (int j = lane; j < D3; j += 32) {
    double p[3] = {0, 0, 0};
    for (int s = 0; s < 3; ++s) {
      const double* Ch = tab.Chat + s * D3 * D3 + j * D3;  // column j of Chat_#
      double acc = 0.0;
      for (int i = 0; i < D3; ++i) acc += __ldg(Ch + i) * uu[i];
      p[s] = acc;
    }
    double w[4];
    for (int l = 0; l < 4; ++l) {
      const double* W = tab.Wlm + (6 * l + int(pm[l]) - 1) * D2 * D3 + j * D2;
      double acc = 0.0;
      for (int i = 0; i < D2; ++i) acc += __ldg(W + i) * lam[l * D2 + i];
      w[l] = acc;
    }
    for (int s = 0; s < 3; ++s) {
      double r = a9[3 * s] * p[0] + a9[3 * s + 1] * p[1] + a9[3 * s + 2] * p[2];
      for (int l = 0; l < 4; ++l) r -= nrm[3 * l + s] * w[l];
      pp[s * D3 + j] = r;
    }
  }
  __syncwarp();
  for (int idx = lane; idx < 3 * D3; idx += 32) {  // y_s = Li r_s
    const int s = idx / D3, i = idx - s * D3;
    double acc = 0.0;
    for (int j = 0; j <= i; ++j) acc += Li[sym_idx(i, j, D3)] * pp[s * D3 + j];
    tv[idx] = acc;
  }
  __syncwarp();
  double* outs[3] = {qx, qy, qz};
  for (int idx = lane; idx < 3 * D3; idx += 32) {  // q_s = Li^T y_s
    const int s = idx / D3, j = idx - s * D3;
    double acc = 0.0;
    for (int i = j; i < D3; ++i) acc += Li[sym_idx(i, j, D3)] * tv[s * D3 + i];
    outs[s][K * D3 + j] = acc;
  }
  for (int i = lane; i < D3; i += 32) uout[K * D3 + i] = uu[i];
}

}  // namespace hdgb
