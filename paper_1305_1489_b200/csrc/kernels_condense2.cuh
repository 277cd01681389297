// K3 v2 (k <= 3): static condensation with explicit inverses.
//
// Same block elimination as kernels_local.cuh, written with M^-1 and S^-1
// instead of triangular factors (only products X M^-1 Y^T appear):
//   Zp = Mi W^T,                         Gw = W Zp                (face Gram)
//   Y_s = Mi C_s^T,  S = D + sum_s C_s Y_s,  H = sum_s C_s Zp N_s  (N_s: per-face n_s)
//   Si = S^-1,  V = H + T^T,  Vs = Si V
//   C  = tauDD + (n_l1.n_l2) o Gw - V^T Vs,   Cf = Vs^T f
// The two d3 x d3 inverses are Gauss-Jordan sweeps held in one warp's
// registers (lane c owns column c; SPD, so no pivoting; the pivots are the
// Cholesky pivots and feed the reference's 1e-14 singularity test). Every
// contraction is a DMMA (mma.sync m8n8k4 f64) tile loop over shared memory;
// a team of NW warps handles one element with 6 named barriers per element.
// The recovery cache is {Mi, Si (packed lower), V, f}.
#pragma once

#include "dev_common.cuh"
#include "gj_sweep.cuh"
#include "kernels_local.cuh"

namespace hdgb {

template <int K_>
struct C2Dims {
  static constexpr int D3 = cdim3(K_), D2 = cdim2(K_), M = 4 * cdim2(K_);
  static constexpr int D3P = round_up(cdim3(K_), 8), MP = round_up(4 * cdim2(K_), 8);
  static constexpr int LD = D3P + 4;  // 4 or 12 (mod 16): conflict-free fragment loads
  static constexpr int NSYM = D3 * (D3 + 1) / 2;
  static constexpr int MT = D3P / 8, NTM = MP / 8, KS = D3P / 4;
  static constexpr int OFF_MI = 0;
  static constexpr int OFF_S = OFF_MI + D3P * LD;
  static constexpr int OFF_Y = OFF_S + D3P * LD;    // Y_s (3), later Vs
  static constexpr int OFF_Z = OFF_Y + 3 * D3P * LD;   // Zp
  static constexpr int OFF_V = OFF_Z + MP * LD;
  static constexpr int OFF_NSC = OFF_V + MP * LD;      // 3 x MP face normals per column
  static constexpr int OFF_TC = OFF_NSC + 3 * MP;      // MP: tau|e| per column
  static constexpr int OFF_WB = OFF_TC + MP;           // MP: W table offset per column (as double)
  static constexpr int OFF_BETA = OFF_WB + MP;         // 3 x MP: beta_#(c) = sum_s a(s,#) n_s(face c)
  static constexpr int OFF_F = OFF_BETA + 3 * MP;      // D3P: f
  static constexpr int OFF_FS = OFF_F + D3P;           // D3P: Si f
  static constexpr int OFF_STG = round_up(OFF_FS + D3P, 2);  // 128: GJ column stage (2 buffers, 16 B aligned)
  static constexpr int OFF_STG2 = OFF_STG + 128;       // 128: second GJ stage
  static constexpr int OFF_GEO = OFF_STG2 + 128;        // 2 x 32: geometry records (cur/next)
  static constexpr int OFF_COL = OFF_GEO + 64;         // second column-data buffer
  static constexpr int PER_ELT = OFF_COL + 8 * MP;
  static constexpr int FACTORS = round_up(NSYM + D3 * M + D3, 2);  // {M^-1 packed, Vs, fs}, 16-B records
  static constexpr int CTA_EXTRA = 0;  // per-CTA shared doubles beyond EPB * PER_ELT
};

template <int K_> struct C2Cfg;
template <> struct C2Cfg<0> { static constexpr int NW = 1, EPB = 8; };
template <> struct C2Cfg<1> { static constexpr int NW = 1, EPB = 16; };
#ifndef HDG_C2_NW2
#define HDG_C2_NW2 2
#define HDG_C2_EPB2 8
#endif
#ifndef HDG_C2_NW3
#define HDG_C2_NW3 4
#define HDG_C2_EPB3 4
#endif
template <> struct C2Cfg<2> { static constexpr int NW = HDG_C2_NW2, EPB = HDG_C2_EPB2; };
template <> struct C2Cfg<3> { static constexpr int NW = HDG_C2_NW3, EPB = HDG_C2_EPB3; };

// Inverse of the SPD N x N matrix held by a warp (lane c owns column c in
// a[]) by the symmetric sweep operator: sweeping pivot k keeps the matrix
// symmetric, so column k is gathered from every lane's own a[k] (one shared
// store per lane + broadcast loads) instead of being broadcast entry by entry.
// After N sweeps a = -A^-1; the sign is folded in on return. No pivoting;
// pmin / pmax return the extreme |pivots| (the LDL^T pivots: p00 and det/p00
// per 2 x 2 block; pmin = 0 if one vanished or is not finite), which the
// rescue screen compares (kernels_rescue.cuh).
// 1/x to full double precision: MUFU reciprocal seed + two Newton steps
// (shorter dependency chain than IEEE division; last-bit rounding may differ).
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

template <int N>
__device__ __forceinline__ void warp_gj_inverse(double (&a)[N], double* stage, int lane, double& pmin,
                                                double& pmax) {
  // stage: 2 buffers x (2 x 32) doubles: the two pivot columns gathered from
  // every lane (column k of a symmetric matrix == every lane's a[k]).
  // Cholesky pivots of each 2x2 block: p00 and det / p00 = 1 / i11, tracked as
  // running extremes (p00, i11, det) instead of stored, to save registers.
  double p00min = 1e300, p00max = 0.0, i11min = 1e300, i11max = 0.0, detmin = 1e300;
  bool finite = true;
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) {
    double* st = stage + ((k >> 1) & 1) * 64;
    if (lane < N) {
      st[lane] = a[k];
      st[32 + lane] = a[k + 1];
    }
    // pivot block straight from the pivot lanes (off the shared-memory path)
    const double p00 = __shfl_sync(0xffffffffu, a[k], k);
    const double p01 = __shfl_sync(0xffffffffu, a[k + 1], k);
    const double p11 = __shfl_sync(0xffffffffu, a[k + 1], k + 1);
    const double det = fma(p00, p11, -p01 * p01);
    const double id = fast_rcp(det);
    const double i00 = p11 * id, i01 = -p01 * id, i11 = p00 * id;  // P^-1 (symmetric)
    p00min = fmin(p00min, fabs(p00));
    p00max = fmax(p00max, fabs(p00));
    i11min = fmin(i11min, fabs(i11));
    i11max = fmax(i11max, fabs(i11));
    detmin = fmin(detmin, fabs(det));
    finite = finite && isfinite(i11) && isfinite(p00);
    const bool m0 = lane == k, m1 = lane == k + 1;
    // w = P^-1 [a_k; a_k+1] for ordinary lanes; pivot lanes hold their own
    // block column, for which "a - v w" must produce A(i,block) P^-1.
    double w0 = fma(i00, a[k], i01 * a[k + 1]);
    double w1 = fma(i01, a[k], i11 * a[k + 1]);
    if (m0) { w0 = 1.0 - i00; w1 = -i01; }
    if (m1) { w0 = -i01; w1 = 1.0 - i11; }
    double nk0 = w0, nk1 = w1;
    if (m0) { nk0 = -i00; nk1 = -i01; }
    if (m1) { nk0 = -i01; nk1 = -i11; }
    __syncwarp();
    // next pivot pair first: it heads the next step's dependency chain
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
      for (int i0 = 0; i0 < N; i0 += 2) {
        if (i0 == k) continue;
        if ((pass == 0) != (i0 == k + 2)) continue;
        const double2 v0 = *reinterpret_cast<const double2*>(st + i0);
        const double2 v1 = *reinterpret_cast<const double2*>(st + 32 + i0);
        a[i0] = fma(-v0.x, w0, fma(-v1.x, w1, a[i0]));
        if (i0 + 1 < N) a[i0 + 1] = fma(-v0.y, w0, fma(-v1.y, w1, a[i0 + 1]));
      }
    }
    a[k] = nk0;
    a[k + 1] = nk1;
  }
  if (N % 2) {  // trailing scalar pivot
    constexpr int k = N - 1;
    double* st = stage + (((k >> 1)) & 1) * 64;
    if (lane < N) st[lane] = a[k];
    const double p = __shfl_sync(0xffffffffu, a[k], k);
    p00min = fmin(p00min, fabs(p));
    p00max = fmax(p00max, fabs(p));
    detmin = fmin(detmin, fabs(p));
    finite = finite && isfinite(p);
    const double ip = fast_rcp(p);
    const bool me = lane == k;
    const double t = me ? 1.0 - ip : a[k] * ip;
    const double nk = me ? -ip : a[k] * ip;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < k; ++i) a[i] = fma(-st[i], t, a[i]);
    a[k] = nk;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = -a[i];
  if (!finite || !(p00min > 0.0) || !(detmin > 0.0)) {
    pmin = 0.0;  // a pivot vanished or overflowed: the rescue kernel decides
    pmax = fmax(pmax, p00max);
  } else {
    const double dmin = N >= 2 ? 1.0 / i11max : 1e300, dmax = N >= 2 ? 1.0 / i11min : 0.0;
    pmin = fmin(pmin, fmin(p00min, dmin));
    pmax = fmax(pmax, fmax(p00max, dmax));
  }
}

// Loads column `lane` of a packed-lower symmetric matrix and inverts it in
// place (warp-wide); pmin / pmax as warp_gj_inverse.
template <int D3>
__device__ __forceinline__ void warp_inverse_packed(const double* __restrict__ P, double (&a)[D3],
                                                    double* stage, int lane, double& pmin, double& pmax) {
#pragma unroll
  for (int i = 0; i < D3; ++i) {
    const int r = i > lane ? i : lane, c = i > lane ? lane : i;
    a[i] = lane < D3 ? P[sym_idx(r, c, D3)] : 0.0;
  }
  pmin = 1e300;
  pmax = 0.0;
  warp_gj_inverse<D3>(a, stage, lane, pmin, pmax);
}

// Column data of element K's faces (per m-column: normals, tau|e|, W offset,
// beta_#(c) = sum_s a(s,#) n_s(l(c))).
template <int D2, int D3, int M, int MP>
__device__ __forceinline__ void build_columns(const double* sg, double* col, int lane) {
  double* nsc = col;
  double* Tc = col + 3 * MP;
  int* wb = reinterpret_cast<int*>(col + 4 * MP);
  double* beta = col + 5 * MP;
  for (int c = lane; c < MP; c += 32) {
    if (c < M) {
      const int l = c / D2, i = c - l * D2;
      const int mu = int(sg[26 + l]);
      const double n0 = sg[10 + 3 * l], n1 = sg[11 + 3 * l], n2 = sg[12 + 3 * l];
      nsc[c] = n0;
      nsc[MP + c] = n1;
      nsc[2 * MP + c] = n2;
#pragma unroll
      for (int h = 0; h < 3; ++h) beta[h * MP + c] = sg[1 + h] * n0 + sg[4 + h] * n1 + sg[7 + h] * n2;
      Tc[c] = sg[22 + l];
      wb[c] = (6 * l + mu - 1) * D2 * D3 + i;
    } else {
#pragma unroll
      for (int h = 0; h < 3; ++h) nsc[h * MP + c] = beta[h * MP + c] = 0.0;
      Tc[c] = 0.0;
      wb[c] = -1;
    }
  }
}

template <int K_>
__global__ void __launch_bounds__(C2Cfg<K_>::NW * 32 * C2Cfg<K_>::EPB)
condense2_kernel(DevTab tab, int nelt, GeoDev geo, const double* __restrict__ Msym,
                 const double* __restrict__ Dsym, const double* __restrict__ fvec,
                 double* __restrict__ Cout, double* __restrict__ Cfout, double* __restrict__ factors,
                 double* __restrict__ pivstat) {
  using Dm = C2Dims<K_>;
  constexpr int NW = C2Cfg<K_>::NW, EPB = C2Cfg<K_>::EPB, NT = NW * 32;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, D3P = Dm::D3P, MP = Dm::MP, LD = Dm::LD;
  constexpr int MT = Dm::MT, NTM = Dm::NTM, KS = Dm::KS;
  constexpr int NLOW = NTM * (NTM + 1) / 2;        // lower tiles of the m x m output
  constexpr int WM = NW > 1 ? 1 : 0;               // warp inverting the next element's M
  constexpr int GW0 = NW > 2 ? 2 : (NW > 1 ? 1 : 0);  // first warp computing W Zp during GJ
  constexpr int NGW = NW - GW0;
  constexpr int TPW = (NLOW + NGW - 1) / NGW;
  constexpr int NLS = MT * (MT + 1) / 2;           // lower tiles of S
  constexpr int NTF = (D2 + 7) / 8 + 1;            // N-tiles a face's columns can span
  extern __shared__ double smem[];
  for (int i = threadIdx.x; i < EPB * Dm::PER_ELT; i += blockDim.x) smem[i] = 0.0;
  __syncthreads();

  Team<NW> tm;
  tm.id = threadIdx.x / NT;
  tm.tid = threadIdx.x % NT;
  tm.warp = tm.tid >> 5;
  tm.lane = tm.tid & 31;
  const int lane = tm.lane, g = lane >> 2, t = lane & 3;
  double* base = smem + tm.id * Dm::PER_ELT;
  double* Mi = base + Dm::OFF_MI;
  double* Sb = base + Dm::OFF_S;
  double* Yb = base + Dm::OFF_Y;   // R_#, later Vs
  double* Zb = base + Dm::OFF_Z;   // Zp, later (W Zp) lower tiles
  double* Vb = base + Dm::OFF_V;
  double* fv = base + Dm::OFF_F;
  double* fs = base + Dm::OFF_FS;
  double* stgS = base + Dm::OFF_STG;
  double* stgM = base + Dm::OFF_STG2;
  auto colbuf = [&](int b) { return base + (b ? Dm::OFF_COL : Dm::OFF_NSC); };
  auto sgbuf = [&](int b) { return base + Dm::OFF_GEO + 32 * b; };
  const double* Wlm = tab.Wlm;
  const double* Ch = tab.Chat;
  const long stride = long(gridDim.x) * EPB;
  int cur = 0;

  // ---- prologue: first element's M^-1, D, f, geometry, column data
  long K = long(blockIdx.x) * EPB + tm.id;
  if (K < nelt) {
    load_geo(geo, K, nelt, sgbuf(0), tm.tid, NT);
    for (int j = 0; j < D3; ++j) {
      const int b0 = sym_idx(j, j, D3);
      for (int i = tm.tid; i < D3 - j; i += NT) Sb[(j + i) + j * LD] = Dsym[K * Dm::NSYM + b0 + i];
    }
    for (int i = tm.tid; i < D3; i += NT) fv[i] = fvec[K * D3 + i];
    if (tm.warp == 0) {
      double a[D3];
      double pmin, pmax;
      warp_inverse_packed<D3>(Msym + K * Dm::NSYM, a, stgM, lane, pmin, pmax);
      if (lane < D3) {
#pragma unroll
        for (int i = 0; i < D3; ++i)  // lower triangle of the sweep result, mirrored
          if (i >= lane) {
            Mi[i + lane * LD] = a[i];
            Mi[lane + i * LD] = a[i];
          }
        if (factors) {
#pragma unroll
          for (int i = 0; i < D3; ++i)
            if (i >= lane) factors[K * Dm::FACTORS + sym_idx(i, lane, D3)] = a[i];
        }
      }
      if (lane == 0) store_pivstat(pivstat, K, 0, pmin, pmax);
    }
    tm.sync();
    if (tm.warp == NW - 1) build_columns<D2, D3, M, MP>(sgbuf(0), colbuf(0), lane);
    tm.sync();
  }

  for (; K < nelt; K += stride) {
    const long Kn = K + stride;
    const bool has_next = Kn < nelt;
    double* Ck = Cout + K * M * M;
    double* F = factors ? factors + K * Dm::FACTORS : nullptr;
    const double* sg = sgbuf(cur);
    const double* a9 = sg + 1;
    const double* nsc = colbuf(cur);
    const double* Tc = colbuf(cur) + 3 * MP;
    const int* wb = reinterpret_cast<const int*>(colbuf(cur) + 4 * MP);
    const double* beta = colbuf(cur) + 5 * MP;

    // -------- P1: Zp = Mi W^T ; R_# = sum_#' g(#,#') Mi Chat_#'^T, g = a^T a
    for (int task = tm.warp; task < NTM + MT; task += NW) {
      if (task < NTM) {
        double acc[MT][2];
#pragma unroll
        for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
        const int wbc = wb[task * 8 + g];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const double b = (wbc >= 0 && k < D3) ? __ldg(Wlm + wbc + k * D2) : 0.0;
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(acc[m][0], acc[m][1], Mi[(m * 8 + g) + k * LD], b);
        }
        const int c0 = task * 8 + 2 * t;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          Zb[(m * 8 + g) + c0 * LD] = acc[m][0];
          Zb[(m * 8 + g) + (c0 + 1) * LD] = acc[m][1];
        }
      } else {
        const int nt = task - NTM;
        const int c = nt * 8 + g;
        double q[3][MT][2];
#pragma unroll
        for (int h = 0; h < 3; ++h)
#pragma unroll
          for (int m = 0; m < MT; ++m) q[h][m][0] = q[h][m][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const bool in = k < D3 && c < D3;
          const int o = c + k * D3;  // Chat_#^T(k, c) = Chat_#(c, k)
          const double b0 = in ? __ldg(Ch + o) : 0.0, b1 = in ? __ldg(Ch + D3 * D3 + o) : 0.0,
                       b2 = in ? __ldg(Ch + 2 * D3 * D3 + o) : 0.0;
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            const double a = Mi[(m * 8 + g) + k * LD];
            dmma(q[0][m][0], q[0][m][1], a, b0);
            dmma(q[1][m][0], q[1][m][1], a, b1);
            dmma(q[2][m][0], q[2][m][1], a, b2);
          }
        }
        double gm[3][3];
#pragma unroll
        for (int h = 0; h < 3; ++h)
#pragma unroll
          for (int h2 = 0; h2 < 3; ++h2)
            gm[h][h2] = a9[h] * a9[h2] + a9[3 + h] * a9[3 + h2] + a9[6 + h] * a9[6 + h2];
        const int c0 = nt * 8 + 2 * t;
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          double* R = Yb + h * D3P * LD;
#pragma unroll
          for (int m = 0; m < MT; ++m)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              R[(m * 8 + g) + (c0 + e) * LD] =
                  gm[h][0] * q[0][m][e] + gm[h][1] * q[1][m][e] + gm[h][2] * q[2][m][e];
        }
      }
    }
    tm.sync();

    // ---- P2: S += sum_# Chat_# R_# (one task per lower tile, two partial
    //      chains) | V_l = Chat_l Zp_l + T_l W_l^T per face l, with
    //      Chat_l = sum_# beta_#(l) Chat_# (H = sum_s C_s Mi E_s^T by faces)
    for (int task = tm.warp; task < NLS + MT * 4; task += NW) {
      if (task < NLS) {
        int mt = 0, rem = task;
        while (rem > mt) { rem -= mt + 1; ++mt; }
        const int j = rem;
        const int r = mt * 8 + g;
        double p0 = 0, p1 = 0, q0 = 0, q1 = 0;
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          const double* R = Yb + h * D3P * LD;
          const double* C = Ch + h * D3 * D3;
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) {
            const int k = kk * 4 + t;
            const double a = (r < D3 && k < D3) ? __ldg(C + r + k * D3) : 0.0;
            if (kk & 1) dmma(q0, q1, a, R[k + (j * 8 + g) * LD]);
            else dmma(p0, p1, a, R[k + (j * 8 + g) * LD]);
          }
        }
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = j * 8 + 2 * t + e;
          if (r < D3 && c <= r)  // BDM (tab.nu < D3): decoupled diagonal outside the P_{k-1} block
            Sb[r + c * LD] = (r >= tab.nu || c >= tab.nu) ? (r == c ? 6.0 * sg[0] : 0.0)
                                                          : Sb[r + c * LD] + (e ? p1 + q1 : p0 + q0);
        }
      } else {
        const int mt = (task - NLS) >> 2, l = (task - NLS) & 3;
        const int r = mt * 8 + g;
        const int cl0 = l * D2, cl1 = cl0 + D2;     // face-l columns [cl0, cl1)
        const int nt0 = cl0 / 8;
        const double b0 = beta[cl0], b1 = beta[MP + cl0], b2 = beta[2 * MP + cl0];
        double acc[NTF][2];
#pragma unroll
        for (int j = 0; j < NTF; ++j) acc[j][0] = acc[j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          double a = 0.0;
          if (r < D3 && k < D3) {
            const int o = r + k * D3;
            a = b0 * __ldg(Ch + o) + b1 * __ldg(Ch + D3 * D3 + o) + b2 * __ldg(Ch + 2 * D3 * D3 + o);
          }
#pragma unroll
          for (int j = 0; j < NTF; ++j) {
            const int c = (nt0 + j) * 8 + g;  // B column of this lane
            const double b = (c >= cl0 && c < cl1) ? Zb[k + c * LD] : 0.0;
            if ((nt0 + j) * 8 < cl1) dmma(acc[j][0], acc[j][1], a, b);
          }
        }
#pragma unroll
        for (int j = 0; j < NTF; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = (nt0 + j) * 8 + 2 * t + e;
            if (c >= cl0 && c < cl1 && r < D3)
              Vb[r + c * LD] = r < tab.nu ? acc[j][e] + Tc[c] * __ldg(Wlm + wb[c] + r * D2) : 0.0;
          }
      }
    }
    tm.sync();

    // --- P3: warp 0 Si = S^-1 | warp WM: M^-1 of the next element | others:
    //         (W Zp) lower tiles in registers; V, f -> recovery cache
    double accz[TPW][2];
#pragma unroll
    for (int i = 0; i < TPW; ++i) accz[i][0] = accz[i][1] = 0.0;
    if (tm.warp == 0) {
      double a[D3];
#pragma unroll
      for (int i = 0; i < D3; ++i) {
        const int r = i > lane ? i : lane, c = i > lane ? lane : i;
        a[i] = lane < D3 ? Sb[r + c * LD] : 0.0;
      }
      double pmin = 1e300, pmax = 0.0;
      warp_gj_inverse<D3>(a, stgS, lane, pmin, pmax);
      if (lane < D3) {
#pragma unroll
        for (int i = 0; i < D3; ++i)  // lower triangle of the sweep result, mirrored
          if (i >= lane) {
            Sb[i + lane * LD] = a[i];
            Sb[lane + i * LD] = a[i];
          }
      }
      if (lane == 0) store_pivstat(pivstat, K, 1, pmin, pmax);
    }
    if (tm.warp == WM && has_next) {  // Mi is dead after P1: invert the next M into it
      double a[D3];
      double pmin, pmax;
      warp_inverse_packed<D3>(Msym + Kn * Dm::NSYM, a, stgM, lane, pmin, pmax);
      if (lane < D3) {
#pragma unroll
        for (int i = 0; i < D3; ++i)  // lower triangle of the sweep result, mirrored
          if (i >= lane) {
            Mi[i + lane * LD] = a[i];
            Mi[lane + i * LD] = a[i];
          }
        if (factors) {
#pragma unroll
          for (int i = 0; i < D3; ++i)
            if (i >= lane) factors[Kn * Dm::FACTORS + sym_idx(i, lane, D3)] = a[i];
        }
      }
      if (lane == 0) store_pivstat(pivstat, Kn, 0, pmin, pmax);
    }
    if (tm.warp >= GW0) {
      const int ow = tm.warp - GW0;
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int tile = ow + i * NGW;
        if (tile >= NLOW) break;
        int mt = 0, rem = tile;
        while (rem > mt) { rem -= mt + 1; ++mt; }
        const int nt = rem;
        const int wbr = wb[mt * 8 + g];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const double aw = (wbr >= 0 && k < D3) ? __ldg(Wlm + wbr + k * D2) : 0.0;
          dmma(accz[i][0], accz[i][1], aw, Zb[k + (nt * 8 + g) * LD]);
        }
      }
    }
    tm.sync();

    // -------- P4: (W Zp) tiles -> Zb | Vs = Si V (into Yb) | fs = Si f | next
    //          element's geometry + column data (double-buffered)
    if (tm.warp >= GW0) {
      const int ow = tm.warp - GW0;
#pragma unroll
      for (int i = 0; i < TPW; ++i) {
        const int tile = ow + i * NGW;
        if (tile >= NLOW) break;
        Zb[tile * 64 + 2 * lane] = accz[i][0];
        Zb[tile * 64 + 2 * lane + 1] = accz[i][1];
      }
    }
    double* Vs = Yb;
    for (int task = tm.warp; task < NTM * MT; task += NW) {
      const int nt = task / MT, m = task % MT;
      double a0 = 0, a1 = 0;
      const int c = nt * 8 + g;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int k = kk * 4 + t;
        dmma(a0, a1, Sb[(m * 8 + g) + k * LD], Vb[k + c * LD]);
      }
      const int r = m * 8 + g, c0 = nt * 8 + 2 * t;
      Vs[r + c0 * LD] = a0;
      Vs[r + (c0 + 1) * LD] = a1;
    }
    for (int r = tm.tid; r < D3; r += NT) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D3; ++k) s += Sb[r + k * LD] * fv[k];
      fs[r] = s;
    }
    if (has_next && tm.warp == NW - 1) {
      const int nxt = cur ^ 1;
      load_geo(geo, Kn, nelt, sgbuf(nxt), lane, 32);
      __syncwarp();
      build_columns<D2, D3, M, MP>(sgbuf(nxt), colbuf(nxt), lane);
    }
    tm.sync();
    if (F)  // recovery cache: Vs = S^-1 V (d3 x m) and fs = S^-1 f after M^-1
      for (int idx = tm.tid; idx < D3 * M + D3; idx += NT) {
        const int r = idx % D3, c = idx / D3;
        F[Dm::NSYM + idx] = c < M ? Vs[r + c * LD] : (r < tab.nu ? fs[r] : 0.0);
      }

    // ---- P5: C = tauDD + (n_l1.n_l2) o (W Zp) - V^T Vs (lower tiles, mirrored);
    //      Cf; then the next element's D and f (Sb, fv are free)
    for (int tile = tm.warp; tile < NLOW; tile += NW) {
      int mt = 0, rem = tile;
      while (rem > mt) { rem -= mt + 1; ++mt; }
      const int nt = rem;
      const int r = mt * 8 + g;
      double v0 = 0, v1 = 0;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int k = kk * 4 + t;
        dmma(v0, v1, Vb[k + r * LD], Vs[k + (nt * 8 + g) * LD]);
      }
      const double z0 = Zb[tile * 64 + 2 * lane], z1 = Zb[tile * 64 + 2 * lane + 1];
      if (r < M) {
        const int l1 = r / D2;
        const double n1x = sg[10 + 3 * l1], n1y = sg[11 + 3 * l1], n1z = sg[12 + 3 * l1];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = nt * 8 + 2 * t + e;
          if (c > r || c >= M) continue;
          const int l2 = c / D2;
          const double nn = n1x * nsc[c] + n1y * nsc[MP + c] + n1z * nsc[2 * MP + c];
          double v = nn * (e ? z1 : z0) - (e ? v1 : v0);
          if (l1 == l2) v += Tc[c] * __ldg(tab.DD + (r - l1 * D2) + (c - l2 * D2) * D2);
          Ck[r + c * M] = v;
          if (c != r) Ck[c + r * M] = v;
        }
      }
    }
    for (int r = tm.tid; r < M; r += NT) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D3; ++k) s += Vb[k + r * LD] * fs[k];
      Cfout[K * M + r] = s;
    }
    if (has_next) {  // Sb and fv are not read in P5

      for (int j = 0; j < D3; ++j) {
        const int b0 = sym_idx(j, j, D3);
        for (int i = tm.tid; i < D3 - j; i += NT) Sb[(j + i) + j * LD] = Dsym[Kn * Dm::NSYM + b0 + i];
      }
      for (int i = tm.tid; i < D3; i += NT) fv[i] = fvec[Kn * D3 + i];
      cur ^= 1;
    }
    tm.sync();
  }
}

// K5 for the cache {Mi, Vs = Si V, fs = Si f}:
//   u = fs + Vs lambda,  q_s = Mi (C_s^T u - E_s^T lambda)
template <int K_>
__global__ void __launch_bounds__(kRecWarps * 32)
recover2_kernel(DevTab tab, int nelt, GeoDev geo, const int* __restrict__ facebyele,
                const double* __restrict__ factors, const double* __restrict__ uhat,
                double* __restrict__ qx, double* __restrict__ qy, double* __restrict__ qz,
                double* __restrict__ uout) {
  using Dm = C2Dims<K_>;
  using Rd = RecDims<K_>;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, NS = Dm::NSYM;
  __shared__ double sh[kRecWarps][Rd::PER_WARP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* lam = sh[warp];
  double* tv = lam + Rd::S1;
  double* uu = tv + Rd::S3;
  double* pp = uu + Rd::SD;
  double* sg = pp + Rd::S3;
  const long K = long(blockIdx.x) * kRecWarps + warp;
  if (K >= nelt) return;
  const double* F = factors + K * Dm::FACTORS;
  const double* Mi = F;
  const double* Vs = F + NS;
  const double* fs = F + NS + D3 * M;
  load_geo(geo, K, nelt, sg, lane, 32);
  for (int i = lane; i < M; i += 32) {
    const int l = i / D2;
    lam[i] = uhat[long(facebyele[long(l) * nelt + K]) * D2 + (i - l * D2)];
  }
  __syncwarp();
  for (int r = lane; r < D3; r += 32) {  // u = S^-1 (f + V lambda) = fs + Vs lambda
    double s = fs[r];
    for (int c = 0; c < M; ++c) s += Vs[r + c * D3] * lam[c];
    uu[r] = s;
  }
  __syncwarp();
  const double* a9 = sg + 1;
  const double* nrm = sg + 10;
  const double* pm = sg + 26;
  for (int j = lane; j < D3; j += 32) {
    double p[3];
    for (int s = 0; s < 3; ++s) {
      const double* C = tab.Chat + s * D3 * D3 + j * D3;
      double acc = 0.0;
      for (int i = 0; i < D3; ++i) acc += __ldg(C + i) * uu[i];
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
  double* outs[3] = {qx, qy, qz};
  for (int idx = lane; idx < 3 * D3; idx += 32) {  // q_s = Mi r_s
    const int s = idx / D3, i = idx - s * D3;
    double acc = 0.0;
    for (int j = 0; j < D3; ++j) acc += Mi[j >= i ? sym_idx(j, i, D3) : sym_idx(i, j, D3)] * pp[s * D3 + j];
    outs[s][K * D3 + i] = acc;
  }
  for (int i = lane; i < D3; i += 32) uout[K * D3 + i] = uu[i];
}

}  // namespace hdgb
