// K3 v6 (k = 3): static condensation, one warp per element, DMMA operands
// chained through registers.
//
// Same algebra as v3 (kernels_condense3.cuh): with Mi = M^-1 and
//   Y_h  = Chat_h Mi                       (d3 x d3, h = reference direction)
//   R'_h = sum_h' g(h', h) Y_h'            (g = a^T a)
//   S    = D + sum_h R'_h Chat_h^T         (= D + sum_s C_s M^-1 C_s^T)
//   V^T  = W_l (sum_h beta_h(l) Y_h + T_l I)^T   per face l (rows of face l)
//   Vs^T = V^T Si,   Zp^T = W Mi,   Si = S^-1
//   C    = tauDD + (n_l1 . n_l2) o (Zp^T W^T) - Vs^T V^T^T,   Cf = Vs^T f
// (C, Cf = A3 A1^-1 A2 + tauDD, A3 A1^-1 Af of local_solver.cpp:71-100).
//
// v3 ran every contraction as a CTA-wide phase over shared-memory operands
// (five CTA barriers per batch, ~1.4 fragment loads per DMMA, the L1/shared
// pipe at 71% while the DMMA pipe sat at 37%). Here one warp owns an
// element from the packed M to the stored C, with no CTA barrier in the
// element loop, and two warps share each SM sub-partition so one's sweep
// inverse (DFMA-latency bound) overlaps the other's DMMA phases (one warp
// with two independent accumulator chains already saturates its
// sub-partition's DMMA issue: 26-cycle latency, 16-cycle issue,
// tools/microbench/dmma_lat.cu).
//
// Register chaining: an accumulator tile holds X[g][2t], X[g][2t+1] in lane
// (g, t); a DMMA A fragment wants A[g][k(t)], a B fragment B[k(t)][g]. So a
// row strip of accumulator tiles IS a set of A (or, for the transposed
// product, B) fragments if the contraction index runs in the permuted order
// kidx: ksteps (tile 0, even), (tile 0, odd), (tile 1, even), (tile 1, odd)
// take k = 2t, 2t + 1, 8 + 2t, 9 + 2t from the lane's own registers; the
// fifth kstep (k = 16 + t, the last 4 of d3 = 20) is gathered by two
// shuffles. The other operand is read in the same order from a k-fastest
// table (row stride 24: two 16-byte loads give four ksteps, conflict-free).
// Per element: 645 DMMA (as v3) and ~80 16-byte fragment loads + 30 8-byte
// loads instead of ~900 8-byte loads.
#pragma once

#include "kernels_condense3.cuh"

namespace hdgb {

struct C6Dims {
  static constexpr int D3 = 20, D2 = 10, M = 40, NSYM = 210;
  static constexpr int LT = 24;  // row stride of the k-fastest operands (Chat, W, V^T)
  static constexpr int LQ = 26;  // Mi / Si storage: (row i, column c) at i * LQ + c
  static constexpr int LS = 24;  // S storage for the sweep (row-major)
  static constexpr int CH_SZ = 24 * LT, WT_SZ = D2 * LT;
  // per CTA: Chat_h row-major (rows / columns >= 20 zero), W^{l,mu} row-major, tauDD
  static constexpr int OFF_CH = 0, OFF_WT = OFF_CH + 3 * CH_SZ, OFF_DD = OFF_WT + 24 * WT_SZ;
  static constexpr int OFF_ZR = round_up(OFF_DD + D2 * D2, 2);  // a zero row (LT)
  static constexpr int CTA_EXTRA = OFF_ZR + LT;
  // per warp (all offsets even: 16-byte aligned)
  static constexpr int P_SQ = 0;                 // Mi (LQ), then S (LS), then Si (LQ)
  static constexpr int P_VT = P_SQ + 24 * LQ;    // V^T, M x LT; packed-Mi staging before that
  static constexpr int P_ST = P_VT + M * LT;     // sweep stage, 128
  static constexpr int P_M = P_ST + 128;         // packed M of the element (cp.async)
  static constexpr int P_D = P_M + NSYM;         // packed D
  static constexpr int FG_SZ = 48;               // f (20) + geometry record (28)
  static constexpr int P_FG = P_D + NSYM;        // 2 slots (current / next element)
  static constexpr int P_DG = P_FG + 2 * FG_SZ;  // derived per-element scalars, 48
  static constexpr int PER_ELT = P_DG + 48;
  static constexpr int FACTORS = round_up(NSYM + D3 * M + D3, 2);
  // derived scalars (DG): g(h,h') 9, beta[f][h] 12, nn[l1][l2] 16, T 4, vol, table row base 4
  static constexpr int DG_G = 0, DG_B = 9, DG_NN = 21, DG_T = 37, DG_VOL = 41, DG_TB = 42;
};
static_assert(C6Dims::P_D % 2 == 0 && C6Dims::P_FG % 2 == 0 && C6Dims::PER_ELT % 2 == 0, "16-byte slots");

#ifndef HDG_C6_NW
#define HDG_C6_NW 8
#endif

struct C6Cfg {
  static constexpr int NW = HDG_C6_NW;
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem_src) : "memory");
}

// contraction index of kstep s (0..4) for lane t: the accumulator-chained order
__device__ __forceinline__ int c6_kidx(int s, int t) { return s < 4 ? (s >> 1) * 8 + 2 * t + (s & 1) : 16 + t; }

// five fragments of one k-fastest row (stride LT, 16-byte aligned) in kidx order
__device__ __forceinline__ void c6_rowfrag(const double* p, int t, double (&f)[5]) {
  const double2 a = *reinterpret_cast<const double2*>(p + 2 * t);
  const double2 b = *reinterpret_cast<const double2*>(p + 8 + 2 * t);
  f[0] = a.x;
  f[1] = a.y;
  f[2] = b.x;
  f[3] = b.y;
  f[4] = p[16 + t];  // 2-way bank conflict: the wavefronts of a 16-byte load + select, no select
}

// the row strip x[n] (n = 0..2 column tiles over d3) of accumulator tiles as
// five kidx-ordered fragments (A of X, or B of X^T)
__device__ __forceinline__ void c6_chain(const double (&x)[3][2], int lane, double (&f)[5]) {
  f[0] = x[0][0];
  f[1] = x[0][1];
  f[2] = x[1][0];
  f[3] = x[1][1];
  const int src = (lane & ~3) | ((lane & 3) >> 1);
  const double v0 = __shfl_sync(0xffffffffu, x[2][0], src);
  const double v1 = __shfl_sync(0xffffffffu, x[2][1], src);
  f[4] = (lane & 1) ? v1 : v0;
}

// B fragments b[s][n] = X[kidx(s)][8n + g] of a symmetric d3 x d3 inverse
// stored by its sweep (Q[i * LQ + c] = lane c's column entry i); every
// symmetric pair reads the lower-index lane's below-diagonal entry (the two
// triangles of a sweep round differently, kernels_condense3.cuh)
__device__ __forceinline__ void c6_symfrag(const double* Q, int g, int t, double (&b)[5][3]) {
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int k = c6_kidx(s, t);
#pragma unroll
    for (int n = 0; n < 3; ++n) {
      const int col = 8 * n + g;
      const int hi = k > col ? k : col, lo = k > col ? col : k;
      b[s][n] = col < C6Dims::D3 ? Q[hi * C6Dims::LQ + lo] : 0.0;
    }
  }
}

__device__ __forceinline__ void c6_sweep(double (&a)[C6Dims::D3], double* stage, int lane, double& pmin, double& pmax) {
  gj_sweep_inverse<C6Dims::D3>(a, stage, lane, pmin, pmax);
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1)
condense6_kernel(DevTab tab, int nelt, GeoDev geo, const double* __restrict__ Msym,
                 const double* __restrict__ Dsym, const double* __restrict__ fvec,
                 double* __restrict__ Cout, double* __restrict__ Cfout, double* __restrict__ factors,
                 double* __restrict__ pivstat) {
  using Dm = C6Dims;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, NSYM = Dm::NSYM, LT = Dm::LT, LQ = Dm::LQ, LS = Dm::LS;
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;

  // ---- CTA tables (the only CTA barrier)
  double* CH = smem + Dm::OFF_CH;
  double* WT = smem + Dm::OFF_WT;
  double* DDs = smem + Dm::OFF_DD;
  for (int i = threadIdx.x; i < 3 * Dm::CH_SZ; i += blockDim.x) {
    const int h = i / Dm::CH_SZ, rem = i - h * Dm::CH_SZ, r = rem / LT, k = rem - r * LT;
    CH[i] = (r < D3 && k < D3) ? tab.Chat[h * D3 * D3 + r + k * D3] : 0.0;
  }
  for (int i = threadIdx.x; i < 24 * Dm::WT_SZ; i += blockDim.x) {
    const int tb = i / Dm::WT_SZ, rem = i - tb * Dm::WT_SZ, r = rem / LT, k = rem - r * LT;
    WT[i] = k < D3 ? tab.Wlm[tb * D2 * D3 + r + k * D2] : 0.0;
  }
  for (int i = threadIdx.x; i < D2 * D2; i += blockDim.x) DDs[i] = tab.DD[i];
  double* ZR = smem + Dm::OFF_ZR;
  for (int i = threadIdx.x; i < LT; i += blockDim.x) ZR[i] = 0.0;
  __syncthreads();

  double* W0 = smem + Dm::CTA_EXTRA + warp * Dm::PER_ELT;
  double* SQ = W0 + Dm::P_SQ;
  double* VT = W0 + Dm::P_VT;
  double* ST = W0 + Dm::P_ST;
  double* Mp = W0 + Dm::P_M;
  double* Dp = W0 + Dm::P_D;
  double* DG = W0 + Dm::P_DG;
  const int nu = tab.nu;
  const bool al16 = ((reinterpret_cast<uintptr_t>(Msym) | reinterpret_cast<uintptr_t>(Dsym) |
                      reinterpret_cast<uintptr_t>(fvec)) & 15) == 0;

  // packed M, D, f and the geometry record of element K -> this warp's slot
  auto prefetch = [&](long K, int slot) {
    double* fg = W0 + Dm::P_FG + slot * Dm::FG_SZ;
    if (al16) {
      for (int q = lane; q < NSYM / 2; q += 32) {
        cp_async16(Mp + 2 * q, Msym + K * NSYM + 2 * q);
        cp_async16(Dp + 2 * q, Dsym + K * NSYM + 2 * q);
      }
      if (lane < D3 / 2) cp_async16(fg + 2 * lane, fvec + K * D3 + 2 * lane);
    } else {
      for (int q = lane; q < NSYM; q += 32) {
        cp_async8(Mp + q, Msym + K * NSYM + q);
        cp_async8(Dp + q, Dsym + K * NSYM + q);
      }
      if (lane < D3) cp_async8(fg + lane, fvec + K * D3 + lane);
    }
    double* sg = fg + D3;  // [0] volume, [1..9] a, [10..21] normals, [22..25] T, [26..27] perm (4 x int32)
    if (lane == 0) cp_async8(sg, geo.volume + K);
    else if (lane < 10) cp_async8(sg + lane, geo.piola + long(lane - 1) * nelt + K);
    else if (lane < 22) cp_async8(sg + lane, geo.normals + long(lane - 10) * nelt + K);
    else if (lane < 26) cp_async8(sg + lane, geo.T + long(lane - 22) * nelt + K);
    else if (lane < 30) cp_async4(reinterpret_cast<int*>(sg + 26) + (lane - 26), geo.perm + long(lane - 26) * nelt + K);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  const long wstride = long(gridDim.x) * NW;
  long K = long(blockIdx.x) * NW + warp;
  int cur = 0;
  // packed M staged in Mp -> lane columns (lane c < D3 owns column c)
  auto load_M = [&](double (&a)[D3], bool) {
#pragma unroll
    for (int i = 0; i < D3; ++i) {
      const int r = i > lane ? i : lane, c = i > lane ? lane : i;
      a[i] = lane < D3 ? Mp[sym_idx(r, c, D3)] : 0.0;
    }
  };
  // M^-1 of element Kx (lane columns) -> SQ (stride LQ), its packed lower part
  // -> recovery cache by one TMA bulk store (staged in VT, retired before VT
  // is rewritten), pivot statistics
  auto store_Mi = [&](const double (&a)[D3], long Kx, double pmin, double pmax) {
    if (lane < D3) {
#pragma unroll
      for (int i = 0; i < D3; ++i) SQ[i * LQ + lane] = a[i];
    }
    if (factors) {
      if (lane < D3) {
        double* dst = VT + lane * (2 * D3 - lane + 1) / 2 - lane;
#pragma unroll
        for (int i = 0; i < D3; ++i)
          if (i >= lane) dst[i] = a[i];
      }
      __syncwarp();
      if (lane == 0) bulk_store(factors + Kx * Dm::FACTORS, VT, NSYM * 8);
    }
    if (lane == 0) store_pivstat(pivstat, Kx, 0, pmin, pmax);
    __syncwarp();
  };
  if (K < nelt) {  // the first element's M^-1 on its own; later ones run inside the previous element's C phase
    prefetch(K, 0);
    cp_async_wait_all();
    __syncwarp();
    double a[D3];
    load_M(a, true);
    __syncwarp();
    double pmin = 1e300, pmax = 0.0;
    c6_sweep(a, ST, lane, pmin, pmax);
    store_Mi(a, K, pmin, pmax);
  }

  for (; K < nelt; K += wstride, cur ^= 1) {
    // (this element's inputs arrived before its M^-1)
    const double* fg = W0 + Dm::P_FG + cur * Dm::FG_SZ;
    const double* sg = fg + D3;
    // ---- derived scalars
    for (int q = lane; q < 46; q += 32) {
      double v;
      if (q < 9) {  // g(h, h') = sum_s a(s, h) a(s, h')
        const int h = q / 3, h2 = q % 3;
        v = sg[1 + h] * sg[1 + h2] + sg[4 + h] * sg[4 + h2] + sg[7 + h] * sg[7 + h2];
      } else if (q < 21) {  // beta_h(f) = sum_s a(s, h) n_f[s]
        const int f = (q - 9) / 3, h = (q - 9) % 3;
        v = sg[1 + h] * sg[10 + 3 * f] + sg[4 + h] * sg[11 + 3 * f] + sg[7 + h] * sg[12 + 3 * f];
      } else if (q < 37) {
        const int l1 = (q - 21) >> 2, l2 = (q - 21) & 3;
        v = sg[10 + 3 * l1] * sg[10 + 3 * l2] + sg[11 + 3 * l1] * sg[11 + 3 * l2] + sg[12 + 3 * l1] * sg[12 + 3 * l2];
      } else if (q < 41) {
        v = sg[22 + (q - 37)];
      } else if (q == 41) {
        v = sg[0];
      } else {  // W^{l, mu} row base of face l in WT
        const int l = q - 42, mu = reinterpret_cast<const int*>(sg + 26)[l];
        v = double((6 * l + mu - 1) * Dm::WT_SZ);
      }
      DG[q] = v;
    }
    double mib[5][3];
    c6_symfrag(SQ, g, t, mib);
    if (factors && lane == 0) bulk_store_wait_read();  // the packed M^-1 staged in VT is read out
    __syncwarp();

    // ---- per d3 row tile i: Y_h, R'_h, S row tiles, V^T column tile
    double gm[3][3];
#pragma unroll
    for (int h = 0; h < 3; ++h)
#pragma unroll
      for (int h2 = 0; h2 < 3; ++h2) gm[h][h2] = DG[Dm::DG_G + 3 * h + h2];
    const double vol = DG[Dm::DG_VOL];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double y[3][3][2];
      double ca[3][5];
#pragma unroll
      for (int h = 0; h < 3; ++h) c6_rowfrag(CH + h * Dm::CH_SZ + (8 * i + g) * LT, t, ca[h]);
#pragma unroll
      for (int h = 0; h < 3; ++h)
#pragma unroll
        for (int n = 0; n < 3; ++n) y[h][n][0] = y[h][n][1] = 0.0;
#pragma unroll
      for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int h = 0; h < 3; ++h)
#pragma unroll
          for (int n = 0; n < 3; ++n) dmma(y[h][n][0], y[h][n][1], ca[h][s], mib[s][n]);
      // S row tiles j <= i: S = D + sum_h R'_h Chat_h^T
      {
        double ra[3][5];
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          double rp[3][2];
#pragma unroll
          for (int n = 0; n < 3; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              rp[n][e] = gm[0][h] * y[0][n][e] + gm[1][h] * y[1][n][e] + gm[2][h] * y[2][n][e];
          c6_chain(rp, lane, ra[h]);
        }
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          if (j > i) break;
          double sa[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            double cb[5];
            if (j == i) {
#pragma unroll
              for (int s = 0; s < 5; ++s) cb[s] = ca[h][s];
            } else {
              c6_rowfrag(CH + h * Dm::CH_SZ + (8 * j + g) * LT, t, cb);
            }
#pragma unroll
            for (int s = 0; s < 5; ++s) dmma(sa[s & 1][0], sa[s & 1][1], ra[h][s], cb[s]);
          }
          // lower entries c <= r, mirrored: the sweep needs S exactly symmetric
          const int r = 8 * i + g;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * j + 2 * t + e;
            if (r < D3 && c <= r) {
              const double v = (r >= nu || c >= nu) ? (r == c ? 6.0 * vol : 0.0)
                                                    : Dp[sym_idx(r, c, D3)] + sa[0][e] + sa[1][e];
              SQ[r * LS + c] = v;
              SQ[c * LS + r] = v;
            }
          }
        }
      }
      // V^T column tile i: V^T[c][r] = sum_k W_l(c)[c'][k] Z_l[r][k], Z_l = sum_h beta_h(l) Y_h + T_l I
      {
        double yb[3][5];
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          double yy[3][2];
#pragma unroll
          for (int n = 0; n < 3; ++n) yy[n][0] = y[h][n][0], yy[n][1] = y[h][n][1];
          c6_chain(yy, lane, yb[h]);
        }
        double zf[4][5];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const double b0 = DG[Dm::DG_B + 3 * f], b1 = DG[Dm::DG_B + 3 * f + 1], b2 = DG[Dm::DG_B + 3 * f + 2];
          const double Tf = DG[Dm::DG_T + f];
#pragma unroll
          for (int s = 0; s < 5; ++s) {
            double z = b0 * yb[0][s] + b1 * yb[1][s] + b2 * yb[2][s];
            if (c6_kidx(s, t) == 8 * i + g) z += Tf;
            zf[f][s] = z;
          }
        }
#pragma unroll
        for (int jc = 0; jc < 5; ++jc) {
          const int c = 8 * jc + g, fc = c / D2;
          const double* wr = WT + int(DG[Dm::DG_TB + fc]) + (c - fc * D2) * LT;
          double va[2] = {0.0, 0.0};
          const int f0 = (8 * jc) / D2, f1 = (8 * jc + 7) / D2;  // faces the tile's rows span
#pragma unroll
          for (int f = f0; f <= f1; ++f) {
            // rows of another face read a zero row (masking by address, not by selects)
            double wa[5];
            c6_rowfrag(f0 == f1 || fc == f ? wr : ZR, t, wa);
#pragma unroll
            for (int s = 0; s < 5; ++s) dmma(va[0], va[1], wa[s], zf[f][s]);
          }
          const int r0 = 8 * i + 2 * t;
          if (r0 < LT) {
            const double v0 = r0 < nu ? va[0] : 0.0, v1 = r0 + 1 < nu ? va[1] : 0.0;
            *reinterpret_cast<double2*>(VT + c * LT + r0) = make_double2(v0, v1);
          }
        }
      }
    }
    __syncwarp();
    const long Kn = K + wstride;
    const bool has_next = Kn < nelt;
    if (has_next) prefetch(Kn, cur ^ 1);  // packed M, D of this element are dead

    // ---- S^-1: sweep (S stored row-major with stride LS), then stored with stride LQ
    double sib[5][3];
    {
      double a[D3];
#pragma unroll
      for (int i = 0; i < D3; ++i) a[i] = lane < D3 ? SQ[i * LS + lane] : 0.0;
      __syncwarp();
      double pmin = 1e300, pmax = 0.0;
      c6_sweep(a, ST, lane, pmin, pmax);
      if (lane < D3) {
#pragma unroll
        for (int i = 0; i < D3; ++i) SQ[i * LQ + lane] = a[i];
      }
      if (lane == 0) store_pivstat(pivstat, K, 1, pmin, pmax);
      __syncwarp();
      c6_symfrag(SQ, g, t, sib);
      if (factors && lane < D3) {  // fs = S^-1 f (canonical entries)
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < D3; ++k) {
          const int hi = k > lane ? k : lane, lo = k > lane ? lane : k;
          s += SQ[hi * LQ + lo] * fg[k];
        }
        factors[K * Dm::FACTORS + NSYM + D3 * M + lane] = lane < nu ? s : 0.0;
      }
    }

    // ---- C, Cf and the Vs record, by m row tiles jc
    // W rows of this lane in every m row tile (V^T and W fragments are
    // reloaded per C tile: fewer live registers, measured faster than keeping them)
    const double* wrow[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int c = 8 * j + g, fc = c / D2;
      wrow[j] = WT + int(DG[Dm::DG_TB + fc]) + (c - fc * D2) * LT;
    }
    double fr[3][2];  // f at this lane's Vs rows 8n + 2t, + 1
#pragma unroll
    for (int n = 0; n < 3; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) fr[n][e] = 8 * n + 2 * t + e < D3 ? fg[8 * n + 2 * t + e] : 0.0;
    double* Ck = Cout + K * M * M;
#pragma unroll
    for (int jc = 0; jc < 5; ++jc) {
      double vfr[5], wfr[5];
      c6_rowfrag(VT + (8 * jc + g) * LT, t, vfr);
      c6_rowfrag(wrow[jc], t, wfr);
      double vs[3][2], zp[3][2];
#pragma unroll
      for (int n = 0; n < 3; ++n) vs[n][0] = vs[n][1] = zp[n][0] = zp[n][1] = 0.0;
#pragma unroll
      for (int s = 0; s < 5; ++s)
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          dmma(vs[n][0], vs[n][1], vfr[s], sib[s][n]);
          dmma(zp[n][0], zp[n][1], wfr[s], mib[s][n]);
        }
      const int r = 8 * jc + g;  // row of C / column of Vs
      {
        double p = 0.0;
#pragma unroll
        for (int n = 0; n < 3; ++n) {
          const int rr = 8 * n + 2 * t;
          if (factors && rr < D3)
            *reinterpret_cast<double2*>(factors + K * Dm::FACTORS + NSYM + rr + r * D3) =
                make_double2(vs[n][0], vs[n][1]);
          p += vs[n][0] * fr[n][0] + vs[n][1] * fr[n][1];
        }
        p += __shfl_xor_sync(FULL, p, 1);
        p += __shfl_xor_sync(FULL, p, 2);
        if (t == 0) Cfout[K * M + r] = p;
      }
      double vsa[5], zpa[5];
      c6_chain(vs, lane, vsa);
      c6_chain(zp, lane, zpa);
      const int l1 = r / D2;
#pragma unroll
      for (int j = 0; j <= jc; ++j) {
        double c1[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0};
        double wb[5], vb[5];
        if (j < jc) {
          c6_rowfrag(wrow[j], t, wb);
          c6_rowfrag(VT + (8 * j + g) * LT, t, vb);
        } else {
#pragma unroll
          for (int s = 0; s < 5; ++s) wb[s] = wfr[s], vb[s] = vfr[s];
        }
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          dmma(c1[0], c1[1], zpa[s], wb[s]);
          dmma(c2[0], c2[1], vsa[s], vb[s]);
        }
        const int c0 = 8 * j + 2 * t;
        double val[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = c0 + e, l2 = c / D2;
          val[e] = DG[Dm::DG_NN + 4 * l1 + l2] * c1[e] - c2[e];
          if (l1 == l2) val[e] += DG[Dm::DG_T + l1] * DDs[(r - l1 * D2) + (c - l2 * D2) * D2];
        }
        if (c0 <= r) Ck[r + c0 * M] = val[0];
        if (c0 + 1 <= r) Ck[r + (c0 + 1) * M] = val[1];
        if (c0 + 1 < r) *reinterpret_cast<double2*>(Ck + c0 + r * M) = make_double2(val[0], val[1]);
        else if (c0 < r) Ck[c0 + r * M] = val[0];
      }
    }
    __syncwarp();
    if (has_next) {  // M^-1 of the next element (measured: interleaving its pivot steps with
                     // this element's C tiles is slower, the sweep's DFMAs share the DMMA pipe)
      double am[D3], pmin = 1e300, pmax = 0.0;
      cp_async_wait_all();
      __syncwarp();
      load_M(am, true);
      __syncwarp();
      c6_sweep(am, ST, lane, pmin, pmax);
      store_Mi(am, Kn, pmin, pmax);
    }
  }
}

}  // namespace hdgb
