// K3 v6 (k = 2, 3): static condensation, one warp per element, DMMA operands
// chained through registers.
//
// Same algebra as the round-1 CTA-phase kernel (v3): with Mi = M^-1 and
//   Y_h  = Chat_h Mi                       (d3 x d3, h = reference direction)
//   R'_h = sum_h' g(h', h) Y_h'            (g = a^T a)
//   S    = D + sum_h R'_h Chat_h^T         (= D + sum_s C_s M^-1 C_s^T)
//   V^T  = W_l (sum_h beta_h(l) Y_h + T_l I)^T   per face l (rows of face l)
//   Vs^T = V^T Si,   Zp^T = W Mi,   Si = S^-1
//   C    = tauDD + (n_l1 . n_l2) o (Zp^T W^T) - Vs^T V,   Cf = Vs^T f
// (C, Cf = A3 A1^-1 A2 + tauDD, A3 A1^-1 Af of local_solver.cpp:71-100).
//
// v3 ran every contraction as a CTA-wide phase over shared-memory operands
// (five CTA barriers per batch, ~1.4 fragment loads per DMMA, the L1/shared
// pipe at 71% while the DMMA pipe sat at 37%). Here one warp owns an
// element from the packed M to the stored C, with no CTA barrier in the
// element loop, and two or more warps share each SM sub-partition so one's
// sweep inverse (DFMA-latency bound) overlaps another's DMMA phases (one
// warp with two independent accumulator chains already saturates its
// sub-partition's DMMA issue: 26-cycle latency, 16-cycle issue,
// tools/microbench/dmma_lat.cu).
//
// Register chaining: an accumulator tile holds X[g][2t], X[g][2t+1] in lane
// (g, t); a DMMA A fragment wants A[g][k(t)], a B fragment B[k(t)][g]. So a
// row strip of accumulator tiles IS a set of A (or, for the transposed
// product, B) fragments if the contraction index runs in the permuted order
// kidx: per whole 8-column tile two ksteps k = 8n + 2t, 8n + 2t + 1 taken
// from the lane's own registers; the d3 remainder (the last 4 of d3 = 20,
// the last 2 of d3 = 10, zero-padded) as one natural kstep k = 8n + t
// gathered by two shuffles. The other operand is read in the same order from
// a k-fastest table (row stride LT = 20 at k = 3, 24 at k = 2, measured: one
// 16-byte load gives a tile's two ksteps).
#pragma once

#include "kernels_condense2.cuh"

namespace hdgb {

template <int K_>
struct C6Dims {
  static constexpr int D3 = cdim3(K_), D2 = cdim2(K_), M = 4 * cdim2(K_), NSYM = D3 * (D3 + 1) / 2;
  static constexpr int NP = D3 / 8;                       // whole 8-wide tiles of d3
  static constexpr int NT3 = (D3 + 7) / 8;                // d3 tiles (row / column)
  static constexpr int KS = 2 * NP + (D3 % 8 ? 1 : 0);    // ksteps over d3
  static constexpr int NTM = M / 8;                       // m tiles
  // d3 <= 16 (k = 2): S^-1 of an element and M^-1 of the warp's next element
  // as one sweep on the two 16-lane halves (gj_sweep_seg)
  static constexpr bool PAIR = D3 <= 16;
#ifndef HDG_C6_LT3
#define HDG_C6_LT3 20
#endif
#ifndef HDG_C6_LT2
#define HDG_C6_LT2 24
#endif
  // row stride of the k-fastest operands (Chat, W, V^T): the fragments read columns < 8 NP + 4 only
  static constexpr int LT = K_ == 3 ? HDG_C6_LT3 : HDG_C6_LT2;
  static_assert(LT % 2 == 0 && LT >= 8 * (D3 / 8) + (D3 % 8 ? 4 : 0), "row stride covers every kstep");
  static constexpr int LQ = K_ == 3 ? 26 : 14;  // Mi / Si storage: (row i, column c) at i * LQ + c
  static constexpr int LS = K_ == 3 ? 24 : 12;  // S storage for the sweep (row-major)
  static constexpr int CH_SZ = NT3 * 8 * LT, WT_SZ = D2 * LT;
  // per CTA: Chat_h row-major (rows / columns >= d3 zero), W^{l,mu} row-major, tauDD, a zero row
  static constexpr int OFF_CH = 0, OFF_WT = OFF_CH + 3 * CH_SZ, OFF_DD = OFF_WT + 24 * WT_SZ;
  static constexpr int OFF_ZR = round_up(OFF_DD + D2 * D2, 2);
  static constexpr int CTA_EXTRA = OFF_ZR + LT;
  // per warp (every slot 16-byte aligned)
  static constexpr int P_SQ = 0;                                 // Mi (LQ), then S (LS), then Si (LQ)
  static constexpr int P_VT = P_SQ + round_up(D3 * LQ, 2);       // V^T, M x LT; packed-Mi staging before that
  static constexpr int P_ST = P_VT + M * LT;                     // sweep stage, 128
  static constexpr int P_M = P_ST + (PAIR ? 256 : 128);          // packed M of the element (cp.async)
  static constexpr int P_D = P_M + round_up(NSYM, 2);            // packed D
  static constexpr int FG_SZ = round_up(D3 + 28, 2);             // f + geometry record
  static constexpr int P_FG = P_D + round_up(NSYM, 2);           // 2 slots (current / next element)
  static constexpr int P_DG = P_FG + 2 * FG_SZ;                  // derived per-element scalars, 48
  // k = 3: M^-1 kept in its own buffer (stride d3), its fragments reloaded per
  // row tile and for the C phase instead of held in registers (measured
  // 4.00 -> 3.94 ms at C2; at k = 2 no gain)
  static constexpr bool MIQ = K_ == 3 || PAIR;
  static constexpr int P_MQ = P_DG + 48;
  static constexpr int MQS = round_up(D3 * D3, 2);  // PAIR: two slots (this element's, the next one's)
  static constexpr int PER_ELT = P_MQ + (MIQ ? (PAIR ? 2 : 1) * MQS : 0);
  static constexpr int FACTORS = round_up(NSYM + D3 * M + D3, 2);
  // the packed M^-1 record goes out by one TMA bulk store (a 16-byte multiple)
  static constexpr bool BULK_MI = (NSYM * 8) % 16 == 0;
  // derived scalars (DG): g(h,h') 9, beta[f][h] 12, nn[l1][l2] 16, T 4, vol, table row base 4
  static constexpr int DG_G = 0, DG_B = 9, DG_NN = 21, DG_T = 37, DG_VOL = 41, DG_TB = 42;
};

#ifndef HDG_C6_NW3
#define HDG_C6_NW3 8
#endif
#ifndef HDG_C6_NW2
#define HDG_C6_NW2 12
#endif
template <int K_>
struct C6Cfg {
  static constexpr int NW = K_ == 3 ? HDG_C6_NW3 : HDG_C6_NW2;
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem_src) : "memory");
}

// Structural zeros of the reference convection matrices. In the
// degree-graded orthonormal basis Chat_h[i][j] = (1/6) int P_i d_h P_j
// vanishes unless deg P_i < deg P_j: its rows i >= dim P_{k-1} are zero and the
// rest is strictly upper triangular. c6_ch_nz says whether the 8 x 4 block
// (row tile, kstep s in the kidx order) of Chat_h holds any nonzero; the
// blocks it denies are skipped as DMMA operands. hdg_b200_set_degree checks
// the pattern against the tables it uploads (capi.cu, check_chat_pattern).
#ifndef HDG_C6_SPARSE
#define HDG_C6_SPARSE 1
#endif
constexpr bool c6_ch_nz(int k, int h, int tile, int s) {
  if (!HDG_C6_SPARSE) return true;
  if (k == 3) {
    if (tile == 0) return !(h == 0 && s == 0);
    if (tile == 1) return s == 4 || (h == 2 && s == 3);
    return false;
  }
  if (k == 2) return tile == 0 && !(h == 0 && s == 0);
  return true;
}
// any nonzero block in the row tile (else Y_h and R'_h vanish on it for every h)
constexpr bool c6_tile_nz(int k, int tile) {
  for (int h = 0; h < 3; ++h)
    for (int s = 0; s < 8; ++s)
      if (c6_ch_nz(k, h, tile, s)) return true;
  return false;
}

// contraction index of kstep s for lane t: the accumulator-chained order
template <int K_>
__device__ __forceinline__ int c6_kidx(int s, int t) {
  constexpr int NP = C6Dims<K_>::NP;
  return s < 2 * NP ? (s >> 1) * 8 + 2 * t + (s & 1) : 8 * NP + t;
}

// the KS fragments of one k-fastest row (stride LT, 16-byte aligned) in kidx order
template <int K_>
__device__ __forceinline__ void c6_rowfrag(const double* p, int t, double (&f)[C6Dims<K_>::KS]) {
  using Dm = C6Dims<K_>;
#pragma unroll
  for (int n = 0; n < Dm::NP; ++n) {
    const double2 a = *reinterpret_cast<const double2*>(p + 8 * n + 2 * t);
    f[2 * n] = a.x;
    f[2 * n + 1] = a.y;
  }
  // remainder kstep: a 2-way bank conflict, the wavefronts of a 16-byte load + select
  if (Dm::KS > 2 * Dm::NP) f[2 * Dm::NP] = p[8 * Dm::NP + t];
}

// the row strip x[n] (n over the d3 column tiles) of accumulator tiles as
// KS kidx-ordered fragments (A of X, or B of X^T)
template <int K_>
__device__ __forceinline__ void c6_chain(const double (&x)[C6Dims<K_>::NT3][2], int lane,
                                         double (&f)[C6Dims<K_>::KS]) {
  using Dm = C6Dims<K_>;
#pragma unroll
  for (int n = 0; n < Dm::NP; ++n) {
    f[2 * n] = x[n][0];
    f[2 * n + 1] = x[n][1];
  }
  if (Dm::KS > 2 * Dm::NP) {
    const int src = (lane & ~3) | ((lane & 3) >> 1);
    const double v0 = __shfl_sync(0xffffffffu, x[Dm::NT3 - 1][0], src);
    const double v1 = __shfl_sync(0xffffffffu, x[Dm::NT3 - 1][1], src);
    f[2 * Dm::NP] = (lane & 1) ? v1 : v0;
  }
}

// B fragments b[s][n] = X[kidx(s)][8n + g] of a symmetric d3 x d3 inverse
// stored by its sweep (Q[i * LQ + c] = lane c's column entry i); every
// symmetric pair reads the lower-index lane's below-diagonal entry (the two
// triangles of a sweep round differently); k-padding
// rows and columns >= d3 read as zero
template <int K_, int LDQ = C6Dims<K_>::LQ>
__device__ __forceinline__ void c6_symfrag(const double* Q, int g, int t,
                                           double (&b)[C6Dims<K_>::KS][C6Dims<K_>::NT3]) {
  using Dm = C6Dims<K_>;
#pragma unroll
  for (int s = 0; s < Dm::KS; ++s) {
    const int k = c6_kidx<K_>(s, t);
#pragma unroll
    for (int n = 0; n < Dm::NT3; ++n) {
      const int col = 8 * n + g;
      const int hi = k > col ? k : col, lo = k > col ? col : k;
      b[s][n] = (col < Dm::D3 && k < Dm::D3) ? Q[hi * LDQ + lo] : 0.0;
    }
  }
}

// SP: the tables passed check_chat_pattern (capi.cu) and the zero blocks of
// Chat_h are skipped; otherwise (a rule too coarse to integrate P_i d_h P_j
// exactly) every block is contracted.
template <int K_, int NW, bool SP = true>
__global__ void __launch_bounds__(NW * 32, 1)
condense6_kernel(DevTab tab, int nelt, GeoDev geo, const double* __restrict__ Msym,
                 const double* __restrict__ Dsym, const double* __restrict__ fvec,
                 double* __restrict__ Cout, double* __restrict__ Cfout, double* __restrict__ factors,
                 double* __restrict__ pivstat) {
  using Dm = C6Dims<K_>;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, NSYM = Dm::NSYM, LT = Dm::LT, LQ = Dm::LQ, LS = Dm::LS;
  constexpr int KS = Dm::KS, NT3 = Dm::NT3, NTM = Dm::NTM;
  constexpr int KSP = SP ? K_ : -1;  // degree handed to the block masks (-1: nothing skipped)
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;

  // ---- CTA tables (the only CTA barrier)
  double* CH = smem + Dm::OFF_CH;
  double* WT = smem + Dm::OFF_WT;
  double* DDs = smem + Dm::OFF_DD;
  double* ZR = smem + Dm::OFF_ZR;
  for (int i = threadIdx.x; i < 3 * Dm::CH_SZ; i += blockDim.x) {
    const int h = i / Dm::CH_SZ, rem = i - h * Dm::CH_SZ, r = rem / LT, k = rem - r * LT;
    CH[i] = (r < D3 && k < D3) ? tab.Chat[h * D3 * D3 + r + k * D3] : 0.0;
  }
  for (int i = threadIdx.x; i < 24 * Dm::WT_SZ; i += blockDim.x) {
    const int tb = i / Dm::WT_SZ, rem = i - tb * Dm::WT_SZ, r = rem / LT, k = rem - r * LT;
    WT[i] = k < D3 ? tab.Wlm[tb * D2 * D3 + r + k * D2] : 0.0;
  }
  for (int i = threadIdx.x; i < D2 * D2; i += blockDim.x) DDs[i] = tab.DD[i];
  for (int i = threadIdx.x; i < LT; i += blockDim.x) ZR[i] = 0.0;
  __syncthreads();

  double* W0 = smem + Dm::CTA_EXTRA + warp * Dm::PER_ELT;
  double* SQ = W0 + Dm::P_SQ;
  double* VT = W0 + Dm::P_VT;
  double* ST = W0 + Dm::P_ST;
  double* Mp = W0 + Dm::P_M;
  double* Dp = W0 + Dm::P_D;
  double* DG = W0 + Dm::P_DG;
  double* MQ = W0 + Dm::P_MQ;
  const int nu = tab.nu;
  const bool al16 = NSYM % 2 == 0 && ((reinterpret_cast<uintptr_t>(Msym) | reinterpret_cast<uintptr_t>(Dsym) |
                                       reinterpret_cast<uintptr_t>(fvec)) & 15) == 0;

  // packed D of element K -> Dp (one cp.async group)
  auto prefetch_D = [&](long K) {
    if (al16) {
      for (int q = lane; q < NSYM / 2; q += 32) cp_async16(Dp + 2 * q, Dsym + K * NSYM + 2 * q);
    } else {
      for (int q = lane; q < NSYM; q += 32) cp_async8(Dp + q, Dsym + K * NSYM + q);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // packed M, f and the geometry record of element K -> Mp and FG slot (one cp.async group)
  auto prefetch_M = [&](long K, int slot) {
    double* fg = W0 + Dm::P_FG + slot * Dm::FG_SZ;
    if (al16) {
      for (int q = lane; q < NSYM / 2; q += 32) cp_async16(Mp + 2 * q, Msym + K * NSYM + 2 * q);
      if (lane < D3 / 2) cp_async16(fg + 2 * lane, fvec + K * D3 + 2 * lane);
    } else {
      for (int q = lane; q < NSYM; q += 32) cp_async8(Mp + q, Msym + K * NSYM + q);
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
  // packed M staged in Mp -> lane columns (lane c < D3 owns column c)
  auto load_M = [&](double (&a)[D3]) {
#pragma unroll
    for (int i = 0; i < D3; ++i) {
      const int r = i > lane ? i : lane, c = i > lane ? lane : i;
      a[i] = lane < D3 ? Mp[sym_idx(r, c, D3)] : 0.0;
    }
  };
  // M^-1 of element Kx (lane columns) -> SQ (stride LQ), its packed lower part
  // -> recovery cache (k = 3: one TMA bulk store staged in VT, retired before
  // VT is rewritten), pivot statistics
  auto store_Mi = [&](const double (&a)[D3], long Kx, double pmin, double pmax) {
    if (lane < D3) {
#pragma unroll
      for (int i = 0; i < D3; ++i) {
        if (Dm::MIQ) MQ[i * D3 + lane] = a[i];
        else SQ[i * LQ + lane] = a[i];
      }
    }
    if (factors) {
      double* dst = (Dm::BULK_MI ? VT : factors + Kx * Dm::FACTORS) + lane * (2 * D3 - lane + 1) / 2 - lane;
      if (lane < D3) {
#pragma unroll
        for (int i = 0; i < D3; ++i)
          if (i >= lane) dst[i] = a[i];
      }
      if (Dm::BULK_MI) {
        __syncwarp();
        if (lane == 0) bulk_store(factors + Kx * Dm::FACTORS, VT, NSYM * 8);
      }
    }
    if (lane == 0) store_pivstat(pivstat, Kx, 0, pmin, pmax);
    __syncwarp();
  };
  // one M^-1: the packed M of element Kx must be in Mp
  auto invert_M = [&](long Kx) {
    double a[D3], pmin = 1e300, pmax = 0.0;
    cp_async_wait_all();
    __syncwarp();
    load_M(a);
    __syncwarp();
    gj_sweep_inverse<D3>(a, ST, lane, pmin, pmax);
    store_Mi(a, Kx, pmin, pmax);
  };

  const long wstride = long(gridDim.x) * NW;
  long K = long(blockIdx.x) * NW + warp;
  int cur = 0;
  if (K < nelt) {  // the first element's M^-1; later ones follow the previous element's C phase
    prefetch_M(K, 0);   //  (PAIR: beside its S^-1)
    prefetch_D(K);
    invert_M(K);
  }

#ifdef HDG_C6_CLK  // diagnostics build: per-phase clocks of each element into Cf[K][0..5]
  long long clk[6];
#define C6_CLK(i) clk[i] = clock64()
#else
#define C6_CLK(i)
#endif
  for (; K < nelt; K += wstride, cur ^= 1) {
    C6_CLK(0);
    const long Kn = K + wstride;
    const bool has_next = Kn < nelt;
    if (Dm::PAIR) {
      cp_async_wait_all();  // this element's D (its M, f, geometry arrived long ago)
      __syncwarp();
      if (has_next) prefetch_M(Kn, cur ^ 1);  // Mp is free: this element's M^-1 is in MQ
    }
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
    double mib[KS][NT3];
    if (!Dm::MIQ) c6_symfrag<K_>(SQ, g, t, mib);
    if (Dm::BULK_MI && factors && lane == 0) bulk_store_wait_read();  // the packed M^-1 staged in VT is read out
    __syncwarp();

    C6_CLK(1);
    // ---- per d3 row tile i: Y_h, R'_h, S row tiles, V^T column tile
    double gm[3][3];
#pragma unroll
    for (int h = 0; h < 3; ++h)
#pragma unroll
      for (int h2 = 0; h2 < 3; ++h2) gm[h][h2] = DG[Dm::DG_G + 3 * h + h2];
    const double vol = DG[Dm::DG_VOL];
#pragma unroll
    for (int i = 0; i < NT3; ++i) {
      if (!c6_tile_nz(KSP, i)) {
        // Chat_h vanishes on these rows for every h: Y_h = R'_h = 0 there, so S
        // keeps D on the tile's rows and V^T[c][r] = T_l(c) W_l(c)[c'][r] on its columns
        const int r = 8 * i + g;
#pragma unroll
        for (int j = 0; j < NT3; ++j) {
          if (j > i) break;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * j + 2 * t + e;
            if (r < D3 && c <= r) {
              const double v = (r >= nu || c >= nu) ? (r == c ? 6.0 * vol : 0.0) : Dp[sym_idx(r, c, D3)];
              SQ[r * LS + c] = v;
              SQ[c * LS + r] = v;
            }
          }
        }
        const int r0 = 8 * i + 2 * t;
        if (r0 < LT) {
#pragma unroll
          for (int jc = 0; jc < NTM; ++jc) {
            const int c = 8 * jc + g, fc = c / D2;
            const double* wr = WT + int(DG[Dm::DG_TB + fc]) + (c - fc * D2) * LT;
            const double Tf = DG[Dm::DG_T + fc];
            const double2 w2 = *reinterpret_cast<const double2*>(wr + r0);
            const double v0 = r0 < nu ? Tf * w2.x : 0.0, v1 = r0 + 1 < nu ? Tf * w2.y : 0.0;
            *reinterpret_cast<double2*>(VT + c * LT + r0) = make_double2(v0, v1);
          }
        }
        continue;
      }
      if (Dm::MIQ) c6_symfrag<K_, D3>(MQ + (Dm::PAIR ? cur * Dm::MQS : 0), g, t, mib);
      double y[3][NT3][2];
      double ca[3][KS];
#pragma unroll
      for (int h = 0; h < 3; ++h) c6_rowfrag<K_>(CH + h * Dm::CH_SZ + (8 * i + g) * LT, t, ca[h]);
#pragma unroll
      for (int h = 0; h < 3; ++h)
#pragma unroll
        for (int n = 0; n < NT3; ++n) y[h][n][0] = y[h][n][1] = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s)
#pragma unroll
        for (int h = 0; h < 3; ++h)
#pragma unroll
          for (int n = 0; n < NT3; ++n)
            if (c6_ch_nz(KSP, h, i, s)) dmma(y[h][n][0], y[h][n][1], ca[h][s], mib[s][n]);
      // S row tiles j <= i: S = D + sum_h R'_h Chat_h^T
      {
        double ra[3][KS];
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          double rp[NT3][2];
#pragma unroll
          for (int n = 0; n < NT3; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              rp[n][e] = gm[0][h] * y[0][n][e] + gm[1][h] * y[1][n][e] + gm[2][h] * y[2][n][e];
          c6_chain<K_>(rp, lane, ra[h]);
        }
#pragma unroll
        for (int j = 0; j < NT3; ++j) {
          if (j > i) break;
          double sa[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            double cb[KS];
            if (j == i) {
#pragma unroll
              for (int s = 0; s < KS; ++s) cb[s] = ca[h][s];
            } else {
              c6_rowfrag<K_>(CH + h * Dm::CH_SZ + (8 * j + g) * LT, t, cb);
            }
#pragma unroll
            for (int s = 0; s < KS; ++s)
              if (c6_ch_nz(KSP, h, j, s)) dmma(sa[s & 1][0], sa[s & 1][1], ra[h][s], cb[s]);
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
        double yb[3][KS];
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          double yy[NT3][2];
#pragma unroll
          for (int n = 0; n < NT3; ++n) yy[n][0] = y[h][n][0], yy[n][1] = y[h][n][1];
          c6_chain<K_>(yy, lane, yb[h]);
        }
        double zf[4][KS];
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const double b0 = DG[Dm::DG_B + 3 * f], b1 = DG[Dm::DG_B + 3 * f + 1], b2 = DG[Dm::DG_B + 3 * f + 2];
          const double Tf = DG[Dm::DG_T + f];
#pragma unroll
          for (int s = 0; s < KS; ++s) {
            double z = b0 * yb[0][s] + b1 * yb[1][s] + b2 * yb[2][s];
            if (c6_kidx<K_>(s, t) == 8 * i + g) z += Tf;
            zf[f][s] = z;
          }
        }
#pragma unroll
        for (int jc = 0; jc < NTM; ++jc) {
          const int c = 8 * jc + g, fc = c / D2;
          const double* wr = WT + int(DG[Dm::DG_TB + fc]) + (c - fc * D2) * LT;
          double va[2] = {0.0, 0.0};
          const int f0 = (8 * jc) / D2, f1 = (8 * jc + 7) / D2;  // faces the tile's rows span
#pragma unroll
          for (int f = f0; f <= f1; ++f) {
            // rows of another face read a zero row (masking by address, not by selects)
            double wa[KS];
            c6_rowfrag<K_>(f0 == f1 || fc == f ? wr : ZR, t, wa);
#pragma unroll
            for (int s = 0; s < KS; ++s) dmma(va[0], va[1], wa[s], zf[f][s]);
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
    C6_CLK(2);
    if (has_next) {
      if (!Dm::PAIR) prefetch_M(Kn, cur ^ 1);
      prefetch_D(Kn);  // the packed M, D of this element are dead
    }

    // ---- S^-1: sweep (S stored row-major with stride LS), then stored with stride LQ
    double sib[KS][NT3];
    {
      double a[D3];
      double pmin = 1e300, pmax = 0.0;
      if constexpr (Dm::PAIR) {
        // lanes 0-15: S of this element; lanes 16-31: M of the next one
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // the next M (its D may stay in flight)
        __syncwarp();
        const int h = lane >> 4, c = lane & 15;
#pragma unroll
        for (int i = 0; i < D3; ++i) {
          double v = 0.0;
          if (c < D3) {
            if (h == 0) v = SQ[i * LS + c];
            else if (has_next) v = Mp[i > c ? sym_idx(i, c, D3) : sym_idx(c, i, D3)];
            else v = i == c ? 1.0 : 0.0;
          }
          a[i] = v;
        }
        __syncwarp();
        gj_sweep_seg<D3, 16, D3>(a, ST + h * 128, c, pmin, pmax);
        if (c < D3) {
          if (h == 0) {
#pragma unroll
            for (int i = 0; i < D3; ++i) SQ[i * LQ + c] = a[i];
          } else if (has_next) {
#pragma unroll
            for (int i = 0; i < D3; ++i) MQ[(cur ^ 1) * Dm::MQS + i * D3 + c] = a[i];  // the other M^-1 slot
            if (factors) {
              double* dst = factors + Kn * Dm::FACTORS + c * (2 * D3 - c + 1) / 2 - c;
#pragma unroll
              for (int i = 0; i < D3; ++i)
                if (i >= c) dst[i] = a[i];
            }
          }
        }
        if (lane == 0) store_pivstat(pivstat, K, 1, pmin, pmax);
        if (lane == 16 && has_next) store_pivstat(pivstat, Kn, 0, pmin, pmax);
      } else {
#pragma unroll
        for (int i = 0; i < D3; ++i) a[i] = lane < D3 ? SQ[i * LS + lane] : 0.0;
        __syncwarp();
        gj_sweep_inverse<D3>(a, ST, lane, pmin, pmax);
        if (lane < D3) {
#pragma unroll
          for (int i = 0; i < D3; ++i) SQ[i * LQ + lane] = a[i];
        }
        if (lane == 0) store_pivstat(pivstat, K, 1, pmin, pmax);
      }
      __syncwarp();
      c6_symfrag<K_>(SQ, g, t, sib);
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

    C6_CLK(3);
    // ---- C, Cf and the Vs record, by m row tiles jc
    // W rows of this lane in every m row tile (V^T and W fragments are
    // reloaded per C tile: fewer live registers, measured faster than keeping them)
    const double* wrow[NTM];
#pragma unroll
    for (int j = 0; j < NTM; ++j) {
      const int c = 8 * j + g, fc = c / D2;
      wrow[j] = WT + int(DG[Dm::DG_TB + fc]) + (c - fc * D2) * LT;
    }
    double fr[NT3][2];  // f at this lane's Vs rows 8n + 2t, + 1
#pragma unroll
    for (int n = 0; n < NT3; ++n)
#pragma unroll
      for (int e = 0; e < 2; ++e) fr[n][e] = 8 * n + 2 * t + e < D3 ? fg[8 * n + 2 * t + e] : 0.0;
    double* Ck = Cout + K * M * M;
    if (Dm::MIQ) c6_symfrag<K_, D3>(MQ + (Dm::PAIR ? cur * Dm::MQS : 0), g, t, mib);
#pragma unroll
    for (int jc = 0; jc < NTM; ++jc) {
      double vfr[KS], wfr[KS];
      c6_rowfrag<K_>(VT + (8 * jc + g) * LT, t, vfr);
      c6_rowfrag<K_>(wrow[jc], t, wfr);
      double vs[NT3][2], zp[NT3][2];
#pragma unroll
      for (int n = 0; n < NT3; ++n) vs[n][0] = vs[n][1] = zp[n][0] = zp[n][1] = 0.0;
#pragma unroll
      for (int s = 0; s < KS; ++s)
#pragma unroll
        for (int n = 0; n < NT3; ++n) {
          dmma(vs[n][0], vs[n][1], vfr[s], sib[s][n]);
          dmma(zp[n][0], zp[n][1], wfr[s], mib[s][n]);
        }
      const int r = 8 * jc + g;  // row of C / column of Vs
      {
        double p = 0.0;
        double* rec = factors + K * Dm::FACTORS + NSYM + r * D3;
#pragma unroll
        for (int n = 0; n < NT3; ++n) {
          const int rr = 8 * n + 2 * t;  // d3 is even: a pair never straddles it
          if (factors && rr < D3) {
            if ((NSYM + D3) % 2 == 0) {  // 16-byte aligned pairs
              *reinterpret_cast<double2*>(rec + rr) = make_double2(vs[n][0], vs[n][1]);
            } else {
              rec[rr] = vs[n][0];
              rec[rr + 1] = vs[n][1];
            }
          }
          p += vs[n][0] * fr[n][0] + vs[n][1] * fr[n][1];
        }
        p += __shfl_xor_sync(FULL, p, 1);
        p += __shfl_xor_sync(FULL, p, 2);
        if (t == 0) Cfout[K * M + r] = p;
      }
      double vsa[KS], zpa[KS];
      c6_chain<K_>(vs, lane, vsa);
      c6_chain<K_>(zp, lane, zpa);
      const int l1 = r / D2;
#pragma unroll
      for (int j = 0; j <= jc; ++j) {
        double c1[2] = {0.0, 0.0}, c2[2] = {0.0, 0.0};
        double wb[KS], vb[KS];
        if (j < jc) {
          c6_rowfrag<K_>(wrow[j], t, wb);
          c6_rowfrag<K_>(VT + (8 * j + g) * LT, t, vb);
        } else {
#pragma unroll
          for (int s = 0; s < KS; ++s) wb[s] = wfr[s], vb[s] = vfr[s];
        }
#pragma unroll
        for (int s = 0; s < KS; ++s) {
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
    // M^-1 of the next element (measured: interleaving its pivot steps with
    // this element's C tiles is slower, the sweep's DFMAs share the DMMA pipe)
    C6_CLK(4);
    if (!Dm::PAIR && has_next) invert_M(Kn);
#ifdef HDG_C6_CLK
    C6_CLK(5);
    __syncwarp();
    if (lane < 5) Cfout[K * M + lane] = double(clk[lane + 1] - clk[lane]);
#endif
  }
}

}  // namespace hdgb
