// K3 v3 (k = 2, 3): CTA-batched static condensation.
//
// Same algebra as kernels_condense2.cuh (explicit M^-1, S^-1 by warp-register
// sweep Gauss-Jordan; every contraction a DMMA tile loop over shared memory),
// but the CTA advances EPB elements phase by phase: every phase pools the
// tasks of all EPB elements over all warps (better balance, 5 CTA barriers
// per EPB elements instead of 5 team barriers per element), and in P3 the
// S^-1 sweeps of the batch run concurrently with the M^-1 sweeps of the next
// batch.
//
// Compact layout: every d3-indexed dimension is stored with stride
// LD = round_up(d3, 4) (20 at k=3, 12 at k=2), so the contraction loops run
// exactly KS = LD/4 DMMA k-steps with no predicates. The k-padding rows /
// columns (k=2 only) are kept zero; tile rows/columns past d3 read whatever
// follows in shared memory and their outputs are never stored.
#pragma once

#include "kernels_condense2.cuh"

namespace hdgb {

#ifdef HDG_PHASE_TIMING
// Diagnostics build only: clock64() at each CTA barrier of the first batches.
__device__ long long g_phase_clk[148][8][8];
#define PHASE_MARK(b, p) \
  if (threadIdx.x == 0 && blockIdx.x < 148 && (b) < 8) g_phase_clk[blockIdx.x][(b)][(p)] = clock64();
#else
#define PHASE_MARK(b, p)
#endif


template <int K_>
struct C3Dims {
  static constexpr int D3 = cdim3(K_), D2 = cdim2(K_), M = 4 * cdim2(K_);
  static constexpr int LD = round_up(D3, 4);        // stride of every d3-indexed dimension
  static constexpr int KS = LD / 4;                 // DMMA k-steps over d3
  static constexpr int D3P = round_up(D3, 8), MP = round_up(M, 8);
  static constexpr int MT = D3P / 8, NTM = MP / 8;  // row tiles over d3, column tiles over m
  static constexpr int NSYM = D3 * (D3 + 1) / 2;
  static constexpr int SQ = round_up(LD * LD + D3P - LD, 2);  // d3 x d3 + tile-row overrun
  static constexpr int RH = LD * D3;                          // one R_# (LD x d3)
  static constexpr int NY = 3 * RH > LD * MP ? 3 * RH : LD * MP;
  static constexpr int OFF_MI = 0;
  static constexpr int OFF_S = OFF_MI + SQ;
  static constexpr int OFF_Y = OFF_S + SQ;       // R_# (3), then Vs (LD x MP)
  static constexpr int OFF_Z = OFF_Y + NY;       // Zp (LD x MP)
  static constexpr int OFF_V = OFF_Z + LD * MP;  // V (LD x MP)
  static constexpr int OFF_NSC = OFF_V + LD * MP;  // column data (8 x MP), see build_columns
  static constexpr int OFF_F = OFF_NSC + 8 * MP;   // LD: f
  static constexpr int OFF_FS = OFF_F + LD;        // LD: Si f
  static constexpr int OFF_STG = round_up(OFF_FS + LD, 2);  // 128: GJ column stage (16 B aligned)
  static constexpr int OFF_STG2 = OFF_STG + 128;            // 128: second GJ stage
  // 2 x 64: element records (cur/next): [0,30) geometry, [32,41) metric
  // G(h,h') = sum_s a(s,h) a(s,h'), [48,64) face normal products n_l1 . n_l2
  static constexpr int OFF_GEO = OFF_STG2 + 128;
  static constexpr int OFF_COL = OFF_GEO + 128;             // second column-data buffer
  static constexpr int OFF_DP = OFF_COL + 8 * MP;           // packed D
  static constexpr int PER_ELT = OFF_DP + round_up(NSYM, 2);
  static constexpr int FACTORS = round_up(NSYM + D3 * M + D3, 2);  // {M^-1 packed, Vs, fs}, 16-B records
  // per CTA: Chat_# [c + k d3] (k < LD, padding zero), tauDD, tile overrun
  static constexpr int CTA_EXTRA = round_up(3 * D3 * LD + D2 * D2 + D3P, 2);
};

// Most 8-column tiles one face's d2 columns (starting at l d2) touch.
constexpr int face_tiles(int d2) {
  int n = 0;
  for (int l = 0; l < 4; ++l) {
    const int t = (l * d2 + d2 - 1) / 8 - (l * d2) / 8 + 1;
    n = t > n ? t : n;
  }
  return n;
}

template <int K_> struct C3Cfg;
#ifndef HDG_C3_EPB2
#define HDG_C3_EPB2 6
#define HDG_C3_NWT2 8
#define HDG_C3_MINB2 2
#endif
#ifndef HDG_C3_EPB3
#define HDG_C3_EPB3 5
#define HDG_C3_NWT3 16
#define HDG_C3_MINB3 1
#endif
template <> struct C3Cfg<2> { static constexpr int EPB = HDG_C3_EPB2, NWT = HDG_C3_NWT2, MINB = HDG_C3_MINB2; };
template <> struct C3Cfg<3> { static constexpr int EPB = HDG_C3_EPB3, NWT = HDG_C3_NWT3, MINB = HDG_C3_MINB3; };

template <int K_>
__global__ void __launch_bounds__(C3Cfg<K_>::NWT * 32, C3Cfg<K_>::MINB)
condense3_kernel(DevTab tab, int nelt, GeoDev geo, const double* __restrict__ Msym,
                 const double* __restrict__ Dsym, const double* __restrict__ fvec,
                 double* __restrict__ Cout, double* __restrict__ Cfout, double* __restrict__ factors,
                 double* __restrict__ pivstat) {
  using Dm = C3Dims<K_>;
  constexpr int EPB = C3Cfg<K_>::EPB, NWT = C3Cfg<K_>::NWT, NT = NWT * 32;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, MP = Dm::MP, LD = Dm::LD, RH = Dm::RH;
  constexpr int MT = Dm::MT, NTM = Dm::NTM, KS = Dm::KS;
  constexpr int NLP = (NTM / 2 + 1) * ((NTM + 1) / 2);  // lower tile pairs of the m x m output
  constexpr int NLS = MT * (MT + 1) / 2;     // lower tiles of S
  constexpr int NTF = face_tiles(D2);        // N-tiles one face's columns span
  static_assert(M % 8 == 0, "P5 pairs columns c0, c0 + 1 < M");
#ifndef HDG_C3_FPT
#define HDG_C3_FPT 4
#endif
  constexpr int FPT = HDG_C3_FPT;            // faces per V task (1, 2 or 4)
#ifndef HDG_C3_PAIR
#define HDG_C3_PAIR 1
#endif
  // d3 <= 16 (k = 2): one warp sweeps two matrices, S of element e and M of
  // the next batch's element e, one per 16-lane half (gj_sweep_seg)
  constexpr bool PAIR = HDG_C3_PAIR && D3 % 2 == 0 && D3 <= 16;
  constexpr int NGJ = PAIR ? EPB : 2 * EPB;  // GJ tasks in P3
  constexpr bool GJ_SEP = NWT > NGJ;         // GJ warps do nothing else in P3
#ifndef HDG_C3_NO_BULK
  // record layout == shared layout (k = 3), packed factors a 16-byte multiple
  const bool BULK_VF = LD == D3 && (Dm::NSYM * 8) % 16 == 0 && tab.nu == D3 && GJ_SEP;
#else
  const bool BULK_VF = false;
#endif
#ifndef HDG_C3_VS_DIRECT
#define HDG_C3_VS_DIRECT 1
#endif
  // Vs, fs go to the recovery cache from P4's registers (1) or by TMA bulk
  // stores from shared memory under P5 (0: measured slower, P5 is
  // shared-memory bound)
  constexpr bool VS_DIRECT = HDG_C3_VS_DIRECT;
  extern __shared__ double smem[];
  // The sweep inverses' two triangles round differently (each lane computes one
  // column), and the Schur-complement products amplify that asymmetry (C at
  // kappa = 1e4 off by 1e-4): every consumer reads one canonical value per
  // symmetric pair, the one the lower-index lane computed (its column below the
  // diagonal: the upper half of a sweep column is measurably less accurate),
  // stored row-wise by that lane at (min, max) = min + max * LD.
  auto sym_at = [](int r, int k) { return r <= k ? r + k * LD : k + r * LD; };
  for (int i = threadIdx.x; i < EPB * Dm::PER_ELT + Dm::CTA_EXTRA; i += blockDim.x) smem[i] = 0.0;
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const double* Wlm = tab.Wlm;
  // CTA copy of Chat_# and tauDD: their fragments are re-read every phase
  double* Ch = smem + EPB * Dm::PER_ELT;
  double* DDs = Ch + 3 * D3 * LD;
  for (int i = threadIdx.x; i < 3 * D3 * D3; i += NT) {
    const int h = i / (D3 * D3);
    Ch[h * D3 * LD + (i - h * D3 * D3)] = tab.Chat[i];
  }
  for (int i = threadIdx.x; i < D2 * D2; i += NT) DDs[i] = tab.DD[i];
  __syncthreads();
  auto B = [&](int e) { return smem + e * Dm::PER_ELT; };
  auto Mi = [&](int e) { return B(e) + Dm::OFF_MI; };
  auto Sb = [&](int e) { return B(e) + Dm::OFF_S; };
  auto Yb = [&](int e) { return B(e) + Dm::OFF_Y; };            // R_#, then Vs
  auto Zb = [&](int e) { return B(e) + Dm::OFF_Z; };            // Zp
  auto Vb = [&](int e) { return B(e) + Dm::OFF_V; };
  auto fv = [&](int e) { return B(e) + Dm::OFF_F; };
  auto fs = [&](int e) { return B(e) + Dm::OFF_FS; };
  auto Dp = [&](int e) { return B(e) + Dm::OFF_DP; };  // packed D
  auto stS = [&](int e) { return B(e) + Dm::OFF_STG; };
  auto stM = [&](int e) { return B(e) + Dm::OFF_STG2; };
  auto colb = [&](int e, int b) { return B(e) + (b ? Dm::OFF_COL : Dm::OFF_NSC); };
  auto sgb = [&](int e, int b) { return B(e) + Dm::OFF_GEO + 64 * b; };
  // per-element tables derived from the geometry record (warp-wide)
  auto build_tables = [&](double* sg) {
    if (lane < 9) {
      const int h = lane / 3, h2 = lane % 3;
      sg[32 + lane] = sg[1 + h] * sg[1 + h2] + sg[4 + h] * sg[4 + h2] + sg[7 + h] * sg[7 + h2];
    } else if (lane >= 16) {
      const int l1 = (lane - 16) >> 2, l2 = lane & 3;
      sg[48 + (lane - 16)] = sg[10 + 3 * l1] * sg[10 + 3 * l2] + sg[11 + 3 * l1] * sg[11 + 3 * l2] +
                             sg[12 + 3 * l1] * sg[12 + 3 * l2];
    }
  };
  // packed lower column `lane` of a symmetric inverse held in registers -> recovery cache.
  // With a shared-memory staging area (k = 3: the packed record is a 16-byte
  // multiple) the packed matrix is assembled there and written by one TMA bulk
  // store, which the caller's lane 0 must retire (bulk_store_wait_read) before
  // the staging area is reused; otherwise straight from the registers.
  auto store_factor = [&](const double (&a)[D3], long K, int off, double* stage) {
    if (!factors) return;
    if (BULK_VF && stage) {
      if (lane < D3) {
        double* dst = stage + lane * (2 * D3 - lane + 1) / 2 - lane;
#pragma unroll
        for (int i = 0; i < D3; ++i)
          if (i >= lane) dst[i] = a[i];
      }
      __syncwarp();
      if (lane == 0) bulk_store(factors + K * Dm::FACTORS + off, stage, Dm::NSYM * 8);
    } else if (lane < D3) {
      double* dst = factors + K * Dm::FACTORS + off + lane * (2 * D3 - lane + 1) / 2 - lane;
#pragma unroll
      for (int i = 0; i < D3; ++i)
        if (i >= lane) dst[i] = a[i];
    }
  };

  const long stride = long(gridDim.x) * EPB;
  long K0 = long(blockIdx.x) * EPB;
  int cur = 0;
  int batch = 0;

  auto load_Df_async = [&](long Kb) {  // packed D and f of batch Kb -> smem (cp.async group)
    for (int idx = threadIdx.x; idx < EPB * Dm::NSYM; idx += NT) {
      const int e = idx / Dm::NSYM, p = idx - e * Dm::NSYM;
      if (Kb + e < nelt) cp_async8(Dp(e) + p, Dsym + (Kb + e) * Dm::NSYM + p);
    }
    for (int idx = threadIdx.x; idx < EPB * D3; idx += NT) {
      const int e = idx / D3, i = idx - e * D3;
      if (Kb + e < nelt) cp_async8(fv(e) + i, fvec + (Kb + e) * D3 + i);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto load_geometry = [&](long Kb, int which, int tid, int nthr) {
    for (int idx = tid; idx < EPB * 32; idx += nthr) {
      const int e = idx >> 5, i = idx & 31;
      if (Kb + e < nelt && i < 30) {
        const long K = Kb + e;
        double v;
        if (i == 0) v = geo.volume[K];
        else if (i < 10) v = geo.piola[long(i - 1) * nelt + K];
        else if (i < 22) v = geo.normals[long(i - 10) * nelt + K];
        else if (i < 26) v = geo.T[long(i - 22) * nelt + K];
        else v = double(geo.perm[long(i - 26) * nelt + K]);
        sgb(e, which)[i] = v;
      }
    }
  };
  // M^-1 of element K (packed M at P, global or the staging copy in Mi(e)):
  // warp-register sweep, full LD-strided result into Mi(e), packed lower part
  // straight from the registers into the recovery cache (warp-wide)
  auto invert_M = [&](int e, long K, const double* P) {
    double a[D3];
#pragma unroll
    for (int i = 0; i < D3; ++i) {
      const int r = i > lane ? i : lane, c = i > lane ? lane : i;
      a[i] = lane < D3 ? P[sym_idx(r, c, D3)] : 0.0;
    }
    __syncwarp();
    double pmin = 1e300, pmax = 0.0;
    gj_sweep_inverse<D3>(a, stM(e), lane, pmin, pmax);
    if (lane < D3) {  // row-wise (conflict-free); consumers read the canonical entries (sym_at)
#pragma unroll
      for (int i = 0; i < D3; ++i) Mi(e)[lane + i * LD] = a[i];
    }
    store_factor(a, K, 0, Yb(e));  // R_# of this slot is dead until the next P1
    if (lane == 0) store_pivstat(pivstat, K, 0, pmin, pmax);
  };

  // ---- prologue: first batch
  if (K0 < nelt) {
    load_Df_async(K0);
    load_geometry(K0, 0, threadIdx.x, NT);
    for (int e = warp; e < EPB; e += NWT)
      if (K0 + e < nelt) invert_M(e, K0 + e, Msym + (K0 + e) * Dm::NSYM);
    if (BULK_VF && lane == 0) bulk_store_wait_read();  // staged M^-1 read before P1 reuses Yb
    cp_async_wait_all();
    __syncthreads();
    for (int e = warp; e < EPB; e += NWT) {
      build_columns<D2, D3, M, MP>(sgb(e, 0), colb(e, 0), lane);
      build_tables(sgb(e, 0));
    }
    __syncthreads();
  }

  for (; K0 < nelt; K0 += stride, ++batch) {
    PHASE_MARK(batch, 0);
    const long Kn0 = K0 + stride;
    const bool has_next = Kn0 < nelt;
    const int nb = int(nelt - K0 < EPB ? nelt - K0 : EPB);  // live elements in this batch

    // -------- P1: Zp = Mi W^T (strips) ; R_# = sum_#' g(#,#') Mi Chat_#'^T (tiles)
    for (int task = warp; task < nb * (MT * MT + NTM); task += NWT) {
      const int e = task / (MT * MT + NTM), sub = task % (MT * MT + NTM);
      const double* sg = sgb(e, cur);
      const double* mi = Mi(e);
      if (sub < MT * MT) {
        const int m = sub / MT, nt = sub % MT;
        const int c = nt * 8 + g;
        double q[3][2] = {{0, 0}, {0, 0}, {0, 0}};
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const int o = c + k * D3;
          const double a = mi[sym_at(m * 8 + g, k)];
          dmma(q[0][0], q[0][1], a, Ch[o]);
          dmma(q[1][0], q[1][1], a, Ch[D3 * LD + o]);
          dmma(q[2][0], q[2][1], a, Ch[2 * D3 * LD + o]);
        }
        const int c0 = nt * 8 + 2 * t, r = m * 8 + g;
        if (r < LD) {
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            const double g0 = sg[32 + 3 * h], g1 = sg[33 + 3 * h], g2 = sg[34 + 3 * h];
            double* R = Yb(e) + h * RH;
            if (c0 < D3) R[r + c0 * LD] = r < D3 ? g0 * q[0][0] + g1 * q[1][0] + g2 * q[2][0] : 0.0;
            if (c0 + 1 < D3) R[r + (c0 + 1) * LD] = r < D3 ? g0 * q[0][1] + g1 * q[1][1] + g2 * q[2][1] : 0.0;
          }
        }
      } else {
        const int nt = sub - MT * MT;
        const double* col = colb(e, cur);
        const int* wb = reinterpret_cast<const int*>(col + 4 * MP);
        const int cz = nt * 8 + g, wbc = wb[cz];
        const double tc = col[3 * MP + cz];
        double* Vi = Vb(e) + cz * LD;  // V starts as T_l W_l^T (the W fragment is at hand)
        double acc[MT][2];
#pragma unroll
        for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const double b = (wbc >= 0 && k < D3) ? __ldg(Wlm + wbc + k * D2) : 0.0;
          Vi[k] = tc * b;
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(acc[m][0], acc[m][1], mi[sym_at(m * 8 + g, k)], b);
        }
        const int c0 = nt * 8 + 2 * t;
        double* Z = Zb(e);
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const int r = m * 8 + g;
          if (r < LD) {
            Z[r + c0 * LD] = r < D3 ? acc[m][0] : 0.0;
            Z[r + (c0 + 1) * LD] = r < D3 ? acc[m][1] : 0.0;
          }
        }
      }
    }
    cp_async_wait_all();  // D, f of this batch (issued during the previous P5)
    __syncthreads();

    PHASE_MARK(batch, 1);
    // next batch's packed M -> Mi(e) (dead after P1), asynchronously under P2
    if (has_next) {
      for (int idx = threadIdx.x; idx < EPB * Dm::NSYM; idx += NT) {
        const int e = idx / Dm::NSYM, p = idx - e * Dm::NSYM;
        if (Kn0 + e < nelt) cp_async8(Mi(e) + p, Msym + (Kn0 + e) * Dm::NSYM + p);
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    // ---- P2: S += sum_# Chat_# R_# (lower tiles) | V_l = Chat_l Zp_l + T_l W_l^T
    constexpr int NP2 = NLS + (4 / FPT) * MT;  // P2 tasks per element
    for (int task = warp; task < nb * NP2; task += NWT) {
      const int e = task / NP2, sub = task % NP2;
      if (sub < NLS) {
        int mt = 0, rem = sub;
        while (rem > mt) { rem -= mt + 1; ++mt; }
        const int j = rem, r = mt * 8 + g;
        double p0 = 0, p1 = 0, q0 = 0, q1 = 0;
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          const double* R = Yb(e) + h * RH;
          const double* C = Ch + h * D3 * LD;
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) {
            const int k = kk * 4 + t;
            const double a = C[r + k * D3];
            if (kk & 1) dmma(q0, q1, a, R[k + (j * 8 + g) * LD]);
            else dmma(p0, p1, a, R[k + (j * 8 + g) * LD]);
          }
        }
        double* S = Sb(e);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = j * 8 + 2 * t + h;
          if (r < D3 && c <= r) {  // BDM (tab.nu < D3): decoupled diagonal outside the P_{k-1} block
            const double v = (r >= tab.nu || c >= tab.nu) ? (r == c ? 6.0 * sgb(e, cur)[0] : 0.0)
                                                          : Dp(e)[sym_idx(r, c, D3)] + (h ? p1 + q1 : p0 + q0);
            S[r + c * LD] = v;
            S[c + r * LD] = v;
          }
        }
      } else {  // V rows of row tile mt for FPT faces: the Chat_# fragments feed every face
        const int mt = (sub - NLS) / (4 / FPT), l0 = ((sub - NLS) % (4 / FPT)) * FPT;
        const int r = mt * 8 + g;
        const double* beta = colb(e, cur) + 5 * MP;
        const double* Z = Zb(e);
        double bl[FPT][3];
        double acc[FPT][NTF][2] = {};
#pragma unroll
        for (int f = 0; f < FPT; ++f)
#pragma unroll
          for (int h = 0; h < 3; ++h) bl[f][h] = beta[h * MP + (l0 + f) * D2];
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const int o = r + k * D3;
          const double c0 = Ch[o], c1 = Ch[D3 * LD + o], c2 = Ch[2 * D3 * LD + o];
#pragma unroll
          for (int f = 0; f < FPT; ++f) {
            const int cl0 = (l0 + f) * D2, cl1 = cl0 + D2, nt0 = cl0 / 8;
            const double a = bl[f][0] * c0 + bl[f][1] * c1 + bl[f][2] * c2;
#pragma unroll
            for (int j = 0; j < NTF; ++j) {
              const int c = (nt0 + j) * 8 + g;
              const double b = (c >= cl0 && c < cl1) ? Z[k + c * LD] : 0.0;
              if ((nt0 + j) * 8 < cl1) dmma(acc[f][j][0], acc[f][j][1], a, b);
            }
          }
        }
        double* V = Vb(e);
        if (r < LD) {
#pragma unroll
          for (int f = 0; f < FPT; ++f) {
            const int cl0 = (l0 + f) * D2, cl1 = cl0 + D2, nt0 = cl0 / 8;
#pragma unroll
            for (int j = 0; j < NTF; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int c = (nt0 + j) * 8 + 2 * t + h;
                if (c >= cl0 && c < cl1) V[r + c * LD] = r < tab.nu ? acc[f][j][h] + V[r + c * LD] : 0.0;
              }
          }
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();

    PHASE_MARK(batch, 2);
    // ---- P3: S^-1 of the batch || M^-1 of the next batch || V, f -> recovery
    //      cache, next geometry
    {
      const bool gj_warp = warp < NGJ;
      if (gj_warp || !GJ_SEP) {
        for (int task = warp; task < NGJ; task += (GJ_SEP ? NGJ : NWT)) {
          const int e = task % EPB;
          if constexpr (PAIR) {
            const int h = lane >> 4, c = lane & 15;
            const bool live = h == 0 ? e < nb : (has_next && Kn0 + e < nelt);
            const long K = h == 0 ? K0 + e : Kn0 + e;
            double* dst = h == 0 ? Sb(e) : Mi(e);  // S stored full (P2); packed M copied into Mi(e) in P2
            double a[D3];
#pragma unroll
            for (int i = 0; i < D3; ++i) {
              double v = i == c ? 1.0 : 0.0;  // dead half / padding lanes: identity
              if (live && c < D3) {
                const int r = i > c ? i : c, cc = i > c ? c : i;
                v = h == 0 ? dst[c + i * LD] : dst[sym_idx(r, cc, D3)];
              }
              a[i] = v;
            }
            __syncwarp();
            double pmin = 1e300, pmax = 0.0;
            gj_sweep_seg<D3, 16, D3>(a, h == 0 ? stS(e) : stM(e), c, pmin, pmax);
            if (live && c < D3) {
#pragma unroll
              for (int i = 0; i < D3; ++i)  // lower triangle mirrored: consistent for sym_at
                if (i >= c) {
                  dst[c + i * LD] = a[i];
                  dst[i + c * LD] = a[i];
                }
              if (factors && h == 1) {  // M^-1 of the next batch (S^-1 is not cached: Vs, fs are)
                double* fd = factors + K * Dm::FACTORS + c * (2 * D3 - c + 1) / 2 - c;
#pragma unroll
                for (int i = 0; i < D3; ++i)
                  if (i >= c) fd[i] = a[i];
              }
            }
            if (live && c == 0) store_pivstat(pivstat, K, h == 0 ? 1 : 0, pmin, pmax);
            continue;
          }
          if (task < EPB) {
            if (e >= nb) continue;
            const long K = K0 + e;
            double a[D3];  // S is stored full (P2), so column `lane` is read row-wise
#pragma unroll
            for (int i = 0; i < D3; ++i) a[i] = lane < D3 ? Sb(e)[lane + i * LD] : 0.0;
            double pmin = 1e300, pmax = 0.0;
#ifndef HDG_DIAG_NO_GJ
            gj_sweep_inverse<D3>(a, stS(e), lane, pmin, pmax);
#else
            pmin = pmax = 1.0;
#endif
            if (lane < D3) {  // row-wise; consumers read canonical (max, min) entries (sym_at)
#pragma unroll
              for (int i = 0; i < D3; ++i) Sb(e)[lane + i * LD] = a[i];
            }
            if (lane == 0) store_pivstat(pivstat, K, 1, pmin, pmax);
          } else if (has_next && Kn0 + e < nelt) {
#ifdef HDG_DIAG_NO_GJ
            continue;
#endif
            invert_M(e, Kn0 + e, Mi(e));  // packed M copied into the dead Mi(e) during P2
          }
        }
        // the staged factors (Dp, Yb) are read before P4 / P5 reuse them
        if (BULK_VF && lane == 0) bulk_store_wait_read();
      }
      if (!gj_warp || !GJ_SEP) {
        // No FP64 here: the sweeps' dependent DFMA chains stall badly behind
        // DMMA traffic on the same pipe, so this phase only moves data.
        const int w0 = GJ_SEP ? warp - NGJ : warp, nw = GJ_SEP ? NWT - NGJ : NWT;
        if (has_next) load_geometry(Kn0, cur ^ 1, w0 * 32 + lane, nw * 32);
      }
    }
    __syncthreads();

    PHASE_MARK(batch, 3);
    // ---- P4: Vs = Si V (into Yb) | fs = Si f | next batch's columns
    for (int task = warp; task < nb * NTM; task += NWT) {  // one column strip per task:
      const int e = task / NTM, nt = task % NTM;           // the V fragment feeds MT chains
      const double* S = Sb(e);
      const double* V = Vb(e);
      double acc[MT][2];
#pragma unroll
      for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
      const int c = nt * 8 + g;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int k = kk * 4 + t;
        const double b = V[k + c * LD];
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma(acc[m][0], acc[m][1], S[sym_at(m * 8 + g, k)], b);
      }
      const int c0 = nt * 8 + 2 * t;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int r = m * 8 + g;
        if (r < LD) {
          Yb(e)[r + c0 * LD] = r < D3 ? acc[m][0] : 0.0;  // Vs (R_# is dead)
          Yb(e)[r + (c0 + 1) * LD] = r < D3 ? acc[m][1] : 0.0;
        }
        if (VS_DIRECT && factors && r < D3) {  // recovery cache, straight from the registers
          double* rec = factors + (K0 + e) * Dm::FACTORS + Dm::NSYM;
          rec[r + c0 * D3] = acc[m][0];
          rec[r + (c0 + 1) * D3] = acc[m][1];
        }
      }
    }
    for (int idx = threadIdx.x; idx < nb * D3; idx += NT) {
      const int e = idx / D3, r = idx % D3;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D3; ++k) s += Sb(e)[sym_at(r, k)] * fv(e)[k];
      fs(e)[r] = s;
      if (VS_DIRECT && factors) factors[(K0 + e) * Dm::FACTORS + Dm::NSYM + D3 * M + r] = r < tab.nu ? s : 0.0;
    }
    __syncthreads();
    // recovery cache: Vs = S^-1 V and fs = S^-1 f after M^-1 (k = 3: already in the
    // record's layout in shared memory, one TMA bulk store each, retired before
    // the end of P5, when Vs's slot is rewritten by the next P1)
    if (VS_DIRECT) {
      // written from P4's registers
    } else if (factors && BULK_VF) {
      if (lane == 0)
        for (int e = warp; e < nb; e += NWT) {
          double* rec = factors + (K0 + e) * Dm::FACTORS + Dm::NSYM;
          bulk_store(rec, Yb(e), D3 * M * 8);
          bulk_store(rec + D3 * M, fs(e), D3 * 8);
        }
    } else if (factors) {
      constexpr int NVF = D3 * M + D3;
      for (int q = threadIdx.x; q < nb * NVF; q += NT) {
        const int e = q / NVF, rem = q - e * NVF, c = rem / D3, r = rem - c * D3;
        factors[(K0 + e) * Dm::FACTORS + Dm::NSYM + rem] =
            c < M ? Yb(e)[r + c * LD] : (r < tab.nu ? fs(e)[r] : 0.0);
      }
    }
    if (has_next)
      for (int e = warp; e < EPB; e += NWT)
        if (Kn0 + e < nelt) {
          build_columns<D2, D3, M, MP>(sgb(e, cur ^ 1), colb(e, cur ^ 1), lane);
          build_tables(sgb(e, cur ^ 1));
        }

    PHASE_MARK(batch, 4);
    if (has_next) load_Df_async(Kn0);  // D, f of this batch are dead after P4
    // ---- P5: C = tauDD + (n_l1.n_l2) o (W Zp) - V^T Vs (lower tiles, mirrored) | Cf
    for (int task = warp; task < nb * NLP; task += NWT) {  // tile pairs (mt, nt0..nt0+1) of a row
      const int e = task / NLP;
      const int tp = task % NLP;  // row mt holds (mt + 2) / 2 pairs; rows < mt hold (mt + 1)^2 / 4
      const int mt = int(2.0f * sqrtf(float(tp) + 0.25f)) - 1;
      const int nt0 = 2 * (tp - (mt + 1) * (mt + 1) / 4), r = mt * 8 + g;
      const bool two = nt0 + 1 <= mt;
      const double* V = Vb(e);
      const double* Vs = Yb(e);
      const double* Z = Zb(e);
      const int wbr = reinterpret_cast<const int*>(colb(e, cur) + 4 * MP)[r];
      double z[2][2] = {{0, 0}, {0, 0}}, v[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int k = kk * 4 + t;
        const double aw = (wbr >= 0 && k < D3) ? __ldg(Wlm + wbr + k * D2) : 0.0;
        const double av = V[k + r * LD];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
          const int cn = (nt0 + u) * 8 + g;
          dmma(z[u][0], z[u][1], aw, Z[k + cn * LD]);
          dmma(v[u][0], v[u][1], av, Vs[k + cn * LD]);
        }
      }
      if (r < M) {
        const int l1 = r / D2;
        const double* nn4 = sgb(e, cur) + 48 + 4 * l1;
        const double* Tc = colb(e, cur) + 3 * MP;
        double* Ck = Cout + (K0 + e) * M * M;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
          const int c0 = (nt0 + u) * 8 + 2 * t;  // c0 + 1 < M: M and the tiles are whole
          double val[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = c0 + h, l2 = c / D2;
            val[h] = nn4[l2] * z[u][h] - v[u][h];
            if (l1 == l2) val[h] += Tc[c] * DDs[(r - l1 * D2) + (c - l2 * D2) * D2];
          }
          // lower entries (c <= r); the mirrored upper ones as one 16-byte
          // store where both columns are strictly below the diagonal
          if (c0 <= r) Ck[r + c0 * M] = val[0];
          if (c0 + 1 <= r) Ck[r + (c0 + 1) * M] = val[1];
          if (c0 + 1 < r) *reinterpret_cast<double2*>(Ck + c0 + r * M) = make_double2(val[0], val[1]);
          else if (c0 < r) Ck[c0 + r * M] = val[0];
        }
      }
    }
    for (int idx = threadIdx.x; idx < nb * M; idx += NT) {
      const int e = idx / M, r = idx % M;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D3; ++k) s += Vb(e)[k + r * LD] * fs(e)[k];
      Cfout[(K0 + e) * M + r] = s;
    }
    if (!VS_DIRECT && factors && BULK_VF && lane == 0 && warp < nb) bulk_store_wait_read();  // Vs, fs read out
    __syncthreads();
    PHASE_MARK(batch, 5);
    cur ^= 1;
  }
}

}  // namespace hdgb
