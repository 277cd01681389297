// K3 v5 (k = 4, 5): static condensation with the v3 algebra (explicit M^-1
// and S^-1, every contraction a DMMA tile loop) for element matrices too
// large for several elements per CTA: d3 = 35 / 56, m = 60 / 84.
//
// One element per CTA iteration, all warps on it:
//   P1  M^-1: M expanded to a full LD-strided matrix, CTA-wide sweep inverse
//   P2  Zp = M^-1 W^T (strips; T_l W_l^T staged into V) | T0 = M^-1 Chat_0^T
//   P3  S = D + Chat'_0 T0 (lower tiles) | T1 = M^-1 Chat_1^T
//   P4  S += Chat'_1 T1 | T0 = M^-1 Chat_2^T
//   P5  S += Chat'_2 T0 | V_l = Chat_l Zp_l (+ T_l W_l^T)
//   P6  S^-1: CTA-wide sweep inverse (S stored full by P3..P5)
//   P7  Vs = S^-1 V (into the dead M^-1 | T0 space) | fs = S^-1 f
//   P8  C = tauDD + (n_l1.n_l2) o (W Zp) - V^T Vs (lower tile pairs) | Cf
// with Chat'_h = sum_# g(#,h) Chat_# (g = a^T a; the 3 loads + FMAs per
// k-step form the A fragment) and Chat_l = sum_# beta_#(l) Chat_#. The
// reference tables (Chat, W) are read through L1/L2 (they do not fit beside
// the element's 180-220 KB of operands). Only two 56 x 56 product buffers
// (T0, T1) exist: the three T_h alternate between them so each S update runs
// beside the next T product.
//
// CTA-wide sweep (cta_sweep_inverse): 2 x 2 pivots as the warp version, each
// thread owning a run of rows of one column, ping-ponging between the matrix
// and a free product buffer (one barrier per pivot pair).
#pragma once

#ifndef HDG_C5_SPARSE  // skip the structurally zero row tiles / ksteps of Chat_h
#define HDG_C5_SPARSE 1
#endif

#include "kernels_condense2.cuh"

namespace hdgb {
// Most 8-column tiles one face's d2 columns (starting at l d2) touch.
constexpr int face_tiles(int d2) {
  int n = 0;
  for (int l = 0; l < 4; ++l) {
    const int t = (l * d2 + d2 - 1) / 8 - (l * d2) / 8 + 1;
    n = t > n ? t : n;
  }
  return n;
}
}  // namespace hdgb

namespace hdgb {

template <int K_>
struct C5Dims {
  static constexpr int D3 = cdim3(K_), D2 = cdim2(K_), M = 4 * cdim2(K_);
  static constexpr int D34 = round_up(D3, 4);                    // contraction length over d3
  static constexpr int KS = D34 / 4;
  static constexpr int LD = (D34 % 16 == 4 || D34 % 16 == 12) ? D34 : D34 + 4;  // conflict-free stride
  static constexpr int D3P = round_up(D3, 8), MP = round_up(M, 8);
  static constexpr int MT = D3P / 8, NTM = MP / 8;
  static constexpr int NSYM = D3 * (D3 + 1) / 2;
  static constexpr int SQ = round_up(LD * LD + (D3P > LD ? D3P - LD : 0), 2);
  static constexpr int OFF_S = 0;
  static constexpr int OFF_MI = OFF_S + SQ;
  static constexpr int OFF_T0 = OFF_MI + SQ;
  static constexpr int OFF_T1 = OFF_T0 + SQ;
  static constexpr int OFF_Z = OFF_T1 + SQ;
  static constexpr int OFF_V = OFF_Z + LD * MP;
  static constexpr int OFF_DP = OFF_V + LD * MP;
  static constexpr int OFF_F = OFF_DP + round_up(NSYM, 2);
  static constexpr int OFF_FS = OFF_F + LD;
  static constexpr int OFF_COL = OFF_FS + LD;
  static constexpr int OFF_SG = OFF_COL + 8 * MP;
  static constexpr int OFF_RED = OFF_SG + 64;
  static constexpr int TOTAL = OFF_RED + 8;
  static constexpr int PER_ELT = TOTAL, CTA_EXTRA = 0;  // launch_condense_impl vocabulary (EPB = 1)
  static constexpr int FACTORS = round_up(NSYM + D3 * M + D3, 2);  // {M^-1 packed, Vs, fs}, 16-B records
  static_assert(2 * SQ >= LD * MP, "Vs must fit in the M^-1 | T0 space");
};

template <int K_> struct C5Cfg { static constexpr int NWT = 16; };
#ifndef HDG_C5_BLOCKINV
#define HDG_C5_BLOCKINV 1  // d3 = 56: block sweep with DMMA trailing updates (cta_block_inverse)
#endif

// Inverse of the full symmetric N x N matrix X (stride LD, shared memory) by
// the sweep operator with 2 x 2 pivots, all NT threads of the CTA. Thread
// layout: NT / N row groups per column, each thread owns one column c and a
// run of rows of it IN REGISTERS for the whole sweep. Each step the owners of
// the pivot rows k, k+1 and the threads of the pivot columns publish them
// (4 N doubles) to a double-buffered stage in Y (8 N doubles), one barrier
// per step, and every thread reads its column's pivot-row entries and its
// rows' pivot-column entries from there: the whole matrix no longer
// round-trips through shared memory each step. (Rows and columns are both
// published although the swept matrix is symmetric in exact arithmetic: the
// pivot columns carry the cancellation A - A (I - P^-1) of the sweep, the rows
// do not, and the update must use the same triangle as the reference order.)
// The result (X^-1, full) is written back to X.
// Returns the pivot test of local_solver.cpp:50-57 (Cholesky pivots).
// pmin / pmax (valid on thread 0) return the extreme |LDL^T pivots|, 0 for a
// vanished or non-finite one (the rescue screen, kernels_rescue.cuh).
template <int N, int LD, int NT>
__device__ __forceinline__ void cta_sweep_inverse(double* X, double* Y, double& pmin, double& pmax) {
  constexpr int RG = NT / N;                  // row groups per column
  constexpr int RPT = (N + RG - 1) / RG;      // rows per thread
  const int c = threadIdx.x / RG, i0 = (threadIdx.x - c * RG) * RPT;
  const bool live = c < N;
  double a[RPT];
#pragma unroll
  for (int u = 0; u < RPT; ++u) a[u] = (live && i0 + u < N) ? X[i0 + u + c * LD] : 0.0;
  pmin = 1e300;
  pmax = 0.0;
  bool bad = false;
  // stage of the pivot pair (k, k+1): [0, N) row k by column, [N, 2N) row
  // k+1, [2N, 3N) column k by row, [3N, 4N) column k+1. The entries a step
  // produces for the next pair are staged from the update loop itself.
  auto put = [&](double* st, int k, int u, bool colk, bool colk1, double v) {
    const int i = i0 + u;
    if (i == k) st[c] = v;
    if (i == k + 1) st[N + c] = v;
    if (colk) st[2 * N + i] = v;
    if (colk1) st[3 * N + i] = v;
  };
  // the pivot columns of the next pair: only their RG threads store (after
  // the update loop, so the other warps skip it)
  auto put_cols = [&](double* st, int k) {
    if (c == k || c == k + 1) {
      double* col = st + (c == k ? 2 : 3) * N;
#pragma unroll
      for (int u = 0; u < RPT; ++u)
        if (i0 + u < N) col[i0 + u] = a[u];
    }
  };
  if (live) {
#pragma unroll
    for (int u = 0; u < RPT; ++u)
      if (i0 + u < N) put(Y, 0, u, c == 0, c == 1, a[u]);
  }
  const bool stats = threadIdx.x < 32;  // the pivot test is returned to thread 0
  int buf = 0;
  for (int k = 0; k < N; k += 2, buf ^= 1) {
    double* st = Y + buf * 4 * N;
    double* nx = Y + (buf ^ 1) * 4 * N;
    __syncthreads();
    if (k + 1 < N) {
      const double p00 = st[k], p01 = st[2 * N + k + 1], p11 = st[N + k + 1];
      const double det = fma(p00, p11, -p01 * p01);
      const double id = gj_rcp(det);
      const double i00 = p11 * id, i01 = -p01 * id, i11 = p00 * id;
      if (stats) {
        const double d0 = fabs(p00), d1 = fabs(det * gj_rcp(p00));  // LDL^T pivots of the pair
        if (!(d0 > 0.0) || !(d1 > 0.0) || !(d0 <= 1.79e308) || !(d1 <= 1.79e308)) bad = true;
        pmin = fmin(pmin, fmin(d0, d1));
        pmax = fmax(pmax, fmax(d0, d1));
      }
      if (live) {
        const double a0 = st[c] - (c == k ? 1.0 : 0.0);
        const double a1 = st[N + c] - (c == k + 1 ? 1.0 : 0.0);
        const double w0 = fma(i00, a0, i01 * a1), w1 = fma(i01, a0, i11 * a1);
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int i = i0 + u;
          if (i < N) {
            double v = a[u] - fma(st[2 * N + i], w0, st[3 * N + i] * w1);
            if (i == k) v = w0 - (c == k ? 1.0 : 0.0);
            if (i == k + 1) v = w1 - (c == k + 1 ? 1.0 : 0.0);
            a[u] = v;
            put(nx, k + 2, u, false, false, v);
          }
        }
        put_cols(nx, k + 2);
      }
    } else {  // trailing scalar pivot
      const double p = st[k];
      if (stats) {
        if (!(fabs(p) > 0.0) || !(fabs(p) <= 1.79e308)) bad = true;
        pmin = fmin(pmin, fabs(p));
        pmax = fmax(pmax, fabs(p));
      }
      const double ip = gj_rcp(p);
      if (live) {
        const double w = (st[c] - (c == k ? 1.0 : 0.0)) * ip;
#pragma unroll
        for (int u = 0; u < RPT; ++u) {
          const int i = i0 + u;
          if (i < N) a[u] = i == k ? w - (c == k ? 1.0 : 0.0) : a[u] - st[2 * N + i] * w;
        }
      }
    }
  }
  // the sweep leaves -X^-1; negate into X
  if (live) {
#pragma unroll
    for (int u = 0; u < RPT; ++u)
      if (i0 + u < N && i0 + u >= c) {  // lower triangle, mirrored: the two halves of a
        X[i0 + u + c * LD] = -a[u];     // Gauss-Jordan inverse round differently
        X[c + (i0 + u) * LD] = -a[u];
      }
  }
  __syncthreads();
  if (bad) pmin = 0.0;
}

// Inverse of the full symmetric positive definite N x N matrix X (stride LD,
// shared memory; N a multiple of 8) by the block sweep operator with 8 x 8
// pivot blocks, all NT threads of the CTA: per block p, (a) one warp inverts
// the pivot block P = A_pp by the register sweep (gj_sweep_inverse, whose
// |LDL^T pivots| are the matrix's own, block by block), (b) Cb_i = A_ip P^-1
// for every other row block (DMMA), (c) A_ij -= Cb_i A_pj for i, j != p, one
// 8 x 8 DMMA tile per warp task (2 k-steps), (d) A_ip <- Cb_i, A_pj <- Cb_j^T,
// A_pp <- -P^-1. Sweeping every block leaves -X^-1; the lower triangle is
// written back negated and mirrored (the consumers' canonical entries, as
// cta_sweep_inverse). 7 block steps at N = 56 instead of 28 scalar 2 x 2
// pivot steps, the trailing updates on the DMMA pipe. Y: >= 712 + 2 N doubles
// of scratch (16-byte aligned). pmin / pmax valid on thread 0.
template <int N, int LD, int NT>
__device__ __forceinline__ void cta_block_inverse(double* X, double* Y, double& pmin, double& pmax) {
  static_assert(N % 8 == 0, "whole 8 x 8 blocks");
  constexpr int NB = N / 8, NW = NT / 32, LC = N + 4, LP = 12;
  double* Cb = Y;             // N x 8, column-major, stride LC
  double* Pi = Y + 8 * LC;    // 8 x 8, stride LP
  double* stage = Pi + 8 * LP + 8;  // gj sweep stage (128), 16-byte aligned
  double* pst = stage + 128;        // |LDL^T pivots| (min, max) of each block's 8 lanes, reduced at the end
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  pmin = 1e300;
  pmax = 0.0;
  for (int p = 0; p < NB; ++p) {
    const int p0 = 8 * p;
    // (a) P^-1 (warp 0, lane c < 8 owns column c)
    if (warp == 0) {
      double a[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = lane < 8 ? X[p0 + i + (p0 + lane) * LD] : 0.0;
      double bmin = 1e300, bmax = 0.0, piv = 1.0;
#pragma unroll
      for (int k = 0; k < 8; k += 2) gj_sweep_step<8>(a, stage, lane, k, piv);
      gj_sweep_finish<8, false>(a, stage, lane, piv, bmin, bmax);  // this lane's pivot: no reduction here
      if (lane < 8) {
        pst[16 * p + lane] = bmin;
        pst[16 * p + 8 + lane] = bmax;
      }
      if (lane < 8) {  // canonical entries: each pair from the lower-index lane's
#pragma unroll      // below-diagonal half (the upper half of a sweep column is less accurate)
        for (int i = 0; i < 8; ++i)
          if (i >= lane) {
            Pi[i + lane * LP] = a[i];
            Pi[lane + i * LP] = a[i];
          }
      }
    }
    __syncthreads();
    // (b) Cb_i = A_ip P^-1, i != p
    for (int i = warp; i < NB; i += NW) {
      if (i == p) continue;
      double c0 = 0.0, c1 = 0.0;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int k = 4 * kk + t;
        dmma(c0, c1, X[8 * i + g + (p0 + k) * LD], Pi[k + g * LP]);
      }
      Cb[8 * i + g + (2 * t) * LC] = c0;
      Cb[8 * i + g + (2 * t + 1) * LC] = c1;
    }
    __syncthreads();
    // (c) A_ij -= Cb_i A_pj, i, j != p (results held until every A_pj is read)
    constexpr int NU = (N / 8 - 1) * (N / 8 - 1);
    constexpr int TPW = (NU + NW - 1) / NW;
    double acc[TPW][2];
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      const int task = warp + u * NW;
      acc[u][0] = acc[u][1] = 0.0;
      if (task < NU) {
        int i = task / (NB - 1), j = task - i * (NB - 1);
        i += i >= p;
        j += j >= p;
        acc[u][0] = X[8 * i + g + (8 * j + 2 * t) * LD];
        acc[u][1] = X[8 * i + g + (8 * j + 2 * t + 1) * LD];
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int k = 4 * kk + t;
          dmma(acc[u][0], acc[u][1], -Cb[8 * i + g + k * LC], X[p0 + k + (8 * j + g) * LD]);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < TPW; ++u) {
      const int task = warp + u * NW;
      if (task < NU) {
        int i = task / (NB - 1), j = task - i * (NB - 1);
        i += i >= p;
        j += j >= p;
        X[8 * i + g + (8 * j + 2 * t) * LD] = acc[u][0];
        X[8 * i + g + (8 * j + 2 * t + 1) * LD] = acc[u][1];
      }
    }
    // (d) the pivot block row and column
    for (int idx = threadIdx.x; idx < 8 * N; idx += NT) {
      const int r = idx % N, c = idx / N;  // row r of column p0 + c
      const double v = (r >= p0 && r < p0 + 8) ? -Pi[(r - p0) + c * LP] : Cb[r + c * LC];
      X[r + (p0 + c) * LD] = v;           // column block
      X[p0 + c + r * LD] = v;             // row block (= its transpose)
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // every block's pivots (the stats were kept off the block steps' chains)
    for (int i = 0; i < 16 * NB; ++i) {
      if ((i & 15) < 8) pmin = fmin(pmin, pst[i]);
      else pmax = fmax(pmax, pst[i]);
    }
  }
  // -X^-1 -> X^-1, lower triangle mirrored
  for (int idx = threadIdx.x; idx < N * N; idx += NT) {
    const int r = idx % N, c = idx / N;
    if (r >= c) {
      const double v = -X[r + c * LD];
      X[r + c * LD] = v;
      if (r > c) X[c + r * LD] = v;
    }
  }
  __syncthreads();
}

template <int K_, bool SP = true>
__global__ void __launch_bounds__(C5Cfg<K_>::NWT * 32, 1)
condense5_kernel(DevTab tab, int nelt, GeoDev geo, const double* __restrict__ Msym,
                 const double* __restrict__ Dsym, const double* __restrict__ fvec,
                 double* __restrict__ Cout, double* __restrict__ Cfout, double* __restrict__ factors,
                 double* __restrict__ pivstat) {
  using Dm = C5Dims<K_>;
  constexpr int NWT = C5Cfg<K_>::NWT, NT = NWT * 32;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, MP = Dm::MP, LD = Dm::LD, KS = Dm::KS;
  constexpr int MT = Dm::MT, NTM = Dm::NTM, NSYM = Dm::NSYM;
  constexpr int NTF = face_tiles(D2);
  constexpr int NLP = (NTM / 2 + 1) * ((NTM + 1) / 2);  // C tile pairs (rows' pairs and singles)
  constexpr bool PAD = Dm::D34 != D3;                    // k-padding present (k = 4)
  // Structural zeros of Chat_h (kernels_condense6.cuh; checked on the host by
  // check_chat_pattern): rows >= dim P_{k-1} vanish and the rest is strictly
  // upper triangular, Chat_h(r, k) = 0 for k <= r. Row tiles >= NT1 of Chat_h
  // are skipped, and a row tile's ksteps start at its first row.
  constexpr int N1 = (HDG_C5_SPARSE && SP) ? cdim3(K_ - 1) : D3;
  constexpr int NT1 = (N1 + 7) / 8;
  constexpr int KSKIP = (HDG_C5_SPARSE && SP) ? 2 : 0;           // ksteps below row tile nt: 2 * nt
  extern __shared__ double smem[];
  for (int i = threadIdx.x; i < Dm::TOTAL; i += NT) smem[i] = 0.0;
  __syncthreads();
  double* S = smem + Dm::OFF_S;
  double* Mi = smem + Dm::OFF_MI;
  double* T0 = smem + Dm::OFF_T0;
  double* T1 = smem + Dm::OFF_T1;
  double* Z = smem + Dm::OFF_Z;
  double* V = smem + Dm::OFF_V;
  double* Vs = smem + Dm::OFF_MI;  // P7..P8: M^-1 and T0 are dead
  double* Dp = smem + Dm::OFF_DP;
  double* fv = smem + Dm::OFF_F;
  double* fs = smem + Dm::OFF_FS;
  double* col = smem + Dm::OFF_COL;
  double* sg = smem + Dm::OFF_SG;
  const double* Tc = col + 3 * MP;
  const int* wb = reinterpret_cast<const int*>(col + 4 * MP);
  const double* beta = col + 5 * MP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const double* Wlm = tab.Wlm;
  const double* Ch = tab.Chat;

  // Chat_h(r, k) from L1/L2 (k-padding and tile rows past d3 read as zero)
  auto chat = [&](int h, int r, int k) -> double {
    if (PAD || D3 % 8) {
      if (r >= D3 || k >= D3) return 0.0;
    }
    return __ldg(Ch + h * D3 * D3 + r + k * D3);
  };
  // T_h = M^-1 Chat_h^T by column strips: column tile nt, row tiles [lo, hi)
  // (three row groups per column): the Chat fragment of a k-step (L1/L2)
  // feeds every row tile of the group
  constexpr int TSG = 3;                           // row groups per column strip
  constexpr int NTS = NT1 * TSG;                   // T strip tasks (column tiles < NT1: the nonzero rows of Chat_h)
  auto t_strip = [&](double* Tb, int h, int task) {
    const int nt = task / TSG, part = task - nt * TSG;
    const int lo = part * MT / TSG, hi = (part + 1) * MT / TSG;
    const int c = nt * 8 + g;
    double acc[(MT + TSG - 1) / TSG][2];
#pragma unroll
    for (int u = 0; u < (MT + TSG - 1) / TSG; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll 2
    for (int kk = KSKIP * nt; kk < KS; ++kk) {
      const int k = kk * 4 + t;
      const double b = chat(h, c, k);
#pragma unroll
      for (int u = 0; u < (MT + TSG - 1) / TSG; ++u)
        if (lo + u < hi) dmma(acc[u][0], acc[u][1], Mi[((lo + u) * 8 + g) + k * LD], b);
    }
    const int c0 = nt * 8 + 2 * t;
#pragma unroll
    for (int u = 0; u < (MT + TSG - 1) / TSG; ++u) {
      const int rr = (lo + u) * 8 + g;
      if (lo + u < hi && rr < LD) {
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2)
          if (c0 + h2 < D3) Tb[rr + (c0 + h2) * LD] = rr < D3 ? acc[u][h2] : 0.0;
      }
    }
  };
  // S (+)= Chat'_h Tb by row strips: row tile mt, column tiles of one chunk
  // (rows split into chunks of <= 3 lower tiles): the combined Chat'_h
  // fragment (3 L1/L2 loads + FMAs) of a k-step feeds the whole chunk
  constexpr int SCH = 3;                           // lower tiles per S task at most
  constexpr int NSS = [] {                         // row tiles < NT1 only: Chat'_h vanishes below
    int n = 0;
    for (int mt = 0; mt < NT1; ++mt) n += (mt + SCH) / SCH;
    return n;
  }();
  auto s_strip = [&](const double* Tb, int h, int task, bool first) {
    int mt = 0, rem = task;
    while (rem >= (mt + SCH) / SCH) { rem -= (mt + SCH) / SCH; ++mt; }
    const int nch = (mt + SCH) / SCH;
    const int jlo = rem * (mt + 1) / nch, jhi = (rem + 1) * (mt + 1) / nch;
    const int r = mt * 8 + g;
    const double g0 = sg[32 + h], g1 = sg[35 + h], g2 = sg[38 + h];  // G symmetric: G(#, h)
    double acc[SCH][2];
#pragma unroll
    for (int u = 0; u < SCH; ++u) acc[u][0] = acc[u][1] = 0.0;
#pragma unroll 2
    for (int kk = KSKIP * mt; kk < KS; ++kk) {
      const int k = kk * 4 + t;
      const double a = g0 * chat(0, r, k) + g1 * chat(1, r, k) + g2 * chat(2, r, k);
#pragma unroll
      for (int u = 0; u < SCH; ++u)
        if (jlo + u < jhi) dmma(acc[u][0], acc[u][1], a, Tb[k + ((jlo + u) * 8 + g) * LD]);
    }
#pragma unroll
    for (int u = 0; u < SCH; ++u) {
      if (jlo + u >= jhi) break;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int c = (jlo + u) * 8 + 2 * t + h2;
        if (r < D3 && c <= r) {
          const double v = (first ? Dp[sym_idx(r, c, D3)] : S[r + c * LD]) + acc[u][h2];
          S[r + c * LD] = v;
          S[c + r * LD] = v;
        }
      }
    }
  };

  // the next element's inputs stream in while this one computes, each as soon
  // as its buffer is dead: packed D after P3, packed M (into T1) after the S
  // inverse, f after P7, the geometry record into registers
  auto geo_value = [&](long Kx) {
    const int i = threadIdx.x;
    if (i == 0) return geo.volume[Kx];
    if (i < 10) return geo.piola[long(i - 1) * nelt + Kx];
    if (i < 22) return geo.normals[long(i - 10) * nelt + Kx];
    if (i < 26) return geo.T[long(i - 22) * nelt + Kx];
    return double(geo.perm[long(i - 26) * nelt + Kx]);
  };
  auto prefetch_packed = [&](double* dst, const double* src, long Kx) {
    for (int p = threadIdx.x; p < NSYM; p += NT) cp_async8(dst + p, src + Kx * NSYM + p);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto prefetch_f = [&](long Kx) {
    for (int i = threadIdx.x; i < D3; i += NT) cp_async8(fv + i, fvec + Kx * D3 + i);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  double gnext = 0.0;
  if (long(blockIdx.x) < nelt) {
    const long K = blockIdx.x;
    if (threadIdx.x < 30) gnext = geo_value(K);
    prefetch_packed(T1, Msym, K);
    prefetch_packed(Dp, Dsym, K);
    prefetch_f(K);
  }

  for (long K = blockIdx.x; K < nelt; K += gridDim.x) {
    const long Kn = K + gridDim.x;
    const bool has_next = Kn < nelt;
    // ---- prologue: geometry, column data, packed M / D / f (prefetched)
    if (threadIdx.x < 30) sg[threadIdx.x] = gnext;
    cp_async_wait_all();
    __syncthreads();
    if (warp == 0) {
      build_columns<D2, D3, M, MP>(sg, col, lane);
      if (lane < 9) {
        const int h = lane / 3, h2 = lane % 3;
        sg[32 + lane] = sg[1 + h] * sg[1 + h2] + sg[4 + h] * sg[4 + h2] + sg[7 + h] * sg[7 + h2];
      } else if (lane >= 16) {
        const int l1 = (lane - 16) >> 2, l2 = lane & 3;
        sg[48 + (lane - 16)] = sg[10 + 3 * l1] * sg[10 + 3 * l2] + sg[11 + 3 * l1] * sg[11 + 3 * l2] +
                               sg[12 + 3 * l1] * sg[12 + 3 * l2];
      }
    }
    // expand packed M (in T1) to the full LD-strided matrix, padding zero
    for (int idx = threadIdx.x; idx < LD * LD; idx += NT) {
      const int c = idx / LD, r = idx - c * LD;
      Mi[idx] = (r < D3 && c < D3) ? T1[r >= c ? sym_idx(r, c, D3) : sym_idx(c, r, D3)] : 0.0;
    }
    __syncthreads();

    // ---- P1: M^-1 (CTA sweep), packed lower part into the recovery cache
    {
      double pmin, pmax;
      if constexpr (D3 % 8 == 0 && HDG_C5_BLOCKINV) cta_block_inverse<D3, LD, NT>(Mi, T0, pmin, pmax);
      else cta_sweep_inverse<D3, LD, NT>(Mi, T0, pmin, pmax);
      if (threadIdx.x == 0) store_pivstat(pivstat, K, 0, pmin, pmax);
    }
    if (factors)  // packed lower, column-major: column c at sym_idx(c, c)
      for (int c = warp; c < D3; c += NWT)
        for (int i = c + lane; i < D3; i += 32) factors[K * Dm::FACTORS + sym_idx(i, c, D3)] = Mi[i + c * LD];

    // ---- P2: Zp strips (T_l W_l^T staged into V) | T0 = M^-1 Chat_0^T
    for (int task = warp; task < NTM + NTS; task += NWT) {
      if (task < NTM) {
        const int nt = task, cz = nt * 8 + g, wbc = wb[cz];
        const double tc = Tc[cz];
        double acc[MT][2];
#pragma unroll
        for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
#pragma unroll 2
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const double b = (wbc >= 0 && k < D3) ? __ldg(Wlm + wbc + k * D2) : 0.0;
          V[k + cz * LD] = tc * b;
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(acc[m][0], acc[m][1], Mi[(m * 8 + g) + k * LD], b);
        }
        const int c0 = nt * 8 + 2 * t;
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const int r = m * 8 + g;
          if (r < LD) {
            Z[r + c0 * LD] = r < D3 ? acc[m][0] : 0.0;
            Z[r + (c0 + 1) * LD] = r < D3 ? acc[m][1] : 0.0;
          }
        }
      } else {
        t_strip(T0, 0, task - NTM);
      }
    }
    __syncthreads();
    // ---- P3..P5: S accumulation beside the next T product / the V rows
    for (int task = warp; task < NSS + NTS; task += NWT) {
      if (task < NSS) s_strip(T0, 0, task, true);
      else t_strip(T1, 1, task - NSS);
    }
    // rows >= 8 NT1 of S are D alone (Chat'_h vanishes there)
    for (int idx = threadIdx.x; idx < (D3 - NT1 * 8) * D3; idx += NT) {
      const int r = NT1 * 8 + idx / D3, c = idx - (idx / D3) * D3;
      if (c <= r) {
        const double v = Dp[sym_idx(r, c, D3)];
        S[r + c * LD] = v;
        S[c + r * LD] = v;
      }
    }
    __syncthreads();
    if (has_next) prefetch_packed(Dp, Dsym, Kn);  // the packed D of this element is dead
    for (int task = warp; task < NSS + NTS; task += NWT) {
      if (task < NSS) s_strip(T1, 1, task, false);
      else t_strip(T0, 2, task - NSS);
    }
    __syncthreads();
    for (int task = warp; task < NSS + 4 * NT1; task += NWT) {  // V: row tiles < NT1 (below, V keeps the staged T_l W_l^T)
      if (task < NSS) {
        s_strip(T0, 2, task, false);
      } else {  // V rows of row tile mt, face l
        const int mt = (task - NSS) >> 2, l = (task - NSS) & 3;
        const int r = mt * 8 + g;
        const int cl0 = l * D2, cl1 = cl0 + D2, nt0 = cl0 / 8;
        const double b0 = beta[cl0], b1 = beta[MP + cl0], b2 = beta[2 * MP + cl0];
        double acc[NTF][2] = {};
#pragma unroll 2
        for (int kk = KSKIP * mt; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const double a = b0 * chat(0, r, k) + b1 * chat(1, r, k) + b2 * chat(2, r, k);
#pragma unroll
          for (int j = 0; j < NTF; ++j) {
            const int c = (nt0 + j) * 8 + g;
            const double b = (c >= cl0 && c < cl1) ? Z[k + c * LD] : 0.0;
            if ((nt0 + j) * 8 < cl1) dmma(acc[j][0], acc[j][1], a, b);
          }
        }
        if (r < LD) {
#pragma unroll
          for (int j = 0; j < NTF; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = (nt0 + j) * 8 + 2 * t + h;
              if (c >= cl0 && c < cl1) V[r + c * LD] = r < D3 ? acc[j][h] + V[r + c * LD] : 0.0;
            }
        }
      }
    }
    __syncthreads();
    if (tab.nu < D3) {  // BDM (bdm_blocks, local_solver.cpp:65-69): the scalar space is P_{k-1}:
      // decouple the remaining modes (identity-scaled S, zero V rows and f)
      const int nu = tab.nu;
      for (int idx = threadIdx.x; idx < D3 * D3; idx += NT) {
        const int r = idx % D3, c = idx / D3;
        if (r >= nu || c >= nu) S[r + c * LD] = r == c ? 6.0 * sg[0] : 0.0;
      }
      for (int idx = threadIdx.x; idx < (D3 - nu) * MP; idx += NT) {
        const int r = nu + idx % (D3 - nu), c = idx / (D3 - nu);
        V[r + c * LD] = 0.0;
      }
      for (int r = nu + threadIdx.x; r < D3; r += NT) fv[r] = 0.0;
      __syncthreads();
    }

    // ---- P6: S^-1 (CTA sweep)
    {
      double pmin, pmax;
      if constexpr (D3 % 8 == 0 && HDG_C5_BLOCKINV) cta_block_inverse<D3, LD, NT>(S, T1, pmin, pmax);
      else cta_sweep_inverse<D3, LD, NT>(S, T1, pmin, pmax);
      if (threadIdx.x == 0) store_pivstat(pivstat, K, 1, pmin, pmax);
    }
    if (has_next) prefetch_packed(T1, Msym, Kn);  // T1 (the inverse's scratch) is dead

    // ---- P7: Vs = S^-1 V strips | fs = S^-1 f
    for (int task = warp; task < NTM; task += NWT) {
      const int nt = task, c = nt * 8 + g;
      double acc[MT][2];
#pragma unroll
      for (int m = 0; m < MT; ++m) acc[m][0] = acc[m][1] = 0.0;
#pragma unroll 2
      for (int kk = 0; kk < KS; ++kk) {
        const int k = kk * 4 + t;
        const double b = V[k + c * LD];
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma(acc[m][0], acc[m][1], S[(m * 8 + g) + k * LD], b);
      }
      const int c0 = nt * 8 + 2 * t;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const int r = m * 8 + g;
        if (r < LD) {
          Vs[r + c0 * LD] = r < D3 ? acc[m][0] : 0.0;
          Vs[r + (c0 + 1) * LD] = r < D3 ? acc[m][1] : 0.0;
        }
      }
    }
    for (int r = threadIdx.x; r < D3; r += NT) {
      double s = 0.0;
      for (int k = 0; k < D3; ++k) s += S[r + k * LD] * fv[k];
      fs[r] = s;
    }
    __syncthreads();
    if (factors) {  // recovery cache: Vs = S^-1 V (d3 x m) and fs = S^-1 f after M^-1
      constexpr int NVF = D3 * M + D3;
      for (int q = threadIdx.x; q < NVF; q += NT) {
        const int c = q / D3, r = q - c * D3;
        factors[K * Dm::FACTORS + NSYM + q] = c < M ? Vs[r + c * LD] : fs[r];
      }
    }

    if (has_next) {
      prefetch_f(Kn);  // f of this element is dead after P7's fs (the barrier above)
      if (threadIdx.x < 30) gnext = geo_value(Kn);
    }
    // ---- P8: C (lower tile pairs, mirrored) | Cf
    for (int task = warp; task < NLP; task += NWT) {
      const int mt = int(2.0f * sqrtf(float(task) + 0.25f)) - 1;
      const int nt0 = 2 * (task - (mt + 1) * (mt + 1) / 4), r = mt * 8 + g;
      const bool two = nt0 + 1 <= mt;
      const int wbr = wb[r];
      double z[2][2] = {{0, 0}, {0, 0}}, v[2][2] = {{0, 0}, {0, 0}};
#pragma unroll 2
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
        const double* nn4 = sg + 48 + 4 * l1;
        double* Ck = Cout + K * M * M;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          if (u == 1 && !two) break;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = (nt0 + u) * 8 + 2 * t + h;
            if (c > r || c >= M) continue;
            const int l2 = c / D2;
            double val = nn4[l2] * z[u][h] - v[u][h];
            if (l1 == l2) val += Tc[c] * __ldg(tab.DD + (r - l1 * D2) + (c - l2 * D2) * D2);
            Ck[r + c * M] = val;
            if (c != r) Ck[c + r * M] = val;
          }
        }
      }
    }
    for (int r = threadIdx.x; r < M; r += NT) {
      double s = 0.0;
      for (int k = 0; k < D3; ++k) s += V[k + r * LD] * fs[k];
      Cfout[K * M + r] = s;
    }
    __syncthreads();
  }
}

}  // namespace hdgb
