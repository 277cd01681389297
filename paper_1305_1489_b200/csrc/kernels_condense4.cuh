// K3 v4 (k = 2, 3): element-batched condensation tasks.
//
// Same algebra as kernels_condense2.cuh (explicit M^-1 and S^-1 by warp
// sweep Gauss-Jordan, every contraction a DMMA tile loop). The CTA holds a
// batch of EPB elements and every task computes ONE output tile for ALL EPB
// elements: the reference-table operand of each DMMA (Chat, W rows) is loaded
// once per k-step and reused EPB times, and each warp carries EPB independent
// accumulator chains, which hides the DMMA latency with only 8 warps per SM.
// In P3 every GJ warp sweeps two matrices in lockstep (S of this batch and M
// of the next batch), so the two latency-bound inversions cost one.
#pragma once

#include "kernels_condense2.cuh"

namespace hdgb {

template <int K_> struct C4Cfg;
template <> struct C4Cfg<2> { static constexpr int EPB = 8, NWT = 8; };
template <> struct C4Cfg<3> { static constexpr int EPB = 4, NWT = 8; };

// Two SPD N x N inverses swept in lockstep by one warp (see warp_gj_inverse).
template <int N>
__device__ __forceinline__ void warp_gj_inverse_pair(double (&a)[2][N], double* stA, double* stB, int lane,
                                                     double (&pmin)[2], double (&pmax)[2]) {
  double piv0[2][N / 2 + 1], pdet[2][N / 2 + 1];
  double* stg[2] = {stA, stB};
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) {
    double w0[2], w1[2], nk0[2], nk1[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      double* st = stg[x] + ((k >> 1) & 1) * 64;
      if (lane < N) {
        st[lane] = a[x][k];
        st[32 + lane] = a[x][k + 1];
      }
      const double p00 = __shfl_sync(0xffffffffu, a[x][k], k);
      const double p01 = __shfl_sync(0xffffffffu, a[x][k + 1], k);
      const double p11 = __shfl_sync(0xffffffffu, a[x][k + 1], k + 1);
      const double det = fma(p00, p11, -p01 * p01);
      piv0[x][k >> 1] = p00;
      pdet[x][k >> 1] = det;
      const double id = fast_rcp(det);
      const double i00 = p11 * id, i01 = -p01 * id, i11 = p00 * id;
      const bool m0 = lane == k, m1 = lane == k + 1;
      w0[x] = fma(i00, a[x][k], i01 * a[x][k + 1]);
      w1[x] = fma(i01, a[x][k], i11 * a[x][k + 1]);
      if (m0) { w0[x] = 1.0 - i00; w1[x] = -i01; }
      if (m1) { w0[x] = -i01; w1[x] = 1.0 - i11; }
      nk0[x] = w0[x];
      nk1[x] = w1[x];
      if (m0) { nk0[x] = -i00; nk1[x] = -i01; }
      if (m1) { nk0[x] = -i01; nk1[x] = -i11; }
    }
    __syncwarp();
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
      for (int i0 = 0; i0 < N; i0 += 2) {
        if (i0 == k) continue;
        if ((pass == 0) != (i0 == k + 2)) continue;
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const double* st = stg[x] + ((k >> 1) & 1) * 64;
          const double2 v0 = *reinterpret_cast<const double2*>(st + i0);
          const double2 v1 = *reinterpret_cast<const double2*>(st + 32 + i0);
          a[x][i0] = fma(-v0.x, w0[x], fma(-v1.x, w1[x], a[x][i0]));
          if (i0 + 1 < N) a[x][i0 + 1] = fma(-v0.y, w0[x], fma(-v1.y, w1[x], a[x][i0 + 1]));
        }
      }
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      a[x][k] = nk0[x];
      a[x][k + 1] = nk1[x];
    }
  }
  if (N % 2) {
    constexpr int k = N - 1;
    double t[2], nk[2];
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      double* st = stg[x] + ((k >> 1) & 1) * 64;
      if (lane < N) st[lane] = a[x][k];
      const double p = __shfl_sync(0xffffffffu, a[x][k], k);
      piv0[x][k >> 1] = p;
      pdet[x][k >> 1] = p * p;
      const double ip = fast_rcp(p);
      const bool me = lane == k;
      t[x] = me ? 1.0 - ip : a[x][k] * ip;
      nk[x] = me ? -ip : a[x][k] * ip;
    }
    __syncwarp();
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const double* st = stg[x] + ((k >> 1) & 1) * 64;
#pragma unroll
      for (int i = 0; i < k; ++i) a[x][i] = fma(-st[i], t[x], a[x][i]);
      a[x][k] = nk[x];
    }
  }
  __syncwarp();
#pragma unroll
  for (int x = 0; x < 2; ++x) {
#pragma unroll
    for (int i = 0; i < N; ++i) a[x][i] = -a[x][i];
#pragma unroll
    for (int j = 0; j < (N + 1) / 2; ++j) {
      const double d1 = pdet[x][j] / piv0[x][j];
      pmin[x] = fmin(pmin[x], fmin(piv0[x][j], d1));
      pmax[x] = fmax(pmax[x], fmax(piv0[x][j], d1));
    }
  }
}

template <int K_>
__global__ void __launch_bounds__(C4Cfg<K_>::NWT * 32)
condense4_kernel(DevTab tab, int nelt, GeoDev geo, const double* __restrict__ Msym,
                 const double* __restrict__ Dsym, const double* __restrict__ fvec,
                 double* __restrict__ Cout, double* __restrict__ Cfout, double* __restrict__ factors,
                 long long* bad_element) {
  using Dm = C2Dims<K_>;
  constexpr int E = C4Cfg<K_>::EPB, NWT = C4Cfg<K_>::NWT, NT = NWT * 32;
  constexpr int D3 = Dm::D3, D2 = Dm::D2, M = Dm::M, D3P = Dm::D3P, MP = Dm::MP, LD = Dm::LD;
  constexpr int MT = Dm::MT, NTM = Dm::NTM, KS = Dm::KS, NS = Dm::NSYM;
  constexpr int NLOW = NTM * (NTM + 1) / 2;
  constexpr int NLS = MT * (MT + 1) / 2;
  constexpr int NTF = (D2 + 7) / 8 + 1;
  constexpr int NGJW = E < NWT ? E : NWT;       // warps sweeping (S_e, M_next_e) pairs
  static_assert(NLOW * 64 <= 3 * D3P * LD, "W Zp tiles must fit in the R buffer");
  extern __shared__ double smem[];
  for (int i = threadIdx.x; i < E * Dm::PER_ELT; i += blockDim.x) smem[i] = 0.0;
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const double* Wlm = tab.Wlm;
  const double* Ch = tab.Chat;
  auto B = [&](int e) { return smem + e * Dm::PER_ELT; };
  auto Mi = [&](int e) { return B(e) + Dm::OFF_MI; };
  auto Sb = [&](int e) { return B(e) + Dm::OFF_S; };
  auto Yb = [&](int e) { return B(e) + Dm::OFF_Y; };  // R_#, then W Zp tiles
  auto Zb = [&](int e) { return B(e) + Dm::OFF_Z; };  // Zp, then Vs
  auto Vb = [&](int e) { return B(e) + Dm::OFF_V; };
  auto fv = [&](int e) { return B(e) + Dm::OFF_F; };
  auto fs = [&](int e) { return B(e) + Dm::OFF_FS; };
  auto stS = [&](int e) { return B(e) + Dm::OFF_STG; };
  auto stM = [&](int e) { return B(e) + Dm::OFF_STG2; };
  auto colb = [&](int e, int b) { return B(e) + (b ? Dm::OFF_COL : Dm::OFF_NSC); };
  auto sgb = [&](int e, int b) { return B(e) + Dm::OFF_GEO + 32 * b; };

  const long stride = long(gridDim.x) * E;
  long K0 = long(blockIdx.x) * E;
  int cur = 0;
  int batch = 0;

  auto load_geo_batch = [&](long Kb, int which) {
    for (int idx = threadIdx.x; idx < E * 32; idx += NT) {
      const int e = idx >> 5, i = idx & 31;
      const long K = Kb + e;
      if (K < nelt && i < 30) {
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
  auto load_Df = [&](long Kb) {  // D (packed lower -> lower of Sb) and f, one warp per element
    for (int e = warp; e < E; e += NWT) {
      const long K = Kb + e;
      if (K >= nelt) continue;
      const double* Dk = Dsym + K * NS;
      double* S = Sb(e);
      for (int j = 0; j < D3; ++j) {
        const int b0 = sym_idx(j, j, D3);
        for (int i = lane; i < D3 - j; i += 32) S[(j + i) + j * LD] = Dk[b0 + i];
      }
      for (int i = lane; i < D3; i += 32) fv(e)[i] = fvec[K * D3 + i];
    }
  };
  auto load_packed = [&](long K, double (&a)[D3]) {  // column `lane` of packed M
#pragma unroll
    for (int i = 0; i < D3; ++i) {
      const int r = i > lane ? i : lane, c = i > lane ? lane : i;
      a[i] = (K < nelt && lane < D3) ? Msym[K * NS + sym_idx(r, c, D3)] : (i == lane ? 1.0 : 0.0);
    }
  };
  auto store_inv = [&](int e, long K, double* dst, int fofs, const double (&a)[D3]) {
    if (K >= nelt || lane >= D3) return;
#pragma unroll
    for (int i = 0; i < D3; ++i) dst[i + lane * LD] = a[i];
    if (factors) {
#pragma unroll
      for (int i = 0; i < D3; ++i)
        if (i >= lane) factors[K * Dm::FACTORS + fofs + sym_idx(i, lane, D3)] = a[i];
    }
  };

  // ---- prologue: first batch's geometry, D, f, M^-1, column data
  if (K0 < nelt) {
    load_geo_batch(K0, 0);
    load_Df(K0);
    for (int e = warp; e < E; e += NWT) {
      double a[D3];
      load_packed(K0 + e, a);
      double pmin = 1e300, pmax = 0.0;
      warp_gj_inverse<D3>(a, stM(e), lane, pmin, pmax);
      store_inv(e, K0 + e, Mi(e), 0, a);
      if (K0 + e < nelt && (!(pmin > 0.0) || pmin < 1e-14 * pmax) && lane == 0) flag_bad(bad_element, K0 + e);
    }
    __syncthreads();
    for (int e = warp; e < E; e += NWT) build_columns<D2, D3, M, MP>(sgb(e, 0), colb(e, 0), lane);
    __syncthreads();
  }

  for (; K0 < nelt; K0 += stride, ++batch) {
    PHASE_MARK(batch, 0);
    const long Kn0 = K0 + stride;
    const bool has_next = Kn0 < nelt;
    const int nb = int(nelt - K0 < E ? nelt - K0 : E);

    // ------------- P1: R_# tiles = g-combinations of Mi Chat^T | Zp strips = Mi W^T
    for (int task = warp; task < MT * MT + NTM; task += NWT) {
      if (task < MT * MT) {
        const int m = task / MT, nt = task % MT;
        const int c = nt * 8 + g, r = m * 8 + g, c0 = nt * 8 + 2 * t;
        double q[E][3][2];
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
          for (int h = 0; h < 3; ++h) q[e][h][0] = q[e][h][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          const bool in = k < D3 && c < D3;
          const int o = c + k * D3;
          const double b0 = in ? __ldg(Ch + o) : 0.0, b1 = in ? __ldg(Ch + D3 * D3 + o) : 0.0,
                       b2 = in ? __ldg(Ch + 2 * D3 * D3 + o) : 0.0;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double a = Mi(e)[r + k * LD];
            dmma(q[e][0][0], q[e][0][1], a, b0);
            dmma(q[e][1][0], q[e][1][1], a, b1);
            dmma(q[e][2][0], q[e][2][1], a, b2);
          }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (e >= nb) break;
          const double* a9 = sgb(e, cur) + 1;
#pragma unroll
          for (int h = 0; h < 3; ++h) {
            const double g0 = a9[h] * a9[0] + a9[3 + h] * a9[3] + a9[6 + h] * a9[6];
            const double g1 = a9[h] * a9[1] + a9[3 + h] * a9[4] + a9[6 + h] * a9[7];
            const double g2 = a9[h] * a9[2] + a9[3 + h] * a9[5] + a9[6 + h] * a9[8];
            double* R = Yb(e) + h * D3P * LD;
            R[r + c0 * LD] = g0 * q[e][0][0] + g1 * q[e][1][0] + g2 * q[e][2][0];
            R[r + (c0 + 1) * LD] = g0 * q[e][0][1] + g1 * q[e][1][1] + g2 * q[e][2][1];
          }
        }
      } else {
        const int nt = task - MT * MT;
        const int c = nt * 8 + g, c0 = nt * 8 + 2 * t;
        double acc[E][MT][2];
        int wbc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          wbc[e] = reinterpret_cast<const int*>(colb(e, cur) + 4 * MP)[c];
#pragma unroll
          for (int m = 0; m < MT; ++m) acc[e][m][0] = acc[e][m][1] = 0.0;
        }
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double b = (wbc[e] >= 0 && k < D3) ? __ldg(Wlm + wbc[e] + k * D2) : 0.0;
#pragma unroll
            for (int m = 0; m < MT; ++m) dmma(acc[e][m][0], acc[e][m][1], Mi(e)[(m * 8 + g) + k * LD], b);
          }
        }
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
          for (int m = 0; m < MT; ++m) {
            Zb(e)[(m * 8 + g) + c0 * LD] = acc[e][m][0];
            Zb(e)[(m * 8 + g) + (c0 + 1) * LD] = acc[e][m][1];
          }
      }
    }
    __syncthreads();

    PHASE_MARK(batch, 1);
    // ---- GJ warps prefetch the next batch's M (sweep in P3) before P2 work
    double mnext[D3];
    if (warp < NGJW) load_packed(has_next ? Kn0 + warp : long(nelt), mnext);

    // ---- P2: S += sum_# Chat_# R_# (lower tiles) | V_l = Chat_l Zp_l + T_l W_l^T
    for (int task = warp; task < NLS + 4 * MT; task += NWT) {
      if (task < NLS) {
        int mt = 0, rem = task;
        while (rem > mt) { rem -= mt + 1; ++mt; }
        const int j = rem, r = mt * 8 + g;
        double acc[E][2];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e][0] = acc[e][1] = 0.0;
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          const double* C = Ch + h * D3 * D3;
#pragma unroll
          for (int kk = 0; kk < KS; ++kk) {
            const int k = kk * 4 + t;
            const double a = (r < D3 && k < D3) ? __ldg(C + r + k * D3) : 0.0;
#pragma unroll
            for (int e = 0; e < E; ++e)
              dmma(acc[e][0], acc[e][1], a, Yb(e)[h * D3P * LD + k + (j * 8 + g) * LD]);
          }
        }
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = j * 8 + 2 * t + h;
            if (r < D3 && c <= r) Sb(e)[r + c * LD] += acc[e][h];
          }
      } else {
        const int mt = (task - NLS) >> 2, l = (task - NLS) & 3;
        const int r = mt * 8 + g;
        const int cl0 = l * D2, cl1 = cl0 + D2, nt0 = cl0 / 8;
        double bt[E][3];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double* beta = colb(e, cur) + 5 * MP;
          bt[e][0] = beta[cl0];
          bt[e][1] = beta[MP + cl0];
          bt[e][2] = beta[2 * MP + cl0];
        }
        double acc[E][NTF][2];
#pragma unroll
        for (int e = 0; e < E; ++e)
#pragma unroll
          for (int j = 0; j < NTF; ++j) acc[e][j][0] = acc[e][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
          double c0 = 0.0, c1 = 0.0, c2 = 0.0;
          if (r < D3 && k < D3) {
            const int o = r + k * D3;
            c0 = __ldg(Ch + o);
            c1 = __ldg(Ch + D3 * D3 + o);
            c2 = __ldg(Ch + 2 * D3 * D3 + o);
          }
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double a = bt[e][0] * c0 + bt[e][1] * c1 + bt[e][2] * c2;
#pragma unroll
            for (int j = 0; j < NTF; ++j) {
              const int c = (nt0 + j) * 8 + g;
              const double b = (c >= cl0 && c < cl1) ? Zb(e)[k + c * LD] : 0.0;
              if ((nt0 + j) * 8 < cl1) dmma(acc[e][j][0], acc[e][j][1], a, b);
            }
          }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double* col = colb(e, cur);
          const double* Tc = col + 3 * MP;
          const int* wb = reinterpret_cast<const int*>(col + 4 * MP);
#pragma unroll
          for (int j = 0; j < NTF; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = (nt0 + j) * 8 + 2 * t + h;
              if (c >= cl0 && c < cl1 && r < D3)
                Vb(e)[r + c * LD] = acc[e][j][h] + Tc[c] * __ldg(Wlm + wb[c] + r * D2);
            }
        }
      }
    }
    __syncthreads();

    PHASE_MARK(batch, 2);
    // ---- P3: GJ warps sweep (S_e, M_next_e) in lockstep | other warps:
    //      (W Zp) tiles -> Yb, V and f -> recovery cache
    if (warp < NGJW) {
      for (int e = warp; e < E; e += NGJW) {
        double a[2][D3];
#pragma unroll
        for (int i = 0; i < D3; ++i) {
          const int r = i > lane ? i : lane, c = i > lane ? lane : i;
          a[0][i] = lane < D3 ? Sb(e)[r + c * LD] : (i == lane ? 1.0 : 0.0);
          a[1][i] = mnext[i];
        }
        double pmin[2] = {1e300, 1e300}, pmax[2] = {0.0, 0.0};
        warp_gj_inverse_pair<D3>(a, stS(e), stM(e), lane, pmin, pmax);
        const long K = K0 + e, Kn = Kn0 + e;
        if (e < nb) {
          double s[D3];
#pragma unroll
          for (int i = 0; i < D3; ++i) s[i] = a[0][i];
          store_inv(e, K, Sb(e), NS, s);
          if ((!(pmin[0] > 0.0) || pmin[0] < 1e-14 * pmax[0]) && lane == 0) flag_bad(bad_element, K);
        }
        if (has_next && Kn < nelt) {
          double s[D3];
#pragma unroll
          for (int i = 0; i < D3; ++i) s[i] = a[1][i];
          store_inv(e, Kn, Mi(e), 0, s);
          if ((!(pmin[1] > 0.0) || pmin[1] < 1e-14 * pmax[1]) && lane == 0) flag_bad(bad_element, Kn);
        }
        if (e + NGJW < E) load_packed(has_next ? Kn0 + e + NGJW : long(nelt), mnext);
      }
    }
    if (warp >= NGJW || NGJW == NWT) {
      const int w0 = NGJW == NWT ? warp : warp - NGJW, nw = NGJW == NWT ? NWT : NWT - NGJW;
      for (int tile = w0; tile < NLOW; tile += nw) {
        int mt = 0, rem = tile;
        while (rem > mt) { rem -= mt + 1; ++mt; }
        const int nt = rem;
        double z[E][2];
        int wbr[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          z[e][0] = z[e][1] = 0.0;
          wbr[e] = reinterpret_cast<const int*>(colb(e, cur) + 4 * MP)[mt * 8 + g];
        }
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
          const int k = kk * 4 + t;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double aw = (wbr[e] >= 0 && k < D3) ? __ldg(Wlm + wbr[e] + k * D2) : 0.0;
            dmma(z[e][0], z[e][1], aw, Zb(e)[k + (nt * 8 + g) * LD]);
          }
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          Yb(e)[tile * 64 + 2 * lane] = z[e][0];
          Yb(e)[tile * 64 + 2 * lane + 1] = z[e][1];
        }
      }
      if (factors) {
        for (int e = w0; e < nb; e += nw) {  // one warp per element: columns of V, then f
          double* F = factors + (K0 + e) * Dm::FACTORS + 2 * NS;
          for (int c = 0; c < M; ++c)
            for (int r = lane; r < D3; r += 32) F[r + c * D3] = Vb(e)[r + c * LD];
          for (int i = lane; i < D3; i += 32) F[D3 * M + i] = fv(e)[i];
        }
      }
    }
    __syncthreads();

    PHASE_MARK(batch, 3);
    // ---- P4: Vs = Si V (into Zb) | fs = Si f | next batch's geometry
    for (int task = warp; task < NTM * MT; task += NWT) {
      const int nt = task / MT, m = task % MT;
      const int c = nt * 8 + g, r = m * 8 + g, c0 = nt * 8 + 2 * t;
      double acc[E][2];
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e][0] = acc[e][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int k = kk * 4 + t;
#pragma unroll
        for (int e = 0; e < E; ++e) dmma(acc[e][0], acc[e][1], Sb(e)[r + k * LD], Vb(e)[k + c * LD]);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        Zb(e)[r + c0 * LD] = acc[e][0];
        Zb(e)[r + (c0 + 1) * LD] = acc[e][1];
      }
    }
    for (int idx = threadIdx.x; idx < nb * D3; idx += NT) {
      const int e = idx / D3, r = idx - (idx / D3) * D3;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D3; ++k) s += Sb(e)[r + k * LD] * fv(e)[k];
      fs(e)[r] = s;
    }
    if (has_next) load_geo_batch(Kn0, cur ^ 1);
    __syncthreads();
    if (has_next)
      for (int e = warp; e < E; e += NWT)
        if (Kn0 + e < nelt) build_columns<D2, D3, M, MP>(sgb(e, cur ^ 1), colb(e, cur ^ 1), lane);

    PHASE_MARK(batch, 4);
    // ---- P5: C = tauDD + (n_l1.n_l2) o (W Zp) - V^T Vs (lower tiles, mirrored) | Cf
    for (int tile = warp; tile < NLOW; tile += NWT) {
      int mt = 0, rem = tile;
      while (rem > mt) { rem -= mt + 1; ++mt; }
      const int nt = rem, r = mt * 8 + g;
      double v[E][2];
#pragma unroll
      for (int e = 0; e < E; ++e) v[e][0] = v[e][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int k = kk * 4 + t;
#pragma unroll
        for (int e = 0; e < E; ++e) dmma(v[e][0], v[e][1], Vb(e)[k + r * LD], Zb(e)[k + (nt * 8 + g) * LD]);
      }
      if (r < M) {
        const int l1 = r / D2;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (e >= nb) break;
          const double* sg = sgb(e, cur);
          const double* nsc = colb(e, cur);
          const double* Tc = nsc + 3 * MP;
          const double n1x = sg[10 + 3 * l1], n1y = sg[11 + 3 * l1], n1z = sg[12 + 3 * l1];
          double* Ck = Cout + (K0 + e) * M * M;
          const double z0 = Yb(e)[tile * 64 + 2 * lane], z1 = Yb(e)[tile * 64 + 2 * lane + 1];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = nt * 8 + 2 * t + h;
            if (c > r || c >= M) continue;
            const int l2 = c / D2;
            const double nn = n1x * nsc[c] + n1y * nsc[MP + c] + n1z * nsc[2 * MP + c];
            double val = nn * (h ? z1 : z0) - v[e][h];
            if (l1 == l2) val += Tc[c] * __ldg(tab.DD + (r - l1 * D2) + (c - l2 * D2) * D2);
            Ck[r + c * M] = val;
            if (c != r) Ck[c + r * M] = val;
          }
        }
      }
    }
    for (int idx = threadIdx.x; idx < nb * M; idx += NT) {
      const int e = idx / M, r = idx - (idx / M) * M;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D3; ++k) s += Vb(e)[k + r * LD] * fs(e)[k];
      Cfout[(K0 + e) * M + r] = s;
    }
    __syncthreads();
    PHASE_MARK(batch, 5);
    if (has_next) {
      load_Df(Kn0);
      cur ^= 1;
    }
    __syncthreads();
  }
}

}  // namespace hdgb
