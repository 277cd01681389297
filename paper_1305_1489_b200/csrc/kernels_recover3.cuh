// K5 v3 (k = 1..3): gather + local recovery from the condensation cache,
// HBM-streaming form.
//
// Per element the cache record {M^-1 (packed lower), Vs = S^-1 V (d3 x m),
// fs = S^-1 f} is read exactly once (k=3: 8,240 B), so the kernel is a stream
// over the cache.
// Each warp owns a chain of elements (persistent grid) and double-buffers the
// records in shared memory with 1-D TMA bulk copies (cp.async.bulk, completion
// on a per-buffer mbarrier): the copies of the next kRec3Bufs-1 elements of the
// chain are in flight while element K is recovered. The skeleton gather (lambda) and the geometry record
// of the next element are prefetched into registers one iteration ahead.
//
// Algebra as recover2_kernel (local_solver.cpp:102-135 restated on the
// condensed factors): u = S^-1 (f + V lambda), q_s = M^-1 (r_s) with
// r_s = sum_# a(s,#) Chat_#^T-contraction of u - sum_l n_l,s W_l lambda_l.
#pragma once

#include "kernels_condense2.cuh"

namespace hdgb {

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}

// Arm the barrier for `bytes` of async-proxy data and start the bulk copy.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "fence.proxy.async.shared::cta;\n"
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%2], %3;\n"
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %3, [%2];\n" ::"r"(d),
      "l"(src), "r"(b), "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned b = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}

// warps per CTA (one CTA per SM) and cache records in flight per warp
template <int K_> struct Rec3Cfg { static constexpr int WARPS = 16, BUFS = 2; };
template <> struct Rec3Cfg<3> { static constexpr int WARPS = 8, BUFS = 2; };

template <int K_>
struct Rec3Dims {
  static constexpr int D3 = cdim3(K_), D2 = cdim2(K_), M = 4 * cdim2(K_), NS = D3 * (D3 + 1) / 2;
  static constexpr int FACTORS = round_up(NS + D3 * M + D3, 2);  // {M^-1 packed, Vs, fs}
  static constexpr int REC = round_up(FACTORS, 2);       // 16-byte multiple
  static constexpr int SCR = round_up(M, 2) + 2 * 32 + 3 * D3 + 32;  // lambda, t, u, r_s, geometry
  static constexpr int PER_WARP = Rec3Cfg<K_>::BUFS * REC + SCR;
  static constexpr int D2P = round_up(D2, 2);
  // per CTA, row-pair interleaved: [h][i / 2][j][i % 2] (Chat^T), [l, perm][i / 2][j][i % 2] (W^T, rows
  // padded to D2P), so that lane j reads rows i, i + 1 of its column with one 16-byte load
  static constexpr int TABLES = 3 * D3 * D3 + 24 * D2P * D3;
  static_assert((FACTORS * 8) % 16 == 0, "cache record must be a 16-byte multiple for cp.async.bulk");
};

template <int K_>
__global__ void __launch_bounds__(Rec3Cfg<K_>::WARPS * 32, 1)
recover3_kernel(DevTab tab, int nelt, GeoDev geo, const int* __restrict__ facebyele,
                const double* __restrict__ factors, const double* __restrict__ uhat,
                double* __restrict__ qx, double* __restrict__ qy, double* __restrict__ qz,
                double* __restrict__ uout) {
  using Rd = Rec3Dims<K_>;
  constexpr int kRec3Warps = Rec3Cfg<K_>::WARPS, kRec3Bufs = Rec3Cfg<K_>::BUFS;
  constexpr int D3 = Rd::D3, D2 = Rd::D2, M = Rd::M, NS = Rd::NS, F = Rd::FACTORS;
  static_assert(M <= 64 && D3 <= 32, "one warp per element: lambda in 2 registers, u in 1");
  extern __shared__ __align__(16) double rsm[];
  __shared__ unsigned long long bars[kRec3Warps][kRec3Bufs];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* buf = rsm + warp * Rd::PER_WARP;
  double* lam = buf + kRec3Bufs * Rd::REC;
  double* tv = lam + round_up(M, 2);
  double* uu = tv + 32;
  double* rs = uu + 32;
  double* sg = rs + 3 * D3;
  constexpr int D2P = Rd::D2P;
  static_assert(D3 % 2 == 0 && M % 2 == 0, "row pairs");
  double* ChT = rsm + kRec3Warps * Rd::PER_WARP;  // CTA copies of Chat^T, Wlm^T (row-pair interleaved)
  double* WT = ChT + 3 * D3 * D3;
  for (int x = threadIdx.x; x < 3 * D3 * D3; x += blockDim.x) {
    const int h = x / (D3 * D3), r = x - h * D3 * D3, i = r / D3, j = r - i * D3;
    ChT[h * D3 * D3 + (i >> 1) * 2 * D3 + 2 * j + (i & 1)] = tab.ChatT[x];
  }
  for (int x = threadIdx.x; x < 24 * D2P * D3; x += blockDim.x) {
    const int b = x / (D2P * D3), r = x - b * D2P * D3, i = r / D3, j = r - i * D3;
    WT[b * D2P * D3 + (i >> 1) * 2 * D3 + 2 * j + (i & 1)] = i < D2 ? tab.WlmT[(b * D2 + i) * D3 + j] : 0.0;
  }
  __syncthreads();
  if (lane == 0) {
    for (int i = 0; i < kRec3Bufs; ++i) mbar_init(&bars[warp][i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();

  const long stride = long(gridDim.x) * kRec3Warps;
  long K = long(blockIdx.x) * kRec3Warps + warp;
  // Register prefetch, software-pipelined so no load is consumed in the
  // iteration that issues it: face ids two elements ahead, lambda and the
  // geometry record one element ahead. Lane i < m owns lambda entry i (and
  // i + 32), lane i < 30 geometry entry i.
  auto face_ids = [&](long Ke, int& f0, int& f1) {
    f0 = f1 = -1;
    if (Ke >= nelt) return;
    if (lane < M) f0 = facebyele[long(lane / D2) * nelt + Ke];
    if (lane + 32 < M) f1 = facebyele[long((lane + 32) / D2) * nelt + Ke];
  };
  auto traces = [&](int f0, int f1, double& l0, double& l1) {
    l0 = f0 >= 0 ? uhat[long(f0) * D2 + lane % D2] : 0.0;
    l1 = f1 >= 0 ? uhat[long(f1) * D2 + (lane + 32) % D2] : 0.0;
  };
  auto geometry = [&](long Ke, double& gv, int& gp) {
    gv = 0.0;
    gp = 0;
    if (Ke >= nelt || lane >= 30) return;
    if (lane == 0) gv = geo.volume[Ke];
    else if (lane < 10) gv = geo.piola[long(lane - 1) * nelt + Ke];
    else if (lane < 22) gv = geo.normals[long(lane - 10) * nelt + Ke];
    else if (lane < 26) gv = geo.T[long(lane - 22) * nelt + Ke];
    else gp = geo.perm[long(lane - 26) * nelt + Ke];
  };
  int f0, f1, fn0, fn1, gp;
  double l0, l1, gv;
  face_ids(K, f0, f1);
  traces(f0, f1, l0, l1);
  geometry(K, gv, gp);
  face_ids(K + stride, fn0, fn1);
  for (int i = 0; i + 1 < kRec3Bufs; ++i) {
    const long Ki = K + i * stride;
    if (Ki < nelt && lane == 0) bulk_load(buf + i * Rd::REC, factors + Ki * F, F * 8, &bars[warp][i]);
  }
  unsigned phase = 0u;  // parity bits, one per buffer
  int b = 0;
  for (; K < nelt; K += stride, b = b + 1 == kRec3Bufs ? 0 : b + 1) {
    const long Kn = K + stride;
    {
      const long Kp = K + (kRec3Bufs - 1) * stride;  // refill the buffer freed last iteration
      const int bp = (b + kRec3Bufs - 1) % kRec3Bufs;
      if (Kp < nelt && lane == 0) bulk_load(buf + bp * Rd::REC, factors + Kp * F, F * 8, &bars[warp][bp]);
    }
    if (lane < M) lam[lane] = l0;
    if (lane + 32 < M) lam[lane + 32] = l1;
    if (lane < 30) sg[lane] = lane < 26 ? gv : double(gp);
    traces(fn0, fn1, l0, l1);  // element Kn
    geometry(Kn, gv, gp);
    face_ids(Kn + stride, fn0, fn1);
    __syncwarp();
    mbar_wait(&bars[warp][b], (phase >> b) & 1u);
    phase ^= 1u << b;
    const double* Mi = buf + b * Rd::REC;
    const double* Vs = Mi + NS;
    const double* fs = Vs + D3 * M;

    if (lane < D3) {  // u = S^-1 (f + V lambda) = fs + Vs lambda
      double s0 = fs[lane], s1 = 0.0;
#pragma unroll
      for (int c = 0; c < M; c += 2) {
        const double2 lc = *reinterpret_cast<const double2*>(lam + c);  // broadcast pair
        s0 = fma(Vs[lane + c * D3], lc.x, s0);
        s1 = fma(Vs[lane + (c + 1) * D3], lc.y, s1);
      }
      const double u = s0 + s1;
      uu[lane] = u;
      uout[K * D3 + lane] = u;
    }
    __syncwarp();
    if (lane < D3) {  // r_s(j) = sum_# a(s,#) (Chat_# u)(j) - sum_l n_l,s (W_l lambda_l)(j)
      const int j = lane;
      double p[3] = {0.0, 0.0, 0.0}, p1[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int i = 0; i < D3; i += 2) {
        const double2 ui = *reinterpret_cast<const double2*>(uu + i);
#pragma unroll
        for (int h = 0; h < 3; ++h) {
          const double2 c = *reinterpret_cast<const double2*>(ChT + h * D3 * D3 + i * D3 + 2 * j);
          p[h] = fma(c.x, ui.x, p[h]);
          p1[h] = fma(c.y, ui.y, p1[h]);
        }
      }
#pragma unroll
      for (int h = 0; h < 3; ++h) p[h] += p1[h];
      double w[4];
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        const double* W = WT + (6 * l + int(sg[26 + l]) - 1) * D2P * D3 + 2 * j;
        double a0 = 0.0, a1 = 0.0;
#pragma unroll
        for (int i = 0; i < D2P; i += 2) {
          const double2 c = *reinterpret_cast<const double2*>(W + i * D3);
          if constexpr (D2 % 2 == 0) {
            const double2 li = *reinterpret_cast<const double2*>(lam + l * D2 + i);
            a0 = fma(c.x, li.x, a0);
            a1 = fma(c.y, li.y, a1);
          } else {
            a0 = fma(c.x, lam[l * D2 + i], a0);
            if (i + 1 < D2) a1 = fma(c.y, lam[l * D2 + i + 1], a1);
          }
        }
        w[l] = a0 + a1;
      }
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        double r = sg[1 + 3 * s] * p[0] + sg[2 + 3 * s] * p[1] + sg[3 + 3 * s] * p[2];
#pragma unroll
        for (int l = 0; l < 4; ++l) r -= sg[10 + 3 * l + s] * w[l];
        rs[s * D3 + j] = r;
      }
    }
    __syncwarp();
    if (lane < D3) {  // q_s = M^-1 r_s, s = x, y, z (one pass over row `lane` of M^-1)
      const int i = lane;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0;
#pragma unroll
      for (int j = 0; j < D3; j += 2) {
        const double m0 = Mi[j >= i ? sym_idx(j, i, D3) : sym_idx(i, j, D3)];
        const double m1 = Mi[j + 1 >= i ? sym_idx(j + 1, i, D3) : sym_idx(i, j + 1, D3)];
        const double2 r0 = *reinterpret_cast<const double2*>(rs + j);
        const double2 r1 = *reinterpret_cast<const double2*>(rs + D3 + j);
        const double2 r2 = *reinterpret_cast<const double2*>(rs + 2 * D3 + j);
        a0 = fma(m1, r0.y, fma(m0, r0.x, a0));
        a1 = fma(m1, r1.y, fma(m0, r1.x, a1));
        a2 = fma(m1, r2.y, fma(m0, r2.x, a2));
      }
      qx[K * D3 + i] = a0;
      qy[K * D3 + i] = a1;
      qz[K * D3 + i] = a2;
    }
    __syncwarp();  // buffer b and the scratch are reused next
  }
}

// K5 v5 (k = 4, 5): the cache record of one element (k=5: 63.6 KB) per CTA
// iteration, one TMA bulk copy into shared memory; all 256 threads recover
// from it (row-parallel matrix-vector products, 4 threads per row with a
// shuffle reduction). Three CTAs per SM keep three records in flight.
constexpr int kRec5Threads = 256;
template <int K_>
struct Rec5Dims {
  static constexpr int D3 = cdim3(K_), D2 = cdim2(K_), M = 4 * cdim2(K_), NS = D3 * (D3 + 1) / 2;
  static constexpr int FACTORS = round_up(NS + D3 * M + D3, 2);  // {M^-1 packed, Vs, fs}
  static constexpr int REC = round_up(FACTORS, 2);
  static constexpr int SCR = round_up(M, 2) + 3 * D3 + 7 * D3 + 3 * D3 + 32;  // lambda, t/u, p|w, r_s, geometry
  static constexpr int TOTAL = REC + SCR;
  static constexpr bool BULK = FACTORS % 2 == 0;  // 16-byte records: one TMA bulk copy (else cp.async)
};

template <int K_>
__global__ void __launch_bounds__(kRec5Threads)
recover5_kernel(DevTab tab, int nelt, GeoDev geo, const int* __restrict__ facebyele,
                const double* __restrict__ factors, const double* __restrict__ uhat,
                double* __restrict__ qx, double* __restrict__ qy, double* __restrict__ qz,
                double* __restrict__ uout) {
  using Rd = Rec5Dims<K_>;
  constexpr int D3 = Rd::D3, D2 = Rd::D2, M = Rd::M, NS = Rd::NS, F = Rd::FACTORS;
  static_assert(4 * D3 <= kRec5Threads, "four threads per row");
  extern __shared__ __align__(16) double r5[];
  __shared__ unsigned long long bar;
  double* rec = r5;
  double* lam = r5 + Rd::REC;
  double* tv = lam + round_up(M, 2);
  double* uu = tv + D3;
  double* pw = uu + 2 * D3;  // p_# (3 D3) then w_l (4 D3)
  double* rs = pw + 7 * D3;  // r_s (3 D3)
  double* sg = rs + 3 * D3;
  const double* Mi = rec;
  const double* Vs = rec + NS;
  const double* fs = Vs + D3 * M;
  const int tid = threadIdx.x, row = tid >> 2, part = tid & 3;
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  unsigned phase = 0u;
  for (long K = blockIdx.x; K < nelt; K += gridDim.x) {
    if constexpr (Rd::BULK) {
      if (tid == 0) bulk_load(rec, factors + K * F, F * 8, &bar);
    } else {
      for (int i = tid; i < F; i += kRec5Threads) cp_async8(rec + i, factors + K * F + i);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
    }
    for (int i = tid; i < M; i += kRec5Threads) {
      const int l = i / D2;
      lam[i] = uhat[long(facebyele[long(l) * nelt + K]) * D2 + (i - l * D2)];
    }
    if (tid < 30) {
      double v;
      if (tid == 0) v = geo.volume[K];
      else if (tid < 10) v = geo.piola[long(tid - 1) * nelt + K];
      else if (tid < 22) v = geo.normals[long(tid - 10) * nelt + K];
      else if (tid < 26) v = geo.T[long(tid - 22) * nelt + K];
      else v = double(geo.perm[long(tid - 26) * nelt + K]);
      sg[tid] = v;
    }
    if constexpr (Rd::BULK) {
      mbar_wait(&bar, phase);
      phase ^= 1u;
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    // u = S^-1 (f + V lambda) = fs + Vs lambda
    double s = 0.0;
    if (row < D3) {
      for (int c = part; c < M; c += 4) s = fma(Vs[row + c * D3], lam[c], s);
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    if (row < D3 && part == 0) {
      uu[row] = fs[row] + s;
      uout[K * D3 + row] = fs[row] + s;
    }
    __syncthreads();
    // p_#(j) = (Chat_# u)(j) over the rows of Chat_#^T, w_l(j) = (W_l lambda_l)(j)
    for (int it = tid; it < 7 * D3; it += kRec5Threads) {
      const int h = it / D3, j = it - h * D3;
      double acc = 0.0;
      if (h < 3) {
        const double* C = tab.ChatT + h * D3 * D3 + j;
        for (int i = 0; i < D3; ++i) acc = fma(__ldg(C + i * D3), uu[i], acc);
      } else {
        const int l = h - 3;
        const double* W = tab.WlmT + (6 * l + int(sg[26 + l]) - 1) * D2 * D3 + j;
        for (int i = 0; i < D2; ++i) acc = fma(__ldg(W + i * D3), lam[l * D2 + i], acc);
      }
      pw[it] = acc;
    }
    __syncthreads();
    for (int it = tid; it < 3 * D3; it += kRec5Threads) {
      const int sd = it / D3, j = it - sd * D3;
      double r = sg[1 + 3 * sd] * pw[j] + sg[2 + 3 * sd] * pw[D3 + j] + sg[3 + 3 * sd] * pw[2 * D3 + j];
#pragma unroll
      for (int l = 0; l < 4; ++l) r -= sg[10 + 3 * l + sd] * pw[(3 + l) * D3 + j];
      rs[it] = r;
    }
    __syncthreads();
    // q_s = M^-1 r_s
    double a0 = 0.0, a1 = 0.0, a2 = 0.0;
    if (row < D3) {
      for (int j = part; j < D3; j += 4) {
        const double m = Mi[j >= row ? sym_idx(j, row, D3) : sym_idx(row, j, D3)];
        a0 = fma(m, rs[j], a0);
        a1 = fma(m, rs[D3 + j], a1);
        a2 = fma(m, rs[2 * D3 + j], a2);
      }
    }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    if (row < D3 && part == 0) {
      qx[K * D3 + row] = a0;
      qy[K * D3 + row] = a1;
      qz[K * D3 + row] = a2;
    }
    __syncthreads();  // the record buffer is refilled next
  }
}

}  // namespace hdgb
