// Warp-register sweep inverse of a small SPD matrix (used by the v3
// condensation kernel, kernels_condense3.cuh). Self-contained: no includes.
#pragma once

#ifndef HDG_GJ_EARLY
#define HDG_GJ_EARLY 1
#endif

// 1/x to full double precision: MUFU reciprocal seed + two Newton steps.
__device__ __forceinline__ double gj_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// Inverse of the symmetric N x N matrix held by a warp (lane c owns column c
// in a[]) by the symmetric sweep operator with 2 x 2 pivots (no pivoting;
// pmin / pmax return the extreme |LDL^T pivots|, 0 for a vanished or
// non-finite one, for the rescue screen of kernels_rescue.cuh). The pivot block columns are
// exchanged through `stage` (2 x 64 doubles, 16-byte aligned). The pivot
// lanes take their diagonal entry minus one into w = P^-1 a_K, which yields
// their special update weights (rows of I - P^-1) without selects, and each
// lane records its own pivot (one warp reduction at the end).
// One 2 x 2 pivot step (pivot rows k, k + 1; k even, a compile-time value
// once the caller's loop is unrolled) of the sweep below. `piv` collects the
// lane's pivot (gj_sweep_finish reduces it).
template <int N>
__device__ __forceinline__ void gj_sweep_step(double (&a)[N], double* stage, int lane, int k, double& piv) {
  double* st = stage + ((k >> 1) & 1) * 64;
  if (lane < N) {
    st[lane] = a[k];
    st[32 + lane] = a[k + 1];
  }
#if HDG_GJ_EARLY
  // barrier right after the stage stores: the pivot block, the next pivot
  // rows and the update's stage loads all issue under the reciprocal chain
  __syncwarp();
  const double2 pk0 = *reinterpret_cast<const double2*>(st + k);       // a[k] of lanes k, k + 1
  const double2 pk1 = *reinterpret_cast<const double2*>(st + 32 + k);  // a[k + 1] of lanes k, k + 1
  const double p00 = pk0.x, p01 = pk1.x, p11 = pk1.y;
  double n0x = 0.0, n0y = 0.0, n1x = 0.0, n1y = 0.0;
  if (k + 2 < N) {
    n0x = st[k + 2];
    n1x = st[32 + k + 2];
    if (k + 3 < N) {
      n0y = st[k + 3];
      n1y = st[32 + k + 3];
    }
  }
#else
  const double p00 = __shfl_sync(0xffffffffu, a[k], k);
  const double p01 = __shfl_sync(0xffffffffu, a[k + 1], k);
  const double p11 = __shfl_sync(0xffffffffu, a[k + 1], k + 1);
  // next pivot pair's rows of the stage by shuffle: keeps shared memory off
  // the step-to-step dependency chain
  double n0x = 0.0, n0y = 0.0, n1x = 0.0, n1y = 0.0;
  if (k + 2 < N) {
    n0x = __shfl_sync(0xffffffffu, a[k], k + 2);
    n1x = __shfl_sync(0xffffffffu, a[k + 1], k + 2);
    if (k + 3 < N) {
      n0y = __shfl_sync(0xffffffffu, a[k], k + 3);
      n1y = __shfl_sync(0xffffffffu, a[k + 1], k + 3);
    }
  }
#endif
  const double det = fma(p00, p11, -p01 * p01);
  const bool m0 = lane == k, m1 = lane == k + 1;
  const double ak0 = m0 ? a[k] - 1.0 : a[k];
  const double ak1 = m1 ? a[k + 1] - 1.0 : a[k + 1];
  // w = P^-1 a_K = adj(P) a_K / det: the adjugate products and the next
  // pivot rows' contractions overlap the reciprocal, one FMA follows it
  const double u0 = fma(p11, ak0, -p01 * ak1);
  const double u1 = fma(p00, ak1, -p01 * ak0);
  double s0 = 0.0, s1 = 0.0;
  if (k + 2 < N) {
    s0 = fma(n0x, u0, n1x * u1);
    if (k + 3 < N) s1 = fma(n0y, u0, n1y * u1);
  }
  const double id = gj_rcp(det);
  if (k + 2 < N) {
    a[k + 2] = fma(-s0, id, a[k + 2]);
    if (k + 3 < N) a[k + 3] = fma(-s1, id, a[k + 3]);
  }
  const double w0 = u0 * id, w1 = u1 * id;
  if (m0) piv = p00;
  if (m1) piv = p00 * id;
#if !HDG_GJ_EARLY
  __syncwarp();
#endif
#pragma unroll
  for (int i0 = 0; i0 < N; i0 += 2) {
    if (i0 == k || i0 == k + 2) continue;
    const double2 v0 = *reinterpret_cast<const double2*>(st + i0);
    const double2 v1 = *reinterpret_cast<const double2*>(st + 32 + i0);
    a[i0] = fma(-v0.x, w0, fma(-v1.x, w1, a[i0]));
    if (i0 + 1 < N) a[i0 + 1] = fma(-v0.y, w0, fma(-v1.y, w1, a[i0 + 1]));
  }
  a[k] = m0 ? w0 - 1.0 : w0;
  a[k + 1] = m1 ? w1 - 1.0 : w1;
}

// The trailing scalar pivot (odd N), the sign flip and the pivot reduction:
// pmin / pmax return the extreme |LDL^T pivots| (0 for a vanished or
// non-finite one).
template <int N, bool REDUCE = true>
__device__ __forceinline__ void gj_sweep_finish(double (&a)[N], double* stage, int lane, double& piv,
                                                double& pmin, double& pmax) {
  if (N % 2) {  // trailing scalar pivot
    constexpr int k = N - 1;
    double* st = stage + (((k >> 1)) & 1) * 64;
    if (lane < N) st[lane] = a[k];
    const double p = __shfl_sync(0xffffffffu, a[k], k);
    const double ip = gj_rcp(p);
    const bool me = lane == k;
    if (me) piv = p;
    const double w = (me ? a[k] - 1.0 : a[k]) * ip;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < k; ++i) a[i] = fma(-st[i], w, a[i]);
    a[k] = me ? w - 1.0 : w;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = -a[i];
  // pivots: even lanes hold p00, odd lanes 1/d1 (the trailing scalar pivot as
  // is); reduced as |d|, a vanished or non-finite pivot as 0
  double d = fabs((lane & 1) && lane < N - (N % 2) ? 1.0 / piv : piv);
  if (!(d <= 1.79e308)) d = 0.0;
  double mn = lane < N ? d : 1e300, mx = lane < N ? d : 0.0;
  if (REDUCE) {  // (else the caller reduces this lane's pivot later, off the critical path)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
  }
  pmin = fmin(pmin, mn);
  pmax = fmax(pmax, mx);
}

// Inverse of the symmetric N x N matrix held by a warp (lane c owns column c
// in a[]) by the symmetric sweep operator with 2 x 2 pivots (no pivoting;
// pmin / pmax return the extreme |LDL^T pivots|, 0 for a vanished or
// non-finite one, for the rescue screen of kernels_rescue.cuh). The pivot block columns are
// exchanged through `stage` (2 x 64 doubles, 16-byte aligned). The pivot
// lanes take their diagonal entry minus one into w = P^-1 a_K, which yields
// their special update weights (rows of I - P^-1) without selects, and each
// lane records its own pivot (one warp reduction at the end).
template <int N>
__device__ __forceinline__ void gj_sweep_inverse(double (&a)[N], double* stage, int lane, double& pmin,
                                                 double& pmax) {
  double piv = 1.0;  // lane c: Cholesky pivot c (odd c: its reciprocal until the end)
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) gj_sweep_step<N>(a, stage, lane, k, piv);
  gj_sweep_finish<N>(a, stage, lane, piv, pmin, pmax);
}

// Sweep inverse of the leading N x N block held by a W-lane segment of the
// warp (lane c < N of the segment owns column c in a[0..N-1]; rows N..R-1 of
// a[] are left untouched). Same algebra as gj_sweep_inverse; shuffles stay
// inside the segment; `stage` is the segment's own 2 x 64 doubles. pmin/pmax
// reduce the |pivots| over the segment (a vanished or non-finite one as 0).
template <int N, int W, int R>
__device__ __forceinline__ void gj_sweep_seg(double (&a)[R], double* stage, int c, double& pmin, double& pmax) {
  static_assert(N % 2 == 0 && N <= W && N <= R, "even N on one segment");
  constexpr unsigned FULL = 0xffffffffu;
  double piv = 1.0;
#pragma unroll
  for (int k = 0; k + 1 < N; k += 2) {
    double* st = stage + ((k >> 1) & 1) * 64;
    if (c < N) {
      st[c] = a[k];
      st[32 + c] = a[k + 1];
    }
#if HDG_GJ_EARLY
    __syncwarp();
    const double2 pk0 = *reinterpret_cast<const double2*>(st + k);
    const double2 pk1 = *reinterpret_cast<const double2*>(st + 32 + k);
    const double p00 = pk0.x, p01 = pk1.x, p11 = pk1.y;
    double n0x = 0.0, n0y = 0.0, n1x = 0.0, n1y = 0.0;
    if (k + 2 < N) {
      const double2 q0 = *reinterpret_cast<const double2*>(st + k + 2);
      const double2 q1 = *reinterpret_cast<const double2*>(st + 32 + k + 2);
      n0x = q0.x, n0y = q0.y, n1x = q1.x, n1y = q1.y;
    }
#else
    const double p00 = __shfl_sync(FULL, a[k], k, W);
    const double p01 = __shfl_sync(FULL, a[k + 1], k, W);
    const double p11 = __shfl_sync(FULL, a[k + 1], k + 1, W);
    double n0x = 0.0, n0y = 0.0, n1x = 0.0, n1y = 0.0;
    if (k + 2 < N) {
      n0x = __shfl_sync(FULL, a[k], k + 2, W);
      n1x = __shfl_sync(FULL, a[k + 1], k + 2, W);
      n0y = __shfl_sync(FULL, a[k], k + 3, W);
      n1y = __shfl_sync(FULL, a[k + 1], k + 3, W);
    }
#endif
    const double det = fma(p00, p11, -p01 * p01);
    const bool m0 = c == k, m1 = c == k + 1;
    const double ak0 = m0 ? a[k] - 1.0 : a[k];
    const double ak1 = m1 ? a[k + 1] - 1.0 : a[k + 1];
    const double u0 = fma(p11, ak0, -p01 * ak1);
    const double u1 = fma(p00, ak1, -p01 * ak0);
    double s0 = 0.0, s1 = 0.0;
    if (k + 2 < N) {
      s0 = fma(n0x, u0, n1x * u1);
      s1 = fma(n0y, u0, n1y * u1);
    }
    const double id = gj_rcp(det);
    if (k + 2 < N) {
      a[k + 2] = fma(-s0, id, a[k + 2]);
      a[k + 3] = fma(-s1, id, a[k + 3]);
    }
    const double w0 = u0 * id, w1 = u1 * id;
    if (m0) piv = p00;
    if (m1) piv = p00 * id;
#if !HDG_GJ_EARLY
    __syncwarp();
#endif
#pragma unroll
    for (int i0 = 0; i0 < N; i0 += 2) {
      if (i0 == k || i0 == k + 2) continue;
      const double2 v0 = *reinterpret_cast<const double2*>(st + i0);
      const double2 v1 = *reinterpret_cast<const double2*>(st + 32 + i0);
      a[i0] = fma(-v0.x, w0, fma(-v1.x, w1, a[i0]));
      a[i0 + 1] = fma(-v0.y, w0, fma(-v1.y, w1, a[i0 + 1]));
    }
    a[k] = m0 ? w0 - 1.0 : w0;
    a[k + 1] = m1 ? w1 - 1.0 : w1;
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = -a[i];
  double d = fabs((c & 1) && c < N ? 1.0 / piv : piv);
  if (!(d <= 1.79e308)) d = 0.0;  // vanished / non-finite pivot
  double mn = c < N ? d : 1e300, mx = c < N ? d : 0.0;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(FULL, mn, o));
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  }
  pmin = fmin(pmin, mn);
  pmax = fmax(pmax, mx);
}
