// Device-side building blocks shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hdg_b200.h"

namespace hdgb {

// ------------------------------------------------------------ compile-time dims
__host__ __device__ constexpr int cdim3(int k) { return (k + 1) * (k + 2) * (k + 3) / 6; }
__host__ __device__ constexpr int cdim2(int k) { return (k + 1) * (k + 2) / 2; }
__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }
__host__ __device__ constexpr int cnq(int deg) { return (deg / 2 + 1) * (deg / 2 + 1) * (deg / 2 + 1); }
__host__ __device__ constexpr int cnqd(int deg) { return (deg / 2 + 1) * (deg / 2 + 1); }
// packed lower-triangle (column-major) index of (i >= j) in an n x n matrix
__host__ __device__ constexpr int sym_idx(int i, int j, int n) { return j * (2 * n - j + 1) / 2 + (i - j); }

// ------------------------------------------------------------------ tables
// One degree's reference-element tables in device memory (host_tables.cpp).
struct DevTab {
  int k, d3, d2, nq, nqd, nqp, nsym, nsymp, d3p;
  int nu;  // scalar-space dimension of the local solve: d3, or d3 - d2 for the BDM variant
  const double* bary;   // nq x 4
  const double* w;      // nq
  const double* P;      // nq x d3
  const double* Pd;     // 3 x (nq x d3)
  const double* Chat;   // 3 x (d3 x d3)
  const double* Shat;   // 9 x (d3 x d3)
  const double* Wlm;    // 24 x (d2 x d3), index 6*l + (mu-1)
  const double* PP;     // 4 x (d3 x d3)
  const double* DD;     // d2 x d2
  const double* tri_bary;  // nqd x 3
  const double* tri_w;     // nqd
  const double* Pface;     // 4 x (nqd x d3)
  const double* Dperm;     // 6 x (nqd x d2)
  const double* Asym;   // fragment-ordered [Wsym | PPsym]: nsymp x (nqp + 4)
  const double* Af;     // fragment-ordered P^T: d3p x nqp
  const double* ChatT;  // 3 x (d3 x d3), Chat transposed
  const double* WlmT;   // 24 x (d3 x d2), Wlm transposed
  const double* ShatP;  // 9 x d3(d3+1)/2, Shat packed lower (column-major)
  const double* Aconv;  // k <= 3: fragment-ordered [P_qi dP_qj/dxhat_#], d3^2 x 3 nqp (kernels_conv2.cuh)
};

// ------------------------------------------------------------------ fields
struct FieldDev {
  int kind;  // HDG_FIELD_*
  int nops;
  double value;
  const double* samples;  // nq x nelt (element's nodes contiguous)
  unsigned char ops[HDG_FIELD_MAX_OPS];
  double consts[HDG_FIELD_MAX_CONSTS];
};

// Postfix VM (opcodes in include/hdg_b200.h). Control flow is uniform across a
// warp (every lane runs the same program), so the switch never diverges.
__device__ __forceinline__ double run_program(const FieldDev& F, double x, double y, double z) {
  double st[HDG_FIELD_MAX_STACK];
  int sp = 0, ci = 0;
  for (int i = 0; i < F.nops; ++i) {
    switch (F.ops[i]) {
      case HDG_OP_X: st[sp++] = x; break;
      case HDG_OP_Y: st[sp++] = y; break;
      case HDG_OP_Z: st[sp++] = z; break;
      case HDG_OP_CONST: st[sp++] = F.consts[ci++]; break;
      case HDG_OP_ADD: --sp; st[sp - 1] = st[sp - 1] + st[sp]; break;
      case HDG_OP_SUB: --sp; st[sp - 1] = st[sp - 1] - st[sp]; break;
      case HDG_OP_MUL: --sp; st[sp - 1] = st[sp - 1] * st[sp]; break;
      case HDG_OP_DIV: --sp; st[sp - 1] = st[sp - 1] / st[sp]; break;
      case HDG_OP_NEG: st[sp - 1] = -st[sp - 1]; break;
      case HDG_OP_SIN: st[sp - 1] = sin(st[sp - 1]); break;
      case HDG_OP_COS: st[sp - 1] = cos(st[sp - 1]); break;
      case HDG_OP_EXP: st[sp - 1] = exp(st[sp - 1]); break;
      case HDG_OP_SQRT: st[sp - 1] = sqrt(st[sp - 1]); break;
      case HDG_OP_ABS: st[sp - 1] = fabs(st[sp - 1]); break;
      case HDG_OP_LT: --sp; st[sp - 1] = st[sp - 1] < st[sp] ? 1.0 : 0.0; break;
      case HDG_OP_POW: --sp; st[sp - 1] = pow(st[sp - 1], st[sp]); break;
      default: break;
    }
  }
  return st[0];
}

// Value of field F at quadrature node q of element K (physical point x,y,z).
__device__ __forceinline__ double eval_field(const FieldDev& F, double x, double y, double z,
                                             int q, long K, int nq) {
  if (F.kind == HDG_FIELD_CONST) return F.value;
  if (F.kind == HDG_FIELD_SAMPLED) return __ldg(F.samples + K * nq + q);
  return run_program(F, x, y, z);
}

// ------------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ------------------------------------------------------ TMA bulk stores
// Shared -> global bulk copy (16-byte aligned addresses, size a multiple of
// 16), tracked by the issuing thread's bulk async-group.
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, unsigned bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(ssrc));
  asm volatile(
      "fence.proxy.async.shared::cta;\n"
      "cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
      "cp.async.bulk.commit_group;\n" ::"l"(gdst), "r"(s), "r"(bytes)
      : "memory");
}
// Wait until the issuing thread's bulk stores have finished reading shared memory.
__device__ __forceinline__ void bulk_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

// ------------------------------------------------------------------ DMMA
// D(8x8) += A(8x4, row) * B(4x8, col), fp64 tensor-core MMA (SASS DMMA.8x8x4).
// Lane layout: a = A[g][t], b = B[t][g], c = {C[g][2t], C[g][2t+1]}, g = lane/4, t = lane%4.
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Named barrier for a team of `nthreads` threads (ids 1..15; 0 is __syncthreads).
__device__ __forceinline__ void team_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// Lowest singular element (reference reports the first detected; with one
// thread that is the lowest, local_solver.cpp:89-98).
__device__ __forceinline__ void flag_bad(long long* bad, long long K) {
  atomicMin(reinterpret_cast<unsigned long long*>(bad), static_cast<unsigned long long>(K));
}

// Pivot statistics of an element's two structured inverses (which = 0: M,
// 1: the Schur complement S): extreme |pivots|, pmin = 0 if a pivot vanished
// or is not finite. kernels_rescue.cuh screens them and re-runs the
// reference's LU path (local_solver.cpp:50-57, :71-100) where they are too
// far apart to vouch for the element.
__device__ __forceinline__ void store_pivstat(double* ps, long long K, int which, double pmin, double pmax) {
  reinterpret_cast<double2*>(ps)[2 * K + which] = make_double2(pmin, pmax);
}

}  // namespace hdgb
