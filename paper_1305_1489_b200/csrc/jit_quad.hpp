// NVRTC specialisation of the K2 node-build kernel (jit_quad.cpp).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <string>
#include <unordered_map>

#include "../../include/hdg_b200.h"

namespace hdgb {
// Field programs -> straight-line device code (shared temporaries across the
// fields of one kernel): emit() returns the expression naming the field's
// value; stmts() the declarations to place before its first use.
class FieldEmitter {
 public:
  std::string emit(const hdg_field& f, const char* sample_ptr);
  const std::string& stmts() const { return stmts_; }

 private:
  std::string stmts_;
  std::unordered_map<std::string, std::string> memo_;
  int ntemp_ = 0;
};
#ifndef HDG_QUAD_THREADS16
#define HDG_QUAD_THREADS16 1024
#endif
// Block size of the JIT node build (measured): EB = 32 runs two 384-thread CTAs per SM;
// EB = 16 (k >= 4, one CTA per SM by shared memory) one 1024-thread CTA.
#ifndef HDG_QUAD_THREADS32
#define HDG_QUAD_THREADS32 384
#endif
// (k <= 2, fewer than 100 nodes: 256 threads, measured faster at C4)
inline int jit_quad_threads(int eb, int nqp) {
  return eb == 16 ? HDG_QUAD_THREADS16 : (nqp >= 100 ? HDG_QUAD_THREADS32 : 256);
}
// Compiled (cached per source and CUDA context) kernel for these fields and EB
// elements per CTA with the block size it was compiled for; fn == nullptr with
// *err set on failure.
struct JitKernel {
  CUfunction fn = nullptr;
  int threads = 0;
};
JitKernel jit_quad_kernel(const hdg_field& kap, const hdg_field& c, const hdg_field& f, int eb, int nqp,
                          std::string* err);
// Kernel sampling a PROGRAM field at every element node (SAMPLED layout), or nullptr.
// A program field sampled at every point of a table (out[K * npoints + p]).
CUfunction jit_sample_kernel(const hdg_field& f, std::string* err);
// w_q / f(x_q) at every element node (out[K * nq + q]; w: the rule's weights).
CUfunction jit_sample_wdiv_kernel(const hdg_field& f, std::string* err);
// The program fields among f[0..2] sampled in one pass at every point of a
// table (out_h[K * npoints + p]; outputs of non-program fields untouched).
CUfunction jit_sample3_kernel(const hdg_field* const f[3], std::string* err);
bool launch_quad_jit(CUfunction fn, cudaStream_t stream, int grid, int block, size_t smem, void** args,
                     std::string* err);
}  // namespace hdgb
