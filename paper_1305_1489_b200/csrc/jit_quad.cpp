// Runtime specialisation of K2 for coefficient programs (NVRTC, sm_100a).
//
// The reference evaluates its coefficient callbacks on the node arrays inside
// build_element_matrices (element_matrices.cpp:94-109, :84-92). Interpreting a
// field program per node is dispatch-bound on the GPU, so K2 is compiled at
// run time with the three field expressions inlined as straight-line device
// code; compiled kernels are cached per source text. If NVRTC or the driver
// module loader fails, the caller keeps using the interpreted kernel (same
// device path, slower) and the failure text is kept for inspection.
#include <cuda.h>
#include <nvrtc.h>

#include <cmath>
#include <cstdio>
#include <mutex>
#include <sstream>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/hdg_b200.h"
#include "jit_quad.hpp"

#ifndef HDG_QUAD_MINB32
#define HDG_QUAD_MINB32 "2"  // EB = 32: two CTAs per SM must fit the registers
#endif
#ifndef HDG_QUAD_UNROLL
#define HDG_QUAD_UNROLL 8  // k-steps of the node GEMM unrolled (A fragments in flight)
#endif

namespace hdgb {

namespace {

const char* kQuadSource = R"CUDA(
// JIT: K2 node build with inlined coefficient fields (see kernels_local.cuh quad_build_kernel).
// EB (elements per CTA, a multiple of 8), QUAD_THREADS (the block size) and
// QUAD_MINB (CTAs per SM the registers must allow) are defined by the host
// before this text
#define LDB (EB + 4)
#define NTI (EB / 8)
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
extern "C" __global__ void __launch_bounds__(QUAD_THREADS, QUAD_MINB)
quad_build_jit(int nelt, int nq, int nqp, int nsym, int nsymp, int d3, int d3p,
               const double* __restrict__ bary, const double* __restrict__ wq,
               const double* __restrict__ Asym, const double* __restrict__ Af,
               const double* __restrict__ vol, const double* __restrict__ T,
               const double* __restrict__ V, const double* __restrict__ sk,
               const double* __restrict__ sc, const double* __restrict__ sf,
               double* __restrict__ Msym, double* __restrict__ Dsym, double* __restrict__ fvec) {
  extern __shared__ double smem[];
  const int rows = nqp + 4;
  double* Bk = smem;
  double* Bc = Bk + rows * LDB;
  double* Bf = Bc + rows * LDB;
  const long K0 = long(blockIdx.x) * EB;
  // blockDim is a multiple of EB: each thread keeps one element (its vertex
  // coordinates and volume in registers) and walks that element's nodes
  const int e = threadIdx.x % EB;
  const long K = K0 + e;
  double vx[12], vk = 0.0;
#pragma unroll
  for (int j = 0; j < 12; ++j) vx[j] = K < nelt ? V[long(j) * nelt + K] : 0.0;
  if (K < nelt) vk = vol[K];
  for (int q = threadIdx.x / EB; q < rows; q += blockDim.x / EB) {
    double bk = 0.0, bc = 0.0, bf = 0.0;
    if (K < nelt) {
      if (q < nq) {
        const double l0 = __ldg(bary + q), l1 = __ldg(bary + nq + q), l2 = __ldg(bary + 2 * nq + q),
                     l3 = __ldg(bary + 3 * nq + q);
        const double x = l0 * vx[0] + l1 * vx[1] + l2 * vx[2] + l3 * vx[3];
        const double y = l0 * vx[4] + l1 * vx[5] + l2 * vx[6] + l3 * vx[7];
        const double z = l0 * vx[8] + l1 * vx[9] + l2 * vx[10] + l3 * vx[11];
        const double wv = __ldg(wq + q) * vk;
        FIELD_STMTS
        bk = wv / (FIELD_KAPPA);
        bc = wv * (FIELD_C);
        bf = wv * (FIELD_F);
      } else if (q >= nqp) {
        bc = T[long(q - nqp) * nelt + K];
      }
    }
    Bk[q * LDB + e] = bk;
    Bc[q * LDB + e] = bc;
    Bf[q * LDB + e] = bf;
  }
  __syncthreads();
  // M and D share the table rows (Wsym): one task loads each A fragment once
  // for both (2 NTI DMMA per load); D's 4 tau PP columns are one extra k-step.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int mts = nsymp / 8, mtf = d3p / 8;
  const int ntasks = mts + mtf;
  for (int task = warp; task < ntasks; task += nwarp) {
    double cm[NTI][2], cd[NTI][2];
#pragma unroll
    for (int j = 0; j < NTI; ++j) cm[j][0] = cm[j][1] = cd[j][0] = cd[j][1] = 0.0;
    const bool sym = task < mts;
    const int mt = sym ? task : task - mts;
    const double* Arow = sym ? Asym + (long(mt) * ((nqp + 4) / 4)) * 32 + lane
                             : Af + (long(mt) * (nqp / 4)) * 32 + lane;
    const double* B0 = sym ? Bk : Bf;
#pragma unroll QUAD_UNROLL
    for (int kk = 0; kk < nqp / 4; ++kk) {
      const double a = __ldg(Arow + kk * 32);
      const int o = (kk * 4 + t) * LDB + g;
#pragma unroll
      for (int j = 0; j < NTI; ++j) dmma(cm[j][0], cm[j][1], a, B0[o + 8 * j]);
      if (sym) {
#pragma unroll
        for (int j = 0; j < NTI; ++j) dmma(cd[j][0], cd[j][1], a, Bc[o + 8 * j]);
      }
    }
    if (sym) {  // tau PP rows (k = nqp .. nqp+3): D only
      const double a = __ldg(Arow + (nqp / 4) * 32);
      const int o = (nqp + t) * LDB + g;
#pragma unroll
      for (int j = 0; j < NTI; ++j) dmma(cd[j][0], cd[j][1], a, Bc[o + 8 * j]);
    }
    const int r = mt * 8 + g;
    const int lim = sym ? nsym : d3;
    if (r < lim) {
#pragma unroll
      for (int j = 0; j < NTI; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long K = K0 + 8 * j + 2 * t + h;
          if (K >= nelt) continue;
          if (sym) {
            Msym[K * lim + r] = cm[j][h];
            Dsym[K * lim + r] = cd[j][h];
          } else {
            fvec[K * lim + r] = cm[j][h];
          }
        }
    }
  }
}
)CUDA";

std::string lit(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "(%a)", v);  // exact hex-float literal
  return buf;
}

// Driver entry points resolved through the runtime (no link-time libcuda
// dependency, so the library still loads on machines without a driver).
struct Drv {
  CUresult (*loadData)(CUmodule*, const void*) = nullptr;
  CUresult (*getFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*setAttr)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                     void**, void**) = nullptr;
  CUresult (*ctxGetCurrent)(CUcontext*) = nullptr;
  bool ok = false;
};
Drv& drv() {
  static Drv d = [] {
    Drv r;
    cudaDriverEntryPointQueryResult q;
    auto get = [&](const char* name, void** fn) {
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn;
    };
    r.ok = get("cuModuleLoadData", reinterpret_cast<void**>(&r.loadData)) &&
           get("cuModuleGetFunction", reinterpret_cast<void**>(&r.getFunction)) &&
           get("cuFuncSetAttribute", reinterpret_cast<void**>(&r.setAttr)) &&
           get("cuLaunchKernel", reinterpret_cast<void**>(&r.launch)) &&
           get("cuCtxGetCurrent", reinterpret_cast<void**>(&r.ctxGetCurrent));
    return r;
  }();
  return d;
}

// Compiled cubins are cached per source text; loaded modules per (context,
// source): a CUfunction belongs to the context that was current when its
// module was loaded, so engines on different devices each load their own.
struct Cache {
  std::mutex mu;
  std::unordered_map<std::string, std::vector<char>> cubin;
  std::unordered_map<std::string, CUfunction> fn;
  std::vector<CUmodule> mods;
  std::string last_error;
};
Cache& cache() {
  static Cache c;
  return c;
}

}  // namespace

// Straight-line device code for the field programs of one kernel. Every
// operation becomes one named temporary, hash-consed across all the fields
// the kernel evaluates (C2's f repeats kappa's sin/cos terms, and x + y feeds
// both exp and cos), products of literals are folded on the host (the same
// IEEE double product the reference's callback computes), and sin/cos of an
// exact multiple of pi use sinpi/cospi (exact argument reduction, no
// Cody-Waite / Payne-Hanek path; differs from sin(fl(pi) m E) by ~1e-16 E).
std::string FieldEmitter::emit(const hdg_field& f, const char* sample_ptr) {
  if (f.kind == HDG_FIELD_CONST) return lit(f.value);
  if (f.kind == HDG_FIELD_SAMPLED) return std::string("__ldg(") + sample_ptr + " + K * nq + q)";
  struct Val {
    std::string s;            // temporary, literal or coordinate
    bool is_const = false;
    double c = 0.0;
    double mul_c = 0.0;       // MUL by a literal: the literal and the other operand
    std::string mul_e;
  };
  auto temp = [&](const std::string& expr) {
    auto it = memo_.find(expr);
    if (it != memo_.end()) return it->second;
    const std::string name = "_t" + std::to_string(ntemp_++);
    stmts_ += "const double " + name + " = " + expr + "; ";
    memo_.emplace(expr, name);
    return name;
  };
  auto konst = [&](double v) { Val r; r.s = lit(v); r.is_const = true; r.c = v; return r; };
  auto node = [&](const std::string& expr) { Val r; r.s = temp(expr); return r; };
  // m with c == m * fl(pi) exactly, m a small multiple of 1/4 (else 0)
  auto pi_multiple = [](double c) {
    const double m = c / 3.141592653589793;
    const double mq = std::nearbyint(m * 4.0) / 4.0;
    return (mq != 0.0 && std::fabs(mq) <= 64.0 && mq * 3.141592653589793 == c) ? mq : 0.0;
  };
  std::vector<Val> st;
  int ci = 0;
  for (int i = 0; i < f.nops; ++i) {
    const int op = f.ops[i];
    auto pop = [&]() { Val v = st.back(); st.pop_back(); return v; };
    switch (op) {
      case HDG_OP_X: { Val v; v.s = "x"; st.push_back(v); break; }
      case HDG_OP_Y: { Val v; v.s = "y"; st.push_back(v); break; }
      case HDG_OP_Z: { Val v; v.s = "z"; st.push_back(v); break; }
      case HDG_OP_CONST: st.push_back(konst(f.consts[ci++])); break;
      case HDG_OP_NEG: {
        const Val a = pop();
        st.push_back(a.is_const ? konst(-a.c) : node("(-" + a.s + ")"));
        break;
      }
      case HDG_OP_SIN:
      case HDG_OP_COS: {
        const Val a = pop();
        const double m = a.mul_e.empty() ? 0.0 : pi_multiple(a.mul_c);
        const char* fn = op == HDG_OP_SIN ? (m != 0.0 ? "sinpi" : "sin") : (m != 0.0 ? "cospi" : "cos");
        st.push_back(node(std::string(fn) + "(" + (m != 0.0 ? (m == 1.0 ? a.mul_e : lit(m) + " * " + a.mul_e) : a.s) + ")"));
        break;
      }
      case HDG_OP_EXP: st.push_back(node("exp(" + pop().s + ")")); break;
      case HDG_OP_SQRT: st.push_back(node("sqrt(" + pop().s + ")")); break;
      case HDG_OP_ABS: st.push_back(node("fabs(" + pop().s + ")")); break;
      default: {
        const Val b = pop(), a = pop();
        if (a.is_const && b.is_const && op >= HDG_OP_ADD && op <= HDG_OP_DIV) {
          st.push_back(konst(op == HDG_OP_ADD ? a.c + b.c : op == HDG_OP_SUB ? a.c - b.c
                             : op == HDG_OP_MUL ? a.c * b.c : a.c / b.c));
          break;
        }
        switch (op) {
          case HDG_OP_ADD: st.push_back(node("(" + a.s + " + " + b.s + ")")); break;
          case HDG_OP_SUB: st.push_back(node("(" + a.s + " - " + b.s + ")")); break;
          case HDG_OP_MUL: {
            Val r = node("(" + a.s + " * " + b.s + ")");
            if (a.is_const) { r.mul_c = a.c; r.mul_e = b.s; }
            else if (b.is_const) { r.mul_c = b.c; r.mul_e = a.s; }
            st.push_back(r);
            break;
          }
          case HDG_OP_DIV: st.push_back(node("(" + a.s + " / " + b.s + ")")); break;
          case HDG_OP_LT: st.push_back(node("((" + a.s + ") < (" + b.s + ") ? 1.0 : 0.0)")); break;
          case HDG_OP_POW: st.push_back(node("pow(" + a.s + ", " + b.s + ")")); break;
          default: st.push_back(konst(0.0));
        }
      }
    }
  }
  return st.empty() ? "0.0" : st.back().s;
}

namespace {
// NVRTC-compile `src` for sm_100a (once per source text) and return its kernel
// `name` loaded in the current context (once per context).
CUfunction compile_cached(const std::string& src, const char* name, std::string* err) {
  Cache& C = cache();
  std::lock_guard<std::mutex> lock(C.mu);
  if (!drv().ok) {
    if (err) *err = "driver entry points unavailable";
    return nullptr;
  }
  CUcontext ctx = nullptr;
  if (drv().ctxGetCurrent(&ctx) != CUDA_SUCCESS || !ctx) {
    if (err) *err = "no current CUDA context";
    return nullptr;
  }
  char key_prefix[32];
  std::snprintf(key_prefix, sizeof key_prefix, "%p\n", static_cast<void*>(ctx));
  const std::string key = key_prefix + std::string(name) + "\n" + src;  // one module may hold several kernels
  auto it = C.fn.find(key);
  if (it != C.fn.end()) return it->second;
  auto bin = C.cubin.find(src);
  if (bin == C.cubin.end()) {
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "hdg_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
      if (err) *err = "nvrtcCreateProgram failed";
      return nullptr;
    }
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo"};
    const nvrtcResult rc = nvrtcCompileProgram(prog, 3, opts);
    if (rc != NVRTC_SUCCESS) {
      size_t n = 0;
      nvrtcGetProgramLogSize(prog, &n);
      std::string log(n, '\0');
      nvrtcGetProgramLog(prog, log.data());
      if (err) *err = "nvrtc: " + log;
      nvrtcDestroyProgram(&prog);
      return nullptr;
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    std::vector<char> cubin(n);
    nvrtcGetCUBIN(prog, cubin.data());
    nvrtcDestroyProgram(&prog);
    bin = C.cubin.emplace(src, std::move(cubin)).first;
  }
  CUmodule mod;
  CUfunction fn;
  if (drv().loadData(&mod, bin->second.data()) != CUDA_SUCCESS ||
      drv().getFunction(&fn, mod, name) != CUDA_SUCCESS) {
    if (err) *err = "cuModuleLoadData/cuModuleGetFunction failed";
    return nullptr;
  }
  C.mods.push_back(mod);
  C.fn.emplace(key, fn);
  return fn;
}

const char* kSampleSource = R"CUDA(
// JIT: a field program sampled at every element node (SAMPLED layout K * nq + q).
extern "C" __global__ void __launch_bounds__(256)
sample_field_jit(int nelt, int nq, const double* __restrict__ bary, const double* __restrict__ V,
                 double* __restrict__ out) {
  const long n = long(nelt) * nq;
  for (long idx = long(blockIdx.x) * blockDim.x + threadIdx.x; idx < n; idx += long(gridDim.x) * blockDim.x) {
    const long K = idx / nq;
    const int q = int(idx - K * nq);
    const double l0 = __ldg(bary + q), l1 = __ldg(bary + nq + q), l2 = __ldg(bary + 2 * nq + q),
                 l3 = __ldg(bary + 3 * nq + q);
    const double x = l0 * V[K] + l1 * V[nelt + K] + l2 * V[2L * nelt + K] + l3 * V[3L * nelt + K];
    const double y = l0 * V[4L * nelt + K] + l1 * V[5L * nelt + K] + l2 * V[6L * nelt + K] + l3 * V[7L * nelt + K];
    const double z = l0 * V[8L * nelt + K] + l1 * V[9L * nelt + K] + l2 * V[10L * nelt + K] + l3 * V[11L * nelt + K];
    FIELD_STMTS
    out[idx] = FIELD_EXPR;
  }
}
)CUDA";

const char* kSampleWSource = R"CUDA(
// JIT: w_q / field at every element node (K * nq + q): the postprocess's
// kappa^-1 weights, the division done here instead of in its epilogue.
extern "C" __global__ void __launch_bounds__(256)
sample_wdiv_jit(int nelt, int nq, const double* __restrict__ bary, const double* __restrict__ V,
                const double* __restrict__ wq, double* __restrict__ out) {
  const long n = long(nelt) * nq;
  for (long idx = long(blockIdx.x) * blockDim.x + threadIdx.x; idx < n; idx += long(gridDim.x) * blockDim.x) {
    const long K = idx / nq;
    const int q = int(idx - K * nq);
    const double l0 = __ldg(bary + q), l1 = __ldg(bary + nq + q), l2 = __ldg(bary + 2 * nq + q),
                 l3 = __ldg(bary + 3 * nq + q);
    const double x = l0 * V[K] + l1 * V[nelt + K] + l2 * V[2L * nelt + K] + l3 * V[3L * nelt + K];
    const double y = l0 * V[4L * nelt + K] + l1 * V[5L * nelt + K] + l2 * V[6L * nelt + K] + l3 * V[7L * nelt + K];
    const double z = l0 * V[8L * nelt + K] + l1 * V[9L * nelt + K] + l2 * V[10L * nelt + K] + l3 * V[11L * nelt + K];
    FIELD_STMTS
    out[idx] = __ldg(wq + q) / (FIELD_EXPR);
  }
}
)CUDA";

const char* kSample3Source = R"CUDA(
// Up to three fields at every point of a table, one pass (shared point and
// temporaries): out_h[K * npts + p] for the fields the host marked present.
extern "C" __global__ void __launch_bounds__(256)
sample_fields3_jit(int nelt, int nq, const double* __restrict__ bary, const double* __restrict__ V,
                   double* __restrict__ out0, double* __restrict__ out1, double* __restrict__ out2) {
  const long n = long(nelt) * nq;
  for (long idx = long(blockIdx.x) * blockDim.x + threadIdx.x; idx < n; idx += long(gridDim.x) * blockDim.x) {
    const long K = idx / nq;
    const int q = int(idx - K * nq);
    const double l0 = __ldg(bary + q), l1 = __ldg(bary + nq + q), l2 = __ldg(bary + 2 * nq + q),
                 l3 = __ldg(bary + 3 * nq + q);
    const double x = l0 * V[K] + l1 * V[nelt + K] + l2 * V[2L * nelt + K] + l3 * V[3L * nelt + K];
    const double y = l0 * V[4L * nelt + K] + l1 * V[5L * nelt + K] + l2 * V[6L * nelt + K] + l3 * V[7L * nelt + K];
    const double z = l0 * V[8L * nelt + K] + l1 * V[9L * nelt + K] + l2 * V[10L * nelt + K] + l3 * V[11L * nelt + K];
    FIELD_STMTS3
    FIELD_OUT0
    FIELD_OUT1
    FIELD_OUT2
  }
}
)CUDA";
}  // namespace

JitKernel jit_quad_kernel(const hdg_field& kap, const hdg_field& c, const hdg_field& f, int eb, int nqp,
                          std::string* err) {
  FieldEmitter fe;
  const std::string ek = fe.emit(kap, "sk"), ec = fe.emit(c, "sc"), ef = fe.emit(f, "sf");
  // the block size is baked into __launch_bounds__ here and returned with the
  // kernel, so the launch always uses the value the kernel was compiled for
  const int threads = jit_quad_threads(eb, nqp);
  const std::string src = "#define EB " + std::to_string(eb) + "\n#define QUAD_THREADS " +
                          std::to_string(threads) + "\n#define QUAD_MINB " + (threads == 384 ? HDG_QUAD_MINB32 : "1") +
                          "\n#define QUAD_UNROLL " +
                          std::to_string(HDG_QUAD_UNROLL) + "\n#define FIELD_STMTS " + fe.stmts() +
                          "\n#define FIELD_KAPPA " + ek + "\n#define FIELD_C " + ec + "\n#define FIELD_F " + ef +
                          "\n" + kQuadSource;
  return JitKernel{compile_cached(src, "quad_build_jit", err), threads};
}

CUfunction jit_sample_kernel(const hdg_field& f, std::string* err) {
  if (f.kind != HDG_FIELD_PROGRAM) {
    if (err) *err = "only program fields are sampled";
    return nullptr;
  }
  FieldEmitter fe;
  const std::string e = fe.emit(f, "nullptr");
  return compile_cached("#define FIELD_STMTS " + fe.stmts() + "\n#define FIELD_EXPR " + e + "\n" + kSampleSource,
                        "sample_field_jit", err);
}

CUfunction jit_sample_wdiv_kernel(const hdg_field& f, std::string* err) {
  if (f.kind != HDG_FIELD_PROGRAM) {
    if (err) *err = "only program fields are sampled";
    return nullptr;
  }
  FieldEmitter fe;
  const std::string e = fe.emit(f, "nullptr");
  return compile_cached("#define FIELD_STMTS " + fe.stmts() + "\n#define FIELD_EXPR " + e + "\n" + kSampleWSource,
                        "sample_wdiv_jit", err);
}

CUfunction jit_sample3_kernel(const hdg_field* const f[3], std::string* err) {
  FieldEmitter fe;
  std::string outs;
  bool any = false;
  for (int h = 0; h < 3; ++h) {
    outs += "#define FIELD_OUT" + std::to_string(h) + " ";
    if (f[h]->kind == HDG_FIELD_PROGRAM) {
      outs += "out" + std::to_string(h) + "[idx] = " + fe.emit(*f[h], "nullptr") + ";";
      any = true;
    }
    outs += "\n";
  }
  if (!any) {
    if (err) *err = "no program field to sample";
    return nullptr;
  }
  return compile_cached("#define FIELD_STMTS3 " + fe.stmts() + "\n" + outs + kSample3Source,
                        "sample_fields3_jit", err);
}

bool launch_quad_jit(CUfunction fn, cudaStream_t stream, int grid, int block, size_t smem, void** args,
                     std::string* err) {
  if (drv().setAttr(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, int(smem)) != CUDA_SUCCESS) {
    if (err) *err = "cuFuncSetAttribute failed";
    return false;
  }
  const CUresult r = drv().launch(fn, grid, 1, 1, block, 1, 1, (unsigned)smem, (CUstream)stream, args, nullptr);
  if (r != CUDA_SUCCESS) {
    if (err) *err = "cuLaunchKernel failed: CUresult " + std::to_string(int(r));
    return false;
  }
  return true;
}

}  // namespace hdgb
