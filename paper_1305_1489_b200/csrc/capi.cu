// C ABI of the engine (include/hdg_b200.h): context, table upload, launch
// dispatch over the polynomial degree, host mesh setup. No exceptions cross
// the ABI; every failure becomes an HDG_E* status plus a thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hdg_b200.h"
#include "dev_common.cuh"
#include "host_internal.hpp"
#include "kernels_local.cuh"
#include "kernels_misc.cuh"
#include "kernels_post.cuh"
#include "kernels_condense2.cuh"
#include "kernels_condense6.cuh"
#include "kernels_condense5.cuh"
#include "kernels_recover3.cuh"
#include "kernels_boundary.cuh"
#include "kernels_solve.cuh"
#include "kernels_errors.cuh"
#include "kernels_post2.cuh"
#include "kernels_rescue.cuh"
#include "kernels_conv2.cuh"
#include "kernels_conv3.cuh"
#include "exchange.cuh"
#include "jit_quad.hpp"
#include "mesh_dev.hpp"

using namespace hdgb;

namespace {

thread_local std::string g_err;

struct HdgError {
  int code;
  std::string msg;
};

#define CUDA_OK(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw HdgError{HDG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};    \
  } while (0)

template <class F>
int guarded(F&& fn) {
  try {
    fn();
    return HDG_OK;
  } catch (const HdgError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const MeshError& e) {
    g_err = e.what();
    return HDG_EMESH;
  } catch (const CudaError& e) {
    g_err = e.what();
    return HDG_ECUDA;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HDG_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HDG_EINVAL;
  }
}

void require(bool cond, int code, const std::string& msg) {
  if (!cond) throw HdgError{code, msg};
}

// Device copy of one degree's tables (one allocation, offsets into it).
struct TabSet {
  bool ready = false;
  bool chat_sparse = false;  // Chat_h has the structural zeros K3 skips (check_chat_pattern)
  HostTables host;
  DevTab dev{};
  double* buf = nullptr;
  size_t doubles = 0;
};

// DMMA fragment order: fragment (mt, kk) = 32 doubles, lane -> A(mt*8 + lane/4, kk*4 + lane%4).
std::vector<double> to_fragments(const std::vector<double>& A, int rows, int cols) {
  std::vector<double> out(size_t(rows) * cols, 0.0);
  const int kc = cols / 4;
  for (int mt = 0; mt < rows / 8; ++mt)
    for (int kk = 0; kk < kc; ++kk)
      for (int lane = 0; lane < 32; ++lane) {
        const int r = mt * 8 + lane / 4, c = kk * 4 + lane % 4;
        out[(size_t(mt) * kc + kk) * 32 + lane] = A[size_t(r) * cols + c];  // A row-major
      }
  return out;
}

// K3 v6 (k = 2, 3) skips the 8 x 4 blocks of Chat_h that c6_ch_nz declares
// structurally zero (rows of top-degree modes, the lower triangle), K3 v5
// (k = 4, 5) the zero row tiles and the ksteps below a row tile. The claim is
// verified on the tables actually built, entry by entry; if a skipped block
// holds anything above rounding (a quadrature rule too coarse to integrate
// P_i d_h P_j exactly), the dense instantiation of the kernel runs instead.
bool check_chat_pattern(const HostTables& h) {
  const int k = h.k, d3 = h.d3;
  if (k < 2) return false;
  double mx = 0.0;
  for (int hh = 0; hh < 3; ++hh)
    for (double v : h.Chat[hh]) mx = std::max(mx, std::fabs(v));
  if (k >= 4) {  // kernels_condense5.cuh: rows >= dim P_{k-1} and, per 8-row tile, the columns below the tile
    const int n1 = pdim3(k - 1);
    for (int hh = 0; hh < 3; ++hh)
      for (int r = 0; r < d3; ++r)
        for (int kk = 0; kk < d3; ++kk)
          if ((r >= n1 || kk < 8 * (r / 8)) && std::fabs(h.Chat[hh][r + size_t(kk) * d3]) > 1e-13 * mx) return false;
    return true;
  }
  const int np = d3 / 8, ks = 2 * np + (d3 % 8 ? 1 : 0), nt3 = (d3 + 7) / 8;
  for (int hh = 0; hh < 3; ++hh)
    for (int tile = 0; tile < nt3; ++tile)
      for (int s = 0; s < ks; ++s) {
        if (c6_ch_nz(k, hh, tile, s)) continue;
        for (int r = 8 * tile; r < std::min(8 * tile + 8, d3); ++r)
          for (int t = 0; t < 4; ++t) {
            const int kk = s < 2 * np ? (s >> 1) * 8 + 2 * t + (s & 1) : 8 * np + t;
            if (kk < d3 && std::fabs(h.Chat[hh][r + size_t(kk) * d3]) > 1e-13 * mx) return false;
          }
      }
  return true;
}

void upload_tables(TabSet& ts, int k, int tet_deg, int tri_deg) {
  if (ts.buf) { cudaFree(ts.buf); ts.buf = nullptr; }
  ts.ready = false;
  ts.chat_sparse = false;
  ts.host = build_host_tables(k, tet_deg, tri_deg);
  const HostTables& h = ts.host;
  const int d3 = h.d3, d2 = h.d2, nq = h.nq, nqd = h.nqd;
  const int nqp = round_up(nq, 4), nsym = d3 * (d3 + 1) / 2, nsymp = round_up(nsym, 8), d3p = round_up(d3, 8);
  // Asym: rows = sym pairs (i >= j), cols = nqp node columns + 4 PP columns (row-major)
  std::vector<double> Asym(size_t(nsymp) * (nqp + 4), 0.0), Af(size_t(d3p) * nqp, 0.0);
  for (int j = 0; j < d3; ++j)
    for (int i = j; i < d3; ++i) {
      const int r = sym_idx(i, j, d3);
      for (int q = 0; q < nq; ++q) Asym[size_t(r) * (nqp + 4) + q] = h.P[q + size_t(i) * nq] * h.P[q + size_t(j) * nq];
      for (int l = 0; l < 4; ++l) Asym[size_t(r) * (nqp + 4) + nqp + l] = h.PP[l][i + size_t(j) * d3];
    }
  for (int i = 0; i < d3; ++i)
    for (int q = 0; q < nq; ++q) Af[size_t(i) * nqp + q] = h.P[q + size_t(i) * nq];
  const std::vector<double> Asym_f = to_fragments(Asym, nsymp, nqp + 4);
  const std::vector<double> Af_f = to_fragments(Af, d3p, nqp);

  std::vector<double> all;
  std::vector<size_t> off;
  auto push = [&](const std::vector<double>& v) {
    off.push_back(all.size());
    all.insert(all.end(), v.begin(), v.end());
    all.resize(round_up(int(all.size()), 32), 0.0);  // 256 B alignment
  };
  auto cat = [](std::initializer_list<const std::vector<double>*> parts) {
    std::vector<double> o;
    for (auto* p : parts) o.insert(o.end(), p->begin(), p->end());
    return o;
  };
  push(h.tet_bary);                                              // 0
  push(h.tet_w);                                                 // 1
  push(h.P);                                                     // 2
  push(cat({&h.Pd[0], &h.Pd[1], &h.Pd[2]}));                     // 3
  push(cat({&h.Chat[0], &h.Chat[1], &h.Chat[2]}));               // 4
  {
    std::vector<double> s;
    for (auto& m : h.Shat) s.insert(s.end(), m.begin(), m.end());
    push(s);                                                     // 5
  }
  {
    std::vector<double> s;
    for (auto& m : h.Wlm) s.insert(s.end(), m.begin(), m.end());
    push(s);                                                     // 6
  }
  push(cat({&h.PP[0], &h.PP[1], &h.PP[2], &h.PP[3]}));           // 7
  push(h.DD);                                                    // 8
  push(h.tri_bary);                                              // 9
  push(h.tri_w);                                                 // 10
  push(cat({&h.Pface[0], &h.Pface[1], &h.Pface[2], &h.Pface[3]}));  // 11
  {
    std::vector<double> s;
    for (auto& m : h.Dperm) s.insert(s.end(), m.begin(), m.end());
    push(s);                                                     // 12
  }
  push(Asym_f);                                                  // 13
  push(Af_f);                                                    // 14
  {  // lane-contiguous transposes for row-per-lane contractions (K5)
    std::vector<double> s(size_t(3) * d3 * d3), w(size_t(24) * d2 * d3);
    for (int h3 = 0; h3 < 3; ++h3)
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < d3; ++i) s[size_t(h3) * d3 * d3 + j + size_t(i) * d3] = h.Chat[h3][i + size_t(j) * d3];
    for (int lm = 0; lm < 24; ++lm)
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < d2; ++i) w[size_t(lm) * d2 * d3 + j + size_t(i) * d3] = h.Wlm[lm][i + size_t(j) * d2];
    push(s);                                                     // 15
    push(w);                                                     // 16
  }
  {  // Shat packed lower (column-major), 9 x d3(d3+1)/2: A operand of the postprocess S GEMM
    const int ns = d3 * (d3 + 1) / 2;
    std::vector<double> sp(size_t(9) * ns);
    for (int hh = 0; hh < 9; ++hh) {
      int p = 0;
      for (int j = 0; j < d3; ++j)
        for (int i = j; i < d3; ++i) sp[size_t(hh) * ns + p++] = h.Shat[hh][i + size_t(j) * d3];
    }
    push(sp);                                                    // 17
  }
  if (k <= 3) {  // K7 v2 volume table: row i + j d3, column # nqp + q: P_qi dP_qj/dxhat_#
    const int rows = round_up(d3 * d3, 8), cols = 3 * nqp;
    std::vector<double> A(size_t(rows) * cols, 0.0);
    for (int j = 0; j < d3; ++j)
      for (int i = 0; i < d3; ++i)
        for (int hh = 0; hh < 3; ++hh)
          for (int q = 0; q < nq; ++q)
            A[size_t(i + j * d3) * cols + hh * nqp + q] = h.P[q + size_t(i) * nq] * h.Pd[hh][q + size_t(j) * nq];
    push(to_fragments(A, rows, cols));                           // 18
  }
  CUDA_OK(cudaMalloc(&ts.buf, all.size() * sizeof(double)));
  CUDA_OK(cudaMemcpy(ts.buf, all.data(), all.size() * sizeof(double), cudaMemcpyHostToDevice));
  ts.doubles = all.size();
  DevTab& t = ts.dev;
  t.k = k; t.d3 = d3; t.d2 = d2; t.nq = nq; t.nqd = nqd; t.nqp = nqp;
  t.nsym = nsym; t.nsymp = nsymp; t.d3p = d3p; t.nu = d3;
  const double* b = ts.buf;
  t.bary = b + off[0]; t.w = b + off[1]; t.P = b + off[2]; t.Pd = b + off[3]; t.Chat = b + off[4];
  t.Shat = b + off[5]; t.Wlm = b + off[6]; t.PP = b + off[7]; t.DD = b + off[8];
  t.tri_bary = b + off[9]; t.tri_w = b + off[10]; t.Pface = b + off[11]; t.Dperm = b + off[12];
  t.Asym = b + off[13]; t.Af = b + off[14]; t.ChatT = b + off[15]; t.WlmT = b + off[16];
  t.ShatP = b + off[17];
  t.Aconv = k <= 3 ? b + off[18] : nullptr;
  ts.ready = true;
}

FieldDev to_dev(const hdg_field& f, const char* name) {
  FieldDev d{};
  d.kind = f.kind;
  d.value = f.value;
  d.samples = f.samples;
  if (f.kind == HDG_FIELD_PROGRAM) {
    require(f.nops > 0 && f.nops <= HDG_FIELD_MAX_OPS && f.nconst >= 0 &&
                f.nconst <= HDG_FIELD_MAX_CONSTS && f.ops,
            HDG_EINVAL, std::string("field program too large or empty: ") + name);
    int depth = 0, maxd = 0, nc = 0;
    for (int i = 0; i < f.nops; ++i) {
      const int op = f.ops[i];
      require(op >= HDG_OP_X && op <= HDG_OP_POW, HDG_EINVAL, std::string("bad opcode in ") + name);
      if (op <= HDG_OP_CONST) ++depth;
      else if (op == HDG_OP_ADD || op == HDG_OP_SUB || op == HDG_OP_MUL || op == HDG_OP_DIV ||
               op == HDG_OP_LT || op == HDG_OP_POW) --depth;
      if (op == HDG_OP_CONST) ++nc;
      require(depth >= 1, HDG_EINVAL, std::string("stack underflow in ") + name);
      maxd = std::max(maxd, depth);
      d.ops[i] = static_cast<unsigned char>(op);
    }
    require(depth == 1 && maxd <= HDG_FIELD_MAX_STACK && nc == f.nconst, HDG_EINVAL,
            std::string("malformed field program: ") + name);
    for (int i = 0; i < f.nconst; ++i) d.consts[i] = f.consts[i];
    d.nops = f.nops;
  } else if (f.kind == HDG_FIELD_SAMPLED) {
    require(f.samples != nullptr, HDG_EINVAL, std::string("sampled field without samples: ") + name);
  } else {
    require(f.kind == HDG_FIELD_CONST, HDG_EINVAL, std::string("bad field kind: ") + name);
  }
  return d;
}

GeoDev to_geo(const hdg_geometry* g) {
  require(g && g->volume && g->piola && g->normals && g->perm && g->T && g->verts, HDG_EINVAL,
          "incomplete hdg_geometry");
  return GeoDev{g->volume, g->piola, g->normals, g->perm, g->T, g->verts};
}

}  // namespace

struct hdg_mesh {
  HostMesh m;
  bool pattern_ready = false;
  SkeletonPattern pat;
};

struct hdg_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  TabSet tab[4];  // [0] degree k, [1] postprocess degree k+1, [2]/[3] degree k / k+1 on the error rule
  int post_tet_deg = -1;
  int tri_deg = 0;
  void* work = nullptr;
  size_t work_bytes = 0;
  long long* d_bad = nullptr;
  long long* h_bad = nullptr;
  int* d_status = nullptr;
  int* h_status = nullptr;
  bool timing = false;
  bool jit = true;          // NVRTC-specialised K2 for program fields
  bool bdm = false;         // bdm_blocks variant (hdg_b200_set_bdm)
  bool tau_allow_zero = false;  // StabilizationField::allow_zero (element_matrices.hpp:24)
  bool build_status_pending = false;  // last build_condense's status not yet reported
  double rescue_screen = 1e-12; // pivot-ratio screen of the rescue kernel (kernels_rescue.cuh)
  double* d_rescue = nullptr;   // rescue kernel scratch
  size_t rescue_len = 0;
  double* d_zero_T = nullptr;  // tau = 0 for the BDM variant
  long zero_T_len = 0;
  int recover_variant = 3;  // k = 1..3: 3 = TMA-streamed cache, 2 = warp per element
  std::string jit_error;    // last JIT failure (kernel then runs interpreted)
  int* d_adj = nullptr;     // boundary face -> 4 K + l (neumann_load)
  double* d_ksamp = nullptr;  // kappa sampled at the postprocess nodes (JIT sampler)
  size_t ksamp_len = 0;
  double* d_bsamp = nullptr;  // program beta components sampled at the convection points (JIT sampler)
  size_t bsamp_len = 0;
  double* d_cbary = nullptr;  // convection points: volume nodes + element-parametrised face points (npts x 4)
  int cbary_k = -1;
  int adj_len = 0;
  cudaEvent_t ev[2 * HDG_NSTAGES] = {};
  bool pending[HDG_NSTAGES] = {};
};

namespace {

void set_device(hdg_ctx* c) { CUDA_OK(cudaSetDevice(c->device)); }

// CUDA events around each stage on the launching stream (hdg_b200_set_timing).
void stage_begin(hdg_ctx* c, int s) {
  if (c->timing) CUDA_OK(cudaEventRecord(c->ev[2 * s], c->stream));
}
void stage_end(hdg_ctx* c, int s) {
  if (!c->timing) return;
  CUDA_OK(cudaEventRecord(c->ev[2 * s + 1], c->stream));
  c->pending[s] = true;
}

void* ctx_work(hdg_ctx* c, size_t bytes) {
  if (bytes > c->work_bytes) {
    if (c->work) cudaFree(c->work);
    c->work = nullptr;
    CUDA_OK(cudaMalloc(&c->work, bytes));
    c->work_bytes = bytes;
  }
  return c->work;
}

// K2 outputs (packed M, packed D, f) then the pivot statistics of K3
// (nelt x 4, 32-byte aligned) screened by the rescue kernel.
size_t pivstat_offset(const DevTab& t, long nelt) { return (size_t(nelt) * (2 * t.nsym + t.d3) + 3) / 4 * 4; }
size_t work_doubles(const DevTab& t, long nelt) { return pivstat_offset(t, nelt) + size_t(nelt) * 4; }

// recovery cache record: {M^-1 packed lower, Vs = S^-1 V (d3 x m), fs = S^-1 f},
// padded to a 16-byte multiple (TMA bulk copies)
int factor_doubles(int k) {
  const int d3 = hdgb::pdim3(k), m = 4 * hdgb::pdim2(k);
  return (d3 * (d3 + 1) / 2 + d3 * m + d3 + 1) / 2 * 2;
}

template <int K_>
struct C6Launch {  // one element per warp
  static constexpr int EPB = C6Cfg<K_>::NW, THREADS = C6Cfg<K_>::NW * 32;
};

template <int K_>
struct C5Launch {  // one element per CTA iteration
  static constexpr int EPB = 1, THREADS = C5Cfg<K_>::NWT * 32;
};

// per-element team kernel (k <= 1): NW warps per element
template <int K_>
struct C2Launch {
  static constexpr int EPB = C2Cfg<K_>::EPB, THREADS = C2Cfg<K_>::NW * 32 * C2Cfg<K_>::EPB;
};

template <class Dm, class Cg, class Kern>
void launch_condense_impl(hdg_ctx* c, Kern kern, int nelt, const GeoDev& geo, const double* Ms,
                          const double* Ds, const double* fv, double* C, double* Cf, double* F, double* ps) {
  const size_t smem = (size_t(Cg::EPB) * Dm::PER_ELT + Dm::CTA_EXTRA) * sizeof(double);
  CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int occ = 0;
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, Cg::THREADS, smem));
  require(occ > 0, HDG_ECUDA, "condense kernel does not fit on an SM");
  const long need = (long(nelt) + Cg::EPB - 1) / Cg::EPB;
  const int grid = int(std::min<long>(need, long(c->sms) * occ));
  DevTab td = c->tab[0].dev;
  if (c->bdm) td.nu = td.d3 - td.d2;  // bdm_blocks (local_solver.cpp:65-69): u truncated to P_{k-1}
  kern<<<grid, Cg::THREADS, smem, c->stream>>>(td, nelt, geo, Ms, Ds, fv, C, Cf, F, ps);
  CUDA_OK(cudaGetLastError());
}

// k <= 1: per-element warp teams (kernels_condense2.cuh); k = 2, 3: one warp
// per element, register-chained DMMA (kernels_condense6.cuh); k = 4, 5: one
// element per CTA iteration (kernels_condense5.cuh). All write the recovery
// cache (factor_doubles) read by launch_recover.
template <int K_>
void launch_condense(hdg_ctx* c, int nelt, const GeoDev& geo, const double* Ms, const double* Ds,
                     const double* fv, double* C, double* Cf, double* F, double* ps) {
#ifndef HDG_TEAM_MAXK
#define HDG_TEAM_MAXK 1  // diagnostics builds: per-element warp teams up to this degree
#endif
  if constexpr (K_ <= HDG_TEAM_MAXK)
    launch_condense_impl<C2Dims<K_>, C2Launch<K_>>(c, condense2_kernel<K_>, nelt, geo, Ms, Ds, fv, C, Cf, F, ps);
  else if constexpr (K_ <= 3) {
    if (c->tab[0].chat_sparse)
      launch_condense_impl<C6Dims<K_>, C6Launch<K_>>(c, condense6_kernel<K_, C6Cfg<K_>::NW, true>, nelt, geo, Ms, Ds,
                                                     fv, C, Cf, F, ps);
    else
      launch_condense_impl<C6Dims<K_>, C6Launch<K_>>(c, condense6_kernel<K_, C6Cfg<K_>::NW, false>, nelt, geo, Ms,
                                                     Ds, fv, C, Cf, F, ps);
  } else {
    if (c->tab[0].chat_sparse)
      launch_condense_impl<C5Dims<K_>, C5Launch<K_>>(c, condense5_kernel<K_, true>, nelt, geo, Ms, Ds, fv, C, Cf, F,
                                                     ps);
    else
      launch_condense_impl<C5Dims<K_>, C5Launch<K_>>(c, condense5_kernel<K_, false>, nelt, geo, Ms, Ds, fv, C, Cf,
                                                     F, ps);
  }
}

// K3b: screen the pivot statistics, re-solve the flagged elements by the
// reference's LU path (kernels_rescue.cuh).
void launch_rescue(hdg_ctx* c, int nelt, const DevTab& td, const GeoDev& geo, const double* Ms,
                   const double* Ds, const double* fv, const double* ps, double* C, double* Cf, double* F) {
  const RescueLayout L(td.d3, td.d2, td.nu);
  const int grid = int(std::max<long>(1, std::min<long>((long(nelt) + kRescueThreads - 1) / kRescueThreads, c->sms)));
  const size_t need = size_t(grid) * L.total;
  if (c->rescue_len < need) {
    if (c->d_rescue) cudaFree(c->d_rescue);
    c->d_rescue = nullptr;
    CUDA_OK(cudaMalloc(&c->d_rescue, need * sizeof(double)));
    c->rescue_len = need;
  }
  rescue_kernel<<<grid, kRescueThreads, 0, c->stream>>>(td, nelt, geo, Ms, Ds, fv, ps, c->rescue_screen, C, Cf, F,
                                                        c->d_rescue, c->d_bad);
  CUDA_OK(cudaGetLastError());
}

template <int K_>
void launch_recover(hdg_ctx* c, int nelt, const GeoDev& geo, const int* fbe, const double* F,
                    const double* uhat, double* qx, double* qy, double* qz, double* u) {
  if constexpr (K_ >= 1 && K_ <= 3) {
    if (c->recover_variant == 3) {  // TMA-streamed cache, persistent warps
      using Rd = Rec3Dims<K_>;
      constexpr int kRec3Warps = Rec3Cfg<K_>::WARPS;
      const size_t smem = (size_t(kRec3Warps) * Rd::PER_WARP + Rd::TABLES) * sizeof(double);
      CUDA_OK(cudaFuncSetAttribute(recover3_kernel<K_>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      const long need = (long(nelt) + kRec3Warps - 1) / kRec3Warps;
      const int grid3 = int(std::min<long>(need, c->sms));
      recover3_kernel<K_><<<grid3, kRec3Warps * 32, smem, c->stream>>>(c->tab[0].dev, nelt, geo, fbe, F, uhat,
                                                                       qx, qy, qz, u);
      CUDA_OK(cudaGetLastError());
      return;
    }
  }
  if constexpr (K_ >= 4 && K_ <= 5) {
    {  // v5 cache {M^-1, S^-1, V, f}: one record per CTA iteration
      using Rd = Rec5Dims<K_>;
      const size_t smem = size_t(Rd::TOTAL) * sizeof(double);
      CUDA_OK(cudaFuncSetAttribute(recover5_kernel<K_>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      int occ = 0;
      CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, recover5_kernel<K_>, kRec5Threads, smem));
      const int grid5 = int(std::min<long>(nelt, long(c->sms) * std::max(occ, 1)));
      recover5_kernel<K_><<<grid5, kRec5Threads, smem, c->stream>>>(c->tab[0].dev, nelt, geo, fbe, F, uhat, qx, qy,
                                                                    qz, u);
      CUDA_OK(cudaGetLastError());
      return;
    }
  }
  if constexpr (K_ <= 3) {  // k = 0, or recover variant 2: one warp per element, direct loads
    const int grid = (nelt + kRecWarps - 1) / kRecWarps;
    recover2_kernel<K_><<<grid, kRecWarps * 32, 0, c->stream>>>(c->tab[0].dev, nelt, geo, fbe, F, uhat, qx,
                                                                 qy, qz, u);
    CUDA_OK(cudaGetLastError());
  }
}

#define DISPATCH_K(k, FN, ...)                              \
  switch (k) {                                              \
    case 0: FN<0>(__VA_ARGS__); break;                      \
    case 1: FN<1>(__VA_ARGS__); break;                      \
    case 2: FN<2>(__VA_ARGS__); break;                      \
    case 3: FN<3>(__VA_ARGS__); break;                      \
    case 4: FN<4>(__VA_ARGS__); break;                      \
    case 5: FN<5>(__VA_ARGS__); break;                      \
    default: throw HdgError{HDG_EINVAL, "degree not compiled (k <= 5)"}; \
  }

// Status of the last build_condense (reset_build_status_kernel words), in the
// reference's order: tau.validate() runs before any factorisation
// (element_matrices.cpp:287), so its invalid_argument wins over a singular
// element.
void raise_build_status(const hdg_ctx* c, int64_t* bad_element) {
  const long long* h = c->h_bad;
  if (bad_element) *bad_element = -1;
  if (h[1] != LLONG_MAX)
    throw HdgError{HDG_EINVAL, "stabilization must be nonnegative (element " + std::to_string(h[1]) + ")"};
  if (h[2] != LLONG_MAX && !c->tau_allow_zero)
    throw HdgError{HDG_EINVAL, "stabilization vanishes identically on element " + std::to_string(h[2])};
  if (h[0] != LLONG_MAX) {
    if (bad_element) *bad_element = h[0];
    throw HdgError{HDG_ESINGULAR, "singular local system on element " + std::to_string(h[0])};
  }
}

void check_bad(hdg_ctx* c, int64_t* bad_element) {
  if (!bad_element) return;
  CUDA_OK(cudaMemcpyAsync(c->h_bad, c->d_bad, 3 * sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  c->build_status_pending = false;
  raise_build_status(c, bad_element);
}

int warps_for(size_t per_warp_bytes) {
  const size_t cap = 200 * 1024;
  int w = int(std::min<size_t>(8, cap / std::max<size_t>(per_warp_bytes, 1)));
  return std::max(1, w);
}

}  // namespace

// K9 driver (template: outside the extern "C" block)
namespace {
// Nonsymmetric skeleton system: right-preconditioned BiCGStab (general
// block-Jacobi), restarted from the true residual until ||b - H x|| <= rtol
// ||r_0||. Scalars on the host (off the timed path).
template <int D2>
void solve_bicgstab(hdg_ctx* c, int nfc, const int64_t* fb, const int* nbr, const double* vals, const double* b,
                    int ndir, const double* ub, double rtol, int maxit, double* x, hdg_solve_info* info) {
  cudaStream_t s = c->stream;
  const long n = long(nfc) * D2;
  const long nd = long(ndir) * D2;
  const int nblk = c->sms * 4;
  auto al = [](size_t v) { return (v + 255) / 256 * 256; };
  const size_t vb = al(size_t(n) * 8), bb = al(size_t(nfc) * D2 * D2 * 8), pb = al(size_t(3) * nblk * 8);
  void* mem = nullptr;
  CUDA_OK(cudaMallocAsync(&mem, 8 * vb + bb + pb + 256, s));
  struct Free {
    void* p; cudaStream_t s;
    ~Free() { cudaFreeAsync(p, s); }
  } guard{mem, s};
  char* base = static_cast<char*>(mem);
  auto vec = [&](int i) { return reinterpret_cast<double*>(base + size_t(i) * vb); };
  double *r = vec(0), *rh = vec(1), *p = vec(2), *v = vec(3), *sv = vec(4), *t = vec(5), *ph = vec(6), *sh = vec(7);
  double* binv = reinterpret_cast<double*>(base + 8 * vb);
  double* part = reinterpret_cast<double*>(base + 8 * vb + bb);
  auto* bad = reinterpret_cast<unsigned long long*>(base + 8 * vb + bb + pb);
  std::vector<double> hp(size_t(3) * nblk);
  auto dots = [&](const double* a0, const double* b0, const double* a1, const double* b1, const double* a2,
                  const double* b2, double (&out)[3]) {
    dots_kernel<<<nblk, kSolveThreads, 0, s>>>(n, a0, b0, a1, b1, a2, b2, part);
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpyAsync(hp.data(), part, hp.size() * 8, cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    for (int q = 0; q < 3; ++q) {
      double acc = 0.0;
      for (int i = 0; i < nblk; ++i) acc += hp[size_t(q) * nblk + i];
      out[q] = acc;
    }
  };
  auto lin = [&](double* out, double a, const double* xx, double bq, const double* yy, double g, const double* zz) {
    lincomb_kernel<<<nblk, kSolveThreads, 0, s>>>(n, out, a, xx, bq, yy, g, zz);
  };
  auto apply = [&](const double* in, double* out) {  // out = mask(H K^-1 in), kin = K^-1 in
    spmv_kernel<D2><<<nblk, kSolveThreads, spmv_smem_bytes<D2>(), s>>>(nfc, fb, nbr, vals, in, out, ndir, nullptr);
  };
  auto precond = [&](const double* in, double* out) {
    precond_general_kernel<D2><<<nblk, kSolveThreads, 0, s>>>(nfc, ndir, binv, in, out);
  };
  // r = mask(b - H x)
  auto residual = [&]() {
    apply(x, t);
    lin(r, 1.0, b, -1.0, t, 0.0, nullptr);
    if (nd > 0) CUDA_OK(cudaMemsetAsync(r, 0, size_t(nd) * 8, s));
  };

  CUDA_OK(cudaMemsetAsync(bad, 0xff, 8, s));
  block_inverse_general_kernel<D2><<<nblk, 128, 0, s>>>(nfc, ndir, fb, nbr, vals, binv, bad);
  CUDA_OK(cudaGetLastError());
  if (ndir > 0) CUDA_OK(cudaMemcpyAsync(x, ub, size_t(nd) * 8, cudaMemcpyDeviceToDevice, s));
  CUDA_OK(cudaMemsetAsync(x + nd, 0, size_t(n - nd) * 8, s));
  unsigned long long hbad = 0;
  CUDA_OK(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, s));
  residual();
  double d[3];
  dots(r, r, nullptr, nullptr, nullptr, nullptr, d);
  if (hbad != ~0ull)
    throw HdgError{HDG_ESOLVE, "sparse LU factorization of the condensed system failed (face " +
                                   std::to_string(hbad) + " diagonal block singular)"};
  const double rr0 = d[0];
  int iters = 0;
  double rel = 0.0, prev_rel = 1e300;
  bool done = !(rr0 > 0.0);
  for (int restart = 0; !done && restart < 20 && iters < maxit; ++restart) {
    CUDA_OK(cudaMemcpyAsync(rh, r, size_t(n) * 8, cudaMemcpyDeviceToDevice, s));
    CUDA_OK(cudaMemsetAsync(p, 0, size_t(n) * 8, s));
    CUDA_OK(cudaMemsetAsync(v, 0, size_t(n) * 8, s));
    double rho = 1.0, alpha = 1.0, omega = 1.0;
    dots(rh, r, nullptr, nullptr, nullptr, nullptr, d);
    double rho_n = d[0];
    while (iters < maxit) {
      if (rho_n == 0.0 || !std::isfinite(rho_n)) break;
      const double beta = (rho_n / rho) * (alpha / omega);
      lin(p, 1.0, r, beta, p, -beta * omega, v);  // p = r + beta (p - omega v)
      precond(p, ph);
      apply(ph, v);
      dots(rh, v, nullptr, nullptr, nullptr, nullptr, d);
      if (d[0] == 0.0 || !std::isfinite(d[0])) break;
      alpha = rho_n / d[0];
      lin(sv, 1.0, r, -alpha, v, 0.0, nullptr);  // s = r - alpha v
      precond(sv, sh);
      apply(sh, t);
      dots(t, sv, t, t, nullptr, nullptr, d);
      omega = d[1] > 0.0 ? d[0] / d[1] : 0.0;
      lin(x, 1.0, x, alpha, ph, omega, sh);      // x += alpha ph + omega sh
      lin(r, 1.0, sv, -omega, t, 0.0, nullptr);  // r = s - omega t
      ++iters;
      rho = rho_n;
      dots(rh, r, r, r, nullptr, nullptr, d);
      rho_n = d[0];
      rel = std::sqrt(std::max(d[1], 0.0) / rr0);
      if (rel <= rtol || omega == 0.0 || !std::isfinite(rel)) break;
    }
    // the recurrence residual drifts: restart from (and test) the true one
    residual();
    dots(r, r, nullptr, nullptr, nullptr, nullptr, d);
    rel = std::sqrt(std::max(d[0], 0.0) / rr0);
    if (!std::isfinite(rel)) break;
    // done at rtol, or at the attainable accuracy: a restart cycle that no
    // longer reduces the true residual once it is within 1e3 rtol
    done = rel <= rtol || (rel <= 1e3 * rtol && rel > 0.5 * prev_rel);
    prev_rel = rel;
  }
  info->iterations = iters;
  info->relres = rel;
  info->converged = done ? 1 : 0;
  if (!done)
    throw HdgError{HDG_ESOLVE, "sparse LU solve of the condensed system failed: BiCGStab relative residual " +
                                   std::to_string(rel) + " after " + std::to_string(iters) + " iterations"};
}

template <int D2>
void solve_cg(hdg_ctx* c, int nfc, const int64_t* fb, const int* nbr, const double* vals, const double* b, int ndir,
              const double* ub, double rtol, int maxit, double* x, hdg_solve_info* info) {
  cudaStream_t s = c->stream;
  const long n = long(nfc) * D2;
  const int nblk = c->sms * 4;
  auto al = [](size_t v) { return (v + 255) / 256 * 256; };
  const size_t vb = al(size_t(n) * 8), pb = al(size_t(nblk) * 8);
  const size_t total = 5 * vb + al(size_t(nfc) * D2 * D2 * 8) + 3 * pb + 256 + 256;
  void* mem = nullptr;
  CUDA_OK(cudaMallocAsync(&mem, total, s));
  struct Free {
    void* p; cudaStream_t s;
    ~Free() { cudaFreeAsync(p, s); }
  } guard{mem, s};
  char* base = static_cast<char*>(mem);
  double* r = reinterpret_cast<double*>(base);
  double* z = reinterpret_cast<double*>(base + vb);
  double* p = reinterpret_cast<double*>(base + 2 * vb);
  double* y = reinterpret_cast<double*>(base + 3 * vb);
  double* r2 = reinterpret_cast<double*>(base + 4 * vb);  // ping-pong partner of r
  float* binv = reinterpret_cast<float*>(base + 5 * vb);
  double* p0 = reinterpret_cast<double*>(base + 5 * vb + al(size_t(nfc) * D2 * D2 * 8));
  double* p1 = p0 + pb / 8;
  double* p2 = p1 + pb / 8;
  auto* sc = reinterpret_cast<SolveScalars*>(reinterpret_cast<char*>(p2) + pb);
  auto* bad = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(sc) + 256);

  CUDA_OK(cudaFuncSetAttribute(spmv_kernel<D2>, cudaFuncAttributeMaxDynamicSharedMemorySize, spmv_smem_bytes<D2>()));
  // reference symmetry test over the free block (global_system.cpp:144-147)
  asym_kernel<D2><<<nblk, kSolveThreads, 0, s>>>(nfc, ndir, fb, nbr, vals, p0, p1);
  CUDA_OK(cudaGetLastError());
  std::vector<double> ha(nblk), hs(nblk);
  CUDA_OK(cudaMemcpyAsync(ha.data(), p0, nblk * 8, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaMemcpyAsync(hs.data(), p1, nblk * 8, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  double asym = 0.0, scale = 0.0;
  for (int i = 0; i < nblk; ++i) { asym += ha[i]; scale += hs[i]; }
  info->asym = asym;
  info->scale = scale;
  if (!(scale == 0.0 || asym < 1e-12 * scale)) {  // the reference's SparseLU branch (global_system.cpp:155-162)
    solve_bicgstab<D2>(c, nfc, fb, nbr, vals, b, ndir, ub, rtol, maxit, x, info);
    return;
  }

  CUDA_OK(cudaMemsetAsync(bad, 0xff, 8, s));
  block_jacobi_kernel<D2><<<nblk, kSolveThreads, 0, s>>>(nfc, ndir, fb, nbr, vals, binv, bad);
  CUDA_OK(cudaGetLastError());
  // x0: u_D on the Dirichlet dofs, 0 on the free ones
  if (ndir > 0) CUDA_OK(cudaMemcpyAsync(x, ub, size_t(ndir) * D2 * 8, cudaMemcpyDeviceToDevice, s));
  CUDA_OK(cudaMemsetAsync(x + long(ndir) * D2, 0, size_t(n - long(ndir) * D2) * 8, s));
  spmv_kernel<D2><<<nblk, kSolveThreads, spmv_smem_bytes<D2>(), s>>>(nfc, fb, nbr, vals, x, y, ndir, nullptr);
  update_kernel<D2><<<nblk, kSolveThreads, 0, s>>>(0, nfc, ndir, binv, b, y, p, x, r, r, z, sc, p1, p2);
  CUDA_OK(cudaMemcpyAsync(r2, r, size_t(n) * 8, cudaMemcpyDeviceToDevice, s));  // zero Dirichlet rows in both
  finalize_kernel<<<1, kSolveThreads, 0, s>>>(0, nblk, p1, p2, sc);
  direction_kernel<<<nblk, kSolveThreads, 0, s>>>(n, z, p, sc, 1);
  CUDA_OK(cudaGetLastError());
  unsigned long long hbad = 0;
  CUDA_OK(cudaMemcpyAsync(&hbad, bad, 8, cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  if (hbad != ~0ull)
    throw HdgError{HDG_ESOLVE, "symmetric factorization of the condensed system failed (face " +
                                   std::to_string(hbad) + " diagonal block not SPD)"};

  // one CG iteration = 5 launches; captured once into a graph of kChunk iterations
  constexpr int kChunk = 16;  // even: r is current again after every chunk
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  // capture on a private stream (the context stream may be the legacy default
  // stream, which cannot be captured); the graph is then launched on s
  cudaStream_t cs = nullptr;
  CUDA_OK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  struct StreamFree {
    cudaStream_t s;
    ~StreamFree() { cudaStreamDestroy(s); }
  } sguard{cs};
  CUDA_OK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  for (int it = 0; it < kChunk; ++it) {
    spmv_kernel<D2><<<nblk, kSolveThreads, spmv_smem_bytes<D2>(), cs>>>(nfc, fb, nbr, vals, p, y, ndir, p0);
    finalize_kernel<<<1, kSolveThreads, 0, cs>>>(1, nblk, p0, nullptr, sc);
    const double* rin = (it & 1) ? r2 : r;
    double* rout = (it & 1) ? r : r2;
    update_kernel<D2><<<nblk, kSolveThreads, 0, cs>>>(1, nfc, ndir, binv, b, y, p, x, rin, rout, z, sc, p1, p2);
    finalize_kernel<<<1, kSolveThreads, 0, cs>>>(2, nblk, p1, p2, sc);
    direction_kernel<<<nblk, kSolveThreads, 0, cs>>>(n, z, p, sc, 0);
  }
  CUDA_OK(cudaStreamEndCapture(cs, &graph));
  struct GraphFree {
    cudaGraph_t g; cudaGraphExec_t* e;
    ~GraphFree() { if (*e) cudaGraphExecDestroy(*e); if (g) cudaGraphDestroy(g); }
  } gguard{graph, &exec};
  CUDA_OK(cudaGraphInstantiate(&exec, graph, 0));
  SolveScalars h{};
  CUDA_OK(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, s));
  CUDA_OK(cudaStreamSynchronize(s));
  int iters = 0;
  double rel = 0.0;
  bool done = !(h.rr0 > 0.0);  // zero right-hand side: x0 is the solution
  while (!done && iters < maxit) {
    CUDA_OK(cudaGraphLaunch(exec, s));
    iters += kChunk;
    CUDA_OK(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    rel = std::sqrt(std::max(h.rr, 0.0) / h.rr0);
    done = rel <= rtol || !(h.pap > 0.0);
  }
  info->iterations = iters;
  info->relres = rel;
  info->converged = rel <= rtol ? 1 : 0;
  if (!info->converged)
    throw HdgError{HDG_ESOLVE, "skeleton CG did not converge: relative residual " + std::to_string(rel) +
                                   " after " + std::to_string(iters) + " iterations"};
}
}  // namespace

// error-functional helpers (outside the extern "C" block: member templates)
namespace {
// inverses of W_{l,mu}[:, t:] (d2 x d2, column-major) for the 24 (l, mu):
// Gauss-Jordan with partial pivoting on the host (level tables)
std::vector<double> face_block_inverses(const HostTables& h) {
  const int d2 = h.d2, d3 = h.d3, t = d3 - d2;
  std::vector<double> out(size_t(24) * d2 * d2);
  for (int lm = 0; lm < 24; ++lm) {
    std::vector<double> a(size_t(d2) * d2), inv(size_t(d2) * d2, 0.0);
    for (int j = 0; j < d2; ++j)
      for (int i = 0; i < d2; ++i) a[i + size_t(j) * d2] = h.Wlm[lm][i + size_t(t + j) * d2];
    for (int i = 0; i < d2; ++i) inv[i + size_t(i) * d2] = 1.0;
    double pmax = 0.0, pmin = 1e300;
    for (int c = 0; c < d2; ++c) {
      int p = c;
      for (int r = c + 1; r < d2; ++r)
        if (std::fabs(a[r + size_t(c) * d2]) > std::fabs(a[p + size_t(c) * d2])) p = r;
      for (int j = 0; j < d2; ++j) {
        std::swap(a[c + size_t(j) * d2], a[p + size_t(j) * d2]);
        std::swap(inv[c + size_t(j) * d2], inv[p + size_t(j) * d2]);
      }
      const double piv = a[c + size_t(c) * d2];
      pmax = std::max(pmax, std::fabs(piv));
      pmin = std::min(pmin, std::fabs(piv));
      require(piv != 0.0, HDG_EINVAL, "singular face block in hdg_project tables");
      for (int j = 0; j < d2; ++j) {
        a[c + size_t(j) * d2] /= piv;
        inv[c + size_t(j) * d2] /= piv;
      }
      for (int r = 0; r < d2; ++r) {
        if (r == c) continue;
        const double m = a[r + size_t(c) * d2];
        if (m == 0.0) continue;
        for (int j = 0; j < d2; ++j) {
          a[r + size_t(j) * d2] -= m * a[c + size_t(j) * d2];
          inv[r + size_t(j) * d2] -= m * inv[c + size_t(j) * d2];
        }
      }
    }
    require(pmin >= 1e-14 * pmax, HDG_EINVAL, "ill-conditioned face block in hdg_project tables");
    std::copy(inv.begin(), inv.end(), out.begin() + size_t(lm) * d2 * d2);
  }
  return out;
}

FieldDev program_field(const hdg_field& f, const char* name) {
  require(f.kind != HDG_FIELD_SAMPLED, HDG_EINVAL,
          std::string("error functionals need CONST or PROGRAM fields (no node samples): ") + name);
  return to_dev(f, name);
}

struct DevBuf {
  void* p = nullptr;
  cudaStream_t s;
  DevBuf(cudaStream_t st, size_t bytes) : s(st) { CUDA_OK(cudaMallocAsync(&p, bytes ? bytes : 8, s)); }
  ~DevBuf() { cudaFreeAsync(p, s); }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

void launch_hdg_project(hdg_ctx* c, int nelt, const GeoDev& geo, const FieldDev* F, double* qx, double* qy,
                        double* qz, double* u) {
  const DevTab& tE = c->tab[2].dev;
  const std::vector<double> wi = face_block_inverses(c->tab[0].host);
  DevBuf dw(c->stream, wi.size() * 8);
  CUDA_OK(cudaMemcpyAsync(dw.p, wi.data(), wi.size() * 8, cudaMemcpyHostToDevice, c->stream));
  set_ll_kernel<<<1, 1, 0, c->stream>>>(c->d_bad + 3, LLONG_MAX);
  const int per_warp = 4 * tE.nq + 4 * tE.nqd + 4 * tE.d3 + 4 * tE.d2 + 32;
  const size_t smem = size_t(kErrWarps) * per_warp * 8;
  CUDA_OK(cudaFuncSetAttribute(hdg_project_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int grid = int(std::min<long>((long(nelt) + kErrWarps - 1) / kErrWarps, long(c->sms) * 16));
  hdg_project_kernel<<<grid, kErrWarps * 32, smem, c->stream>>>(tE, c->tab[0].dev, nelt, geo, F[0], F[1], F[2],
                                                                F[3], dw.as<double>(), qx, qy, qz, u, c->d_bad + 3,
                                                                per_warp);
  CUDA_OK(cudaGetLastError());
  CUDA_OK(cudaMemcpyAsync(c->h_bad + 3, c->d_bad + 3, sizeof(long long), cudaMemcpyDeviceToHost, c->stream));
  CUDA_OK(cudaStreamSynchronize(c->stream));
  if (c->h_bad[3] != LLONG_MAX)
    throw HdgError{HDG_ESINGULAR, "singular projection system on element " + std::to_string(c->h_bad[3])};
}
}  // namespace

extern "C" {

const char* hdg_b200_version(void) { return "hdg_b200 1.0 (sm_100a)"; }
const char* hdg_b200_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------ mesh
int hdg_b200_mesh_box(int nx, int ny, int nz, int bc_rule, double perturb_frac, uint64_t seed,
                      double keep_plane_z, hdg_mesh** out) {
  return guarded([&] {
    require(out != nullptr, HDG_EINVAL, "out is NULL");
    require(bc_rule >= 0 && bc_rule <= 2, HDG_EINVAL, "unknown boundary rule");
    auto m = std::make_unique<hdg_mesh>();
    box_mesh(nx, ny, nz, BoundaryRule(bc_rule), m->m);
    if (perturb_frac > 0) perturb_interior(m->m, nx, ny, nz, perturb_frac, seed, keep_plane_z);
    *out = m.release();
  });
}

int hdg_b200_mesh_create(int nver, const double* h_coords, int nelt, const int* h_elements, int ndir,
                         const int* h_dirichlet, int nneu, const int* h_neumann, hdg_mesh** out) {
  return guarded([&] {
    require(out && nver > 0 && nelt > 0 && ndir >= 0 && nneu >= 0 && h_coords && h_elements,
            HDG_EINVAL, "bad raw mesh arguments");
    auto m = std::make_unique<hdg_mesh>();
    HostMesh& r = m->m;
    r.nver = nver; r.nelt = nelt; r.ndir = ndir; r.nneu = nneu;
    r.coords.assign(h_coords, h_coords + size_t(nver) * 3);
    r.elements.assign(h_elements, h_elements + size_t(nelt) * 4);
    for (int v : r.elements) require(v >= 0 && v < nver, HDG_EMESH, "vertex index out of range");
    if (ndir) r.dirichlet.assign(h_dirichlet, h_dirichlet + size_t(ndir) * 3);
    if (nneu) r.neumann.assign(h_neumann, h_neumann + size_t(nneu) * 3);
    *out = m.release();
  });
}

int hdg_b200_mesh_expand(hdg_mesh* m) {
  return guarded([&] {
    require(m != nullptr, HDG_EINVAL, "mesh is NULL");
    expand_mesh(m->m);
    m->pattern_ready = false;
  });
}

int hdg_b200_mesh_dims(const hdg_mesh* m, int64_t dims[6]) {
  return guarded([&] {
    require(m && dims, HDG_EINVAL, "NULL argument");
    const HostMesh& r = m->m;
    dims[0] = r.nver; dims[1] = r.nelt; dims[2] = r.nfc; dims[3] = r.ndir; dims[4] = r.nneu;
    dims[5] = r.expanded;
  });
}

int hdg_b200_mesh_copy(const hdg_mesh* m, int what, void* dst) {
  return guarded([&] {
    require(m && dst, HDG_EINVAL, "NULL argument");
    const HostMesh& r = m->m;
    auto cp = [&](const auto& v) { std::memcpy(dst, v.data(), v.size() * sizeof(v[0])); };
    switch (what) {
      case HDG_MESH_COORDS: cp(r.coords); break;
      case HDG_MESH_ELEMENTS: cp(r.elements); break;
      case HDG_MESH_DIRICHLET: cp(r.dirichlet); break;
      case HDG_MESH_NEUMANN: cp(r.neumann); break;
      case HDG_MESH_FACES: require(r.expanded, HDG_ESTATE, "mesh not expanded"); cp(r.faces); break;
      case HDG_MESH_FACETYPE: require(r.expanded, HDG_ESTATE, "mesh not expanded"); cp(r.facetype); break;
      case HDG_MESH_FACEBYELE: require(r.expanded, HDG_ESTATE, "mesh not expanded"); cp(r.facebyele); break;
      default: throw HdgError{HDG_EINVAL, "unknown mesh array"};
    }
  });
}

void hdg_b200_mesh_free(hdg_mesh* m) { delete m; }

int hdg_b200_pattern_dims(const hdg_mesh* mc, int64_t* nnbr_total) {
  return guarded([&] {
    require(mc && nnbr_total, HDG_EINVAL, "NULL argument");
    auto* m = const_cast<hdg_mesh*>(mc);
    require(m->m.expanded, HDG_ESTATE, "mesh not expanded");
    if (!m->pattern_ready) { build_pattern(m->m, m->pat); m->pattern_ready = true; }
    *nnbr_total = m->pat.facebase.back();
  });
}

int hdg_b200_pattern_build(const hdg_mesh* mc, int64_t* h_facebase, int* h_nbr, uint8_t* h_slot) {
  return guarded([&] {
    require(mc, HDG_EINVAL, "NULL mesh");
    auto* m = const_cast<hdg_mesh*>(mc);
    require(m->m.expanded, HDG_ESTATE, "mesh not expanded");
    if (!m->pattern_ready) { build_pattern(m->m, m->pat); m->pattern_ready = true; }
    if (h_facebase) std::memcpy(h_facebase, m->pat.facebase.data(), m->pat.facebase.size() * 8);
    if (h_nbr) std::memcpy(h_nbr, m->pat.nbr.data(), m->pat.nbr.size() * 4);
    if (h_slot) std::memcpy(h_slot, m->pat.slot.data(), m->pat.slot.size());
  });
}

int hdg_b200_pattern_build_raw(int nelt, int nfc, const int* h_facebyele, int64_t* nnbr_total,
                               int64_t* h_facebase, int* h_nbr, uint8_t* h_slot) {
  return guarded([&] {
    require(nelt > 0 && nfc > 0 && h_facebyele, HDG_EINVAL, "bad argument");
    SkeletonPattern p;
    build_pattern_raw(nelt, nfc, h_facebyele, p);
    if (nnbr_total) *nnbr_total = p.facebase.back();
    if (h_facebase) std::memcpy(h_facebase, p.facebase.data(), p.facebase.size() * 8);
    if (h_nbr) std::memcpy(h_nbr, p.nbr.data(), p.nbr.size() * 4);
    if (h_slot) std::memcpy(h_slot, p.slot.data(), p.slot.size());
  });
}

// --------------------------------------------------------------- context
int hdg_b200_create(int device, void* stream, hdg_ctx** out) {
  return guarded([&] {
    require(out != nullptr, HDG_EINVAL, "out is NULL");
    auto c = std::make_unique<hdg_ctx>();
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    set_device(c.get());
    CUDA_OK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device));
    // [0..2] build_condense status (reset_build_status_kernel), [3] hdg_project,
    // [4] elements re-solved by the rescue kernel
    CUDA_OK(cudaMalloc(&c->d_bad, 8 * sizeof(long long)));
    CUDA_OK(cudaMallocHost(&c->h_bad, 8 * sizeof(long long)));
    for (int i = 0; i < 8; ++i) c->h_bad[i] = i == 4 ? 0 : LLONG_MAX;
    CUDA_OK(cudaMemcpy(c->d_bad, c->h_bad, 8 * sizeof(long long), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMalloc(&c->d_status, 2 * sizeof(int)));
    CUDA_OK(cudaMallocHost(&c->h_status, 2 * sizeof(int)));
    c->h_status[0] = c->h_status[1] = INT_MAX;
    CUDA_OK(cudaMemcpy(c->d_status, c->h_status, 2 * sizeof(int), cudaMemcpyHostToDevice));
    *out = c.release();
  });
}

void hdg_b200_destroy(hdg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  for (auto& t : c->tab)
    if (t.buf) cudaFree(t.buf);
  if (c->work) cudaFree(c->work);
  if (c->d_adj) cudaFree(c->d_adj);
  if (c->d_zero_T) cudaFree(c->d_zero_T);
  if (c->d_ksamp) cudaFree(c->d_ksamp);
  if (c->d_bsamp) cudaFree(c->d_bsamp);
  if (c->d_cbary) cudaFree(c->d_cbary);
  if (c->d_rescue) cudaFree(c->d_rescue);
  if (c->d_bad) cudaFree(c->d_bad);
  if (c->h_bad) cudaFreeHost(c->h_bad);
  if (c->d_status) cudaFree(c->d_status);
  if (c->h_status) cudaFreeHost(c->h_status);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  delete c;
}

int hdg_b200_set_stream(hdg_ctx* c, void* stream) {
  return guarded([&] {
    require(c != nullptr, HDG_EINVAL, "ctx is NULL");
    c->stream = static_cast<cudaStream_t>(stream);
  });
}

int hdg_b200_set_degree(hdg_ctx* c, int k, int tet_deg, int tri_deg) {
  return guarded([&] {
    require(c != nullptr, HDG_EINVAL, "ctx is NULL");
    require(k >= 0 && k <= 5, HDG_EINVAL, "degree must be in 0..5");
    set_device(c);
    upload_tables(c->tab[0], k, tet_deg, tri_deg);
    c->tab[0].chat_sparse = check_chat_pattern(c->tab[0].host);
    c->tri_deg = tri_deg;
    c->tab[1].ready = false;
    if (c->post_tet_deg >= 0) upload_tables(c->tab[1], k + 1, c->post_tet_deg, tri_deg);
    c->tab[2].ready = c->tab[3].ready = false;
  });
}

int hdg_b200_set_postprocess_rule(hdg_ctx* c, int tet_deg) {
  return guarded([&] {
    require(c && c->tab[0].ready, HDG_ESTATE, "set_degree first");
    set_device(c);
    c->post_tet_deg = tet_deg;
    // degree k+1 tables on the postprocess tet rule; the level's tri rule is
    // reused as in study.cpp:34
    upload_tables(c->tab[1], c->tab[0].host.k + 1, tet_deg, c->tri_deg);
  });
}

int hdg_b200_dims(const hdg_ctx* c, int64_t dims[8]) {
  return guarded([&] {
    require(c && dims && c->tab[0].ready, HDG_ESTATE, "set_degree first");
    const DevTab& t = c->tab[0].dev;
    dims[0] = t.k; dims[1] = t.d3; dims[2] = t.d2; dims[3] = t.nq; dims[4] = t.nqd;
    dims[5] = factor_doubles(t.k);
    dims[6] = c->tab[1].ready ? c->tab[1].dev.nq : 0;
    dims[7] = c->tab[1].ready ? c->tab[1].dev.d3 : 0;
  });
}

namespace {
void copy_table(const HostTables& h, int which, double* dst, int64_t cap) {
    std::vector<double> v;
    auto cat = [&](const auto& arr) { for (auto& m : arr) v.insert(v.end(), m.begin(), m.end()); };
    switch (which) {
      case HDG_TABLE_TET_BARY: v = h.tet_bary; break;
      case HDG_TABLE_TET_W: v = h.tet_w; break;
      case HDG_TABLE_P: v = h.P; break;
      case HDG_TABLE_CHAT: cat(h.Chat); break;
      case HDG_TABLE_WLM: cat(h.Wlm); break;
      case HDG_TABLE_PP: cat(h.PP); break;
      case HDG_TABLE_DD: v = h.DD; break;
      case HDG_TABLE_TRI_BARY: v = h.tri_bary; break;
      case HDG_TABLE_TRI_W: v = h.tri_w; break;
      default: throw HdgError{HDG_EINVAL, "unknown table"};
    }
    require(int64_t(v.size()) <= cap, HDG_EINVAL, "destination too small");
    std::memcpy(dst, v.data(), v.size() * sizeof(double));
}
}  // namespace

int hdg_b200_copy_table(const hdg_ctx* c, int which, double* dst, int64_t cap) {
  return guarded([&] {
    require(c && dst && c->tab[0].ready, HDG_ESTATE, "set_degree first");
    copy_table(c->tab[0].host, which, dst, cap);
  });
}

int hdg_b200_host_table(int k, int tet_deg, int tri_deg, int which, double* dst, int64_t cap) {
  return guarded([&] {
    require(dst != nullptr, HDG_EINVAL, "dst is NULL");
    copy_table(build_host_tables(k, tet_deg, tri_deg), which, dst, cap);
  });
}

// ------------------------------------------------------------------- K1
int hdg_b200_geometry(hdg_ctx* c, int nver, int nelt, int nfc, const double* d_coords,
                      const int* d_elements, const int* d_faces, const int* d_facebyele,
                      const double* d_tau, double tau_const, hdg_geometry* g) {
  return guarded([&] {
    require(c && g && d_coords && d_elements && d_faces && d_facebyele && g->area, HDG_EINVAL,
            "NULL argument");
    require(nver > 0 && nelt > 0 && nfc > 0, HDG_EINVAL, "empty mesh");
    to_geo(g);
    set_device(c);
    const int init[2] = {INT_MAX, INT_MAX};
    std::memcpy(c->h_status, init, sizeof(init));
    CUDA_OK(cudaMemcpyAsync(c->d_status, c->h_status, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    stage_begin(c, 0);
    face_area_kernel<<<(nfc + 255) / 256, 256, 0, c->stream>>>(nver, nfc, d_coords, d_faces, g->area);
    geometry_kernel<<<(nelt + 127) / 128, 128, 0, c->stream>>>(
        nver, nelt, nfc, d_coords, d_elements, d_faces, d_facebyele, d_tau, tau_const, g->area,
        g->volume, g->piola, g->normals, g->perm, g->T, g->verts, c->d_status);
    CUDA_OK(cudaGetLastError());
    stage_end(c, 0);
  });
}

int hdg_b200_upwind_tau(hdg_ctx* c, int nelt, const hdg_geometry* g, hdg_field bx, hdg_field by,
                        hdg_field bz, double* d_tau) {
  return guarded([&] {
    require(c && d_tau && nelt > 0, HDG_EINVAL, "bad argument");
    const GeoDev geo = to_geo(g);
    require(bx.kind != HDG_FIELD_SAMPLED && by.kind != HDG_FIELD_SAMPLED && bz.kind != HDG_FIELD_SAMPLED,
            HDG_EINVAL, "upwind tau needs CONST or PROGRAM fields");
    set_device(c);
    upwind_tau_kernel<<<(nelt + 127) / 128, 128, 0, c->stream>>>(nelt, geo, to_dev(bx, "bx"),
                                                                  to_dev(by, "by"), to_dev(bz, "bz"), d_tau);
    CUDA_OK(cudaGetLastError());
  });
}

int hdg_b200_quad_points(hdg_ctx* c, int nelt, const hdg_geometry* g, int which, double* X, double* Y,
                         double* Z) {
  return guarded([&] {
    require(c && X && Y && Z && (which == 0 || which == 1), HDG_EINVAL, "bad argument");
    require(c->tab[which].ready, HDG_ESTATE, "tables not set");
    const GeoDev geo = to_geo(g);
    set_device(c);
    const DevTab& t = c->tab[which].dev;
    const long n = long(nelt) * t.nq;
    quad_points_kernel<<<int((n + 255) / 256), 256, 0, c->stream>>>(nelt, t.nq, t.bary, geo.verts, X, Y, Z);
    CUDA_OK(cudaGetLastError());
  });
}

// ---------------------------------------------------------------- K2 + K3
int64_t hdg_b200_work_size(const hdg_ctx* c, int nelt) {
  if (!c || !c->tab[0].ready) return -1;
  return int64_t(work_doubles(c->tab[0].dev, nelt) * sizeof(double));
}

int hdg_b200_build_condense(hdg_ctx* c, int nelt, const hdg_geometry* g, hdg_field kappa, hdg_field cf,
                            hdg_field f, double* d_C, double* d_Cf, double* d_factors, void* d_work,
                            int64_t* bad_element) {
  return guarded([&] {
    require(c && d_C && d_Cf && nelt > 0, HDG_EINVAL, "bad argument");
    require(c->tab[0].ready, HDG_ESTATE, "set_degree first");
    const GeoDev geo = to_geo(g);
    const FieldDev fk = to_dev(kappa, "kappa"), fc = to_dev(cf, "c"), ff = to_dev(f, "f");
    set_device(c);
    const DevTab& t = c->tab[0].dev;
    reset_build_status_kernel<<<1, 32, 0, c->stream>>>(c->d_bad);
    c->build_status_pending = true;
    tau_check_kernel<<<int(std::min<long>((long(nelt) + 255) / 256, long(c->sms) * 4)), 256, 0, c->stream>>>(
        nelt, geo.T, c->d_bad);
    GeoDev geo_b = geo;
    if (c->bdm) {  // bdm_blocks ignores tau entirely (local_solver.cpp:36-43): run with T = 0
      require(t.k >= 1, HDG_EINVAL, "the BDM variant needs degree k >= 1");
      if (c->zero_T_len < 4L * nelt) {
        if (c->d_zero_T) cudaFree(c->d_zero_T);
        c->d_zero_T = nullptr;
        CUDA_OK(cudaMalloc(&c->d_zero_T, sizeof(double) * 4 * size_t(nelt)));
        c->zero_T_len = 4L * nelt;
      }
      CUDA_OK(cudaMemsetAsync(c->d_zero_T, 0, sizeof(double) * 4 * size_t(nelt), c->stream));
      geo_b.T = c->d_zero_T;
    }
    double* work = static_cast<double*>(d_work ? d_work : ctx_work(c, work_doubles(t, nelt) * sizeof(double)));
    double* Ms = work;
    double* Ds = Ms + size_t(nelt) * t.nsym;
    double* fv = Ds + size_t(nelt) * t.nsym;
    const int eb = quad_eb(t.nqp);
    const size_t qsmem = quad_smem_bytes(eb, t.nqp);
    const int qgrid = (nelt + eb - 1) / eb;
    const bool any_prog = kappa.kind == HDG_FIELD_PROGRAM || cf.kind == HDG_FIELD_PROGRAM || f.kind == HDG_FIELD_PROGRAM;
    JitKernel jk;
    if (c->jit && any_prog) {
      std::string err;
      jk = jit_quad_kernel(kappa, cf, f, eb, t.nqp, &err);
      if (!jk.fn) c->jit_error = err;
    }
    stage_begin(c, 1);
    bool launched = false;
    if (jk.fn) {
      int nel = nelt, nq = t.nq, nqp = t.nqp, nsym = t.nsym, nsymp = t.nsymp, d3 = t.d3, d3p = t.d3p;
      const double *bary = t.bary, *w = t.w, *As = t.Asym, *Af = t.Af, *vol = geo_b.volume, *T = geo_b.T,
                   *V = geo_b.verts, *sk = kappa.samples, *sc = cf.samples, *sf = f.samples;
      void* args[] = {&nel, &nq, &nqp, &nsym, &nsymp, &d3, &d3p, &bary, &w, &As, &Af, &vol, &T, &V,
                      &sk, &sc, &sf, &Ms, &Ds, &fv};
      std::string err;
      launched = launch_quad_jit(jk.fn, c->stream, qgrid, jk.threads, qsmem, args, &err);
      c->jit_error = launched ? std::string() : err;
    }
    if (!launched) {
      if (eb == 32) {
        CUDA_OK(cudaFuncSetAttribute(quad_build_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(qsmem)));
        quad_build_kernel<32><<<qgrid, 256, qsmem, c->stream>>>(t, nelt, geo_b, fk, fc, ff, Ms, Ds, fv);
      } else {
        CUDA_OK(cudaFuncSetAttribute(quad_build_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(qsmem)));
        quad_build_kernel<16><<<qgrid, 256, qsmem, c->stream>>>(t, nelt, geo_b, fk, fc, ff, Ms, Ds, fv);
      }
    }
    CUDA_OK(cudaGetLastError());
    stage_end(c, 1);
    double* ps = work + pivstat_offset(t, nelt);
    stage_begin(c, 2);
    DISPATCH_K(t.k, launch_condense, c, nelt, geo_b, Ms, Ds, fv, d_C, d_Cf, d_factors, ps);
    stage_end(c, 2);
    stage_begin(c, 6);
    {
      DevTab td = t;
      if (c->bdm) td.nu = td.d3 - td.d2;
      launch_rescue(c, nelt, td, geo_b, Ms, Ds, fv, ps, d_C, d_Cf, d_factors);
    }
    stage_end(c, 6);
    check_bad(c, bad_element);
  });
}

// ------------------------------------------------------------------- K5
int hdg_b200_recover(hdg_ctx* c, int nelt, const hdg_geometry* g, const int* d_facebyele,
                     const double* d_factors, const double* d_uhat, double* d_qx, double* d_qy,
                     double* d_qz, double* d_u) {
  return guarded([&] {
    require(c && d_facebyele && d_factors && d_uhat && d_qx && d_qy && d_qz && d_u && nelt > 0,
            HDG_EINVAL, "bad argument");
    require(c->tab[0].ready, HDG_ESTATE, "set_degree first");
    const GeoDev geo = to_geo(g);
    set_device(c);
    stage_begin(c, 3);
    DISPATCH_K(c->tab[0].dev.k, launch_recover, c, nelt, geo, d_facebyele, d_factors, d_uhat, d_qx, d_qy,
               d_qz, d_u);
    stage_end(c, 3);
  });
}

// ------------------------------------------------------------------- K4
int hdg_b200_pattern_fill(hdg_ctx* c, int nfc, int d2, const int64_t* d_facebase, const int* d_nbr,
                          int64_t* d_rowptr, int* d_colidx) {
  return guarded([&] {
    require(c && d_facebase && d_nbr && d_rowptr && d_colidx && nfc > 0 && d2 > 0, HDG_EINVAL,
            "bad argument");
    set_device(c);
    const long rows = long(nfc) * d2 + 1;
    pattern_fill_kernel<<<int((rows + 255) / 256), 256, 0, c->stream>>>(nfc, d2, d_facebase, d_nbr, d_rowptr,
                                                                      d_colidx);
    CUDA_OK(cudaGetLastError());
  });
}

int hdg_b200_scatter(hdg_ctx* c, int nelt, int d2, const int* d_facebyele, const uint8_t* d_slot,
                     const int64_t* d_facebase, const double* d_C, const double* d_Cf, double* d_vals,
                     double* d_b) {
  return guarded([&] {
    require(c && d_facebyele && d_slot && d_facebase && d_C && d_Cf && d_vals && d_b && nelt > 0 && d2 > 0,
            HDG_EINVAL, "bad argument");
    set_device(c);
    stage_begin(c, 4);
    const int m = 4 * d2;
    const size_t smem = size_t(kScatterWarps) * (m * m + 64) * sizeof(double);
    if (smem <= 200 * 1024) {
      CUDA_OK(cudaFuncSetAttribute(scatter2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      int occ = 0;
      CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, scatter2_kernel, kScatterWarps * 32, smem));
      const long need = (long(nelt) + kScatterWarps - 1) / kScatterWarps;
      const int grid = int(std::min<long>(need, long(c->sms) * std::max(occ, 1)));
      scatter2_kernel<<<grid, kScatterWarps * 32, smem, c->stream>>>(nelt, d2, d_facebyele, d_slot, d_facebase,
                                                                     d_C, d_Cf, d_vals, d_b);
    } else {  // k = 5: the C slice does not fit eight warps' shared memory
      scatter_kernel<<<(nelt + 7) / 8, 256, 0, c->stream>>>(nelt, d2, d_facebyele, d_slot, d_facebase, d_C,
                                                           d_Cf, d_vals, d_b);
    }
    CUDA_OK(cudaGetLastError());
    stage_end(c, 4);
  });
}

int hdg_b200_face_sides(hdg_ctx* c, int nelt, int nfc, const int* d_facebyele, int* d_sides) {
  return guarded([&] {
    require(c && d_facebyele && d_sides && nelt > 0 && nfc > 0, HDG_EINVAL, "bad argument");
    set_device(c);
    const int grid = int(std::min<long>((long(nfc) + 255) / 256, long(c->sms) * 8));
    face_sides_init_kernel<<<grid, 256, 0, c->stream>>>(nfc, d_sides);
    const int grid2 = int(std::min<long>((4L * nelt + 255) / 256, long(c->sms) * 8));
    face_sides_kernel<<<grid2, 256, 0, c->stream>>>(nelt, d_facebyele, d_sides);
    face_sides_fix_kernel<<<grid, 256, 0, c->stream>>>(nfc, d_sides);
    CUDA_OK(cudaGetLastError());
  });
}

int hdg_b200_scatter_faces(hdg_ctx* c, int nfc, int d2, const int* d_sides, const uint8_t* d_slot,
                           const int64_t* d_facebase, const double* d_C, const double* d_Cf, double* d_vals,
                           double* d_b) {
  return guarded([&] {
    require(c && d_sides && d_slot && d_facebase && d_C && d_Cf && d_vals && d_b && nfc > 0, HDG_EINVAL,
            "bad argument");
    set_device(c);
    stage_begin(c, 4);
    auto go = [&](auto kern, int D2) {
      const int m = 4 * D2;
      const size_t per_warp = size_t(2 * m * D2 + 8) * sizeof(double);
      const int nw = int(std::min<size_t>(kFaceRowWarps, (200 * 1024) / per_warp));
      const size_t smem = per_warp * kFaceRowWarps;  // every warp's slice (the surplus warps exit)
      const size_t smem_used = per_warp * nw;
      CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_used)));
      int occ = 0;
      CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kFaceRowWarps * 32, smem_used));
      const long need = (long(nfc) + nw - 1) / nw;
      const int grid = int(std::min<long>(need, long(c->sms) * std::max(occ, 1)));
      (void)smem;
      kern<<<grid, kFaceRowWarps * 32, smem_used, c->stream>>>(nfc, d_sides, d_slot, d_facebase, d_C, d_Cf, d_vals,
                                                            d_b, nw);
    };
    switch (d2) {
      case 1: go(scatter_faces_kernel<1>, 1); break;
      case 3: go(scatter_faces_kernel<3>, 3); break;
      case 6: go(scatter_faces_kernel<6>, 6); break;
      case 10: go(scatter_faces_kernel<10>, 10); break;
      case 15: go(scatter_faces_kernel<15>, 15); break;
      case 21: go(scatter_faces_kernel<21>, 21); break;
      default: throw HdgError{HDG_EINVAL, "scatter_faces: d2 must be dim P_k(triangle), k <= 5"};
    }
    CUDA_OK(cudaGetLastError());
    stage_end(c, 4);
  });
}

// ------------------------------------------------------------------- K6
int hdg_b200_postprocess(hdg_ctx* c, int nelt, const hdg_geometry* g, hdg_field kappa, const double* qx,
                         const double* qy, const double* qz, const double* u, double* ustar) {
  return guarded([&] {
    require(c && qx && qy && qz && u && ustar && nelt > 0, HDG_EINVAL, "bad argument");
    require(c->tab[0].ready && c->tab[1].ready, HDG_ESTATE, "set_postprocess_rule first");
    const GeoDev geo = to_geo(g);
    FieldDev fk = to_dev(kappa, "kappa");
    set_device(c);
    const DevTab& tp = c->tab[1].dev;
    const int n = tp.d3;
    require(n - 1 <= 96, HDG_EINVAL, "postprocess degree too high (d3(k+1) <= 97)");
    int kap_wdiv = 0;
    if (c->jit && kappa.kind == HDG_FIELD_PROGRAM) {
      // a program kappa is sampled once at the P_{k+1} nodes by an NVRTC-compiled
      // sampler, so the postprocess reads samples instead of interpreting it per node
      std::string err;
      // k + 1 <= 4 (postprocess2_kernel): w_q / kappa, no division in K6's epilogue
      const bool wdiv = n <= 40;
      CUfunction fn = wdiv ? jit_sample_wdiv_kernel(kappa, &err) : jit_sample_kernel(kappa, &err);
      if (fn) {
        const size_t len = size_t(tp.nq) * nelt;
        if (c->ksamp_len < len) {
          if (c->d_ksamp) cudaFree(c->d_ksamp);
          c->d_ksamp = nullptr;
          CUDA_OK(cudaMalloc(&c->d_ksamp, len * sizeof(double)));
          c->ksamp_len = len;
        }
        int nel = nelt, nq = tp.nq;
        const double *bary = tp.bary, *V = geo.verts, *wq = tp.w;
        double* out = c->d_ksamp;
        void* args_w[] = {&nel, &nq, &bary, &V, &wq, &out};
        void* args_k[] = {&nel, &nq, &bary, &V, &out};
        void** args = wdiv ? args_w : args_k;
        const int grid = int(std::min<long>((long(len) + 255) / 256, long(c->sms) * 16));
        if (launch_quad_jit(fn, c->stream, grid, 256, 0, args, &err)) {
          fk.kind = HDG_FIELD_SAMPLED;
          fk.samples = c->d_ksamp;
          kap_wdiv = wdiv ? 1 : 0;
          c->jit_error.clear();
        } else {
          c->jit_error = err;
        }
      } else {
        c->jit_error = err;
      }
    }
    if (n <= 40) {  // k <= 3: CTA-batched DMMA version (kernels_post2.cuh)
      const Post2Dims pd(n, tp.nq, c->tab[0].dev.d3);
      const size_t smem2 = size_t(pd.total) * sizeof(double);
      const long need2 = (long(nelt) + kPost2EB - 1) / kPost2EB;
      auto go = [&](auto kern) {
        CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem2)));
        int occ = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kPost2Warps * 32, smem2));
        const int grid2 = int(std::min<long>(need2, long(c->sms) * std::max(occ, 1)));
        kern<<<grid2, kPost2Warps * 32, smem2, c->stream>>>(tp, c->tab[0].dev.d3, nelt, geo, fk, kap_wdiv, qx, qy,
                                                            qz, u, ustar);
      };
      stage_begin(c, 5);
      switch (n - 1) {  // trailing system size for k + 1 = 1..4
        case 3: go(postprocess2_kernel<3>); break;
        case 9: go(postprocess2_kernel<9>); break;
        case 19: go(postprocess2_kernel<19>); break;
        case 34: go(postprocess2_kernel<34>); break;
        default: throw HdgError{HDG_EINVAL, "postprocess: unexpected P_{k+1} dimension"};
      }
      CUDA_OK(cudaGetLastError());
      stage_end(c, 5);
      return;
    }
    const int per_warp = post_per_warp(n, tp.nq, c->tab[0].dev.d3);
    const size_t smem = size_t(kPostWarps) * per_warp * sizeof(double);
    CUDA_OK(cudaFuncSetAttribute(postprocess_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const long need = (long(nelt) + kPostWarps - 1) / kPostWarps;
    const int grid = int(std::min<long>(need, long(c->sms) * 16));
    stage_begin(c, 5);
    postprocess_kernel<<<grid, kPostWarps * 32, smem, c->stream>>>(tp, c->tab[0].dev.d3, nelt, geo, fk, qx, qy, qz,
                                                                  u, ustar, per_warp);
    CUDA_OK(cudaGetLastError());
    stage_end(c, 5);
  });
}

// ------------------------------------------------- device mesh expansion
int hdg_b200_expand_device(hdg_ctx* c, int nver, const double* d_coords, int nelt, const int* d_elements,
                           int ndir, const int* d_dirichlet, int nneu, const int* d_neumann, int* d_faces,
                           uint8_t* d_facetype, int* d_facebyele, int* nfc_out) {
  return guarded([&] {
    require(c && d_coords && d_elements && d_faces && d_facetype && d_facebyele && nver > 0 && nelt > 0 &&
                ndir >= 0 && nneu >= 0 && (ndir == 0 || d_dirichlet) && (nneu == 0 || d_neumann),
            HDG_EINVAL, "bad argument");
    set_device(c);
    expand_device(c->stream, nver, d_coords, nelt, d_elements, ndir, d_dirichlet, nneu, d_neumann, d_faces,
                  d_facetype, d_facebyele);
    if (nfc_out) *nfc_out = expanded_face_count(nelt, ndir, nneu);
  });
}

int hdg_b200_pattern_device(hdg_ctx* c, int nelt, int nfc, const int* d_facebyele, int64_t* d_facebase,
                            int* d_nbr, uint8_t* d_slot, int* maxnbr) {
  return guarded([&] {
    require(c && d_facebyele && d_facebase && d_nbr && d_slot && nelt > 0 && nfc > 0, HDG_EINVAL,
            "bad argument");
    set_device(c);
    const int mx = pattern_device(c->stream, nelt, nfc, d_facebyele, d_facebase, d_nbr, d_slot);
    if (maxnbr) *maxnbr = mx;
  });
}

// ------------------------------------------------------------ K9: solve

int hdg_b200_solve_skeleton(hdg_ctx* c, int nfc, int d2, const int64_t* d_facebase, const int* d_nbr,
                            const double* d_vals, const double* d_b, int ndir, const double* d_ub, double rtol,
                            int maxit, double* d_uhat, hdg_solve_info* info) {
  hdg_solve_info local{};
  hdg_solve_info* inf = info ? info : &local;
  *inf = hdg_solve_info{};
  return guarded([&] {
    require(c && d_facebase && d_nbr && d_vals && d_b && d_uhat && nfc > 0 && ndir >= 0 && ndir <= nfc &&
                (ndir == 0 || d_ub) && rtol > 0.0 && maxit > 0,
            HDG_EINVAL, "bad argument");
    set_device(c);
    switch (d2) {
      case 1: solve_cg<1>(c, nfc, d_facebase, d_nbr, d_vals, d_b, ndir, d_ub, rtol, maxit, d_uhat, inf); break;
      case 3: solve_cg<3>(c, nfc, d_facebase, d_nbr, d_vals, d_b, ndir, d_ub, rtol, maxit, d_uhat, inf); break;
      case 6: solve_cg<6>(c, nfc, d_facebase, d_nbr, d_vals, d_b, ndir, d_ub, rtol, maxit, d_uhat, inf); break;
      case 10: solve_cg<10>(c, nfc, d_facebase, d_nbr, d_vals, d_b, ndir, d_ub, rtol, maxit, d_uhat, inf); break;
      case 15: solve_cg<15>(c, nfc, d_facebase, d_nbr, d_vals, d_b, ndir, d_ub, rtol, maxit, d_uhat, inf); break;
      case 21: solve_cg<21>(c, nfc, d_facebase, d_nbr, d_vals, d_b, ndir, d_ub, rtol, maxit, d_uhat, inf); break;
      default: throw HdgError{HDG_EINVAL, "d2 must be dim2(k) for k <= 5"};
    }
  });
}

// --------------------------------------------- error functionals (§8(f)4)

int hdg_b200_set_error_rule(hdg_ctx* c, int deg) {
  return guarded([&] {
    require(c && c->tab[0].ready, HDG_ESTATE, "set_degree first");
    set_device(c);
    const int k = c->tab[0].host.k;
    const int d = deg >= 0 ? deg : 2 * k + 4;  // postprocess.cpp:182-183
    upload_tables(c->tab[2], k, d, d);
    upload_tables(c->tab[3], k + 1, d, d);
  });
}

int hdg_b200_hdg_project(hdg_ctx* c, int nelt, const hdg_geometry* g, hdg_field qx, hdg_field qy, hdg_field qz,
                         hdg_field u, double* d_qx, double* d_qy, double* d_qz, double* d_u, int64_t* bad_element) {
  if (bad_element) *bad_element = -1;
  return guarded([&] {
    require(c && d_qx && d_qy && d_qz && d_u && nelt > 0, HDG_EINVAL, "bad argument");
    require(c->tab[0].ready && c->tab[2].ready, HDG_ESTATE, "set_error_rule first");
    const GeoDev geo = to_geo(g);
    const FieldDev F[4] = {program_field(qx, "qx"), program_field(qy, "qy"), program_field(qz, "qz"),
                           program_field(u, "u")};
    set_device(c);
    try {
      launch_hdg_project(c, nelt, geo, F, d_qx, d_qy, d_qz, d_u);
    } catch (const HdgError& e) {
      if (e.code == HDG_ESINGULAR && bad_element) *bad_element = c->h_bad[3];
      throw;
    }
  });
}

int hdg_b200_compute_errors(hdg_ctx* c, int nelt, const hdg_geometry* g, int nver, const double* d_coords, int nfc,
                            const int* d_faces, hdg_field qx, hdg_field qy, hdg_field qz, hdg_field u,
                            const double* d_uhat, const double* d_qx, const double* d_qy, const double* d_qz,
                            const double* d_u, const double* d_ustar, hdg_error_report* out) {
  return guarded([&] {
    require(c && out && d_coords && d_faces && d_uhat && d_qx && d_qy && d_qz && d_u && nelt > 0 && nfc > 0 &&
                nver > 0,
            HDG_EINVAL, "bad argument");
    require(c->tab[0].ready && c->tab[2].ready && c->tab[3].ready, HDG_ESTATE, "set_error_rule first");
    require(g && g->area, HDG_EINVAL, "compute_errors needs the face areas (hdg_geometry.area)");
    const GeoDev geo = to_geo(g);
    const FieldDev F[4] = {program_field(qx, "qx"), program_field(qy, "qy"), program_field(qz, "qz"),
                           program_field(u, "u")};
    set_device(c);
    cudaStream_t s = c->stream;
    const DevTab& tE = c->tab[2].dev;
    const DevTab& tE1 = c->tab[3].dev;
    require(tE.nqd <= 64, HDG_EINVAL, "error tri rule too large (nqd <= 64)");
    const int d3 = tE.d3;
    // superconvergence reference (postprocess.cpp:226-232): HDG projection,
    // or the L2 projection when tau == 0 everywhere (BDM)
    double tmax = 0.0;
    {
      std::vector<double> T(size_t(4) * nelt);
      CUDA_OK(cudaMemcpyAsync(T.data(), g->T, T.size() * 8, cudaMemcpyDeviceToHost, s));
      CUDA_OK(cudaStreamSynchronize(s));
      for (double v : T) tmax = std::max(tmax, std::fabs(v));
    }
    DevBuf proj(s, size_t(4) * d3 * nelt * 8);
    double* pq = proj.as<double>();
    double* pu = pq + size_t(3) * d3 * nelt;
    if (tmax == 0.0) {
      const size_t smem = size_t(kErrWarps) * tE.nq * 8;
      CUDA_OK(cudaFuncSetAttribute(l2_project_volume_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(smem)));
      const int grid = int(std::min<long>((long(nelt) + kErrWarps - 1) / kErrWarps, long(c->sms) * 16));
      l2_project_volume_kernel<<<grid, kErrWarps * 32, smem, s>>>(tE, nelt, geo, F[3], pu, tE.nq);
      CUDA_OK(cudaGetLastError());
    } else {
      launch_hdg_project(c, nelt, geo, F, pq, pq + size_t(d3) * nelt, pq + size_t(2) * d3 * nelt, pu);
    }
    const int nblk = c->sms * 4;
    DevBuf part(s, size_t(nblk) * sizeof(ErrSums));
    CUDA_OK(cudaMemsetAsync(part.p, 0, size_t(nblk) * sizeof(ErrSums), s));
    const int per_warp = 4 * d3 + tE1.d3;
    const size_t smem = size_t(kErrWarps) * per_warp * 8;
    CUDA_OK(cudaFuncSetAttribute(volume_errors_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    volume_errors_kernel<<<nblk, kErrWarps * 32, smem, s>>>(tE, tE1, nelt, geo, F[0], F[1], F[2], F[3], d_qx, d_qy,
                                                          d_qz, d_u, d_ustar, pu, part.as<ErrSums>(), per_warp);
    face_errors_kernel<<<nblk, kErrWarps * 32, 0, s>>>(tE, nfc, d_coords, nver, d_faces, g->area, F[3], d_uhat,
                                                       part.as<ErrSums>());
    CUDA_OK(cudaGetLastError());
    std::vector<ErrSums> h(nblk);
    CUDA_OK(cudaMemcpyAsync(h.data(), part.p, size_t(nblk) * sizeof(ErrSums), cudaMemcpyDeviceToHost, s));
    CUDA_OK(cudaStreamSynchronize(s));
    double S[9] = {0};
    for (const auto& b : h)
      for (int j = 0; j < 9; ++j) S[j] += b.v[j];
    auto rel = [](double e2, double n2) { return std::sqrt(n2 > 0 ? e2 / n2 : e2); };
    out->e_q = rel(S[1], S[0]);
    out->e_u = rel(S[3], S[2]);
    out->e_star = d_ustar ? rel(S[4], S[2]) : 0.0;
    out->eps_u = rel(S[5], S[2]);
    out->e_uhat = rel(S[7], S[6]);
    out->eps_uhat = rel(S[8], S[6]);
  });
}

// ----------------------------------------------------------- boundary data
namespace {
void launch_face_moments(hdg_ctx* c, int mode, int f0, int f1, int nver, const double* coords, int nfc,
                         const int* faces, const int* adj, const double* normals, int nelt, const FieldDev& g0,
                         const FieldDev& g1, const FieldDev& g2, double scale, double* out) {
  const DevTab& t = c->tab[0].dev;
  require(t.nqd <= kFaceMaxNodes, HDG_EINVAL, "face rule too large for the face-moment kernel");
  if (f1 <= f0) return;
  const long need = (long(f1 - f0) + kFaceWarps - 1) / kFaceWarps;
  const int grid = int(std::min<long>(need, long(c->sms) * 8));
  face_moments_kernel<<<grid, kFaceWarps * 32, 0, c->stream>>>(t, mode, f0, f1, coords, nver, faces, nfc, adj,
                                                               normals, nelt, g0, g1, g2, scale, out);
  CUDA_OK(cudaGetLastError());
}
}  // namespace

int hdg_b200_dirichlet_project(hdg_ctx* c, int nver, const double* d_coords, int nfc, const int* d_faces,
                               int ndir, hdg_field g, double* d_out) {
  return guarded([&] {
    require(c && d_coords && d_faces && d_out && nver > 0 && nfc > 0 && ndir >= 0 && ndir <= nfc, HDG_EINVAL,
            "bad argument");
    require(c->tab[0].ready, HDG_ESTATE, "set_degree first");
    const FieldDev fg = to_dev(g, "g");
    set_device(c);
    launch_face_moments(c, 0, 0, ndir, nver, d_coords, nfc, d_faces, nullptr, nullptr, 0, fg, fg, fg, 0.5, d_out);
  });
}

int hdg_b200_skeleton_project(hdg_ctx* c, int nver, const double* d_coords, int nfc, const int* d_faces,
                              hdg_field g, double* d_out) {
  return guarded([&] {
    require(c && d_coords && d_faces && d_out && nver > 0 && nfc > 0, HDG_EINVAL, "bad argument");
    require(c->tab[0].ready, HDG_ESTATE, "set_degree first");
    const FieldDev fg = to_dev(g, "g");
    set_device(c);
    launch_face_moments(c, 0, 0, nfc, nver, d_coords, nfc, d_faces, nullptr, nullptr, 0, fg, fg, fg, 0.5, d_out);
  });
}

int hdg_b200_neumann_load(hdg_ctx* c, int nver, const double* d_coords, int nfc, const int* d_faces, int nelt,
                          const int* d_facebyele, const hdg_geometry* g, int ndir, int nneu, hdg_field gx,
                          hdg_field gy, hdg_field gz, double alpha, double* d_b) {
  return guarded([&] {
    require(c && d_coords && d_faces && d_facebyele && d_b && nver > 0 && nfc > 0 && nelt > 0 && ndir >= 0 &&
                nneu >= 0 && ndir + nneu <= nfc,
            HDG_EINVAL, "bad argument");
    require(c->tab[0].ready, HDG_ESTATE, "set_degree first");
    require(g && g->normals, HDG_EINVAL, "neumann_load needs the element normals");
    const FieldDev fx = to_dev(gx, "gx"), fy = to_dev(gy, "gy"), fz = to_dev(gz, "gz");
    set_device(c);
    if (nneu == 0) return;
    const int nbdy = ndir + nneu;
    if (c->adj_len < nbdy) {
      if (c->d_adj) cudaFree(c->d_adj);
      c->d_adj = nullptr;
      CUDA_OK(cudaMalloc(&c->d_adj, size_t(nbdy) * sizeof(int)));
      c->adj_len = nbdy;
    }
    boundary_adjacency_kernel<<<int((4L * nelt + 255) / 256), 256, 0, c->stream>>>(nelt, d_facebyele, nbdy,
                                                                                   c->d_adj);
    CUDA_OK(cudaGetLastError());
    launch_face_moments(c, 1, ndir, nbdy, nver, d_coords, nfc, d_faces, c->d_adj, g->normals, nelt, fx, fy, fz,
                        alpha, d_b);
  });
}

// ------------------------------------------------------------------- K7
int hdg_b200_convection_block(hdg_ctx* c, int nelt, const hdg_geometry* g, hdg_field bx, hdg_field by,
                              hdg_field bz, double* vol, double* dp, double* dd) {
  return guarded([&] {
    require(c && vol && dp && dd && nelt > 0, HDG_EINVAL, "bad argument");
    require(c->tab[0].ready, HDG_ESTATE, "set_degree first");
    require(bx.kind != HDG_FIELD_SAMPLED && by.kind != HDG_FIELD_SAMPLED && bz.kind != HDG_FIELD_SAMPLED,
            HDG_EINVAL, "convection block needs CONST or PROGRAM fields (face nodes are not sampled)");
    const GeoDev geo = to_geo(g);
    set_device(c);
    const DevTab& t = c->tab[0].dev;
    if (t.Aconv) {  // k <= 3: the DMMA kernels (kernels_conv3.cuh, k <= 2; kernels_conv2.cuh, k = 3)
      const Conv2Dims cd(t.d3, t.d2, t.nq, t.nqd);
      // program beta components are sampled once per point by an NVRTC-compiled
      // sampler (the volume nodes, then the element-parametrised face points),
      // so the kernel reads samples instead of interpreting the programs
      FieldDev fb[3] = {to_dev(bx, "bx"), to_dev(by, "by"), to_dev(bz, "bz")};
      const hdg_field* hb[3] = {&bx, &by, &bz};
      const int npts = t.nq + 4 * t.nqd;
      if (c->jit && (bx.kind == HDG_FIELD_PROGRAM || by.kind == HDG_FIELD_PROGRAM || bz.kind == HDG_FIELD_PROGRAM)) {
        if (c->cbary_k != t.k) {
          if (c->d_cbary) cudaFree(c->d_cbary);
          c->d_cbary = nullptr;
          CUDA_OK(cudaMalloc(&c->d_cbary, sizeof(double) * 4 * npts));
          conv_points_kernel<<<1, 256, 0, c->stream>>>(t, c->d_cbary);
          CUDA_OK(cudaGetLastError());
          c->cbary_k = t.k;
        }
        const size_t len = size_t(3) * npts * nelt;
        if (c->bsamp_len < len) {
          if (c->d_bsamp) cudaFree(c->d_bsamp);
          c->d_bsamp = nullptr;
          CUDA_OK(cudaMalloc(&c->d_bsamp, len * sizeof(double)));
          c->bsamp_len = len;
        }
        std::string err;
        CUfunction fn = jit_sample3_kernel(hb, &err);  // all program components in one pass
        if (fn) {
          int nel = nelt, np = npts;
          const double *bary = c->d_cbary, *V = geo.verts;
          double* o[3];
          for (int h = 0; h < 3; ++h) o[h] = c->d_bsamp + size_t(h) * npts * nelt;
          void* args[] = {&nel, &np, &bary, &V, &o[0], &o[1], &o[2]};
          const int grid = int(std::min<long>((long(npts) * nelt + 255) / 256, long(c->sms) * 16));
          if (launch_quad_jit(fn, c->stream, grid, 256, 0, args, &err)) {
            for (int h = 0; h < 3; ++h)
              if (hb[h]->kind == HDG_FIELD_PROGRAM) {
                fb[h].kind = HDG_FIELD_SAMPLED;
                fb[h].samples = o[h];
              }
            c->jit_error.clear();
          } else {
            c->jit_error = err;
          }
        } else {
          c->jit_error = err;
        }
      }
      const size_t smem = size_t(cd.total) * sizeof(double);
      auto go3 = [&](auto kern, auto dims) -> bool {  // one warp per element (kernels_conv3.cuh)
        using Dm = decltype(dims);
        if (t.nq != Dm::NQ || t.nqd != Dm::NQD) return false;  // another rule: the generic kernels
        constexpr int NW = 16;
        const size_t smem3 = size_t(Dm::CTA_EXTRA + NW * Dm::PER_WARP) * sizeof(double);
        CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem3)));
        const long need = (long(nelt) + NW - 1) / NW;
        const int grid = int(std::min<long>(need, long(c->sms)));
        kern<<<grid, NW * 32, smem3, c->stream>>>(t, nelt, geo, fb[0], fb[1], fb[2], vol, dp, dd);
        CUDA_OK(cudaGetLastError());
        return true;
      };
      bool done3 = false;
      switch (t.k) {
        case 0: done3 = go3(convection3_kernel<0>, Conv3Dims<0>{}); break;
        case 1: done3 = go3(convection3_kernel<1>, Conv3Dims<1>{}); break;
        case 2: done3 = go3(convection3_kernel<2>, Conv3Dims<2>{}); break;
        default: break;
      }
      if (done3) return;
      auto go = [&](auto kern) {
        CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        int occ = 0;
        CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kConv2Threads, smem));
        const long need = (long(nelt) + kConv2EB - 1) / kConv2EB;
        const int grid = int(std::min<long>(need, long(c->sms) * std::max(occ, 1)));
        kern<<<grid, kConv2Threads, smem, c->stream>>>(t, nelt, geo, fb[0], fb[1], fb[2], npts, vol, dp, dd);
      };
      switch (t.k) {
        case 0: go(convection2_kernel<0>); break;
        case 1: go(convection2_kernel<1>); break;
        case 2: go(convection2_kernel<2>); break;
        default: go(convection2_kernel<3>); break;
      }
      CUDA_OK(cudaGetLastError());
      return;
    }
    const int per_warp = 3 * t.nq + 4 * t.nqd + 32;
    const int nw = warps_for(size_t(per_warp) * 8);
    const size_t smem = size_t(nw) * per_warp * sizeof(double);
    CUDA_OK(cudaFuncSetAttribute(convection_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    const int grid = int(std::min<long>((long(nelt) + nw - 1) / nw, long(c->sms) * 8));
    convection_kernel<<<grid, nw * 32, smem, c->stream>>>(t, nelt, geo, to_dev(bx, "bx"), to_dev(by, "by"),
                                                         to_dev(bz, "bz"), vol, dp, dd, per_warp);
    CUDA_OK(cudaGetLastError());
  });
}

int hdg_b200_element_matrices(hdg_ctx* c, int nelt, const hdg_geometry* g, hdg_field kappa, hdg_field cf,
                              hdg_field f, hdg_element_matrices* out) {
  return guarded([&] {
    require(c && out && nelt > 0, HDG_EINVAL, "bad argument");
    require(c->tab[0].ready, HDG_ESTATE, "set_degree first");
    const GeoDev geo = to_geo(g);
    set_device(c);
    const DevTab& t = c->tab[0].dev;
    const int per_warp = 3 * t.nq + 32;
    const int nw = warps_for(size_t(per_warp) * 8);
    const size_t smem = size_t(nw) * per_warp * sizeof(double);
    CUDA_OK(cudaFuncSetAttribute(element_matrices_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    EmsOut o{out->Mkinv, out->Mc, out->Cx, out->Cy, out->Cz, out->tauPP, out->tauDP,
             out->nxDP, out->nyDP, out->nzDP, out->tauDD, out->fvec};
    const int grid = int(std::min<long>((long(nelt) + nw - 1) / nw, long(c->sms) * 8));
    element_matrices_kernel<<<grid, nw * 32, smem, c->stream>>>(t, nelt, geo, to_dev(kappa, "kappa"),
                                                               to_dev(cf, "c"), to_dev(f, "f"), o, per_warp);
    CUDA_OK(cudaGetLastError());
  });
}

int hdg_b200_set_timing(hdg_ctx* c, int enabled) {
  return guarded([&] {
    require(c != nullptr, HDG_EINVAL, "ctx is NULL");
    set_device(c);
    if (enabled && !c->ev[0])
      for (auto& e : c->ev) CUDA_OK(cudaEventCreate(&e));
    c->timing = enabled != 0;
  });
}

int hdg_b200_stage_times(hdg_ctx* c, double ms[HDG_NSTAGES]) {
  return guarded([&] {
    require(c && ms, HDG_EINVAL, "NULL argument");
    set_device(c);
    for (int s = 0; s < HDG_NSTAGES; ++s) {
      ms[s] = -1.0;
      if (!c->pending[s]) continue;
      CUDA_OK(cudaEventSynchronize(c->ev[2 * s + 1]));
      float t = 0.f;
      CUDA_OK(cudaEventElapsedTime(&t, c->ev[2 * s], c->ev[2 * s + 1]));
      ms[s] = t;
      c->pending[s] = false;
    }
  });
}

int hdg_b200_set_jit(hdg_ctx* c, int enabled) {
  return guarded([&] {
    require(c != nullptr, HDG_EINVAL, "ctx is NULL");
    c->jit = enabled != 0;
  });
}

const char* hdg_b200_jit_status(const hdg_ctx* c) { return c ? c->jit_error.c_str() : ""; }

int hdg_b200_set_rescue_screen(hdg_ctx* c, double screen) {
  return guarded([&] {
    require(c != nullptr && screen >= 0.0, HDG_EINVAL, "screen must be >= 0");
    c->rescue_screen = screen;
  });
}

int hdg_b200_rescued_elements(hdg_ctx* c, int64_t* count) {
  return guarded([&] {
    require(c && count, HDG_EINVAL, "NULL argument");
    set_device(c);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    long long v = 0;
    CUDA_OK(cudaMemcpy(&v, c->d_bad + 4, sizeof(long long), cudaMemcpyDeviceToHost));
    *count = v;
  });
}

int hdg_b200_set_tau_allow_zero(hdg_ctx* c, int enabled) {
  return guarded([&] {
    require(c != nullptr, HDG_EINVAL, "ctx is NULL");
    c->tau_allow_zero = enabled != 0;
  });
}

int hdg_b200_set_bdm(hdg_ctx* c, int enabled) {
  return guarded([&] {
    require(c != nullptr, HDG_EINVAL, "ctx is NULL");
    c->bdm = enabled != 0;
  });
}

int hdg_b200_set_recover_variant(hdg_ctx* c, int variant) {
  return guarded([&] {
    require(c != nullptr && (variant == 2 || variant == 3), HDG_EINVAL, "recover variant must be 2 or 3");
    c->recover_variant = variant;
  });
}

int hdg_b200_set_chat_sparsity(hdg_ctx* c, int enabled, int* active) {
  return guarded([&] {
    require(c && c->tab[0].ready, HDG_ESTATE, "set_degree first");
    c->tab[0].chat_sparse = enabled != 0 && check_chat_pattern(c->tab[0].host);
    if (active) *active = c->tab[0].chat_sparse ? 1 : 0;
  });
}

// ------------------------------------------- interface exchange (§8(e))
}  // extern "C"

struct hdg_exchange {
  int device = 0;
  int d2 = 0;
  struct Peer {
    int rank = 0, nfaces = 0;
    long n = 0, nv = 0;           // entries, of which value positions
    int64_t* idx = nullptr;       // device positions (values | b)
    double* send = nullptr;       // device staging
    double* recv = nullptr;
  };
  std::vector<Peer> peers;
  ~hdg_exchange() {
    cudaSetDevice(device);
    for (auto& p : peers) {
      if (p.idx) cudaFree(p.idx);
      if (p.send) cudaFree(p.send);
      if (p.recv) cudaFree(p.recv);
    }
  }
};

namespace {
void require_nccl() {
  const NcclApi& a = nccl_api();
  if (!a.ok) throw HdgError{HDG_ENCCL, a.why};
}
void nccl_ok(int rc, const char* what) {
  if (rc != 0) throw HdgError{HDG_ENCCL, std::string(what) + ": " + nccl_api().errorString(rc)};
}
int exchange_grid(const hdg_ctx* c, long n) { return int(std::max<long>(1, std::min<long>((n + 255) / 256, c->sms * 4L))); }
}  // namespace

extern "C" {

int hdg_b200_exchange_positions(int nfc, int d2, const int64_t* h_facebase, const int* h_nbr, int nfaces,
                                const int* h_faces, int64_t* h_pos) {
  return guarded([&] {
    require(nfc > 0 && d2 > 0 && h_facebase && h_nbr && nfaces >= 0 && (nfaces == 0 || (h_faces && h_pos)),
            HDG_EINVAL, "bad argument");
    std::vector<int64_t> pos;
    std::string err;
    require(interface_positions(nfc, d2, h_facebase, h_nbr, nfaces, h_faces, pos, &err), HDG_EINVAL, err);
    std::copy(pos.begin(), pos.end(), h_pos);
  });
}

int hdg_b200_exchange_plan(hdg_ctx* c, int nfc, int d2, const int64_t* h_facebase, const int* h_nbr, int npeers,
                           const int* h_peer_rank, const int* h_peer_nfaces, const int* h_faces,
                           hdg_exchange** out) {
  return guarded([&] {
    require(c && out && nfc > 0 && d2 > 0 && h_facebase && h_nbr && npeers >= 0 &&
                (npeers == 0 || (h_peer_rank && h_peer_nfaces && h_faces)),
            HDG_EINVAL, "bad argument");
    set_device(c);
    auto plan = std::make_unique<hdg_exchange>();
    plan->device = c->device;
    plan->d2 = d2;
    const int* fp = h_faces;
    for (int q = 0; q < npeers; ++q) {
      hdg_exchange::Peer p;
      p.rank = h_peer_rank[q];
      p.nfaces = h_peer_nfaces[q];
      require(p.nfaces >= 0, HDG_EINVAL, "negative interface face count");
      std::vector<int64_t> pos;
      std::string err;
      require(interface_positions(nfc, d2, h_facebase, h_nbr, p.nfaces, fp, pos, &err), HDG_EINVAL, err);
      fp += p.nfaces;
      p.n = long(pos.size());
      p.nv = long(p.nfaces) * d2 * d2;
      if (p.n) {
        CUDA_OK(cudaMalloc(&p.idx, size_t(p.n) * sizeof(int64_t)));
        CUDA_OK(cudaMalloc(&p.send, size_t(p.n) * sizeof(double)));
        CUDA_OK(cudaMalloc(&p.recv, size_t(p.n) * sizeof(double)));
        CUDA_OK(cudaMemcpy(p.idx, pos.data(), size_t(p.n) * sizeof(int64_t), cudaMemcpyHostToDevice));
      }
      plan->peers.push_back(p);
    }
    *out = plan.release();
  });
}

void hdg_b200_exchange_free(hdg_exchange* plan) { delete plan; }

int hdg_b200_exchange_pack(hdg_ctx* c, const hdg_exchange* plan, int peer, const double* d_vals, const double* d_b,
                           double* d_buf) {
  return guarded([&] {
    require(c && plan && peer >= 0 && peer < int(plan->peers.size()) && d_vals && d_b && d_buf, HDG_EINVAL,
            "bad argument");
    set_device(c);
    const auto& p = plan->peers[peer];
    if (!p.n) return;
    exchange_pack_kernel<<<exchange_grid(c, p.n), 256, 0, c->stream>>>(p.n, p.idx, d_vals, p.nv, d_b, d_buf);
    CUDA_OK(cudaGetLastError());
  });
}

int hdg_b200_exchange_unpack_add(hdg_ctx* c, const hdg_exchange* plan, int peer, const double* d_buf,
                                 double* d_vals, double* d_b) {
  return guarded([&] {
    require(c && plan && peer >= 0 && peer < int(plan->peers.size()) && d_vals && d_b && d_buf, HDG_EINVAL,
            "bad argument");
    set_device(c);
    const auto& p = plan->peers[peer];
    if (!p.n) return;
    exchange_unpack_add_kernel<<<exchange_grid(c, p.n), 256, 0, c->stream>>>(p.n, p.idx, d_buf, p.nv, d_vals, d_b);
    CUDA_OK(cudaGetLastError());
  });
}

int hdg_b200_exchange_interface(hdg_ctx* c, const hdg_exchange* plan, void* comm, double* d_vals, double* d_b) {
  return guarded([&] {
    require(c && plan && d_vals && d_b, HDG_EINVAL, "bad argument");
    set_device(c);
    if (plan->peers.empty()) return;
    require(comm != nullptr, HDG_EINVAL, "NULL communicator");
    require_nccl();
    const NcclApi& a = nccl_api();
    for (const auto& p : plan->peers)
      if (p.n) exchange_pack_kernel<<<exchange_grid(c, p.n), 256, 0, c->stream>>>(p.n, p.idx, d_vals, p.nv, d_b, p.send);
    CUDA_OK(cudaGetLastError());
    nccl_ok(a.groupStart(), "ncclGroupStart");
    for (const auto& p : plan->peers) {
      if (!p.n) continue;
      nccl_ok(a.send(p.send, size_t(p.n), kNcclDouble, p.rank, comm, c->stream), "ncclSend");
      nccl_ok(a.recv(p.recv, size_t(p.n), kNcclDouble, p.rank, comm, c->stream), "ncclRecv");
    }
    nccl_ok(a.groupEnd(), "ncclGroupEnd");
    for (const auto& p : plan->peers)
      if (p.n)
        exchange_unpack_add_kernel<<<exchange_grid(c, p.n), 256, 0, c->stream>>>(p.n, p.idx, p.recv, p.nv, d_vals,
                                                                                 d_b);
    CUDA_OK(cudaGetLastError());
  });
}

int hdg_b200_nccl_get_unique_id(unsigned char id[128]) {
  return guarded([&] {
    require(id != nullptr, HDG_EINVAL, "NULL id");
    require_nccl();
    NcclApi::UniqueId u;
    nccl_ok(nccl_api().getUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, 128);
  });
}

int hdg_b200_nccl_comm_init(hdg_ctx* c, int nranks, int rank, const unsigned char id[128], void** comm) {
  return guarded([&] {
    require(c && id && comm && nranks > 0 && rank >= 0 && rank < nranks, HDG_EINVAL, "bad argument");
    set_device(c);
    require_nccl();
    NcclApi::UniqueId u;
    std::memcpy(u.internal, id, 128);
    nccl_ok(nccl_api().commInitRank(comm, nranks, u, rank), "ncclCommInitRank");
  });
}

int hdg_b200_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    if (!comm) return;
    require_nccl();
    nccl_ok(nccl_api().commDestroy(comm), "ncclCommDestroy");
  });
}

#ifdef HDG_PHASE_TIMING
extern "C" int hdg_b200_debug_phase_clocks(long long* out) {
  return guarded([&] { CUDA_OK(cudaMemcpyFromSymbol(out, g_phase_clk, sizeof(g_phase_clk))); });
}
#endif

int hdg_b200_synchronize(hdg_ctx* c) {
  return guarded([&] {
    require(c != nullptr, HDG_EINVAL, "ctx is NULL");
    set_device(c);
    CUDA_OK(cudaStreamSynchronize(c->stream));
    CUDA_OK(cudaGetLastError());
    CUDA_OK(cudaMemcpy(c->h_status, c->d_status, 2 * sizeof(int), cudaMemcpyDeviceToHost));
    require(c->h_status[0] == INT_MAX, HDG_EMESH,
            "element " + std::to_string(c->h_status[0]) + " has non-positive orientation");
    require(c->h_status[1] == INT_MAX, HDG_EMESH, "face vertex triples do not match as sets");
    // deferred status of the last build_condense run without bad_element
    // (reported once)
    if (c->build_status_pending) {
      CUDA_OK(cudaMemcpy(c->h_bad, c->d_bad, 3 * sizeof(long long), cudaMemcpyDeviceToHost));
      c->build_status_pending = false;
      raise_build_status(c, nullptr);
    }
  });
}

}  // extern "C"
