// Interface-face exchange between z-slabs over NCCL.
//
// Each rank scatters its slab into a slab-local CSR. Two tets share at most
// one face, so off-diagonal face blocks never straddle ranks: the only shared
// entries of the global system are the interface faces' d2 x d2 diagonal
// blocks of H and their d2 entries of b (assemble, global_system.cpp:31-56,
// sums both sides' triplets in setFromTriplets). A plan holds, per neighbour
// rank, the CSR / b positions of those entries (interface faces in ascending
// global order on both sides, so the two lists pair up entry by entry); the
// exchange gathers them into a send buffer, runs one grouped ncclSend /
// ncclRecv per neighbour on the context stream, and adds what it receives.
// Both sides end with a + b == b + a: bit-identical to the single-GPU
// assembly. NCCL is resolved at run time (dlopen of libnccl.so.2, the copy
// torch already loaded if any), so the library loads without it.
#pragma once

#include <dlfcn.h>

#include <cstdint>
#include <string>
#include <vector>

namespace hdgb {

// ---- NCCL entry points (types restated from nccl.h: the ABI is stable)
struct NcclApi {
  using Comm = void*;
  struct UniqueId { char internal[128]; };
  int (*getUniqueId)(UniqueId*) = nullptr;
  int (*commInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*commDestroy)(Comm) = nullptr;
  int (*send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*groupStart)() = nullptr;
  int (*groupEnd)() = nullptr;
  const char* (*errorString)(int) = nullptr;
  bool ok = false;
  std::string why;
};
constexpr int kNcclDouble = 8;  // ncclFloat64

inline NcclApi& nccl_api() {
  static NcclApi a = [] {
    NcclApi r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      r.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return r;
    }
    auto get = [&](const char* n, auto& fn) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, n));
      return fn != nullptr;
    };
    r.ok = get("ncclGetUniqueId", r.getUniqueId) && get("ncclCommInitRank", r.commInitRank) &&
           get("ncclCommDestroy", r.commDestroy) && get("ncclSend", r.send) && get("ncclRecv", r.recv) &&
           get("ncclGroupStart", r.groupStart) && get("ncclGroupEnd", r.groupEnd) &&
           get("ncclGetErrorString", r.errorString);
    if (!r.ok) r.why = "libnccl.so.2 lacks a required entry point";
    return r;
  }();
  return a;
}

// ---- device side
__global__ void exchange_pack_kernel(long n, const int64_t* __restrict__ idx, const double* __restrict__ vals,
                                     long nv, const double* __restrict__ b, double* __restrict__ out) {
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x)
    out[i] = i < nv ? vals[idx[i]] : b[idx[i]];
}

__global__ void exchange_unpack_add_kernel(long n, const int64_t* __restrict__ idx, const double* __restrict__ in,
                                           long nv, double* __restrict__ vals, double* __restrict__ b) {
  for (long i = long(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += long(gridDim.x) * blockDim.x) {
    double* dst = i < nv ? vals + idx[i] : b + idx[i];
    *dst += in[i];
  }
}

// ---- host side: positions of interface entries in the slab-local CSR
// Face f's block row is one contiguous run of nb * d2 * d2 values starting at
// facebase[f] * d2 * d2, row i of the run holding nb blocks of d2 columns in
// the ascending neighbour order of nbr (pattern_fill_kernel); its own
// diagonal block is the slot where nbr[f][s] == f. b's entries are f*d2 + i.
// Per face: d2*d2 value positions (row-major within the block), then the d2
// b positions come after all faces' value positions.
inline bool interface_positions(int nfc, int d2, const int64_t* facebase, const int* nbr, int nfaces,
                                const int* faces, std::vector<int64_t>& out, std::string* err) {
  out.clear();
  out.reserve(size_t(nfaces) * (d2 * d2 + d2));
  for (int a = 0; a < nfaces; ++a) {
    const int f = faces[a];
    if (f < 0 || f >= nfc) {
      if (err) *err = "interface face id out of range";
      return false;
    }
    const int nb = int(facebase[f + 1] - facebase[f]);
    int self = -1;
    for (int s = 0; s < nb && s < 8; ++s)
      if (nbr[size_t(f) * 8 + s] == f) self = s;
    if (self < 0) {
      if (err) *err = "face missing from its own neighbour list";
      return false;
    }
    const int64_t base = facebase[f] * int64_t(d2) * d2;
    for (int i = 0; i < d2; ++i)
      for (int j = 0; j < d2; ++j) out.push_back(base + int64_t(i) * nb * d2 + int64_t(self) * d2 + j);
  }
  for (int a = 0; a < nfaces; ++a)
    for (int i = 0; i < d2; ++i) out.push_back(int64_t(faces[a]) * d2 + i);
  return true;
}

}  // namespace hdgb
