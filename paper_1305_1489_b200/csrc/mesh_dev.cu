// GPU mesh expansion and skeleton pattern, bit-exact with the
// host restatement in host_mesh.cpp and with proj/src/mesh.cpp:74-171 and
// global_system.cpp:31-56.
//
// expand: every element face occurrence (K, l) gets the 63-bit key of its
// sorted vertex triple (21 bits per vertex id, so integer order ==
// std::map's lexicographic order of the triples). A stable radix sort of
// (key, 4K + l) groups the occurrences of each face with the lowest element
// first. Boundary rows are matched by binary search; the unmatched groups
// are the interior faces, numbered after all boundary faces in key order and
// parametrised by their lowest element's occurrence. The reference's checks
// become error codes with the reference's precedence (orientation, then
// boundary rows in input order, then interior faces in key order).
//
// pattern: per face the sorted, de-duplicated faces of its (one or two)
// elements; per element the slot of each (l1, l2) pair in row face l1's
// list; facebase = exclusive scan of the list lengths.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <string>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "host_internal.hpp"
#include "mesh_dev.hpp"

namespace hdgb {

namespace {

#define MCUDA(call)                                                                 \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) throw CudaError(std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kKeyBits = 21;  // per vertex id
// error word: (rank << 4) | code, minimum wins (the reference's first failure)
enum : unsigned long long {
  kErrNone = ~0ull,
  kErrNoMatch = 1,       // boundary face matches no element face
  kErrBdyShared = 2,     // boundary face shared by more than one element
  kErrTwice = 3,         // boundary face listed twice
  kErrUnlisted = 4,      // element face on the boundary is not listed
  kErrInterior3 = 5,     // interior face shared by more than two elements
  kErrOrient = 6,        // element K has non-positive orientation
  kErrCount = 7,         // face count identity violated
  kErrRange = 8,         // vertex id out of range
  kErrPatFace = 9,       // facebyele entry out of range
  kErrPat3 = 10,         // face belongs to more than two elements
};

__device__ __forceinline__ void raise(unsigned long long* err, unsigned long long rank, unsigned long long code) {
  atomicMin(err, (rank << 4) | code);
}

__device__ __forceinline__ unsigned long long tri_key(int a, int b, int c) {
  int t;
  if (a > b) { t = a; a = b; b = t; }
  if (b > c) { t = b; b = c; c = t; }
  if (a > b) { t = a; a = b; b = t; }
  return (static_cast<unsigned long long>(a) << (2 * kKeyBits)) |
         (static_cast<unsigned long long>(b) << kKeyBits) | static_cast<unsigned long long>(c);
}

__constant__ int cLocalFace[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {3, 1, 2}};

// orientation (mesh.cpp:79-81) + occurrence keys
__global__ void occ_keys_kernel(int nver, const double* __restrict__ X, int nelt, const int* __restrict__ el,
                                unsigned long long* __restrict__ keys, int* __restrict__ vals,
                                unsigned long long* err) {
  const long K = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (K >= nelt) return;
  int v[4];
  bool ok = true;
  for (int c = 0; c < 4; ++c) {
    v[c] = el[K + long(c) * nelt];
    ok = ok && v[c] >= 0 && v[c] < nver;
  }
  if (!ok) {
    raise(err, 0, kErrRange);
    for (int l = 0; l < 4; ++l) { keys[4 * K + l] = 0; vals[4 * K + l] = int(4 * K + l); }
    return;
  }
  double B[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) B[r][c] = X[v[c + 1] + long(r) * nver] - X[v[0] + long(r) * nver];
  const double det = B[0][0] * (B[1][1] * B[2][2] - B[2][1] * B[1][2]) -
                     B[1][0] * (B[0][1] * B[2][2] - B[2][1] * B[0][2]) +
                     B[2][0] * (B[0][1] * B[1][2] - B[1][1] * B[0][2]);
  if (!(det > 0)) raise(err, 1 + K, kErrOrient);
  for (int l = 0; l < 4; ++l) {
    keys[4 * K + l] = tri_key(v[cLocalFace[l][0]], v[cLocalFace[l][1]], v[cLocalFace[l][2]]);
    vals[4 * K + l] = int(4 * K + l);
  }
}

__global__ void heads_kernel(long n, const unsigned long long* __restrict__ keys, int* __restrict__ head) {
  const long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// seg_id = inclusive scan of head, minus one
__global__ void seg_start_kernel(long n, const int* __restrict__ head, const int* __restrict__ seg_incl,
                                 int* __restrict__ seg_start, int* __restrict__ nuniq,
                                 int* __restrict__ first_row) {
  const long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int u = seg_incl[i] - 1;
  if (head[i]) {
    seg_start[u] = int(i);
    first_row[u] = INT_MAX;
  }
  if (i == n - 1) {
    seg_start[u + 1] = int(n);
    *nuniq = u + 1;
  }
}

__device__ long lower_bound_key(const unsigned long long* keys, long n, unsigned long long key) {
  long lo = 0, hi = n;
  while (lo < hi) {
    const long mid = (lo + hi) >> 1;
    if (keys[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// boundary row b (Dirichlet rows, then Neumann rows) -> its group
__global__ void boundary_match_kernel(int ndir, const int* __restrict__ dir, int nneu, const int* __restrict__ neu,
                                      int nver, long nocc, const unsigned long long* __restrict__ keys,
                                      const int* __restrict__ seg_incl, const int* __restrict__ seg_start,
                                      int* __restrict__ row_seg, int* __restrict__ first_row, long rank0,
                                      unsigned long long* err) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= ndir + nneu) return;
  const bool d = b < ndir;
  const int r = d ? b : b - ndir, nr = d ? ndir : nneu;
  const int* rows = d ? dir : neu;
  const int a0 = rows[r], a1 = rows[r + nr], a2 = rows[r + 2 * nr];
  row_seg[b] = -1;
  if (a0 < 0 || a0 >= nver || a1 < 0 || a1 >= nver || a2 < 0 || a2 >= nver) {
    raise(err, rank0 + b, kErrNoMatch);
    return;
  }
  const unsigned long long key = tri_key(a0, a1, a2);
  const long p = lower_bound_key(keys, nocc, key);
  if (p == nocc || keys[p] != key) {
    raise(err, rank0 + b, kErrNoMatch);
    return;
  }
  const int u = seg_incl[p] - 1;
  if (seg_start[u + 1] - seg_start[u] != 1) {
    raise(err, rank0 + b, kErrBdyShared);
    return;
  }
  row_seg[b] = u;
  atomicMin(&first_row[u], b);
}

__global__ void boundary_twice_kernel(int nbdy, const int* __restrict__ row_seg, const int* __restrict__ first_row,
                                      long rank0, unsigned long long* err) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbdy) return;
  const int u = row_seg[b];
  if (u >= 0 && first_row[u] != b) raise(err, rank0 + b, kErrTwice);
}

// interior groups: counts checked, flag for the numbering scan (size nocc: tail zero)
__global__ void interior_flag_kernel(long nocc, const int* __restrict__ nuniq, const int* __restrict__ seg_start,
                                     const int* __restrict__ first_row, int* __restrict__ is_int, long rank0,
                                     unsigned long long* err) {
  const long u = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= nocc) return;
  int f = 0;
  if (u < *nuniq && first_row[u] == INT_MAX) {
    const int cnt = seg_start[u + 1] - seg_start[u];
    if (cnt == 1) raise(err, rank0 + u, kErrUnlisted);
    else if (cnt > 2) raise(err, rank0 + u, kErrInterior3);
    f = 1;
  }
  is_int[u] = f;
}

__global__ void number_faces_kernel(int nbdy, int nfc, const int* __restrict__ nuniq,
                                    const int* __restrict__ first_row, const int* __restrict__ is_int,
                                    const int* __restrict__ int_excl, const int* __restrict__ seg_start,
                                    const int* __restrict__ svals, int nelt, const int* __restrict__ el,
                                    int* __restrict__ face_of, int* __restrict__ faces,
                                    uint8_t* __restrict__ facetype, unsigned long long* err) {
  const long u = long(blockIdx.x) * blockDim.x + threadIdx.x;
  const int nu = *nuniq;
  if (u >= nu) return;
  if (u == nu - 1 && nbdy + int_excl[u] + is_int[u] != nfc) raise(err, ~0ull >> 8, kErrCount);
  if (!is_int[u]) {
    face_of[u] = first_row[u];  // INT_MAX only on an error path
    return;
  }
  const int F = nbdy + int_excl[u];
  face_of[u] = F;
  if (F >= nfc) return;
  const int val = svals[seg_start[u]];  // lowest element's occurrence
  const long K = val >> 2;
  const int l = val & 3;
  for (int i = 0; i < 3; ++i) faces[F + long(i) * nfc] = el[K + long(cLocalFace[l][i]) * nelt];
  facetype[F] = kInterior;
}

__global__ void boundary_faces_kernel(int ndir, const int* __restrict__ dir, int nneu, const int* __restrict__ neu,
                                      int nfc, int* __restrict__ faces, uint8_t* __restrict__ facetype) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= ndir + nneu || b >= nfc) return;
  const bool d = b < ndir;
  const int r = d ? b : b - ndir, nr = d ? ndir : nneu;
  const int* rows = d ? dir : neu;
  for (int i = 0; i < 3; ++i) faces[b + long(i) * nfc] = rows[r + long(i) * nr];
  facetype[b] = d ? kDirichlet : kNeumann;
}

__global__ void facebyele_kernel(long nocc, int nelt, int nfc, const int* __restrict__ seg_incl,
                                 const int* __restrict__ svals, const int* __restrict__ face_of,
                                 int* __restrict__ fbe) {
  const long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nocc) return;
  const int val = svals[i];
  const int F = face_of[seg_incl[i] - 1];
  fbe[(val >> 2) + long(val & 3) * nelt] = F < nfc ? F : -1;
}

// ---------------------------------------------------------------- pattern
__global__ void face_elements_kernel(int nelt, int nfc, const int* __restrict__ fbe, int* __restrict__ cnt,
                                     int* __restrict__ occK, unsigned long long* err) {
  const long i = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 4L * nelt) return;
  const int f = fbe[i];
  const long K = i % nelt;
  if (f < 0 || f >= nfc) {
    raise(err, 0, kErrPatFace);
    return;
  }
  const int s = atomicAdd(&cnt[f], 1);
  if (s < 2) occK[2L * f + s] = int(K);
  else raise(err, 1, kErrPat3);
}

__global__ void neighbours_kernel(int nelt, int nfc, const int* __restrict__ fbe, const int* __restrict__ cnt,
                                  const int* __restrict__ occK, int* __restrict__ nbr, long long* __restrict__ nnbr,
                                  int* __restrict__ maxnbr) {
  const long f = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (f >= nfc) return;
  int c[8];
  int n = 0;
  const int ne = min(cnt[f], 2);
  for (int e = 0; e < ne; ++e) {
    const long K = occK[2 * f + e];
    for (int l = 0; l < 4; ++l) {
      const int g = fbe[K + long(l) * nelt];
      int j = n++;
      while (j > 0 && c[j - 1] > g) { c[j] = c[j - 1]; --j; }  // insertion sort
      c[j] = g;
    }
  }
  int nu = 0;
  for (int j = 0; j < n; ++j)
    if (nu == 0 || c[j] != c[nu - 1]) c[nu++] = c[j];
  for (int j = 0; j < 8; ++j) nbr[8 * f + j] = j < nu ? c[j] : -1;
  nnbr[f] = nu;
  atomicMax(maxnbr, nu);
}

__global__ void slots_kernel(int nelt, const int* __restrict__ fbe, const int* __restrict__ nbr,
                             const long long* __restrict__ nnbr, uint8_t* __restrict__ slot) {
  const long K = long(blockIdx.x) * blockDim.x + threadIdx.x;
  if (K >= nelt) return;
  int f[4];
  for (int l = 0; l < 4; ++l) f[l] = fbe[K + long(l) * nelt];
  for (int l1 = 0; l1 < 4; ++l1) {
    const int* nb = nbr + 8L * f[l1];
    const int nn = int(nnbr[f[l1]]);
    for (int l2 = 0; l2 < 4; ++l2) {
      int pos = 0;
      while (pos < nn && nb[pos] < f[l2]) ++pos;  // lower_bound
      slot[16 * K + 4 * l1 + l2] = uint8_t(pos);
    }
  }
}

inline int blocks(long n, int t = 256) { return int((n + t - 1) / t); }

// stream-ordered scratch, freed on scope exit
struct Scratch {
  cudaStream_t s;
  void* p = nullptr;
  Scratch(cudaStream_t st, size_t bytes) : s(st) { MCUDA(cudaMallocAsync(&p, bytes ? bytes : 1, s)); }
  ~Scratch() { cudaFreeAsync(p, s); }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

std::string mesh_message(unsigned long long e, long nelt) {
  const unsigned code = unsigned(e & 15ull);
  const unsigned long long rank = e >> 4;
  switch (code) {
    case kErrNoMatch: return "boundary face matches no element face";
    case kErrBdyShared: return "boundary face shared by more than one element";
    case kErrTwice: return "boundary face listed twice";
    case kErrUnlisted: return "element face on the boundary is not listed as Dirichlet or Neumann";
    case kErrInterior3: return "interior face shared by more than two elements";
    case kErrOrient: return "element " + std::to_string(long(rank) - 1) + " has non-positive orientation";
    case kErrCount: return "face count identity violated";
    case kErrRange: return "element vertex id out of range";
    case kErrPatFace: return "facebyele entry out of range";
    case kErrPat3: return "face belongs to more than two elements";
    default: (void)nelt; return "mesh error";
  }
}

void check_err(cudaStream_t s, const unsigned long long* d_err, long nelt) {
  unsigned long long h = kErrNone;
  MCUDA(cudaMemcpyAsync(&h, d_err, sizeof(h), cudaMemcpyDeviceToHost, s));
  MCUDA(cudaStreamSynchronize(s));
  if (h != kErrNone) throw MeshError(mesh_message(h, nelt));
}

}  // namespace

int expanded_face_count(int nelt, int ndir, int nneu) { return (4 * nelt + ndir + nneu) / 2; }

void expand_device(cudaStream_t s, int nver, const double* coords, int nelt, const int* elements, int ndir,
                   const int* dir, int nneu, const int* neu, int* faces, uint8_t* facetype, int* facebyele) {
  if (nver >= (1 << kKeyBits)) throw std::invalid_argument("GPU expansion packs 21-bit vertex ids (nver < 2^21)");
  if (nelt <= 0) throw MeshError("mesh has no elements");
  const long nocc = 4L * nelt;
  const int nbdy = ndir + nneu;
  const int nfc = expanded_face_count(nelt, ndir, nneu);
  // scratch layout
  size_t sort_bytes = 0, scan_bytes = 0;
  MCUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, (unsigned long long*)nullptr,
                                        (unsigned long long*)nullptr, (int*)nullptr, (int*)nullptr, nocc, 0,
                                        3 * kKeyBits, s));
  MCUDA(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, (int*)nullptr, (int*)nullptr, nocc, s));
  size_t scan2 = 0;
  MCUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan2, (int*)nullptr, (int*)nullptr, nocc, s));
  const size_t tmp_bytes = std::max(sort_bytes, std::max(scan_bytes, scan2));
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t o_k0 = 0, o_k1 = o_k0 + al(nocc * 8), o_v0 = o_k1 + al(nocc * 8), o_v1 = o_v0 + al(nocc * 4),
               o_head = o_v1 + al(nocc * 4), o_seg = o_head + al(nocc * 4), o_start = o_seg + al(nocc * 4),
               o_first = o_start + al((nocc + 1) * 4), o_isint = o_first + al(nocc * 4),
               o_excl = o_isint + al(nocc * 4), o_faceof = o_excl + al(nocc * 4),
               o_rowseg = o_faceof + al(nocc * 4), o_misc = o_rowseg + al(size_t(nbdy + 1) * 4),
               o_tmp = o_misc + 256, total = o_tmp + al(tmp_bytes);
  Scratch sc(s, total);
  char* base = sc.as<char>();
  auto* k0 = reinterpret_cast<unsigned long long*>(base + o_k0);
  auto* k1 = reinterpret_cast<unsigned long long*>(base + o_k1);
  int* v0 = reinterpret_cast<int*>(base + o_v0);
  int* v1 = reinterpret_cast<int*>(base + o_v1);
  int* head = reinterpret_cast<int*>(base + o_head);
  int* seg = reinterpret_cast<int*>(base + o_seg);
  int* start = reinterpret_cast<int*>(base + o_start);
  int* first = reinterpret_cast<int*>(base + o_first);
  int* isint = reinterpret_cast<int*>(base + o_isint);
  int* excl = reinterpret_cast<int*>(base + o_excl);
  int* faceof = reinterpret_cast<int*>(base + o_faceof);
  int* rowseg = reinterpret_cast<int*>(base + o_rowseg);
  auto* err = reinterpret_cast<unsigned long long*>(base + o_misc);
  int* nuniq = reinterpret_cast<int*>(base + o_misc + 8);
  void* tmp = base + o_tmp;

  MCUDA(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), s));
  occ_keys_kernel<<<blocks(nelt), 256, 0, s>>>(nver, coords, nelt, elements, k0, v0, err);
  size_t tb = tmp_bytes;
  MCUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, nocc, 0, 3 * kKeyBits, s));
  heads_kernel<<<blocks(nocc), 256, 0, s>>>(nocc, k1, head);
  tb = tmp_bytes;
  MCUDA(cub::DeviceScan::InclusiveSum(tmp, tb, head, seg, nocc, s));
  seg_start_kernel<<<blocks(nocc), 256, 0, s>>>(nocc, head, seg, start, nuniq, first);
  const long rank_b = 1L + nelt, rank_i = rank_b + nbdy;
  if (nbdy > 0) {
    boundary_match_kernel<<<blocks(nbdy), 256, 0, s>>>(ndir, dir, nneu, neu, nver, nocc, k1, seg, start, rowseg,
                                                      first, rank_b, err);
    boundary_twice_kernel<<<blocks(nbdy), 256, 0, s>>>(nbdy, rowseg, first, rank_b, err);
  }
  interior_flag_kernel<<<blocks(nocc), 256, 0, s>>>(nocc, nuniq, start, first, isint, rank_i, err);
  tb = tmp_bytes;
  MCUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, isint, excl, nocc, s));
  number_faces_kernel<<<blocks(nocc), 256, 0, s>>>(nbdy, nfc, nuniq, first, isint, excl, start, v1, nelt, elements,
                                                   faceof, faces, facetype, err);
  if (nbdy > 0)
    boundary_faces_kernel<<<blocks(nbdy), 256, 0, s>>>(ndir, dir, nneu, neu, nfc, faces, facetype);
  facebyele_kernel<<<blocks(nocc), 256, 0, s>>>(nocc, nelt, nfc, seg, v1, faceof, facebyele);
  MCUDA(cudaGetLastError());
  check_err(s, err, nelt);
}

int pattern_device(cudaStream_t s, int nelt, int nfc, const int* facebyele, int64_t* facebase, int* nbr,
                   uint8_t* slot) {
  if (nelt <= 0 || nfc <= 0) throw std::invalid_argument("empty mesh");
  size_t scan_bytes = 0;
  MCUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (long long*)nullptr, (long long*)nullptr, nfc + 1, s));
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  const size_t o_cnt = 0, o_occ = al(size_t(nfc) * 4), o_nn = o_occ + al(size_t(nfc) * 8),
               o_misc = o_nn + al(size_t(nfc + 1) * 8), o_tmp = o_misc + 256, total = o_tmp + al(scan_bytes);
  Scratch sc(s, total);
  char* base = sc.as<char>();
  int* cnt = reinterpret_cast<int*>(base + o_cnt);
  int* occ = reinterpret_cast<int*>(base + o_occ);
  auto* nn = reinterpret_cast<long long*>(base + o_nn);
  auto* err = reinterpret_cast<unsigned long long*>(base + o_misc);
  int* maxnbr = reinterpret_cast<int*>(base + o_misc + 8);
  MCUDA(cudaMemsetAsync(cnt, 0, size_t(nfc) * 4, s));
  MCUDA(cudaMemsetAsync(nn + nfc, 0, 8, s));
  MCUDA(cudaMemsetAsync(err, 0xff, 8, s));
  MCUDA(cudaMemsetAsync(maxnbr, 0, 4, s));
  face_elements_kernel<<<blocks(4L * nelt), 256, 0, s>>>(nelt, nfc, facebyele, cnt, occ, err);
  neighbours_kernel<<<blocks(nfc), 256, 0, s>>>(nelt, nfc, facebyele, cnt, occ, nbr, nn, maxnbr);
  size_t tb = scan_bytes;
  MCUDA(cub::DeviceScan::ExclusiveSum(base + o_tmp, tb, nn, reinterpret_cast<long long*>(facebase), nfc + 1, s));
  slots_kernel<<<blocks(nelt), 256, 0, s>>>(nelt, facebyele, nbr, nn, slot);
  MCUDA(cudaGetLastError());
  check_err(s, err, nelt);
  int h = 0;
  MCUDA(cudaMemcpyAsync(&h, maxnbr, 4, cudaMemcpyDeviceToHost, s));
  MCUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace hdgb
