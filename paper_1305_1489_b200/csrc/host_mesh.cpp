// Host-side mesh setup for the engine (input generation + numbering; not timed).
//
//  * box_mesh      — Kuhn 6-tet split, restating proj/src/mesh.cpp:185-253
//                    (vertex ids, element order, boundary-row order are bit-exact)
//  * expand_mesh   — global face numbering, restating proj/src/mesh.cpp:74-171:
//                    Dirichlet rows, then Neumann rows (input order), then
//                    interior faces in ascending sorted-vertex-triple order
//                    (std::map order) taken from the lower-numbered element.
//                    Implemented with a radix-style key sort instead of a
//                    std::map so C5 (6.3M face occurrences) expands in ~1 s.
//  * build_pattern — the skeleton system's block sparsity (global_system.cpp:31-56).
// Geometry (volumes, normals, perm codes, areas) is computed on the GPU (K1).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "host_internal.hpp"

namespace hdgb {

namespace {

inline void sort3(int& a, int& b, int& c) {
  if (a > b) std::swap(a, b);
  if (b > c) std::swap(b, c);
  if (a > b) std::swap(a, b);
}

// Packed sorted vertex triple; lexicographic order of (a,b,c) == integer order.
inline unsigned __int128 tri_key(int a, int b, int c) {
  sort3(a, b, c);
  return (static_cast<unsigned __int128>(uint32_t(a)) << 64) |
         (static_cast<unsigned __int128>(uint32_t(b)) << 32) | uint32_t(c);
}

double det_of(const std::vector<double>& X, int nver, const int v[4]) {
  double B[3][3];
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) B[r][c] = X[v[c + 1] + size_t(r) * nver] - X[v[0] + size_t(r) * nver];
  return B[0][0] * (B[1][1] * B[2][2] - B[2][1] * B[1][2]) -
         B[1][0] * (B[0][1] * B[2][2] - B[2][1] * B[0][2]) +
         B[2][0] * (B[0][1] * B[1][2] - B[1][1] * B[0][2]);
}

uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

// mesh.cpp:185-253
void box_mesh(int nx, int ny, int nz, BoundaryRule bc, HostMesh& m) {
  if (nx < 1 || ny < 1 || nz < 1) throw MeshError("box_mesh: cell counts must be >= 1");
  const int nvx = nx + 1, nvy = ny + 1, nvz = nz + 1;
  m = HostMesh{};
  m.nver = nvx * nvy * nvz;
  m.coords.assign(size_t(m.nver) * 3, 0.0);
  auto vid = [&](int i, int j, int k) { return (k * nvy + j) * nvx + i; };
  for (int k = 0; k < nvz; ++k)
    for (int j = 0; j < nvy; ++j)
      for (int i = 0; i < nvx; ++i) {
        const int v = vid(i, j, k);
        m.coords[v] = 0.0 + (1.0 - 0.0) * i / nx;
        m.coords[m.nver + v] = 0.0 + (1.0 - 0.0) * j / ny;
        m.coords[2 * size_t(m.nver) + v] = 0.0 + (1.0 - 0.0) * k / nz;
      }
  constexpr int axis_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  constexpr bool odd_perm[6] = {false, true, true, false, false, true};
  m.nelt = 6 * nx * ny * nz;
  m.elements.assign(size_t(m.nelt) * 4, 0);
  int K = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        for (int p = 0; p < 6; ++p, ++K) {
          int step[3] = {0, 0, 0}, v[4];
          v[0] = vid(i, j, k);
          for (int s = 0; s < 3; ++s) {
            step[axis_perm[p][s]] = 1;
            v[s + 1] = vid(i + step[0], j + step[1], k + step[2]);
          }
          if (odd_perm[p]) std::swap(v[1], v[2]);
          for (int c = 0; c < 4; ++c) m.elements[K + size_t(c) * m.nelt] = v[c];
        }
  // boundary faces = element faces whose vertex set occurs once; scan K, l
  const size_t nocc = size_t(m.nelt) * 4;
  std::vector<unsigned __int128> keys(nocc);
  for (int e = 0; e < m.nelt; ++e)
    for (int l = 0; l < 4; ++l)
      keys[size_t(e) * 4 + l] = tri_key(m.elements[e + size_t(kLocalFace[l][0]) * m.nelt],
                                        m.elements[e + size_t(kLocalFace[l][1]) * m.nelt],
                                        m.elements[e + size_t(kLocalFace[l][2]) * m.nelt]);
  std::vector<unsigned __int128> sorted = keys;
  std::sort(sorted.begin(), sorted.end());
  std::vector<int> dir, neu;
  for (int e = 0; e < m.nelt; ++e)
    for (int l = 0; l < 4; ++l) {
      const auto key = keys[size_t(e) * 4 + l];
      const auto lo = std::lower_bound(sorted.begin(), sorted.end(), key);
      if (lo + 1 != sorted.end() && *(lo + 1) == key) continue;  // shared
      int t[3];
      for (int i = 0; i < 3; ++i) t[i] = m.elements[e + size_t(kLocalFace[l][i]) * m.nelt];
      double u[3], w[3], n[3];
      for (int c = 0; c < 3; ++c) {
        u[c] = m.coords[t[1] + size_t(c) * m.nver] - m.coords[t[0] + size_t(c) * m.nver];
        w[c] = m.coords[t[2] + size_t(c) * m.nver] - m.coords[t[0] + size_t(c) * m.nver];
      }
      n[0] = 0.5 * (u[1] * w[2] - u[2] * w[1]);
      n[1] = 0.5 * (u[2] * w[0] - u[0] * w[2]);
      n[2] = 0.5 * (u[0] * w[1] - u[1] * w[0]);
      const double nn = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
      for (int c = 0; c < 3; ++c) n[c] = kFaceNormalSign[l] * n[c] / nn;
      bool is_dir = true;  // mesh.cpp:173-183 + SURVEY §8(d) dirichlet_x
      if (bc == kDirichletTopBottom) is_dir = std::abs(n[2]) > 0.5;
      if (bc == kDirichletX) is_dir = std::abs(n[0]) > 0.5;
      auto& dst = is_dir ? dir : neu;
      dst.insert(dst.end(), t, t + 3);
    }
  m.ndir = int(dir.size() / 3);
  m.nneu = int(neu.size() / 3);
  m.dirichlet.assign(size_t(m.ndir) * 3, 0);
  m.neumann.assign(size_t(m.nneu) * 3, 0);
  for (int r = 0; r < m.ndir; ++r)
    for (int c = 0; c < 3; ++c) m.dirichlet[r + size_t(c) * m.ndir] = dir[size_t(r) * 3 + c];
  for (int r = 0; r < m.nneu; ++r)
    for (int c = 0; c < 3; ++c) m.neumann[r + size_t(c) * m.nneu] = neu[size_t(r) * 3 + c];
}

// Builder-defined C3 jitter: every interior vertex, in id
// order, moves by U(-frac*h, frac*h) per coordinate drawn from a splitmix64
// stream; vertices on the plane z = keep_plane_z move in x and y only; a move
// is redrawn (up to 16 times, else dropped) unless every incident tet keeps
// det B > 0.25 * h^3 (non-inverted, not degenerate).
void perturb_interior(HostMesh& m, int nx, int ny, int nz, double frac, uint64_t seed,
                      double keep_plane_z) {
  if (frac <= 0) return;
  const int nvx = nx + 1, nvy = ny + 1;
  const double hx = 1.0 / nx, hy = 1.0 / ny, hz = 1.0 / nz;
  const double h3 = hx * hy * hz;
  std::vector<std::vector<int>> inc(m.nver);
  for (int K = 0; K < m.nelt; ++K)
    for (int c = 0; c < 4; ++c) inc[m.elements[K + size_t(c) * m.nelt]].push_back(K);
  uint64_t s = seed;
  auto uni = [&]() { return double(splitmix64(s) >> 11) * 0x1.0p-53; };
  for (int v = 0; v < m.nver; ++v) {
    const int i = v % nvx, j = (v / nvx) % nvy, k = v / (nvx * nvy);
    if (i == 0 || j == 0 || k == 0 || i == nx || j == ny || k == nz) continue;
    double* X = &m.coords[v];
    double* Y = &m.coords[size_t(m.nver) + v];
    double* Z = &m.coords[2 * size_t(m.nver) + v];
    const double x0 = *X, y0 = *Y, z0 = *Z;
    const bool on_plane = std::fabs(z0 - keep_plane_z) < 1e-12;
    for (int attempt = 0; attempt < 16; ++attempt) {
      const double dx = (2.0 * uni() - 1.0) * frac * hx;
      const double dy = (2.0 * uni() - 1.0) * frac * hy;
      const double dz = (2.0 * uni() - 1.0) * frac * hz;
      *X = x0 + dx;
      *Y = y0 + dy;
      *Z = on_plane ? z0 : z0 + dz;
      bool ok = true;
      for (int K : inc[v]) {
        int vv[4];
        for (int c = 0; c < 4; ++c) vv[c] = m.elements[K + size_t(c) * m.nelt];
        if (!(det_of(m.coords, m.nver, vv) > 0.25 * h3)) { ok = false; break; }
      }
      if (ok) break;
      *X = x0;
      *Y = y0;
      *Z = z0;
    }
  }
}

// mesh.cpp:74-171 (numbering only; geometry is K1 on the device)
void expand_mesh(HostMesh& m) {
  const int nelt = m.nelt, nbdy = m.ndir + m.nneu;
  for (int K = 0; K < nelt; ++K) {
    int v[4];
    for (int c = 0; c < 4; ++c) v[c] = m.elements[K + size_t(c) * nelt];
    if (!(det_of(m.coords, m.nver, v) > 0))
      throw MeshError("element " + std::to_string(K) + " has non-positive orientation");
  }
  const size_t nocc = size_t(nelt) * 4;
  struct Occ { unsigned __int128 key; int K, l; };
  std::vector<Occ> occ(nocc);
  for (int K = 0; K < nelt; ++K)
    for (int l = 0; l < 4; ++l)
      occ[size_t(K) * 4 + l] = {tri_key(m.elements[K + size_t(kLocalFace[l][0]) * nelt],
                                        m.elements[K + size_t(kLocalFace[l][1]) * nelt],
                                        m.elements[K + size_t(kLocalFace[l][2]) * nelt]), K, l};
  std::vector<Occ> srt = occ;
  std::sort(srt.begin(), srt.end(), [](const Occ& a, const Occ& b) {
    return a.key < b.key || (a.key == b.key && (a.K < b.K || (a.K == b.K && a.l < b.l)));
  });
  // unique keys with their occurrence ranges
  std::vector<size_t> ustart;
  for (size_t i = 0; i < nocc; ++i)
    if (i == 0 || srt[i].key != srt[i - 1].key) ustart.push_back(i);
  const size_t nuniq = ustart.size();
  ustart.push_back(nocc);
  std::vector<int> face_of(nuniq, -1);
  auto find = [&](unsigned __int128 key) -> size_t {
    size_t lo = 0, hi = nuniq;
    while (lo < hi) {
      const size_t mid = (lo + hi) / 2;
      if (srt[ustart[mid]].key < key) lo = mid + 1; else hi = mid;
    }
    if (lo == nuniq || srt[ustart[lo]].key != key) return size_t(-1);
    return lo;
  };
  std::vector<int> faces;
  faces.reserve(size_t(nuniq) * 3);
  m.facetype.clear();
  auto add_boundary = [&](const std::vector<int>& rows, int nr, FaceType type) {
    for (int r = 0; r < nr; ++r) {
      const int a = rows[r], b = rows[r + size_t(nr)], c = rows[r + 2 * size_t(nr)];
      const size_t u = find(tri_key(a, b, c));
      if (u == size_t(-1)) throw MeshError("boundary face matches no element face");
      if (ustart[u + 1] - ustart[u] != 1) throw MeshError("boundary face shared by more than one element");
      if (face_of[u] >= 0) throw MeshError("boundary face listed twice");
      face_of[u] = int(m.facetype.size());
      faces.insert(faces.end(), {a, b, c});
      m.facetype.push_back(type);
    }
  };
  add_boundary(m.dirichlet, m.ndir, kDirichlet);
  add_boundary(m.neumann, m.nneu, kNeumann);
  for (size_t u = 0; u < nuniq; ++u) {
    if (face_of[u] >= 0) continue;
    const size_t cnt = ustart[u + 1] - ustart[u];
    if (cnt == 1) throw MeshError("element face on the boundary is not listed as Dirichlet or Neumann");
    if (cnt > 2) throw MeshError("interior face shared by more than two elements");
    const Occ& o = srt[ustart[u]];  // lowest element first (sorted by K)
    face_of[u] = int(m.facetype.size());
    for (int i = 0; i < 3; ++i) faces.push_back(m.elements[o.K + size_t(kLocalFace[o.l][i]) * nelt]);
    m.facetype.push_back(kInterior);
  }
  m.nfc = int(m.facetype.size());
  if (4 * nelt != 2 * (m.nfc - nbdy) + nbdy) throw MeshError("face count identity violated");
  m.faces.assign(size_t(m.nfc) * 3, 0);
  for (int f = 0; f < m.nfc; ++f)
    for (int i = 0; i < 3; ++i) m.faces[f + size_t(i) * m.nfc] = faces[size_t(f) * 3 + i];
  m.facebyele.assign(size_t(nelt) * 4, 0);
  for (size_t u = 0; u < nuniq; ++u)
    for (size_t i = ustart[u]; i < ustart[u + 1]; ++i)
      m.facebyele[srt[i].K + size_t(srt[i].l) * nelt] = face_of[u];
  m.expanded = true;
}

// global_system.cpp:31-56: entry (face f1 row i, face f2 col j) exists iff f1
// and f2 are faces of a common element; structurally symmetric, so the CSR
// pattern equals Eigen's CSC pattern (rows sorted, duplicates summed).
void build_pattern(const HostMesh& m, SkeletonPattern& p) {
  build_pattern_raw(m.nelt, m.nfc, m.facebyele.data(), p);
}

// Same from a bare facebyele (nelt x 4, column-major): used for slab-local
// patterns in multi-GPU runs, where a slab's faces are renumbered locally.
void build_pattern_raw(int nelt, int nfc, const int* facebyele, SkeletonPattern& p) {
  struct {
    const int* fbe;
    int fb(size_t i) const { return fbe[i]; }
  } m{facebyele};
  p.nfc = nfc;
  p.nbr.assign(size_t(nfc) * 8, -1);
  p.nnbr.assign(nfc, 0);
  std::vector<int> cand(size_t(nfc) * 8, -1), ncand(nfc, 0);
  for (int K = 0; K < nelt; ++K)
    for (int l1 = 0; l1 < 4; ++l1) {
      const int f1 = m.fb(K + size_t(l1) * nelt);
      if (f1 < 0 || f1 >= nfc) throw MeshError("facebyele entry out of range");
      for (int l2 = 0; l2 < 4; ++l2) {
        if (ncand[f1] >= 8) throw MeshError("face belongs to more than two elements");
        cand[size_t(f1) * 8 + ncand[f1]++] = m.fb(K + size_t(l2) * nelt);
      }
    }
  p.maxnbr = 0;
  for (int f = 0; f < nfc; ++f) {
    int* c = &cand[size_t(f) * 8];
    std::sort(c, c + ncand[f]);
    const int nu = int(std::unique(c, c + ncand[f]) - c);
    p.nnbr[f] = nu;
    std::copy(c, c + nu, &p.nbr[size_t(f) * 8]);
    p.maxnbr = std::max(p.maxnbr, nu);
  }
  p.facebase.assign(size_t(nfc) + 1, 0);
  for (int f = 0; f < nfc; ++f) p.facebase[f + 1] = p.facebase[f] + p.nnbr[f];
  p.slot.assign(size_t(nelt) * 16, 0);
  for (int K = 0; K < nelt; ++K)
    for (int l1 = 0; l1 < 4; ++l1) {
      const int f1 = m.fb(K + size_t(l1) * nelt);
      const int* nb = &p.nbr[size_t(f1) * 8];
      for (int l2 = 0; l2 < 4; ++l2) {
        const int f2 = m.fb(K + size_t(l2) * nelt);
        const int pos = int(std::lower_bound(nb, nb + p.nnbr[f1], f2) - nb);
        p.slot[size_t(K) * 16 + l1 * 4 + l2] = uint8_t(pos);
      }
    }
}

}  // namespace hdgb
