// TEST INFRASTRUCTURE ONLY — see hdg_oracle.hpp. CPU restatement of the
// reference element-local HDG path; every function cites what it restates
// (paths relative to /root/reference/proj).
#include "hdg_oracle.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <numeric>
#include <thread>

namespace hdgo {

// ---------------------------------------------------------------------------
// batch.hpp:42-58
void parallel_for(int n, int nthreads, const std::function<void(int, int)>& fn) {
  if (n <= 0) return;
  nthreads = std::max(1, std::min(nthreads, n));
  if (nthreads == 1) { fn(0, n); return; }
  std::vector<std::thread> pool;
  const int chunk = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    const int b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    pool.emplace_back(fn, b, e);
  }
  for (auto& th : pool) th.join();
}

// ---------------------------------------------------------------- fields
// Postfix program VM; opcodes mirror include/hdg_b200.h (HDG_OP_*).
ScalarField program_field(const int* ops, int nops, const double* consts, int nconst) {
  std::vector<int> o(ops, ops + nops);
  std::vector<double> cs(consts, consts + nconst);
  return [o, cs](double x, double y, double z) {
    double st[32];
    int sp = 0, ci = 0;
    for (int op : o) {
      switch (op) {
        case 0: st[sp++] = x; break;
        case 1: st[sp++] = y; break;
        case 2: st[sp++] = z; break;
        case 3: st[sp++] = cs[ci++]; break;
        case 4: --sp; st[sp - 1] = st[sp - 1] + st[sp]; break;
        case 5: --sp; st[sp - 1] = st[sp - 1] - st[sp]; break;
        case 6: --sp; st[sp - 1] = st[sp - 1] * st[sp]; break;
        case 7: --sp; st[sp - 1] = st[sp - 1] / st[sp]; break;
        case 8: st[sp - 1] = -st[sp - 1]; break;
        case 9: st[sp - 1] = std::sin(st[sp - 1]); break;
        case 10: st[sp - 1] = std::cos(st[sp - 1]); break;
        case 11: st[sp - 1] = std::exp(st[sp - 1]); break;
        case 12: st[sp - 1] = std::sqrt(st[sp - 1]); break;
        case 13: st[sp - 1] = std::fabs(st[sp - 1]); break;
        case 14: --sp; st[sp - 1] = st[sp - 1] < st[sp] ? 1.0 : 0.0; break;
        case 15: --sp; st[sp - 1] = std::pow(st[sp - 1], st[sp]); break;
        default: throw std::invalid_argument("bad field opcode");
      }
    }
    return st[0];
  };
}

ScalarField constant_field(double v) {
  return [v](double, double, double) { return v; };
}

// --------------------------------------------------------------------- mesh
namespace {
std::array<int, 3> sorted_triple(int a, int b, int c) {
  std::array<int, 3> t{a, b, c};
  std::sort(t.begin(), t.end());
  return t;
}
// mesh.cpp:24-32
int find_perm(const std::array<int, 3>& g, const std::array<int, 3>& l) {
  for (int mu = 1; mu <= 6; ++mu) {
    bool ok = true;
    for (int i = 0; i < 3; ++i)
      if (g[kVertexImage[mu - 1][i]] != l[i]) { ok = false; break; }
    if (ok) return mu;
  }
  throw MeshError("face vertex triples do not match as sets");
}
// mesh.cpp:34-39
void half_cross(const Mat& X, const std::array<int, 3>& t, double out[3]) {
  double u[3], v[3];
  for (int c = 0; c < 3; ++c) {
    u[c] = X(t[1], c) - X(t[0], c);
    v[c] = X(t[2], c) - X(t[0], c);
  }
  out[0] = 0.5 * (u[1] * v[2] - u[2] * v[1]);
  out[1] = 0.5 * (u[2] * v[0] - u[0] * v[2]);
  out[2] = 0.5 * (u[0] * v[1] - u[1] * v[0]);
}
double norm3v(const double v[3]) { return std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }
}  // namespace

// mesh.cpp:43-66
ElementGeometry geometry(const RawMesh& raw, int K) {
  if (K < 0 || K >= raw.n_elements()) throw MeshError("element index out of range");
  ElementGeometry g;
  const Mat& X = raw.coordinates;
  auto v = [&](int i, int c) { return X(raw.elements(K, i), c); };
  for (int c = 0; c < 3; ++c)
    for (int r = 0; r < 3; ++r) g.B[r + 3 * c] = v(c + 1, r) - v(0, r);
  const double* B = g.B;
  // Eigen's 3x3 determinant: cofactor expansion along column 0
  g.detB = B[0] * (B[4] * B[8] - B[7] * B[5]) - B[1] * (B[3] * B[8] - B[6] * B[5]) +
           B[2] * (B[3] * B[7] - B[6] * B[4]);
  const double x1 = v(0, 0), x2 = v(1, 0), x3 = v(2, 0), x4 = v(3, 0);
  const double y1 = v(0, 1), y2 = v(1, 1), y3 = v(2, 1), y4 = v(3, 1);
  const double z1 = v(0, 2), z2 = v(1, 2), z3 = v(2, 2), z4 = v(3, 2);
  g.a[0] = (y3 - y1) * (z4 - z1) - (y4 - y1) * (z3 - z1);
  g.a[1] = (y4 - y1) * (z2 - z1) - (y2 - y1) * (z4 - z1);
  g.a[2] = (y2 - y1) * (z3 - z1) - (y3 - y1) * (z2 - z1);
  g.a[3] = (x4 - x1) * (z3 - z1) - (x3 - x1) * (z4 - z1);
  g.a[4] = (x2 - x1) * (z4 - z1) - (x4 - x1) * (z2 - z1);
  g.a[5] = (x3 - x1) * (z2 - z1) - (x2 - x1) * (z3 - z1);
  g.a[6] = (x3 - x1) * (y4 - y1) - (x4 - x1) * (y3 - y1);
  g.a[7] = (x4 - x1) * (y2 - y1) - (x2 - x1) * (y4 - y1);
  g.a[8] = (x2 - x1) * (y3 - y1) - (x3 - x1) * (y2 - y1);
  return g;
}

// mesh.cpp:74-171
ExpandedMesh expand(const RawMesh& raw) {
  const int nelt = raw.n_elements(), ndir = raw.dirichlet.r, nneu = raw.neumann.r;
  for (int K = 0; K < nelt; ++K)
    if (geometry(raw, K).detB <= 0)
      throw MeshError("element " + std::to_string(K) + " has non-positive orientation");
  std::map<std::array<int, 3>, std::vector<std::pair<int, int>>> incidence;
  for (int K = 0; K < nelt; ++K)
    for (int l = 0; l < 4; ++l)
      incidence[sorted_triple(raw.elements(K, kLocalFace[l][0]), raw.elements(K, kLocalFace[l][1]),
                              raw.elements(K, kLocalFace[l][2]))]
          .emplace_back(K, l);
  ExpandedMesh em;
  em.raw = raw;
  std::map<std::array<int, 3>, int> face_number;
  const int nbdy = ndir + nneu;
  std::vector<std::array<int, 3>> tri;
  auto add_boundary = [&](const IMat& rows, FaceType type) {
    for (int r = 0; r < rows.r; ++r) {
      const std::array<int, 3> t{rows(r, 0), rows(r, 1), rows(r, 2)};
      const auto key = sorted_triple(t[0], t[1], t[2]);
      const auto it = incidence.find(key);
      if (it == incidence.end()) throw MeshError("boundary face matches no element face");
      if (it->second.size() != 1) throw MeshError("boundary face shared by more than one element");
      if (face_number.count(key)) throw MeshError("boundary face listed twice");
      face_number[key] = int(tri.size());
      tri.push_back(t);
      em.facetype.push_back(type);
    }
  };
  add_boundary(raw.dirichlet, Dirichlet);
  add_boundary(raw.neumann, Neumann);
  for (const auto& [key, occ] : incidence) {
    if (face_number.count(key)) continue;
    if (occ.size() == 1)
      throw MeshError("element face on the boundary is not listed as Dirichlet or Neumann");
    if (occ.size() > 2) throw MeshError("interior face shared by more than two elements");
    const auto [K, l] = occ.front().first <= occ.back().first ? occ.front() : occ.back();
    face_number[key] = int(tri.size());
    tri.push_back({raw.elements(K, kLocalFace[l][0]), raw.elements(K, kLocalFace[l][1]),
                   raw.elements(K, kLocalFace[l][2])});
    em.facetype.push_back(Interior);
  }
  const int nfc = int(tri.size());
  if (4 * nelt != 2 * (nfc - nbdy) + nbdy) throw MeshError("face count identity violated");
  em.faces = IMat(nfc, 3);
  for (int f = 0; f < nfc; ++f)
    for (int i = 0; i < 3; ++i) em.faces(f, i) = tri[f][i];
  for (int f = 0; f < nfc; ++f) {
    if (em.facetype[f] == Dirichlet) em.dirfaces.push_back(f);
    if (em.facetype[f] == Neumann) em.neufaces.push_back(f);
  }
  em.facebyele = IMat(nelt, 4);
  em.perm = IMat(nelt, 4);
  em.volume.assign(nelt, 0.0);
  em.area.assign(nfc, 0.0);
  em.normals = Mat(nelt, 12);
  for (int f = 0; f < nfc; ++f) {
    double h[3];
    half_cross(raw.coordinates, tri[f], h);
    em.area[f] = norm3v(h);
  }
  for (int K = 0; K < nelt; ++K) {
    em.volume[K] = geometry(raw, K).detB / 6.0;
    for (int l = 0; l < 4; ++l) {
      const std::array<int, 3> loc{raw.elements(K, kLocalFace[l][0]),
                                   raw.elements(K, kLocalFace[l][1]),
                                   raw.elements(K, kLocalFace[l][2])};
      const int f = face_number.at(sorted_triple(loc[0], loc[1], loc[2]));
      em.facebyele(K, l) = f;
      em.perm(K, l) = find_perm(tri[f], loc);
      double h[3];
      half_cross(raw.coordinates, loc, h);
      for (int c = 0; c < 3; ++c) em.normals(K, 3 * l + c) = kFaceNormalSign[l] * h[c];
    }
  }
  return em;
}

// mesh.cpp:173-183
FaceClassifier all_dirichlet() {
  return [](const double*, const double*) { return Dirichlet; };
}
FaceClassifier dirichlet_top_bottom() {
  return [](const double*, const double* nu) {
    return std::abs(nu[2]) > 0.5 ? Dirichlet : Neumann;
  };
}
FaceClassifier dirichlet_x() {
  return [](const double*, const double* nu) {
    return std::abs(nu[0]) > 0.5 ? Dirichlet : Neumann;
  };
}

// mesh.cpp:185-253
RawMesh box_mesh(int nx, int ny, int nz, const BoxBounds& bd, const FaceClassifier& bc) {
  if (nx < 1 || ny < 1 || nz < 1) throw MeshError("box_mesh: cell counts must be >= 1");
  if (!(bd.x1 > bd.x0) || !(bd.y1 > bd.y0) || !(bd.z1 > bd.z0))
    throw MeshError("box_mesh: degenerate bounds");
  RawMesh m;
  const int nvx = nx + 1, nvy = ny + 1, nvz = nz + 1;
  m.coordinates = Mat(nvx * nvy * nvz, 3);
  auto vid = [&](int i, int j, int k) { return (k * nvy + j) * nvx + i; };
  for (int k = 0; k < nvz; ++k)
    for (int j = 0; j < nvy; ++j)
      for (int i = 0; i < nvx; ++i) {
        const int v = vid(i, j, k);
        m.coordinates(v, 0) = bd.x0 + (bd.x1 - bd.x0) * i / nx;
        m.coordinates(v, 1) = bd.y0 + (bd.y1 - bd.y0) * j / ny;
        m.coordinates(v, 2) = bd.z0 + (bd.z1 - bd.z0) * k / nz;
      }
  constexpr int axis_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                   {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  constexpr bool odd_perm[6] = {false, true, true, false, false, true};
  m.elements = IMat(6 * nx * ny * nz, 4);
  int K = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i)
        for (int p = 0; p < 6; ++p, ++K) {
          int step[3] = {0, 0, 0};
          int v[4];
          v[0] = vid(i, j, k);
          for (int s = 0; s < 3; ++s) {
            step[axis_perm[p][s]] = 1;
            v[s + 1] = vid(i + step[0], j + step[1], k + step[2]);
          }
          if (odd_perm[p]) std::swap(v[1], v[2]);
          for (int c = 0; c < 4; ++c) m.elements(K, c) = v[c];
        }
  std::map<std::array<int, 3>, int> count;
  const int ne = m.elements.r;
  for (int e = 0; e < ne; ++e)
    for (int l = 0; l < 4; ++l)
      ++count[sorted_triple(m.elements(e, kLocalFace[l][0]), m.elements(e, kLocalFace[l][1]),
                            m.elements(e, kLocalFace[l][2]))];
  std::vector<std::array<int, 3>> dir, neu;
  for (int e = 0; e < ne; ++e)
    for (int l = 0; l < 4; ++l) {
      const std::array<int, 3> t{m.elements(e, kLocalFace[l][0]), m.elements(e, kLocalFace[l][1]),
                                 m.elements(e, kLocalFace[l][2])};
      if (count.at(sorted_triple(t[0], t[1], t[2])) != 1) continue;
      double cen[3], n[3];
      for (int c = 0; c < 3; ++c)
        cen[c] = (m.coordinates(t[0], c) + m.coordinates(t[1], c) + m.coordinates(t[2], c)) / 3.0;
      half_cross(m.coordinates, t, n);
      const double nn = norm3v(n);
      for (int c = 0; c < 3; ++c) n[c] = kFaceNormalSign[l] * n[c] / nn;
      (bc(cen, n) == Dirichlet ? dir : neu).push_back(t);
    }
  m.dirichlet = IMat(int(dir.size()), 3);
  for (size_t r = 0; r < dir.size(); ++r)
    for (int c = 0; c < 3; ++c) m.dirichlet(int(r), c) = dir[r][c];
  m.neumann = IMat(int(neu.size()), 3);
  for (size_t r = 0; r < neu.size(); ++r)
    for (int c = 0; c < 3; ++c) m.neumann(int(r), c) = neu[r][c];
  return m;
}

// --------------------------------------------------------------- quadrature
namespace {
// Symmetric tridiagonal eigenproblem by implicit QL with Wilkinson-type
// shifts (the published Golub-Welsch ingredient; the reference uses Eigen's
// SelfAdjointEigenSolver::computeFromTridiagonal, quadrature.cpp:23-24).
// d: diagonal (n), e: off-diagonal (n-1). Returns ascending eigenvalues and
// the first component of each normalised eigenvector.
void tridiag_eig(std::vector<double> d, std::vector<double> e, std::vector<double>& lam,
                 std::vector<double>& v0) {
  const int n = int(d.size());
  e.resize(n, 0.0);
  std::vector<double> z(size_t(n) * n, 0.0);  // z(i,j) eigenvector matrix, col-major
  for (int i = 0; i < n; ++i) z[i + size_t(i) * n] = 1.0;
  for (int l = 0; l < n; ++l) {
    for (int iter = 0; iter < 200; ++iter) {
      int m = l;
      for (; m < n - 1; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 1e-300 + 2.220446049250313e-16 * dd) break;
      }
      if (m == l) break;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[m] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
      double s = 1.0, c = 1.0, p = 0.0;
      int i = m - 1;
      bool underflow = false;
      for (; i >= l; --i) {
        double f = s * e[i];
        const double b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) { d[i + 1] -= p; e[m] = 0.0; underflow = true; break; }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        for (int k = 0; k < n; ++k) {
          f = z[k + size_t(i + 1) * n];
          z[k + size_t(i + 1) * n] = s * z[k + size_t(i) * n] + c * f;
          z[k + size_t(i) * n] = c * z[k + size_t(i) * n] - s * f;
        }
      }
      if (underflow) continue;
      d[l] -= p;
      e[l] = g;
      e[m] = 0.0;
    }
  }
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return d[a] < d[b]; });
  lam.resize(n);
  v0.resize(n);
  for (int j = 0; j < n; ++j) {
    lam[j] = d[idx[j]];
    v0[j] = z[0 + size_t(idx[j]) * n];
  }
}

// quadrature.cpp:12-32
void gauss_jacobi_biunit(int n, int alpha, std::vector<double>& x, std::vector<double>& w) {
  std::vector<double> diag(n), off(std::max(0, n - 1));
  const double a = alpha;
  diag[0] = -a / (a + 2.0);
  for (int k = 1; k < n; ++k) diag[k] = -a * a / ((2.0 * k + a) * (2.0 * k + a + 2.0));
  for (int k = 1; k < n; ++k)
    off[k - 1] = std::sqrt(4.0 * k * (k + a) * k * (k + a) /
                           ((2.0 * k + a) * (2.0 * k + a) * (2.0 * k + a + 1.0) *
                            (2.0 * k + a - 1.0)));
  std::vector<double> v0;
  tridiag_eig(diag, off, x, v0);
  const double mu0 = std::pow(2.0, a + 1.0) / (a + 1.0);
  w.resize(n);
  for (int i = 0; i < n; ++i) w[i] = mu0 * v0[i] * v0[i];
}
}  // namespace

// quadrature.cpp:36-41
void gauss_jacobi01(int n, int alpha, std::vector<double>& x, std::vector<double>& w) {
  gauss_jacobi_biunit(n, alpha, x, w);
  const double s = std::pow(2.0, alpha + 1.0);
  for (int i = 0; i < n; ++i) { x[i] = (x[i] + 1.0) / 2.0; w[i] /= s; }
}

// quadrature.cpp:43-67
TetRule tet_rule(int degree) {
  if (degree < 0 || degree > 60) throw std::invalid_argument("tet_rule: unsupported degree");
  const int n = degree / 2 + 1;
  std::vector<double> ta, wa, tb, wb, tc, wc;
  gauss_jacobi01(n, 0, ta, wa);
  gauss_jacobi01(n, 1, tb, wb);
  gauss_jacobi01(n, 2, tc, wc);
  TetRule r;
  r.exactness = degree;
  r.barycentric = Mat(n * n * n, 4);
  r.weights.resize(n * n * n);
  int q = 0;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i, ++q) {
        const double z = tc[k], y = tb[j] * (1.0 - z), x = ta[i] * (1.0 - tb[j]) * (1.0 - z);
        r.barycentric(q, 0) = 1.0 - x - y - z;
        r.barycentric(q, 1) = x;
        r.barycentric(q, 2) = y;
        r.barycentric(q, 3) = z;
        r.weights[q] = 6.0 * wa[i] * wb[j] * wc[k];
      }
  return r;
}

// quadrature.cpp:69-90
TriRule tri_rule(int degree) {
  if (degree < 0 || degree > 60) throw std::invalid_argument("tri_rule: unsupported degree");
  const int n = degree / 2 + 1;
  std::vector<double> ta, wa, tb, wb;
  gauss_jacobi01(n, 0, ta, wa);
  gauss_jacobi01(n, 1, tb, wb);
  TriRule r;
  r.exactness = degree;
  r.barycentric = Mat(n * n, 3);
  r.weights.resize(n * n);
  int q = 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i, ++q) {
      const double t = tb[j], s = ta[i] * (1.0 - t);
      r.barycentric(q, 0) = 1.0 - s - t;
      r.barycentric(q, 1) = s;
      r.barycentric(q, 2) = t;
      r.weights[q] = 2.0 * wa[i] * wb[j];
    }
  return r;
}

// quadrature.cpp:92-102
std::array<Mat, 4> boundary_points(const TriRule& tri) {
  const int nq = tri.size();
  std::array<Mat, 4> bp;
  for (auto& m : bp) m = Mat(nq, 3);
  for (int r = 0; r < nq; ++r) {
    const double s = tri.barycentric(r, 1), t = tri.barycentric(r, 2);
    bp[0](r, 0) = s; bp[0](r, 1) = t; bp[0](r, 2) = 0.0;
    bp[1](r, 0) = s; bp[1](r, 1) = 0.0; bp[1](r, 2) = t;
    bp[2](r, 0) = 0.0; bp[2](r, 1) = s; bp[2](r, 2) = t;
    bp[3](r, 0) = s; bp[3](r, 1) = t; bp[3](r, 2) = 1.0 - s - t;
  }
  return bp;
}

// -------------------------------------------------------------------- basis
namespace {
// basis.cpp:12-33
void jacobi_homog(int nmax, int alpha, double a, double b, double* p, double* pa, double* pb) {
  const double al = alpha;
  p[0] = 1.0;
  if (pa) { pa[0] = 0.0; pb[0] = 0.0; }
  if (nmax == 0) return;
  p[1] = 0.5 * ((al + 2.0) * a + al * b);
  if (pa) { pa[1] = 0.5 * (al + 2.0); pb[1] = 0.5 * al; }
  for (int n = 2; n <= nmax; ++n) {
    const double c0 = 2.0 * n * (n + al) * (2.0 * n + al - 2.0);
    const double A = (2.0 * n + al - 1.0) * (2.0 * n + al) * (2.0 * n + al - 2.0);
    const double B = (2.0 * n + al - 1.0) * al * al;
    const double C = 2.0 * (n + al - 1.0) * (n - 1.0) * (2.0 * n + al);
    const double lin = A * a + B * b;
    p[n] = (lin * p[n - 1] - C * b * b * p[n - 2]) / c0;
    if (pa) {
      pa[n] = (A * p[n - 1] + lin * pa[n - 1] - C * b * b * pa[n - 2]) / c0;
      pb[n] = (B * p[n - 1] + lin * pb[n - 1] - C * (2.0 * b * p[n - 2] + b * b * pb[n - 2])) / c0;
    }
  }
}

// basis.cpp:37-54 + 56-101
void eval3(int k, const Mat& pts, Mat* P, Mat* Px, Mat* Py, Mat* Pz) {
  const int n = pts.r, d3 = dim3(k);
  const bool grad = Px != nullptr;
  if (P) *P = Mat(n, d3);
  if (grad) { *Px = Mat(n, d3); *Py = Mat(n, d3); *Pz = Mat(n, d3); }
  struct Idx { int i, j, m; };
  std::vector<Idx> idx;
  for (int d = 0; d <= k; ++d)
    for (int i = 0; i <= d; ++i)
      for (int j = 0; i + j <= d; ++j) idx.push_back({i, j, d - i - j});
  std::vector<double> q(k + 1), qa(k + 1), qb(k + 1), s(k + 1), sa(k + 1), sb(k + 1);
  std::vector<std::vector<double>> r(k + 1, std::vector<double>(k + 1)),
      ra(k + 1, std::vector<double>(k + 1)), rb(k + 1, std::vector<double>(k + 1));
  for (int p = 0; p < n; ++p) {
    const double x = pts(p, 0), y = pts(p, 1), z = pts(p, 2);
    const double b1 = 1.0 - y - z, a1 = 2.0 * x - b1;
    const double b2 = 1.0 - z, a2 = 2.0 * y - b2;
    const double t3 = 2.0 * z - 1.0;
    jacobi_homog(k, 0, a1, b1, q.data(), grad ? qa.data() : nullptr, grad ? qb.data() : nullptr);
    for (int i = 0; i <= k; ++i)
      jacobi_homog(k - i, 2 * i + 1, a2, b2, r[i].data(), grad ? ra[i].data() : nullptr,
                   grad ? rb[i].data() : nullptr);
    int prev_alpha = -1;
    for (int col = 0; col < d3; ++col) {
      const auto [i, j, m] = idx[col];
      const int alpha = 2 * i + 2 * j + 2;
      if (alpha != prev_alpha) {
        jacobi_homog(k - i - j, alpha, t3, 1.0, s.data(), grad ? sa.data() : nullptr,
                     grad ? sb.data() : nullptr);
        prev_alpha = alpha;
      }
      const double N = std::sqrt(2.0 * (2 * i + 1) * (i + j + 1) * (2 * i + 2 * j + 2 * m + 3));
      const double qi = q[i], rj = r[i][j], sm = s[m];
      if (P) (*P)(p, col) = N * qi * rj * sm;
      if (grad) {
        const double qd = qa[i] - qb[i];
        const double rd = ra[i][j] - rb[i][j];
        (*Px)(p, col) = N * 2.0 * qa[i] * rj * sm;
        (*Py)(p, col) = N * (qd * rj + qi * 2.0 * ra[i][j]) * sm;
        (*Pz)(p, col) = N * (qd * rj * sm + qi * rd * sm + qi * rj * 2.0 * sa[m]);
      }
    }
  }
}
}  // namespace

Mat eval_dubiner3d(int k, const Mat& pts) {
  Mat P;
  eval3(k, pts, &P, nullptr, nullptr, nullptr);
  return P;
}
void eval_dubiner3d_grad(int k, const Mat& pts, Mat& Px, Mat& Py, Mat& Pz) {
  eval3(k, pts, nullptr, &Px, &Py, &Pz);
}

// basis.cpp:116-134
Mat eval_dubiner2d(int k, const Mat& pts) {
  const int n = pts.r;
  Mat D(n, dim2(k));
  std::vector<double> q(k + 1), s(k + 1);
  for (int p = 0; p < n; ++p) {
    const double sx = pts(p, 0), t = pts(p, 1);
    const double b = 1.0 - t, a = 2.0 * sx - b;
    jacobi_homog(k, 0, a, b, q.data(), nullptr, nullptr);
    int col = 0;
    for (int d = 0; d <= k; ++d)
      for (int i = 0; i <= d; ++i, ++col) {
        const int j = d - i;
        jacobi_homog(j, 2 * i + 1, 2.0 * t - 1.0, 1.0, s.data(), nullptr, nullptr);
        D(p, col) = std::sqrt(2.0 * (2 * i + 1) * (i + j + 1)) * q[i] * s[j];
      }
  }
  return D;
}

// basis.cpp:136-165
BasisTables build_tables(int k, const TetRule& tet, const TriRule& tri) {
  BasisTables tb;
  tb.k = k;
  tb.d3 = dim3(k);
  tb.d2 = dim2(k);
  Mat vol(tet.size(), 3);
  for (int q = 0; q < tet.size(); ++q)
    for (int c = 0; c < 3; ++c) vol(q, c) = tet.barycentric(q, c + 1);
  eval3(k, vol, &tb.P, &tb.Px, &tb.Py, &tb.Pz);
  const auto bp = boundary_points(tri);
  for (int l = 0; l < 4; ++l) tb.Pface[l] = eval_dubiner3d(k, bp[l]);
  const int nq = tri.size();
  Mat tp(nq, 2);
  for (int r = 0; r < nq; ++r) { tp(r, 0) = tri.barycentric(r, 1); tp(r, 1) = tri.barycentric(r, 2); }
  tb.D = eval_dubiner2d(k, tp);
  for (int mu = 0; mu < 6; ++mu) {
    Mat mp(nq, 2);
    for (int r = 0; r < nq; ++r) {
      const double s = tp(r, 0), t = tp(r, 1), u = 1.0 - s - t;
      const double F[6][2] = {{s, t}, {t, s}, {t, u}, {s, u}, {u, s}, {u, t}};
      mp(r, 0) = F[mu][0];
      mp(r, 1) = F[mu][1];
    }
    tb.Dperm[mu] = eval_dubiner2d(k, mp);
  }
  return tb;
}

// ---------------------------------------------------------- element matrices
// element_matrices.cpp:25-46
StabilizationField StabilizationField::constant(const ExpandedMesh& em, double v) {
  StabilizationField s;
  s.tau = Mat(em.n_elements(), 4, v);
  return s;
}
Mat StabilizationField::scaled(const ExpandedMesh& em) const {
  Mat T(tau.r, 4);
  for (int K = 0; K < tau.r; ++K)
    for (int l = 0; l < 4; ++l) T(K, l) = tau(K, l) * em.area[em.facebyele(K, l)];
  return T;
}
void StabilizationField::validate() const {
  for (double t : tau.a)
    if (t < 0) throw std::invalid_argument("stabilization must be nonnegative");
  if (allow_zero) return;
  for (int K = 0; K < tau.r; ++K) {
    double mx = tau(K, 0);
    for (int l = 1; l < 4; ++l) mx = std::max(mx, tau(K, l));
    if (mx <= 0)
      throw std::invalid_argument("stabilization vanishes identically on element " +
                                  std::to_string(K));
  }
}

// element_matrices.cpp:48-57
Mat piola_coefficients(const ExpandedMesh& em) {
  const int nelt = em.n_elements();
  Mat a(nelt, 9);
  for (int K = 0; K < nelt; ++K) {
    const ElementGeometry g = geometry(em.raw, K);
    for (int i = 0; i < 9; ++i) a(K, i) = g.a[i];
  }
  return a;
}
// element_matrices.cpp:59-64
Mat normal_weights(const ExpandedMesh& em, int star) {
  Mat n(em.n_elements(), 4);
  for (int K = 0; K < em.n_elements(); ++K)
    for (int l = 0; l < 4; ++l) n(K, l) = em.normals(K, 3 * l + star);
  return n;
}

namespace {
// lambda (nq x 4) * nodal (4 x Nelt) — mesh.cpp:255-268 + element_matrices.cpp:66-70
PhysicalPoints map_points(const ExpandedMesh& em, const Mat& lambda) {
  const int nelt = em.n_elements(), nq = lambda.r;
  PhysicalPoints pp{Mat(nq, nelt), Mat(nq, nelt), Mat(nq, nelt)};
  const Mat& X = em.raw.coordinates;
  for (int K = 0; K < nelt; ++K) {
    double xv[4][3];
    for (int i = 0; i < 4; ++i)
      for (int c = 0; c < 3; ++c) xv[i][c] = X(em.raw.elements(K, i), c);
    for (int q = 0; q < nq; ++q) {
      double s[3] = {0, 0, 0};
      for (int i = 0; i < 4; ++i)
        for (int c = 0; c < 3; ++c) s[c] += lambda(q, i) * xv[i][c];
      pp.X(q, K) = s[0];
      pp.Y(q, K) = s[1];
      pp.Z(q, K) = s[2];
    }
  }
  return pp;
}
// xi(K,l) * 1{perm(K,l) == mu} — element_matrices.cpp:15-21
std::vector<double> masked_column(const ExpandedMesh& em, const Mat& xi, int l, int mu) {
  std::vector<double> out(em.n_elements(), 0.0);
  for (int K = 0; K < em.n_elements(); ++K)
    if (em.perm(K, l) == mu) out[K] = xi(K, l);
  return out;
}
// flat += vecW * coef^T   (the reference's rank-one batch update)
void rank1(Batch3& out, const std::vector<double>& vecW, const double* coef) {
  const size_t rc = size_t(out.rows) * out.cols;
  for (int K = 0; K < out.count; ++K) {
    const double c = coef[K];
    double* s = out.slice(K);
    for (size_t i = 0; i < rc; ++i) s[i] += vecW[i] * c;
  }
}
}  // namespace

PhysicalPoints quad_points_physical(const ExpandedMesh& em, const TetRule& rule) {
  return map_points(em, rule.barycentric);
}
// element_matrices.cpp:72-82
PhysicalPoints face_points_physical(const ExpandedMesh& em, const TriRule& tri, int l) {
  const auto bp = boundary_points(tri);
  Mat lambda(bp[l].r, 4);
  for (int r = 0; r < bp[l].r; ++r) {
    lambda(r, 0) = 1.0 - (bp[l](r, 0) + bp[l](r, 1) + bp[l](r, 2));
    for (int c = 0; c < 3; ++c) lambda(r, c + 1) = bp[l](r, c);
  }
  return map_points(em, lambda);
}
Mat sample(const ScalarField& f, const PhysicalPoints& pp) {
  Mat out(pp.X.r, pp.X.c);
  for (size_t i = 0; i < out.a.size(); ++i) out.a[i] = f(pp.X.a[i], pp.Y.a[i], pp.Z.a[i]);
  return out;
}

// element_matrices.cpp:84-92
Mat source_vectors(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule,
                   const ScalarField& f) {
  const int nelt = em.n_elements(), nq = rule.size(), d3 = tb.d3;
  const Mat fv = sample(f, quad_points_physical(em, rule));
  Mat out(d3, nelt);
  for (int K = 0; K < nelt; ++K) {
    for (int i = 0; i < d3; ++i) {
      double s = 0;
      for (int q = 0; q < nq; ++q) s += tb.P(q, i) * (rule.weights[q] * fv(q, K));
      out(i, K) = s * em.volume[K];
    }
  }
  return out;
}

// element_matrices.cpp:94-109
Batch3 mass_matrices(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule,
                     const ScalarField& m) {
  const int d3 = tb.d3, nelt = em.n_elements();
  Mat M = sample(m, quad_points_physical(em, rule));
  for (int K = 0; K < nelt; ++K)
    for (int q = 0; q < M.r; ++q) M(q, K) *= em.volume[K];
  Batch3 out(d3, d3, nelt);
  std::vector<double> W(size_t(d3) * d3), row(nelt);
  for (int q = 0; q < rule.size(); ++q) {
    for (int j = 0; j < d3; ++j)
      for (int i = 0; i < d3; ++i) W[i + size_t(j) * d3] = rule.weights[q] * tb.P(q, i) * tb.P(q, j);
    for (int K = 0; K < nelt; ++K) row[K] = M(q, K);
    rank1(out, W, row.data());
  }
  return out;
}

// element_matrices.cpp:111-128
void convection_matrices(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule,
                         Batch3& Cx, Batch3& Cy, Batch3& Cz) {
  const int d3 = tb.d3, nelt = em.n_elements(), nq = rule.size();
  const Mat a = piola_coefficients(em);
  const Mat* Pd[3] = {&tb.Px, &tb.Py, &tb.Pz};
  std::array<std::vector<double>, 3> Chat;
  for (int s = 0; s < 3; ++s) {
    Chat[s].assign(size_t(d3) * d3, 0.0);
    for (int j = 0; j < d3; ++j)
      for (int i = 0; i < d3; ++i) {
        double acc = 0;
        for (int q = 0; q < nq; ++q) acc += (rule.weights[q] * tb.P(q, i)) * (*Pd[s])(q, j);
        Chat[s][i + size_t(j) * d3] = acc / 6.0;
      }
  }
  Batch3* out[3] = {&Cx, &Cy, &Cz};
  std::vector<double> col(nelt);
  for (int star = 0; star < 3; ++star) {
    *out[star] = Batch3(d3, d3, nelt);
    for (int sharp = 0; sharp < 3; ++sharp) {
      for (int K = 0; K < nelt; ++K) col[K] = a(K, 3 * star + sharp);
      rank1(*out[star], Chat[sharp], col.data());
    }
  }
}

// element_matrices.cpp:130-153
void variable_convection_matrices(const ExpandedMesh& em, const BasisTables& tb,
                                  const TetRule& rule, const ScalarField& m, Batch3& Cx,
                                  Batch3& Cy, Batch3& Cz) {
  const int d3 = tb.d3, nelt = em.n_elements();
  const Mat a = piola_coefficients(em);
  const Mat M = sample(m, quad_points_physical(em, rule));
  Batch3* out[3] = {&Cx, &Cy, &Cz};
  const Mat* Pd[3] = {&tb.Px, &tb.Py, &tb.Pz};
  for (int s = 0; s < 3; ++s) *out[s] = Batch3(d3, d3, nelt);
  std::vector<double> W(size_t(d3) * d3), coef(nelt);
  for (int q = 0; q < rule.size(); ++q)
    for (int sharp = 0; sharp < 3; ++sharp) {
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < d3; ++i)
          W[i + size_t(j) * d3] = (rule.weights[q] / 6.0) * tb.P(q, i) * (*Pd[sharp])(q, j);
      for (int star = 0; star < 3; ++star) {
        for (int K = 0; K < nelt; ++K) coef[K] = M(q, K) * a(K, 3 * star + sharp);
        rank1(*out[star], W, coef.data());
      }
    }
}

// element_matrices.cpp:155-167
Batch3 type_a(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri, const Mat& xi) {
  const int d3 = tb.d3, nq = tri.size();
  Batch3 out(d3, d3, em.n_elements());
  std::vector<double> W(size_t(d3) * d3);
  for (int l = 0; l < 4; ++l) {
    for (int j = 0; j < d3; ++j)
      for (int i = 0; i < d3; ++i) {
        double s = 0;
        for (int r = 0; r < nq; ++r) s += tb.Pface[l](r, i) * tri.weights[r] * tb.Pface[l](r, j);
        W[i + size_t(j) * d3] = s;
      }
    rank1(out, W, xi.col(l));
  }
  return out;
}

// element_matrices.cpp:169-180
Batch3 type_b(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri, const Mat& xi) {
  const int d2 = tb.d2, nelt = em.n_elements(), nq = tri.size(), m = 4 * d2;
  Mat W(d2, d2);
  for (int j = 0; j < d2; ++j)
    for (int i = 0; i < d2; ++i) {
      double s = 0;
      for (int r = 0; r < nq; ++r) s += tb.D(r, i) * tri.weights[r] * tb.D(r, j);
      W(i, j) = s;
    }
  Batch3 out(m, m, nelt);
  for (int K = 0; K < nelt; ++K) {
    double* S = out.slice(K);
    for (int l = 0; l < 4; ++l)
      for (int j = 0; j < d2; ++j)
        for (int i = 0; i < d2; ++i) S[(l * d2 + i) + size_t(l * d2 + j) * m] = xi(K, l) * W(i, j);
  }
  return out;
}

namespace {
// copy a d2 x cols block batch into rows [l*d2, (l+1)*d2) of a 4d2 x cols batch
void place_rows(Batch3& out, const Batch3& block, int l) {
  const int d2 = block.rows, cols = block.cols;
  for (int K = 0; K < out.count; ++K) {
    double* S = out.slice(K);
    const double* B = block.slice(K);
    for (int j = 0; j < cols; ++j)
      for (int i = 0; i < d2; ++i) S[(l * d2 + i) + size_t(j) * out.rows] = B[i + size_t(j) * d2];
  }
}
void place_diag(Batch3& out, const Batch3& block, int l) {
  const int d2 = block.rows;
  for (int K = 0; K < out.count; ++K) {
    double* S = out.slice(K);
    const double* B = block.slice(K);
    for (int j = 0; j < d2; ++j)
      for (int i = 0; i < d2; ++i)
        S[(l * d2 + i) + size_t(l * d2 + j) * out.rows] = B[i + size_t(j) * d2];
  }
}
}  // namespace

// element_matrices.cpp:182-202
Batch3 type_c(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri, const Mat& xi) {
  const int d2 = tb.d2, d3 = tb.d3, nelt = em.n_elements(), nq = tri.size();
  Batch3 out(4 * d2, d3, nelt);
  std::vector<double> W(size_t(d2) * d3);
  for (int l = 0; l < 4; ++l) {
    Batch3 block(d2, d3, nelt);
    for (int mu = 1; mu <= 6; ++mu) {
      const auto coef = masked_column(em, xi, l, mu);
      bool any = false;
      for (double c : coef) any |= (c != 0.0);
      if (!any) continue;
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < d2; ++i) {
          double s = 0;
          for (int r = 0; r < nq; ++r)
            s += tb.Dperm[mu - 1](r, i) * tri.weights[r] * tb.Pface[l](r, j);
          W[i + size_t(j) * d2] = s;
        }
      rank1(block, W, coef.data());
    }
    place_rows(out, block, l);
  }
  return out;
}

// element_matrices.cpp:204-229
Batch3 variable_surface_dp(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri,
                           const ScalarField& alpha, const Mat& xi) {
  const int d2 = tb.d2, d3 = tb.d3, nelt = em.n_elements();
  Batch3 out(4 * d2, d3, nelt);
  std::vector<double> W(size_t(d2) * d3), c2(nelt);
  for (int l = 0; l < 4; ++l) {
    const Mat A = sample(alpha, face_points_physical(em, tri, l));
    Batch3 block(d2, d3, nelt);
    for (int mu = 1; mu <= 6; ++mu) {
      const auto coef = masked_column(em, xi, l, mu);
      bool any = false;
      for (double c : coef) any |= (c != 0.0);
      if (!any) continue;
      for (int r = 0; r < tri.size(); ++r) {
        for (int j = 0; j < d3; ++j)
          for (int i = 0; i < d2; ++i)
            W[i + size_t(j) * d2] = tri.weights[r] * tb.Dperm[mu - 1](r, i) * tb.Pface[l](r, j);
        for (int K = 0; K < nelt; ++K) c2[K] = coef[K] * A(r, K);
        rank1(block, W, c2.data());
      }
    }
    place_rows(out, block, l);
  }
  return out;
}

// element_matrices.cpp:231-256
Batch3 variable_surface_dd(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri,
                           const ScalarField& alpha, const Mat& xi) {
  const int d2 = tb.d2, nelt = em.n_elements();
  Batch3 out(4 * d2, 4 * d2, nelt);
  std::vector<double> W(size_t(d2) * d2), c2(nelt);
  for (int l = 0; l < 4; ++l) {
    const Mat A = sample(alpha, face_points_physical(em, tri, l));
    Batch3 block(d2, d2, nelt);
    for (int mu = 1; mu <= 6; ++mu) {
      const auto coef = masked_column(em, xi, l, mu);
      bool any = false;
      for (double c : coef) any |= (c != 0.0);
      if (!any) continue;
      for (int r = 0; r < tri.size(); ++r) {
        for (int j = 0; j < d2; ++j)
          for (int i = 0; i < d2; ++i)
            W[i + size_t(j) * d2] =
                tri.weights[r] * tb.Dperm[mu - 1](r, i) * tb.Dperm[mu - 1](r, j);
        for (int K = 0; K < nelt; ++K) c2[K] = coef[K] * A(r, K);
        rank1(block, W, c2.data());
      }
    }
    place_diag(out, block, l);
  }
  return out;
}

// element_matrices.cpp:258-280
Batch3 stiffness_matrices(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule) {
  const int d3 = tb.d3, nelt = em.n_elements(), nq = rule.size();
  const Mat a = piola_coefficients(em);
  const Mat* Pd[3] = {&tb.Px, &tb.Py, &tb.Pz};
  Batch3 out(d3, d3, nelt);
  std::vector<double> S(size_t(d3) * d3), g(nelt);
  for (int s1 = 0; s1 < 3; ++s1)
    for (int s2 = 0; s2 < 3; ++s2) {
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < d3; ++i) {
          double acc = 0;
          for (int q = 0; q < nq; ++q) acc += (*Pd[s1])(q, i) * rule.weights[q] * (*Pd[s2])(q, j);
          S[i + size_t(j) * d3] = acc / 6.0;
        }
      for (int K = 0; K < nelt; ++K) {
        double acc = 0;
        for (int star = 0; star < 3; ++star) acc += a(K, 3 * star + s1) * a(K, 3 * star + s2);
        g[K] = acc / (6.0 * em.volume[K]);
      }
      rank1(out, S, g.data());
    }
  return out;
}

// element_matrices.cpp:282-309
ElementMatrixSet build_element_matrices(const ExpandedMesh& em, const BasisTables& tb,
                                        const TetRule& tet, const TriRule& tri,
                                        const ScalarField& kappa, const ScalarField& c,
                                        const ScalarField& f, const StabilizationField& tau) {
  tau.validate();
  ElementMatrixSet ms;
  ms.k = tb.k;
  ms.d3 = tb.d3;
  ms.d2 = tb.d2;
  const ScalarField kinv = [&kappa](double x, double y, double z) { return 1.0 / kappa(x, y, z); };
  ms.Mkinv = mass_matrices(em, tb, tet, kinv);
  ms.Mc = mass_matrices(em, tb, tet, c);
  convection_matrices(em, tb, tet, ms.Cx, ms.Cy, ms.Cz);
  const Mat T = tau.scaled(em);
  ms.tauPP = type_a(em, tb, tri, T);
  ms.tauDP = type_c(em, tb, tri, T);
  ms.nxDP = type_c(em, tb, tri, normal_weights(em, 0));
  ms.nyDP = type_c(em, tb, tri, normal_weights(em, 1));
  ms.nzDP = type_c(em, tb, tri, normal_weights(em, 2));
  ms.tauDD = type_b(em, tb, tri, T);
  ms.fvec = source_vectors(em, tb, tet, f);
  return ms;
}

// convdiff.cpp:5-28
ConvectionBilinearSet convection_bilinear_matrices(const ExpandedMesh& em, const BasisTables& tb,
                                                   const TetRule& tet, const TriRule& tri,
                                                   const VectorField& beta) {
  const int d3 = tb.d3, d2 = tb.d2, nelt = em.n_elements();
  ConvectionBilinearSet out{Batch3(d3, d3, nelt), Batch3(4 * d2, d3, nelt),
                            Batch3(4 * d2, 4 * d2, nelt)};
  const ScalarField* comp[3] = {&beta.x, &beta.y, &beta.z};
  for (int star = 0; star < 3; ++star) {
    Batch3 Cx, Cy, Cz;
    variable_convection_matrices(em, tb, tet, *comp[star], Cx, Cy, Cz);
    const Batch3* pick[3] = {&Cx, &Cy, &Cz};
    for (size_t i = 0; i < out.vol.data.size(); ++i) out.vol.data[i] += pick[star]->data[i];
    const Mat nw = normal_weights(em, star);
    const Batch3 dp = variable_surface_dp(em, tb, tri, *comp[star], nw);
    const Batch3 dd = variable_surface_dd(em, tb, tri, *comp[star], nw);
    for (size_t i = 0; i < out.dp.data.size(); ++i) out.dp.data[i] += dp.data[i];
    for (size_t i = 0; i < out.dd.data.size(); ++i) out.dd.data[i] += dd.data[i];
  }
  return out;
}

// -------------------------------------------------------------- local solver
// Eigen PartialPivLU semantics: at step k pick the row with the largest |a(i,k)|
// (first on ties), swap, scale, rank-1 update.
void PartialPivLU::compute(const double* A, int nn) {
  n = nn;
  lu.assign(A, A + size_t(n) * n);
  perm.resize(n);
  std::iota(perm.begin(), perm.end(), 0);
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = std::fabs(lu[k + size_t(k) * n]);
    for (int i = k + 1; i < n; ++i) {
      const double v = std::fabs(lu[i + size_t(k) * n]);
      if (v > best) { best = v; p = i; }
    }
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(lu[k + size_t(j) * n], lu[p + size_t(j) * n]);
      std::swap(perm[k], perm[p]);
    }
    const double piv = lu[k + size_t(k) * n];
    if (piv != 0.0)
      for (int i = k + 1; i < n; ++i) lu[i + size_t(k) * n] /= piv;
    for (int j = k + 1; j < n; ++j) {
      const double ukj = lu[k + size_t(j) * n];
      if (ukj == 0.0) continue;
      double* cj = &lu[size_t(j) * n];
      const double* ck = &lu[size_t(k) * n];
      for (int i = k + 1; i < n; ++i) cj[i] -= ck[i] * ukj;
    }
  }
}
void PartialPivLU::solve(double* B, int ncols) const {
  std::vector<double> tmp(n);
  for (int c = 0; c < ncols; ++c) {
    double* b = B + size_t(c) * n;
    for (int i = 0; i < n; ++i) tmp[i] = b[perm[i]];
    for (int j = 0; j < n; ++j) {  // L (unit) forward, column-oriented
      const double v = tmp[j];
      if (v == 0.0) continue;
      const double* cj = &lu[size_t(j) * n];
      for (int i = j + 1; i < n; ++i) tmp[i] -= cj[i] * v;
    }
    for (int j = n - 1; j >= 0; --j) {  // U backward
      tmp[j] /= lu[j + size_t(j) * n];
      const double v = tmp[j];
      const double* cj = &lu[size_t(j) * n];
      for (int i = 0; i < j; ++i) tmp[i] -= cj[i] * v;
    }
    for (int i = 0; i < n; ++i) b[i] = tmp[i];
  }
}
double PartialPivLU::min_abs_diag() const {
  double m = HUGE_VAL;
  for (int i = 0; i < n; ++i) m = std::min(m, std::fabs(lu[i + size_t(i) * n]));
  return m;
}
double PartialPivLU::max_abs_diag() const {
  double m = 0;
  for (int i = 0; i < n; ++i) m = std::max(m, std::fabs(lu[i + size_t(i) * n]));
  return m;
}

namespace {
// local_solver.cpp:12-48
LocalBlocks assemble_blocks(const ElementMatrixSet& ms, int nu, bool with_tau) {
  const int d3 = ms.d3, d2 = ms.d2, nelt = ms.fvec.c, m = 4 * d2;
  LocalBlocks lb;
  lb.d3 = d3;
  lb.d2 = d2;
  lb.nu = nu;
  lb.n = 3 * d3 + nu;
  const int n = lb.n;
  lb.A1 = Batch3(n, n, nelt);
  lb.A2 = Batch3(n, m, nelt);
  lb.A3 = Batch3(m, n, nelt);
  lb.Af = Mat(n, nelt);
  lb.tauDD = with_tau ? ms.tauDD : Batch3(m, m, nelt);
  const Batch3* C[3] = {&ms.Cx, &ms.Cy, &ms.Cz};
  const Batch3* nDP[3] = {&ms.nxDP, &ms.nyDP, &ms.nzDP};
  for (int K = 0; K < nelt; ++K) {
    double* A1 = lb.A1.slice(K);
    double* A2 = lb.A2.slice(K);
    double* A3 = lb.A3.slice(K);
    const double* Mk = ms.Mkinv.slice(K);
    for (int s = 0; s < 3; ++s) {
      const double* Cs = C[s]->slice(K);
      const double* Ns = nDP[s]->slice(K);
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < d3; ++i) A1[(s * d3 + i) + size_t(s * d3 + j) * n] = Mk[i + j * d3];
      for (int j = 0; j < nu; ++j)  // -C^T (d3 x nu)
        for (int i = 0; i < d3; ++i) A1[(s * d3 + i) + size_t(3 * d3 + j) * n] = -Cs[j + i * d3];
      for (int j = 0; j < d3; ++j)  // C top rows (nu x d3)
        for (int i = 0; i < nu; ++i) A1[(3 * d3 + i) + size_t(s * d3 + j) * n] = Cs[i + j * d3];
      for (int j = 0; j < m; ++j)  // nDP^T (d3 x m)
        for (int i = 0; i < d3; ++i) A2[(s * d3 + i) + size_t(j) * n] = Ns[j + size_t(i) * m];
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < m; ++i) A3[i + size_t(s * d3 + j) * m] = Ns[i + size_t(j) * m];
    }
    const double* Mc = ms.Mc.slice(K);
    const double* PP = ms.tauPP.slice(K);
    const double* TD = ms.tauDP.slice(K);
    for (int j = 0; j < nu; ++j)
      for (int i = 0; i < nu; ++i) {
        double v = Mc[i + j * d3];
        if (with_tau) v += PP[i + j * d3];
        A1[(3 * d3 + i) + size_t(3 * d3 + j) * n] = v;
      }
    if (with_tau) {
      for (int j = 0; j < m; ++j)
        for (int i = 0; i < nu; ++i) A2[(3 * d3 + i) + size_t(j) * n] = -TD[j + size_t(i) * m];
      for (int j = 0; j < nu; ++j)
        for (int i = 0; i < m; ++i) A3[i + size_t(3 * d3 + j) * m] = TD[i + size_t(j) * m];
    }
    for (int i = 0; i < nu; ++i) lb.Af(3 * d3 + i, K) = ms.fvec(i, K);
  }
  return lb;
}

// local_solver.cpp:50-57
void factor_checked(PartialPivLU& lu, const double* A, int n, int K) {
  lu.compute(A, n);
  const double mx = lu.max_abs_diag();
  if (mx == 0.0 || lu.min_abs_diag() < 1e-14 * mx)
    throw LocalSolverError(K, "singular local system on element " + std::to_string(K));
}
}  // namespace

LocalBlocks local_blocks(const ElementMatrixSet& ms) { return assemble_blocks(ms, ms.d3, true); }
LocalBlocks bdm_blocks(const ElementMatrixSet& ms) {
  if (ms.k < 1) throw std::invalid_argument("the BDM variant needs degree k >= 1");
  return assemble_blocks(ms, ms.d3 - ms.d2, false);
}

// local_solver.cpp:71-100
CondensedSystem condense(const LocalBlocks& lb, int nthreads) {
  const int nelt = lb.A1.count, m = 4 * lb.d2, n = lb.n;
  CondensedSystem cs{Batch3(m, m, nelt), Mat(m, nelt)};
  std::atomic<int> bad{-1};
  parallel_for(nelt, nthreads, [&](int begin, int end) {
    std::vector<double> rhs(size_t(n) * (m + 1));
    PartialPivLU lu;
    for (int K = begin; K < end; ++K) {
      try {
        factor_checked(lu, lb.A1.slice(K), n, K);
      } catch (const LocalSolverError&) {
        int expect = -1;
        bad.compare_exchange_strong(expect, K);
        return;
      }
      std::copy(lb.A2.slice(K), lb.A2.slice(K) + size_t(n) * m, rhs.begin());
      for (int i = 0; i < n; ++i) rhs[size_t(m) * n + i] = lb.Af(i, K);
      lu.solve(rhs.data(), m + 1);
      const double* A3 = lb.A3.slice(K);
      double* C = cs.C.slice(K);
      const double* DD = lb.tauDD.slice(K);
      for (int j = 0; j <= m; ++j) {
        double* out = j < m ? C + size_t(j) * m : cs.Cf.col(K);
        for (int i = 0; i < m; ++i) out[i] = 0.0;
        const double* x = rhs.data() + size_t(j) * n;
        for (int p = 0; p < n; ++p) {
          const double v = x[p];
          const double* a = A3 + size_t(p) * m;
          for (int i = 0; i < m; ++i) out[i] += a[i] * v;
        }
        if (j < m)
          for (int i = 0; i < m; ++i) out[i] += DD[i + size_t(j) * m];
      }
    }
  });
  if (bad.load() >= 0)
    throw LocalSolverError(bad.load(),
                           "singular local system on element " + std::to_string(bad.load()));
  return cs;
}

// local_solver.cpp:102-135
LocalSolution local_recover(const LocalBlocks& lb, const Mat& uhat, int nthreads) {
  const int nelt = lb.A1.count, d3 = lb.d3, n = lb.n, m = 4 * lb.d2;
  LocalSolution out{Mat(d3, nelt), Mat(d3, nelt), Mat(d3, nelt), Mat(d3, nelt)};
  std::atomic<int> bad{-1};
  parallel_for(nelt, nthreads, [&](int begin, int end) {
    std::vector<double> rhs(n);
    PartialPivLU lu;
    for (int K = begin; K < end; ++K) {
      try {
        factor_checked(lu, lb.A1.slice(K), n, K);
      } catch (const LocalSolverError&) {
        int expect = -1;
        bad.compare_exchange_strong(expect, K);
        return;
      }
      for (int i = 0; i < n; ++i) rhs[i] = lb.Af(i, K);
      const double* A2 = lb.A2.slice(K);
      for (int j = 0; j < m; ++j) {
        const double v = uhat(j, K);
        for (int i = 0; i < n; ++i) rhs[i] -= A2[i + size_t(j) * n] * v;
      }
      lu.solve(rhs.data(), 1);
      for (int i = 0; i < d3; ++i) {
        out.qx(i, K) = rhs[i];
        out.qy(i, K) = rhs[d3 + i];
        out.qz(i, K) = rhs[2 * d3 + i];
      }
      for (int i = 0; i < lb.nu; ++i) out.u(i, K) = rhs[3 * d3 + i];
    }
  });
  if (bad.load() >= 0)
    throw LocalSolverError(bad.load(),
                           "singular local system on element " + std::to_string(bad.load()));
  return out;
}

// ------------------------------------------------------------ global system
// global_system.cpp:31-56 — triplets in (K,l1,l2,j,i) order then a compressed
// column-major matrix with duplicates summed (Eigen setFromTriplets).
SkeletonSystem assemble(const ExpandedMesh& em, const CondensedSystem& cs) {
  const int m = cs.C.rows, d2 = m / 4, nelt = em.n_elements();
  const int64_t ndof = int64_t(em.n_faces()) * d2;
  SkeletonSystem sys;
  sys.d2 = d2;
  sys.ndof = ndof;
  sys.b.assign(ndof, 0.0);
  // column c holds rows of every element touching face(c/d2): build per face
  // the sorted list of neighbour faces (pattern), then accumulate.
  const int nfc = em.n_faces();
  std::vector<std::vector<int>> nbr(nfc);
  for (int K = 0; K < nelt; ++K)
    for (int l1 = 0; l1 < 4; ++l1)
      for (int l2 = 0; l2 < 4; ++l2) nbr[em.facebyele(K, l2)].push_back(em.facebyele(K, l1));
  for (auto& v : nbr) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  sys.colptr.assign(ndof + 1, 0);
  for (int f = 0; f < nfc; ++f)
    for (int j = 0; j < d2; ++j) sys.colptr[int64_t(f) * d2 + j + 1] = int64_t(nbr[f].size()) * d2;
  for (int64_t c = 0; c < ndof; ++c) sys.colptr[c + 1] += sys.colptr[c];
  sys.rowidx.resize(sys.colptr[ndof]);
  sys.vals.assign(sys.colptr[ndof], 0.0);
  for (int f = 0; f < nfc; ++f)
    for (int j = 0; j < d2; ++j) {
      int64_t p = sys.colptr[int64_t(f) * d2 + j];
      for (int g : nbr[f])
        for (int i = 0; i < d2; ++i) sys.rowidx[p++] = g * d2 + i;
    }
  for (int K = 0; K < nelt; ++K) {
    const double* C = cs.C.slice(K);
    for (int l1 = 0; l1 < 4; ++l1) {
      const int f1 = em.facebyele(K, l1);
      for (int i = 0; i < d2; ++i) sys.b[int64_t(f1) * d2 + i] += cs.Cf(l1 * d2 + i, K);
      for (int l2 = 0; l2 < 4; ++l2) {
        const int f2 = em.facebyele(K, l2);
        const auto& nb = nbr[f2];
        const int pos = int(std::lower_bound(nb.begin(), nb.end(), f1) - nb.begin());
        for (int j = 0; j < d2; ++j) {
          const int64_t base = sys.colptr[int64_t(f2) * d2 + j] + int64_t(pos) * d2;
          for (int i = 0; i < d2; ++i)
            sys.vals[base + i] += C[(l1 * d2 + i) + size_t(l2 * d2 + j) * m];
        }
      }
    }
  }
  return sys;
}

// global_system.cpp:9-29
void face_quad_points(const ExpandedMesh& em, const std::vector<int>& faces, const TriRule& tri,
                      Mat& X, Mat& Y, Mat& Z) {
  const int n = int(faces.size()), nq = tri.size();
  X = Mat(nq, n);
  Y = Mat(nq, n);
  Z = Mat(nq, n);
  const Mat& C = em.raw.coordinates;
  for (int j = 0; j < n; ++j) {
    const int f = faces[j];
    for (int r = 0; r < nq; ++r) {
      const double s = tri.barycentric(r, 1), t = tri.barycentric(r, 2);
      double p[3];
      for (int c = 0; c < 3; ++c)
        p[c] = (1.0 - s - t) * C(em.faces(f, 0), c) + s * C(em.faces(f, 1), c) +
               t * C(em.faces(f, 2), c);
      X(r, j) = p[0];
      Y(r, j) = p[1];
      Z(r, j) = p[2];
    }
  }
}

namespace {
Mat tri_points(const TriRule& tri) {
  Mat tp(tri.size(), 2);
  for (int r = 0; r < tri.size(); ++r) { tp(r, 0) = tri.barycentric(r, 1); tp(r, 1) = tri.barycentric(r, 2); }
  return tp;
}
}  // namespace

// global_system.cpp:58-70
std::vector<double> dirichlet_project(const ExpandedMesh& em, int k, const TriRule& tri,
                                      const ScalarField& g) {
  const int d2 = dim2(k), n = em.n_dirichlet(), nq = tri.size();
  Mat X, Y, Z;
  face_quad_points(em, em.dirfaces, tri, X, Y, Z);
  const Mat D = eval_dubiner2d(k, tri_points(tri));
  std::vector<double> out(size_t(n) * d2);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < d2; ++i) {
      double s = 0;
      for (int r = 0; r < nq; ++r) s += D(r, i) * tri.weights[r] * g(X(r, j), Y(r, j), Z(r, j));
      out[size_t(j) * d2 + i] = 0.5 * s;
    }
  return out;
}

// global_system.cpp:72-104
std::vector<double> neumann_load(const ExpandedMesh& em, int k, const TriRule& tri,
                                 const VectorField& g) {
  const int d2 = dim2(k), n = em.n_neumann(), nq = tri.size();
  std::vector<double> out(size_t(em.n_faces()) * d2, 0.0);
  if (n == 0) return out;
  std::vector<int> adjK(em.n_faces(), -1), adjl(em.n_faces(), -1);
  for (int K = 0; K < em.n_elements(); ++K)
    for (int l = 0; l < 4; ++l) {
      const int f = em.facebyele(K, l);
      if (adjK[f] < 0) { adjK[f] = K; adjl[f] = l; }
    }
  Mat X, Y, Z;
  face_quad_points(em, em.neufaces, tri, X, Y, Z);
  const Mat D = eval_dubiner2d(k, tri_points(tri));
  for (int j = 0; j < n; ++j) {
    const int f = em.neufaces[j];
    const double nx = em.normals(adjK[f], 3 * adjl[f]), ny = em.normals(adjK[f], 3 * adjl[f] + 1),
                 nz = em.normals(adjK[f], 3 * adjl[f] + 2);
    std::vector<double> gn(nq);
    for (int r = 0; r < nq; ++r) {
      const double x = X(r, j), y = Y(r, j), z = Z(r, j);
      gn[r] = g.x(x, y, z) * nx + g.y(x, y, z) * ny + g.z(x, y, z) * nz;
    }
    for (int i = 0; i < d2; ++i) {
      double s = 0;
      for (int r = 0; r < nq; ++r) s += D(r, i) * (tri.weights[r] * gn[r]);
      out[size_t(f) * d2 + i] = s;
    }
  }
  return out;
}

// global_system.cpp:167-175
Mat gather_traces(const ExpandedMesh& em, int d2, const double* uhat) {
  Mat out(4 * d2, em.n_elements());
  for (int K = 0; K < em.n_elements(); ++K)
    for (int l = 0; l < 4; ++l)
      for (int i = 0; i < d2; ++i) out(l * d2 + i, K) = uhat[size_t(em.facebyele(K, l)) * d2 + i];
  return out;
}

// ---------------------------------------------------------------- postprocess
// postprocess.cpp:33-74
Mat postprocess_star(const ExpandedMesh& em, const BasisTables& tb1, const TetRule& rule,
                     const ScalarField& kappa, const LocalSolution& ls, int nthreads) {
  const int d31 = tb1.d3, nelt = em.n_elements(), d3 = ls.u.r, nq = rule.size();
  const double kSqrt6 = 2.449489742783178;
  const Batch3 S = stiffness_matrices(em, tb1, rule);
  const PhysicalPoints pp = quad_points_physical(em, rule);
  Mat Kinv = sample(kappa, pp);
  for (double& v : Kinv.a) v = 1.0 / v;
  const Mat a = piola_coefficients(em);
  const Mat* Pd[3] = {&tb1.Px, &tb1.Py, &tb1.Pz};
  const Mat* Qc[3] = {&ls.qx, &ls.qy, &ls.qz};
  Mat R(d31, nelt);
  std::vector<double> Qs(size_t(3) * nq), G(nq);
  for (int K = 0; K < nelt; ++K) {
    for (int s = 0; s < 3; ++s)
      for (int q = 0; q < nq; ++q) {
        double v = 0;
        for (int i = 0; i < d3; ++i) v += tb1.P(q, i) * (*Qc[s])(i, K);
        Qs[s * nq + q] = v * Kinv(q, K);
      }
    for (int sharp = 0; sharp < 3; ++sharp) {
      for (int q = 0; q < nq; ++q) {
        double g = 0;
        for (int star = 0; star < 3; ++star) g += Qs[star * nq + q] * a(K, 3 * star + sharp);
        G[q] = g;
      }
      for (int i = 0; i < d31; ++i) {
        double acc = 0;
        for (int q = 0; q < nq; ++q) acc += (*Pd[sharp])(q, i) * (rule.weights[q] * G[q]);
        R(i, K) -= (1.0 / 6.0) * acc;
      }
    }
  }
  Mat out(d31, nelt);
  parallel_for(nelt, nthreads, [&](int begin, int end) {
    std::vector<double> A(size_t(d31) * d31), rhs(d31);
    PartialPivLU lu;
    for (int K = begin; K < end; ++K) {
      const double detB = 6.0 * em.volume[K];
      std::copy(S.slice(K), S.slice(K) + size_t(d31) * d31, A.begin());
      for (int i = 0; i < d31; ++i) rhs[i] = R(i, K);
      for (int j = 0; j < d31; ++j) A[0 + size_t(j) * d31] = 0.0;
      A[0] = detB / kSqrt6;
      rhs[0] = detB / kSqrt6 * ls.u(0, K);
      lu.compute(A.data(), d31);
      lu.solve(rhs.data(), 1);
      for (int i = 0; i < d31; ++i) out(i, K) = rhs[i];
    }
  });
  return out;
}

// postprocess.cpp:76-82
Mat l2_project_volume(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule,
                      const ScalarField& f) {
  const Mat F = sample(f, quad_points_physical(em, rule));
  Mat out(tb.d3, em.n_elements());
  for (int K = 0; K < em.n_elements(); ++K)
    for (int i = 0; i < tb.d3; ++i) {
      double s = 0;
      for (int q = 0; q < rule.size(); ++q) s += tb.P(q, i) * (rule.weights[q] * F(q, K));
      out(i, K) = s / 6.0;
    }
  return out;
}

// postprocess.cpp:84-93
Mat l2_project_skeleton(const ExpandedMesh& em, int k, const TriRule& tri, const ScalarField& fn) {
  std::vector<int> all(em.n_faces());
  std::iota(all.begin(), all.end(), 0);
  Mat X, Y, Z;
  face_quad_points(em, all, tri, X, Y, Z);
  const Mat D = eval_dubiner2d(k, tri_points(tri));
  const int d2 = dim2(k), nq = tri.size();
  Mat out(d2, em.n_faces());
  for (int f = 0; f < em.n_faces(); ++f)
    for (int i = 0; i < d2; ++i) {
      double s = 0;
      for (int r = 0; r < nq; ++r) s += D(r, i) * (tri.weights[r] * fn(X(r, f), Y(r, f), Z(r, f)));
      out(i, f) = 0.5 * s;
    }
  return out;
}

// postprocess.cpp:95-177
LocalSolution hdg_project(const ExpandedMesh& em, const ElementMatrixSet& ms,
                          const BasisTables& tb, const TetRule& tet, const TriRule& tri,
                          const StabilizationField& tau, const VectorField& q,
                          const ScalarField& u, int nthreads) {
  const int d3 = tb.d3, d2 = tb.d2, nelt = em.n_elements(), t = d3 - d2, n = 4 * d3;
  const int nq = tet.size(), nqd = tri.size();
  const PhysicalPoints pp = quad_points_physical(em, tet);
  const ScalarField* comps[4] = {&q.x, &q.y, &q.z, &u};
  std::array<Mat, 4> Vm;
  for (int c = 0; c < 4; ++c) {
    const Mat F = sample(*comps[c], pp);
    Vm[c] = Mat(d3, nelt);
    for (int K = 0; K < nelt; ++K)
      for (int i = 0; i < d3; ++i) {
        double s = 0;
        for (int qq = 0; qq < nq; ++qq) s += tet.weights[qq] * tb.P(qq, i) * F(qq, K);
        Vm[c](i, K) = s;
      }
  }
  const Mat T = tau.scaled(em);
  Mat Bmom(4 * d2, nelt);
  for (int l = 0; l < 4; ++l) {
    const PhysicalPoints fp = face_points_physical(em, tri, l);
    for (int K = 0; K < nelt; ++K) {
      const int mu = em.perm(K, l);
      for (int i = 0; i < d2; ++i) {
        double s = 0;
        for (int r = 0; r < nqd; ++r) {
          const double x = fp.X(r, K), y = fp.Y(r, K), z = fp.Z(r, K);
          const double g = q.x(x, y, z) * em.normals(K, 3 * l) + q.y(x, y, z) * em.normals(K, 3 * l + 1) +
                           q.z(x, y, z) * em.normals(K, 3 * l + 2) + u(x, y, z) * T(K, l);
          s += tb.Dperm[mu - 1](r, i) * (tri.weights[r] * g);
        }
        Bmom(l * d2 + i, K) += s;
      }
    }
  }
  LocalSolution out{Mat(d3, nelt), Mat(d3, nelt), Mat(d3, nelt), Mat(d3, nelt)};
  const Batch3* nDP[3] = {&ms.nxDP, &ms.nyDP, &ms.nzDP};
  std::atomic<int> bad{-1};
  parallel_for(nelt, nthreads, [&](int begin, int end) {
    std::vector<double> A(size_t(n) * n), rhs(n);
    PartialPivLU lu;
    for (int K = begin; K < end; ++K) {
      const double vol = em.volume[K];
      std::fill(A.begin(), A.end(), 0.0);
      for (int c = 0; c < 4; ++c)
        for (int mm = 0; mm < t; ++mm) {
          A[(c * t + mm) + size_t(c * d3 + mm) * n] = 6.0 * vol;
          rhs[c * t + mm] = vol * Vm[c](mm, K);
        }
      const int m4 = 4 * d2;
      for (int s = 0; s < 3; ++s) {
        const double* N = nDP[s]->slice(K);
        for (int j = 0; j < d3; ++j)
          for (int i = 0; i < m4; ++i) A[(4 * t + i) + size_t(s * d3 + j) * n] = N[i + size_t(j) * m4];
      }
      const double* TD = ms.tauDP.slice(K);
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < m4; ++i) A[(4 * t + i) + size_t(3 * d3 + j) * n] = TD[i + size_t(j) * m4];
      for (int i = 0; i < m4; ++i) rhs[4 * t + i] = Bmom(i, K);
      lu.compute(A.data(), n);
      const double mx = lu.max_abs_diag();
      if (mx == 0.0 || lu.min_abs_diag() < 1e-14 * mx) {
        int expect = -1;
        bad.compare_exchange_strong(expect, K);
        return;
      }
      lu.solve(rhs.data(), 1);
      for (int i = 0; i < d3; ++i) {
        out.qx(i, K) = rhs[i];
        out.qy(i, K) = rhs[d3 + i];
        out.qz(i, K) = rhs[2 * d3 + i];
        out.u(i, K) = rhs[3 * d3 + i];
      }
    }
  });
  if (bad.load() >= 0) throw LocalSolverError(bad.load(), "singular projection system");
  return out;
}

// postprocess.cpp:189-263
ErrorReport compute_errors(const ExpandedMesh& em, const ElementMatrixSet& ms,
                           const StabilizationField& tau, const ScalarField& u_exact,
                           const VectorField& q_exact, int k, const double* uhat,
                           const LocalSolution& fields, const Mat* ustar, int nthreads) {
  const int d2 = dim2(k), nelt = em.n_elements();
  const TetRule tet = tet_rule(2 * k + 4);
  const TriRule tri = tri_rule(2 * k + 4);
  const BasisTables tb = build_tables(k, tet, tri);
  const PhysicalPoints pp = quad_points_physical(em, tet);
  const int nq = tet.size();
  auto vol_err = [&](const Mat& P, const Mat* C, const Mat& F) {
    double tot = 0;
    for (int K = 0; K < nelt; ++K) {
      double per = 0;
      for (int q = 0; q < nq; ++q) {
        double d = F(q, K);
        if (C)
          for (int i = 0; i < C->r; ++i) d -= P(q, i) * (*C)(i, K);
        per += tet.weights[q] * d * d;
      }
      tot += per * em.volume[K];
    }
    return tot;
  };
  const Mat Qx = sample(q_exact.x, pp), Qy = sample(q_exact.y, pp), Qz = sample(q_exact.z, pp);
  const Mat U = sample(u_exact, pp);
  const double nq2 = vol_err(tb.P, nullptr, Qx) + vol_err(tb.P, nullptr, Qy) + vol_err(tb.P, nullptr, Qz);
  const double eq2 = vol_err(tb.P, &fields.qx, Qx) + vol_err(tb.P, &fields.qy, Qy) +
                     vol_err(tb.P, &fields.qz, Qz);
  const double nu2 = vol_err(tb.P, nullptr, U);
  const double eu2 = vol_err(tb.P, &fields.u, U);
  auto rel = [](double e2, double n2) { return std::sqrt(n2 > 0 ? e2 / n2 : e2); };
  ErrorReport rep;
  rep.e_q = rel(eq2, nq2);
  rep.e_u = rel(eu2, nu2);
  std::vector<int> all(em.n_faces());
  std::iota(all.begin(), all.end(), 0);
  Mat Xf, Yf, Zf;
  face_quad_points(em, all, tri, Xf, Yf, Zf);
  const Mat D = eval_dubiner2d(k, tri_points(tri));
  double nhat2 = 0, ehat2 = 0;
  for (int f = 0; f < em.n_faces(); ++f) {
    double sU = 0, sD = 0;
    for (int r = 0; r < tri.size(); ++r) {
      const double Uf = u_exact(Xf(r, f), Yf(r, f), Zf(r, f));
      double v = 0;
      for (int i = 0; i < d2; ++i) v += D(r, i) * uhat[size_t(f) * d2 + i];
      sU += tri.weights[r] * Uf * Uf;
      sD += tri.weights[r] * (Uf - v) * (Uf - v);
    }
    const double a2 = em.area[f] * em.area[f];
    nhat2 += sU * a2;
    ehat2 += sD * a2;
  }
  rep.e_uhat = rel(ehat2, nhat2);
  double taumax = 0;
  for (double t : tau.tau.a) taumax = std::max(taumax, std::fabs(t));
  Mat proj_u = taumax == 0.0 ? l2_project_volume(em, tb, tet, u_exact)
                             : hdg_project(em, ms, tb, tet, tri, tau, q_exact, u_exact, nthreads).u;
  double du = 0;
  for (int K = 0; K < nelt; ++K) {
    double s = 0;
    for (int i = 0; i < tb.d3; ++i) {
      const double d = proj_u(i, K) - fields.u(i, K);
      s += d * d;
    }
    du += s * 6.0 * em.volume[K];
  }
  rep.eps_u = rel(du, nu2);
  const Mat Pu = l2_project_skeleton(em, k, tri, u_exact);
  double dh = 0;
  for (int f = 0; f < em.n_faces(); ++f) {
    double s = 0;
    for (int i = 0; i < d2; ++i) {
      const double d = Pu(i, f) - uhat[size_t(f) * d2 + i];
      s += d * d;
    }
    dh += 2.0 * s * em.area[f] * em.area[f];
  }
  rep.eps_uhat = rel(dh, nhat2);
  if (ustar && ustar->a.size() > 0) {
    const BasisTables tb1 = build_tables(k + 1, tet, tri);
    rep.e_star = rel(vol_err(tb1.P, ustar, U), nu2);
  }
  return rep;
}

}  // namespace hdgo
