// Internal host-side types of the B200 engine (setup layer, not timed).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace hdgb {

constexpr int kMaxDegree = 6;  // kernels are instantiated for k = 0..6

inline int pdim3(int k) { return (k + 1) * (k + 2) * (k + 3) / 6; }
inline int pdim2(int k) { return (k + 1) * (k + 2) / 2; }

struct MeshError : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- tables
struct HostTables {
  int k = 0, d3 = 0, d2 = 0, nq = 0, nqd = 0;
  std::vector<double> tet_bary, tet_w;  // nq x 4 (col-major), nq
  std::vector<double> tri_bary, tri_w;  // nqd x 3, nqd
  std::vector<double> P;                // nq x d3
  std::array<std::vector<double>, 3> Pd;
  std::array<std::vector<double>, 4> Pface;  // nqd x d3
  std::vector<double> D;                     // nqd x d2
  std::array<std::vector<double>, 6> Dperm;  // nqd x d2
  std::array<std::vector<double>, 3> Chat;   // d3 x d3
  std::array<std::vector<double>, 9> Shat;   // d3 x d3 (3*#+#')
  std::array<std::vector<double>, 4> PP;     // d3 x d3
  std::array<std::vector<double>, 24> Wlm;   // d2 x d3, index 6*l + (mu-1)
  std::vector<double> DD;                    // d2 x d2
};

void gauss_jacobi01(int n, int alpha, std::vector<double>& x, std::vector<double>& w);
void tet_rule(int degree, std::vector<double>& bary, std::vector<double>& w);
void tri_rule(int degree, std::vector<double>& bary, std::vector<double>& w);
void dubiner3d(int k, int npts, const double* x, const double* y, const double* z, double* P,
               double* Px, double* Py, double* Pz);
void dubiner2d(int k, int npts, const double* s, const double* t, double* D);
HostTables build_host_tables(int k, int tet_deg, int tri_deg);

// ------------------------------------------------------------------ mesh
enum FaceType : uint8_t { kInterior = 0, kDirichlet = 1, kNeumann = 2 };
enum BoundaryRule : int { kAllDirichlet = 0, kDirichletTopBottom = 1, kDirichletX = 2 };

// mesh.hpp:38-44
constexpr int kLocalFace[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {3, 1, 2}};
constexpr double kFaceNormalSign[4] = {-1.0, 1.0, -1.0, 1.0};
constexpr int kVertexImage[6][3] = {{0, 1, 2}, {0, 2, 1}, {2, 0, 1},
                                    {2, 1, 0}, {1, 2, 0}, {1, 0, 2}};

struct HostMesh {
  int nver = 0, nelt = 0, nfc = 0, ndir = 0, nneu = 0;
  std::vector<double> coords;      // nver x 3 (col-major)
  std::vector<int> elements;       // nelt x 4
  std::vector<int> dirichlet;      // ndir x 3
  std::vector<int> neumann;        // nneu x 3
  std::vector<int> faces;          // nfc x 3 (intrinsic parametrisation)
  std::vector<uint8_t> facetype;   // nfc
  std::vector<int> facebyele;      // nelt x 4
  bool expanded = false;
};

void box_mesh(int nx, int ny, int nz, BoundaryRule bc, HostMesh& m);
void perturb_interior(HostMesh& m, int nx, int ny, int nz, double frac, uint64_t seed,
                      double keep_plane_z);
void expand_mesh(HostMesh& m);

// Skeleton sparsity: per face the sorted neighbour faces (faces sharing an
// element with it, itself included) and per element the slot of each
// (l1, l2) face pair inside row-face l1's neighbour list.
struct SkeletonPattern {
  int nfc = 0, maxnbr = 0;
  std::vector<int> nnbr;        // nfc
  std::vector<int> nbr;         // nfc x 8 (padded with -1)
  std::vector<int64_t> facebase;  // nfc + 1 : first CSR value of each face's rows / d2^2
  std::vector<uint8_t> slot;    // nelt x 16
};
void build_pattern(const HostMesh& m, SkeletonPattern& p);
void build_pattern_raw(int nelt, int nfc, const int* facebyele, SkeletonPattern& p);

}  // namespace hdgb
