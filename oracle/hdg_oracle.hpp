// =============================================================================
// TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle") of the reference HDG
// element-local path (arXiv 1305.1489, /root/reference/proj). It exists so the
// tests, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg can CHECK
// the CUDA product against the reference algorithm. The product
// (paper_1305_1489_b200/) never links, imports or calls anything here.
//
// Parity pinning: the reference cannot be compiled in this image (Eigen3, the
// doctest/CLI11 `vendor/` headers are absent — see DESIGN.md §Oracle), so this
// restatement is pinned against the reference's own known-answer tests and the
// README golden errors (tests/test_oracle_kats.py), not against reference
// binaries.
//
// Every function cites the reference file:line it restates. Storage follows the
// reference: column-major dense matrices (Eigen default), `Batch3` slices
// contiguous (proj/include/hdg/batch.hpp:14-38), 0-based indices.
// =============================================================================
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace hdgo {

// ---------------------------------------------------------------- dense types
struct Mat {  // column-major, like Eigen::MatrixXd
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rr, int cc, double v = 0.0) : r(rr), c(cc), a(size_t(rr) * cc, v) {}
  double& operator()(int i, int j) { return a[size_t(i) + size_t(j) * r]; }
  double operator()(int i, int j) const { return a[size_t(i) + size_t(j) * r]; }
  double* col(int j) { return a.data() + size_t(j) * r; }
  const double* col(int j) const { return a.data() + size_t(j) * r; }
};
struct IMat {
  int r = 0, c = 0;
  std::vector<int> a;
  IMat() = default;
  IMat(int rr, int cc, int v = 0) : r(rr), c(cc), a(size_t(rr) * cc, v) {}
  int& operator()(int i, int j) { return a[size_t(i) + size_t(j) * r]; }
  int operator()(int i, int j) const { return a[size_t(i) + size_t(j) * r]; }
};

// batch.hpp:14-38 — rows x cols x count, slice K contiguous, column-major.
struct Batch3 {
  int rows = 0, cols = 0, count = 0;
  std::vector<double> data;
  Batch3() = default;
  Batch3(int r, int c, int n) : rows(r), cols(c), count(n), data(size_t(r) * c * n, 0.0) {}
  double* slice(int K) { return data.data() + size_t(rows) * cols * K; }
  const double* slice(int K) const { return data.data() + size_t(rows) * cols * K; }
};

// batch.hpp:42-58 — deterministic contiguous-chunk thread loop.
void parallel_for(int n, int nthreads, const std::function<void(int, int)>& fn);

// ------------------------------------------------------------------- fields
// coefficient.hpp:13 — a scalar field evaluated at physical points.
using ScalarField = std::function<double(double, double, double)>;
struct VectorField { ScalarField x, y, z; };

// Field "programs": postfix expressions over (x,y,z) — the same encoding the
// product's C ABI accepts (include/hdg_b200.h, HDG_OP_*).
ScalarField program_field(const int* ops, int nops, const double* consts, int nconst);
ScalarField constant_field(double v);

// --------------------------------------------------------------------- mesh
enum FaceType : uint8_t { Interior = 0, Dirichlet = 1, Neumann = 2 };

// mesh.hpp:38-44
constexpr int kLocalFace[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {3, 1, 2}};
constexpr double kFaceNormalSign[4] = {-1.0, 1.0, -1.0, 1.0};
constexpr int kVertexImage[6][3] = {{0, 1, 2}, {0, 2, 1}, {2, 0, 1},
                                    {2, 1, 0}, {1, 2, 0}, {1, 0, 2}};

struct RawMesh {  // mesh.hpp:24-32
  Mat coordinates;  // Nver x 3
  IMat elements;    // Nelt x 4
  IMat dirichlet;   // Ndir x 3
  IMat neumann;     // Nneu x 3
  int n_vertices() const { return coordinates.r; }
  int n_elements() const { return elements.r; }
};

struct ExpandedMesh {  // mesh.hpp:46-67
  RawMesh raw;
  IMat faces;  // Nfc x 3
  std::vector<uint8_t> facetype;
  std::vector<int> dirfaces, neufaces;
  IMat facebyele;  // Nelt x 4
  IMat perm;       // Nelt x 4, 1..6
  std::vector<double> volume, area;
  Mat normals;  // Nelt x 12
  int n_elements() const { return raw.n_elements(); }
  int n_faces() const { return faces.r; }
  int n_dirichlet() const { return int(dirfaces.size()); }
  int n_neumann() const { return int(neufaces.size()); }
};

struct ElementGeometry {  // mesh.hpp:69-73
  double B[9];  // column-major 3x3
  double detB;
  double a[9];  // a(r,c) at 3r+c (row-major, as piola_coefficients column order)
};

struct MeshError : std::runtime_error { using std::runtime_error::runtime_error; };

ElementGeometry geometry(const RawMesh& raw, int K);
ExpandedMesh expand(const RawMesh& raw);
using FaceClassifier = std::function<FaceType(const double* centroid, const double* nu)>;
struct BoxBounds { double x0 = 0, x1 = 1, y0 = 0, y1 = 1, z0 = 0, z1 = 1; };
RawMesh box_mesh(int nx, int ny, int nz, const BoxBounds& b, const FaceClassifier& bc);
FaceClassifier all_dirichlet();
FaceClassifier dirichlet_top_bottom();
FaceClassifier dirichlet_x();  // C2/C5 classifier: Dirichlet iff |nu_x| > 0.5

// --------------------------------------------------------------- quadrature
struct TetRule { Mat barycentric; std::vector<double> weights; int exactness = 0;
                 int size() const { return int(weights.size()); } };
struct TriRule { Mat barycentric; std::vector<double> weights; int exactness = 0;
                 int size() const { return int(weights.size()); } };
void gauss_jacobi01(int n, int alpha, std::vector<double>& x, std::vector<double>& w);
TetRule tet_rule(int degree);
TriRule tri_rule(int degree);
std::array<Mat, 4> boundary_points(const TriRule& tri);

// -------------------------------------------------------------------- basis
inline int dim3(int k) { return (k + 1) * (k + 2) * (k + 3) / 6; }
inline int dim2(int k) { return (k + 1) * (k + 2) / 2; }
Mat eval_dubiner3d(int k, const Mat& pts);
void eval_dubiner3d_grad(int k, const Mat& pts, Mat& Px, Mat& Py, Mat& Pz);
Mat eval_dubiner2d(int k, const Mat& pts);
struct BasisTables {  // basis.hpp:32-39
  int k = 0, d3 = 0, d2 = 0;
  Mat P, Px, Py, Pz;
  std::array<Mat, 4> Pface;
  Mat D;
  std::array<Mat, 6> Dperm;
};
BasisTables build_tables(int k, const TetRule& tet, const TriRule& tri);

// ---------------------------------------------------------- element matrices
struct StabilizationField {  // element_matrices.hpp:22-30
  Mat tau;  // Nelt x 4
  bool allow_zero = false;
  static StabilizationField constant(const ExpandedMesh& em, double v);
  Mat scaled(const ExpandedMesh& em) const;
  void validate() const;
};
Mat piola_coefficients(const ExpandedMesh& em);
Mat normal_weights(const ExpandedMesh& em, int star);
struct PhysicalPoints { Mat X, Y, Z; };
PhysicalPoints quad_points_physical(const ExpandedMesh& em, const TetRule& rule);
PhysicalPoints face_points_physical(const ExpandedMesh& em, const TriRule& tri, int l);
Mat sample(const ScalarField& f, const PhysicalPoints& pp);
Mat source_vectors(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule,
                   const ScalarField& f);
Batch3 mass_matrices(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule,
                     const ScalarField& m);
void convection_matrices(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule,
                         Batch3& Cx, Batch3& Cy, Batch3& Cz);
void variable_convection_matrices(const ExpandedMesh& em, const BasisTables& tb,
                                  const TetRule& rule, const ScalarField& m, Batch3& Cx,
                                  Batch3& Cy, Batch3& Cz);
Batch3 type_a(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri, const Mat& xi);
Batch3 type_b(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri, const Mat& xi);
Batch3 type_c(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri, const Mat& xi);
Batch3 variable_surface_dp(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri,
                           const ScalarField& alpha, const Mat& xi);
Batch3 variable_surface_dd(const ExpandedMesh& em, const BasisTables& tb, const TriRule& tri,
                           const ScalarField& alpha, const Mat& xi);
Batch3 stiffness_matrices(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule);

struct ElementMatrixSet {  // element_matrices.hpp:86-93
  int k = 0, d3 = 0, d2 = 0;
  Batch3 Mkinv, Mc, Cx, Cy, Cz, tauPP, tauDP, nxDP, nyDP, nzDP, tauDD;
  Mat fvec;
};
ElementMatrixSet build_element_matrices(const ExpandedMesh& em, const BasisTables& tb,
                                        const TetRule& tet, const TriRule& tri,
                                        const ScalarField& kappa, const ScalarField& c,
                                        const ScalarField& f, const StabilizationField& tau);

struct ConvectionBilinearSet { Batch3 vol, dp, dd; };  // convdiff.hpp:13-17
ConvectionBilinearSet convection_bilinear_matrices(const ExpandedMesh& em, const BasisTables& tb,
                                                   const TetRule& tet, const TriRule& tri,
                                                   const VectorField& beta);

// -------------------------------------------------------------- local solver
struct LocalBlocks {  // local_solver.hpp:22-31
  int d3 = 0, d2 = 0, nu = 0, n = 0;
  Batch3 A1, A2, A3;
  Mat Af;
  Batch3 tauDD;
};
LocalBlocks local_blocks(const ElementMatrixSet& ms);
LocalBlocks bdm_blocks(const ElementMatrixSet& ms);
struct CondensedSystem { Batch3 C; Mat Cf; };
struct LocalSolverError : std::runtime_error {
  int element;
  LocalSolverError(int K, const std::string& w) : std::runtime_error(w), element(K) {}
};
CondensedSystem condense(const LocalBlocks& lb, int nthreads = 1);
struct LocalSolution { Mat qx, qy, qz, u; };
LocalSolution local_recover(const LocalBlocks& lb, const Mat& uhat, int nthreads = 1);

// Eigen-style PartialPivLU (max |a| in the column, first index on ties).
struct PartialPivLU {
  int n = 0;
  std::vector<double> lu;   // column-major n x n
  std::vector<int> perm;    // row permutation applied
  void compute(const double* A, int n);
  void solve(double* B, int ncols) const;  // in place, column-major n x ncols
  double min_abs_diag() const;
  double max_abs_diag() const;
};

// ------------------------------------------------------------ global system
struct SkeletonSystem {  // global_system.hpp:25-29 (CSC like Eigen's ColMajor)
  int64_t ndof = 0;
  std::vector<int64_t> colptr;
  std::vector<int> rowidx;
  std::vector<double> vals;
  std::vector<double> b;
  int d2 = 0;
};
SkeletonSystem assemble(const ExpandedMesh& em, const CondensedSystem& cs);
void face_quad_points(const ExpandedMesh& em, const std::vector<int>& faces, const TriRule& tri,
                      Mat& X, Mat& Y, Mat& Z);
std::vector<double> dirichlet_project(const ExpandedMesh& em, int k, const TriRule& tri,
                                      const ScalarField& g);
std::vector<double> neumann_load(const ExpandedMesh& em, int k, const TriRule& tri,
                                 const VectorField& g);
Mat gather_traces(const ExpandedMesh& em, int d2, const double* uhat);

// ---------------------------------------------------------------- postprocess
Mat postprocess_star(const ExpandedMesh& em, const BasisTables& tb1, const TetRule& rule,
                     const ScalarField& kappa, const LocalSolution& ls, int nthreads = 1);
Mat l2_project_volume(const ExpandedMesh& em, const BasisTables& tb, const TetRule& rule,
                      const ScalarField& f);
Mat l2_project_skeleton(const ExpandedMesh& em, int k, const TriRule& tri, const ScalarField& f);
LocalSolution hdg_project(const ExpandedMesh& em, const ElementMatrixSet& ms,
                          const BasisTables& tb, const TetRule& tet, const TriRule& tri,
                          const StabilizationField& tau, const VectorField& q,
                          const ScalarField& u, int nthreads = 1);
struct ErrorReport { double e_q = 0, e_u = 0, e_uhat = 0, eps_u = 0, eps_uhat = 0, e_star = 0; };
ErrorReport compute_errors(const ExpandedMesh& em, const ElementMatrixSet& ms,
                           const StabilizationField& tau, const ScalarField& u_exact,
                           const VectorField& q_exact, int k, const double* uhat,
                           const LocalSolution& fields, const Mat* ustar, int nthreads = 1);

}  // namespace hdgo
