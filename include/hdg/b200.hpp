// hdg/b200.hpp — reference-shaped C++ host API over the C ABI (hdg_b200.h).
//
// What a caller of the reference library (/root/reference/proj, namespace
// hdg) uses on the element-local path, with the same call shapes, value types
// and exceptions, but running on the B200 engine:
//
//   reference (Eigen, CPU)                       here
//   --------------------------------------------------------------------------
//   ScalarField (coefficient.hpp:13-14)          ScalarField: callback over
//     callbacks over point arrays                  point arrays, sampled at the
//                                                  device's physical nodes
//   build_element_matrices -> local_blocks       condense(level, kappa, c, f)
//     -> condense (element_matrices.hpp:95-99,     -> CondensedSystem {C, Cf}
//     local_solver.hpp:33, :51)
//   gather_traces + local_recover                local_recover(level, cs, uhat)
//     (global_system.hpp:55-56,                    -> LocalSolution {qx,qy,qz,u}
//     local_solver.hpp:58-59)
//   postprocess_star (postprocess.hpp:26-28)     postprocess_star(level, kappa, ls)
//   LocalSolverError{element}                    LocalSolverError{element}
//     (local_solver.hpp:45-49)
//   MeshError (mesh.hpp:75-78)                   MeshError
//   GlobalSolverError (global_system.hpp:44-46)  GlobalSolverError
//   std::invalid_argument (tau, BDM k < 1)       std::invalid_argument
//
// Storage keeps the reference layouts without Eigen: Matrix is column-major
// (Eigen::MatrixXd), Batch3 slice K is contiguous column-major
// (batch.hpp:14-38). Results are host copies (as the reference returns owning
// Eigen values); the recovery cache stays in device memory inside
// CondensedSystem. Header-only; link libhdg_b200.so and cudart.
#ifndef HDG_B200_HPP
#define HDG_B200_HPP

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../hdg_b200.h"

namespace hdg {
namespace b200 {

// ------------------------------------------------------------ value types
struct Matrix {  // column-major, Eigen::MatrixXd layout
  int rows = 0, cols = 0;
  std::vector<double> a;
  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), a(size_t(r) * c, 0.0) {}
  double& operator()(int i, int j) { return a[size_t(i) + size_t(j) * rows]; }
  double operator()(int i, int j) const { return a[size_t(i) + size_t(j) * rows]; }
  double* col(int j) { return a.data() + size_t(j) * rows; }
};

struct Batch3 {  // batch.hpp:14-38: rows x cols x count, slice K contiguous
  int rows = 0, cols = 0, count = 0;
  std::vector<double> data;
  Batch3() = default;
  Batch3(int r, int c, int n) : rows(r), cols(c), count(n), data(size_t(r) * c * n, 0.0) {}
  double* slice(int K) { return data.data() + size_t(rows) * cols * K; }
  const double* slice(int K) const { return data.data() + size_t(rows) * cols * K; }
  double operator()(int K, int i, int j) const { return slice(K)[size_t(i) + size_t(j) * rows]; }
};

// coefficient.hpp:13-14: evaluates a field at n points (the reference passes
// Eigen arrays of the quadrature-node coordinates and returns their shape).
using ScalarField = std::function<void(const double* X, const double* Y, const double* Z, double* out, size_t n)>;

inline ScalarField constant_field(double v) {
  return [v](const double*, const double*, const double*, double* out, size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = v;
  };
}
inline ScalarField pointwise_field(std::function<double(double, double, double)> f) {
  return [f = std::move(f)](const double* X, const double* Y, const double* Z, double* out, size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = f(X[i], Y[i], Z[i]);
  };
}

// -------------------------------------------------------------- exceptions
struct LocalSolverError : std::runtime_error {  // local_solver.hpp:45-49
  int element;
  LocalSolverError(int K, const std::string& what) : std::runtime_error(what), element(K) {}
};
struct MeshError : std::runtime_error { using std::runtime_error::runtime_error; };
struct GlobalSolverError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

// Rethrows an HDG_E* status as the reference's exception type.
inline void check(int status, int64_t bad_element = -1) {
  if (status == HDG_OK) return;
  const std::string msg = hdg_b200_last_error();
  switch (status) {
    case HDG_ESINGULAR: throw LocalSolverError(int(bad_element), msg);
    case HDG_EMESH: throw MeshError(msg);
    case HDG_ESOLVE: throw GlobalSolverError(msg);
    case HDG_EINVAL: throw std::invalid_argument(msg);
    default: throw DeviceError(msg);
  }
}
inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------- device buffers
template <class T>
class DeviceArray {
 public:
  DeviceArray() = default;
  explicit DeviceArray(size_t n) : n_(n) { cuda_check(cudaMalloc(&p_, (n ? n : 1) * sizeof(T)), "cudaMalloc"); }
  DeviceArray(const T* host, size_t n) : DeviceArray(n) { upload(host); }
  ~DeviceArray() { if (p_) cudaFree(p_); }
  DeviceArray(DeviceArray&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceArray& operator=(DeviceArray&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  DeviceArray(const DeviceArray&) = delete;
  DeviceArray& operator=(const DeviceArray&) = delete;
  T* get() const { return p_; }
  size_t size() const { return n_; }
  void upload(const T* host) { cuda_check(cudaMemcpy(p_, host, n_ * sizeof(T), cudaMemcpyHostToDevice), "H2D"); }
  void download(T* host) const { cuda_check(cudaMemcpy(host, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "D2H"); }
  std::vector<T> to_host() const {
    std::vector<T> v(n_);
    download(v.data());
    return v;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// ------------------------------------------------------------------ level
// One discretisation level on one device: the expanded mesh (box_mesh +
// expand, mesh.cpp:74-253, numbering bit-exact), the degree-k tables
// (study.cpp:13-15), and the per-element geometry with tau
// (StabilizationField, element_matrices.hpp:22-30). The mesh is generated and
// expanded by the engine's host layer, then uploaded.
class Level {
 public:
  // box_mesh(nx, ny, nz) with a boundary rule (HDG_BC_*), tau constant on every face.
  Level(int device, int k, int nx, int ny, int nz, int bc_rule, double tau, double perturb = 0.0,
        uint64_t seed = 1305)
      : device_(device), k_(k) {
    check(hdg_b200_create(device, nullptr, &ctx_));
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    check(hdg_b200_set_degree(ctx_, k, 2 * k + 2, 2 * k + 2));
    hdg_mesh* m = nullptr;
    check(hdg_b200_mesh_box(nx, ny, nz, bc_rule, perturb, seed, 0.5, &m));
    upload_mesh(m);
    hdg_b200_mesh_free(m);
    set_tau(tau);
  }
  ~Level() { if (ctx_) hdg_b200_destroy(ctx_); }
  Level(const Level&) = delete;
  Level& operator=(const Level&) = delete;

  hdg_ctx* ctx() const { return ctx_; }
  int k() const { return k_; }
  int nelt() const { return nelt_; }
  int nfc() const { return nfc_; }
  int d3() const { return (k_ + 1) * (k_ + 2) * (k_ + 3) / 6; }
  int d2() const { return (k_ + 1) * (k_ + 2) / 2; }
  const hdg_geometry& geometry() const { return geo_; }
  const int* facebyele() const { return facebyele_.get(); }
  const std::vector<int>& host_facebyele() const { return h_facebyele_; }

  // StabilizationField::constant (element_matrices.cpp:25-29) or per face
  // (Nelt x 4 column-major, the reference's tau matrix); recomputes geometry.
  void set_tau(double tau) { geometry_with(nullptr, tau); }
  void set_tau(const Matrix& tau) {
    if (tau.rows != nelt_ || tau.cols != 4) throw std::invalid_argument("tau must be Nelt x 4");
    DeviceArray<double> d(tau.a.data(), tau.a.size());
    geometry_with(d.get(), 0.0);
  }

  // The caller's callback sampled at the device's physical nodes (which = 0:
  // degree-k rule, 1: postprocess rule): device array, nq x nelt.
  DeviceArray<double> sample(const ScalarField& f, int which = 0) {
    int64_t dims[8];
    check(hdg_b200_dims(ctx_, dims));
    const size_t nq = size_t(which == 0 ? dims[3] : dims[6]);
    const size_t n = nq * size_t(nelt_);
    DeviceArray<double> X(n), Y(n), Z(n), out(n);
    check(hdg_b200_quad_points(ctx_, nelt_, &geo_, which, X.get(), Y.get(), Z.get()));
    check(hdg_b200_synchronize(ctx_));
    const std::vector<double> hx = X.to_host(), hy = Y.to_host(), hz = Z.to_host();
    std::vector<double> v(n);
    f(hx.data(), hy.data(), hz.data(), v.data(), n);
    out.upload(v.data());
    return out;
  }

 private:
  void upload_mesh(hdg_mesh* m) {
    check(hdg_b200_mesh_expand(m));
    int64_t d[6];
    check(hdg_b200_mesh_dims(m, d));
    nver_ = int(d[0]);
    nelt_ = int(d[1]);
    nfc_ = int(d[2]);
    std::vector<double> coords(size_t(nver_) * 3);
    std::vector<int> el(size_t(nelt_) * 4), faces(size_t(nfc_) * 3);
    h_facebyele_.resize(size_t(nelt_) * 4);
    check(hdg_b200_mesh_copy(m, HDG_MESH_COORDS, coords.data()));
    check(hdg_b200_mesh_copy(m, HDG_MESH_ELEMENTS, el.data()));
    check(hdg_b200_mesh_copy(m, HDG_MESH_FACES, faces.data()));
    check(hdg_b200_mesh_copy(m, HDG_MESH_FACEBYELE, h_facebyele_.data()));
    coords_ = DeviceArray<double>(coords.data(), coords.size());
    elements_ = DeviceArray<int>(el.data(), el.size());
    faces_ = DeviceArray<int>(faces.data(), faces.size());
    facebyele_ = DeviceArray<int>(h_facebyele_.data(), h_facebyele_.size());
    const size_t n = size_t(nelt_);
    volume_ = DeviceArray<double>(n);
    piola_ = DeviceArray<double>(9 * n);
    normals_ = DeviceArray<double>(12 * n);
    perm_ = DeviceArray<int>(4 * n);
    T_ = DeviceArray<double>(4 * n);
    verts_ = DeviceArray<double>(12 * n);
    area_ = DeviceArray<double>(size_t(nfc_));
    geo_ = hdg_geometry{volume_.get(), piola_.get(), normals_.get(), perm_.get(), T_.get(), verts_.get(),
                        area_.get()};
  }
  void geometry_with(const double* d_tau, double tau) {
    check(hdg_b200_geometry(ctx_, nver_, nelt_, nfc_, coords_.get(), elements_.get(), faces_.get(),
                            facebyele_.get(), d_tau, tau, &geo_));
    check(hdg_b200_synchronize(ctx_));  // MeshError for a non-positive orientation
  }

  int device_ = 0, k_ = 0, nver_ = 0, nelt_ = 0, nfc_ = 0;
  hdg_ctx* ctx_ = nullptr;
  DeviceArray<double> coords_, volume_, piola_, normals_, T_, verts_, area_;
  DeviceArray<int> elements_, faces_, facebyele_, perm_;
  std::vector<int> h_facebyele_;
  hdg_geometry geo_{};
};

// ----------------------------------------------------- local solver (K2-K6)
struct CondensedSystem {  // local_solver.hpp:39-42
  Batch3 C;                       // 4 d2 x 4 d2 per element
  Matrix Cf;                      // 4 d2 x Nelt
  DeviceArray<double> d_C, d_Cf;  // device copies (scatter input)
  DeviceArray<double> factors;    // device recovery cache (local_recover)
};

struct LocalSolution {  // local_solver.hpp:53-55
  Matrix qx, qy, qz, u;  // d3 x Nelt
  DeviceArray<double> d_qx, d_qy, d_qz, d_u;
};

inline hdg_field sampled(const DeviceArray<double>& s) {
  hdg_field f{};
  f.kind = HDG_FIELD_SAMPLED;
  f.samples = s.get();
  return f;
}

// build_element_matrices -> local_blocks -> condense (element_matrices.cpp:
// 282-309, local_solver.cpp:12-100): one fused device call. Throws
// std::invalid_argument for an invalid tau (element_matrices.cpp:38-46) and
// LocalSolverError{lowest element} for a singular element (:50-57).
inline CondensedSystem condense(Level& lv, const ScalarField& kappa, const ScalarField& c, const ScalarField& f) {
  const int n = lv.nelt(), m = 4 * lv.d2();
  int64_t dims[8];
  check(hdg_b200_dims(lv.ctx(), dims));
  DeviceArray<double> sk = lv.sample(kappa), sc = lv.sample(c), sf = lv.sample(f);
  CondensedSystem cs;
  cs.d_C = DeviceArray<double>(size_t(n) * m * m);
  cs.d_Cf = DeviceArray<double>(size_t(n) * m);
  cs.factors = DeviceArray<double>(size_t(n) * size_t(dims[5]));
  int64_t bad = -1;
  const hdg_geometry g = lv.geometry();
  const int st = hdg_b200_build_condense(lv.ctx(), n, &g, sampled(sk), sampled(sc), sampled(sf), cs.d_C.get(),
                                         cs.d_Cf.get(), cs.factors.get(), nullptr, &bad);
  check(st, bad);  // (bad is set by the call: not an argument of the same expression)
  cs.C = Batch3(m, m, n);
  cs.Cf = Matrix(m, n);
  cs.d_C.download(cs.C.data.data());
  cs.d_Cf.download(cs.Cf.a.data());
  return cs;
}

// gather_traces + local_recover (global_system.cpp:167-175,
// local_solver.cpp:102-135): uhat is the skeleton vector (dof = f d2 + i).
inline LocalSolution local_recover(Level& lv, const CondensedSystem& cs, const std::vector<double>& uhat) {
  const int n = lv.nelt(), d3 = lv.d3();
  if (uhat.size() != size_t(lv.nfc()) * lv.d2()) throw std::invalid_argument("uhat must hold Nfc * d2 entries");
  DeviceArray<double> du(uhat.data(), uhat.size());
  LocalSolution ls;
  ls.d_qx = DeviceArray<double>(size_t(n) * d3);
  ls.d_qy = DeviceArray<double>(size_t(n) * d3);
  ls.d_qz = DeviceArray<double>(size_t(n) * d3);
  ls.d_u = DeviceArray<double>(size_t(n) * d3);
  const hdg_geometry g = lv.geometry();
  check(hdg_b200_recover(lv.ctx(), n, &g, lv.facebyele(), cs.factors.get(), du.get(), ls.d_qx.get(),
                         ls.d_qy.get(), ls.d_qz.get(), ls.d_u.get()));
  check(hdg_b200_synchronize(lv.ctx()));
  for (auto [h, d] : {std::pair<Matrix*, const DeviceArray<double>*>{&ls.qx, &ls.d_qx}, {&ls.qy, &ls.d_qy},
                      {&ls.qz, &ls.d_qz}, {&ls.u, &ls.d_u}}) {
    *h = Matrix(d3, n);
    d->download(h->a.data());
  }
  return ls;
}

// postprocess_star (postprocess.cpp:33-74) on tet_rule(2(k+1)+2) (study.cpp:33-34):
// u* of degree k+1, d3(k+1) x Nelt.
inline Matrix postprocess_star(Level& lv, const ScalarField& kappa, const LocalSolution& ls) {
  check(hdg_b200_set_postprocess_rule(lv.ctx(), 2 * (lv.k() + 1) + 2));
  int64_t dims[8];
  check(hdg_b200_dims(lv.ctx(), dims));
  const int n = lv.nelt(), d3p = int(dims[7]);
  DeviceArray<double> sk = lv.sample(kappa, 1), us(size_t(n) * d3p);
  const hdg_geometry g = lv.geometry();
  check(hdg_b200_postprocess(lv.ctx(), n, &g, sampled(sk), ls.d_qx.get(), ls.d_qy.get(), ls.d_qz.get(),
                             ls.d_u.get(), us.get()));
  check(hdg_b200_synchronize(lv.ctx()));
  Matrix out(d3p, n);
  us.download(out.a.data());
  return out;
}

}  // namespace b200
}  // namespace hdg

#endif  // HDG_B200_HPP
