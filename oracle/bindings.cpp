// TEST INFRASTRUCTURE ONLY — pybind11 bindings exposing the CPU oracle to the
// pytest suite, smoke() and bench.py's cpu_baseline leg. Arrays come back as
// numpy copies in the reference's layout: dense matrices F-ordered (Eigen
// column-major), Batch3 as (count, rows, cols) with each slice F-ordered.
#include <pybind11/functional.h>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <atomic>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstring>
#include <random>
#include <tuple>

#include "hdg_oracle.hpp"

namespace py = pybind11;
using namespace hdgo;

namespace {

using DArr = py::array_t<double, py::array::f_style | py::array::forcecast>;
using IArr = py::array_t<int, py::array::f_style | py::array::forcecast>;

py::array_t<double> np_mat(const Mat& m) {
  py::array_t<double> out({m.r, m.c}, {sizeof(double), sizeof(double) * m.r});
  std::memcpy(out.mutable_data(), m.a.data(), m.a.size() * sizeof(double));
  return out;
}
py::array_t<int> np_imat(const IMat& m) {
  py::array_t<int> out({m.r, m.c}, {sizeof(int), sizeof(int) * m.r});
  std::memcpy(out.mutable_data(), m.a.data(), m.a.size() * sizeof(int));
  return out;
}
py::array_t<double> np_batch(const Batch3& b) {
  py::array_t<double> out({b.count, b.rows, b.cols},
                          {sizeof(double) * b.rows * b.cols, sizeof(double),
                           sizeof(double) * b.rows});
  std::memcpy(out.mutable_data(), b.data.data(), b.data.size() * sizeof(double));
  return out;
}
template <class T>
py::array_t<T> np_vec(const std::vector<T>& v) {
  py::array_t<T> out(v.size());
  std::memcpy(out.mutable_data(), v.data(), v.size() * sizeof(T));
  return out;
}
Mat mat_from(const DArr& a) {
  if (a.ndim() != 2) throw std::invalid_argument("expected a 2-D array");
  Mat m(int(a.shape(0)), int(a.shape(1)));
  std::memcpy(m.a.data(), a.data(), m.a.size() * sizeof(double));
  return m;
}
IMat imat_from(const IArr& a) {
  if (a.ndim() != 2) throw std::invalid_argument("expected a 2-D int array");
  IMat m(int(a.shape(0)), int(a.shape(1)));
  std::memcpy(m.a.data(), a.data(), m.a.size() * sizeof(int));
  return m;
}

struct Field { ScalarField f; };
struct VField { VectorField f; };
struct Tables {
  TetRule tet;
  TriRule tri;
  BasisTables tb;
};

FaceClassifier classifier(const std::string& name) {
  if (name == "all_dirichlet") return all_dirichlet();
  if (name == "dirichlet_top_bottom") return dirichlet_top_bottom();
  if (name == "dirichlet_x") return dirichlet_x();
  throw std::invalid_argument("unknown classifier " + name);
}

}  // namespace

PYBIND11_MODULE(_hdg_oracle, m) {
  m.doc() = "CPU oracle of the reference HDG element-local path (test infrastructure only)";

  py::register_exception<MeshError>(m, "MeshError", PyExc_RuntimeError);
  static py::exception<LocalSolverError> lse(m, "LocalSolverError", PyExc_RuntimeError);
  py::register_exception_translator([](std::exception_ptr p) {
    try {
      if (p) std::rethrow_exception(p);
    } catch (const LocalSolverError& e) {
      PyErr_SetObject(lse.ptr(), py::make_tuple(e.what(), e.element).ptr());
    }
  });

  py::class_<Field>(m, "Field")
      .def_static("constant", [](double v) { return Field{constant_field(v)}; })
      .def_static("program",
                  [](std::vector<int> ops, std::vector<double> consts) {
                    return Field{program_field(ops.data(), int(ops.size()), consts.data(),
                                               int(consts.size()))};
                  })
      .def_static("python", [](py::function fn) {
        return Field{[fn](double x, double y, double z) {
          py::gil_scoped_acquire g;
          return fn(x, y, z).cast<double>();
        }};
      })
      .def("__call__", [](const Field& f, double x, double y, double z) { return f.f(x, y, z); });
  py::class_<VField>(m, "VField").def(py::init([](const Field& x, const Field& y, const Field& z) {
    return VField{{x.f, y.f, z.f}};
  }));

  // ------------------------------------------------------------------ mesh
  py::class_<ExpandedMesh>(m, "ExpandedMesh")
      .def_property_readonly("coordinates", [](const ExpandedMesh& e) { return np_mat(e.raw.coordinates); })
      .def_property_readonly("elements", [](const ExpandedMesh& e) { return np_imat(e.raw.elements); })
      .def_property_readonly("dirichlet", [](const ExpandedMesh& e) { return np_imat(e.raw.dirichlet); })
      .def_property_readonly("neumann", [](const ExpandedMesh& e) { return np_imat(e.raw.neumann); })
      .def_property_readonly("faces", [](const ExpandedMesh& e) { return np_imat(e.faces); })
      .def_property_readonly("facetype", [](const ExpandedMesh& e) { return np_vec(e.facetype); })
      .def_property_readonly("dirfaces", [](const ExpandedMesh& e) { return np_vec(e.dirfaces); })
      .def_property_readonly("neufaces", [](const ExpandedMesh& e) { return np_vec(e.neufaces); })
      .def_property_readonly("facebyele", [](const ExpandedMesh& e) { return np_imat(e.facebyele); })
      .def_property_readonly("perm", [](const ExpandedMesh& e) { return np_imat(e.perm); })
      .def_property_readonly("volume", [](const ExpandedMesh& e) { return np_vec(e.volume); })
      .def_property_readonly("area", [](const ExpandedMesh& e) { return np_vec(e.area); })
      .def_property_readonly("normals", [](const ExpandedMesh& e) { return np_mat(e.normals); })
      .def_property_readonly("n_elements", &ExpandedMesh::n_elements)
      .def_property_readonly("n_faces", &ExpandedMesh::n_faces);

  m.def("box_mesh_raw",
        [](int nx, int ny, int nz, const std::string& bc, std::vector<double> bounds) {
          BoxBounds b;
          if (bounds.size() == 6) b = {bounds[0], bounds[1], bounds[2], bounds[3], bounds[4], bounds[5]};
          RawMesh r = box_mesh(nx, ny, nz, b, classifier(bc));
          return py::make_tuple(np_mat(r.coordinates), np_imat(r.elements), np_imat(r.dirichlet),
                                np_imat(r.neumann));
        },
        py::arg("nx"), py::arg("ny"), py::arg("nz"), py::arg("bc"),
        py::arg("bounds") = std::vector<double>{});
  m.def("expand", [](const DArr& coords, const IArr& elements, const IArr& dir, const IArr& neu) {
    RawMesh r;
    r.coordinates = mat_from(coords);
    r.elements = imat_from(elements);
    r.dirichlet = imat_from(dir);
    r.neumann = imat_from(neu);
    return expand(r);
  });
  m.def("geometry", [](const ExpandedMesh& em, int K) {
    const ElementGeometry g = geometry(em.raw, K);
    return py::make_tuple(np_vec(std::vector<double>(g.B, g.B + 9)), g.detB,
                          np_vec(std::vector<double>(g.a, g.a + 9)));
  });
  m.def("piola_coefficients", [](const ExpandedMesh& em) { return np_mat(piola_coefficients(em)); });

  // -------------------------------------------------------------- tables
  m.def("gauss_jacobi01", [](int n, int alpha) {
    std::vector<double> x, w;
    gauss_jacobi01(n, alpha, x, w);
    return py::make_tuple(np_vec(x), np_vec(w));
  });
  py::class_<Tables>(m, "Tables")
      .def_property_readonly("k", [](const Tables& t) { return t.tb.k; })
      .def_property_readonly("d3", [](const Tables& t) { return t.tb.d3; })
      .def_property_readonly("d2", [](const Tables& t) { return t.tb.d2; })
      .def_property_readonly("tet_bary", [](const Tables& t) { return np_mat(t.tet.barycentric); })
      .def_property_readonly("tet_w", [](const Tables& t) { return np_vec(t.tet.weights); })
      .def_property_readonly("tri_bary", [](const Tables& t) { return np_mat(t.tri.barycentric); })
      .def_property_readonly("tri_w", [](const Tables& t) { return np_vec(t.tri.weights); })
      .def_property_readonly("P", [](const Tables& t) { return np_mat(t.tb.P); })
      .def_property_readonly("Px", [](const Tables& t) { return np_mat(t.tb.Px); })
      .def_property_readonly("Py", [](const Tables& t) { return np_mat(t.tb.Py); })
      .def_property_readonly("Pz", [](const Tables& t) { return np_mat(t.tb.Pz); })
      .def_property_readonly("D", [](const Tables& t) { return np_mat(t.tb.D); })
      .def("Pface", [](const Tables& t, int l) { return np_mat(t.tb.Pface.at(l)); })
      .def("Dperm", [](const Tables& t, int mu) { return np_mat(t.tb.Dperm.at(mu)); });
  m.def("tables", [](int k, int tet_deg, int tri_deg) {
    Tables t{tet_rule(tet_deg), tri_rule(tri_deg), {}};
    t.tb = build_tables(k, t.tet, t.tri);
    return t;
  });
  m.def("eval_dubiner3d", [](int k, const DArr& pts) { return np_mat(eval_dubiner3d(k, mat_from(pts))); });
  m.def("eval_dubiner3d_grad", [](int k, const DArr& pts) {
    Mat a, b, c;
    eval_dubiner3d_grad(k, mat_from(pts), a, b, c);
    return py::make_tuple(np_mat(a), np_mat(b), np_mat(c));
  });
  m.def("eval_dubiner2d", [](int k, const DArr& pts) { return np_mat(eval_dubiner2d(k, mat_from(pts))); });

  // ----------------------------------------------------- element matrices
  py::class_<StabilizationField>(m, "Stabilization")
      .def(py::init([](const DArr& tau, bool allow_zero) {
             StabilizationField s;
             s.tau = mat_from(tau);
             s.allow_zero = allow_zero;
             return s;
           }),
           py::arg("tau"), py::arg("allow_zero") = false)
      .def("scaled", [](const StabilizationField& s, const ExpandedMesh& em) { return np_mat(s.scaled(em)); })
      .def("validate", &StabilizationField::validate);

  py::class_<ElementMatrixSet>(m, "ElementMatrixSet")
      .def("get", [](const ElementMatrixSet& s, const std::string& n) -> py::object {
        if (n == "fvec") return np_mat(s.fvec);
        const std::map<std::string, const Batch3*> tbl = {
            {"Mkinv", &s.Mkinv}, {"Mc", &s.Mc},       {"Cx", &s.Cx},       {"Cy", &s.Cy},
            {"Cz", &s.Cz},       {"tauPP", &s.tauPP}, {"tauDP", &s.tauDP}, {"nxDP", &s.nxDP},
            {"nyDP", &s.nyDP},   {"nzDP", &s.nzDP},   {"tauDD", &s.tauDD}};
        return np_batch(*tbl.at(n));
      });
  m.def("build_element_matrices",
        [](const ExpandedMesh& em, const Tables& t, const Field& kappa, const Field& c,
           const Field& f, const StabilizationField& tau) {
          py::gil_scoped_release r;
          return build_element_matrices(em, t.tb, t.tet, t.tri, kappa.f, c.f, f.f, tau);
        });
  m.def("mass_matrices", [](const ExpandedMesh& em, const Tables& t, const Field& f) {
    return np_batch(mass_matrices(em, t.tb, t.tet, f.f));
  });
  m.def("source_vectors", [](const ExpandedMesh& em, const Tables& t, const Field& f) {
    return np_mat(source_vectors(em, t.tb, t.tet, f.f));
  });
  m.def("convection_matrices", [](const ExpandedMesh& em, const Tables& t) {
    Batch3 a, b, c;
    convection_matrices(em, t.tb, t.tet, a, b, c);
    return py::make_tuple(np_batch(a), np_batch(b), np_batch(c));
  });
  m.def("variable_convection_matrices", [](const ExpandedMesh& em, const Tables& t, const Field& f) {
    Batch3 a, b, c;
    variable_convection_matrices(em, t.tb, t.tet, f.f, a, b, c);
    return py::make_tuple(np_batch(a), np_batch(b), np_batch(c));
  });
  m.def("type_a", [](const ExpandedMesh& em, const Tables& t, const DArr& xi) {
    return np_batch(type_a(em, t.tb, t.tri, mat_from(xi)));
  });
  m.def("type_b", [](const ExpandedMesh& em, const Tables& t, const DArr& xi) {
    return np_batch(type_b(em, t.tb, t.tri, mat_from(xi)));
  });
  m.def("type_c", [](const ExpandedMesh& em, const Tables& t, const DArr& xi) {
    return np_batch(type_c(em, t.tb, t.tri, mat_from(xi)));
  });
  m.def("variable_surface_dp", [](const ExpandedMesh& em, const Tables& t, const Field& a, const DArr& xi) {
    return np_batch(variable_surface_dp(em, t.tb, t.tri, a.f, mat_from(xi)));
  });
  m.def("variable_surface_dd", [](const ExpandedMesh& em, const Tables& t, const Field& a, const DArr& xi) {
    return np_batch(variable_surface_dd(em, t.tb, t.tri, a.f, mat_from(xi)));
  });
  m.def("stiffness_matrices", [](const ExpandedMesh& em, const Tables& t) {
    return np_batch(stiffness_matrices(em, t.tb, t.tet));
  });
  m.def("normal_weights", [](const ExpandedMesh& em, int s) { return np_mat(normal_weights(em, s)); });
  m.def("quad_points_physical", [](const ExpandedMesh& em, const Tables& t) {
    const PhysicalPoints p = quad_points_physical(em, t.tet);
    return py::make_tuple(np_mat(p.X), np_mat(p.Y), np_mat(p.Z));
  });
  m.def("face_points_physical", [](const ExpandedMesh& em, const Tables& t, int l) {
    const PhysicalPoints p = face_points_physical(em, t.tri, l);
    return py::make_tuple(np_mat(p.X), np_mat(p.Y), np_mat(p.Z));
  });
  m.def("convection_bilinear_matrices",
        [](const ExpandedMesh& em, const Tables& t, const VField& beta) {
          py::gil_scoped_release r;
          ConvectionBilinearSet s = convection_bilinear_matrices(em, t.tb, t.tet, t.tri, beta.f);
          py::gil_scoped_acquire g;
          return py::make_tuple(np_batch(s.vol), np_batch(s.dp), np_batch(s.dd));
        });

  // --------------------------------------------------------- local solver
  py::class_<LocalBlocks>(m, "LocalBlocks")
      .def_readonly("n", &LocalBlocks::n)
      .def_readonly("nu", &LocalBlocks::nu)
      .def_property_readonly("A1", [](const LocalBlocks& b) { return np_batch(b.A1); })
      .def_property_readonly("A2", [](const LocalBlocks& b) { return np_batch(b.A2); })
      .def_property_readonly("A3", [](const LocalBlocks& b) { return np_batch(b.A3); })
      .def_property_readonly("Af", [](const LocalBlocks& b) { return np_mat(b.Af); })
      .def_property_readonly("tauDD", [](const LocalBlocks& b) { return np_batch(b.tauDD); })
      .def("zero_A1_slice", [](LocalBlocks& b, int K) {
        std::fill(b.A1.slice(K), b.A1.slice(K) + size_t(b.n) * b.n, 0.0);
      });
  m.def("local_blocks", &local_blocks);
  m.def("bdm_blocks", &bdm_blocks);
  m.def("condense", [](const LocalBlocks& lb, int nthreads) {
    CondensedSystem cs;
    {
      py::gil_scoped_release r;
      cs = condense(lb, nthreads);
    }
    return py::make_tuple(np_batch(cs.C), np_mat(cs.Cf));
  }, py::arg("lb"), py::arg("nthreads") = 1);
  m.def("local_recover", [](const LocalBlocks& lb, const DArr& uhat, int nthreads) {
    const Mat U = mat_from(uhat);
    LocalSolution ls;
    {
      py::gil_scoped_release r;
      ls = local_recover(lb, U, nthreads);
    }
    return py::make_tuple(np_mat(ls.qx), np_mat(ls.qy), np_mat(ls.qz), np_mat(ls.u));
  }, py::arg("lb"), py::arg("uhat"), py::arg("nthreads") = 1);

  // ------------------------------------------------------- global system
  m.def("assemble", [](const ExpandedMesh& em, const py::array_t<double>& C, const DArr& Cf) {
    // C: (nelt, m, m) slices F-ordered
    CondensedSystem cs;
    const int nelt = int(C.shape(0)), mm = int(C.shape(1));
    cs.C = Batch3(mm, mm, nelt);
    auto Cu = C.unchecked<3>();
    for (int K = 0; K < nelt; ++K)
      for (int j = 0; j < mm; ++j)
        for (int i = 0; i < mm; ++i) cs.C.slice(K)[i + size_t(j) * mm] = Cu(K, i, j);
    cs.Cf = mat_from(Cf);
    const SkeletonSystem s = assemble(em, cs);
    return py::make_tuple(np_vec(s.colptr), np_vec(s.rowidx), np_vec(s.vals), np_vec(s.b));
  });
  m.def("dirichlet_project", [](const ExpandedMesh& em, int k, int tri_deg, const Field& g) {
    return np_vec(dirichlet_project(em, k, tri_rule(tri_deg), g.f));
  });
  m.def("neumann_load", [](const ExpandedMesh& em, int k, int tri_deg, const VField& g) {
    return np_vec(neumann_load(em, k, tri_rule(tri_deg), g.f));
  });
  m.def("gather_traces", [](const ExpandedMesh& em, int d2, const py::array_t<double>& uhat) {
    return np_mat(gather_traces(em, d2, uhat.data()));
  });

  // ---------------------------------------------------------- postprocess
  m.def("postprocess_star",
        [](const ExpandedMesh& em, const Tables& t1, const Field& kappa, const DArr& qx,
           const DArr& qy, const DArr& qz, const DArr& u, int nthreads) {
          LocalSolution ls{mat_from(qx), mat_from(qy), mat_from(qz), mat_from(u)};
          Mat out;
          {
            py::gil_scoped_release r;
            out = postprocess_star(em, t1.tb, t1.tet, kappa.f, ls, nthreads);
          }
          return np_mat(out);
        },
        py::arg("em"), py::arg("t1"), py::arg("kappa"), py::arg("qx"), py::arg("qy"),
        py::arg("qz"), py::arg("u"), py::arg("nthreads") = 1);
  m.def("l2_project_volume", [](const ExpandedMesh& em, const Tables& t, const Field& f) {
    return np_mat(l2_project_volume(em, t.tb, t.tet, f.f));
  });
  m.def("l2_project_skeleton", [](const ExpandedMesh& em, int k, int tri_deg, const Field& f) {
    return np_mat(l2_project_skeleton(em, k, tri_rule(tri_deg), f.f));
  });
  m.def("hdg_project", [](const ExpandedMesh& em, const ElementMatrixSet& ms, const Tables& t,
                          const StabilizationField& tau, const VField& q, const Field& u) {
    const LocalSolution ls = hdg_project(em, ms, t.tb, t.tet, t.tri, tau, q.f, u.f, 1);
    return py::make_tuple(np_mat(ls.qx), np_mat(ls.qy), np_mat(ls.qz), np_mat(ls.u));
  });
  m.def("compute_errors",
        [](const ExpandedMesh& em, const ElementMatrixSet& ms, const StabilizationField& tau,
           const Field& u, const VField& q, int k, const py::array_t<double>& uhat,
           const DArr& qx, const DArr& qy, const DArr& qz, const DArr& uu,
           py::object ustar) {
          LocalSolution ls{mat_from(qx), mat_from(qy), mat_from(qz), mat_from(uu)};
          Mat us;
          const Mat* usp = nullptr;
          if (!ustar.is_none()) {
            us = mat_from(ustar.cast<DArr>());
            usp = &us;
          }
          ErrorReport r = compute_errors(em, ms, tau, u.f, q.f, k, uhat.data(), ls, usp, 1);
          return std::vector<double>{r.e_q, r.e_u, r.e_uhat, r.eps_u, r.eps_uhat, r.e_star};
        });

  // problems.cpp:40-46 — poly-k monomials from std::mt19937(12345 + degree)
  m.def("poly_k_terms", [](int degree) {
    std::mt19937 gen(12345u + static_cast<unsigned>(degree));
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    std::vector<std::tuple<int, int, int, double>> terms;
    for (int d = 0; d <= degree; ++d)
      for (int a = d; a >= 0; --a)
        for (int b = d - a; b >= 0; --b) {
          const double c = dist(gen);
          terms.emplace_back(a, b, d - a - b, c);
        }
    return terms;
  });

  // ------------------------------------------- CPU baseline (bench.py)
  // Times the reference-faithful path on an element range: build (1 thread),
  // local_blocks (1 thread), condense + recover (nthreads). Returns seconds per
  // stage; uhat is the per-element stacked trace (4 d2 x nelt).
  // "all-cores" CPU baseline: every stage of the path parallel
  // over contiguous element chunks (same per-element math and summation order).
  m.def("time_pipeline_all_cores",
        [](const ExpandedMesh& em, const Tables& t, const Field& kappa, const Field& c,
           const Field& f, const StabilizationField& tau, const DArr& uhat, int nthreads) {
          const Mat U = mat_from(uhat);
          py::gil_scoped_release r;
          const int nelt = em.n_elements();
          auto rows = [](const auto& src, int k0, int k1, auto& dst) {
            dst.r = k1 - k0;
            dst.c = src.c;
            dst.a.assign(size_t(dst.r) * dst.c, {});
            for (int j = 0; j < src.c; ++j)
              for (int i = k0; i < k1; ++i) dst.a[size_t(i - k0) + size_t(j) * dst.r] = src.a[size_t(i) + size_t(j) * src.r];
          };
          std::vector<ExpandedMesh> sub(nthreads, em);
          std::vector<StabilizationField> stau(nthreads, tau);
          std::vector<Mat> su(nthreads);
          std::vector<int> k0s(nthreads + 1);
          for (int i = 0; i <= nthreads; ++i) k0s[i] = int(long(nelt) * i / nthreads);
          for (int i = 0; i < nthreads; ++i) {  // chunk views (setup, not timed)
            const int k0 = k0s[i], k1 = k0s[i + 1];
            rows(em.raw.elements, k0, k1, sub[i].raw.elements);
            rows(em.facebyele, k0, k1, sub[i].facebyele);
            rows(em.perm, k0, k1, sub[i].perm);
            rows(em.normals, k0, k1, sub[i].normals);
            sub[i].volume.assign(em.volume.begin() + k0, em.volume.begin() + k1);
            rows(tau.tau, k0, k1, stau[i].tau);
            su[i] = Mat(U.r, k1 - k0);
            for (int K = k0; K < k1; ++K)
              for (int j = 0; j < U.r; ++j) su[i](j, K - k0) = U(j, K);
          }
          std::vector<double> chk(nthreads, 0.0);
          using clk = std::chrono::steady_clock;
          auto t0 = clk::now();
          parallel_for(nthreads, nthreads, [&](int b, int e) {
            for (int i = b; i < e; ++i) {
              if (k0s[i + 1] == k0s[i]) continue;
              ElementMatrixSet ms = build_element_matrices(sub[i], t.tb, t.tet, t.tri, kappa.f, c.f, f.f, stau[i]);
              LocalBlocks lb = local_blocks(ms);
              CondensedSystem cs = condense(lb, 1);
              LocalSolution ls = local_recover(lb, su[i], 1);
              chk[i] = cs.C.data[0] + ls.u.a[0];
            }
          });
          auto t1 = clk::now();
          double sum = 0.0;
          for (double v : chk) sum += v;
          return std::vector<double>{std::chrono::duration<double>(t1 - t0).count(), sum};
        });
  // Config C2's coefficient callbacks as compiled C++ lambdas (what a user of
  // the reference writes as ScalarField, coefficient.hpp:13-14), so the CPU
  // baseline does not pay the field-program interpreter. Same expressions as
  // paper_1305_1489_b200/configs.py (_C2_KAPPA, c = 1 + xyz, _C2 f).
  m.def("c2_native_fields", []() {
    const double pi = 3.141592653589793;
    auto kap = [pi](double x, double y, double) { return 1 + 0.5 * std::sin(2 * pi * x) * std::cos(2 * pi * y); };
    auto c = [](double x, double y, double z) { return 1 + x * y * z; };
    auto f = [pi, kap](double x, double y, double z) {
      return std::exp(x + y) * std::sin(pi * z) *
             (-pi * std::cos(2 * pi * (x + y)) - kap(x, y, z) * (2 - pi * pi) + 1 + x * y * z);
    };
    return py::make_tuple(Field{kap}, Field{c}, Field{f});
  });

  // Whole-mesh CPU baseline in element chunks (<= 16,384
  // elements per chunk, because the materialised reference path needs
  // ~190 KB per element at k = 3): nthreads workers pull chunks of `chunk`
  // contiguous elements and run build_element_matrices -> local_blocks ->
  // condense -> local_recover on each (the reference's per-element math and
  // summation order; every stage on all cores, the "all-cores" mode).
  // Per-thread mesh views (global coordinates and face areas, per-chunk
  // element rows) are set up outside the timed region; the per-chunk row
  // copies are inside it. Returns {seconds, checksum}.
  m.def("time_pipeline_chunked",
        [](const ExpandedMesh& em, const Tables& t, const Field& kappa, const Field& c,
           const Field& f, const StabilizationField& tau, const DArr& uhat, int nthreads, int chunk) {
          const Mat U = mat_from(uhat);
          py::gil_scoped_release r;
          const int nelt = em.n_elements();
          const int nchunks = (nelt + chunk - 1) / chunk;
          nthreads = std::max(1, std::min(nthreads, nchunks));
          std::vector<ExpandedMesh> sub(nthreads);
          std::vector<StabilizationField> stau(nthreads, tau);
          for (auto& s : sub) {  // setup: global arrays the element code indexes
            s.raw.coordinates = em.raw.coordinates;
            s.faces = em.faces;
            s.area = em.area;
            s.facetype = em.facetype;
          }
          auto rows = [](const auto& src, int k0, int k1, auto& dst) {
            dst.r = k1 - k0;
            dst.c = src.c;
            dst.a.resize(size_t(dst.r) * dst.c);
            for (int j = 0; j < src.c; ++j)
              std::memcpy(&dst.a[size_t(j) * dst.r], &src.a[size_t(k0) + size_t(j) * src.r],
                          sizeof(src.a[0]) * size_t(dst.r));
          };
          std::atomic<int> next{0};
          std::vector<double> chk(nthreads, 0.0);
          using clk = std::chrono::steady_clock;
          auto t0 = clk::now();
          std::vector<std::thread> pool;
          for (int w = 0; w < nthreads; ++w)
            pool.emplace_back([&, w] {
              ExpandedMesh& s = sub[w];
              StabilizationField& st = stau[w];
              Mat su;
              for (int ci = next++; ci < nchunks; ci = next++) {
                const int k0 = ci * chunk, k1 = std::min(nelt, k0 + chunk);
                rows(em.raw.elements, k0, k1, s.raw.elements);
                rows(em.facebyele, k0, k1, s.facebyele);
                rows(em.perm, k0, k1, s.perm);
                rows(em.normals, k0, k1, s.normals);
                s.volume.assign(em.volume.begin() + k0, em.volume.begin() + k1);
                rows(tau.tau, k0, k1, st.tau);
                su = Mat(U.r, k1 - k0);
                std::memcpy(su.a.data(), U.col(k0), sizeof(double) * size_t(U.r) * (k1 - k0));
                ElementMatrixSet ms = build_element_matrices(s, t.tb, t.tet, t.tri, kappa.f, c.f, f.f, st);
                LocalBlocks lb = local_blocks(ms);
                CondensedSystem cs = condense(lb, 1);
                LocalSolution ls = local_recover(lb, su, 1);
                chk[w] += cs.C.data[0] + ls.u.a[0];
              }
            });
          for (auto& th : pool) th.join();
          auto t1 = clk::now();
          double sum = 0.0;
          for (double v : chk) sum += v;
          return std::vector<double>{std::chrono::duration<double>(t1 - t0).count(), sum};
        },
        py::arg("em"), py::arg("t"), py::arg("kappa"), py::arg("c"), py::arg("f"), py::arg("tau"),
        py::arg("uhat"), py::arg("nthreads"), py::arg("chunk") = 1024);
  // The reference path (build -> local_blocks -> condense -> local_recover) on
  // the element range [k0, k1) of a full mesh, over nthreads contiguous
  // sub-ranges: returns C (k1-k0, m, m), Cf (m, k1-k0), qx, qy, qz, u
  // (d3, k1-k0). uhat: per-element stacked traces (4 d2, k1-k0). For parity
  // over whole full-size meshes in bounded-memory chunks (tests).
  m.def("pipeline_range",
        [](const ExpandedMesh& em, const Tables& t, const Field& kappa, const Field& c, const Field& f,
           const StabilizationField& tau, const DArr& uhat, int k0, int k1, int nthreads) {
          const Mat U = mat_from(uhat);
          const int ne = k1 - k0, d3 = t.tb.d3, m = 4 * t.tb.d2;
          if (k0 < 0 || k1 > em.n_elements() || ne <= 0 || U.c != ne || U.r != m)
            throw std::invalid_argument("pipeline_range: bad range or uhat shape");
          Batch3 C(m, m, ne);
          Mat Cf(m, ne), qx(d3, ne), qy(d3, ne), qz(d3, ne), u(d3, ne);
          {
            py::gil_scoped_release r;
            auto rows = [](const auto& src, int a, int b, auto& dst) {
              dst.r = b - a;
              dst.c = src.c;
              dst.a.resize(size_t(dst.r) * dst.c);
              for (int j = 0; j < src.c; ++j)
                std::memcpy(&dst.a[size_t(j) * dst.r], &src.a[size_t(a) + size_t(j) * src.r],
                            sizeof(src.a[0]) * size_t(dst.r));
            };
            parallel_for(ne, nthreads, [&](int b, int e) {
              ExpandedMesh s;
              s.raw.coordinates = em.raw.coordinates;
              s.faces = em.faces;
              s.area = em.area;
              rows(em.raw.elements, k0 + b, k0 + e, s.raw.elements);
              rows(em.facebyele, k0 + b, k0 + e, s.facebyele);
              rows(em.perm, k0 + b, k0 + e, s.perm);
              rows(em.normals, k0 + b, k0 + e, s.normals);
              s.volume.assign(em.volume.begin() + k0 + b, em.volume.begin() + k0 + e);
              StabilizationField st = tau;
              rows(tau.tau, k0 + b, k0 + e, st.tau);
              Mat su(m, e - b);
              std::memcpy(su.a.data(), U.col(b), sizeof(double) * size_t(m) * (e - b));
              ElementMatrixSet ms = build_element_matrices(s, t.tb, t.tet, t.tri, kappa.f, c.f, f.f, st);
              LocalBlocks lb = local_blocks(ms);
              CondensedSystem cs = condense(lb, 1);
              LocalSolution ls = local_recover(lb, su, 1);
              std::memcpy(C.slice(b), cs.C.data.data(), cs.C.data.size() * sizeof(double));
              std::memcpy(Cf.col(b), cs.Cf.a.data(), cs.Cf.a.size() * sizeof(double));
              std::memcpy(qx.col(b), ls.qx.a.data(), ls.qx.a.size() * sizeof(double));
              std::memcpy(qy.col(b), ls.qy.a.data(), ls.qy.a.size() * sizeof(double));
              std::memcpy(qz.col(b), ls.qz.a.data(), ls.qz.a.size() * sizeof(double));
              std::memcpy(u.col(b), ls.u.a.data(), ls.u.a.size() * sizeof(double));
            });
          }
          return py::make_tuple(np_batch(C), np_mat(Cf), np_mat(qx), np_mat(qy), np_mat(qz), np_mat(u));
        });
  m.def("time_pipeline",
        [](const ExpandedMesh& em, const Tables& t, const Field& kappa, const Field& c,
           const Field& f, const StabilizationField& tau, const DArr& uhat, int nthreads) {
          const Mat U = mat_from(uhat);
          py::gil_scoped_release r;
          using clk = std::chrono::steady_clock;
          auto t0 = clk::now();
          ElementMatrixSet ms = build_element_matrices(em, t.tb, t.tet, t.tri, kappa.f, c.f, f.f, tau);
          auto t1 = clk::now();
          LocalBlocks lb = local_blocks(ms);
          auto t2 = clk::now();
          CondensedSystem cs = condense(lb, nthreads);
          auto t3 = clk::now();
          LocalSolution ls = local_recover(lb, U, nthreads);
          auto t4 = clk::now();
          auto sec = [](clk::duration d) { return std::chrono::duration<double>(d).count(); };
          return std::vector<double>{sec(t1 - t0), sec(t2 - t1), sec(t3 - t2), sec(t4 - t3),
                                     cs.C.data[0] + ls.u.a[0]};
        });
}
