// Compiled C++ client of the drop-in boundary (include/hdg_b200.h through the
// reference-shaped adapter include/hdg/b200.hpp), built by
// __graft_entry__.build() and run by tests/test_capi_smoke.py on the GPU:
// condense -> local_recover -> postprocess_star on the 2x2x2 box at k = 2
// with callbacks sampled at the device's nodes, outputs written for the test
// to compare with the oracle; then the reference's exception contract
// (LocalSolverError{lowest element}, std::invalid_argument for tau < 0).
#include <cmath>
#include <cstdio>
#include <limits>
#include <stdexcept>
#include <vector>

#include "hdg/b200.hpp"

using namespace hdg::b200;

namespace {
int failures = 0;
void expect(bool ok, const char* what) {
  if (!ok) {
    std::fprintf(stderr, "FAILED: %s\n", what);
    ++failures;
  }
}
void write(std::FILE* fh, const std::vector<double>& v) { std::fwrite(v.data(), sizeof(double), v.size(), fh); }
}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: capi_smoke OUT.bin\n");
    return 2;
  }
  const int k = 2;
  Level lv(0, k, 2, 2, 2, HDG_BC_DIRICHLET_TOP_BOTTOM, 1.0);
  const ScalarField kappa = pointwise_field([](double x, double y, double z) { return 2 + std::sin(x) * std::sin(y) * std::sin(z); });
  const ScalarField c = pointwise_field([](double x, double y, double z) { return 1 + 0.5 * (x * x + y * y + z * z); });
  const ScalarField f = pointwise_field([](double x, double y, double z) { return std::cos(x + 2 * y - z); });

  CondensedSystem cs = condense(lv, kappa, c, f);
  const int m = 4 * lv.d2();
  double asym = 0.0;
  for (int K = 0; K < lv.nelt(); ++K)
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j) asym = std::fmax(asym, std::fabs(cs.C(K, i, j) - cs.C(K, j, i)));
  expect(asym < 1e-12, "C symmetric");  // test_local_solver.cpp:96-106

  std::vector<double> uhat(size_t(lv.nfc()) * lv.d2());
  for (size_t i = 0; i < uhat.size(); ++i) uhat[i] = std::sin(0.37 * double(i));
  LocalSolution ls = local_recover(lv, cs, uhat);
  Matrix ustar = postprocess_star(lv, kappa, ls);

  std::FILE* fh = std::fopen(argv[1], "wb");
  if (!fh) return 2;
  const int hdr[4] = {lv.nelt(), m, lv.d3(), ustar.rows};
  std::fwrite(hdr, sizeof(int), 4, fh);
  write(fh, cs.C.data);
  write(fh, cs.Cf.a);
  write(fh, ls.qx.a);
  write(fh, ls.qy.a);
  write(fh, ls.qz.a);
  write(fh, ls.u.a);
  write(fh, ustar.a);
  std::fclose(fh);

  // singular element: kappa = inf on element 3 only (kappa^-1 = 0 there)
  {
    Level lv2(0, 1, 2, 2, 2, HDG_BC_DIRICHLET_TOP_BOTTOM, 1.0);
    int64_t dims[8];
    check(hdg_b200_dims(lv2.ctx(), dims));
    const size_t nq = size_t(dims[3]);
    std::vector<double> kv(nq * lv2.nelt(), 1.0);
    for (size_t q = 0; q < nq; ++q) kv[3 * nq + q] = std::numeric_limits<double>::infinity();
    size_t calls = 0;
    const ScalarField kap_sing = [&](const double*, const double*, const double*, double* out, size_t n) {
      for (size_t i = 0; i < n; ++i) out[i] = kv[i];
      ++calls;
    };
    bool thrown = false;
    try {
      condense(lv2, kap_sing, constant_field(1.0), constant_field(1.0));
      std::fprintf(stderr, "condense returned without LocalSolverError\n");
    } catch (const LocalSolverError& e) {
      thrown = e.element == 3;
      if (!thrown) std::fprintf(stderr, "LocalSolverError on element %d (%s)\n", e.element, e.what());
    }
    expect(thrown && calls == 1, "LocalSolverError on element 3");
    // negative tau on element 2: std::invalid_argument (element_matrices.cpp:38-46)
    Matrix tau(lv2.nelt(), 4);
    for (double& t : tau.a) t = 1.0;
    tau(2, 1) = -1.0;
    lv2.set_tau(tau);
    thrown = false;
    try {
      condense(lv2, constant_field(1.0), constant_field(1.0), constant_field(1.0));
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    expect(thrown, "invalid_argument for tau < 0");
  }
  std::printf("capi_smoke: nelt=%d m=%d failures=%d\n", lv.nelt(), m, failures);
  return failures ? 1 : 0;
}
