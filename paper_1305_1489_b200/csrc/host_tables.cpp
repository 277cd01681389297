// Host-side reference-element tables for the B200 kernels (not timed).
//
// Restates the reference's L0 layer (proj/src/quadrature.cpp, proj/src/basis.cpp)
// and pre-contracts the per-degree reference matrices the kernels consume, so
// the device never re-derives them:
//   Chat[#]   = (1/6) sum_q w_q P_qi dP_qj/dx#        (element_matrices.cpp:117-122)
//   Wlm[l][mu]= sum_r w_r Dperm[mu]_ri Pface[l]_rj    (element_matrices.cpp:197-198)
//   PP[l]     = sum_r w_r Pface[l]_ri Pface[l]_rj     (element_matrices.cpp:163-164)
//   DD        = sum_r w_r D_ri D_rj                   (element_matrices.cpp:172)
//   Shat[#][#'] = (1/6) sum_q w_q dP_qi/dx# dP_qj/dx#'  (element_matrices.cpp:270-271)
// Gauss–Jacobi nodes come from the Jacobi matrix the reference builds
// (quadrature.cpp:12-22), solved here by Sturm-sequence bisection with
// Christoffel weights instead of a QL sweep (same nodes to ~1 ulp).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "host_internal.hpp"

namespace hdgb {

namespace {

// Eigenvalues of the symmetric tridiagonal (a, b) by bisection on Sturm counts.
std::vector<double> tridiag_eigenvalues(const std::vector<double>& a, const std::vector<double>& b) {
  const int n = int(a.size());
  double lo = a[0], hi = a[0];
  for (int i = 0; i < n; ++i) {  // Gershgorin bounds
    const double r = (i > 0 ? std::fabs(b[i - 1]) : 0.0) + (i + 1 < n ? std::fabs(b[i]) : 0.0);
    lo = std::min(lo, a[i] - r);
    hi = std::max(hi, a[i] + r);
  }
  auto count_below = [&](double x) {
    int cnt = 0;
    double q = a[0] - x;
    if (q < 0) ++cnt;
    for (int i = 1; i < n; ++i) {
      if (q == 0.0) q = 1e-300;
      q = (a[i] - x) - b[i - 1] * b[i - 1] / q;
      if (q < 0) ++cnt;
    }
    return cnt;
  };
  std::vector<double> ev(n);
  for (int j = 0; j < n; ++j) {
    double l = lo, h = hi;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (l + h);
      if (mid == l || mid == h) break;
      if (count_below(mid) > j) h = mid; else l = mid;
    }
    ev[j] = 0.5 * (l + h);
  }
  return ev;
}

}  // namespace

// quadrature.cpp:12-41 (Jacobi matrix for (1-x)^alpha on [-1,1], mapped to [0,1])
void gauss_jacobi01(int n, int alpha, std::vector<double>& x, std::vector<double>& w) {
  const double al = alpha;
  std::vector<double> a(n), b(std::max(0, n - 1));
  a[0] = -al / (al + 2.0);
  for (int k = 1; k < n; ++k) a[k] = -al * al / ((2.0 * k + al) * (2.0 * k + al + 2.0));
  for (int k = 1; k < n; ++k)
    b[k - 1] = std::sqrt(4.0 * k * (k + al) * k * (k + al) /
                         ((2.0 * k + al) * (2.0 * k + al) * (2.0 * k + al + 1.0) *
                          (2.0 * k + al - 1.0)));
  const std::vector<double> lam = tridiag_eigenvalues(a, b);
  const double mu0 = std::pow(2.0, al + 1.0) / (al + 1.0);
  x.resize(n);
  w.resize(n);
  for (int i = 0; i < n; ++i) {
    // Christoffel number: 1 / sum_k phat_k(lambda)^2 with the orthonormal recurrence.
    double p0 = 1.0, p1 = 0.0, s = 1.0;
    if (n > 1) {
      p1 = (lam[i] - a[0]) * p0 / b[0];
      s += p1 * p1;
      for (int k = 1; k + 1 < n; ++k) {
        const double p2 = ((lam[i] - a[k]) * p1 - b[k - 1] * p0) / b[k];
        s += p2 * p2;
        p0 = p1;
        p1 = p2;
      }
    }
    x[i] = (lam[i] + 1.0) / 2.0;
    w[i] = mu0 / s / std::pow(2.0, al + 1.0);
  }
}

// quadrature.cpp:43-67 — collapsed tensor rule, loop order k(z), j, i.
void tet_rule(int degree, std::vector<double>& bary, std::vector<double>& w) {
  if (degree < 0 || degree > 60) throw std::invalid_argument("tet_rule: unsupported degree");
  const int n = degree / 2 + 1;
  std::vector<double> ta, wa, tb, wb, tc, wc;
  gauss_jacobi01(n, 0, ta, wa);
  gauss_jacobi01(n, 1, tb, wb);
  gauss_jacobi01(n, 2, tc, wc);
  const int nq = n * n * n;
  bary.assign(size_t(nq) * 4, 0.0);
  w.assign(nq, 0.0);
  int q = 0;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i, ++q) {
        const double z = tc[k], y = tb[j] * (1.0 - z), x = ta[i] * (1.0 - tb[j]) * (1.0 - z);
        bary[q] = 1.0 - x - y - z;
        bary[nq + q] = x;
        bary[2 * nq + q] = y;
        bary[3 * nq + q] = z;
        w[q] = 6.0 * wa[i] * wb[j] * wc[k];
      }
}

// quadrature.cpp:69-90
void tri_rule(int degree, std::vector<double>& bary, std::vector<double>& w) {
  if (degree < 0 || degree > 60) throw std::invalid_argument("tri_rule: unsupported degree");
  const int n = degree / 2 + 1;
  std::vector<double> ta, wa, tb, wb;
  gauss_jacobi01(n, 0, ta, wa);
  gauss_jacobi01(n, 1, tb, wb);
  const int nq = n * n;
  bary.assign(size_t(nq) * 3, 0.0);
  w.assign(nq, 0.0);
  int r = 0;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i, ++r) {
      const double t = tb[j], s = ta[i] * (1.0 - t);
      bary[r] = 1.0 - s - t;
      bary[nq + r] = s;
      bary[2 * nq + r] = t;
      w[r] = 2.0 * wa[i] * wb[j];
    }
}

namespace {

// Homogenised Jacobi recurrence p_n(a,b) = b^n P_n^(alpha,0)(a/b) and its
// partials (basis.cpp:12-33).
void jac(int nmax, int alpha, double a, double b, double* p, double* pa, double* pb) {
  const double al = alpha;
  p[0] = 1.0;
  if (pa) pa[0] = pb[0] = 0.0;
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

}  // namespace

// Orthonormal Dubiner basis on the reference tet, hierarchical by degree with
// (i,j,m) lexicographic inside a degree (basis.cpp:37-101). Column-major
// (npts x d3) outputs; grad outputs may be null.
void dubiner3d(int k, int npts, const double* x, const double* y, const double* z, double* P,
               double* Px, double* Py, double* Pz) {
  const int d3 = pdim3(k);
  const bool grad = Px != nullptr;
  std::vector<double> q(k + 1), qa(k + 1), qb(k + 1), s(k + 1), sa(k + 1), sb(k + 1);
  std::vector<double> r((k + 1) * (k + 1)), ra((k + 1) * (k + 1)), rb((k + 1) * (k + 1));
  for (int p = 0; p < npts; ++p) {
    const double b1 = 1.0 - y[p] - z[p], a1 = 2.0 * x[p] - b1;
    const double b2 = 1.0 - z[p], a2 = 2.0 * y[p] - b2;
    const double t3 = 2.0 * z[p] - 1.0;
    jac(k, 0, a1, b1, q.data(), grad ? qa.data() : nullptr, grad ? qb.data() : nullptr);
    for (int i = 0; i <= k; ++i)
      jac(k - i, 2 * i + 1, a2, b2, &r[i * (k + 1)], grad ? &ra[i * (k + 1)] : nullptr,
          grad ? &rb[i * (k + 1)] : nullptr);
    int col = 0;
    for (int d = 0; d <= k; ++d)
      for (int i = 0; i <= d; ++i)
        for (int j = 0; i + j <= d; ++j, ++col) {
          const int m = d - i - j;
          jac(k - i - j, 2 * i + 2 * j + 2, t3, 1.0, s.data(), grad ? sa.data() : nullptr,
              grad ? sb.data() : nullptr);
          const double N = std::sqrt(2.0 * (2 * i + 1) * (i + j + 1) * (2 * i + 2 * j + 2 * m + 3));
          const double qi = q[i], rj = r[i * (k + 1) + j], sm = s[m];
          const size_t o = p + size_t(col) * npts;
          if (P) P[o] = N * qi * rj * sm;
          if (grad) {
            const double qd = qa[i] - qb[i];
            const double rd = ra[i * (k + 1) + j] - rb[i * (k + 1) + j];
            Px[o] = N * 2.0 * qa[i] * rj * sm;
            Py[o] = N * (qd * rj + qi * 2.0 * ra[i * (k + 1) + j]) * sm;
            Pz[o] = N * (qd * rj * sm + qi * rd * sm + qi * rj * 2.0 * sa[m]);
          }
        }
    (void)d3;
  }
}

// basis.cpp:116-134
void dubiner2d(int k, int npts, const double* sx, const double* t, double* D) {
  std::vector<double> q(k + 1), s(k + 1);
  for (int p = 0; p < npts; ++p) {
    const double b = 1.0 - t[p], a = 2.0 * sx[p] - b;
    jac(k, 0, a, b, q.data(), nullptr, nullptr);
    int col = 0;
    for (int d = 0; d <= k; ++d)
      for (int i = 0; i <= d; ++i, ++col) {
        const int j = d - i;
        jac(j, 2 * i + 1, 2.0 * t[p] - 1.0, 1.0, s.data(), nullptr, nullptr);
        D[p + size_t(col) * npts] = std::sqrt(2.0 * (2 * i + 1) * (i + j + 1)) * q[i] * s[j];
      }
  }
}

// Builds every table for degree k on (tet_deg, tri_deg) rules.
HostTables build_host_tables(int k, int tet_deg, int tri_deg) {
  if (k < 0 || k > kMaxDegree) throw std::invalid_argument("unsupported degree");
  HostTables t;
  t.k = k;
  t.d3 = pdim3(k);
  t.d2 = pdim2(k);
  tet_rule(tet_deg, t.tet_bary, t.tet_w);
  tri_rule(tri_deg, t.tri_bary, t.tri_w);
  const int nq = int(t.tet_w.size()), nqd = int(t.tri_w.size()), d3 = t.d3, d2 = t.d2;
  t.nq = nq;
  t.nqd = nqd;
  const double* vx = &t.tet_bary[nq];
  const double* vy = &t.tet_bary[2 * nq];
  const double* vz = &t.tet_bary[3 * nq];
  t.P.assign(size_t(nq) * d3, 0.0);
  for (auto& g : t.Pd) g.assign(size_t(nq) * d3, 0.0);
  dubiner3d(k, nq, vx, vy, vz, t.P.data(), t.Pd[0].data(), t.Pd[1].data(), t.Pd[2].data());
  // face images q^l of the triangle points (quadrature.cpp:92-102)
  const double* ts = &t.tri_bary[nqd];
  const double* tt = &t.tri_bary[2 * nqd];
  std::vector<double> fx(nqd), fy(nqd), fz(nqd);
  for (int l = 0; l < 4; ++l) {
    for (int r = 0; r < nqd; ++r) {
      const double s = ts[r], u = tt[r];
      const double px[4] = {s, s, 0.0, s}, py[4] = {u, 0.0, s, u}, pz[4] = {0.0, u, u, 1.0 - s - u};
      fx[r] = px[l];
      fy[r] = py[l];
      fz[r] = pz[l];
    }
    t.Pface[l].assign(size_t(nqd) * d3, 0.0);
    dubiner3d(k, nqd, fx.data(), fy.data(), fz.data(), t.Pface[l].data(), nullptr, nullptr, nullptr);
  }
  t.D.assign(size_t(nqd) * d2, 0.0);
  dubiner2d(k, nqd, ts, tt, t.D.data());
  std::vector<double> ms(nqd), mt(nqd);
  for (int mu = 0; mu < 6; ++mu) {  // F_mu maps (basis.cpp:142-147)
    for (int r = 0; r < nqd; ++r) {
      const double s = ts[r], u = tt[r], v = 1.0 - s - u;
      const double F[6][2] = {{s, u}, {u, s}, {u, v}, {s, v}, {v, s}, {v, u}};
      ms[r] = F[mu][0];
      mt[r] = F[mu][1];
    }
    t.Dperm[mu].assign(size_t(nqd) * d2, 0.0);
    dubiner2d(k, nqd, ms.data(), mt.data(), t.Dperm[mu].data());
  }
  // contracted reference matrices
  for (int s = 0; s < 3; ++s) {
    t.Chat[s].assign(size_t(d3) * d3, 0.0);
    for (int j = 0; j < d3; ++j)
      for (int i = 0; i < d3; ++i) {
        double acc = 0;
        for (int q = 0; q < nq; ++q) acc += (t.tet_w[q] * t.P[q + size_t(i) * nq]) * t.Pd[s][q + size_t(j) * nq];
        t.Chat[s][i + size_t(j) * d3] = acc / 6.0;
      }
  }
  for (int s1 = 0; s1 < 3; ++s1)
    for (int s2 = 0; s2 < 3; ++s2) {
      auto& S = t.Shat[3 * s1 + s2];
      S.assign(size_t(d3) * d3, 0.0);
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < d3; ++i) {
          double acc = 0;
          for (int q = 0; q < nq; ++q)
            acc += t.Pd[s1][q + size_t(i) * nq] * t.tet_w[q] * t.Pd[s2][q + size_t(j) * nq];
          S[i + size_t(j) * d3] = acc / 6.0;
        }
    }
  for (int l = 0; l < 4; ++l) {
    t.PP[l].assign(size_t(d3) * d3, 0.0);
    for (int j = 0; j < d3; ++j)
      for (int i = 0; i < d3; ++i) {
        double acc = 0;
        for (int r = 0; r < nqd; ++r)
          acc += t.Pface[l][r + size_t(i) * nqd] * t.tri_w[r] * t.Pface[l][r + size_t(j) * nqd];
        t.PP[l][i + size_t(j) * d3] = acc;
      }
    for (int mu = 0; mu < 6; ++mu) {
      auto& W = t.Wlm[l * 6 + mu];
      W.assign(size_t(d2) * d3, 0.0);
      for (int j = 0; j < d3; ++j)
        for (int i = 0; i < d2; ++i) {
          double acc = 0;
          for (int r = 0; r < nqd; ++r)
            acc += t.Dperm[mu][r + size_t(i) * nqd] * t.tri_w[r] * t.Pface[l][r + size_t(j) * nqd];
          W[i + size_t(j) * d2] = acc;
        }
    }
  }
  t.DD.assign(size_t(d2) * d2, 0.0);
  for (int j = 0; j < d2; ++j)
    for (int i = 0; i < d2; ++i) {
      double acc = 0;
      for (int r = 0; r < nqd; ++r) acc += t.D[r + size_t(i) * nqd] * t.tri_w[r] * t.D[r + size_t(j) * nqd];
      t.DD[i + size_t(j) * d2] = acc;
    }
  return t;
}

}  // namespace hdgb
