// Host-side 1D numerics: quadrature rules, collocation derivative matrices
// and Modified_A / Lagrange-GLL basis tables in element storage order.
//
// Restates, in C++ with extended-precision Newton iterations:
//   quadrature.py:57-102   legendre / jacobi / jacobi_deriv recurrences
//   quadrature.py:153-185  GLL, GL and Gauss-Radau(-1) rules
//   quadrature.py:224-260  barycentric interpolation / derivative matrices
//   basis.py:78-114        Modified_A values+derivatives, boundary-first order
//   basis.py:99-108        Lagrange basis through GLL nodes (nodal storage:
//                          endpoints first, stdregions.py:56-67)
#include "tables.h"

#include <cmath>
#include <stdexcept>

namespace sphp {

typedef long double ld;

static void legendre(int n, ld x, ld* p, ld* dp) {
  ld p0 = 1, p1 = x;
  if (n == 0) {
    *p = 1;
    *dp = 0;
    return;
  }
  for (int k = 1; k < n; ++k) {
    ld p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
    p0 = p1;
    p1 = p2;
  }
  *p = p1;
  if (std::fabs(std::fabs(x) - 1.0L) < 1e-30L) {
    ld s = (x > 0) ? 1.0L : ((n - 1) % 2 == 0 ? 1.0L : -1.0L);
    *dp = s * n * (n + 1) / 2.0L;
  } else {
    *dp = n * (p0 - x * p1) / (1 - x * x);
  }
}

ld jacobi(int n, ld a, ld b, ld x) {
  if (n == 0) return 1;
  ld p0 = 1, p1 = 0.5L * ((a + b + 2) * x + (a - b));
  for (int k = 2; k <= n; ++k) {
    ld c = 2 * k + a + b;
    ld a1 = 2 * k * (k + a + b) * (c - 2);
    ld a2 = (c - 1) * (a * a - b * b);
    ld a3 = (c - 2) * (c - 1) * c;
    ld a4 = 2 * (k + a - 1) * (k + b - 1) * c;
    ld p2 = ((a2 + a3 * x) * p1 - a4 * p0) / a1;
    p0 = p1;
    p1 = p2;
  }
  return p1;
}

static ld jacobi_deriv(int n, ld a, ld b, ld x) {
  if (n == 0) return 0;
  return 0.5L * (n + a + b + 1) * jacobi(n - 1, a + 1, b + 1, x);
}

template <class F>
static ld newton(F f, ld x) {
  for (int it = 0; it < 100; ++it) {
    ld fx, dfx;
    f(x, &fx, &dfx);
    ld step = fx / dfx;
    x -= step;
    if (std::fabs(step) < 1e-21L) break;
  }
  return x;
}

void make_rule(int q, int ptype, std::vector<double>& z, std::vector<double>& w) {
  z.assign(q, 0.0);
  w.assign(q, 0.0);
  const ld pi = 3.141592653589793238462643383279502884L;
  if (ptype == 1) {  // Gauss-Lobatto-Legendre (quadrature.py:153-166)
    if (q < 2) throw std::invalid_argument("Gauss-Lobatto-Legendre needs at least 2 points");
    int n = q - 1;
    std::vector<ld> x(q);
    x[0] = -1;
    x[q - 1] = 1;
    for (int i = 1; i < q - 1; ++i) {
      ld g = -std::cos(pi * i / n);
      x[i] = newton(
          [n](ld t, ld* f, ld* df) {
            ld p, dp;
            legendre(n, t, &p, &dp);
            *f = dp;
            *df = (2 * t * dp - n * (n + 1) * p) / (1 - t * t);
          },
          g);
    }
    for (int i = 0; i < q; ++i) {
      ld p, dp;
      legendre(n, x[i], &p, &dp);
      z[i] = (double)x[i];
      w[i] = (double)(2.0L / (q * n * p * p));
    }
  } else if (ptype == 0) {  // Gauss-Legendre (quadrature.py:146-150)
    if (q < 1) throw std::invalid_argument("num_points must be positive");
    if (q == 1) {
      z[0] = 0;
      w[0] = 2;
      return;
    }
    for (int i = 0; i < q; ++i) {
      ld g = -std::cos(pi * (i + 0.75L) / (q + 0.5L));
      ld x = newton(
          [q](ld t, ld* f, ld* df) { legendre(q, t, f, df); }, g);
      ld p, dp;
      legendre(q, x, &p, &dp);
      z[i] = (double)x;
      w[i] = (double)(2.0L / ((1 - x * x) * dp * dp));
    }
  } else if (ptype == 2) {  // Gauss-Radau, endpoint -1 (quadrature.py:169-185)
    if (q < 1) throw std::invalid_argument("num_points must be positive");
    if (q == 1) {
      z[0] = -1;
      w[0] = 2;
      return;
    }
    int n = q - 1;
    z[0] = -1;
    w[0] = 2.0 / ((double)q * q);
    for (int i = 1; i < q; ++i) {
      ld g = -std::cos(2 * pi * i / (2 * q - 1));
      ld x = newton(
          [n](ld t, ld* f, ld* df) {
            *f = jacobi(n, 0, 1, t);
            *df = jacobi_deriv(n, 0, 1, t);
          },
          g);
      ld p, dp;
      legendre(n, x, &p, &dp);
      z[i] = (double)x;
      w[i] = (double)((1 - x) / ((ld)q * q * p * p));
    }
  } else {
    throw std::invalid_argument("unknown points type");
  }
}

// barycentric collocation derivative (quadrature.py:246-260)
void diff_matrix(const std::vector<double>& z, std::vector<double>& D) {
  int q = (int)z.size();
  std::vector<double> bw(q);
  for (int i = 0; i < q; ++i) {
    double prod = 1.0;
    for (int j = 0; j < q; ++j)
      if (j != i) prod *= (z[i] - z[j]);
    bw[i] = 1.0 / prod;
  }
  D.assign((size_t)q * q, 0.0);
  for (int i = 0; i < q; ++i) {
    double s = 0.0;
    for (int j = 0; j < q; ++j) {
      if (i == j) continue;
      D[i * q + j] = (bw[j] / bw[i]) / (z[i] - z[j]);
    }
    for (int j = 0; j < q; ++j)
      if (j != i) s += D[i * q + j];
    D[i * q + i] = -s;
  }
}

// interpolation matrix from nodes to points (quadrature.py:224-243)
static void interp_matrix(const std::vector<double>& nodes, const std::vector<double>& pts,
                          std::vector<double>& I) {
  int n = (int)nodes.size(), q = (int)pts.size();
  std::vector<double> bw(n);
  for (int i = 0; i < n; ++i) {
    double prod = 1.0;
    for (int j = 0; j < n; ++j)
      if (j != i) prod *= (nodes[i] - nodes[j]);
    bw[i] = 1.0 / prod;
  }
  I.assign((size_t)q * n, 0.0);
  for (int i = 0; i < q; ++i) {
    int hit = -1;
    for (int j = 0; j < n; ++j)
      if (pts[i] - nodes[j] == 0.0) {
        hit = j;
        break;
      }
    if (hit >= 0) {
      I[(size_t)i * n + hit] = 1.0;
      continue;
    }
    double s = 0;
    for (int j = 0; j < n; ++j) s += bw[j] / (pts[i] - nodes[j]);
    for (int j = 0; j < n; ++j) I[(size_t)i * n + j] = (bw[j] / (pts[i] - nodes[j])) / s;
  }
}

// Modified_A in storage order (basis.py:78-96, :111-114); Lagrange-GLL
// nodal in storage order endpoints-first (basis.py:99-108, stdregions.py:63-66)
void basis_table(int btype, int m, const std::vector<double>& z, std::vector<double>& B,
                 std::vector<double>& Bd) {
  int q = (int)z.size();
  B.assign((size_t)m * q, 0.0);
  Bd.assign((size_t)m * q, 0.0);
  if (btype == 0) {
    if (m < 2) throw std::invalid_argument("modified basis needs num_modes >= 2");
    for (int i = 0; i < q; ++i) {
      double x = z[i];
      double lo = 0.5 * (1.0 - x), hi = 0.5 * (1.0 + x);
      B[0 * q + i] = lo;
      Bd[0 * q + i] = -0.5;
      B[1 * q + i] = hi;
      Bd[1 * q + i] = 0.5;
      for (int k = 2; k < m; ++k) {
        // evaluate the recurrences in double to stay on the reference's
        // arithmetic path (basis.py:92-95)
        double j = (double)jacobi(k - 2, 1, 1, (ld)x);
        double dj = (double)jacobi_deriv(k - 2, 1, 1, (ld)x);
        B[k * q + i] = lo * hi * j;
        Bd[k * q + i] = -0.5 * x * j + lo * hi * dj;
      }
    }
  } else if (btype == 2) {
    std::vector<double> nodes, nw;
    make_rule(m, 1, nodes, nw);
    std::vector<double> I, Dn;
    interp_matrix(nodes, z, I);  // (q, m)
    diff_matrix(nodes, Dn);      // (m, m)
    // storage permutation [0, m-1, 1..m-2]
    std::vector<int> perm;
    perm.push_back(0);
    perm.push_back(m - 1);
    for (int k = 1; k < m - 1; ++k) perm.push_back(k);
    for (int s = 0; s < m; ++s) {
      int c = perm[s];
      for (int i = 0; i < q; ++i) {
        B[(size_t)s * q + i] = I[(size_t)i * m + c];
        double d = 0;
        for (int l = 0; l < m; ++l) d += I[(size_t)i * m + l] * Dn[(size_t)l * m + c];
        Bd[(size_t)s * q + i] = d;
      }
    }
  } else {
    throw std::invalid_argument("basis type not supported by the tensor-product kernels");
  }
}


// Modified_B (basis.py:117-157): rows in storage order, block p = 0..Pa,
// q = 0..Pb-p within a block (block 0 = the Modified_A table of order Pb).
// pidx[n] = p of row n; bstart[p] = first row of block p (Pa + 2 entries).
void modified_b_table(int Pa, int Pb, const std::vector<double>& z, std::vector<double>& B,
                      std::vector<double>& Bd, std::vector<int>& pidx, std::vector<int>& bstart) {
  if (Pa < 1 || Pb < 1) throw std::invalid_argument("orders must be >= 1");
  if (Pb < Pa) throw std::invalid_argument("second-direction order must be >= first (P_b >= P_a)");
  const int q = (int)z.size();
  std::vector<double> seg, dseg;
  basis_table(0, Pb + 1, z, seg, dseg);
  B.clear();
  Bd.clear();
  pidx.clear();
  bstart.clear();
  for (int p = 0; p <= Pa; ++p) {
    bstart.push_back((int)pidx.size());
    if (p == 0) {
      for (int r = 0; r <= Pb; ++r) {
        B.insert(B.end(), seg.begin() + (size_t)r * q, seg.begin() + (size_t)(r + 1) * q);
        Bd.insert(Bd.end(), dseg.begin() + (size_t)r * q, dseg.begin() + (size_t)(r + 1) * q);
        pidx.push_back(0);
      }
      continue;
    }
    std::vector<double> lop(q), dlop(q), hi(q);
    for (int i = 0; i < q; ++i) {
      const double lo = 0.5 * (1.0 - z[i]);
      double pw = 1.0, pw1 = 1.0;
      for (int k = 0; k < p; ++k) pw *= lo;
      for (int k = 0; k < p - 1; ++k) pw1 *= lo;
      lop[i] = pw;
      dlop[i] = -0.5 * p * pw1;
      hi[i] = 0.5 * (1.0 + z[i]);
    }
    B.insert(B.end(), lop.begin(), lop.end());
    Bd.insert(Bd.end(), dlop.begin(), dlop.end());
    pidx.push_back(p);
    for (int r = 1; r <= Pb - p; ++r) {
      for (int i = 0; i < q; ++i) {
        const double j = (double)jacobi(r - 1, 2 * p - 1, 1, (ld)z[i]);
        const double dj = (double)jacobi_deriv(r - 1, 2 * p - 1, 1, (ld)z[i]);
        B.push_back(lop[i] * hi[i] * j);
        Bd.push_back((dlop[i] * hi[i] + 0.5 * lop[i]) * j + lop[i] * hi[i] * dj);
      }
      pidx.push_back(p);
    }
  }
  bstart.push_back((int)pidx.size());
}

}  // namespace sphp
