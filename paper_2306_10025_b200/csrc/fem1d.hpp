// 1D tables shared by the input generator (generator.cpp) and the model
// problems (model_problem.cpp): tensor Gauss-Legendre rules on [0,1] and the
// equispaced Lagrange basis of degree p (values and derivatives at the
// quadrature points).  Changing the arithmetic here changes the generated
// matrices, whose sha256 the full-size fixtures record (tests/golden).
#pragma once

#include <cmath>
#include <vector>

namespace pdb {

struct Gauss {
  std::vector<double> x, w;  // on [0,1]
};

inline Gauss gauss_legendre01(int n) {
  Gauss g;
  g.x.resize(n);
  g.w.resize(n);
  // Legendre P_n and P_n' at z by the three-term recurrence.
  auto legendre = [n](double z, double& pn, double& dpn) {
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= n; ++k) {
      const double pk = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = pk;
    }
    pn = p1;
    dpn = n * (z * p1 - p0) / (z * z - 1.0);
  };
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double pn, dp;
    for (int it = 0; it < 100; ++it) {
      legendre(z, pn, dp);
      const double dz = pn / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    legendre(z, pn, dp);
    g.x[n - 1 - i] = 0.5 * (1.0 + z);
    g.w[n - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);  // 2/((1-z^2)P'^2) mapped to [0,1]
  }
  return g;
}

// 1D Lagrange basis on nodes a/p: values and derivatives at the Gauss points.
inline void lagrange_tables(int p, const Gauss& g, std::vector<double>& val, std::vector<double>& der) {
  const int nq = static_cast<int>(g.x.size());
  val.assign((p + 1) * nq, 0.0);
  der.assign((p + 1) * nq, 0.0);
  for (int a = 0; a <= p; ++a) {
    const double xa = static_cast<double>(a) / p;
    for (int q = 0; q < nq; ++q) {
      const double x = g.x[q];
      double v = 1.0;
      for (int b = 0; b <= p; ++b)
        if (b != a) v *= (x - static_cast<double>(b) / p) / (xa - static_cast<double>(b) / p);
      double d = 0.0;
      for (int c = 0; c <= p; ++c) {
        if (c == a) continue;
        double t = 1.0 / (xa - static_cast<double>(c) / p);
        for (int b = 0; b <= p; ++b)
          if (b != a && b != c) t *= (x - static_cast<double>(b) / p) / (xa - static_cast<double>(b) / p);
        d += t;
      }
      val[a * nq + q] = v;
      der[a * nq + q] = d;
    }
  }
}

}  // namespace pdb
