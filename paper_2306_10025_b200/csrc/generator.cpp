// Seeded synthetic inputs for the BASELINE.json configurations.
//
// The reference's assembler (fem.cpp:248-346) only builds uniform meshes
// with a manufactured right-hand side, so the jittered / random-coefficient
// configs are produced here.  Discretisation conventions
// follow the reference so that patch detection behaves identically:
//   * Q_p Lagrange on equispaced nodes, DoFs lexicographic with x fastest on
//     the (cells*p+1)^dim lattice (fem.hpp:12-35, fem.cpp:71-86);
//   * tensor Gauss-Legendre with p+1 points per axis (fem.cpp:255);
//   * Dirichlet rows replaced by identity rows WITHOUT column elimination
//     (fem.cpp:323-342), so patch rows on the boundary keep the
//     single-nonzero signature boundary_pattern keys on (patch.cpp:101-111);
//   * stored entries are never pruned (sparse.hpp:17-19).
// Geometry: cell corners off the boundary are jittered by U(+-jitter*h) per
// coordinate and each cell is mapped multilinearly from its corners.
// Randomness: std::mt19937_64 streams with u = (rng() >> 11) * 2^-53
// (jitter: seed; coefficient blocks: seed+1; right-hand side: seed+2).
// Assembly is cell-parallel over 2^dim parity colours (cells of one colour
// share no DoF), so the accumulated values do not depend on thread count.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <random>
#include <thread>

#include "fem1d.hpp"
#include "host.hpp"

namespace pdb {

ElasticHook g_elastic_device_hook = nullptr;

namespace {

inline double unit(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }

template <typename F>
void parallel_for(Index n, int threads, F&& fn) {
  if (n <= 0) return;
  const Index workers = std::max<Index>(1, std::min<Index>(threads, n));
  if (workers == 1) {
    fn(Index{0}, n);
    return;
  }
  const Index chunk = (n + workers - 1) / workers;
  std::vector<std::thread> pool;
  for (Index t = 0; t < workers; ++t) {
    const Index b = std::min(t * chunk, n), e = std::min(b + chunk, n);
    if (b >= e) break;
    pool.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

void generate_scalar(const pdb_gen_options& o, pdb_problem_s& out, const RowWindow* win) {
  require(o.dim == 2 || o.dim == 3, Errc::invalid_argument, "mesh dimension must be 2 or 3");
  require(o.cells >= 1, Errc::invalid_argument, "mesh needs at least one cell per axis");
  require(o.degree >= 1, Errc::invalid_degree, "polynomial degree must be >= 1");
  require(o.jitter >= 0.0 && o.jitter < 0.5, Errc::invalid_argument, "jitter must be in [0, 0.5)");
  const int d = o.dim, p = o.degree;
  const Index C = o.cells;
  const Index npa = C * p + 1;
  const Index n = d == 3 ? npa * npa * npa : npa * npa;
  const Index nva = C + 1;  // vertices per axis
  const Index nv = d == 3 ? nva * nva * nva : nva * nva;
  const double h = 1.0 / static_cast<double>(C);
  int threads = o.threads > 0 ? o.threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));

  // --- geometry: jittered cell corners -----------------------------------
  std::vector<double> X(static_cast<size_t>(nv * d));
  {
    std::mt19937_64 rng(o.seed);
    for (Index v = 0; v < nv; ++v) {
      Index lat[3] = {v % nva, (v / nva) % nva, d == 3 ? v / (nva * nva) : 0};
      bool interior = true;
      for (int k = 0; k < d; ++k)
        if (lat[k] == 0 || lat[k] == C) interior = false;
      for (int k = 0; k < d; ++k) {
        const double u = unit(rng);
        double x = static_cast<double>(lat[k]) * h;
        if (interior) x += (2.0 * u - 1.0) * o.jitter * h;
        X[static_cast<size_t>(v * d + k)] = x;
      }
    }
  }
  // --- coefficient per cell ----------------------------------------------
  const Index ncells = d == 3 ? C * C * C : C * C;
  std::vector<double> rho(static_cast<size_t>(ncells), o.coeff_value);
  if (o.coeff_kind == 1) {
    require(o.block_cells >= 1 && o.n_levels >= 1 && o.n_levels <= 8, Errc::invalid_argument,
            "random-block coefficient needs block_cells >= 1 and 1..8 levels");
    for (int k = 0; k < o.n_levels; ++k)
      require(o.levels[k] > 0.0, Errc::non_positive_coefficient, "coefficient must be positive");
    const Index nb = (C + o.block_cells - 1) / o.block_cells;
    const Index nblocks = d == 3 ? nb * nb * nb : nb * nb;
    std::vector<double> bval(static_cast<size_t>(nblocks));
    std::mt19937_64 rng(o.seed + 1);
    for (Index b = 0; b < nblocks; ++b) {
      Index k = static_cast<Index>(unit(rng) * o.n_levels);
      if (k >= o.n_levels) k = o.n_levels - 1;
      bval[static_cast<size_t>(b)] = o.levels[k];
    }
    for (Index c = 0; c < ncells; ++c) {
      const Index cx = c % C, cy = (c / C) % C, cz = d == 3 ? c / (C * C) : 0;
      const Index bx = cx / o.block_cells, by = cy / o.block_cells, bz = cz / o.block_cells;
      rho[static_cast<size_t>(c)] = bval[static_cast<size_t>(bx + nb * (by + nb * bz))];
    }
  } else {
    require(o.coeff_value > 0.0, Errc::non_positive_coefficient, "coefficient must be positive");
  }

  // --- CSR pattern: tensor ranges of the cells touching each node ----------
  auto axis_range = [&](Index i, Index& lo, Index& w) {
    const Index cmin = i == 0 ? 0 : (i - 1) / p;
    const Index cmax = std::min<Index>(C - 1, i / p);
    lo = cmin * p;
    w = cmax * p + p - lo + 1;
  };
  auto on_boundary = [&](Index i) {
    const Index ix = i % npa, iy = (i / npa) % npa, iz = d == 3 ? i / (npa * npa) : 0;
    if (ix == 0 || ix == npa - 1 || iy == 0 || iy == npa - 1) return true;
    if (d == 3 && (iz == 0 || iz == npa - 1)) return true;
    return false;
  };
  RowWindow all;
  all.ranges = {{0, n}};
  const RowWindow& Wn = win ? *win : all;
  const Index nr = Wn.rows();
  HostCsr& A = out.a;
  A.n = nr;
  A.row_ptr.assign(static_cast<size_t>(nr + 1), 0);
  parallel_for(nr, threads, [&](Index b, Index e) {
    for (Index li = b; li < e; ++li) {
      const Index i = Wn.global(li);
      if (on_boundary(i)) {
        A.row_ptr[static_cast<size_t>(li + 1)] = 1;
        continue;
      }
      Index cnt = 1;
      const Index lat[3] = {i % npa, (i / npa) % npa, d == 3 ? i / (npa * npa) : 0};
      for (int k = 0; k < d; ++k) {
        Index lo, w;
        axis_range(lat[k], lo, w);
        cnt *= w;
      }
      A.row_ptr[static_cast<size_t>(li + 1)] = cnt;
    }
  });
  for (Index i = 0; i < nr; ++i) A.row_ptr[static_cast<size_t>(i + 1)] += A.row_ptr[static_cast<size_t>(i)];
  const Index nnz = A.row_ptr[static_cast<size_t>(nr)];
  require(n < (Index{1} << 31), Errc::invalid_argument, "generator: more than 2^31 rows");
  A.col.resize(static_cast<size_t>(nnz));
  A.val.assign(static_cast<size_t>(nnz), 0.0);
  parallel_for(nr, threads, [&](Index b, Index e) {
    for (Index li = b; li < e; ++li) {
      const Index i = Wn.global(li);
      Index pos = A.row_ptr[static_cast<size_t>(li)];
      if (on_boundary(i)) {
        A.col[static_cast<size_t>(pos)] = static_cast<int32_t>(i);
        A.val[static_cast<size_t>(pos)] = 1.0;
        continue;
      }
      const Index lat[3] = {i % npa, (i / npa) % npa, d == 3 ? i / (npa * npa) : 0};
      Index lo[3] = {0, 0, 0}, w[3] = {1, 1, 1};
      for (int k = 0; k < d; ++k) axis_range(lat[k], lo[k], w[k]);
      for (Index z = 0; z < w[2]; ++z)
        for (Index y = 0; y < w[1]; ++y)
          for (Index x = 0; x < w[0]; ++x)
            A.col[static_cast<size_t>(pos++)] =
                static_cast<int32_t>((lo[0] + x) + npa * ((lo[1] + y) + npa * (lo[2] + z)));
    }
  });

  // --- element matrices, scattered colour by colour ------------------------
  const Gauss g = gauss_legendre01(p + 1);
  const int nq1 = p + 1;
  std::vector<double> val1, der1;
  lagrange_tables(p, g, val1, der1);
  const int nloc1 = p + 1;
  const int nloc = d == 3 ? nloc1 * nloc1 * nloc1 : nloc1 * nloc1;
  const int nq = d == 3 ? nq1 * nq1 * nq1 : nq1 * nq1;
  const int ncorner = d == 3 ? 8 : 4;
  // reference-element tables: grad_xi phi_a at q, d comps; corner shape grads.
  std::vector<double> gref(static_cast<size_t>(nq * nloc * d));
  std::vector<double> cgrad(static_cast<size_t>(nq * ncorner * d));
  std::vector<double> qw(static_cast<size_t>(nq));
  for (int q = 0; q < nq; ++q) {
    const int qx = q % nq1, qy = (q / nq1) % nq1, qz = d == 3 ? q / (nq1 * nq1) : 0;
    qw[q] = g.w[qx] * g.w[qy] * (d == 3 ? g.w[qz] : 1.0);
    for (int a = 0; a < nloc; ++a) {
      const int ax = a % nloc1, ay = (a / nloc1) % nloc1, az = d == 3 ? a / (nloc1 * nloc1) : 0;
      const double vx = val1[ax * nq1 + qx], vy = val1[ay * nq1 + qy], vz = d == 3 ? val1[az * nq1 + qz] : 1.0;
      const double dx = der1[ax * nq1 + qx], dy = der1[ay * nq1 + qy], dz = d == 3 ? der1[az * nq1 + qz] : 0.0;
      double* gr = &gref[static_cast<size_t>((q * nloc + a) * d)];
      gr[0] = dx * vy * vz;
      gr[1] = vx * dy * vz;
      if (d == 3) gr[2] = vx * vy * dz;
    }
    const double xi[3] = {g.x[qx], g.x[qy], d == 3 ? g.x[qz] : 0.0};
    for (int c = 0; c < ncorner; ++c) {
      const int b[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
      double f[3], df[3];
      for (int k = 0; k < 3; ++k) {
        f[k] = b[k] ? xi[k] : 1.0 - xi[k];
        df[k] = b[k] ? 1.0 : -1.0;
      }
      double* cg = &cgrad[static_cast<size_t>((q * ncorner + c) * d)];
      if (d == 2) {
        cg[0] = df[0] * f[1];
        cg[1] = f[0] * df[1];
      } else {
        cg[0] = df[0] * f[1] * f[2];
        cg[1] = f[0] * df[1] * f[2];
        cg[2] = f[0] * f[1] * df[2];
      }
    }
  }

  const int ncolors = 1 << d;
  for (int color = 0; color < ncolors; ++color) {
    const int px = color & 1, py = (color >> 1) & 1, pz = (color >> 2) & 1;
    const Index cxn = (C - px + 1) / 2, cyn = (C - py + 1) / 2, czn = d == 3 ? (C - pz + 1) / 2 : 1;
    const Index ncol = cxn * cyn * czn;
    parallel_for(ncol, threads, [&](Index b, Index e) {
      std::vector<double> K(static_cast<size_t>(nloc * nloc));
      std::vector<double> G(static_cast<size_t>(nloc * d));
      std::vector<Index> dofs(static_cast<size_t>(nloc));
      for (Index t = b; t < e; ++t) {
        const Index cx = px + 2 * (t % cxn), cy = py + 2 * ((t / cxn) % cyn), cz = d == 3 ? pz + 2 * (t / (cxn * cyn)) : 0;
        const Index cell = cx + C * (cy + C * cz);
        const Index slow = d == 3 ? cz : cy;
        if (slow < Wn.cell_lo || slow > Wn.cell_hi) continue;  // touches no window row
        double Xc[8][3];
        for (int c = 0; c < ncorner; ++c) {
          const Index v = (cx + (c & 1)) + nva * ((cy + ((c >> 1) & 1)) + nva * (cz + ((c >> 2) & 1)));
          for (int k = 0; k < d; ++k) Xc[c][k] = X[static_cast<size_t>(v * d + k)];
        }
        std::fill(K.begin(), K.end(), 0.0);
        const double rc = rho[static_cast<size_t>(cell)];
        for (int q = 0; q < nq; ++q) {
          double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // J[r][s] = dx_r/dxi_s
          for (int c = 0; c < ncorner; ++c) {
            const double* cg = &cgrad[static_cast<size_t>((q * ncorner + c) * d)];
            for (int r = 0; r < d; ++r)
              for (int s = 0; s < d; ++s) J[r][s] += Xc[c][r] * cg[s];
          }
          double inv[3][3], det;
          if (d == 2) {
            det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
            inv[0][0] = J[1][1] / det;
            inv[0][1] = -J[0][1] / det;
            inv[1][0] = -J[1][0] / det;
            inv[1][1] = J[0][0] / det;
          } else {
            const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
            const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
            const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
            det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
            inv[0][0] = c00 / det;
            inv[1][0] = c01 / det;
            inv[2][0] = c02 / det;
            inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
            inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
            inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
            inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
            inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
            inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
          }
          require(det > 0.0, Errc::invalid_argument, "generator: inverted cell (jitter too large)");
          // grad_x phi_a = J^{-T} grad_xi phi_a:  G[a][r] = sum_s inv[s][r] gxi[s]
          for (int a = 0; a < nloc; ++a) {
            const double* gx = &gref[static_cast<size_t>((q * nloc + a) * d)];
            for (int r = 0; r < d; ++r) {
              double s = 0.0;
              for (int k = 0; k < d; ++k) s += inv[k][r] * gx[k];
              G[static_cast<size_t>(a * d + r)] = s;
            }
          }
          const double wq = qw[q] * det * rc;
          for (int a = 0; a < nloc; ++a)
            for (int bb = 0; bb < nloc; ++bb) {
              double s = 0.0;
              for (int r = 0; r < d; ++r) s += G[static_cast<size_t>(a * d + r)] * G[static_cast<size_t>(bb * d + r)];
              K[static_cast<size_t>(a * nloc + bb)] += wq * s;
            }
        }
        // local DoF a = ax + (p+1)(ay + (p+1) az), ascending global order
        for (int a = 0; a < nloc; ++a) {
          const int ax = a % nloc1, ay = (a / nloc1) % nloc1, az = d == 3 ? a / (nloc1 * nloc1) : 0;
          dofs[static_cast<size_t>(a)] = (cx * p + ax) + npa * ((cy * p + ay) + npa * (cz * p + az));
        }
        for (int a = 0; a < nloc; ++a) {
          const Index gi = dofs[static_cast<size_t>(a)];
          if (on_boundary(gi)) continue;  // row replaced (fem.cpp:323)
          const Index li = win ? Wn.local(gi) : gi;
          if (li < 0) continue;
          const Index lat[3] = {gi % npa, (gi / npa) % npa, d == 3 ? gi / (npa * npa) : 0};
          Index lo[3] = {0, 0, 0}, w[3] = {1, 1, 1};
          for (int k = 0; k < d; ++k) axis_range(lat[k], lo[k], w[k]);
          const Index base = A.row_ptr[static_cast<size_t>(li)];
          for (int bb = 0; bb < nloc; ++bb) {
            const Index gj = dofs[static_cast<size_t>(bb)];
            const Index jl[3] = {gj % npa, (gj / npa) % npa, d == 3 ? gj / (npa * npa) : 0};
            const Index off = (jl[0] - lo[0]) + w[0] * ((jl[1] - lo[1]) + w[1] * (jl[2] - lo[2]));
            A.val[static_cast<size_t>(base + off)] += K[static_cast<size_t>(a * nloc + bb)];
          }
        }
      }
    });
  }

  // --- right-hand side ----------------------------------------------------
  out.rhs.assign(static_cast<size_t>(nr), 0.0);
  {
    std::mt19937_64 rng(o.seed + 2);  // one draw per global row
    Index at = 0, li = 0;
    for (const auto& g : Wn.ranges) {
      rng.discard(static_cast<unsigned long long>(g.first - at));
      for (Index i = g.first; i < g.second; ++i, ++li) {
        const double u = unit(rng);
        if (!on_boundary(i)) out.rhs[static_cast<size_t>(li)] = 2.0 * u - 1.0;
      }
      at = g.second;
    }
  }
  out.has_exact = false;
  out.dim = d;
  out.cells = C;
  out.degree = p;
  out.components = 1;
  out.n_global = n;
  if (win) out.row_ranges.assign(win->ranges.begin(), win->ranges.end());
}

// ---- vector systems: Stokes (config 4) and linear elasticity (config 5) ----
//
// DoFs are node-major: the ncomp = dim components of lattice node v are DoFs
// ncomp*v + c, nodes lexicographic with x fastest on the (cells*p+1)^dim
// lattice (so every row's columns come out ascending).  Stokes pressure DoFs
// follow all velocity DoFs, lexicographic on the (cells*(p-1)+1)^dim lattice
// of the continuous Q_{p-1} pressure space (Taylor-Hood).  Dirichlet: every
// velocity / displacement component of a boundary node gets an identity row
// (no column elimination, as fem.cpp:323-342); pressure rows are left
// unconstrained and there is no pressure-pressure block.  Element forms:
//   Stokes     a(u,v) = int 2 mu eps(u):eps(v),   b(v,q) = -int q div v
//   elasticity a(u,v) = int lambda div u div v + 2 mu eps(u):eps(v)
// i.e. K[(a,c),(b,e)] = int lam d_c phi_a d_e phi_b
//                       + mu (delta_ce grad phi_a . grad phi_b + d_e phi_a d_c phi_b).
// With symmetric gradients a cell-interior node couples to both components of
// every node of its cell, so the Vanka rows of a Q2-Q1 cell have 2*9 + 4 = 22
// entries and the interior rows of a Q3 hex 3*64 = 192.
// Coefficients: coeff_kind 1 = random blocks (seed+1 stream, as generate_scalar),
// 2 = lognormal exp(coeff_value * z), z ~ N(0,1) by Box-Muller on the seed+1
// stream.  Right-hand side: U[-1,1] on free velocity / displacement rows,
// 0 on Dirichlet and pressure rows (seed+2 stream, one draw per DoF).
void generate_system(const pdb_gen_options& o, pdb_problem_s& out, const RowWindow* win) {
  require(o.physics == 1 || o.physics == 2, Errc::invalid_argument, "physics must be 1 (Stokes) or 2 (elasticity)");
  const bool stokes = o.physics == 1;
  require(o.dim == 2 || o.dim == 3, Errc::invalid_argument, "mesh dimension must be 2 or 3");
  require(!stokes || o.dim == 2, Errc::invalid_argument, "the Stokes generator is two-dimensional");
  require(o.cells >= 1, Errc::invalid_argument, "mesh needs at least one cell per axis");
  require(o.degree >= (stokes ? 2 : 1), Errc::invalid_degree,
          stokes ? "Taylor-Hood needs velocity degree >= 2" : "polynomial degree must be >= 1");
  require(o.jitter >= 0.0 && o.jitter < 0.5, Errc::invalid_argument, "jitter must be in [0, 0.5)");
  const int d = o.dim, p = o.degree, pp = p - 1, ncomp = d;
  const Index C = o.cells;
  const Index npa = C * p + 1, ppa = C * pp + 1;
  const Index nnodes = d == 3 ? npa * npa * npa : npa * npa;
  const Index npres = stokes ? (d == 3 ? ppa * ppa * ppa : ppa * ppa) : 0;
  const Index nu = ncomp * nnodes, n = nu + npres;
  require(n < (Index{1} << 31), Errc::invalid_argument, "generator: more than 2^31 rows");
  const Index nva = C + 1;
  const Index nv = d == 3 ? nva * nva * nva : nva * nva;
  const double h = 1.0 / static_cast<double>(C);
  const int threads = o.threads > 0 ? o.threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  double lam_f = 0.0, mu_f = 1.0;  // Lame factors per unit coefficient
  if (!stokes) {
    const double nu_ = o.poisson_ratio;
    require(nu_ > -1.0 && nu_ < 0.5, Errc::invalid_argument, "Poisson ratio must be in (-1, 0.5)");
    lam_f = nu_ / ((1.0 + nu_) * (1.0 - 2.0 * nu_));
    mu_f = 1.0 / (2.0 * (1.0 + nu_));
  }

  // geometry: jittered cell corners (same stream use as generate_scalar)
  std::vector<double> X(static_cast<size_t>(nv * d));
  {
    std::mt19937_64 rng(o.seed);
    for (Index v = 0; v < nv; ++v) {
      Index lat[3] = {v % nva, (v / nva) % nva, d == 3 ? v / (nva * nva) : 0};
      bool interior = true;
      for (int k = 0; k < d; ++k)
        if (lat[k] == 0 || lat[k] == C) interior = false;
      for (int k = 0; k < d; ++k) {
        const double u = unit(rng);
        double x = static_cast<double>(lat[k]) * h;
        if (interior) x += (2.0 * u - 1.0) * o.jitter * h;
        X[static_cast<size_t>(v * d + k)] = x;
      }
    }
  }
  // coefficient per cell
  const Index ncells = d == 3 ? C * C * C : C * C;
  std::vector<double> coef(static_cast<size_t>(ncells), o.coeff_value);
  if (o.coeff_kind == 1) {
    require(o.block_cells >= 1 && o.n_levels >= 1 && o.n_levels <= 8, Errc::invalid_argument,
            "random-block coefficient needs block_cells >= 1 and 1..8 levels");
    for (int k = 0; k < o.n_levels; ++k)
      require(o.levels[k] > 0.0, Errc::non_positive_coefficient, "coefficient must be positive");
    const Index nb = (C + o.block_cells - 1) / o.block_cells;
    const Index nblocks = d == 3 ? nb * nb * nb : nb * nb;
    std::vector<double> bval(static_cast<size_t>(nblocks));
    std::mt19937_64 rng(o.seed + 1);
    for (Index b = 0; b < nblocks; ++b) {
      Index k = static_cast<Index>(unit(rng) * o.n_levels);
      if (k >= o.n_levels) k = o.n_levels - 1;
      bval[static_cast<size_t>(b)] = o.levels[k];
    }
    for (Index c = 0; c < ncells; ++c) {
      const Index cx = c % C, cy = (c / C) % C, cz = d == 3 ? c / (C * C) : 0;
      coef[static_cast<size_t>(c)] =
          bval[static_cast<size_t>(cx / o.block_cells + nb * (cy / o.block_cells + nb * (cz / o.block_cells)))];
    }
  } else if (o.coeff_kind == 2) {
    require(o.coeff_value >= 0.0, Errc::invalid_argument, "lognormal sigma must be >= 0");
    std::mt19937_64 rng(o.seed + 1);
    for (Index c = 0; c < ncells; ++c) {
      const double u1 = 1.0 - unit(rng), u2 = unit(rng);  // u1 in (0, 1]
      const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
      coef[static_cast<size_t>(c)] = std::exp(o.coeff_value * z);
    }
  } else {
    require(o.coeff_value > 0.0, Errc::non_positive_coefficient, "coefficient must be positive");
  }

  // lattice helpers: node / pressure-node ranges of the cells around a point
  auto cell_span = [&](Index i, int deg, Index& cmin, Index& cmax) {
    cmin = i == 0 ? 0 : (i - 1) / deg;
    cmax = std::min<Index>(C - 1, i / deg);
  };
  auto lattice = [&](Index v, Index per, Index* l) {
    l[0] = v % per;
    l[1] = (v / per) % per;
    l[2] = d == 3 ? v / (per * per) : 0;
  };
  auto boundary_node = [&](Index v) {
    Index l[3];
    lattice(v, npa, l);
    for (int k = 0; k < d; ++k)
      if (l[k] == 0 || l[k] == npa - 1) return true;
    return false;
  };
  // for a velocity row at node lattice l: velocity node range (lo, w) and pressure range (plo, pw)
  struct Range {
    Index lo[3] = {0, 0, 0}, w[3] = {1, 1, 1}, plo[3] = {0, 0, 0}, pw[3] = {1, 1, 1};
    Index nvel = 0, npr = 0;
  };
  auto node_ranges = [&](const Index* l) {
    Range r;
    r.nvel = ncomp;
    r.npr = stokes ? 1 : 0;
    for (int k = 0; k < d; ++k) {
      Index cmin, cmax;
      cell_span(l[k], p, cmin, cmax);
      r.lo[k] = cmin * p;
      r.w[k] = (cmax - cmin) * p + p + 1;
      r.nvel *= r.w[k];
      if (stokes) {
        r.plo[k] = cmin * pp;
        r.pw[k] = (cmax - cmin) * pp + pp + 1;
        r.npr *= r.pw[k];
      }
    }
    return r;
  };
  auto pres_ranges = [&](const Index* q) {  // velocity node range of the cells around pressure node q
    Range r;
    r.nvel = ncomp;
    for (int k = 0; k < d; ++k) {
      Index cmin, cmax;
      cell_span(q[k], pp, cmin, cmax);
      r.lo[k] = cmin * p;
      r.w[k] = (cmax - cmin) * p + p + 1;
      r.nvel *= r.w[k];
    }
    return r;
  };

  RowWindow all;
  all.ranges = {{0, n}};
  const RowWindow& Wn = win ? *win : all;
  const Index nr = Wn.rows();
  HostCsr& A = out.a;
  A.n = nr;
  A.row_ptr.assign(static_cast<size_t>(nr + 1), 0);
  parallel_for(nr, threads, [&](Index b, Index e) {
    for (Index li = b; li < e; ++li) {
      const Index i = Wn.global(li);
      Index cnt;
      if (i < nu) {
        const Index v = i / ncomp;
        if (boundary_node(v)) {
          cnt = 1;
        } else {
          Index l[3];
          lattice(v, npa, l);
          const Range r = node_ranges(l);
          cnt = r.nvel + r.npr;
        }
      } else {
        Index q[3];
        lattice(i - nu, ppa, q);
        cnt = pres_ranges(q).nvel;
      }
      A.row_ptr[static_cast<size_t>(li + 1)] = cnt;
    }
  });
  for (Index i = 0; i < nr; ++i) A.row_ptr[static_cast<size_t>(i + 1)] += A.row_ptr[static_cast<size_t>(i)];
  const Index nnz = A.row_ptr[static_cast<size_t>(nr)];
  A.col.resize(static_cast<size_t>(nnz));
  A.val.assign(static_cast<size_t>(nnz), 0.0);
  parallel_for(nr, threads, [&](Index b, Index e) {
    for (Index li = b; li < e; ++li) {
      const Index i = Wn.global(li);
      Index pos = A.row_ptr[static_cast<size_t>(li)];
      if (i < nu && boundary_node(i / ncomp)) {
        A.col[static_cast<size_t>(pos)] = static_cast<int32_t>(i);
        A.val[static_cast<size_t>(pos)] = 1.0;
        continue;
      }
      Range r;
      if (i < nu) {
        Index l[3];
        lattice(i / ncomp, npa, l);
        r = node_ranges(l);
      } else {
        Index q[3];
        lattice(i - nu, ppa, q);
        r = pres_ranges(q);
      }
      for (Index z = 0; z < r.w[2]; ++z)
        for (Index y = 0; y < r.w[1]; ++y)
          for (Index x = 0; x < r.w[0]; ++x) {
            const Index node = (r.lo[0] + x) + npa * ((r.lo[1] + y) + npa * (r.lo[2] + z));
            for (int c = 0; c < ncomp; ++c) A.col[static_cast<size_t>(pos++)] = static_cast<int32_t>(ncomp * node + c);
          }
      if (i < nu && stokes)
        for (Index z = 0; z < r.pw[2]; ++z)
          for (Index y = 0; y < r.pw[1]; ++y)
            for (Index x = 0; x < r.pw[0]; ++x)
              A.col[static_cast<size_t>(pos++)] =
                  static_cast<int32_t>(nu + (r.plo[0] + x) + ppa * ((r.plo[1] + y) + ppa * (r.plo[2] + z)));
    }
  });

  // reference-element tables
  const Gauss g = gauss_legendre01(p + 1);
  const int nq1 = p + 1;
  std::vector<double> val1, der1, pval1, pder1;
  lagrange_tables(p, g, val1, der1);
  if (stokes) lagrange_tables(pp, g, pval1, pder1);
  const int nl1 = p + 1, pl1 = pp + 1;
  const int nloc = d == 3 ? nl1 * nl1 * nl1 : nl1 * nl1;
  const int ploc = stokes ? (d == 3 ? pl1 * pl1 * pl1 : pl1 * pl1) : 0;
  const int nq = d == 3 ? nq1 * nq1 * nq1 : nq1 * nq1;
  const int ncorner = d == 3 ? 8 : 4;
  const int ndof = nloc * ncomp;
  std::vector<double> gref(static_cast<size_t>(nq * nloc * d)), cgrad(static_cast<size_t>(nq * ncorner * d));
  std::vector<double> qw(static_cast<size_t>(nq)), pref(static_cast<size_t>(nq * std::max(ploc, 1)));
  for (int q = 0; q < nq; ++q) {
    const int qx = q % nq1, qy = (q / nq1) % nq1, qz = d == 3 ? q / (nq1 * nq1) : 0;
    qw[q] = g.w[qx] * g.w[qy] * (d == 3 ? g.w[qz] : 1.0);
    for (int a = 0; a < nloc; ++a) {
      const int ax = a % nl1, ay = (a / nl1) % nl1, az = d == 3 ? a / (nl1 * nl1) : 0;
      const double vx = val1[ax * nq1 + qx], vy = val1[ay * nq1 + qy], vz = d == 3 ? val1[az * nq1 + qz] : 1.0;
      const double dx = der1[ax * nq1 + qx], dy = der1[ay * nq1 + qy], dz = d == 3 ? der1[az * nq1 + qz] : 0.0;
      double* gr = &gref[static_cast<size_t>((q * nloc + a) * d)];
      gr[0] = dx * vy * vz;
      gr[1] = vx * dy * vz;
      if (d == 3) gr[2] = vx * vy * dz;
    }
    for (int i = 0; i < ploc; ++i) {
      const int ix = i % pl1, iy = (i / pl1) % pl1, iz = d == 3 ? i / (pl1 * pl1) : 0;
      pref[static_cast<size_t>(q * ploc + i)] =
          pval1[ix * nq1 + qx] * pval1[iy * nq1 + qy] * (d == 3 ? pval1[iz * nq1 + qz] : 1.0);
    }
    const double xi[3] = {g.x[qx], g.x[qy], d == 3 ? g.x[qz] : 0.0};
    for (int c = 0; c < ncorner; ++c) {
      const int bb[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
      double f[3], df[3];
      for (int k = 0; k < 3; ++k) {
        f[k] = bb[k] ? xi[k] : 1.0 - xi[k];
        df[k] = bb[k] ? 1.0 : -1.0;
      }
      double* cg = &cgrad[static_cast<size_t>((q * ncorner + c) * d)];
      if (d == 2) {
        cg[0] = df[0] * f[1];
        cg[1] = f[0] * df[1];
      } else {
        cg[0] = df[0] * f[1] * f[2];
        cg[1] = f[0] * df[1] * f[2];
        cg[2] = f[0] * f[1] * df[2];
      }
    }
  }

  bool on_device = false;
  if (!stokes && g_elastic_device_hook != nullptr) {
    const char* ge = getenv("PDB_GEN_DEVICE");
    if (!(ge && ge[0] == '0')) {
      ElasticAssembly ea{d, p, ncomp, nloc, nq, ncorner, C, nva, npa, X.data(), coef.data(), gref.data(),
                         cgrad.data(), qw.data(), lam_f, mu_f, Wn.cell_lo, Wn.cell_hi, Wn.ranges,
                         A.row_ptr.data(), A.val.data(), nnz};
      on_device = g_elastic_device_hook(ea);
    }
  }
  const int ncolors = on_device ? 0 : 1 << d;
  for (int color = 0; color < ncolors; ++color) {
    const int px = color & 1, py = (color >> 1) & 1, pz = (color >> 2) & 1;
    const Index cxn = (C - px + 1) / 2, cyn = (C - py + 1) / 2, czn = d == 3 ? (C - pz + 1) / 2 : 1;
    parallel_for(cxn * cyn * czn, threads, [&](Index b, Index e) {
      std::vector<double> K(static_cast<size_t>(ndof * ndof)), B(static_cast<size_t>(std::max(ploc, 1) * ndof));
      std::vector<double> G(static_cast<size_t>(nloc * d));
      std::vector<Index> node(static_cast<size_t>(nloc)), pnode(static_cast<size_t>(std::max(ploc, 1)));
      for (Index t = b; t < e; ++t) {
        const Index cx = px + 2 * (t % cxn), cy = py + 2 * ((t / cxn) % cyn), cz = d == 3 ? pz + 2 * (t / (cxn * cyn)) : 0;
        const Index cell = cx + C * (cy + C * cz);
        const Index slow = d == 3 ? cz : cy;
        if (slow < Wn.cell_lo || slow > Wn.cell_hi) continue;  // touches no window row
        double Xc[8][3];
        for (int c = 0; c < ncorner; ++c) {
          const Index v = (cx + (c & 1)) + nva * ((cy + ((c >> 1) & 1)) + nva * (cz + ((c >> 2) & 1)));
          for (int k = 0; k < d; ++k) Xc[c][k] = X[static_cast<size_t>(v * d + k)];
        }
        std::fill(K.begin(), K.end(), 0.0);
        std::fill(B.begin(), B.end(), 0.0);
        const double cc = coef[static_cast<size_t>(cell)];
        const double lam = lam_f * cc, mu = mu_f * cc;
        for (int q = 0; q < nq; ++q) {
          double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
          for (int c = 0; c < ncorner; ++c) {
            const double* cg = &cgrad[static_cast<size_t>((q * ncorner + c) * d)];
            for (int r = 0; r < d; ++r)
              for (int s2 = 0; s2 < d; ++s2) J[r][s2] += Xc[c][r] * cg[s2];
          }
          double inv[3][3], det;
          if (d == 2) {
            det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
            inv[0][0] = J[1][1] / det;
            inv[0][1] = -J[0][1] / det;
            inv[1][0] = -J[1][0] / det;
            inv[1][1] = J[0][0] / det;
          } else {
            const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
            const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
            const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
            det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
            inv[0][0] = c00 / det;
            inv[1][0] = c01 / det;
            inv[2][0] = c02 / det;
            inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
            inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
            inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
            inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
            inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
            inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
          }
          require(det > 0.0, Errc::invalid_argument, "generator: inverted cell (jitter too large)");
          for (int a = 0; a < nloc; ++a) {
            const double* gx = &gref[static_cast<size_t>((q * nloc + a) * d)];
            for (int r = 0; r < d; ++r) {
              double s2 = 0.0;
              for (int k = 0; k < d; ++k) s2 += inv[k][r] * gx[k];
              G[static_cast<size_t>(a * d + r)] = s2;
            }
          }
          const double wq = qw[q] * det;
          for (int a = 0; a < nloc; ++a) {
            const double* Ga = &G[static_cast<size_t>(a * d)];
            for (int bn = 0; bn < nloc; ++bn) {
              const double* Gb = &G[static_cast<size_t>(bn * d)];
              double dot = 0.0;
              for (int r = 0; r < d; ++r) dot += Ga[r] * Gb[r];
              for (int c = 0; c < ncomp; ++c)
                for (int e2 = 0; e2 < ncomp; ++e2) {
                  double v = lam * Ga[c] * Gb[e2] + mu * Ga[e2] * Gb[c];
                  if (c == e2) v += mu * dot;
                  K[static_cast<size_t>((a * ncomp + c) * ndof + bn * ncomp + e2)] += wq * v;
                }
            }
          }
          for (int i = 0; i < ploc; ++i) {
            const double psi = pref[static_cast<size_t>(q * ploc + i)];
            for (int bn = 0; bn < nloc; ++bn)
              for (int e2 = 0; e2 < ncomp; ++e2)
                B[static_cast<size_t>(i * ndof + bn * ncomp + e2)] -= wq * psi * G[static_cast<size_t>(bn * d + e2)];
          }
        }
        for (int a = 0; a < nloc; ++a) {
          const int ax = a % nl1, ay = (a / nl1) % nl1, az = d == 3 ? a / (nl1 * nl1) : 0;
          node[static_cast<size_t>(a)] = (cx * p + ax) + npa * ((cy * p + ay) + npa * (cz * p + az));
        }
        for (int i = 0; i < ploc; ++i) {
          const int ix = i % pl1, iy = (i / pl1) % pl1, iz = d == 3 ? i / (pl1 * pl1) : 0;
          pnode[static_cast<size_t>(i)] = (cx * pp + ix) + ppa * ((cy * pp + iy) + ppa * (cz * pp + iz));
        }
        // velocity / displacement rows
        for (int a = 0; a < nloc; ++a) {
          const Index gv = node[static_cast<size_t>(a)];
          if (boundary_node(gv)) continue;  // identity rows (fem.cpp:323)
          Index l[3];
          lattice(gv, npa, l);
          const Range r = node_ranges(l);
          for (int c = 0; c < ncomp; ++c) {
            const Index li = win ? Wn.local(ncomp * gv + c) : ncomp * gv + c;
            if (li < 0) continue;
            const Index base = A.row_ptr[static_cast<size_t>(li)];
            for (int bn = 0; bn < nloc; ++bn) {
              Index jl[3];
              lattice(node[static_cast<size_t>(bn)], npa, jl);
              const Index off = ((jl[0] - r.lo[0]) + r.w[0] * ((jl[1] - r.lo[1]) + r.w[1] * (jl[2] - r.lo[2]))) * ncomp;
              for (int e2 = 0; e2 < ncomp; ++e2)
                A.val[static_cast<size_t>(base + off + e2)] += K[static_cast<size_t>((a * ncomp + c) * ndof + bn * ncomp + e2)];
            }
            for (int i = 0; i < ploc; ++i) {  // B^T block
              Index ql[3];
              lattice(pnode[static_cast<size_t>(i)], ppa, ql);
              const Index off = r.nvel + (ql[0] - r.plo[0]) + r.pw[0] * ((ql[1] - r.plo[1]) + r.pw[1] * (ql[2] - r.plo[2]));
              A.val[static_cast<size_t>(base + off)] += B[static_cast<size_t>(i * ndof + a * ncomp + c)];
            }
          }
        }
        // pressure rows
        for (int i = 0; i < ploc; ++i) {
          Index ql[3];
          lattice(pnode[static_cast<size_t>(i)], ppa, ql);
          const Range r = pres_ranges(ql);
          const Index li = win ? Wn.local(nu + pnode[static_cast<size_t>(i)]) : nu + pnode[static_cast<size_t>(i)];
          if (li < 0) continue;
          const Index base = A.row_ptr[static_cast<size_t>(li)];
          for (int bn = 0; bn < nloc; ++bn) {
            Index jl[3];
            lattice(node[static_cast<size_t>(bn)], npa, jl);
            const Index off = ((jl[0] - r.lo[0]) + r.w[0] * ((jl[1] - r.lo[1]) + r.w[1] * (jl[2] - r.lo[2]))) * ncomp;
            for (int e2 = 0; e2 < ncomp; ++e2)
              A.val[static_cast<size_t>(base + off + e2)] += B[static_cast<size_t>(i * ndof + bn * ncomp + e2)];
          }
        }
      }
    });
  }

  out.rhs.assign(static_cast<size_t>(nr), 0.0);
  {
    std::mt19937_64 rng(o.seed + 2);  // one draw per global row
    Index at = 0, li = 0;
    for (const auto& g : Wn.ranges) {
      rng.discard(static_cast<unsigned long long>(g.first - at));
      for (Index i = g.first; i < g.second; ++i, ++li) {
        const double u = unit(rng);
        if (i < nu && !boundary_node(i / ncomp)) out.rhs[static_cast<size_t>(li)] = 2.0 * u - 1.0;
      }
      at = g.second;
    }
  }
  out.n_global = n;
  if (win) out.row_ranges.assign(win->ranges.begin(), win->ranges.end());
  out.has_exact = false;
  out.dim = d;
  out.cells = C;
  out.degree = p;
  out.components = 0;  // vector / mixed DoFs: no scalar lattice
}

RowWindow slab_window(const pdb_gen_options& o, int rank, int nranks) {
  require(nranks >= 1 && rank >= 0 && rank < nranks, Errc::invalid_argument, "rank must be in [0, nranks)");
  const Index C = o.cells;
  require(nranks == 1 || C / nranks >= 2, Errc::invalid_argument,
          "slab partition too thin: every rank needs at least two cell layers");
  return cells_window(o, C * rank / nranks, C * (rank + 1) / nranks);
}

RowWindow cells_window(const pdb_gen_options& o, Index s0, Index s1) {
  const Index C = o.cells;
  require(s0 >= 0 && s1 <= C && s0 < s1, Errc::invalid_argument, "cell layer range must satisfy 0 <= c0 < c1 <= cells");
  const int d = o.dim, p = o.degree;
  const Index npa = C * p + 1;
  const Index layer = d == 3 ? npa * npa : npa;  // nodes per slowest-axis layer
  RowWindow w;
  w.cell_lo = s0 > 0 ? s0 - 1 : 0;
  w.cell_hi = std::min<Index>(C - 1, s1);
  if (o.physics == 0) {
    w.ranges.push_back({s0 * p * layer, (s1 * p + 1) * layer});
  } else {
    const Index ncomp = d;
    w.ranges.push_back({ncomp * s0 * p * layer, ncomp * (s1 * p + 1) * layer});
    if (o.physics == 1) {
      const Index pp = p - 1, ppa = C * pp + 1;
      const Index player = d == 3 ? ppa * ppa : ppa;
      const Index nu = ncomp * (d == 3 ? npa * npa * npa : npa * npa);
      w.ranges.push_back({nu + s0 * pp * player, nu + (s1 * pp + 1) * player});
    }
  }
  return w;
}

void gen_options_defaults(pdb_gen_options* o) {
  if (o == nullptr) return;
  *o = pdb_gen_options{};
  o->dim = 2;
  o->degree = 2;
  o->cells = 32;
  o->seed = 42;
  o->coeff_value = 1.0;
  o->block_cells = 1;
  o->poisson_ratio = 0.3;
}

// 1 = 2D Q2 32^2 jitter 0.1; 2 = 2D Q4 256^2 jitter 0.05, rho on 8x8-cell
// blocks from {1,10,100,1000}; 3 = 3D Q2 64^3 jitter 0.1; 4 = 2D Stokes
// Q2-Q1 512^2, mu lognormal(0,1) per cell; 5 = 3D elasticity Q3 96^3,
// E from {1,100} on 4^3-cell blocks, nu 0.3.
bool gen_options_preset(int config, int64_t cells, pdb_gen_options* o) {
  gen_options_defaults(o);
  switch (config) {
    case 1:
      o->dim = 2, o->degree = 2, o->cells = 32, o->jitter = 0.1;
      break;
    case 2:
      o->dim = 2, o->degree = 4, o->cells = 256, o->jitter = 0.05, o->coeff_kind = 1, o->block_cells = 8;
      o->n_levels = 4;
      o->levels[0] = 1.0, o->levels[1] = 10.0, o->levels[2] = 100.0, o->levels[3] = 1000.0;
      break;
    case 3:
      o->dim = 3, o->degree = 2, o->cells = 64, o->jitter = 0.1;
      break;
    case 4:
      o->physics = 1, o->dim = 2, o->degree = 2, o->cells = 512, o->coeff_kind = 2, o->coeff_value = 1.0;
      break;
    case 5:
      o->physics = 2, o->dim = 3, o->degree = 3, o->cells = 96, o->coeff_kind = 1, o->block_cells = 4;
      o->n_levels = 2, o->poisson_ratio = 0.3;
      o->levels[0] = 1.0, o->levels[1] = 100.0;
      break;
    default:
      return false;
  }
  if (cells > 0) o->cells = cells;
  return true;
}

}  // namespace pdb
