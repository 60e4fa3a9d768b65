// Device assembly of the linear-elasticity element matrices (config 5) for
// the seeded generator (generator.cpp, generate_system with physics 2).
//
// One CTA per cell of a colour (cells of one colour share no DoF, so their
// additions into the CSR values never collide), colours launched in order on
// one stream.  Per cell: the corner Jacobian, its inverse and determinant at
// every quadrature point (thread per point), the physical basis gradients
// G[q][a][r] in shared memory (64 x 64 x 3 for Q3), then thread per node pair
// (a, b): the 3 x 3 component block summed over the quadrature points in
// order, added into the rows of a's components.  Compiled with --fmad=false
// and written in the host loop's expression order, so the values are bitwise
// the host assembly's (tests/test_generator_device.py); the pattern, the
// geometry, the coefficients and the right-hand side stay on the host.
#include <cstdlib>
#include <vector>

#include "host.hpp"

namespace pdb {

namespace {

constexpr int kAsmThreads = 256;
constexpr int kMaxRanges = 2;

struct AsmArgs {
  int d, p, ncomp, nloc, nq, ncorner, px, py, pz;
  int64_t C, nva, npa, cxn, cyn, czn;
  const double *X, *coef, *gref, *cgrad, *qw;
  double lam_f, mu_f;
  int64_t cell_lo, cell_hi;
  int nrng;
  int64_t rlo[kMaxRanges], rhi[kMaxRanges], roff[kMaxRanges];
  const int64_t* row_ptr;
  double* val;
  int* bad;
};

__device__ __forceinline__ int64_t local_row(const AsmArgs& a, int64_t g) {
  for (int k = 0; k < a.nrng; ++k)
    if (g >= a.rlo[k] && g < a.rhi[k]) return a.roff[k] + g - a.rlo[k];
  return -1;
}

__global__ void __launch_bounds__(kAsmThreads) elastic_cells_kernel(AsmArgs a) {
  extern __shared__ double sm[];
  const int d = a.d, nloc = a.nloc, nq = a.nq, nc = a.ncorner, ncomp = a.ncomp;
  double* G = sm;                                   // [nq][nloc][d]
  double* WQ = G + (size_t)nq * nloc * d;           // [nq]
  double* INV = WQ + nq;                            // [nq][9]
  __shared__ double Xc[8][3];
  const int64_t t = blockIdx.x;
  const int64_t cx = a.px + 2 * (t % a.cxn), cy = a.py + 2 * ((t / a.cxn) % a.cyn),
                cz = d == 3 ? a.pz + 2 * (t / (a.cxn * a.cyn)) : 0;
  const int64_t slow = d == 3 ? cz : cy;
  if (slow < a.cell_lo || slow > a.cell_hi) return;  // touches no window row (block-uniform)
  const int64_t cell = cx + a.C * (cy + a.C * cz);
  if (threadIdx.x < (unsigned)(nc * d)) {
    const int c = threadIdx.x / d, k = threadIdx.x % d;
    const int64_t v = (cx + (c & 1)) + a.nva * ((cy + ((c >> 1) & 1)) + a.nva * (cz + ((c >> 2) & 1)));
    Xc[c][k] = a.X[v * d + k];
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nq; q += kAsmThreads) {
    double J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // J[r][s] = dx_r / dxi_s
    for (int c = 0; c < nc; ++c) {
      const double* cg = a.cgrad + (size_t)(q * nc + c) * d;
      for (int r = 0; r < d; ++r)
        for (int s2 = 0; s2 < d; ++s2) J[r][s2] = __dadd_rn(J[r][s2], __dmul_rn(Xc[c][r], cg[s2]));
    }
    double inv[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, det;
    if (d == 2) {
      det = __dsub_rn(__dmul_rn(J[0][0], J[1][1]), __dmul_rn(J[0][1], J[1][0]));
      inv[0][0] = __ddiv_rn(J[1][1], det);
      inv[0][1] = __ddiv_rn(-J[0][1], det);
      inv[1][0] = __ddiv_rn(-J[1][0], det);
      inv[1][1] = __ddiv_rn(J[0][0], det);
    } else {
      const double c00 = __dsub_rn(__dmul_rn(J[1][1], J[2][2]), __dmul_rn(J[1][2], J[2][1]));
      const double c01 = __dsub_rn(__dmul_rn(J[1][2], J[2][0]), __dmul_rn(J[1][0], J[2][2]));
      const double c02 = __dsub_rn(__dmul_rn(J[1][0], J[2][1]), __dmul_rn(J[1][1], J[2][0]));
      det = __dadd_rn(__dadd_rn(__dmul_rn(J[0][0], c00), __dmul_rn(J[0][1], c01)), __dmul_rn(J[0][2], c02));
      inv[0][0] = __ddiv_rn(c00, det);
      inv[1][0] = __ddiv_rn(c01, det);
      inv[2][0] = __ddiv_rn(c02, det);
      inv[0][1] = __ddiv_rn(__dsub_rn(__dmul_rn(J[0][2], J[2][1]), __dmul_rn(J[0][1], J[2][2])), det);
      inv[1][1] = __ddiv_rn(__dsub_rn(__dmul_rn(J[0][0], J[2][2]), __dmul_rn(J[0][2], J[2][0])), det);
      inv[2][1] = __ddiv_rn(__dsub_rn(__dmul_rn(J[0][1], J[2][0]), __dmul_rn(J[0][0], J[2][1])), det);
      inv[0][2] = __ddiv_rn(__dsub_rn(__dmul_rn(J[0][1], J[1][2]), __dmul_rn(J[0][2], J[1][1])), det);
      inv[1][2] = __ddiv_rn(__dsub_rn(__dmul_rn(J[0][2], J[1][0]), __dmul_rn(J[0][0], J[1][2])), det);
      inv[2][2] = __ddiv_rn(__dsub_rn(__dmul_rn(J[0][0], J[1][1]), __dmul_rn(J[0][1], J[1][0])), det);
    }
    if (!(det > 0.0)) atomicOr(a.bad, 1);  // inverted cell (jitter too large)
    WQ[q] = __dmul_rn(a.qw[q], det);
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) INV[q * 9 + r * 3 + k] = inv[r][k];
  }
  __syncthreads();
  // G[q][a][r] = sum_k inv[k][r] * gref[q][a][k]  (grad_x = J^{-T} grad_xi)
  for (int e = threadIdx.x; e < nq * nloc; e += kAsmThreads) {
    const int q = e / nloc, an = e % nloc;
    const double* gx = a.gref + (size_t)(q * nloc + an) * d;
    const double* iv = INV + q * 9;
    for (int r = 0; r < d; ++r) {
      double s2 = 0.0;
      for (int k = 0; k < d; ++k) s2 = __dadd_rn(s2, __dmul_rn(iv[k * 3 + r], gx[k]));
      G[(size_t)e * d + r] = s2;
    }
  }
  __syncthreads();
  const double cc = a.coef[cell];
  const double lam = __dmul_rn(a.lam_f, cc), mu = __dmul_rn(a.mu_f, cc);
  const int nl1 = a.p + 1;
  for (int pr = threadIdx.x; pr < nloc * nloc; pr += kAsmThreads) {
    const int an = pr / nloc, bn = pr % nloc;
    // row node (an) and its lattice / pattern range
    const int ax = an % nl1, ay = (an / nl1) % nl1, az = d == 3 ? an / (nl1 * nl1) : 0;
    const int64_t l0 = cx * a.p + ax, l1 = cy * a.p + ay, l2 = d == 3 ? cz * a.p + az : 0;
    bool boundary = l0 == 0 || l0 == a.npa - 1 || l1 == 0 || l1 == a.npa - 1;
    if (d == 3) boundary = boundary || l2 == 0 || l2 == a.npa - 1;
    if (boundary) continue;  // identity rows (fem.cpp:323)
    const int64_t gv = l0 + a.npa * (l1 + a.npa * l2);
    int64_t li[3];
    bool any = false;
    for (int c = 0; c < ncomp; ++c) {
      li[c] = local_row(a, ncomp * gv + c);
      any = any || li[c] >= 0;
    }
    if (!any) continue;
    double acc[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int q = 0; q < nq; ++q) {
      const double* Ga = G + ((size_t)q * nloc + an) * d;
      const double* Gb = G + ((size_t)q * nloc + bn) * d;
      double dot = 0.0;
      for (int r = 0; r < d; ++r) dot = __dadd_rn(dot, __dmul_rn(Ga[r], Gb[r]));
      const double wq = WQ[q];
      for (int c = 0; c < ncomp; ++c)
        for (int e2 = 0; e2 < ncomp; ++e2) {
          double v = __dadd_rn(__dmul_rn(__dmul_rn(lam, Ga[c]), Gb[e2]), __dmul_rn(__dmul_rn(mu, Ga[e2]), Gb[c]));
          if (c == e2) v = __dadd_rn(v, __dmul_rn(mu, dot));
          acc[c][e2] = __dadd_rn(acc[c][e2], __dmul_rn(wq, v));
        }
    }
    // column node (bn) offset inside the row's tensor range
    int64_t lo[3], w[3];
    const int64_t lrow[3] = {l0, l1, l2};
    for (int k = 0; k < 3; ++k) {
      if (k >= d) {
        lo[k] = 0;
        w[k] = 1;
        continue;
      }
      const int64_t cmin = lrow[k] == 0 ? 0 : (lrow[k] - 1) / a.p;
      const int64_t cmax = min((int64_t)(a.C - 1), lrow[k] / a.p);
      lo[k] = cmin * a.p;
      w[k] = (cmax - cmin) * a.p + a.p + 1;
    }
    const int bx = bn % nl1, by = (bn / nl1) % nl1, bz = d == 3 ? bn / (nl1 * nl1) : 0;
    const int64_t j0 = cx * a.p + bx, j1 = cy * a.p + by, j2 = d == 3 ? cz * a.p + bz : 0;
    const int64_t off = ((j0 - lo[0]) + w[0] * ((j1 - lo[1]) + w[1] * (j2 - lo[2]))) * ncomp;
    for (int c = 0; c < ncomp; ++c) {
      if (li[c] < 0) continue;
      double* row = a.val + a.row_ptr[li[c]] + off;
      for (int e2 = 0; e2 < ncomp; ++e2) row[e2] = __dadd_rn(row[e2], acc[c][e2]);
    }
  }
}

bool elastic_device(const ElasticAssembly& ea) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return false;
  }
  if (ea.ranges.size() > (size_t)kMaxRanges || ea.ncomp > 3 || ea.d > 3) return false;
  const size_t smem = ((size_t)ea.nq * ea.nloc * ea.d + ea.nq + (size_t)ea.nq * 9) * sizeof(double);
  if (smem > 200 * 1024) return false;
  cudaStream_t s = cudaStreamPerThread;
  const int64_t nr = ea.ranges.empty() ? 0 : [&] {
    int64_t r = 0;
    for (const auto& g : ea.ranges) r += g.second - g.first;
    return r;
  }();
  auto up = [&](const double* h, size_t n) {
    DevBuf<double> b(n);
    b.upload(h, n, s);
    return b;
  };
  const int64_t nv = ea.d == 3 ? ea.nva * ea.nva * ea.nva : ea.nva * ea.nva;
  const int64_t ncells = ea.d == 3 ? ea.C * ea.C * ea.C : ea.C * ea.C;
  DevBuf<double> X = up(ea.X, (size_t)(nv * ea.d)), coef = up(ea.coef, (size_t)ncells);
  DevBuf<double> gref = up(ea.gref, (size_t)ea.nq * ea.nloc * ea.d);
  DevBuf<double> cgrad = up(ea.cgrad, (size_t)ea.nq * ea.ncorner * ea.d), qw = up(ea.qw, (size_t)ea.nq);
  DevBuf<int64_t> rp((size_t)(nr + 1));
  rp.upload(ea.row_ptr, (size_t)(nr + 1), s);
  DevBuf<double> val((size_t)std::max<int64_t>(ea.nnz, 1));
  if (ea.nnz > 0) val.upload(ea.val, (size_t)ea.nnz, s);  // zeros and the Dirichlet identity rows' 1.0
  DevBuf<int> bad(1);
  PDB_CUDA(cudaMemsetAsync(bad.get(), 0, sizeof(int), s));
  AsmArgs a{};
  a.d = ea.d, a.p = ea.p, a.ncomp = ea.ncomp, a.nloc = ea.nloc, a.nq = ea.nq, a.ncorner = ea.ncorner;
  a.C = ea.C, a.nva = ea.nva, a.npa = ea.npa;
  a.X = X.get(), a.coef = coef.get(), a.gref = gref.get(), a.cgrad = cgrad.get(), a.qw = qw.get();
  a.lam_f = ea.lam_f, a.mu_f = ea.mu_f, a.cell_lo = ea.cell_lo, a.cell_hi = ea.cell_hi;
  a.nrng = (int)ea.ranges.size();
  int64_t off = 0;
  for (int k = 0; k < a.nrng; ++k) {
    a.rlo[k] = ea.ranges[(size_t)k].first;
    a.rhi[k] = ea.ranges[(size_t)k].second;
    a.roff[k] = off;
    off += a.rhi[k] - a.rlo[k];
  }
  a.row_ptr = rp.get(), a.val = val.get(), a.bad = bad.get();
  PDB_CUDA(cudaFuncSetAttribute(elastic_cells_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int ncolors = 1 << ea.d;
  for (int color = 0; color < ncolors; ++color) {
    a.px = color & 1, a.py = (color >> 1) & 1, a.pz = (color >> 2) & 1;
    a.cxn = (ea.C - a.px + 1) / 2, a.cyn = (ea.C - a.py + 1) / 2, a.czn = ea.d == 3 ? (ea.C - a.pz + 1) / 2 : 1;
    const int64_t ncol = a.cxn * a.cyn * a.czn;
    if (ncol > 0) elastic_cells_kernel<<<(unsigned)ncol, kAsmThreads, smem, s>>>(a);
    PDB_LAUNCH_CHECK();
  }
  int bh = 0;
  PDB_CUDA(cudaMemcpyAsync(&bh, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  PDB_CUDA(cudaMemcpyAsync(ea.val, val.get(), (size_t)ea.nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
  sync(s);
  require(bh == 0, Errc::invalid_argument, "generator: inverted cell (jitter too large)");
  return true;
}

struct Register {
  Register() { g_elastic_device_hook = &elastic_device; }
} register_hook;

}  // namespace

}  // namespace pdb
