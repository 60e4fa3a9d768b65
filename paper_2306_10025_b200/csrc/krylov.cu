// Device Krylov drivers.  Vectors and the recurrence scalars stay in HBM;
// only the small Hessenberg / Givens recurrences and the convergence tests
// run on the host, with one host synchronisation per iteration (GMRES: the
// column of h_ij and ||w|| read in one copy; PCG: ||r||^2, with alpha and
// beta formed on the device).
//   gmres: reference gmres.cpp:27-169 (restarted GMRES(m), modified
//          Gram-Schmidt, Givens rotations, right preconditioning by default,
//          true residual at the end of each cycle).
//   pcg:   preconditioned CG (absent from the reference), the
//          same recurrence as oracle/pdb_oracle.c orc_pcg.
// Dots use the deterministic fixed-tree reduction of kernels/blas.cu.  The
// GMRES Gram-Schmidt sweep is one cooperative kernel per Arnoldi step
// (k::mgs_fused: the new vector stays in registers across the j + 2
// grid-wide reductions) instead of 3 (j + 1) + 2 launches; work vectors come
// from the stream-ordered pool, so a solve does no device-wide allocation.
#include <cfloat>
#include <cmath>

#include "host.hpp"
#include "kernels.hpp"

namespace pdb {

namespace {

struct Ops {
  const DeviceCsr& a;
  const pdb_precond_s* pc;
  cudaStream_t s;
  k::SpmvPlan plan;
  Scratch<double> partials;
  Scratch<double> scal;  // device scalars
  Ops(const DeviceCsr& a_, const pdb_precond_s* pc_, cudaStream_t s_, size_t nscal = 64)
      : a(a_), pc(pc_), s(s_), plan(plan_of(a_)), partials(static_cast<size_t>(k::dot_partials()), s_),
        scal(std::max<size_t>(nscal, 64), s_) {}
  void spmv(const double* x, double* y) {
    k::spmv(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), x, y, s);
  }
  void apply(const double* r, double* z) { precond_apply_device(*pc, r, z, s); }
  // dot into device scalar slot `slot`
  double* dot_dev(const double* x, const double* y, int slot) {
    k::dot(a.n, x, y, partials.get(), scal.get() + slot, s);
    return scal.get() + slot;
  }
  double dot(const double* x, const double* y) {
    double* d = dot_dev(x, y, 63);
    double h = 0.0;
    PDB_CUDA(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, s));
    sync(s);
    return h;
  }
  double norm(const double* x) { return std::sqrt(dot(x, x)); }
};

}  // namespace

void gmres_device(const DeviceCsr& a, const double* b_host, const pdb_precond_s* pc, const pdb_gmres_options& o,
                  double* x_host, pdb_report_s& rep, cudaStream_t s) {
  require_device();
  const int64_t n = a.n;
  require(o.restart >= 1, Errc::invalid_argument, "restart length must be >= 1");
  if (pc) require(pc->n == n, Errc::dimension_mismatch, "preconditioner does not match the matrix");
  Ops ops(a, pc, s, static_cast<size_t>(o.restart) + 2);
  const size_t un = static_cast<size_t>(std::max<int64_t>(n, 1));
  // pool (stream-ordered) allocations: no device-wide synchronisation per solve
  Scratch<double> b(un, s), x(un, s), r0(un, s), tmp(un, s), corr(un, s);
  b.upload(b_host, static_cast<size_t>(n));
  x.zero();
  rep = pdb_report_s();
  const double bnorm = ops.norm(b.get());
  if (bnorm == 0.0) {
    rep.converged = true;
    rep.final_relative_residual = 0.0;
    for (int64_t i = 0; i < n; ++i) x_host[i] = 0.0;
    return;
  }
  const bool left = o.left_precond != 0;
  auto apply_op = [&](const double* v, double* out) {
    if (!pc) {
      ops.spmv(v, out);
    } else if (left) {
      ops.spmv(v, tmp.get());
      ops.apply(tmp.get(), out);
    } else {
      ops.apply(v, tmp.get());
      ops.spmv(tmp.get(), out);
    }
  };
  auto true_relres = [&]() {
    ops.spmv(x.get(), corr.get());
    k::sub(n, b.get(), corr.get(), corr.get(), s);
    return ops.norm(corr.get()) / bnorm;
  };
  const size_t m = static_cast<size_t>(o.restart);
  Scratch<double> V((m + 1) * un, s);
  auto Vp = [&](size_t i) { return V.get() + i * un; };
  std::vector<std::vector<double>> h(m + 1, std::vector<double>(m, 0.0));
  std::vector<double> cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0), y(m, 0.0);
  bool first_cycle = true;
  for (;;) {
    if (first_cycle) {
      PDB_CUDA(cudaMemcpyAsync(r0.get(), b.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else {
      ops.spmv(x.get(), r0.get());
      k::sub(n, b.get(), r0.get(), r0.get(), s);
    }
    if (pc && left) {
      ops.apply(r0.get(), tmp.get());
      PDB_CUDA(cudaMemcpyAsync(r0.get(), tmp.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    const double beta = ops.norm(r0.get());
    if (first_cycle) rep.residual_history.push_back(beta);
    const double refnorm = rep.residual_history.front();
    if (beta == 0.0) {
      rep.converged = true;
      break;
    }
    k::div_scalar(n, r0.get(), beta, Vp(0), s);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    size_t steps = 0;
    bool breakdown = false;
    for (size_t j = 0; j < m; ++j) {
      apply_op(Vp(j), Vp(j + 1));
      // modified Gram-Schmidt: one cooperative kernel (vector in registers,
      // j + 2 grid-wide reductions), else per-i dot + axpy launches with h_ij
      // in device slot i feeding the axpy
      if (!k::mgs_fused(n, static_cast<int>(j), V.get(), static_cast<int64_t>(un), Vp(j + 1), ops.scal.get(), s)) {
        for (size_t i = 0; i <= j; ++i) {
          double* hij = ops.dot_dev(Vp(j + 1), Vp(i), static_cast<int>(i));
          k::axpy(n, hij, true, Vp(i), Vp(j + 1), s);
        }
        ops.dot_dev(Vp(j + 1), Vp(j + 1), static_cast<int>(j + 1));
      }
      std::vector<double> hv(j + 2);
      PDB_CUDA(cudaMemcpyAsync(hv.data(), ops.scal.get(), (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, s));
      sync(s);  // the iteration's only host synchronisation
      for (size_t i = 0; i <= j; ++i) h[i][j] = hv[i];
      const double hj1 = std::sqrt(hv[j + 1]);
      h[j + 1][j] = hj1;
      if (hj1 > 0.0) k::div_scalar(n, Vp(j + 1), hj1, Vp(j + 1), s);
      for (size_t i = 0; i < j; ++i) {
        const double t1 = cs[i] * h[i][j] + sn[i] * h[i + 1][j];
        const double t2 = -sn[i] * h[i][j] + cs[i] * h[i + 1][j];
        h[i][j] = t1;
        h[i + 1][j] = t2;
      }
      const double denom = std::hypot(h[j][j], h[j + 1][j]);
      cs[j] = h[j][j] / denom;
      sn[j] = h[j + 1][j] / denom;
      h[j][j] = denom;
      h[j + 1][j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++steps;
      ++rep.iterations;
      const double est = std::abs(g[j + 1]);
      rep.residual_history.push_back(std::max(est, DBL_MIN));
      if (hj1 == 0.0) {
        breakdown = true;
        break;
      }
      if (est <= o.tol * refnorm || rep.iterations >= o.max_iters) break;
    }
    for (size_t i = steps; i-- > 0;) {
      double sacc = g[i];
      for (size_t kk = i + 1; kk < steps; ++kk) sacc -= h[i][kk] * y[kk];
      y[i] = sacc / h[i][i];
    }
    tmp.zero();
    for (size_t i = 0; i < steps; ++i) k::axpy_val(n, y[i], Vp(i), tmp.get(), s);
    if (pc && !left) {
      ops.apply(tmp.get(), corr.get());
      k::axpy_val(n, 1.0, corr.get(), x.get(), s);
    } else {
      k::axpy_val(n, 1.0, tmp.get(), x.get(), s);
    }
    rep.final_relative_residual = true_relres();
    if (rep.final_relative_residual <= o.tol || breakdown) {
      rep.converged = rep.final_relative_residual <= o.tol || breakdown;
      break;
    }
    if (rep.iterations >= o.max_iters) break;
    ++rep.restarts;
    first_cycle = false;
  }
  rep.final_relative_residual = true_relres();
  x.download(x_host, static_cast<size_t>(n));
  sync(s);
}

// Reproducible PCG: the oracle's orc_pcg sequence bit for bit -- the bitwise
// SpMV, the patch solves in lu_solve_into's order (PDB_APPLY=lu factors), the
// ordered scatter, unfused axpys and the blocked inner products (chunks of
// 256 summed in order, chunk sums in groups of 256 in order, then the groups;
// oracle/pdb_oracle.c dot_blocked) -- so iteration counts and residual
// histories are identical to the CPU restatement's.  Host-driven (a few
// synchronisations per iteration): a verification mode, not the fast path.
static void pcg_reproducible(const DeviceCsr& a, const double* b_host, const pdb_precond_s* pc, double tol,
                             int64_t max_iters, double* x_host, pdb_report_s& rep, cudaStream_t s) {
  constexpr int kChunk = 256;
  const int64_t n = a.n;
  const size_t un = static_cast<size_t>(std::max<int64_t>(n, 1));
  const int64_t nch = (n + kChunk - 1) / kChunk;
  Scratch<double> b(un, s), x(un, s), r(un, s), z(un, s), p(un, s), q(un, s);
  Scratch<double> chunks(static_cast<size_t>(std::max<int64_t>(nch, 1)), s);
  std::vector<double> ch(static_cast<size_t>(std::max<int64_t>(nch, 1)));
  const k::SpmvPlan plan = plan_of(a);
  auto dotb = [&](const double* u, const double* v) {
    k::dot_chunks(n, kChunk, u, v, chunks.get(), s);
    PDB_CUDA(cudaMemcpyAsync(ch.data(), chunks.get(), nch * sizeof(double), cudaMemcpyDeviceToHost, s));
    sync(s);
    double total = 0.0;
    for (int64_t g0 = 0; g0 < nch; g0 += kChunk) {
      double gs = 0.0;
      for (int64_t c = g0; c < nch && c < g0 + kChunk; ++c) gs += ch[static_cast<size_t>(c)];
      total += gs;
    }
    return total;
  };
  auto precond = [&]() {
    if (pc) precond_apply_device(*pc, r.get(), z.get(), s, /*symmetric=*/true, /*reference_order=*/true);
    else PDB_CUDA(cudaMemcpyAsync(z.get(), r.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  };
  b.upload(b_host, static_cast<size_t>(n));
  x.zero();
  PDB_CUDA(cudaMemcpyAsync(r.get(), b.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  rep = pdb_report_s();
  const double bnorm = std::sqrt(dotb(b.get(), b.get()));
  if (bnorm == 0.0) {
    rep.converged = true;
  } else {
    rep.residual_history.push_back(1.0);
    precond();
    PDB_CUDA(cudaMemcpyAsync(p.get(), z.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    double rz = dotb(r.get(), z.get());
    while (rep.iterations < max_iters) {
      k::spmv(plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), p.get(), q.get(), s);
      const double alpha = rz / dotb(p.get(), q.get());
      k::axpy_ref(n, alpha, p.get(), x.get(), 0, s);
      k::axpy_ref(n, alpha, q.get(), r.get(), 1, s);
      ++rep.iterations;
      const double rel = std::sqrt(dotb(r.get(), r.get())) / bnorm;
      rep.residual_history.push_back(rel);
      if (rel <= tol) {
        rep.converged = true;
        break;
      }
      precond();
      const double rz_new = dotb(r.get(), z.get());
      const double beta = rz_new / rz;
      rz = rz_new;
      k::axpy_ref(n, beta, z.get(), p.get(), 2, s);
    }
  }
  PDB_LAUNCH_CHECK();
  rep.final_relative_residual = rep.residual_history.empty() ? 0.0 : rep.residual_history.back();
  x.download(x_host, static_cast<size_t>(n));
  sync(s);
}

void pcg_device(const DeviceCsr& a, const double* b_host, const pdb_precond_s* pc, double tol, int64_t max_iters,
                double* x_host, pdb_report_s& rep, cudaStream_t s, bool reproducible) {
  require_device();
  if (reproducible) {
    if (pc) require(pc->n == a.n, Errc::dimension_mismatch, "preconditioner does not match the matrix");
    pcg_reproducible(a, b_host, pc, tol, max_iters, x_host, rep, s);
    return;
  }
  const int64_t n = a.n;
  if (pc) require(pc->n == n, Errc::dimension_mismatch, "preconditioner does not match the matrix");
  Ops ops(a, pc, s);
  const size_t un = static_cast<size_t>(std::max<int64_t>(n, 1));
  Scratch<double> b(un, s), r(un, s), z(un, s), p(un, s), q(un, s);
  Scratch<double> xb[2] = {Scratch<double>(un, s), Scratch<double>(un, s)};  // x_k alternates buffers
  const int nparts = std::max(ops.plan.blocks, k::dot_partials());
  Scratch<double> part1(static_cast<size_t>(nparts), s), part2(static_cast<size_t>(nparts), s);
  b.upload(b_host, static_cast<size_t>(n));
  xb[0].zero();
  PDB_CUDA(cudaMemcpyAsync(r.get(), b.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  rep = pdb_report_s();
  const double bnorm = ops.norm(b.get());
  int xres = 0;  // buffer holding the returned iterate
  if (bnorm == 0.0) {
    rep.converged = true;
  } else {
    rep.residual_history.push_back(1.0);
    auto precond = [&]() {
      if (pc) precond_apply_device(*pc, r.get(), z.get(), s, /*symmetric=*/true);
      else PDB_CUDA(cudaMemcpyAsync(z.get(), r.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    };
    // device scalar slots; RR + (k & 1): the residual norms of two consecutive iterations
    constexpr int RZ = 0, ALPHA = 2, BETA = 5, RR = 6;
    double* sc = ops.scal.get();
    static thread_local double* rr_host = nullptr;  // pinned, 2 slots
    if (!rr_host) PDB_CUDA(cudaMallocHost(&rr_host, 2 * sizeof(double)));
    cudaEvent_t ev[2];
    for (auto& e : ev) PDB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    precond();
    PDB_CUDA(cudaMemcpyAsync(p.get(), z.get(), n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    k::dot_partial(n, r.get(), z.get(), part2.get(), s);
    k::finish_sum(part2.get(), k::dot_partials(), sc + RZ, false, s);
    // Iteration k: q = A p with (p, q) fused, alpha = rz / (p, q); x and r
    // updated with r.r fused; ||r||^2 copied to the host slot k & 1; then the
    // preconditioner, rz_new and p for iteration k + 1.  The host enqueues
    // iteration k + 1 before it reads the norm of iteration k, so the GPU never
    // waits for the convergence test; a converged solve returns x_{k+1}, kept
    // in its own buffer while the speculative iteration writes the other.
    auto enqueue = [&](int64_t k) {
      k::spmv_dot(ops.plan, a.n, a.row_ptr.get(), a.col.get(), a.val.get(), p.get(), q.get(), part1.get(), s);
      k::finish_ratio(part1.get(), ops.plan.blocks, sc + RZ, sc + ALPHA, false, s);
      k::cg_update(n, sc + ALPHA, p.get(), q.get(), xb[k & 1].get(), xb[(k + 1) & 1].get(), r.get(), part2.get(), s);
      k::finish_sum(part2.get(), k::dot_partials(), sc + RR + (k & 1), false, s);
      PDB_CUDA(cudaMemcpyAsync(rr_host + (k & 1), sc + RR + (k & 1), sizeof(double), cudaMemcpyDeviceToHost, s));
      PDB_CUDA(cudaEventRecord(ev[k & 1], s));
      precond();
      k::dot_partial(n, r.get(), z.get(), part1.get(), s);
      k::finish_ratio(part1.get(), k::dot_partials(), sc + RZ, sc + BETA, true, s);  // beta = rz_new / rz; rz = rz_new
      k::xpay(n, z.get(), sc + BETA, p.get(), s);
    };
    const char* la = getenv("PDB_PCG_LOOKAHEAD");
    const bool lookahead = !(la && la[0] == '0');
    int64_t enq = 0;
    if (max_iters > 0) enqueue(enq++);
    for (int64_t k = 0; k < enq; ++k) {
      if (lookahead && enq < max_iters) enqueue(enq++);
      PDB_CUDA(cudaEventSynchronize(ev[k & 1]));
      const double rr = rr_host[k & 1];
      ++rep.iterations;
      xres = static_cast<int>((k + 1) & 1);
      const double rel = std::sqrt(rr) / bnorm;
      rep.residual_history.push_back(rel);
      if (rel <= tol) {
        rep.converged = true;
        break;
      }
      if (!lookahead && enq < max_iters) enqueue(enq++);
    }
    sync(s);
    for (auto& e : ev) cudaEventDestroy(e);
  }
  rep.final_relative_residual = rep.residual_history.empty() ? 0.0 : rep.residual_history.back();
  xb[xres].download(x_host, static_cast<size_t>(n));
  sync(s);
}

}  // namespace pdb
