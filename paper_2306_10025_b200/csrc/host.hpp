// Host orchestration entry points shared between the C-ABI (capi.cpp) and
// the per-subsystem sources.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/patchdb/patchdb.h"
#include "kernels.hpp"
#include "objects.hpp"

struct pdb_shard_s;
struct pdb_slab_s;
struct pdb_comm_s;
struct pdb_shard_plan_s;

namespace pdb {

// matrix.cpp
void upload_csr(const HostCsr& h, DeviceCsr& d, cudaStream_t s);
// the two halves of upload_csr for callers that fill d's arrays themselves:
// allocation (with the kernels' tail padding), then the residual structures
// (warp items, SELL copy; h is read only by the opt-in host SELL build)
void alloc_csr(Index n, Index nnz, DeviceCsr& d, cudaStream_t s);
// host -> device copy of a large pageable array through pinned staging buffers (synchronous)
void h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t s);
void finish_csr(const HostCsr& h, const std::vector<int64_t>& row_ptr, DeviceCsr& d, cudaStream_t s);
HostCsr validated_csr(Index n, const int64_t* rp, const int64_t* ci, const double* v);
HostCsr download_csr(const DeviceCsr& d, cudaStream_t s);
void spmv_device(const DeviceCsr& a, const double* x, double* y, cudaStream_t s);
k::SpmvPlan plan_of(const DeviceCsr& a);  // SpMV launch plan (streaming partition when available)
// Column-pattern classes of the SELL copy (every row's columns are row + one
// of a few offset lists); false when the rows do not share patterns.
bool sell_classes(const HostCsr& h, std::vector<int32_t>& cls, std::vector<int32_t>& tab, std::vector<int32_t>& tstart);
// sell_build.cu: the same SELL copy built on the device from d's CSR arrays
void build_sell_device(DeviceCsr& d, cudaStream_t s);

// sell_mirror.cpp: the half-storage residual layout (see there).
struct MirrorHost {
  int64_t nslices = 0;
  std::vector<int64_t> soff;       // per slice: value index of (slot 0, lane 0)
  std::vector<int32_t> rows;       // per slice lane: row (-1: padding), length | (class + 1) << 16
  std::vector<double> val;
  std::vector<int32_t> clo;        // per class: lower (mirrored) entries
  std::vector<int32_t> rbase;      // per row: value index of its slot 0
  std::vector<int32_t> kslot;      // per class offset (tab index): 32 * slot of the mirrored value
  std::vector<int64_t> win_slice;  // first slice per window (+ end)
  int64_t virtual_rows = 0;
  std::string why;                 // reason when not built
};
bool build_mirror_host(const HostCsr& h, const std::vector<int32_t>& cls, const std::vector<int32_t>& tab,
                       const std::vector<int32_t>& tstart, int64_t sigma, MirrorHost& out);
void mirror_spmv_host(const MirrorHost& m, const std::vector<int32_t>& tab, const std::vector<int32_t>& tstart,
                      const double* x, double* y);
HostCsr read_matrix_market_host(const std::string& path);
void write_matrix_market_host(const HostCsr& a, const std::string& path);

// generator.cpp
// Rows a generator assembles: sorted disjoint global ranges [lo, hi), and the
// cells along the slowest axis that touch them (inclusive).  Default: all.
struct RowWindow {
  std::vector<std::pair<Index, Index>> ranges;
  Index cell_lo = 0, cell_hi = INT64_MAX;
  Index rows() const {
    Index r = 0;
    for (const auto& g : ranges) r += g.second - g.first;
    return r;
  }
  Index global(Index li) const {
    for (const auto& g : ranges) {
      if (li < g.second - g.first) return g.first + li;
      li -= g.second - g.first;
    }
    return -1;
  }
  Index local(Index gi) const {
    Index off = 0;
    for (const auto& g : ranges) {
      if (gi >= g.first && gi < g.second) return off + gi - g.first;
      off += g.second - g.first;
    }
    return -1;
  }
};
// win == nullptr: the whole problem.  Otherwise only the window's rows, with
// global column ids, bitwise equal to the same rows of the whole problem
// (cells are assembled colour by colour in the same order; skipping cells
// that touch no window row removes no contribution to a window row).
void generate_scalar(const pdb_gen_options& o, pdb_problem_s& out, const RowWindow* win = nullptr);
// physics 1 (Stokes Q_p-Q_{p-1}, 2D) and 2 (linear elasticity): node-major vector DoFs
void generate_system(const pdb_gen_options& o, pdb_problem_s& out, const RowWindow* win = nullptr);
// Device assembly of the elasticity element matrices (generator_dev.cu).  The
// generator (host C++, also built into the CUDA-free libpdbgen.so) calls it
// through this hook, which libpatchdb sets when it loads; it returns false
// (host assembly) when no device is usable.  Same per-entry operation order
// as the host loop (colour by colour, cells of a colour sharing no DoF, the
// element sums over quadrature points in order, no FMA): bitwise equal.
struct ElasticAssembly {
  int d, p, ncomp, nloc, nq, ncorner;
  Index C, nva, npa;
  const double *X, *coef, *gref, *cgrad, *qw;  // host tables
  double lam_f, mu_f;
  Index cell_lo, cell_hi;                       // slowest-axis cells touching the rows
  std::vector<std::pair<Index, Index>> ranges;  // global row ranges held (local = concatenation)
  const int64_t* row_ptr;                       // host, local rows + 1
  double* val;                                  // host, filled (nnz)
  Index nnz;
};
using ElasticHook = bool (*)(const ElasticAssembly&);
extern ElasticHook g_elastic_device_hook;

// Slab of rank r of W along the slowest axis: cells [C r / W, C (r+1) / W);
// the rows are every DoF of those cells (both faces included).
RowWindow slab_window(const pdb_gen_options& o, int rank, int nranks);
// Rows of the DoFs of the cells [c0, c1) along the slowest axis.
RowWindow cells_window(const pdb_gen_options& o, Index c0, Index c1);
// pdb_gen_options defaults and the BASELINE config presets (false: config not in 1..5)
void gen_options_defaults(pdb_gen_options* o);
bool gen_options_preset(int config, int64_t cells, pdb_gen_options* o);

// model_problem.cpp -- the reference's uniform-mesh model problems and the
// two-level coarse space (pdb_problem_assemble, pdb_precond_create_combo)
struct ModelConfig {
  int dim = 2;
  Index cells = 60;
  int degree = 2;
  std::string kind;  // "", "constant", "smooth", "piecewise"
  double value = 1.0;
  Index blocks_x = 4, blocks_y = 4;
  std::vector<double> block_values;
  int experiment = 1;
  enum Coeff { Constant, Smooth, Piecewise } coeff = Constant;
};
ModelConfig parse_model_config(const std::string& json);
// An explicit coefficient.kind wins, else `fallback` ("constant" for
// pdb_problem_assemble, "smooth"/"piecewise" by experiment for export).
void resolve_model_coefficient(ModelConfig& m, const char* fallback = "constant");
void assemble_model_problem(const ModelConfig& m, pdb_problem_s& out);
double model_l2_error(const pdb_problem_s& p, const double* u);
// Rectangular CSR operator (rows x cols).
struct CoarseOp {
  Index rows = 0, cols = 0;
  std::vector<int64_t> ptr;
  std::vector<int32_t> col;
  std::vector<double> val;
};
struct CoarseSpaceHost {
  CoarseOp p0;      // fine DoFs x coarse vertices (bilinear interpolation)
  CoarseOp r0;      // P0^T, rows in ascending fine order
  CoarseOp coarse;  // R0 A P0
};
CoarseSpaceHost build_coarse_space(const pdb_problem_s& p);

// coarse.cu -- device coarse correction z += P0 (R0 A P0)^{-1} R0 r
void coarse_setup(const CoarseSpaceHost& cs, pdb::CoarseDev& out, cudaStream_t s);
void coarse_correct(const pdb::CoarseDev& c, const double* r, double* z, cudaStream_t s);

// patchset.cpp
void detect_patches(const DeviceCsr& a, Index ps, pdb_patchset_s& out, cudaStream_t s);
void extract_patches(const DeviceCsr& a, const pdb_patchset_s& ps, DevBuf<double>& mats, cudaStream_t s);
std::vector<int64_t> patches_host(const pdb_patchset_s& ps, cudaStream_t s);
void write_patchset_json(const pdb_patchset_s& ps, const std::string& path, cudaStream_t s);

// database.cpp
// A communicator for the sharded setup (k-means assignment split across ranks).
struct ShardComm {
  struct ncclComm* comm = nullptr;
  int rank = 0, nranks = 1;
};

pdb_comm_s* comm_create(const unsigned char* id128, int rank, int nranks);
void comm_delete(pdb_comm_s* c);
const ShardComm& comm_of(const pdb_comm_s* c);

struct BuildParams {
  int method = PDB_METHOD_GREEDY_L1;
  double eps = 1e-7;
  int64_t db_size = 0;
  uint64_t seed = 42;
  int max_iters = 50;
  bool best_match = false;
  int64_t abort_above = -1;  // greedy only
  const ShardComm* comm = nullptr;  // k-means: patches' assignment sharded over comm->nranks ranks
};
// Returns false when a capped greedy pass aborted (no database).
bool build_database(const DeviceCsr& a, const pdb_patchset_s& ps, const BuildParams& p, pdb_database_s& out,
                    cudaStream_t s);
bool build_database_from_mats(const DevBuf<double>& mats, int64_t np, int64_t ps, const BuildParams& p,
                              pdb_database_s& out, cudaStream_t s);
double bisect_database(const DeviceCsr& a, const pdb_patchset_s& ps, const BuildParams& p, int64_t lo, int64_t hi,
                       pdb_database_s& out, cudaStream_t s);
void import_database(const std::string& json_path, const std::string& bin_path, pdb_database_s& db, cudaStream_t s);
double database_objective(const DeviceCsr& a, const pdb_patchset_s& ps, const pdb_database_s& db, double beta,
                          cudaStream_t s);
void compressibility_curve(const DeviceCsr& a, const pdb_patchset_s& ps, bool spectral, const double* grid,
                           int64_t count, int64_t* sizes, double* ratios, cudaStream_t s);
void export_database(const pdb_database_s& db, const std::string& json_path, const std::string& bin_path,
                     cudaStream_t s);

// database.cu: the reference's lu_factor failure text (dense.cpp:59-61)
std::string singular_msg(int32_t status, double best);
// split_budget (compress.cpp:336-392): the k-means budget per boundary partition
std::vector<int64_t> split_budget(int64_t m_p, const std::vector<int64_t>& sizes);

// precond.cpp
void precond_exact(const DeviceCsr& a, const pdb_patchset_s& ps, double omega, pdb_precond_s& out, cudaStream_t s);
void precond_compressed(const pdb_patchset_s& ps, const pdb_database_s& db, double omega, pdb_precond_s& out,
                        cudaStream_t s);
void precond_compressed_shard(const pdb_patchset_s& ps, const pdb_database_s& db, double omega, pdb_precond_s& out,
                              cudaStream_t s);
void patch_stage(const pdb_precond_s& pc, const double* r, const double* in_scale, double* sols, cudaStream_t s);
// DoF -> (patch, slot) map of pc.patches (inv_ptr / inv, ascending patch), plus the padded copy
void build_inverse(pdb_precond_s& pc, cudaStream_t s, const int32_t* slot_of = nullptr);
void common_setup(const pdb_patchset_s& ps, double omega, pdb_precond_s& pc, cudaStream_t s);
// z = M^{-1} r on device pointers (symmetric: omega W^1/2 S W^1/2, used by PCG).
// reference_order: the patch solves in lu_solve_into's order (reproducible PCG; needs lu_apply)
void precond_apply_device(const pdb_precond_s& pc, const double* r, double* z, cudaStream_t s,
                          bool symmetric = false, bool reference_order = false);
// sweeps of smooth(); history (device, may be null) gets sweeps+1 norms.
void relax_device(const DeviceCsr& a, const pdb_precond_s& pc, const double* b, double* x, int64_t sweeps,
                  double* history, cudaStream_t s);
// Same sweeps with CUDA events around each kernel: ms_phase[3] = average ms of
// residual, patch_solve, scatter_update.
void relax_host(const DeviceCsr& a, const pdb_precond_s& pc, const double* b_h, double* x_h, int64_t sweeps,
                double* history_h, cudaStream_t s);
void relax_profile(const DeviceCsr& a, const pdb_precond_s& pc, const double* b, double* x, int64_t sweeps,
                   double* ms_phase, cudaStream_t s);

// shard_plan.cpp -- slab partition of the sweep (host-only planning)
struct ShardPlan {
  int rank = 0, nranks = 1;
  Index k0 = 0, k1 = 0;              // local patch range (global patch ids)
  std::vector<int64_t> dofs;         // local index -> global DoF (ascending)
  std::vector<int64_t> rp;           // local CSR (rows = local DoFs; non-patch rows empty)
  std::vector<int32_t> ci;
  std::vector<double> val;
  std::vector<int32_t> patches;      // local patch DoF lists (local indices)
  std::vector<double> weights;       // global overlap weights at local DoFs
  std::vector<int32_t> owned;        // local indices of owned DoFs (ascending)
  std::vector<int32_t> up, up_peer;  // interface partials sent to the owner: local idx, destination rank
  std::vector<int32_t> pin, pin_peer;  // interface partials received: local idx (owned), source rank
  std::vector<int32_t> xs, xs_peer;  // x halo sent: local idx (owned), destination rank
  std::vector<int32_t> xr, xr_peer;  // x halo received: local idx, source rank
};
ShardPlan plan_shard(Index n, const int64_t* rp, const int32_t* ci, const double* val, Index np, Index ps,
                     const int32_t* patches, const double* weights, int rank, int nranks);
}  // namespace pdb
struct pdb_shard_plan_s {
  pdb::ShardPlan p;
};
namespace pdb {
// shard.cu (pdb_shard_s is defined there: it holds the NCCL communicator)
pdb_shard_s* shard_new();
void shard_delete(pdb_shard_s* sh);
int64_t shard_local_size(const pdb_shard_s& sh);
const ShardPlan& shard_plan(const pdb_shard_s& sh);
void comm_unique_id(unsigned char* id128);
void shard_create(const HostCsr& A, const pdb_patchset_s& gps, const pdb_database_s* db, double omega, int rank,
                  int nranks, pdb_shard_s& sh, cudaStream_t s);
void shard_attach(pdb_shard_s& sh, const unsigned char* id);
void shard_relax(pdb_shard_s& sh, const double* b, double* x, int64_t sweeps, cudaStream_t s);

// krylov.cpp
void gmres_device(const DeviceCsr& a, const double* b_host, const pdb_precond_s* pc, const pdb_gmres_options& o,
                  double* x_host, pdb_report_s& rep, cudaStream_t s);
// reproducible: the oracle's orc_pcg sequence bit for bit (verification mode)
void pcg_device(const DeviceCsr& a, const double* b_host, const pdb_precond_s* pc, double tol, int64_t max_iters,
                double* x_host, pdb_report_s& rep, cudaStream_t s, bool reproducible = false);

// slab.cu -- multi-GPU sweep shards with rank-local data
struct SlabRank;
// emulated: one state per rank in `ranks` (all ranks, or a subset whose absent
// neighbours' messages are empty -- single-GPU slices of a larger job)
pdb_slab_s* slab_new(int rank, int nranks, bool emulated, const std::vector<int>& ranks = {});
void slab_delete(pdb_slab_s* g);
void slab_attach(pdb_slab_s& g, const unsigned char* id128);
// db: replicated database (phi sliced by the global patch offset); build:
// construct the compressed database from the ranks' own patches instead
// (greedy-l1); neither: exact factors of the local patches.
void slab_setup(pdb_slab_s& g, std::vector<pdb_problem_s*>& probs, int64_t patch_size, const pdb_database_s* db,
                double omega, cudaStream_t s, const BuildParams* build = nullptr);
int64_t slab_database_size(const pdb_slab_s& g);
void slab_phi(const pdb_slab_s& g, int i, int64_t* out);
void slab_creators(const pdb_slab_s& g, int64_t* out);
void slab_relax(pdb_slab_s& g, const std::vector<const double*>& b, const std::vector<double*>& x, int64_t sweeps,
                cudaStream_t s);
// per local rank i: sizes / lists for the C-ABI getters
struct SlabInfo {
  int rank, nranks;
  int64_t n_local, n_rows, n_patches, first_patch, split, n_owned, n_up, n_pin, n_xs, n_xr;
};
SlabInfo slab_info(const pdb_slab_s& g, int i);
void slab_local_dofs(const pdb_slab_s& g, int i, int64_t* out);
void slab_owned(const pdb_slab_s& g, int i, int64_t* out);
int slab_local_ranks(const pdb_slab_s& g);
double slab_upload_seconds(const pdb_slab_s& g);  // matrix upload + residual structures inside the setup
void slab_relax_one(pdb_slab_s& g, int i, const double* b, double* x, int64_t sweeps, cudaStream_t s);
}  // namespace pdb
