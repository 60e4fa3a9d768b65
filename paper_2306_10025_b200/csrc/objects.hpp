// Handle types behind the opaque pointers of include/patchdb/patchdb.h.
//
// Layout in HBM:
//   matrix    CSR, row_ptr int64[n+1], col int32[nnz], val fp64[nnz]
//   patchset  patches int32[np*ps] (ascending per patch), weights fp64[n]
//   database  reps / lu fp64[m*ps*ps] row-major (reference layout), piv int32[m*ps], phi int32[np]
//   precond   factors fp64[nf*ps*ps] COLUMN-major per factor (lane i reads L(i,j)/U(i,j) of
//             column j at consecutive addresses), piv int32[nf*ps], phi int32[np],
//             omega_w fp64[n], DOF->(patch,slot) inverse map inv_ptr int32[n+1], inv int32[np*ps]
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "common.hpp"

namespace pdb {

struct HostCsr {
  Index n = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col;
  std::vector<double> val;
  Index nnz() const { return static_cast<Index>(col.size()); }
};

struct DeviceCsr {
  Index n = 0;
  Index nnz = 0;
  DevBuf<int64_t> row_ptr;
  DevBuf<int32_t> col;
  DevBuf<double> val;
  // warp items of the CSR residual (v5): nitems + 1 row starts and row_ptr there
  DevBuf<int32_t> item_start;
  DevBuf<int64_t> item_base;
  int nitems = 0;
  // SELL-C-sigma copy (v9 residual): slices of 32 rows of similar length,
  // entry j of slice row l at sell_off[s] + 32 j + l; sell_row = {row, length}
  DevBuf<int64_t> sell_off;
  DevBuf<int32_t> sell_row;
  DevBuf<double> sell_val;
  DevBuf<int32_t> sell_col;
  int64_t nslices = 0;  // 0: not built
  // Column-pattern classes (build_sell): when every row's columns are
  // row + one of a few offset lists (structured FEM lattices: one list per
  // node type), no column indices are stored; sell_row.y packs
  // length | (class + 1) << 16 and the offsets sit in sell_tab.
  DevBuf<int32_t> sell_tab, sell_tstart;
  int64_t sell_classes = 0;  // 0: explicit columns
  // Half ("mirror") storage (sell_mirror.cpp): slices as above but holding
  // only each row's upper entries; lower entry m of a class-c row i reads
  // value mir_rbase[j] + mir_kslot[tstart[c] + m], j = i + offset (the row
  // that stores a_ji == a_ij).  mirror == false: the plain SELL layout above.
  bool mirror = false;
  DevBuf<int32_t> mir_clo, mir_rbase, mir_kslot;
  int64_t mir_virtual = 0;
  std::string mir_why;             // why the mirror layout is not in use
  std::vector<int64_t> win_slice;  // first slice of each kSellSigma-row window (+ end)
};

// Two-level coarse correction of the combo preconditioner (reference
// ComboPreconditioner, precond.cpp:103-121): P0 and R0 = P0^T as CSR, the
// banded LU of R0 A P0 in COLUMN-major band storage (column j holds band
// rows 0..ldab-1 of the reference's LAPACK-style layout, banded.cpp:11-60).
struct CoarseDev {
  Index fine_n = 0, nc = 0, kl = 0, ku = 0, ldab = 0;
  DevBuf<int32_t> p0_ptr, p0_col, r0_ptr, r0_col;
  DevBuf<double> p0_val, r0_val;
  DevBuf<double> band;   // [nc][ldab]
  DevBuf<int32_t> ipiv;  // absolute pivot row per column
  DevBuf<double> rdiag;  // 1 / U(j, j)
  DevBuf<double> inv;    // dense (R0 A P0)^{-1}, row-major [nc][ld], when ld > 0
  Index ld = 0;
  // blocked solve (nblk > 0): forward maps F_k [m_k][m_k] and backward maps
  // G_k [bk_k][bk_k + nr_k], row-major, concatenated at foff / goff
  Index bk = 0, nblk = 0, vmax = 0;
  DevBuf<int64_t> foff, goff;
  DevBuf<double> fblk, gblk;
};

struct BuildWork {
  int64_t pair_evals = 0;
  int64_t power_iters = 0;
  int64_t lu_count = 0;
};

}  // namespace pdb

struct pdb_problem_s {
  pdb::HostCsr a;
  std::vector<double> rhs;
  bool has_exact = false;
  std::vector<double> exact;  // manufactured solution (uniform-mesh assembler only)
  int dim = 2;
  int64_t cells = 0;
  int degree = 1;
  int components = 1;  // DoFs per lattice node (vector generators: > 1)
  // slab problems (pdb_problem_generate_slab): the global row ranges held,
  // the global size; a.n is the local row count, a.col holds global ids
  std::vector<std::pair<int64_t, int64_t>> row_ranges;
  int64_t n_global = 0;
  int slab_rank = 0, slab_ranks = 1;
  bool is_slab() const { return !row_ranges.empty(); }
};

struct pdb_matrix_s {
  pdb::DeviceCsr a;
};

struct pdb_patchset_s {
  int64_t n = 0;   // rows of the matrix it was detected on
  int64_t np = 0;  // patches
  int64_t ps = 0;  // patch size
  pdb::DevBuf<int32_t> patches;
  pdb::DevBuf<double> weights;
};

struct pdb_database_s {
  int64_t m = 0, np = 0, ps = 0;
  pdb::DevBuf<double> reps;
  pdb::DevBuf<double> lu;
  pdb::DevBuf<int32_t> piv;
  pdb::DevBuf<int32_t> phi;
  std::string method;
  double eps = 0.0;
  std::vector<std::vector<uint8_t>> entry_patterns;  // per entry, partitioned k-means only
  pdb::BuildWork work;
};

struct pdb_precond_s {
  int64_t n = 0, np = 0, ps = 0, nf = 0;
  double omega = 1.0;
  bool compressed = false;
  bool lu_apply = false;  // true: triangular solves on column-major LU; false: explicit inverses
  pdb::DevBuf<int32_t> patches;
  pdb::DevBuf<double> omega_w;
  pdb::DevBuf<double> sqrt_w;    // W^{1/2} and omega W^{1/2}: the symmetric weighting PCG uses
  pdb::DevBuf<double> omega_sw;
  pdb::DevBuf<double> factors;  // column-major per factor
  pdb::DevBuf<int32_t> piv;
  pdb::DevBuf<int32_t> phi;     // compressed mode only
  // cluster-grouped apply (compressed mode): patches sorted by entry, tiled
  pdb::DevBuf<int32_t> order, slot_of, tile_entry, tile_start, tile_idx;
  int ntiles = 0, max_tile = 0;
  pdb::DevBuf<double> frag;  // inverses in DMMA A-fragment order (tensor-core grouped apply), when allocated
  pdb::FragTensorMap frag_map{};  // TMA descriptor of frag (patches above 32 DoFs)
  bool has_frag_map = false;
  int maxc = 0;  // largest slot count when <= 8 and the weights are 1/count: the templated scatter
  pdb::DevBuf<int32_t> inv_ptr;
  pdb::DevBuf<int32_t> inv;
  std::shared_ptr<pdb::CoarseDev> coarse;  // combo preconditioner only
};

struct pdb_report_s {
  int64_t iterations = 0;
  int64_t restarts = 0;
  bool converged = false;
  double final_relative_residual = 0.0;
  std::vector<double> residual_history;
};
