"""C-ABI contract checks that need no GPU: exported symbols, struct layouts,
defaults, NULL handling and status strings (reference capi.cpp:37-430,
patchdb.h:25-168), and the loud no-device failure of compute entry points."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "patchdb", "patchdb.h")
LIB = os.path.join(ROOT, "paper_2306_10025_b200", "lib", "libpatchdb.so.0")

# The 44 symbols the reference library exports (nm -D of libpatchdb.so.0.1.0,
# SURVEY.md §8b); the drop-in must export every one of them.
REFERENCE_SYMBOLS = """
pdb_status_string pdb_last_error pdb_matrix_read_matrix_market pdb_matrix_write_matrix_market pdb_matrix_rows
pdb_matrix_nnz pdb_matrix_spmv pdb_matrix_free pdb_problem_assemble pdb_problem_ndofs pdb_problem_matrix
pdb_problem_rhs pdb_problem_exact_solution pdb_problem_l2_error pdb_problem_free pdb_patchset_detect
pdb_patchset_count pdb_patchset_patch_size pdb_patchset_write_json pdb_patchset_free pdb_compress_options_init
pdb_database_build pdb_database_size pdb_database_n_patches pdb_database_phi pdb_database_export pdb_database_free
pdb_precond_create pdb_precond_create_combo pdb_precond_apply pdb_precond_free pdb_gmres_options_init
pdb_gmres_solve pdb_report_iterations pdb_report_restarts pdb_report_converged pdb_report_final_relative_residual
pdb_report_residual_history_size pdb_report_residual_history pdb_report_free pdb_run_experiment pdb_run_analyze
pdb_run_benchmark pdb_export_matrix
""".split()


def exported():
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if line.strip()}


def declared():
    text = open(HEADER).read()
    return set(re.findall(r"PDB_API[^;(]*?\b(pdb_\w+)\s*\(", text))


def test_reference_symbol_count():
    assert len(REFERENCE_SYMBOLS) == 44


def test_exports_every_declared_symbol_and_nothing_else():
    ex = exported()
    decl = declared()
    assert set(REFERENCE_SYMBOLS) <= decl
    assert decl <= ex, sorted(decl - ex)
    assert all(s.startswith("pdb_") for s in ex), sorted(s for s in ex if not s.startswith("pdb_"))


def test_soname():
    out = subprocess.run(["readelf", "-d", LIB], capture_output=True, text=True, check=True).stdout
    assert "Library soname: [libpatchdb.so.0]" in out


def test_struct_layouts(P):
    O = P.CompressOptions
    assert C.sizeof(O) == 48
    assert [getattr(O, f).offset for f in ("method", "eps", "db_size", "seed", "max_iters", "best_match",
                                           "threads")] == [0, 8, 16, 24, 32, 36, 40]
    G = P.GmresOptions
    assert C.sizeof(G) == 32
    assert [getattr(G, f).offset for f in ("restart", "tol", "max_iters", "left_precond", "threads")] == \
        [0, 8, 16, 24, 28]


def test_option_defaults(P):
    o = P.CompressOptions()
    P.lib.pdb_compress_options_init(C.byref(o))
    assert (o.method, o.eps, o.db_size, o.seed, o.max_iters, o.best_match, o.threads) == \
        (P.GREEDY_L1, 1e-7, 0, 42, 50, 0, 1)  # capi.cpp:238-247
    g = P.GmresOptions()
    P.lib.pdb_gmres_options_init(C.byref(g))
    assert (g.restart, g.tol, g.max_iters, g.left_precond, g.threads) == (20, 1e-8, 2000, 0, 1)  # :346-353
    P.lib.pdb_compress_options_init(None)  # NULL is ignored
    P.lib.pdb_gmres_options_init(None)


def test_status_strings(P):
    want = ["ok", "invalid argument", "dimension mismatch", "singular matrix", "index out of range",
            "duplicate index", "parse error", "non-square matrix", "no patches found", "empty cluster",
            "budget too small", "invalid degree", "non-positive coefficient", "io error", "internal error"]
    assert [P.lib.pdb_status_string(i).decode() for i in range(15)] == want
    assert P.lib.pdb_status_string(99).decode() == "unknown status"


def test_null_handling(P):
    L = P.lib
    for getter in (L.pdb_matrix_rows, L.pdb_matrix_nnz, L.pdb_patchset_count, L.pdb_patchset_patch_size,
                   L.pdb_database_size, L.pdb_database_n_patches, L.pdb_report_iterations, L.pdb_report_restarts,
                   L.pdb_report_converged, L.pdb_report_residual_history_size, L.pdb_problem_ndofs):
        assert getter(None) == 0
    assert L.pdb_report_final_relative_residual(None) == 0.0
    for free in (L.pdb_matrix_free, L.pdb_patchset_free, L.pdb_database_free, L.pdb_precond_free,
                 L.pdb_report_free, L.pdb_problem_free):
        free(None)
    out = C.c_void_p()
    assert L.pdb_matrix_spmv(None, None, None) == P.PDB_ERR_INVALID_ARGUMENT
    assert L.pdb_last_error().decode() == "null argument"
    assert L.pdb_patchset_detect(None, 9, C.byref(out)) == P.PDB_ERR_INVALID_ARGUMENT
    assert L.pdb_precond_create(None, None, None, 1.0, 1, C.byref(out)) == P.PDB_ERR_INVALID_ARGUMENT
    assert L.pdb_database_phi(None, None) == P.PDB_ERR_INVALID_ARGUMENT
    assert L.pdb_gmres_solve(None, None, None, None, None, None) == P.PDB_ERR_INVALID_ARGUMENT


def test_matrix_market_parse_errors_before_device(P, tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("not a banner\n")
    with pytest.raises(P.PatchdbError) as e:
        P.Matrix.read_matrix_market(str(bad))
    assert e.value.status == P.PDB_ERR_PARSE
    assert e.value.message == f"{bad}: line 1: missing %%MatrixMarket banner"
    rect = tmp_path / "rect.mtx"
    rect.write_text("%%MatrixMarket matrix coordinate real general\n2 3 0\n")
    with pytest.raises(P.PatchdbError) as e:
        P.Matrix.read_matrix_market(str(rect))
    assert e.value.status == P.PDB_ERR_NON_SQUARE_MATRIX
    with pytest.raises(P.PatchdbError) as e:
        P.Matrix.read_matrix_market(str(tmp_path / "missing.mtx"))
    assert e.value.status == P.PDB_ERR_IO


def test_csr_validation_errors(P):
    import numpy as np
    with pytest.raises(P.PatchdbError) as e:
        P.Matrix.from_csr(np.array([0, 1]), np.array([5]), np.array([1.0]))
    assert e.value.status == P.PDB_ERR_INDEX_OUT_OF_RANGE
    with pytest.raises(P.PatchdbError) as e:
        P.Matrix.from_csr(np.array([0, 2, 2]), np.array([1, 0]), np.array([1.0, 2.0]))
    assert e.value.status == P.PDB_ERR_INVALID_ARGUMENT


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", None) is None and
                    os.path.exists("/dev/nvidia0"), reason="a GPU is present")
def test_no_cpu_fallback(P):
    """Without a device every compute entry point fails loudly (no CPU path)."""
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    prob = P.Problem.generate(1, 4)
    with pytest.raises(P.PatchdbError) as e:
        prob.matrix()
    assert e.value.status == P.PDB_ERR_INTERNAL and "CUDA" in e.value.message


def test_out_of_scope_entry_points_fail_cleanly(P):
    L = P.lib
    # the experiment drivers (CSV reproduction of the paper's tables) are out of scope
    assert L.pdb_run_experiment(b"{}", b"/tmp/x.csv") == P.PDB_ERR_INTERNAL
    assert "outside the B200 hot path" in L.pdb_last_error().decode()
    assert L.pdb_run_benchmark(b"{}", b"/tmp/x.csv") == P.PDB_ERR_INTERNAL
    assert L.pdb_run_analyze(b"{}", b"/tmp/x.csv", b"/tmp/y.csv") == P.PDB_ERR_INTERNAL


def test_sharded_setup_entry_points_validate_before_device(P):
    L = P.lib
    out = C.c_void_p()
    uid = (C.c_ubyte * 128)()
    assert L.pdb_comm_create(None, 0, 1, C.byref(out)) == P.PDB_ERR_INVALID_ARGUMENT
    assert L.pdb_comm_create(uid, 2, 2, C.byref(out)) == P.PDB_ERR_INVALID_ARGUMENT
    assert "rank" in L.pdb_last_error().decode()
    assert L.pdb_database_build_sharded(None, None, None, None, C.byref(out)) == P.PDB_ERR_INVALID_ARGUMENT
    L.pdb_comm_free(None)


def test_database_import_errors_before_device(P, tmp_path):
    with pytest.raises(P.PatchdbError) as e:
        P.Database.load(str(tmp_path / "missing.json"), str(tmp_path / "missing.bin"))
    assert e.value.status == P.PDB_ERR_IO
    bad = tmp_path / "bad.json"
    bad.write_text('{"method": "kmeans", "eps": 0, "m_p": 2, "n_p": 3, "entries": [{"rows": 9, "cols": 9}]}')
    (tmp_path / "bad.bin").write_bytes(b"")
    with pytest.raises(P.PatchdbError) as e:
        P.Database.load(str(bad), str(tmp_path / "bad.bin"))
    assert e.value.status == P.PDB_ERR_PARSE
    ok = tmp_path / "ok.json"
    ok.write_text('{"method": "m", "eps": 0.5, "m_p": 1, "n_p": 2, "entries": [{"rows": 2, "cols": 2}], "phi": [0, 0]}')
    (tmp_path / "short.bin").write_bytes(b"\0" * 8)
    with pytest.raises(P.PatchdbError) as e:
        P.Database.load(str(ok), str(tmp_path / "short.bin"))
    assert e.value.status == P.PDB_ERR_PARSE and "expected 4 doubles" in e.value.message
