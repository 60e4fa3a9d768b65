"""Drop-in check at the C-ABI (pytest -m gpu).

tests/dropin/dropin.c is compiled against the UNMODIFIED reference header
(/root/reference/proj/include/patchdb/patchdb.h) and linked by SONAME
(libpatchdb.so.0) by `make -C oracle dropin` (run by __graft_entry__.build()
where the reference exists; the binary and the reference's own
libpatchdb.so.0 -- unmodified capi.cpp + core -- travel prebuilt).  The SAME
binary runs once against the reference library and once against this repo's
library, selected by LD_LIBRARY_PATH, on the config-1 matrix read from a
Matrix Market file: detect, all seven database methods, export, precondition,
apply, GMRES, error paths.  Outputs must agree: struct sizes, defaults,
status codes and messages, sizes, phi, the SpMV, the patch-set JSON and the
exported database JSON and binary bytes exactly; applies within 1e-11;
GMRES iteration counts exactly, histories within 1e-6 relative.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "dropin")
REFLIB = os.path.join(ROOT, "oracle", "_ref", "capi")
OURLIB = os.path.join(ROOT, "paper_2306_10025_b200", "lib")


def write_mtx(path):
    sys.path.insert(0, os.path.join(ROOT, "inputs"))
    import pdbgen
    g = pdbgen.Generated(1, 0)
    rp, ci, v = g.csr()
    with open(path, "w") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{g.ndofs} {g.ndofs} {g.nnz}\n")
        for i in range(g.ndofs):
            for q in range(rp[i], rp[i + 1]):
                f.write(f"{i + 1} {ci[q] + 1} {v[q]:.17g}\n")


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    if not (os.path.exists(DRIVER) and os.path.exists(os.path.join(REFLIB, "libpatchdb.so.0"))):
        pytest.skip("drop-in driver / reference C-ABI not built (make -C oracle dropin)")
    d = tmp_path_factory.mktemp("dropin")
    mtx = str(d / "c1.mtx")
    write_mtx(mtx)
    out = {}
    for tag, lib in (("ref", REFLIB), ("ours", OURLIB)):
        od = d / tag
        od.mkdir()
        env = dict(os.environ, LD_LIBRARY_PATH=lib)
        subprocess.run([DRIVER, mtx, str(od)], check=True, env=env, timeout=600)
        out[tag] = od
    return out


def test_libraries_actually_differ(runs):
    ldd = subprocess.run(["ldd", DRIVER], capture_output=True, text=True, env=dict(os.environ, LD_LIBRARY_PATH=OURLIB))
    assert OURLIB in ldd.stdout


def test_summary_identical(runs):
    a = (runs["ref"] / "summary.txt").read_text().splitlines()
    b = (runs["ours"] / "summary.txt").read_text().splitlines()
    assert len(a) == len(b)
    for x, y in zip(a, b):
        if "missing.mtx" in x:  # the temp directory differs between the runs
            x, y = x.split("error=")[0], y.split("error=")[0]
        assert x == y


@pytest.mark.parametrize("name", ["patchset.json", "spmv.bin"] + [f"phi_m{m}.bin" for m in range(7)] +
                         [f"db_m{m}.{e}" for m in range(7) for e in ("json", "bin")])
def test_bytes_identical(runs, name):
    assert (runs["ours"] / name).read_bytes() == (runs["ref"] / name).read_bytes()


@pytest.mark.parametrize("m", range(7))
def test_apply_and_gmres(runs, m):
    za = np.fromfile(runs["ref"] / f"apply_m{m}.bin")
    zb = np.fromfile(runs["ours"] / f"apply_m{m}.bin")
    np.testing.assert_allclose(zb, za, rtol=1e-11, atol=1e-11 * np.abs(za).max())
    ha = np.fromfile(runs["ref"] / f"gmres_hist_m{m}.bin")
    hb = np.fromfile(runs["ours"] / f"gmres_hist_m{m}.bin")
    assert len(ha) == len(hb)
    np.testing.assert_allclose(hb, ha, rtol=1e-6)
