"""Device assembly of the elasticity element matrices (csrc/generator_dev.cu,
pytest -m gpu): the generator's values assembled on the GPU are bitwise the
host assembly's (PDB_GEN_DEVICE=0), whole problems and slabs; the host-only
libpdbgen.so (no device hook) agrees too."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def same(a, b):
    return all(np.array_equal(np.asarray(x).view(np.uint64) if np.asarray(x).dtype == np.float64 else x,
                              np.asarray(y).view(np.uint64) if np.asarray(y).dtype == np.float64 else y)
               for x, y in zip(a, b))


@pytest.mark.parametrize("cells,jitter", [(3, 0.0), (4, 0.0), (6, 0.1)])
def test_device_assembly_equals_host(P, monkeypatch, cells, jitter):
    dev = P.Problem.generate(5, cells, jitter=jitter)
    monkeypatch.setenv("PDB_GEN_DEVICE", "0")
    host = P.Problem.generate(5, cells, jitter=jitter)
    monkeypatch.delenv("PDB_GEN_DEVICE")
    assert same(dev.csr(), host.csr())
    assert np.array_equal(dev.rhs(), host.rhs())


@pytest.mark.parametrize("cells,ranks", [(8, 2), (9, 4)])
def test_device_assembly_slabs(P, monkeypatch, cells, ranks):
    g = P.Problem.generate(5, cells)
    rp, ci, v = g.csr()
    for r in range(ranks):
        s = P.Problem.generate_slab(5, cells, r, ranks)
        rows = s.row_ids()
        srp, sci, sv = s.csr()
        take = np.concatenate([np.arange(rp[i], rp[i + 1]) for i in rows])
        assert np.array_equal(sv.view(np.uint64), v[take].view(np.uint64))


def test_device_assembly_equals_standalone_library(P):
    sys.path.insert(0, os.path.join(ROOT, "inputs"))
    import pdbgen
    a = pdbgen.Generated(5, 4)
    b = P.Problem.generate(5, 4)
    assert same(a.csr(), b.csr())
