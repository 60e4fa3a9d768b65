"""pdb_problem_assemble / _exact_solution / _l2_error against the compiled
reference (CPU only: assembly is host setup).

The reference assembles its model problems with fem.cpp:248-346 after
parse_config (experiments.cpp:45-95) and resolve_coefficient with the
constant fallback (capi.cpp:169-179).  The quadrature rule and Lagrange
tables are the input generator's own (fem1d.hpp), whose nodes and weights
may differ from quadrature.cpp in the last bit: the sparsity pattern and the
exact solution must be identical, matrix values, right-hand side and L2 error
equal to rounding (1e-13 relative to the row scale); error statuses must match
the reference's for every malformed configuration.
"""
import json

import numpy as np
import pytest

CONFIGS = [
    "",  # defaults: 2D, 60 cells, Q2, constant 1
    dict(cells=8, degree=3),
    dict(cells=6, degree=2, coefficient=dict(kind="smooth")),
    dict(cells=8, degree=2, coefficient=dict(kind="piecewise")),
    dict(cells=8, degree=1, coefficient=dict(kind="piecewise", blocks=[2, 2], values=[1, 5, 7, 3])),
    dict(cells=12, degree=2, coefficient=dict(kind="piecewise", blocks=[3, 4], values=list(range(1, 13)))),
    dict(cells=5, degree=5, coefficient=dict(kind="constant", value=3.25)),
    dict(dim=3, cells=4, degree=2),
    dict(dim=3, cells=3, degree=3, coefficient=dict(kind="constant", value=2.5)),
    dict(cells=1, degree=1),
    # keys outside the problem are parsed and ignored
    dict(cells=7, degree=2, experiment=2, methods=["full"], db_sizes=[3], seed=7, left_precond=True, omega=0.5),
]


def _js(c):
    return c if isinstance(c, str) else json.dumps(c)


@pytest.mark.parametrize("cfg", CONFIGS, ids=lambda c: _js(c) or "default")
def test_assemble_matches_reference(P, ref, cfg):
    p = P.Problem.assemble(_js(cfg))
    r = ref.problem(_js(cfg))
    (rp, ci, v), (rrp, rci, rv) = p.csr(), r.csr()
    assert np.array_equal(rp, rrp) and np.array_equal(ci, rci)
    scale = np.repeat(np.maximum.reduceat(np.abs(rv), rrp[:-1]), np.diff(rrp))
    assert np.all(np.abs(v - rv) <= 1e-13 * scale)
    b, rb = p.rhs(), r.rhs()
    np.testing.assert_allclose(b, rb, rtol=1e-13, atol=1e-13 * np.abs(rb).max())
    assert np.array_equal(p.exact_solution(), r.exact())
    u = np.random.default_rng(3).uniform(-1, 1, p.ndofs)
    np.testing.assert_allclose(p.l2_error(u), r.l2_error(u), rtol=1e-12)
    np.testing.assert_allclose(p.l2_error(p.exact_solution()), r.l2_error(r.exact()), rtol=1e-9)


def test_default_problem(P):
    p = P.Problem.assemble("")
    assert p.ndofs == 121 * 121
    rp, ci, v = p.csr()
    # Dirichlet rows are identity rows without column elimination
    b = p.rhs()
    u = p.exact_solution()
    lat = np.arange(p.ndofs)
    ix, iy = lat % 121, lat // 121
    bnd = (ix == 0) | (ix == 120) | (iy == 0) | (iy == 120)
    for d in np.flatnonzero(bnd)[:50]:
        assert rp[d + 1] - rp[d] == 1 and ci[rp[d]] == d and v[rp[d]] == 1.0
        assert b[d] == u[d]


def test_dict_and_keywords(P):
    a = P.Problem.assemble(dict(cells=4), degree=3)
    b = P.Problem.assemble('{"cells": 4, "degree": 3}')
    assert a.ndofs == b.ndofs == 13 * 13
    assert all(np.array_equal(x, y) for x, y in zip(a.csr(), b.csr()))


BAD = [
    ('{"cells": ', 6),                      # syntax
    ('[1, 2]', 6),                          # not an object
    ('{"dim": 4}', 1),
    ('{"cells": 0}', 1),
    ('{"degree": 0}', 11),
    ('{"coefficient": {"kind": "banana"}}', 1),
    ('{"dim": 3, "cells": 2, "coefficient": {"kind": "smooth"}}', 1),
    ('{"cells": 4, "coefficient": {"kind": "piecewise", "blocks": [2, 2], "values": [1, 2, 3]}}', 1),
    ('{"coefficient": {"kind": "piecewise", "blocks": [2]}}', 6),
    ('{"cells": "many"}', 14),              # json type error
    ('{"cells": 4, "coefficient": {"kind": "constant", "value": -1}}', 12),
    ('{"cells": 4, "coefficient": {"kind": "piecewise", "blocks": [1, 2], "values": [1, 0]}}', 12),
]


@pytest.mark.parametrize("text,code", BAD)
def test_assemble_errors_match_reference(P, ref, text, code):
    with pytest.raises(P.PatchdbError) as e:
        P.Problem.assemble(text)
    assert e.value.status == code
    import oracle as O
    with pytest.raises(O.CheckerError) as er:
        ref.problem(text)
    assert er.value.status == code


def test_generated_problem_has_no_manufactured_solution(P):
    p = P.Problem.generate(1, 4)
    with pytest.raises(P.PatchdbError):
        p.exact_solution()
    with pytest.raises(P.PatchdbError):
        p.l2_error(np.zeros(p.ndofs))


def test_discretisation_error_decreases(P):
    """Sanity of the manufactured problem: the nodal interpolant's L2 error
    falls with h at the Q_p rate (a direct solve is not needed for this)."""
    errs = []
    for cells in (4, 8, 16):
        p = P.Problem.assemble(dict(cells=cells, degree=2))
        errs.append(p.l2_error(p.exact_solution()))
    assert errs[0] > errs[1] > errs[2]
    assert errs[1] / errs[2] > 6.0  # ~ h^3 for Q2


@pytest.mark.parametrize("cfg", [dict(cells=6, degree=2), dict(cells=4, degree=3, experiment=2),
                                 dict(cells=5, degree=2, coefficient=dict(kind="constant", value=2.0))])
def test_export_matrix_matches_reference(P, ref, tmp_path, cfg):
    """pdb_export_matrix writes the reference's Matrix Market layout (header,
    1-based entries row by row, %.17g values); values equal to rounding."""
    a, b = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    P.export_matrix(cfg, str(a))
    ref.export_matrix(json.dumps(cfg), str(b))
    la, lb = a.read_text().splitlines(), b.read_text().splitlines()
    assert la[:2] == lb[:2] and len(la) == len(lb)
    ea = np.array([x.split() for x in la[2:]], dtype=float)
    eb = np.array([x.split() for x in lb[2:]], dtype=float)
    assert np.array_equal(ea[:, :2], eb[:, :2])
    np.testing.assert_allclose(ea[:, 2], eb[:, 2], rtol=1e-13, atol=1e-13 * np.abs(eb[:, 2]).max())


def test_export_matrix_errors(P, tmp_path):
    with pytest.raises(P.PatchdbError) as e:
        P.export_matrix(dict(cells=2), str(tmp_path / "no" / "such" / "dir.mtx"))
    assert e.value.status == 13
    with pytest.raises(P.PatchdbError) as e:
        P.export_matrix("{", str(tmp_path / "x.mtx"))
    assert e.value.status == 6
