"""pdb_problem_assemble / _exact_solution / _l2_error against the compiled
reference (CPU only: assembly is host setup).

The reference assembles its model problems with fem.cpp:248-346 after
parse_config (experiments.cpp:45-95) and resolve_coefficient with the
constant fallback (capi.cpp:169-179).  Matrix, right-hand side, exact
solution and L2 error must be bitwise identical; error statuses must match
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
def test_assemble_bitwise(P, ref, cfg):
    p = P.Problem.assemble(_js(cfg))
    r = ref.problem(_js(cfg))
    for a, b in zip(p.csr(), r.csr()):
        assert np.array_equal(a, b)
    assert np.array_equal(p.rhs(), r.rhs())
    assert np.array_equal(p.exact_solution(), r.exact())
    u = np.random.default_rng(3).uniform(-1, 1, p.ndofs)
    assert p.l2_error(u) == r.l2_error(u)
    assert p.l2_error(p.exact_solution()) == r.l2_error(r.exact())


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
def test_export_matrix_bytes_match_reference(P, ref, tmp_path, cfg):
    """pdb_export_matrix writes the same Matrix Market bytes (%.17g values)."""
    a, b = tmp_path / "ours.mtx", tmp_path / "ref.mtx"
    P.export_matrix(cfg, str(a))
    ref.export_matrix(json.dumps(cfg), str(b))
    assert a.read_bytes() == b.read_bytes()


def test_export_matrix_errors(P, tmp_path):
    with pytest.raises(P.PatchdbError) as e:
        P.export_matrix(dict(cells=2), str(tmp_path / "no" / "such" / "dir.mtx"))
    assert e.value.status == 13
    with pytest.raises(P.PatchdbError) as e:
        P.export_matrix("{", str(tmp_path / "x.mtx"))
    assert e.value.status == 6
