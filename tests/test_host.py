"""Host-side logic (no GPU): the CSR container's structural operations, the
stencil recognition of externally built problems (whole-CSR verification),
supplied-splitting checks, and the exact-solution sentinel."""

import numpy as np
import pytest

import paper_2512_21164_b200 as g
from paper_2512_21164_b200 import sparsemat as M
from paper_2512_21164_b200.problems import Problem
from paper_2512_21164_b200.stencil import csr_equals, recognise, splitting_matches


def _rand(rng, n, m, d=0.3):
    return rng.standard_normal((n, m)) * (rng.random((n, m)) < d)


def test_sparsemat_structure_matches_dense():
    rng = np.random.default_rng(4)
    for _ in range(10):
        a, b = _rand(rng, 11, 11), _rand(rng, 3, 4)
        ma, mb = M.SparseMatrix.from_dense(a), M.SparseMatrix.from_dense(b)
        assert np.array_equal(ma.to_dense(), a)
        assert np.array_equal(M.kron(ma, mb).to_dense(), np.kron(a, b))
        assert np.array_equal(M.transpose(mb).to_dense(), b.T)
        m, n = M.symm_skew_split(ma)
        assert np.array_equal(m.to_dense(), (a + a.T) * 0.5) and np.array_equal(n.to_dense(), (a - a.T) * 0.5)
        assert np.array_equal(M.shift_diagonal(ma, 0.25).to_dense(), a + 0.25 * np.eye(11))
        # canonical form: ascending unique columns, no stored zeros
        for i in range(ma.nrows):
            c = ma.col_indices[ma.row_offsets[i]:ma.row_offsets[i + 1]]
            assert np.all(np.diff(c) > 0)
        assert np.all(ma.values != 0)
    t = M.tridiag(6, -1.0, 2.0, -0.5).to_dense()
    assert np.array_equal(t, np.diag(np.full(5, -1.0), -1) + 2 * np.eye(6) + np.diag(np.full(5, -0.5), 1))
    with pytest.raises(ValueError):
        M.SparseMatrix([0, 1], [3], [1.0], (1, 2))  # column outside the matrix
    with pytest.raises(ValueError):
        M.SparseMatrix([0, 2, 1], [0, 1], [1.0, 1.0], (2, 2))  # decreasing offsets
    with pytest.raises(g.errors.NonSquare):
        M.symm_skew_split(M.SparseMatrix.from_dense(np.ones((2, 3))))


def _csr_problem(p, tweak=None):
    """The problem's A as a plain CSR (as the reference builds it)."""
    a = M.SparseMatrix.from_scipy(p.A.to_scipy())
    if tweak is not None:
        v = a.values.copy()
        v[tweak] = np.nextafter(v[tweak], np.inf)
        a = M.SparseMatrix(a.row_offsets, a.col_indices, v, a.shape)
    return Problem(A=a, b=np.zeros(a.nrows), exact_solution=None, label=p.label, params=dict(p.params))


@pytest.mark.parametrize("build,ng", [(g.build_cdr_2d, 9), (g.build_cd_3d, 5), (g.build_complex_rd, 6)])
def test_recognition_verifies_every_entry(build, ng):
    p = build(ng)
    assert recognise(_csr_problem(p)) is not None
    # one value bit changed anywhere (here: the middle entry) -> not the stencil
    nnz = p.A.to_scipy().nnz
    assert recognise(_csr_problem(p, tweak=nnz // 2)) is None
    assert recognise(_csr_problem(p, tweak=nnz - 1)) is None


def test_supplied_splitting_must_be_the_stencils():
    p = g.build_cd_3d(5)
    sp = g.make_hss_splitting(p.A, 0.5, "bf16")
    assert splitting_matches(sp, p.A.spec)
    # a splitting of a different build of the same problem still matches
    assert splitting_matches(g.make_hss_splitting(g.build_cd_3d(5).A, 0.5, "bf16"), p.A.spec)
    # a CSR splitting equal to the stencil's matches; a modified one does not
    csr = M.SparseMatrix.from_scipy(p.A.to_scipy())
    sc = g.make_hss_splitting(csr, 0.5, "bf16")
    assert splitting_matches(sc, p.A.spec)
    h = sc.H_low
    v = h.values.copy()
    v[3] *= 2.0
    import dataclasses

    bad = dataclasses.replace(sc, H_low=M.SparseMatrix(h.row_offsets, h.col_indices, v, h.shape))
    assert not splitting_matches(bad, p.A.spec)
    assert csr_equals(csr, p.A)


def test_exact_solution_sentinel():
    p = g.build_cd_3d(4)
    assert p.exact_is_ones
    p.exact_solution = None  # explicit: no exact solution (ferr / mu become None)
    assert not p.exact_is_ones and p.exact_solution is None
    q = g.build_cd_3d(4)
    assert np.array_equal(q.exact_solution, np.ones(64)) and not q.exact_is_ones
