"""Second-order P2^- system on the Kuhn tet mesh (BASELINE config 4).

The reference's P2^- is 2-D only (form_space.cpp:41-166), so these checks are
(1) the product's exact-rational element tables against the oracle's
independent floating-point derivation, (2) the product's numbering and
assembled operators against the oracle's (oracle/p2_oracle.py), and (3) the
invariants the reference's tests assert for its spaces:
counts (App. A), D C = 0 exactly, exact symmetry, SPD masses, d of a
constant 1-form = 0, nested SPAI patterns and a least-squares SPAI check.
"""
import re
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2301_01753_b200 as S
from oracle import p2_oracle as P2
from oracle import tetmesh_oracle as TO

ROOT = Path(__file__).resolve().parents[1]
PAT2 = "m1sq"


def _csr(a):
    return sp.csr_matrix((a.val, a.col_idx, a.row_ptr), shape=(a.rows, a.cols))


def _rows_to_dense(rows, ncols):
    m = np.zeros((len(rows), ncols))
    for r, row in enumerate(rows):
        for c, v in row:
            m[r, c] = v
    return m


@pytest.fixture(scope="module")
def element():
    return P2.P2Element()


def test_exact_tables_match_the_oracle_derivation(element):
    txt = (ROOT / "paper_2301_01753_b200/csrc/p2_tables.hpp").read_text()
    tab = element.tables()
    for name, shape in (("C", (15, 20)), ("D", (4, 15)), ("I1", (20, 20, 3, 3)),
                        ("I2", (15, 15, 3, 3))):
        body = re.search(r"k" + name + r"(?:\[\d+\])+ = \{(.*?)\};", txt, re.S).group(1)
        a = np.array([float(x) for x in body.replace("\n", "").split(",") if x.strip()])
        a = a.reshape(shape)
        assert np.abs(a - tab[name]).max() <= 1e-13 * max(1.0, np.abs(a).max()), name


def test_generator_reproduces_committed_header(tmp_path):
    import importlib.util
    spec = importlib.util.spec_from_file_location("gen", ROOT / "tools/gen_p2_tables.py")
    gen = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gen)
    out = tmp_path / "p2.hpp"
    gen.write_header(gen.build(), out)
    assert out.read_text() == (ROOT / "paper_2301_01753_b200/csrc/p2_tables.hpp").read_text()


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_counts_match_appendix_a(n):
    n1, n2, n3 = S.TetMesh(n, 0.1, 1).p2_counts()
    assert n1 == 38 * n**3 - 30 * n**2 + 6 * n
    assert n2 == 54 * n**3 + 18 * n**2
    assert n3 == 24 * n**3


@pytest.mark.parametrize("n,seed", [(2, 3), (3, 5)])
def test_operators_match_oracle(element, n, seed):
    m = S.TetMesh(n, 0.1, seed)
    o = P2.OracleP2(TO.OracleTetMesh(n, 0.1, seed), element)
    n1, n2, n3 = m.p2_counts()
    assert (n1, n2, n3) == (o.n1, o.n2, o.n3)
    for name, rows, shape in (("c", o.curl_rows(), (n2, n1)), ("d", o.div_rows(), (n3, n2)),
                              ("m1", o.mass_rows(1), (n1, n1)), ("m2", o.mass_rows(2), (n2, n2))):
        a = _csr(m.p2_operator(name)).toarray()
        b = _rows_to_dense(rows, shape[1])
        assert a.shape == shape
        scale = np.abs(b).max()
        assert np.abs(a - b).max() <= 1e-13 * scale, name
        # same sparsity up to entries that vanish analytically
        assert np.all((a != 0) | (np.abs(b) <= 1e-14 * scale)), name
        assert np.all((b != 0) | (np.abs(a) <= 1e-14 * scale)), name


@pytest.mark.parametrize("n", [2, 4])
def test_invariants(n):
    m = S.TetMesh(n, 0.1, 7)
    c, d = _csr(m.p2_operator("c")), _csr(m.p2_operator("d"))
    m1, m2 = _csr(m.p2_operator("m1")), _csr(m.p2_operator("m2"))
    assert (d @ c).count_nonzero() == 0 or np.abs((d @ c).data).max() == 0.0
    assert (m1 != m1.T).nnz == 0 and (m2 != m2.T).nnz == 0
    if n == 2:
        assert np.linalg.eigvalsh(m1.toarray()).min() > 0
        assert np.linalg.eigvalsh(m2.toarray()).min() > 0


def test_d_of_constant_one_form_vanishes():
    """Canonical DOFs of a constant 1-form (edge moments c.tau and 0, face
    moments 1/2 c.(x_c - x_a) and -1/2 c.(x_b - x_a)); C annihilates them on
    rows whose entity has no PEC-dropped neighbour DOFs."""
    n = 4
    m = S.TetMesh(n, 0.1, 9)
    xyz, ev, fv, tv = m.geometry()
    ent1, ks1 = m.p2_dofs(1)
    cvec = np.array([0.3, -1.1, 0.7])
    p = np.zeros(len(ent1))
    for r, (e, ks) in enumerate(zip(ent1, ks1)):
        kind, slot = ks & 1, ks >> 1
        if kind == 0:
            a, b = ev[e]
            p[r] = cvec @ (xyz[b] - xyz[a]) if slot == 0 else 0.0
        else:
            a, b, cc = fv[e]
            p[r] = 0.5 * cvec @ (xyz[cc] - xyz[a]) if slot == 0 else -0.5 * cvec @ (xyz[b] - xyz[a])
    c = _csr(m.p2_operator("c"))
    ent2, ks2 = m.p2_dofs(2)
    onb = lambda v: np.any((xyz[v] <= 1e-12) | (xyz[v] >= 1 - 1e-12))  # noqa: E731
    inner = [r for r, (e, ks) in enumerate(zip(ent2, ks2))
             if not onb(tv[e] if ks & 1 else fv[e])]
    assert len(inner) > 100
    assert np.abs((c @ p)[inner]).max() <= 1e-13


def test_spai_pattern_nesting_and_lstsq():
    """S(M1) subset of S(M1^2) on P2 M1 and the product SPAI (LDLT path of
    spai.cpp:127-286) against a numpy least-squares solve per column."""
    m = S.TetMesh(2, 0.1, 4)
    m1 = m.p2_operator("m1")
    p1, p2 = S.make_pattern(m1, "m1"), S.make_pattern(m1, PAT2)
    a1, a2 = _csr(p1), _csr(p2)
    assert ((a1 != 0).astype(int) - (a1 != 0).multiply(a2 != 0).astype(int)).nnz == 0
    q, rep = S.spai_approximate_inverse(m1, PAT2)
    M = _csr(m1).toarray()
    Q = _csr(q).toarray()
    pat = [np.nonzero(a2[:, l].toarray().ravel())[0] for l in range(M.shape[0])]
    for l in range(0, M.shape[0], 7):
        I = pat[l]
        x, *_ = np.linalg.lstsq(M[:, I], np.eye(M.shape[0])[:, l], rcond=None)
        assert np.abs(Q[I, l] - x).max() <= 1e-9 * max(1.0, np.abs(x).max())
    assert rep["fallback_columns"] == 0
