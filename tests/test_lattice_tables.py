"""CPU: the generated Kuhn-lattice stencils (tools/gen_lattice_tables.py ->
csrc/lattice_tables.hpp) against the host mesh builder: at an interior vertex
every row type's slots are exactly the columns of the M1 / M2 / C rows, in
ascending column order, and the checked-in header is the generator's output."""
import importlib.util
import os

import numpy as np
import pytest

import paper_2301_01753_b200 as S
from tests.conftest import ROOT

GEN = os.path.join(ROOT, "tools", "gen_lattice_tables.py")


def _gen():
    spec = importlib.util.spec_from_file_location("gen_lattice_tables", GEN)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _entities(mesh, faces):
    xyz, ev, fv, _ = mesh.geometry()
    n1 = mesh.n + 1
    base = (fv if faces else ev)[:, 0]
    coords = np.stack([base % n1, (base // n1) % n1, base // (n1 * n1)], axis=1)
    other = (fv[:, 1:] if faces else ev[:, 1:2])
    off = lambda v: np.stack([v % n1, (v // n1) % n1, v // (n1 * n1)], axis=1) - coords
    return coords, [off(other[:, k]) for k in range(other.shape[1])]


def test_header_is_the_generator_output(tmp_path):
    g = _gen()
    out = tmp_path / "lattice_tables.hpp"
    g.OUT = str(out)
    g.emit()
    with open(os.path.join(ROOT, "paper_2301_01753_b200", "csrc", "lattice_tables.hpp")) as f:
        assert f.read() == out.read_text()


@pytest.mark.parametrize("which", ["mass1", "mass2", "curl"])
def test_interior_stencils_equal_the_mesh_rows(which):
    g = _gen()
    n, v = 6, (3, 3, 3)
    mesh = S.TetMesh(n, 0.1, 5)
    op = getattr(mesh, which)()
    rows_faces = which != "mass1"
    cols_faces = which == "mass2"
    rc, rofs = _entities(mesh, rows_faces)
    cc, cofs = _entities(mesh, cols_faces)
    ET, FT = g.ET, g.FT

    def etype(o):
        return ET.index(tuple(int(x) for x in o))

    def row_type(r):
        if not rows_faces:
            return etype(rofs[0][r])
        return FT.index((etype(rofs[0][r]), etype(rofs[1][r])))

    def col_key(c):
        t = (FT.index((etype(cofs[0][c]), etype(cofs[1][c]))) if cols_faces
             else etype(cofs[0][c]))
        return t, tuple(int(x) for x in cc[c] - np.array(v))

    at_v = np.flatnonzero(np.all(rc == np.array(v), axis=1))
    assert at_v.size == (12 if rows_faces else 7)
    for r in at_v:
        t = row_type(r)
        cols = [col_key(c) for c in op.row_cols(r)]
        if which == "mass1":
            want = g.edge_neighbours(t)
        elif which == "mass2":
            want = g.face_neighbours(t)
        else:
            want = [(et, off) for (et, off, _) in g.curl_row(t)]
            signs = [s for (_, _, s) in g.curl_row(t)]
            assert list(op.row_vals(r)) == signs
        assert cols == want, (which, t)
