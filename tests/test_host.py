"""CPU: the product's host-side C++ (setup builders, CSR utilities) and the C
ABI surface. No GPU compute is called here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2301_01753_b200 as S
from paper_2301_01753_b200 import _lib as L
from oracle import oracle as O
from tests.conftest import ROOT


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "sfeec_b200.h")).read()
    declared = set(re.findall(r"\b(sfeec_\w+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = L.lib()
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in sfeec_b200.h but not exported"
    assert declared == set(L.EXPORTED_SYMBOLS), "python binding out of sync with the header"


def test_no_cpu_fallback_without_device():
    if S.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(S.DeviceError, match="no CUDA device"):
        S.YeeScheme(4, 4, 4, 1, 1, 1, 0.1)
    c, _ = S.yee_operators(2, 2, 2, 1, 1, 1)
    q = S.scaled_identity(c.cols, 1.0)
    m2 = S.scaled_identity(c.rows, 1.0)
    with pytest.raises(S.DeviceError):
        S.SplitScheme(S.SplitKind.Strang, 0.1, q, c, m2)


def test_invalid_parameters_raise_before_device_use():
    c, _ = S.yee_operators(2, 2, 2, 1, 1, 1)
    q = S.scaled_identity(c.cols, 1.0)
    m2 = S.scaled_identity(c.rows, 1.0)
    with pytest.raises(S.InvalidParameter, match="dt must be >= 0"):
        S.SplitScheme(S.SplitKind.Strang, -0.1, q, c, m2)
    with pytest.raises(S.InvalidParameter, match="inconsistent"):
        S.SplitScheme(S.SplitKind.Strang, 0.1, S.scaled_identity(c.cols + 1, 1.0), c, m2)
    bad = S.SparseOperator(2, 3, [0, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(S.InvalidParameter, match="square"):
        S.SplitScheme(S.SplitKind.Strang, 0.1, bad, c, m2)


@pytest.mark.parametrize("tag", ["unit4", "aniso345", "nondyadic"])
def test_periodic_curl_bitwise_equals_reference(golden, tag):
    g = golden("cubical_curl.npz")
    nx, ny, nz = (int(v) for v in g[f"{tag}_dims"])
    dx, dy, dz = (float(v) for v in g[f"{tag}_d"])
    c, _ = S.yee_operators(nx, ny, nz, dx, dy, dz, bc=L.BC_PERIODIC)
    assert np.array_equal(c.row_ptr, g[f"{tag}_rp"])
    assert np.array_equal(c.col_idx, g[f"{tag}_ci"])
    assert np.array_equal(c.val, g[f"{tag}_va"])


def test_from_triplets_symmetric_part_transpose_match_reference(golden):
    t = golden("triplets.npz")
    m = S.operator_from_triplets(7, 5, t["r"], t["c"], t["v"])
    assert np.array_equal(m.row_ptr, t["rp"]) and np.array_equal(m.col_idx, t["ci"])
    assert np.array_equal(m.val, t["va"])
    g = golden("scheme.npz")
    n1 = int(g["n1"])
    q = S.SparseOperator(n1, n1, g["q_rp"], g["q_ci"], g["q_va"])
    qs = S.symmetric_part(q)
    assert np.array_equal(qs.row_ptr, g["qsym_rp"]) and np.array_equal(qs.col_idx, g["qsym_ci"])
    assert np.array_equal(qs.val, g["qsym_va"])
    ct = S.transpose(S.SparseOperator(int(g["n2"]), n1, g["c_rp"], g["c_ci"], g["c_va"]))
    ref = O.port_transpose((int(g["n2"]), n1, g["c_rp"], g["c_ci"], g["c_va"]))
    assert np.array_equal(ct.row_ptr, ref[2]) and np.array_equal(ct.col_idx, ref[3])
    assert np.array_equal(ct.val, ref[4])


def test_from_triplets_rejects_out_of_range():
    with pytest.raises(S.InvalidParameter, match="out of range"):
        S.operator_from_triplets(2, 2, [0, 2], [0, 0], [1.0, 1.0])


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_pec_yee_counts_and_exact_complex(n):
    """Appendix A (Yee, PEC): interior edges 3n(n-1)^2, faces 3n^2(n+1); D C = 0."""
    c, d = S.yee_operators(n, n, n, 1.0, 0.5, 2.0, bc=L.BC_PEC)
    assert c.cols == 3 * n * (n - 1) ** 2
    assert c.rows == 3 * n * n * (n + 1)
    assert d.rows == n ** 3 and d.cols == c.rows
    dc = d.to_dense() @ c.to_dense()
    assert np.all(dc == 0.0)
    # every row of C has <= 4 entries; boundary faces have none
    assert np.all(np.diff(c.row_ptr) <= 4)


def test_pec_numbering_roundtrip_and_orientation():
    """PEC face rows: a face strictly inside the box has the full 4-edge
    boundary with the reference orientation (+e_a1(p), +e_a2(p+a1),
    -e_a1(p+a2), -e_a2(p)), entries +-|edge|/|face|."""
    nx, ny, nz = 3, 4, 5
    dx, dy, dz = 1.0, 0.5, 2.0
    c, _ = S.yee_operators(nx, ny, nz, dx, dy, dz, bc=L.BC_PEC)
    # x-face (a=0) at (i,j,k)=(1,1,1): edges y(1,1,1)+, z(1,2,1)+, y(1,1,2)-, z(1,1,1)-
    def face_id(a, i, j, k):
        ext = {0: (nx + 1, ny, nz), 1: (nx, ny + 1, nz), 2: (nx, ny, nz + 1)}
        off = [0, (nx + 1) * ny * nz, (nx + 1) * ny * nz + nx * (ny + 1) * nz]
        e = ext[a]
        return off[a] + i + e[0] * (j + e[1] * k)

    def edge_id(a, i, j, k):
        ext = {0: (nx, ny - 1, nz - 1), 1: (nx - 1, ny, nz - 1), 2: (nx - 1, ny - 1, nz)}
        lo = {0: (0, 1, 1), 1: (1, 0, 1), 2: (1, 1, 0)}
        off = [0, nx * (ny - 1) * (nz - 1), nx * (ny - 1) * (nz - 1) + (nx - 1) * ny * (nz - 1)]
        e, l = ext[a], lo[a]
        return off[a] + (i - l[0]) + e[0] * ((j - l[1]) + e[1] * (k - l[2]))

    f = face_id(0, 1, 1, 1)
    row = dict(zip(c.row_cols(f), c.row_vals(f)))
    area = dy * dz
    want = {edge_id(1, 1, 1, 1): dy / area, edge_id(2, 1, 2, 1): dz / area,
            edge_id(1, 1, 1, 2): -dy / area, edge_id(2, 1, 1, 1): -dz / area}
    assert row == want
    # boundary face x = 0 has no interior edges
    assert c.row_ptr[face_id(0, 0, 1, 1) + 1] == c.row_ptr[face_id(0, 0, 1, 1)]


@pytest.mark.parametrize("n,npulses", [(6, 1), (9, 8)])
def test_host_pulse_projection_matches_numpy(n, npulses):
    """sfeec_tetmesh_pulse (host C++) = inputs.pulse_one_form (numpy), to
    rounding; edge sub-ranges are slices of the whole."""
    from paper_2301_01753_b200 import inputs
    m = S.TetMesh(n, 0.1, 2023)
    xyz, ev, _, _ = m.geometry(faces=False, tets=False)
    want = inputs.pulse_one_form(xyz, ev, 7, 0.1, npulses)
    got = m.pulse(7, 0.1, npulses)
    assert np.abs(got - want).max() <= 1e-14 * np.abs(want).max()
    assert np.array_equal(m.pulse(7, 0.1, npulses, 10, 200), got[10:200])


def test_reference_arm_maps_no_product_library():
    """bench.py --impl reference times the reference step on operators built by
    the oracle restatements: the process never maps libsfeec_b200.so (VERDICT
    r1: the arm used to build its operators with the product)."""
    import subprocess
    import sys
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    code = ("import sys; sys.path.insert(0, %r); import bench; "
            "r = bench.cpu_reference_sample('tet16', budget_s=0.5, max_steps=3); "
            "assert r['value'] > 0, r; "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT' if 'libsfeec_b200' in maps else 'CLEAN')" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("CLEAN"), out.stdout
