#!/usr/bin/env python
"""Generates paper_2301_01753_b200/csrc/lattice_tables.hpp: the stencils of
the first-order Kuhn-lattice operators (C, C^T, M2, Q_sym = S(M1) pattern) at
an interior vertex, for the lattice layout of the device leapfrog
(csrc/lattice.cu).

Entities at vertex v = (i, j, k): edge (v, t) from v to v + ET[t]; face (v, f)
with vertices v, v + ET[FT[f][0]], v + ET[FT[f][1]] (ascending ids). A slot is
(neighbour type, offset (di, dj, dk)), ordered by (dk, dj, type, di): the
ascending column order of the k-major DOF numbering for a row away from the
32-vertex x-block edges, so the lattice kernels sum a row in CSR order.

Symmetric operators (Q_sym, M2) store each off-diagonal pair once: a slot is
"canonical" when its offset is lexicographically positive in (dk, dj, di), or
zero with the neighbour type >= the row type. A non-canonical slot reads the
value of its mirror -- the neighbour's canonical slot pointing back -- at the
neighbour's position.

  python tools/gen_lattice_tables.py  (rewrites the header; deterministic)
"""
from __future__ import annotations

import itertools
import os

ET = [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (0, 1, 1), (1, 0, 1), (1, 1, 1)]
FT = [(0, 3), (1, 3), (1, 4), (2, 4), (0, 5), (2, 5), (0, 6), (1, 6), (2, 6), (3, 6), (4, 6),
      (5, 6)]
PERM = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
LE = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
LF = [(1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2301_01753_b200", "csrc", "lattice_tables.hpp")


def add(a, b):
    return tuple(x + y for x, y in zip(a, b))


def sub(a, b):
    return tuple(x - y for x, y in zip(a, b))


def tets_near(v):
    """all Kuhn tets (as vertex-coordinate 4-tuples) of the 8 cubes at v"""
    out = []
    for d in itertools.product((-1, 0), repeat=3):
        c = add(v, d)
        for p in PERM:
            vs, cc = [c], list(c)
            for a in p:
                cc[a] += 1
                vs.append(tuple(cc))
            out.append(tuple(vs))
    return out


def edge_of(a, b):
    """(base, type) of the edge between vertices a < b (coordinates)"""
    return a, ET.index(sub(b, a))


def face_of(a, b, c):
    t1, t2 = ET.index(sub(b, a)), ET.index(sub(c, a))
    return a, FT.index((t1, t2))


def key(slot):
    t, (di, dj, dk) = slot
    return (dk, dj, t, di)


def edge_neighbours(t, v=(0, 0, 0)):
    a, b = v, add(v, ET[t])
    nb = set()
    for tet in tets_near(v) + tets_near(b):
        if a in tet and b in tet:
            for p, q in LE:
                base, tt = edge_of(tet[p], tet[q])
                nb.add((tt, sub(base, v)))
    return sorted(nb, key=key)


def face_vertices(f, v=(0, 0, 0)):
    return v, add(v, ET[FT[f][0]]), add(v, ET[FT[f][1]])


def face_neighbours(f, v=(0, 0, 0)):
    fv = face_vertices(f, v)
    nb = set()
    for tet in tets_near(v):
        if all(x in tet for x in fv):
            for lf in LF:
                base, ff = face_of(*(tet[i] for i in lf))
                nb.add((ff, sub(base, v)))
    return sorted(nb, key=key)


def curl_row(f):
    """[(edge type, offset, sign)]: +[v1,v2] - [v0,v2] + [v0,v1]"""
    v0, v1, v2 = face_vertices(f)
    out = []
    for (a, b), s in (((v1, v2), 1), ((v0, v2), -1), ((v0, v1), 1)):
        base, t = edge_of(a, b)
        out.append((t, base, s))
    return sorted(out, key=lambda x: key((x[0], x[1])))


def curl_t_row(t):
    """[(face type, offset, sign)] of the faces containing edge (0, t)"""
    out = []
    for f in range(12):
        for (et, off, s) in curl_row(f):
            if et == t:
                out.append((f, tuple(-x for x in off), s))
    return sorted(out, key=lambda x: key((x[0], x[1])))


def canonical(row_t, slot):
    t, off = slot
    o = (off[2], off[1], off[0])
    return o > (0, 0, 0) or (o == (0, 0, 0) and t >= row_t)


def sym_tables(rows):
    """rows[t] = sorted slots -> (canonical index lists, per-slot source)"""
    canon = [[s for s in rows[t] if canonical(t, s)] for t in range(len(rows))]
    table = []
    for t, slots in enumerate(rows):
        ent = []
        for (tt, off) in slots:
            if canonical(t, (tt, off)):
                ent.append((tt, off, 0, t, canon[t].index((tt, off))))
            else:
                back = (t, tuple(-x for x in off))
                assert back in rows[tt], (t, tt, off)
                ent.append((tt, off, 1, tt, canon[tt].index(back)))
        table.append(ent)
    return canon, table


def emit():
    q_rows = [edge_neighbours(t) for t in range(7)]
    m_rows = [face_neighbours(f) for f in range(12)]
    q_canon, q_tab = sym_tables(q_rows)
    m_canon, m_tab = sym_tables(m_rows)
    # symmetric check: every (t, t', off) has its reverse
    for t in range(7):
        for (tt, off) in q_rows[t]:
            assert (t, tuple(-x for x in off)) in q_rows[tt]
    L = []
    w = L.append
    w("// GENERATED by tools/gen_lattice_tables.py -- do not edit.")
    w("// Interior-vertex stencils of the first-order Kuhn-lattice operators")
    w("// (DESIGN.md 3.4). Slot = {neighbour type, di, dj, dk, mirror, src type,")
    w("// src index}: the value is coefficient array (src type, src index) at the")
    w("// row's vertex (mirror 0) or at the neighbour's (mirror 1).")
    w("#pragma once")
    w("")
    w("#ifdef __CUDACC__")
    w("#define SFEEC_HD __host__ __device__")
    w("#else")
    w("#define SFEEC_HD")
    w("#endif")
    w("")
    w("namespace sfeec_b200 {")
    w("namespace lat {")
    w("")
    w("struct Slot {")
    w("  int t, di, dj, dk, mirror, st, si;")
    w("};")
    w("struct CSlot {")
    w("  int t, di, dj, dk, sign;")
    w("};")
    w("")
    for name, rows, canon, tab, n in (("Q", q_rows, q_canon, q_tab, 7),
                                      ("M", m_rows, m_canon, m_tab, 12)):
        w(f"// {name}: {n} row types; slots per type {[len(r) for r in rows]}, "
          f"canonical {[len(c) for c in canon]}")
        w(f"inline constexpr int k{name}Types = {n};")

        off = [0]
        for c in canon:
            off.append(off[-1] + len(c))
        w(f"SFEEC_HD constexpr int k{name}CanonOff(int t) {{")
        w(f"  constexpr int v[{n + 1}] = {{{', '.join(map(str, off))}}};")
        w("  return v[t];")
        w("}")
        w(f"inline constexpr int k{name}Arrays = {off[-1]};")
        so = [0]
        for r in rows:
            so.append(so[-1] + len(r))
        w(f"SFEEC_HD constexpr int k{name}SlotOff(int t) {{")
        w(f"  constexpr int v[{n + 1}] = {{{', '.join(map(str, so))}}};")
        w("  return v[t];")
        w("}")
        w(f"SFEEC_HD constexpr Slot k{name}Tab(int s) {{")
        w(f"  constexpr Slot v[{so[-1]}] = {{")
        for t in range(n):
            for (tt, o, mir, st, si) in tab[t]:
                w(f"      {{{tt}, {o[0]}, {o[1]}, {o[2]}, {mir}, {st}, {si}}},  // row type {t}")
        w("  };")
        w("  return v[s];")
        w("}")
        w("")
    c_rows = [curl_row(f) for f in range(12)]
    ct_rows = [curl_t_row(t) for t in range(7)]
    w("// C: face type -> 3 (edge type, offset, sign); C^T: edge type -> faces")
    w("SFEEC_HD constexpr CSlot kCTab(int s) {")
    w("  constexpr CSlot v[36] = {")
    for f in range(12):
        for (t, o, s) in c_rows[f]:
            w(f"      {{{t}, {o[0]}, {o[1]}, {o[2]}, {s}}},  // face type {f}")
    w("  };")
    w("  return v[s];")
    w("}")
    so = [0]
    for r in ct_rows:
        so.append(so[-1] + len(r))
    w("SFEEC_HD constexpr int kCTOff(int t) {")
    w(f"  constexpr int v[8] = {{{', '.join(map(str, so))}}};")
    w("  return v[t];")
    w("}")
    w("SFEEC_HD constexpr CSlot kCTTab(int s) {")
    w(f"  constexpr CSlot v[{so[-1]}] = {{")
    for t in range(7):
        for (f, o, s) in ct_rows[t]:
            w(f"      {{{f}, {o[0]}, {o[1]}, {o[2]}, {s}}},  // edge type {t}")
    w("  };")
    w("  return v[s];")
    w("}")
    w("")
    w("}  // namespace lat")
    w("}  // namespace sfeec_b200")
    with open(OUT, "w") as fh:
        fh.write("\n".join(L) + "\n")
    print(OUT, [len(r) for r in q_rows], sum(len(r) for r in q_rows),
          [len(c) for c in q_canon], sum(len(c) for c in q_canon),
          [len(r) for r in m_rows], sum(len(c) for c in m_canon), so[-1])


if __name__ == "__main__":
    emit()
