"""Marching-cubes case table: the classic 256-case triangulation the
reference walks (recon.py:39-108 over _mc_tables.py:13-331, the Bourke /
Lorensen lineage table), held in OUR cell conventions so the device emits
exactly the reference's triangles, in the reference's order.

Conventions (ours): corner c of a cell sits at offset (c & 1, (c >> 1) & 1,
(c >> 2) & 1); cell edge e = 4*axis + (bit pattern of the two other
coordinates, lower axis first); the case index sets bit c when corner c is
OUTSIDE (value <= iso), as in the reference (ties count as outside).  The
re-indexed table is generated once by tools/gen_mc_table.py into
``_mc_cases`` (case and edge indices permuted, triangle and vertex order
kept); tests/test_mc.py checks the faces against the reference's own
marching_cubes output (golden fixtures).
"""

from __future__ import annotations

import numpy as np

from ._mc_cases import CASES

CORNERS = np.array([[(c >> 0) & 1, (c >> 1) & 1, (c >> 2) & 1] for c in range(8)])


def _edges():
    edges = []
    for axis in range(3):
        others = [a for a in range(3) if a != axis]
        for bits in range(4):
            p = [0, 0, 0]
            p[others[0]] = bits & 1
            p[others[1]] = (bits >> 1) & 1
            q = list(p)
            q[axis] = 1
            c0 = p[0] + 2 * p[1] + 4 * p[2]
            c1 = q[0] + 2 * q[1] + 4 * q[2]
            edges.append((axis, c0, c1))
    return edges


EDGES = _edges()                       # e -> (axis, corner0, corner1)
EDGE_AXIS = np.array([e[0] for e in EDGES])
EDGE_BASE = np.array([CORNERS[e[1]] for e in EDGES])  # offset of the lower corner


def build():
    """(TRI_TABLE (256, 3*MAX_TRIS) int8, -1 padded; TRI_COUNT (256,) int8)
    decoded from the classic table in our conventions (_mc_cases)."""
    tokens = CASES.split()
    assert len(tokens) == 256
    rows = [[] if t == "-" else [int(ch, 16) for ch in t] for t in tokens]
    max_t = max(len(r) for r in rows) // 3
    table = -np.ones((256, 3 * max_t), dtype=np.int8)
    count = np.zeros(256, dtype=np.int8)
    for c, r in enumerate(rows):
        assert len(r) % 3 == 0 and all(0 <= e < 12 for e in r)
        count[c] = len(r) // 3
        table[c, :len(r)] = r
    return table, count


TRI_TABLE, TRI_COUNT = build()
MAX_TRIS = TRI_TABLE.shape[1] // 3
