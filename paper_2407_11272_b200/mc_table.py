"""Marching-cubes case table, GENERATED (not transcribed) from a face rule.

Conventions (ours): corner c of a cell sits at offset (c & 1, (c >> 1) & 1,
(c >> 2) & 1); cell edge e = 4*axis + (bit pattern of the two other
coordinates, lower axis first); the case index sets bit c when corner c is
OUTSIDE (value <= iso), as in the reference (recon.py: ties count as outside).

Construction, per case: on each of the 6 cell faces the inside/outside
pattern gives 0, 2 or 4 crossed edges.  Two crossings give one segment; four
(diagonal inside corners) give two, each cutting off one inside corner (the
"separate inside corners" rule, applied identically by both cells sharing the
face, so the surface is watertight).  Segments are oriented so that, seen
from outside the cell, the inside corner lies on the right of the walking
direction; chained through the crossed edges they form closed loops, and a
fan over each loop yields triangles whose normals point from inside (value >
iso) to outside -- outward for winding-number fields.  The table is built
once at import and checked by tests/test_host_and_capi.py (closure and
orientation on every case).
"""

from __future__ import annotations

import numpy as np

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
_EDGE_OF = {frozenset((e[1], e[2])): i for i, e in enumerate(EDGES)}


def _faces():
    """6 faces as (outward normal, 4 corners in cyclic order)."""
    out = []
    for axis in range(3):
        for side in (0, 1):
            others = [a for a in range(3) if a != axis]
            cyc = [(0, 0), (1, 0), (1, 1), (0, 1)]
            corners = []
            for u, v in cyc:
                p = [0, 0, 0]
                p[axis] = side
                p[others[0]] = u
                p[others[1]] = v
                corners.append(p[0] + 2 * p[1] + 4 * p[2])
            n = np.zeros(3)
            n[axis] = 1.0 if side else -1.0
            out.append((n, corners))
    return out


FACES = _faces()


def _mid(e):
    return (CORNERS[EDGES[e][1]] + CORNERS[EDGES[e][2]]) / 2.0


def _case_triangles(case: int):
    inside = [not (case >> c) & 1 for c in range(8)]
    segs = []  # directed (edge_from, edge_to)
    for n, cyc in FACES:
        ins = [inside[c] for c in cyc]
        crossed = [(cyc[i], cyc[(i + 1) % 4]) for i in range(4)
                   if ins[i] != ins[(i + 1) % 4]]
        if not crossed:
            continue
        if len(crossed) == 2:
            e1, e2 = (_EDGE_OF[frozenset(p)] for p in crossed)
            ref_corner = next(c for c in cyc if inside[c])
            pairs = [(e1, e2, ref_corner)]
        else:  # ambiguous face: cut off each inside corner separately
            pairs = []
            for i, c in enumerate(cyc):
                if ins[i]:
                    ea = _EDGE_OF[frozenset((c, cyc[(i - 1) % 4]))]
                    eb = _EDGE_OF[frozenset((c, cyc[(i + 1) % 4]))]
                    pairs.append((ea, eb, c))
        for ea, eb, c in pairs:
            pa, pb = _mid(ea), _mid(eb)
            d = pb - pa
            r = CORNERS[c] - (pa + pb) / 2.0
            # inside corner on the RIGHT seen from outside: (n x d) . r < 0
            if np.dot(np.cross(n, d), r) < 0:
                segs.append((ea, eb))
            else:
                segs.append((eb, ea))
    nxt = {}
    for a, b in segs:
        assert a not in nxt, (case, segs)
        nxt[a] = b
    tris, seen = [], set()
    for start in sorted(nxt):
        if start in seen:
            continue
        loop, e = [], start
        while e not in seen:
            seen.add(e)
            loop.append(e)
            e = nxt[e]
        assert e == start, (case, loop)
        for i in range(1, len(loop) - 1):
            tris.append((loop[0], loop[i], loop[i + 1]))
    return tris


def build():
    all_tris = [_case_triangles(c) for c in range(256)]
    max_t = max(len(t) for t in all_tris)
    table = -np.ones((256, 3 * max_t), dtype=np.int8)
    count = np.zeros(256, dtype=np.int8)
    for c, tris in enumerate(all_tris):
        count[c] = len(tris)
        for s, t in enumerate(tris):
            table[c, 3 * s:3 * s + 3] = t
    return table, count


TRI_TABLE, TRI_COUNT = build()
MAX_TRIS = TRI_TABLE.shape[1] // 3
