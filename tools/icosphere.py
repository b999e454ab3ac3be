"""Deterministic icosphere centroid geometry (host-side producer helper, not the hot path).

BASELINE.json configs 1-4 name an icosphere mesh; the reference has no mesh code
(SURVEY.md §0.1), so the builder writes this generator: icosahedron (12 vertices,
20 faces), ``level`` rounds of midpoint 4-split with vertices projected to the
unit sphere.  Points are flat-triangle centroids, weights are flat-triangle areas.
Face order is deterministic: each parent face is replaced in place by its four
children (corner a, corner b, corner c, centre).
"""

from __future__ import annotations

import numpy as np


def _icosahedron():
    p = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array(
        [[-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0],
         [0, -1, p], [0, 1, p], [0, -1, -p], [0, 1, -p],
         [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1]],
        dtype=np.float64,
    )
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    f = np.array(
        [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
         [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
         [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
         [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]],
        dtype=np.int64,
    )
    return v, f


def icosphere(level: int):
    """Return (vertices, faces) of the icosphere refined ``level`` times."""
    verts, faces = _icosahedron()
    verts = [tuple(x) for x in verts]
    for _ in range(level):
        cache: dict[tuple[int, int], int] = {}

        def mid(a: int, b: int) -> int:
            key = (a, b) if a < b else (b, a)
            idx = cache.get(key)
            if idx is None:
                m = (np.asarray(verts[a]) + np.asarray(verts[b])) * 0.5
                m /= np.linalg.norm(m)
                idx = len(verts)
                verts.append(tuple(m))
                cache[key] = idx
            return idx

        new_faces = np.empty((4 * len(faces), 3), dtype=np.int64)
        for i, (a, b, c) in enumerate(faces):
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            new_faces[4 * i + 0] = (a, ab, ca)
            new_faces[4 * i + 1] = (b, bc, ab)
            new_faces[4 * i + 2] = (c, ca, bc)
            new_faces[4 * i + 3] = (ab, bc, ca)
        faces = new_faces
    return np.asarray(verts, dtype=np.float64), faces


def icosphere_centroids(level: int):
    """(points, weights): flat-triangle centroids and areas, N = 20 * 4**level."""
    v, f = icosphere(level)
    a, b, c = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]
    pts = (a + b + c) / 3.0
    area = 0.5 * np.linalg.norm(np.cross(b - a, c - a), axis=1)
    return pts, area
