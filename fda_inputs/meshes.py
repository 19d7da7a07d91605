"""Mesh generators (vertex/triangle arrays only; no element geometry).

* ``icosphere(s, radius)``: regular icosahedron (12 vertices, cyclic
  permutations of (0, ±1, ±φ), normalised), subdivided s times 1:4 at edge
  midpoints projected to the sphere.  20·4^s triangles, CCW seen from outside,
  generation order = caller order.
* ``geodesic_sphere(nu, radius)``: icosahedron with every face split at
  edge frequency ν into ν² triangles, vertices projected to the sphere;
  20·ν² triangles (ν = 73: 106,580 ≈ the 106,032 of PAPER.md Table 3).
* ``octasphere(n, radius)``: regular octahedron subdivided the same way;
  8·4^n triangles, the N sequence of PAPER.md Table 2.
* ``graded_spheroid(...)``: prolate spheroid x²/a² + (y²+z²)/b² = 1 meshed in
  rings graded 8:1 toward the tips (SURVEY.md §8(d) config-4 recipe).
"""
from __future__ import annotations

import math

import numpy as np


def _subdivide(verts: list, faces: list, times: int, radius: float):
    """1:4 midpoint subdivision, new vertices projected to the sphere.

    Face (a,b,c) -> (a,ab,ca), (ab,b,bc), (ca,bc,c), (ab,bc,ca), emitted in
    that order per parent face; midpoints numbered by sorted unique edge.
    """
    V = np.array(verts, dtype=np.float64).reshape(-1, 3)
    F = np.array(faces, dtype=np.int64).reshape(-1, 3)
    for _ in range(times):
        e = np.stack([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]], axis=1)  # (m,3,2)
        e_sorted = np.sort(e, axis=2).reshape(-1, 2)
        uniq, inv = np.unique(e_sorted, axis=0, return_inverse=True)
        inv = inv.reshape(-1, 3)
        M = 0.5 * (V[uniq[:, 0]] + V[uniq[:, 1]])
        M *= (radius / np.linalg.norm(M, axis=1))[:, None]
        base = V.shape[0]
        V = np.concatenate([V, M], axis=0)
        ab, bc, ca = (base + inv[:, 0], base + inv[:, 1], base + inv[:, 2])
        a, b, c = F[:, 0], F[:, 1], F[:, 2]
        F = np.stack([
            np.stack([a, ab, ca], 1), np.stack([ab, b, bc], 1),
            np.stack([ca, bc, c], 1), np.stack([ab, bc, ca], 1)], axis=1).reshape(-1, 3)
    return V, F


def _orient_outward(verts, faces):
    out = []
    for (a, b, c) in faces:
        pa, pb, pc = (np.asarray(verts[i]) for i in (a, b, c))
        if np.dot(np.cross(pb - pa, pc - pa), pa + pb + pc) < 0:
            b, c = c, b
        out.append((a, b, c))
    return out


def _finish(verts, faces):
    V = np.ascontiguousarray(np.array(verts, dtype=np.float64).reshape(-1, 3))
    F = np.ascontiguousarray(np.array(faces, dtype=np.int32).reshape(-1, 3))
    return V, F


def icosphere(s: int, radius: float = 0.5):
    """Icosphere with 20·4^s triangles of the given radius, centred at 0."""
    if s < 0 or s > 10:
        raise ValueError("subdivision level out of range [0, 10]")
    phi = (1.0 + math.sqrt(5.0)) / 2.0
    base = []
    for sa in (-1.0, 1.0):
        for sb in (-1.0, 1.0):
            base.append((0.0, sa, sb * phi))
            base.append((sa, sb * phi, 0.0))
            base.append((sb * phi, 0.0, sa))
    base = sorted(base)
    # faces = vertex triples mutually at the icosahedron edge length 2
    faces = []
    n = len(base)
    P = np.array(base)
    for a in range(n):
        for b in range(a + 1, n):
            if abs(np.linalg.norm(P[a] - P[b]) - 2.0) > 1e-9:
                continue
            for c in range(b + 1, n):
                if (abs(np.linalg.norm(P[a] - P[c]) - 2.0) < 1e-9
                        and abs(np.linalg.norm(P[b] - P[c]) - 2.0) < 1e-9):
                    faces.append((a, b, c))
    assert len(faces) == 20
    verts = [p * (radius / np.linalg.norm(p)) for p in P]
    faces = _orient_outward(verts, faces)
    verts, faces = _subdivide(verts, faces, s, radius)
    return _finish(verts, faces)


def geodesic_sphere(nu: int, radius: float = 1.0):
    """Frequency-ν geodesic icosphere: 20·ν² triangles, CCW seen from outside;
    caller order = (face of the icosahedron, row i, column j, up/down)."""
    if nu < 1 or nu > 1000:
        raise ValueError("frequency out of range [1, 1000]")
    V0, F0 = icosphere(0, 1.0)
    pts, tris = [], []
    nloc = (nu + 1) * (nu + 2) // 2
    for f, (a, b, c) in enumerate(F0):
        A, B, C = V0[a], V0[b], V0[c]
        ij = [(i, j) for i in range(nu + 1) for j in range(nu + 1 - i)]
        idx = {p: f * nloc + q for q, p in enumerate(ij)}
        for (i, j) in ij:
            pts.append(A + (i / nu) * (B - A) + (j / nu) * (C - A))
        for i in range(nu):
            for j in range(nu - i):
                tris.append((idx[(i, j)], idx[(i + 1, j)], idx[(i, j + 1)]))
                if i + j < nu - 1:
                    tris.append((idx[(i + 1, j)], idx[(i + 1, j + 1)], idx[(i, j + 1)]))
    P = np.array(pts)
    P /= np.linalg.norm(P, axis=1)[:, None]
    # merge the copies of shared edge / corner vertices
    key = np.round(P * 1e9).astype(np.int64)
    uniq, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first)                    # keep first-appearance order
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    V = P[first[order]] * radius
    F = rank[inv.reshape(-1)][np.array(tris)]
    # orient CCW seen from outside (vectorised _orient_outward)
    pa, pb, pc = V[F[:, 0]], V[F[:, 1]], V[F[:, 2]]
    flip = np.einsum("ij,ij->i", np.cross(pb - pa, pc - pa), pa + pb + pc) < 0
    F[flip] = F[flip][:, [0, 2, 1]]
    return _finish(V, F)


def octasphere(n: int, radius: float = 1.0):
    """Octahedral sphere with 8·4^n triangles (Table 2 family)."""
    if n < 0 or n > 10:
        raise ValueError("subdivision level out of range [0, 10]")
    verts = [np.array(v, dtype=np.float64) * radius for v in
             [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]]
    faces = []
    for xi in (0, 1):
        for yi in (2, 3):
            for zi in (4, 5):
                faces.append((xi, yi, zi))
    faces = _orient_outward(verts, faces)
    verts, faces = _subdivide(verts, faces, n, radius)
    return _finish(verts, faces)


def graded_spheroid(a: float = 0.5, b: float = 0.125, h_eq: float = 2.4809e-3,
                    grading: float = 8.0):
    """Prolate spheroid x²/a² + (y²+z²)/b² = 1, rings graded toward the tips.

    Recipe: meridian arc length s from tip to tip;
    size function h(x) = h_eq·(1/g + (1-1/g)(1 - |x|/a)); rings at
    s_{m+1} = s_m + (√3/2) h(x(s_m)), rescaled to end exactly at the far tip;
    ring m has max(3, round(2πρ_m/h_m)) nodes, rotated by half a step per ring;
    consecutive rings zipped choosing the shorter diagonal; tips are fans.
    """
    # meridian parametrised by angle t in [0, π]: x = a cos t, ρ = b sin t
    nt = 200001
    t = np.linspace(0.0, math.pi, nt)
    x = a * np.cos(t)
    rho = b * np.sin(t)
    ds = np.hypot(np.diff(x), np.diff(rho))
    s = np.concatenate([[0.0], np.cumsum(ds)])
    L = s[-1]

    def hfun(xx):
        return h_eq * (1.0 / grading + (1.0 - 1.0 / grading) * (1.0 - abs(xx) / a))

    ring_s = [0.0]
    while True:
        xm = np.interp(ring_s[-1], s, x)
        nxt = ring_s[-1] + (math.sqrt(3.0) / 2.0) * hfun(xm)
        if nxt >= L:
            break
        ring_s.append(nxt)
    ring_s = np.array(ring_s)
    # rescale so that the last step ends exactly at the far tip
    nsteps = len(ring_s)
    ring_s = ring_s * (L / (ring_s[-1] + (math.sqrt(3.0) / 2.0) * hfun(np.interp(ring_s[-1], s, x))))
    ring_s = np.concatenate([ring_s, [L]])
    verts = []
    faces = []
    # tip 0
    verts.append((a, 0.0, 0.0))
    rings = []
    offset = 0.0
    for m in range(1, nsteps):
        sm = ring_s[m]
        xm = float(np.interp(sm, s, x))
        rm = float(np.interp(sm, s, rho))
        hm = hfun(xm)
        nm = max(3, int(round(2.0 * math.pi * rm / hm)))
        offset += 0.5
        idx = []
        for q in range(nm):
            ang = 2.0 * math.pi * (q + offset) / nm
            verts.append((xm, rm * math.cos(ang), rm * math.sin(ang)))
            idx.append(len(verts) - 1)
        rings.append(idx)
    verts.append((-a, 0.0, 0.0))
    tip1 = len(verts) - 1
    P = np.array(verts)
    # fan at tip 0
    r0 = rings[0]
    for q in range(len(r0)):
        faces.append((0, r0[q], r0[(q + 1) % len(r0)]))
    # zip rings
    for m in range(len(rings) - 1):
        A, B = rings[m], rings[m + 1]
        ia = ib = 0
        na, nb = len(A), len(B)
        # start B at the node closest in angle to A[0]
        angA = math.atan2(P[A[0], 2], P[A[0], 1])
        angsB = np.arctan2(P[B, 2], P[B, 1])
        start = int(np.argmin(np.abs(np.angle(np.exp(1j * (angsB - angA))))))
        Bs = B[start:] + B[:start]
        while ia < na or ib < nb:
            a0, a1 = A[ia % na], A[(ia + 1) % na]
            b0, b1 = Bs[ib % nb], Bs[(ib + 1) % nb]
            if ia >= na:
                adv_a = False
            elif ib >= nb:
                adv_a = True
            else:      # the shorter diagonal (squared lengths, plain floats: same order as the norms)
                adv_a = _d2(verts[a1], verts[b0]) <= _d2(verts[a0], verts[b1])
            if adv_a:
                faces.append((a0, a1, b0))
                ia += 1
            else:
                faces.append((a0, b1, b0))
                ib += 1
    rl = rings[-1]
    for q in range(len(rl)):
        faces.append((tip1, rl[(q + 1) % len(rl)], rl[q]))
    faces = _orient_outward_convex(P, faces)
    return _finish(P, faces)


def _d2(p, q):
    dx, dy, dz = p[0] - q[0], p[1] - q[1], p[2] - q[2]
    return dx * dx + dy * dy + dz * dz


def _orient_outward_convex(P, faces):
    """Flip faces whose CCW normal points towards the origin (convex, origin inside)."""
    Fa = np.asarray(faces, dtype=np.int64)
    pa, pb, pc = P[Fa[:, 0]], P[Fa[:, 1]], P[Fa[:, 2]]
    flip = np.einsum("ij,ij->i", np.cross(pb - pa, pc - pa), pa + pb + pc) < 0
    Fa[flip, 1], Fa[flip, 2] = Fa[flip, 2], Fa[flip, 1].copy()
    return [tuple(f) for f in Fa.tolist()]
