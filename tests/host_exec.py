"""Test helper: apply the library's exported build tables on the CPU in
complex128 (host-logic test; NOT a product path).

It checks that the tables produced by fda_build (tree, lists, states,
compressed S̃/M̃/K̃/L̃/T̃, corrections) reproduce the oracle operator to the
FDA tolerance, independently of the CUDA kernels.  Near-field Q3 values come
from the oracle kernels (oracle/kernels.py)."""
from __future__ import annotations

import numpy as np

import oracle as O


def _mat(pool, mats, m):
    off, rows, cols = mats[m]
    return pool[off:off + rows * cols].astype(np.complex128).reshape(cols, rows).T


def apply_tables(f, x: np.ndarray, far: bool = True, near: bool = True, corr: bool = True,
                 kind: str = "lhs", exchange=None) -> np.ndarray:
    """y = A x (kind 'lhs') or y = B x (kind 'rhs', needs rhs_operator=1).
    exchange(ob) (sharded builds): called between the passes with this rank's
    partial outgoing states; must add the peers' partials (xsend / xrecv)."""
    sfx = "_rhs" if kind == "rhs" else ""
    n = f.n
    perm = f.table("perm")
    V = f.table("verts").reshape(n, 3, 3)
    lr = f.table("leaf_range").reshape(-1, 2)
    nl = lr.shape[0]
    xt = np.asarray(x, dtype=np.complex128)[perm]
    y = np.zeros(n, dtype=np.complex128)
    a = V[:, 1] - V[:, 0]
    b = V[:, 2] - V[:, 0]
    cr = np.cross(a, b)
    area = 0.5 * np.linalg.norm(cr, axis=1)
    nrm = -cr / (2 * area)[:, None]
    cen = V.mean(axis=1)
    P3, W3 = O.RULE_Q3
    Yq = np.einsum("qa,jad->jqd", P3, V)             # (n,3,3) quadrature points
    k, alpha = f.k, f.alpha
    own = f.table("owned")          # sharded builds: this rank's leaves [l0, l1) / elements [e0, e1)
    l0, l1, e0, e1 = (int(v) for v in own)
    if near:
        nptr, nidx = f.table("near_ptr"), f.table("near_idx")
        for i in range(l0, l1):
            tb, te = lr[i]
            src = np.concatenate([np.arange(*lr[j]) for j in nidx[nptr[i]:nptr[i + 1]]])
            X = cen[tb:te][:, None, None, :]
            NX = nrm[tb:te][:, None, None, :]
            Y = Yq[src][None]
            NY = nrm[src][None, :, None, :]
            K = (O.lhs_kernel(X, NX, Y, NY, k, alpha) if kind == "lhs"
                 else O.rhs_kernel(X, NX, Y, k, alpha))       # (nt, ns, 3)
            A = (K @ W3) * area[src][None, :]
            y[tb:te] += A @ xt[src]
    if corr:
        cp, cc = f.table("corr_ptr" + sfx), f.table("corr_col" + sfx)
        cv = f.table("corr_val" + sfx).astype(np.complex128)
        rows = np.repeat(np.arange(n), np.diff(cp))
        m = (rows >= e0) & (rows < e1)
        np.add.at(y, rows[m], (cv * xt[cc])[m])
    if far:
        pool = f.table("pool")
        mats = f.table("mats").reshape(-1, 3)
        oo, io = f.table("out_offset"), f.table("in_offset")
        osz, isz = f.table("sizes")
        lev = f.table("levels").reshape(-1, 4)
        rank = lev[:, 3].astype(int)
        boxes = f.table("boxes").reshape(-1, 8)
        outs = f.table("out_states").reshape(-1, 2)
        ins = f.table("in_states").reshape(-1, 2)
        ob = np.zeros(osz, dtype=np.complex128)
        ib = np.zeros(isz, dtype=np.complex128)

        def T_out(s):
            return rank[boxes[outs[s, 0], 0]]

        def T_in(s):
            return rank[boxes[ins[s, 0], 0]]
        lS, lT, lo, li = f.table("leaf_S" + sfx), f.table("leaf_T"), f.table("leaf_out"), f.table("leaf_in")
        for i in range(nl):
            if lS[i] >= 0:
                s = lo[i]
                ob[oo[s]:oo[s] + T_out(s)] = _mat(pool, mats, lS[i]) @ xt[lr[i, 0]:lr[i, 1]]
        for (i, s, m) in f.table("hf_s2m" + sfx).reshape(-1, 3):    # HF leaves: one op per wedge
            ob[oo[s]:oo[s] + T_out(s)] = _mat(pool, mats, m) @ xt[lr[i, 0]:lr[i, 1]]
        m2m = f.table("m2m").reshape(-1, 4)
        for l in sorted(set(m2m[:, 0]), reverse=True):
            for (_, s, d, m) in m2m[m2m[:, 0] == l]:
                ob[oo[d]:oo[d] + T_out(d)] += _mat(pool, mats, m) @ ob[oo[s]:oo[s] + T_out(s)]
        if exchange is not None:
            exchange(ob)
        for (_, s, d, m) in f.table("m2l").reshape(-1, 4):
            ib[io[d]:io[d] + T_in(d)] += _mat(pool, mats, m) @ ob[oo[s]:oo[s] + T_out(s)]
        for (_, s, d, mv, mu, _t) in f.table("m2l_lr").reshape(-1, 6):   # §4.2: Û (V̂ src)
            ib[io[d]:io[d] + T_in(d)] += _mat(pool, mats, mu) @ (_mat(pool, mats, mv) @ ob[oo[s]:oo[s] + T_out(s)])
        l2l = f.table("l2l").reshape(-1, 4)
        for l in sorted(set(l2l[:, 0])):
            for (_, s, d, m) in l2l[l2l[:, 0] == l]:
                ib[io[d]:io[d] + T_in(d)] += _mat(pool, mats, m) @ ib[io[s]:io[s] + T_in(s)]
        for i in range(nl):
            if lT[i] >= 0:
                s = li[i]
                y[lr[i, 0]:lr[i, 1]] += _mat(pool, mats, lT[i]) @ ib[io[s]:io[s] + T_in(s)]
        for (i, s, m) in f.table("hf_l2t").reshape(-1, 3):           # HF leaves: one op per wedge
            y[lr[i, 0]:lr[i, 1]] += _mat(pool, mats, m) @ ib[io[s]:io[s] + T_in(s)]
    out = np.empty(n, dtype=np.complex128)
    out[perm] = y
    return out
