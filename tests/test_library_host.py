"""Host-logic tests of libfda.so (no GPU): the C ABI loads and exports every
symbol of include/fda.h, argument/mesh errors, tree/list/direction
invariants (readings C7-C11, C18), and the host build tables reproduce the
oracle when applied in complex128 (tests/host_exec.py)."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle as O
from oracle import fast
from fda_inputs import icosphere, octasphere, config_mesh, CONFIGS, random_density
from paper_1403_4747_b200 import FDA, FdaError, EXPORTS, load_library
from paper_1403_4747_b200.build import build as build_lib
from host_exec import apply_tables

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _lib():
    build_lib()
    return load_library()


def test_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "fda.h")).read()
    declared = set(re.findall(r"^\s*(?:fda_status|const char\*|void)\s+(\w+)\(", hdr, re.M))
    assert declared == set(EXPORTS), declared ^ set(EXPORTS)
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1403_4747_b200", "libfda.so"))
    for name in declared:
        assert hasattr(lib, name), name


def test_argument_and_mesh_errors():
    V, F = icosphere(1, 0.5)
    with pytest.raises(FdaError) as e:
        FDA(V, F, -1.0, 1j, 1e-4, device=-1)
    assert e.value.status == 1
    with pytest.raises(FdaError) as e:
        FDA(V, F, 1.0, 1j, 0.5, device=-1)
    assert e.value.status == 1
    with pytest.raises(FdaError) as e:
        FDA(V, F, 1.0, 0.0, 1e-4, device=-1)          # Im α = 0
    assert e.value.status == 1
    with pytest.raises(FdaError) as e:
        FDA(V, F[:-1], 1.0, 1j, 1e-4, device=-1)      # open mesh
    assert e.value.status == 2
    with pytest.raises(FdaError) as e:
        FDA(V, F[:, ::-1], 1.0, 1j, 1e-4, device=-1)  # inward orientation
    assert e.value.status == 2
    F2 = F.copy()
    F2[0, 1] = F2[0, 0]
    with pytest.raises(FdaError) as e:
        FDA(V, F2, 1.0, 1j, 1e-4, device=-1)
    assert e.value.status == 2
    F3 = F.copy()
    F3[0, 0] = len(V) + 5
    with pytest.raises(FdaError) as e:
        FDA(V, F3, 1.0, 1j, 1e-4, device=-1)
    assert e.value.status == 1


def test_host_only_context_refuses_matvec():
    V, F = icosphere(1, 0.5)
    f = FDA(V, F, 3.0, 1j / 3, 1e-4, device=-1)
    with pytest.raises(FdaError) as e:
        f.matvec(np.zeros(len(F), complex))
    assert e.value.status == 7


def test_config1_tree_and_list_counts():
    """272 leaves, 14,432 M2L pairs, 1.457e6
    direct element pairs; ≈74 corrections per row (A.7)."""
    V, F = config_mesh(1)
    c = CONFIGS[1]
    f = FDA(V, F, c.k, c.alpha, 1e-4, device=-1)
    s = f.stats()
    assert s["n_leaves"] == 272
    assert s["n_m2l_pairs"] == 14432
    assert abs(s["n_direct_element_pairs"] / 1.457e6 - 1) < 0.01
    assert 70 < s["n_corrections"] / len(F) < 78


def _coverage(f):
    """Brute-force pair coverage: for every ordered element pair, the number
    of M2L pairs between ancestors plus direct leaf pairs containing it."""
    n = f.n
    boxes = f.table("boxes").reshape(-1, 8)
    lr = f.table("leaf_range").reshape(-1, 2)
    cov = np.zeros((n, n), dtype=np.int32)
    nptr, nidx = f.table("near_ptr"), f.table("near_idx")
    for i in range(lr.shape[0]):
        for j in nidx[nptr[i]:nptr[i + 1]]:
            cov[lr[i, 0]:lr[i, 1], lr[j, 0]:lr[j, 1]] += 1
    outs = f.table("out_states").reshape(-1, 2)
    ins = f.table("in_states").reshape(-1, 2)
    pairs = [(s, d) for (_, s, d, _) in f.table("m2l").reshape(-1, 4)]
    pairs += [(s, d) for (_, s, d, _, _, _) in f.table("m2l_lr").reshape(-1, 6)]   # §4.2 factored ops
    for s, d in pairs:
        C, B = boxes[outs[s, 0]], boxes[ins[d, 0]]
        cov[B[5]:B[6], C[5]:C[6]] += 1
    return cov


@pytest.mark.parametrize("s,k,ml,hfl", [(3, 60.0, 8, 0), (3, 120.0, 4, 0), (2, 10.0, 4, 0), (3, 60.0, 64, 1),
                                         (3, 120.0, 16, 1)])
def test_pair_coverage_exact(s, k, ml, hfl):
    """Every ordered element pair is covered exactly once (reading C11;
    SURVEY A.13), with HF boxes split (C9) or kept as HF leaves (hfl = 1,
    PAPER.md P:344-346)."""
    V, F = icosphere(s, 0.5)
    f = FDA(V, F, k, 1j / k, 1e-3, device=-1, max_leaf=ml, hf_leaves=hfl)
    if hfl:
        assert len(f.table("hf_s2m")) > 0 and len(f.table("hf_l2t")) > 0
    assert (_coverage(f) == 1).all()


def test_direct_all_covers_everything_directly():
    V, F = icosphere(2, 0.5)
    f = FDA(V, F, 10.0, 0.1j, 1e-4, device=-1, direct_all=1, max_leaf=8)
    assert f.stats()["n_m2l_pairs"] == 0
    assert (_coverage(f) == 1).all()


def test_config1_tables_match_oracle():
    """LF-only FDA (config 1 is pure kernel-independent FMM, SURVEY §0.1 item
    6) applied from the exported tables vs the dense oracle."""
    V, F = config_mesh(1)
    c = CONFIGS[1]
    f = FDA(V, F, c.k, c.alpha, 1e-4, device=-1)
    x = random_density(len(F), c.x_seed)
    y = apply_tables(f, x)
    el = O.element_geometry(V, F)
    yo = fast.matvec_rows(el, np.arange(len(F)), x, c.k, c.alpha)
    assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < 1e-4
    # direct path alone (near + corrections, no far field) is NOT the operator
    yn = apply_tables(f, x, far=False)
    assert np.linalg.norm(yn - yo) / np.linalg.norm(yo) > 1e-3


def test_hf_leaf_tables_match_oracle():
    """Paper-faithful adaptivity (opt.hf_leaves): HF
    leaves with directional S2M / L2T per used wedge, applied from the
    exported tables vs the dense oracle."""
    V, F = icosphere(3, 0.5)
    k = 60.0
    f = FDA(V, F, k, 1j / k, 1e-4, device=-1, max_leaf=64, hf_leaves=1)
    assert len(f.table("hf_s2m")) // 3 > 100      # many (leaf, wedge) S2M ops
    x = random_density(len(F), 4)
    y = apply_tables(f, x)
    el = O.element_geometry(V, F)
    yo = fast.matvec_rows(el, np.arange(len(F)), x, k, 1j / k)
    assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < 1e-3


def test_hf_tables_match_oracle():
    """Three HF levels (384/96/24 wedges) on a 5,120-element sphere, kD = 40."""
    V, F = icosphere(4, 0.5)
    k = 40.0
    f = FDA(V, F, k, 1j / k, 1e-4, device=-1, max_leaf=16)
    s = f.stats()
    assert s["n_hf_levels"] >= 3 and s["dirs"][:3] == [384, 96, 24]
    x = random_density(len(F), 11)
    y = apply_tables(f, x)
    el = O.element_geometry(V, F)
    rows = np.arange(0, len(F), 3)
    yo = fast.matvec_rows(el, rows, x, k, 1j / k)
    err = np.linalg.norm(y[rows] - yo) / np.linalg.norm(yo)
    assert err < 1e-3, err


def test_eps_convergence():
    """FDA error falls with ε (the invariant of BASELINE north_star): the
    tables at ε = 1e-2, 1e-3, 1e-4 give decreasing errors."""
    V, F = icosphere(3, 0.5)
    k = 30.0
    el = O.element_geometry(V, F)
    x = random_density(len(F), 3)
    yo = fast.matvec_rows(el, np.arange(len(F)), x, k, 1j / k)
    errs = []
    for eps in (1e-2, 1e-3, 1e-4):
        f = FDA(V, F, k, 1j / k, eps, device=-1, max_leaf=8)
        y = apply_tables(f, x)
        errs.append(np.linalg.norm(y - yo) / np.linalg.norm(yo))
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-3, errs


def test_rhs_pass_tables_match_oracle():
    """The second fast directional pass (G sources, same target kernel and
    translations) applied from the tables vs the oracle's dense
    B = -(α/2)I + S + αK'."""
    V, F = octasphere(4, 1.0)
    k = 2 * np.pi
    f = FDA(V, F, k, 1j / k, 1e-4, device=-1, rhs_operator=1, max_leaf=32)
    el = O.element_geometry(V, F)
    x = random_density(len(F), 3)
    for kind in ("lhs", "rhs"):
        y = apply_tables(f, x, kind=kind)
        yo = fast.matvec_rows(el, np.arange(len(F)), x, k, 1j / k, kind=kind)
        assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < 1e-4, kind


def test_m2l_routing_dense_on_low_sharing_levels():
    """§4.2 factored K̃ (r < T/2) on every level where a factored K̃ is
    shared by ≥ 16 ops; the coarse HF level of config 2 (L2: ~10 ops per K̃)
    keeps the dense K̃.  Every M2L pair is routed exactly once."""
    V, F = config_mesh(2)
    c = CONFIGS[2]
    f = FDA(V, F, c.k, c.alpha, c.eps, device=-1)
    dense = f.table("m2l").reshape(-1, 4)
    lr = f.table("m2l_lr").reshape(-1, 6)
    assert len(dense) + len(lr) == f.stats()["n_m2l_pairs"]
    lr_levels = set(lr[:, 0].tolist())
    dense_levels = set(dense[:, 0].tolist())
    assert 2 in dense_levels and 2 not in lr_levels
    assert {3, 4, 5} <= lr_levels
    for l in lr_levels:
        o = lr[lr[:, 0] == l]
        assert len(o) >= 16 * len(set(o[:, 3].tolist()))


def test_correction_pairs_brute_force_graded():
    """The correction pair list (every pair with ρ_ij = |x_i − c_j|/h_j < 3, reading C6; the
    size-class hash grids of corrections.cpp) equals the brute-force O(N²) search on a graded
    spheroid whose element size varies 8× (the case the per-class grids exist for)."""
    from fda_inputs.meshes import graded_spheroid
    V, F = graded_spheroid(h_eq=0.03)
    n = len(F)
    assert 3000 < n < 30000
    f = FDA(V, F, 20.0, -1j / 20.0, 1e-3, device=-1)
    perm = f.table("perm")                              # tree position → caller index
    ptr, col = f.table("corr_ptr"), f.table("corr_col")
    P = V[F]
    cen = P.mean(axis=1)
    h = np.max(np.linalg.norm(P - np.roll(P, 1, axis=1), axis=2), axis=1)
    assert h.max() / h.min() > 4.0                      # several size classes
    got = {}
    for ti in range(n):
        i = perm[ti]
        got[i] = np.sort(perm[col[ptr[ti]:ptr[ti + 1]]])
    for i0 in range(0, n, 512):
        rows = np.arange(i0, min(n, i0 + 512))
        rho = np.linalg.norm(cen[rows, None, :] - cen[None, :, :], axis=2) / h[None, :]
        for a, i in enumerate(rows):
            want = np.nonzero(rho[a] < 3.0)[0]
            assert np.array_equal(got[i], want), i
