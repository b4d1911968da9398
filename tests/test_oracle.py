"""CPU suite: pins the oracle (oracle/rst_oracle.c) to the reference.

Three anchors: (1) the reference's own doctest golden vectors
(proj/tests/test_*.cpp), restated here; (2) committed fixtures produced by
the reference itself (tests/golden/make_golden.py); (3) when oracle/_ref is
built (this container), live side-by-side runs against the compiled
reference on random graphs.
"""
import ctypes
import glob
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = sorted(glob.glob(os.path.join(HERE, "golden", "*.npz")))
INF = np.iinfo(np.int64).max


def fixture_graph(O, d):
    return O.Graph(int(d["n"]), d["eu"], d["ev"])


@pytest.mark.parametrize("path", [p for p in GOLDEN if "euler_ranks" not in p],
                         ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_matches_reference_fixtures(O, path):
    d = np.load(path)
    g = fixture_graph(O, d)
    labels, te = O.cc_spanning_forest(g)
    assert np.array_equal(labels, d["cc_labels"])
    assert np.array_equal(te, d["cc_tree_edges"])
    for root in d["roots"]:
        for algo, tag in ((0, "bfs"), (1, "cc_euler"), (2, "pr_rst")):
            p, r, lv = O.run(g, algo, int(root))
            assert np.array_equal(p, d[f"{tag}_r{root}_parent"]), (tag, root)
            assert np.array_equal(r, d[f"{tag}_r{root}_roots"]), (tag, root)
            if algo == 0:
                assert np.array_equal(lv, d[f"{tag}_r{root}_levels"])
                p2, r2, lv2 = O.run(g, 0, int(root), fast_bfs=False)  # literal restatement
                assert np.array_equal(p2, p) and np.array_equal(lv2, lv)


def test_oracle_euler_ranks_fixture(O):
    d = np.load(os.path.join(HERE, "golden", "euler_ranks.npz"))
    for t in range(20):
        n = int(d[f"t{t}_n"][0])
        te = d[f"t{t}_edges"]
        E = 2 * len(te)
        rank = np.zeros(E, np.int64)
        rc = O.lib().og_list_rank(ctypes.c_int64(E), O._p(np.ascontiguousarray(d[f"t{t}_succ"])),
                                  O._p(rank))
        assert rc == 0 and np.array_equal(rank, d[f"t{t}_rank"])
        p, r, rk = O.euler_root_forest(n, te, np.zeros(n, np.int64), 0, ranks=True)
        assert np.array_equal(rk, d[f"t{t}_rank"])


# ---- the reference's doctest golden vectors -------------------------------
def test_cc_triangle_hook(O):
    # test_cc.cpp:41-55
    g = O.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    rep = np.array([0, 1, 2], np.int64)
    tf = np.zeros(3, np.uint8)
    slot = np.full(3, INF, np.int64)
    assert O.hook_step(g, 0, rep, tf, slot)
    assert list(rep) == [0, 0, 0] and list(tf) == [1, 1, 0]
    assert not O.hook_step(g, 1, rep, tf, slot)


def test_cc_uncompressed_throws(O):
    # test_cc.cpp:57-66
    g = O.from_edges(3, [(0, 1), (1, 2)])
    with pytest.raises(O.OracleError, match="hooking ran on uncompressed labels"):
        O.hook_step(g, 0, np.array([1, 2, 2], np.int64), np.zeros(2, np.uint8),
                    np.full(3, INF, np.int64))


def test_jump_steps(O):
    # test_cc.cpp:68-94: chain of 8 in 3 steps; compressed input 1 step; odd cycle throws
    rep = np.array([0, 0, 1, 2, 3, 4, 5, 6], np.int64)
    assert O.jump_to_convergence(rep) == 3 and list(rep) == [0] * 8
    rep = np.array([0, 0, 2, 2], np.int64)
    assert O.jump_to_convergence(rep) == 1
    with pytest.raises(O.OracleError, match="pointer jumping failed to converge"):
        O.jump_to_convergence(np.array([1, 2, 0, 3], np.int64))


def test_spanning_forest_partition(O):
    # test_cc.cpp:96-103
    for g in [O.gen("path", 64), O.gen("star", 64), O.gen("grid", 9, 11),
              O.from_edges(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])] + \
             [O.gen("random", 500, 0.004, seed=s) for s in range(1, 6)]:
        labels, te = O.cc_spanning_forest(g)
        want = O.components(g)
        canon = {}
        norm = np.array([canon.setdefault(int(l), v) for v, l in enumerate(labels)])
        assert np.array_equal(norm, want)
        assert len(te) == g.n - len(set(want.tolist()))


def test_euler_star3_worked_example(O):
    # test_euler.cpp:169-197
    n, T = 3, 2
    tu = np.array([0, 0], np.int64)
    tv = np.array([1, 2], np.int64)
    fr, to, nx = (np.zeros(4, np.int64) for _ in range(3))
    first, last = np.zeros(3, np.int64), np.zeros(3, np.int64)
    O.lib().og_build_euler(ctypes.c_int64(n), ctypes.c_int64(T), O._p(tu), O._p(tv), O._p(fr),
                           O._p(to), O._p(first), O._p(last), O._p(nx))
    assert list(fr) == [0, 0, 1, 2] and list(to) == [1, 2, 0, 0]
    assert first[0] == 0 and nx[0] == 1 and last[0] == 1
    p, r, rk = O.euler_root_forest(3, [(0, 1), (0, 2)], [0, 0, 0], -1, ranks=True)
    assert list(rk) == [0, 2, 1, 3] and list(p) == [0, 0, 0] and list(r) == [0]


def test_euler_errors_and_multicomponent(O):
    # test_euler.cpp:257-281
    p, r = O.euler_root_forest(3, [(0, 1)], [0, 0, 2], 1)
    assert list(p) == [1, 1, 2] and list(r) == [1, 2]
    with pytest.raises(O.OracleError, match="edge count does not match a spanning forest"):
        O.euler_root_forest(3, [(0, 1), (1, 2), (0, 2)], [0, 0, 0], 0)
    with pytest.raises(O.OracleError):
        O.euler_root_forest(3, [(0, 1)], [0, 0], 0)


def test_pr_small(O):
    # test_pr.cpp:254-288
    assert list(O.run(O.gen("path", 3), 2, 0)[0]) == [0, 0, 1]
    g = O.from_edges(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])
    assert list(O.run(g, 2, 4)[1]) == [0, 4]
    assert list(O.run(O.gen("path", 1), 2, 0)[0]) == [0]
    with pytest.raises(O.OracleError, match=r"jump batch out of range \[1, 20\]"):
        O.run(O.gen("path", 4), 2, 0, jump_batch=0)
    with pytest.raises(O.OracleError, match="root 4 out of range"):
        O.run(O.gen("path", 4), 2, 4)


def test_bfs_vectors(O):
    # test_bfs.cpp:22-75
    p, r, lv = O.run(O.gen("path", 10), 0, 0)
    assert list(lv) == list(range(10))
    g = O.from_edges(4, [(0, 1), (0, 2), (1, 3), (2, 3)])
    p, r, lv = O.run(g, 0, 0)
    assert p[3] == 1 and list(lv) == [0, 1, 1, 2]
    g = O.from_edges(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])
    p, r, lv = O.run(g, 0, 0)
    assert list(r) == [0, 3] and p[4] == 3 and p[5] == 3 and lv[3] == 0 and lv[4] == 1
    p, r, lv = O.run(O.gen("path", 8), 0, 3)
    assert O.forest_depth(p) == 4


def test_generators_pinned(O):
    # road R=1000 -> m=1,201,120; kron s=16 -> m=909,106, 18,656 comps
    assert O.gen("road", 1000).m == 1201120
    g = O.gen("kron", 16)
    assert g.m == 909106 and len(np.unique(O.components(g))) == 18656
    assert O.gen("grid", 100, 100).m == 19800


def test_validate_restatement(O):
    g = O.gen("grid", 12, 9)
    p, r, _ = O.run(g, 2, 5)
    assert O.validate(g, p, r, 5)[0]
    bad = p.copy()
    bad[0] = 107
    ok, msg = O.validate(g, bad, None, 5)
    assert not ok and "not a graph edge" in msg


# ---- live comparison with the compiled reference --------------------------
ref_needed = pytest.mark.skipif(
    not os.path.exists(os.path.join(os.path.dirname(HERE), "oracle", "_ref", "librst_ref.so")),
    reason="oracle/_ref not built (no /root/reference here)")


@ref_needed
@pytest.mark.parametrize("seed", range(1, 41))
def test_oracle_vs_reference_random(O, seed):
    rs = np.random.RandomState(seed)
    n = int(rs.randint(1, 400))
    p = float(rs.choice([0.001, 0.003, 0.006, 0.01, 0.03]))
    g = O.gen("random", n, p, seed=seed)
    rg = O.ref_generate(f"random:{n}:{p}", seed)
    assert np.array_equal(g.eu, rg.eu) and np.array_equal(g.ev, rg.ev)
    root = int(rs.randint(0, n))
    for algo in (0, 1, 2):
        a, b = O.run(g, algo, root), O.ref_run(g, algo, root)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        if algo == 0:
            assert np.array_equal(a[2], b[2])
    for jb in (1, 3, 20):
        assert np.array_equal(O.run(g, 2, root, jump_batch=jb)[0], O.ref_run(g, 2, root, jump_batch=jb)[0])


@ref_needed
@pytest.mark.parametrize("spec", ["road:120", "kron:12", "grid:40:70", "path:5000"])
def test_oracle_vs_reference_shapes(O, spec):
    kind, *ps = spec.split(":")
    g = O.gen(kind, *[int(x) for x in ps])
    deg = np.diff(g.offsets)
    root = int(np.argmax(deg))
    for algo in (0, 1, 2):
        a, b = O.run(g, algo, root), O.ref_run(g, algo, root)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---- the config-5 checker (oracle/kron_uf.c) ------------------------------------
@pytest.mark.parametrize("scale,ef", [(10, 16), (12, 16), (13, 4)])
def test_kron_uf_matches_reference_components(O, scale, ef):
    # host union-find over regenerated tuples == the partition of the
    # normalized graph (reference cc labels when the reference is built)
    g = O.gen("kron", scale, ef)
    root, c = O.kron_uf(scale, ef, threads=4)
    labels = O.ref_cc_spanning_forest(g)[0] if O.have_ref() else O.cc_spanning_forest(g)[0]
    assert O.same_partition(labels, root)
    _, te = O.cc_spanning_forest(g)
    assert c == g.n - len(te)
    # tree edges form a forest with the same classes; one extra edge makes a cycle
    tuv = np.stack([g.eu[te], g.ev[te]], 1)
    troot, tc = O.uf_edges(g.n, tuv, threads=3)
    assert tc == g.n - len(te) and np.array_equal(troot, root)
    extra = np.array([[g.eu[0], g.ev[0]]]) if 0 not in set(te.tolist()) else None
    if extra is not None:
        _, tc2 = O.uf_edges(g.n, np.concatenate([tuv, extra]))
        assert tc2 == tc  # the non-tree edge merges nothing: T + 1 edges, same classes


def test_same_partition_detects_differences(O):
    root = np.array([0, 0, 2, 2, 4], np.int32)
    assert O.same_partition(np.array([1, 1, 3, 3, 4]), root)
    assert not O.same_partition(np.array([1, 1, 1, 3, 4]), root)   # merges two classes
    assert not O.same_partition(np.array([0, 1, 2, 2, 4]), root)   # splits a class
    assert not O.same_partition(np.array([0, 0, 2, 2, 9]), root)   # out of range


def corruptions(g, parent, rs, count):
    """Random corruptions of a valid forest: re-pointed parents (edges and
    non-edges), 2-cycles, extra roots, roots removed."""
    n = g.n
    out = []
    for _ in range(count):
        p = parent.copy()
        kind = rs.randint(0, 5)
        v = int(rs.randint(0, n))
        if kind == 0:  # any vertex
            p[v] = int(rs.randint(0, n))
        elif kind == 1:  # a neighbour (an edge: may close a cycle or stay valid)
            nb = g.nbrs[g.offsets[v]:g.offsets[v + 1]]
            if len(nb):
                p[v] = int(nb[rs.randint(0, len(nb))])
        elif kind == 2:  # 2-cycle on an edge
            nb = g.nbrs[g.offsets[v]:g.offsets[v + 1]]
            if len(nb):
                u = int(nb[rs.randint(0, len(nb))])
                p[v], p[u] = u, v
        elif kind == 3:  # extra root
            p[v] = v
        else:  # a root removed (points at a neighbour)
            roots = np.flatnonzero(p == np.arange(n))
            r = int(roots[rs.randint(0, len(roots))])
            nb = g.nbrs[g.offsets[r]:g.offsets[r + 1]]
            if len(nb):
                p[r] = int(nb[0])
        out.append(p)
    return out


def validation_class(msg):
    """The reference's first validation error -> the device validator's code."""
    for key, code in (("is not a graph edge", 2), ("parent chain cycle", 3), ("has two roots", 4),
                      ("roots but graph has", 4), ("reaches a root in a different", 5),
                      ("was requested as root", 6)):
        if key in msg:
            return code
    return -1


@ref_needed
@pytest.mark.parametrize("spec", [("grid", 9, 13), ("random", 300, 0.01), ("kron", 9)])
def test_validate_restatement_vs_reference_corruptions(O, spec):
    g = O.gen(*spec) if spec[0] != "random" else O.ref_generate(f"random:{spec[1]}:{spec[2]}", 7)
    p, r, _ = O.run(g, 1, 0)
    rs = np.random.RandomState(11)
    for q in corruptions(g, p, rs, 60):
        roots = np.flatnonzero(q == np.arange(g.n))
        want = O.ref_validate(g, q, roots, 0)
        got = O.validate(g, q, roots, 0)
        assert got[0] == want[0], (want, got)
        if not want[0]:
            assert validation_class(got[1]) == validation_class(want[1]), (want, got)
