"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bit-exact on every integer output: parent arrays, roots (in the reference's
order), BFS levels, CC labels and tree-edge ids. The oracle itself is pinned
to the reference in tests/test_oracle.py.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ALGOS = [0, 1, 2]  # bfs, cc-euler, pr-rst


def dev_graph(rst, g):
    return rst.DeviceGraph.from_host(g.n, np.stack([g.eu, g.ev], 1), g.offsets, g.nbrs, g.origin)


def check_all(rst, O, g, root, algos=ALGOS, jump_batch=5):
    dg = dev_graph(rst, g)
    for algo in algos:
        p, r, lv, st = dg.run(algo, root, jump_batch)
        ep, er, elv = O.run(g, algo, root, jump_batch)
        assert np.array_equal(p, ep), f"algo {algo}: parent mismatch at {np.nonzero(p != ep)[0][:10]}"
        assert np.array_equal(r, er), f"algo {algo}: roots mismatch"
        if algo == 0:
            assert np.array_equal(lv, elv), "bfs levels mismatch"
    labels, te = dg.cc_spanning_forest()
    el, ete = O.cc_spanning_forest(g)
    assert np.array_equal(labels, el)
    assert np.array_equal(te, ete)
    dg.close()


SMALL = [("path", 1), ("path", 2), ("path", 3), ("path", 10), ("path", 100), ("star", 10),
         ("star", 1000), ("grid", 5, 7), ("grid", 9, 11), ("grid", 12, 9), ("complete", 12),
         ("road", 40), ("kron", 10)]


@pytest.mark.parametrize("spec", SMALL, ids=lambda s: ":".join(map(str, s)))
def test_small_generators(rst, O, spec):
    g = O.gen(*spec)
    for root in sorted({0, g.n // 2, g.n - 1}):
        check_all(rst, O, g, root)


@pytest.mark.parametrize("seed", range(1, 16))
def test_random_graphs(rst, O, seed):
    rs = np.random.RandomState(seed)
    n = int(rs.randint(2, 400))
    p = float(rs.choice([0.002, 0.005, 0.01, 0.03]))
    g = O.gen("random", n, p, seed=seed)
    check_all(rst, O, g, int(rs.randint(0, n)))


def test_two_triangles(rst, O):
    # tests/oracles.hpp:521-523; test_bfs.cpp:64-75, test_euler.cpp:305-311
    g = O.from_edges(6, [(0, 1), (1, 2), (0, 2), (3, 4), (4, 5), (3, 5)])
    check_all(rst, O, g, 0)
    check_all(rst, O, g, 4)
    dg = dev_graph(rst, g)
    p, r, lv, _ = dg.run(0, 0)
    assert list(r) == [0, 3] and p[4] == 3 and p[5] == 3 and lv[3] == 0 and lv[4] == 1
    assert list(dg.run(1, 4)[1]) == [0, 4]
    assert list(dg.run(2, 4)[1]) == [0, 4]


def test_edgeless_and_isolated(rst, O):
    g = O.Graph(5, np.zeros(0, np.int64), np.zeros(0, np.int64))
    check_all(rst, O, g, 2)
    g = O.from_edges(8, [(1, 2), (5, 6), (6, 7)])
    for root in range(8):
        check_all(rst, O, g, root)


def test_bfs_smallest_id_tiebreak(rst, O):
    # test_bfs.cpp:55-62: 3 is reachable via 1 and 2; 1 wins
    g = O.from_edges(4, [(0, 1), (0, 2), (1, 3), (2, 3)])
    p, r, lv, _ = dev_graph(rst, g).run(0, 0)
    assert p[3] == 1 and list(lv) == [0, 1, 1, 2]


def test_pr_golden(rst, O):
    # test_pr.cpp:254-260: path:3 root 0 -> {0, 0, 1}
    g = O.gen("path", 3)
    assert list(dev_graph(rst, g).run(2, 0)[0]) == [0, 0, 1]


@pytest.mark.parametrize("cap", ["1", "3", "0", "100000"])
def test_pr_reroot_short_path_and_fallback(rst, O, monkeypatch, cap):
    # the re-rooting's path, and every round's paths, walked on the parents
    # when short (cap hops), else the skip structure rebuilt and the paths
    # marked by ascent + descent: both give the reference's parents
    monkeypatch.setenv("RSTG_PR_SHORT_PATH", cap)
    monkeypatch.setenv("RSTG_PR_SHORT_PATHS", cap)
    monkeypatch.setenv("RSTG_PR_SHORT_PATHS_ROOTS", "1000000000")
    for spec, root in ((("grid", 20, 30), 377), (("road", 40), 999), (("kron", 10), 3),
                       (("path", 3000), 1500)):
        g = O.gen(*spec)
        dg = dev_graph(rst, g)
        p, r, _, _ = dg.run(2, root)
        ep, er, _ = O.run(g, 2, root)
        assert np.array_equal(p, ep) and np.array_equal(r, er), (spec, cap)
        dg.close()


def test_jump_batch_invariance(rst, O):
    # acceptance.cpp:386-401, test_pr.cpp:300-311
    g = O.gen("path", 4096)
    dg = dev_graph(rst, g)
    a = dg.run(2, 0, 1)[0]
    b = dg.run(2, 0, 5)[0]
    c = dg.run(2, 0, 20)[0]
    assert np.array_equal(a, b) and np.array_equal(a, c)


def test_root_out_of_range(rst, O):
    g = O.gen("path", 4)
    dg = dev_graph(rst, g)
    for algo in ALGOS:
        for root in (4, -1):
            with pytest.raises(rst.RSTError, match=f"root {root} out of range"):
                dg.run(algo, root)


def test_jump_batch_out_of_range(rst, O):
    g = O.gen("path", 4)
    with pytest.raises(rst.RSTError, match=r"jump batch out of range \[1, 20\]"):
        dev_graph(rst, g).run(2, 0, 0)


def test_handle_after_failed_builds(rst, O):
    # a build that throws midway (after its first grafts) leaves the state
    # a repeated build skips re-initialising (slots, scratch, marks) unknown:
    # the next builds on the same handle must re-initialise and stay exact
    g = O.gen("road", 60)
    dg = dev_graph(rst, g)
    ep = {a: O.run(g, a, 7)[0] for a in (0, 1, 2)}
    for _ in range(2):
        assert np.array_equal(dg.run(2, 7)[0], ep[2])
        with pytest.raises(rst.RSTError, match=r"jump batch out of range"):
            dg.run(2, 7, 0)
        for a in (2, 1, 2, 0):
            assert np.array_equal(dg.run(a, 7)[0], ep[a]), a
    dg.close()


def test_determinism_repeats(rst, O):
    g = O.gen("random", 1500, 0.002, seed=31)
    dg = dev_graph(rst, g)
    for algo in ALGOS:
        ref = dg.run(algo, 0)[0]
        for _ in range(3):
            assert np.array_equal(dg.run(algo, 0)[0], ref)


# ---- kernel-level golden vectors (reference doctest cases) ----------------
def test_hook_step_triangle(rst):
    # test_cc.cpp:41-55
    e = [(0, 1), (0, 2), (1, 2)]
    rep = np.array([0, 1, 2], np.int64)
    tf = np.zeros(3, np.uint8)
    slot = np.full(3, np.iinfo(np.int64).max, np.int64)
    assert rst.hook_step(3, e, 0, rep, tf, slot)
    assert list(rep) == [0, 0, 0] and list(tf) == [1, 1, 0]
    assert not rst.hook_step(3, e, 1, rep, tf, slot)


def test_hook_step_uncompressed(rst):
    # test_cc.cpp:57-66
    rep = np.array([1, 2, 2], np.int64)
    with pytest.raises(rst.RSTError, match="hooking ran on uncompressed labels"):
        rst.hook_step(3, [(0, 1), (1, 2)], 0, rep, np.zeros(2, np.uint8),
                      np.full(3, np.iinfo(np.int64).max, np.int64))


def test_jump_chain(rst):
    # test_cc.cpp:68-94
    rep = np.array([0] + list(range(7)), np.int64)
    rst.jump_to_convergence(rep)
    assert list(rep) == [0] * 8
    rep = np.array([0, 0, 2, 2], np.int64)
    rst.jump_to_convergence(rep)
    assert list(rep) == [0, 0, 2, 2]
    with pytest.raises(rst.RSTError, match="pointer jumping failed to converge"):
        rst.jump_to_convergence(np.array([1, 2, 0, 3], np.int64))


def test_list_rank_star3(rst):
    # test_euler.cpp:169-197: succ after the cut, ranks {0, 2, 1, 3}
    succ = [2, 3, 1, -1]
    assert list(rst.list_rank(succ)) == [0, 2, 1, 3]


def test_list_rank_random_lists(rst, O):
    rs = np.random.RandomState(7)
    for E in (1, 2, 33, 1000, 100000):
        perm = rs.permutation(E)
        succ = np.full(E, -1, np.int64)
        cut = set(rs.choice(E, size=min(5, E), replace=False).tolist())
        for i in range(E - 1):
            if i not in cut:
                succ[perm[i]] = perm[i + 1]
        exp = np.zeros(E, np.int64)
        import ctypes
        O.lib().og_list_rank(ctypes.c_int64(E), O._p(succ), O._p(exp))
        assert np.array_equal(rst.list_rank(succ), exp)


def test_list_rank_cycle(rst):
    # test_euler.cpp:283-295
    with pytest.raises(rst.RSTError, match="list ranking failed to converge: not a forest"):
        rst.list_rank([1, 2, 0, -1])


def test_euler_root_forest_worked(rst, O):
    # test_euler.cpp:169-197, 257-264, 266-281
    p, r = rst.euler_root_forest(3, [(0, 1), (0, 2)], [0, 0, 0], -1)
    assert list(p) == [0, 0, 0] and list(r) == [0]
    p, r = rst.euler_root_forest(3, [(0, 1)], [0, 0, 2], 1)
    assert list(p) == [1, 1, 2] and list(r) == [1, 2]
    with pytest.raises(rst.RSTError, match="edge count does not match a spanning forest"):
        rst.euler_root_forest(3, [(0, 1), (1, 2), (0, 2)], [0, 0, 0], 0)
    with pytest.raises(rst.RSTError):
        rst.euler_root_forest(3, [(0, 1)], [0, 0], 0)


def test_euler_root_forest_random_trees(rst, O):
    # test_euler.cpp:243-255 (random attachment trees, seed 2026 in C++)
    rs = np.random.RandomState(2026)
    for _ in range(30):
        n = int(rs.randint(1, 257))
        te = [(int(rs.randint(0, v)), v) for v in range(1, n)]
        root = int(rs.randint(0, n))
        p, r = rst.euler_root_forest(n, te, [0] * n, root)
        ep, er = O.euler_root_forest(n, te, [0] * n, root)
        assert np.array_equal(p, ep) and list(r) == [root]


# ---- device validator ------------------------------------------------------
def test_device_validator(rst, O):
    g = O.gen("grid", 20, 30)
    dg = dev_graph(rst, g)
    p = O.run(g, 1, 7)[0]
    assert dg.validate(p, 7)[0]
    bad = p.copy(); bad[5] = 5  # extra root in a one-component graph
    assert dg.validate(bad)[1] == 4
    bad = p.copy(); bad[0] = 599  # not an edge
    assert dg.validate(bad)[1] == 2
    cyc = p.copy(); cyc[7] = 8; cyc[8] = 7
    assert dg.validate(cyc)[1] in (3, 4)
    assert dg.validate(p, 8)[1] == 6


@pytest.mark.parametrize("spec", [("grid", 9, 13), ("random", 300, 0.01), ("kron", 9),
                                  ("road", 30)])
def test_device_validator_vs_reference_corruptions(rst, O, spec):
    # validate_rooted_forest (validate.cpp:108-211) of the reference itself
    # on random corruptions: same verdict, same error class (first error),
    # and for a non-edge parent the same (smallest) offending vertex
    from test_oracle import corruptions, validation_class
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    g = O.gen(*spec) if spec[0] != "random" else O.ref_generate(f"random:{spec[1]}:{spec[2]}", 7)
    dg = dev_graph(rst, g)
    p = O.run(g, 1, 0)[0]
    rs = np.random.RandomState(5)
    for q in corruptions(g, p, rs, 80):
        roots = np.flatnonzero(q == np.arange(g.n))
        want_ok, want_msg = O.ref_validate(g, q, roots, 0)
        ok, code, bad = dg.validate(q, 0)
        assert ok == want_ok, (want_msg, code, bad)
        if not ok:
            assert code == validation_class(want_msg), (want_msg, code, bad)
            if code == 2:
                assert want_msg.startswith(f"parent edge ({bad}, "), (want_msg, bad)
    dg.close()


# ---- medium shapes -----------------------------------------------------------
@pytest.mark.parametrize("spec,root", [(("grid", 1024, 1024), 0), (("road", 1000), 0),
                                        (("kron", 16), None), (("path", 1 << 18), 0)])
def test_medium_shapes(rst, O, spec, root):
    g = O.gen(*spec)
    if root is None:
        deg = np.diff(g.offsets)
        root = int(np.argmax(deg))  # max-degree vertex, smallest id on ties
    check_all(rst, O, g, root)


def test_device_generators_match_host(rst, O):
    for spec, host in [("path:1000", ("path", 1000)), ("star:77", ("star", 77)),
                       ("grid:31:17", ("grid", 31, 17)), ("road:300", ("road", 300)),
                       ("kron:12", ("kron", 12))]:
        dg = rst.DeviceGraph.generate(spec)
        g = O.gen(*host)
        e = dg.edges()
        assert dg.n == g.n and dg.m == g.m, spec
        assert np.array_equal(e[:, 0], g.eu) and np.array_equal(e[:, 1], g.ev), spec
        # device-built CSR drives BFS: parity with the oracle checks it too
        p, r, lv, _ = dg.run(0, 0)
        ep, er, elv = O.run(g, 0, 0)
        assert np.array_equal(p, ep) and np.array_equal(lv, elv), spec


# ---- the reference's own outputs (tests/golden, from make_golden.py) -------
import glob as _glob
import os as _os

_GOLDEN = sorted(p for p in _glob.glob(_os.path.join(_os.path.dirname(__file__), "golden", "*.npz"))
                 if "euler_ranks" not in p)


@pytest.mark.parametrize("path", _GOLDEN, ids=lambda p: _os.path.basename(p)[:-4])
def test_golden_fixtures(rst, path):
    d = np.load(path)
    n = int(d["n"])
    dg = rst.DeviceGraph.from_host(n, np.stack([d["eu"], d["ev"]], 1))  # CSR built on device
    labels, te = dg.cc_spanning_forest()
    assert np.array_equal(labels, d["cc_labels"]) and np.array_equal(te, d["cc_tree_edges"])
    for root in d["roots"]:
        for algo, tag in ((0, "bfs"), (1, "cc_euler"), (2, "pr_rst")):
            p, r, lv, _ = dg.run(algo, int(root))
            assert np.array_equal(p, d[f"{tag}_r{root}_parent"]), (tag, root)
            assert np.array_equal(r, d[f"{tag}_r{root}_roots"]), (tag, root)
            if algo == 0:
                assert np.array_equal(lv, d[f"{tag}_r{root}_levels"]), (tag, root)


def test_golden_euler_ranks(rst):
    d = np.load(_os.path.join(_os.path.dirname(__file__), "golden", "euler_ranks.npz"))
    for t in range(20):
        assert np.array_equal(rst.list_rank(d[f"t{t}_succ"]), d[f"t{t}_rank"])


# ---- edge-partitioned CC (multi-GPU path, run here as parts on one GPU) ----
def test_kron_parts_concatenate_to_full(rst, O):
    g = O.gen("kron", 12)
    for k in (1, 2, 3, 5):
        parts = [rst.DeviceGraph.generate_part("kron:12", r, k) for r in range(k)]
        e = np.concatenate([p.edges() for p in parts])
        assert np.array_equal(e[:, 0], g.eu) and np.array_equal(e[:, 1], g.ev)


def test_distcc_one_rank_matches_exact_cc(rst, O):
    import torch

    from paper_2603_11645_b200.distcc import distributed_cc

    for spec in ("kron:12", "kron:14", "kron:10:4"):
        s, ef = int(spec.split(":")[1]), int((spec.split(":") + ["16"])[2])
        g = O.gen("kron", s, ef)
        labels, te = O.cc_spanning_forest(g)
        dg = rst.DeviceGraph.generate_part(spec, 0, 1)
        tflag = torch.zeros(max(dg.m, 1), dtype=torch.uint8, device="cuda")
        rep, st = distributed_cc(dg, dg.n, 1, tflag)
        assert np.array_equal(rep.cpu().numpy().astype(np.int64), labels)
        assert st["tree_edges"] == len(te)
        assert np.array_equal(np.nonzero(tflag[: dg.m].cpu().numpy())[0], te)


def _distcc_worker(rank, world, port, spec, out):
    import os

    import torch
    import torch.distributed as dist

    import paper_2603_11645_b200 as P
    from paper_2603_11645_b200.distcc import SlotExchange, distributed_cc, edge_base

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)  # every rank on the one GPU
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dg = P.DeviceGraph.generate_part(spec, rank, world)
    base = edge_base(dg.m, rank, world, "cpu")
    dg.set_edge_base(base)
    tflag = torch.zeros(max(dg.m, 1), dtype=torch.uint8, device="cuda")
    ex = SlotExchange(dg.n, "cuda", world, staged=True)
    rep, st = distributed_cc(dg, dg.n, world, tflag, ex)
    te = np.nonzero(tflag[: dg.m].cpu().numpy())[0] + base
    out[rank] = (rep.cpu().numpy().astype(np.int64), st["tree_edges"], te, list(ex.calls))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,spec", [(2, "kron:13"), (3, "kron:12"), (4, "kron:10:4")])
def test_distcc_multiprocess_cuda(rst, O, world, spec):
    """The CUDA edge-partitioned rounds (rstg_cc_labels + SlotExchange) in
    `world` processes sharing one GPU, gloo host-staged exchange: labels on
    every rank and the union of the ranks' tree edges equal the 1-GPU
    reference (cc_spanning_forest)."""
    import socket

    import torch.multiprocessing as mp

    s, ef = int(spec.split(":")[1]), int((spec.split(":") + ["16"])[2])
    g = O.gen("kron", s, ef)
    labels, te = O.cc_spanning_forest(g)
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    out = mp.Manager().dict()
    mp.spawn(_distcc_worker, args=(world, port, spec, out), nprocs=world, join=True)
    for r in range(world):
        rep, total, _, calls = out[r]
        assert np.array_equal(rep, labels), f"rank {r}"
        assert total == len(te)
        assert calls == out[0][3]
    assert np.array_equal(np.concatenate([out[r][2] for r in range(world)]), te)
    assert out[0][3][0] == (0, g.n) and all(c < g.n for _, c in out[0][3][1:])


def test_distcc_simulated_ranks_on_one_gpu(rst, O):
    """k partitions hooked into one slot array (the MIN all-reduce of k
    ranks equals applying their atomicMin proposals to one slot array)."""
    import torch

    g = O.gen("kron", 13)
    labels, _ = O.cc_spanning_forest(g)
    k = 3
    parts = [rst.DeviceGraph.generate_part("kron:13", r, k) for r in range(k)]
    base = 0
    for p in parts:
        p.set_edge_base(base)
        base += p.m
    n = parts[0].n
    rep = torch.empty(n, dtype=torch.int32, device="cuda")
    slot = torch.empty(n, dtype=torch.int64, device="cuda")
    parts[0].cc_init(rep.data_ptr(), slot.data_ptr())
    mode = 0
    while True:
        for p in parts:
            p.cc_hook(mode, rep.data_ptr(), slot.data_ptr())
        if parts[0].cc_apply(rep.data_ptr(), slot.data_ptr()) == 0:
            break
        parts[0].cc_compress(rep.data_ptr())
        mode ^= 1
    assert np.array_equal(rep.cpu().numpy().astype(np.int64), labels)


# ---- BASELINE.json configs at full size ---------------------------------------
# Device-generated graph (the bench's input), copied out and handed to the
# oracle as the same normalized edge list; every strategy bit-exact against
# it. The device generators equal the host ones (test_device_generators_
# match_host above, and the survey's m / component counts below).
FULL = [("grid:1024:1024", 2095104), ("path:16777216", 16777215), ("road:4899", 28858008),
        ("kron:24:16", 260382979)]


@pytest.mark.slow
@pytest.mark.parametrize("spec,m_expect", FULL, ids=[s for s, _ in FULL])
def test_full_size_configs(rst, O, spec, m_expect):
    dg = rst.DeviceGraph.generate(spec)
    assert dg.m == m_expect
    e = dg.edges()
    g = O.Graph(dg.n, e[:, 0], e[:, 1])
    del e
    root = 0
    if spec.startswith("kron"):
        root = int(np.argmax(np.diff(g.offsets)))  # max degree, smallest id on ties
    for algo in ALGOS:
        p, r, lv, _ = dg.run(algo, root)
        ep, er, elv = O.run(g, algo, root)
        assert np.array_equal(p, ep), f"{spec} algo {algo}: parent mismatch at {np.nonzero(p != ep)[0][:10]}"
        assert np.array_equal(r, er), f"{spec} algo {algo}: roots mismatch"
        if algo == 0:
            assert np.array_equal(lv, elv), f"{spec}: bfs levels mismatch"
        assert dg.validate(p, root)[0]
    dg.close()


# ---- list-ranking parameters never change the result --------------------------
# Ruler density, walks in flight, walk CTAs, chunking, the ruler-level path
# and forced short walks (dynamic rulers split off mid-walk, walked by
# follow-up launches) are performance knobs only.
_WALK_KNOBS = [{"RSTG_LR_LOGK0": "1"}, {"RSTG_LR_LOGK0": "7"}, {"RSTG_LR_BLOCKS": "2"},
               {"RSTG_LR_BLOCKS": "1"}, {"RSTG_LR_CHUNK": "1"},
               {"RSTG_LR_LOGK1": "1"}, {"RSTG_LR_LOGK1": "6"}, {"RSTG_LR_COOP": "1"},
               {"RSTG_LR_WALKCAP": "4"}, {"RSTG_LR_WALKCAP": "17", "RSTG_LR_LOGK0": "6"}]
# the ruling-set walk (RSTG_LR_TILES=0) and tile contraction with its knobs
LR_KNOBS = ([dict(k, RSTG_LR_TILES="0") for k in _WALK_KNOBS] +
            [{"RSTG_LR_TILES": "1"}, {"RSTG_LR_TILES": "1", "RSTG_LR_TILELEVELS": "0"},
             {"RSTG_LR_TILES": "1", "RSTG_LR_TILELEVELS": "0", "RSTG_LR_LOGK1": "1"},
             {"RSTG_LR_TILES": "1", "RSTG_LR_TILELEVELS": "0", "RSTG_LR_LOGK1": "6"}])


@pytest.mark.parametrize("spec,root", [(("road", 300), 0), (("kron", 14), None), (("path", 5000), 77),
                                        (("grid", 40, 60), 123)])
def test_list_rank_knobs_invariant(rst, O, spec, root, monkeypatch):
    g = O.gen(*spec)
    if root is None:
        root = int(np.argmax(np.diff(g.offsets)))
    ep, er, _ = O.run(g, 1, root)
    dg = dev_graph(rst, g)
    for knobs in LR_KNOBS:
        for k, v in knobs.items():
            monkeypatch.setenv(k, v)
        p, r, _, _ = dg.run(1, root)
        assert np.array_equal(p, ep), f"{spec} {knobs}: parent mismatch"
        assert np.array_equal(r, er), f"{spec} {knobs}: roots mismatch"
        for k in knobs:
            monkeypatch.delenv(k)
    # explicit forests and raw lists take the same knobs
    monkeypatch.setenv("RSTG_LR_WALKCAP", "3")
    succ = np.full(1000, -1, np.int64)
    perm = np.random.RandomState(3).permutation(1000)
    for i in range(999):
        succ[perm[i]] = perm[i + 1]
    exp = np.zeros(1000, np.int64)
    import ctypes
    O.lib().og_list_rank(ctypes.c_int64(1000), O._p(succ), O._p(exp))
    assert np.array_equal(rst.list_rank(succ), exp)
    dg.close()


def test_tile_levels_overflow_fallback(rst, monkeypatch):
    # tile-contraction levels sized for an impossible contraction: the top
    # tile overflows (a 9M-vertex mesh leaves far more than 8192 segments)
    # and the ranking falls back to list_prefix on the level-1 segments --
    # the same parents as the ruling-set walk (itself pinned to the oracle
    # in the other tests)
    g = rst.DeviceGraph.generate("road:3000")
    out = {}
    for tag, knobs in (("walk", {"RSTG_LR_TILES": "0"}),
                       ("tiles", {"RSTG_LR_TILES": "1"}),
                       ("overflow", {"RSTG_LR_TILES": "1", "RSTG_LR_TILECONTRACT": "1000000"}),
                       # a repeated build sizes the levels from the previous
                       # count; a short bound overflows and is settled after
                       # the build (tile_rank_settle)
                       ("shortbound", {"RSTG_LR_TILES": "1", "RSTG_LR_SEGBOUND": "20000"})):
        for k, v in knobs.items():
            monkeypatch.setenv(k, v)
        out[tag] = g.run(1, 7)[0]
        for k in knobs:
            monkeypatch.delenv(k)
    assert np.array_equal(out["tiles"], out["walk"])
    assert np.array_equal(out["overflow"], out["walk"])
    assert np.array_equal(out["shortbound"], out["walk"])
    g.close()


def test_handle_reuse_across_graph_sizes(rst, O):
    # one handle, graphs of shrinking and growing size, many and few
    # components: per-build state kept between builds (the Euler min table,
    # clean slot buffers) must never leak from one graph into the next
    sparse = O.gen("random", 150000, 0.000003, seed=5)  # ~116K components: flagged table
    gs = [O.gen("kron", 13), O.gen("grid", 20, 30), O.gen("kron", 13), sparse,
          O.gen("random", 3000, 0.002, seed=4), sparse, O.gen("path", 9000), O.gen("kron", 12)]
    h = rst.DeviceGraph.from_host(gs[0].n, np.stack([gs[0].eu, gs[0].ev], 1))
    for g in gs:
        root = int(np.argmax(np.diff(g.offsets)))
        h.upload(g.n, np.stack([g.eu, g.ev], 1))
        for algo in (1, 0, 1):  # cc-euler, BFS (borrows the min table), cc-euler
            p, r, _, _ = h.run(algo, root)
            ep, er, _ = O.run(g, algo, root)
            assert np.array_equal(p, ep), (g.n, algo)
            assert np.array_equal(r, er), (g.n, algo)
    h.close()


def test_step_counts_rerun_identical(rst, O):
    # acceptance.cpp:330-363 (criterion 7): parents, steps and work are
    # bit-identical across reruns -- with the CSR given or built on the
    # device, and whether round 0 reads upload keys, recomputed keys or CSR
    for g in (O.gen("random", 1000, 0.01, seed=3), O.gen("grid", 50, 50), O.gen("kron", 12)):
        for csr in (True, False):
            extra = (g.offsets, g.nbrs, g.origin) if csr else ()
            dg = rst.DeviceGraph.from_host(g.n, np.stack([g.eu, g.ev], 1), *extra)
            for algo in ALGOS:
                res = [dg.run(algo, 0) for _ in range(3)]
                for p, _, _, st in res[1:]:
                    assert np.array_equal(p, res[0][0])
                    assert (st["steps"], st["work"]) == (res[0][3]["steps"], res[0][3]["work"]), (algo, csr)
            dg.close()


# ---- device forest_depth --------------------------------
def test_forest_depth_device(rst, O):
    for spec, root in ((("road", 300), 0), (("kron", 13), 5), (("path", 5000), 4999), (("grid", 40, 60), 77)):
        g = O.gen(*spec)
        dg = dev_graph(rst, g)
        for algo in ALGOS:
            p = O.run(g, algo, root)[0]
            depth, rmax, best = dg.forest_depth(p)
            assert best == O.forest_depth(p), (spec, algo)
            # per-vertex depth against a direct walk, per-root maxima against the depths
            for v in range(0, g.n, max(1, g.n // 97)):
                d, x = 0, v
                while p[x] != x:
                    x, d = p[x], d + 1
                assert depth[v] == d
            roots = np.nonzero(p == np.arange(g.n))[0]
            assert (rmax[roots] >= 0).all() and (np.delete(rmax, roots) == -1).all()
        dg.close()
    g = O.gen("path", 8)
    dg = dev_graph(rst, g)
    cyc = np.array([1, 2, 0, 3, 3, 4, 5, 6], np.int64)
    with pytest.raises(rst.RSTError, match="parent array contains a cycle at vertex 0"):
        dg.forest_depth(cyc)
    with pytest.raises(rst.RSTError, match="parent out of range at vertex 2"):
        dg.forest_depth(np.array([0, 0, 9, 2, 3, 4, 5, 6], np.int64))
    tail = np.array([5, 0, 1, 3, 3, 6, 5, 6], np.int64)  # 0 -> 5 -> 6 -> 5: the walk meets 5 twice
    with pytest.raises(rst.RSTError, match="parent array contains a cycle at vertex 5"):
        dg.forest_depth(tail)
    with pytest.raises(O.OracleError, match="cycle at vertex 5"):
        O.forest_depth(tail)
    dg.close()


def test_handle_reuse_unconsumed_upload(rst, O):
    # an upload whose round-0 keys are never consumed,
    # then a smaller graph that completes cc-euler, then a larger one: the
    # slot entries past the smaller graph's n must not leak into the third
    a, b, c = O.gen("kron", 12), O.gen("grid", 20, 25), O.gen("road", 70)
    h = rst.DeviceGraph.from_host(a.n, np.stack([a.eu, a.ev], 1))  # keys left in the slots
    for g in (b, c, a, b, a):
        h.upload(g.n, np.stack([g.eu, g.ev], 1))
        p, r, _, _ = h.run(1, 0)
        ep, er, _ = O.run(g, 1, 0)
        assert np.array_equal(p, ep) and np.array_equal(r, er), g.n
    # uploads never consumed in between, larger then smaller
    h.upload(a.n, np.stack([a.eu, a.ev], 1))
    h.upload(b.n, np.stack([b.eu, b.ev], 1))
    p, r, _, _ = h.run(1, 0)
    assert np.array_equal(p, O.run(b, 1, 0)[0])
    h.upload(a.n, np.stack([a.eu, a.ev], 1))
    for algo in ALGOS:
        assert np.array_equal(h.run(algo, 0)[0], O.run(a, algo, 0)[0]), algo
    h.close()


@pytest.mark.parametrize("algo", [2, 1, 0])
@pytest.mark.parametrize("spec,root", [(("road", 60), 0), (("kron", 11), 5), (("grid", 30, 40), 77)])
def test_edge_list_upload_each_strategy_first(rst, O, spec, root, algo):
    # an edge-list upload leaves the CSR pending (built on first use): each
    # strategy run FIRST on such a handle takes its no-CSR path (PR-RST: the
    # graft loop instead of the fused round-0 pass; cc-euler: keyed round 0)
    g = O.gen(*spec)
    h = rst.DeviceGraph.from_host(g.n, np.stack([g.eu, g.ev], 1))
    p, r, _, _ = h.run(algo, root)
    ep, er, _ = O.run(g, algo, root)
    assert np.array_equal(p, ep) and np.array_equal(r, er)
    # and then the others on the same handle
    for a2 in (0, 1, 2):
        assert np.array_equal(h.run(a2, root)[0], O.run(g, a2, root)[0])
    h.close()


def test_edge_upload_rejects_bad_edge_lists(rst, O):
    # build_csr's argument checks (graph.cpp:145-156),
    # on the device, in the reference's order, for the edge-list upload
    ok = np.array([[0, 1], [1, 2], [2, 3]], np.int64)
    cases = [
        (np.array([[0, 1], [1, 7], [2, 3]]), "edge endpoint out of range"),
        (np.array([[0, 1], [-1, 2], [2, 3]]), "edge endpoint out of range"),
        (np.array([[0, 1], [2, 2], [2, 3]]), "self-loop in normalized EdgeList"),
        (np.array([[0, 1], [2, 2], [2, 9]]), "self-loop in normalized EdgeList"),  # first offender
        (np.array([[0, 1], [2, 3], [1, 2]]), "EdgeList not normalized"),
        (np.array([[0, 1], [1, 2], [1, 2]]), "EdgeList not normalized"),  # duplicate
    ]
    for edges, msg in cases:
        with pytest.raises(rst.RSTArgError, match=msg):
            rst.DeviceGraph.from_host(4, edges.astype(np.int64))
    h = rst.DeviceGraph.from_host(4, ok)
    with pytest.raises(rst.RSTArgError, match="edge endpoint out of range"):
        h.upload(4, np.array([[0, 1], [1, 4]], np.int64))
    # the handle is usable again after a rejected upload
    h.upload(4, ok)
    assert list(h.run(1, 0)[0]) == [0, 0, 1, 2]
    h.close()
    # chunk boundaries (4M edges per staging chunk): an order violation
    # exactly across the boundary is seen
    g = O.gen("path", (1 << 22) + 3)
    e = np.stack([g.eu, g.ev], 1).copy()
    e[[(1 << 22) - 1, 1 << 22]] = e[[1 << 22, (1 << 22) - 1]]
    with pytest.raises(rst.RSTArgError, match="EdgeList not normalized"):
        rst.DeviceGraph.from_host(g.n, e)


def test_euler_root_forest_error_order(rst, O):
    # the edge count is checked before the tour
    # (euler_rooting.cpp:205-208); duplicate/self-loop tree edges with the
    # right count fail in list ranking; labels out of range are rejected
    with pytest.raises(rst.RSTError, match="edge count does not match a spanning forest"):
        rst.euler_root_forest(3, [(0, 1), (0, 1), (1, 2)], [0, 0, 0], -1)
    with pytest.raises(rst.RSTError, match="edge count does not match a spanning forest"):
        rst.euler_root_forest(4, [(0, 1), (2, 2)], [0, 0, 0, 0], -1)
    with pytest.raises(rst.RSTError, match="list ranking failed to converge: not a forest"):
        rst.euler_root_forest(3, [(0, 1), (0, 1)], [0, 0, 0], -1)
    with pytest.raises(rst.RSTError, match="list ranking failed to converge: not a forest"):
        rst.euler_root_forest(3, [(0, 1), (2, 2)], [0, 0, 0], -1)
    with pytest.raises(rst.RSTError, match="label out of range at vertex 1"):
        rst.euler_root_forest(3, [(0, 1), (1, 2)], [0, 5, 0], -1)
    with pytest.raises(rst.RSTError, match="label out of range at vertex 2"):
        rst.euler_root_forest(3, [(0, 1), (1, 2)], [0, 0, -1], -1)
    # unsorted, reversed tree edges are fine (arc order never changes parents)
    p, r = rst.euler_root_forest(4, [(3, 2), (1, 0), (2, 0)], [0] * 4, 3)
    ep, er = O.euler_root_forest(4, [(3, 2), (1, 0), (2, 0)], [0] * 4, 3)
    assert np.array_equal(p, ep) and list(r) == [3]


def test_euler_structure_api(rst, O):
    # the reference's arc-level API (euler_rooting.hpp:18-59) on the device:
    # build_euler layout against a direct restatement, successors and ranks
    # against the reference's own values (tests/golden/euler_ranks.npz, made
    # by the reference's compute_successor/break_cycles/list_rank), parents
    # against euler_root_forest
    d = np.load(_os.path.join(_os.path.dirname(__file__), "golden", "euler_ranks.npz"))
    for t in range(20):
        n, te = int(d[f"t{t}_n"][0]), d[f"t{t}_edges"]
        es = rst.EulerStructure(n, te)
        T = len(te)
        fr = np.concatenate([te[:, 0], te[:, 1]]); to = np.concatenate([te[:, 1], te[:, 0]])
        assert np.array_equal(es.from_, fr) and np.array_equal(es.to, to)
        order = np.lexsort((to, fr))
        first = np.full(n, -1); last = np.full(n, -1); nxt = np.full(2 * T, -1)
        for k, e in enumerate(order):
            v = fr[e]
            if k == 0 or fr[order[k - 1]] != v:
                first[v] = e
            if k + 1 < len(order) and fr[order[k + 1]] == v:
                nxt[e] = order[k + 1]
            else:
                last[v] = e
        assert np.array_equal(es.first, first) and np.array_equal(es.last, last)
        assert np.array_equal(es.next, nxt)
        es.compute_successor()
        es.break_cycles([0])
        assert np.array_equal(es.succ, d[f"t{t}_succ"]), t
        rank = es.list_rank()
        assert np.array_equal(rank, d[f"t{t}_rank"]), t
        p = es.derive_parents(rank)
        ep, _ = O.euler_root_forest(n, te, [0] * n, 0)
        assert np.array_equal(p, ep), t
    # edge cases: no arcs, and a root without arcs in a forest
    es = rst.EulerStructure(3, np.zeros((0, 2), np.int64))
    assert list(es.first) == [-1, -1, -1] and es.num_arcs == 0
    es = rst.EulerStructure(4, [(1, 2), (2, 3)])
    es.compute_successor()
    es.break_cycles([0, 1])
    assert list(es.derive_parents(es.list_rank())) == [0, 1, 1, 2]


def test_reference_acceptance_binary_unchanged():
    # the reference's OWN acceptance suite (proj/tests/acceptance.cpp),
    # compiled unchanged against the rst:: mirror headers (Makefile
    # build/ref_acceptance) and run on the GPU library: 9 PASS lines
    import os
    import subprocess
    exe = _os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))), "build",
                        "ref_acceptance")
    if not os.path.exists(exe):
        pytest.skip("build/ref_acceptance not built (reference sources absent at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS  criterion") == 9 and "all 9 criteria passed" in r.stdout


# ---- full-size parity pinned to the REFERENCE itself ----------------------------
# tests/golden/full_digests.json: sha256 of the reference's own outputs
# (oracle/_ref run_algorithm / cc_spanning_forest on 8 host cores,
# tests/golden/make_full_digests.py) for every BASELINE config that fits one
# host, and of the edge list the reference was given.
import hashlib as _hashlib
import json as _json

_DIGESTS_PATH = _os.path.join(_os.path.dirname(__file__), "golden", "full_digests.json")
_DIGESTS = _json.load(open(_DIGESTS_PATH)) if _os.path.exists(_DIGESTS_PATH) else {}


def _sha(*arrays):
    h = _hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a, dtype="<i8").tobytes())
    return h.hexdigest()


@pytest.mark.slow
@pytest.mark.parametrize("name", sorted(_DIGESTS))
def test_full_size_reference_digests(rst, name):
    rec = _DIGESTS[name]
    dg = rst.DeviceGraph.generate(name)
    assert (dg.n, dg.m) == (rec["n"], rec["m"])
    e = dg.edges()
    assert _sha(e[:, 0], e[:, 1]) == rec["edges"], "device generator != the reference's input"
    del e
    root = rec["root"]
    labels, te = dg.cc_spanning_forest()
    assert _sha(labels) == rec["cc_labels"] and _sha(te) == rec["cc_tree_edges"]
    for algo, tag in ((1, "cc_euler"), (2, "pr_rst"), (0, "bfs")):
        if algo == 0 and name.startswith("path"):
            continue  # 16.7M BFS levels: minutes per build (bench excludes it too)
        p, r, lv, _ = dg.run(algo, root)
        want = rec[tag]
        assert _sha(p) == want["parent"], f"{name} {tag}: parent differs from the {want['source']}"
        assert _sha(r) == want["roots"] and len(r) == want["num_roots"], f"{name} {tag}: roots"
        if algo == 0:
            assert _sha(lv) == want["levels"], f"{name}: bfs levels"
    dg.close()


def test_kron_verification_script_small(tmp_path):
    # scripts/verify_kron28.py (the config-5 record) end to end at scale 16,
    # including the 2-process partitioned run sharing the GPU
    import json
    import subprocess
    import sys
    root = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
    out = tmp_path / "v.json"
    r = subprocess.run([sys.executable, _os.path.join(root, "scripts", "verify_kron28.py"),
                        "--scale", "16", "--ranks", "2", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    rec = json.load(open(out))
    assert rec["verified"] and rec["components"] == 18656  # SURVEY.md Appendix B, s=16
    assert all(x["labels_equal_1gpu"] for x in rec["partitioned"]["per_rank"])
