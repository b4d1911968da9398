"""The edge-list / MatrixMarket loader (load_edge_list,
graph.cpp:48-127) against the reference's own loader (oracle/_ref).

CPU: the parse stage (rstg_parse_edge_text: host threads, no device) --
accepted pairs in file order, and the error message AND line number of the
first offending line, on hand-made texts (comments, MatrixMarket banner and
size line, CRLF, tabs, blank lines) and on random texts with injected
faults, chunked over several threads.
GPU: the full load (parse + device id remap + device normalize) equals the
reference's EdgeList (num_vertices, edges, original_ids) bit for bit, and a
graph made from it builds the same RST.
"""
import numpy as np
import pytest

VALID = [
    b"0 1\n1 2\n2 0\n",
    b"# comment\n\n  % other\n0\t1\n1 2 \n  3    2\n",
    b"%%MatrixMarket matrix coordinate pattern general\n% c\n4 4 3\n1 2\n2 3\n3 4\n",
    b"%%MatrixMarket\n3 3\n",                       # banner but a 2-token first line: data
    b"0 1\r\n1 2\r\n\r\n2 3",                         # CRLF, no final newline
    b"5 7\n7 5\n5 5\n9 7\n",                          # sparse ids, duplicate, self-loop
    b"100 200\n300 100\n200 300\n",
    b"0 0\n1 1\n0 1\n",
    b"  # indented comment\n\t% tab comment\n10 20\n",
    b"0 1\n" * 5,
]
ERRORS = [
    b"0 1\n1 x\n",            # expected integer, got 'x'
    b"0 1\n1 2 3\n",          # expected 2 integer tokens, got 3
    b"0 1\n1\n",              # got 1
    b"0 -1\n",                # negative vertex id
    b"0 1\n1 2 3 4\n",        # got 4
    b"4 4 3\n1 2\n",          # size line without banner
    b"%%MatrixMarket\n4 4 3 9\n1 2\n",
    b"0 1\n1 2\r3\n",         # a CR inside a token
    b"0 1\n99999999999999999999 1\n",  # out of int64 range
    b"0 1\n+1 2\n",
    b"",
    b"# nothing\n% at all\n",
    b"%%MatrixMarket\n3 3 2\n",
]


def _random_text(rs, lines, fault=None):
    out = []
    for i in range(lines):
        r = rs.rand()
        if r < 0.05:
            out.append("# c %d" % i)
        elif r < 0.08:
            out.append("")
        else:
            u, v = rs.randint(0, 5000), rs.randint(0, 5000)
            sep = " " if rs.rand() < 0.7 else "\t"
            out.append("%d%s%d" % (u, sep, v) + (" " if rs.rand() < 0.1 else ""))
    if fault is not None:
        k, bad = fault
        out[k] = bad
    return ("\n".join(out) + "\n").encode()


def _ref_parse(O, text):
    try:
        return O.ref_load_edge_list(text), None
    except O.OracleError as e:
        return None, (str(e), e.line)


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_parse_matches_reference_errors(rsth, O, threads):
    if not O.have_ref():
        pytest.skip("reference not built")
    for text in VALID + ERRORS:
        ref, err = _ref_parse(O, text)
        if err is not None and err[1] >= 0:
            with pytest.raises(rsth.RSTParseError) as ei:
                rsth.parse_edge_text(text, threads)
            assert str(ei.value) == err[0] and ei.value.line == err[1], text
        else:
            pairs = rsth.parse_edge_text(text, threads)  # (empty text: no pairs, no parse error)
            if ref is not None:
                n, eu, ev, ids = ref
                assert len(pairs) >= len(eu)


def test_parse_pairs_in_file_order(rsth):
    pairs = rsth.parse_edge_text(b"# c\n3 4\n\n1\t2\r\n5 6", 4)
    assert pairs.tolist() == [[3, 4], [1, 2], [5, 6]]
    mm = b"%%MatrixMarket matrix coordinate pattern general\n% c\n4 4 3\n1 2\n2 3\n3 4\n"
    assert rsth.parse_edge_text(mm).tolist() == [[1, 2], [2, 3], [3, 4]]


@pytest.mark.parametrize("seed", range(6))
def test_parse_random_texts_chunked(rsth, O, seed):
    # >1 MiB so the parse is cut into per-thread chunks; a fault on a random
    # line must be reported with the reference's line number and message
    rs = np.random.RandomState(seed)
    lines = 120000
    faults = [None, (int(rs.randint(0, lines)), "1 2 3"), (int(rs.randint(0, lines)), "7 q"),
              (int(rs.randint(0, lines)), "-4 2"), (int(rs.randint(lines - 10, lines)), "1"),
              (int(rs.randint(0, 50)), "x")]
    text = _random_text(rs, lines, faults[seed])
    assert len(text) > (1 << 20)
    ref, err = _ref_parse(O, text) if O.have_ref() else (None, None)
    for threads in (1, 5, 16):
        if faults[seed] is None:
            pairs = rsth.parse_edge_text(text, threads)
            want = [ln.split() for ln in text.decode().split("\n")
                    if ln.strip() and not ln.strip().startswith("#")]
            assert len(pairs) == len(want)
            assert pairs[:50].tolist() == [[int(a), int(b)] for a, b in want[:50]]
        else:
            with pytest.raises(rsth.RSTParseError) as ei:
                rsth.parse_edge_text(text, threads)
            assert ei.value.line == faults[seed][0] + 1
            if err is not None:
                assert (str(ei.value), ei.value.line) == err


# ---- full load on the device ---------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("text", VALID, ids=range(len(VALID)))
def test_load_matches_reference(rst, O, text):
    n, eu, ev, ids = O.ref_load_edge_list(text)
    gn, e, gids = rst.load_edge_list(text)
    assert gn == n and np.array_equal(e[:, 0], eu) and np.array_equal(e[:, 1], ev)
    assert np.array_equal(gids, ids)


@pytest.mark.gpu
def test_load_errors_match_reference(rst, O):
    for text in ERRORS:
        ref, err = _ref_parse(O, text)
        assert err is not None
        if err[1] >= 0:
            with pytest.raises(rst.RSTParseError) as ei:
                rst.load_edge_list(text)
            assert (str(ei.value), ei.value.line) == err
        else:
            with pytest.raises(rst.RSTError, match=err[0]):
                rst.load_edge_list(text)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,sparse", [(1, False), (2, True), (3, True)])
def test_load_random_graph_then_rst(rst, O, seed, sparse):
    # a road-like file (dense or sparse ids), loaded on the device, equals the
    # reference's EdgeList; the graph built from it gives the reference's RST
    g = O.gen("road", 150)
    rs = np.random.RandomState(seed)
    perm = rs.permutation(g.n).astype(np.int64)
    ids = perm * 1000 + 7 if sparse else perm
    order = rs.permutation(g.m)
    lines = ["%d %d" % (ids[g.ev[i]], ids[g.eu[i]]) for i in order]
    text = ("# road\n" + "\n".join(lines) + "\n").encode()
    n, eu, ev, oids = O.ref_load_edge_list(text)
    gn, e, gids = rst.load_edge_list(text)
    assert gn == n and np.array_equal(e[:, 0], eu) and np.array_equal(e[:, 1], ev)
    assert np.array_equal(gids, oids)
    dg = rst.DeviceGraph.from_edge_list_text(text)
    h = O.Graph(n, eu, ev)
    for algo in (0, 1, 2):
        assert np.array_equal(dg.run(algo, 3)[0], O.run(h, algo, 3)[0]), algo
    dg.close()
