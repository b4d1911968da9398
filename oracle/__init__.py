"""TEST INFRASTRUCTURE ONLY -- the checker, never the product.

ctypes bindings for the plain-C oracle restatement (``librst_oracle.so``) and
for the unmodified reference core compiled from /root/reference
(``_ref/librst_ref.so``). Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package. The product package (``paper_2603_11645_b200``) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "librst_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librst_ref.so")

_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
I64 = np.int64

ALGO_BFS, ALGO_CC_EULER, ALGO_PR_RST = 0, 1, 2  # bench.hpp:16 AlgoKind order


def build() -> None:
    """Compile the oracle (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "-j4"], check=True)


def _p(a):
    if a is None:
        return None
    if a.dtype == np.uint8:
        return a.ctypes.data_as(_u8p)
    assert a.dtype == I64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


class OracleError(RuntimeError):
    pass


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        L.og_last_error.restype = ctypes.c_char_p
        for name in ("og_normalize", "og_gen_path", "og_gen_star", "og_gen_grid",
                     "og_gen_random", "og_gen_complete", "og_gen_road", "og_gen_kron",
                     "og_cc_spanning_forest", "og_jump_to_convergence", "og_forest_depth",
                     "og_kron_uf", "og_uf_edges"):
            getattr(L, name).restype = ctypes.c_int64
        L.og_splitmix64.restype = ctypes.c_uint64
        L.og_splitmix64.argtypes = [ctypes.c_uint64]
        L.og_kron_perm.restype = ctypes.c_uint64
        L.og_kron_perm.argtypes = [ctypes.c_uint64, ctypes.c_int]
        _lib = L
    return _lib


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not have_ref():
            raise OracleError("reference library oracle/_ref/librst_ref.so not built")
        L = ctypes.CDLL(REF_SO)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_graph_create.restype = ctypes.c_void_p
        L.ref_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p]
        L.ref_graph_destroy.argtypes = [ctypes.c_void_p]
        L.ref_graph_run.restype = ctypes.c_double
        L.ref_graph_run.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_int64, _i64p]
        L.ref_generate.restype = ctypes.c_int64
        L.ref_generate.argtypes = [ctypes.c_char_p, ctypes.c_uint64, _i64p, _i64p, _i64p]
        L.ref_forest_depth.restype = ctypes.c_int64
        L.ref_load_edge_list.restype = ctypes.c_int64
        L.ref_load_edge_list.argtypes = [ctypes.c_char_p, ctypes.c_int64] + [_i64p] * 6
        _ref = L
    return _ref


def _err(L, fn="og_last_error"):
    return getattr(L, fn)().decode()


# ---------------------------------------------------------------- graphs
class Graph:
    """Host graph in the reference layout (graph.hpp:29-43), int64."""

    def __init__(self, n, eu, ev, normalized=True):
        eu = np.ascontiguousarray(eu, dtype=I64)
        ev = np.ascontiguousarray(ev, dtype=I64)
        if not normalized:
            eu, ev = eu.copy(), ev.copy()
            m = lib().og_normalize(len(eu), _p(eu), _p(ev))
            eu, ev = eu[:m].copy(), ev[:m].copy()
        self.n, self.m = int(n), int(len(eu))
        self.eu, self.ev = eu, ev
        self.offsets = np.zeros(self.n + 1, dtype=I64)
        self.nbrs = np.zeros(2 * self.m, dtype=I64)
        self.origin = np.zeros(2 * self.m, dtype=I64)
        rc = lib().og_build_csr(ctypes.c_int64(self.n), ctypes.c_int64(self.m), _p(self.eu),
                                _p(self.ev), _p(self.offsets), _p(self.nbrs), _p(self.origin))
        if rc != 0:
            raise ValueError(_err(lib()))


def _take_edges(m, peu, pev):
    L = lib()
    if m < 0:
        raise ValueError(_err(L))
    eu = np.ctypeslib.as_array(peu, shape=(m,)).copy() if m else np.zeros(0, I64)
    ev = np.ctypeslib.as_array(pev, shape=(m,)).copy() if m else np.zeros(0, I64)
    L.og_free(peu)
    L.og_free(pev)
    return eu, ev


def gen(kind: str, *params, seed: int = 0) -> Graph:
    """Oracle-side generators (graph.cpp:181-313 + SURVEY road/kron)."""
    L = lib()
    peu, pev = _i64p(), _i64p()
    if kind == "path":
        n = int(params[0]); m = L.og_gen_path(ctypes.c_int64(n), ctypes.byref(peu), ctypes.byref(pev))
    elif kind == "star":
        n = int(params[0]); m = L.og_gen_star(ctypes.c_int64(n), ctypes.byref(peu), ctypes.byref(pev))
    elif kind == "grid":
        r, c = int(params[0]), int(params[1]); n = r * c
        m = L.og_gen_grid(ctypes.c_int64(r), ctypes.c_int64(c), ctypes.byref(peu), ctypes.byref(pev))
    elif kind == "random":
        n = int(params[0])
        m = L.og_gen_random(ctypes.c_int64(n), ctypes.c_double(float(params[1])),
                            ctypes.c_uint64(seed), ctypes.byref(peu), ctypes.byref(pev))
    elif kind == "complete":
        n = int(params[0]); m = L.og_gen_complete(ctypes.c_int64(n), ctypes.byref(peu), ctypes.byref(pev))
    elif kind == "road":
        R = int(params[0]); p = float(params[1]) if len(params) > 1 else 0.2026; n = R * R
        m = L.og_gen_road(ctypes.c_int64(R), ctypes.c_double(p), ctypes.byref(peu), ctypes.byref(pev))
    elif kind == "kron":
        s = int(params[0]); ef = int(params[1]) if len(params) > 1 else 16; n = 1 << s
        m = L.og_gen_kron(ctypes.c_int(s), ctypes.c_int(ef), ctypes.byref(peu), ctypes.byref(pev))
    else:
        raise ValueError(f"unknown generator kind: {kind}")
    eu, ev = _take_edges(m, peu, pev)
    return Graph(n, eu, ev)


def from_edges(n, edges) -> Graph:
    """graph_from_edges (tests/oracles.hpp:487-493): normalize + CSR."""
    e = np.array(edges, dtype=I64).reshape(-1, 2)
    return Graph(n, e[:, 0], e[:, 1], normalized=False)


# ------------------------------------------------------------ algorithms
def cc_spanning_forest(g: Graph):
    L = lib()
    labels = np.zeros(g.n, I64)
    flag = np.zeros(max(g.m, 1), np.uint8)
    rounds = ctypes.c_int64(0)
    T = L.og_cc_spanning_forest(ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu), _p(g.ev),
                                _p(labels), _p(flag), ctypes.byref(rounds))
    if T < 0:
        raise OracleError(_err(L))
    return labels, np.nonzero(flag[: g.m])[0].astype(I64)


def hook_step(g: Graph, mode: int, rep, tree_flag, slot):
    r = lib().og_hook_step(ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu), _p(g.ev),
                           ctypes.c_int(mode), _p(rep), _p(tree_flag), _p(slot))
    if r < 0:
        raise OracleError(_err(lib()))
    return bool(r)


def jump_to_convergence(rep):
    s = lib().og_jump_to_convergence(ctypes.c_int64(len(rep)), _p(rep))
    if s < 0:
        raise OracleError(_err(lib()))
    return int(s)


def euler_root_forest(n, tree_edges, labels, designated_root=-1, ranks=False):
    te = np.array(tree_edges, dtype=I64).reshape(-1, 2)
    tu, tv = np.ascontiguousarray(te[:, 0]), np.ascontiguousarray(te[:, 1])
    labels = np.ascontiguousarray(labels, dtype=I64)
    if len(labels) != n:
        raise OracleError("labels size does not match vertex count")
    parent = np.zeros(n, I64)
    roots = np.zeros(max(n, 1), I64)
    nr = ctypes.c_int64(0)
    rk = np.zeros(max(2 * len(tu), 1), I64) if ranks else None
    rc = lib().og_euler_root_forest(ctypes.c_int64(n), ctypes.c_int64(len(tu)), _p(tu), _p(tv),
                                    _p(labels), ctypes.c_int64(designated_root), _p(parent),
                                    _p(roots), ctypes.byref(nr), _p(rk))
    if rc != 0:
        raise OracleError(_err(lib()))
    if ranks:
        return parent, roots[: nr.value].copy(), rk[: 2 * len(tu)].copy()
    return parent, roots[: nr.value].copy()


def run(g: Graph, algo: int, root: int = 0, jump_batch: int = 5, fast_bfs: bool = True):
    """Returns (parent, roots, levels|None) like run_algorithm's RootedForest."""
    L = lib()
    parent = np.zeros(g.n, I64)
    roots = np.zeros(max(g.n, 1), I64)
    nr = ctypes.c_int64(0)
    levels = None
    if algo == ALGO_CC_EULER:
        rc = L.og_cc_euler_rst(ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu), _p(g.ev),
                               ctypes.c_int64(root), _p(parent), _p(roots), ctypes.byref(nr))
    elif algo == ALGO_PR_RST:
        rc = L.og_pr_rst(ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu), _p(g.ev),
                         ctypes.c_int64(root), ctypes.c_int64(jump_batch), _p(parent), _p(roots),
                         ctypes.byref(nr))
    elif algo == ALGO_BFS:
        levels = np.zeros(g.n, I64)
        fn = L.og_bfs_rst_fast if fast_bfs else L.og_bfs_rst
        rc = fn(ctypes.c_int64(g.n), _p(g.offsets), _p(g.nbrs), ctypes.c_int64(root), _p(parent),
                _p(levels), _p(roots), ctypes.byref(nr))
    else:
        raise ValueError("bad algo")
    if rc != 0:
        raise OracleError(_err(L))
    return parent, roots[: nr.value].copy(), levels


def components(g: Graph):
    lab = np.zeros(g.n, I64)
    lib().og_components(ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu), _p(g.ev), _p(lab))
    return lab


def kron_uf(scale: int, edge_factor: int = 16, threads: int | None = None):
    """Host union-find over every Kronecker tuple, regenerated on the fly
    (kron_uf.c; the checker of config 5). Returns (root int32[n] = smallest
    id of each class, number of classes)."""
    n = 1 << scale
    root = np.empty(n, np.int32)
    c = lib().og_kron_uf(ctypes.c_int(scale), ctypes.c_int(edge_factor),
                         ctypes.c_int(threads or os.cpu_count() or 1),
                         root.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    if c < 0:
        raise OracleError("kron_uf: bad parameters")
    return root, int(c)


def uf_edges(n: int, uv, threads: int | None = None):
    """Host union-find over an explicit edge list (int32 pairs): (root, classes)."""
    uv = np.ascontiguousarray(np.asarray(uv, dtype=np.int32).reshape(-1, 2))
    root = np.empty(max(n, 1), np.int32)
    c = lib().og_uf_edges(ctypes.c_int64(n), ctypes.c_int64(len(uv)),
                          uv.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                          ctypes.c_int(threads or os.cpu_count() or 1),
                          root.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return root[:n], int(c)


def same_partition(labels, root) -> bool:
    """labels (any class representative per vertex, each a member of its
    class) and root (smallest id per class) describe the same partition:
    every vertex shares its label's class, and the class counts agree."""
    labels = np.asarray(labels)
    root = np.asarray(root)
    n = len(root)
    if len(labels) != n:
        return False
    if n == 0:
        return True
    if labels.min() < 0 or labels.max() >= n:
        return False
    if not np.array_equal(root[labels], root):
        return False
    return len(np.unique(labels)) == int(np.count_nonzero(root == np.arange(n)))


def validate(g: Graph, parent, roots=None, required_root=-1):
    parent = np.ascontiguousarray(parent, dtype=I64)
    r = None if roots is None else np.ascontiguousarray(roots, dtype=I64)
    ok = lib().og_validate(ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu), _p(g.ev),
                           _p(g.offsets), _p(g.nbrs), _p(parent), _p(r),
                           ctypes.c_int64(0 if r is None else len(r)),
                           ctypes.c_int64(required_root))
    return bool(ok), _err(lib())


def forest_depth(parent):
    parent = np.ascontiguousarray(parent, dtype=I64)
    d = lib().og_forest_depth(ctypes.c_int64(len(parent)), _p(parent))
    if d < 0:
        raise OracleError(_err(lib()))
    return int(d)


# ----------------------------------------------------- reference (_ref)
def ref_generate(spec: str, seed: int = 0) -> Graph:
    R = ref()
    n = ctypes.c_int64(0)
    m = R.ref_generate(spec.encode(), seed, ctypes.byref(n), None, None)
    if m < 0:
        raise ValueError(_err(R, "ref_last_error"))
    eu = np.zeros(m, I64)
    ev = np.zeros(m, I64)
    R.ref_generate(spec.encode(), seed, ctypes.byref(n), _p(eu), _p(ev))
    return Graph(n.value, eu, ev)


def ref_load_edge_list(text: bytes):
    """The reference's load_edge_list (graph.cpp:48-127) on an in-memory
    text: (n, eu, ev, original_ids), or raises OracleError(message) with
    .line set for a ParseError."""
    R = ref()
    n, nids, line = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(-1)
    m = R.ref_load_edge_list(text, len(text), ctypes.byref(n), None, None, None,
                             ctypes.byref(nids), ctypes.byref(line))
    if m < 0:
        e = OracleError(_err(R, "ref_last_error"))
        e.line = line.value
        raise e
    eu, ev, ids = np.zeros(max(m, 1), I64), np.zeros(max(m, 1), I64), np.zeros(max(nids.value, 1), I64)
    R.ref_load_edge_list(text, len(text), ctypes.byref(n), _p(eu), _p(ev), _p(ids),
                         ctypes.byref(nids), ctypes.byref(line))
    return n.value, eu[:m], ev[:m], ids[: nids.value]


def ref_run(g: Graph, algo: int, root: int = 0, workers: int = 1, jump_batch: int = 5):
    R = ref()
    parent = np.zeros(g.n, I64)
    levels = np.zeros(g.n, I64)
    roots = np.zeros(max(g.n, 1), I64)
    nr, steps, work = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
    rc = R.ref_run(ctypes.c_int(algo), ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu),
                   _p(g.ev), ctypes.c_int64(root), ctypes.c_int(workers),
                   ctypes.c_int64(jump_batch), _p(parent), _p(levels), _p(roots),
                   ctypes.byref(nr), ctypes.byref(steps), ctypes.byref(work))
    if rc != 0:
        raise OracleError(_err(R, "ref_last_error"))
    return parent, roots[: nr.value].copy(), (levels if algo == ALGO_BFS else None)


def ref_validate(g: Graph, parent, roots, required_root=-1):
    """The reference's validate_rooted_forest (validate.cpp:108-211):
    (valid, first error message or "")."""
    R = ref()
    parent = np.ascontiguousarray(parent, dtype=I64)
    roots = np.ascontiguousarray(roots, dtype=I64)
    rc = R.ref_validate(ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu), _p(g.ev), _p(parent),
                        _p(roots), ctypes.c_int64(len(roots)), ctypes.c_int64(required_root))
    if rc < 0:
        raise OracleError(_err(R, "ref_last_error"))
    return rc == 1, _err(R, "ref_last_error")


def ref_cc_spanning_forest(g: Graph, workers: int = 1):
    R = ref()
    labels = np.zeros(g.n, I64)
    te = np.zeros(max(g.m, 1), I64)
    T = ctypes.c_int64(0)
    rc = R.ref_cc_spanning_forest(ctypes.c_int64(g.n), ctypes.c_int64(g.m), _p(g.eu), _p(g.ev),
                                  ctypes.c_int(workers), _p(labels), _p(te), ctypes.byref(T), None)
    if rc != 0:
        raise OracleError(_err(R, "ref_last_error"))
    return labels, te[: T.value].copy()


def ref_euler_ranks(n, tree_edges, roots):
    te = np.array(tree_edges, dtype=I64).reshape(-1, 2)
    tu, tv = np.ascontiguousarray(te[:, 0]), np.ascontiguousarray(te[:, 1])
    roots = np.ascontiguousarray(roots, dtype=I64)
    E = 2 * len(tu)
    succ = np.zeros(max(E, 1), I64)
    rank = np.zeros(max(E, 1), I64)
    rc = ref().ref_euler_ranks(ctypes.c_int64(n), ctypes.c_int64(len(tu)), _p(tu), _p(tv),
                               _p(roots), ctypes.c_int64(len(roots)), _p(succ), _p(rank))
    if rc != 0:
        raise OracleError(_err(ref(), "ref_last_error"))
    return succ[:E].copy(), rank[:E].copy()


class RefGraph:
    """A reference Graph held across timing calls (bench --impl reference)."""

    def __init__(self, g: Graph):
        self.g = g
        self.h = ref().ref_graph_create(g.n, g.m, _p(g.eu), _p(g.ev))
        if not self.h:
            raise OracleError(_err(ref(), "ref_last_error"))

    def run_ms(self, algo, root=0, workers=1, jump_batch=5, parent=None):
        ms = ref().ref_graph_run(self.h, algo, root, workers, jump_batch, _p(parent))
        if ms < 0:
            raise OracleError(_err(ref(), "ref_last_error"))
        return ms

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_graph_destroy(self.h)
            self.h = None
