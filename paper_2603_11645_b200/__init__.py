"""B200-native rooted-spanning-tree engine (arXiv 2603.11645 strategies).

Python binding over the C ABI in ``include/rstg.h`` (``librstg.so``, built
in-tree by ``make``). The reference is C++; its drop-in host API is the C++
``rst::`` mirror in ``host/`` (``librst_b200.so``). This module exists for
the tests and ``bench.py``: the same entry points, numpy in/out.

There is no CPU fallback: if the CUDA library cannot be loaded, or no GPU is
visible, calls raise.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# (RSTG_LIB_PATH: an experiment's alternative build of the same library)
LIB_PATH = os.environ.get("RSTG_LIB_PATH") or os.path.join(HERE, "librstg.so")

BFS, CC_EULER, PR_RST = 0, 1, 2  # bench.hpp:16 AlgoKind
ALGOS = {"bfs": BFS, "cc-euler": CC_EULER, "pr-rst": PR_RST}

RSTG_OK, RSTG_ERR_ARG, RSTG_ERR_ALGO, RSTG_ERR_CUDA, RSTG_ERR_PARSE = 0, 1, 2, 3, 4

# Symbols include/rstg.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "rstg_last_error", "rstg_device_count", "rstg_graph_create", "rstg_graph_create_device", "rstg_graph_upload",
    "rstg_graph_generate", "rstg_graph_info", "rstg_graph_edges", "rstg_graph_edges_flagged",
    "rstg_graph_destroy", "rstg_edge_list_load", "rstg_edge_list_info", "rstg_edge_list_copy",
    "rstg_edge_list_destroy", "rstg_graph_from_edge_list", "rstg_parse_edge_text",
    "rstg_set_stream", "rstg_set_timing", "rstg_phase_times", "rstg_run", "rstg_run_device",
    "rstg_cc_spanning_forest", "rstg_euler_root_forest", "rstg_validate", "rstg_forest_depth",
    "rstg_graph_generate_part", "rstg_graph_set_edge_base", "rstg_cc_init", "rstg_cc_hook",
    "rstg_cc_apply", "rstg_cc_compress", "rstg_cc_labels", "rstg_k_hook_step",
    "rstg_k_jump", "rstg_k_list_rank", "rstg_k_build_euler", "rstg_k_compute_successor",
    "rstg_k_break_cycles", "rstg_k_derive_parents",
)

_i64p = ctypes.POINTER(ctypes.c_int64)
# int (*rstg_reduce_min_fn)(void* ctx, int which, int64_t count)
REDUCE_MIN_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_vp = ctypes.c_void_p


class Stats(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int64), ("work", ctypes.c_int64), ("rounds", ctypes.c_int64),
                ("launches", ctypes.c_int64), ("tree_edges", ctypes.c_int64),
                ("components", ctypes.c_int64), ("levels", ctypes.c_int64),
                ("device_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class RSTError(RuntimeError):
    """Algorithm failure; message = the reference's std::runtime_error text."""


class RSTParseError(ValueError):
    """Malformed edge-list text (rst::ParseError); .line = 1-based line."""

    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


class RSTArgError(ValueError):
    """Invalid argument (reference: std::invalid_argument)."""


class CudaError(RuntimeError):
    pass


_lib = None


def lib():
    """Loads librstg.so (raises if it is missing: no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        L.rstg_last_error.restype = ctypes.c_char_p
        L.rstg_graph_create.argtypes = [_i64p, _i64p, _i64p, _i64p, ctypes.c_int64, ctypes.c_int64,
                                        ctypes.c_int, ctypes.POINTER(_vp)]
        L.rstg_graph_upload.argtypes = [_vp, _i64p, _i64p, _i64p, _i64p, ctypes.c_int64,
                                        ctypes.c_int64]
        L.rstg_graph_create_device.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_int, ctypes.POINTER(_vp)]
        L.rstg_graph_generate.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(_vp)]
        L.rstg_graph_info.argtypes = [_vp, _i64p, _i64p]
        L.rstg_graph_edges.argtypes = [_vp, _i64p]
        L.rstg_graph_edges_flagged.argtypes = [_vp, _vp, _i64p, ctypes.c_int64, _i64p]
        L.rstg_edge_list_load.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(_vp), _i64p]
        L.rstg_edge_list_info.argtypes = [_vp, _i64p, _i64p, _i64p]
        L.rstg_edge_list_copy.argtypes = [_vp, _i64p, _i64p]
        L.rstg_edge_list_destroy.argtypes = [_vp]
        L.rstg_graph_from_edge_list.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(_vp)]
        L.rstg_parse_edge_text.argtypes = [ctypes.c_char_p, ctypes.c_int64, ctypes.c_int, _i64p,
                                           ctypes.c_int64, _i64p, _i64p]
        L.rstg_graph_destroy.argtypes = [_vp]
        L.rstg_set_stream.argtypes = [_vp, _vp]
        L.rstg_set_timing.argtypes = [_vp, ctypes.c_int]
        L.rstg_phase_times.argtypes = [_vp, ctypes.c_char_p, ctypes.c_int64]
        L.rstg_run.argtypes = [_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _i64p, _i64p,
                               _i64p, _i64p, ctypes.POINTER(Stats)]
        L.rstg_run_device.argtypes = [_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _vp, _vp,
                                      ctypes.POINTER(Stats)]
        L.rstg_cc_spanning_forest.argtypes = [_vp, _i64p, _i64p, _i64p, ctypes.POINTER(Stats)]
        L.rstg_euler_root_forest.argtypes = [ctypes.c_int64, _i64p, ctypes.c_int64, _i64p,
                                             ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _i64p,
                                             _i64p, _i64p]
        L.rstg_forest_depth.argtypes = [_vp, _i64p, _i64p, _i64p, _i64p]
        L.rstg_validate.argtypes = [_vp, _i64p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_int), _i64p]
        L.rstg_graph_generate_part.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                               ctypes.c_int, ctypes.POINTER(_vp)]
        L.rstg_graph_set_edge_base.argtypes = [_vp, ctypes.c_int64]
        L.rstg_cc_init.argtypes = [_vp, _vp, _vp]
        L.rstg_cc_hook.argtypes = [_vp, ctypes.c_int, _vp, _vp]
        L.rstg_cc_apply.argtypes = [_vp, _vp, _vp, _vp, _i64p]
        L.rstg_cc_compress.argtypes = [_vp, _vp]
        L.rstg_cc_labels.argtypes = [_vp, _vp, _vp, _vp, _vp, REDUCE_MIN_FN, _vp,
                                     ctypes.POINTER(Stats)]
        L.rstg_k_hook_step.argtypes =[ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int, _i64p,
                                       _u8p, _i64p, ctypes.POINTER(ctypes.c_int)]
        L.rstg_k_jump.argtypes = [ctypes.c_int64, _i64p]
        L.rstg_k_list_rank.argtypes = [ctypes.c_int64, _i64p, _i64p]
        L.rstg_k_build_euler.argtypes = [ctypes.c_int64, _i64p, ctypes.c_int64] + [_i64p] * 5
        L.rstg_k_compute_successor.argtypes = [ctypes.c_int64, ctypes.c_int64] + [_i64p] * 4
        L.rstg_k_break_cycles.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i64p,
                                          ctypes.c_int64, _i64p]
        L.rstg_k_derive_parents.argtypes = [ctypes.c_int64, ctypes.c_int64] + [_i64p] * 4
        _lib = L
    return _lib


def _check(rc):
    if rc == RSTG_OK:
        return
    msg = lib().rstg_last_error().decode()
    if rc == RSTG_ERR_ALGO:
        raise RSTError(msg)
    if rc == RSTG_ERR_ARG:
        raise RSTArgError(msg)
    raise CudaError(msg)


def _p64(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def device_count() -> int:
    c = ctypes.c_int(0)
    _check(lib().rstg_device_count(ctypes.byref(c)))
    return c.value


class DeviceGraph:
    """Device-resident graph handle (rstg_graph)."""

    def __init__(self, handle):
        self._h = _vp(handle) if not isinstance(handle, _vp) else handle
        n, m = ctypes.c_int64(0), ctypes.c_int64(0)
        _check(lib().rstg_graph_info(self._h, ctypes.byref(n), ctypes.byref(m)))
        self.n, self.m = n.value, m.value

    # -- constructors --------------------------------------------------
    @classmethod
    def from_host(cls, n, edges_uv, offsets=None, neighbors=None, edge_origin=None, device=0):
        """From the reference's host layout (int64). edges_uv: (m, 2)."""
        e = np.ascontiguousarray(np.asarray(edges_uv, dtype=np.int64).reshape(-1, 2))
        h = _vp()
        _check(lib().rstg_graph_create(_p64(offsets), _p64(neighbors), _p64(edge_origin),
                                       _p64(e), int(n), len(e), device, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def generate(cls, spec: str, device=0):
        h = _vp()
        _check(lib().rstg_graph_generate(spec.encode(), device, ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, n, d_edges, d_offsets=None, d_nbrs=None, d_arc_edge=None, m=None,
                    device=0):
        """From device pointers (ints) to int32 arrays."""
        h = _vp()
        _check(lib().rstg_graph_create_device(_vp(d_edges), _vp(d_offsets), _vp(d_nbrs),
                                              _vp(d_arc_edge), int(n), int(m), device,
                                              ctypes.byref(h)))
        return cls(h)

    @classmethod
    def from_edge_list_text(cls, text: bytes, threads: int = 0, device=0):
        """load_edge_list on the device, then the graph from it (no host round trip)."""
        L = lib()
        el, line = _vp(), ctypes.c_int64(-1)
        rc = L.rstg_edge_list_load(text, len(text), threads or os.cpu_count() or 1, device,
                                   ctypes.byref(el), ctypes.byref(line))
        if rc == RSTG_ERR_PARSE:
            raise RSTParseError(L.rstg_last_error().decode(), line.value)
        _check(rc)
        try:
            h = _vp()
            _check(L.rstg_graph_from_edge_list(el, device, ctypes.byref(h)))
        finally:
            L.rstg_edge_list_destroy(el)
        return cls(h)

    @classmethod
    def generate_part(cls, spec: str, part: int, nparts: int, device=0):
        """Kronecker edges whose smaller endpoint is in part/nparts of [0, n)."""
        h = _vp()
        _check(lib().rstg_graph_generate_part(spec.encode(), part, nparts, device,
                                              ctypes.byref(h)))
        return cls(h)

    def set_edge_base(self, e_base: int):
        _check(lib().rstg_graph_set_edge_base(self._h, int(e_base)))

    # -- per-round connectivity kernels on caller device buffers (dist CC) --
    def cc_init(self, d_rep: int, d_slot: int):
        _check(lib().rstg_cc_init(self._h, _vp(d_rep), _vp(d_slot)))

    def cc_hook(self, mode: int, d_rep: int, d_slot: int):
        _check(lib().rstg_cc_hook(self._h, int(mode), _vp(d_rep), _vp(d_slot)))

    def cc_apply(self, d_rep: int, d_slot: int, d_tflag: int = 0) -> int:
        a = ctypes.c_int64(0)
        _check(lib().rstg_cc_apply(self._h, _vp(d_rep), _vp(d_slot), _vp(d_tflag or None),
                                   ctypes.byref(a)))
        return a.value

    def cc_compress(self, d_rep: int):
        _check(lib().rstg_cc_compress(self._h, _vp(d_rep)))

    def cc_labels(self, d_rep: int, d_tflag: int = 0, d_slot: int = 0, d_xbuf: int = 0,
                  reduce_min=None) -> dict:
        """rstg_cc_labels: converged labels (int32, device) through the
        optimised rounds; reduce_min(which, count) -> 0 MIN-combines the
        slots across ranks (edge-partitioned mode), None = one GPU."""
        st = Stats()
        cb = REDUCE_MIN_FN(lambda ctx, which, count: int(reduce_min(which, count))) \
            if reduce_min is not None else REDUCE_MIN_FN()
        _check(lib().rstg_cc_labels(self._h, _vp(d_rep), _vp(d_tflag or None),
                                    _vp(d_slot or None), _vp(d_xbuf or None), cb, None,
                                    ctypes.byref(st)))
        return st.as_dict()

    def upload(self, n, edges_uv, offsets=None, neighbors=None, edge_origin=None):
        """Re-uploads a graph into this handle (edges_uv int64, (m, 2) or flat)."""
        e = np.asarray(edges_uv)
        m = e.size // 2
        _check(lib().rstg_graph_upload(self._h, _p64(offsets), _p64(neighbors), _p64(edge_origin),
                                       e.ctypes.data_as(_i64p), int(n), int(m)))
        self.n, self.m = int(n), int(m)

    def close(self):
        if self._h:
            lib().rstg_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- accessors -----------------------------------------------------
    def edges(self) -> np.ndarray:
        out = np.zeros(2 * self.m, np.int64)
        _check(lib().rstg_graph_edges(self._h, _p64(out)))
        return out.reshape(-1, 2)

    def edges_flagged(self, d_flags: int, cap: int) -> np.ndarray:
        """Edges whose device uint8 flag is set, id order, (count, 2) int64."""
        out = np.zeros(2 * max(cap, 1), np.int64)
        c = ctypes.c_int64(0)
        _check(lib().rstg_graph_edges_flagged(self._h, _vp(d_flags), _p64(out), int(cap),
                                              ctypes.byref(c)))
        return out[: 2 * c.value].reshape(-1, 2)

    def set_stream(self, stream_ptr: int):
        _check(lib().rstg_set_stream(self._h, _vp(stream_ptr)))

    def set_timing(self, on: bool):
        _check(lib().rstg_set_timing(self._h, 1 if on else 0))

    def phase_times(self) -> dict:
        buf = ctypes.create_string_buffer(1 << 16)
        _check(lib().rstg_phase_times(self._h, buf, len(buf)))
        return json.loads(buf.value.decode() or "{}")

    # -- algorithms ----------------------------------------------------
    def run(self, algo, root=0, jump_batch=5, want_levels=None, out=None, want_roots=True):
        """run_algorithm: returns (parent, roots, levels|None, stats dict).

        out: optional int64 array (e.g. pinned) receiving the parent array."""
        algo = ALGOS.get(algo, algo)
        parent = out if out is not None else np.zeros(self.n, np.int64)
        levels = np.zeros(self.n, np.int64) if (algo == BFS and want_levels is not False) else None
        roots = np.zeros(max(self.n, 1), np.int64) if want_roots else None
        if roots is None:
            st = Stats()
            nr = ctypes.c_int64(0)
            _check(lib().rstg_run(self._h, algo, int(root), int(jump_batch), _p64(parent),
                                  _p64(levels), None, ctypes.byref(nr), ctypes.byref(st)))
            return parent, None, levels, st.as_dict()
        nr = ctypes.c_int64(0)
        st = Stats()
        _check(lib().rstg_run(self._h, algo, int(root), int(jump_batch), _p64(parent),
                              _p64(levels), _p64(roots), ctypes.byref(nr), ctypes.byref(st)))
        return parent, roots[: nr.value].copy(), levels, st.as_dict()

    def run_device(self, algo, root, d_parent: int, d_levels: int = 0, jump_batch=5):
        algo = ALGOS.get(algo, algo)
        st = Stats()
        _check(lib().rstg_run_device(self._h, algo, int(root), int(jump_batch), _vp(d_parent),
                                     _vp(d_levels or None), ctypes.byref(st)))
        return st.as_dict()

    def cc_spanning_forest(self):
        labels = np.zeros(self.n, np.int64)
        te = np.zeros(max(self.m, 1), np.int64)
        T = ctypes.c_int64(0)
        st = Stats()
        _check(lib().rstg_cc_spanning_forest(self._h, _p64(labels), _p64(te), ctypes.byref(T),
                                             ctypes.byref(st)))
        return labels, te[: T.value].copy()

    def forest_depth(self, parent):
        """forest_depth (rooted_forest.cpp:12-95) on the device:
        (depth per vertex, max depth per root (-1 off roots), max depth)."""
        p = np.ascontiguousarray(parent, dtype=np.int64)
        depth = np.zeros(max(self.n, 1), np.int64)
        rmax = np.zeros(max(self.n, 1), np.int64)
        best = ctypes.c_int64(0)
        _check(lib().rstg_forest_depth(self._h, _p64(p), _p64(depth), _p64(rmax),
                                       ctypes.byref(best)))
        return depth[: self.n], rmax[: self.n], best.value

    def validate(self, parent, required_root=-1):
        p = np.ascontiguousarray(parent, dtype=np.int64)
        valid, code, bad = ctypes.c_int(0), ctypes.c_int(0), ctypes.c_int64(0)
        _check(lib().rstg_validate(self._h, _p64(p), int(required_root), ctypes.byref(valid),
                                   ctypes.byref(code), ctypes.byref(bad)))
        return bool(valid.value), code.value, bad.value


def euler_root_forest(n, tree_edges, labels, designated_root=-1, device=0):
    te = np.ascontiguousarray(np.asarray(tree_edges, dtype=np.int64).reshape(-1, 2))
    lab = np.ascontiguousarray(np.asarray(labels, dtype=np.int64))
    parent = np.zeros(max(n, 1), np.int64)
    roots = np.zeros(max(n, 1), np.int64)
    nr = ctypes.c_int64(0)
    _check(lib().rstg_euler_root_forest(int(n), _p64(te), len(te), _p64(lab), len(lab),
                                        int(designated_root), device, _p64(parent), _p64(roots),
                                        ctypes.byref(nr)))
    return parent[:n], roots[: nr.value].copy()


def hook_step(n, edges_uv, mode, rep, tree_flag, slot):
    """hook_step on device; rep/tree_flag/slot updated in place."""
    e = np.ascontiguousarray(np.asarray(edges_uv, dtype=np.int64).reshape(-1, 2))
    applied = ctypes.c_int(0)
    _check(lib().rstg_k_hook_step(int(n), len(e), _p64(e), int(mode), _p64(rep),
                                  tree_flag.ctypes.data_as(_u8p), _p64(slot),
                                  ctypes.byref(applied)))
    return bool(applied.value)


def jump_to_convergence(rep):
    _check(lib().rstg_k_jump(len(rep), _p64(rep)))


def list_rank(succ):
    s = np.ascontiguousarray(np.asarray(succ, dtype=np.int64))
    rank = np.zeros(max(len(s), 1), np.int64)
    _check(lib().rstg_k_list_rank(len(s), _p64(s), _p64(rank)))
    return rank[: len(s)]


class EulerStructure:
    """The reference's arc-level Euler structure (euler_rooting.hpp:18-31),
    int64 arrays in its layout, each step one device call."""

    def __init__(self, n, tree_edges):
        te = np.ascontiguousarray(np.asarray(tree_edges, dtype=np.int64).reshape(-1, 2))
        self.num_vertices, self.num_arcs = int(n), 2 * len(te)
        E = self.num_arcs
        self.from_, self.to, self.next = (np.zeros(max(E, 1), np.int64) for _ in range(3))
        self.first, self.last = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), np.int64)
        _check(lib().rstg_k_build_euler(int(n), _p64(te), len(te), _p64(self.from_), _p64(self.to),
                                        _p64(self.first), _p64(self.last), _p64(self.next)))
        self.from_, self.to, self.next = self.from_[:E], self.to[:E], self.next[:E]
        self.first, self.last = self.first[:n], self.last[:n]
        self.succ = None

    def compute_successor(self):
        self.succ = np.zeros(max(self.num_arcs, 1), np.int64)
        _check(lib().rstg_k_compute_successor(self.num_vertices, self.num_arcs, _p64(self.from_),
                                              _p64(self.first), _p64(self.next), _p64(self.succ)))
        self.succ = self.succ[: self.num_arcs]

    def break_cycles(self, roots):
        r = np.ascontiguousarray(np.asarray(roots, dtype=np.int64))
        _check(lib().rstg_k_break_cycles(self.num_vertices, self.num_arcs, _p64(self.last), _p64(r),
                                         len(r), _p64(self.succ)))

    def list_rank(self):
        return list_rank(self.succ)

    def derive_parents(self, rank):
        parent = np.zeros(max(self.num_vertices, 1), np.int64)
        rk = np.ascontiguousarray(np.asarray(rank, dtype=np.int64))
        _check(lib().rstg_k_derive_parents(self.num_vertices, self.num_arcs, _p64(self.from_),
                                           _p64(self.to), _p64(rk), _p64(parent)))
        return parent[: self.num_vertices]


def parse_edge_text(text: bytes, threads: int = 0):
    """The loader's parse stage alone (host threads): raw (u, v) pairs in
    file order, int64 (count, 2); RSTParseError on malformed text."""
    L = lib()
    threads = threads or os.cpu_count() or 1
    c, line = ctypes.c_int64(0), ctypes.c_int64(-1)
    rc = L.rstg_parse_edge_text(text, len(text), threads, None, 0, ctypes.byref(c), ctypes.byref(line))
    if rc == RSTG_ERR_PARSE:
        raise RSTParseError(L.rstg_last_error().decode(), line.value)
    _check(rc)
    out = np.zeros(2 * max(c.value, 1), np.int64)
    _check(L.rstg_parse_edge_text(text, len(text), threads, _p64(out), c.value, ctypes.byref(c),
                                  ctypes.byref(line)))
    return out[: 2 * c.value].reshape(-1, 2)


def load_edge_list(text: bytes, threads: int = 0, device: int = 0):
    """load_edge_list (graph.cpp:48-127): (n, edges int64 (m, 2), original_ids)."""
    L = lib()
    h, line = _vp(), ctypes.c_int64(-1)
    rc = L.rstg_edge_list_load(text, len(text), threads or os.cpu_count() or 1, device,
                               ctypes.byref(h), ctypes.byref(line))
    if rc == RSTG_ERR_PARSE:
        raise RSTParseError(L.rstg_last_error().decode(), line.value)
    _check(rc)
    try:
        n, m, k = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_int64(0)
        _check(L.rstg_edge_list_info(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(k)))
        e = np.zeros(2 * max(m.value, 1), np.int64)
        ids = np.zeros(max(k.value, 1), np.int64)
        _check(L.rstg_edge_list_copy(h, _p64(e), _p64(ids)))
        return n.value, e[: 2 * m.value].reshape(-1, 2), ids[: k.value]
    finally:
        L.rstg_edge_list_destroy(h)
