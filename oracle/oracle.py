"""TEST INFRASTRUCTURE — ctypes front-ends for the two CPU checkers.

* ``RefOracle``  — the UNMODIFIED reference engine (oracle/_ref/libwfref.so, built
  by ``make -C oracle ref`` from /root/reference/proj sources + ref_harness.cpp).
* ``PortOracle`` — the plain-C restatement (oracle/liboracle.so, wf_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from paper_2107_11983_b200.abi import RunMetricsC, raise_for
from paper_2107_11983_b200.host import (ExecOptions, Graph, QuerySpec, RunMetrics, RunResult,
                                        WalkSet)

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libwfref.so")
PORT_LIB = os.path.join(HERE, "liboracle.so")

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_f64p = C.POINTER(C.c_double)
_f32p = C.POINTER(C.c_float)


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _digest_mix(x: np.ndarray) -> np.ndarray:
    x = x ^ (x >> np.uint64(30))
    x = x * np.uint64(0xBF58476D1CE4E5B9)
    x = x ^ (x >> np.uint64(27))
    x = x * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def walk_digest(walks, qid0: int, chunk: int = 1 << 17, threads: int = 0) -> int:
    """The 64-bit digest ref_harness.cpp:wfref_run_digest gives the block of
    query ids [qid0, qid0 + len(walks)): per walk mix(qid*K1 + (len << 8 |
    status) + K3) + sum over positions of mix(qid*K1 + pos*K2 + vertex), summed
    mod 2^64.  Chunks of walks are folded on a thread pool (numpy releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    k1, k2, k3 = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xC2B2AE3D27D4EB4F), np.uint64(0x632BE59BD9B4E019)
    n = len(walks)
    offsets = np.asarray(walks.offsets, dtype=np.uint64)

    def fold(a):
        b = min(n, a + chunk)
        with np.errstate(over="ignore"):
            lens = np.diff(offsets[a:b + 1])
            base = (np.arange(a, b, dtype=np.uint64) + np.uint64(qid0)) * k1
            head = base + ((lens << np.uint64(8)) | walks.status[a:b].astype(np.uint64)) + k3
            total = _digest_mix(head).sum(dtype=np.uint64)
            v0, v1 = int(offsets[a]), int(offsets[b])
            reps = lens.astype(np.int64)
            term = np.arange(v1 - v0, dtype=np.uint64) - np.repeat(offsets[a:b] - np.uint64(v0), reps)
            term *= k2
            term += np.repeat(base, reps)
            term += walks.vertices[v0:v1]
            return total + _digest_mix(term).sum(dtype=np.uint64)

    starts = range(0, n, chunk)
    if len(starts) <= 1:
        parts = [fold(a) for a in starts]
    else:
        with ThreadPoolExecutor(threads or min(16, os.cpu_count() or 1)) as pool:
            parts = list(pool.map(fold, starts))
    with np.errstate(over="ignore"):
        return int(np.sum(np.asarray(parts, dtype=np.uint64), dtype=np.uint64))


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


class _WfoGraph(C.Structure):
    _fields_ = [("offsets", _u64p), ("neighbors", _u32p), ("weights", _f32p),
                ("labels", _u8p), ("vertex_count", C.c_uint32), ("edge_count", C.c_uint64)]


class _WfoResult(C.Structure):
    _fields_ = [("n", C.c_uint64), ("offsets", _u64p), ("vertices", _u32p), ("status", _u8p),
                ("total_steps", C.c_uint64), ("exec_seconds", C.c_double),
                ("preprocess_seconds", C.c_double)]


class _WfoCsr(C.Structure):
    _fields_ = [("vertex_count", C.c_uint32), ("edge_count", C.c_uint64), ("offsets", _u64p),
                ("neighbors", _u32p), ("weights", _f32p), ("labels", _u8p)]


class PortOracle:
    """The C restatement (wf_oracle.c)."""

    def rmat(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, weighted=False,
             label_count=0, threads=0) -> Graph:
        """CPU R-MAT CSR (same definition as the device generator)."""
        g = _WfoCsr()
        rc = self.lib.wfo_rmat_csr(C.c_uint32(scale), C.c_uint32(edge_factor), C.c_double(a),
                                   C.c_double(b), C.c_double(c), C.c_uint64(seed),
                                   C.c_int(int(weighted)), C.c_uint32(label_count),
                                   C.c_int(threads), C.byref(g))
        raise_for(rc, "bad R-MAT parameters")
        try:
            V, E = g.vertex_count, g.edge_count
            off = np.ctypeslib.as_array(g.offsets, shape=(V + 1,)).copy()
            nbr = np.ctypeslib.as_array(g.neighbors, shape=(E,)).copy() if E else np.zeros(0, np.uint32)
            w = np.ctypeslib.as_array(g.weights, shape=(E,)).copy() if weighted and E else None
            lab = (np.ctypeslib.as_array(g.labels, shape=(E,)).copy()
                   if label_count and E else None)
        finally:
            self.lib.wfo_rmat_free(C.byref(g))
        return Graph(off, nbr, w, lab)

    def __init__(self, path: str = PORT_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        lib = C.CDLL(path)
        lib.wfo_run.restype = C.c_int
        lib.wfo_static_tables.restype = C.c_int
        lib.wfo_alias_init.restype = C.c_int
        self.lib = lib

    def _graph(self, g: Graph) -> _WfoGraph:
        if g.weights is not None and g.weights.dtype != np.float32:
            raise ValueError("the C restatement holds f32 weights; f64 graphs are checked against RefOracle")
        cg = _WfoGraph()
        cg.offsets = _ptr(g.offsets, _u64p)
        cg.neighbors = _ptr(g.neighbors, _u32p)
        cg.weights = _ptr(g.weights, _f32p)
        cg.labels = _ptr(g.labels, _u8p)
        cg.vertex_count = g.vertex_count
        cg.edge_count = g.edge_count
        return cg

    def rng_probe(self, seed: int, stream: int, draws: int) -> np.ndarray:
        out = np.zeros(draws, dtype=np.uint64)
        self.lib.wfo_rng_probe(C.c_uint64(seed), C.c_uint64(stream), C.c_uint32(draws),
                               _ptr(out, _u64p))
        return out

    def rng_index_real(self, seed, stream, n, bound):
        idx = C.c_uint32()
        real = C.c_double()
        self.lib.wfo_rng_index_real(C.c_uint64(seed), C.c_uint64(stream), C.c_uint32(n),
                                    C.c_double(bound), C.byref(idx), C.byref(real))
        return idx.value, real.value

    def alias_init(self, weights):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        n = w.size
        split = np.zeros(n, np.float64)
        first = np.zeros(n, np.uint32)
        second = np.zeros(n, np.uint32)
        err = C.create_string_buffer(256)
        rc = self.lib.wfo_alias_init(_ptr(w, _f64p), C.c_uint32(n), _ptr(split, _f64p),
                                     _ptr(first, _u32p), _ptr(second, _u32p), err, 256)
        raise_for(rc, err.value.decode())
        return split, first, second

    def run(self, g: Graph, spec: QuerySpec, prog, opts: ExecOptions,
            qids: Optional[np.ndarray] = None, threads: int = 1, discard: bool = False) -> RunResult:
        cg = self._graph(g)
        desc = prog.to_c()
        cspec = spec.to_c()
        copts = opts.to_c()
        res = _WfoResult()
        err = C.create_string_buffer(256)
        q = None if qids is None else np.ascontiguousarray(qids, dtype=np.uint64)
        rc = self.lib.wfo_run(C.byref(cg), C.byref(desc), C.byref(cspec), C.byref(copts),
                              _ptr(q, _u64p), C.c_uint64(0 if q is None else q.size),
                              C.c_int(threads), C.c_int(1 if discard else 0), C.byref(res),
                              err, 256)
        raise_for(rc, err.value.decode())
        try:
            n = res.n
            metrics = RunMetrics(res.preprocess_seconds, res.exec_seconds, res.total_steps, 1)
            if discard:
                ws = WalkSet(np.zeros(1, np.uint64), np.zeros(0, np.uint32), np.zeros(0, np.uint8))
            else:
                offsets = np.ctypeslib.as_array(res.offsets, shape=(n + 1,)).copy()
                verts = (np.ctypeslib.as_array(res.vertices, shape=(int(offsets[-1]),)).copy()
                         if offsets[-1] else np.zeros(0, np.uint32))
                status = (np.ctypeslib.as_array(res.status, shape=(n,)).copy()
                          if n else np.zeros(0, np.uint8))
                ws = WalkSet(offsets, verts, status, q)
        finally:
            self.lib.wfo_result_free(C.byref(res))
        return RunResult(ws, metrics)

    def static_tables(self, g: Graph, prog, sampler: int):
        v, e = g.vertex_count, g.edge_count
        out = dict(alias_split=np.zeros(e, np.float64), alias_first_dst=np.zeros(e, np.uint32),
                   alias_second_dst=np.zeros(e, np.uint32), its=np.zeros(e, np.float64),
                   rej_p_star=np.zeros(v, np.float64), exhausted=np.zeros(v, np.uint8))
        cg = self._graph(g)
        desc = prog.to_c()
        err = C.create_string_buffer(256)
        rc = self.lib.wfo_static_tables(C.byref(cg), C.byref(desc), C.c_int(sampler),
                                        _ptr(out["alias_split"], _f64p),
                                        _ptr(out["alias_first_dst"], _u32p),
                                        _ptr(out["alias_second_dst"], _u32p),
                                        _ptr(out["its"], _f64p), _ptr(out["rej_p_star"], _f64p),
                                        _ptr(out["exhausted"], _u8p), err, 256)
        raise_for(rc, err.value.decode())
        return out


class RefOracle:
    """The unmodified reference, through oracle/_ref/libwfref.so."""

    def __init__(self, path: str = REF_LIB):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference is mounted")
        lib = C.CDLL(path)
        lib.wfref_last_error.restype = C.c_char_p
        lib.wfref_synthetic_weight.restype = C.c_double
        lib.wfref_synthetic_label.restype = C.c_uint32
        lib.wfref_hardware_threads.restype = C.c_uint
        self.lib = lib

    def _check(self, rc):
        raise_for(rc, (self.lib.wfref_last_error() or b"").decode())

    # -- graphs ------------------------------------------------------------------
    def graph(self, g: Graph) -> "RefGraph":
        """Graph::from_csr over the device formats (f32 weights widened to f64,
        u8 labels widened to u32 inside the reference's own vectors)."""
        h = C.c_void_p()
        if g.weights is not None and g.weights.dtype == np.float64:
            lab = None if g.labels is None else np.ascontiguousarray(g.labels, dtype=np.uint32)
            self._check(self.lib.wfref_graph_create(
                _ptr(g.offsets, _u64p), _ptr(g.neighbors, _u32p), _ptr(g.weights, _f64p),
                _ptr(lab, _u32p), C.c_uint32(g.vertex_count), C.c_uint64(g.edge_count), C.byref(h)))
            return RefGraph(self, h)
        self._check(self.lib.wfref_graph_create_f32(
            _ptr(g.offsets, _u64p), _ptr(g.neighbors, _u32p), _ptr(g.weights, _f32p),
            _ptr(g.labels, _u8p), C.c_uint32(g.vertex_count), C.c_uint64(g.edge_count),
            C.byref(h)))
        return RefGraph(self, h)

    def rmat(self, scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, weighted=False,
             label_count=0, threads=0) -> "RefGraph":
        """The seeded R-MAT CSR built on the CPU by the C restatement of the
        generator (wfo_rmat_csr, bit-identical to the device build,
        tests/test_rmat_cpu.py) and handed straight to Graph::from_csr: no
        Python copies, so s26 (2.1 B edges) fits the host beside the
        reference's own f64 arrays and 24 B/edge alias tables."""
        port = PortOracle()
        g = _WfoCsr()
        rc = port.lib.wfo_rmat_csr(C.c_uint32(scale), C.c_uint32(edge_factor), C.c_double(a),
                                   C.c_double(b), C.c_double(c), C.c_uint64(seed),
                                   C.c_int(int(weighted)), C.c_uint32(label_count),
                                   C.c_int(threads), C.byref(g))
        raise_for(rc, "bad R-MAT parameters")
        try:
            h = C.c_void_p()
            self._check(self.lib.wfref_graph_create_f32(
                C.cast(g.offsets, _u64p), C.cast(g.neighbors, _u32p),
                C.cast(g.weights, _f32p) if weighted else None,
                C.cast(g.labels, _u8p) if label_count else None,
                C.c_uint32(g.vertex_count), C.c_uint64(g.edge_count), C.byref(h)))
        finally:
            port.lib.wfo_rmat_free(C.byref(g))
        return RefGraph(self, h)

    def power_law(self, vertex_count, edge_count, seed, exponent=0.8, weighted=False,
                  label_count=0) -> "RefGraph":
        h = C.c_void_p()
        self._check(self.lib.wfref_graph_power_law(C.c_uint32(vertex_count),
                                                   C.c_uint64(edge_count), C.c_double(exponent),
                                                   C.c_uint64(seed), C.c_int(int(weighted)),
                                                   C.c_uint32(label_count), C.byref(h)))
        return RefGraph(self, h)

    def load_edge_list(self, path, undirected=False, weights=0, labels=0, label_count=5,
                       seed=0):
        """load_edge_list through the reference; returns (RefGraph, original_ids)."""
        h = C.c_void_p()
        n = C.c_uint64()
        self._check(self.lib.wfref_load_edge_list(path.encode(), C.c_int(int(undirected)),
                                                  C.c_int(weights), C.c_int(labels),
                                                  C.c_uint32(label_count), C.c_uint64(seed),
                                                  C.byref(h), C.byref(n), None, C.c_uint64(0)))
        self.lib.wfref_graph_destroy(h)
        ids = np.zeros(n.value, np.uint64)
        h = C.c_void_p()
        self._check(self.lib.wfref_load_edge_list(path.encode(), C.c_int(int(undirected)),
                                                  C.c_int(weights), C.c_int(labels),
                                                  C.c_uint32(label_count), C.c_uint64(seed),
                                                  C.byref(h), C.byref(n), _ptr(ids, _u64p),
                                                  C.c_uint64(ids.size)))
        return RefGraph(self, h), ids

    def read_binary(self, path) -> "RefGraph":
        h = C.c_void_p()
        self._check(self.lib.wfref_graph_read_binary(path.encode(), C.byref(h)))
        return RefGraph(self, h)

    def ring(self, n, seed=0, weighted=False, label_count=0) -> "RefGraph":
        h = C.c_void_p()
        self._check(self.lib.wfref_graph_ring(C.c_uint32(n), C.c_uint64(seed),
                                              C.c_int(int(weighted)), C.c_uint32(label_count),
                                              C.byref(h)))
        return RefGraph(self, h)

    def build(self, vertex_count, edges, weights=None, labels=None) -> "RefGraph":
        e = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint32)
        h = C.c_void_p()
        self._check(self.lib.wfref_graph_build(C.c_uint32(vertex_count), _ptr(e, _u32p),
                                               C.c_uint64(e.shape[0]), _ptr(w, _f64p),
                                               _ptr(lab, _u32p), C.byref(h)))
        return RefGraph(self, h)

    # -- RNG ---------------------------------------------------------------------
    def rng_probe(self, seed, stream, draws):
        out = np.zeros(draws, dtype=np.uint64)
        self.lib.wfref_rng_probe(C.c_uint64(seed), C.c_uint64(stream), C.c_uint32(draws),
                                 _ptr(out, _u64p))
        return out

    def rng_index_real(self, seed, stream, n, bound):
        idx = C.c_uint32()
        real = C.c_double()
        self.lib.wfref_rng_index_real(C.c_uint64(seed), C.c_uint64(stream), C.c_uint32(n),
                                      C.c_double(bound), C.byref(idx), C.byref(real))
        return idx.value, real.value

    def alias_init(self, weights):
        w = np.ascontiguousarray(weights, dtype=np.float64)
        n = w.size
        split = np.zeros(n, np.float64)
        first = np.zeros(n, np.uint32)
        second = np.zeros(n, np.uint32)
        self._check(self.lib.wfref_alias_init(_ptr(w, _f64p), C.c_uint32(n), _ptr(split, _f64p),
                                              _ptr(first, _u32p), _ptr(second, _u32p)))
        return split, first, second

    def synthetic_weight(self, seed, edge):
        return self.lib.wfref_synthetic_weight(C.c_uint64(seed), C.c_uint64(edge))

    def synthetic_label(self, seed, edge, count):
        return self.lib.wfref_synthetic_label(C.c_uint64(seed), C.c_uint64(edge),
                                              C.c_uint32(count))

    def hardware_threads(self) -> int:
        return int(self.lib.wfref_hardware_threads())


class RefGraph:
    def __init__(self, ref: RefOracle, handle: C.c_void_p):
        self.ref = ref
        self.h = handle

    def __del__(self):
        try:
            if self.h:
                self.ref.lib.wfref_graph_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def info(self):
        v = C.c_uint32()
        e = C.c_uint64()
        hw = C.c_int()
        hl = C.c_int()
        md = C.c_uint64()
        mw = C.c_double()
        so = C.c_int()
        self.ref.lib.wfref_graph_info(self.h, C.byref(v), C.byref(e), C.byref(hw), C.byref(hl),
                                      C.byref(md), C.byref(mw), C.byref(so))
        return dict(V=v.value, E=e.value, has_weights=bool(hw.value), has_labels=bool(hl.value),
                    max_degree=md.value, max_weight=mw.value, sorted=bool(so.value))

    def export(self):
        """CSR arrays (weights f64, labels u32) as the reference holds them."""
        i = self.info()
        off = np.zeros(i["V"] + 1, np.uint64)
        nbr = np.zeros(i["E"], np.uint32)
        w = np.zeros(i["E"], np.float64) if i["has_weights"] else None
        lab = np.zeros(i["E"], np.uint32) if i["has_labels"] else None
        self.ref.lib.wfref_graph_export(self.h, _ptr(off, _u64p), _ptr(nbr, _u32p),
                                        _ptr(w, _f64p), _ptr(lab, _u32p))
        return off, nbr, w, lab

    def write_binary(self, path) -> None:
        self.ref._check(self.ref.lib.wfref_graph_write_binary(self.h, path.encode()))

    def has_edge(self, u, v) -> bool:
        return bool(self.ref.lib.wfref_has_edge(self.h, C.c_uint32(u), C.c_uint32(v)))

    def _collect(self, h, metrics: RunMetricsC, qids_given) -> RunResult:
        lib = self.ref.lib
        n = C.c_uint64()
        tv = C.c_uint64()
        lib.wfref_result_info(h, C.byref(n), C.byref(tv))
        qids = np.zeros(n.value, np.uint64)
        offsets = np.zeros(n.value + 1, np.uint64)
        verts = np.zeros(tv.value, np.uint32)
        status = np.zeros(n.value, np.uint8)
        lib.wfref_result_copy(h, _ptr(qids, _u64p), _ptr(offsets, _u64p), _ptr(verts, _u32p),
                              _ptr(status, _u8p))
        lib.wfref_result_destroy(h)
        m = RunMetrics(metrics.preprocess_seconds, metrics.exec_seconds, metrics.total_steps,
                       metrics.max_in_flight)
        return RunResult(WalkSet(offsets, verts, status, qids), m)

    def run(self, spec: QuerySpec, prog, opts: ExecOptions, interleaved: bool = False,
            discard: bool = False) -> RunResult:
        desc = prog.to_c()
        cspec = spec.to_c()
        copts = opts.to_c()
        h = C.c_void_p()
        m = RunMetricsC()
        self.ref._check(self.ref.lib.wfref_run(self.h, C.byref(desc), C.byref(cspec),
                                               C.byref(copts), C.c_int(int(interleaved)),
                                               C.c_int(int(discard)), C.byref(h), C.byref(m)))
        return self._collect(h, m, None)

    def run_encoded(self, spec: QuerySpec, prog, opts: ExecOptions, fmt: int,
                    path: Optional[str] = None) -> bytes:
        """run_sequential, then the reference's own record writers: the encoded
        bytes (append_text_record / append_binary_record), and with `path` the
        file written by DoubleBufferedWriter."""
        lib = self.ref.lib
        desc, cspec, copts = prog.to_c(), spec.to_c(), opts.to_c()
        h = C.c_void_p()
        m = RunMetricsC()
        self.ref._check(lib.wfref_run(self.h, C.byref(desc), C.byref(cspec), C.byref(copts),
                                      C.c_int(0), C.c_int(0), C.byref(h), C.byref(m)))
        try:
            n = C.c_uint64()
            self.ref._check(lib.wfref_encode(h, C.c_int(fmt), None, C.c_uint64(0), C.byref(n)))
            buf = C.create_string_buffer(max(n.value, 1))
            self.ref._check(lib.wfref_encode(h, C.c_int(fmt), buf, C.c_uint64(n.value), C.byref(n)))
            if path is not None:
                self.ref._check(lib.wfref_write_file(h, path.encode(), C.c_int(fmt)))
            return buf.raw[:n.value]
        finally:
            lib.wfref_result_destroy(h)

    def run_qids(self, spec: QuerySpec, prog, opts: ExecOptions, qids) -> RunResult:
        desc = prog.to_c()
        cspec = spec.to_c()
        copts = opts.to_c()
        q = np.ascontiguousarray(qids, dtype=np.uint64)
        h = C.c_void_p()
        m = RunMetricsC()
        self.ref._check(self.ref.lib.wfref_run_qids(self.h, C.byref(desc), C.byref(cspec),
                                                    C.byref(copts), _ptr(q, _u64p),
                                                    C.c_uint64(q.size), C.byref(h), C.byref(m)))
        return self._collect(h, m, q)

    def run_digest(self, spec: QuerySpec, prog, opts: ExecOptions, block_qids: int,
                   threads: int = 0):
        """Every query of the spec walked by the reference (ResolvedRun + StepDriver
        on `threads` host threads) and folded into one 64-bit digest per block of
        `block_qids` query ids, nothing stored: full-size parity (walk_digest is the
        same fold over a WalkSet).  Returns (digests u64[n_blocks], total_steps,
        preprocess_seconds)."""
        desc = prog.to_c()
        cspec = spec.to_c()
        copts = opts.to_c()
        n = (int(spec.sources.size) if spec.sources is not None
             else spec.count if spec.count else self.info()["V"])
        nb = (n + block_qids - 1) // block_qids
        out = np.zeros(nb, dtype=np.uint64)
        m = RunMetricsC()
        self.ref._check(self.ref.lib.wfref_run_digest(
            self.h, C.byref(desc), C.byref(cspec), C.byref(copts),
            C.c_uint32(threads or self.ref.hardware_threads()), C.c_uint64(block_qids),
            _ptr(out, _u64p), C.c_uint64(nb), C.byref(m)))
        return out, int(m.total_steps), float(m.preprocess_seconds)

    def run_test_program(self, which: int, params, spec: QuerySpec, opts: ExecOptions,
                         interleaved: bool = False):
        """One of the reference-API test programs in ref_harness.cpp (Counting,
        AvoidVertex, NegativeWeight, LabelWeight, LabelStop); returns
        (RunResult, update() calls of CountingProgram)."""
        cspec = spec.to_c()
        copts = opts.to_c()
        h = C.c_void_p()
        m = RunMetricsC()
        upd = C.c_uint64()
        self.ref._check(self.ref.lib.wfref_run_test_program(
            self.h, C.c_int(which), C.byref(params), C.byref(cspec), C.byref(copts),
            C.c_int(int(interleaved)), C.byref(h), C.byref(m), C.byref(upd)))
        return self._collect(h, m, None), upd.value

    def static_tables(self, prog, sampler: int):
        i = self.info()
        e, v = i["E"], i["V"]
        out = dict(alias_split=np.zeros(e, np.float64), alias_first=np.zeros(e, np.uint32),
                   alias_second=np.zeros(e, np.uint32), alias_first_dst=np.zeros(e, np.uint32),
                   alias_second_dst=np.zeros(e, np.uint32), its=np.zeros(e, np.float64),
                   rej_p_star=np.zeros(v, np.float64), exhausted=np.zeros(v, np.uint8))
        secs = C.c_double()
        desc = prog.to_c()
        self.ref._check(self.ref.lib.wfref_static_tables(
            self.h, C.byref(desc), C.c_int(sampler), _ptr(out["alias_split"], _f64p),
            _ptr(out["alias_first"], _u32p), _ptr(out["alias_second"], _u32p),
            _ptr(out["alias_first_dst"], _u32p), _ptr(out["alias_second_dst"], _u32p),
            _ptr(out["its"], _f64p), _ptr(out["rej_p_star"], _f64p), _ptr(out["exhausted"], _u8p),
            C.byref(secs)))
        out["seconds"] = secs.value
        return out
