"""Python mirror of the reference's engine interface over the CUDA C-ABI.

    run_sequential(g, spec, prog, opts)            engine.hpp:440-504
    run_interleaved(g, spec, prog, k, k', opts)    interleave.hpp:391-556
    Session  ~ detail::ResolvedRun                 engine.hpp:275-294
    DeviceGraph ~ Graph resident in HBM            graph.hpp:17-107

All compute goes through paper_2107_11983_b200/libwalkforge_b200.so (sm_100a
kernels).  There is no CPU fallback: if the library or a device is missing,
every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import abi
from . import host as host_mod
from .abi import (ExecOptionsC, GraphInfoC, ProgramDesc, QuerySpecC, RmatParamsC, RunMetricsC,
                  raise_for)
from .host import ExecOptions, Graph, QuerySpec, RunMetrics, RunResult, WalkSet

LIB_PATH = os.environ.get("WF_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                 "libwalkforge_b200.so")

_u64p = C.POINTER(C.c_uint64)
# wf_block_fn: int (*)(void* user, uint64_t block, uint64_t qid_begin, uint64_t qid_end, uint64_t vertex_begin)
_BLOCK_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)
_f32p = C.POINTER(C.c_float)
_f64p = C.POINTER(C.c_double)
_vp = C.c_void_p

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Loads the engine; raises if it was not built (no silent fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: run paper_2107_11983_b200/build.py "
                           "(or __graft_entry__.build())")
    lib = C.CDLL(path)
    lib.wf_last_error.restype = C.c_char_p
    lib.wf_kernel_launches.restype = C.c_uint64
    for name in abi.EXPORTED_SYMBOLS:
        getattr(lib, name)  # every declared symbol must resolve
    _lib = lib
    return lib


_nccl_preloaded = False


def _preload_nccl() -> None:
    """The library dlopens "libnccl.so.2" at the first multi-device / communicator
    call and takes whatever is already loaded under that SONAME.  In a Python
    process that later imports torch, loading the SYSTEM libnccl first would
    leave torch resolving its own (newer) NCCL symbols against it and failing
    to import: so load the NCCL torch ships (site-packages/nvidia/nccl) first
    when it exists.  No torch NCCL: the system library, as before."""
    global _nccl_preloaded
    if _nccl_preloaded:
        return
    _nccl_preloaded = True
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations if spec else []):
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                C.CDLL(cand, mode=C.RTLD_GLOBAL)
                return
    except Exception:
        pass


def _check(rc: int) -> None:
    if rc != 0:
        raise_for(rc, (_lib.wf_last_error() or b"").decode())


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


def kernel_launches() -> int:
    return int(load_library().wf_kernel_launches())


class DeviceGraph:
    """A Graph resident in HBM (wf_graph)."""

    def __init__(self, handle: C.c_void_p):
        self.h = handle
        self._info = None

    @classmethod
    def from_host(cls, g: Graph, device: int = 0) -> "DeviceGraph":
        lib = load_library()
        h = _vp()
        # Graph::from_csr takes vectors: an empty attribute array means "absent"
        # (graph.cpp:118-159), which only shows on a graph without edges
        weights = g.weights if g.weights is not None and g.weights.size else None
        lab = None if g.labels is None or g.labels.size == 0 else g.labels.astype(np.uint32)
        if weights is not None and weights.dtype == np.float64:
            # the reference's f64 weights (wf_graph_create_f64)
            w = np.ascontiguousarray(weights)
            _check(lib.wf_graph_create_f64(_ptr(g.offsets, _u64p), _ptr(g.neighbors, _u32p),
                                           w.ctypes.data_as(C.POINTER(C.c_double)), _ptr(lab, _u32p),
                                           C.c_uint32(g.vertex_count), C.c_uint64(g.edge_count),
                                           C.c_int(device), C.byref(h)))
            return cls(h)
        _check(lib.wf_graph_create(_ptr(g.offsets, _u64p), _ptr(g.neighbors, _u32p),
                                   _ptr(weights, _f32p), _ptr(lab, _u32p),
                                   C.c_uint32(g.vertex_count), C.c_uint64(g.edge_count),
                                   C.c_int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def from_device(cls, offsets_ptr: int, neighbors_ptr: int, weights_ptr: int, labels_ptr: int,
                    vertex_count: int, edge_count: int, device: int = 0) -> "DeviceGraph":
        """From device pointers (e.g. torch tensor .data_ptr()); 0 = absent."""
        lib = load_library()
        h = _vp()
        _check(lib.wf_graph_create_device(_vp(offsets_ptr), _vp(neighbors_ptr),
                                          _vp(weights_ptr or None), _vp(labels_ptr or None),
                                          C.c_uint32(vertex_count), C.c_uint64(edge_count),
                                          C.c_int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def rmat(cls, scale: int, edge_factor: int = 16, a: float = 0.57, b: float = 0.19,
             c: float = 0.19, seed: int = 1, weighted: bool = False, label_count: int = 0,
             device: int = 0) -> "DeviceGraph":
        """Synthetic R-MAT (SURVEY §8 d), generated and CSR-built on the device."""
        lib = load_library()
        p = RmatParamsC(scale, edge_factor, a, b, c, seed, 1 if weighted else 0, label_count)
        h = _vp()
        _check(lib.wf_graph_generate_rmat(C.byref(p), C.c_int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def read_wfg1(cls, path: str, device: int = 0) -> "DeviceGraph":
        """Graph::read_binary (graph.cpp:215-277)."""
        h = _vp()
        _check(load_library().wf_graph_read_wfg1(path.encode(), C.c_int(device), C.byref(h)))
        return cls(h)

    @classmethod
    def load_edge_list(cls, path: str, undirected: bool = False, weights: int = 0,
                       labels: int = 0, label_count: int = 5, seed: int = 0,
                       device: int = 0) -> "DeviceGraph":
        """load_edge_list (graph.cpp:307-453); weights/labels: 0 none, 1 from
        file, 2 random (EdgeListOptions, graph.hpp:80-87)."""
        o = abi.EdgeListOptionsC(1 if undirected else 0, weights, labels, label_count, seed)
        h = _vp()
        _check(load_library().wf_graph_load_edge_list(path.encode(), C.byref(o), C.c_int(device),
                                                      C.byref(h)))
        return cls(h)

    def write_wfg1(self, path: str) -> None:
        """Graph::write_binary (graph.cpp:190-213)."""
        _check(load_library().wf_graph_write_wfg1(self.h, path.encode()))

    def original_ids(self) -> np.ndarray:
        out = np.zeros(self.vertex_count, np.uint64)
        _check(load_library().wf_graph_original_ids(self.h, _ptr(out, _u64p)))
        return out

    def __del__(self):
        try:
            if self.h:
                _lib.wf_graph_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def info(self) -> dict:
        if self._info is None:
            i = GraphInfoC()
            _check(load_library().wf_graph_info_get(self.h, C.byref(i)))
            self._info = dict(V=i.vertex_count, E=i.edge_count, max_degree=i.max_degree,
                              max_weight=i.max_weight, has_weights=bool(i.has_weights),
                              has_labels=bool(i.has_labels), sorted=bool(i.adjacency_sorted),
                              device=i.device, label_count=i.label_count,
                              weights_f64=bool(i.weights_f64))
        return self._info

    @property
    def vertex_count(self) -> int:
        return self.info()["V"]

    @property
    def edge_count(self) -> int:
        return self.info()["E"]

    def download(self) -> Graph:
        i = self.info()
        off = np.zeros(i["V"] + 1, np.uint64)
        nbr = np.zeros(i["E"], np.uint32)
        w = np.zeros(i["E"], np.float32) if i["has_weights"] else None
        lab = np.zeros(i["E"], np.uint8) if i["has_labels"] else None
        _check(load_library().wf_graph_download(self.h, _ptr(off, _u64p), _ptr(nbr, _u32p),
                                                _ptr(w, _f32p), _ptr(lab, _u8p)))
        if i.get("weights_f64"):  # weights that are not float32-exact: the f64 values
            w = np.zeros(i["E"], np.float64)
            _check(load_library().wf_graph_download_weights_f64(self.h, w.ctypes.data_as(C.POINTER(C.c_double))))
        return Graph(off, nbr, w, lab)

    def has_edge(self, src, dst) -> np.ndarray:
        s = np.ascontiguousarray(src, dtype=np.uint32)
        d = np.ascontiguousarray(dst, dtype=np.uint32)
        out = np.zeros(s.size, np.uint8)
        _check(load_library().wf_graph_has_edge(self.h, _ptr(s, _u32p), _ptr(d, _u32p),
                                                C.c_uint64(s.size), _ptr(out, _u8p)))
        return out.astype(bool)


class DeviceWalkSet:
    """RunResult's WalkSet kept in HBM (wf_walkset)."""

    def __init__(self, handle, metrics: RunMetrics, n_queries: int, vertex_count: int):
        self.h = handle
        self.metrics = metrics
        self.n = n_queries
        self.V = vertex_count

    def __del__(self):
        try:
            if self.h:
                _lib.wf_walkset_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def info(self):
        n = C.c_uint64()
        tv = C.c_uint64()
        ml = C.c_uint32()
        _check(load_library().wf_walkset_info(self.h, C.byref(n), C.byref(tv), C.byref(ml)))
        return dict(n=n.value, total_vertices=tv.value, max_length=ml.value)

    def to_host(self, qid_begin: int = 0, qid_end: Optional[int] = None) -> WalkSet:
        qe = self.n if qid_end is None else qid_end
        n = qe - qid_begin
        off = np.zeros(n + 1, np.uint64)
        st = np.zeros(n, np.uint8)
        lib = load_library()
        _check(lib.wf_walkset_copy(self.h, C.c_uint64(qid_begin), C.c_uint64(qe),
                                   _ptr(off, _u64p), None, _ptr(st, _u8p)))
        verts = np.zeros(int(off[-1]), np.uint32)
        _check(lib.wf_walkset_copy(self.h, C.c_uint64(qid_begin), C.c_uint64(qe), None,
                                   _ptr(verts, _u32p), None))
        return WalkSet(off, verts, st, np.arange(qid_begin, qe, dtype=np.uint64))

    def copy_into(self, offsets_ptr: int, vertices_ptr: int, status_ptr: int,
                  qid_begin: int = 0, qid_end: Optional[int] = None) -> None:
        """Raw copy into caller buffers (host or device pointers)."""
        qe = self.n if qid_end is None else qid_end
        _check(load_library().wf_walkset_copy(self.h, C.c_uint64(qid_begin), C.c_uint64(qe),
                                              _vp(offsets_ptr or None), _vp(vertices_ptr or None),
                                              _vp(status_ptr or None)))

    def write(self, path: str, fmt: int = 0, qid_begin: int = 0, qid_end: int = 0) -> int:
        """wf_walkset_write: the walk set as text (0) or binary (1) records."""
        n = C.c_uint64()
        _check(load_library().wf_walkset_write(self.h, path.encode(), C.c_int(fmt),
                                               C.c_uint64(qid_begin), C.c_uint64(qid_end),
                                               C.byref(n)))
        return n.value

    def visit_counts(self) -> np.ndarray:
        out = np.zeros(self.V, np.uint32)
        _check(load_library().wf_walkset_visit_counts(self.h, _ptr(out, _u32p)))
        return out


class Session:
    """A program bound to a device graph with its sampler resolved and static
    tables built (ResolvedRun)."""

    def __init__(self, graph: DeviceGraph, prog, opts: Optional[ExecOptions] = None):
        self.graph = graph
        self.prog = prog
        self.opts = opts or ExecOptions()
        self._copts = self.opts.to_c()
        h = _vp()
        if isinstance(prog, host_mod.DeviceProgram):
            self._desc = ProgramDesc()
            self._desc.kind = -1
            _check(load_library().wf_session_create_custom(graph.h, _vp(prog.ops), _vp(prog.object_pointer()),
                                                           C.byref(self._copts), C.byref(h)))
        else:
            self._desc = prog.to_c()
            _check(load_library().wf_session_create(graph.h, C.byref(self._desc),
                                                    C.byref(self._copts), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                _lib.wf_session_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def describe(self):
        s = C.c_int32()
        f = C.c_int32()
        p = C.c_double()
        _check(load_library().wf_session_describe(self.h, C.byref(s), C.byref(f), C.byref(p)))
        return abi.Sampler(s.value), abi.Flow(f.value), p.value

    def run(self, spec: QuerySpec) -> DeviceWalkSet:
        cs = spec.to_c()
        m = RunMetricsC()
        h = _vp()
        _check(load_library().wf_session_run(self.h, C.byref(cs), C.byref(h), C.byref(m)))
        metrics = RunMetrics(m.preprocess_seconds, m.exec_seconds, m.total_steps, m.max_in_flight)
        n = spec.total(self.graph) if spec.mode == abi.QueryMode.ONE_PER_VERTEX else spec.count
        return DeviceWalkSet(h, metrics, n, self.graph.vertex_count)

    def launch(self, spec: QuerySpec, qid_begin: int, qid_end: int, paths_ptr: int, stride: int,
               lengths_ptr: int, status_ptr: int, visit_counts_ptr: int = 0,
               steps_ptr: int = 0, overflow_ptr: int = 0, stream: int = 0,
               sources_dev_ptr: int = 0) -> None:
        """wf_session_launch into caller-owned device buffers (async)."""
        cs = spec.to_c()
        if sources_dev_ptr:
            cs.sources = C.cast(_vp(sources_dev_ptr), _u32p)
        _check(load_library().wf_session_launch(
            self.h, C.byref(cs), C.c_uint64(qid_begin), C.c_uint64(qid_end), _vp(paths_ptr),
            C.c_uint32(stride), _vp(lengths_ptr), _vp(status_ptr), _vp(visit_counts_ptr or None),
            _vp(steps_ptr or None), _vp(overflow_ptr or None), _vp(stream or None)))

    def run_host(self, spec: QuerySpec, offsets_ptr: int, vertices_ptr: int, capacity: int,
                 status_ptr: int, chunk: int = 0, qid_begin: int = 0,
                 qid_end: int = 0) -> RunMetrics:
        """wf_session_run_host: run and stream the walk set into HOST buffers
        (pointers; pinned memory for full bandwidth)."""
        cs = spec.to_c()
        m = RunMetricsC()
        _check(load_library().wf_session_run_host(
            self.h, C.byref(cs), C.c_uint64(qid_begin), C.c_uint64(qid_end),
            _vp(offsets_ptr or None), _vp(vertices_ptr), C.c_uint64(capacity),
            _vp(status_ptr or None), C.c_uint64(chunk), C.byref(m)))
        return RunMetrics(m.preprocess_seconds, m.exec_seconds, m.total_steps, m.max_in_flight)

    def run_host_records(self, spec: QuerySpec, records_ptr: int, vertices_ptr: int, capacity: int,
                         chunk: int = 0, qid_begin: int = 0, qid_end: int = 0) -> RunMetrics:
        """wf_session_run_host_records: records u32[n] (length | status << 31)
        and the paths back to back, into HOST buffers (pinned for full bandwidth)."""
        cs = spec.to_c()
        m = RunMetricsC()
        _check(load_library().wf_session_run_host_records(
            self.h, C.byref(cs), C.c_uint64(qid_begin), C.c_uint64(qid_end), _vp(records_ptr),
            _vp(vertices_ptr), C.c_uint64(capacity), C.c_uint64(chunk), C.byref(m)))
        return RunMetrics(m.preprocess_seconds, m.exec_seconds, m.total_steps, m.max_in_flight)

    def run_host_blocks(self, spec: QuerySpec, records_ptr: int, vertices_ptr: int, capacity: int,
                        on_block, chunk: int = 0, qid_begin: int = 0, qid_end: int = 0) -> RunMetrics:
        """wf_session_run_host_blocks (the BlockSink form): as run_host_records,
        and on_block(block, qid_begin, qid_end, vertex_begin) -> bool|None is
        called in qid order as each block lands; returning True stops the run
        (IoError)."""
        def tramp(_user, block, q0, q1, v0):
            try:
                return 1 if on_block(block, q0, q1, v0) else 0
            except Exception:  # a Python error stops the run instead of crossing the C frame
                return 1
        cb = _BLOCK_FN(tramp)
        cs = spec.to_c()
        m = RunMetricsC()
        _check(load_library().wf_session_run_host_blocks(
            self.h, C.byref(cs), C.c_uint64(qid_begin), C.c_uint64(qid_end), _vp(records_ptr),
            _vp(vertices_ptr), C.c_uint64(capacity), C.c_uint64(chunk), cb, None, C.byref(m)))
        return RunMetrics(m.preprocess_seconds, m.exec_seconds, m.total_steps, m.max_in_flight)

    def run_to_numpy(self, spec: QuerySpec, chunk: int = 0) -> RunResult:
        """Convenience over run_host with numpy (pageable) buffers.  Unbounded
        programs (PPR, custom programs without max_path_vertices) have no host
        capacity to size in advance: they run into HBM (wf_session_run, which
        re-runs walks that outgrow their row) and are copied out after."""
        n = self.graph.vertex_count if spec.mode == abi.QueryMode.ONE_PER_VERTEX else spec.count
        if self.unbounded():
            ws = self.run(spec)
            return RunResult(ws.to_host(), ws.metrics)
        cap = n * self.row_capacity()  # fixed-length programs fit exactly
        off = np.zeros(n + 1, np.uint64)
        verts = np.zeros(max(cap, 1), np.uint32)
        st = np.zeros(max(n, 1), np.uint8)
        m = self.run_host(spec, off.ctypes.data, verts.ctypes.data, cap, st.ctypes.data, chunk)
        return RunResult(WalkSet(off, verts[:int(off[-1])], st[:n]), m)

    def unbounded(self) -> bool:
        p = self.prog
        if isinstance(p, host_mod.DeviceProgram):
            return p.max_path() == 0
        return isinstance(p, host_mod.PprProgram)

    def row_capacity(self) -> int:
        p = self.prog
        if isinstance(p, host_mod.DeviceProgram):
            return p.max_path() or self.opts.path_stride or 64
        if isinstance(p, host_mod.MetaPathProgram):
            return len(p.schema) + 1
        if isinstance(p, host_mod.PprProgram):
            return self.opts.path_stride or 64
        return p.target_length

    def layout(self) -> int:
        f = C.c_uint32()
        _check(load_library().wf_session_layout(self.h, C.byref(f)))
        return f.value

    def tune(self, spec: QuerySpec, qid_begin: int = 0, qid_end: int = 0,
             sources_dev_ptr: int = 0) -> tuple:
        """wf_session_tune: time whole launches of the range at each candidate
        blocks/SM and keep the fastest for launches of that size.  Returns
        (blocks_per_sm, best_ms)."""
        cs = spec.to_c()
        if sources_dev_ptr:
            cs.sources = C.cast(_vp(sources_dev_ptr), _u32p)
        b = C.c_int32()
        ms = C.c_double()
        _check(load_library().wf_session_tune(self.h, C.byref(cs), C.c_uint64(qid_begin),
                                              C.c_uint64(qid_end), C.byref(b), C.byref(ms)))
        return b.value, ms.value

    def set_stats(self, enable: bool) -> None:
        _check(load_library().wf_session_set_stats(self.h, C.c_int(1 if enable else 0)))

    def stats(self) -> dict:
        out = np.zeros(6, np.uint64)
        _check(load_library().wf_session_stats_n(self.h, _ptr(out, _u64p), C.c_uint32(6)))
        d = dict(trials=int(out[0]), probes=int(out[1]), scanned=int(out[2]))
        kind = int(self._desc.kind)
        if kind == abi.ProgramKind.NODE2VEC:
            d["ref_probes"] = int(out[3])
        if kind == abi.ProgramKind.METAPATH:
            d["ref_label_sectors"] = int(out[4])
            d["step_attempts"] = int(out[5])
        return d

    def sync(self, stream: int = 0) -> None:
        _check(load_library().wf_session_sync(self.h, _vp(stream or None)))

    def tables(self) -> dict:
        i = self.graph.info()
        e, v = i["E"], i["V"]
        out = dict(alias_thr=np.zeros(e, np.uint64), alias_first_dst=np.zeros(e, np.uint32),
                   alias_second_dst=np.zeros(e, np.uint32), its=np.zeros(e, np.float64),
                   rej_p_star=np.zeros(v, np.float64), exhausted=np.zeros(v, np.uint8))
        _check(load_library().wf_session_tables(
            self.h, _ptr(out["alias_thr"], _u64p), _ptr(out["alias_first_dst"], _u32p),
            _ptr(out["alias_second_dst"], _u32p), _ptr(out["its"], _f64p),
            _ptr(out["rej_p_star"], _f64p), _ptr(out["exhausted"], _u8p)))
        return out


def _as_device(g) -> DeviceGraph:
    return g if isinstance(g, DeviceGraph) else DeviceGraph.from_host(g)


def run_sequential(g, spec: QuerySpec, prog, opts: Optional[ExecOptions] = None) -> RunResult:
    """run_sequential (engine.hpp:440-504): every query to completion; the walk
    set is a pure function of (graph, spec, program, seed)."""
    dg = _as_device(g)
    if isinstance(prog, host_mod.DeviceProgram):
        sess = Session(dg, prog, opts)
        ws = sess.run(spec)
        return RunResult(ws.to_host(), ws.metrics)
    cs = spec.to_c()
    # validate the spec before resolving the program, like the reference
    desc = prog.to_c()
    copts = (opts or ExecOptions()).to_c()
    m = RunMetricsC()
    h = _vp()
    _check(load_library().wf_run(dg.h, C.byref(desc), C.byref(cs), C.byref(copts), C.byref(h),
                                 C.byref(m)))
    n = dg.vertex_count if spec.mode == abi.QueryMode.ONE_PER_VERTEX else spec.count
    ws = DeviceWalkSet(h, RunMetrics(m.preprocess_seconds, m.exec_seconds, m.total_steps,
                                     m.max_in_flight), n, dg.vertex_count)
    return RunResult(ws.to_host(), ws.metrics)


def run_interleaved(g, spec: QuerySpec, prog, k: int, k_prime: int,
                    opts: Optional[ExecOptions] = None) -> RunResult:
    """run_interleaved (interleave.hpp:391-556): same walks as run_sequential;
    k / k' are validated like the reference and otherwise only launch hints."""
    o = opts or ExecOptions()
    o = ExecOptions(**{**o.__dict__, "k": k, "k_prime": k_prime})
    if k == 0:
        raise abi.ConfigError("task ring size must be >= 1")
    if k_prime == 0 or k_prime > k:
        raise abi.ConfigError("search ring size must be in [1, k]")
    return run_sequential(g, spec, prog, o)


def encode_walks(ws: WalkSet, fmt: int = 0, qid_base: int = 0) -> bytes:
    """wf_encode_walks over a host WalkSet: the reference's record bytes."""
    lib = load_library()
    off = np.ascontiguousarray(ws.offsets, dtype=np.uint64)
    verts = np.ascontiguousarray(ws.vertices, dtype=np.uint32)
    st = np.ascontiguousarray(ws.status, dtype=np.uint8)
    n = C.c_uint64()
    _check(lib.wf_encode_walks(_ptr(off, _u64p), _ptr(verts, _u32p), _ptr(st, _u8p),
                               C.c_uint64(len(ws)), C.c_uint64(qid_base), C.c_int(fmt), None,
                               C.c_uint64(0), C.byref(n)))
    buf = C.create_string_buffer(max(n.value, 1))
    _check(lib.wf_encode_walks(_ptr(off, _u64p), _ptr(verts, _u32p), _ptr(st, _u8p),
                               C.c_uint64(len(ws)), C.c_uint64(qid_base), C.c_int(fmt), buf,
                               C.c_uint64(n.value), C.byref(n)))
    return buf.raw[:n.value]


def rng_probe(seed: int, streams, draws: int) -> np.ndarray:
    s = np.ascontiguousarray(streams, dtype=np.uint64)
    out = np.zeros((s.size, draws), np.uint64)
    _check(load_library().wf_rng_probe(C.c_uint64(seed), _ptr(s, _u64p), C.c_uint64(s.size),
                                       C.c_uint32(draws), _ptr(out, _u64p)))
    return out


_SHARD_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32),
                        C.POINTER(C.c_uint32), C.c_uint64)


def worker_range(n: int, workers: int, w: int):
    """worker_range (engine.hpp:296-298) through the library: [n*w/W, n*(w+1)/W)."""
    b, e = C.c_uint64(), C.c_uint64()
    _check(load_library().wf_worker_range(C.c_uint64(n), C.c_uint32(workers), C.c_uint32(w), C.byref(b),
                                          C.byref(e)))
    return b.value, e.value


def device_count() -> int:
    n = C.c_int32()
    _check(load_library().wf_device_count(C.byref(n)))
    return n.value


class MultiDevice:
    """run_*'s workers over devices (wf_multi_*): the graph replicated on every
    listed device, the static tables built once and peer-copied, `workers`
    contiguous qid blocks walked by one host thread per device and delivered
    in worker order; PPR visit counts reduced with one NCCL all-reduce (or a
    device sum when a device is listed twice)."""

    def __init__(self, graph: DeviceGraph, devices, prog, opts: Optional[ExecOptions] = None):
        self.graph = graph
        self.prog = prog
        self.opts = opts or ExecOptions()
        self._copts = self.opts.to_c()
        devs = (C.c_int32 * len(devices))(*devices)
        h = _vp()
        _preload_nccl()
        lib = load_library()
        if isinstance(prog, host_mod.DeviceProgram):
            _check(lib.wf_multi_create_custom(graph.h, devs, C.c_uint32(len(devices)), _vp(prog.ops),
                                              _vp(prog.object_pointer()), C.byref(self._copts), C.byref(h)))
        else:
            self._desc = prog.to_c()
            _check(lib.wf_multi_create(graph.h, devs, C.c_uint32(len(devices)), C.byref(self._desc),
                                       C.byref(self._copts), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                _lib.wf_multi_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def info(self):
        n = C.c_uint32()
        coll = C.c_int32()
        _check(load_library().wf_multi_info(self.h, C.byref(n), C.byref(coll)))
        return dict(devices=n.value, nccl=bool(coll.value))

    def run(self, spec: QuerySpec, workers: int = 0, on_block=None, counts: bool = False):
        """Runs every query; returns (RunResult, visit counts or None, blocks
        [(worker, qid_begin, qid_end)] in delivery order).  on_block(worker,
        q0, q1, WalkSet) is called in worker order."""
        n = self.graph.vertex_count if spec.mode == abi.QueryMode.ONE_PER_VERTEX else spec.count
        offs = [np.zeros(1, np.uint64)]
        verts, stats, order = [], [], []
        err = []
        total = [0]  # vertices delivered so far (a worker block may be empty)

        def tramp(_user, w, q0, q1, rec, vp, nv):
            try:
                r = np.ctypeslib.as_array(rec, shape=(q1 - q0,)).copy() if q1 > q0 else np.zeros(0, np.uint32)
                v = np.ctypeslib.as_array(vp, shape=(nv,)).copy() if nv else np.zeros(0, np.uint32)
                lens = (r & 0x7FFFFFFF).astype(np.uint64)
                st = (r >> 31).astype(np.uint8)
                order.append((w, q0, q1))
                o = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint64)
                if on_block is not None:
                    on_block(w, q0, q1, WalkSet(o, v, st))
                offs.append(o[1:] + np.uint64(total[0]))
                total[0] += int(o[-1])
                verts.append(v)
                stats.append(st)
                return 0
            except Exception as e:  # stop the run, re-raise here
                err.append(e)
                return 1

        cb = _SHARD_FN(tramp)
        cs = spec.to_c()
        m = RunMetricsC()
        cnt = np.zeros(self.graph.vertex_count, np.uint32) if counts else None
        rc = load_library().wf_multi_run(self.h, C.byref(cs), C.c_uint32(workers), cb, None,
                                         _ptr(cnt, _u32p), C.byref(m))
        if err:
            raise err[0]
        _check(rc)
        ws = WalkSet(np.concatenate(offs).astype(np.uint64),
                     np.concatenate(verts) if verts else np.zeros(0, np.uint32),
                     np.concatenate(stats) if stats else np.zeros(0, np.uint8))
        assert len(ws) == n
        return (RunResult(ws, RunMetrics(m.preprocess_seconds, m.exec_seconds, m.total_steps, m.max_in_flight)),
                cnt, order)


class Comm:
    """The library's own NCCL communicator for one-process-per-GPU jobs
    (wf_comm_*): rank 0 makes the id (unique_id()), the caller ships it to the
    other ranks; allreduce_u32 sums a device u32 vector in place."""

    ID_BYTES = 128

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * Comm.ID_BYTES)()
        _preload_nccl()
        _check(load_library().wf_comm_unique_id(buf))
        return bytes(buf)

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        buf = (C.c_uint8 * Comm.ID_BYTES)(*uid)
        h = _vp()
        _preload_nccl()
        _check(load_library().wf_comm_create(buf, C.c_int32(nranks), C.c_int32(rank), C.c_int32(device),
                                             C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                _lib.wf_comm_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def allreduce_u32(self, dev_ptr: int, count: int, stream: int = 0) -> None:
        _check(load_library().wf_comm_allreduce_u32(self.h, _vp(dev_ptr), C.c_uint64(count), _vp(stream or None)))


def nccl_version() -> int:
    _preload_nccl()
    v = C.c_int32()
    _check(load_library().wf_nccl_version(C.byref(v)))
    return v.value
