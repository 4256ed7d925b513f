"""Host-side mirror of the reference's value types (no device code here).

Graph            proj/include/walkforge/graph.hpp:17-107 (CSR arrays; from_csr, build_graph)
QuerySpec        proj/include/walkforge/walker.hpp:61-84
ExecOptions      proj/include/walkforge/engine.hpp:81-89
PprProgram ...   proj/include/walkforge/algorithms.hpp:20-193 (parameters only; the
                 device functors live in csrc/programs.cuh)
WalkSet          proj/include/walkforge/walker.hpp:47-55 as ragged arrays

Weights are float32 (the device stores f32; the reference widens them to f64
exactly, graph.hpp:24-25) and labels uint8 (labels < 256).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from .abi import (ConfigError, ExecOptionsC, ProgramDesc, ProgramKind, QueryMode, QuerySpecC,
                  Sampler, WalkStatus)


class Graph:
    """CSR graph: offsets u64[V+1], neighbors u32[E], weights f32[E] or f64[E]
    (the reference's own type, graph.hpp:102; kept when given), labels u8[E]?"""

    def __init__(self, offsets, neighbors, weights=None, labels=None):
        self.offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        self.neighbors = np.ascontiguousarray(neighbors, dtype=np.uint32)
        if weights is not None:
            w = np.asarray(weights)
            weights = np.ascontiguousarray(w, dtype=np.float64 if w.dtype == np.float64 else np.float32)
        self.weights = weights
        self.labels = None if labels is None else np.ascontiguousarray(labels, dtype=np.uint8)

    @classmethod
    def from_csr(cls, offsets, neighbors, weights=None, labels=None) -> "Graph":
        """Graph::from_csr (proj/src/graph.cpp:118-159) structural validation."""
        offsets = np.asarray(offsets, dtype=np.uint64)
        neighbors = np.asarray(neighbors, dtype=np.uint32)
        if offsets.size < 2:
            raise ConfigError("graph must have at least one vertex")
        if int(offsets[0]) != 0 or int(offsets[-1]) != neighbors.size:
            raise ConfigError("CSR offsets do not frame the neighbor array")
        if np.any(offsets[1:] < offsets[:-1]):
            raise ConfigError("CSR offsets must be non-decreasing")
        v = offsets.size - 1
        if neighbors.size and int(neighbors.max()) >= v:
            raise ConfigError(f"neighbor id {int(neighbors.max())} out of range")
        if weights is not None:
            w64 = np.asarray(weights)
            if w64.size != neighbors.size:
                raise ConfigError("weight array does not match edge count")
            wd = w64.astype(np.float64)
            if not np.all(np.isfinite(wd)) or np.any(wd < 0):
                raise ConfigError("edge weights must be finite and non-negative")
            w32 = wd.astype(np.float32)
            # float32-exact weights are stored as f32; others keep their f64 values
            weights = w32 if np.array_equal(w32.astype(np.float64), wd) else wd
        if labels is not None:
            labels = np.asarray(labels)
            if labels.size != neighbors.size:
                raise ConfigError("label array does not match edge count")
            if labels.size and int(labels.max()) > 255:
                raise ConfigError("edge labels must be < 256 on the device")
        return cls(offsets, neighbors, weights, labels)

    @property
    def vertex_count(self) -> int:
        return self.offsets.size - 1

    @property
    def edge_count(self) -> int:
        return self.neighbors.size

    def degree(self, v: int) -> int:
        return int(self.offsets[v + 1] - self.offsets[v])

    def has_weights(self) -> bool:
        return self.weights is not None

    def has_labels(self) -> bool:
        return self.labels is not None

    def max_weight(self) -> float:
        return float(self.weights.max()) if self.weights is not None and self.weights.size else 0.0

    def neighbors_of(self, v: int) -> np.ndarray:
        return self.neighbors[int(self.offsets[v]):int(self.offsets[v + 1])]


def build_graph(vertex_count: int, edges: Sequence[tuple[int, int]], weights=None,
                labels=None) -> Graph:
    """build_graph / assemble_csr (proj/src/graph.cpp:37-102, 289-304): bucket by
    source, sort each list by destination with input order breaking ties."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if e.size and (e.min() < 0 or e.max() >= vertex_count):
        raise ConfigError("edge endpoint out of range")
    order = np.lexsort((np.arange(len(e)), e[:, 1], e[:, 0]))
    src = e[order, 0]
    offsets = np.zeros(vertex_count + 1, dtype=np.uint64)
    np.add.at(offsets, src + 1, 1)
    offsets = np.cumsum(offsets, dtype=np.uint64)
    w = None if weights is None else np.asarray(weights, dtype=np.float64)[order]
    lab = None if labels is None else np.asarray(labels)[order]
    return Graph.from_csr(offsets, e[order, 1].astype(np.uint32), w, lab)


@dataclass
class QuerySpec:
    """QuerySpec (walker.hpp:61-84).  `from_list` is from_file after parsing."""

    mode: QueryMode = QueryMode.ONE_PER_VERTEX
    source: int = 0
    count: int = 0
    sources: Optional[np.ndarray] = None

    @classmethod
    def one_per_vertex(cls) -> "QuerySpec":
        return cls(QueryMode.ONE_PER_VERTEX)

    @classmethod
    def from_source(cls, source: int, count: int) -> "QuerySpec":
        return cls(QueryMode.FROM_SOURCE, source=source, count=count)

    @classmethod
    def from_file(cls, path: str) -> "QuerySpec":
        """QuerySpec::from_file (walker.cpp:22-78): `vertex [count]` per line,
        '#' comments, blank lines skipped; the reference's messages and classes."""
        from .abi import ParseError, WalkforgeError
        try:
            f = open(path, "r", encoding="utf-8", errors="surrogateescape")
        except OSError:
            raise WalkforgeError(f"cannot open query file '{path}'") from None
        out = []
        with f:
            for line_no, line in enumerate(f, 1):
                line = line.rstrip("\n").split("#", 1)[0]
                tok = line.split()
                if not tok:
                    continue
                if len(tok) > 2:
                    raise ParseError(f"{path}:{line_no}: too many columns")
                vals = []
                for t in tok:
                    # std::from_chars on uint64: decimal digits only, no sign, no overflow
                    if not t.isascii() or not t.isdigit() or int(t) >= 1 << 64:
                        raise ParseError(f"{path}:{line_no}: expected `vertex [count]`")
                    vals.append(int(t))
                v, c = vals[0], (vals[1] if len(vals) == 2 else 1)
                if v > 0xFFFFFFFF:
                    raise ParseError(f"{path}:{line_no}: vertex id out of range")
                out.extend([v] * c)
        if not out:
            raise ParseError(f"{path}: no queries")
        return cls.from_list(np.asarray(out, dtype=np.uint32))

    @classmethod
    def from_list(cls, sources) -> "QuerySpec":
        s = np.ascontiguousarray(sources, dtype=np.uint32)
        return cls(QueryMode.FROM_LIST, count=s.size, sources=s)

    def total(self, g: Graph) -> int:
        return g.vertex_count if self.mode == QueryMode.ONE_PER_VERTEX else self.count

    def to_c(self) -> QuerySpecC:
        c = QuerySpecC()
        c.mode = int(self.mode)
        c.source = self.source
        c.count = self.total_hint()
        c.sources = (self.sources.ctypes.data_as(C.POINTER(C.c_uint32))
                     if self.sources is not None else None)
        return c

    def total_hint(self) -> int:
        return self.count


@dataclass
class ExecOptions:
    """ExecOptions (engine.hpp:81-89)."""

    threads: int = 1
    seed: int = 0
    sampler: Optional[Sampler] = None
    use_static_tables: bool = True
    rej_trial_cap: int = 1 << 20
    k: int = 64
    k_prime: int = 32
    path_stride: int = 0
    layout_flags: int = 0

    def to_c(self) -> ExecOptionsC:
        c = ExecOptionsC()
        c.seed = self.seed
        c.sampler = int(Sampler.DEFAULT if self.sampler is None else self.sampler)
        c.use_static_tables = 1 if self.use_static_tables else 0
        c.rej_trial_cap = self.rej_trial_cap
        c.threads = self.threads
        c.k = self.k
        c.k_prime = self.k_prime
        c.path_stride = self.path_stride
        c.layout_flags = self.layout_flags
        return c


class DeviceProgram:
    """A user's device program (the WalkProgram concept, program.hpp:49-93,
    written against include/walkforge_b200/device_program.cuh and compiled
    into the user's own shared library).  `ops` is the address of the
    wf_program_ops table its WF_DEVICE_PROGRAM(Type, symbol) exports (or a
    (library path, symbol) pair); `obj` the program object: a ctypes
    Structure with the C++ type's layout (or its raw bytes)."""

    kind = -1  # kCustomProgram

    def __init__(self, ops, obj):
        if isinstance(ops, tuple):
            lib = C.CDLL(ops[0])
            fn = getattr(lib, ops[1])
            fn.restype = C.c_void_p
            self._lib = lib
            ops = fn()
        self.ops = int(ops)
        self.obj = obj
        self._buf = C.create_string_buffer(bytes(obj), max(len(bytes(obj)), 1))

    def object_pointer(self) -> int:
        return C.addressof(self._buf)

    def table(self) -> "ProgramOpsC":
        return ProgramOpsC.from_address(self.ops)

    def max_path(self) -> int:
        """max_path_vertices() of the object (0 = unbounded)."""
        t = self.table()
        return int(t.max_path(C.c_void_p(self.object_pointer()))) if t.max_path else 0


class ProgramOpsC(C.Structure):  # wf_program_ops (walkforge_b200.h)
    _fields_ = [("abi_version", C.c_uint32), ("launch_size", C.c_uint32), ("name", C.c_char_p),
                ("walker_type", C.c_int32), ("preferred_sampler", C.c_int32), ("has_max_weight", C.c_int32),
                ("prechecked", C.c_int32), ("program_size", C.c_uint32), ("engine_abi", C.c_uint32),
                ("launch", C.c_void_p), ("occupancy", C.c_void_p), ("static_weights", C.c_void_p),
                ("max_weight", C.CFUNCTYPE(C.c_double, C.c_void_p)),
                ("max_path", C.CFUNCTYPE(C.c_uint32, C.c_void_p))]


class _Program:
    kind: ProgramKind

    def to_c(self) -> ProgramDesc:
        raise NotImplementedError


@dataclass
class PprProgram(_Program):
    termination: float = 0.2
    kind = ProgramKind.PPR

    def to_c(self):
        d = ProgramDesc()
        d.kind = int(self.kind)
        d.termination = self.termination
        return d


@dataclass
class DeepWalkProgram(_Program):
    target_length: int = 80
    weighted: bool = False
    kind = ProgramKind.DEEPWALK

    def to_c(self):
        d = ProgramDesc()
        d.kind = int(self.kind)
        d.target_length = self.target_length
        d.weighted = 1 if self.weighted else 0
        return d


@dataclass
class Node2VecProgram(_Program):
    a: float = 2.0
    b: float = 0.5
    target_length: int = 80
    weighted: bool = False
    kind = ProgramKind.NODE2VEC

    def to_c(self):
        d = ProgramDesc()
        d.kind = int(self.kind)
        d.a, d.b = self.a, self.b
        d.target_length = self.target_length
        d.weighted = 1 if self.weighted else 0
        return d


@dataclass
class MetaPathProgram(_Program):
    schema: Sequence[int] = (0,)
    kind = ProgramKind.METAPATH
    _buf: np.ndarray = field(default=None, repr=False)

    def to_c(self):
        self._buf = np.ascontiguousarray(self.schema, dtype=np.uint32)
        d = ProgramDesc()
        d.kind = int(self.kind)
        d.schema = self._buf.ctypes.data_as(C.POINTER(C.c_uint32))
        d.schema_len = self._buf.size
        return d


@dataclass
class UniformProgram(_Program):
    target_length: int = 80
    kind = ProgramKind.UNIFORM

    def to_c(self):
        d = ProgramDesc()
        d.kind = int(self.kind)
        d.target_length = self.target_length
        return d


@dataclass
class WalkSet:
    """WalkSet as ragged arrays: path of query i = vertices[offsets[i]:offsets[i+1]]."""

    offsets: np.ndarray
    vertices: np.ndarray
    status: np.ndarray
    qids: Optional[np.ndarray] = None

    def __len__(self):
        return self.status.size

    def path(self, i: int) -> np.ndarray:
        return self.vertices[int(self.offsets[i]):int(self.offsets[i + 1])]

    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets)

    def equals(self, other: "WalkSet") -> bool:
        return (np.array_equal(self.offsets, other.offsets)
                and np.array_equal(self.vertices, other.vertices)
                and np.array_equal(self.status, other.status))

    def first_mismatch(self, other: "WalkSet") -> Optional[int]:
        n = min(len(self), len(other))
        for i in range(n):
            if self.status[i] != other.status[i] or not np.array_equal(self.path(i), other.path(i)):
                return i
        return None if len(self) == len(other) else n


@dataclass
class RunMetrics:
    preprocess_seconds: float = 0.0
    exec_seconds: float = 0.0
    total_steps: int = 0
    max_in_flight: int = 0


@dataclass
class RunResult:
    walks: WalkSet
    metrics: RunMetrics
