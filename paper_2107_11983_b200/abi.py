"""ctypes mirror of include/walkforge_b200.h (plain data only).

Enum values and struct layouts must match the C header byte for byte; the
no-GPU test suite checks sizes and the exported symbol list.  The exception
classes mirror the reference hierarchy (proj/include/walkforge/error.hpp:8-48)
so callers catch the same names they catch around the reference.
"""
from __future__ import annotations

import ctypes as C
import enum


class Sampler(enum.IntEnum):
    """SamplerKind, proj/include/walkforge/sampler.hpp:21."""

    DEFAULT = -1
    NAIVE = 0
    ITS = 1
    ALIAS = 2
    REJ = 3
    OREJ = 4

    @classmethod
    def parse(cls, name: str) -> "Sampler":
        """parse_sampler, proj/src/sampler.cpp:19-26."""
        table = {"naive": cls.NAIVE, "its": cls.ITS, "alias": cls.ALIAS, "rej": cls.REJ,
                 "orej": cls.OREJ, "o-rej": cls.OREJ}
        if name not in table:
            raise ConfigError(f"unknown sampler '{name}'")
        return table[name]


class ProgramKind(enum.IntEnum):
    PPR = 0
    DEEPWALK = 1
    NODE2VEC = 2
    METAPATH = 3
    UNIFORM = 4


class WalkStatus(enum.IntEnum):
    """WalkStatus, proj/include/walkforge/walker.hpp:12."""

    COMPLETE = 0
    DEAD_END = 1


class QueryMode(enum.IntEnum):
    ONE_PER_VERTEX = 0
    FROM_SOURCE = 1
    FROM_LIST = 2


class Flow(enum.IntEnum):
    """ExecFlow, proj/include/walkforge/engine.hpp:58-62."""

    DIRECT = 0
    TABLES = 1
    GATHERED = 2


# ---- exceptions: proj/include/walkforge/error.hpp:8-48 -------------------------
class WalkforgeError(RuntimeError):
    """Error base (error.hpp:8-10)."""


class ParseError(WalkforgeError):
    pass


class FormatError(WalkforgeError):
    pass


class ConfigError(WalkforgeError):
    pass


class DistributionError(WalkforgeError):
    pass


class ContractError(WalkforgeError):
    pass


class RejectionCapError(WalkforgeError):
    pass


class IoError(WalkforgeError):
    pass


class CudaError(WalkforgeError):
    """Device fault or no device; no reference counterpart."""


class InvalidArgument(WalkforgeError):
    pass


STATUS_TO_ERROR = {
    1: ParseError,
    2: FormatError,
    3: ConfigError,
    4: DistributionError,
    5: ContractError,
    6: RejectionCapError,
    7: IoError,
    8: CudaError,
    9: CudaError,
    10: InvalidArgument,
}


def raise_for(code: int, message: str) -> None:
    if code != 0:
        raise STATUS_TO_ERROR.get(code, WalkforgeError)(message)


# ---- structs ------------------------------------------------------------------
class ProgramDesc(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("target_length", C.c_uint32),
        ("weighted", C.c_int32),
        ("reserved0", C.c_int32),
        ("termination", C.c_double),
        ("a", C.c_double),
        ("b", C.c_double),
        ("schema", C.POINTER(C.c_uint32)),
        ("schema_len", C.c_uint32),
        ("reserved1", C.c_uint32),
    ]


class ExecOptionsC(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("sampler", C.c_int32),
        ("use_static_tables", C.c_int32),
        ("rej_trial_cap", C.c_uint32),
        ("threads", C.c_uint32),
        ("k", C.c_uint32),
        ("k_prime", C.c_uint32),
        ("path_stride", C.c_uint32),
        ("layout_flags", C.c_uint32),
    ]


LAYOUT_COMPACT_ALIAS = 1
LAYOUT_NO_ADJ = 2
LAYOUT_MP_SUCC = 4
LAYOUT_FORCE_ADJ = 8
LAYOUT_SEARCH_TREE = 16
LAYOUT_NO_MP_SUCC = 32
LAYOUT_NO_EDGE_FILTER = 64
LAYOUT_ADJ8 = 128
LAYOUT_WIDE_ALIAS = 256

HAS_WIDE_ALIAS = 1
HAS_ADJ = 2
HAS_MP_SUCC = 4
HAS_LABEL_INDEX = 8
HAS_ADJ8 = 128
HAS_SEARCH_INDEX = 16
HAS_EDGE_HASH = 32
HAS_EDGE_FILTER = 64


class QuerySpecC(C.Structure):
    _fields_ = [
        ("mode", C.c_int32),
        ("source", C.c_uint32),
        ("count", C.c_uint64),
        ("sources", C.POINTER(C.c_uint32)),
    ]


class RunMetricsC(C.Structure):
    _fields_ = [
        ("preprocess_seconds", C.c_double),
        ("exec_seconds", C.c_double),
        ("total_steps", C.c_uint64),
        ("max_in_flight", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


class GraphInfoC(C.Structure):
    _fields_ = [
        ("vertex_count", C.c_uint32),
        ("max_degree", C.c_uint32),
        ("edge_count", C.c_uint64),
        ("max_weight", C.c_double),
        ("has_weights", C.c_int32),
        ("has_labels", C.c_int32),
        ("adjacency_sorted", C.c_int32),
        ("device", C.c_int32),
        ("label_count", C.c_uint32),
        ("weights_f64", C.c_uint32),
    ]


class EdgeListOptionsC(C.Structure):
    _fields_ = [
        ("undirected", C.c_int32),
        ("weights", C.c_int32),
        ("labels", C.c_int32),
        ("label_count", C.c_uint32),
        ("seed", C.c_uint64),
    ]


class RmatParamsC(C.Structure):
    _fields_ = [
        ("scale", C.c_uint32),
        ("edge_factor", C.c_uint32),
        ("a", C.c_double),
        ("b", C.c_double),
        ("c", C.c_double),
        ("seed", C.c_uint64),
        ("weighted", C.c_int32),
        ("label_count", C.c_uint32),
    ]


# Every symbol include/walkforge_b200.h declares (checked by the CPU suite).
EXPORTED_SYMBOLS = [
    "wf_abi_version", "wf_last_error", "wf_kernel_launches", "wf_device_count",
    "wf_graph_create", "wf_graph_create_f64", "wf_graph_download_weights_f64",
    "wf_graph_create_device", "wf_graph_generate_rmat",
    "wf_graph_info_get", "wf_graph_download", "wf_graph_has_edge", "wf_graph_labels_present", "wf_graph_destroy",
    "wf_graph_read_wfg1", "wf_graph_write_wfg1", "wf_graph_load_edge_list", "wf_graph_original_ids",
    "wf_session_create", "wf_session_describe", "wf_session_destroy", "wf_session_run",
    "wf_session_launch", "wf_session_sync", "wf_session_run_host", "wf_session_run_host_records",
    "wf_session_run_host_blocks",
    "wf_session_set_stats",
    "wf_session_stats", "wf_session_stats_n", "wf_session_layout", "wf_session_tune",
    "wf_session_create_custom",
    "wf_worker_range", "wf_multi_create", "wf_multi_create_custom", "wf_multi_info", "wf_multi_run",
    "wf_multi_destroy", "wf_comm_unique_id", "wf_comm_create", "wf_comm_allreduce_u32", "wf_comm_destroy",
    "wf_nccl_version",
    "wf_walkset_info", "wf_walkset_copy", "wf_walkset_visit_counts", "wf_walkset_destroy",
    "wf_run", "wf_rng_probe", "wf_session_tables", "wf_encode_walks", "wf_walkset_write",
]
