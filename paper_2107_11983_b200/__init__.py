"""B200-native random-walk engine (ThunderRW's Gather–Move–Update path).

The compute path is hand-written sm_100a CUDA behind the C-ABI in
include/walkforge_b200.h (library: paper_2107_11983_b200/libwalkforge_b200.so).
This package holds the Python mirror of the reference interface (engine.py) and
plain-data helpers; there is no CPU fallback.
"""
from .abi import (ConfigError, ContractError, DistributionError, FormatError, IoError,  # noqa: F401
                  ParseError, RejectionCapError, Sampler, WalkStatus, WalkforgeError)
from .host import (DeepWalkProgram, ExecOptions, Graph, MetaPathProgram, Node2VecProgram,  # noqa: F401
                   PprProgram, QuerySpec, RunMetrics, RunResult, UniformProgram, WalkSet,
                   build_graph)
