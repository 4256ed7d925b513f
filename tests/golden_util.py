"""Loads the committed golden fixtures (tests/golden/, made by make_golden.py
from the unmodified reference)."""
from __future__ import annotations

import json
import os

import numpy as np

from paper_2107_11983_b200.abi import Sampler
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, Graph, MetaPathProgram,
                                        Node2VecProgram, PprProgram, QuerySpec, UniformProgram,
                                        WalkSet)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

_cache = {}


def _npz(name):
    if name not in _cache:
        with np.load(os.path.join(GOLDEN, name)) as z:
            _cache[name] = {k: z[k] for k in z.files}
    return _cache[name]


def cases():
    with open(os.path.join(GOLDEN, "cases.json")) as f:
        return json.load(f)


def graph(name) -> Graph:
    z = _npz("graphs.npz")
    return Graph(z[f"{name}/offsets"], z[f"{name}/neighbors"], z.get(f"{name}/weights"),
                 z.get(f"{name}/labels"))


def walks(case) -> WalkSet:
    z = _npz("walks.npz")
    n = case["name"]
    return WalkSet(z[f"{n}/offsets"], z[f"{n}/vertices"], z[f"{n}/status"])


def tables():
    return _npz("tables.npz")


def rng():
    return _npz("rng.npz")


def program(d):
    k = d["program"]
    if k == "ppr":
        return PprProgram(d.get("termination", 0.2))
    if k == "deepwalk":
        return DeepWalkProgram(d["length"], d.get("weighted", False))
    if k == "node2vec":
        return Node2VecProgram(d.get("a", 2.0), d.get("b", 0.5), d["length"],
                               d.get("weighted", False))
    if k == "metapath":
        return MetaPathProgram(d["schema"])
    if k == "uniform":
        return UniformProgram(d["length"])
    raise ValueError(k)


def spec(d):
    s = d.get("spec", {"mode": "one_per_vertex"})
    if s["mode"] == "one_per_vertex":
        return QuerySpec.one_per_vertex()
    if s["mode"] == "from_source":
        return QuerySpec.from_source(s["source"], s["count"])
    return QuerySpec.from_list(np.asarray(s["sources"], dtype=np.uint32))


def opts(d):
    smp = d.get("sampler")
    return ExecOptions(seed=d.get("seed", 1), sampler=None if smp is None else Sampler.parse(smp),
                       use_static_tables=d.get("tables", True))
