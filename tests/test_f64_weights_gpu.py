"""Weights that are not float32-exact (the reference stores f64, graph.hpp:102):
the engine keeps an f64 copy resident and every sampler, table and program
reads it, so walks equal the unmodified reference's on the same f64 graph —
for weights given at the ABI (wf_graph_create_f64), read from a WFG1 file the
reference wrote with its own synthetic f64 weights, and parsed from a text
edge list with decimal weights."""
import os
import tempfile

import numpy as np
import pytest

from oracle.oracle import RefOracle, ref_available
from paper_2107_11983_b200 import abi
from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import DeepWalkProgram, ExecOptions, Graph, Node2VecProgram, QuerySpec

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def ref_graph():
    # the reference's power-law fixture with its own f64 synthetic weights
    return RefOracle().power_law(3000, 40000, seed=5, weighted=True, label_count=0)


def same(got, want):
    bad = got.walks.first_mismatch(want.walks)
    assert bad is None, f"walk {bad} differs"
    assert got.metrics.total_steps == want.metrics.total_steps


@pytest.mark.parametrize("sampler,tables", [(abi.Sampler.ALIAS, True), (abi.Sampler.ITS, True),
                                            (abi.Sampler.REJ, True), (abi.Sampler.OREJ, True),
                                            (abi.Sampler.ALIAS, False), (abi.Sampler.ITS, False)])
def test_f64_weights_deepwalk_every_sampler(ref_graph, sampler, tables):
    off, nbr, w, _ = ref_graph.export()
    assert not np.array_equal(w.astype(np.float32).astype(np.float64), w)  # really f64
    dg = E.DeviceGraph.from_host(Graph(off, nbr, w))
    assert dg.info()["weights_f64"] and dg.info()["max_weight"] == w.max()
    opts = ExecOptions(seed=4, sampler=int(sampler), use_static_tables=tables)
    prog = DeepWalkProgram(25, True)
    same(E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts),
         ref_graph.run(QuerySpec.one_per_vertex(), prog, opts))


def test_f64_weights_node2vec_and_download(ref_graph):
    off, nbr, w, _ = ref_graph.export()
    dg = E.DeviceGraph.from_host(Graph(off, nbr, w))
    opts = ExecOptions(seed=2)
    prog = Node2VecProgram(2.0, 0.5, 20, True)
    same(E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts),
         ref_graph.run(QuerySpec.one_per_vertex(), prog, opts))
    back = dg.download()
    assert back.weights.dtype == np.float64 and np.array_equal(back.weights, w)


def test_reference_written_wfg1_with_f64_weights(ref_graph):
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "g.wfg")
        ref_graph.write_binary(path)
        dg = E.DeviceGraph.read_wfg1(path)
        opts = ExecOptions(seed=8)
        prog = DeepWalkProgram(30, True)
        same(E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts),
             ref_graph.run(QuerySpec.one_per_vertex(), prog, opts))
        # and written back: the same f64 bytes the reference wrote
        path2 = os.path.join(d, "g2.wfg")
        dg.write_wfg1(path2)
        assert open(path, "rb").read() == open(path2, "rb").read()


def test_decimal_edge_list_weights():
    rng = np.random.default_rng(3)
    lines = []
    for _ in range(6000):
        a, b = rng.integers(0, 800, 2)
        lines.append(f"{a} {b} {rng.integers(1, 1000) / 10.0}")  # 0.1 .. 99.9: not float32-exact
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "e.txt")
        open(path, "w").write("\n".join(lines) + "\n")
        dg = E.DeviceGraph.load_edge_list(path, undirected=True, weights=1)
        rg, _ = RefOracle().load_edge_list(path, undirected=True, weights=1)
        assert dg.info()["weights_f64"]
        for sampler in (abi.Sampler.ALIAS, abi.Sampler.OREJ):
            opts = ExecOptions(seed=6, sampler=int(sampler))
            prog = DeepWalkProgram(15, True)
            same(E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts),
                 rg.run(QuerySpec.one_per_vertex(), prog, opts))
        # random (synthetic_weight) attributes are f64 too (graph.cpp:279-287)
        dgr = E.DeviceGraph.load_edge_list(path, undirected=True, weights=2, seed=9)
        rgr, _ = RefOracle().load_edge_list(path, undirected=True, weights=2, seed=9)
        opts = ExecOptions(seed=6)
        same(E.run_sequential(dgr, QuerySpec.one_per_vertex(), DeepWalkProgram(15, True), opts),
             rgr.run(QuerySpec.one_per_vertex(), DeepWalkProgram(15, True), opts))
