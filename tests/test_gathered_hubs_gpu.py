"""Gathered flows (a gather over all d edges per step, engine.hpp:134-184) on an
R-MAT graph whose hubs have thousands of edges: hub steps run warp-
cooperatively (coop_step: weights 32 edges per round, the ITS pick by a
warp-wide exact scan, ALIAS over the warp's scratch row, REJ's p* as a warp
max), lighter vertices per lane.  Every walk must equal the unmodified
reference's, including where the exactness certificate fails (f64 weights)
and the owner falls back to the reference's edge-order sum."""
import numpy as np
import pytest

from oracle.oracle import RefOracle, ref_available
from paper_2107_11983_b200 import abi
from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, Graph, MetaPathProgram, Node2VecProgram,
                                        QuerySpec)

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]

GATHERED = [abi.Sampler.ITS, abi.Sampler.ALIAS, abi.Sampler.REJ]


@pytest.fixture(scope="module")
def rmat():
    # 10 labels: more than the label index holds, so MetaPath ITS also gathers
    dg = E.DeviceGraph.rmat(14, 16, seed=3, weighted=True, label_count=10)
    hg = dg.download()
    assert np.diff(hg.offsets).max() > 1000  # real hubs
    return dg, hg, RefOracle().graph(hg)


def same(got, want):
    bad = got.walks.first_mismatch(want.walks)
    assert bad is None, f"walk {bad} differs"
    assert got.metrics.total_steps == want.metrics.total_steps


@pytest.mark.parametrize("sampler", GATHERED)
@pytest.mark.parametrize("prog", [DeepWalkProgram(30, True), Node2VecProgram(2.0, 0.5, 30, False),
                                  Node2VecProgram(0.5, 2.0, 30, True), MetaPathProgram([i % 10 for i in range(20)])],
                         ids=["deepwalk_w", "node2vec", "node2vec_w", "metapath10"])
def test_gathered_hub_steps_match_reference(rmat, prog, sampler):
    dg, hg, rg = rmat
    opts = ExecOptions(seed=12, sampler=int(sampler), use_static_tables=False)
    spec = QuerySpec.one_per_vertex()
    sess = E.Session(dg, prog, opts)
    s, f, _ = sess.describe()
    assert f == abi.Flow.GATHERED
    same(E.run_sequential(dg, spec, prog, opts), rg.run(spec, prog, opts))


def test_gathered_hubs_without_exactness_certificate():
    """f64 weights that are not float32-exact: the reordered sum is not
    certified, so ITS scans in the owner lane and ALIAS sums the scratch row
    in edge order — still the reference's walks."""
    ref = RefOracle()
    rg = ref.power_law(3000, 60000, seed=17, weighted=True)
    off, nbr, w, _ = rg.export()
    assert np.diff(off).max() >= 64
    dg = E.DeviceGraph.from_host(Graph(off, nbr, w))
    for sampler in GATHERED:
        opts = ExecOptions(seed=4, sampler=int(sampler), use_static_tables=False)
        prog = DeepWalkProgram(25, True)
        same(E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts),
             rg.run(QuerySpec.one_per_vertex(), prog, opts))


def test_quantum_certificate_mixed_scales():
    """Weights of very different scales (1e-12 .. 1e12, exactly representable
    in f32): the certificate must reject the reordered sum where it would
    round, and the walks still match."""
    rng = np.random.default_rng(8)
    V = 400
    deg = np.where(np.arange(V) < 4, 300, 3)
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    nbr = np.concatenate([np.sort(rng.choice(V, d, replace=False)) for d in deg]).astype(np.uint32)
    scale = rng.choice([1e-12, 1.0, 3.0, 1e12], nbr.size)
    w = (scale * rng.integers(1, 100, nbr.size)).astype(np.float32)
    hg = Graph(off, nbr, w)
    dg = E.DeviceGraph.from_host(hg)
    rg = RefOracle().graph(hg)
    for sampler in GATHERED:
        opts = ExecOptions(seed=2, sampler=int(sampler), use_static_tables=False)
        prog = DeepWalkProgram(20, True)
        same(E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts),
             rg.run(QuerySpec.one_per_vertex(), prog, opts))


def _ceil53(split):
    from fractions import Fraction
    x = Fraction(split) * (1 << 53)
    n = x.numerator // x.denominator
    return n + (1 if n < x else 0)


@pytest.mark.parametrize("f64", [False, True])
def test_static_tables_hub_warps_bit_exact(f64):
    """preprocess_static (engine.hpp:190-251): ITS / REJ hub vertices (>= 64
    edges) are built by a warp each (certified reordered sums / segmented ITS
    scan, warp max for REJ), light ones and every ALIAS vertex per thread.
    Every table equals the reference's, with f32 weights and with f64 ones
    (no certificate: edge-order sums)."""
    dg0 = E.DeviceGraph.rmat(14, 16, seed=7, weighted=True)
    hg = dg0.download()
    if f64:
        w = hg.weights.astype(np.float64) * (1.0 + 1e-9)  # not float32-exact
        hg = Graph(hg.offsets, hg.neighbors, w)
    dg = E.DeviceGraph.from_host(hg)
    assert np.diff(hg.offsets).max() >= 1000 and dg.info()["weights_f64"] == f64
    rg = RefOracle().graph(hg)
    prog = DeepWalkProgram(20, True)
    deg = np.diff(hg.offsets).astype(np.int64)
    for s in GATHERED:
        got = E.Session(dg, prog, ExecOptions(sampler=int(s))).tables()
        want = rg.static_tables(prog, int(s))
        assert np.array_equal(got["exhausted"], want["exhausted"])
        live = np.repeat(want["exhausted"] == 0, deg)
        if s == abi.Sampler.ALIAS:
            thr = np.array([_ceil53(x) for x in want["alias_split"]], dtype=np.uint64)
            assert np.array_equal(got["alias_thr"][live], thr[live])
            assert np.array_equal(got["alias_first_dst"][live], want["alias_first_dst"][live])
            assert np.array_equal(got["alias_second_dst"][live], want["alias_second_dst"][live])
        elif s == abi.Sampler.ITS:
            assert np.array_equal(got["its"], want["its"])
        else:
            assert np.array_equal(got["rej_p_star"], want["rej_p_star"])


def _merge_graph(weighted):
    """Sorted adjacency with multi-edges and self-loops: hubs of 200-3000
    edges (several 128-entry merge windows), mid vertices of 32-120 edges
    whose previous vertex is a hub more than 8x larger (the per-edge test
    path) or comparable (the merge path), and light vertices below 32."""
    rng = np.random.default_rng(21)
    V = 2500
    deg = np.where(np.arange(V) < 12, rng.integers(200, 3000, V),
                   np.where(np.arange(V) < 400, rng.integers(32, 120, V), rng.integers(1, 31, V)))
    lists = []
    for v in range(V):
        d = int(deg[v])
        # half the picks among the hubs and mid vertices (shared neighbourhoods), repeats allowed
        pool = np.where(rng.random(d) < 0.5, rng.integers(0, 400, d), rng.integers(0, V, d))
        if v % 7 == 0:
            pool[0] = v  # self-loop
        lists.append(np.sort(pool))
    off = np.concatenate([[0], np.cumsum([len(x) for x in lists])]).astype(np.uint64)
    nbr = np.concatenate(lists).astype(np.uint32)
    w = (rng.integers(1, 9, nbr.size) * 0.5).astype(np.float32) if weighted else None
    return Graph(off, nbr, w)


@pytest.mark.parametrize("weighted", [False, True])
@pytest.mark.parametrize("sampler", GATHERED)
def test_node2vec_merge_intersection_matches_reference(weighted, sampler):
    """Node2Vec hub gathers take the warp merge of N(cur) and N(prev)
    (n2v_merge_weights) on sorted adjacency: duplicates, self-loops, window
    boundaries and the fallback to per-edge tests must all give the
    reference's walks."""
    hg = _merge_graph(weighted)
    dg = E.DeviceGraph.from_host(hg)
    assert dg.info()["sorted"]
    rg = RefOracle().graph(hg)
    prog = Node2VecProgram(0.5, 2.0, 40, weighted)
    opts = ExecOptions(seed=31, sampler=int(sampler))
    spec = QuerySpec.one_per_vertex()
    same(E.run_sequential(dg, spec, prog, opts), rg.run(spec, prog, opts))


def _big_hub_graph(kind):
    """Hubs of 4500-13000 edges (several 128-entry staging batches per
    cursor, both replay phases): their ALIAS gathers go through the warp's
    staged replay (vose_bucket_staged).  `kind` picks the
    weights: "u15" uniform [1, 5) f32, "wide" mixed scales with zeros, "int"
    small integers (many exact ties with 1.0 after scaling)."""
    rng = np.random.default_rng({"u15": 3, "wide": 5, "int": 7}[kind])
    V = 1500
    deg = np.array([4500, 6100, 9000, 13000] + list(rng.integers(2, 60, V - 4)))
    lists = [np.sort(np.where(rng.random(d) < 0.3, rng.integers(0, 4, d), rng.integers(0, V, d))) for d in deg]
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    nbr = np.concatenate(lists).astype(np.uint32)
    if kind == "u15":
        w = rng.uniform(1, 5, nbr.size).astype(np.float32)
    elif kind == "wide":
        w = (rng.choice([0.0, 0.25, 1.0, 3.0, 1024.0], nbr.size) * rng.integers(1, 50, nbr.size)).astype(np.float32)
    else:
        w = rng.integers(1, 4, nbr.size).astype(np.float32)
    labels = rng.integers(0, 3, nbr.size).astype(np.uint8)
    return Graph(off, nbr, w, labels)


@pytest.mark.parametrize("kind", ["u15", "wide", "int"])
def test_alias_gather_above_lane_row_matches_reference(kind):
    hg = _big_hub_graph(kind)
    dg = E.DeviceGraph.from_host(hg)
    rg = RefOracle().graph(hg)
    opts = ExecOptions(seed=44, sampler=int(abi.Sampler.ALIAS), use_static_tables=False)
    spec = QuerySpec.from_list(np.repeat(np.arange(8, dtype=np.uint32), 40))  # many walks through the hubs
    for prog in [DeepWalkProgram(30, True), MetaPathProgram([i % 3 for i in range(25)]),
                 Node2VecProgram(0.5, 2.0, 25, True)]:
        same(E.run_sequential(dg, spec, prog, opts), rg.run(spec, prog, opts))


@pytest.mark.parametrize("label_p", [0.03, 0.2, 0.5, 0.9, 1.0])
def test_alias_gather_uniform_weights_closed_form(label_p):
    """Every positive weight equal (MetaPath's 0/1 weights; unweighted
    DeepWalk): the hub's Vose replay is a closed form (vose_bucket_uniform)
    with the chain only for larges the first phase leaves; the share of
    matching edges sets c = n/m (integer and fractional), both phases and the
    leftovers."""
    rng = np.random.default_rng(int(label_p * 100) + 3)
    V = 1200
    deg = np.array([40, 97, 256, 1000, 3001, 7000] + list(rng.integers(1, 50, V - 6)))
    lists = [np.sort(rng.integers(0, V, d)) for d in deg]
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    nbr = np.concatenate(lists).astype(np.uint32)
    labels = np.where(rng.random(nbr.size) < label_p, 1, 0).astype(np.uint8)
    hg = Graph(off, nbr, rng.uniform(1, 5, nbr.size).astype(np.float32), labels)
    dg = E.DeviceGraph.from_host(hg)
    rg = RefOracle().graph(hg)
    spec = QuerySpec.from_list(np.repeat(np.arange(6, dtype=np.uint32), 60))
    opts = ExecOptions(seed=9, sampler=int(abi.Sampler.ALIAS), use_static_tables=False)
    for prog in [MetaPathProgram([1] * 12), DeepWalkProgram(12, False)]:
        same(E.run_sequential(dg, spec, prog, opts), rg.run(spec, prog, opts))
