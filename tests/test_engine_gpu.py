"""GPU parity: the CUDA engine (through the C-ABI) against the reference.

* golden fixtures made by the unmodified reference (tests/golden/): RNG vectors,
  every program x sampler x flow combination, edge cases, error classes, static
  tables — bit-exact;
* synthetic R-MAT graphs generated on the device, compared with the reference
  engine (oracle/_ref) or the C restatement on the same CSR — bit-exact walks;
* size-independent properties at full BASELINE sizes (tests/test_configs_gpu.py).
"""
import os

import numpy as np
import pytest

from oracle.oracle import PortOracle, RefOracle, ref_available
from paper_2107_11983_b200 import abi
from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, MetaPathProgram,
                                        Node2VecProgram, PprProgram, QuerySpec, UniformProgram)
from tests import golden_util as gu
from oracle.rmat_ref import rmat_csr

pytestmark = pytest.mark.gpu

CASES = gu.cases()
_graphs = {}


def dgraph(name):
    if name not in _graphs:
        _graphs[name] = E.DeviceGraph.from_host(gu.graph(name))
    return _graphs[name]


def oracle():
    return RefOracle() if ref_available() else None


def test_rng_matches_reference_vectors():
    z = gu.rng()
    for (s, q), draws in zip(z["pairs"], z["draws"]):
        got = E.rng_probe(int(s), [int(q)], 16)[0]
        assert np.array_equal(got, draws)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_golden_case(case):
    g = dgraph(case["graph"])
    if "error" in case:
        with pytest.raises(getattr(abi, case["error"])):
            E.run_sequential(g, gu.spec(case), gu.program(case), gu.opts(case))
        return
    res = E.run_sequential(g, gu.spec(case), gu.program(case), gu.opts(case))
    want = gu.walks(case)
    bad = res.walks.first_mismatch(want)
    assert bad is None, (bad, res.walks.path(bad) if bad is not None and bad < len(res.walks) else None,
                         want.path(bad) if bad is not None and bad < len(want) else None)
    assert res.metrics.total_steps == case["total_steps"]


def test_golden_cases_interleaved_entry_point():
    case = next(c for c in CASES if c["name"] == "pl_node2vec_w_orej")
    res = E.run_interleaved(dgraph(case["graph"]), gu.spec(case), gu.program(case), 64, 32,
                            gu.opts(case))
    assert res.walks.equals(gu.walks(case))
    with pytest.raises(abi.ConfigError):
        E.run_interleaved(dgraph(case["graph"]), gu.spec(case), gu.program(case), 4, 8,
                          gu.opts(case))


@pytest.mark.parametrize("gname", ["powerlaw", "zeroweights", "ring"])
def test_static_tables_bit_exact(gname):
    t = gu.tables()
    g = dgraph(gname)
    prog = DeepWalkProgram(20, True)
    for s in [abi.Sampler.ALIAS, abi.Sampler.ITS, abi.Sampler.REJ]:
        sess = E.Session(g, prog, ExecOptions(sampler=s))
        out = sess.tables()
        key = f"{gname}/{s.name.lower()}"
        ex = t[f"{key}/exhausted"]
        assert np.array_equal(out["exhausted"], ex)
        if s == abi.Sampler.ALIAS:
            split = t[f"{key}/alias_split"]
            thr = np.array([_ceil53(x) for x in split], dtype=np.uint64)
            # slots of exhausted vertices are never read (the reference leaves them zeroed)
            live = np.repeat(ex == 0, np.diff(gu.graph(gname).offsets).astype(np.int64))
            assert np.array_equal(out["alias_thr"][live], thr[live])
            assert np.array_equal(out["alias_first_dst"][live], t[f"{key}/alias_first_dst"][live])
            assert np.array_equal(out["alias_second_dst"][live], t[f"{key}/alias_second_dst"][live])
        elif s == abi.Sampler.ITS:
            assert np.array_equal(out["its"], t[f"{key}/its"])
        else:
            assert np.array_equal(out["rej_p_star"], t[f"{key}/rej_p_star"])


def _ceil53(split: float) -> int:
    from fractions import Fraction
    x = Fraction(split) * (1 << 53)
    n = x.numerator // x.denominator
    return n + (1 if n < x else 0)


def test_unit_threshold_equivalence():
    """(r >> 11) < ceil(c * 2^53) <=> uniform_real(1.0) < c, over random r and
    adversarial c next to the draw."""
    rng = np.random.default_rng(0)
    port = PortOracle()
    for _ in range(2000):
        seed, stream = (int(x) for x in rng.integers(0, 2 ** 63, 2))
        r = int(port.rng_probe(seed, stream, 1)[0])
        k = r >> 11
        u = k * 2.0 ** -53
        for c in [u, np.nextafter(u, 0), np.nextafter(u, 1), 0.2, 1.0, 0.5]:
            if not (0 < c <= 1):
                continue
            assert (k < _ceil53(c)) == (u < c)


@pytest.mark.parametrize("scale,weighted,labels", [(6, False, 0), (9, True, 5), (10, True, 3)])
def test_rmat_generator_matches_reference_restatement(scale, weighted, labels):
    g = E.DeviceGraph.rmat(scale, 16, seed=7, weighted=weighted, label_count=labels).download()
    off, nbr, w, lab = rmat_csr(scale, 16, seed=7, weighted=weighted, label_count=labels)
    assert np.array_equal(g.offsets, off)
    assert np.array_equal(g.neighbors, nbr)
    if weighted:
        assert np.array_equal(g.weights, w)
    if labels:
        assert np.array_equal(g.labels, lab)


def test_rmat_weights_are_reference_synthetic_weights():
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    ref = RefOracle()
    g = E.DeviceGraph.rmat(8, 16, seed=3, weighted=True, label_count=5).download()
    for e in range(0, g.edge_count, 97):
        assert g.weights[e] == np.float32(ref.synthetic_weight(3, e))
        assert g.labels[e] == ref.synthetic_label(3, e, 5)


def _compare_with_reference(dg, hg, spec, prog, opts, qids=None):
    ref = RefOracle() if ref_available() else None
    if ref is not None:
        rg = ref.graph(hg)
        want = rg.run_qids(spec, prog, opts, qids) if qids is not None else rg.run(spec, prog, opts)
    else:
        want = PortOracle().run(hg, spec, prog, opts, qids=qids, threads=4)
    got = E.run_sequential(dg, spec, prog, opts)
    if qids is not None:
        gw = got.walks
        for i, q in enumerate(qids):
            assert gw.status[q] == want.walks.status[i]
            assert np.array_equal(gw.path(int(q)), want.walks.path(i)), int(q)
    else:
        bad = got.walks.first_mismatch(want.walks)
        assert bad is None, bad
        assert got.metrics.total_steps == want.metrics.total_steps
    return got


RMAT_PROGRAMS = [
    ("ppr_naive", lambda: PprProgram(0.2), None),
    ("ppr_alias", lambda: PprProgram(0.2), abi.Sampler.ALIAS),
    ("deepwalk_alias_w", lambda: DeepWalkProgram(80, True), None),
    ("deepwalk_its_w", lambda: DeepWalkProgram(40, True), abi.Sampler.ITS),
    ("deepwalk_rej_w", lambda: DeepWalkProgram(40, True), abi.Sampler.REJ),
    ("node2vec_orej", lambda: Node2VecProgram(2.0, 0.5, 80, False), None),
    ("node2vec_orej_w", lambda: Node2VecProgram(2.0, 0.5, 40, True), None),
    ("node2vec_its", lambda: Node2VecProgram(2.0, 0.5, 12, False), abi.Sampler.ITS),
    ("metapath_its", lambda: MetaPathProgram([i % 5 for i in range(79)]), None),
    ("metapath_rej", lambda: MetaPathProgram([i % 5 for i in range(20)]), abi.Sampler.REJ),
    ("metapath_alias", lambda: MetaPathProgram([i % 5 for i in range(10)]), abi.Sampler.ALIAS),
    ("uniform_naive", lambda: UniformProgram(30), None),
]


@pytest.fixture(scope="module")
def rmat12():
    dg = E.DeviceGraph.rmat(12, 16, seed=1, weighted=True, label_count=5)
    return dg, dg.download()


@pytest.mark.parametrize("name,mk,sampler", RMAT_PROGRAMS, ids=[p[0] for p in RMAT_PROGRAMS])
def test_rmat12_all_walks_match_reference(rmat12, name, mk, sampler):
    dg, hg = rmat12
    spec = QuerySpec.one_per_vertex()
    if name.startswith("ppr"):
        spec = QuerySpec.from_list(np.random.default_rng(5).integers(0, hg.vertex_count, 20000))
    _compare_with_reference(dg, hg, spec, mk(), ExecOptions(seed=11, sampler=sampler))


def test_ppr_row_overflow_rerun_is_exact(rmat12):
    """Walks longer than the row capacity are re-run into their own rows."""
    dg, hg = rmat12
    spec = QuerySpec.from_list(np.random.default_rng(9).integers(0, hg.vertex_count, 5000))
    opts = ExecOptions(seed=3, path_stride=2)
    got = _compare_with_reference(dg, hg, spec, PprProgram(0.1), opts)
    assert got.walks.lengths().max() > 2


def test_visit_counts_match_paths(rmat12):
    dg, hg = rmat12
    spec = QuerySpec.from_list(np.random.default_rng(2).integers(0, hg.vertex_count, 30000))
    sess = E.Session(dg, PprProgram(0.2), ExecOptions(seed=5, path_stride=4))
    ws = sess.run(spec)
    host = ws.to_host()
    want = np.bincount(host.vertices, minlength=hg.vertex_count).astype(np.uint32)
    assert np.array_equal(ws.visit_counts(), want)
    sess2 = E.Session(dg, DeepWalkProgram(10, True), ExecOptions(seed=5))
    ws2 = sess2.run(QuerySpec.one_per_vertex())
    h2 = ws2.to_host()
    assert np.array_equal(ws2.visit_counts(),
                          np.bincount(h2.vertices, minlength=hg.vertex_count).astype(np.uint32))


def test_label_index_path_equals_label_scan_path(rmat12):
    """MetaPath through the label-partitioned CSR equals the generic per-step
    label scan (the reference's gather) on the same queries."""
    dg, hg = rmat12
    schema = [i % 5 for i in range(40)]
    fast = E.run_sequential(dg, QuerySpec.one_per_vertex(), MetaPathProgram(schema),
                            ExecOptions(seed=4))
    want = PortOracle().run(hg, QuerySpec.one_per_vertex(), MetaPathProgram(schema),
                            ExecOptions(seed=4), threads=4)
    assert fast.walks.equals(want.walks)


def test_results_independent_of_launch_and_repeat(rmat12):
    dg, _ = rmat12
    prog = Node2VecProgram(2.0, 0.5, 30, False)
    a = E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, ExecOptions(seed=8))
    b = E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, ExecOptions(seed=8, k=1, k_prime=1))
    assert a.walks.equals(b.walks)


def test_session_launch_chunks_equal_whole_run(rmat12):
    """Query ranges launched separately (the multi-GPU shard path) reproduce the
    whole run: walks depend only on (seed, qid)."""
    import torch
    dg, hg = rmat12
    prog = DeepWalkProgram(20, True)
    opts = ExecOptions(seed=13)
    whole = E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts).walks
    sess = E.Session(dg, prog, opts)
    n = hg.vertex_count
    paths = torch.zeros(n * 20, dtype=torch.int32, device="cuda")
    lens = torch.zeros(n, dtype=torch.int32, device="cuda")
    st = torch.zeros(n, dtype=torch.uint8, device="cuda")
    steps = torch.zeros(1, dtype=torch.int64, device="cuda")
    bounds = [0, 1000, 1001, 2500, n]
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        sess.launch(QuerySpec.one_per_vertex(), lo, hi, paths.data_ptr() + lo * 20 * 4, 20,
                    lens.data_ptr() + lo * 4, st.data_ptr() + lo, 0, steps.data_ptr())
    sess.sync()
    rows = paths.view(n, 20).cpu().numpy().view(np.uint32)
    L = lens.cpu().numpy()
    assert np.array_equal(L, whole.lengths())
    for q in range(0, n, 7):
        assert np.array_equal(rows[q, :L[q]], whole.path(q))
    assert int(steps.item()) == int(whole.lengths().sum() - n)


def test_errors_surface_as_reference_classes(rmat12):
    import torch
    dg, hg = rmat12
    with pytest.raises(abi.ConfigError):
        E.Session(dg, MetaPathProgram([0, 1]), ExecOptions(sampler=abi.Sampler.OREJ))
    with pytest.raises(abi.ConfigError):
        E.Session(dg, DeepWalkProgram(5, True), ExecOptions(sampler=abi.Sampler.NAIVE))
    with pytest.raises(abi.ConfigError):
        E.run_sequential(dg, QuerySpec.from_source(hg.vertex_count + 3, 4), PprProgram(0.2))
    # a source list with a non-vertex: the host list through run_host (checked by
    # the walk kernel, named on the host) and a device list through launch
    bad = np.arange(64, dtype=np.uint32)
    bad[37] = hg.vertex_count + 9
    sess = E.Session(dg, PprProgram(0.2), ExecOptions(seed=1, path_stride=64))
    off = np.zeros(65, np.uint64)
    verts = np.zeros(64 * 64, np.uint32)
    st = np.zeros(64, np.uint8)
    with pytest.raises(abi.ConfigError, match=str(hg.vertex_count + 9)):
        sess.run_host(QuerySpec.from_list(bad), off.ctypes.data, verts.ctypes.data, verts.size,
                      st.ctypes.data)
    d_src = torch.from_numpy(bad.view(np.int32)).cuda()
    paths = torch.empty(64 * 64, dtype=torch.int32, device="cuda")
    lens = torch.empty(64, dtype=torch.int32, device="cuda")
    stat = torch.empty(64, dtype=torch.uint8, device="cuda")
    with pytest.raises(abi.ConfigError):
        sess.launch(QuerySpec.from_list(bad), 0, 64, paths.data_ptr(), 64, lens.data_ptr(),
                    stat.data_ptr(), 0, 0, 0, 0, sources_dev_ptr=d_src.data_ptr())
        sess.sync(0)
    # the session is usable again after the error
    good = QuerySpec.from_list(np.arange(64, dtype=np.uint32))
    sess.run_host(good, off.ctypes.data, verts.ctypes.data, verts.size, st.ctypes.data)
    # a trial cap the bound cannot meet: RejectionCapError raised after the sync
    with pytest.raises(abi.RejectionCapError):
        E.run_sequential(dg, QuerySpec.one_per_vertex(), Node2VecProgram(0.01, 0.5, 10, False),
                         ExecOptions(seed=1, rej_trial_cap=1))


def test_graph_validation_like_from_csr():
    from paper_2107_11983_b200.host import Graph
    bad = Graph(np.array([0, 2, 1], np.uint64), np.array([1, 0], np.uint32))
    with pytest.raises(abi.ConfigError):
        E.DeviceGraph.from_host(bad)
    bad2 = Graph(np.array([0, 1, 2], np.uint64), np.array([1, 5], np.uint32))
    with pytest.raises(abi.ConfigError):
        E.DeviceGraph.from_host(bad2)
    bad3 = Graph(np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint32),
                 np.array([1.0, -2.0], np.float32))
    with pytest.raises(abi.ConfigError):
        E.DeviceGraph.from_host(bad3)


def test_has_edge_matches_reference(rmat12):
    dg, hg = rmat12
    rng = np.random.default_rng(1)
    src = rng.integers(0, hg.vertex_count, 5000)
    dst = np.where(rng.random(5000) < 0.5, rng.integers(0, hg.vertex_count, 5000),
                   [hg.neighbors_of(int(s))[0] if hg.degree(int(s)) else 0 for s in src])
    got = dg.has_edge(src, dst)
    want = np.array([d in set(hg.neighbors_of(int(s)).tolist()) for s, d in zip(src, dst)])
    assert np.array_equal(got, want)


LAYOUT_CASES = [
    ("deepwalk_compact_alias", lambda: DeepWalkProgram(40, True), abi.LAYOUT_COMPACT_ALIAS, 0),
    ("deepwalk_wide_alias", lambda: DeepWalkProgram(40, True), abi.LAYOUT_WIDE_ALIAS, abi.HAS_WIDE_ALIAS),
    ("deepwalk_default_alias", lambda: DeepWalkProgram(40, True), 0, 0),  # small graph: compact
    ("ppr_adj", lambda: PprProgram(0.2), abi.LAYOUT_FORCE_ADJ, abi.HAS_ADJ),
    ("ppr_no_adj", lambda: PprProgram(0.2), abi.LAYOUT_NO_ADJ, 0),
    ("node2vec_adj", lambda: Node2VecProgram(2.0, 0.5, 40, False), abi.LAYOUT_FORCE_ADJ,
     abi.HAS_ADJ | abi.HAS_EDGE_HASH),
    ("node2vec_w_adj", lambda: Node2VecProgram(0.5, 3.0, 30, True), abi.LAYOUT_FORCE_ADJ,
     abi.HAS_ADJ | abi.HAS_EDGE_HASH),
    ("node2vec_no_adj", lambda: Node2VecProgram(2.0, 0.5, 40, False), abi.LAYOUT_NO_ADJ,
     abi.HAS_EDGE_HASH | abi.HAS_EDGE_FILTER),
    ("node2vec_no_filter", lambda: Node2VecProgram(2.0, 0.5, 40, False), abi.LAYOUT_NO_EDGE_FILTER,
     abi.HAS_EDGE_HASH),
    ("node2vec_w_no_filter_tree", lambda: Node2VecProgram(0.5, 3.0, 30, True),
     abi.LAYOUT_NO_EDGE_FILTER | abi.LAYOUT_SEARCH_TREE, abi.HAS_SEARCH_INDEX),
    ("node2vec_search_tree", lambda: Node2VecProgram(2.0, 0.5, 40, False),
     abi.LAYOUT_SEARCH_TREE | abi.LAYOUT_FORCE_ADJ, abi.HAS_ADJ | abi.HAS_SEARCH_INDEX),
    ("node2vec_w_search_tree", lambda: Node2VecProgram(0.5, 3.0, 30, True),
     abi.LAYOUT_SEARCH_TREE, abi.HAS_SEARCH_INDEX),
    ("metapath_succ", lambda: MetaPathProgram([i % 5 for i in range(40)]), abi.LAYOUT_MP_SUCC,
     abi.HAS_MP_SUCC | abi.HAS_LABEL_INDEX),
    ("metapath_succ_irregular", lambda: MetaPathProgram([0, 1, 0, 2, 3, 1, 4]), abi.LAYOUT_MP_SUCC,
     abi.HAS_LABEL_INDEX),  # successor of 0 is not unique: falls back to records
    ("metapath_records", lambda: MetaPathProgram([i % 5 for i in range(40)]), abi.LAYOUT_NO_MP_SUCC,
     abi.HAS_LABEL_INDEX),
    ("metapath_default_succ", lambda: MetaPathProgram([i % 5 for i in range(40)]), 0,
     abi.HAS_MP_SUCC | abi.HAS_LABEL_INDEX),
    ("ppr_adj8", lambda: PprProgram(0.15), abi.LAYOUT_ADJ8, abi.HAS_ADJ8),
    ("node2vec_adj8", lambda: Node2VecProgram(2.0, 0.5, 40, False), abi.LAYOUT_ADJ8,
     abi.HAS_ADJ8 | abi.HAS_EDGE_HASH | abi.HAS_EDGE_FILTER),
    ("node2vec_w_adj8", lambda: Node2VecProgram(0.5, 3.0, 30, True), abi.LAYOUT_ADJ8, abi.HAS_ADJ8),
]


@pytest.mark.parametrize("name,mk,flags,expect", LAYOUT_CASES, ids=[c[0] for c in LAYOUT_CASES])
def test_every_hbm_layout_is_bit_exact(rmat12, name, mk, flags, expect):
    """Each decorated / compact layout (abi.LAYOUT_*) gives the reference's walks."""
    dg, hg = rmat12
    prog = mk()
    spec = QuerySpec.one_per_vertex()
    if name.startswith("ppr"):
        spec = QuerySpec.from_list(np.random.default_rng(8).integers(0, hg.vertex_count, 20000))
    opts = ExecOptions(seed=23, layout_flags=flags)
    sess = E.Session(dg, prog, opts)
    assert sess.layout() & expect == expect
    if not expect & abi.HAS_WIDE_ALIAS and name.startswith("deepwalk"):
        assert not sess.layout() & abi.HAS_WIDE_ALIAS
    _compare_with_reference(dg, hg, spec, prog, opts)


@pytest.mark.parametrize("prog,chunk,nsrc", [(PprProgram(0.1), 1000, 9000),
                                             (PprProgram(0.2), 1 << 14, 1 << 18),
                                             (DeepWalkProgram(24, True), 777, 9000),
                                             (Node2VecProgram(2.0, 0.5, 16, False), 0, 9000),
                                             (MetaPathProgram([i % 5 for i in range(12)]), 513, 9000)])
def test_run_host_streaming_equals_run(rmat12, prog, chunk, nsrc):
    """wf_session_run_host (chunked compute/copy pipeline into host buffers),
    called repeatedly on one session and on qid sub-ranges, equals the walk set
    of run_sequential — including PPR walks that outgrow their row (stride 8)."""
    dg, hg = rmat12
    src = np.random.default_rng(3).integers(0, hg.vertex_count, nsrc).astype(np.uint32)
    spec = QuerySpec.from_list(src)
    opts = ExecOptions(seed=17, path_stride=8)
    whole = E.run_sequential(dg, spec, prog, opts).walks
    sess = E.Session(dg, prog, opts)
    for rep in range(3):
        res = sess.run_to_numpy(spec, chunk=chunk)
        assert res.walks.equals(whole), rep
        assert res.metrics.total_steps == int(whole.lengths().sum()) - len(whole)
    # a shard [lo, hi) through the raw call
    lo, hi = 2500, min(nsrc, 7100 + nsrc // 2)
    n = hi - lo
    off = np.zeros(n + 1, np.uint64)
    cap = int(whole.offsets[hi] - whole.offsets[lo]) + 16
    verts = np.zeros(cap, np.uint32)
    st = np.zeros(n, np.uint8)
    sess.run_host(spec, off.ctypes.data, verts.ctypes.data, cap, st.ctypes.data, chunk=chunk,
                  qid_begin=lo, qid_end=hi)
    base = whole.offsets[lo]
    assert np.array_equal(off, whole.offsets[lo:hi + 1] - base)
    assert np.array_equal(verts[:int(off[-1])], whole.vertices[int(base):int(whole.offsets[hi])])
    assert np.array_equal(st, whole.status[lo:hi])


@pytest.mark.parametrize("mode", ["whole", "chunks"])
@pytest.mark.parametrize("stage_bytes", [None, 3 << 17])
def test_run_host_modes_and_segments(rmat12, monkeypatch, mode, stage_bytes):
    """Both host-streaming modes (whole-launch publication for short walks,
    in-kernel chunk reports for long ones) give every program's exact walk
    set, also when a small staging budget splits the run into several
    launches (segments) and the chunks into batches."""
    dg, hg = rmat12
    monkeypatch.setenv("WF_STREAM_MODE", mode)
    if stage_bytes:
        monkeypatch.setenv("WF_STREAM_STAGE_BYTES", str(stage_bytes))
    src = np.random.default_rng(21).integers(0, hg.vertex_count, 30000).astype(np.uint32)
    spec = QuerySpec.from_list(src)
    for prog, chunk in [(PprProgram(0.2), 1 << 10), (DeepWalkProgram(20, True), 0),
                        (Node2VecProgram(2.0, 0.5, 12, False), 1 << 12), (UniformProgram(9), 100),
                        (MetaPathProgram([i % 5 for i in range(10)]), 1 << 11)]:
        opts = ExecOptions(seed=29, path_stride=16)
        whole = E.run_sequential(dg, spec, prog, opts).walks
        sess = E.Session(dg, prog, opts)
        res = sess.run_to_numpy(spec, chunk=chunk)
        assert res.walks.equals(whole), (type(prog).__name__, mode, stage_bytes)
        n, total = src.size, int(whole.offsets[-1])
        rec = np.zeros(n, np.uint32)
        verts = np.zeros(total, np.uint32)
        sess.run_host_records(spec, rec.ctypes.data, verts.ctypes.data, total, chunk=chunk)
        assert np.array_equal(rec & 0x7FFFFFFF, np.diff(whole.offsets).astype(np.uint32))
        assert np.array_equal((rec >> 31).astype(np.uint8), whole.status)
        assert np.array_equal(verts, whole.vertices)
        # a pinned source list streams in while the kernels run (src_ready)
        import torch
        pinned = torch.from_numpy(src.view(np.int32)).pin_memory()
        h_rec = torch.zeros(n, dtype=torch.int32).pin_memory()
        h_vert = torch.zeros(total, dtype=torch.int32).pin_memory()
        sess.run_host_records(QuerySpec.from_list(pinned.numpy().view(np.uint32)), h_rec.data_ptr(),
                              h_vert.data_ptr(), total, chunk=chunk)
        assert np.array_equal(h_rec.numpy().view(np.uint32), rec)
        assert np.array_equal(h_vert.numpy().view(np.uint32), whole.vertices)


@pytest.mark.parametrize("mode", ["whole", "chunks"])
def test_run_host_errors_in_both_modes(rmat12, monkeypatch, mode):
    """Device-side errors surface from the streaming pipeline as the reference's
    exception classes, with pinned (streamed) and pageable source lists, and
    the session stays usable: a non-vertex source (ConfigError) and a trial cap
    the O-REJ bound cannot meet (RejectionCapError)."""
    import torch
    dg, hg = rmat12
    monkeypatch.setenv("WF_STREAM_MODE", mode)
    n = 1 << 16
    src = np.random.default_rng(4).integers(0, hg.vertex_count, n).astype(np.uint32)
    src[n - 5] = hg.vertex_count + 3
    pinned = torch.from_numpy(src.view(np.int32)).pin_memory()
    sess = E.Session(dg, PprProgram(0.2), ExecOptions(seed=2, path_stride=64))
    verts = torch.zeros(n * 64, dtype=torch.int32).pin_memory()
    rec = torch.zeros(n, dtype=torch.int32).pin_memory()
    for sources in (src, pinned.numpy().view(np.uint32)):
        with pytest.raises(abi.ConfigError, match=str(hg.vertex_count + 3)):
            sess.run_host_records(QuerySpec.from_list(sources), rec.data_ptr(), verts.data_ptr(), n * 64,
                                  chunk=1 << 12)
    good = src.copy()
    good[n - 5] = 7
    whole = E.run_sequential(dg, QuerySpec.from_list(good), PprProgram(0.2), ExecOptions(seed=2)).walks
    sess.run_host_records(QuerySpec.from_list(good), rec.data_ptr(), verts.data_ptr(), n * 64, chunk=1 << 12)
    total = int(whole.offsets[-1])
    assert np.array_equal(verts.numpy()[:total].view(np.uint32), whole.vertices)
    n2v = E.Session(dg, Node2VecProgram(0.01, 0.5, 10, False), ExecOptions(seed=1, rej_trial_cap=1))
    with pytest.raises(abi.RejectionCapError):
        n2v.run_to_numpy(QuerySpec.one_per_vertex())


@pytest.mark.parametrize("mode", ["whole", "chunks"])
@pytest.mark.parametrize("prog,stride", [(PprProgram(0.2), 64), (PprProgram(0.1), 8),
                                         (DeepWalkProgram(24, True), 0),
                                         (Node2VecProgram(2.0, 0.5, 16, False), 0)])
def test_run_host_blocks_deliver_final_bytes_in_order(rmat12, monkeypatch, mode, prog, stride):
    """wf_session_run_host_blocks (the BlockSink form): blocks arrive in qid
    order, consecutive, covering the run, and what the host buffers hold for a
    block AT ITS CALLBACK is already the final walk set (blocks with walks
    longer than their row, stride 8, come after the patch).  A callback that
    returns non-zero stops the run with IoError; the session stays usable."""
    import torch
    dg, hg = rmat12
    monkeypatch.setenv("WF_STREAM_MODE", mode)
    src = np.random.default_rng(31).integers(0, hg.vertex_count, 1 << 17).astype(np.uint32)
    spec = QuerySpec.from_list(src)
    opts = ExecOptions(seed=47, path_stride=stride)
    whole = E.run_sequential(dg, spec, prog, opts).walks
    n, total = src.size, int(whole.offsets[-1])
    sess = E.Session(dg, prog, opts)
    h_rec = torch.zeros(n, dtype=torch.int32).pin_memory()
    h_vert = torch.zeros(total + 64, dtype=torch.int32).pin_memory()
    rec_np, vert_np = h_rec.numpy().view(np.uint32), h_vert.numpy().view(np.uint32)
    seen = []

    def on_block(b, q0, q1, v0):
        rec = rec_np[q0:q1].copy()
        nv = int((rec & 0x7FFFFFFF).astype(np.int64).sum())
        seen.append((b, q0, q1, v0, rec, vert_np[v0:v0 + nv].copy()))

    m = sess.run_host_blocks(spec, h_rec.data_ptr(), h_vert.data_ptr(), total + 64, on_block, chunk=1 << 12)
    assert m.total_steps == total - n
    assert [b for b, *_ in seen] == list(range(len(seen))) and len(seen) > 1
    assert seen[0][1] == 0 and seen[-1][2] == n
    for (_, q0, q1, v0, rec, verts), nxt in zip(seen, seen[1:] + [None]):
        if nxt is not None:
            assert nxt[1] == q1
        assert v0 == int(whole.offsets[q0])
        assert np.array_equal(rec & 0x7FFFFFFF, np.diff(whole.offsets[q0:q1 + 1]).astype(np.uint32))
        assert np.array_equal((rec >> 31).astype(np.uint8), whole.status[q0:q1])
        assert np.array_equal(verts, whole.vertices[v0:int(whole.offsets[q1])])
    # a shard [lo, hi): qids and vertex offsets relative to lo
    lo, hi = 12345, 100000
    got = []
    sess.run_host_blocks(spec, h_rec.data_ptr(), h_vert.data_ptr(), total + 64,
                         lambda b, q0, q1, v0: got.append((q0, q1, v0)), chunk=1 << 12, qid_begin=lo, qid_end=hi)
    assert got[0][0] == 0 and got[-1][1] == hi - lo
    base = int(whole.offsets[lo])
    for q0, q1, v0 in got:
        assert v0 == int(whole.offsets[lo + q0]) - base
    nv = int(whole.offsets[hi]) - base
    assert np.array_equal(vert_np[:nv], whole.vertices[base:base + nv])
    # stopping the run from the callback
    with pytest.raises(abi.IoError):
        sess.run_host_blocks(spec, h_rec.data_ptr(), h_vert.data_ptr(), total + 64,
                             lambda b, *_: b == 1, chunk=1 << 12)
    h_vert.fill_(0)
    sess.run_host_records(spec, h_rec.data_ptr(), h_vert.data_ptr(), total + 64, chunk=1 << 12)
    assert np.array_equal(vert_np[:total], whole.vertices)


def test_launch_tuner_keeps_results(rmat12):
    """wf_session_tune only changes the grid: walks are identical before and after."""
    import torch
    dg, hg = rmat12
    rng = np.random.default_rng(5)
    src = rng.integers(0, hg.vertex_count, 20000, dtype=np.uint32)
    spec = QuerySpec.from_list(src)
    sess = E.Session(dg, PprProgram(0.2), ExecOptions(seed=3, path_stride=64))
    n = src.size

    def run():
        d_src = torch.from_numpy(src.view(np.int32)).cuda()
        paths = torch.zeros(n * 64, dtype=torch.int32, device="cuda")
        lens = torch.zeros(n, dtype=torch.int32, device="cuda")
        st = torch.zeros(n, dtype=torch.uint8, device="cuda")
        counts = torch.zeros(hg.vertex_count, dtype=torch.int32, device="cuda")
        sess.launch(spec, 0, n, paths.data_ptr(), 64, lens.data_ptr(), st.data_ptr(), counts.data_ptr(),
                    sources_dev_ptr=d_src.data_ptr())
        sess.sync(0)
        L = lens.cpu().numpy()
        P = paths.cpu().numpy().reshape(n, 64)
        rows = [P[i, :min(L[i], 64)].copy() for i in range(n)]
        return L, rows, st.cpu().numpy(), counts.cpu().numpy()

    before = run()
    blocks, ms = sess.tune(spec)
    assert 1 <= blocks <= 8 and ms > 0
    after = run()
    assert np.array_equal(before[0], after[0])
    assert all(np.array_equal(a, b) for a, b in zip(before[1], after[1]))
    assert np.array_equal(before[2], after[2])
    assert np.array_equal(before[3], after[3])


def test_degree_escape_vertex_matches_reference():
    """A vertex of degree >= 2^24 - 1 does not fit the packed vertex word and is
    read through the offsets (kDegEscape): walks through it stay bit-exact."""
    from paper_2107_11983_b200.host import Graph
    D = (1 << 24) + 37
    V = D + 1
    offsets = np.empty(V + 1, np.uint64)
    offsets[0] = 0
    offsets[1:] = D + np.arange(0, V, dtype=np.uint64)
    nbr = np.empty(2 * D, np.uint32)
    nbr[:D] = np.arange(1, V, dtype=np.uint32)
    nbr[D:] = 0
    w = np.random.default_rng(1).uniform(1.0, 5.0, 2 * D).astype(np.float32)
    hg = Graph(offsets, nbr, w)
    dg = E.DeviceGraph.from_host(hg)
    src = np.where(np.arange(512) % 2 == 0, 0, np.random.default_rng(2).integers(1, V, 512)).astype(np.uint32)
    spec = QuerySpec.from_list(src)
    for prog, sampler in [(PprProgram(0.2), None), (DeepWalkProgram(12, True), None),
                          (DeepWalkProgram(12, True), abi.Sampler.ITS),
                          (Node2VecProgram(2.0, 0.5, 12, False), None), (UniformProgram(12), None)]:
        opts = ExecOptions(seed=31, sampler=sampler)
        _compare_with_reference(dg, hg, spec, prog, opts)


@pytest.mark.parametrize("prog,chunk,stride", [(PprProgram(0.2), 1 << 14, 64), (PprProgram(0.1), 5000, 8),
                                               (DeepWalkProgram(24, True), 7777, 0),
                                               (MetaPathProgram([i % 5 for i in range(12)]), 0, 0)])
def test_run_host_pinned_equals_run(rmat12, prog, chunk, stride):
    """Pinned host buffers (the bench's e2e path): the same bytes as the walk
    set of run_sequential, including walks that outgrow their row, and a
    too-small capacity is an error, not an overrun."""
    import torch
    dg, hg = rmat12
    src = np.random.default_rng(9).integers(0, hg.vertex_count, 1 << 17).astype(np.uint32)
    spec = QuerySpec.from_list(src)
    opts = ExecOptions(seed=41, path_stride=stride)
    whole = E.run_sequential(dg, spec, prog, opts).walks
    n = src.size
    total = int(whole.offsets[-1])
    sess = E.Session(dg, prog, opts)
    h_off = torch.zeros(n + 1, dtype=torch.int64).pin_memory()
    h_vert = torch.zeros(total + 64, dtype=torch.int32).pin_memory()
    h_stat = torch.zeros(n, dtype=torch.uint8).pin_memory()
    for rep in range(2):
        h_vert.fill_(-1)
        m = sess.run_host(spec, h_off.data_ptr(), h_vert.data_ptr(), total + 64, h_stat.data_ptr(), chunk=chunk)
        assert np.array_equal(h_off.numpy().view(np.uint64), whole.offsets), rep
        assert np.array_equal(h_vert.numpy()[:total].view(np.uint32), whole.vertices), rep
        assert np.array_equal(h_stat.numpy(), whole.status), rep
        assert m.total_steps == total - n
    # too small a capacity is an error, not an overrun
    with pytest.raises(abi.InvalidArgument):
        sess.run_host(spec, h_off.data_ptr(), h_vert.data_ptr(), total - 1, h_stat.data_ptr(), chunk=chunk)


@pytest.mark.parametrize("prog,chunk,stride", [(PprProgram(0.2), 1 << 14, 64), (PprProgram(0.1), 5000, 8),
                                               (Node2VecProgram(2.0, 0.5, 16, False), 0, 0)])
def test_run_host_records_equals_run(rmat12, prog, chunk, stride):
    """wf_session_run_host_records: length | status << 31 per query and the
    paths back to back — the same walk set, including walks that outgrow their row."""
    import torch
    dg, hg = rmat12
    src = np.random.default_rng(12).integers(0, hg.vertex_count, 1 << 17).astype(np.uint32)
    spec = QuerySpec.from_list(src)
    opts = ExecOptions(seed=43, path_stride=stride)
    whole = E.run_sequential(dg, spec, prog, opts).walks
    n = src.size
    total = int(whole.offsets[-1])
    sess = E.Session(dg, prog, opts)
    h_rec = torch.zeros(n, dtype=torch.int32).pin_memory()
    h_vert = torch.zeros(total + 64, dtype=torch.int32).pin_memory()
    for rep in range(2):
        m = sess.run_host_records(spec, h_rec.data_ptr(), h_vert.data_ptr(), total + 64, chunk=chunk)
        rec = h_rec.numpy().view(np.uint32)
        assert np.array_equal(rec & 0x7FFFFFFF, np.diff(whole.offsets).astype(np.uint32)), rep
        assert np.array_equal((rec >> 31).astype(np.uint8), whole.status), rep
        assert np.array_equal(h_vert.numpy()[:total].view(np.uint32), whole.vertices), rep
        assert m.total_steps == total - n


def test_degenerate_inputs_match_reference():
    """Edgeless graphs, a single vertex, and empty query sets."""
    from paper_2107_11983_b200.host import Graph
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    ref = RefOracle()
    for V in [1, 4]:
        hg = Graph(np.zeros(V + 1, np.uint64), np.zeros(0, np.uint32))
        dg = E.DeviceGraph.from_host(hg)
        rg = ref.graph(hg)
        for prog in [PprProgram(0.2), DeepWalkProgram(9, False), UniformProgram(5),
                     Node2VecProgram(2.0, 0.5, 7, False)]:
            for spec in [QuerySpec.one_per_vertex(), QuerySpec.from_source(V - 1, 6),
                         QuerySpec.from_source(0, 0)]:
                opts = ExecOptions(seed=2)
                got = E.run_sequential(dg, spec, prog, opts)
                want = rg.run(spec, prog, opts)
                assert got.walks.equals(want.walks), (V, prog, spec.mode)
                assert got.metrics.total_steps == want.metrics.total_steps == 0
                # and through the host-streaming pipeline
                streamed = E.Session(dg, prog, opts).run_to_numpy(spec)
                assert streamed.walks.equals(want.walks), (V, prog, spec.mode)
                assert streamed.metrics.total_steps == 0


@pytest.mark.parametrize("cap", [1, 2, 3, 4, 6, 10, 40])
@pytest.mark.parametrize("sampler", [abi.Sampler.OREJ, abi.Sampler.REJ])
def test_trial_cap_outcome_matches_reference(rmat12, cap, sampler):
    """The walk kernel makes one rejection trial per iteration and counts a
    move's trials across iterations (Walker::trials): for every cap the run
    either raises RejectionCapError exactly when the reference does, or gives
    its walks (sampler.hpp:27, interleave.hpp:286-380)."""
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    dg, hg = rmat12
    spec = QuerySpec.from_list(np.arange(0, hg.vertex_count, 7, dtype=np.uint32))
    if sampler == abi.Sampler.OREJ:
        prog = Node2VecProgram(0.25, 4.0, 12, True)  # acceptance as low as 1/16: caps below ~40 bind
        opts = ExecOptions(seed=5, rej_trial_cap=cap)
    else:
        prog = DeepWalkProgram(12, True)
        opts = ExecOptions(seed=5, sampler=int(sampler), rej_trial_cap=cap)
    rg = RefOracle().graph(hg)
    try:
        want = rg.run(spec, prog, opts)
    except abi.RejectionCapError:
        want = None
    if want is None:
        with pytest.raises(abi.RejectionCapError):
            E.run_sequential(dg, spec, prog, opts)
    else:
        got = E.run_sequential(dg, spec, prog, opts)
        assert got.walks.first_mismatch(want.walks) is None
        assert got.metrics.total_steps == want.metrics.total_steps


def test_randomised_differential_parity_sample():
    """tools/fuzz_parity.py: random graphs (hubs, multi-edges, weight families,
    labels) x programs x samplers x layouts x query specs against the
    unmodified reference — outcome class, every walk, the step total.  A
    sample here; profiles/r02_fuzz_parity.log holds the 33 k-case runs."""
    import subprocess
    import sys
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_parity.py"), "--cases", "250",
                        "--seed", "5"], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "250 cases (seed 5), 0 differing" in p.stdout, p.stdout[-3000:] + p.stderr[-2000:]
