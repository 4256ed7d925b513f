"""Statistical and property checks of the device engine, mirroring the
reference's acceptance gate (proj/tests/acceptance.cpp):

* sampler distributions: L-inf < 0.01 and chi-square p >= 1e-4 over 20 random
  weight vectors for every sampling method, 2^20 draws each (acceptance.cpp:59-145);
* REJ mean trials 3.0 +- 5 % (acceptance.cpp:150-164);
* PPR mean walk length 5.0 in [4.9, 5.1] (acceptance.cpp:317-327);
* Node2Vec on all 38 connected labelled 4-vertex graphs against the
  brute-force second-order transition probabilities (acceptance.cpp:332-427);
* MetaPath label soundness and dead-end truth (acceptance.cpp:432-488).

Bit-exact parity with the reference (test_engine_gpu.py) already implies
these; they are kept because they check the engine against the model, not
against another implementation.
"""
import itertools

import numpy as np
import pytest
from scipy import stats

from paper_2107_11983_b200 import abi
from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, MetaPathProgram,
                                        Node2VecProgram, PprProgram, QuerySpec, UniformProgram,
                                        build_graph)

pytestmark = pytest.mark.gpu

DRAWS = 1 << 20


def _star(weights):
    """Vertex 0 -> leaves 1..d with the given weights; leaves point back to 0."""
    d = len(weights)
    edges = [(0, i + 1) for i in range(d)] + [(i + 1, 0) for i in range(d)]
    w = list(weights) + [1.0] * d
    return build_graph(d + 1, edges, weights=np.asarray(w, np.float32))


def _first_step_counts(g, prog, opts, d):
    res = E.run_sequential(g, QuerySpec.from_source(0, DRAWS), prog, opts)
    ws = res.walks
    assert np.all(np.diff(ws.offsets) == 2)
    dst = ws.vertices.reshape(-1, 2)[:, 1].astype(np.int64)
    return np.bincount(dst - 1, minlength=d)[:d]


METHODS = [
    ("alias_tables", lambda: DeepWalkProgram(2, True), dict(sampler=abi.Sampler.ALIAS)),
    ("its_tables", lambda: DeepWalkProgram(2, True), dict(sampler=abi.Sampler.ITS)),
    ("rej_tables", lambda: DeepWalkProgram(2, True), dict(sampler=abi.Sampler.REJ)),
    ("alias_gathered", lambda: DeepWalkProgram(2, True),
     dict(sampler=abi.Sampler.ALIAS, use_static_tables=False)),
    ("its_gathered", lambda: DeepWalkProgram(2, True),
     dict(sampler=abi.Sampler.ITS, use_static_tables=False)),
    ("rej_gathered", lambda: DeepWalkProgram(2, True),
     dict(sampler=abi.Sampler.REJ, use_static_tables=False)),
    # O-REJ: Node2Vec's first move weighs max(1/a, 1, 1/b) * w_e, i.e. w_e
    ("orej", lambda: Node2VecProgram(1.0, 1.0, 2, True), dict(sampler=abi.Sampler.OREJ)),
    ("naive", lambda: UniformProgram(2), dict(sampler=abi.Sampler.NAIVE)),
]


@pytest.mark.parametrize("name,mk,kw", METHODS, ids=[m[0] for m in METHODS])
def test_sampler_distributions(name, mk, kw):
    rng = np.random.default_rng(2024)
    for trial in range(20):
        d = int(rng.integers(2, 65))
        w = rng.uniform(0.05, 10.0, d).astype(np.float32)
        if trial % 4 == 3:
            w[rng.integers(0, d, max(1, d // 4))] = 0.0  # zero-weight edges are never taken
            if not w.any():
                w[0] = 1.0
        g = _star(w)
        counts = _first_step_counts(g, mk(), ExecOptions(seed=trial + 11, **kw), d)
        p = np.full(d, 1.0 / d) if name == "naive" else w.astype(np.float64) / w.astype(np.float64).sum()
        emp = counts / counts.sum()
        assert np.max(np.abs(emp - p)) < 0.01, (name, trial)
        assert np.all(counts[p == 0] == 0), (name, trial)
        live = p > 0
        chi = stats.chisquare(counts[live], p[live] / p[live].sum() * counts.sum())
        assert chi.pvalue >= 1e-4, (name, trial, chi)


def test_rej_mean_trials():
    """p* d / sum(w) = 3 * 6 / 6 = 3 trials per move on average."""
    g = _star([3.0, 1.0, 1.0, 1.0, 0.0, 0.0])
    sess = E.Session(E.DeviceGraph.from_host(g), DeepWalkProgram(2, True),
                     ExecOptions(seed=5, sampler=abi.Sampler.REJ))
    sess.set_stats(True)
    res = sess.run(QuerySpec.from_source(0, DRAWS))
    trials = sess.stats()["trials"]
    moves = res.metrics.total_steps
    assert moves == DRAWS
    assert abs(trials / moves - 3.0) <= 0.15, trials / moves


def test_ppr_mean_length():
    """On a graph without dead ends a PPR walk takes geometric(0.2) moves: mean 5."""
    n = 32
    edges = [(u, v) for u in range(n) for v in range(n) if u != v]
    g = E.DeviceGraph.from_host(build_graph(n, edges))
    src = np.random.default_rng(3).integers(0, n, DRAWS).astype(np.uint32)
    res = E.run_sequential(g, QuerySpec.from_list(src), PprProgram(0.2), ExecOptions(seed=9))
    moves = np.diff(res.walks.offsets).astype(np.float64) - 1
    assert 4.9 <= moves.mean() <= 5.1, moves.mean()
    assert moves.min() >= 1


def _connected_4_vertex_graphs():
    pairs = list(itertools.combinations(range(4), 2))
    out = []
    for mask in range(1, 1 << 6):
        es = [pairs[i] for i in range(6) if mask >> i & 1]
        adj = {v: set() for v in range(4)}
        for a, b in es:
            adj[a].add(b)
            adj[b].add(a)
        seen, todo = {0}, [0]
        while todo:
            for y in adj[todo.pop()]:
                if y not in seen:
                    seen.add(y)
                    todo.append(y)
        if len(seen) == 4:
            out.append((es, adj))
    return out


@pytest.mark.parametrize("a,b", [(2.0, 0.5), (0.25, 4.0)])
def test_node2vec_all_connected_4_vertex_graphs(a, b):
    graphs = _connected_4_vertex_graphs()
    assert len(graphs) == 38
    n_walks = 1 << 16
    for gi, (es, adj) in enumerate(graphs):
        edges = [(x, y) for x, y in es] + [(y, x) for x, y in es]
        g = E.DeviceGraph.from_host(build_graph(4, edges))
        for s in range(4):
            res = E.run_sequential(g, QuerySpec.from_source(s, n_walks), Node2VecProgram(a, b, 3, False),
                                   ExecOptions(seed=100 * gi + s))
            P = res.walks.vertices.reshape(-1, 3).astype(np.int64)
            # first move: uniform over the neighbours of s
            c1 = np.bincount(P[:, 1], minlength=4)
            nb = sorted(adj[s])
            if len(nb) > 1:
                chi = stats.chisquare(c1[nb])
                assert chi.pvalue >= 1e-4, (gi, s, "first", chi)
            # second move given (prev, cur): Eq. 1 weights 1/a, 1, 1/b
            for cur in nb:
                sel = P[P[:, 1] == cur, 2]
                nxt = sorted(adj[cur])
                w = np.array([1.0 / a if x == s else (1.0 if x in adj[s] else 1.0 / b) for x in nxt])
                cnt = np.bincount(sel, minlength=4)[nxt]
                if len(nxt) < 2:  # a single neighbour: every walk must take it
                    assert cnt.sum() == sel.size
                    continue
                if cnt.sum() < 1000:
                    continue
                chi = stats.chisquare(cnt, w / w.sum() * cnt.sum())
                assert chi.pvalue >= 1e-4, (gi, s, cur, chi)


def test_metapath_label_soundness_and_dead_ends():
    dg = E.DeviceGraph.rmat(12, 16, seed=5, weighted=True, label_count=5)
    hg = dg.download()
    schema = [(3 * i + 1) % 5 for i in range(25)]
    res = E.run_sequential(dg, QuerySpec.one_per_vertex(), MetaPathProgram(schema), ExecOptions(seed=4))
    off = hg.offsets.astype(np.int64)
    nbr = hg.neighbors
    lab = hg.labels
    ws = res.walks
    n_dead = 0
    for q in range(len(ws)):
        p = ws.path(q).astype(np.int64)
        for i in range(len(p) - 1):
            u, v = p[i], p[i + 1]
            lst = nbr[off[u]:off[u + 1]]
            j = np.searchsorted(lst, v)
            assert j < lst.size and lst[j] == v
            assert lab[off[u] + j] == schema[i], (q, i)
        moves = len(p) - 1
        if ws.status[q] == abi.WalkStatus.COMPLETE:
            assert moves == len(schema)
        else:
            n_dead += 1
            u = p[-1]
            assert moves < len(schema)
            assert not np.any(lab[off[u]:off[u + 1]] == schema[moves]), q
    assert n_dead > 0
