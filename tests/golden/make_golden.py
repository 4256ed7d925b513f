"""Generates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the container that mounts /root/reference (after `make -C oracle ref`):

    python tests/golden/make_golden.py

Everything is produced by calling the reference's own code through
oracle/_ref/libwfref.so (RngStream, alias_init, make_power_law_graph,
make_ring_graph, build_graph, run_sequential, preprocess_static).  The fixture
graphs' weights are rounded to float32 and the graph is rebuilt through
Graph::from_csr, so the stored graph is exactly what the device engine holds
(the reference then widens the f32 values back to f64 exactly).

Outputs: graphs.npz, walks.npz, tables.npz, rng.npz, cases.json.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefOracle  # noqa: E402
from paper_2107_11983_b200.abi import Sampler, WalkforgeError  # noqa: E402
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, Graph,  # noqa: E402
                                        MetaPathProgram, Node2VecProgram, PprProgram, QuerySpec,
                                        UniformProgram)

ref = RefOracle()


def f32_graph(rg):
    """Round the reference graph's weights to f32 and rebuild via from_csr."""
    off, nbr, w, lab = rg.export()
    w32 = None if w is None else w.astype(np.float32)
    g = Graph(off, nbr, w32, None if lab is None else lab.astype(np.uint8))
    return g


def program_from(d):
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


def spec_from(d):
    s = d.get("spec", {"mode": "one_per_vertex"})
    if s["mode"] == "one_per_vertex":
        return QuerySpec.one_per_vertex()
    if s["mode"] == "from_source":
        return QuerySpec.from_source(s["source"], s["count"])
    return QuerySpec.from_list(np.asarray(s["sources"], dtype=np.uint32))


def opts_from(d):
    smp = d.get("sampler")
    return ExecOptions(seed=d.get("seed", 1), sampler=None if smp is None else Sampler.parse(smp),
                       use_static_tables=d.get("tables", True))


def main():
    graphs = {}

    # -- graphs ------------------------------------------------------------------
    graphs["powerlaw"] = f32_graph(ref.power_law(1000, 10000, seed=42, weighted=True,
                                                 label_count=5))
    graphs["ring"] = f32_graph(ref.ring(64, seed=3, weighted=True, label_count=5))
    graphs["triangle"] = f32_graph(ref.build(3, [(0, 1), (1, 2), (2, 0)]))
    graphs["line4"] = f32_graph(ref.build(4, [(0, 1), (1, 2), (2, 3)]))
    graphs["clique4"] = f32_graph(ref.build(4, [(i, j) for i in range(4) for j in range(4)
                                                if i != j]))
    graphs["star5"] = f32_graph(ref.build(6, [p for i in range(1, 6) for p in ((0, i), (i, 0))]))
    graphs["fan"] = f32_graph(ref.build(3, [(0, 1), (0, 2)], weights=[1.0, 3.0]))
    graphs["labelled4"] = f32_graph(ref.build(4, [(0, 1), (0, 2), (1, 2), (2, 3), (3, 0)],
                                              labels=[0, 1, 1, 2, 0]))
    graphs["deadend3"] = f32_graph(ref.build(3, [(0, 1), (1, 2)]))
    # zero-weight edges: vertex 1's only out-edge has weight 0 (exhausted for
    # static tables), vertex 0 mixes zero and positive weights.
    graphs["zeroweights"] = f32_graph(ref.build(
        4, [(0, 1), (0, 2), (0, 3), (1, 0), (2, 0), (2, 3), (3, 0)],
        weights=[0.0, 2.0, 1.0, 0.0, 1.5, 0.0, 4.0]))
    # unsorted adjacency (from_csr keeps it): has_edge falls back to a scan.
    pl = graphs["powerlaw"]
    rng = np.random.default_rng(5)
    nbr = pl.neighbors.copy()
    w = pl.weights.copy()
    lab = pl.labels.copy()
    for v in range(pl.vertex_count):
        a, b = int(pl.offsets[v]), int(pl.offsets[v + 1])
        perm = rng.permutation(b - a) + a
        nbr[a:b], w[a:b], lab[a:b] = nbr[perm], w[perm], lab[perm]
    graphs["powerlaw_unsorted"] = Graph(pl.offsets, nbr, w, lab)

    # -- runs --------------------------------------------------------------------
    cases = []

    def add(name, graph, **d):
        d.update(name=name, graph=graph)
        cases.append(d)

    samplers_all = ["naive", "its", "alias", "rej", "orej"]
    for s in samplers_all:
        add(f"pl_ppr_{s}", "powerlaw", program="ppr", termination=0.2, sampler=s, seed=7)
    for s in ["its", "alias", "rej", "orej"]:
        add(f"pl_deepwalk_w_{s}", "powerlaw", program="deepwalk", length=20, weighted=True,
            sampler=s, seed=7)
    for s in ["its", "alias", "rej"]:
        add(f"pl_deepwalk_w_{s}_gathered", "powerlaw", program="deepwalk", length=20,
            weighted=True, sampler=s, seed=7, tables=False)
    add("pl_deepwalk_w80_alias", "powerlaw", program="deepwalk", length=80, weighted=True,
        sampler="alias", seed=1)
    add("pl_deepwalk_u_default", "powerlaw", program="deepwalk", length=20, weighted=False,
        seed=3)
    for s in ["its", "alias", "rej", "orej"]:
        add(f"pl_node2vec_w_{s}", "powerlaw", program="node2vec", a=2.0, b=0.5, length=20,
            weighted=True, sampler=s, seed=7)
    add("pl_node2vec_u_orej", "powerlaw", program="node2vec", a=2.0, b=0.5, length=20,
        weighted=False, seed=1)
    add("pl_node2vec_u_orej_q", "powerlaw", program="node2vec", a=0.25, b=4.0, length=20,
        weighted=False, seed=2)
    add("pl_node2vec_unsorted", "powerlaw_unsorted", program="node2vec", a=2.0, b=0.5,
        length=20, weighted=False, seed=1)
    for s in ["its", "alias", "rej"]:
        add(f"pl_metapath_{s}", "powerlaw", program="metapath", schema=[0, 1, 2, 3], sampler=s,
            seed=7)
    add("pl_metapath_long", "powerlaw", program="metapath", schema=[i % 5 for i in range(19)],
        seed=1)
    add("pl_uniform_naive", "powerlaw", program="uniform", length=20, seed=11)
    add("pl_uniform_alias", "powerlaw", program="uniform", length=20, sampler="alias", seed=11)
    add("ring_deepwalk_w", "ring", program="deepwalk", length=6, weighted=True, seed=1)
    add("ring_ppr_from0", "ring", program="ppr", termination=0.2, seed=1,
        spec={"mode": "from_source", "source": 0, "count": 200})
    add("ring_ppr_stop1", "ring", program="ppr", termination=1.0, seed=2,
        spec={"mode": "from_source", "source": 5, "count": 50})
    add("ring_metapath", "ring", program="metapath", schema=[0, 1, 2, 3, 4, 0, 1], seed=4)
    add("pl_ppr_list", "powerlaw", program="ppr", termination=0.15, seed=9,
        spec={"mode": "from_list", "sources": [int(x) for x in
                                               np.random.default_rng(1).integers(0, 1000, 500)]})
    add("triangle_len12", "triangle", program="deepwalk", length=12, seed=0)
    add("triangle_len1", "triangle", program="deepwalk", length=1, seed=0)
    add("line_deadend", "line4", program="deepwalk", length=10, seed=0,
        spec={"mode": "from_source", "source": 0, "count": 1})
    add("labelled_exact", "labelled4", program="metapath", schema=[0, 1, 2], seed=0,
        spec={"mode": "from_source", "source": 0, "count": 50})
    add("labelled_deadend", "labelled4", program="metapath", schema=[0, 1, 2], seed=0,
        spec={"mode": "from_source", "source": 1, "count": 50})
    add("star_node2vec", "star5", program="node2vec", a=2.0, b=0.5, length=9, seed=5)
    add("clique_node2vec_its", "clique4", program="node2vec", a=2.0, b=0.5, length=9,
        sampler="its", seed=5)
    add("fan_deepwalk_alias", "fan", program="deepwalk", length=2, weighted=True,
        sampler="alias", seed=21, spec={"mode": "from_source", "source": 0, "count": 2000})
    add("fan_deepwalk_its", "fan", program="deepwalk", length=2, weighted=True,
        sampler="its", seed=21, spec={"mode": "from_source", "source": 0, "count": 2000})
    add("fan_deepwalk_rej", "fan", program="deepwalk", length=2, weighted=True,
        sampler="rej", seed=21, spec={"mode": "from_source", "source": 0, "count": 2000})
    for s in ["its", "alias", "rej"]:
        add(f"zero_deepwalk_w_{s}", "zeroweights", program="deepwalk", length=8, weighted=True,
            sampler=s, seed=3)
        add(f"zero_deepwalk_w_{s}_gathered", "zeroweights", program="deepwalk", length=8,
            weighted=True, sampler=s, seed=3, tables=False)
    # illegal pairings refused up front (engine.hpp:255-272, 103-114)
    add("err_naive_static", "triangle", program="deepwalk", length=5, sampler="naive",
        error="ConfigError")
    add("err_orej_metapath", "labelled4", program="metapath", schema=[0, 0, 1], sampler="orej",
        error="ConfigError")
    add("err_bad_source", "triangle", program="ppr", termination=0.2,
        spec={"mode": "from_source", "source": 9, "count": 5}, error="ConfigError")
    add("err_metapath_label", "labelled4", program="metapath", schema=[0, 7], error="ConfigError")
    add("err_ppr_term", "triangle", program="ppr", termination=1.5, error="ConfigError")
    add("err_weighted_unweighted", "triangle", program="deepwalk", length=5, weighted=True,
        error="ConfigError")

    walks = {}
    ref_graphs = {name: ref.graph(g) for name, g in graphs.items()}
    for c in cases:
        rg = ref_graphs[c["graph"]]
        try:
            res = rg.run(spec_from(c), program_from(c), opts_from(c))
        except WalkforgeError as e:
            if c.get("error") != type(e).__name__:
                raise
            c["message"] = str(e)
            continue
        assert "error" not in c, c
        walks[c["name"] + "/offsets"] = res.walks.offsets
        walks[c["name"] + "/vertices"] = res.walks.vertices
        walks[c["name"] + "/status"] = res.walks.status
        c["total_steps"] = int(res.metrics.total_steps)

    # -- static tables (preprocess_static) --------------------------------------
    tables = {}
    for gname in ["powerlaw", "zeroweights", "ring"]:
        for s in [Sampler.ALIAS, Sampler.ITS, Sampler.REJ]:
            t = ref_graphs[gname].static_tables(DeepWalkProgram(20, True), int(s))
            key = f"{gname}/{s.name.lower()}"
            if s == Sampler.ALIAS:
                for k in ["alias_split", "alias_first", "alias_second", "alias_first_dst",
                          "alias_second_dst", "exhausted"]:
                    tables[f"{key}/{k}"] = t[k]
            elif s == Sampler.ITS:
                tables[f"{key}/its"] = t["its"]
                tables[f"{key}/exhausted"] = t["exhausted"]
            else:
                tables[f"{key}/rej_p_star"] = t["rej_p_star"]
                tables[f"{key}/exhausted"] = t["exhausted"]

    # -- RNG + alias_init --------------------------------------------------------
    rng_out = {}
    pairs = [(0, 0), (1, 0), (1, 1), (1, 65535), (42, 7), (2 ** 63 + 5, 2 ** 40 + 3),
             (0xFFFFFFFFFFFFFFFF, 0xFFFFFFFFFFFFFFFF)]
    rng_out["pairs"] = np.array(pairs, dtype=np.uint64)
    rng_out["draws"] = np.stack([ref.rng_probe(s, q, 16) for s, q in pairs])
    ir = [(s, q, n, b) for (s, q) in pairs for (n, b) in [(1, 1.0), (7, 0.001), (1000, 123.5),
                                                          (2 ** 32 - 1, 2.0), (3, 5.0)]]
    rng_out["ir_args_u"] = np.array([(s, q) for s, q, _, _ in ir], dtype=np.uint64)
    rng_out["ir_args_n"] = np.array([n for _, _, n, _ in ir], dtype=np.uint32)
    rng_out["ir_args_b"] = np.array([b for _, _, _, b in ir], dtype=np.float64)
    res = [ref.rng_index_real(s, q, n, b) for s, q, n, b in ir]
    rng_out["ir_idx"] = np.array([r[0] for r in res], dtype=np.uint32)
    rng_out["ir_real"] = np.array([r[1] for r in res], dtype=np.float64)
    g = np.random.default_rng(20260822)
    dists = []
    for i in range(40):
        n = int(g.integers(1, 200))
        w = (0.5 + 9.5 * g.random(n)).astype(np.float32).astype(np.float64)
        if i % 4 == 3:
            w[g.integers(0, n)] = 0.0
        if i % 7 == 0:
            w[:] = 1.0
        dists.append(w)
    flat = np.concatenate(dists)
    offs = np.cumsum([0] + [len(d) for d in dists]).astype(np.uint64)
    rng_out["alias_weights"] = flat
    rng_out["alias_offsets"] = offs
    sp, fi, se = [], [], []
    for d in dists:
        a, b, c = ref.alias_init(d)
        sp.append(a), fi.append(b), se.append(c)
    rng_out["alias_split"] = np.concatenate(sp)
    rng_out["alias_first"] = np.concatenate(fi)
    rng_out["alias_second"] = np.concatenate(se)
    rng_out["synthetic_weight"] = np.array([ref.synthetic_weight(1, e) for e in range(64)])
    rng_out["synthetic_label"] = np.array([ref.synthetic_label(1, e, 5) for e in range(64)],
                                          dtype=np.uint32)

    gz = {}
    for name, gr in graphs.items():
        gz[f"{name}/offsets"] = gr.offsets
        gz[f"{name}/neighbors"] = gr.neighbors
        if gr.weights is not None:
            gz[f"{name}/weights"] = gr.weights
        if gr.labels is not None:
            gz[f"{name}/labels"] = gr.labels
    np.savez_compressed(os.path.join(HERE, "graphs.npz"), **gz)
    np.savez_compressed(os.path.join(HERE, "walks.npz"), **walks)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **tables)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **rng_out)
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(cases, f, indent=1)
    print(f"{len(cases)} cases, {len(graphs)} graphs")


if __name__ == "__main__":
    main()
