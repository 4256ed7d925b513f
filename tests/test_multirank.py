"""World-size-2 gloo test of bench.py's own multi-rank code on CPU: its shard
plan (bench.query_plan -> worker_range, engine.hpp:296-298), its visit-count
reduction (bench.reduce_counts; on GPUs the engine's ncclAllReduce through
wf_comm, here the gloo process group) and its max-over-ranks combination
(bench.combine_ranks).  Each rank walks its shard with the C oracle (a
stand-in for the device engine, which needs a GPU); the shards must reproduce
the single-rank job exactly."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

CFG = dict(bench.CONFIGS["c2"], n_queries=1500)  # PPR, random sources, weak scaling
CFG_V = dict(bench.CONFIGS["c1"], length=12)     # one walk per vertex, strong scaling


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import PortOracle
    from paper_2107_11983_b200.host import DeepWalkProgram, ExecOptions, PprProgram
    from tests import golden_util as gu
    g = gu.graph("powerlaw")
    res = {}
    for name, cfg, prog in [("ppr", CFG, PprProgram(0.2)), ("dw", CFG_V, DeepWalkProgram(12, True))]:
        spec, lo, hi = bench.query_plan(cfg, g.vertex_count, rank, world)
        walks = PortOracle().run(g, spec, prog, ExecOptions(seed=3), qids=np.arange(lo, hi, dtype=np.uint64))
        counts = torch.from_numpy(np.bincount(walks.walks.vertices, minlength=g.vertex_count).astype(np.int64))
        bench.reduce_counts(counts, None, dist)
        t, e, eo, mv = bench.combine_ranks(dist, "cpu", 10.0 + rank, 1.0, 2.0 * rank, walks.metrics.total_steps)
        gathered = [None] * world
        dist.all_gather_object(gathered, (lo, hi, walks.walks.vertices.tolist()))
        res[name] = (counts.numpy().tolist(), gathered, (t, e, eo, mv), spec.count)
    if rank == 0:
        out.put(res)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_bench_shards_reduce_and_combine():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    from oracle.oracle import PortOracle
    from paper_2107_11983_b200.host import DeepWalkProgram, ExecOptions, PprProgram
    from tests import golden_util as gu
    g = gu.graph("powerlaw")
    for name, cfg, prog in [("ppr", CFG, PprProgram(0.2)), ("dw", CFG_V, DeepWalkProgram(12, True))]:
        counts, gathered, (t, e, eo, mv), n = res[name]
        spec, _, _ = bench.query_plan(cfg, g.vertex_count, 0, 2)
        whole = PortOracle().run(g, spec, prog, ExecOptions(seed=3))
        assert np.array_equal(np.asarray(counts), np.bincount(whole.walks.vertices, minlength=g.vertex_count))
        # shards are contiguous, cover the job, and concatenate to the whole walk set
        assert gathered[0][0] == 0 and gathered[0][1] == gathered[1][0] and gathered[1][1] == n
        verts = np.concatenate([np.asarray(x[2], np.uint32) for x in gathered])
        assert np.array_equal(verts, whole.walks.vertices)
        # the line's value: max of the ranks' times, sum of their moves
        assert (t, e, eo) == (11.0, 1.0, 2.0) and mv == whole.metrics.total_steps
    # weak scaling for random sources (a batch per rank), strong for per-vertex
    assert res["ppr"][3] == 2 * CFG["n_queries"] and res["dw"][3] == g.vertex_count


@pytest.mark.parametrize("n,world", [(10, 3), (1 << 26, 8), (5, 8)])
def test_shard_ranges_partition(n, world):
    spans = [bench.worker_range(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert spans == [(n * r // world, n * (r + 1) // world) for r in range(world)]
