"""World-size-2 gloo test of the multi-GPU data flow on CPU: contiguous qid
shards (worker_range) walked independently and the PPR visit counts summed by
all-reduce reproduce the single-rank job exactly.  The per-rank walker here is
the C oracle (a stand-in for the device engine, which needs a GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2107_11983_b200.shard import reduce_visit_counts, shard_queries


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
    from paper_2107_11983_b200.host import ExecOptions, PprProgram, QuerySpec
    from tests import golden_util as gu
    g = gu.graph("powerlaw")
    src = np.random.default_rng(4).integers(0, g.vertex_count, 3001).astype(np.uint32)
    spec = QuerySpec.from_list(src)
    lo, hi = shard_queries(src.size, world, rank)
    res = PortOracle().run(g, spec, PprProgram(0.2), ExecOptions(seed=3),
                           qids=np.arange(lo, hi, dtype=np.uint64))
    counts = torch.from_numpy(np.bincount(res.walks.vertices, minlength=g.vertex_count)
                              .astype(np.int64))
    reduce_visit_counts(counts, dist)
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, res.walks.offsets.tolist(),
                                      res.walks.vertices.tolist()))
    if rank == 0:
        out.put((counts.numpy().tolist(), gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_and_count_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, gathered = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    from oracle.oracle import PortOracle
    from paper_2107_11983_b200.host import ExecOptions, PprProgram, QuerySpec
    from tests import golden_util as gu
    g = gu.graph("powerlaw")
    src = np.random.default_rng(4).integers(0, g.vertex_count, 3001).astype(np.uint32)
    whole = PortOracle().run(g, QuerySpec.from_list(src), PprProgram(0.2), ExecOptions(seed=3))
    want = np.bincount(whole.walks.vertices, minlength=g.vertex_count)
    assert np.array_equal(np.asarray(counts), want)
    # shards are contiguous, cover the job, and concatenate to the whole walk set
    assert gathered[0][0] == 0 and gathered[0][1] == gathered[1][0] and gathered[1][1] == 3001
    verts = np.concatenate([np.asarray(g_[3], np.uint32) for g_ in gathered])
    assert np.array_equal(verts, whole.walks.vertices)


@pytest.mark.parametrize("n,world", [(10, 3), (1 << 26, 8), (5, 8)])
def test_shard_ranges_partition(n, world):
    spans = [shard_queries(n, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
