"""Multi-device execution in the library (wf_multi_*, wf_comm_*) on the one GPU
a test box has.

* Workers over devices: `workers` contiguous qid blocks (worker_range,
  engine.hpp:296-298), delivered once each in worker order (BlockSink,
  engine.hpp:76-79), must concatenate to the single-device walk set — which the
  golden tests pin to the reference.  Device lists [0] (a one-rank NCCL
  communicator for the visit counts) and [0, 0] (two replicas sharing the GPU:
  no NCCL, counts summed on the device) exercise both reduction paths.
* bench.py's per-rank path: its shard plan run as two ranks' launches on one
  device equals the whole run.
* wf_comm: the library's own NCCL all-reduce (one rank).
"""
import os
import sys

import numpy as np
import pytest

from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, MetaPathProgram, Node2VecProgram,
                                        PprProgram, QuerySpec)

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dg():
    return E.DeviceGraph.rmat(14, 16, seed=1, weighted=True, label_count=5)


def single(dg, spec, prog, opts):
    return E.run_sequential(dg, spec, prog, opts)


@pytest.mark.parametrize("devices,workers", [([0], 0), ([0], 4), ([0, 0], 0), ([0, 0], 5)])
@pytest.mark.parametrize("prog", [PprProgram(0.2), DeepWalkProgram(20, True), Node2VecProgram(2.0, 0.5, 15, False),
                                  MetaPathProgram([i % 5 for i in range(9)])], ids=["ppr", "deepwalk", "node2vec",
                                                                                     "metapath"])
def test_workers_over_devices_equal_single_device(dg, devices, workers, prog):
    V = dg.vertex_count
    spec = (QuerySpec.from_list(np.random.default_rng(5).integers(0, V, 7001, dtype=np.uint32))
            if isinstance(prog, PprProgram) else QuerySpec.one_per_vertex())
    opts = ExecOptions(seed=9)
    want = single(dg, spec, prog, opts)
    m = E.MultiDevice(dg, devices, prog, opts)
    info = m.info()
    assert info["devices"] == len(devices)
    # NCCL only for PPR (its visit counts are the one collective) on distinct devices
    assert info["nccl"] == (isinstance(prog, PprProgram) and len(set(devices)) == len(devices))
    got, counts, order = m.run(spec, workers=workers, counts=isinstance(prog, PprProgram))
    assert got.walks.first_mismatch(want.walks) is None
    assert got.metrics.total_steps == want.metrics.total_steps
    W = workers or len(devices)
    n = spec.count if spec.count else V
    assert [w for w, _, _ in order] == list(range(W))
    assert [(a, b) for _, a, b in order] == [E.worker_range(n, W, w) for w in range(W)]
    if isinstance(prog, PprProgram):
        assert np.array_equal(counts, np.bincount(want.walks.vertices, minlength=V).astype(np.uint32))


def test_multi_sink_error_stops_the_run(dg):
    m = E.MultiDevice(dg, [0, 0], DeepWalkProgram(10, True), ExecOptions(seed=1))

    def boom(w, q0, q1, ws):
        if w == 1:
            raise RuntimeError("sink full")

    with pytest.raises(RuntimeError, match="sink full"):
        m.run(QuerySpec.one_per_vertex(), workers=3, on_block=boom)


def test_bench_rank_shards_on_one_device(dg):
    """bench.py's shard plan (query_plan -> worker_range) run as two ranks'
    launches on one GPU reproduces the whole run, and the summed per-rank
    visit counts equal the whole run's."""
    import torch
    sys.path.insert(0, ROOT)
    import bench
    cfg = dict(bench.CONFIGS["c2"], n_queries=6000)
    prog = PprProgram(0.2)
    V = dg.vertex_count
    sess = E.Session(dg, prog, ExecOptions(seed=1, path_stride=64))
    spec, _, _ = bench.query_plan(cfg, V, 0, 2)
    want = sess.run(spec).to_host()
    counts = torch.zeros(V, dtype=torch.int32, device="cuda")
    d_src = torch.from_numpy(spec.sources.view(np.int32)).cuda()
    verts = []
    for rank in range(2):
        _, lo, hi = bench.query_plan(cfg, V, rank, 2)
        n = hi - lo
        paths = torch.empty(n * 64, dtype=torch.int32, device="cuda")
        lens = torch.empty(n, dtype=torch.int32, device="cuda")
        st = torch.empty(n, dtype=torch.uint8, device="cuda")
        sess.launch(spec, lo, hi, paths.data_ptr(), 64, lens.data_ptr(), st.data_ptr(), counts.data_ptr(),
                    sources_dev_ptr=d_src.data_ptr())
        sess.sync()
        L = lens.cpu().numpy()
        P = paths.cpu().numpy().reshape(n, 64)
        assert L.max() <= 64
        verts += [P[i, :L[i]] for i in range(n)]
    got = np.concatenate(verts).astype(np.uint32)
    assert np.array_equal(got, want.vertices)
    assert np.array_equal(counts.cpu().numpy(), np.bincount(want.vertices, minlength=V).astype(np.int32))


def test_comm_allreduce_one_rank():
    """The library's own NCCL communicator (what bench.py's torchrun path uses
    for the PPR counts): one rank sums to itself."""
    import torch
    assert E.nccl_version() >= 21800
    comm = E.Comm(E.Comm.unique_id(), 1, 0, 0)
    x = torch.arange(1000, dtype=torch.int32, device="cuda")
    comm.allreduce_u32(x.data_ptr(), x.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(x.cpu(), torch.arange(1000, dtype=torch.int32))


def test_more_workers_than_queries_delivers_empty_blocks(dg):
    """worker_range gives some workers nothing when workers > queries (and all of
    them nothing for an empty query set): every worker still gets its block, in
    order, and the walks are the single-device run's (found by tools/fuzz_parity.py:
    the Python block collector indexed into an empty offsets array)."""
    prog, opts = DeepWalkProgram(12, True), ExecOptions(seed=9)
    for spec, workers in [(QuerySpec.from_source(3, 2), 7), (QuerySpec.from_source(3, 0), 3),
                          (QuerySpec.from_list(np.asarray([5, 1, 4], np.uint32)), 5)]:
        m = E.MultiDevice(dg, [0, 0], prog, opts)
        got, _, order = m.run(spec, workers=workers)
        assert [w for w, _, _ in order] == list(range(workers))
        want = E.run_sequential(dg, spec, prog, opts)
        assert got.walks.first_mismatch(want.walks) is None and len(got.walks) == len(want.walks)
