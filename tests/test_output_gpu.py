"""Walk-record encoding (SURVEY §8 f row 1): device-encoded text and binary
records are byte-identical to the reference's append_text_record /
append_binary_record (proj/src/output.cpp:26-47), and files written by
wf_walkset_write equal the reference's DoubleBufferedWriter files."""
import os
import tempfile

import numpy as np
import pytest

from oracle.oracle import RefOracle, ref_available
from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, MetaPathProgram,
                                        Node2VecProgram, PprProgram, QuerySpec)
from tests import golden_util as gu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def graphs():
    pl = gu.graph("powerlaw")
    return pl, E.DeviceGraph.from_host(pl), RefOracle().graph(pl)


CASES = [
    (PprProgram(0.2), QuerySpec.from_source(7, 5000)),
    (DeepWalkProgram(30, True), QuerySpec.one_per_vertex()),
    (Node2VecProgram(2.0, 0.5, 25, False), QuerySpec.one_per_vertex()),
    (MetaPathProgram([0, 1, 2, 3, 4, 0]), QuerySpec.one_per_vertex()),  # dead ends
]


@pytest.mark.parametrize("i", range(len(CASES)))
@pytest.mark.parametrize("fmt", [0, 1])
def test_encoded_records_are_reference_bytes(graphs, i, fmt):
    hg, dg, rg = graphs
    prog, spec = CASES[i]
    opts = ExecOptions(seed=5)
    want = rg.run_encoded(spec, prog, opts, fmt)
    got_ws = E.run_sequential(dg, spec, prog, opts).walks
    assert E.encode_walks(got_ws, fmt) == want


@pytest.mark.parametrize("fmt", [0, 1])
def test_walkset_file_equals_reference_writer_file(graphs, fmt):
    hg, dg, rg = graphs
    prog, spec = PprProgram(0.15), QuerySpec.from_list(
        np.random.default_rng(2).integers(0, hg.vertex_count, 30000).astype(np.uint32))
    opts = ExecOptions(seed=9, path_stride=8)  # some walks outgrow their rows
    with tempfile.TemporaryDirectory() as d:
        ref_path = os.path.join(d, "ref.out")
        ours = os.path.join(d, "ours.out")
        rg.run_encoded(spec, prog, opts, fmt, path=ref_path)
        ws = E.Session(dg, prog, opts).run(spec)
        n = ws.write(ours, fmt)
        a = open(ref_path, "rb").read()
        b = open(ours, "rb").read()
        assert n == len(b)
        assert a == b


def test_large_walkset_file_multiple_blocks():
    """> 1 Mi records: several encode/write blocks, still one ordered file."""
    dg = E.DeviceGraph.rmat(21, 4, seed=3)
    ws = E.Session(dg, PprProgram(0.5), ExecOptions(seed=1)).run(QuerySpec.one_per_vertex())
    host = ws.to_host()
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "w.bin")
        n = ws.write(p, 1)
        data = open(p, "rb").read()
    assert n == len(data) == 13 * len(host) + 4 * host.vertices.size
    assert data == E.encode_walks(host, 1)
