"""Custom device programs (the WalkProgram concept, program.hpp:49-93) against
the unmodified reference running the same programs.

The programs are the reference's own test programs (CountingProgram,
AvoidVertexProgram, NegativeWeightProgram: proj/tests/test_engine.cpp:17-47)
plus a weighted meta-path and an unbounded stop-coin program
that reads the traversed edge in update().  The device side is user code
compiled against include/walkforge_b200/device_program.cuh
(tests/programs/test_programs.cu -> libwf_test_programs.so); the reference
side is the same programs written against the reference API
(oracle/ref_harness.cpp wfref_run_test_program).  Walks must be bit-identical.
"""
import ctypes as C
import os

import numpy as np
import pytest

from oracle.oracle import RefOracle, ref_available
from paper_2107_11983_b200 import abi
from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import DeviceProgram, ExecOptions, Graph, QuerySpec

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROGRAMS = os.path.join(ROOT, "tests", "programs", "libwf_test_programs.so")


class TestParams(C.Structure):  # ref_harness.cpp TestProgramParams
    __test__ = False
    _fields_ = [("length", C.c_uint32), ("banned", C.c_uint32), ("stop", C.c_double),
                ("stop_label", C.c_uint32), ("schema_len", C.c_uint32), ("schema", C.c_uint32 * 48)]


class CountingC(C.Structure):
    _fields_ = [("length", C.c_uint32), ("updates", C.c_void_p)]


class AvoidVertexC(C.Structure):
    _fields_ = [("banned", C.c_uint32), ("length", C.c_uint32)]


class NegativeWeightC(C.Structure):
    _fields_ = [("unused", C.c_uint32)]


class LabelWeightC(C.Structure):
    _fields_ = [("schema_len", C.c_uint32), ("schema", C.c_uint32 * 48)]


class LabelStopC(C.Structure):
    _fields_ = [("stop", C.c_double), ("stop_label", C.c_uint32)]


@pytest.fixture(scope="module")
def graphs():
    ref = RefOracle()
    # the reference's own power-law fixture (synthetic.cpp:46-66): weighted,
    # labelled, hubs, multi-edges and self-loops
    rg = ref.power_law(2000, 20000, seed=42, weighted=True, label_count=5)
    off, nbr, w, lab = rg.export()
    hg = Graph(off, nbr, w.astype(np.float32), lab.astype(np.uint8))
    rg32 = ref.graph(hg)  # the reference over the f32-rounded weights the device holds
    dg = E.DeviceGraph.from_host(hg)
    return rg32, dg, hg


def program(symbol, obj):
    return DeviceProgram((PROGRAMS, symbol), obj)


def assert_same(got, want):
    bad = got.walks.first_mismatch(want.walks)
    assert bad is None, f"walk {bad} differs"
    assert got.metrics.total_steps == want.metrics.total_steps


def test_counting_program_updates_once_per_move(graphs):
    rg, dg, hg = graphs
    import torch
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    prog = program("wf_test_counting_program", CountingC(10, ctr.data_ptr()))
    opts = ExecOptions(seed=7)
    got = E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts)
    want, updates = rg.run_test_program(0, TestParams(length=10), QuerySpec.one_per_vertex(), opts)
    assert_same(got, want)
    assert int(ctr.item()) == got.metrics.total_steps == updates


@pytest.mark.parametrize("sampler,tables", [(-1, True), (abi.Sampler.ALIAS, True), (abi.Sampler.ITS, True),
                                            (abi.Sampler.REJ, True), (abi.Sampler.OREJ, True),
                                            (abi.Sampler.ALIAS, False), (abi.Sampler.ITS, False),
                                            (abi.Sampler.REJ, False)])
def test_avoid_vertex_program_every_flow(graphs, sampler, tables):
    rg, dg, hg = graphs
    banned = int(np.argmax(np.diff(hg.offsets)))  # the biggest hub
    prog = program("wf_test_avoid_vertex_program", AvoidVertexC(banned, 12))
    opts = ExecOptions(seed=3, sampler=None if sampler == -1 else int(sampler), use_static_tables=tables)
    tp = TestParams(length=12, banned=banned)
    if sampler == abi.Sampler.OREJ:
        # O-REJ never accepts at a vertex whose only neighbour is the banned
        # one: both engines hit the trial cap (sampler.hpp:152-164) and raise
        with pytest.raises(abi.RejectionCapError):
            rg.run_test_program(1, tp, QuerySpec.one_per_vertex(), opts)
        with pytest.raises(abi.RejectionCapError):
            E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts)
        # ... and walk identically when no vertex depends on the banned one alone
        deg = np.diff(hg.offsets)
        only = {int(hg.neighbors_of(u)[0]) for u in range(hg.vertex_count)
                if deg[u] and np.all(hg.neighbors_of(u) == hg.neighbors_of(u)[0])}
        banned = int(max((v for v in range(hg.vertex_count) if v not in only), key=lambda v: deg[v]))
        prog = program("wf_test_avoid_vertex_program", AvoidVertexC(banned, 12))
        tp = TestParams(length=12, banned=banned)
    got = E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts)
    want, _ = rg.run_test_program(1, tp, QuerySpec.one_per_vertex(), opts)
    assert_same(got, want)
    ws = got.walks
    for i in range(len(ws)):
        assert banned not in ws.path(i)[1:]
    if sampler == -1:
        s, f, _ = E.Session(dg, prog, opts).describe()
        assert s == abi.Sampler.ALIAS and f == abi.Flow.TABLES  # static default, like the reference


def test_negative_weight_program_raises_contract_error(graphs):
    rg, dg, hg = graphs
    prog = program("wf_test_negative_weight_program", NegativeWeightC(0))
    with pytest.raises(abi.ContractError):
        E.Session(dg, prog, ExecOptions(seed=1))  # preprocess_static checks every weight
    with pytest.raises(abi.ContractError):
        rg.run_test_program(2, TestParams(), QuerySpec.one_per_vertex(), ExecOptions(seed=1))
    # gathered: the first gather of a walk raises (engine.hpp:134-184)
    opts = ExecOptions(seed=1, use_static_tables=False)
    with pytest.raises(abi.ContractError):
        E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts)
    with pytest.raises(abi.ContractError):
        rg.run_test_program(2, TestParams(), QuerySpec.one_per_vertex(), opts)


@pytest.mark.parametrize("sampler", [-1, abi.Sampler.ALIAS, abi.Sampler.REJ])
def test_label_weight_program_dynamic(graphs, sampler):
    rg, dg, hg = graphs
    schema = [i % 5 for i in range(9)]
    arr = (C.c_uint32 * 48)(*schema)
    prog = program("wf_test_label_weight_program", LabelWeightC(len(schema), arr))
    opts = ExecOptions(seed=11, sampler=None if sampler == -1 else int(sampler))
    tp = TestParams(schema_len=len(schema), schema=arr)
    got = E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, opts)
    want, _ = rg.run_test_program(3, tp, QuerySpec.one_per_vertex(), opts)
    assert_same(got, want)


@pytest.mark.parametrize("sampler,stride", [(-1, 0), (abi.Sampler.OREJ, 0), (-1, 4)])
def test_label_stop_program_unbounded(graphs, sampler, stride):
    """Unbounded walks; update() draws and reads the traversed edge's label.
    stride 4 forces walks past their row capacity (the overflow re-run)."""
    rg, dg, hg = graphs
    prog = program("wf_test_label_stop_program", LabelStopC(0.1, 4))
    opts = ExecOptions(seed=5, sampler=None if sampler == -1 else int(sampler), path_stride=stride)
    spec = QuerySpec.from_list(np.random.default_rng(2).integers(0, hg.vertex_count, 5000, dtype=np.uint32))
    got = E.run_sequential(dg, spec, prog, opts)
    want, _ = rg.run_test_program(4, TestParams(stop=0.1, stop_label=4), spec, opts)
    assert_same(got, want)
    # the streaming host path (run_host) gives the same walks
    sess = E.Session(dg, prog, opts)
    res = sess.run_to_numpy(spec)
    bad = res.walks.first_mismatch(want.walks)
    assert bad is None, f"streamed walk {bad} differs"


def test_custom_session_rejects_illegal_pairings(graphs):
    rg, dg, hg = graphs
    schema = (C.c_uint32 * 48)(0, 1)
    dyn = program("wf_test_label_weight_program", LabelWeightC(2, schema))
    with pytest.raises(abi.ConfigError):  # NAIVE needs an unbiased program (engine.hpp:258-262)
        E.Session(dg, dyn, ExecOptions(sampler=int(abi.Sampler.NAIVE)))
    with pytest.raises(abi.ConfigError):  # O-REJ needs max_weight() (engine.hpp:103-114)
        E.Session(dg, dyn, ExecOptions(sampler=int(abi.Sampler.OREJ)))


def test_randomised_custom_program_parity_sample():
    """tools/fuzz_custom.py: the test programs on random graphs x samplers x
    tables x specs against the reference running the same programs (walks, step
    total, update() count).  A sample; profiles/r02_fuzz_custom.log holds 8000."""
    import subprocess
    import sys
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_custom.py"), "--cases", "200",
                        "--seed", "7"], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "200 cases (seed 7), 0 differing" in p.stdout, p.stdout[-3000:] + p.stderr[-2000:]
