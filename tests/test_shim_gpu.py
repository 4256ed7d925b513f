"""The header-only C++ shim compiled as a reference caller would use it
(include/walkforge_b200/engine.hpp, WALKFORGE_B200_DROP_IN) reproduces the
reference's golden walk sets."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2107_11983_b200 import engine as E
from tests import golden_util as gu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def fnv(ws):
    h = 1469598103934665603
    mask = (1 << 64) - 1

    def mix(x):
        nonlocal h
        for i in range(8):
            h ^= (x >> (8 * i)) & 0xFF
            h = (h * 1099511628211) & mask
    for q in range(len(ws)):
        p = ws.path(q)
        mix(q)
        mix(int(ws.status[q]))
        mix(len(p))
        for v in p:
            mix(int(v))
    return h


PROGRAMS = os.path.join(ROOT, "tests", "programs")


def build_shim(tmp):
    """A reference caller's build: plain g++ against the C header and the
    shim, linked with the engine and with a separately compiled user
    device-program library (tests/programs)."""
    exe = os.path.join(tmp, "shim_test")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", "shim_test.cpp"), "-o", exe,
                           "-L", os.path.dirname(E.LIB_PATH), "-lwalkforge_b200",
                           f"-Wl,-rpath,{os.path.dirname(E.LIB_PATH)}",
                           "-L", PROGRAMS, "-l:libwf_test_programs.so", f"-Wl,-rpath,{PROGRAMS}"])
    return exe


def test_shim_compiles_cpu_only():
    """The shim is plain C++20 against the C header (no CUDA types leak)."""
    with tempfile.TemporaryDirectory() as d:
        assert os.path.exists(build_shim(d))


@pytest.mark.gpu
def test_shim_reproduces_golden_walks():
    g = gu.graph("powerlaw")
    with tempfile.TemporaryDirectory() as d:
        exe = build_shim(d)
        path = os.path.join(d, "g.bin")
        with open(path, "wb") as f:
            f.write(np.uint32(g.vertex_count).tobytes())
            f.write(np.uint64(g.edge_count).tobytes())
            f.write(g.offsets.tobytes())
            f.write(g.neighbors.tobytes())
            f.write(g.weights.tobytes())
            f.write(g.labels.astype(np.uint32).tobytes())
        out = subprocess.check_output([exe, path], text=True).splitlines()
        res = {l.split()[0]: l.split()[1:] for l in out}
        # output.hpp's writer + ordered sink: the reference's record bytes
        # (wf_encode_walks is pinned byte-identical to output.cpp elsewhere)
        dw = gu.walks({c["name"]: c for c in gu.cases()}["pl_deepwalk_w_alias"])
        for key, fmt in [("written_txt", 0), ("written_bin", 1), ("written_txt_workers", 0)]:
            with open(res[key][0], "rb") as f:
                assert f.read() == E.encode_walks(dw, fmt), key
        assert res["written_txt_workers"][1] == "each_once"
        assert res["empty_workers"] == ["1", "1", "1"]
    cases = {c["name"]: c for c in gu.cases()}
    for key, case in [("deepwalk_alias", "pl_deepwalk_w_alias"),
                      ("node2vec_orej", "pl_node2vec_w_orej"),
                      ("metapath_its", "pl_metapath_its")]:
        ws = gu.walks(cases[case])
        assert res[key][0] == f"{fnv(ws):016x}", key
        assert int(res[key][1]) == cases[case]["total_steps"]
    assert res["metapath_its"][2] == "sink_empty=1"
    assert res["naive_static"] == ["ConfigError"]
    assert res["graph_accessors"] == ["ok"]
    assert res["tune"] == ["64", "32", "1"]
    assert res["writer_open"] == ["IoError"]
    assert res["query_file"] == ["3", "3", "3", "7"]  # walker.cpp:22-78 on test_cli.cpp:188's file
    assert res["query_file_error"] == ["ParseError", ":1:", "too", "many", "columns"]
    # unbounded walks, worker blocks and user device programs against the
    # unmodified reference on the same graph
    import ctypes as C
    from oracle.oracle import RefOracle, ref_available
    from paper_2107_11983_b200.host import ExecOptions, PprProgram, QuerySpec
    if not ref_available():
        return
    from tests.test_custom_programs_gpu import TestParams
    rg = RefOracle().graph(g)
    want = rg.run(QuerySpec.from_source(0, 3), PprProgram(1e-4), ExecOptions(seed=3))
    assert res["ppr_long"] == [f"{fnv(want.walks):016x}", str(want.metrics.total_steps), "3"]
    src = np.array([(i * 37) % g.vertex_count for i in range(200)], np.uint32)
    want = rg.run(QuerySpec.from_list(src), PprProgram(0.2), ExecOptions(seed=3, threads=3))
    assert res["ppr_workers"] == [f"{fnv(want.walks):016x}", str(want.metrics.total_steps), "order=012", "n=3"]
    want, _ = rg.run_test_program(1, TestParams(length=12, banned=0), QuerySpec.one_per_vertex(), ExecOptions(seed=3))
    assert res["custom_avoid"] == [f"{fnv(want.walks):016x}", str(want.metrics.total_steps)]
    want, _ = rg.run_test_program(4, TestParams(stop=0.1, stop_label=4), QuerySpec.one_per_vertex(),
                                  ExecOptions(seed=5), interleaved=True)
    assert res["custom_stop"] == [f"{fnv(want.walks):016x}", str(want.metrics.total_steps)]
