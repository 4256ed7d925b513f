"""The CLI front-end (paper_2107_11983_b200/cli/walkforge.cpp) driven like the
reference's `walkforge convert|run` (proj/tools/walkforge.cpp:128-216): same
flags, WFG1 files and walk files byte-identical to the reference's."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle.oracle import RefOracle, ref_available
from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, MetaPathProgram,
                                        Node2VecProgram, PprProgram, QuerySpec, Sampler)

CLI = os.path.join(os.path.dirname(E.LIB_PATH), "walkforge_b200")


def test_cli_built_and_rejects_bad_usage():
    assert os.path.exists(CLI)
    r = subprocess.run([CLI, "frobnicate"], capture_output=True, text=True)
    assert r.returncode == 2


pytestmark_gpu = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


def _edge_list(path):
    rng = np.random.default_rng(4)
    with open(path, "w") as f:
        f.write("# cli test graph\n")
        for _ in range(4000):
            s, d = rng.integers(0, 500, 2)
            f.write(f"{s} {d} {rng.choice(['1.5', '2', '0.25', '3.75'])} {rng.integers(0, 4)}\n")


RUNS = [
    (["--algorithm", "deepwalk", "--weighted", "--length", "20"], DeepWalkProgram(20, True), {}),
    (["--algorithm", "ppr", "--termination", "0.3", "--queries", "source:7:300"], PprProgram(0.3),
     {"spec": QuerySpec.from_source(7, 300)}),
    (["--algorithm", "node2vec", "-a", "0.5", "-b", "2", "--length", "15", "--binary-output"],
     Node2VecProgram(0.5, 2.0, 15, False), {"fmt": 1}),
    (["--algorithm", "metapath", "--schema", "0,1,2,3", "--sampler", "rej"],
     MetaPathProgram([0, 1, 2, 3]), {"sampler": Sampler.REJ}),
    (["--algorithm", "deepwalk", "--weighted", "--length", "12", "--no-static-tables",
      "--sampler", "its", "--interleave", "off"], DeepWalkProgram(12, True),
     {"sampler": Sampler.ITS, "tables": False}),
]


@pytest.mark.gpu
@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("i", range(len(RUNS)))
def test_cli_convert_and_run_match_reference(i):
    flags, prog, extra = RUNS[i]
    ref = RefOracle()
    with tempfile.TemporaryDirectory() as d:
        el = os.path.join(d, "g.txt")
        _edge_list(el)
        wfg = os.path.join(d, "g.wfg")
        out = subprocess.run([CLI, "convert", el, wfg, "--undirected", "--weights", "file",
                              "--labels", "file"], capture_output=True, text=True, check=True).stdout
        assert out.startswith("V=")
        rg, _ = ref.load_edge_list(el, True, 1, 1)
        ref_wfg = os.path.join(d, "ref.wfg")
        rg.write_binary(ref_wfg)
        assert open(wfg, "rb").read() == open(ref_wfg, "rb").read()
        walks = os.path.join(d, "walks.out")
        res = subprocess.run([CLI, "run", wfg, "-o", walks, "--seed", "9"] + flags,
                             capture_output=True, text=True, check=True).stdout
        metrics = dict(line.split(" ", 1) for line in res.strip().splitlines())
        opts = ExecOptions(seed=9, sampler=extra.get("sampler"),
                           use_static_tables=extra.get("tables", True))
        spec = extra.get("spec", QuerySpec.one_per_vertex())
        want_path = os.path.join(d, "ref.out")
        rg.run_encoded(spec, prog, opts, extra.get("fmt", 0), path=want_path)
        assert open(walks, "rb").read() == open(want_path, "rb").read()
        want = rg.run(spec, prog, opts)
        assert int(metrics["total_steps"]) == want.metrics.total_steps


@pytest.mark.gpu
def test_cli_tune_reports_launch_choice():
    with tempfile.TemporaryDirectory() as d:
        el = os.path.join(d, "g.txt")
        _edge_list(el)
        wfg = os.path.join(d, "g.wfg")
        r = subprocess.run([CLI, "convert", el, wfg], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([CLI, "tune", wfg], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        assert "launch tuner:" in r.stdout and "blocks/SM" in r.stdout
