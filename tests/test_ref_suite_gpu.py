"""The reference's own "engine", "interleave", "algorithms" and "graph" unit
suites (/root/reference/proj/tests/test_engine.cpp, test_interleave.cpp,
test_algorithms.cpp, test_graph.cpp) re-expressed
against the drop-in shim (tests/cpp/ref_suite.cpp: same case names and call
patterns, custom programs as device programs) compiled with plain g++ the way a
reference caller would, and run on the GPU."""
import os
import subprocess
import tempfile

import pytest

from paper_2107_11983_b200 import engine as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROGRAMS = os.path.join(ROOT, "tests", "programs")


def build_suite(tmp, name="ref_suite"):
    exe = os.path.join(tmp, name)
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                           os.path.join(ROOT, "tests", "cpp", name + ".cpp"), "-o", exe, "-lpthread",
                           "-L", os.path.dirname(E.LIB_PATH), "-lwalkforge_b200",
                           f"-Wl,-rpath,{os.path.dirname(E.LIB_PATH)}",
                           "-L", PROGRAMS, "-l:libwf_test_programs.so", f"-Wl,-rpath,{PROGRAMS}"])
    return exe


def test_ref_suite_compiles_cpu_only():
    with tempfile.TemporaryDirectory() as d:
        assert os.path.exists(build_suite(d))


@pytest.mark.gpu
def test_reference_engine_and_interleave_suites_pass_through_the_shim():
    with tempfile.TemporaryDirectory() as d:
        exe = build_suite(d)
        p = subprocess.run([exe, d], capture_output=True, text=True, timeout=900)
    lines = p.stdout.strip().splitlines()
    failed = [ln for ln in lines if ln.startswith("FAIL") or ln.startswith("    ")]
    assert p.returncode == 0 and not failed, p.stdout[-4000:] + p.stderr[-2000:]
    assert lines[-1] == "42 cases, 0 failed", lines[-1]
    assert sum((ln.startswith("ok") and " engine: " in ln) for ln in lines) == 14
    assert sum((ln.startswith("ok") and " interleave: " in ln) for ln in lines) == 8
    assert sum((ln.startswith("ok") and " algorithms: " in ln) for ln in lines) == 8
    assert sum((ln.startswith("ok") and " graph: " in ln) for ln in lines) == 12


def test_reference_output_suite_passes_on_the_shim_headers():
    """test_output.cpp's ten cases against walkforge_b200/output.hpp (host-only: CPU suite)."""
    with tempfile.TemporaryDirectory() as d:
        exe = build_suite(d, "ref_output_suite")
        p = subprocess.run([exe, d], capture_output=True, text=True, timeout=300)
    lines = p.stdout.strip().splitlines()
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-1000:]
    assert lines[-1] == "11 cases, 0 failed", lines[-1]  # the 10 reference cases + one of the shim's own
