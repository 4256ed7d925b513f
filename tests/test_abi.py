"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/walkforge_b200.h declares, and the ctypes mirror matches
the C struct layouts.  No compute call is made (no GPU here)."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2107_11983_b200 import abi
from paper_2107_11983_b200 import build as wfbuild
from paper_2107_11983_b200 import engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "walkforge_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(engine.LIB_PATH):
        wfbuild.build()
    return engine.load_library()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(wf_[a-z_0-9]+)\s*\(", text)
    return sorted(set(names))


def test_header_declarations_match_python_list():
    assert declared_functions() == sorted(abi.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", engine.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (wf_[a-z_0-9]+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing
    assert lib.wf_abi_version() == 1


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", engine.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_struct_layouts_match_header():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "walkforge_b200.h"
#define S(t) printf(#t " %zu\n", sizeof(t));
#define O(t, f) printf(#t "." #f " %zu\n", offsetof(t, f));
int main(void) {
  S(wf_program_desc) O(wf_program_desc, termination) O(wf_program_desc, schema) O(wf_program_desc, schema_len)
  S(wf_exec_options) O(wf_exec_options, sampler) O(wf_exec_options, path_stride)
  S(wf_query_spec) O(wf_query_spec, count) O(wf_query_spec, sources)
  S(wf_run_metrics) O(wf_run_metrics, total_steps)
  S(wf_graph_info) O(wf_graph_info, max_weight) O(wf_graph_info, label_count)
  S(wf_rmat_params) O(wf_rmat_params, seed) O(wf_rmat_params, label_count)
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        exe = os.path.join(d, "l")
        open(c, "w").write(src)
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        lines = dict(l.rsplit(" ", 1) for l in subprocess.check_output([exe], text=True).splitlines())
    m = {"wf_program_desc": abi.ProgramDesc, "wf_exec_options": abi.ExecOptionsC,
         "wf_query_spec": abi.QuerySpecC, "wf_run_metrics": abi.RunMetricsC,
         "wf_graph_info": abi.GraphInfoC, "wf_rmat_params": abi.RmatParamsC}
    for key, val in lines.items():
        if "." in key:
            t, f = key.split(".")
            cf = "max_degree" if f == "max_degree_lo" else f
            assert getattr(m[t], cf).offset == int(val), key
        else:
            assert C.sizeof(m[key]) == int(val), key


def test_no_cpu_fallback_without_device(lib):
    """Compute calls fail loudly (WF_ERR_CUDA) where there is no GPU."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(abi.CudaError):
        engine.rng_probe(1, [0], 2)
