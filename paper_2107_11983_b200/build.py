"""Builds the engine library in-tree: paper_2107_11983_b200/libwalkforge_b200.so.

nvcc for sm_100a only (`-gencode arch=compute_100a,code=sm_100a`), -lineinfo so
ncu's source page maps to the kernels, -fmad=false so no fp64 multiply-add is
ever contracted (the sampler tables and draws must round exactly like the
reference's separate multiply and add).  Objects are rebuilt when any source or
header is newer.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# experiment hooks (tools only): alternative defines build into another object dir / library
EXTRA = os.environ.get("WF_BUILD_DEFINES", "").split()
OBJ = os.environ.get("WF_BUILD_DIR", os.path.join(HERE, "_build"))
LIB = os.environ.get("WF_LIB", os.path.join(HERE, "libwalkforge_b200.so"))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC",
                     "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
                     f"-I{os.path.join(ROOT, 'include')}"] + EXTRA


def nvcc() -> str:
    for cand in [shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"]:
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def source_hash() -> str:
    """sha256 (16 hex) over the library's sources, headers and nvcc flags: the
    stamp that ties a committed ncu capture (profiles/ncu_traffic.json) to the
    kernels it measured."""
    import hashlib
    files = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                   + glob.glob(os.path.join(CSRC, "*.hpp"))
                   + glob.glob(os.path.join(ROOT, "include", "walkforge_b200", "**", "*"), recursive=True)
                   + [os.path.join(ROOT, "include", "walkforge_b200.h")])
    h = hashlib.sha256()
    for f in files:
        if os.path.isfile(f):
            h.update(os.path.relpath(f, ROOT).encode())
            with open(f, "rb") as fh:
                h.update(fh.read())
    h.update(" ".join(a for a in NVCC_FLAGS if not a.startswith("-I")).encode())
    return h.hexdigest()[:16]


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def build(verbose: bool = False, jobs: int = 4) -> str:
    os.makedirs(OBJ, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.hpp"))
               + glob.glob(os.path.join(ROOT, "include", "walkforge_b200", "device", "*"))
               + [os.path.join(ROOT, "include", "walkforge_b200.h")])
    hdr_time = _newest(headers)
    procs = []
    objs = []
    for src in sources:
        obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time):
            continue
        cmd = [nvcc()] + NVCC_FLAGS + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        while len([p for _, p in procs if p.poll() is None]) >= jobs:
            procs[0][1].wait()
    failed = []
    for src, p in procs:
        out, _ = p.communicate()
        text = out.decode(errors="replace")
        if p.returncode != 0:
            failed.append(f"{src}:\n{text}")
        elif verbose and text.strip():
            print(text, file=sys.stderr)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-lrt",
                                                               "-lpthread", "-ldl"]
        subprocess.check_call(cmd)
    # the reference CLI's front-end (cli/walkforge.cpp) over the C-ABI
    cli_src = os.path.join(HERE, "cli", "walkforge.cpp")
    cli = os.path.join(os.path.dirname(LIB), "walkforge_b200")
    if os.path.exists(cli_src) and (not os.path.exists(cli) or os.path.getmtime(cli) < max(
            os.path.getmtime(cli_src), os.path.getmtime(LIB))):
        subprocess.check_call(["g++", "-std=c++20", "-O2", f"-I{os.path.join(ROOT, 'include')}",
                               cli_src, "-o", cli, f"-L{os.path.dirname(LIB)}",
                               f"-l:{os.path.basename(LIB)}", "-Wl,-rpath,$ORIGIN"])
    return LIB


def build_user_program(src: str, out: str) -> str:
    """Compiles a user's device-program translation unit (one that includes
    walkforge_b200/device_program.cuh and uses WF_DEVICE_PROGRAM) into a
    shared library, with the engine's own flags: the way a user of the
    library builds a custom program."""
    deps = [src] + glob.glob(os.path.join(ROOT, "include", "walkforge_b200", "**", "*"), recursive=True) + [
        os.path.join(ROOT, "include", "walkforge_b200.h")]
    if os.path.exists(out) and os.path.getmtime(out) >= _newest(deps):
        return out
    subprocess.check_call([nvcc()] + NVCC_FLAGS + ["-shared", "-o", out, src])
    return out


def build_test_programs() -> str:
    """tests/programs/libwf_test_programs.so (test code: the reference's own
    custom test programs written against the device program API)."""
    d = os.path.join(ROOT, "tests", "programs")
    return build_user_program(os.path.join(d, "test_programs.cu"), os.path.join(d, "libwf_test_programs.so"))


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
