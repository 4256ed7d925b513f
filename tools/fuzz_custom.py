"""Randomised differential parity for USER device programs (the WalkProgram
concept, include/walkforge_b200/device_program.cuh) against the unmodified
reference running the same programs through its own API
(oracle/ref_harness.cpp: wfref_run_test_program).

    python tools/fuzz_custom.py [--cases 600] [--seed 0] [--log gpurun_out/fuzz_custom.log]

Graphs, query specs, samplers, tables on/off and trial caps are drawn as in
tools/fuzz_parity.py; the programs are tests/programs/test_programs.cu's:
CountingProgram (unbiased, counts update() calls), AvoidVertexProgram (static,
zero weights), LabelWeightProgram (dynamic, weight = label match ? w_e : 0),
LabelStopProgram (unbounded, draws in update(), reads the traversed edge).
Same exception class, or the same walks, step total and update() count.
Test infrastructure: the reference is the checker.  Exit code = differing cases.
"""
import argparse
import ctypes as C
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from fuzz_parity import draw_graph, draw_spec, outcome, ref_outcome  # noqa: E402
from oracle.oracle import RefOracle  # noqa: E402
from paper_2107_11983_b200 import abi  # noqa: E402
from paper_2107_11983_b200 import engine as E  # noqa: E402
from paper_2107_11983_b200.host import DeviceProgram, ExecOptions  # noqa: E402

PROGRAMS = os.path.join(ROOT, "tests", "programs", "libwf_test_programs.so")


class TestParams(C.Structure):  # ref_harness.cpp TestProgramParams
    _fields_ = [("length", C.c_uint32), ("banned", C.c_uint32), ("stop", C.c_double),
                ("stop_label", C.c_uint32), ("schema_len", C.c_uint32), ("schema", C.c_uint32 * 48)]


class CountingC(C.Structure):
    _fields_ = [("length", C.c_uint32), ("updates", C.c_void_p)]


class AvoidVertexC(C.Structure):
    _fields_ = [("banned", C.c_uint32), ("length", C.c_uint32)]


class LabelWeightC(C.Structure):
    _fields_ = [("schema_len", C.c_uint32), ("schema", C.c_uint32 * 48)]


class LabelStopC(C.Structure):
    _fields_ = [("stop", C.c_double), ("stop_label", C.c_uint32)]


def main():
    import torch
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=600)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--log", default="")
    args = ap.parse_args()
    log = open(args.log, "w") if args.log else sys.stdout
    ref = RefOracle()
    rng = np.random.default_rng(args.seed)
    bad, outcomes = 0, {}
    t0 = time.time()
    for case in range(args.cases):
        g, meta = draw_graph(rng)
        kinds = ["counting", "avoid"] + (["label_stop"] if meta["labels"] else []) + \
            (["label_weight"] * 2 if meta["labels"] and g.weights is not None else [])
        kind = str(rng.choice(kinds))
        ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
        if kind == "counting":
            n = int(rng.choice([1, 2, 10, 33]))
            prog, which, tp = DeviceProgram((PROGRAMS, "wf_test_counting_program"), CountingC(n, ctr.data_ptr())), 0, \
                TestParams(length=n)
        elif kind == "avoid":
            n, banned = int(rng.choice([1, 5, 20])), int(rng.integers(0, meta["V"]))
            prog, which, tp = DeviceProgram((PROGRAMS, "wf_test_avoid_vertex_program"), AvoidVertexC(banned, n)), 1, \
                TestParams(length=n, banned=banned)
        elif kind == "label_weight":
            schema = [int(x) for x in rng.integers(0, meta["labels"], int(rng.choice([1, 6, 20])))]
            arr = (C.c_uint32 * 48)(*schema)
            prog, which, tp = DeviceProgram((PROGRAMS, "wf_test_label_weight_program"),
                                            LabelWeightC(len(schema), arr)), 3, \
                TestParams(schema_len=len(schema), schema=arr)
        else:
            stop, sl = float(rng.choice([0.05, 0.3, 1.0])), int(rng.integers(0, meta["labels"]))
            prog, which, tp = DeviceProgram((PROGRAMS, "wf_test_label_stop_program"), LabelStopC(stop, sl)), 4, \
                TestParams(stop=stop, stop_label=sl)
        spec, sname = draw_spec(rng, meta["V"])
        sampler = rng.choice([None, abi.Sampler.NAIVE, abi.Sampler.ITS, abi.Sampler.ALIAS, abi.Sampler.REJ,
                              abi.Sampler.OREJ])
        opts = ExecOptions(seed=int(rng.integers(0, 1 << 40)), sampler=None if sampler is None else int(sampler),
                           use_static_tables=bool(rng.random() < 0.5),
                           rej_trial_cap=int(rng.choice([1 << 20, 1 << 20, 64])),
                           path_stride=int(rng.choice([0, 0, 4])) if kind == "label_stop" else 0)
        desc = (f"case {case}: {meta} {kind} {sname} sampler={sampler} tables={opts.use_static_tables} "
                f"cap={opts.rej_trial_cap} stride={opts.path_stride} seed={opts.seed}")
        try:
            rg = ref.graph(g)
            dg = E.DeviceGraph.from_host(g)
            rerr, want = ref_outcome(lambda: rg.run_test_program(which, tp, spec, opts, interleaved=bool(case & 1)))
            gerr, got = outcome(lambda: E.run_sequential(dg, spec, prog, opts))
            outcomes[rerr] = outcomes.get(rerr, 0) + 1
            ok = rerr == gerr
            why = ""
            if ok and want is not None:
                res, updates = want
                fm = got.walks.first_mismatch(res.walks)
                ok = fm is None and got.metrics.total_steps == res.metrics.total_steps
                if not ok:
                    why = (f" first_mismatch={fm} steps gpu={got.metrics.total_steps} ref={res.metrics.total_steps}"
                           + (f" gpu_path={got.walks.path(fm)[:6]} st={got.walks.status[fm]} "
                              f"ref_path={res.walks.path(fm)[:6]} st={res.walks.status[fm]}" if fm is not None
                              and fm < min(len(got.walks), len(res.walks)) else ""))
                if ok and kind == "counting":
                    ok = int(ctr.item()) == updates == got.metrics.total_steps
                    why = f" update() calls gpu={int(ctr.item())} ref={updates} steps={got.metrics.total_steps}"
                if ok and case % 3 == 0:
                    herr, hres = outcome(lambda: E.Session(dg, prog, opts).run_to_numpy(spec))
                    ok = herr is None and hres.walks.first_mismatch(res.walks) is None
                    why = f" streaming path: err={herr}"
            if not ok:
                bad += 1
                print("DIFF " + desc + f" params=({tp.length},{tp.banned},{tp.schema_len}) ref={rerr} gpu={gerr}" + why,
                      file=log, flush=True)
        except Exception:
            bad += 1
            print("CRASH " + desc + "\n" + traceback.format_exc(), file=log, flush=True)
    msg = f"{args.cases} cases (seed {args.seed}), {bad} differing, outcomes {outcomes}, {time.time() - t0:.0f} s"
    print(msg, file=log, flush=True)
    if log is not sys.stdout:
        print(msg)
    return bad


if __name__ == "__main__":
    sys.exit(min(main(), 100))
