"""Randomised differential parity against the unmodified reference (oracle/_ref).

    python tools/fuzz_parity.py [--cases 300] [--seed 0] [--log gpurun_out/fuzz.log]

Each case draws a small graph (random degrees with a few hubs of 31..20000
edges so the warp-cooperative gathered paths run, sorted or unsorted adjacency,
multi-edges and self-loops, weights from several families — equal, small
integers, U[1,5) f32, mixed scales, zeros, f64 not float32-exact — and labels),
a program, a sampling method, static tables on/off, a query spec and a seed,
runs it on the engine (device walk set; every third case also the host-streaming
path with a random chunk size, every third the worker blocks over devices
[0] / [0, 0] with PPR's visit counts, every fifth the encoded walk file,
text or binary, against the reference writer's bytes) and on the reference, and compares outcome class (same exception
or none), every walk and the step total.  Test infrastructure: the reference is
the checker.  Exit code = number of differing cases.
"""
import argparse
import os
import sys
import tempfile
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.oracle import RefOracle  # noqa: E402
from paper_2107_11983_b200 import abi  # noqa: E402
from paper_2107_11983_b200 import engine as E  # noqa: E402
from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, Graph, MetaPathProgram,  # noqa: E402
                                        Node2VecProgram, PprProgram, QuerySpec, UniformProgram)


def draw_graph(rng):
    V = int(rng.choice([3, 17, 64, 300, 1500, 5000]))
    base = rng.integers(0, 6, V)
    if rng.random() < 0.3:
        base[rng.random(V) < 0.2] = 0  # dead ends
    n_hubs = int(rng.integers(0, 6))
    for _ in range(n_hubs):
        base[int(rng.integers(0, V))] = int(rng.choice([31, 32, 33, 64, 127, 128, 129, 255, 257, 300, 1000, 4097, 6000, 20000]))
    deg = base.astype(np.int64)
    off = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint64)
    Etot = int(off[-1])
    style = rng.choice(["sorted_simple", "sorted_multi", "unsorted"])
    nbr = np.empty(Etot, np.uint32)
    for v in range(V):
        d = int(deg[v])
        if d == 0:
            continue
        if style == "sorted_simple" and d <= V:
            nb = np.sort(rng.choice(V, d, replace=False))
        else:
            nb = rng.integers(0, V, d)
            if style != "unsorted":
                nb = np.sort(nb)
        nbr[int(off[v]):int(off[v + 1])] = nb
    wkind = rng.choice(["none", "equal", "ints", "u15", "mixed", "zeros", "f64"])
    w = None
    if Etot and wkind != "none":
        if wkind == "equal":
            w = np.full(Etot, float(rng.choice([1.0, 2.5, 0.125])), np.float32)
        elif wkind == "ints":
            w = rng.integers(1, 6, Etot).astype(np.float32)
        elif wkind == "u15":
            w = (1.0 + 4.0 * rng.random(Etot)).astype(np.float32)
        elif wkind == "mixed":
            w = (rng.choice([1e-6, 1.0, 3.0, 1e6], Etot) * rng.integers(1, 50, Etot)).astype(np.float32)
        elif wkind == "zeros":
            w = rng.integers(0, 4, Etot).astype(np.float32)
        else:
            w = 0.1 + rng.random(Etot) * 3.0  # float64, not f32-exact
    elif wkind != "none":
        w = np.zeros(0, np.float32)
    labels = None
    lc = int(rng.choice([0, 0, 3, 5, 12]))
    if lc:
        labels = rng.integers(0, lc, Etot).astype(np.uint8)
    return Graph(off, nbr, w, labels), dict(V=V, E=Etot, style=str(style), wkind=str(wkind), labels=lc,
                                            maxdeg=int(deg.max()) if V else 0)


def draw_program(rng, g, meta):
    weighted = g.weights is not None and rng.random() < 0.7
    kinds = ["ppr", "deepwalk", "node2vec", "uniform"] + (["metapath"] * 2 if meta["labels"] else [])
    k = rng.choice(kinds)
    if k == "ppr":
        return PprProgram(float(rng.choice([0.2, 0.5, 0.05, 1.0]))), "ppr"
    if k == "deepwalk":
        return DeepWalkProgram(int(rng.choice([1, 2, 9, 40])), weighted), f"deepwalk(w={weighted})"
    if k == "node2vec":
        a, b = float(rng.choice([0.25, 0.5, 1.0, 2.0, 4.0])), float(rng.choice([0.25, 0.5, 1.0, 2.0, 4.0]))
        return Node2VecProgram(a, b, int(rng.choice([2, 9, 30])), weighted), f"node2vec({a},{b},w={weighted})"
    if k == "uniform":
        return UniformProgram(int(rng.choice([1, 5, 25]))), "uniform"
    n = int(rng.choice([1, 4, 19]))
    present = np.unique(g.labels) if g.labels.size else np.array([0])
    pool = present if rng.random() < 0.9 else np.arange(meta["labels"])
    return MetaPathProgram([int(x) for x in rng.choice(pool, n)]), f"metapath(len={n})"


def draw_spec(rng, V):
    m = rng.choice(["per_vertex", "source", "list"])
    if m == "per_vertex":
        return QuerySpec.one_per_vertex(), "one_per_vertex"
    if m == "source":
        return QuerySpec.from_source(int(rng.integers(0, V)), int(rng.choice([0, 1, 257, 3000]))), "from_source"
    return QuerySpec.from_list(rng.integers(0, V, int(rng.choice([1, 100, 4097]))).astype(np.uint32)), "from_list"


def outcome(fn):
    try:
        return None, fn()
    except abi.WalkforgeError as e:
        return type(e).__name__, None


def ref_outcome(fn):
    try:
        return None, fn()
    except Exception as e:  # the oracle wrapper raises the same classes by name
        return type(e).__name__, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=300)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--log", default="")
    args = ap.parse_args()
    log = open(args.log, "w") if args.log else sys.stdout
    ref = RefOracle()
    rng = np.random.default_rng(args.seed)
    bad = 0
    errors = {}
    t0 = time.time()
    for case in range(args.cases):
        g, meta = draw_graph(rng)
        try:
            prog, pname = draw_program(rng, g, meta)
        except abi.WalkforgeError as e:  # constructor validation (same on both sides: host class)
            continue
        spec, sname = draw_spec(rng, meta["V"])
        sampler = rng.choice([None, abi.Sampler.NAIVE, abi.Sampler.ITS, abi.Sampler.ALIAS, abi.Sampler.REJ,
                              abi.Sampler.OREJ])
        layout = int(rng.choice([0, 0, 0, abi.LAYOUT_COMPACT_ALIAS, abi.LAYOUT_WIDE_ALIAS,
                                 abi.LAYOUT_FORCE_ADJ, abi.LAYOUT_NO_ADJ, abi.LAYOUT_ADJ8,
                                 abi.LAYOUT_SEARCH_TREE, abi.LAYOUT_NO_EDGE_FILTER,
                                 abi.LAYOUT_NO_MP_SUCC]))
        opts = ExecOptions(seed=int(rng.integers(0, 1 << 40)), sampler=None if sampler is None else int(sampler),
                           use_static_tables=bool(rng.random() < 0.5),
                           rej_trial_cap=int(rng.choice([1 << 20, 1 << 20, 64])), layout_flags=layout,
                           # PPR rows shorter than some walks: the overflow re-run path
                           path_stride=int(rng.choice([0, 0, 4, 16])) if pname == "ppr" else 0)
        chunk = int(rng.choice([0, 1, 256, 4096, 65536]))
        workers = int(rng.integers(1, 8))
        devices = [0, 0] if rng.random() < 0.5 else [0]
        desc = (f"case {case}: {meta} {pname} {sname} sampler={sampler} tables={opts.use_static_tables} "
                f"cap={opts.rej_trial_cap} layout={layout} stride={opts.path_stride} chunk={chunk} workers={workers} "
                f"devices={devices} seed={opts.seed}")
        try:
            rg = ref.graph(g)
            dg = E.DeviceGraph.from_host(g)
            rerr, want = ref_outcome(lambda: rg.run(spec, prog, opts, interleaved=bool(case & 1)))
            gerr, got = outcome(lambda: E.run_sequential(dg, spec, prog, opts))
            ok = rerr == gerr
            if ok and want is not None:
                ok = got.walks.first_mismatch(want.walks) is None and \
                    got.metrics.total_steps == want.metrics.total_steps
            if ok and want is not None and case % 3 == 0:  # host streaming (chunk = publication granularity)
                herr, hres = outcome(lambda: E.Session(dg, prog, opts).run_to_numpy(spec, chunk))
                ok = herr is None and hres.walks.first_mismatch(want.walks) is None
            if ok and want is not None and case % 3 == 1:  # worker blocks over devices, in worker order
                is_ppr = pname == "ppr"
                merr, mres = outcome(lambda: E.MultiDevice(dg, devices, prog, opts).run(spec, workers, counts=is_ppr))
                ok = merr is None
                if ok:
                    res, cnt, order = mres
                    ok = res.walks.first_mismatch(want.walks) is None and \
                        [w for w, _, _ in order] == list(range(workers))
                    if ok and is_ppr:
                        ok = np.array_equal(cnt, np.bincount(want.walks.vertices, minlength=meta["V"]))
            if ok and want is not None and case % 5 == 2:  # the qid-ordered file (wf_walkset_write) vs the reference writer
                fmt = int(case // 5) & 1
                with tempfile.TemporaryDirectory() as td:
                    fp = os.path.join(td, "walks.out")
                    E.Session(dg, prog, opts).run(spec).write(fp, fmt)
                    ok = open(fp, "rb").read() == rg.run_encoded(spec, prog, opts, fmt)
            errors[rerr] = errors.get(rerr, 0) + 1
            if not ok:
                bad += 1
                print("DIFF " + desc + f" ref={rerr} gpu={gerr}", file=log, flush=True)
        except Exception:
            bad += 1
            print("CRASH " + desc + "\n" + traceback.format_exc(), file=log, flush=True)
    print(f"{args.cases} cases (seed {args.seed}), {bad} differing, outcomes {errors}, "
          f"{time.time() - t0:.0f} s", file=log, flush=True)
    if log is not sys.stdout:
        print(f"{args.cases} cases (seed {args.seed}), {bad} differing, outcomes {errors}")
    return bad


if __name__ == "__main__":
    sys.exit(min(main(), 100))
