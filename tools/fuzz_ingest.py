"""Randomised differential check of the device edge-list ingest
(wf_graph_load_edge_list, csrc/graph_io.cu) against the unmodified reference's
load_edge_list (graph.cpp:307-453).

    python tools/fuzz_ingest.py [--cases 400] [--seed 0] [--log gpurun_out/fuzz_ingest.log]

Each case writes a random text edge list — dense or sparse 64-bit ids, comments
(whole-line and trailing), blank lines, tabs / runs of spaces / CRLF, weight and
label columns in decimal, scientific or integer form, duplicates, self-loops —
and, in a third of the cases, one malformed line (a word, a missing or extra
column, a negative or non-finite weight, a label out of range, an id that
overflows).  Both loaders run with the same random options (directedness,
weights / labels none | from file | random, label count, seed); they must raise
the same error class with the same message, or give the same CSR (offsets,
neighbours, f64 weights, labels) and original ids, and the WFG1 file written
from the device graph must equal the reference's byte for byte.  The one
documented difference — a label >= 256, which the u8 device labels refuse — is
counted apart.
Test infrastructure: the reference is the checker.  Exit code = differing cases.
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
from paper_2107_11983_b200 import engine as E  # noqa: E402


def fmt_weight(rng, w):
    k = rng.integers(0, 5)
    if k == 0:
        return repr(float(w))
    if k == 1:
        return f"{w:.3f}"
    if k == 2:
        return f"{w:.6e}"
    if k == 3:
        return str(int(w) + 1)
    return f"{w:g}"


def draw_file(rng):
    n_ids = int(rng.choice([1, 2, 5, 40, 400]))
    if rng.random() < 0.5:
        ids = np.arange(n_ids, dtype=np.uint64)
    else:
        ids = np.unique(rng.integers(0, int(rng.choice([50, 10**6, 2**40, 2**63])), n_ids, dtype=np.uint64))
    n_lines = int(rng.choice([1, 3, 30, 300, 3000]))
    cols = int(rng.choice([2, 3, 4]))  # src dst [weight [label]]
    sep = rng.choice([" ", "\t", "  ", " \t "])
    eol = "\r\n" if rng.random() < 0.15 else "\n"
    lines = []
    for _ in range(n_lines):
        r = rng.random()
        if r < 0.05:
            lines.append("# " + "x" * int(rng.integers(0, 20)))
            continue
        if r < 0.09:
            lines.append("" if rng.random() < 0.5 else "   ")
            continue
        u, v = ids[rng.integers(0, ids.size)], ids[rng.integers(0, ids.size)]
        tok = [str(int(u)), str(int(v))]
        if cols >= 3:
            tok.append(fmt_weight(rng, rng.random() * 9.0 + (0.0 if rng.random() < 0.9 else 1e6)))
        if cols >= 4:
            tok.append(str(int(rng.integers(0, 5))))
        line = (" " if rng.random() < 0.1 else "") + sep.join(tok)
        if rng.random() < 0.1:
            line += " # trailing"
        lines.append(line)
    bad = None
    if rng.random() < 0.33 and lines:
        bad = rng.choice(["word", "one_col", "extra_col", "neg_w", "nan_w", "inf_w", "big_label", "neg_id",
                          "overflow_id", "float_id", "hex_id", "plus_id"])
        at = int(rng.integers(0, len(lines)))
        w = "1.5" if cols >= 3 else ""
        lab = "1" if cols >= 4 else ""
        tail = (" " + w if w else "") + (" " + lab if lab else "")
        lines[at] = {
            "word": "nonsense here",
            "one_col": "7",
            "extra_col": "0 1 1.0 2 9",
            "neg_w": "0 1 -2.5" + (" 1" if cols >= 4 else ""),
            "nan_w": "0 1 nan" + (" 1" if cols >= 4 else ""),
            "inf_w": "0 1 inf" + (" 1" if cols >= 4 else ""),
            "big_label": "0 1 1.0 4000000000" if cols >= 4 else "0 1 1.0 7",
            "neg_id": "-3 1" + tail,
            "overflow_id": "18446744073709551616 1" + tail,
            "float_id": "1.5 2" + tail,
            "hex_id": "0x10 2" + tail,
            "plus_id": "+4 2" + tail,
        }[str(bad)]
    text = eol.join(lines) + (eol if rng.random() < 0.8 else "")
    return text, cols, bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=400)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--log", default="")
    args = ap.parse_args()
    log = open(args.log, "w") if args.log else sys.stdout
    ref = RefOracle()
    rng = np.random.default_rng(args.seed)
    differing, outcomes = 0, {}
    t0 = time.time()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "edges.txt")
        for case in range(args.cases):
            text, cols, bad = draw_file(rng)
            with open(path, "w", newline="") as f:
                f.write(text)
            undirected = bool(rng.random() < 0.4)
            wmode = int(rng.choice([0, 1, 2])) if cols >= 3 else int(rng.choice([0, 1, 2], p=[0.6, 0.1, 0.3]))
            lmode = int(rng.choice([0, 1, 2])) if cols >= 4 else int(rng.choice([0, 1, 2], p=[0.6, 0.1, 0.3]))
            label_count = int(rng.choice([1, 3, 5, 200]))
            seed = int(rng.integers(0, 1 << 40))
            desc = (f"case {case}: cols={cols} bad={bad} undirected={undirected} weights={wmode} labels={lmode} "
                    f"label_count={label_count} seed={seed} bytes={len(text)}")
            try:
                try:
                    rg, rids = ref.load_edge_list(path, undirected, wmode, lmode, label_count, seed)
                    rerr = None
                except Exception as e:
                    rerr, rmsg = type(e).__name__, str(e)
                try:
                    dg = E.DeviceGraph.load_edge_list(path, undirected, wmode, lmode, label_count, seed)
                    gerr = None
                except Exception as e:
                    gerr, gmsg = type(e).__name__, str(e)
                outcomes[rerr] = outcomes.get(rerr, 0) + 1
                if bad == "big_label" and rerr is None and gerr == "ConfigError" and "label" in gmsg:
                    # the one documented difference: device labels are u8 (north star: "uint8 edge
                    # labels"), a label >= 256 is refused where the reference keeps a u32
                    outcomes["label>=256 refused (documented)"] = outcomes.get("label>=256 refused (documented)", 0) + 1
                    continue
                ok = rerr == gerr
                why = f"ref={rerr} gpu={gerr}"
                if ok and rerr is not None:
                    ok = rmsg == gmsg
                    why = f"messages differ: ref={rmsg!r} gpu={gmsg!r}"
                if ok and rerr is None:
                    off, nbr, w, lab = rg.export()
                    hg = dg.download()
                    ok = (np.array_equal(off, hg.offsets) and np.array_equal(nbr, hg.neighbors)
                          and np.array_equal(rids, dg.original_ids())
                          and (w is None) == (hg.weights is None)
                          and (w is None or np.array_equal(w, hg.weights.astype(np.float64)))
                          and (lab is None) == (hg.labels is None)
                          and (lab is None or np.array_equal(lab, hg.labels.astype(np.uint32))))
                    why = "CSR / attributes / original ids differ"
                    if ok:
                        a, b = os.path.join(d, "a.wfg"), os.path.join(d, "b.wfg")
                        rg.write_binary(a)
                        dg.write_wfg1(b)
                        ok = open(a, "rb").read() == open(b, "rb").read()
                        why = "WFG1 bytes differ"
                if not ok:
                    differing += 1
                    print("DIFF " + desc + " " + why, file=log, flush=True)
                    keep = os.path.join(os.path.dirname(args.log) or ".", f"fuzz_ingest_case{args.seed}_{case}.txt")
                    with open(keep, "w", newline="") as f:
                        f.write(text[:20000])
            except Exception:
                differing += 1
                print("CRASH " + desc + "\n" + traceback.format_exc(), file=log, flush=True)
    msg = f"{args.cases} cases (seed {args.seed}), {differing} differing, outcomes {outcomes}, {time.time() - t0:.0f} s"
    print(msg, file=log, flush=True)
    if log is not sys.stdout:
        print(msg)
    return differing


if __name__ == "__main__":
    sys.exit(min(main(), 100))
