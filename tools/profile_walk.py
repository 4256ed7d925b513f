"""Launch the walk kernel of one bench config a few times (for ncu / timing).

    python tools/profile_walk.py --config c5 [--scale 24] [--launches 3]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--scale", type=int, default=0)
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--layout", type=int, default=0)
    ap.add_argument("--queries", type=int, default=0, help="override the batch size (random-source configs)")
    ap.add_argument("--counts", action="store_true", help="PPR: also accumulate visit counts")
    ap.add_argument("--diag-times", action="store_true",
                    help="library built with -DWF_DIAG_FINISH_TIME: print walk completion-time percentiles")
    ap.add_argument("--tune", action="store_true", help="run the launch tuner first (wf_session_tune)")
    ap.add_argument("--graph", action="store_true", help="replay the launch as a captured CUDA graph")
    ap.add_argument("--flush", action="store_true", help="write 256 MiB between launches (cold L2, as bench.py)")
    ap.add_argument("--stride", type=int, default=0, help="path row stride override (vertices)")
    ap.add_argument("--per-vertex", action="store_true",
                    help="random-source configs: one walk per vertex in vertex order instead")
    args = ap.parse_args()
    import torch

    from paper_2107_11983_b200 import engine as E
    from paper_2107_11983_b200.host import ExecOptions
    cfg = dict(bench.CONFIGS[args.config] if args.config in bench.CONFIGS else bench.GATHERED[args.config])
    if args.scale:
        cfg["scale"] = args.scale
    dg = E.DeviceGraph.rmat(cfg["scale"], 16, seed=1, weighted=cfg["weighted"],
                            label_count=cfg["labels"])
    V = dg.info()["V"]
    sess = E.Session(dg, bench.program_of(cfg), ExecOptions(seed=1, path_stride=bench.row_capacity(cfg),
                                                            layout_flags=args.layout, **bench.exec_extra(cfg)))
    if args.queries and cfg["queries"] == "random":
        cfg["n_queries"] = args.queries
    if args.per_vertex:
        cfg["queries"] = "per_vertex"
    spec, lo, hi = bench.query_plan(cfg, V, 0, 1)
    n = hi - lo
    stride = args.stride or bench.row_capacity(cfg)
    d_src = torch.from_numpy(spec.sources.view("int32")).cuda()
    paths = torch.empty(n * stride, dtype=torch.int32, device="cuda")
    lens = torch.empty(n, dtype=torch.int32, device="cuda")
    st = torch.empty(n, dtype=torch.uint8, device="cuda")
    steps = torch.zeros(1, dtype=torch.int64, device="cuda")
    counts = torch.zeros(V, dtype=torch.int32, device="cuda") if args.counts else None
    stream = torch.cuda.current_stream()
    l2buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if args.flush else None
    def launch():
        s = torch.cuda.current_stream()
        sess.launch(spec, lo, hi, paths.data_ptr(), stride, lens.data_ptr(), st.data_ptr(),
                    counts.data_ptr() if counts is not None else 0, steps.data_ptr(), 0, s.cuda_stream,
                    sources_dev_ptr=d_src.data_ptr())

    if args.tune:
        print("tuned blocks/SM, ms:", sess.tune(spec, lo, hi, sources_dev_ptr=d_src.data_ptr()), flush=True)
    graph = None
    if args.graph:
        launch()  # warm (no allocation inside the capture)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            launch()
        torch.cuda.synchronize()
    # ncu --nvtx --nvtx-include "timed/" captures only these launches (not the tuner's)
    torch.cuda.nvtx.range_push("timed")
    for i in range(args.launches):
        steps.zero_()
        if l2buf is not None:
            bench.flush_l2(l2buf)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            launch()
        e1.record(stream)
        sess.sync(stream.cuda_stream)
        dt = time.perf_counter() - t
        ms = e0.elapsed_time(e1)
        print(f"launch {i}: {steps.item()} moves {ms:.3f} ms (events; wall {dt*1e3:.2f}) "
              f"{steps.item()/ms/1e6:.2f} G steps/s V={V} E={dg.info()['E']} layout={sess.layout()}",
              flush=True)
        if args.diag_times:
            import numpy as np
            raw = lens.cpu().numpy().view(np.uint32).astype(np.int64)
            t = raw >> 8
            t = ((t - t.min()) % (1 << 24)) * 32e-3  # us
            ln = raw & 255
            qs = [50, 90, 99, 99.9, 99.99, 100]
            print("  finish us: " + " ".join(f"p{q}={np.percentile(t, q):.1f}" for q in qs), flush=True)
            last = np.argsort(t)[-8:]
            print("  last walks (finish us, length): " + " ".join(f"({t[i]:.0f},{ln[i]})" for i in last))
            for lo, hi in [(1, 8), (8, 16), (16, 32), (32, 64), (64, 256)]:
                sel = (ln >= lo) & (ln < hi)
                if sel.any():
                    print(f"  length [{lo},{hi}): n={sel.sum()} mean finish {t[sel].mean():.1f} us, "
                          f"max {t[sel].max():.1f} us")

    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main()
