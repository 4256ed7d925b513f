#!/usr/bin/env python
"""Benchmark: RW steps/sec of the B200 walk engine (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5]
                    [--impl ours|reference] [--no-extras]

One "step" = one pass of the hot path over one batch of queries of the named
configuration (BASELINE.json `configs`, SURVEY §8 d shorthand):

  c1  DeepWalk s16 weighted ALIAS, one walk per vertex, L=80
  c2  PPR s20, NAIVE, 2^20 uniform random sources, stop 0.2, + visit counts
  c3  Node2Vec s22 (a=2, b=0.5) O-REJ, one walk per vertex, L=80
  c4  MetaPath s22, 5 labels, schema [i%5]x79, one walk per vertex
  c5  DeepWalk s26 weighted ALIAS, 2^26 walks, L=80                      [default]

The default is C5, BASELINE.json's box-scale config for the 1/2/4/8-GPU sweep
(the largest single-GPU configuration); C1-C4 are reported under
`per_algorithm`, each with its own reference CPU baseline.

Graphs are synthetic R-MAT (a,b,c,d = .57/.19/.19/.05, edge factor 16, seed 1)
generated on the device; the paper's real graphs are not in this container.

value     device-resident throughput: moves / s, inputs in HBM, CUDA events on
          the launching stream, max over ranks.
e2e       same metric through the C-ABI call that returns walks in HOST memory
          (wf_session_run_host_records; offsets_api: wf_session_run_host): H2D
          of the step's source list from pinned host memory + D2H of the whole
          walk set (ragged) into pinned host memory; L2 flushed before each
          step as for `value` (small graphs).
roofline  algorithmic bytes per launch (SURVEY §8 d S_alg x moves) / mean launch
          time vs the measured HBM copy bandwidth (MEASURED_PEAKS.json).  S_alg
          is §8 d's per-move figure for the reference CSR layout (ALIAS / NAIVE
          2.375 sectors = 76 B; O-REJ and MetaPath from instrumented logical
          counts); `layout` gives the same for the decorated layouts this
          engine uses; measured_sectors: HBM bandwidth / measured DRAM bytes per
          move (ncu, profiles/ncu_traffic.json, stamped with the source hash it
          was captured from; a capture of other sources is reported stale).
cpu_baseline  the unmodified reference (oracle/_ref, run_interleaved k=64 k'=32,
          all host threads, no-op sink) on a bounded sample, rank 0 at N=1.

Multi-GPU (torchrun): graph replicated per rank, queries sharded in contiguous
qid blocks (worker_range, engine.hpp:296-298).  One-walk-per-vertex configs
(C1, C3-C5) split the fixed walk set over the ranks (strong scaling: BASELINE's
"2^26 walks sharded evenly across GPUs"); C2 gives every rank its own batch of
2^20 random sources (weak scaling); PPR visit counts are summed with one NCCL
all-reduce inside the timed step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RW steps/sec at 1/2/4/8 B200 per algorithm; % of HBM random-access roofline"
SECTOR = 32

CONFIGS = {
    "c1": dict(workload="C1 DeepWalk R-MAT s16 ef16, weighted f32 [1,5), ALIAS tables, one walk "
                        "per vertex, length 80, seed 1", scale=16, program="deepwalk", length=80,
               weighted=True, labels=0, queries="per_vertex", scaling="strong"),
    "c2": dict(workload="C2 PPR R-MAT s20 ef16, unweighted, NAIVE, 2^20 uniform random sources, "
                        "stop 0.2, walks + visit counts", scale=20, program="ppr", weighted=False,
               labels=0, queries="random", n_queries=1 << 20, scaling="weak"),
    "c3": dict(workload="C3 Node2Vec R-MAT s22 ef16, p=a=2 q=b=0.5, O-REJ, one walk per vertex, "
                        "length 80", scale=22, program="node2vec", length=80, weighted=False,
               labels=0, queries="per_vertex", scaling="strong"),
    "c4": dict(workload="C4 MetaPath R-MAT s22 ef16, labels u8 {0..4}, f32 weights (unused), "
                        "schema [i%5]x79, one walk per vertex", scale=22, program="metapath",
               weighted=True, labels=5, queries="per_vertex", scaling="strong"),
    "c5": dict(workload="C5 DeepWalk R-MAT s26 ef16, weighted f32 [1,5), ALIAS tables, 2^26 walks, "
                        "length 80", scale=26, program="deepwalk", length=80, weighted=True,
               labels=0, queries="per_vertex", scaling="strong"),
}

# Gathered flows (a per-step gather over every edge of the current vertex,
# engine.hpp:134-184) on the s22 graph: not BASELINE configs, but the flows
# whose hub steps run warp-cooperatively (coop_step); reported under
# per_algorithm with their own reference baselines.
GATHERED = {
    "g1": dict(workload="G1 Node2Vec R-MAT s22 (a=2, b=0.5), ITS gathered (per-step gather), 2^16 walks from "
                        "uniform random sources, length 80", scale=22, program="node2vec", length=80, weighted=False,
               labels=0, queries="random", n_queries=1 << 16, scaling="weak", sampler="ITS", tables=True),
    "g2": dict(workload="G2 MetaPath R-MAT s22, ALIAS gathered (Vose per step), schema [i%5]x79, 2^16 walks "
                        "from uniform random sources", scale=22, program="metapath", weighted=True, labels=5,
               queries="random", n_queries=1 << 16, scaling="weak", sampler="ALIAS", tables=True),
    "g3": dict(workload="G3 DeepWalk R-MAT s22 weighted, ALIAS without static tables (Vose per step), 2^16 "
                        "walks from uniform random sources, length 80", scale=22, program="deepwalk", length=80,
               weighted=True, labels=0, queries="random", n_queries=1 << 16, scaling="weak", sampler="ALIAS",
               tables=False),
}


def exec_extra(cfg):
    """ExecOptions overrides of a config (sampler / static tables)."""
    from paper_2107_11983_b200 import abi
    out = {}
    if cfg.get("sampler"):
        out["sampler"] = int(getattr(abi.Sampler, cfg["sampler"]))
    if "tables" in cfg:
        out["use_static_tables"] = bool(cfg["tables"])
    return out


# CPU-baseline samples (queries), sized for ~10-30 s of reference work on 16 cores
CPU_SAMPLE = {"c1": 1 << 16, "c2": 1 << 20, "c3": 1 << 20, "c4": 1 << 15, "c5": 1 << 22,
              "g1": 1 << 12, "g2": 1 << 12, "g3": 1 << 12}


def program_of(cfg):
    from paper_2107_11983_b200.host import (DeepWalkProgram, MetaPathProgram, Node2VecProgram,
                                            PprProgram)
    p = cfg["program"]
    if p == "deepwalk":
        return DeepWalkProgram(cfg["length"], cfg["weighted"])
    if p == "ppr":
        return PprProgram(0.2)
    if p == "node2vec":
        return Node2VecProgram(2.0, 0.5, cfg["length"], False)
    return MetaPathProgram([i % 5 for i in range(79)])


def row_capacity(cfg):
    if cfg["program"] == "ppr":
        return 64
    if cfg["program"] == "metapath":
        return 80
    return cfg["length"]


def worker_range(n, workers, w):
    """worker_range (engine.hpp:296-298) from the engine library (wf_worker_range),
    or its formula where no library is built (CPU-only tests)."""
    try:
        from paper_2107_11983_b200 import engine as E
        return E.worker_range(n, workers, w)
    except (OSError, FileNotFoundError):
        return n * w // workers, n * (w + 1) // workers


def query_plan(cfg, V, rank, world):
    """(QuerySpec over the whole job, qid_begin, qid_end) for this rank: the
    job's contiguous worker_range shard (engine.hpp:296-298)."""
    from paper_2107_11983_b200.host import QuerySpec
    if cfg["queries"] == "random":
        # weak scaling: the job is world batches of 2^20 random sources, so
        # every rank's shard is one batch
        total = cfg["n_queries"] * world
        src = np.random.default_rng(1).integers(0, V, total, dtype=np.uint32)
        spec = QuerySpec.from_list(src)
    else:
        # one walk per vertex; the vertex list is sharded (C5: 2^26 walks split
        # evenly).  FROM_LIST with sources[q] = q is the same walk set as
        # one_per_vertex and gives the e2e path a real H2D input.
        spec = QuerySpec.from_list(np.arange(V, dtype=np.uint32))
    lo, hi = worker_range(spec.count, world, rank)
    return spec, lo, hi


def make_comm(dist, rank, world, device):
    """The engine's own NCCL communicator (wf_comm_*) for the PPR visit-count
    reduction: rank 0's id travels over the torch process group (plumbing
    only); the reduction itself is the library's ncclAllReduce."""
    if dist is None:
        return None
    from paper_2107_11983_b200 import engine as E
    obj = [E.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return E.Comm(obj[0], world, rank, device)


def reduce_counts(counts, comm, dist, stream=0):
    """Sum the ranks' visit-count vectors in place: the path's one collective
    (SURVEY 8(e)).  On GPUs through the library communicator; without one
    (CPU tests, gloo) through the process group."""
    if comm is not None:
        comm.allreduce_u32(counts.data_ptr(), counts.numel(), stream)
    elif dist is not None and dist.get_world_size() > 1:
        dist.all_reduce(counts)


def combine_ranks(dist, device, total_ms, e2e_s, e2e_off_s, moves):
    """Max over ranks of the device times, sum of the moves (the contract's
    whole-job value)."""
    if dist is None:
        return total_ms, e2e_s, e2e_off_s, moves
    import torch
    t = torch.tensor([total_ms, e2e_s or 0.0, e2e_off_s or 0.0], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    mv = torch.tensor([moves], dtype=torch.int64, device=device)
    dist.all_reduce(mv)
    return float(t[0]), float(t[1]), float(t[2]), int(mv.item())


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def s_alg(cfg, stats, moves, layout, steps=None):
    """Algorithmic 32 B sectors per move, two ways.

    ref (SURVEY §8 d, the figure `roofline.frac` uses): the reference's CSR
    layout, no cache reuse, no overfetch.
      ALIAS (C1, C5) and NAIVE (C2): offsets pair 1.25 + bucket / neighbour 1
        + path 1/8 = 2.375 sectors = 76 B (PPR's visit counts live in L2 and
        are not counted).
      O-REJ (C3): 1.25 + per trial (1 neighbour + ceil(log2(d_prev + 1))
        binary-search probes when the reference's weight() tests adjacency)
        + 1/8, from the instrumented counters (`ref_probes`).
      MetaPath (C4): per step 1.25 + ceil(d_v / 32) label sectors, per move
        + 1 neighbour + 1/8 (`ref_label_sectors`, `steps`).
    layout: the same count for the decorated layouts this engine uses (abi.HAS_*).
    Returns dict(ref=sectors, ref_model=text, layout=sectors, layout_model=text,
    requests=random requests per move)."""
    from paper_2107_11983_b200 import abi
    p = cfg["program"]
    mv = max(moves, 1)
    if cfg.get("sampler") and (p in ("node2vec", "metapath") or not cfg.get("tables", True)):
        # gathered flows: the per-step gather reads every edge's weight input
        # (u8 label, f32 weight, or u32 neighbour + adjacency test)
        eb = {"metapath": 1, "deepwalk": 4, "node2vec": 4}[p]
        sc = stats.get("scanned", 0) / mv
        pr = stats.get("probes", 0) / mv
        ref = 1.25 + sc * eb / SECTOR + pr + 1.0 + 0.125
        text = (f"gathered: offsets 1.25 + {sc:.1f} edges x {eb} B / 32 + {pr:.2f} adjacency-test sectors "
                f"+ neighbour 1 + 1/8 = {ref:.3f} sectors (instrumented edges scanned per move)")
        return dict(ref=ref, ref_model=text, layout=ref, layout_model=text, requests=1.0 + pr)
    one = {"deepwalk": abi.HAS_WIDE_ALIAS, "ppr": abi.HAS_ADJ, "metapath": abi.HAS_MP_SUCC}
    if p in one:
        reads = 1.0 if layout & one[p] else 2.0
        if reads == 1.0:
            desc = {"deepwalk": "32 B alias bucket carrying the next vertex word",
                    "ppr": "16 B adjacency entry carrying the next vertex word",
                    "metapath": "16 B partitioned edge carrying the next label group"}[p]
        else:
            desc = {"deepwalk": "16 B alias bucket + 8 B vertex word",
                    "ppr": "4 B neighbour + 8 B vertex word",
                    "metapath": "32 B label record + 4 B partitioned neighbour"}[p]
        lay, lay_text = reads + 0.125, f"{desc} + 1/8 path = {reads + 0.125:.3f} sectors"
    else:
        trials = stats.get("trials", 0) / mv
        probes = stats.get("probes", 0) / mv
        base = 0.0 if layout & abi.HAS_ADJ else 1.0
        reads = base + trials + probes
        lay = reads + 0.125
        lay_text = (f"{trials:.3f} trial adjacency sectors + {probes:.3f} filter/hash sectors"
                    f"{' + vertex word' if base else ''} + 1/8 path = {lay:.3f} sectors")
    if p in ("deepwalk", "ppr"):
        ref = 2.375
        ref_text = ("SURVEY 8(d): offsets pair 1.25 + " + ("16 B alias bucket" if p == "deepwalk" else "neighbour")
                    + " 1 + path 1/8 = 2.375 sectors = 76 B per move")
    elif p == "node2vec" and "ref_probes" in stats:
        trials = stats["trials"] / mv
        rp = stats["ref_probes"] / mv
        ref = 1.25 + trials + rp + 0.125
        ref_text = (f"SURVEY 8(d): offsets 1.25 + {trials:.3f} trial neighbour sectors + {rp:.3f} binary-search "
                    f"probes (instrumented ceil(log2(d_prev+1)) per adjacency test) + 1/8 = {ref:.3f} sectors")
    elif p == "metapath" and "ref_label_sectors" in stats and steps:
        st = steps / mv
        ls = stats["ref_label_sectors"] / mv
        ref = 1.25 * st + ls + 1.0 + 0.125
        ref_text = (f"SURVEY 8(d): offsets 1.25 x {st:.3f} steps + {ls:.3f} label sectors (instrumented "
                    f"ceil(d_v/32) per step) + neighbour 1 + 1/8 = {ref:.3f} sectors")
    else:
        ref, ref_text = lay, "no instrumented reference counts: layout figure"
    return dict(ref=ref, ref_model=ref_text, layout=lay, layout_model=lay_text, requests=reads)


def random_access_block(moves_per_s, reads_per_move):
    """Random HBM requests per second against the measured B200 ceiling for
    random 32 B requests (tools/randbw.cu: every random sector miss fetches a
    128 B line; profiles/random_access.json)."""
    ceiling = None
    try:
        with open(os.path.join(ROOT, "profiles", "random_access.json")) as f:
            ceiling = float(json.load(f)["random_sector_requests_per_s"])
    except Exception:
        pass
    req = moves_per_s * reads_per_move
    return {"logical_requests_per_move": reads_per_move, "logical_requests_per_s": req,
            "measured_dram_miss_ceiling_requests_per_s": ceiling,
            "frac_of_ceiling": (req / ceiling) if ceiling else None,
            "note": "ceiling = random 32 B requests that all miss L2 (each a 128 B DRAM fetch); "
                    "requests served by L2 (hot vertices, search index) can push frac above 1"}


def source_sha():
    from paper_2107_11983_b200.build import source_hash
    return source_hash()


def ncu_traffic():
    """profiles/ncu_traffic.json: DRAM bytes (read + write) per walk-kernel launch
    and per move, from ncu captures of each config at its tuned grid, stamped
    with the library source hash they were captured from."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def traffic_for(key, moves):
    """(bytes per launch, bytes per move, stamp) of the committed capture for
    this config; None values when missing or captured from other sources."""
    t = ncu_traffic()
    ent = t.get("configs", {}).get(key)
    cur = source_sha()
    stamp = {"captured_src_sha": (ent or {}).get("src_sha"), "current_src_sha": cur,
             "source": "profiles/ncu_traffic.json (dram__bytes_read.sum + dram__bytes_write.sum, "
                       "one ncu launch of this config's walk kernel at its tuned grid)"}
    if not ent:
        stamp["stale"] = None
        return None, None, stamp
    stamp["stale"] = ent.get("src_sha") != cur
    stamp["captured_moves"] = ent.get("moves")
    if stamp["stale"] or ent.get("moves") != moves:
        if ent.get("moves") != moves:
            stamp["note"] = "capture ran a different number of moves"
        return None, None, stamp
    return ent["bytes"], ent["bytes"] / moves, stamp


# What bounds each config's walk kernel; the numbers in
# the note are computed from the run and the stamped capture (bound_note).
BOUND_CAUSE = {
    "c1": "the graph is L2-resident; the 65 Ki walks' dependent L2 chains bound it",
    "c2": "the bulk saturates the L2/atomic queue and the longest geometric walks finish in an unloaded tail",
    "c3": "one 128 B DRAM line per O-REJ trial (adjacency entry) plus the L2-resident pair filter",
    "c4": "one random DRAM request per move (successor-decorated partitioned edge, 64 B fetch)",
    "c5": "one random DRAM request per move (wide alias bucket, 64 B fetch): the random-request rate of HBM",
    "g1": "per-step gathers over the current vertex's edges (hub steps warp-cooperative), each a Node2Vec "
          "adjacency test",
    "g2": "per-step gathers of the current vertex's labels and Vose's construction per step",
    "g3": "per-step gathers of the current vertex's weights and Vose's construction per step",
}


def bound_note(key, moves_per_s, bytes_per_move, peak):
    cause = BOUND_CAUSE.get(key, "")
    if bytes_per_move is None:
        return f"{cause}; no current ncu capture for these sources, DRAM rate not computed"
    dram = moves_per_s * bytes_per_move / 1e9
    f = dram / peak
    kind = "DRAM-bound" if f >= 0.6 else "not DRAM-bound"
    return (f"{kind}: {cause}. ncu measured {bytes_per_move:.1f} B of DRAM traffic per move "
            f"({bytes_per_move / SECTOR:.2f} sectors); at this run's rate that is {dram:.0f} GB/s "
            f"= {f:.1%} of the measured copy bandwidth")


def roofline_block(key, cfg, r, moves, ms_per_launch, peak, peak_kind):
    """The line's roofline object for one config (see the module docstring)."""
    sa = s_alg(cfg, r["stats"], moves, r["layout"], steps=r.get("step_attempts") or r["stats"].get("step_attempts"))
    launch_s = ms_per_launch * 1e-3
    rate = moves / launch_s
    ach = moves * sa["ref"] * SECTOR / launch_s / 1e9
    lay = moves * sa["layout"] * SECTOR / launch_s / 1e9
    traffic, bpm, stamp = traffic_for(key, moves)
    return {
        "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
        "traffic": traffic,
        "peak_source": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
        "bytes_per_move": sa["ref"] * SECTOR, "bytes_model": sa["ref_model"],
        "layout": {"bytes_per_move": sa["layout"] * SECTOR, "model": sa["layout_model"],
                   "achieved": lay, "frac": lay / peak},
        "measured_sectors": None if bpm is None else {
            "bytes_per_move": bpm, "ceiling_steps_per_s": peak / bpm * 1e9,
            "frac": rate / (peak / bpm * 1e9)},
        "traffic_stamp": stamp,
        "note": bound_note(key, rate, bpm, peak),
        **({"caveat": "frac > 1: SURVEY 8(d)'s S_alg counts the sectors the reference's layout would touch "
                      "(binary-search probes, label scans) that this engine's layout does not read; "
                      "layout.frac and measured_sectors.frac are the bytes actually moved"}
           if ach / peak > 1 else {}),
    }, sa

def flush_l2(buf):
    buf.add_(1)


def run_ours(args, cfg, rank, world, local_rank, dist, comm=None):
    import torch

    from paper_2107_11983_b200 import engine as E
    from paper_2107_11983_b200.host import ExecOptions

    torch.cuda.set_device(local_rank)
    dev = local_rank
    t_setup = time.time()
    dg = E.DeviceGraph.rmat(cfg["scale"], 16, seed=1, weighted=cfg["weighted"],
                            label_count=cfg["labels"], device=dev)
    info = dg.info()
    V = info["V"]
    prog = program_of(cfg)
    opts = ExecOptions(seed=1, path_stride=row_capacity(cfg), **exec_extra(cfg))
    sess = E.Session(dg, prog, opts)
    sampler, flow, pre_s = sess.describe()
    layout = sess.layout()
    spec, lo, hi = query_plan(cfg, V, rank, world)
    n = hi - lo
    stride = row_capacity(cfg)
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    d_src = torch.from_numpy(spec.sources.view(np.int32)).to(f"cuda:{dev}")
    paths = torch.empty(n * stride, dtype=torch.int32, device=dev)
    lens = torch.empty(n, dtype=torch.int32, device=dev)
    stat = torch.empty(n, dtype=torch.uint8, device=dev)
    steps = torch.zeros(1, dtype=torch.int64, device=dev)
    over = torch.zeros(1, dtype=torch.int64, device=dev)
    counts = torch.zeros(V, dtype=torch.int32, device=dev) if cfg["program"] == "ppr" else None
    small = cfg["scale"] <= 20  # working set near L2 size: flush between steps
    l2buf = torch.zeros((256 << 20) // 4, dtype=torch.float32, device=dev) if small else None

    def device_step():
        s = torch.cuda.current_stream()
        steps.zero_()
        if counts is not None:
            counts.zero_()
        sess.launch(spec, lo, hi, paths.data_ptr(), stride, lens.data_ptr(), stat.data_ptr(),
                    counts.data_ptr() if counts is not None else 0, steps.data_ptr(),
                    over.data_ptr(), s.cuda_stream, sources_dev_ptr=d_src.data_ptr())

    graph = None

    def one_step():
        if graph is not None:
            graph.replay()
        else:
            device_step()
        if counts is not None:
            reduce_counts(counts, comm, dist, torch.cuda.current_stream().cuda_stream)

    # launch tuner (wf_session_tune, the device analogue of the reference's
    # tune_ring_sizes): picks blocks/SM for launches of this size; untimed
    tuned = None
    if not args.no_tune:
        tuned = sess.tune(spec, lo, hi, sources_dev_ptr=d_src.data_ptr())[0]

    # logical access counts for S_alg (one instrumented pass, untimed)
    sess.set_stats(True)
    one_step()
    sess.sync(sptr)
    stats = sess.stats()
    moves_per_step = int(steps.item())
    sess.set_stats(False)
    # The step's device work (counter resets + the walk kernel) is captured
    # once as a CUDA graph and replayed: a 0.2 ms kernel otherwise waits
    # ~20 us per step for the host to submit it.  Every replay runs the whole
    # walk kernel; wf_session_launch is capturable (no host sync, no allocation
    # once warm).
    launches_c0 = E.kernel_launches()
    if not args.no_graph:
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            device_step()
        torch.cuda.synchronize()
    kernels_per_step = E.kernel_launches() - launches_c0 if graph is not None else None
    for _ in range(args.warmup):
        one_step()
    sess.sync(sptr)
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup

    launches0 = E.kernel_launches()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            if small:
                flush_l2(l2buf)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            ev[k][0].record(stream)
            one_step()
            ev[k][1].record(stream)
            torch.cuda.synchronize()
    sess.sync(sptr)
    launches = E.kernel_launches() - launches0
    if kernels_per_step is not None:  # replays do not pass the host-side counter
        launches = kernels_per_step * args.steps
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    assert int(steps.item()) == moves_per_step, "walks are deterministic per step"

    # end to end through the C-ABI with host buffers (pinned)
    e2e = None
    if not args.no_e2e:
        cap = n * stride  # >= total vertices: rows hold whole walks; PPR averages ~5
        h_src = torch.from_numpy(spec.sources.view(np.int32)).pin_memory()
        h_off = torch.empty(n + 1, dtype=torch.int64).pin_memory()
        h_vert = torch.empty(cap, dtype=torch.int32).pin_memory()
        h_stat = torch.empty(n, dtype=torch.uint8).pin_memory()
        from paper_2107_11983_b200.host import QuerySpec
        hspec = QuerySpec.from_list(spec.sources)
        hspec_c_sources = h_src  # keep alive
        hspec.sources = h_src.numpy().view(np.uint32)
        for _ in range(1):
            sess.run_host(hspec, h_off.data_ptr(), h_vert.data_ptr(), cap, h_stat.data_ptr(),
                          qid_begin=lo, qid_end=hi)
        # the offsets form is a secondary API: a few steps suffice when a step
        # moves gigabytes (C5: 11 GB)
        off_steps = args.steps if n * stride * 4 < (1 << 30) else min(args.steps, 3)
        e2e_s = []
        for _ in range(off_steps):
            if l2buf is not None:
                flush_l2(l2buf)  # cold L2 for every timed step, as for `value`
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m = sess.run_host(hspec, h_off.data_ptr(), h_vert.data_ptr(), cap, h_stat.data_ptr(),
                              qid_begin=lo, qid_end=hi)
            e2e_s.append(time.perf_counter() - t0)
        total_vertices = int(h_off[n].item())
        assert m.total_steps == moves_per_step
        e2e_off = dict(seconds=float(sum(e2e_s)), steps=off_steps, h2d=n * 4, d2h=total_vertices * 4 + (n + 1) * 8 + n,
                       api="wf_session_run_host (offsets u64 + status u8, pinned host buffers)")
        # the records form (length | status << 31 per query, walker.hpp:47-55's
        # WalkRecord without the implicit qid): 4 B per query instead of 9
        h_rec = torch.empty(n, dtype=torch.int32).pin_memory()
        sess.run_host_records(hspec, h_rec.data_ptr(), h_vert.data_ptr(), cap, qid_begin=lo, qid_end=hi)
        e2e_s = []
        for _ in range(args.steps):
            if l2buf is not None:
                flush_l2(l2buf)
            if dist:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m = sess.run_host_records(hspec, h_rec.data_ptr(), h_vert.data_ptr(), cap, qid_begin=lo, qid_end=hi)
            e2e_s.append(time.perf_counter() - t0)
        assert m.total_steps == moves_per_step
        assert int((h_rec.numpy().view(np.uint32) & 0x7FFFFFFF).astype(np.int64).sum()) == total_vertices
        e2e = dict(seconds=float(sum(e2e_s)), steps=args.steps, h2d=n * 4, d2h=total_vertices * 4 + n * 4,
                   api="wf_session_run_host_records (pinned host buffers)", offsets_api=e2e_off)
        del hspec_c_sources

    return dict(moves=moves_per_step, total_ms=total_ms, step_ms=step_ms, stats=stats,
                launches=launches, clocks=clk.summary(), info=info, sampler=sampler.name,
                flow=flow.name, preprocess_s=pre_s, setup_s=setup_s, e2e=e2e, n=n, dg=dg, layout=layout,
                spec=spec, sess=sess, tuned=tuned)


def cpu_baseline(key, cfg, dg, spec, threads=None):
    """The unmodified reference (oracle/_ref) on a bounded sample — measurement
    only; never on the product path."""
    from oracle.oracle import PortOracle, RefOracle, ref_available
    from paper_2107_11983_b200.host import ExecOptions, QuerySpec
    threads = threads or os.cpu_count()
    m = min(CPU_SAMPLE[key], spec.count)
    sample = QuerySpec.from_list(spec.sources[:m])
    hg = dg.download()
    prog = program_of(cfg)
    opts = ExecOptions(seed=1, threads=threads, **exec_extra(cfg))
    if ref_available():
        rg = RefOracle().graph(hg)
        del hg
        run = lambda: rg.run(sample, prog, opts, interleaved=True, discard=True)  # noqa: E731
        kind = "reference"
    else:
        port = PortOracle()
        run = lambda: port.run(hg, sample, prog, opts, threads=threads, discard=True)  # noqa: E731
        kind = "port"
    run()  # warm-up (first-touch page faults skew cold runs, SURVEY §8 d)
    moves, secs, pre, reps, t0 = 0, 0.0, 0.0, 0, time.time()
    while reps < 1 or (time.time() - t0 < 3.0 and reps < 200):  # >= ~3 s of CPU work
        res = run()
        moves += res.metrics.total_steps
        secs += res.metrics.exec_seconds
        pre = res.metrics.preprocess_seconds
        reps += 1
    rate = moves / max(secs, 1e-9)
    return dict(value=rate, unit="steps/s", cores=threads, kind=kind,
                sample=f"first {m} of the config's queries x {reps} runs ({moves} moves, "
                       f"{secs:.2f} s exec; preprocess {pre:.2f} s per run excluded as in "
                       f"engine.hpp:455,498), run_interleaved k=64 k'=32, {threads} threads, "
                       f"no-op sink, one warm-up run")


def extras(args, rank, world, local_rank, dist):
    """GPU numbers for the other configs (not bench lines; evidence), each with
    its own reference CPU baseline."""
    out = {}
    peak, peak_kind = measured_peak()
    for key in ["c1", "c2", "c3", "c4", "c5"] + sorted(GATHERED):
        if key == args.config:
            continue
        try:
            # e2e evidence too, except for C5 (10.9 GB of pinned host buffers per step)
            a = argparse.Namespace(**{**vars(args), "steps": 3, "warmup": 1,
                                      "no_e2e": key == "c5" or key in GATHERED})
            cfg = CONFIGS[key] if key in CONFIGS else GATHERED[key]
            r = run_ours(a, cfg, rank, world, local_rank, dist)
            ms = r["total_ms"] / 3
            roof, sa = roofline_block(key, cfg, r, r["moves"], ms, peak, peak_kind)
            rate = r["moves"] / (ms * 1e-3)
            ent = dict(workload=cfg["workload"], steps_per_s=rate, blocks_per_sm=r["tuned"],
                       ms_per_step=ms, moves=r["moves"], roofline=roof,
                       e2e=None if not r["e2e"] else {
                           "value": r["moves"] * r["e2e"]["steps"] / r["e2e"]["seconds"], "unit": "steps/s",
                           "h2d_bytes_per_step": r["e2e"]["h2d"], "d2h_bytes_per_step": r["e2e"]["d2h"],
                           "api": r["e2e"]["api"]},
                       random_access=random_access_block(rate, sa["requests"]),
                       preprocess_seconds=r["preprocess_s"], E=r["info"]["E"])
            if not args.no_cpu and key != "c5":
                try:
                    ent["cpu_baseline"] = cpu_baseline(key, cfg, r["dg"], r["spec"])
                    ent["vs_cpu_baseline"] = rate / ent["cpu_baseline"]["value"]
                except Exception as e:
                    ent["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"}
            out[key] = ent
            del r
            import torch
            torch.cuda.empty_cache()
        except Exception as e:  # evidence only; never fail the headline
            out[key] = dict(error=f"{type(e).__name__}: {e}")
    return out


def reference_arm(args, cfg, rank, world):
    """--impl reference: the reference's own CPU path, rank 0 only.  Its input
    is built on the CPU (RefOracle.rmat: the oracle's C R-MAT, bit-identical
    to the device generator, handed straight to Graph::from_csr); no engine
    code runs on this arm."""
    if rank != 0:
        return
    from oracle.oracle import PortOracle, RefOracle, ref_available
    from paper_2107_11983_b200.host import ExecOptions, QuerySpec
    threads = os.cpu_count()
    t0 = time.time()
    kind = "reference" if ref_available() else "port"
    if kind == "reference":
        rg = RefOracle().rmat(cfg["scale"], 16, seed=1, weighted=cfg["weighted"],
                              label_count=cfg["labels"])
        info = rg.info()
        V, E_count = info["V"], info["E"]
    else:
        hg = PortOracle().rmat(cfg["scale"], 16, seed=1, weighted=cfg["weighted"],
                               label_count=cfg["labels"])
        V, E_count = hg.vertex_count, hg.edge_count
    graph_s = time.time() - t0
    spec, lo, hi = query_plan(cfg, V, 0, 1)
    # Every run_interleaved call rebuilds the static tables (ResolvedRun,
    # engine.hpp:275-294; 39 s at C5), so the K steps run as ONE call over K
    # consecutive samples of m queries (preprocessing excluded from the metric,
    # engine.hpp:455,498, as in the reference), after one warm-up call over one
    # sample (first-touch page faults).
    n_all = hi - lo
    m = min(CPU_SAMPLE[args.config], max(1, n_all // max(args.steps, 1)))
    prog = program_of(cfg)
    opts = ExecOptions(seed=1, threads=threads, **exec_extra(cfg))

    def run(queries):
        sample = QuerySpec.from_list(spec.sources[:queries])
        if kind == "reference":
            return rg.run(sample, prog, opts, interleaved=True, discard=True)
        return PortOracle().run(hg, sample, prog, opts, threads=threads, discard=True)

    if args.warmup > 0:
        run(m)
    r = run(m * args.steps)
    moves, secs, pre = r.metrics.total_steps, r.metrics.exec_seconds, r.metrics.preprocess_seconds
    value = moves / secs
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "int64+f64", "data": "synthetic R-MAT",
        "config": {"workload": cfg["workload"], "sample_queries_per_step": m,
                   "graph": "CPU R-MAT (oracle/wf_oracle.c wfo_rmat_csr, bit-identical to the device build) "
                            "-> Graph::from_csr", "graph_build_seconds": graph_s,
                   "vertices": int(V), "edges": int(E_count)},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": threads, "kind": kind,
                         "sample": f"{args.steps} steps of {m} queries (the first {m * args.steps} of the "
                                   f"config's queries) in one run_interleaved call, k=64 k'=32, no-op sink, "
                                   f"preprocessing ({pre:.2f} s) excluded (engine.hpp:455,498); one warm-up "
                                   f"call over {m} queries"},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit_line(line)


# The JSON line is the only thing on stdout: native libraries that print there
# (NCCL's version banner under torchrun) are pointed at stderr at the file
# descriptor level, and the line itself goes to the saved stdout.
_JSON_FD = None


def _stdout_for_json_only():
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit_line(line):
    text = json.dumps(line) + "\n"
    if _JSON_FD is None:
        print(text, end="", flush=True)
    else:
        os.write(_JSON_FD, text.encode())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS) + sorted(GATHERED))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tune", action="store_true", help="skip the launch tuner (occupancy grid)")
    ap.add_argument("--no-graph", action="store_true", help="launch each step from the host instead of a CUDA graph replay")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    cfg = CONFIGS[args.config] if args.config in CONFIGS else GATHERED[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, cfg, rank, world)
        return

    import torch
    dist = None
    if world > 1 or "RANK" in os.environ:  # any torchrun launch, even N=1
        _stdout_for_json_only()
        # NCCL's init log names every rank of the communicators (the engine's
        # own for the visit counts and torch's for the barriers)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # ... on stderr: stdout carries only rank 0's JSON line
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        dist = tdist
    comm = make_comm(dist, rank, world, local_rank) if cfg["program"] == "ppr" else None

    r = run_ours(args, cfg, rank, world, local_rank, dist, comm)
    total_ms = r["total_ms"]
    moves = r["moves"]
    e2e_s = r["e2e"]["seconds"] if r["e2e"] else None
    e2e_off_s = r["e2e"]["offsets_api"]["seconds"] if r["e2e"] else None
    total_ms, e2e_max, e2e_off_max, all_moves = combine_ranks(dist, "cuda", total_ms, e2e_s, e2e_off_s, moves)
    value = all_moves * args.steps / (total_ms * 1e-3)

    peak, peak_kind = measured_peak()
    roof, sa = roofline_block(args.config, cfg, r, moves, total_ms / args.steps, peak, peak_kind)
    line = {
        "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": cfg["scaling"], "vs_baseline": None, "dtype": "int64+f64",
        "data": "synthetic R-MAT (seed 1) generated on device; paper graphs not available",
        "config": {"workload": cfg["workload"], "queries_per_gpu": r["n"],
                   "vertices": r["info"]["V"], "edges": r["info"]["E"],
                   "sampler": r["sampler"], "flow": r["flow"],
                   "parallelism": f"query shards x{world}, graph replicated"
                                  + (", visit counts summed by the engine's ncclAllReduce (wf_comm)" if comm else ""),
                   "l2": "flushed between steps (256 MiB write)" if cfg["scale"] <= 20
                   else "inputs larger than L2",
                   "launch": "host launch per step" if args.no_graph
                   else "CUDA graph replay per step (counter resets + walk kernel)",
                   "blocks_per_sm": r["tuned"] if r["tuned"] is not None else "occupancy max (untuned)"},
        "roofline": roof,
        "random_access": random_access_block(moves * args.steps / (total_ms * 1e-3), sa["requests"]),
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "preprocess_seconds": r["preprocess_s"],
    }
    if r["e2e"]:
        eo = r["e2e"]["offsets_api"]
        line["e2e"] = {"value": all_moves * r["e2e"]["steps"] / e2e_max, "unit": "steps/s",
                       "h2d_bytes_per_step": r["e2e"]["h2d"], "d2h_bytes_per_step": r["e2e"]["d2h"],
                       "steps": r["e2e"]["steps"], "api": r["e2e"]["api"],
                       "offsets_api": {"value": all_moves * eo["steps"] / e2e_off_max, "steps": eo["steps"],
                                       "h2d_bytes_per_step": eo["h2d"], "d2h_bytes_per_step": eo["d2h"],
                                       "api": eo["api"]}}
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config, cfg, r["dg"], r["spec"])
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"}
    if world == 1 and not args.no_extras:
        del r
        torch.cuda.empty_cache()
        line["per_algorithm"] = extras(args, rank, world, local_rank, dist)
    if rank == 0:
        emit_line(line)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
