"""Multi-GPU query sharding (SURVEY §8 e).

Walk queries are independent — each depends only on (graph, seed, qid)
(R/SPEC.md:269,295) — so a job is split into contiguous qid blocks exactly as
the reference splits it over worker threads (worker_range,
proj/include/walkforge/engine.hpp:296-298).  Each rank holds a replica of the
graph; the only exchange is the PPR visit-count vector, summed with one
all-reduce (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Tuple


def worker_range(n: int, workers: int, w: int) -> Tuple[int, int]:
    """[n*w/W, n*(w+1)/W) — engine.hpp:296-298."""
    return n * w // workers, n * (w + 1) // workers


def shard_queries(n_queries: int, world: int, rank: int) -> Tuple[int, int]:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return worker_range(n_queries, world, rank)


def reduce_visit_counts(counts, dist=None):
    """Sum per-shard visit counts across ranks (in place); no-op single rank."""
    if dist is not None and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(counts)
    return counts
