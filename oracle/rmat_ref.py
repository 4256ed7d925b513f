"""Independent numpy restatement of the synthetic R-MAT generator (SURVEY §8 d)
used to check the device generator bit for bit at small scales.

Draw i uses RngStream(seed ^ RMAT_SALT, i) (rng.hpp:23-30); each 64-bit draw
decides two recursion levels (high 32 bits, then low 32 bits) against
floor(a 2^32), floor((a+b) 2^32), floor((a+b+c) 2^32).  Symmetrise, drop
self-loops, dedup, sort.  Weights: f32(1 + uniform_real(4)) of
RngStream(seed ^ WEIGHT_SALT, e); labels uniform_index(L) of
RngStream(seed ^ LABEL_SALT, e) (graph.cpp:279-287), e = final CSR edge index.
"""
from __future__ import annotations

import math

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
SALT = np.uint64(0xA3EC647659359ACD)
RMAT_SALT = 0x524D4154454447
WEIGHT_SALT = 0x57464757454947
LABEL_SALT = 0x5746474C41424C


def mix(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def stream_state(seed: int, streams):
    with np.errstate(over="ignore"):
        pre = mix(np.uint64(seed) + GAMMA)
        return mix(pre ^ mix(np.asarray(streams, dtype=np.uint64) ^ SALT))


def next_u64(state):
    with np.errstate(over="ignore"):
        state = state + GAMMA
    return state, mix(state)


def rmat_edges(scale, edge_factor, a, b, c, seed):
    n = edge_factor << scale
    st = stream_state(seed ^ RMAT_SALT, np.arange(n, dtype=np.uint64))
    t1 = np.uint64(min(math.floor(a * 2 ** 32), 2 ** 32 - 1))
    t2 = np.uint64(min(math.floor((a + b) * 2 ** 32), 2 ** 32 - 1))
    t3 = np.uint64(min(math.floor((a + b + c) * 2 ** 32), 2 ** 32 - 1))
    s = np.zeros(n, np.uint64)
    d = np.zeros(n, np.uint64)
    for lvl in range(0, scale, 2):
        st, x = next_u64(st)
        for h in range(2):
            l = lvl + h
            if l >= scale:
                break
            u = (x >> np.uint64(32)) if h == 0 else (x & np.uint64(0xFFFFFFFF))
            bit = np.uint64(1 << (scale - 1 - l))
            q1 = (u >= t1) & (u < t2)
            q2 = (u >= t2) & (u < t3)
            q3 = u >= t3
            d |= np.where(q1 | q3, bit, np.uint64(0))
            s |= np.where(q2 | q3, bit, np.uint64(0))
    return s, d


def rmat_csr(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, weighted=False,
             label_count=0):
    s, d = rmat_edges(scale, edge_factor, a, b, c, seed)
    keep = s != d
    s, d = s[keep], d[keep]
    src = np.concatenate([s, d])
    dst = np.concatenate([d, s])
    key = np.unique((src << np.uint64(32)) | dst)
    src = (key >> np.uint64(32)).astype(np.int64)
    dst = (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    V = 1 << scale
    off = np.zeros(V + 1, np.uint64)
    np.add.at(off, src + 1, 1)
    off = np.cumsum(off, dtype=np.uint64)
    E = dst.size
    w = lab = None
    if weighted:
        stw = stream_state(seed ^ WEIGHT_SALT, np.arange(E, dtype=np.uint64))
        _, r = next_u64(stw)
        u = (r >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        x = u * 4.0
        x = np.where(x < 4.0, x, np.nextafter(4.0, 0.0))
        w = (1.0 + x).astype(np.float32)
    if label_count:
        stl = stream_state(seed ^ LABEL_SALT, np.arange(E, dtype=np.uint64))
        _, r = next_u64(stl)
        # (r * n) >> 64 for n < 2^32: split r into 32-bit halves
        hi = r >> np.uint64(32)
        lo = r & np.uint64(0xFFFFFFFF)
        n = np.uint64(label_count)
        lab = ((hi * n + ((lo * n) >> np.uint64(32))) >> np.uint64(32)).astype(np.uint8)
    return off, dst, w, lab
