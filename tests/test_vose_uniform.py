"""The closed form the gathered ALIAS hub step uses when every positive weight
is equal (engine.cuh: vose_bucket_uniform), restated in Python floats (IEEE
doubles) and checked bucket by bucket against a straight transcription of the
reference's FIFO Vose build (proj/include/walkforge/sampler.hpp:89-120).
CPU only; the device path is checked against the reference's walks in
tests/test_gathered_hubs_gpu.py."""
import math
import random


def vose_reference(weights):
    """sampler.hpp:89-120: bucket i -> (split, alias)."""
    n = len(weights)
    total = 0.0
    for w in weights:
        total += w
    scaled = [w * n / total for w in weights]
    small = [i for i in range(n) if scaled[i] < 1.0]
    large = [i for i in range(n) if not scaled[i] < 1.0]
    out, sh, lh = {}, 0, 0
    while sh < len(small) and lh < len(large):
        s = small[sh]
        sh += 1
        lg = large[lh]
        out[s] = (scaled[s], lg)
        scaled[lg] -= 1.0 - scaled[s]
        if scaled[lg] < 1.0:
            lh += 1
            small.append(lg)
    for i in small[sh:] + large[lh:]:
        out[i] = (1.0, i)
    return out, total


def vose_uniform(weights, total, x):
    """Mirror of vose_bucket_uniform; None where the device falls back to the chain."""
    n = len(weights)
    pos = [i for i in range(n) if weights[i] > 0]
    m = len(pos)
    c = weights[pos[0]] * n / total
    if m == n or not c >= 1.0 or not c < 2.0 ** 52:
        return (1.0, x) if m == n else None
    K = int(c)
    f = c - K
    Z = n - m
    before = sum(1 for i in range(x) if weights[i] > 0)
    if not weights[x] > 0:
        j = (x - before) // K
        return (0.0, pos[j]) if j < m else (1.0, x)
    D = Z // K
    if before >= D:
        return None
    e = math.frexp(c)[1] - 53  # ulp(c) = 2^e
    t = 1.0 - f
    v0 = c - (Z - D * K)
    T = int(math.ldexp(t, -e))
    assert math.ldexp(t, -e) == T and math.ldexp(v0 - 1.0, -e).is_integer()  # exact unit arithmetic
    a0 = int(math.ldexp(v0 - 1.0, -e)) // T + 1
    ac = int(math.ldexp(c - 1.0, -e)) // T + 1
    head = D if before < a0 else D + 1 + (before - a0) // ac
    return (f, pos[head]) if head < m else (1.0, x)


def test_uniform_closed_form_matches_vose():
    rng = random.Random(1)
    checked = 0
    for _ in range(700):
        n = rng.randint(2, 240)
        m = rng.randint(1, n) if rng.random() < 0.5 else max(1, n // rng.choice([2, 3, 5, 7, 10]))
        w = rng.choice([1.0, 3.0, 0.1, 0.7, 2.5, 1e-3, 7.25, 1 / 3])
        idx = set(rng.sample(range(n), m))
        weights = [w if i in idx else 0.0 for i in range(n)]
        ref, total = vose_reference(weights)
        for x in range(n):
            got = vose_uniform(weights, total, x)
            if got is not None:
                assert got == ref[x], (n, m, w, x, got, ref[x])
                checked += 1
    assert checked > 50000
