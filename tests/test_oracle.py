"""Pins the C restatement (oracle/wf_oracle.c) against golden vectors produced
by the unmodified reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from oracle.oracle import PortOracle, RefOracle, ref_available
from paper_2107_11983_b200 import abi
from tests import golden_util as gu

port = PortOracle()
CASES = gu.cases()


def test_rng_golden_vectors():
    z = gu.rng()
    for (s, q), draws in zip(z["pairs"], z["draws"]):
        assert np.array_equal(port.rng_probe(int(s), int(q), 16), draws)
    for (s, q), n, b, idx, real in zip(z["ir_args_u"], z["ir_args_n"], z["ir_args_b"],
                                       z["ir_idx"], z["ir_real"]):
        i, r = port.rng_index_real(int(s), int(q), int(n), float(b))
        assert i == idx and r == real  # bit-exact doubles


def test_rng_survey_appendix():
    # SURVEY appendix (RngStream(0,0) x3) — independent of the fixtures
    assert [hex(x) for x in port.rng_probe(0, 0, 3)] == [
        "0xa8bfb5fcd49d1301", "0x710d36dd6711cdb2", "0x617cc292e13a6f46"]


def test_alias_init_golden():
    z = gu.rng()
    offs = z["alias_offsets"]
    for i in range(len(offs) - 1):
        a, b = int(offs[i]), int(offs[i + 1])
        w = z["alias_weights"][a:b]
        if w.sum() == 0:
            continue
        split, first, second = port.alias_init(w)
        assert np.array_equal(split, z["alias_split"][a:b])
        assert np.array_equal(first, z["alias_first"][a:b])
        assert np.array_equal(second, z["alias_second"][a:b])


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_port_matches_reference_walks(case):
    g = gu.graph(case["graph"])
    if "error" in case:
        with pytest.raises(getattr(abi, case["error"])):
            port.run(g, gu.spec(case), gu.program(case), gu.opts(case))
        return
    res = port.run(g, gu.spec(case), gu.program(case), gu.opts(case))
    want = gu.walks(case)
    assert res.walks.first_mismatch(want) is None
    assert res.metrics.total_steps == case["total_steps"]


@pytest.mark.parametrize("threads", [2, 5])
def test_port_thread_invariance(threads):
    case = next(c for c in CASES if c["name"] == "pl_ppr_naive")
    g = gu.graph(case["graph"])
    res = port.run(g, gu.spec(case), gu.program(case), gu.opts(case), threads=threads)
    assert res.walks.equals(gu.walks(case))


def test_port_static_tables_golden():
    t = gu.tables()
    for gname in ["powerlaw", "zeroweights", "ring"]:
        g = gu.graph(gname)
        prog = gu.program({"program": "deepwalk", "length": 20, "weighted": True})
        out = port.static_tables(g, prog, int(abi.Sampler.ALIAS))
        assert np.array_equal(out["alias_split"], t[f"{gname}/alias/alias_split"])
        assert np.array_equal(out["alias_first_dst"], t[f"{gname}/alias/alias_first_dst"])
        assert np.array_equal(out["alias_second_dst"], t[f"{gname}/alias/alias_second_dst"])
        assert np.array_equal(out["exhausted"], t[f"{gname}/alias/exhausted"])
        out = port.static_tables(g, prog, int(abi.Sampler.ITS))
        assert np.array_equal(out["its"], t[f"{gname}/its/its"])
        out = port.static_tables(g, prog, int(abi.Sampler.REJ))
        assert np.array_equal(out["rej_p_star"], t[f"{gname}/rej/rej_p_star"])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_port_matches_live_reference_on_random_graphs():
    """Where the reference library is present, compare the port with it live on
    fresh random graphs (beyond the committed fixtures)."""
    ref = RefOracle()
    rng = np.random.default_rng(3)
    for trial in range(4):
        rg = ref.power_law(300 + 100 * trial, 3000, seed=100 + trial, weighted=True,
                           label_count=4)
        off, nbr, w, lab = rg.export()
        g = gu.Graph(off, nbr, w.astype(np.float32), lab.astype(np.uint8))
        rg32 = ref.graph(g)
        for d in [dict(program="ppr", termination=0.3),
                  dict(program="deepwalk", length=15, weighted=True),
                  dict(program="node2vec", length=15, a=1.5, b=0.7, weighted=trial % 2 == 0),
                  dict(program="metapath", schema=[0, 1, 2, 3, 0])]:
            d["seed"] = int(rng.integers(0, 2 ** 63))
            want = rg32.run(gu.spec(d), gu.program(d), gu.opts(d))
            got = port.run(g, gu.spec(d), gu.program(d), gu.opts(d))
            assert got.walks.equals(want.walks)
            assert got.metrics.total_steps == want.metrics.total_steps


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_run_digest_is_the_fold_of_the_reference_walks():
    """wfref_run_digest (the whole-run digest the full-size C4 / C5 parity tests
    compare) equals oracle.walk_digest over the walks the reference's
    run_sequential returns, block by block; one changed vertex or status moves it."""
    from oracle.oracle import walk_digest
    from paper_2107_11983_b200.host import (DeepWalkProgram, ExecOptions, MetaPathProgram,
                                            PprProgram, QuerySpec, WalkSet)
    rg = RefOracle().rmat(11, 16, seed=1, weighted=True, label_count=5)
    src = np.random.default_rng(3).integers(0, 2048, 3000, dtype=np.uint32)
    block = 700
    for prog, spec in [(DeepWalkProgram(40, True), QuerySpec.one_per_vertex()),
                       (PprProgram(0.2), QuerySpec.from_list(src)),
                       (MetaPathProgram([i % 5 for i in range(19)]), QuerySpec.one_per_vertex())]:
        opts = ExecOptions(seed=7)
        res = rg.run(spec, prog, opts)
        w, n = res.walks, len(res.walks)
        got, steps, _ = rg.run_digest(spec, prog, opts, block, threads=3)
        assert steps == res.metrics.total_steps and got.size == (n + block - 1) // block
        for b in range(got.size):
            a0, a1 = b * block, min(n, (b + 1) * block)
            v0, v1 = int(w.offsets[a0]), int(w.offsets[a1])
            sub = WalkSet(w.offsets[a0:a1 + 1] - w.offsets[a0], w.vertices[v0:v1].copy(),
                          w.status[a0:a1].copy())
            assert walk_digest(sub, a0, chunk=256) == int(got[b]) == walk_digest(sub, a0)
            if b == 0:
                sub.vertices[v1 - v0 - 1] ^= 1
                assert walk_digest(sub, a0) != int(got[b])
                sub.vertices[v1 - v0 - 1] ^= 1
                sub.status[0] ^= 1
                assert walk_digest(sub, a0) != int(got[b])
                assert walk_digest(sub, a0 + 1) != int(got[b])
