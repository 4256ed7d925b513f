"""bench.py's reference arm runs on the host alone (no GPU): the JSON line the
driver parses carries the contract's keys.  (The GPU arm is exercised by the
driver on a B200.)"""
import json
import os
import subprocess
import sys

import pytest

from oracle.oracle import ref_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "config", "impl", "cpu_baseline", "e2e"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "steps/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1


def _fake_run(program, layout, stats=None, steps=None):
    return {"stats": stats or {}, "layout": layout, "step_attempts": steps}


def test_roofline_frac_recomputes_from_the_line():
    """roofline.frac = moves x S_alg (SURVEY 8(d), 76 B for ALIAS / NAIVE) /
    mean launch time / peak, recomputed from the block's own fields."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2107_11983_b200 import abi
    moves, ms, peak = 2_591_505_019, 61.3, 6534.5
    for key, layout in [("c5", abi.HAS_WIDE_ALIAS), ("c1", 0), ("c2", abi.HAS_ADJ)]:
        cfg = bench.CONFIGS[key]
        roof, sa = bench.roofline_block(key, cfg, _fake_run(cfg["program"], layout), moves, ms, peak, "measured")
        assert roof["bytes_per_move"] == 76.0
        want = moves * roof["bytes_per_move"] / (ms * 1e-3) / 1e9
        assert abs(roof["achieved"] - want) < 1e-6 * want
        assert abs(roof["frac"] - want / peak) < 1e-9
        assert abs(roof["layout"]["frac"] - moves * roof["layout"]["bytes_per_move"] / (ms * 1e-3) / 1e9 / peak) < 1e-9
        assert roof["note"]
    # instrumented reference counts for O-REJ and MetaPath
    cfg = bench.CONFIGS["c3"]
    roof, _ = bench.roofline_block("c3", cfg, _fake_run("node2vec", abi.HAS_ADJ,
                                   {"trials": 106, "probes": 50, "ref_probes": 982}), 100, 1.0, peak, "m")
    assert abs(roof["bytes_per_move"] - (1.25 + 1.06 + 9.82 + 0.125) * 32) < 1e-9
    cfg = bench.CONFIGS["c4"]
    roof, _ = bench.roofline_block("c4", cfg, _fake_run("metapath", abi.HAS_MP_SUCC,
                                   {"ref_label_sectors": 300}, steps=110), 100, 1.0, peak, "m")
    assert abs(roof["bytes_per_move"] - (1.25 * 1.1 + 3.0 + 1.125) * 32) < 1e-9


def test_stale_traffic_capture_is_not_reported(tmp_path, monkeypatch):
    """A capture stamped with other library sources is reported stale: no
    traffic, no measured-sector fraction."""
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setattr(bench, "ncu_traffic", lambda: {"configs": {"c5": {
        "bytes": 3.4e11, "moves": 1000, "src_sha": "0" * 16}}})
    t, bpm, stamp = bench.traffic_for("c5", 1000)
    assert t is None and bpm is None and stamp["stale"] is True
    monkeypatch.setattr(bench, "ncu_traffic", lambda: {"configs": {"c5": {
        "bytes": 3.4e11, "moves": 1000, "src_sha": bench.source_sha()}}})
    t, bpm, stamp = bench.traffic_for("c5", 1000)
    assert t == 3.4e11 and bpm == 3.4e8 and stamp["stale"] is False
