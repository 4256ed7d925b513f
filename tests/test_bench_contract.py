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


def test_roofline_evidence_covers_every_config():
    """Every config's bench entry can carry BASELINE's measured-sector roofline
    (profiles/ncu_traffic.json, from committed ncu captures) and a note on what
    bounds its kernel."""
    sys.path.insert(0, ROOT)
    import bench
    for key in bench.CONFIGS:
        assert bench.ROOFLINE_NOTES.get(key), key
        block = bench.measured_sectors_block(key, 1e10, 6547.5)
        assert block is not None and block["bytes_per_move"] > 0, key
        assert 0 < block["frac"] and block["ceiling_steps_per_s"] > 0, key
