"""The reference's "cli" suite (/root/reference/proj/tests/test_cli.cpp:57-259)
re-expressed, case by case under the reference's case names, against this
repo's CLI (paper_2107_11983_b200/walkforge_b200: same sub-commands and flags):
a black box over the binary, stdout and stderr merged, exactly as the
reference drives its own."""
import os
import struct
import subprocess

import pytest

from paper_2107_11983_b200 import engine as E

pytestmark = pytest.mark.gpu

CLI = os.path.join(os.path.dirname(E.LIB_PATH), "walkforge_b200")


def run_cli(*args):
    p = subprocess.run([CLI, *args], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, timeout=300)
    return p.returncode, p.stdout


def ring_edge_list():
    """12-vertex directed graph with no dead ends: a ring with chords."""
    return "".join(f"{v} {(v + 1) % 12}\n{v} {(v + 5) % 12}\n" for v in range(12))


@pytest.fixture
def d(tmp_path):
    (tmp_path / "g.txt").write_text(ring_edge_list())
    return tmp_path


def test_convert_then_run_produces_one_well_formed_record_per_query(d):  # :58
    rc, out = run_cli("convert", str(d / "g.txt"), str(d / "g.wfg"))
    assert rc == 0 and "V=12" in out and "E=24" in out
    rc, out = run_cli("run", str(d / "g.wfg"), "-o", str(d / "w.out"), "--algorithm", "deepwalk", "--length", "7",
                      "--seed", "3", "--threads", "2")
    assert rc == 0 and "total_steps 72" in out, out
    lines = (d / "w.out").read_text().splitlines()
    assert len(lines) == 12
    for i, line in enumerate(lines):
        qid, status, rest = line.split("\t")
        path = [int(x) for x in rest.split()]
        assert int(qid) == i and status == "complete" and len(path) == 7 and path[0] == i


def test_a_fixed_seed_reproduces_the_output_bytes_exactly(d):  # :91
    run_cli("convert", str(d / "g.txt"), str(d / "g.wfg"))
    base = ["run", str(d / "g.wfg"), "--algorithm", "ppr", "--termination", "0.3", "--queries", "source:0:400"]
    assert run_cli(*base, "--seed", "11", "-o", str(d / "a.out"))[0] == 0
    assert run_cli(*base, "--seed", "11", "-o", str(d / "b.out"))[0] == 0
    a = (d / "a.out").read_bytes()
    assert a and a == (d / "b.out").read_bytes()
    assert run_cli(*base, "--seed", "12", "-o", str(d / "c.out"))[0] == 0
    assert a != (d / "c.out").read_bytes()


def test_interleaving_does_not_change_the_walks(d):  # :112
    run_cli("convert", str(d / "g.txt"), str(d / "g.wfg"), "--weights", "random", "--seed", "4")
    base = ["run", str(d / "g.wfg"), "--algorithm", "node2vec", "--weighted", "--length", "9", "--seed", "6", "-o"]
    assert run_cli(*base, str(d / "on.out"), "--interleave", "on", "-k", "16", "--k-prime", "8")[0] == 0
    assert run_cli(*base, str(d / "off.out"), "--interleave", "off")[0] == 0
    on = (d / "on.out").read_bytes()
    assert on and on == (d / "off.out").read_bytes()


def test_binary_output_lays_out_records_back_to_back(d):  # :128
    run_cli("convert", str(d / "g.txt"), str(d / "g.wfg"))
    assert run_cli("run", str(d / "g.wfg"), "--algorithm", "deepwalk", "--length", "5", "--seed", "2",
                   "--binary-output", "-o", str(d / "w.bin"))[0] == 0
    data = (d / "w.bin").read_bytes()
    pos, expected_qid = 0, 0
    while pos < len(data):
        assert pos + 13 <= len(data)
        qid, status, length = struct.unpack_from("<QBI", data, pos)
        assert qid == expected_qid and status == 0 and length == 5
        assert pos + 13 + 4 * length <= len(data)
        assert struct.unpack_from("<I", data, pos + 13)[0] == qid
        pos += 13 + 4 * length
        expected_qid += 1
    assert expected_qid == 12


def test_label_constrained_runs_stop_where_the_schema_does(d):  # :159
    run_cli("convert", str(d / "g.txt"), str(d / "g.wfg"), "--labels", "random", "--label-count", "3", "--seed", "9")
    rc, out = run_cli("run", str(d / "g.wfg"), "--algorithm", "metapath", "--schema", "0,1,2", "--seed", "1", "-o",
                      str(d / "w.out"))
    assert rc == 0, out
    lines = (d / "w.out").read_text().splitlines()
    assert len(lines) == 12
    for line in lines:
        complete, dead = "\tcomplete\t" in line, "\tdead_end\t" in line
        assert complete or dead
        if complete:
            assert len(line.rsplit("\t", 1)[1].split()) == 4


def test_query_files_drive_the_sources(d):  # :184
    run_cli("convert", str(d / "g.txt"), str(d / "g.wfg"))
    (d / "q.txt").write_text("# sources\n3 2\n7\n")
    rc, out = run_cli("run", str(d / "g.wfg"), "--algorithm", "deepwalk", "--length", "4", "--queries",
                      "file:" + str(d / "q.txt"), "-o", str(d / "w.out"))
    assert rc == 0, out
    lines = (d / "w.out").read_text().splitlines()
    assert len(lines) == 3
    assert lines[0].startswith("0\tcomplete\t3 ") and lines[1].startswith("1\tcomplete\t3 ")
    assert lines[2].startswith("2\tcomplete\t7 ")


def test_the_ring_sweep_reports_every_power_of_two_and_a_recommendation(d):  # :200
    """On the device k / k' are launch hints (resident walkers replace the rings): the
    sweep runs the reference's probe at every ring size and prints the reference's
    report format, so the curve is flat; the launch tuner's choice follows it."""
    rc, out = run_cli("tune", str(d / "g.txt"), "--budget", "60", "--seed", "5")
    assert rc == 0, out
    assert "task ring sweep" in out and "search ring sweep" in out and "recommended k=" in out
    lines = out.splitlines()
    assert any(ln.startswith("1\t") for ln in lines)
    ks = [int(ln.split("\t")[0]) for ln in lines[:lines.index(next(x for x in lines if x.startswith("search ring")))]
          if ln[:1].isdigit()]
    assert ks == [1 << i for i in range(11)]
    assert all(float(ln.split("\t")[1]) > 0 for ln in lines if ln[:1].isdigit())
    assert "device launch tuner:" in out and "blocks/SM" in out


def test_failures_exit_non_zero_with_a_pointed_message(d):  # :215
    # malformed edge list names the line
    (d / "bad.txt").write_text("0 1\n0 x\n")
    rc, out = run_cli("run", str(d / "bad.txt"))
    assert rc != 0 and "bad.txt:2" in out
    # missing graph file
    rc, out = run_cli("run", str(d / "nope.wfg"))
    assert rc != 0 and "error:" in out
    # metapath without labels
    run_cli("convert", str(d / "g.txt"), str(d / "g.wfg"))
    rc, out = run_cli("run", str(d / "g.wfg"), "--algorithm", "metapath", "--schema", "0")
    assert rc != 0 and "error:" in out
    # naive sampling with a weighted program
    rc, out = run_cli("run", str(d / "g.txt"), "--algorithm", "deepwalk", "--sampler", "naive", "-o",
                      str(d / "w.out"))
    assert rc != 0 and "error:" in out
    # unknown flag; no subcommand
    assert run_cli("run", "g.wfg", "--frobnicate")[0] != 0
    assert run_cli()[0] != 0
