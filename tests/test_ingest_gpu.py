"""Graph ingest (SURVEY §8 f row 2) against the reference: the text edge-list
loader (load_edge_list, graph.cpp:307-453) and WFG1 binary files
(write_binary / read_binary, graph.cpp:190-277)."""
import os
import tempfile

import numpy as np
import pytest

from oracle.oracle import RefOracle, ref_available
from paper_2107_11983_b200 import abi
from paper_2107_11983_b200 import engine as E
from paper_2107_11983_b200.host import DeepWalkProgram, ExecOptions, Node2VecProgram, QuerySpec

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]


def random_edge_list(path, seed, m=3000, sparse=True, with_w=True, with_l=True):
    rng = np.random.default_rng(seed)
    pool = (rng.integers(0, 2 ** 40, 400) if sparse else np.arange(400)).astype(np.uint64)
    lines = ["# synthetic edge list", ""]
    for i in range(m):
        s, d = pool[rng.integers(0, 400)], pool[rng.integers(0, 400)]
        if i % 97 == 0:
            d = s  # self-loops survive (no dedup in the reference loader)
        cols = [str(s), str(d)]
        if with_w:
            cols.append(rng.choice(["2.5", "0.125", "3", "1e0", "7.75", "0", "4.0625"]))
        if with_l:
            cols.append(str(int(rng.integers(0, 5))))
        sep = "\t" if i % 5 == 0 else " "
        line = sep.join(cols)
        if i % 11 == 0:
            line += "   # trailing comment"
        lines.append(line)
        if i % 13 == 0:
            lines.append(line)  # duplicate edges survive too
    open(path, "w").write("\n".join(lines) + "\n")


def same_graph(dg, rg, ids_ref=None):
    """The same CSR, labels and weights: f64 weights (e.g. synthetic_weight,
    graph.cpp:279-282) come back as the same doubles."""
    h = dg.download()
    off, nbr, w, lab = rg.export()
    assert np.array_equal(h.offsets, off)
    assert np.array_equal(h.neighbors, nbr)
    assert (h.weights is None) == (w is None)
    if w is not None:
        assert np.array_equal(h.weights.astype(np.float64), w)
    assert (h.labels is None) == (lab is None)
    if lab is not None:
        assert np.array_equal(h.labels.astype(np.uint32), lab)
    if ids_ref is not None:
        assert np.array_equal(dg.original_ids(), ids_ref)


@pytest.mark.parametrize("undirected", [False, True])
@pytest.mark.parametrize("weights,labels", [(0, 0), (1, 1), (2, 2), (1, 2), (2, 0)])
def test_edge_list_loader_matches_reference(undirected, weights, labels):
    ref = RefOracle()
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.txt")
        random_edge_list(p, seed=weights * 7 + labels + int(undirected))
        rg, ids = ref.load_edge_list(p, undirected, weights, labels, 5, seed=11)
        dg = E.DeviceGraph.load_edge_list(p, undirected, weights, labels, 5, seed=11)
        same_graph(dg, rg, ids)
        # walks on the loaded graphs agree too (ingest -> run end to end)
        prog = DeepWalkProgram(12, weights != 0) if weights else Node2VecProgram(2.0, 0.5, 12, False)
        want = rg.run(QuerySpec.one_per_vertex(), prog, ExecOptions(seed=3))
        got = E.run_sequential(dg, QuerySpec.one_per_vertex(), prog, ExecOptions(seed=3))
        assert got.walks.equals(want.walks)


@pytest.mark.parametrize("text,err", [
    ("1\n", abi.ParseError),
    ("1 2 3 4 5\n", abi.ParseError),
    ("a b\n", abi.ParseError),
    ("-1 2\n", abi.ParseError),
    ("# nothing\n\n", abi.ParseError),
])
def test_edge_list_parse_errors(text, err):
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "bad.txt")
        open(p, "w").write(text)
        with pytest.raises(err):
            RefOracle().load_edge_list(p)
        with pytest.raises(err):
            E.DeviceGraph.load_edge_list(p)


@pytest.mark.parametrize("text,wmode", [("0 1\n1 2 x\n", 1), ("0 1 1.5\n1 2 -2\n", 1),
                                        ("0 1 2.5\n1 2\n", 1), ("0 1 2.5\n", 0)])
def test_edge_list_weight_column_errors(text, wmode):
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "w.txt")
        open(p, "w").write(text)
        try:
            RefOracle().load_edge_list(p, weights=wmode)
            ref_ok = True
        except abi.WalkforgeError as e:
            ref_ok, ref_err = False, type(e)
        if ref_ok:
            E.DeviceGraph.load_edge_list(p, weights=wmode)
        else:
            with pytest.raises(ref_err):
                E.DeviceGraph.load_edge_list(p, weights=wmode)


def test_wfg1_round_trip_is_byte_identical():
    ref = RefOracle()
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.txt")
        random_edge_list(p, seed=5)
        rg, _ = ref.load_edge_list(p, True, 1, 1)
        dg = E.DeviceGraph.load_edge_list(p, True, 1, 1)
        a, b = os.path.join(d, "ref.wfg"), os.path.join(d, "ours.wfg")
        rg.write_binary(a)
        dg.write_wfg1(b)
        assert open(a, "rb").read() == open(b, "rb").read()
        back = E.DeviceGraph.read_wfg1(a)
        same_graph(back, ref.read_binary(b))
        # an R-MAT graph (no labels) too
        g2 = E.DeviceGraph.rmat(10, 8, seed=2, weighted=True)
        c = os.path.join(d, "rmat.wfg")
        g2.write_wfg1(c)
        same_graph(E.DeviceGraph.read_wfg1(c), ref.read_binary(c))


def test_wfg1_format_errors():
    with tempfile.TemporaryDirectory() as d:
        good = os.path.join(d, "g.wfg")
        E.DeviceGraph.rmat(6, 4, seed=1).write_wfg1(good)
        data = open(good, "rb").read()
        for name, blob in [("magic", b"XFG1" + data[4:]), ("trunc", data[:-3]),
                           ("trail", data + b"\0"), ("flags", data[:20] + b"\x08" + data[21:])]:
            p = os.path.join(d, name)
            open(p, "wb").write(blob)
            with pytest.raises(abi.FormatError):
                RefOracle().read_binary(p)
            with pytest.raises(abi.FormatError):
                E.DeviceGraph.read_wfg1(p)
        with pytest.raises(abi.IoError):
            E.DeviceGraph.read_wfg1(os.path.join(d, "missing.wfg"))


def test_randomised_edge_list_ingest_sample():
    """tools/fuzz_ingest.py: random text edge lists (sparse 64-bit ids, comments,
    blanks, CRLF, number formats, a malformed line in a third of them) through
    the device loader and the reference's load_edge_list: the same error class
    and message, or the same CSR, attributes, original ids and WFG1 bytes.  A
    sample here; profiles/r02_fuzz_ingest.log holds the 16 k-case runs."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_ingest.py"), "--cases", "300",
                        "--seed", "9"], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "300 cases (seed 9), 0 differing" in p.stdout, p.stdout[-3000:] + p.stderr[-2000:]
