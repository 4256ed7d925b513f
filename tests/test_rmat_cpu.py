"""The two CPU restatements of the synthetic R-MAT generator (numpy and C,
oracle/) agree bit for bit; the device generator is checked against them in
tests/test_engine_gpu.py."""
import numpy as np
import pytest

from oracle.oracle import PortOracle
from oracle.rmat_ref import rmat_csr


@pytest.mark.parametrize("scale,weighted,labels", [(5, False, 0), (9, True, 5), (11, True, 3)])
def test_c_rmat_matches_numpy_rmat(scale, weighted, labels):
    g = PortOracle().rmat(scale, 16, seed=7, weighted=weighted, label_count=labels, threads=3)
    off, nbr, w, lab = rmat_csr(scale, 16, seed=7, weighted=weighted, label_count=labels)
    assert np.array_equal(g.offsets, off)
    assert np.array_equal(g.neighbors, nbr)
    if weighted:
        assert np.array_equal(g.weights, w)
    if labels:
        assert np.array_equal(g.labels, lab)


def test_rmat_graph_properties():
    g = PortOracle().rmat(12, 16, seed=1)
    V = g.vertex_count
    src = np.repeat(np.arange(V), np.diff(g.offsets).astype(np.int64))
    assert not np.any(src == g.neighbors)  # no self-loops
    for v in range(0, V, 97):  # sorted, deduplicated adjacency
        ns = g.neighbors_of(v)
        assert np.all(ns[1:] > ns[:-1])
    # symmetric
    fwd = set(zip(src.tolist(), g.neighbors.tolist()))
    assert all((d, s) in fwd for s, d in list(fwd)[:5000])
