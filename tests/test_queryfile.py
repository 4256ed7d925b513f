"""QuerySpec.from_file (walker.cpp:22-78) in the Python mirror: the
reference's own CLI test file (test_cli.cpp:184-196) and its error classes."""
import os
import re
import tempfile

import numpy as np
import pytest

from paper_2107_11983_b200 import abi
from paper_2107_11983_b200.host import QuerySpec


def _write(d, text):
    p = os.path.join(d, "q.txt")
    with open(p, "w") as f:
        f.write(text)
    return p


def test_reference_cli_query_file():
    with tempfile.TemporaryDirectory() as d:
        q = QuerySpec.from_file(_write(d, "# sources\n3 2\n7\n"))
        assert np.array_equal(q.sources, [3, 3, 7])
        assert q.count == 3


@pytest.mark.parametrize("text,msg", [
    ("1 2 3\n", "q.txt:1: too many columns"),
    ("\n\n-4\n", "q.txt:3: expected `vertex [count]`"),
    ("5 x\n", "q.txt:1: expected `vertex [count]`"),
    ("4294967296\n", "q.txt:1: vertex id out of range"),
    ("# only a comment\n\n", "q.txt: no queries"),
    ("7 0\n", "q.txt: no queries"),
])
def test_query_file_errors(text, msg):
    with tempfile.TemporaryDirectory() as d:
        with pytest.raises(abi.ParseError, match=re.escape(msg)):
            QuerySpec.from_file(_write(d, text))


def test_missing_query_file():
    with pytest.raises(abi.WalkforgeError, match="cannot open query file"):
        QuerySpec.from_file("/nonexistent/q.txt")


def test_comments_and_whitespace():
    with tempfile.TemporaryDirectory() as d:
        q = QuerySpec.from_file(_write(d, "  9\t3   # three from 9\n\n0\n"))
        assert np.array_equal(q.sources, [9, 9, 9, 0])
