"""GRID text I/O (reference measures.py:138-216) against fixtures produced by
the live reference (tests/golden/make_grid_golden.py): parsed dims and masses
bit for bit, dump text byte for byte, and the same exception class, message,
line and token on malformed input.  CPU only."""

from __future__ import annotations

import io
import json
import os

import numpy as np
import pytest

import paper_2506_00976_b200 as G

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "grid_io.json")))


@pytest.mark.parametrize("case", CASES, ids=[f"c{i}" for i in range(len(CASES))])
def test_grid_io_matches_reference(case):
    text = case["text"]
    if case["ok"]:
        m = G.load_grid_measure(text)
        assert list(m.grid.dims) == case["dims"]
        assert m.mass.tobytes().hex() == case["mass"]
        assert G.dump_grid_measure(m) == case["dump"]
        # str, bytes and file objects parse alike
        for src in (text.encode("ascii"), io.StringIO(text), io.BytesIO(text.encode("ascii"))):
            assert G.load_grid_measure(src).mass.tobytes() == m.mass.tobytes()
    else:
        with pytest.raises(G.GridotError) as ei:
            G.load_grid_measure(text)
        exc = ei.value
        assert type(exc).__name__ == case["error"]
        assert str(exc) == case["message"]
        assert getattr(exc, "line", None) == case["line"]
        assert getattr(exc, "token", None) == case["token"]
        assert getattr(exc, "index", None) == case["index"]


def test_round_trip_bitwise():
    rng = np.random.default_rng(11)
    for dims in ((3, 5), (2, 3, 4), (9,)):
        m = G.GridMeasure(G.GridSpec(dims), rng.random(int(np.prod(dims))) * 1e-7)
        back = G.load_grid_measure(G.dump_grid_measure(m))
        assert back.grid.dims == m.grid.dims and back.mass.tobytes() == m.mass.tobytes()


def test_unreadable_source():
    with pytest.raises(TypeError):
        G.load_grid_measure(3.5)
