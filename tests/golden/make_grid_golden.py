"""GRID text-format fixtures from the LIVE reference (build container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_grid_golden.py

Runs the reference's ``load_grid_measure`` / ``dump_grid_measure``
(measures.py:138-216) on valid and malformed inputs and writes
``tests/golden/grid_io.json``: per case the parsed dims and mass bytes (hex)
and the reference's dump text, or the exception class with its line / token /
message.  The inputs are written out here (small hand-made strings and seeded
random masses), not taken from any dataset.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("GRIDOT_REF", "/root/reference/pkg/src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import gridot as G  # noqa: E402


def cases():
    rng = np.random.default_rng(20250601)
    out = [
        "2 2 2\n1 0 0 1\n", "1 3\n0.5 0.5\n0\n", "# comment\n\n2 2 2\n1 0\n\n0 1\n",
        "  # indented comment\n3 2 1 2\n1e-300 2.5E3\n 7 0.125 \n", "1 1\n1_000\n",
        "1 2\n  inf 1\n", "1 2\n-0.0 +3\n", "2 2 2\r\n1 0\r\n0 1\r\n", "1 2\n1\t2\n",
        "", "\n\n# only comments\n", "0 4\n1 1 1 1\n", "2 2\n1 1 1 1\n", "1 0\n", "1 x\n1\n",
        "1 4\n1 1 1\n", "1 2\n1 1 1\n", "1 2\n1 oops\n", "1 2\n1 nan\n", "1 2\n1 -inf\n",
        "2 2 2\n1 -1 0 1\n", "# note\n2 2 x\n1 1 1 1\n", "1 3\n0.5 0.5\nbogus\n",
        "x 2\n1 1\n", "2.0 2 2\n1 1 1 1\n", "1 -3\n1 1 1\n", "1 3\n1 2 -0.5\n",
    ]
    for dims in ((3, 5), (4, 3, 2), (7,), (16, 16)):
        m = rng.random(int(np.prod(dims)))
        m[rng.random(m.size) < 0.2] = 0.0
        m *= 10.0 ** rng.integers(-12, 12, m.size)
        out.append(G.dump_grid_measure(G.GridMeasure(G.GridSpec(dims), m)))
    return out


def main():
    rec = []
    for text in cases():
        r = {"text": text}
        try:
            m = G.load_grid_measure(text)
            r.update(ok=True, dims=list(m.grid.dims), mass=m.mass.tobytes().hex(),
                     dump=G.dump_grid_measure(m))
        except Exception as exc:  # recorded, compared by the tests
            r.update(ok=False, error=type(exc).__name__, message=str(exc),
                     line=getattr(exc, "line", None), token=getattr(exc, "token", None),
                     index=getattr(exc, "index", None))
        rec.append(r)
    with open(os.path.join(HERE, "grid_io.json"), "w") as fh:
        json.dump(rec, fh, indent=0)
    print(f"{len(rec)} cases, {sum(r['ok'] for r in rec)} valid")


if __name__ == "__main__":
    main()
