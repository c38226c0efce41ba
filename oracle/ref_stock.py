"""ORACLE / TEST INFRASTRUCTURE ONLY: the stock reference package as the CPU arm.

The reference (``gridot``, ``/root/reference/pkg/src/gridot``) is pure Python
(numpy, scipy, a numba simplex).  It cannot be imported from
``/root/reference`` on the GPU box, so ``stage()`` -- run by
``__graft_entry__.build()`` in the build container -- copies its modules
BYTE-IDENTICAL into ``oracle/_ref/gridot/`` (git-ignored, not gpurun-ignored:
it travels to the box like a built ``.so``), and ``load()`` imports it from
there only after checking every file against the SHA-256 manifest committed
here (``REF_SHA256``).  Nothing is edited, nothing is re-implemented: the CPU
arm of ``bench.py`` calls the reference's own four bound functions
(``quantized.py:172,199,288,487``) exactly as ``cli._dispatch`` does
(``cli.py:211-232``).

The product package never imports this module.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF_ROOT = os.path.join(HERE, "_ref")
REF_PKG = os.path.join(REF_ROOT, "gridot")
SOURCE = os.environ.get("GRIDOT_REF", "/root/reference/pkg/src")

# sha256 of /root/reference/pkg/src/gridot/*.py (the reference as surveyed)
REF_SHA256 = {
    "__init__.py": "333e335a9c7cbbb9558bbeaa03a99e412803a365e76e678377cbaa1d6ad0ad15",
    "_simplex.py": "88c816266e51208088ad9684409c86b0a92cae6f24ca242a4e181d7c423f4754",
    "cli.py": "ff777224de6ddef063eb7af9fc032b03810c7fb0c7e97317257a0d15376486cb",
    "costs.py": "33219b6a0a61d00d188b8b94fc6bf44be35d135979f6a7b6089a56baa1231867",
    "errors.py": "91f2dd28bd91bcf3c92935f3f0214b763f1f0ca20a8219436d5287389fd83b4e",
    "exact.py": "2635b81faa1a1bf702c32788765dc62c999d16ca05774bf064900713d18d0ec9",
    "measures.py": "09eed80ebfb68d8210540b6e7d695e61bf9c0d7e1d13347c36b4298bf331d55b",
    "quantized.py": "3a78b246efd42c58cb5a027bc382e0104e535626508436dfbbbee7ef7224d304",
    "reports.py": "00c4fba00a5845cc2f757ebff4356329f7aefa4b097e225159d9405c6797b373",
    "sinkhorn.py": "beab400bae3da24d16f9456fc0e178cef2c45c7b26ebdc503f24ee5e33a5bbe7",
}


class ReferenceUnavailable(RuntimeError):
    """The staged copy of the reference is missing or does not match the manifest."""


def _sha(path: str) -> str:
    with open(path, "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def verify(pkg: str = REF_PKG) -> None:
    """Every module present and byte-identical to the manifest."""
    for name, want in REF_SHA256.items():
        path = os.path.join(pkg, name)
        if not os.path.exists(path):
            raise ReferenceUnavailable(f"{path} missing (run __graft_entry__.build() where "
                                       f"{SOURCE} exists)")
        got = _sha(path)
        if got != want:
            raise ReferenceUnavailable(f"{path}: sha256 {got[:16]}... != manifest {want[:16]}...")


def stage() -> bool:
    """Copy the reference modules into oracle/_ref/gridot when the source tree is
    present (build container); returns whether a verified copy exists."""
    src = os.path.join(SOURCE, "gridot")
    if os.path.isdir(src):
        verify(src)
        os.makedirs(REF_PKG, exist_ok=True)
        for name in REF_SHA256:
            shutil.copyfile(os.path.join(src, name), os.path.join(REF_PKG, name))
    try:
        verify()
        return True
    except ReferenceUnavailable:
        return False


_gridot = None


def load():
    """Import the staged, checksum-verified reference package."""
    global _gridot
    if _gridot is not None:
        return _gridot
    verify()
    if not os.environ.get("NUMBA_CACHE_DIR"):
        # _simplex uses @njit(cache=True); the package dir must stay untouched
        os.environ["NUMBA_CACHE_DIR"] = os.path.join(tempfile.gettempdir(), "gdt_numba_cache")
    if "gridot" in sys.modules:
        mod = sys.modules["gridot"]
        if os.path.dirname(os.path.abspath(mod.__file__)) != REF_PKG:
            raise ReferenceUnavailable(f"another gridot is imported: {mod.__file__}")
    sys.path.insert(0, REF_ROOT)
    try:
        import gridot
    finally:
        sys.path.remove(REF_ROOT)
    if os.path.dirname(os.path.abspath(gridot.__file__)) != REF_PKG:
        raise ReferenceUnavailable(f"imported {gridot.__file__}, expected {REF_PKG}")
    _gridot = gridot
    return gridot


def warm_up() -> float:
    """JIT-compile (or load from the numba cache) the reference simplex on a tiny
    problem, untimed; returns the seconds it took."""
    import numpy as np

    G = load()
    t0 = time.perf_counter()
    grid = G.GridSpec((8, 8))
    rng = np.random.default_rng(0)
    a, b = rng.random(64) + 0.1, rng.random(64) + 0.1
    mu, nu = G.GridMeasure(grid, a / a.sum()), G.GridMeasure(grid, b / b.sum())
    for p in (1.0, 2.0):
        four_bounds(mu, nu, 4, p, None, 10_000)
    return time.perf_counter() - t0


def four_bounds(mu, nu, kappa, p, xi, max_iter):
    """The four QUANT_METHODS through the reference's own functions, in the
    order and with the arguments of ``cli._dispatch`` (cli.py:211-232)."""
    G = load()
    return {
        "weighted_cost": G.weighted_cost_upper_bound(mu, nu, kappa, p),
        "min_cost": G.min_cost_lower_bound(mu, nu, kappa, p),
        "primal_upscaling": G.primal_upscaling_upper_bound(mu, nu, kappa, p, xi=xi,
                                                           max_iter=max_iter),
        "dual_upscaling": G.dual_upscaling_lower_bound(mu, nu, kappa, p),
    }


def pair_bounds(cfg: int, pair: int, combos=None):
    """One seeded pair of a BASELINE config, every (kappa, p), all four bounds.

    Returns (seconds, {(kappa, p): {method: raw_value}})."""
    sys.path.insert(0, os.path.dirname(HERE))
    from paper_2506_00976_b200 import synthetic as S  # the shared seeded generator

    G = load()
    wl = S.WORKLOADS[cfg]
    combos = wl.combos if combos is None else combos
    mu_h, nu_h = S.measure(cfg, pair, 0), S.measure(cfg, pair, 1)
    t0 = time.perf_counter()
    grid = G.GridSpec(wl.dims)
    mu, nu = G.GridMeasure(grid, mu_h), G.GridMeasure(grid, nu_h)
    out = {}
    for k, p in combos:
        reps = four_bounds(mu, nu, int(k), float(p), wl.xi, wl.max_iter)
        out[(int(k), float(p))] = {m: r.raw_value for m, r in reps.items()}
    return time.perf_counter() - t0, out


if __name__ == "__main__":
    ok = stage()
    print(f"reference staged in {REF_PKG}: {'verified' if ok else 'UNAVAILABLE'}")
