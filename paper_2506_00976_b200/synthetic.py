"""Seeded synthetic measure pairs for the five BASELINE.json configurations.

The reference measures its bounds on DOTmark / EMDB data that is not present
here; these generators stand in for it with the shapes, sizes and value
distributions BASELINE.json names.  Every measure
is generated in float64 on the host, laid out axis-1-fastest (``ravel("F")``
of an array indexed ``[x1, x2(, x3)]``, the flat order of
``pkg/src/gridot/measures.py:3-6``) and normalised to total mass 1 like
``normalize`` (``measures.py:228-233``).

Seeds follow ``cli.bench_run`` (``pkg/src/gridot/cli.py:288-291``):
``np.random.default_rng([BASE_SEED, cfg_id, pair_idx, side])`` with side 0 =
mu, 1 = nu.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BASE_SEED = 2506_00976


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json configuration (configs[cfg_id - 1])."""

    cfg_id: int
    dims: tuple
    pairs: int
    combos: tuple          # ((kappa, p), ...)
    precision: str         # "fp64" | "fp32"
    xi: float | None       # None -> reference default 1e-9 * |supports|
    max_iter: int
    kind: str


WORKLOADS = {
    1: Workload(1, (32, 32), 1, ((4, 2.0),), "fp64", 0.0, 50, "gaussians3"),
    2: Workload(2, (64, 64), 45, ((4, 2.0),), "fp32", 0.0, 100, "white_noise"),
    3: Workload(3, (128, 128), 45, ((4, 1.0), (4, 2.0), (8, 1.0), (8, 2.0)),
                "fp32", None, 10_000, "smooth_field"),
    4: Workload(4, (256, 256), 360, ((8, 2.0),), "fp32", 0.0, 200, "cauchy"),
    5: Workload(5, (32, 32, 32), 64, ((4, 2.0),), "fp64", None, 10_000,
                "gaussians5_aniso"),
}


def _coords(dims):
    idx = np.unravel_index(np.arange(int(np.prod(dims))), dims, order="F")
    return np.stack(idx, axis=1).astype(np.float64) + 1.0


def _normalise(x):
    x = np.asarray(x, dtype=np.float64)
    return x / float(np.sum(x))


def _gaussians_iso(rng, dims, count, sig_lo, sig_hi):
    X = _coords(dims)
    d = len(dims)
    w = rng.dirichlet(np.ones(count))
    dens = np.zeros(X.shape[0])
    for i in range(count):
        c = rng.uniform(1.0, dims[0], size=d)
        s = rng.uniform(sig_lo, sig_hi)
        sq = np.sum((X - c[None, :]) ** 2, axis=1)
        dens += w[i] * np.exp(-sq / (2.0 * s * s)) / (2.0 * np.pi * s * s) ** (d / 2.0)
    return _normalise(dens + 1e-6)


def _gaussians_aniso(rng, dims, count, s_lo, s_hi):
    X = _coords(dims)
    d = len(dims)
    w = rng.dirichlet(np.ones(count))
    dens = np.zeros(X.shape[0])
    for i in range(count):
        c = rng.uniform(1.0, dims[0], size=d)
        s = rng.uniform(s_lo, s_hi, size=d)
        q, r = np.linalg.qr(rng.standard_normal((d, d)))
        q = q * np.sign(np.diag(r))[None, :]          # Haar-distributed rotation
        cov = q @ np.diag(s * s) @ q.T
        prec = np.linalg.inv(cov)
        df = X - c[None, :]
        quad = np.einsum("ni,ij,nj->n", df, prec, df)
        norm = 1.0 / np.sqrt((2.0 * np.pi) ** d * np.linalg.det(cov))
        dens += w[i] * norm * np.exp(-0.5 * quad)
    return _normalise(dens + 1e-6)


def _smooth_field(rng, dims, sigma=8.0):
    z = rng.standard_normal(dims)
    # circular convolution with a Gaussian of std sigma pixels, via FFT
    kern = np.ones(dims)
    for a, n in enumerate(dims):
        k = np.arange(n)
        k = np.minimum(k, n - k).astype(np.float64)
        g = np.exp(-0.5 * (k / sigma) ** 2)
        g /= g.sum()
        shape = [1] * len(dims)
        shape[a] = n
        kern = kern * g.reshape(shape)
    field = np.real(np.fft.ifftn(np.fft.fftn(z) * np.fft.fftn(kern)))
    field = (field - field.mean()) / field.std()
    return _normalise(np.exp(field).ravel(order="F"))


def _cauchy(rng, dims):
    X = _coords(dims)
    c = rng.uniform(1.0, dims[0], size=len(dims))
    gam = rng.uniform(5.0, 40.0)
    sq = np.sum((X - c[None, :]) ** 2, axis=1)
    return _normalise((1.0 + sq / (gam * gam)) ** -1.5)


def measure(cfg_id: int, pair_idx: int, side: int, seed: int = BASE_SEED) -> np.ndarray:
    """Flat float64 masses of one side of one pair of configuration cfg_id."""
    wl = WORKLOADS[cfg_id]
    rng = np.random.default_rng([seed, cfg_id, pair_idx, side])
    if wl.kind == "gaussians3":
        return _gaussians_iso(rng, wl.dims, 3, 1.5, 6.0)
    if wl.kind == "white_noise":
        return _normalise(rng.random(int(np.prod(wl.dims))))
    if wl.kind == "smooth_field":
        return _smooth_field(rng, wl.dims)
    if wl.kind == "cauchy":
        return _cauchy(rng, wl.dims)
    if wl.kind == "gaussians5_aniso":
        return _gaussians_aniso(rng, wl.dims, 5, 2.0, 8.0)
    raise ValueError(wl.kind)


def batch(cfg_id: int, pair_lo: int, pair_hi: int, seed: int = BASE_SEED):
    """(mu, nu) float64 arrays of shape [pairs, cells] for pairs [lo, hi)."""
    mus = np.stack([measure(cfg_id, i, 0, seed) for i in range(pair_lo, pair_hi)])
    nus = np.stack([measure(cfg_id, i, 1, seed) for i in range(pair_lo, pair_hi)])
    return mus, nus
