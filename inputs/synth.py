"""Seeded synthetic inputs for the LE-MPR gap-filling hot path.

This module is shared by the oracle tests, the GPU tests and bench.py. It holds
NONE of the method's arithmetic (no transform, energy, temperature or Metropolis
step): it only draws fields and masks, with the shapes and structure of the
paper's workloads (BASELINE.json configs).

Recipe:
- Field: Whittle–Matérn Gaussian random field on the torus via FFT, spectral density
  S(k) ∝ (kappa^2 + |k|^2)^-(nu+1) (2-D), unit variance.
- Heterogeneous variance: sigma(s) = exp(a*g(s)), g a standardised smooth field with
  correlation length L/8, a = ln(10)/2 so sigma spans ~100x (two regimes, as in the
  Walker-lake "near-constant vs highly variable domains").
- Optional skew: z <- exp(0.79*x) (skewness ~3.6 like Walker lake).
- Masks: ``mask != 0`` marks a known sample. Random gaps: exactly round(p*L^2) sites
  drawn by a permutation. Cloud gaps: the round(p*L^2) largest sites of a smooth
  field (nu=1.5, correlation length L/32), stable argsort.
- Seeds: field 2212, mask 1317, simulation 20221202.
"""
from __future__ import annotations

import numpy as np

SEED_FIELD = 2212
SEED_MASK = 1317
SEED_SIM = 20221202


def matern_field(Ly: int, Lx: int, nu: float = 1.5, corr_len: float = 16.0,
                 seed: int = SEED_FIELD) -> np.ndarray:
    """Unit-variance Whittle–Matérn field (float64) of shape (Ly, Lx)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    ky = np.fft.fftfreq(Ly) * 2.0 * np.pi
    kx = np.fft.rfftfreq(Lx) * 2.0 * np.pi
    kappa = 1.0 / float(corr_len)
    k2 = ky[:, None] ** 2 + kx[None, :] ** 2
    amp = (kappa * kappa + k2) ** (-(nu + 1.0) / 2.0)
    noise = rng.standard_normal((Ly, Lx))
    f = np.fft.irfft2(np.fft.rfft2(noise) * amp, s=(Ly, Lx))
    f -= f.mean()
    sd = f.std()
    return f / sd if sd > 0 else f


def heterogeneous_field(L: int, nu: float = 1.5, corr_len: float = 16.0,
                        spread: float = 100.0, skew: bool = False,
                        seed: int = SEED_FIELD, Lx: int | None = None) -> np.ndarray:
    """Field with spatially varying standard deviation; float32, shape (L, Lx or L)."""
    Ly, Lx = L, (Lx if Lx is not None else L)
    x = matern_field(Ly, Lx, nu=nu, corr_len=corr_len, seed=seed)
    g = matern_field(Ly, Lx, nu=1.5, corr_len=max(Ly, Lx) / 8.0, seed=seed + 1)
    a = np.log(np.sqrt(spread)) / 2.0
    z = np.exp(a * g) * x
    if skew:
        z = np.exp(0.79 * z / max(z.std(), 1e-30))
    return z.astype(np.float32)


def domain_wall_field(L: int, tile: int = 64, low: float = 0.1, high: float = 10.0, nu: float = 1.5,
                      corr_len: float = 8.0, seed: int = SEED_FIELD) -> np.ndarray:
    """A field with SHARP variance domain walls: unit-variance Matern x scaled by `high` on
    the tiles (tile x tile) of one checkerboard colour and by `low` on the others — the
    "domains of almost constant values as well as domains with large spatial fluctuations"
    of PAPER.md:100, with walls the smoothing of SST removes. float32."""
    x = matern_field(L, L, nu=nu, corr_len=corr_len, seed=seed)
    rr, cc = np.meshgrid(np.arange(L) // tile, np.arange(L) // tile, indexing="ij")
    sigma = np.where(((rr + cc) & 1) == 1, high, low)
    return (sigma * x).astype(np.float32)


def random_mask(Ly: int, Lx: int, p: float, seed: int = SEED_MASK) -> np.ndarray:
    """uint8 mask, 1 = known sample; exactly round(p*Ly*Lx) gaps (P = pL^2)."""
    n = Ly * Lx
    P = int(round(p * n))
    rng = np.random.Generator(np.random.PCG64(seed))
    m = np.ones(n, dtype=np.uint8)
    m[rng.permutation(n)[:P]] = 0
    return m.reshape(Ly, Lx)


def cloud_mask(Ly: int, Lx: int, p: float, seed: int = SEED_MASK) -> np.ndarray:
    """uint8 mask with clustered (cloud-like) gaps: the round(p*n) highest sites of a smooth field."""
    n = Ly * Lx
    P = int(round(p * n))
    f = matern_field(Ly, Lx, nu=1.5, corr_len=max(Ly, Lx) / 32.0, seed=seed).ravel()
    order = np.argsort(-f, kind="stable")
    m = np.ones(n, dtype=np.uint8)
    m[order[:P]] = 0
    return m.reshape(Ly, Lx)


def make_problem(L: int, p: float, gaps: str = "random", nu: float = 1.5,
                 corr_len: float = 16.0, seed_field: int = SEED_FIELD,
                 seed_mask: int = SEED_MASK, Lx: int | None = None):
    """Return (truth float32 (Ly,Lx), z float32 with NaN at gaps, mask uint8)."""
    Ly, Lx = L, (Lx if Lx is not None else L)
    truth = heterogeneous_field(Ly, nu=nu, corr_len=corr_len, seed=seed_field, Lx=Lx)
    if gaps == "random":
        mask = random_mask(Ly, Lx, p, seed=seed_mask)
    elif gaps == "cloud":
        mask = cloud_mask(Ly, Lx, p, seed=seed_mask)
    else:
        raise ValueError(f"unknown gap kind {gaps!r}")
    z = truth.copy()
    z[mask == 0] = np.nan
    return truth, z, mask


# BASELINE.json configs (the workloads the paper's sizes map to).
CONFIGS = {
    "C1": dict(L=64, p=0.5, gaps="random", nu=1.5, M=10, sweeps=30),
    "C2": dict(L=1024, p=0.33, gaps="random", nu=0.5, M=100, sweeps=30),
    "C3": dict(L=4096, p=0.7, gaps="cloud", nu=1.5, M=64, sweeps=30),
    "C4": dict(L=16384, p=0.5, gaps="random", nu=1.5, M=10, sweeps=30),
}
