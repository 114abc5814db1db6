"""Seeded synthetic inputs shaped like the paper's workloads (shared by tests,
bench.py and smoke()).

This module holds NONE of the method's arithmetic: it never evaluates the
Matérn correlation, a variance matrix, a factorisation or a likelihood.  The
spatial field in the response is simulated with random Fourier features drawn
from the Matérn spectral measure (a Student-t mixture of Gaussians), which is a
different computation from anything on the hot path.

Recipe:
  * sites: the paper's simulation-study density, 224 sites on a 9 km × 9 km
    square, so side = 9 km·sqrt(n/224); uniform with a minimum
    separation of 0.25 × the mean spacing.  C2 is "villages-shaped" after the
    Loaloa coordinates (190 clustered villages, φX = 50 km): 25 parent
    centres uniform on 600 km, children N(parent, (9 km)²), min separation 100 m.
  * covariates: intercept, X1 = x/1e4 (villages: x/1e5), X2 = X1²,
    then sin(2πx/L), cos(2πy/L) for p = 4, 5.
  * response: y' = Xβ + U + ε, β = (5, 1, 1, 0.5, −0.5)[:p],
    U Matérn with σ² = 1, κ = 2, φX = 1000 m (villages 50 km), φR = 2,
    φA = 0.2 (isotropic configs φR = 1), τ = 0.8; then y = (1 + λ0 y')^{1/λ0}
    with λ0 = 0.5 (the Swiss λ̂); ε is redrawn where 1 + λ0 y' ≤ 0.
  * parameter points ("representative-like", P:229-238 internal coordinates):
    γ1 ~ N(γ1⁰, 0.4²), log κ ~ N(log 2, 0.6²) clipped to [log 0.2, log 20],
    ν = 0.8 + N(0, 0.25²), ν² = max(ν, 0.1)²  (parity floor ν² ≥ 0.01),
    (γ2, γ3) ~ N(truth, 0.3² I) (isotropic: φR = 1, φA = 0), plus a 20 %
    κ-fixed share over κ ∈ {0.5, 0.9, 10, 20, 100}.
  * λ grid: M equally spaced values in [0.2, 0.8].
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

SEED_BASE = 230504318


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    p: int
    K: int
    M: int
    iso: bool
    layout: str  # "uniform" | "villages"
    desc: str


# BASELINE.json configs[0..4]; M for C3/C4 is not stated there -> 5.
CONFIGS = {
    "C1": Config("C1", 100, 2, 16, 3, True, "uniform",
                 "isotropic Matérn, n=100, p=2, 16 points × 3 λ"),
    "C2": Config("C2", 200, 3, 1000, 5, False, "villages",
                 "anisotropic Matérn, n=200 villages-shaped, p=3, 1,000 points × 5 λ"),
    "C3": Config("C3", 1000, 4, 10000, 5, False, "uniform",
                 "anisotropic Matérn, n=1,000, p=4, 10,000 points × 5 λ"),
    "C4": Config("C4", 2000, 5, 20000, 5, False, "uniform",
                 "anisotropic Matérn, n=2,000, p=5, 20,000 points × 5 λ (headline)"),
    "C5": Config("C5", 5000, 3, 4000, 10, True, "uniform",
                 "isotropic Matérn, n=5,000, p=3, 4,000 points × 10 λ (stress)"),
}

TRUTH = dict(kappa=2.0, phiR=2.0, phiA=0.2, sigma2=1.0, tau=0.8)
KAPPA_FIXED = (0.5, 0.9, 10.0, 20.0, 100.0)
LAMBDA0 = 0.5


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _truth_phiX(cfg: Config) -> float:
    return 50_000.0 if cfg.layout == "villages" else 1000.0


def _sites(cfg: Config, rng: np.random.Generator) -> np.ndarray:
    n = cfg.n
    if cfg.layout == "villages":
        side, dmin = 600_000.0, 100.0
        parents = rng.uniform(0.0, side, size=(25, 2))
    else:
        side = 9000.0 * math.sqrt(n / 224.0)
        dmin = 0.25 * side / math.sqrt(n)
    cell = dmin
    grid: dict[tuple[int, int], list[int]] = {}
    pts = np.empty((n, 2))
    k = 0
    while k < n:
        if cfg.layout == "villages":
            c = parents[rng.integers(0, 25)]
            cand = c + rng.normal(0.0, 9000.0, size=2)
        else:
            cand = rng.uniform(0.0, side, size=2)
        gx, gy = int(math.floor(cand[0] / cell)), int(math.floor(cand[1] / cell))
        ok = True
        for dx in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for j in grid.get((gx + dx, gy + dy), ()):
                    if (pts[j, 0] - cand[0]) ** 2 + (pts[j, 1] - cand[1]) ** 2 < dmin * dmin:
                        ok = False
                        break
                if not ok:
                    break
            if not ok:
                break
        if ok:
            pts[k] = cand
            grid.setdefault((gx, gy), []).append(k)
            k += 1
    return pts


def _covariates(cfg: Config, coords: np.ndarray) -> np.ndarray:
    n, p = cfg.n, cfg.p
    scale = 1e5 if cfg.layout == "villages" else 1e4
    L = float(np.ptp(coords[:, 0])) or 1.0
    x1 = coords[:, 0] / scale
    cols = [np.ones(n), x1, x1 * x1,
            np.sin(2 * math.pi * coords[:, 0] / L), np.cos(2 * math.pi * coords[:, 1] / L)]
    return np.stack(cols[:p], axis=1)


def _field_rff(coords, kappa, phiX, phiR, phiA, rng, J=2000) -> np.ndarray:
    """Gaussian field with Matérn spectral measure via random Fourier features.

    Spectral measure of a Matérn with argument sqrt(8κ)·|u| in 2-D is a
    Student-t: ω = α Z / sqrt(2 G), Z ~ N(0, I2), G ~ Gamma(κ, 1), α = sqrt(8κ),
    applied to u = diag(1/φX, 1/φY) Rot(φA) s.
    """
    phiY = phiX / phiR
    c, s = math.cos(phiA), math.sin(phiA)
    u = np.stack([(c * coords[:, 0] - s * coords[:, 1]) / phiX,
                  (s * coords[:, 0] + c * coords[:, 1]) / phiY], axis=1)
    alpha = math.sqrt(8.0 * kappa)
    Z = rng.normal(size=(J, 2))
    G = rng.gamma(kappa, 1.0, size=J)
    W = alpha * Z / np.sqrt(2.0 * G)[:, None]
    b = rng.uniform(0.0, 2 * math.pi, size=J)
    return math.sqrt(2.0 / J) * np.cos(u @ W.T + b).sum(axis=1)


def make_dataset(cfg: Config | str, seed: int | None = None):
    """Returns (coords n×2, y n (>0), X n×p) for a config, seeded."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    idx = list(CONFIGS).index(cfg.name) if cfg.name in CONFIGS else 0
    rng = _rng(SEED_BASE + idx if seed is None else seed)
    coords = _sites(cfg, rng)
    X = _covariates(cfg, coords)
    beta = np.array([5.0, 1.0, 1.0, 0.5, -0.5])[: cfg.p]
    phiR = 1.0 if cfg.iso else TRUTH["phiR"]
    phiA = 0.0 if cfg.iso else TRUTH["phiA"]
    U = math.sqrt(TRUTH["sigma2"]) * _field_rff(coords, TRUTH["kappa"], _truth_phiX(cfg), phiR,
                                                phiA, rng)
    mean = X @ beta + U
    eps = rng.normal(0.0, TRUTH["tau"], size=cfg.n)
    for _ in range(100):
        bad = 1.0 + LAMBDA0 * (mean + eps) <= 0.0
        if not bad.any():
            break
        eps[bad] = rng.normal(0.0, TRUTH["tau"], size=int(bad.sum()))
    ystar = mean + eps
    y = (1.0 + LAMBDA0 * ystar) ** (1.0 / LAMBDA0)
    return coords, y, X


def internal_to_natural(g1, logk, nu, g2, g3):
    """Internal ω' = (γ1, log κ, ν, γ2, γ3) -> natural (φX, κ, ν², φR, φA).

    φR = 1 + γ2² + γ3², φA = atan2(γ3, γ2)/2, φX φY = e^{γ1}, φY = φX/φR.
    """
    phiR = 1.0 + g2 * g2 + g3 * g3
    phiA = 0.5 * np.arctan2(g3, g2)
    phiX = np.sqrt(np.exp(g1) * phiR)
    return np.stack([phiX, np.exp(logk), nu * nu, phiR, phiA], axis=-1)


def make_params(cfg: Config | str, K: int | None = None, seed: int | None = None,
                kappa_fixed_share: float = 0.2) -> np.ndarray:
    """K×5 parameter points {φX, κ, ν², φR, φA}, seeded."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    K = cfg.K if K is None else K
    idx = list(CONFIGS).index(cfg.name) if cfg.name in CONFIGS else 0
    rng = _rng((SEED_BASE + 1000 + idx) if seed is None else seed)
    phiX0 = _truth_phiX(cfg)
    phiR0 = 1.0 if cfg.iso else TRUTH["phiR"]
    g1_0 = math.log(phiX0) + math.log(phiX0 / phiR0)
    g1 = rng.normal(g1_0, 0.4, size=K)
    logk = np.clip(rng.normal(math.log(2.0), 0.6, size=K), math.log(0.2), math.log(20.0))
    nu = np.maximum(0.8 + rng.normal(0.0, 0.25, size=K), 0.1)
    if cfg.iso:
        g2 = np.zeros(K)
        g3 = np.zeros(K)
    else:
        r0 = math.sqrt(phiR0 - 1.0)
        g2 = rng.normal(r0 * math.cos(2 * TRUTH["phiA"]), 0.3, size=K)
        g3 = rng.normal(r0 * math.sin(2 * TRUTH["phiA"]), 0.3, size=K)
    nfix = int(round(kappa_fixed_share * K))
    sel = rng.permutation(K)[:nfix]
    logk[sel] = np.log(np.array(KAPPA_FIXED)[np.arange(nfix) % len(KAPPA_FIXED)])
    P = internal_to_natural(g1, logk, nu, g2, g3)
    if cfg.iso:
        P[:, 3] = 1.0
        P[:, 4] = 0.0
    return np.ascontiguousarray(P)


def make_stress_params(cfg: Config | str, K: int, seed: int = SEED_BASE + 77) -> np.ndarray:
    """Stress set: nugget-repaired points (ν² = 0 for half) and κ ∈ {10, 20}."""
    P = make_params(cfg, K, seed=seed, kappa_fixed_share=0.0)
    P[::2, 2] = 0.0
    P[1::4, 1] = 10.0
    P[3::4, 1] = 20.0
    return P


def make_lambdas(M: int) -> np.ndarray:
    return np.linspace(0.2, 0.8, M) if M > 1 else np.array([0.5])


def make_inputs(name: str, K: int | None = None):
    cfg = CONFIGS[name]
    coords, y, X = make_dataset(cfg)
    params = make_params(cfg, K)
    lambdas = make_lambdas(cfg.M)
    return coords, y, X, params, lambdas


def input_hash(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:16]
