"""Representative parameter points (paper Step 2, §3).

Builds the quadratic approximation of the profile log-likelihood around an MLE
and places parameter points on χ² contour ellipsoids, plus the Box-Cox λ grid —
the workloads the batched likelihood (lik_eval_batch) is run on.  The 51·3 (or
33·3) stencil likelihoods of the numerical Hessian are evaluated in one batched
call through the C ABI ("computed on GPU in parallel"); the rest is small
dense algebra on the host (5×5 eigen-decomposition, sphere packing).

Readings (R21-R25):
  R21 internal coordinates ω' = (γ1, κ̃, ν, γ2, γ3) with ν = √ν²; φR < 1 is
      mapped to the equivalent (φX/φR, 1/φR, φA + π/2) first, so γ2, γ3 are real.
  R22 the Hessian is taken in ω' at λ = λ̂; the λ curvature from ℓ_p(ω̂', λ̂ ± δ)
      (second derivatives between λ and ω' assumed zero); central differences,
      step δ = 1e-3·max(1, |ω̂'_i|).
  R23 eigenvalue repair: |d|, and if max(d) > 100 every d < 0.1 → 0.1.
  R24 ellipsoid map: the printed x' = E⁻² D^{1/2} x + ω̂' is garbled; the map
      ω' = ω̂' + √c E D^{−1/2} x makes (ω'−ω̂')ᵀ(−H)(ω'−ω̂') = c for |x| = 1 (the
      region of P:267-269 with −H in the quadratic form, not (−H)⁻¹).
  R25 nugget repair: among points with ν < 0, a seeded random half get ν² = 0
      and the other half ν² ~ U(0, 2).
"""
from __future__ import annotations

import functools
import math
from dataclasses import dataclass, field

import numpy as np

DEFAULT_ALPHAS = (0.00001, 0.01, 0.1, 0.2, 0.25, 0.3, 0.5, 0.8, 0.9, 0.95, 0.99, 0.999)


# --------------------------------------------------------------------------- parametrisation
def kappa_regime(kappa_hat: float) -> str:
    """κ̃ = log κ if κ̂ < 4 else κ^{−1/2}."""
    return "log" if kappa_hat < 4 else "invroot"


def to_internal(nat, regime: str) -> np.ndarray:
    """Natural {φX, κ, ν², φR, φA} (…×5) -> internal (γ1, κ̃, ν, γ2, γ3)."""
    nat = np.atleast_2d(np.asarray(nat, dtype=np.float64))
    phiX, kappa, nug, phiR, phiA = nat.T
    flip = phiR < 1.0  # R21: (φX, φR, φA) ≡ (φX/φR, 1/φR, φA + π/2)
    phiX = np.where(flip, phiX / phiR, phiX)
    phiA = np.where(flip, phiA + math.pi / 2, phiA)
    phiR = np.where(flip, 1.0 / phiR, phiR)
    phiY = phiX / phiR
    g1 = np.log(phiX) + np.log(phiY)
    rad = np.sqrt(phiR - 1.0)
    kt = np.log(kappa) if regime == "log" else kappa ** -0.5
    return np.stack([g1, kt, np.sqrt(nug), rad * np.cos(2 * phiA), rad * np.sin(2 * phiA)], axis=-1)


def to_natural(internal, regime: str, kappa_fixed: float | None = None) -> np.ndarray:
    """Internal (…×5, or …×4 without κ̃ when κ is fixed) -> natural {φX, κ, ν², φR, φA}."""
    w = np.atleast_2d(np.asarray(internal, dtype=np.float64))
    if kappa_fixed is not None and w.shape[-1] == 4:
        w = np.insert(w, 1, np.nan, axis=-1)
    g1, kt, nu, g2, g3 = w.T
    phiR = 1.0 + g2 * g2 + g3 * g3
    phiA = 0.5 * np.arctan2(g3, g2)
    phiX = np.exp(0.5 * g1) * np.sqrt(phiR)
    if kappa_fixed is not None:
        kappa = np.full_like(g1, kappa_fixed)
    else:
        kappa = np.exp(kt) if regime == "log" else kt ** -2.0
    return np.stack([phiX, kappa, nu * nu, phiR, phiA], axis=-1)


# --------------------------------------------------------------------------- Hessian stencil
def stencil(center, delta) -> np.ndarray:
    """Central-difference stencil: center, ±δ_i e_i, (±δ_i e_i ±δ_j e_j) for i < j:
    1 + 2d + 4·d(d−1)/2 points (51 for d = 5, 33 for d = 4)."""
    c = np.asarray(center, dtype=np.float64)
    d = c.shape[0]
    pts = [c.copy()]
    for i in range(d):
        for s in (1, -1):
            x = c.copy()
            x[i] += s * delta[i]
            pts.append(x)
    for i in range(d):
        for j in range(i + 1, d):
            for si in (1, -1):
                for sj in (1, -1):
                    x = c.copy()
                    x[i] += si * delta[i]
                    x[j] += sj * delta[j]
                    pts.append(x)
    return np.array(pts)


def hessian_from_stencil(f, delta) -> np.ndarray:
    """Second derivatives from the values f on stencil(center, delta)."""
    d = len(delta)
    H = np.zeros((d, d))
    f0 = f[0]
    idx = 1
    fp, fm = np.zeros(d), np.zeros(d)
    for i in range(d):
        fp[i], fm[i] = f[idx], f[idx + 1]
        idx += 2
    for i in range(d):
        H[i, i] = (fp[i] - 2 * f0 + fm[i]) / (delta[i] ** 2)
    for i in range(d):
        for j in range(i + 1, d):
            fpp, fpm, fmp, fmm = f[idx:idx + 4]
            idx += 4
            H[i, j] = H[j, i] = (fpp - fpm - fmp + fmm) / (4 * delta[i] * delta[j])
    return H


def repair_eigenvalues(d) -> np.ndarray:
    """R23."""
    d = np.abs(np.asarray(d, dtype=np.float64))
    if not np.any(d > 0):
        raise ValueError("degenerate Hessian")
    if d.max() > 100:
        d = np.where(d < 0.1, 0.1, d)
    return d


# --------------------------------------------------------------------------- sphere points
def sphere_points(dim: int, n: int, seed: int = 0, iters: int = 100) -> np.ndarray:
    """n points on the unit (dim−1)-sphere spread out by a seeded repulsion optimiser
    (maximising the minimum pairwise distance).  Deterministic for a seed;
    cached, since every fit of the same dimension shares one set."""
    return _sphere_points(dim, n, seed, iters).copy()


@functools.lru_cache(maxsize=16)
def _sphere_points(dim: int, n: int, seed: int, iters: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(n, dim))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    # characteristic spacing of n points on the sphere
    step = 0.5 * (2.0 * math.pi ** (dim / 2) / math.gamma(dim / 2) / n) ** (1.0 / (dim - 1))
    best, best_d = x.copy(), 0.0
    eye = np.eye(n) * 1e9
    for it in range(iters):
        # on the unit sphere |x_i − x_j|² = 2 − 2 x_i·x_j (Gram matrix: O(n²) memory, not O(n²d))
        d2 = np.maximum(2.0 - 2.0 * (x @ x.T), 1e-300) + eye
        dmin = math.sqrt(d2.min())
        if dmin > best_d:
            best, best_d = x.copy(), dmin
        w = d2 ** (-(dim + 1) / 2)                 # short-range repulsion
        force = x * w.sum(1, keepdims=True) - w @ x   # Σ_j w_ij (x_i − x_j)
        force -= (force * x).sum(1, keepdims=True) * x   # tangential part
        fn = np.linalg.norm(force, axis=1, keepdims=True)
        x = x + step * (1.0 - it / iters) * force / np.maximum(fn, 1e-300)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
    return best


def min_distance(x) -> float:
    diff = x[:, None, :] - x[None, :, :]
    d2 = (diff * diff).sum(-1) + np.eye(len(x)) * 1e9
    return float(math.sqrt(d2.min()))


# --------------------------------------------------------------------------- contours, λ, nugget
def chi2_quantile(df: int, upper_alpha: float) -> float:
    """Upper-α point of χ²_df: P(χ² > c) = α."""
    from scipy.stats import chi2
    return float(chi2.isf(upper_alpha, df))


def contour_points(center, negH, alphas, sphere) -> tuple[np.ndarray, np.ndarray]:
    """R24: ω' = ω̂' + √c E D^{−1/2} x for each α and sphere point x; returns (points, α labels)."""
    d, E = np.linalg.eigh(np.asarray(negH, dtype=np.float64))
    d = repair_eigenvalues(d)
    A = E @ np.diag(d ** -0.5)
    pts, labs = [], []
    for a in alphas:
        c = chi2_quantile(len(center), a)
        pts.append(np.asarray(center) + math.sqrt(c) * sphere @ A.T)
        labs.append(np.full(len(sphere), a))
    return np.concatenate(pts), np.concatenate(labs)


def repaired_neg_hessian(negH) -> np.ndarray:
    d, E = np.linalg.eigh(np.asarray(negH, dtype=np.float64))
    return E @ np.diag(repair_eigenvalues(d)) @ E.T


def repair_nugget(nu, rng) -> np.ndarray:
    """R25: returns ν² with negative ν repaired (half → 0, half → U(0, 2))."""
    nu = np.asarray(nu, dtype=np.float64)
    nug = nu * nu
    neg = np.nonzero(nu < 0)[0]
    if len(neg):
        perm = rng.permutation(neg)
        half = len(perm) // 2
        nug[perm[:half]] = 0.0
        nug[perm[half:]] = rng.uniform(0.0, 2.0, size=len(perm) - half)
    return nug


def lambda_grid(center: float, curvature: float, m: int) -> np.ndarray:
    """m equally spaced values between the 0.01 and 0.99 quantiles of the 1-D quadratic
    approximation N(λ̂, −1/curvature), plus λ̂."""
    if m <= 1:
        return np.array([center])
    sd = (-curvature) ** -0.5 if curvature < 0 else 1.0
    z = 2.3263478740408408  # Φ⁻¹(0.99)
    g = np.linspace(center - z * sd, center + z * sd, m)
    return np.unique(np.append(g, center))


# --------------------------------------------------------------------------- driver
@dataclass
class Fit:
    """An MLE to build contours around: natural parameters {φX, κ, ν², φR, φA}, λ̂,
    and optionally the fixed κ of a κ-fixed fit (4-D Hessian)."""
    natural: np.ndarray
    lambda_hat: float
    kappa_fixed: float | None = None


@dataclass
class RepresentativeSet:
    params: np.ndarray                  # K×5 natural
    lambdas: np.ndarray                 # M
    alpha: np.ndarray                   # K (NaN for the MLEs themselves)
    source: np.ndarray                  # K: index of the fit each point came from
    neg_hessians: list = field(default_factory=list)
    lambda_curvature: float = float("nan")
    stencil_loglik: list = field(default_factory=list)  # per fit: stencil points × (λ̂−δ, λ̂, λ̂+δ)


def configure_params(ctx, coords, y, X, fits, alphas=DEFAULT_ALPHAS, n5: int = 726, n4: int = 120,
                     m_lambda: int = 33, seed: int = 0, rel_step: float = 1e-3,
                     alphas_fixed=None) -> RepresentativeSet:
    """The paper's configParams: the stencil likelihoods of all fits in one
    batched lik_eval_batch call (each fit's λ̂ − δ, λ̂, λ̂ + δ), then per fit the Hessian in internal
    coordinates, eigen-repair, contour points at each α, nugget repair; plus the
    MLEs themselves and the λ grid of the first fit.  `alphas_fixed`: the contour
    levels of the κ-fixed fits (default `alphas`; the paper's examples use 11 resp.
    10 of their 12 levels there, R26)."""
    rng = np.random.default_rng(seed)
    # all fits' stencils in ONE batched call: the dataset is shared, and the λ columns
    # are the union of every fit's {λ̂ − δ, λ̂, λ̂ + δ} (each stencil reads its own three)
    setup = []
    for fit in fits:
        regime = kappa_regime(float(fit.natural[1]))
        w0 = to_internal(fit.natural, regime)[0]
        if fit.kappa_fixed is not None:
            w0 = np.delete(w0, 1)
        delta = rel_step * np.maximum(1.0, np.abs(w0))
        dl = rel_step * max(1.0, abs(fit.lambda_hat))
        setup.append((regime, w0, delta, dl, to_natural(stencil(w0, delta), regime, fit.kappa_fixed)))
    lam_all = np.concatenate([[f.lambda_hat - su[3], f.lambda_hat, f.lambda_hat + su[3]]
                              for f, su in zip(fits, setup)])
    res = ctx.eval_batch(coords, y, X, np.concatenate([su[4] for su in setup]), lam_all)
    out_p, out_a, out_s, negHs, stencil_ll = [], [], [], [], []
    curv0 = None
    row = 0
    for f_i, (fit, (regime, w0, delta, dl, nat)) in enumerate(zip(fits, setup)):
        rows = slice(row, row + len(nat))
        row += len(nat)
        if not np.all(res["status"][rows] == 0):
            raise RuntimeError(f"fit {f_i}: stencil point with status {res['status'][rows]}")
        ll = res["loglik"][rows, 3 * f_i:3 * f_i + 3]
        stencil_ll.append(ll)
        negH = -hessian_from_stencil(ll[:, 1], delta)
        curv = (ll[0, 2] - 2 * ll[0, 1] + ll[0, 0]) / dl ** 2
        if curv0 is None:
            curv0 = curv
        negHs.append(negH)
        sph = sphere_points(len(w0), n5 if len(w0) == 5 else n4, seed=seed)
        levels = alphas if (fit.kappa_fixed is None or alphas_fixed is None) else alphas_fixed
        cp, al = contour_points(w0, negH, levels, sph)
        nu_col = 2 if fit.kappa_fixed is None else 1
        nug = repair_nugget(cp[:, nu_col], rng)
        cp[:, nu_col] = np.sqrt(nug)
        nat_pts = to_natural(cp, regime, fit.kappa_fixed)
        out_p.append(nat_pts)
        out_a.append(al)
        out_s.append(np.full(len(nat_pts), f_i))
    # the MLEs themselves ("including 6 MLEs")
    out_p.append(np.array([np.asarray(f.natural, dtype=np.float64) for f in fits]))
    out_a.append(np.full(len(fits), np.nan))
    out_s.append(np.arange(len(fits)))
    return RepresentativeSet(np.concatenate(out_p), lambda_grid(fits[0].lambda_hat, curv0, m_lambda),
                             np.concatenate(out_a), np.concatenate(out_s), negHs, curv0, stencil_ll)


# --------------------------------------------------------------------------- profiles (NEXT-4)
def upper_hull(x, y):
    """Upper convex hull of the 2-D cloud (x, y): vertices sorted by x."""
    o = np.lexsort((y, x))
    x, y = np.asarray(x, dtype=np.float64)[o], np.asarray(y, dtype=np.float64)[o]
    hull = []
    for px, py in zip(x, y):
        while len(hull) >= 2:
            (ax, ay), (bx, by) = hull[-2], hull[-1]
            if (bx - ax) * (py - ay) - (by - ay) * (px - ax) >= 0:  # b is not above a→p
                hull.pop()
            else:
                break
        if hull and hull[-1][0] == px:  # same abscissa: keep the larger y
            if py > hull[-1][1]:
                hull[-1] = (px, py)
            continue
        hull.append((px, py))
    h = np.array(hull)
    return h[:, 0], h[:, 1]


def profile_1d(theta, loglik):
    """1-D profile curve: the upper convex hull of (θ_k, max_m ℓ_p(k, m)),
    linearly interpolated.  Returns (vertices x, vertices y, callable curve)."""
    ok = np.isfinite(loglik)
    hx, hy = upper_hull(np.asarray(theta)[ok], np.asarray(loglik)[ok])
    return hx, hy, (lambda t: np.interp(t, hx, hy, left=np.nan, right=np.nan))


def likelihood_ci(hx, hy, level: float = 0.95):
    """Likelihood-based CI (Eq. likelihood): {θ : ℓ_p(θ) ≥ max − c/2},
    c = χ²_1 quantile at `level`, on the piecewise-linear hull curve; an end that
    never drops below the threshold is reported at the cloud's boundary."""
    from scipy.stats import chi2
    thr = hy.max() - 0.5 * chi2.ppf(level, 1)
    i0 = int(np.argmax(hy))

    def cross(i_in, i_out):
        x0, y0, x1, y1 = hx[i_in], hy[i_in], hx[i_out], hy[i_out]
        return x0 + (thr - y0) * (x1 - x0) / (y1 - y0)
    lo = hx[0]
    for i in range(i0, 0, -1):
        if hy[i - 1] < thr:
            lo = cross(i, i - 1)
            break
    hi = hx[-1]
    for i in range(i0, len(hx) - 1):
        if hy[i + 1] < thr:
            hi = cross(i, i + 1)
            break
    return float(hx[i0]), float(lo), float(hi)


def profile_2d(ti, tj, loglik, query):
    """2-D profile surface: 3-D convex hull of (θ_i, θ_j, ℓ), bottom facets
    removed, linear interpolation on the upper facets.  query: Q×2 -> Q values (NaN
    outside the hull's projection)."""
    from scipy.spatial import ConvexHull
    P = np.column_stack([ti, tj, loglik])
    P = P[np.isfinite(P).all(axis=1)]
    hull = ConvexHull(P)
    out = np.full(len(query), np.nan)
    q = np.asarray(query, dtype=np.float64)
    for simplex, eq in zip(hull.simplices, hull.equations):
        if eq[2] <= 0:  # facet normal points down: bottom facet
            continue
        a, b, c = P[simplex]
        T = np.array([[b[0] - a[0], c[0] - a[0]], [b[1] - a[1], c[1] - a[1]]])
        if abs(np.linalg.det(T)) < 1e-300:
            continue
        lam = np.linalg.solve(T, (q - a[:2]).T).T
        inside = (lam[:, 0] >= -1e-12) & (lam[:, 1] >= -1e-12) & (lam.sum(1) <= 1 + 1e-12)
        val = a[2] + lam[:, 0] * (b[2] - a[2]) + lam[:, 1] * (c[2] - a[2])
        out = np.where(inside & np.isnan(out), val, out)
    return out
