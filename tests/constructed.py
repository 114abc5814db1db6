"""Hand-constructed inputs whose point status is fixed by exact arithmetic, not by
either implementation (test data only; no method arithmetic).

xvx_singular()   Step 5 fails: XᵀV⁻¹X is singular in FP64 although X passes the
                 full-rank check.  100 sites on a 10 × 10 grid 1e6 range units apart, so
                 every off-diagonal ρ underflows to exactly 0 and ν² = 0 gives V = I
                 exactly; X = [1, 1 + 2⁻³⁰e] with small integers e, Σe = 0.  Exactly,
                 XᵀX = [[n, n], [n, n + 2⁻⁶⁰Σe²]] is positive definite (det = n·2⁻⁶⁰Σe² > 0,
                 and the Gram-Schmidt residual of column 2 is 2⁻⁶⁰Σe²/n ≈ 2e-17 of its
                 norm², above the 1e-20 rank threshold), but every FP64 partial sum of
                 x₁·x₂ = Σ(1 + 2⁻³⁰e_i) and of x₂·x₂ = Σ(1 + 2⁻²⁹e_i + 2⁻⁶⁰e_i²) is exact
                 except for the 2⁻⁶⁰e_i² terms (below half an ulp of any partial sum ≥ 1 for
                 |e_i| ≤ 7), so both products round to exactly n and the second pivot of
                 XᵀV⁻¹X is exactly 0 ≤ p·ε·max diag: status XVX_NOT_PD on any summation order.
resid_in_span()  Step 8 cancels: for λ = 1, y' = y − 1 = 1 + 3t lies in span(X),
                 X = [1, t], up to the rounding of the Box-Cox transform (≲ 1e-16 relative),
                 so q = (y' − Xβ̂)ᵀV⁻¹(y' − Xβ̂) ≲ 1e-30·y'ᵀV⁻¹y' exactly, and Step 8's
                 subtraction leaves only rounding noise (≲ 1e-14·y'ᵀV⁻¹y'): the column
                 fails R12 (q ≤ 1e-10·y'ᵀV⁻¹y') on both sides and the point's status is
                 NEG_RESID.  The λ = 0.5 column (y' = 2(√y − 1), not in the span; q/yy ≈
                 1e-3) stays valid and is compared element by element.
"""
from __future__ import annotations

import math

import numpy as np


def xvx_singular():
    g = np.arange(10) * 1e6
    coords = np.array([(a, b) for a in g for b in g], dtype=np.float64)
    n = coords.shape[0]
    rng = np.random.default_rng(230504318)
    v = rng.integers(1, 8, size=n // 2) * rng.choice([-1, 1], size=n // 2)
    e = rng.permutation(np.r_[v, -v]).astype(np.float64)  # Σe = 0, |e| ≤ 7
    X = np.column_stack([np.ones(n), 1.0 + e * 2.0 ** -30])
    y = np.exp(rng.normal(1.0, 0.3, size=n))
    P = np.array([[1.0, 0.5, 0.0, 1.0, 0.0],     # φX = 1 ≪ 1e6 spacing: ρ = 0 off the diagonal
                  [2.0, 2.5, 0.0, 1.5, 0.3],
                  [5.0, 40.0, 0.0, 1.0, 0.0]])
    lam = np.array([0.5, 1.0])
    return coords, y, X, P, lam, e


def resid_in_span():
    rng = np.random.default_rng(2305)
    n = 150
    side = 9000.0 * math.sqrt(n / 224.0)
    coords = rng.uniform(0.0, side, size=(n, 2))
    t = coords[:, 0] / side * 3.0           # t ∈ [0, 3]
    X = np.column_stack([np.ones(n), t])
    y = 2.0 + 3.0 * t                       # y ∈ [2, 11]; y − 1 = 1 + 3t ∈ span(X)
    P = np.array([[900.0, 1.5, 0.2, 1.0, 0.0],
                  [1500.0, 0.5, 0.05, 2.0, 0.7],
                  [600.0, 10.0, 0.5, 1.0, 0.0]])
    lam = np.array([1.0, 0.5])
    return coords, y, X, P, lam
