"""Closed-form likelihoods used as pins (no oracle, no CUDA): shared by the CPU
oracle pins and the large-n GPU tests."""
import numpy as np


def ou_loglik(t, g, y, X, lam):
    """κ = 1/2, ν² = 0, collinear sites: V_ij = exp(−2 g |t_i − t_j|) is the
    covariance of a stationary Ornstein-Uhlenbeck process, whose inverse is
    tridiagonal: log|V| = Σ log(1 − r_i²),
    aᵀV⁻¹b = a_1 b_1 + Σ (a_{i+1} − r_i a_i)(b_{i+1} − r_i b_i)/(1 − r_i²)."""
    o = np.argsort(t)
    t, y, X = t[o], y[o], X[o]
    r = np.exp(-2 * g * np.diff(t))
    yp = np.log(y) if lam == 0 else (y ** lam - 1) / lam
    B = np.column_stack([yp, X])
    W = np.vstack([B[:1], (B[1:] - r[:, None] * B[:-1]) / np.sqrt(1 - r * r)[:, None]])
    C = W.T @ W
    XX, Xy, yy = C[1:, 1:], C[1:, 0], C[0, 0]
    beta = np.linalg.solve(XX, Xy)
    q = yy - Xy @ beta
    n = len(y)
    logdet = np.log1p(-r * r).sum()
    m2l = n * np.log(q / n) + logdet - 2 * (lam - 1) * np.log(y).sum() + n * np.log(2 * np.pi) + n
    return -m2l / 2, beta, q / n, logdet
