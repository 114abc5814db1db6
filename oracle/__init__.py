"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/liboracle.so`` (built from ``oracle/oracle.cpp``
with plain g++).  The oracle is a slow, obviously-correct FP64 CPU
implementation of the profile log-likelihood of arXiv 2305.04318
(PAPER.md P:59-66).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2305_04318_b200`` never imports it, and the two share
no code.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_D = ctypes.c_double
_I = ctypes.c_int
_PD = ctypes.POINTER(ctypes.c_double)
_PI = ctypes.POINTER(ctypes.c_int)


def build(force: bool = False) -> str:
    """Compile liboracle.so with g++ (-O2, no fast-math: IEEE FP64)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC",
               "-shared", "-pthread", "-o", _LIB, _SRC]
        subprocess.check_call(cmd)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        for name in ("oracle_boxcox", "oracle_log_bessel_k", "oracle_log_bessel_k_integral",
                     "oracle_matern_rho"):
            getattr(L, name).restype = _D
            getattr(L, name).argtypes = [_D, _D]
        L.oracle_aniso_distance.restype = _D
        L.oracle_aniso_distance.argtypes = [_D, _D, _D, _D, _D]
        L.oracle_build_V.restype = None
        L.oracle_build_V.argtypes = [_I, _PD, _PD, _PD]
        L.oracle_ldl.restype = _I
        L.oracle_ldl.argtypes = [_I, _PD, _PD]
        L.oracle_validate.restype = _I
        L.oracle_validate.argtypes = [_I, _I, _PD, _PD, _PD, _I, _PD, _I, _PD]
        L.oracle_eval.restype = _I
        L.oracle_eval.argtypes = [_I, _I, _PD, _PD, _PD, _I, _PD, _I, _PD,
                                  _PD, _PD, _PD, _PD, _PI, _PD, _PD, _PD, _PD, _PD, _PD, _PD, _I]
        L.oracle_profiles.restype = None
        L.oracle_profiles.argtypes = [_I, _I, _I, _I, _PD, _PD, _PI, _PD, _PD, _I, _PD, _PD, _I,
                                      _PD, _PD, _PD]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_PD)


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def boxcox(y: float, lam: float) -> float:
    return lib().oracle_boxcox(float(y), float(lam))


def aniso_distance(x1, x2, phiX, phiR, phiA) -> float:
    return lib().oracle_aniso_distance(float(x1), float(x2), float(phiX), float(phiR), float(phiA))


def log_bessel_k(nu: float, z: float) -> float:
    return lib().oracle_log_bessel_k(float(nu), float(z))


def log_bessel_k_integral(nu: float, z: float) -> float:
    return lib().oracle_log_bessel_k_integral(float(nu), float(z))


def matern_rho(d: float, kappa: float) -> float:
    return lib().oracle_matern_rho(float(d), float(kappa))


def build_V(coords, params5) -> np.ndarray:
    coords = _c(coords)
    n = coords.shape[0]
    w = _c(params5)
    V = np.empty((n, n))
    lib().oracle_build_V(n, _p(coords), _p(w), _p(V))
    return V


def ldl(A):
    """Returns (L unit-lower, D, status) for a symmetric matrix A."""
    A = _c(A).copy()
    n = A.shape[0]
    D = np.zeros(n)
    st = lib().oracle_ldl(n, _p(A), _p(D))
    L = np.tril(A, -1) + np.eye(n)
    return L, D, st


def validate(coords, y, X, params, lambdas) -> int:
    coords, y, X, params, lambdas = map(_c, (coords, y, X, params, lambdas))
    n, p = X.shape
    return lib().oracle_validate(n, p, _p(coords), _p(y), _p(X), params.shape[0], _p(params),
                                 lambdas.shape[0], _p(lambdas))


def eval_batch(coords, y, X, params, lambdas, nthreads: int | None = None, summaries=False):
    """Batched profile log-likelihood, ABI output layout.

    Returns dict(rc, loglik K×M, betahat K×M×p, sigma2hat K×M, logdetV K, status K
    [, ssqYX K×r×r, detReml K, ssqResidual K×M, qdirect K×M, ssqBetahat K×M,
       loglik_reml K×M, sigma2_reml K×M]).
    """
    coords, y, X, lambdas = map(_c, (coords, y, X, lambdas))
    params = _c(params).reshape(-1, 5)
    n, p = X.shape
    K, M = params.shape[0], lambdas.shape[0]
    r = M + p
    out = dict(loglik=np.full((K, M), np.nan), betahat=np.full((K, M, p), np.nan),
               sigma2hat=np.full((K, M), np.nan), logdetV=np.full(K, np.nan),
               status=np.full(K, -1, dtype=np.int32))
    if summaries:
        out.update(ssqYX=np.full((K, r, r), np.nan), detReml=np.full(K, np.nan),
                   ssqResidual=np.full((K, M), np.nan), qdirect=np.full((K, M), np.nan),
                   ssqBetahat=np.full((K, M), np.nan), loglik_reml=np.full((K, M), np.nan),
                   sigma2_reml=np.full((K, M), np.nan))
    nt = nthreads or (os.cpu_count() or 1)
    nul = ctypes.cast(None, _PD)
    rc = lib().oracle_eval(
        n, p, _p(coords), _p(y), _p(X), K, _p(params), M, _p(lambdas),
        _p(out["loglik"]), _p(out["betahat"]), _p(out["sigma2hat"]), _p(out["logdetV"]),
        out["status"].ctypes.data_as(_PI),
        _p(out["ssqYX"]) if summaries else nul, _p(out["detReml"]) if summaries else nul,
        _p(out["ssqResidual"]) if summaries else nul, _p(out["qdirect"]) if summaries else nul,
        _p(out["ssqBetahat"]) if summaries else nul, _p(out["loglik_reml"]) if summaries else nul,
        _p(out["sigma2_reml"]) if summaries else nul, int(nt))
    out["rc"] = rc
    return out


def profiles(n, p, ssqYX, logdetV, status, lambdas, y, beta_grid, sigma_grid):
    """β_a, σ and λ profile log-likelihoods over the K×M grid from summaries.
    Returns (prof_beta p×G, prof_sigma Sg, prof_lambda M)."""
    ssqYX, logdetV, lambdas, y = map(_c, (ssqYX, logdetV, lambdas, y))
    status = np.ascontiguousarray(status, dtype=np.int32)
    beta_grid = _c(beta_grid).reshape(p, -1)
    sigma_grid = _c(sigma_grid)
    K, M, G, Sg = logdetV.shape[0], lambdas.shape[0], beta_grid.shape[1], sigma_grid.shape[0]
    ob, os_, ol = np.empty((p, G)), np.empty(Sg), np.empty(M)
    lib().oracle_profiles(n, p, K, M, _p(ssqYX), _p(logdetV), status.ctypes.data_as(_PI), _p(lambdas),
                          _p(y), G, _p(beta_grid), _p(ob), Sg, _p(sigma_grid), _p(os_), _p(ol))
    return ob, os_, ol
