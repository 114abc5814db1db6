"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each pin is chosen so that a plausible mistake in oracle/oracle.cpp (a dropped
term, a wrong sign or index, a transposed operand, a wrong prefactor) fails it:

* worked examples printed in SPEC.md / derived by hand (tests/golden/*.json);
* closed forms of the Matérn at κ = 1/2, 3/2, 5/2 (independent of Bessel K);
* mpmath besselk at 40 digits, mpmath det/inverse at 50 digits (brute force);
* the Ornstein-Uhlenbeck (κ = 1/2, collinear sites) closed-form likelihood;
* scipy LAPACK (cho_factor) + scipy.stats multivariate-normal log-density;
* invariances (translation, joint rotation, permutation, scale, period π);
* the Box-Cox Jacobian as a change of variables with a numerical derivative.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest
from closed_forms import ou_loglik  # noqa: E402
import scipy.linalg as sla
import scipy.stats as sst

import synthgen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------- Box-Cox
def test_boxcox_spec_examples(orc):
    for y, lam, want in _gold("spec_examples.json")["boxcox"]["cases"]:
        assert orc.boxcox(y, lam) == pytest.approx(want, rel=1e-15, abs=1e-15)


def test_boxcox_continuity_and_monotone(orc):
    # |b(y, 1e-8) − log y| ≤ 1e-6 on [0.1, 100]
    for y in np.geomspace(0.1, 100, 37):
        assert abs(orc.boxcox(y, 1e-8) - math.log(y)) <= 1e-6
        assert orc.boxcox(y, 0.0) == math.log(y)
    # strictly increasing in y for fixed λ; mpmath reference (y^λ − 1)/λ at 40 digits
    mpmath.mp.dps = 40
    for lam in (-1.3, -0.2, 0.3, 0.5, 1.0, 2.0):
        ys = np.geomspace(0.05, 500, 25)
        vals = [orc.boxcox(y, lam) for y in ys]
        assert all(b > a for a, b in zip(vals, vals[1:]))
        for y, v in zip(ys, vals):
            ref = (mpmath.mpf(y) ** lam - 1) / lam
            assert v == pytest.approx(float(ref), rel=2e-15, abs=1e-300)


# --------------------------------------------------------------------------- distance
def test_distance_spec_examples(orc):
    for x1, x2, phiX, phiR, phiA, want in _gold("spec_examples.json")["distance"]["cases"]:
        assert orc.aniso_distance(x1, x2, phiX, phiR, phiA) == pytest.approx(want, rel=1e-15)


def test_distance_invariants(orc):
    rng = np.random.default_rng(1)
    for _ in range(200):
        h = rng.normal(size=2) * 100
        phiX, phiR, phiA, th = rng.uniform(10, 200), rng.uniform(0.3, 9), rng.uniform(-3, 3), rng.uniform(-3, 3)
        d = orc.aniso_distance(h[0], h[1], phiX, phiR, phiA)
        # joint rotation: d(Rot(-θ) h; φA + θ) = d(h; φA)
        c, s = math.cos(-th), math.sin(-th)
        hr = (c * h[0] - s * h[1], s * h[0] + c * h[1])
        assert orc.aniso_distance(hr[0], hr[1], phiX, phiR, phiA + th) == pytest.approx(d, rel=1e-12)
        # period π in φA, symmetry in h, isotropy when φR = 1
        assert orc.aniso_distance(h[0], h[1], phiX, phiR, phiA + math.pi) == pytest.approx(d, rel=1e-12)
        assert orc.aniso_distance(-h[0], -h[1], phiX, phiR, phiA) == d
        assert orc.aniso_distance(h[0], h[1], phiX, 1.0, phiA) == pytest.approx(
            math.hypot(h[0], h[1]) / phiX, rel=1e-14)
        # (φR, φA) ≡ (1/φR, φA + π/2) with φX -> φX/φR (R5)
        assert orc.aniso_distance(h[0], h[1], phiX / phiR, 1 / phiR, phiA + math.pi / 2) == pytest.approx(d, rel=1e-12)


# --------------------------------------------------------------------------- Matérn
def test_matern_spec_examples(orc):
    for d, kappa, want in _gold("spec_examples.json")["matern"]["cases"]:
        assert orc.matern_rho(d, kappa) == pytest.approx(want, rel=1e-13)


@pytest.mark.parametrize("kappa,closed", [
    (0.5, lambda d: math.exp(-2 * d)),
    (1.5, lambda d: (1 + math.sqrt(12) * d) * math.exp(-math.sqrt(12) * d)),
    (2.5, lambda d: (1 + math.sqrt(20) * d + (math.sqrt(20) * d) ** 2 / 3) * math.exp(-math.sqrt(20) * d)),
])
def test_matern_half_integer_closed_forms(orc, kappa, closed):
    # K_{1/2}, K_{3/2}, K_{5/2} are elementary; these pin prefactor, sqrt(8κ) scaling
    # and the Bessel evaluation together (R1, R2).
    for d in np.concatenate([np.geomspace(1e-7, 1, 40), np.linspace(1, 150, 40)]):
        want = closed(d)
        got = orc.matern_rho(d, kappa)
        if want < 1e-290:
            assert got < 1e-280
        else:
            assert got == pytest.approx(want, rel=2e-13), (kappa, d)


def _mp_rho(d, kappa):
    mpmath.mp.dps = 40
    d, k = mpmath.mpf(d), mpmath.mpf(kappa)
    z = mpmath.sqrt(8 * k) * d
    return 2 ** (1 - k) / mpmath.gamma(k) * z ** k * mpmath.besselk(k, z)


KGRID = [0.05, 0.2, 0.37, 0.5, 0.9, 1.0, 1.83, 2.0, 3.7, 10.0, 20.0, 47.3, 100.0, 200.0]
ZGRID = [1e-8, 1e-4, 0.01, 0.3, 1.0, 1.99, 2.01, 5.0, 30.0, 200.0, 700.0]


def test_log_bessel_k_vs_mpmath(orc):
    """ln K_ν(z) vs mpmath at 40 digits, including the overflow region where the
    library routine returns inf and the oracle switches to the integral (R9)."""
    mpmath.mp.dps = 40
    worst = 0.0
    for nu in KGRID:
        for z in ZGRID:
            ref = float(mpmath.log(mpmath.besselk(nu, z)))
            got = orc.log_bessel_k(nu, z)
            err = abs(got - ref) / max(1.0, abs(ref))
            worst = max(worst, err)
            assert err <= 2e-14, (nu, z, got, ref)
            # the integral branch is checked everywhere too (it is the fallback)
            gi = orc.log_bessel_k_integral(nu, z)
            assert abs(gi - ref) / max(1.0, abs(ref)) <= 5e-14, (nu, z, gi, ref)


def test_matern_vs_mpmath(orc):
    for kappa in KGRID:
        for d in (1e-9, 1e-5, 1e-3, 0.02, 0.1, 0.4, 1.0, 2.5, 8.0, 30.0):
            ref = _mp_rho(d, kappa)
            got = orc.matern_rho(d, kappa)
            if ref < mpmath.mpf("1e-290"):
                assert got < 1e-280
                continue
            assert got == pytest.approx(float(ref), rel=5e-14), (kappa, d)


def test_matern_limits_and_monotone(orc):
    for kappa in KGRID:
        assert orc.matern_rho(0.0, kappa) == 1.0
        if kappa >= 0.5:
            assert abs(orc.matern_rho(1e-10, kappa) - 1.0) < 1e-6
        else:
            # 1 − ρ ~ Γ(1−κ)/Γ(1+κ) (z/2)^{2κ} as z → 0 (small-argument expansion of K_κ)
            z = math.sqrt(8 * kappa) * 1e-12
            lead = math.gamma(1 - kappa) / math.gamma(1 + kappa) * (z / 2) ** (2 * kappa)
            assert 1 - orc.matern_rho(1e-12, kappa) == pytest.approx(lead, rel=0.02)
        ds = np.linspace(1e-4, 5, 200)
        vals = [orc.matern_rho(d, kappa) for d in ds]
        assert all(b <= a for a, b in zip(vals, vals[1:]))
    # Gaussian limit κ → ∞: exp(−2 d²); κ = 1e4 within 1e-4
    for d in (0.1, 0.3, 0.9):
        assert orc.matern_rho(d, 1e4) == pytest.approx(math.exp(-2 * d * d), rel=1e-15)
        assert abs(orc.matern_rho(d, 999.0) - math.exp(-2 * d * d)) < 1e-3


# --------------------------------------------------------------------------- V and LDLᵀ
def test_build_V_structure(orc):
    coords, y, X = synthgen.make_dataset("C1")
    w = np.array([800.0, 1.7, 0.3, 2.5, 0.4])
    V = orc.build_V(coords, w)
    assert np.array_equal(V, V.T)
    assert np.all(np.diag(V) == 1.3)
    # elementwise against the scalar functions (distance from the paper's matrix product)
    i, j = 17, 3
    h = coords[i] - coords[j]
    S = np.diag([1 / w[0], w[3] / w[0]])
    R = np.array([[math.cos(w[4]), -math.sin(w[4])], [math.sin(w[4]), math.cos(w[4])]])
    d = np.linalg.norm(S @ R @ h)
    assert V[i, j] == pytest.approx(float(_mp_rho(d, w[1])), rel=1e-13)
    # isotropy degeneracy: φR = 1 -> φA irrelevant
    V1 = orc.build_V(coords, [800.0, 1.7, 0.3, 1.0, 0.0])
    V2 = orc.build_V(coords, [800.0, 1.7, 0.3, 1.0, 1.1])
    np.testing.assert_allclose(V1, V2, rtol=1e-12, atol=1e-300)
    # positive definite (all eigenvalues ≥ ν²·(1 − 1e-9)), LAPACK eigvalsh
    ev = np.linalg.eigvalsh(V)
    assert ev.min() > 0.3 * (1 - 1e-9)


def test_ldl_examples(orc):
    g = _gold("spec_examples.json")["ldl"]
    L, D, st = orc.ldl(np.array(g["V"]))
    assert st == 0
    np.testing.assert_array_equal(L, np.array(g["L"]))
    np.testing.assert_array_equal(D, np.array(g["D"]))
    L, D, st = orc.ldl(np.eye(4))
    assert st == 0 and np.array_equal(L, np.eye(4)) and np.array_equal(D, np.ones(4))
    _, _, st = orc.ldl(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert st == 1
    rng = np.random.default_rng(0)
    A = rng.normal(size=(40, 40))
    A = A @ A.T + 40 * np.eye(40)
    L, D, st = orc.ldl(A)
    assert st == 0
    np.testing.assert_allclose(L @ np.diag(D) @ L.T, A, rtol=0, atol=1e-12 * np.abs(A).max())
    # log|A| against LAPACK
    assert np.log(D).sum() == pytest.approx(np.linalg.slogdet(A)[1], rel=1e-13)


# --------------------------------------------------------------------------- whole likelihood
def _far_sites(n, rng):
    # sites 1e7 apart with φX = 1: ρ underflows to exactly 0, V = (1+ν²) I
    return np.stack([np.arange(n) * 1e7, rng.uniform(0, 1, n)], axis=1)


def test_spec_n3_ols_example(orc):
    g = _gold("spec_n3_ols.json")
    coords = _far_sites(3, np.random.default_rng(0))
    yprime = np.array(g["y_prime"])
    y = yprime + 1.0                      # λ = 1: b(y;1) = y − 1, Jacobian 0
    X = np.ones((3, 1))
    out = orc.eval_batch(coords, y, X, [[1.0, 0.7, 0.0, 1.0, 0.0]], [1.0])
    assert out["rc"] == 0 and out["status"][0] == 0
    assert out["logdetV"][0] == 0.0
    assert out["betahat"][0, 0, 0] == pytest.approx(g["betahat"], rel=1e-15)
    assert out["sigma2hat"][0, 0] == pytest.approx(g["sigma2hat"], rel=1e-15)
    assert -2 * out["loglik"][0, 0] == pytest.approx(g["minus2_loglik"], rel=1e-15)


def test_far_sites_reduce_to_ols(orc):
    rng = np.random.default_rng(3)
    n, p, M = 60, 3, 4
    coords = _far_sites(n, rng)
    X = np.column_stack([np.ones(n), rng.normal(size=(n, p - 1))])
    y = np.exp(rng.normal(1.0, 0.3, size=n))
    lam = np.array([-0.5, 0.0, 0.4, 1.3])
    nug = 0.37
    out = orc.eval_batch(coords, y, X, [[1.0, 1.3, nug, 1.0, 0.0]], lam)
    assert out["logdetV"][0] == pytest.approx(n * math.log(1 + nug), rel=1e-14)
    for m, l in enumerate(lam):
        yp = np.log(y) if l == 0 else (y ** l - 1) / l
        beta, rss, *_ = np.linalg.lstsq(X, yp, rcond=None)
        np.testing.assert_allclose(out["betahat"][0, m], beta, rtol=1e-11, atol=1e-12)
        assert out["sigma2hat"][0, m] == pytest.approx(float(rss[0]) / (n * (1 + nug)), rel=1e-11)


def _mp_loglik(coords, y, X, w, lam):
    """Brute force at 50 digits: mpmath Bessel, det, inverse (n ≤ 10)."""
    mpmath.mp.dps = 50
    n, p = X.shape
    V = mpmath.matrix(n, n)
    for i in range(n):
        for j in range(n):
            if i == j:
                V[i, j] = 1 + mpmath.mpf(w[2])
            else:
                h = coords[i] - coords[j]
                S = np.diag([1 / w[0], w[3] / w[0]])
                R = np.array([[math.cos(w[4]), -math.sin(w[4])], [math.sin(w[4]), math.cos(w[4])]])
                u = R @ h
                d = mpmath.sqrt((mpmath.mpf(u[0]) * S[0, 0]) ** 2 + (mpmath.mpf(u[1]) * S[1, 1]) ** 2)
                V[i, j] = _mp_rho(d, w[1]) if d > 0 else 1
    mpmath.mp.dps = 50
    Vi = V ** -1
    Xm = mpmath.matrix(X.tolist())
    yp = mpmath.matrix([(mpmath.mpf(v) ** lam - 1) / lam if lam != 0 else mpmath.log(v) for v in y])
    XtVi = Xm.T * Vi
    beta = (XtVi * Xm) ** -1 * (XtVi * yp)
    r = yp - Xm * beta
    q = (r.T * Vi * r)[0, 0]
    logdet = mpmath.log(mpmath.det(V))
    m2l = n * mpmath.log(q / n) + logdet - 2 * (lam - 1) * sum(mpmath.log(v) for v in y) \
        + n * mpmath.log(2 * mpmath.pi) + n
    return float(-m2l / 2), [float(b) for b in beta], float(q / n), float(logdet)


def test_brute_force_mpmath_small(orc):
    rng = np.random.default_rng(11)
    for trial in range(4):
        n, p = 7 + trial, 1 + trial % 3
        coords = rng.uniform(0, 1000, size=(n, 2))
        X = np.column_stack([np.ones(n)] + [rng.normal(size=n) for _ in range(p - 1)])
        y = np.exp(rng.normal(2.0, 0.4, size=n))
        w = [rng.uniform(200, 900), [0.3, 1.0, 2.7, 13.0][trial], rng.uniform(0.05, 0.5),
             rng.uniform(0.5, 4.0), rng.uniform(-1.5, 1.5)]
        lam = [0.0, 0.35, 1.0]
        out = orc.eval_batch(coords, y, X, [w], lam)
        assert out["status"][0] == 0
        for m, l in enumerate(lam):
            ll, beta, s2, ld = _mp_loglik(coords, y, X, w, l)
            assert out["loglik"][0, m] == pytest.approx(ll, rel=1e-11)
            np.testing.assert_allclose(out["betahat"][0, m], beta, rtol=1e-9, atol=1e-10)
            assert out["sigma2hat"][0, m] == pytest.approx(s2, rel=1e-10)
            assert out["logdetV"][0] == pytest.approx(ld, rel=1e-11, abs=1e-12)


@pytest.mark.parametrize("n", [50, 600])
def test_ou_closed_form(orc, n):
    rng = np.random.default_rng(n)
    phiX, phiR, phiA = 300.0, 2.5, 0.6
    u = np.array([math.cos(1.1), math.sin(1.1)])
    g = orc.aniso_distance(u[0], u[1], phiX, phiR, phiA)
    # spacing so that r_i = exp(−2 g Δt) ≤ 0.9 (well conditioned)
    gaps = rng.uniform(-math.log(0.9) / (2 * g), 3.0 / g, size=n - 1)
    t = np.concatenate([[0.0], np.cumsum(gaps)])
    t = rng.permutation(t)
    coords = np.outer(t, u) + np.array([1234.5, -987.0])
    X = np.column_stack([np.ones(n), rng.normal(size=n), rng.normal(size=n)])
    y = np.exp(rng.normal(2.0, 0.3, size=n))
    lam = [0.0, 0.5]
    out = orc.eval_batch(coords, y, X, [[phiX, 0.5, 0.0, phiR, phiA]], lam)
    assert out["status"][0] == 0
    for m, l in enumerate(lam):
        ll, beta, s2, ld = ou_loglik(t, g, y, X, l)
        assert out["logdetV"][0] == pytest.approx(ld, rel=1e-10)
        assert out["loglik"][0, m] == pytest.approx(ll, rel=1e-10)
        np.testing.assert_allclose(out["betahat"][0, m], beta, rtol=1e-8, atol=1e-9)
        assert out["sigma2hat"][0, m] == pytest.approx(s2, rel=1e-9)


def test_kappa_3_2_against_lapack_and_scipy_density(orc):
    """κ = 3/2 closed form V, LAPACK Cholesky, and the scipy multivariate-normal
    log-density of Eq. 2 with the Box-Cox Jacobian taken as a change of variables
    whose derivative is computed numerically (pins the Jacobian sign and factor)."""
    coords, y, X = synthgen.make_dataset("C1")
    n = len(y)
    w = [900.0, 1.5, 0.2, 1.0, 0.0]
    lam = [0.3, 0.8]
    out = orc.eval_batch(coords, y, X, [w], lam)
    D = np.sqrt(((coords[:, None, :] - coords[None, :, :]) ** 2).sum(-1)) / w[0]
    z = math.sqrt(12) * D
    V = (1 + z) * np.exp(-z) + w[2] * np.eye(n)
    cf = sla.cho_factor(V, lower=True)
    assert out["logdetV"][0] == pytest.approx(2 * np.log(np.diag(cf[0])).sum(), rel=1e-12)
    for m, l in enumerate(lam):
        yp = (y ** l - 1) / l
        XtViX = X.T @ sla.cho_solve(cf, X)
        beta = np.linalg.solve(XtViX, X.T @ sla.cho_solve(cf, yp))
        r = yp - X @ beta
        s2 = r @ sla.cho_solve(cf, r) / n
        h = 1e-6 * y
        dbdy = (((y + h) ** l - 1) / l - ((y - h) ** l - 1) / l) / (2 * h)
        ll = sst.multivariate_normal(mean=X @ beta, cov=s2 * V).logpdf(yp) + np.log(dbdy).sum()
        assert out["loglik"][0, m] == pytest.approx(ll, rel=1e-9)
        np.testing.assert_allclose(out["betahat"][0, m], beta, rtol=1e-10)
        # maximality (β̂, σ̂² maximise Eq. 2)
        for db in (np.full(X.shape[1], 1e-3), -np.full(X.shape[1], 1e-3)):
            assert sst.multivariate_normal(mean=X @ (beta + db), cov=s2 * V).logpdf(yp) < \
                sst.multivariate_normal(mean=X @ beta, cov=s2 * V).logpdf(yp)
        for f in (0.9, 1.1):
            assert sst.multivariate_normal(mean=X @ beta, cov=f * s2 * V).logpdf(yp) < \
                sst.multivariate_normal(mean=X @ beta, cov=s2 * V).logpdf(yp)


def test_invariances(orc):
    coords, y, X = synthgen.make_dataset("C1")
    X = X[:, :1]  # intercept only: invariant under moving the sites
    P = np.array([[700.0, 1.3, 0.25, 2.2, 0.35], [1500.0, 0.7, 0.5, 1.0, 0.0]])
    lam = [0.1, 0.6]
    base = orc.eval_batch(coords, y, X, P, lam)["loglik"]
    # translation
    np.testing.assert_allclose(orc.eval_batch(coords + [5e4, -3e3], y, X, P, lam)["loglik"], base, rtol=1e-11)
    # joint rotation of sites by θ and φA -> φA − θ... (d(Rot(θ)s; φA − θ) = d(s; φA))
    th = 0.77
    Rm = np.array([[math.cos(th), -math.sin(th)], [math.sin(th), math.cos(th)]])
    P2 = P.copy()
    P2[:, 4] -= th
    np.testing.assert_allclose(orc.eval_batch(coords @ Rm.T, y, X, P2, lam)["loglik"], base, rtol=1e-11)
    # φA + π periodicity
    P3 = P.copy()
    P3[:, 4] += math.pi
    np.testing.assert_allclose(orc.eval_batch(coords, y, X, P3, lam)["loglik"], base, rtol=1e-11)
    # scale coordinates and φX together
    P4 = P.copy()
    P4[:, 0] *= 3.5
    np.testing.assert_allclose(orc.eval_batch(coords * 3.5, y, X, P4, lam)["loglik"], base, rtol=1e-11)
    # permutation of sites (with y, X rows)
    perm = np.random.default_rng(5).permutation(len(y))
    np.testing.assert_allclose(orc.eval_batch(coords[perm], y[perm], X[perm], P, lam)["loglik"], base, rtol=1e-11)


def test_lambda_column_equivalence(orc):
    # evaluating at λ0 on y equals evaluating the pre-transformed data at λ = 1
    # (y_new = b(y; λ0) + 1, Jacobian 0), after removing the Jacobian (λ0 − 1)Σ log y
    coords, y, X = synthgen.make_dataset("C1")
    P = synthgen.make_params("C1", 4)
    l0 = 0.45
    a = orc.eval_batch(coords, y, X, P, [l0])
    ynew = (y ** l0 - 1) / l0 + 1.0
    assert ynew.min() > 0
    b = orc.eval_batch(coords, ynew, X, P, [1.0])
    np.testing.assert_allclose(a["loglik"][:, 0] - (l0 - 1) * np.log(y).sum(), b["loglik"][:, 0], rtol=1e-11)
    np.testing.assert_allclose(a["betahat"], b["betahat"], rtol=1e-10)


def test_step8_subtraction_agrees_with_eq4(orc):
    coords, y, X, P, lam = synthgen.make_inputs("C2", K=24)
    out = orc.eval_batch(coords, y, X, P, lam, summaries=True)
    ok = out["status"] == 0
    rel = np.abs(out["ssqResidual"][ok] - out["qdirect"][ok]) / np.abs(out["qdirect"][ok])
    assert rel.max() < 1e-9
    # ssqYX is symmetric and its diagonal is positive
    S = out["ssqYX"][ok]
    np.testing.assert_allclose(S, np.transpose(S, (0, 2, 1)), rtol=1e-10)


def test_status_and_errors(orc):
    coords, y, X = synthgen.make_dataset("C1")
    good = [900.0, 1.5, 0.2, 1.0, 0.0]
    bad = [[-1.0, 1.5, 0.2, 1.0, 0.0], [900.0, 0.0, 0.2, 1.0, 0.0], [900.0, 1.5, -0.1, 1.0, 0.0],
           [900.0, 1.5, 0.2, 0.0, 0.0], [900.0, float("nan"), 0.2, 1.0, 0.0]]
    out = orc.eval_batch(coords, y, X, [good] + bad, [0.5])
    assert out["status"][0] == 0
    assert np.all(out["status"][1:] == 4)
    assert np.all(np.isneginf(out["loglik"][1:])) and np.all(np.isnan(out["logdetV"][1:]))
    # not PD: huge range, smooth, no nugget on dense sites
    c2 = np.stack([np.arange(40) * 1.0, np.zeros(40)], axis=1)
    out = orc.eval_batch(c2, np.ones(40) + np.arange(40), np.ones((40, 1)), [[1e5, 10.0, 0.0, 1.0, 0.0]], [0.5])
    assert out["status"][0] == 1
    # call-level errors
    assert orc.validate(coords, y, X, [good], [0.5]) == 0
    y2 = y.copy()
    y2[7] = -1.0
    assert orc.validate(coords, y2, X, [good], [0.5]) == -2
    c3 = coords.copy()
    c3[9] = c3[4]
    assert orc.validate(c3, y, X, [good], [0.5]) == -2
    X2 = np.column_stack([X, 2 * X[:, 1]])
    assert orc.validate(coords, y, X2, [good], [0.5]) == -3
    assert orc.validate(coords[:3], y[:3], X[:3], [good], [0.5]) == -1


def test_xvx_not_pd_constructed(orc):
    """Step 5: the constructed X of tests/constructed.py passes the full-rank check
    but XᵀV⁻¹X (V = I exactly) is singular in FP64 — pinned by exact rational arithmetic,
    not by the oracle: the exact Gram matrix is PD, yet its FP64 entries are exactly n."""
    from fractions import Fraction
    import constructed
    coords, y, X, P, lam, e = constructed.xvx_singular()
    n = X.shape[0]
    x2 = [Fraction(float(v)) for v in X[:, 1]]
    g12, g22 = sum(x2), sum(v * v for v in x2)
    assert g12 == n and g22 - n == Fraction(int((e * e).sum()), 2 ** 60)  # det = n·2⁻⁶⁰Σe² > 0
    acc = 0.0
    for v in X[:, 1]:  # the FP64 left-to-right sum of x2·x2 (any order gives the same)
        acc += v * v
    assert acc == float(n) and float(np.sum(X[:, 1] * X[:, 1])) == float(n)
    # ρ underflows to exactly 0 off the diagonal: V = I
    for w in P:
        V = orc.build_V(coords, w)
        assert np.array_equal(V, np.eye(n))
    assert orc.validate(coords, y, X, P, lam) == 0  # not ERANK
    out = orc.eval_batch(coords, y, X, P, lam, summaries=True)
    assert np.all(out["status"] == 2)
    assert np.all(np.isneginf(out["loglik"])) and np.all(np.isnan(out["betahat"]))
    assert np.all(np.isnan(out["logdetV"])) and np.all(np.isnan(out["sigma2hat"]))


def test_neg_resid_constructed(orc):
    """Step 8 and R12: y' of the λ = 1 column lies in span(X) (tests/constructed.py),
    so Eq. 4's q vanishes up to Box-Cox rounding and Step 8's subtraction is noise: that
    column fails (status NEG_RESID, ℓ_p = −∞, σ̂² and β̂ NaN), the λ = 0.5 column stands."""
    import constructed
    coords, y, X, P, lam = constructed.resid_in_span()
    out = orc.eval_batch(coords, y, X, P, lam, summaries=True)
    assert np.all(out["status"] == 3)
    yy = out["ssqYX"][:, 0, 0]
    assert np.all(np.abs(out["ssqResidual"][:, 0]) <= 1e-13 * yy)
    assert np.all(np.isneginf(out["loglik"][:, 0])) and np.all(np.isnan(out["sigma2hat"][:, 0]))
    assert np.all(np.isnan(out["betahat"][:, 0])) and np.all(np.isneginf(out["loglik_reml"][:, 0]))
    # the other column: finite, and Step 8 agrees with the direct Eq. 4 form
    assert np.all(np.isfinite(out["loglik"][:, 1])) and np.all(out["sigma2hat"][:, 1] > 0)
    q8, q4 = out["ssqResidual"][:, 1], out["qdirect"][:, 1]
    assert np.all(q4 > 1e-6 * out["ssqYX"][:, 1, 1])
    assert np.abs(q8 - q4).max() <= 1e-9 * q4.min()
    # log|V| and the Table-1 summaries of a NEG_RESID point stay valid
    assert np.all(np.isfinite(out["logdetV"])) and np.all(np.isfinite(out["ssqYX"]))
    # the profiles use the valid column only (R12): λ-profile of column 0 is −∞
    grid = np.linspace(-1.0, 4.0, 5).reshape(1, -1).repeat(X.shape[1], 0)
    pb, ps, pl = orc.profiles(X.shape[0], X.shape[1], out["ssqYX"], out["logdetV"], out["status"], lam, y,
                              grid, np.array([0.5, 1.0]))
    assert np.isneginf(pl[0]) and pl[1] == pytest.approx(out["loglik"][:, 1].max(), rel=1e-12)
    assert np.all(np.isfinite(pb)) and np.all(np.isfinite(ps))


def test_thread_determinism(orc):
    coords, y, X, P, lam = synthgen.make_inputs("C2", K=16)
    a = orc.eval_batch(coords, y, X, P, lam, nthreads=1)
    b = orc.eval_batch(coords, y, X, P, lam, nthreads=5)
    for k in ("loglik", "betahat", "sigma2hat", "logdetV", "status"):
        assert np.array_equal(a[k], b[k])


# --------------------------------------------------------------------------- REML (Appendix)
def test_spec_n3_reml_example(orc):
    g = _gold("spec_n3_ols.json")
    coords = _far_sites(3, np.random.default_rng(0))
    y = np.array(g["y_prime"]) + 1.0
    out = orc.eval_batch(coords, y, np.ones((3, 1)), [[1.0, 0.7, 0.0, 1.0, 0.0]], [1.0], summaries=True)
    assert out["sigma2_reml"][0, 0] == pytest.approx(g["sigma2hat_reml"], rel=1e-15)
    assert -2 * out["loglik_reml"][0, 0] == pytest.approx(g["minus2_loglik_reml"], rel=1e-15)
    assert out["detReml"][0] == pytest.approx(math.log(3.0), rel=1e-15)


def test_reml_searle_identities(orc):
    """Appendix: with an explicit full-rank contrast A (AX = 0, orthonormal
    rows, scipy null space), y* = A y' and the exact REML likelihood of y*,
      y*ᵀ(AVAᵀ)⁻¹y* = (y'−Xβ̂)ᵀV⁻¹(y'−Xβ̂)                 (Searle, 2nd identity)
      −2ℓ*_p(paper) − (−2ℓ*_p(y*)) + 2(λ−1)Σ log y = p log 2π + log|XᵀX|
    (the paper's |AVAᵀ| = |V||XᵀV⁻¹X| holds up to the constant |XᵀX|⁻¹ for orthonormal A).
    V from the κ = 3/2 closed form (no Bessel), dense linear algebra from numpy."""
    coords, y, X = synthgen.make_dataset("C1")
    n, p = X.shape
    A = sla.null_space(X.T).T  # (n−p) × n, orthonormal rows, A X = 0
    const = p * math.log(2 * math.pi) + np.linalg.slogdet(X.T @ X)[1]
    lam = [0.25, 0.9]
    for w in ([900.0, 1.5, 0.2, 1.0, 0.0], [400.0, 1.5, 0.7, 1.0, 0.0]):
        out = orc.eval_batch(coords, y, X, [w], lam, summaries=True)
        D = np.sqrt(((coords[:, None, :] - coords[None, :, :]) ** 2).sum(-1)) / w[0]
        z = math.sqrt(12) * D
        V = (1 + z) * np.exp(-z) + w[2] * np.eye(n)
        AVA = A @ V @ A.T
        for m, l in enumerate(lam):
            yp = (y ** l - 1) / l
            ys = A @ yp
            qstar = ys @ np.linalg.solve(AVA, ys)
            assert qstar == pytest.approx(out["qdirect"][0, m], rel=1e-10)
            s2 = qstar / (n - p)
            assert out["sigma2_reml"][0, m] == pytest.approx(s2, rel=1e-10)
            m2l_exact = (n - p) * math.log(s2) + np.linalg.slogdet(AVA)[1] + (n - p) * (1 + math.log(2 * math.pi))
            jac = -2 * (l - 1) * np.log(y).sum()
            assert -2 * out["loglik_reml"][0, m] - m2l_exact - jac == pytest.approx(const, abs=1e-9)
        # detReml = log|XᵀV⁻¹X| (Table 1)
        assert out["detReml"][0] == pytest.approx(np.linalg.slogdet(X.T @ np.linalg.solve(V, X))[1], rel=1e-11)
        # ssqYX blocks (Table 1): y'ᵀV⁻¹y' on the diagonal, XᵀV⁻¹X lower-right, XᵀV⁻¹y' lower-left
        B = np.column_stack([(y ** l - 1) / l for l in lam] + [X])
        np.testing.assert_allclose(out["ssqYX"][0], B.T @ np.linalg.solve(V, B), rtol=1e-10)


# --------------------------------------------------------------------------- profiles (§3.4-3.6)
def _closed_form_case(K=3, M=2, seed=5):
    """C1 sites, κ = 3/2 closed-form V (no Bessel) for an independent brute force."""
    coords, y, X = synthgen.make_dataset("C1")
    rng = np.random.default_rng(seed)
    P = np.column_stack([rng.uniform(500, 1500, K), np.full(K, 1.5), rng.uniform(0.1, 0.8, K),
                         np.ones(K), np.zeros(K)])
    lam = np.linspace(0.3, 0.7, M)
    return coords, y, X, P, lam


def _V32(coords, w):
    D = np.sqrt(((coords[:, None, :] - coords[None, :, :]) ** 2).sum(-1)) / w[0]
    z = math.sqrt(12) * D
    return (1 + z) * np.exp(-z) + w[2] * np.eye(len(coords))


def test_beta_profile_vs_direct_maximisation(orc):
    """ℓ_p(β_a = b) equals max over (k, m) of the full log-likelihood Eq. 2
    maximised numerically over β_{−a} and σ² at β_a = b (scipy, explicit V)."""
    import scipy.optimize as so
    coords, y, X, P, lam = _closed_form_case()
    n, p = X.shape
    out = orc.eval_batch(coords, y, X, P, lam, summaries=True)
    bh = out["betahat"][0, 0]
    grid = np.stack([v + np.array([-0.3, 0.05, 0.4]) * max(1.0, abs(v)) for v in bh])
    prof, _, _ = orc.profiles(n, p, out["ssqYX"], out["logdetV"], out["status"], lam, y, grid, [1.0])
    for a in range(p):
        for g, b in enumerate(grid[a]):
            best = -np.inf
            for k in range(len(P)):
                V = _V32(coords, P[k])
                Vi = np.linalg.inv(V)
                ld = np.linalg.slogdet(V)[1]
                for m, l in enumerate(lam):
                    yp = (y ** l - 1) / l
                    keep = [i for i in range(p) if i != a]

                    def nll(th):
                        beta = np.empty(p)
                        beta[a] = b
                        beta[keep] = th[:-1]
                        s2 = math.exp(th[-1])
                        r = yp - X @ beta
                        return 0.5 * (r @ Vi @ r / s2 + n * math.log(s2) + ld + n * math.log(2 * math.pi)) \
                            - (l - 1) * np.log(y).sum()
                    x0 = np.append(bh[keep], math.log(out["sigma2hat"][k, m]))
                    res = so.minimize(nll, x0, method="BFGS", options=dict(gtol=1e-10))
                    best = max(best, -res.fun)
            assert prof[a, g] == pytest.approx(best, rel=1e-7, abs=1e-7)


def test_sigma_and_lambda_profiles(orc):
    """σ profile vs the scipy multivariate-normal density at (β̂, σ²V) maximised
    over the grid; λ profile = max_k ℓ_p(ω_k, λ_m); both peak at the global maximum."""
    coords, y, X, P, lam = _closed_form_case(K=2, M=3)
    n, p = X.shape
    out = orc.eval_batch(coords, y, X, P, lam, summaries=True)
    sig = np.array([0.5, 1.0, 2.0, float(np.sqrt(out["sigma2hat"][0, 1]))])
    _, ps, pl = orc.profiles(n, p, out["ssqYX"], out["logdetV"], out["status"], lam, y,
                             np.zeros((p, 1)), sig)
    np.testing.assert_allclose(pl, out["loglik"].max(axis=0), rtol=1e-12)
    for t, s in enumerate(sig):
        best = -np.inf
        for k in range(len(P)):
            V = _V32(coords, P[k])
            for m, l in enumerate(lam):
                yp = (y ** l - 1) / l
                ll = sst.multivariate_normal(mean=X @ out["betahat"][k, m], cov=s * s * V).logpdf(yp) \
                    + (l - 1) * np.log(y).sum()
                best = max(best, ll)
        assert ps[t] == pytest.approx(best, rel=1e-10)
    assert ps.max() <= out["loglik"].max() + 1e-9
