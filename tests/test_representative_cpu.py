"""Representative points (paper Step 2) and profile curves / CIs
(P:168-173): host logic, pinned against closed forms and the oracle.
SURVEY §8(f) NEXT-3 / NEXT-4."""
import math

import numpy as np
import pytest

from paper_2305_04318_b200 import representative as rp


# ------------------------------------------------------------------ reparametrisation (R21)
@pytest.mark.parametrize("regime", ["log", "invroot"])
def test_internal_round_trip(regime):
    rng = np.random.default_rng(3)
    nat = np.column_stack([rng.uniform(50, 5000, 40), rng.uniform(0.3, 20, 40), rng.uniform(0, 2, 40),
                           rng.uniform(1.0, 8.0, 40), rng.uniform(-math.pi / 2, math.pi / 2, 40)])
    back = rp.to_natural(rp.to_internal(nat, regime), regime)
    np.testing.assert_allclose(back, nat, rtol=1e-12, atol=1e-12)


def test_internal_coordinates_closed_form():
    """γ1 = log φX + log φY, γ2 = √(φR−1)cos 2φA, γ3 = √(φR−1)sin 2φA, ν = √ν²,
    κ̃ = log κ (κ̂ < 4) or κ^{−1/2}."""
    nat = np.array([200.0, 9.0, 0.25, 5.0, math.pi / 8])
    w_inv = rp.to_internal(nat, rp.kappa_regime(9.0))[0]
    w_log = rp.to_internal(nat, rp.kappa_regime(1.5))[0]
    phiY = 200.0 / 5.0
    np.testing.assert_allclose(w_inv, [math.log(200 * phiY), 1 / 3, 0.5, 2 * math.cos(math.pi / 4),
                                       2 * math.sin(math.pi / 4)], rtol=1e-14)
    assert w_log[1] == pytest.approx(math.log(9.0))


def test_phiR_below_one_is_the_same_model(orc):
    """R21: (φX, φR, φA) and (φX/φR, 1/φR, φA + π/2) give the same V (checked with the
    oracle's literal distance matrix)."""
    rng = np.random.default_rng(5)
    coords = rng.uniform(0, 1000, size=(30, 2))
    nat = np.array([[300.0, 1.5, 0.3, 0.4, 0.7]])
    w = rp.to_internal(nat, "log")
    nat2 = rp.to_natural(w, "log")
    assert nat2[0, 3] > 1.0
    np.testing.assert_allclose(orc.build_V(coords, nat2[0]), orc.build_V(coords, nat[0]), rtol=1e-12, atol=1e-14)


# ------------------------------------------------------------------ Hessian stencil (R22)
@pytest.mark.parametrize("d, npts", [(5, 51), (4, 33)])
def test_stencil_size(d, npts):
    assert len(rp.stencil(np.zeros(d), np.ones(d))) == npts


def test_hessian_of_quadratic_is_exact():
    """A quadratic's central differences are exact (up to rounding)."""
    rng = np.random.default_rng(0)
    A = rng.normal(size=(5, 5))
    H = A + A.T
    g = rng.normal(size=5)
    c = rng.normal(size=5)
    f = lambda x: 0.5 * (x - c) @ H @ (x - c) + g @ x
    delta = np.array([1e-2, 2e-2, 5e-3, 1e-2, 3e-2])
    pts = rp.stencil(np.ones(5), delta)
    Hn = rp.hessian_from_stencil(np.array([f(x) for x in pts]), delta)
    np.testing.assert_allclose(Hn, H, atol=1e-8)


def test_hessian_of_smooth_function():
    """Second-order accuracy on a non-polynomial function (closed-form Hessian)."""
    f = lambda x: math.exp(x[0]) * math.sin(x[1]) + x[2] ** 4 + x[0] * x[3] ** 3
    x0 = np.array([0.3, 0.7, 1.1, -0.4])
    Hx = np.array([[math.exp(.3) * math.sin(.7), math.exp(.3) * math.cos(.7), 0, 3 * .16],
                   [math.exp(.3) * math.cos(.7), -math.exp(.3) * math.sin(.7), 0, 0],
                   [0, 0, 12 * 1.21, 0],
                   [3 * .16, 0, 0, 6 * .3 * -.4]])
    delta = 1e-3 * np.ones(4)
    Hn = rp.hessian_from_stencil(np.array([f(x) for x in rp.stencil(x0, delta)]), delta)
    np.testing.assert_allclose(Hn, Hx, atol=1e-5)


# ------------------------------------------------------------------ eigen repair (R23)
def test_repair_eigenvalues_examples():
    np.testing.assert_array_equal(rp.repair_eigenvalues([4, -3, 2]), [4, 3, 2])
    np.testing.assert_array_equal(rp.repair_eigenvalues([150, 0.01, 5]), [150, 0.1, 5])
    np.testing.assert_array_equal(rp.repair_eigenvalues([50, 0.01, -5]), [50, 0.01, 5])


# ------------------------------------------------------------------ sphere + contours (R24)
def test_sphere_points_spread_and_seeded():
    s = rp.sphere_points(5, 200, seed=1)
    np.testing.assert_allclose(np.linalg.norm(s, axis=1), 1.0, rtol=1e-14)
    np.testing.assert_array_equal(s, rp.sphere_points(5, 200, seed=1))
    r = np.random.default_rng(1).normal(size=(200, 5))
    r /= np.linalg.norm(r, axis=1, keepdims=True)
    assert rp.min_distance(s) > 3 * rp.min_distance(r)


def test_sphere_points_small_cases_reach_the_optimum():
    """4 points on a circle: a square (min distance √2); 6 on S² : octahedron (√2)."""
    assert rp.min_distance(rp.sphere_points(2, 4, seed=0, iters=400)) == pytest.approx(math.sqrt(2), rel=2e-3)
    assert rp.min_distance(rp.sphere_points(3, 6, seed=0, iters=400)) == pytest.approx(math.sqrt(2), rel=2e-2)


def test_chi2_quantile():
    assert rp.chi2_quantile(1, 0.05) == pytest.approx(1.959963984540054 ** 2, rel=1e-12)
    assert rp.chi2_quantile(2, 0.1) == pytest.approx(-2 * math.log(0.1), rel=1e-12)  # χ²_2 = Exp(½)


def test_contour_points_lie_on_the_quadratic_form():
    """(ω'−ω̂')ᵀ(−H)(ω'−ω̂') = c_α for every contour point (R24)."""
    rng = np.random.default_rng(2)
    A = rng.normal(size=(5, 5))
    negH = A @ A.T + 0.5 * np.eye(5)
    center = rng.normal(size=5)
    sph = rp.sphere_points(5, 60, seed=4)
    pts, lab = rp.contour_points(center, negH, rp.DEFAULT_ALPHAS, sph)
    assert pts.shape == (60 * 12, 5)
    dv = pts - center
    qf = np.einsum("ki,ij,kj->k", dv, negH, dv)
    c = np.array([rp.chi2_quantile(5, a) for a in lab])
    np.testing.assert_allclose(qf, c, rtol=1e-8)


def test_contour_points_use_the_repaired_hessian():
    negH = np.diag([400.0, 0.01, -2.0, 1.0])  # repaired: (400, 0.1, 2, 1)
    sph = rp.sphere_points(4, 30, seed=0)
    pts, lab = rp.contour_points(np.zeros(4), negH, [0.5], sph)
    qf = np.einsum("ki,ij,kj->k", pts, np.diag([400.0, 0.1, 2.0, 1.0]), pts)
    np.testing.assert_allclose(qf, rp.chi2_quantile(4, 0.5), rtol=1e-8)
    np.testing.assert_allclose(rp.repaired_neg_hessian(negH), np.diag([400.0, 0.1, 2.0, 1.0]), atol=1e-12)


# ------------------------------------------------------------------ nugget + λ grid
def test_repair_nugget():
    rng = np.random.default_rng(0)
    nu = np.array([0.5, -0.1, -0.2, 0.3, -0.7, -1.0, -0.05])
    nug = rp.repair_nugget(nu, rng)
    neg = nu < 0
    np.testing.assert_allclose(nug[~neg], nu[~neg] ** 2)
    assert int(np.sum(nug[neg] == 0.0)) == 2          # floor(5/2) set to zero
    rest = nug[neg][nug[neg] != 0.0]
    assert len(rest) == 3 and np.all((rest > 0) & (rest < 2))


def test_lambda_grid():
    g = rp.lambda_grid(0.4, -100.0, 9)
    sd, z = 0.1, 2.3263478740408408
    assert 0.4 in g and len(g) == 9  # λ̂ is the middle node
    assert g[0] == pytest.approx(0.4 - z * sd) and g[-1] == pytest.approx(0.4 + z * sd)
    assert len(rp.lambda_grid(0.33, -100.0, 8)) == 9
    np.testing.assert_array_equal(rp.lambda_grid(0.5, -1.0, 1), [0.5])


# ------------------------------------------------------------------ configure_params driver
class QuadraticCtx:
    """Stands in for the GPU context: ℓ = −½(ω'−w*)ᵀA(ω'−w*) + b(λ−λ*)² in internal
    coordinates, so the stencil Hessian must come back as −A and the λ curvature 2b."""

    def __init__(self, A, wstar, regime, b=-30.0, lam_star=0.3):
        self.A, self.wstar, self.regime, self.b, self.lam_star = A, wstar, regime, b, lam_star
        self.calls = 0

    def eval_batch(self, coords, y, X, params, lambdas):
        self.calls += 1
        w = rp.to_internal(params, self.regime)
        dv = w - self.wstar
        base = -0.5 * np.einsum("ki,ij,kj->k", dv, self.A, dv)
        ll = base[:, None] + self.b * (np.asarray(lambdas)[None, :] - self.lam_star) ** 2
        return {"loglik": ll, "status": np.zeros(len(params), dtype=np.int32)}


def test_configure_params_recovers_the_hessian_and_counts():
    nat0 = np.array([800.0, 1.2, 0.5, 2.0, 0.3])
    regime = rp.kappa_regime(nat0[1])
    w0 = rp.to_internal(nat0, regime)[0]
    rng = np.random.default_rng(8)
    B = rng.normal(size=(5, 5))
    A = B @ B.T + np.eye(5)
    ctx = QuadraticCtx(A, w0, regime)
    fits = [rp.Fit(nat0, 0.3), rp.Fit(nat0, 0.3, kappa_fixed=1.2)]
    rs = rp.configure_params(ctx, None, None, None, fits, n5=40, n4=20, m_lambda=7)
    assert ctx.calls == 1  # all stencils in one batched call
    np.testing.assert_allclose(rs.neg_hessians[0], A, rtol=1e-5, atol=1e-5 * np.abs(A).max())
    A4 = np.delete(np.delete(A, 1, 0), 1, 1)
    np.testing.assert_allclose(rs.neg_hessians[1], A4, rtol=1e-5, atol=1e-5 * np.abs(A).max())
    assert rs.lambda_curvature == pytest.approx(-60.0, rel=1e-6)
    assert rs.params.shape == (12 * 40 + 12 * 20 + 2, 5)
    assert np.all(rs.params[:, 2] >= 0) and np.all(rs.params[:, 3] >= 1.0)
    np.testing.assert_allclose(rs.params[12 * 40:12 * 60, 1], 1.2)  # κ held fixed
    assert 0.3 in rs.lambdas and len(rs.lambdas) == 7


# ------------------------------------------------------------------ profiles + CIs (NEXT-4)
def test_upper_hull_dominates_and_is_concave():
    rng = np.random.default_rng(1)
    x = rng.uniform(-3, 3, 500)
    y = -x ** 2 - rng.exponential(2.0, 500)
    hx, hy = rp.upper_hull(x, y)
    curve = np.interp(x, hx, hy)
    assert np.all(curve >= y - 1e-12)
    slopes = np.diff(hy) / np.diff(hx)
    assert np.all(np.diff(slopes) <= 1e-12)
    assert hy.max() == y.max()


def test_hull_of_concave_samples_is_the_samples():
    x = np.linspace(-2, 2, 41)
    hx, hy = rp.upper_hull(x, -x ** 2)
    np.testing.assert_array_equal(hx, x)


def test_likelihood_ci_of_a_quadratic_profile():
    """ℓ_p(θ) = −(θ−μ)²/(2s²): the 95% likelihood CI is μ ± 1.95996 s."""
    mu, s = 1.3, 0.2
    th = np.linspace(0, 3, 3001)
    rng = np.random.default_rng(0)
    ll = -(th - mu) ** 2 / (2 * s * s)
    # add dominated points (the profile takes the max over the other parameters)
    th2 = np.concatenate([th, rng.uniform(0, 3, 2000)])
    ll2 = np.concatenate([ll, -(th2[3001:] - mu) ** 2 / (2 * s * s) - rng.exponential(1, 2000)])
    hx, hy, f = rp.profile_1d(th2, ll2)
    best, lo, hi = rp.likelihood_ci(hx, hy, 0.95)
    assert best == pytest.approx(mu, abs=1e-3)
    assert lo == pytest.approx(mu - 1.959963984540054 * s, abs=1e-5)
    assert hi == pytest.approx(mu + 1.959963984540054 * s, abs=1e-5)


def test_likelihood_ci_open_end_reports_the_boundary():
    th = np.linspace(0, 1, 11)
    hx, hy, _ = rp.profile_1d(th, -0.1 * th)
    best, lo, hi = rp.likelihood_ci(hx, hy, 0.95)
    assert (best, lo, hi) == (0.0, 0.0, 1.0)


def test_profile_2d_concave_surface():
    rng = np.random.default_rng(0)
    a = rng.uniform(-1, 1, 400)
    b = rng.uniform(-1, 1, 400)
    f = -(a ** 2) - 2 * b ** 2 + 0.5 * a * b
    extra_a, extra_b = rng.uniform(-1, 1, 300), rng.uniform(-1, 1, 300)
    g = -(extra_a ** 2) - 2 * extra_b ** 2 + 0.5 * extra_a * extra_b - rng.exponential(0.5, 300)
    A, B, L = np.concatenate([a, extra_a]), np.concatenate([b, extra_b]), np.concatenate([f, g])
    surf = rp.profile_2d(A, B, L, np.column_stack([A, B]))
    ok = np.isfinite(surf)
    assert ok.mean() > 0.9
    assert np.all(surf[ok] >= L[ok] - 1e-9)  # upper facets dominate every sample
    q = np.array([[0.0, 0.0], [0.3, -0.2]])
    exact = -(q[:, 0] ** 2) - 2 * q[:, 1] ** 2 + 0.5 * q[:, 0] * q[:, 1]
    np.testing.assert_allclose(rp.profile_2d(A, B, L, q), exact, atol=0.05)
    assert np.isnan(rp.profile_2d(A, B, L, np.array([[5.0, 5.0]]))[0])


def test_configure_params_paper_shapes():
    """The paper's point counts (R26): Swiss 15,318 = 6 + 12·726 + 5·11·120;
    soil 12,316 = 4 + 12·726 + 3·10·120."""
    nat0 = np.array([800.0, 1.2, 0.5, 2.0, 0.3])
    regime = rp.kappa_regime(nat0[1])
    ctx = QuadraticCtx(np.eye(5), rp.to_internal(nat0, regime)[0], regime)
    for kfix, nlev, total in (((0.5, 0.9, 10.0, 20.0, 100.0), 11, 15318), ((0.5, 0.8, 1.0), 10, 12316)):
        fits = [rp.Fit(nat0, 0.3)] + [rp.Fit(np.r_[nat0[0], k, nat0[2:]], 0.3, kappa_fixed=k) for k in kfix]
        rs = rp.configure_params(ctx, None, None, None, fits, alphas_fixed=rp.DEFAULT_ALPHAS[12 - nlev:])
        assert rs.params.shape == (total, 5)
