"""Representative points on the GPU (paper Step 2):
the stencil Hessian from CUDA likelihoods vs the same stencil evaluated by the
oracle, and the whole Step-2 → Step-3 → profile pipeline with sampled parity."""
import math
import os

import numpy as np
import pytest

import synthgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2305_04318_b200 as lik  # noqa: E402
from paper_2305_04318_b200 import representative as rp  # noqa: E402

NTHREADS = os.cpu_count() or 8


class Recorder:
    """Wraps an eval_batch provider and keeps the stencil values it returned."""

    def __init__(self, fn):
        self.fn, self.ll = fn, []

    def eval_batch(self, coords, y, X, params, lambdas):
        r = self.fn(coords, y, X, params, lambdas)
        self.ll.append(r["loglik"].copy())
        return r


def assert_status_or_borderline(orc, coords, params, st_g, st_r):
    """Statuses must agree, except where the R11 non-PD decision (pivot ≤ n·ε·max V_ii,
    P:853) sits within rounding of its threshold: nugget-repaired points (ν² = 0,
    P:277) with long ranges give nearly singular V, and the two sides factor it by
    different FP64 algorithms (blocked LLᵀ vs unblocked LDLᵀ, R10), so a pivot within
    a few n·ε·‖V‖ of the threshold may land on either side."""
    n = coords.shape[0]
    for i in np.nonzero(st_g != st_r)[0]:
        assert {int(st_g[i]), int(st_r[i])} == {lik.PT_OK, lik.PT_V_NOT_PD}, (i, st_g[i], st_r[i])
        _, D, _ = orc.ldl(orc.build_V(coords, params[i]))
        tol = n * np.finfo(float).eps * (1.0 + params[i][2])
        dmin = D[D != 0].min() if np.any(D != 0) else 0.0
        assert dmin < 100 * tol, (i, params[i], dmin / tol)


@pytest.fixture(scope="module")
def ctx():
    c = lik.create(0)
    yield c
    c.close()


def _truth(cfg):
    iso = synthgen.CONFIGS[cfg].iso
    phiX = 50_000.0 if synthgen.CONFIGS[cfg].layout == "villages" else 1000.0
    return np.array([phiX, 2.0, 0.64, 1.0 if iso else 2.0, 0.0 if iso else 0.2])


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_stencil_hessian_matches_oracle(ctx, orc, cfg):
    coords, y, X = synthgen.make_dataset(cfg)
    fits = [rp.Fit(_truth(cfg), 0.5), rp.Fit(_truth(cfg), 0.5, kappa_fixed=2.0)]
    g = Recorder(ctx.eval_batch)
    o = Recorder(lambda *a: orc.eval_batch(*a, nthreads=NTHREADS))
    rs_g = rp.configure_params(g, coords, y, X, fits, n5=20, n4=12, m_lambda=9)
    rs_o = rp.configure_params(o, coords, y, X, fits, n5=20, n4=12, m_lambda=9)
    assert len(g.ll) == len(o.ll) == 1  # one batched call for all fits' stencils
    for f_i, fit in enumerate(fits):
        e = np.abs(rs_g.stencil_loglik[f_i] - rs_o.stencil_loglik[f_i])
        assert (e / np.abs(rs_o.stencil_loglik[f_i])).max() <= 1e-8  # the stencil values themselves
        w0 = rp.to_internal(fit.natural, rp.kappa_regime(fit.natural[1]))[0]
        if fit.kappa_fixed is not None:
            w0 = np.delete(w0, 1)
        delta = 1e-3 * np.maximum(1.0, np.abs(w0))
        # central-difference error propagation: |ΔH_ii| ≤ 4e/δ_i², |ΔH_ij| ≤ e/(δ_i δ_j)
        emax = e[:, 1].max()
        bound = emax / np.outer(delta, delta) * (1.0 + 3.0 * np.eye(len(delta))) + 1e-12
        dH = np.abs(rs_g.neg_hessians[f_i] - rs_o.neg_hessians[f_i])
        assert np.all(dH <= bound), (f_i, dH.max(), bound.min())
        # the contour map uses the repaired eigenvalues; |·| and the 0.1 clamp are
        # 1-Lipschitz, so by Weyl |Δd_i| ≤ ‖ΔH‖_2 ≤ ‖ΔH‖_F (the points themselves scale
        # with d^{−1/2} and are ill-conditioned when −H is nearly singular)
        dg = np.sort(rp.repair_eigenvalues(np.linalg.eigvalsh(rs_g.neg_hessians[f_i])))
        do = np.sort(rp.repair_eigenvalues(np.linalg.eigvalsh(rs_o.neg_hessians[f_i])))
        assert np.all(np.abs(dg - do) <= np.linalg.norm(bound) + 1e-12)
    # λ curvature (R22): |Δ| ≤ 4e/δ_λ²
    dl = 1e-3 * max(1.0, 0.5)
    e0 = np.abs(rs_g.stencil_loglik[0][0] - rs_o.stencil_loglik[0][0]).max()
    assert abs(rs_g.lambda_curvature - rs_o.lambda_curvature) <= 4 * e0 / dl ** 2 + 1e-12
    assert len(rs_g.params) == len(rs_o.params) == 12 * 20 + 12 * 12 + 2


def test_representative_pipeline_profiles(ctx, orc):
    """Step 2 on the GPU, Step 3 (the batched evaluation) on the GPU, 1-D λ profile and
    its likelihood CI; sampled parity of the evaluated grid vs the oracle."""
    coords, y, X = synthgen.make_dataset("C2")
    fits = [rp.Fit(_truth("C2"), 0.5)]
    rs = rp.configure_params(ctx, coords, y, X, fits, n5=40, m_lambda=9)
    res = ctx.eval_batch(coords, y, X, rs.params, rs.lambdas)
    assert res["status"].shape == (len(rs.params),)
    assert np.mean(res["status"] == 0) > 0.95
    sel = np.random.default_rng(0).choice(len(rs.params), 24, replace=False)
    ref = orc.eval_batch(coords, y, X, rs.params[sel], rs.lambdas, nthreads=NTHREADS)
    st_g = res["status"][sel]
    assert_status_or_borderline(orc, coords, rs.params[sel], st_g, ref["status"])
    ok = (ref["status"] == 0) & (st_g == 0)
    rel = np.abs(res["loglik"][sel][ok] - ref["loglik"][ok]) / np.abs(ref["loglik"][ok])
    assert rel.max() <= 1e-8
    # λ profile: max over points of ℓ_p(ω_k, λ_m), then the CI
    llk = np.where(res["status"][:, None] == 0, res["loglik"], -np.inf)
    prof_l = llk.max(axis=0)
    hx, hy, _ = rp.profile_1d(rs.lambdas, prof_l)
    best, lo, hi = rp.likelihood_ci(hx, hy, 0.95)
    assert lo <= best <= hi
    assert 0.0 < best < 1.0  # data generated with λ = 0.5 (synthgen.LAMBDA0)
    # φX profile over the representative cloud (max over λ per point)
    hx, hy, _ = rp.profile_1d(np.log(rs.params[:, 0]), llk.max(axis=1))
    best, lo, hi = rp.likelihood_ci(hx, hy, 0.95)
    assert lo <= best <= hi and math.isfinite(best)
