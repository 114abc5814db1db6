"""GPU tests (-m gpu), through the C ABI:

* the constructed Step-5 and Step-8 failures of tests/constructed.py (XVX_NOT_PD and
  NEG_RESID, R12) — statuses, failed columns and the valid column vs the
  oracle; the β/σ/λ profiles of a NEG_RESID batch vs the oracle's;
* the Matérn build against mpmath (ρ = 2^{1−κ}/Γ(κ) z^κ K_κ(z) at 50 digits,
  Eq. matern), not against the oracle, on a (κ, z) grid at R8's bar
  2e-14·max(1, |ln ρ|);
* ordering of calls on one context enqueued on different streams (shared workspace).
"""
import math
import os

import numpy as np
import pytest

import constructed
import synthgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2305_04318_b200 as lik  # noqa: E402
from test_gpu_parity import assert_parity  # noqa: E402

NTHREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def ctx():
    c = lik.create(0)
    yield c
    c.close()


def test_xvx_not_pd_constructed(ctx, orc):
    coords, y, X, P, lam, _ = constructed.xvx_singular()
    gpu = ctx.eval_batch(coords, y, X, P, lam)
    ref = orc.eval_batch(coords, y, X, P, lam, nthreads=NTHREADS)
    assert list(gpu["status"]) == [lik.PT_XVX_NOT_PD] * P.shape[0]
    assert_parity(gpu, ref, label="xvx")
    assert np.all(np.isneginf(gpu["loglik"])) and np.all(np.isnan(gpu["betahat"]))
    assert np.all(np.isnan(gpu["sigma2hat"])) and np.all(np.isnan(gpu["logdetV"]))


def test_neg_resid_constructed(ctx, orc):
    coords, y, X, P, lam = constructed.resid_in_span()
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    ex = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device_ex(*t).items()}
    ref = orc.eval_batch(coords, y, X, P, lam, nthreads=NTHREADS, summaries=True)
    assert list(ex["status"]) == [lik.PT_NEG_RESID] * P.shape[0]
    assert_parity(ex, ref, label="neg_resid")
    # column 0 failed (R12), column 1 valid on both sides; no +inf anywhere
    assert np.all(np.isneginf(ex["loglik"][:, 0])) and np.all(np.isfinite(ex["loglik"][:, 1]))
    assert not np.any(np.isposinf(ex["loglik"])) and not np.any(np.isposinf(ex["loglik_reml"]))
    assert np.all(np.abs(ex["ssqResidual"][:, 0]) <= 1e-10 * ex["ssqYX"][:, 0, 0])
    # the summaries of a NEG_RESID point are valid (Table 1)
    sc = np.abs(ref["ssqYX"]).max(axis=(1, 2), keepdims=True)
    assert (np.abs(ex["ssqYX"] - ref["ssqYX"]) / sc).max() <= 1e-8
    # profiles: the failed column is skipped, the valid one used (GPU vs oracle)
    n, p = X.shape
    grid = np.stack([np.linspace(-2.0, 4.0, 9) for _ in range(p)])
    sig = np.sqrt(np.linspace(0.5, 2.0, 5) * np.nanmedian(ref["sigma2hat"]))
    summ = ctx.eval_batch_device_ex(*t)
    pb, ps, pl = ctx.profiles_device(n, t[1], summ, t[4], torch.tensor(grid, device="cuda"),
                                     torch.tensor(sig, device="cuda"))
    torch.cuda.synchronize()
    rb, rs, rl = orc.profiles(n, p, ref["ssqYX"], ref["logdetV"], ref["status"], lam, y, grid, sig)
    pl = pl.cpu().numpy()
    assert np.isneginf(pl[0]) and np.isneginf(rl[0])
    assert abs(pl[1] - rl[1]) <= 1e-8 * abs(rl[1])
    assert np.all(np.abs(pb.cpu().numpy() - rb) <= 1e-8 * np.abs(rb))
    assert np.all(np.abs(ps.cpu().numpy() - rs) <= 1e-8 * np.abs(rs))


# --------------------------------------------------------------------------- ρ vs mpmath
KAPPAS = [0.05, 0.37, 1.83, 47.3, 100.0, 200.0, 0.5, 2.5, 10.0, 999.0]


def _mp_log_rho(kappa, z):
    import mpmath
    mpmath.mp.dps = 50
    k, z = mpmath.mpf(kappa), mpmath.mpf(z)
    return (1 - k) * mpmath.log(2) - mpmath.loggamma(k) + k * mpmath.log(z) + mpmath.log(mpmath.besselk(k, z))


@pytest.mark.parametrize("n", [61, 300])  # both table layouts (whole octaves below n = 256, quarters above)
def test_matern_build_vs_mpmath(ctx, n):
    """V[i, 0] = ρ(z_i) for sites on a line at x_i (φX = √(8κ), isotropic, so
    z_i = √(8κ)·x_i/φX ≈ x_i), z ∈ [1e-8, 700] log-spaced — through the table and the
    exact path of the build — against mpmath at 50 digits, at R8's bar
    |Δρ| ≤ 2e-14·max(1, |ln ρ|)·ρ for ρ ≥ 1e-290; where ln ρ < −745 the GPU gives
    ρ < 1e-300 (R8: ρ := 0, or an underflowing subnormal)."""
    import mpmath
    zs = np.r_[0.0, np.geomspace(1e-8, 700.0, n - 1)]
    coords = np.column_stack([zs, np.zeros(n)])
    worst = 0.0
    for kappa in KAPPAS:
        phiX = math.sqrt(8.0 * kappa)
        P = np.array([[phiX, kappa, 0.0, 1.0, 0.0]])
        V = ctx.debug_build_V(torch.tensor(coords, device="cuda"), torch.tensor(P, device="cuda"))
        col = V.cpu().numpy()[0][:, 0]
        assert col[0] == 1.0
        for i in range(1, n, 1 if n < 100 else 3):
            mpmath.mp.dps = 50
            z = mpmath.sqrt(8 * mpmath.mpf(kappa)) * mpmath.mpf(float(zs[i])) / mpmath.mpf(phiX)
            if kappa >= 1e3:  # R7: the Gaussian limit exp(−2d²), d = x_i/φX
                lr = -2 * (mpmath.mpf(float(zs[i])) / mpmath.mpf(phiX)) ** 2
            else:
                lr = _mp_log_rho(kappa, z)
            if lr < -745:
                assert col[i] < 1e-300, (kappa, zs[i], col[i])
                continue
            rho = float(mpmath.exp(lr))
            if rho < 1e-290:
                continue
            err = abs(col[i] - rho) / rho / max(1.0, abs(float(lr)))
            worst = max(worst, err)
            assert err <= 2e-14, (kappa, float(zs[i]), col[i], rho, err)
    print(f"n={n}: worst |Δρ|/ρ/max(1,|ln ρ|) = {worst:.2e}")


# --------------------------------------------------------------------------- streams
def test_calls_on_different_streams_are_ordered(ctx):
    """Two calls on one context enqueued back to back on different streams (no host
    synchronisation in between) share the workspace; each must equal its result computed
    alone (the second call waits for the first one's event)."""
    coords, y, X, P, lam = synthgen.make_inputs("C3", K=600)
    P2 = np.ascontiguousarray(P[::-1])
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    p2 = torch.tensor(P2, device="cuda")
    a = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(*t).items()}
    b = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(t[0], t[1], t[2], p2, t[4]).items()}
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        o1 = ctx.eval_batch_device(*t, stream=s1)
        o2 = ctx.eval_batch_device(t[0], t[1], t[2], p2, t[4], stream=s2)
        o3 = ctx.eval_batch(coords, y, X, P, lam)  # host API on the context's own stream
        torch.cuda.synchronize()
        for key in a:
            assert np.array_equal(o1[key].cpu().numpy(), a[key], equal_nan=True), key
            assert np.array_equal(o2[key].cpu().numpy(), b[key], equal_nan=True), key
            assert np.array_equal(o3[key], a[key], equal_nan=True), key


# --------------------------------------------------------------------------- small path
@pytest.mark.parametrize("name,K", [("C1", 16), ("C2", 400), ("swiss", 300)])
def test_small_path_matches_fused_path(name, K):
    """chol_small (build + factor of the whole augmented matrix in shared memory, taken
    for n_pad + r_pad ≤ 216) against chol_fused (64-tiles through HBM, LIK_NO_SMALL) on
    the same inputs: two independent factorisations agree to rounding."""
    if name == "swiss":  # the paper's Swiss-rainfall shape: n = 100, p = 2, M = 34
        cfg = synthgen.Config("sw", 100, 2, K, 34, True, "uniform", "swiss-shaped")
        coords, y, X = synthgen.make_dataset(cfg, seed=5)
        P, lam = synthgen.make_params(cfg, K, seed=6), np.linspace(-1.0, 2.0, 34)
    else:
        coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
    a = lik.create(0).eval_batch(coords, y, X, P, lam)
    os.environ["LIK_NO_SMALL"] = "1"
    try:
        c = lik.create(0)
    finally:
        del os.environ["LIK_NO_SMALL"]
    b = c.eval_batch(coords, y, X, P, lam)
    c.close()
    assert np.array_equal(a["status"], b["status"])
    ok = a["status"] == 0
    np.testing.assert_allclose(a["loglik"][ok], b["loglik"][ok], rtol=1e-11)
    np.testing.assert_allclose(a["logdetV"][ok], b["logdetV"][ok], rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(a["sigma2hat"][ok], b["sigma2hat"][ok], rtol=1e-10)
    sc = np.abs(b["betahat"][ok]).max(axis=-1, keepdims=True)
    assert (np.abs(a["betahat"][ok] - b["betahat"][ok]) / sc).max() <= 1e-9


@pytest.mark.parametrize("name,K", [("C2", 400), ("swiss", 300)])
def test_small_path_bitwise_repeatable_and_k_independent(ctx, name, K):
    """chol_small (one CTA per point, matrix in shared memory): a point's outputs do not
    depend on the other points of the call, its position in the grid, or the run —
    bitwise, for the whole-octave table (one unit grid per three octaves) included."""
    if name == "swiss":
        cfg = synthgen.Config("sw", 100, 2, K, 34, True, "uniform", "swiss-shaped")
        coords, y, X = synthgen.make_dataset(cfg, seed=5)
        P, lam = synthgen.make_params(cfg, K, seed=6), np.linspace(-1.0, 2.0, 34)
    else:
        coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
    full = ctx.eval_batch(coords, y, X, P, lam)
    again = ctx.eval_batch(coords, y, X, P, lam)
    sub = ctx.eval_batch(coords, y, X, np.ascontiguousarray(P[K // 2:][::-1]), lam)
    for key in full:
        assert np.array_equal(full[key], again[key], equal_nan=True), key
        assert np.array_equal(full[key][K // 2:][::-1], sub[key], equal_nan=True), key
