"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by
element on the same seeded inputs (-m gpu).

Tolerances (north_star / DESIGN.md §6): relative 1e-8 on ℓ_p, σ̂² and log|V|
(absolute 1e-8 when |log|V|| < 1); max_j |Δβ̂_j| ≤ 1e-8·‖β̂‖∞; V elements
relative 1e-13 (+ κ and |ln ρ| terms, see test_matern_build_elementwise).  Status codes must agree exactly.
"""
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

NTHREADS = os.cpu_count() or 8


@pytest.fixture(scope="module")
def ctx():
    c = lik.create(0)
    yield c
    c.close()


def assert_parity(gpu, ref, tol=1e-8, label=""):
    """Statuses equal; on OK points and on the valid λ columns of NEG_RESID points (R12)
    ℓ_p, σ̂² relative ≤ tol, log|V| relative (absolute below 1), β̂ ≤ tol·‖β̂‖∞; a
    NEG_RESID point's failed columns are −∞ on both sides."""
    st_g, st_r = gpu["status"], ref["status"]
    assert np.array_equal(st_g, st_r), f"{label} status mismatch {np.nonzero(st_g != st_r)}"
    neg = st_r == 3
    if neg.any():
        fg, fr = np.isneginf(gpu["loglik"][neg]), np.isneginf(ref["loglik"][neg])
        assert np.array_equal(fg, fr), f"{label} NEG_RESID columns differ"
        assert np.all(np.isnan(gpu["sigma2hat"][neg][fg])) and np.all(np.isnan(gpu["betahat"][neg][fg]))
    col = (st_r == 0)[:, None] | (neg[:, None] & np.isfinite(ref["loglik"]))
    pts = (st_r == 0) | neg
    if not col.any():
        return
    ll_g, ll_r = gpu["loglik"][col], ref["loglik"][col]
    rel = np.abs(ll_g - ll_r) / np.abs(ll_r)
    assert rel.max() <= tol, f"{label} loglik rel {rel.max():.3e} at {np.nonzero(col)[0][rel.argmax()]}"
    s_g, s_r = gpu["sigma2hat"][col], ref["sigma2hat"][col]
    rel = np.abs(s_g - s_r) / np.abs(s_r)
    assert rel.max() <= tol, f"{label} sigma2 rel {rel.max():.3e}"
    ld_g, ld_r = gpu["logdetV"][pts], ref["logdetV"][pts]
    err = np.abs(ld_g - ld_r) / np.maximum(np.abs(ld_r), 1.0)
    assert err.max() <= tol, f"{label} logdetV err {err.max():.3e}"
    b_g, b_r = gpu["betahat"][col], ref["betahat"][col]
    scale = np.abs(b_r).max(axis=-1, keepdims=True)
    err = np.abs(b_g - b_r) / scale
    assert err.max() <= tol, f"{label} betahat err {err.max():.3e}"


def stratified_sample(P, count, seed, W=None):
    """SURVEY §8(d)'s stratified parity subset: κ = 100, κ = ½, κ ≥ 20, the smallest κ,
    the largest ν² and φX, the first and last point of every wave of W points (the
    bench's launch configuration), then uniform random points up to `count`."""
    K = P.shape[0]
    rng = np.random.default_rng(seed)
    pick = [np.nonzero(P[:, 1] > 99)[0][:3], np.nonzero(np.isclose(P[:, 1], 0.5))[0][:3],
            np.nonzero((P[:, 1] >= 20) & (P[:, 1] < 99))[0][:3], np.argsort(P[:, 1])[:2],
            np.argsort(P[:, 2])[-2:], np.argsort(P[:, 0])[-2:], [0, K - 1]]
    if W:
        starts = np.arange(0, K, W)
        pick += [starts, np.minimum(starts + W - 1, K - 1)]
    sel = np.unique(np.concatenate([np.asarray(a, dtype=np.int64) for a in pick]))
    rest = np.setdiff1d(np.arange(K), sel)
    extra = max(0, count - sel.size)
    return np.unique(np.r_[sel, rng.choice(rest, min(extra, rest.size), replace=False)])


def default_wave(K, n, r):
    """The library's automatic wave size (lik_api.cpp run_device) for this GPU."""
    nt = (n + 63) // 64
    slot = (nt * (nt + 1) // 2 + nt) * 64 * 64 * 8
    free, _ = torch.cuda.mem_get_info()
    res = torch.cuda.get_device_properties(0).multi_processor_count * 2
    half = max(1, int(0.5 * free) // slot)
    wmax = min(16 * res, half, 65535)
    if wmax >= res:
        wmax -= wmax % res
    nw = -(-K // wmax)
    w = -(-K // nw)
    if w > res:
        w = min(wmax, -(-w // res) * res, K)
    return w


def _oracle(orc, coords, y, X, P, lam):
    return orc.eval_batch(coords, y, X, P, lam, nthreads=NTHREADS)


# --------------------------------------------------------------------------- matern_build
def _inputs_n(n, K, seed=11):
    """C3-shaped inputs with an arbitrary number of sites."""
    base = synthgen.CONFIGS["C3"]
    cfg = synthgen.Config(f"n{n}", n, base.p, K, base.M, base.iso, base.layout, f"n{n}")
    coords, y, X = synthgen.make_dataset(cfg, seed=seed)
    return coords, y, X, synthgen.make_params(cfg, K, seed=seed + 1), synthgen.make_lambdas(cfg.M)


# C1 / C2 take the whole-octave table (n < 256), n300 the quarter-octave one (as C3-C5)
@pytest.mark.parametrize("name", ["C1", "C2", "n300"])
def test_matern_build_elementwise(ctx, orc, name):
    coords, y, X, P, lam = _inputs_n(300, 64) if name == "n300" else synthgen.make_inputs(name, K=64)
    P = P[:12].copy()
    P[0, 1] = 100.0     # κ-fixed extremes
    P[1, 1] = 0.5
    P[2, 1] = 2000.0    # Gaussian limit (R7)
    P[3, 1] = 0.21
    # large κ at long range: ln ρ far below −746 inside the last non-zero table octave
    P[4] = [40751.846, 230.364234, 1.22954009, 4.43248760, 0.496259428]
    dc = torch.tensor(coords, device="cuda")
    dp = torch.tensor(P, device="cuda")
    V = ctx.debug_build_V(dc, dp).cpu().numpy()
    for k in range(P.shape[0]):
        ref = orc.build_V(coords, P[k])
        # ρ = exp(ln ρ) on both sides, so the relative error of ρ is the absolute error
        # of ln ρ: ~ε·|ln ρ| from the distance and the exponent, plus the cancelling
        # O(κ ln z) terms of ln(2^{1−κ}/Γ(κ)) + κ ln z + ln K_κ(z).
        tol = (1e-13 * max(1.0, P[k, 1] / 10.0) if P[k, 1] < 1e3 else 1e-14) \
            + 2e-15 * np.abs(np.log(np.maximum(ref, 1e-300)))
        err = np.abs(V[k] - ref) - tol * np.abs(ref)
        assert err.max() <= 1e-300, (k, P[k], float((np.abs(V[k] - ref) / np.maximum(np.abs(ref), 1e-300)).max()))


# --------------------------------------------------------------------------- whole path
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_parity_full_config(ctx, orc, name):
    coords, y, X, P, lam = synthgen.make_inputs(name)
    gpu = ctx.eval_batch(coords, y, X, P, lam)
    ref = _oracle(orc, coords, y, X, P, lam)
    assert_parity(gpu, ref, label=name)


@pytest.mark.parametrize("n,p,M", [(5, 1, 1), (8, 3, 2), (63, 2, 3), (64, 2, 4), (65, 3, 3),
                                   (127, 4, 5), (129, 1, 7), (191, 5, 11), (250, 2, 30),
                                   # both Matérn table layouts at their switch (n = 256)
                                   (255, 3, 5), (256, 2, 4), (300, 4, 7)])
def test_parity_ragged_sizes(ctx, orc, n, p, M):
    rng = np.random.default_rng(1000 + n)
    side = 9000.0 * math.sqrt(n / 224.0)
    coords = rng.uniform(0, side, size=(n, 2))
    X = np.column_stack([np.ones(n)] + [rng.normal(size=n) for _ in range(p - 1)])
    y = np.exp(rng.normal(2.0, 0.4, size=n))
    cfg = synthgen.Config("R", n, p, 24, M, False, "uniform", "")
    P = synthgen.make_params(cfg, 24, seed=77 + n)
    lam = np.linspace(-0.5, 1.2, M)
    gpu = ctx.eval_batch(coords, y, X, P, lam)
    ref = _oracle(orc, coords, y, X, P, lam)
    assert_parity(gpu, ref, label=f"n={n}")


def test_parity_C3_subset(ctx, orc):
    """C3 on the GPU (full K in the bench's launch configuration); the stratified subset of
    256 points recomputed by the oracle."""
    coords, y, X, P, lam = synthgen.make_inputs("C3")
    W = default_wave(P.shape[0], X.shape[0], X.shape[1] + lam.shape[0])
    dc, dy, dX, dp, dl = (torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam))
    out = ctx.eval_batch_device(dc, dy, dX, dp, dl)
    torch.cuda.synchronize()
    gpu = {k: v.cpu().numpy() for k, v in out.items()}
    sel = stratified_sample(P, 256, seed=3, W=W)
    assert sel.size >= 256
    ref = _oracle(orc, coords, y, X, P[sel], lam)
    assert_parity({k: v[sel] for k, v in gpu.items()}, ref, label="C3")
    assert np.all(gpu["status"] == 0) and np.all(np.isfinite(gpu["loglik"]))


def test_parity_C4_bench_launch_sampled(ctx, orc):
    """Full C4 (K = 20,000, the bench workload and launch configuration) on the
    GPU; the stratified sample of 64 points, incl. the first and last
    point of every wave, recomputed one by one by the oracle."""
    coords, y, X, P, lam = synthgen.make_inputs("C4")
    W = default_wave(P.shape[0], X.shape[0], X.shape[1] + lam.shape[0])
    dc, dy, dX, dp, dl = (torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam))
    out = ctx.eval_batch_device(dc, dy, dX, dp, dl)
    torch.cuda.synchronize()
    gpu = {k: v.cpu().numpy() for k, v in out.items()}
    sel = stratified_sample(P, 64, seed=4, W=W)
    assert sel.size >= 64
    ref = _oracle(orc, coords, y, X, P[sel], lam)
    assert_parity({k: v[sel] for k, v in gpu.items()}, ref, label="C4")
    assert np.all(gpu["status"] == 0)
    assert np.all(np.isfinite(gpu["loglik"]))


def test_parity_C5_sampled(ctx, orc):
    """C5 (n = 5,000, the large-matrix stress config): full K on the GPU, the stratified
    sample of 16 points (incl. κ = 100 and κ = ½) recomputed by the oracle."""
    coords, y, X, P, lam = synthgen.make_inputs("C5")
    W = default_wave(P.shape[0], X.shape[0], X.shape[1] + lam.shape[0])
    gpu = ctx.eval_batch(coords, y, X, P, lam)
    sel = stratified_sample(P, 16, seed=5, W=W)  # the strata and the wave ends: ~30 points
    assert sel.size >= 16
    ref = _oracle(orc, coords, y, X, P[sel], lam)
    assert_parity({k: v[sel] for k, v in gpu.items()}, ref, label="C5")
    assert np.all(gpu["status"] == 0)


# --------------------------------------------------------------------------- edge cases
def test_status_codes(ctx, orc):
    coords, y, X = synthgen.make_dataset("C1")
    good = [900.0, 1.5, 0.2, 1.0, 0.0]
    P = np.array([good, [-1.0, 1.5, 0.2, 1.0, 0.0], [900.0, 0.0, 0.2, 1.0, 0.0],
                  [900.0, 1.5, -0.1, 1.0, 0.0], [900.0, 1.5, 0.2, 0.0, 0.0],
                  [900.0, float("nan"), 0.2, 1.0, 0.0], [900.0, float("inf"), 0.2, 1.0, 0.0], good])
    gpu = ctx.eval_batch(coords, y, X, P, [0.3, 0.7])
    ref = _oracle(orc, coords, y, X, P, [0.3, 0.7])
    assert list(gpu["status"]) == [0, 4, 4, 4, 4, 4, 4, 0]
    assert_parity(gpu, ref)
    assert np.all(np.isneginf(gpu["loglik"][1:7])) and np.all(np.isnan(gpu["logdetV"][1:7]))
    assert np.all(np.isnan(gpu["betahat"][1:7]))
    # V not PD (dense sites, long smooth range, no nugget): both sides flag it
    c2 = np.stack([np.arange(70) * 1.0, np.zeros(70)], axis=1)
    y2 = 1.0 + np.arange(70.0)
    P2 = [[1e5, 10.0, 0.0, 1.0, 0.0], [5.0, 0.5, 0.1, 1.0, 0.0]]
    g2 = ctx.eval_batch(c2, y2, np.ones((70, 1)), P2, [0.5])
    r2 = _oracle(orc, c2, y2, np.ones((70, 1)), P2, [0.5])
    assert g2["status"][0] == 1 and r2["status"][0] == 1
    assert_parity(g2, r2)


def test_call_level_errors(ctx):
    coords, y, X = synthgen.make_dataset("C1")
    P = [[900.0, 1.5, 0.2, 1.0, 0.0]]
    assert ctx.eval_batch_rc(coords, y, X, P, [0.5])[0] == lik.LIK_OK
    y2 = y.copy()
    y2[7] = -1.0
    rc, msg = ctx.eval_batch_rc(coords, y2, X, P, [0.5])
    assert rc == lik.LIK_EDOMAIN and "y[7]" in msg
    c3 = coords.copy()
    c3[9] = c3[4]
    rc, msg = ctx.eval_batch_rc(c3, y, X, P, [0.5])
    assert rc == lik.LIK_EDOMAIN and "4" in msg and "9" in msg
    rc, _ = ctx.eval_batch_rc(coords, y, np.column_stack([X, 2 * X[:, 1]]), P, [0.5])
    assert rc == lik.LIK_ERANK
    rc, _ = ctx.eval_batch_rc(coords[:3], y[:3], X[:3], P, [0.5])
    assert rc == lik.LIK_EINVAL
    rc, _ = ctx.eval_batch_rc(coords, y, np.column_stack([X] * 32), P, [0.5])  # p = 64 > 63
    assert rc == lik.LIK_EINVAL
    c4 = coords.copy()
    c4[3, 0] = float("nan")
    assert ctx.eval_batch_rc(c4, y, X, P, [0.5])[0] == lik.LIK_EINVAL


def test_many_lambdas_in_chunks(ctx, orc):
    """M + p > 64: the λ are evaluated in chunks of 64 − p (one factorisation per chunk)
    and copied into place — vs the oracle, and each chunk's columns bitwise equal to a
    call with just that chunk's λ; the summaries and prepared datasets refuse it."""
    coords, y, X = synthgen.make_dataset("C1")
    p = X.shape[1]
    lam = np.linspace(-1.0, 2.0, 150)  # 3 chunks of 62 (p = 2)
    P = np.array([[900.0, 1.5, 0.2, 1.0, 0.0], [600.0, 0.7, 0.4, 1.0, 0.0], [-1.0, 1.5, 0.2, 1.0, 0.0]])
    gpu = ctx.eval_batch(coords, y, X, P, lam)
    assert_parity(gpu, _oracle(orc, coords, y, X, P, lam), label="chunks")
    Mc = 64 - p
    for m0 in range(0, len(lam), Mc):
        part = ctx.eval_batch(coords, y, X, P, lam[m0:m0 + Mc])
        for key in ("loglik", "sigma2hat", "betahat"):
            assert np.array_equal(gpu[key][:, m0:m0 + Mc], part[key], equal_nan=True), (m0, key)
        assert np.array_equal(gpu["logdetV"], part["logdetV"], equal_nan=True)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    with pytest.raises(lik.LikError) as e:
        ctx.eval_batch_device_ex(*t)
    assert e.value.code == lik.LIK_ENOTIMPL
    with pytest.raises(lik.LikError) as e:
        ctx.dataset(coords, y, X, lam)
    assert e.value.code == lik.LIK_ENOTIMPL


def test_wide_r_and_gaussian_limit(ctx, orc):
    # M + p = 64 (the ABI maximum) and κ ≥ 1e3 (Gaussian limit, R7)
    coords, y, X = synthgen.make_dataset("C1")
    lam = np.linspace(-1.0, 1.5, 62)
    P = np.array([[900.0, 1.5, 0.2, 1.0, 0.0], [600.0, 3000.0, 0.3, 1.0, 0.0]])
    assert_parity(ctx.eval_batch(coords, y, X, P, lam), _oracle(orc, coords, y, X, P, lam))


def test_determinism_waves_and_apis(ctx):
    coords, y, X, P, lam = synthgen.make_inputs("C2", K=300)
    a = ctx.eval_batch(coords, y, X, P, lam)
    for w in (1, 7, 64):
        ctx.set_wave_points(w)
        b = ctx.eval_batch(coords, y, X, P, lam)
        for key in a:
            assert np.array_equal(a[key], b[key], equal_nan=True), (w, key)
    ctx.set_wave_points(0)
    # permuting points permutes outputs bitwise
    perm = np.random.default_rng(2).permutation(P.shape[0])
    c = ctx.eval_batch(coords, y, X, P[perm], lam)
    for key in a:
        assert np.array_equal(a[key][perm], c[key], equal_nan=True)
    # device API on torch tensors, on a side stream
    dc, dy, dX, dp, dl = (torch.tensor(v, device="cuda") for v in (coords, y, X, P, lam))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = ctx.eval_batch_device(dc, dy, dX, dp, dl, stream=s)
    s.synchronize()
    for key in a:
        assert np.array_equal(a[key], out[key].cpu().numpy(), equal_nan=True), key


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shard_assembly_bitwise_vs_one_gpu(ctx, world):
    """§8(e): the sharded table equals the 1-GPU table bitwise.  Each rank's strided
    shard is evaluated in turn on this one GPU (independent calls, no collective),
    packed as all_gather_results packs it and un-strided by unpack_global."""
    from paper_2305_04318_b200 import multi
    coords, y, X, P, lam = synthgen.make_inputs("C2", K=301)
    K, M, p = P.shape[0], len(lam), X.shape[1]
    dc, dy, dX, dl = (torch.tensor(v, device="cuda") for v in (coords, y, X, lam))
    full = ctx.eval_batch_device(dc, dy, dX, torch.tensor(P, device="cuda"), dl)
    Kmax = multi.local_count(K, 0, world)
    bufs = []
    for g in range(world):
        out = ctx.eval_batch_device(dc, dy, dX, torch.tensor(P[multi.shard_indices(K, g, world)], device="cuda"), dl)
        bufs.append(multi.pack(out, M, p, Kmax))
    table = multi.unpack_global(torch.stack(bufs).cpu().numpy(), K, M, p, world)
    for key in table:
        assert np.array_equal(table[key], full[key].cpu().numpy(), equal_nan=True), (world, key)


@pytest.mark.parametrize("name, K, reps", [("C3", 1776, 3), ("C4", 1184, 2), ("C2", 2960, 3),
                                            ("n1020", 1776, 3)])
def test_bitwise_repeatability_over_cta_rounds(ctx, name, K, reps):
    """Repeated calls give bitwise identical outputs with several rounds of resident
    CTAs per launch (K = 6 resp. 4 / 10 × 296): CTAs that start on an SM after another
    finished see its shared memory and a different timing mix, which is where a
    race in the k-loop's stage protocol showed (a stage released before the warp's
    loads of it completed; ~0.5 % of the points).  n = 1020 takes the
    separate augmented tile row (no merged tail); C2 is diagonal-factorisation bound."""
    if name == "n1020":
        base = synthgen.CONFIGS["C3"]
        cfg = synthgen.Config("n1020", 1020, base.p, K, base.M, base.iso, base.layout, "n1020")
        coords, y, X = synthgen.make_dataset(cfg, seed=7)
        P, lam = synthgen.make_params(cfg, K, seed=8), synthgen.make_lambdas(cfg.M)
    else:
        coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
    t = [torch.tensor(v, device="cuda") for v in (coords, y, X, P, lam)]
    first = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(*t).items()}
    for _ in range(reps):
        nxt = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(*t).items()}
        for key in first:
            same = np.array_equal(first[key], nxt[key], equal_nan=True)
            assert same, (key, np.nonzero(np.any((first[key] != nxt[key]).reshape(K, -1), axis=1))[0][:10])


@pytest.mark.parametrize("name, K", [("C2", 300), ("C4", 900)])
def test_dataset_api_bitwise(ctx, name, K):
    """lik_dataset_eval_device: bitwise equal to lik_eval_batch_device; two evaluations
    enqueued back to back without synchronisation each equal their separate result."""
    coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
    t = [torch.tensor(v, device="cuda") for v in (coords, y, X, P, lam)]
    ref = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(*t).items()}
    ds = ctx.dataset(coords, y, X, lam)
    try:
        P2 = P[::-1].copy()
        o1 = ds.eval_device(t[3])
        o2 = ds.eval_device(torch.tensor(P2, device="cuda"))  # no sync in between
        torch.cuda.synchronize()
        for key in ref:
            assert np.array_equal(o1[key].cpu().numpy(), ref[key], equal_nan=True), key
            assert np.array_equal(o2[key].cpu().numpy(), ref[key][::-1], equal_nan=True), key
    finally:
        ds.close()


def test_dataset_api_errors(ctx):
    coords, y, X, P, lam = synthgen.make_inputs("C1")
    bad = y.copy()
    bad[3] = -1.0
    with pytest.raises(lik.LikError) as e:
        ctx.dataset(coords, bad, X, lam)
    assert e.value.code == lik.LIK_EDOMAIN and "y[3]" in ctx.last_error()
    ds = ctx.dataset(coords, y, X, lam)
    try:
        with pytest.raises(lik.LikError) as e:
            ds.eval_device(torch.zeros((0, 5), dtype=torch.float64, device="cuda"))
        assert e.value.code == lik.LIK_EINVAL
    finally:
        ds.close()


@pytest.mark.parametrize("name, per_wave", [("C2", 1), ("C3", 2)])
def test_stage_timing_api(name, per_wave):
    """Stage timers: per wave the table (+ the build kernel when the matrix does not fit
    chol_small, which builds its own tiles) and one factorisation launch."""
    c = lik.create(0, lik.FLAG_TIMING)
    coords, y, X, P, lam = synthgen.make_inputs(name, K=200)
    c.eval_batch(coords, y, X, P, lam)
    t = c.stage_times()
    assert t["chol_fused"][1] >= 1 and t["chol_fused"][0] > 0
    assert t["matern_build"][1] == per_wave * t["chol_fused"][1]
    c.reset_stage_times()
    assert c.stage_times()["chol_fused"] == (0.0, 0)
    c.close()


def test_reml_and_table1_summaries(ctx, orc):
    """NEXT-1: Table-1 summaries and the REML profile likelihood (Appendix) vs the oracle;
    the ML outputs of the _ex entry point are bitwise those of lik_eval_batch_device."""
    for name, K in (("C1", 16), ("C2", 64)):
        coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
        t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
        ex = ctx.eval_batch_device_ex(*t)
        base = ctx.eval_batch_device(*t)
        torch.cuda.synchronize()
        ex = {k: v.cpu().numpy() for k, v in ex.items()}
        for k2, v in base.items():
            assert np.array_equal(v.cpu().numpy(), ex[k2], equal_nan=True), k2
        ref = orc.eval_batch(coords, y, X, P, lam, nthreads=NTHREADS, summaries=True)
        ok = ref["status"] == 0
        assert np.array_equal(ex["status"], ref["status"])
        rel = lambda a, b: np.abs(a - b) / np.maximum(np.abs(b), 1.0)
        assert rel(ex["detReml"][ok], ref["detReml"][ok]).max() <= 1e-8
        sc = np.abs(ref["ssqYX"][ok]).max(axis=(1, 2), keepdims=True)
        assert (np.abs(ex["ssqYX"][ok] - ref["ssqYX"][ok]) / sc).max() <= 1e-8
        yy = np.stack([np.diagonal(ref["ssqYX"][kk])[:lam.shape[0]] for kk in range(len(P))])[ok]
        assert (np.abs(ex["ssqBetahat"][ok] - ref["ssqBetahat"][ok]) / yy).max() <= 1e-8
        assert (np.abs(ex["ssqResidual"][ok] - ref["ssqResidual"][ok]) / yy).max() <= 1e-8
        assert (np.abs(ex["loglik_reml"][ok] - ref["loglik_reml"][ok]) / np.abs(ref["loglik_reml"][ok])).max() <= 1e-8
        assert (np.abs(ex["sigma2hat_reml"][ok] - ref["sigma2_reml"][ok]) / ref["sigma2_reml"][ok]).max() <= 1e-8


def test_site_order_invariance():
    """The default Morton site order and the caller's natural order give the same
    likelihoods (a symmetric permutation of V leaves |V| and the quadratic forms
    unchanged; only the rounding order differs)."""
    coords, y, X, P, lam = synthgen.make_inputs("C2", K=48)
    a = lik.create(0).eval_batch(coords, y, X, P, lam)
    b = lik.create(0, lik.FLAG_NATURAL_ORDER).eval_batch(coords, y, X, P, lam)
    assert np.array_equal(a["status"], b["status"])
    np.testing.assert_allclose(a["loglik"], b["loglik"], rtol=1e-11)
    np.testing.assert_allclose(a["logdetV"], b["logdetV"], rtol=1e-11, atol=1e-11)
    np.testing.assert_allclose(a["betahat"], b["betahat"], rtol=1e-9, atol=1e-9 * np.abs(a["betahat"]).max())


@pytest.mark.parametrize("name,K", [("C1", 16), ("C2", 200)])
def test_profiles_vs_oracle(ctx, orc, name, K):
    """NEXT-2: β_a, σ, λ profile log-likelihoods over the K×M grid from the
    GPU summaries vs the oracle's profiles from its own summaries."""
    coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
    n, p = X.shape
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    summ = ctx.eval_batch_device_ex(*t)
    ref = orc.eval_batch(coords, y, X, P, lam, nthreads=NTHREADS, summaries=True)
    bh = ref["betahat"][ref["status"] == 0].reshape(-1, p)
    lo, hi = bh.min(axis=0), bh.max(axis=0)
    span = np.maximum(hi - lo, 1e-3 * np.maximum(1.0, np.abs(bh).max(axis=0)))
    grid = np.stack([np.linspace(lo[a] - span[a], hi[a] + span[a], 33) for a in range(p)])
    sig = np.sqrt(np.linspace(0.3, 3.0, 17) * np.median(ref["sigma2hat"]))
    pb, ps, pl = ctx.profiles_device(n, t[1], summ, t[4], torch.tensor(grid, device="cuda"),
                                     torch.tensor(sig, device="cuda"))
    torch.cuda.synchronize()
    rb, rs, rl = orc.profiles(n, p, ref["ssqYX"], ref["logdetV"], ref["status"], lam, y, grid, sig)
    rel = lambda a, b: np.abs(a - b) / np.abs(b)
    assert rel(pb.cpu().numpy(), rb).max() <= 1e-8
    assert rel(ps.cpu().numpy(), rs).max() <= 1e-8
    assert rel(pl.cpu().numpy(), rl).max() <= 1e-8
    # the β profile peaks at the global maximum of ℓ_p over the grid
    assert pb.cpu().numpy().max() <= ref["loglik"].max() + 1e-9


def test_bounds_checked_build():
    """The LIK_BOUNDS_CHECK build traps if any bulk copy or tile pointer leaves the point's
    workspace slot; run the sanitizer case (C1, ragged C2, merged and separate augmented
    tails, profiles, debug V) in a subprocess with it (compute-sanitizer is closed on
    the pool)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_b = os.path.join(root, "paper_2305_04318_b200", "liblik_bounds.so")
    from paper_2305_04318_b200 import build as b
    if b._stale(lib_b):  # rebuilt whenever a source is newer (a stale variant would test old code)
        b.build(force=True, defines=("LIK_BOUNDS_CHECK",), out=lib_b)
    env = dict(os.environ, LIK_LIBRARY=lib_b)
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "debug", "sanitize_case.py")], cwd=root,
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "lik bounds" not in r.stdout + r.stderr


def test_eval_sharded_nccl_world1(ctx):
    """multi.eval_sharded (the multi-GPU entry point: shard, evaluate, NCCL all-gather,
    un-stride) under a one-rank NCCL group equals eval_batch bitwise."""
    import torch.distributed as dist
    from paper_2305_04318_b200 import multi
    coords, y, X, P, lam = synthgen.make_inputs("C2", K=77)
    ref = ctx.eval_batch(coords, y, X, P, lam)
    store = dist.HashStore()
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        got = multi.eval_sharded(ctx, coords, y, X, P, lam, torch.device("cuda", 0))
    finally:
        dist.destroy_process_group()
    for key in ref:
        assert np.array_equal(ref[key], got[key], equal_nan=True), key


def test_golden_n3_example_on_gpu(ctx):
    """The hand-computed worked example (tests/golden/spec_n3_ols.json: n = 3, V = I,
    X = 1, y' = (1, 2, 3); Eq. profile P:145-148 and Eq. remlpro) through
    the CUDA path directly, independent of the oracle: sites 1e6 ranges apart make
    every off-diagonal ρ underflow to 0 and ν² = 0 gives V = I; λ = 1 gives
    y' = y − 1 with zero Jacobian."""
    import json
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_n3_ols.json")))
    coords = np.array([[0.0, 0.0], [1e6, 0.0], [0.0, 1e6]])
    y = np.array(g["y_prime"]) + 1.0
    X = np.ones((3, 1))
    P = np.array([[1.0, 2.5, 0.0, 1.0, 0.0]])
    lam = np.array([1.0])
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    out = ctx.eval_batch_device_ex(*t)
    assert int(out["status"][0]) == 0
    assert float(out["logdetV"][0]) == 0.0
    assert float(out["betahat"][0, 0, 0]) == pytest.approx(g["betahat"], rel=1e-14)
    assert float(out["sigma2hat"][0, 0]) == pytest.approx(g["sigma2hat"], rel=1e-14)
    assert -2.0 * float(out["loglik"][0, 0]) == pytest.approx(g["minus2_loglik"], rel=1e-14)
    assert float(out["sigma2hat_reml"][0, 0]) == pytest.approx(g["sigma2hat_reml"], rel=1e-14)
    assert -2.0 * float(out["loglik_reml"][0, 0]) == pytest.approx(g["minus2_loglik_reml"], rel=1e-14)
