"""Time the paper's own batched-likelihood runs (shapes only; synthetic data):
  Swiss rainfall: n = 100, p = 2, K = 15,318 points × M = 34 λ
  Soil mercury: n = 829, p = 18, K = 12,316 points × M = 31 λ
through lik_eval_batch_device_ex (ℓ_p, β̂, σ̂², Table-1 summaries, REML) and
lik_profiles_device (β_a profiles on a 100-point grid per coefficient, σ on 100
values, λ), 1 GPU.  The paper reports no timings for these runs."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_04318_b200 as lik
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2305_04318_b200 import representative as rp


from bench_paper_workloads_lib import workload  # noqa: E402


ctx = lik.create(0, lik.FLAG_TIMING)
for name, n, p, K, M in (("swiss", 100, 2, 15318, 34), ("soil", 829, 18, 12316, 31)):
    coords, y, X, P, lam = workload(name, n, p, K, M, 2305 + n)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    summ = ctx.eval_batch_device_ex(*t)
    torch.cuda.synchronize()
    ok = summ["status"] == 0
    bh = summ["betahat"][ok].reshape(-1, p)
    grid = torch.stack([torch.linspace(float(bh[:, a].min()), float(bh[:, a].max()), 100, dtype=torch.float64)
                        for a in range(p)]).cuda()
    sig = torch.linspace(0.3, 3.0, 100, dtype=torch.float64).cuda() * float(summ["sigma2hat"][ok].median().sqrt())
    ctx.profiles_device(n, t[1], summ, t[4], grid, sig)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    reps = 3
    ctx.reset_stage_times()
    e[0].record()
    for _ in range(reps):
        summ = ctx.eval_batch_device_ex(*t)
    e[1].record()
    for _ in range(reps):
        pb, ps, pl = ctx.profiles_device(n, t[1], summ, t[4], grid, sig)
    e[2].record()
    torch.cuda.synchronize()
    ev_ms, pr_ms = e[0].elapsed_time(e[1]) / reps, e[1].elapsed_time(e[2]) / reps
    r = M + p
    F = n ** 3 / 3 + n * n * r + n * r * r
    # Step 2: 6 fits (κ free + the 5 κ-fixed of P:582), stencil Hessians on the
    # GPU (51·3 / 33·3 likelihoods each), 726 / 120 sphere points × 12 α, λ grid of M−1 + λ̂
    # the paper's shapes (R26): Swiss — κ free + fixed at 0.5, 0.9, 10, 20, 100, the fixed fits
    # on 11 of the 12 levels (15,318 points); soil — κ free + fixed at 0.5, 0.8, 1 on
    # 10 levels (12,316 points)
    nat = np.array(P[0]); nat[1] = 2.0
    kfix, nlev = ((0.5, 0.9, 10.0, 20.0, 100.0), 11) if name == "swiss" else ((0.5, 0.8, 1.0), 10)
    fits = [rp.Fit(nat, 0.5)] + [rp.Fit(np.r_[nat[0], kf, nat[2:]], 0.5, kappa_fixed=kf) for kf in kfix]
    afix = rp.DEFAULT_ALPHAS[len(rp.DEFAULT_ALPHAS) - nlev:]
    import time
    t0 = time.perf_counter(); rs = rp.configure_params(ctx, coords, y, X, fits, m_lambda=M - 1, alphas_fixed=afix)
    t1 = time.perf_counter(); rs = rp.configure_params(ctx, coords, y, X, fits, m_lambda=M - 1, alphas_fixed=afix)
    t2 = time.perf_counter()
    print(json.dumps({"workload": name, "n": n, "p": p, "K": K, "M": M,
                      "eval_ms": round(ev_ms, 3), "points_per_s": K / (ev_ms / 1e3),
                      "likelihoods_per_s": K * M / (ev_ms / 1e3), "dense_fp64_tflops": K * F / (ev_ms / 1e3) / 1e12,
                      "profiles_ms": round(pr_ms, 3),
                      "step2_ms_cold": round((t1 - t0) * 1e3, 1), "step2_ms_warm": round((t2 - t1) * 1e3, 1),
                      "step2_points": int(len(rs.params)), "step2_lambdas": int(len(rs.lambdas)), "status_ok": int(ok.sum()),
                      "stages_ms": {k: round(v[0] / reps, 3) for k, v in ctx.stage_times().items()}}), flush=True)
