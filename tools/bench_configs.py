"""Time the hot path on every BASELINE.json config (C1..C5) at full K, 1 GPU.
Reports points/s, dense FP64 TFLOP/s (n³/3 + n²r + nr² per point) and stage times."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik

names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
ctx = lik.create(0, lik.FLAG_TIMING)
for nm in names:
    cfg = synthgen.CONFIGS[nm]
    coords, y, X, P, lam = synthgen.make_inputs(nm)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    out = lik.Ctx.alloc_outputs(cfg.K, cfg.M, cfg.p, "cuda")
    reps = 3 if cfg.n <= 2000 else 1
    ctx.eval_batch_device(*t, out=out)  # warm
    torch.cuda.synchronize()
    ctx.reset_stage_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ctx.eval_batch_device(*t, out=out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    r = cfg.M + cfg.p
    F = cfg.n ** 3 / 3 + cfg.n ** 2 * r + cfg.n * r * r
    st = {k: round(v[0] / reps, 3) for k, v in ctx.stage_times().items()}
    chol_tf = cfg.K * F / (st["chol_fused"] / 1e3) / 1e12
    print(json.dumps({"config": nm, "n": cfg.n, "K": cfg.K, "M": cfg.M, "p": cfg.p, "ms": round(ms, 3),
                      "points_per_s": cfg.K / (ms / 1e3), "fp64_tflops": cfg.K * F / (ms / 1e3) / 1e12,
                      "chol_fused_tflops": chol_tf, "stages_ms": st,
                      "status_ok": int((out["status"] == 0).sum().item())}), flush=True)
