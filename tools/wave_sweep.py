"""Chol/build time vs wave size W (points per launch) on C4 — the per-launch tail
effect (all CTAs of a launch start together; the launch ends with the slowest)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik

K = int(sys.argv[1]) if len(sys.argv) > 1 else 2960
coords, y, X, P, lam = synthgen.make_inputs("C4", K=K)
t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
ctx = lik.create(0, lik.FLAG_TIMING)
for W in [int(w) for w in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["296", "592", "1480", "2960"])]:
    ctx.set_wave_points(W)
    ctx.eval_batch_device(*t)
    torch.cuda.synchronize()
    ctx.reset_stage_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        out = ctx.eval_batch_device(*t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    st = {k: round(v[0] / 2, 2) for k, v in ctx.stage_times().items()}
    F = 2000 ** 3 / 3 + 2000 ** 2 * 10 + 2000 * 100
    print(json.dumps({"W": W, "K": K, "ms": round(ms, 2), "points_per_s": round(K / ms * 1e3, 1),
                      "chol_tflops": round(K * F / (st["chol_fused"] / 1e3) / 1e12, 2), "stages_ms": st}), flush=True)
