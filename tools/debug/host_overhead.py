import sys, time, os
sys.path.insert(0, '.')
import numpy as np, torch, synthgen, paper_2305_04318_b200 as lik
coords, y, X, P, lam = synthgen.make_inputs("C4", K=296)
t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
ctx = lik.create(0)
for W in (296, 2960):
    ctx.set_wave_points(W)
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); ctx.eval_batch_device(*t); t1 = time.perf_counter()
        torch.cuda.synchronize(); t2 = time.perf_counter()
        print(W, it, f"host call {1e3*(t1-t0):.2f} ms, total {1e3*(t2-t0):.2f} ms")
