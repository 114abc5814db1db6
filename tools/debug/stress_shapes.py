"""Bitwise repeatability over shapes: several (n, p, M, K) cases, each evaluated
twice in one context with other shapes in between; reports any difference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
ctx = lik.create(0)
cases = [("C5", None, None), ("C2", None, None), ("C3", 1776, None)]
for n, p, M in [(65, 1, 1), (129, 3, 7), (250, 2, 30), (777, 4, 5), (1500, 5, 20)]:
    cases.append((synthgen.Config(f"r{n}", n, p, 900, M, False, "uniform", "ragged"), 900, None))
def run(c, K):
    cfg = synthgen.CONFIGS[c] if isinstance(c, str) else c
    coords, y, X = synthgen.make_dataset(cfg, seed=7)
    P = synthgen.make_params(cfg, K if K else cfg.K, seed=11)
    lam = synthgen.make_lambdas(cfg.M)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    out = ctx.eval_batch_device(*t)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}
first = [run(c, K) for c, K, _ in cases]
bad = 0
for i, (c, K, _) in enumerate(cases):
    again = run(c, K)
    for key in first[i]:
        if not np.array_equal(first[i][key], again[key], equal_nan=True):
            bad += 1
            print("DIFF", getattr(c, "name", c), key, flush=True)
            break
    else:
        print("same", getattr(c, "name", c), "ok", int((again["status"] == 0).sum()), flush=True)
print("cases with differences:", bad)
