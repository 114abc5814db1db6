"""Launch list helper: one eval_batch_device call on the Swiss shape (n = 100, p = 2,
15,318 points × 34 λ) and one on the soil shape, for `ncu --metrics gpu__time_duration.sum`."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2305_04318_b200 as lik
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from bench_paper_workloads_lib import workload  # noqa: E402

ctx = lik.create(0, 0)
for name, n, p, K, M in (("swiss", 100, 2, 15318, 34), ("soil", 829, 18, 12316, 31)):
    coords, y, X, P, lam = workload(name, n, p, K, M, 2305 + n)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    for _ in range(2):
        ctx.eval_batch_device(*t)
    torch.cuda.synchronize()
