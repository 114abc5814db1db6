"""Host-side trace of eval_batch_device_ex calls on the Swiss shape (LIK_HOST_TRACE)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2305_04318_b200 as lik
from bench_paper_workloads_lib import workload

ctx = lik.create(0, lik.FLAG_TIMING)
coords, y, X, P, lam = workload("swiss", 100, 2, 15318, 34, 2405)
t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.eval_batch_device_ex(*t)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"call {i}: host {1e3 * (t1 - t0):.2f} ms, total {1e3 * (t2 - t0):.2f} ms", file=sys.stderr, flush=True)
