"""A/B timing of the small-matrix path: ms per lik_eval_batch_device call on C2 (n = 200,
1,000 points × 5 λ) and the paper's Swiss shape (n = 100, p = 2, 15,318 points × 34 λ),
CUDA events around 20 calls after 5 warm-up calls (and through a prepared lik_dataset), for each library given (LIK_LIBRARY
per process: run one process per library).  usage: python tools/small_ab.py [C2|swiss ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import synthgen, paper_2305_04318_b200 as lik
from bench_paper_workloads_lib import workload

ctx = lik.create(0, 0)
res = []
for name in sys.argv[1:] or ["C2", "swiss"]:
    if name == "swiss":
        arrs = workload("swiss", 100, 2, 15318, 34, 2405)
    else:
        arrs = synthgen.make_inputs(name)
    t = [torch.tensor(a, device="cuda") for a in arrs]
    for _ in range(5):
        ctx.eval_batch_device(*t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ctx.eval_batch_device(*t)
    e1.record()
    torch.cuda.synchronize()
    res.append(f"{name} {e0.elapsed_time(e1) / 20:.3f} ms")
    # the prepare-once dataset path (validation and site ordering done once)
    ds = ctx.dataset(*arrs[:3], arrs[4])
    out = None
    for _ in range(5):
        out = ds.eval_device(t[3], out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        ds.eval_device(t[3], out=out)
    e1.record()
    torch.cuda.synchronize()
    ds.close()
    res[-1] += f" (dataset {e0.elapsed_time(e1) / 20:.3f} ms)"
print(os.path.basename(os.environ.get("LIK_LIBRARY", "liblik.so")), " | ".join(res))
