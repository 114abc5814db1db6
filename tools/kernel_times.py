"""One evaluation per named config (full K unless K is given as NAME:K), meant to run
under `ncu --metrics gpu__time_duration.sum` for per-kernel launch times
(table / build / chol split of the build stage, which the stage timer reports together)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synthgen, paper_2305_04318_b200 as lik

ctx = lik.create(0)
for arg in sys.argv[1:] or ["C2", "C4:4144"]:
    nm, _, k = arg.partition(":")
    coords, y, X, P, lam = synthgen.make_inputs(nm, K=int(k) if k else None)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    ctx.eval_batch_device(*t)
    torch.cuda.synchronize()
