"""Determinism stress per configuration: CONFIG evaluated REPS times (optionally with
other configurations in between); prints how many points differ from the first run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
name, reps, inter = sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else ""
K = int(sys.argv[4]) if len(sys.argv) > 4 else None
ctx = lik.create(0)
def run(nm, K=None):
    coords, y, X, P, lam = synthgen.make_inputs(nm, K=K)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    out = ctx.eval_batch_device(*t)
    torch.cuda.synchronize()
    return out["loglik"].cpu().numpy(), P
base, P = run(name, K)
for r in range(reps):
    for nm in inter.split(",") if inter else []:
        run(nm, K=200)
    cur, _ = run(name, K)
    d = np.nonzero(np.any(base != cur, axis=1))[0]
    rel = np.max(np.abs(base - cur) / np.abs(base)) if len(d) else 0.0
    print(f"{name} rep {r} inter={inter or '-'}: {len(d)} points differ, max rel {rel:.2e}", (d[:6].tolist(), P[d[:3], 1].tolist()) if len(d) else "", flush=True)
