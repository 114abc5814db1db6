"""Repeated identical calls: which outputs differ between runs, at how many points,
and by how much (relative).  usage: repeat_diff.py CONFIG K REPS"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
name, K, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
t = [torch.tensor(v, device="cuda") for v in (coords, y, X, P, lam)]
ctx = lik.create(0)
first = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(*t).items()}
for r in range(reps):
    nxt = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(*t).items()}
    for key in ("logdetV", "loglik", "betahat", "sigma2hat", "status"):
        a, b = first[key].reshape(K, -1).astype(float), nxt[key].reshape(K, -1).astype(float)
        bad = np.nonzero(~((a == b) | (np.isnan(a) & np.isnan(b))).all(axis=1))[0]
        if len(bad):
            rel = np.abs(a[bad] - b[bad]) / np.maximum(np.abs(a[bad]), 1e-300)
            print(f"rep {r} {key}: {len(bad)} points {bad[:6].tolist()} max rel {np.nanmax(rel):.3e} "
                  f"(slot = point mod 296: {(bad[:6] % 296).tolist()}, round {(bad[:6] // 296).tolist()})", flush=True)
print("done")
