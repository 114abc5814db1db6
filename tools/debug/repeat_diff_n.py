"""repeat_diff for an arbitrary n (C3-like inputs): merged vs separate augmented tail.
usage: repeat_diff_n.py n K reps"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
n, K, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = synthgen.CONFIGS["C3"]
cfg = synthgen.Config("X", n, cfg.p, K, cfg.M, cfg.iso, cfg.layout, "X")
coords, y, X = synthgen.make_dataset(cfg, seed=7)
P = synthgen.make_params(cfg, K, seed=8)
lam = synthgen.make_lambdas(cfg.M)
t = [torch.tensor(v, device="cuda") for v in (coords, y, X, P, lam)]
ctx = lik.create(0)
first = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(*t).items()}
nbad = 0
for r in range(reps):
    nxt = {k: v.cpu().numpy() for k, v in ctx.eval_batch_device(*t).items()}
    for key in ("logdetV", "loglik", "betahat"):
        a, b = first[key].reshape(K, -1), nxt[key].reshape(K, -1)
        bad = np.nonzero(~((a == b) | (np.isnan(a) & np.isnan(b))).all(axis=1))[0]
        nbad += len(bad)
print(f"n={n} r={cfg.M + cfg.p} n%64={n % 64} differing={nbad}")
