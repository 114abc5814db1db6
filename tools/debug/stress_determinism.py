"""Bitwise determinism stress: the full C4 launch evaluated repeatedly in one
context, interleaved with other configurations; any difference is reported with
the first differing point.  usage: stress_determinism.py [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
ctx = lik.create(0)
def run(name, K=None):
    coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    out = ctx.eval_batch_device(*t)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}
base = run("C4")
bad = 0
for r in range(reps):
    run("C3", K=500); run("C2"); run("C1")
    cur = run("C4")
    for key in ("loglik", "logdetV", "sigma2hat", "betahat", "status"):
        a, b = base[key], cur[key]
        diff = np.nonzero(~((a == b) | (np.isnan(a) & np.isnan(b))).reshape(a.shape[0], -1).all(axis=1))[0]
        if len(diff):
            bad += 1
            k = diff[0]
            print(f"rep {r}: {key} differs at {len(diff)} points, first {k}: {a[k].ravel()[:3]} vs {b[k].ravel()[:3]}", flush=True)
            if r == 0:
                import oracle
                oracle.build()
                coords, y, X, P, lam = synthgen.make_inputs("C4")
                ref = oracle.eval_batch(coords, y, X, P[k:k + 1], lam, nthreads=16)
                print("   oracle", ref["loglik"][0][:3], "params", P[k].tolist(), flush=True)
                print("   differing points:", diff[:20].tolist(), flush=True)
            break
    else:
        print(f"rep {r}: identical", flush=True)
print("differing reps:", bad)
