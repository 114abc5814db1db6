"""Diagnose one parameter point: V elements (debug_build_V) and ℓ_p vs the oracle.
usage: diag_point.py CONFIG INDEX   (INDEX into synthgen.make_inputs(CONFIG) params)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synthgen, oracle, paper_2305_04318_b200 as lik
name, idx = sys.argv[1], int(sys.argv[2])
coords, y, X, P, lam = synthgen.make_inputs(name)
oracle.build()
p = P[idx:idx + 1].copy()
print("params", p[0].tolist())
ctx = lik.create(0)
g = ctx.eval_batch(coords, y, X, p, lam)
r = oracle.eval_batch(coords, y, X, p, lam, nthreads=16)
print("loglik gpu", g["loglik"][0][:3], "oracle", r["loglik"][0][:3])
V = ctx.debug_build_V(torch.tensor(coords, device="cuda"), torch.tensor(p, device="cuda")).cpu().numpy()[0]
Vr = oracle.build_V(coords, p[0])
rel = np.abs(V - Vr) / np.maximum(np.abs(Vr), 1e-300)
i, j = np.unravel_index(np.argmax(rel), rel.shape)
print("max rel V err", rel.max(), "at", (i, j), "gpu", V[i, j], "ref", Vr[i, j], "d", np.linalg.norm(coords[i] - coords[j]))
big = rel > 1e-10
print("elements with rel err > 1e-10:", int(big.sum()), "of", big.size)
if big.any():
    d = np.array([np.linalg.norm(coords[a] - coords[b]) for a, b in zip(*np.nonzero(big))])
    print("their distances: min", d.min(), "max", d.max(), " values ref min", Vr[big].min(), "max", Vr[big].max())
