"""Write a config's outputs to an .npz (for bitwise comparisons between library builds).
usage: dump_outputs.py CONFIG K OUT.npz"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
name, K, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
t = [torch.tensor(v, device="cuda") for v in (coords, y, X, P, lam)]
res = lik.create(0).eval_batch_device(*t)
np.savez(out, **{k: v.cpu().numpy() for k, v in res.items()})
