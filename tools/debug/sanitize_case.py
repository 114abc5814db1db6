"""Small end-to-end cases for compute-sanitizer: C1, a ragged C2 subset, n = 300 (the fused
path) and the Swiss shape (M = 34) through
lik_eval_batch_device_ex, lik_profiles_device and lik_debug_build_V."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
ctx = lik.create(0)
for name, K in (("C1", 16), ("C2", 6)):
    coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
    t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
    s = ctx.eval_batch_device_ex(*t)
    n, p = X.shape
    grid = torch.tensor(np.tile(np.linspace(-1, 6, 5), (p, 1)), device="cuda")
    ctx.profiles_device(n, t[1], s, t[4], grid, torch.tensor([0.5, 1.0], device="cuda"))
    ctx.debug_build_V(t[0], t[3][:2].contiguous())
    torch.cuda.synchronize()
    print(name, s["status"].cpu().numpy(), float(s["loglik"][0, 0]))
# non-merged tail (n multiple of 64) and the separate augmented row
cfg = synthgen.Config("R", 128, 2, 4, 3, False, "uniform", "")
coords, y, X = synthgen.make_dataset(cfg, seed=3)
P = synthgen.make_params(cfg, 4, seed=4)
out = ctx.eval_batch(coords, y, X, P, synthgen.make_lambdas(3))
print("n=128", out["status"], out["loglik"][0, 0])
# the large-n path (quarter-octave table, build_kernel, chol_fused) and the Swiss shape
cfg = synthgen.Config("L", 300, 3, 3, 2, False, "uniform", "")
coords, y, X = synthgen.make_dataset(cfg, seed=5)
out = ctx.eval_batch(coords, y, X, synthgen.make_params(cfg, 3, seed=6), synthgen.make_lambdas(2))
print("n=300", out["status"], out["loglik"][0, 0])
cfg = synthgen.Config("S", 100, 2, 4, 34, True, "uniform", "")
coords, y, X = synthgen.make_dataset(cfg, seed=7)
out = ctx.eval_batch(coords, y, X, synthgen.make_params(cfg, 4, seed=8), np.linspace(-1.0, 2.0, 34))
print("swiss-shaped", out["status"], out["loglik"][0, 0])
