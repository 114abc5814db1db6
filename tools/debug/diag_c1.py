import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle, synthgen, paper_2305_04318_b200 as lik
name = sys.argv[1] if len(sys.argv) > 1 else 'C1'
coords, y, X, P, lam = synthgen.make_inputs(name, K=16)
ctx = lik.create(0)
g = ctx.eval_batch(coords, y, X, P, lam)
r = oracle.eval_batch(coords, y, X, P, lam, summaries=True)
np.set_printoptions(precision=6, linewidth=200)
print("status", g['status'], r['status'])
print("logdet rel", (g['logdetV'] - r['logdetV']) / np.abs(r['logdetV']))
print("sigma2 rel", ((g['sigma2hat'] - r['sigma2hat']) / r['sigma2hat'])[:, 0])
print("beta", g['betahat'][0, 0], r['betahat'][0, 0])
print("loglik rel", ((g['loglik'] - r['loglik']) / np.abs(r['loglik']))[:, 0])
# V check
V = ctx.debug_build_V(torch.tensor(coords, device='cuda'), torch.tensor(P, device='cuda')).cpu().numpy()
for k in range(4):
    ref = oracle.build_V(coords, P[k])
    print(k, P[k], "V max rel", (np.abs(V[k] - ref) / np.maximum(np.abs(ref), 1e-300)).max())
# single-point variants: sizes
for n in (64, 65, 128, 129):
    c2, y2, X2 = coords[:n] if n <= 100 else None, None, None
