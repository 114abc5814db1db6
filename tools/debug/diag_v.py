import sys, numpy as np, torch, mpmath
sys.path.insert(0, '.')
import oracle, synthgen, paper_2305_04318_b200 as lik
mpmath.mp.dps = 40
coords, y, X, P, lam = synthgen.make_inputs('C2', K=64)
P = P[:12].copy(); P[0,1]=100.0; P[1,1]=0.5; P[2,1]=2000.0; P[3,1]=0.21
ctx = lik.create(0)
V = ctx.debug_build_V(torch.tensor(coords, device='cuda'), torch.tensor(P, device='cuda')).cpu().numpy()
for k in range(12):
    ref = oracle.build_V(coords, P[k])
    rel = np.abs(V[k]-ref)/np.maximum(np.abs(ref),1e-300)
    rel[ref < 1e-300] = 0
    i, j = np.unravel_index(rel.argmax(), rel.shape)
    w = P[k]
    h = coords[i]-coords[j]
    c, s = np.cos(w[4]), np.sin(w[4]); phiY = w[0]/w[3]
    u = (c*h[0]-s*h[1])/w[0]; v = (s*h[0]+c*h[1])/phiY
    d = mpmath.sqrt(mpmath.mpf(u)**2+mpmath.mpf(v)**2); kap = mpmath.mpf(w[1])
    if w[1] < 1e3:
        z = mpmath.sqrt(8*kap)*d
        mp = 2**(1-kap)/mpmath.gamma(kap)*z**kap*mpmath.besselk(kap,z)
    else:
        mp = mpmath.exp(-2*d*d); z = 0
    print(k, "kappa %.3g" % w[1], "worst rel %.2e" % rel.max(), "z=%.4g lnrho=%.1f" % (float(z), float(mpmath.log(mp))),
          "gpu rel vs mp %.2e" % float(abs((V[k][i,j]-mp)/mp)), "oracle rel vs mp %.2e" % float(abs((ref[i,j]-mp)/mp)))
