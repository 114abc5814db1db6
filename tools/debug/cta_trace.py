"""Per-SM timeline of chol_fused CTAs (debug build with LIK_CTA_TRACE): busy time
vs span, gaps between consecutive CTAs on a slot, and the launch tail.
usage: PHASE_LIB=liblik_trace.so cta_trace.py CONFIG K"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["LIK_LIBRARY"] = os.path.abspath(os.environ.get("PHASE_LIB", "paper_2305_04318_b200/liblik_trace.so"))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2960
coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
ctx = lik.create(0)
ctx.set_wave_points(K)
t = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
ctx.eval_batch_device(*t); torch.cuda.synchronize()
ctx.eval_batch_device(*t); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (3 * K))()
lik.lib().lik_debug_cta_trace(buf, K)
a = np.array(list(buf), dtype=np.float64).reshape(K, 3)
t0 = a[:, 0].min()
st, en, sm = (a[:, 0] - t0) / 1e6, (a[:, 1] - t0) / 1e6, a[:, 2].astype(int)
span = en.max()
dur = en - st
print(f"{name} K={K}: launch span {span:.2f} ms, CTA duration mean {dur.mean():.2f} ms (min {dur.min():.2f}, max {dur.max():.2f})")
busy = 0.0; gaps = []
for s in np.unique(sm):
    idx = np.nonzero(sm == s)[0]
    o = idx[np.argsort(st[idx])]
    busy += dur[o].sum()
    # two slots per SM: greedy assign
    ends = [0.0, 0.0]
    for i in o:
        k = int(np.argmin(ends))
        gaps.append(st[i] - ends[k]); ends[k] = en[i]
nsm = len(np.unique(sm))
print(f"SMs {nsm}; busy (CTA-time) / (2 x SMs x span) = {busy / (2 * nsm * span) * 100:.1f} %")
g = np.array(gaps)
print(f"gaps between consecutive CTAs on a slot: mean {g.mean()*1e3:.1f} us, p50 {np.median(g)*1e3:.1f} us, sum/slot {g.sum()/(2*nsm):.2f} ms")
last = np.sort(en)
print(f"tail: first CTA end of last round at {np.percentile(en, 90):.2f} ms, last at {span:.2f} ms")
