"""Per-phase cycle breakdown of chol_fused (debug build with LIK_PHASE_TIMERS)."""
import ctypes, os, sys
sys.path.insert(0, '.')
os.environ["LIK_LIBRARY"] = os.path.abspath(os.environ.get("PHASE_LIB", "paper_2305_04318_b200/liblik_phase.so"))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 296
coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
ctx = lik.create(0)
L = lik.lib()
buf = (ctypes.c_ulonglong * 16)()
t = lambda a: torch.tensor(a, device="cuda")
args = [t(a) for a in (coords, y, X, P, lam)]
ctx.eval_batch_device(*args); torch.cuda.synchronize()
L.lik_debug_phase_cycles(buf, 1)
ctx.eval_batch_device(*args); torch.cuda.synchronize()
L.lik_debug_phase_cycles(buf, 1)
v = np.array(list(buf[:16]), dtype=float)
names = ["frag_load", "kloop", "bar_after_kloop", "staging_store", "potrf", "trinv", "trsm+store", "fence+bar", "final+epilogue"]
tot = v[:9].sum()
print(f"kloop data wait: first chunk {v[9]/K/1e6:.3f} Mcyc/point, later chunks {v[15]/K/1e6:.3f} Mcyc/point")
for i, nm in enumerate(names):
    print(f"{nm:18s} {v[i]/tot*100:6.2f}%  {v[i]/K/1e6:8.3f} Mcyc/point")
print("total Mcyc/point (thread 0)", tot / K / 1e6)
for i, nm in zip(range(10, 15), ["potrf.warp0_16x16", "potrf.bar_after_warp0", "potrf.panel_product", "potrf.trailing", "inverse_levels"]):
    print(f"  {nm:22s} {v[i]/K/1e6:8.3f} Mcyc/point")
