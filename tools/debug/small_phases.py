"""Per-phase cycle breakdown of chol_small (debug build with LIK_PHASE_TIMERS), for the
lead warp and warp 0.  usage: python tools/debug/small_phases.py [C2|swiss] [K]"""
import ctypes, os, sys
sys.path.insert(0, '.')
os.environ["LIK_LIBRARY"] = os.path.abspath(os.environ.get("PHASE_LIB", "paper_2305_04318_b200/liblik_phase.so"))
import numpy as np, torch
import synthgen, paper_2305_04318_b200 as lik
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
if name == "swiss":
    cfg = synthgen.Config("sw", 100, 2, K, 34, True, "uniform", "swiss")
    coords, y, X = synthgen.make_dataset(cfg, seed=5)
    P, lam = synthgen.make_params(cfg, K, seed=6), np.linspace(-1.0, 2.0, 34)
else:
    coords, y, X, P, lam = synthgen.make_inputs(name, K=K)
ctx = lik.create(0)
L = lik.lib()
buf = (ctypes.c_ulonglong * 16)()
args = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
ctx.eval_batch_device(*args); torch.cuda.synchronize()
L.lik_debug_small_phase_cycles(buf, 1)
ctx.eval_batch_device(*args); torch.cuda.synchronize()
L.lik_debug_small_phase_cycles(buf, 1)
v = np.array(list(buf[:16]), dtype=float).reshape(2, 8)
names = ["load", "build", "factor0+bar", "(lead: G work before factor8)", "(lead: factor8)", "step work", "step barrier", "epilogue"]
for w, lab in ((0, "lead warp"), (1, "warp 0")):
    tot = v[w].sum()
    print(f"--- {lab}: total {tot / K / 1e3:.2f} kcyc/point")
    for i, nm in enumerate(names):
        print(f"  {nm:32s} {v[w, i]/K/1e3:8.2f} kcyc/point")
