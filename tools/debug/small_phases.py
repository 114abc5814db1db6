"""Per-phase cycle breakdown of chol_small (debug build with LIK_PHASE_TIMERS), for the
lead warp, warp 0 (update group U) and warp NW-4 (a panel helper).  usage: python tools/debug/small_phases.py [C2|swiss] [K]"""
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
buf = (ctypes.c_ulonglong * 36)()
args = [torch.tensor(a, device="cuda") for a in (coords, y, X, P, lam)]
ctx.eval_batch_device(*args); torch.cuda.synchronize()
L.lik_debug_small_phase_cycles(buf, 1)
ctx.eval_batch_device(*args); torch.cuda.synchronize()
L.lik_debug_small_phase_cycles(buf, 1)
v = np.array(list(buf[:36]), dtype=float).reshape(3, 12)
names = ["load", "build", "panel 0", "G: next-panel update", "G: after the named barrier (helpers: row solves)",
         "U: trailing update", "step barrier", "epilogue", "G: before the named barrier (lead: factor8s)",
         "G: named-barrier wait", "-", "-"]
# (a BAR.SYNC blocks the warp at a later instruction than the clock read after it, so a
# barrier's wait can show up in the phase after it)
for w, lab in ((0, "lead warp"), (1, "warp 0 (U)"), (2, "warp NW-4 (a panel helper)")):
    tot = v[w].sum()
    print(f"--- {lab}: total {tot / K / 1e3:.2f} kcyc/point")
    for i, nm in enumerate(names):
        print(f"  {nm:32s} {v[w, i]/K/1e3:8.2f} kcyc/point")
