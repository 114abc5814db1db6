"""Library baseline for context (not a product path): batched FP64 Cholesky of SPD
matrices of the C4 size through torch.linalg.cholesky_ex (cuSOLVER), and the
triangular solve with r = 10 right-hand sides (torch.linalg.solve_triangular),
timed with CUDA events.  Compares with chol_fused, which does the factorisation,
the solve and the cross products in one pass.  Usage: library_baseline.py [n] [batch]"""
import json, sys
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
r = 10
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.randn(B, n, n, device="cuda", dtype=torch.float64, generator=g) / n ** 0.5
V = A @ A.transpose(-1, -2) + torch.eye(n, device="cuda", dtype=torch.float64)
Bm = torch.randn(B, n, r, device="cuda", dtype=torch.float64, generator=g)
torch.cuda.synchronize()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


ms_chol, (L, info) = timed(lambda: torch.linalg.cholesky_ex(V))
ms_solve, _ = timed(lambda: torch.linalg.solve_triangular(L, Bm, upper=False))
F_chol = n ** 3 / 3
F_solve = n * n * r
print(json.dumps({
    "kind": "library_baseline", "n": n, "batch": B, "r": r,
    "cholesky_ms": round(ms_chol, 3), "cholesky_tflops": B * F_chol / (ms_chol / 1e3) / 1e12,
    "solve_ms": round(ms_solve, 3), "solve_tflops": B * F_solve / (ms_solve / 1e3) / 1e12,
    "points_per_s_chol_plus_solve": B / ((ms_chol + ms_solve) / 1e3),
    "info_ok": bool((info == 0).all()), "torch": torch.__version__,
}))
