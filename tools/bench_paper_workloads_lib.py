"""Synthetic inputs with the shapes of the paper's own runs (used by
bench_paper_workloads.py and tools/debug/swiss_launches.py)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synthgen


def workload(name, n, p, K, M, seed):
    cfg = synthgen.Config(name, n, min(p, 5), K, M, False, "uniform", name)
    coords, y, X5 = synthgen.make_dataset(cfg, seed=seed)
    rng = np.random.default_rng(seed)
    X = np.column_stack([X5] + [rng.normal(size=n) for _ in range(p - X5.shape[1])])
    P = synthgen.make_params(cfg, K, seed=seed + 1)
    lam = np.linspace(0.2, 0.8, M)
    return coords, y, X, P, lam
