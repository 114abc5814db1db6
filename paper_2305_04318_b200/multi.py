"""Multi-GPU plumbing for the batched likelihood.

Parameter points are independent units, so the path shards
with no data-path collective: rank g evaluates the points k ≡ g (mod G)
(strided, which balances the κ-dependent cost of the Matérn build), and the
one exchange step is an all-gather of the per-rank result tables over
torch.distributed (NCCL over NVLink on B200, gloo in the CPU tests), after
which every rank un-strides the table into global point order.  Host logic
only; the likelihood itself runs in liblik.so.
"""
from __future__ import annotations

import numpy as np


def dataset_checksum(*arrays) -> int:
    """A 60-bit checksum of the dataset arrays (SHA-256 of their bytes)."""
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return int(h.hexdigest()[:15], 16)


def check_same_dataset(*arrays, device=None) -> None:
    """Every rank generated / loaded the same dataset: all-reduce the
    checksum with MAX over (h, −h); raises on any disagreement."""
    import torch
    import torch.distributed as dist
    h = dataset_checksum(*arrays)
    t = torch.tensor([h, -h], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if int(t[0]) != h or int(t[1]) != -h:
        raise RuntimeError("ranks disagree on the dataset")


def shard_indices(K: int, rank: int, world: int) -> np.ndarray:
    """Global point indices owned by `rank` (strided assignment)."""
    return np.arange(rank, K, world)


def local_count(K: int, rank: int, world: int) -> int:
    return len(range(rank, K, world))


def pack_width(M: int, p: int) -> int:
    """Doubles per point in the gathered table: loglik M, sigma2hat M, betahat M·p, logdetV, status."""
    return M * (2 + p) + 2


def pack(out: dict, M: int, p: int, Kmax: int):
    """Pack a rank's outputs (torch tensors) into a Kmax × W float64 tensor (zero-padded)."""
    import torch
    K = out["loglik"].shape[0]
    W = pack_width(M, p)
    buf = torch.zeros((Kmax, W), dtype=torch.float64, device=out["loglik"].device)
    if K:
        buf[:K] = torch.cat([out["loglik"].reshape(K, M), out["sigma2hat"].reshape(K, M),
                             out["betahat"].reshape(K, M * p), out["logdetV"].reshape(K, 1),
                             out["status"].reshape(K, 1).to(torch.float64)], 1)
    return buf


def unpack_global(gathered, K: int, M: int, p: int, world: int) -> dict:
    """gathered: world × Kmax × W (numpy) -> global-order dict of numpy arrays."""
    Kmax = gathered.shape[1]
    table = np.empty((K, pack_width(M, p)))
    for g in range(world):
        idx = shard_indices(K, g, world)
        table[idx] = gathered[g, :len(idx)]
    assert Kmax >= max(len(shard_indices(K, g, world)) for g in range(world))
    return dict(loglik=table[:, :M], sigma2hat=table[:, M:2 * M],
                betahat=table[:, 2 * M:2 * M + M * p].reshape(K, M, p),
                logdetV=table[:, -2], status=table[:, -1].astype(np.int32))


def all_gather_results(out: dict, K: int, M: int, p: int, group=None) -> dict:
    """All-gather every rank's outputs and return the global table (numpy) on all ranks."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    Kmax = local_count(K, 0, world)
    buf = pack(out, M, p, Kmax)
    gathered = torch.empty((world * Kmax, buf.shape[1]), dtype=buf.dtype, device=buf.device)
    dist.all_gather_into_tensor(gathered, buf, group=group)
    return unpack_global(gathered.view(world, Kmax, -1).cpu().numpy(), K, M, p, world)


def eval_sharded(ctx, coords, y, X, params, lambdas, device, group=None, stream=None) -> dict:
    """Evaluate all K points across the ranks of `group`; every rank returns the full table."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    params = np.ascontiguousarray(params, dtype=np.float64).reshape(-1, 5)
    K = params.shape[0]
    mine = shard_indices(K, rank, world)
    n, p = np.asarray(X).reshape(len(y), -1).shape
    M = len(lambdas)
    t = lambda a: torch.tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)
    if len(mine):
        out = ctx.eval_batch_device(t(coords), t(y), t(np.asarray(X).reshape(n, p)), t(params[mine]),
                                    t(lambdas), stream=stream)
    else:
        out = {k: torch.empty((0,) + s, dtype=d, device=device) for k, s, d in
               (("loglik", (M,), torch.float64), ("sigma2hat", (M,), torch.float64),
                ("betahat", (M, p), torch.float64), ("logdetV", (), torch.float64),
                ("status", (), torch.int32))}
    return all_gather_results(out, K, M, p, group)
