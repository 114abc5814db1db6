"""World-size-2 gloo tests (CPU) of the N>1 host logic: strided sharding, the
all-gather of the result tables and the un-striding into global point order
(-m "not gpu").  The per-rank "results" are synthetic tensors derived from the
global point index, so any mis-ordering or dropped point is detected."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_04318_b200 import multi


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fake_outputs(idx, M, p):
    K = len(idx)
    k = torch.tensor(idx, dtype=torch.float64)
    return dict(loglik=k[:, None] * 10 + torch.arange(M, dtype=torch.float64),
                sigma2hat=k[:, None] + 0.5 + torch.zeros(M, dtype=torch.float64),
                betahat=k[:, None, None] * 100 + torch.arange(M * p, dtype=torch.float64).reshape(1, M, p),
                logdetV=-k, status=(torch.tensor(idx) % 5).to(torch.int32))


def _worker(rank, world, port, K, M, p, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        idx = multi.shard_indices(K, rank, world)
        out = _fake_outputs(idx, M, p)
        full = multi.all_gather_results(out, K, M, p)
        q.put((rank, {k: v.tolist() for k, v in full.items()}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("K", [1, 7, 20])
def test_sharded_gather_world2(K):
    M, p, world = 3, 2, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, M, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    ref = _fake_outputs(np.arange(K), M, p)
    for r in range(world):
        for key, v in ref.items():
            np.testing.assert_array_equal(np.asarray(res[r][key]), v.numpy(), err_msg=f"rank {r} {key}")


def test_shard_partition_properties():
    for K in (1, 5, 148, 20000):
        for world in (1, 2, 4, 8):
            parts = [multi.shard_indices(K, g, world) for g in range(world)]
            allidx = np.sort(np.concatenate(parts))
            assert np.array_equal(allidx, np.arange(K))
            sizes = [len(x) for x in parts]
            assert max(sizes) - min(sizes) <= 1
            assert multi.local_count(K, 0, world) == max(sizes)


def _check_worker(rank, world, port, same, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        coords = np.arange(10.0).reshape(5, 2)
        y = np.ones(5) + (0 if same else rank * 1e-12)
        try:
            multi.check_same_dataset(coords, y)
            q.put((rank, "ok"))
        except RuntimeError as e:
            q.put((rank, str(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("same", [True, False])
def test_dataset_agreement_world2(same):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_check_worker, args=(r, 2, port, same, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    if same:
        assert res == {0: "ok", 1: "ok"}
    else:
        assert all("disagree" in v for v in res.values())
