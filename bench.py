"""Benchmark of the hot path: profile-likelihood parameter points per second at
n = 2000 (BASELINE.json configs[3], "C4"), FP64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4|C5|...]
                    [--scaling strong|weak] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

A "step" is one lik_eval_batch_device call over the rank's share of the batch
(all of SURVEY §8(a): prep, matern_build, Cholesky, solve, cross products,
epilogue), inputs resident in HBM, plus the one exchange step at N > 1: an
all-gather of the result tables over NCCL.  C4 = 20,000 parameter points × 5
Box-Cox λ; C5 (the 8-GPU large-matrix stress config) = 4,000 points × 10 λ at
n = 5,000.  Multi-GPU defaults to STRONG scaling, as BASELINE.json states the
configs ("20,000 points sharded across 1/2/4/8 B200"): the config's K points are
sharded k ≡ rank (mod N) (strided, balancing the κ-dependent cost);
`--scaling weak` gives every rank its own K points instead.  `value` = all points
processed ÷ the max-over-ranks device time.  The L2 (126 MB) is flushed with a
256 MiB write before every timed step.

With `--gpus N > 1` and no torchrun environment (WORLD_SIZE unset), bench.py
starts the N ranks itself through torch.distributed.run (127.0.0.1) and passes
rank 0's line through; under torchrun, --gpus must equal WORLD_SIZE.  NCCL's
communicator-init lines (NCCL_DEBUG=INFO, subsystem INIT, unless set) go to
stderr, stdout carries only the JSON line.

`e2e` is the same metric through the host-pointer API: lik_eval_batch at N = 1
(host→device copy of the step's inputs, the path, device→host copy of the
outputs, all inside the timed region) and multi.eval_sharded at N > 1.

`--impl reference` times the CPU oracle (oracle/, the parity reference) on the
host cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthgen  # noqa: E402

WORKLOAD = "C4"  # default workload (--config)
METRIC = "profile-likelihood param points/sec at n=2000 (1/2/4/8 B200); FP64 TFLOP/s vs peak"
UNIT = "points/s"
PHASE0 = os.path.join(ROOT, "profiles", "r01", "phase0_fp64_peaks.jsonl")
TRAFFIC = os.path.join(ROOT, "profiles", "chol_traffic.json")


def dense_flops_per_point(n, r):
    """algorithmic FP64 flops per point = n³/3 + n²r + n r²."""
    return n ** 3 / 3.0 + n * n * r + n * r * r


def fp64_peak():
    """Measured DMMA.8x8x4 FP64 peak (tools/phase0, TFLOP/s) else 37.2 nominal."""
    try:
        vals = [json.loads(l) for l in open(PHASE0)]
        best = max(v["tflops"] for v in vals if v.get("kind") == "dmma_sustained")
        return best, ("measured: DMMA.8x8x4 loop, tools/phase0 (profiles/r01/phase0_fp64_peaks.jsonl); "
                      "MEASURED_PEAKS.json has no FP64 entry and its bf16 x nominal-ratio route "
                      "(~27 TF/s) is below what this kernel sustains (DESIGN.md sec. 5)")
    except Exception:
        return 37.2, "nominal: 148 SM x 64 FMA/clk x 2 x 1.965 GHz"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def slot_bytes(n: int, r: int) -> int:
    """Workspace bytes the build writes per point: the lower tile triangle of V plus one
    row of augmented tiles, 64×64 FP64 each (lik_internal.cuh SlotGeom)."""
    nt = (n + 63) // 64
    return (nt * (nt + 1) // 2 + nt) * 64 * 64 * 8


BUILD_INSTR_PER_ELEMENT = 79.7 / 32  # warp instructions per element, build_kernel<4> (ncu, profiles/r02/ncu_build_summary.txt: 3.19e9 for 592 points)


def build_issue_roofline(K, n, build_ms_per_step, sm_mhz, nsm=148):
    """Issue-bound roofline of the Matérn build: elements (whole 64-tiles of the lower
    tile triangle) x warp instructions per element over 4 sub-partitions x SMs x clock."""
    if not build_ms_per_step or not sm_mhz:
        return None
    nt = (n + 63) // 64
    elements = K * nt * (nt + 1) // 2 * 64 * 64
    rate = elements * BUILD_INSTR_PER_ELEMENT / (build_ms_per_step / 1e3)  # warp instr/s
    peak = 4 * nsm * sm_mhz * 1e6
    return {"bound": "issue", "achieved": rate / 1e12, "peak": peak / 1e12, "unit": "Twarp-instr/s",
            "frac": rate / peak, "instr_per_element": BUILD_INSTR_PER_ELEMENT,
            "note": "table kernel time included (0.4 % of the stage)"}


def hbm_peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs")
    except Exception:
        return None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cfg, coords, y, X, P, lam, budget_s=20.0):
    """The oracle, as it stands, on the host cores over a bounded sample of points."""
    import oracle
    T = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.eval_batch(coords, y, X, P[:T], lam, nthreads=T)  # one point per thread
    t1 = time.perf_counter()
    per_round = t1 - t0
    rounds = max(1, min(4, int(budget_s / max(per_round, 1e-3)) - 1))
    npts = T
    tt = per_round
    if rounds > 1:
        t0 = time.perf_counter()
        oracle.eval_batch(coords, y, X, P[T:T * rounds], lam, nthreads=T)
        tt += time.perf_counter() - t0
        npts += T * (rounds - 1)
    return {"value": npts / tt, "unit": UNIT, "cores": T, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{npts} points of {cfg.name} (n={cfg.n}, p={cfg.p}, M={cfg.M}) over {T} threads, {tt:.1f} s",
            "extrapolated_full_config_hours": cfg.K / (npts / tt) / 3600.0}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle timed on the box's host cores (rank 0 only;
    the other ranks exit without work)."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    cfg = synthgen.CONFIGS[args.config]
    coords, y, X = synthgen.make_dataset(cfg)
    P = synthgen.make_params(cfg)
    lam = synthgen.make_lambdas(cfg.M)
    T = os.cpu_count() or 1
    pts_per_step = T  # one point per host thread per step (C4: ~3 s of CPU each)
    for w in range(args.warmup):
        oracle.eval_batch(coords, y, X, P[w * T:(w + 1) * T][:1], lam, nthreads=1)
    times = []
    for s in range(args.steps):
        sl = P[(s * pts_per_step) % cfg.K:][:pts_per_step]
        t0 = time.perf_counter()
        oracle.eval_batch(coords, y, X, sl, lam, nthreads=T)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    value = pts_per_step / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.desc}", "n": cfg.n, "p": cfg.p, "M": cfg.M,
                       "K_per_step": pts_per_step, "parallelism": "host threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": T, "kind": "oracle",
                             "sample": f"{pts_per_step} points of {cfg.name} per step, {T} threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


def _reserve_stdout():
    """Return a stream on the original stdout and send fd 1 to stderr from here on:
    native libraries (NCCL's version / NCCL_DEBUG lines) write to fd 1 directly, and
    stdout must carry only the one JSON line."""
    sys.stdout.flush()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    return out


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: start the N ranks through
    torch.distributed.run on 127.0.0.1; rank 0's JSON line reaches our stdout."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd, cwd=ROOT)


def probe_ranks(args, rank, world):
    """--probe-ranks: the launch check used by the CPU tests — every rank joins a gloo
    group and rank 0 prints who came (no GPU work)."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.tensor([rank, int(os.environ.get("LOCAL_RANK", "0"))], dtype=torch.int64)
    got = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(got, t)
    if rank == 0:
        print(json.dumps({"probe": True, "world": world, "gpus": args.gpus, "backend": dist.get_backend(),
                          "ranks": [int(g[0]) for g in got], "local_ranks": [int(g[1]) for g in got]}),
              flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default=WORKLOAD, choices=sorted(synthgen.CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's K points sharded over the ranks (default); "
                         "weak: K points per rank")
    ap.add_argument("--points", type=int, default=None,
                    help="points (strong: in total, weak: per rank; default: the config's K)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use torch.distributed (NCCL) even with one process: runs the multi-GPU "
                         "code path (checksum, all-gather, max over ranks) on a single GPU")
    ap.add_argument("--probe-ranks", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and args.gpus != world:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.probe_ranks:
        probe_ranks(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator-init lines on stderr
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    json_out = _reserve_stdout()
    import torch
    import torch.distributed as dist

    import paper_2305_04318_b200 as lik
    from paper_2305_04318_b200 import multi

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.dist
    if use_dist:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(_free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)

    cfg = synthgen.CONFIGS[args.config]
    strong = args.scaling == "strong"
    K_total = (args.points or cfg.K) * (1 if strong else world)
    coords, y, X = synthgen.make_dataset(cfg)
    Pall = synthgen.make_params(cfg, K_total)
    P = np.ascontiguousarray(Pall[rank::world])  # strided sharding balances κ-dependent cost
    K = P.shape[0]
    K_max = multi.local_count(K_total, 0, world)  # the largest shard (rank 0)
    lam = synthgen.make_lambdas(cfg.M)
    n, p, M = cfg.n, cfg.p, cfg.M
    r = M + p

    if use_dist:  # every rank generated the same dataset (§8(e))
        multi.check_same_dataset(coords, y, X, lam, device=dev)
    ctx = lik.create(local, lik.FLAG_TIMING)
    st = torch.cuda.Stream(dev)
    dc, dy, dX, dp, dl = (torch.tensor(a, device=dev) for a in (coords, y, X, P, lam))
    out = lik.Ctx.alloc_outputs(K, M, p, dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    pack_w = multi.pack_width(M, p)
    gathered = torch.empty((world * K_max, pack_w), dtype=torch.float64, device=dev) if use_dist else None

    def step():
        if K:
            ctx.eval_batch_device(dc, dy, dX, dp, dl, out=out, stream=st)
        if use_dist:  # the one exchange step: all-gather of the result tables (NCCL / NVLink)
            with torch.cuda.stream(st):
                dist.all_gather_into_tensor(gathered, multi.pack(out, M, p, K_max))

    for _ in range(args.warmup):
        with torch.cuda.stream(st):
            flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    ctx.reset_stage_times()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t_wall0 = time.perf_counter()
        for s in range(args.steps):
            with torch.cuda.stream(st):
                flush.fill_(float(s))
            evs[s][0].record(st)
            step()
            evs[s][1].record(st)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    if use_dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms_local = float(np.mean(step_ms))
    stages = ctx.stage_times()
    # max over ranks
    t = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = K_total / (ms / 1e3)
    F = dense_flops_per_point(n, r)
    ok_frac = float((out["status"] == 0).float().mean().item()) if K else 1.0

    # ---- e2e through the host-pointer API (pinned host inputs, copies inside the timed region)
    hin = [torch.tensor(a).pin_memory() for a in (coords, y, X, P, lam)]
    hn = [h.numpy() for h in hin]
    e2e_ctx = lik.create(local)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    e2e_steps = max(1, min(args.steps, 2))
    if not use_dist:
        # lik_eval_batch: host inputs in, host outputs back (one C-ABI call)
        e2e_ctx.eval_batch(*hn)  # warm (allocations)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = e2e_ctx.eval_batch(*hn)
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        h2d = sum(a.nbytes for a in hn)
        d2h = sum(v.nbytes for v in res.values())
    else:
        # multi.eval_sharded: this rank's shard up, the all-gathered table of every
        # rank's results back to the host (the multi-GPU public entry point)
        multi.eval_sharded(e2e_ctx, coords, y, X, Pall, lam, dev)  # warm
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = multi.eval_sharded(e2e_ctx, coords, y, X, Pall, lam, dev)
        e2e_s = (time.perf_counter() - t0) / e2e_steps
        h2d = sum(a.nbytes for a in hn)  # coords, y, X, this rank's params, λ
        d2h = world * K_max * pack_w * 8
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if use_dist:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = K_total / float(te.item())
    e2e_ctx.close()

    if rank == 0:
        chol_ms, chol_n = stages["chol_fused"]
        build_ms, build_n = stages["matern_build"]
        clk_med = clk.summary().get("sm_mhz")
        peak, peak_src = fp64_peak()
        achieved = (args.steps * K * F) / (chol_ms / 1e3) / 1e12 if chol_ms > 0 else None
        traffic, traffic_note, ncu_dmma = None, None, None
        try:
            tj = json.load(open(TRAFFIC))
            ncu_dmma = tj.get("dmma_pipe_pct")
            if tj.get("n", 2000) == n:
                pts_per_launch = args.steps * K / chol_n if chol_n else K
                traffic = tj["dram_bytes_per_point"] * pts_per_launch
                traffic_note = (f"dram_bytes_read+write per point from one ncu --set full capture "
                                f"({tj['points_per_launch']}-point launch, {tj['source']}) x "
                                f"{pts_per_launch:.0f} points per launch here")
        except Exception:
            pass
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.desc}", "n": n, "p": p, "M": M,
                       "K_total": K_total, "K_rank0": K,
                       "parallelism": f"points sharded k = rank mod {world} over {world} GPU(s), "
                                      f"one NCCL all-gather of the result tables" if use_dist else
                                      "1 GPU",
                       "l2": "flushed (256 MiB write) before every timed step",
                       "wall_s_timed_region": round(t_wall, 3)},
            "fp64_tflops": value * F / 1e12,
            "fp64_tflops_per_gpu": value * F / 1e12 / world,
            "roofline": {"bound": "tensor", "kernel": "chol_fused (DMMA.8x8x4)",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "traffic_note": traffic_note,
                         "peak_source": peak_src,
                         "ncu_dmma_pipe_pct": ncu_dmma,  # the DMMA pipe's busy share in the committed capture (hardware counter, no peak assumed)
                         "algorithmic": "n^3/3 + n^2 r + n r^2 FP64 flops per point (SURVEY §8(d)), "
                                        "x points per launch / launch duration (CUDA events on the launching stream), rank 0",
                         "share_of_step": chol_ms / (args.steps * ms_local) if ms_local else None},
            "matern_build": {  # table + build per step: ρ evaluations and workspace bytes written
                "evals_per_s": K * n * (n - 1) / 2 / (build_ms / args.steps / 1e3) if build_ms > 0 else None,
                "gb_per_s_written": K * slot_bytes(n, r) / (build_ms / args.steps / 1e3) / 1e9 if build_ms > 0 else None,
                "hbm_peak_gbs": hbm_peak(),
                # its bound is instruction issue: the build kernel's warp
                # instructions per element from the committed ncu capture, against one
                # issue per cycle on every SM sub-partition at the median SM clock
                "issue_roofline": build_issue_roofline(K, n, build_ms / args.steps, clk_med)},
            "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items()},
            "launches_per_step": {k: v[1] / args.steps for k, v in stages.items()},
            "gpu_launches": int(sum(v[1] for v in stages.values())),
            "clocks": clk.summary(),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "status_ok_fraction": ok_frac,
            "input_hash": synthgen.input_hash(coords, y, X, P, lam),
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(cfg, coords, y, X, P, lam)
        print(json.dumps(line), file=json_out, flush=True)
    ctx.close()
    if use_dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
