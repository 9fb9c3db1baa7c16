"""Benchmark: batched env-step throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--scenario simple_spread]
                    [--envs B] [--strong] [--impl b200|reference] [--dry-run]

One JSON line on rank 0.  A "step" is one Env.step of the whole batch on
every GPU.  Weak scaling (default): B envs per GPU; rank r holds the global
env range [r*B, (r+1)*B) of one N*B-env batch, so the sharded run is the
1-GPU run of N*B envs, random stream included.  --strong keeps the batch
global (BASELINE config 5: 262144 envs sharded over 1/2/4/8 GPUs).
`--gpus N` without a launcher spawns the N ranks itself (one process per
GPU, RANK / WORLD_SIZE / LOCAL_RANK / MASTER_ADDR=127.0.0.1); under torchrun
it checks WORLD_SIZE == N.  Inputs are device-resident synthetic uniform
actions; working sets that fit the 126 MB L2 cycle enough action buffers to
exceed it (config.l2 says which).

  value  — agent-steps/s over all GPUs, kernel path (actions resident in HBM):
           CUDA-graph replays of the validated step (NaN scan + guarded fused
           launch, as Env.step), CUDA-event timed, max over ranks.
  e2e    — the same metric through the public API with host buffers: pinned
           host actions in (Env.step), obs/rewards/dones copied out to pinned
           host memory on a second stream every step (step k's device->host
           copy overlaps step k+1's host->device copy and compute).
  roofline — the fused step kernel: algorithmic bytes / launch time vs the
           measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline — the reference's CPU path on one host core, bounded sample:
           the unmodified reference (swarmsim, installed in baseline/_ref)
           when present ("reference"), else the oracle port ("port").

--impl reference: the reference's CPU path on every host core (one process
per core, a start barrier, wall clock around all of them), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
L2_BYTES = 126_000_000


# algorithmic HBM bytes per env-step: state r/w once,
# actions read, obs/reward/done written, step_count r/w.  Split into what
# every step moves (actions in, outputs out) and what a launch moves once
# (state read + written, static entities, step_count): a fused rollout of S
# steps pays the second part once per S steps.
def step_bytes(scenario: str, A: int, n_other: int, obs_dim: int) -> tuple[int, int]:
    io = 8 * A + 4 * A * obs_dim + 4 * A + 1
    if scenario == "simple_spread":
        return io, 32 * A + 8 * A + 16            # agents r/w, markers, step_count r/w
    if scenario == "transport":
        return io, 32 * (A + 1) + 8 + 8 + 16      # agents + package r/w, goal, package rot
    if scenario == "flocking":
        return io, 32 * A + 8 * (1 + n_other) + 16
    if scenario == "dispersion":
        return io + 4, 32 * A + 8 * n_other + 16 + 8   # + fresh-bites aux / eaten flags
    if scenario == "discovery":
        return io + 8 * n_other, 32 * A + 8 * n_other + 16 + 8   # + point relocations
    raise ValueError(scenario)


def bytes_per_env_step(scenario: str, A: int, n_other: int, obs_dim: int, steps_per_launch: int = 1) -> float:
    per_step, per_launch = step_bytes(scenario, A, n_other, obs_dim)
    return per_step + per_launch / steps_per_launch


# name: scenario, overrides, envs (per GPU, or global with --strong),
# (1-core cpu_baseline sample envs, steps), reference-arm sample envs per step
WORKLOADS = {
    # cpu_baseline samples (envs, steps): ~10 s of one host core each
    "simple_spread": ("simple_spread", {"n_agents": 3}, 1_000_000, (1_000_000, 20), 1_000_000),
    "transport": ("transport", {"n_agents": 4}, 100_000, (100_000, 200), 100_000),
    "flocking": ("flocking", {"n_agents": 5, "n_obstacles": 3, "lidar_rays": 12}, 100_000, (20_000, 50), 100_000),
    "dispersion": ("dispersion", {"n_agents": 64, "n_food": 64}, 262_144, (1024, 7), 8192),
    "discovery": ("discovery", {"n_agents": 64}, 262_144, (2048, 25), 32768),
}


def workload_string(name: str, B: int, Bg: int, world: int, strong: bool) -> str:
    scen, ov = WORKLOADS[name][0], WORKLOADS[name][1]
    if strong:
        return f"{scen} {ov}, {Bg} envs sharded over {world} GPU(s)"
    return f"{scen} {ov}, {B} envs per GPU"


def ncu_traffic(scenario: str, envs: int, rollout: int = 0):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the fused
    kernel from the committed ncu --set full captures (profiles/r02, then
    r01), if one was taken at this batch size; else None.  rollout=S: the
    capture of the S-step rollout kernel, its bytes per launch / S (per
    step, like roofline.achieved)."""
    for rnd in ("r02", "r01"):
        p = ROOT / "profiles" / rnd / "ncu_traffic.json"
        if not p.exists():
            continue
        d = json.loads(p.read_text()).get(scenario)
        if not d:
            continue
        if "envs" in d:                      # r01 layout: one capture per scenario
            d = {str(d["envs"]): d}
        hit = d.get(f"{envs}@rollout{rollout}" if rollout else str(envs))
        if hit:
            return hit["dram_bytes_per_launch"] / hit.get("steps_per_launch", 1), f"profiles/{rnd}/ncu_traffic.json"
    return None, None


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons, sampled every 50 ms by a reader
    thread for as long as the context is open (soak + warm-up + timed steps)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.rows: list[list[str]] = []
        self.error = None

    def _reader(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7 and parts[0].isdigit():
                self.rows.append(parts)

    def __enter__(self):
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True, bufsize=1)
            self.thread = threading.Thread(target=self._reader, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError) as exc:
            self.proc, self.error = None, str(exc)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [f"nvidia-smi unavailable: {self.error}"]}
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        import statistics

        sm = [int(r[0]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][1]),
                "reasons": sorted(reasons), "samples": len(rows)}


# ---------------------------------------------------------------------------
# process launch: one process per GPU
# ---------------------------------------------------------------------------
def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks of this script
    (rank r on GPU r), forward their output, return the worst exit code."""
    port = str(_free_port())
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, str(Path(__file__).resolve()), *sys.argv[1:]], env=env))
    rc = 0
    for p in procs:
        rc = max(rc, p.wait())
    return rc


def dist_setup(n_gpus: int, use_cuda: bool = True):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"bench.py --gpus {n_gpus} launched with WORLD_SIZE={world}")
    # SS_DIST_BACKEND=gloo exercises the multi-rank path where there is no
    # NCCL peer (several ranks on one GPU, or --dry-run on a CPU host)
    backend = os.environ.get("SS_DIST_BACKEND", "nccl" if use_cuda else "gloo")
    if use_cuda:
        local = local % max(1, torch.cuda.device_count())
    if world > 1:
        if use_cuda:
            torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif use_cuda and torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world: int, dev) -> None:
    import torch
    import torch.distributed as dist

    if world > 1:
        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[dev.index])
        else:
            dist.barrier()
    if dev is not None and dev.type == "cuda":
        torch.cuda.synchronize(dev)


def max_over_ranks(x: float, world: int, dev) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# the reference's CPU path
# ---------------------------------------------------------------------------
def load_reference():
    """The unmodified reference package (swarmsim) from baseline/_ref."""
    p = ROOT / "baseline" / "_ref"
    if not (p / "swarmsim" / "__init__.py").exists():
        return None
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    try:
        import swarmsim

        return swarmsim
    except Exception:       # broken install: fall back to the oracle port
        return None


class CpuRun:
    """One CPU process stepping B envs of a workload through the reference's
    public API (Env.step, plus lidar_scan per agent for the Lidar-extended
    flocking config, appended to the observations as the B200 path does),
    or through the oracle port when the reference is not installed.  Actions
    are pre-drawn as the reference's bench does (bench.py:35-47)."""

    def __init__(self, name: str, B: int, n_steps: int, seed: int = 0):
        import numpy as np

        scen, ov = WORKLOADS[name][0], dict(WORKLOADS[name][1])
        self.ref = load_reference()
        rays = ov.pop("lidar_rays", 0) if self.ref is not None else 0
        if self.ref is not None:
            R = self.ref
            self.kind = "reference"
            self.env = R.Env(R.create_scenario(scen, **ov), batch_size=B, seed=seed)
            self.lidar = R.Lidar(n_rays=rays, max_range=1.0) if rays else None
            A = len(self.env.agents)
        else:
            from oracle import swarm_oracle as O

            self.kind = "port"
            self.env = O.OracleEnv(scen, B, seed=seed, **ov)
            self.lidar = None
            A = self.env.ws.n_agents
        self.A, self.B = A, B
        g = np.random.Generator(np.random.Philox(seed + 1))
        self.acts = [[g.uniform(-1.0, 1.0, (B, 2)).astype(np.float32) for _ in range(A)] for _ in range(n_steps)]

    def step(self, k: int) -> None:
        import numpy as np

        res = self.env.step(self.acts[k])
        if self.lidar is not None:
            scan = self.ref.lidar_scan
            _ = [np.concatenate([o, scan(a, self.lidar, self.env.world)], axis=1)
                 for o, a in zip(res.obs, self.env.agents)]

    def describe(self) -> str:
        if self.kind == "reference":
            return "the unmodified reference (swarmsim 0.1.0 from baseline/_ref, numpy) through Env.step"
        return "oracle/swarm_oracle.py (numpy restatement pinned bit-exact to the reference)"


def cpu_rate(name: str, B: int, steps: int, warmup: int = 1) -> dict:
    """Single-process env-steps/s of the reference's CPU path on a bounded sample."""
    run = CpuRun(name, B, warmup + steps)
    for t in range(warmup):
        run.step(t)
    t0 = time.perf_counter()
    for t in range(warmup, warmup + steps):
        run.step(t)
    sec = time.perf_counter() - t0
    return {"env_steps_per_s": B * steps / sec, "agent_steps_per_s": B * run.A * steps / sec,
            "seconds": sec, "B": B, "steps": steps, "kind": run.kind, "what": run.describe()}


def _ref_worker(name, B, W, K, seed, bar, q):
    run = CpuRun(name, B, W + K, seed)
    for t in range(W):
        run.step(t)
    bar.wait()
    t0 = time.perf_counter()           # CLOCK_MONOTONIC: comparable across processes
    for t in range(W, W + K):
        run.step(t)
    q.put((t0, time.perf_counter(), run.kind, run.describe(), run.A))


def run_reference(args, rank, world) -> None:
    """--impl reference: the reference's CPU path on every host core (rank 0)."""
    if rank != 0:
        return
    import multiprocessing as mp

    name = args.scenario
    default_b, sample = WORKLOADS[name][2], WORKLOADS[name][4]
    B = args.envs or default_b
    Bg = B if args.strong else B * world
    cores = len(os.sched_getaffinity(0))
    total = min(Bg, sample)               # envs stepped per timed step (bounded sample)
    per = max(1, total // cores)
    ctx = mp.get_context("fork")
    bar, q = ctx.Barrier(cores), ctx.Queue()
    procs = [ctx.Process(target=_ref_worker, args=(name, per, args.warmup, args.steps, 1000 + c, bar, q))
             for c in range(cores)]
    for p in procs:
        p.start()
    got = [q.get() for _ in procs]
    for p in procs:
        p.join()
    sec = max(g[1] for g in got) - min(g[0] for g in got)     # wall clock around all workers
    kind, what, A = got[0][2], got[0][3], got[0][4]
    envs = per * cores
    value = envs * A * args.steps / sec
    line = {
        "impl": "reference", "metric": "agent-steps/sec", "value": value, "unit": "agent-steps/s",
        "env_steps_per_s": envs * args.steps / sec, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000 * sec / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_string(name, B, Bg, world, args.strong), "scenario": WORKLOADS[name][0],
                   "envs_per_gpu": B if not args.strong else None, "global_envs": Bg},
        "cpu_baseline": {"value": value, "unit": "agent-steps/s", "cores": cores, "kind": kind,
                         "sample": f"{envs} of the workload's {Bg} envs per step ({per} per process), "
                                   f"{args.steps} timed steps after {args.warmup} warm-up; {what}; "
                                   f"{cores} processes, one per host core, started on a barrier, "
                                   f"wall clock around all"},
        "e2e": {"value": value, "unit": "agent-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the B200 path
# ---------------------------------------------------------------------------
def pinned_copy_gbs(dev, nbytes: int = 256 << 20) -> dict:
    """Measured pinned-host <-> device bandwidth (the e2e link ceiling)."""
    import torch

    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    out = {}
    for name, (dst, src) in {"h2d": (d, h), "d2h": (h, d)}.items():
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(4):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize(dev)
        out[name] = 4 * nbytes / (time.perf_counter() - t0) / 1e9
    return out


def e2e_rate(env, host_acts, K, A, B, O, dev, keep_obs_on_device: bool):
    """Env.step with pinned host actions; each step's outputs copied to pinned
    host buffers on a copy stream (double-buffered), so step k's D2H overlaps
    step k+1's H2D + compute.  Returns seconds for K steps."""
    import torch

    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    nb = 2
    obs_h = [torch.empty((A, B, O), dtype=torch.float32).pin_memory() for _ in range(nb)] if not keep_obs_on_device else None
    rew_h = [torch.empty((A, B), dtype=torch.float32).pin_memory() for _ in range(nb)]
    done_h = [torch.empty(B, dtype=torch.bool).pin_memory() for _ in range(nb)]
    ready = [None] * nb
    checksum = 0.0

    def step(k):
        nonlocal checksum
        j = k % nb
        if ready[j] is not None:
            ready[j].synchronize()               # buffer j's result is on the host: read it
            checksum += float(rew_h[j][0, 0])
        res = env.step(host_acts[k % len(host_acts)])
        ev = torch.cuda.Event()
        ev.record(comp)
        copy.wait_event(ev)
        with torch.cuda.stream(copy):
            if obs_h is not None:
                for a in range(A):
                    obs_h[j][a].copy_(res.obs[a], non_blocking=True)
                    res.obs[a].record_stream(copy)
            for a in range(A):
                rew_h[j][a].copy_(res.rewards[a], non_blocking=True)
                res.rewards[a].record_stream(copy)
            done_h[j].copy_(res.dones, non_blocking=True)
            res.dones.record_stream(copy)
        done_ev = torch.cuda.Event()
        done_ev.record(copy)
        ready[j] = done_ev

    step(0)
    torch.cuda.synchronize(dev)
    ready[:] = [None] * nb
    t0 = time.perf_counter()
    for k in range(1, K + 1):
        step(k)
    for ev in ready:
        if ev is not None:
            ev.synchronize()
    return time.perf_counter() - t0


def run_b200(args, rank, world, local) -> None:
    import numpy as np
    import torch

    from paper_2207_03530_b200 import Env, create_scenario

    dev = torch.device("cuda", local)
    name = args.scenario
    scen, ov, default_b = WORKLOADS[name][0], WORKLOADS[name][1], WORKLOADS[name][2]
    if args.strong:
        from paper_2207_03530_b200.parallel import shard_range

        Bg = args.envs or default_b
        off, B = shard_range(rank, world, Bg)
    else:
        B = args.envs or default_b
        off, Bg = rank * B, world * B
    env = Env(create_scenario(scen, **ov), B, seed=0, device=dev, validate=False,
              env_offset=off, global_batch=Bg)
    A = len(env.agents)
    O = len(env.observations()[0][0])
    n_other = len(env.world.entities) - A
    K, W = args.steps, args.warmup
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    # a pool of distinct action sets, cycled; together they span > 2x L2 (or
    # one set alone exceeds L2), so no step reads actions left in L2
    set_bytes = A * B * 8
    pool = 1 if set_bytes > L2_BYTES else max(2, min(8, -(-2 * L2_BYTES // set_bytes)))
    acts = [torch.rand((A, B, 2), device=dev, generator=gen).mul_(2.0).sub_(1.0) for _ in range(pool)]
    stream = torch.cuda.current_stream(dev)
    # Env.step as CUDA-graph replays of S consecutive validated fused steps
    # (NaN scan + guarded launch, the eager Env.step's work without its host
    # sync), S the largest divisor of K up to 10 while the S steps' outputs
    # (distinct graph-owned buffers) stay under 32 GB of the 180 GB HBM: the
    # GPU runs step after step as in a long rollout, each step's scan
    # overlapping the previous step
    out_bytes = A * B * (O * 4 + 4) + B
    cap = 32e9
    S = max(s for s in range(1, 11) if K % s == 0 and s * out_bytes <= cap) if out_bytes <= cap else 1
    graph = env.step_graph(acts, steps_per_replay=S, validate=True, fused_rollout=False if args.per_step else None)
    # the step kernel alone (its share of the validated step): the same
    # replays without the NaN scan, captured now so that its timing follows
    # the value loop without an idle gap (same clocks / power state)
    kgraph = env.step_graph(acts, steps_per_replay=S, fused_rollout=False if args.per_step else None)
    R = K // S
    # a fused rollout kernel moves the state once per S steps
    bpe = bytes_per_env_step(scen, A, n_other, O, S if graph.fused_rollout else 1)
    launches_per_replay = graph.launches_per_replay

    # ---- kernel-path throughput (device-resident inputs) -------------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
    with ClockSampler(dev.index) as clocks:
        t_soak, n = time.perf_counter(), 0     # clock soak: nvidia-smi sees loaded clocks
        while time.perf_counter() - t_soak < args.soak:
            graph.step(n % pool)
            n += 1
            if n % max(1, 64 // S) == 0:
                torch.cuda.synchronize(dev)
        for t in range(-(-W // S)):            # >= W warm-up steps
            graph.step(t % pool)
        barrier(world, dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(R):
            starts[k].record(stream)
            graph.step((W + k) % pool)
            ends[k].record(stream)
        t1.record(stream)
        # the kernel-only replays, back to back with the value loop
        kst = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        ken = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
        kgraph.step(0)
        for k in range(R):
            kst[k].record(stream)
            kgraph.step((W + k) % pool)
            ken[k].record(stream)
        torch.cuda.synchronize(dev)
    graph.check()                              # no NaN was replayed
    barrier(world, dev)
    ms_total = max_over_ranks(t0.elapsed_time(t1), world, dev)
    ms_step = float(np.median(sorted(s.elapsed_time(e) / S for s, e in zip(starts, ends))))
    env_steps = Bg * K
    value = env_steps * A / (ms_total / 1000.0)

    ms_launch = float(np.median(sorted(s.elapsed_time(e) / S for s, e in zip(kst, ken))))
    achieved = bpe * B / (ms_launch / 1e3) / 1e9
    graph_fused = graph.fused_rollout
    del graph, kgraph

    # ---- end to end through the public API with host buffers --------------
    env_e2e = Env(create_scenario(scen, **ov), B, seed=0, device=dev, validate=True,
                  env_offset=off, global_batch=Bg)
    host_acts = [[torch.from_numpy(np.random.default_rng(7 + k).uniform(-1, 1, (B, 2)).astype(np.float32)).pin_memory()
                  for _ in range(A)] for k in range(4)]
    # enough steps for ~0.3 s of end-to-end stepping (10..300): a 10-step
    # loop of a small workload lasts a few ms, within reach of one host hiccup
    calib = max_over_ranks(e2e_rate(env_e2e, host_acts, 3, A, B, O, dev, False), world, dev) / 3
    E2E_K = int(max_over_ranks(float(min(300, max(10, int(0.3 / max(calib, 1e-6))))), world, dev))
    barrier(world, dev)
    e2e_sec = max_over_ranks(e2e_rate(env_e2e, host_acts, E2E_K, A, B, O, dev, False), world, dev)
    barrier(world, dev)
    metric_sec = max_over_ranks(e2e_rate(env_e2e, host_acts, E2E_K, A, B, O, dev, True), world, dev)
    e2e_value = Bg * A * E2E_K / e2e_sec
    h2d = A * B * 8
    d2h = A * B * O * 4 + A * B * 4 + B
    link = pinned_copy_gbs(dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cb, cs = WORKLOADS[name][3]
        r = cpu_rate(name, min(B, cb), cs)
        cpu = {"value": r["agent_steps_per_s"], "unit": "agent-steps/s", "cores": 1, "kind": r["kind"],
               "sample": f"{r['B']} envs x {cs} steps of the same workload, {r['what']}, 1 core"}

    # episode statistics of the e2e rollout, all-reduced over NVLink (NCCL)
    # once, outside every timed region — the only collective of the run
    from paper_2207_03530_b200.parallel import EpisodeStats

    stats = EpisodeStats(B, dev)
    res = env_e2e.step(host_acts[0])
    stats.update(res.rewards, res.dones)
    episode = stats.reduce()

    if rank == 0:
        pk = peaks()
        traffic, tsrc = ncu_traffic(scen, B, S if graph_fused else 0)
        line = {
            "metric": "agent-steps/sec", "value": value, "unit": "agent-steps/s",
            "env_steps_per_s": env_steps / (ms_total / 1000.0),
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_total / K,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic uniform actions in [-1,1]; env state from the scenario's reset distribution",
            "config": {"workload": workload_string(name, B, Bg, world, args.strong), "scenario": scen,
                       "envs_per_gpu": B, "global_envs": Bg, "agents": A, "obs_dim": O,
                       "l2": ("working set > L2 (no flush needed)" if bpe * B > L2_BYTES else
                              f"L2-resident step: {pool} action buffers cycled, {pool * set_bytes >> 20} MiB"),
                       "validate": True,
                       "stepping": (f"Env.step_graph(steps_per_replay={S}, validate=True): CUDA-graph replays of "
                                    + (f"the {S} action scans + ONE fused rollout kernel of {S} steps (state on "
                                       "chip between them)" if graph_fused else
                                       f"{S} consecutive validated fused steps (NaN scan + guarded launch)")
                                    + f", {pool} action buffer(s) cycled; e2e: eager Env.step(validate=True) with "
                                      "host buffers")},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": traffic,
                         "traffic_source": tsrc and (f"{tsrc} (ncu --set full, one launch at {B} envs"
                                                     + (f", the {S}-step rollout kernel's bytes / {S})"
                                                        if graph_fused else ")")),
                         "bytes_per_env_step": bpe,
                         "bytes_model": (f"per step {step_bytes(scen, A, n_other, O)[0]} B (actions, outputs) + "
                                         f"{step_bytes(scen, A, n_other, O)[1]} B (state r/w, static, step_count) "
                                         f"per launch of {S if graph_fused else 1} step(s)"),
                         "kernel_ms": ms_launch, "step_ms": ms_step,
                         "kernel_timing": "CUDA events around each kernel-only replay, back to back with the "
                                          "timed value loop (same clocks / power state)",
                         "kernel_share_of_step": ms_launch / ms_step, "peak_source": pk["source"]},
            "e2e": {"value": e2e_value, "unit": "agent-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": E2E_K,
                    # the host link: the step's D2H (obs dominate) overlaps the
                    # next step's H2D; fraction of the measured pinned D2H copy rate
                    "link_gbs": (h2d + d2h) * E2E_K / e2e_sec / 1e9,
                    "pinned_copy_gbs": link,
                    "d2h_frac_of_pinned": d2h * E2E_K / e2e_sec / 1e9 / link["d2h"],
                    "obs_on_device": {"value": Bg * A * E2E_K / metric_sec, "h2d_bytes_per_step": h2d,
                                      "d2h_bytes_per_step": A * B * 4 + B}},
            # per replay: one action-scan launch (per 16 steps) + the S step kernels or one rollout kernel
            "gpu_launches": R * launches_per_replay,
            "fused_rollout": graph_fused,
            "steps_per_replay": S,
            "episode_stats": {"mean_return_1step": episode["mean_return"], "envs": episode["envs"],
                              "reduced_over_ranks": world},
            "clock_soak_s": args.soak,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


def run_dry(args, rank, world) -> None:
    """--dry-run: the launch path only (rendezvous, barriers, max over ranks)
    with a host-timed placeholder step; no GPU work, value null."""
    t0 = time.perf_counter()
    time.sleep(0.01 * (rank + 1))
    barrier(world, None)
    sec = max_over_ranks(time.perf_counter() - t0, world, None)
    if rank == 0:
        name = args.scenario
        B = args.envs or WORKLOADS[name][2]
        Bg = B if args.strong else B * world
        print(json.dumps({"metric": "agent-steps/sec", "value": None, "dry_run": True, "n_gpus": world,
                          "max_rank_seconds": sec, "steps": args.steps, "warmup": args.warmup,
                          "config": {"workload": workload_string(name, B, Bg, world, args.strong)}}), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--scenario", choices=sorted(WORKLOADS), default="simple_spread")
    ap.add_argument("--envs", type=int, default=0, help="envs per GPU (default: the workload's)")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: --envs / the workload's batch is the global batch, sharded over ranks")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--per-step", action="store_true",
                    help="per-step graph replays even where a fused rollout kernel exists (A/B)")
    ap.add_argument("--soak", type=float, default=1.5, help="seconds of untimed steps for clock sampling")
    ap.add_argument("--dry-run", action="store_true", help="launch path only (no GPU work)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        if args.impl == "reference":
            pass                               # rank 0 alone runs the CPU reference
        else:
            raise SystemExit(spawn_ranks(args.gpus))
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
        run_reference(args, rank, world)
        return
    rank, world, local = dist_setup(args.gpus, use_cuda=not args.dry_run)
    if args.dry_run:
        run_dry(args, rank, world)
    else:
        run_b200(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
