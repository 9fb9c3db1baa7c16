"""Benchmark: batched env-step throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--scenario simple_spread]
                    [--envs B_PER_GPU] [--strong] [--impl b200|reference]

One JSON line on rank 0.  A "step" is one Env.step of the whole batch on
every GPU (weak scaling: B envs per GPU; rank r holds the global env range
[r*B, (r+1)*B) of one N*B-env batch, so the sharded run is the 1-GPU run of
N*B envs, random stream included).  --strong keeps the batch global (e.g.
dispersion / discovery: 262144 envs sharded over 1/2/4/8 GPUs, BASELINE
config 5) and reports "scaling": "strong".  Inputs are device-resident synthetic
uniform actions; the working set (341 B/env at 1M envs = 341 MB) exceeds the
126 MB L2, so no flush is needed between steps.

  value  — agent-steps/s over all GPUs, kernel path (actions resident in HBM),
           CUDA-event timed, max over ranks.
  e2e    — the same metric through the public API with host buffers: pinned
           host actions copied in and obs/rewards/dones copied out every step
           (e2e.obs_on_device: the same with observations left in HBM for a
           GPU policy, only rewards / dones copied out).
  roofline — the fused step kernel: algorithmic bytes / launch time vs the
           measured HBM copy bandwidth (MEASURED_PEAKS.json).
  cpu_baseline — the reference algorithm (oracle/swarm_oracle.py, a numpy
           port pinned bit-exact to the reference) timed on this host.

--impl reference: the reference's CPU path (the oracle port; the Python
reference itself cannot travel to the GPU box), sharded over every host core.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# algorithmic HBM bytes per env-step: state r/w once,
# actions read, obs/reward/done written, step_count r/w.
def bytes_per_env_step(scenario: str, A: int, n_other: int, obs_dim: int) -> int:
    if scenario == "simple_spread":
        M, S = A, A                           # movable agents, static markers
        return 8 * A + 32 * M + 8 * S + 4 * A * obs_dim + 4 * A + 1 + 16
    if scenario == "transport":
        return 8 * A + 32 * (A + 1) + 8 + 8 + 4 * A * obs_dim + 4 * A + 1 + 16
    if scenario == "flocking":
        return 8 * A + 32 * A + 8 * (1 + n_other) + 4 * A * obs_dim + 4 * A + 1 + 16
    if scenario == "dispersion":
        return 8 * A + 32 * A + 8 * n_other + 4 * A * obs_dim + 4 * A + 1 + 16 + 8 + 4
    if scenario == "discovery":
        return 8 * A + 32 * A + 8 * n_other + 8 * n_other + 4 * A * obs_dim + 4 * A + 1 + 16 + 8
    raise ValueError(scenario)


WORKLOADS = {
    # name: (scenario, overrides, default envs per GPU)
    "simple_spread": ("simple_spread", {"n_agents": 3}, 1_000_000),
    "transport": ("transport", {"n_agents": 4}, 100_000),
    "flocking": ("flocking", {"n_agents": 5, "n_obstacles": 3, "lidar_rays": 12}, 100_000),
    "dispersion": ("dispersion", {"n_agents": 64, "n_food": 64}, 262_144),
    "discovery": ("discovery", {"n_agents": 64}, 262_144),
}


def ncu_traffic(scenario: str, envs: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the fused
    kernel from the committed ncu --set full capture (profiles/r01), if that
    capture was taken at this batch size; else None."""
    p = ROOT / "profiles" / "r01" / "ncu_traffic.json"
    if not p.exists():
        return None
    d = json.loads(p.read_text()).get(scenario)
    if not d or d["envs"] != envs:
        return None
    return d["dram_bytes_per_launch"]


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


def dist_setup(n_gpus: int):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SS_DIST_BACKEND=gloo lets the multi-rank path be exercised with several
    # ranks on one GPU (launch logic only); real runs use NCCL, one GPU per rank
    backend = os.environ.get("SS_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
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
    torch.cuda.synchronize(dev)


def max_over_ranks(x: float, world: int, dev) -> float:
    import torch
    import torch.distributed as dist

    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_oracle_rate(scen: str, overrides: dict, B: int, steps: int, warmup: int = 1) -> dict:
    """Single-process oracle (reference algorithm) env-steps/s on a bounded sample."""
    import numpy as np

    from oracle import swarm_oracle as O

    ov = dict(overrides)
    env = O.OracleEnv(scen, B, seed=0, **ov)
    A = env.ws.n_agents
    g = np.random.Generator(np.random.Philox(1))
    acts = [[g.uniform(-1.0, 1.0, (B, 2)).astype(np.float32) for _ in range(A)] for _ in range(warmup + steps)]
    for t in range(warmup):
        env.step(acts[t])
    t0 = time.perf_counter()
    for t in range(warmup, warmup + steps):
        env.step(acts[t])
    sec = time.perf_counter() - t0
    return {"env_steps_per_s": B * steps / sec, "agent_steps_per_s": B * A * steps / sec,
            "seconds": sec, "B": B, "steps": steps}


def _shard_worker(args):
    scen, overrides, B, steps, warmup = args
    r = cpu_oracle_rate(scen, overrides, B, steps, warmup)
    return r["seconds"]


def run_reference(args, rank, world) -> None:
    """--impl reference: the reference algorithm on every host core (rank 0 only)."""
    if rank != 0:
        return
    import multiprocessing as mp

    scen, ov, default_b = WORKLOADS[args.scenario]
    cores = len(os.sched_getaffinity(0))
    B_total = args.envs or default_b
    per = max(1, B_total // cores)
    A = ov.get("n_agents", 3)
    total_steps = args.steps
    # each step: all cores advance their shard one step; time = slowest shard
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        secs = pool.map(_shard_worker, [(scen, ov, per, total_steps, args.warmup)] * cores)
    sec = max(secs)
    envs = per * cores
    value = envs * A * total_steps / sec
    line = {
        "impl": "reference", "metric": "agent-steps/sec", "value": value, "unit": "agent-steps/s",
        "env_steps_per_s": envs * total_steps / sec, "n_gpus": world, "steps": total_steps,
        "warmup": args.warmup, "ms_per_step": 1000 * sec / total_steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{scen} {ov} , {envs} envs (sharded over {cores} processes)",
                   "scenario": scen, "envs": envs},
        "cpu_baseline": {"value": value, "unit": "agent-steps/s", "cores": cores, "kind": "port",
                         "sample": f"{envs} envs x {total_steps} steps, oracle/swarm_oracle.py "
                                   f"(numpy restatement pinned bit-exact to the reference), {cores} processes"},
        "e2e": {"value": value, "unit": "agent-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args, rank, world, local) -> None:
    import numpy as np
    import torch

    from paper_2207_03530_b200 import Env, create_scenario

    dev = torch.device("cuda", local)
    scen, ov, default_b = WORKLOADS[args.scenario]
    if args.strong:
        # strong scaling: the workload's batch is the GLOBAL batch, sharded
        # over the ranks with the global random-stream layout (parallel.py)
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
    bpe = bytes_per_env_step(scen, A, n_other, O)
    K, W = args.steps, args.warmup
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    # a pool of distinct action sets, cycled; together they span > 2x L2 (or
    # one set alone exceeds L2), so no step reads actions left in L2
    set_bytes = A * B * 8
    pool = 1 if set_bytes > 126_000_000 else max(2, min(8, -(-2 * 126_000_000 // set_bytes)))
    acts = [torch.rand((A, B, 2), device=dev, generator=gen).mul_(2.0).sub_(1.0) for _ in range(pool)]
    stream = torch.cuda.current_stream(dev)
    # Env.step as CUDA-graph replays of S consecutive fused steps each (no
    # host launch between them), S the largest divisor of K up to 10 while S
    # steps' outputs stay under ~4 GB (S = 1 for the 13 GB-per-step obs of
    # dispersion-64): the GPU runs step after step as in a long rollout
    out_bytes = A * B * (O * 4 + 4) + B
    S = max(s for s in range(1, 11) if K % s == 0 and s * out_bytes <= 4e9) if out_bytes <= 4e9 else 1
    graph = env.step_graph(acts, steps_per_replay=S)
    R = K // S

    # ---- kernel-path throughput (device-resident inputs) -------------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(R)]
    with ClockSampler(dev.index) as clocks:
        # clock soak: untimed steps so nvidia-smi sees the loaded clocks
        t_soak, n = time.perf_counter(), 0
        while time.perf_counter() - t_soak < args.soak:
            graph.step(n % pool)
            n += 1
            if n % max(1, 64 // S) == 0:
                torch.cuda.synchronize(dev)
        for t in range(-(-W // S)):         # >= W warm-up steps
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
        torch.cuda.synchronize(dev)
    barrier(world, dev)
    ms_total = max_over_ranks(t0.elapsed_time(t1), world, dev)
    # per-step device time of the fused kernel: each replay's events / S
    per_launch = sorted(s.elapsed_time(e) / S for s, e in zip(starts, ends))
    ms_launch = float(np.median(per_launch))
    env_steps = Bg * K
    value = env_steps * A / (ms_total / 1000.0)
    achieved = bpe * B / (ms_launch / 1e3) / 1e9

    # ---- end to end through the public API with host buffers --------------
    # the reference-facing call: Env.step with validation on (NaN scan +
    # guard), host actions in, observations / rewards / dones back to host
    del graph
    env_e2e = Env(create_scenario(scen, **ov), B, seed=0, device=dev, validate=True,
                  env_offset=off, global_batch=Bg)
    E2E_K = max(3, min(K, 10))
    host_acts = [[torch.from_numpy(np.random.default_rng(7 + k).uniform(-1, 1, (B, 2)).astype(np.float32)).pin_memory()
                  for _ in range(A)] for k in range(E2E_K + 1)]
    obs_h = torch.empty((A, B, O), dtype=torch.float32).pin_memory()
    rew_h = torch.empty((A, B), dtype=torch.float32).pin_memory()
    done_h = torch.empty(B, dtype=torch.bool).pin_memory()

    def e2e_step(k):
        res = env_e2e.step(host_acts[k])
        for a in range(A):
            obs_h[a].copy_(res.obs[a], non_blocking=True)
        rew_h.copy_(torch.stack(res.rewards), non_blocking=True)
        done_h.copy_(res.dones, non_blocking=True)
        torch.cuda.synchronize(dev)

    e2e_step(0)
    barrier(world, dev)
    t0e = time.perf_counter()
    for k in range(1, E2E_K + 1):
        e2e_step(k)
    e2e_sec = max_over_ranks(time.perf_counter() - t0e, world, dev)
    e2e_value = Bg * A * E2E_K / e2e_sec
    h2d = A * B * 8
    d2h = A * B * O * 4 + A * B * 4 + B

    # the same loop for a policy that runs on the GPU: observations stay in
    # HBM, only rewards / dones (the logged metric) come back to the host
    def e2e_metric_step(k):
        res = env_e2e.step(host_acts[k])
        rew_h.copy_(torch.stack(res.rewards), non_blocking=True)
        done_h.copy_(res.dones, non_blocking=True)
        torch.cuda.synchronize(dev)

    barrier(world, dev)
    t0m = time.perf_counter()
    for k in range(1, E2E_K + 1):
        e2e_metric_step(k)
    metric_sec = max_over_ranks(time.perf_counter() - t0m, world, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cb = min(B, args.cpu_envs)
        r = cpu_oracle_rate(scen, ov, cb, args.cpu_steps)
        cpu = {"value": r["agent_steps_per_s"], "unit": "agent-steps/s", "cores": 1, "kind": "port",
               "sample": f"{cb} envs x {args.cpu_steps} steps of the same workload, oracle/swarm_oracle.py "
                         "(numpy restatement pinned bit-exact to the reference), 1 core"}

    # episode statistics of the e2e rollout, all-reduced over NVLink (NCCL)
    # once, outside every timed region — the only collective of the run
    from paper_2207_03530_b200.parallel import EpisodeStats

    stats = EpisodeStats(B, dev)
    res = env_e2e.step(host_acts[0])
    stats.update(res.rewards, res.dones)
    episode = stats.reduce()

    if rank == 0:
        pk = peaks()
        line = {
            "metric": "agent-steps/sec", "value": value, "unit": "agent-steps/s",
            "env_steps_per_s": env_steps / (ms_total / 1000.0),
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": ms_total / K,
            "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic uniform actions in [-1,1]; env state from the scenario's reset distribution",
            "config": {"workload": (f"{scen} {ov}, {Bg} envs sharded over {world} GPU(s)" if args.strong
                                    else f"{scen} {ov}, {B} envs per GPU"), "scenario": scen,
                       "envs_per_gpu": B, "global_envs": Bg, "agents": A, "obs_dim": O,
                       "l2": "working set > L2 (no flush needed)" if bpe * B > 126e6 else "L2-resident",
                       "stepping": f"Env.step_graph(steps_per_replay={S}): CUDA-graph replays of {S} consecutive "
                                   f"fused steps, {pool} action buffer(s) cycled; e2e uses eager Env.step(validate=True)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / pk["hbm_gbs"], "traffic": ncu_traffic(scen, B),
                         "traffic_source": "profiles/r01/ncu_traffic.json (ncu --set full, one launch)",
                         "bytes_per_env_step": bpe, "kernel_ms": ms_launch, "peak_source": pk["source"]},
            "e2e": {"value": e2e_value, "unit": "agent-steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    # the host link carries every step's actions in and obs / rewards /
                    # dones out: achieved PCIe GB/s per GPU (one direction at a time)
                    "link_gbs": (h2d + d2h) * E2E_K / e2e_sec / 1e9,
                    "obs_on_device": {"value": Bg * A * E2E_K / metric_sec, "h2d_bytes_per_step": h2d,
                                      "d2h_bytes_per_step": A * B * 4 + B}},
            "gpu_launches": K,
            "steps_per_replay": S,
            "episode_stats": {"mean_return_1step": episode["mean_return"], "envs": episode["envs"],
                              "reduced_over_ranks": world},
            "clock_soak_s": args.soak,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)


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
    ap.add_argument("--cpu-envs", type=int, default=1_000_000)
    ap.add_argument("--cpu-steps", type=int, default=5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--soak", type=float, default=1.5, help="seconds of untimed steps for clock sampling")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference(args, rank, world)
        return
    rank, world, local = dist_setup(args.gpus)
    run_b200(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
