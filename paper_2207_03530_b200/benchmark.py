"""Throughput sweeps with the reference harness's API (swarmsim/bench.py).

bench_throughput(...) keeps the reference's rows and CSV schema
(n_envs, mode, steps, seconds; bench.py:22-130) and adds the device modes:

  vectorized  one batched Env of n envs, eager Env.step (validated public
              API) with actions pre-drawn on the host (bench.py:35-60)
  graph       the same batch stepped by CUDA-graph replay of the fused step
              with device-resident actions (Env.step_graph)
  sequential  n independent B=1 Envs stepped in a Python loop (bench.py:63-75)

Times are device times: CUDA events around the timed steps after
synchronising, wall clock only for the host-bound sequential loop.
write_csv(rows, path, extended=True) appends gpus / agents /
env_steps_per_s / agent_steps_per_s / hbm_gbs / roofline_frac columns.
"""
from __future__ import annotations

import csv
import json
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from .batching import SeededRng
from .env import Env
from .scenarios import create_scenario


@dataclass
class BenchRow:
    n_envs: int
    mode: str
    steps: int
    seconds: float
    agents: int = 0
    bytes_per_env_step: int | None = None
    extra: dict = field(default_factory=dict)


def _env(name, n, seed, overrides, device, validate=True):
    return Env(create_scenario(name, **(overrides or {})), batch_size=n, seed=seed, device=device,
               validate=validate)


def _pregen(env: Env, n_steps: int, seed: int) -> list:
    rng = SeededRng(seed)
    return [[None if a.action_script is not None else rng.uniform(-a.u_range, a.u_range, (env.batch_size, 2))
             for a in env.agents] for _ in range(n_steps)]


def _time_vectorized(name, n, n_steps, seed, warmup, overrides, device) -> float:
    env = _env(name, n, seed, overrides, device)
    acts = _pregen(env, warmup + n_steps, seed + 1)
    for t in range(warmup):
        env.step(acts[t])
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for t in range(warmup, warmup + n_steps):
        env.step(acts[t])
    torch.cuda.synchronize(device)
    return time.perf_counter() - t0


def _time_graph(name, n, n_steps, seed, warmup, overrides, device) -> float:
    env = _env(name, n, seed, overrides, device, validate=False)
    A = len(env.agents)
    g = torch.Generator(device=device)
    g.manual_seed(seed + 1)
    acts = [torch.rand((A, n, 2), device=device, generator=g) * 2 - 1 for _ in range(2)]
    graph = env.step_graph(acts)
    for t in range(warmup):
        graph.step(t % 2)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(device)
    s.record()
    for t in range(n_steps):
        graph.step(t % 2)
    e.record()
    torch.cuda.synchronize(device)
    return s.elapsed_time(e) / 1e3


def _time_sequential(name, n, n_steps, seed, warmup, overrides, device) -> float:
    envs = [_env(name, 1, seed + k, overrides, device) for k in range(n)]
    plans = [_pregen(envs[k], warmup + n_steps, seed + 1 + k) for k in range(n)]
    for env, acts in zip(envs, plans):
        for t in range(warmup):
            env.step(acts[t])
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for env, acts in zip(envs, plans):
        for t in range(warmup, warmup + n_steps):
            env.step(acts[t])
    torch.cuda.synchronize(device)
    return time.perf_counter() - t0


_TIMERS = {"vectorized": _time_vectorized, "graph": _time_graph, "sequential": _time_sequential}


def bench_throughput(scenario_name: str = "simple_spread", env_counts: list[int] | None = None,
                     n_steps: int = 100, mode: str = "both", seed: int = 0, warmup: int = 5,
                     overrides: dict | None = None, threads: int = 1, device=None) -> list[BenchRow]:
    """One row per (mode, size), sorted by (mode, n_envs) (bench.py:78-115).

    mode: "both" (= vectorized + sequential, as the reference), "vectorized",
    "graph", "sequential" or "all".
    """
    if env_counts is None:
        env_counts = [1, 1000]
    modes = {"both": ["vectorized", "sequential"], "all": ["graph", "sequential", "vectorized"]}.get(
        mode, [mode])
    if any(m not in _TIMERS for m in modes):
        raise ValueError(f"unknown bench mode {mode!r}")
    device = torch.device(device or "cuda")
    rows = []
    for m in modes:
        for n in sorted(env_counts):
            try:
                sec = _TIMERS[m](scenario_name, n, n_steps, seed, warmup, overrides, device)
            except torch.cuda.OutOfMemoryError:
                sec = float("nan")
            rows.append(BenchRow(n_envs=n, mode=m, steps=n_steps, seconds=sec))
    with torch.cuda.device(device):
        probe = _env(scenario_name, 1, seed, overrides, device)
    for r in rows:
        r.agents = len(probe.agents)
    rows.sort(key=lambda r: (r.mode, r.n_envs))
    return rows


def steps_per_second(row: BenchRow) -> float:
    """Env-steps per second (bench.py:126-130)."""
    if not row.seconds or row.seconds != row.seconds:
        return float("nan")
    return row.n_envs * row.steps / row.seconds


def write_csv(rows: list[BenchRow], path: str, extended: bool = False, hbm_gbs: float | None = None,
              bytes_per_env_step: int | None = None, gpus: int = 1) -> None:
    """The reference schema n_envs,mode,steps,seconds (+ device columns)."""
    if hbm_gbs is None:
        p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
        hbm_gbs = json.loads(p.read_text())["hbm_gbs"] if p.exists() else 6650.0
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        head = ["n_envs", "mode", "steps", "seconds"]
        if extended:
            head += ["gpus", "agents", "env_steps_per_s", "agent_steps_per_s", "hbm_gbs", "roofline_frac"]
        w.writerow(head)
        for r in sorted(rows, key=lambda r: (r.mode, r.n_envs)):
            line = [r.n_envs, r.mode, r.steps, f"{r.seconds:.6f}"]
            if extended:
                rate = steps_per_second(r)
                gbs = rate * bytes_per_env_step / 1e9 if bytes_per_env_step else float("nan")
                line += [gpus, r.agents, f"{rate:.6g}", f"{rate * r.agents:.6g}", f"{gbs:.6g}",
                         f"{gbs / hbm_gbs:.4f}" if bytes_per_env_step else "nan"]
            w.writerow(line)
