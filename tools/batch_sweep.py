"""Throughput vs number of parallel envs on one GPU (the paper's scaling sweep).

    python tools/batch_sweep.py SCENARIO B1 B2 ... [--steps K]

For each batch size: a fresh Env stepped by CUDA-graph replays of --spr
consecutive fused steps with device-resident random actions (two buffers
cycled), 0.3 s clock soak, then K timed steps.  `probe` instead times a
graph of one 1-element kernel: the harness floor.  Prints one JSON line per size: per-launch median
kernel time (CUDA events around each replay), ms per step over the whole
timed loop, env-steps/s, agent-steps/s and the HBM roofline fraction
(algorithmic bytes per env-step).
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import WORKLOADS, bytes_per_env_step, peaks  # noqa: E402
from paper_2207_03530_b200 import Env, create_scenario  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("scenario")
    ap.add_argument("sizes", type=int, nargs="+")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--spr", type=int, default=10, help="steps per graph replay")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    if args.scenario == "probe":
        # the timing floor of this harness: a graph of one 1-element kernel
        x = torch.zeros(1, device=dev)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
            x.add_(1.0)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(1000):
            g.replay()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
        torch.cuda.synchronize()
        for a, b in ev:
            a.record()
            g.replay()
            b.record()
        torch.cuda.synchronize()
        print(json.dumps({"probe": "1-element kernel graph", "kernel_ms": float(np.median([a.elapsed_time(b) for a, b in ev])),
                          "ms_per_step": ev[0][0].elapsed_time(ev[-1][1]) / len(ev)}))
        return
    scen, ov, _ = WORKLOADS[args.scenario][:3]
    hbm = peaks()["hbm_gbs"]
    for B in args.sizes:
        env = Env(create_scenario(scen, **ov), B, seed=0, device=dev, validate=False)
        A = len(env.agents)
        O = env.observations()[0].shape[1]
        bpe = bytes_per_env_step(scen, A, len(env.world.entities) - A, O)
        acts = [torch.rand((A, B, 2), device=dev) * 2 - 1 for _ in range(2)]
        S = args.spr if A * B * (O * 4 + 4) * args.spr <= 4e9 else 1
        g = env.step_graph(acts, steps_per_replay=S)
        t0, n = time.perf_counter(), 0
        while time.perf_counter() - t0 < 0.3:
            g.step(n % 2)
            n += 1
            if n % 16 == 0:
                torch.cuda.synchronize()
        K = max(1, args.steps // S)
        s = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        torch.cuda.synchronize()
        ends = []
        for k in range(K):
            s[k].record()
            g.step(k % 2)
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            ends.append(e)
        s[K].record()
        torch.cuda.synchronize()
        launch = float(np.median([s[k].elapsed_time(ends[k]) for k in range(K)])) / S
        total = s[0].elapsed_time(s[K]) / (K * S)
        rate = B / (total / 1e3)
        print(json.dumps({"scenario": args.scenario, "envs": B, "steps_per_replay": S, "kernel_ms": launch,
                          "ms_per_step": total,
                          "env_steps_per_s": rate, "agent_steps_per_s": rate * A,
                          "bytes_per_env_step": bpe, "hbm_frac": bpe * B / (launch / 1e3) / 1e9 / hbm,
                          "working_set_mb": bpe * B / 1e6}), flush=True)
        del g, env
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
