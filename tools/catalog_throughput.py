"""Step throughput of every catalog task on one GPU (eager Env.step).

    python tools/catalog_throughput.py [B] [STEPS]

The five BASELINE tasks run their fused kernel; the other eight run
k_generic_physics plus their torch-on-device reward / observation ports.
Actions are device-resident uniform forces ((A, B, 2) tensor, validate=False);
prints one JSON line per task: eager Env.step and Env.step_graph (10 steps
per replay).
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2207_03530_b200 as S  # noqa: E402


def main() -> None:
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    dev = torch.device("cuda:0")
    for name in S.scenario_names():
        env = S.Env(S.create_scenario(name), B, seed=0, device=dev, validate=False)
        A = len(env.agents)
        acts = torch.rand((A, B, 2), device=dev) * 2 - 1
        scripted = any(a.action_script is not None for a in env.agents)
        plan = [None if a.action_script is not None else acts[i] for i, a in enumerate(env.agents)] \
            if scripted else acts
        for _ in range(3):
            env.step(plan)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            env.step(plan)
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / K
        # the same step captured in CUDA graphs of 10 steps (Env.step_graph)
        graph = env.step_graph([acts, acts.clone()], steps_per_replay=10)
        graph.step(0)
        torch.cuda.synchronize()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for k in range(max(1, K // 10)):
            graph.step(k % 2)
        s1.record()
        torch.cuda.synchronize()
        gsec = s0.elapsed_time(s1) / 1e3 / (max(1, K // 10) * 10)
        print(json.dumps({"scenario": name, "envs": B, "agents": A, "fused": bool(env.fused),
                          "ms_per_step": sec * 1e3, "env_steps_per_s": B / sec,
                          "agent_steps_per_s": B * A / sec, "graph_ms_per_step": gsec * 1e3,
                          "graph_agent_steps_per_s": B * A / gsec}), flush=True)
        del graph
        del env
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
