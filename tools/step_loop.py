"""Minimal step loop for profiling: python tools/step_loop.py SCENARIO ENVS STEPS [ROLLOUT].

Runs STEPS fused Env.step calls (validate=False, device-resident actions) of
the bench workload SCENARIO with ENVS envs on cuda:0 — short enough to run
under `ncu --set full` (see profiles/README.md for the exact commands).
ROLLOUT=S > 0: STEPS replays of a StepGraph of S steps with the fused
rollout kernel (one ss_env_rollout launch per replay) instead.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from bench import WORKLOADS  # noqa: E402
from paper_2207_03530_b200 import Env, create_scenario  # noqa: E402


def main() -> None:
    name = sys.argv[1] if len(sys.argv) > 1 else "simple_spread"
    scen, ov, default_b = WORKLOADS[name][:3]
    B = int(sys.argv[2]) if len(sys.argv) > 2 and int(sys.argv[2]) > 0 else default_b
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    env = Env(create_scenario(scen, **ov), B, seed=0, device="cuda:0", validate=False)
    A = len(env.agents)
    acts = torch.rand((A, B, 2), device="cuda:0") * 2 - 1
    roll = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    if roll > 0:
        bufs = [torch.rand((A, B, 2), device="cuda:0") * 2 - 1 for _ in range(2)]
        graph = env.step_graph(bufs, steps_per_replay=roll, fused_rollout=True)
        assert graph.fused_rollout, name
        for k in range(steps):
            graph.step(k % 2)
    for _ in range(steps if roll <= 0 else 0):
        env.step(acts)
    torch.cuda.synchronize()
    print(f"{name}: {steps} steps of {B} envs ok")


if __name__ == "__main__":
    main()
