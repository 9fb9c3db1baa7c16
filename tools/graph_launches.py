"""Replay a few CUDA-graph steps of one scenario (for an ncu launch list).

    python tools/graph_launches.py SCENARIO [B] [REPLAYS]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2207_03530_b200 as S  # noqa: E402

name = sys.argv[1]
B = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
R = int(sys.argv[3]) if len(sys.argv) > 3 else 3
env = S.Env(S.create_scenario(name), B, seed=0, device="cuda:0", validate=False)
acts = torch.rand((len(env.agents), B, 2), device="cuda:0") * 2 - 1
g = env.step_graph(acts)
for _ in range(R):
    g.step(0)
torch.cuda.synchronize()
print(f"{name}: {R} graph replays of {B} envs ok")
