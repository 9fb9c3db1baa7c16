"""e2e loop of bench.py with Env(validate=True / False), a few repetitions:
is the per-step NaN verdict read (.item()) serialised behind the big
observation copies on the device-to-host copy engine?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2207_03530_b200 import Env, create_scenario  # noqa: E402

dev = torch.device("cuda:0")
B, A = 1_000_000, 3
host_acts = [[torch.from_numpy(np.random.default_rng(7 + k).uniform(-1, 1, (B, 2)).astype(np.float32)).pin_memory()
              for _ in range(A)] for k in range(4)]
for validate in (True, False, True, False):
    env = Env(create_scenario("simple_spread", n_agents=A), B, seed=0, device=dev, validate=validate)
    O = len(env.observations()[0][0])
    sec = bench.e2e_rate(env, host_acts, 10, A, B, O, dev, False)
    print("validate", validate, "e2e %.3g" % (B * A * 10 / sec), "ms/step %.3f" % (sec / 10 * 1e3), flush=True)
