"""Golden 10-seed episode returns from the reference (run in the build
container, where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_episode_returns.py

The protocol of the reference's acceptance test
(pkg/tests/test_acceptance.py:319-346, frozen in pkg/docs/scenarios.md:13-27):
for every task and seeds 0..9, run_episode (rollout.py:46-69) of a batch-1
Env(seed=s) under HeuristicPolicy() and under RandomPolicy(seed=1000 + s).
Writes episode_returns.json with every per-seed return at full float64
precision, so the device run can be compared bitwise, not just to the doc's
two decimals.
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from swarmsim import Env, HeuristicPolicy, RandomPolicy, create_scenario, run_episode, scenario_names  # noqa: E402


def main() -> None:
    out = {}
    for name in sorted(scenario_names()):
        heur = [float(run_episode(Env(create_scenario(name), 1, seed=s), HeuristicPolicy())[0]) for s in range(10)]
        rand = [float(run_episode(Env(create_scenario(name), 1, seed=s), RandomPolicy(seed=1000 + s))[0])
                for s in range(10)]
        out[name] = {"scripted": heur, "random": rand,
                     "scripted_mean": float(np.mean(heur)), "random_mean": float(np.mean(rand))}
        print(f"{name}: scripted {np.mean(heur):.3f} vs random {np.mean(rand):.3f}", flush=True)
    Path(__file__).with_name("episode_returns.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
