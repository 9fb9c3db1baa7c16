"""Golden runs of the decode paths the fused-kernel fixtures do not cover:
Gaussian action / observation noise (env.py:139-142, 203-205; drawn from the
Env's Philox stream by numpy's standard_normal) and the discrete action mode
(env.py:100-135).  Generated from the reference (build container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_noise_golden.py

Writes noise_golden.npz: per case and step the observations, rewards, dones
and the final entity state, for bitwise comparison on the device
(tests/test_gpu_noise_discrete.py).
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import swarmsim as R  # noqa: E402

# (tag, scenario, overrides, batch, steps, action_mode, {agent: (action_noise, obs_noise)})
CASES = [
    ("noise_spread", "simple_spread", {}, 16, 25, "continuous", {0: (0.1, 0.0), 1: (0.0, 0.05), 2: (0.2, 0.02)}),
    ("noise_transport", "transport", {}, 12, 25, "continuous", {1: (0.3, 0.0), 3: (0.0, 0.1)}),
    ("discrete_spread", "simple_spread", {}, 16, 25, "discrete", {}),
    ("discrete_flocking", "flocking", {}, 10, 25, "discrete", {2: (0.05, 0.0)}),
]


def state(env):
    return np.stack([np.stack([e.state.pos.x, e.state.pos.y, e.state.vel.x, e.state.vel.y, e.state.rot,
                               e.state.ang_vel]).astype(np.float32) for e in env.world.entities])


def actions(g, A, B, mode):
    if mode == "discrete":
        return [g.integers(0, 5, (B,)) for _ in range(A)]
    return [g.uniform(-1.0, 1.0, (B, 2)).astype(np.float32) for _ in range(A)]


def main() -> None:
    out = {}
    for tag, name, ov, B, steps, mode, noise in CASES:
        env = R.Env(R.create_scenario(name, **ov), batch_size=B, seed=7, action_mode=mode)
        for k, (an, on) in noise.items():
            env.agents[k].action_noise_std = an
            env.agents[k].obs_noise_std = on
        obs0 = env.reset()
        g = np.random.Generator(np.random.Philox(99))
        A = len(env.agents)
        acts, obs, rew, done = [], [], [], []
        for _ in range(steps):
            a = actions(g, A, B, mode)
            r = env.step(a)
            acts.append(np.stack(a))
            obs.append(np.stack(r.obs).astype(np.float32))
            rew.append(np.stack(r.rewards).astype(np.float32))
            done.append(r.dones.copy())
        out[tag + "_obs0"] = np.stack(obs0).astype(np.float32)
        out[tag + "_actions"] = np.stack(acts)
        out[tag + "_obs"] = np.stack(obs)
        out[tag + "_rew"] = np.stack(rew)
        out[tag + "_done"] = np.stack(done)
        out[tag + "_state"] = state(env)
    np.savez_compressed(Path(__file__).with_name("noise_golden.npz"), **out)
    print(sorted(out))


if __name__ == "__main__":
    main()
