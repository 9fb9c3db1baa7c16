"""Decode paths outside the fused kernels' continuous decode, pinned bitwise
to reference runs (tests/golden/noise_golden.npz, generated from the
reference by tests/golden/make_noise_golden.py): Gaussian action noise
(env.py:139-142) and observation noise (env.py:203-205), drawn from the Env's
own Philox stream interleaved with the reset draws, and the discrete action
mode (env.py:100-135)."""
from pathlib import Path

import numpy as np
import pytest

import paper_2207_03530_b200 as S

pytestmark = pytest.mark.gpu

G = np.load(Path(__file__).parent / "golden" / "noise_golden.npz")
CASES = [
    ("noise_spread", "simple_spread", 16, "continuous", {0: (0.1, 0.0), 1: (0.0, 0.05), 2: (0.2, 0.02)}),
    ("noise_transport", "transport", 12, "continuous", {1: (0.3, 0.0), 3: (0.0, 0.1)}),
    ("discrete_spread", "simple_spread", 16, "discrete", {}),
    ("discrete_flocking", "flocking", 10, "discrete", {2: (0.05, 0.0)}),
]


def state(env):
    return env.world.state_array().cpu().numpy()


@pytest.mark.parametrize("tag,name,B,mode,noise", CASES, ids=[c[0] for c in CASES])
def test_noise_and_discrete_match_reference(cuda, tag, name, B, mode, noise):
    env = S.Env(S.create_scenario(name), B, seed=7, device=cuda, action_mode=mode)
    for k, (an, on) in noise.items():
        env.agents[k].action_noise_std = an
        env.agents[k].obs_noise_std = on
    obs0 = env.reset()
    np.testing.assert_array_equal(np.stack([o.cpu().numpy() for o in obs0]), G[tag + "_obs0"])
    acts = G[tag + "_actions"]
    for t in range(acts.shape[0]):
        r = env.step(list(acts[t]))
        np.testing.assert_array_equal(np.stack([o.cpu().numpy() for o in r.obs]), G[tag + "_obs"][t],
                                      err_msg=f"obs @ {t}")
        np.testing.assert_array_equal(np.stack([x.cpu().numpy() for x in r.rewards]), G[tag + "_rew"][t])
        np.testing.assert_array_equal(r.dones.cpu().numpy(), G[tag + "_done"][t])
    np.testing.assert_array_equal(state(env), G[tag + "_state"])
