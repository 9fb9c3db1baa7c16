"""Device parity against the golden fixtures generated from the reference.

For every config in tests/golden/manifest.json the B200 Env (public API,
through the C-ABI) must reproduce the reference bit-for-bit:
  * the state after construction (numpy-Philox reset on the device),
  * every step's full state and observations (canonical sha256),
  * every step's rewards and dones (exact arrays),
  * the Philox stream state after the run,
  * a per-index reset, a multi-index reset (as reset_at) and a whole reset.
Free-running for the full horizon: any 1-ulp deviation would compound and
show up as a hash mismatch (SURVEY.md finding 5).
"""
import numpy as np
import pytest
import torch

import golden_util as G

pytestmark = pytest.mark.gpu

CONFIGS = [m["tag"] for m in G.manifest()]


def _make_env(meta, cuda):
    from paper_2207_03530_b200 import Env, create_scenario

    ov = dict(meta["overrides"])
    if meta["lidar_rays"]:
        ov["lidar_rays"] = meta["lidar_rays"]
    return Env(create_scenario(meta["scenario"], **ov), meta["batch"], seed=meta["seed"], device=cuda)


def _rng_words(env) -> dict:
    st = env.rng.state()
    return {"counter": [int(x) for x in st["state"]["counter"]], "key": [int(x) for x in st["state"]["key"]],
            "buffer": [int(x) for x in st["buffer"]], "buffer_pos": int(st["buffer_pos"])}


def _state(env) -> np.ndarray:
    return env.world.state_array().cpu().numpy()


@pytest.mark.parametrize("tag", CONFIGS)
def test_free_running_bitwise(tag, cuda):
    meta = next(m for m in G.manifest() if m["tag"] == tag)
    g = G.load(tag)
    env = _make_env(meta, cuda)
    assert [e.name for e in env.world.entities] == meta["entities"]
    np.testing.assert_array_equal(_state(env), g["state0"])
    assert G.canon_hash([o.cpu().numpy() for o in env.observations()]) == str(g["obs0_hash"])
    assert _rng_words(env) == G.rng_dict(g["rng0"])
    A = len(env.agents)
    plans = G.pregen_actions(A, meta["batch"], meta["steps"], meta["action_seed"])
    assert G.canon_hash([np.stack(p) for p in plans]) == str(g["actions_hash"])
    ck = {int(t): i for i, t in enumerate(g["ckpt_steps"])}
    for t, plan in enumerate(plans, start=1):
        res = env.step(plan)
        st = _state(env)
        obs = [o.cpu().numpy() for o in res.obs]
        if t in ck:
            np.testing.assert_array_equal(st, g["ckpt_state"][ck[t]], err_msg=f"{tag} state @ step {t}")
        assert G.canon_hash([st]) == str(g["state_hash"][t - 1]), f"{tag}: state diverged at step {t}"
        np.testing.assert_array_equal(torch.stack(res.rewards).cpu().numpy(), g["rew"][t - 1],
                                      err_msg=f"{tag} rewards @ step {t}")
        np.testing.assert_array_equal(res.dones.cpu().numpy(), g["done"][t - 1], err_msg=f"{tag} dones @ {t}")
        assert G.canon_hash(obs) == str(g["obs_hash"][t - 1]), f"{tag}: observations diverged at step {t}"
    for a, o in enumerate(obs):
        np.testing.assert_array_equal(o, g[f"ckpt_obs_{a}"])
    assert _rng_words(env) == G.rng_dict(g["rng_final"])

    # per-index reset, then the multi-index reset as ONE masked launch
    env.reset(env_index=int(g["reset_single_index"]))
    np.testing.assert_array_equal(_state(env), g["reset_single_state"])
    assert _rng_words(env) == G.rng_dict(g["reset_single_rng"])
    obs = env.reset_at([int(i) for i in g["reset_multi_index"]])
    np.testing.assert_array_equal(_state(env), g["reset_multi_state"])
    assert _rng_words(env) == G.rng_dict(g["reset_multi_rng"])
    assert G.canon_hash([o.cpu().numpy() for o in obs]) == str(g["reset_multi_obs_hash"])
    np.testing.assert_array_equal(env.step_count.cpu().numpy(), g["reset_multi_step_count"])
    env.reset()
    np.testing.assert_array_equal(_state(env), g["reset_all_state"])
    assert _rng_words(env) == G.rng_dict(g["reset_all_rng"])
