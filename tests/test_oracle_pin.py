"""The oracle is pinned before it is trusted (CPU).

1. Against the committed golden fixtures (generated from the reference by
   tests/golden/make_golden.py): every step's state / obs hashes, rewards,
   dones, the Philox state, and the reset sequences — bit-exact.
2. Against the reference itself, imported from /root/reference (skipped on
   the GPU box where it does not exist), on configs and seeds the fixtures
   do not cover: random batch sizes, other seeds, multi-index resets.
"""
import json

import numpy as np
import pytest

import golden_util as G
from oracle import swarm_oracle as O


def _oracle_env(meta):
    ov = dict(meta["overrides"])
    if meta["lidar_rays"]:
        ov["lidar_rays"] = meta["lidar_rays"]
    return O.OracleEnv(meta["scenario"], meta["batch"], seed=meta["seed"], **ov)


def _state(env) -> np.ndarray:
    ws = env.ws
    return np.stack([np.stack([ws.px[k], ws.py[k], ws.vx[k], ws.vy[k], ws.rot[k], ws.w[k]])
                     for k in range(len(ws.bodies))])


def _rng(env) -> dict:
    st = env.rng.bit_generator.state
    return {"counter": [int(x) for x in st["state"]["counter"]], "key": [int(x) for x in st["state"]["key"]],
            "buffer": [int(x) for x in st["buffer"]], "buffer_pos": int(st["buffer_pos"])}


@pytest.mark.parametrize("tag", [m["tag"] for m in G.manifest() if m.get("oracle", True)])
def test_oracle_matches_golden(tag):
    meta = next(m for m in G.manifest() if m["tag"] == tag)
    g = G.load(tag)
    env = _oracle_env(meta)
    assert [b.name for b in env.ws.bodies] == meta["entities"]
    np.testing.assert_array_equal(_state(env), g["state0"])
    assert G.canon_hash(env.observations()) == str(g["obs0_hash"])
    assert _rng(env) == G.rng_dict(g["rng0"])
    plans = G.pregen_actions(env.ws.n_agents, meta["batch"], meta["steps"], meta["action_seed"])
    for t, plan in enumerate(plans, start=1):
        obs, rew, done = env.step(plan)
        assert G.canon_hash([_state(env)]) == str(g["state_hash"][t - 1]), f"state @ {t}"
        assert G.canon_hash(obs) == str(g["obs_hash"][t - 1]), f"obs @ {t}"
        np.testing.assert_array_equal(np.stack(rew), g["rew"][t - 1])
        np.testing.assert_array_equal(done, g["done"][t - 1])
    assert _rng(env) == G.rng_dict(g["rng_final"])
    env.reset(int(g["reset_single_index"]))
    np.testing.assert_array_equal(_state(env), g["reset_single_state"])
    env.reset_mask(np.isin(np.arange(meta["batch"]), g["reset_multi_index"]))
    np.testing.assert_array_equal(_state(env), g["reset_multi_state"])
    assert _rng(env) == G.rng_dict(g["reset_multi_rng"])
    env.reset()
    np.testing.assert_array_equal(_state(env), g["reset_all_state"])
    assert _rng(env) == G.rng_dict(g["reset_all_rng"])


LIVE = [
    ("simple_spread", {"n_agents": 4}, 37, 40, 5),
    ("transport", {"n_agents": 3}, 29, 60, 9),
    ("flocking", {"n_agents": 6, "n_obstacles": 2}, 23, 40, 11),
    ("dispersion", {"n_agents": 7, "n_food": 9}, 31, 60, 3),
    ("discovery", {"n_agents": 9, "n_points": 4}, 19, 60, 4),
]


def _ref_state(env) -> np.ndarray:
    rows = []
    for e in env.world.entities:
        s = e.state
        rows.append(np.stack([s.pos.x, s.pos.y, s.vel.x, s.vel.y, s.rot, s.ang_vel]).astype(np.float32))
    return np.stack(rows)


@pytest.mark.reference
@pytest.mark.parametrize("name,ov,B,steps,seed", LIVE)
def test_oracle_matches_reference_live(reference, name, ov, B, steps, seed):
    ref = reference.Env(reference.create_scenario(name, **ov), batch_size=B, seed=seed)
    orc = O.OracleEnv(name, B, seed=seed, **ov)
    np.testing.assert_array_equal(_state(orc), _ref_state(ref))
    plans = G.pregen_actions(len(ref.agents), B, steps, seed + 100)
    for t, plan in enumerate(plans):
        r = ref.step(plan)
        obs, rew, done = orc.step(plan)
        np.testing.assert_array_equal(_state(orc), _ref_state(ref), err_msg=f"step {t}")
        for a, b in zip(obs, r.obs):
            np.testing.assert_array_equal(a, b)
        for a, b in zip(rew, r.rewards):
            np.testing.assert_array_equal(a, b.astype(np.float32))
        np.testing.assert_array_equal(done, r.dones)
        if t == steps // 2:
            sel = np.zeros(B, dtype=bool)
            sel[[1, B // 2, B - 2]] = True
            for i in np.flatnonzero(sel):
                ref.reset(env_index=int(i))
            orc.reset_mask(sel)
            np.testing.assert_array_equal(_state(orc), _ref_state(ref))
    assert json.dumps(_rng(orc)) == json.dumps({
        "counter": [int(x) for x in ref.rng.state()["state"]["counter"]],
        "key": [int(x) for x in ref.rng.state()["state"]["key"]],
        "buffer": [int(x) for x in ref.rng.state()["buffer"]],
        "buffer_pos": int(ref.rng.state()["buffer_pos"])})


@pytest.mark.reference
def test_oracle_lidar_matches_reference(reference):
    """The oracle's lidar restatement vs the reference's lidar_scan."""
    ref = reference.Env(reference.create_scenario("flocking", n_agents=5, n_obstacles=3), batch_size=64, seed=3)
    orc = O.OracleEnv("flocking", 64, seed=3, n_agents=5, n_obstacles=3)
    lid = reference.Lidar(n_rays=16, max_range=0.8)
    for i, agent in enumerate(ref.agents):
        np.testing.assert_array_equal(O.lidar(orc.ws, i, 16, 0.8), reference.lidar_scan(agent, lid, ref.world))
