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


def _ref_step_substeps(reference, env, plan, k):
    """The reference's Env.step (env.py:209-235) with world_step replaced by k
    reference world_step calls at PhysParams(dt=dt/k) on the held decoded
    actions: the definition of the sub-step extension (core.PhysParams)."""
    import dataclasses

    from swarmsim.dynamics import world_step
    from swarmsim.env import decode_action

    actions = [decode_action(raw, spec, agent, env.rng) for raw, agent, spec in
               zip(plan, env.agents, env.action_specs)]
    base = env.world.params
    env.world.params = dataclasses.replace(base, dt=base.dt / k)
    try:
        for _ in range(k):
            world_step(env.world, actions)
    finally:
        env.world.params = base
    env.scenario.post_step(env.world)
    env.step_count += 1
    rew = [env.scenario.reward(a, env.world).astype(np.float32) for a in env.agents]
    done = env.scenario.done(env.world) | (env.step_count >= env.max_steps)
    return env.observations(), rew, done


@pytest.mark.reference
@pytest.mark.parametrize("name,ov,k", [("simple_spread", {"n_agents": 3}, 4), ("transport", {"n_agents": 4}, 3),
                                       ("flocking", {"n_agents": 5, "n_obstacles": 3}, 2),
                                       ("discovery", {"n_agents": 6}, 3)])
def test_oracle_substeps_match_reference_composition(reference, name, ov, k):
    """Oracle with Phys.substeps = k == k reference world_step calls of dt / k
    per step (pins the sub-step extension to the reference's own functions)."""
    B, steps = 48, 25
    ref = reference.Env(reference.create_scenario(name, **ov), batch_size=B, seed=5)
    orc = O.OracleEnv(name, B, seed=5, substeps=k, **ov)
    for t, plan in enumerate(G.pregen_actions(len(ref.agents), B, steps, 77)):
        r_obs, r_rew, r_done = _ref_step_substeps(reference, ref, plan, k)
        obs, rew, done = orc.step(plan)
        np.testing.assert_array_equal(_state(orc), _ref_state(ref), err_msg=f"step {t}")
        for a, b in zip(obs, r_obs):
            np.testing.assert_array_equal(a, b)
        for a, b in zip(rew, r_rew):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(done, r_done)


def test_oracle_joint_newton_and_pull():
    """Joint forces are equal and opposite (bitwise) and pull a stretched
    pair together / push a compressed pair apart."""
    bodies = [O.Body("a", "sphere", (0.05,), movable=True), O.Body("b", "sphere", (0.05,), movable=True)]
    ws = O.WorldState(bodies, 64)
    rng = np.random.default_rng(0)
    ws.px[0] = rng.uniform(-1, 1, 64).astype(np.float32)
    ws.py[0] = rng.uniform(-1, 1, 64).astype(np.float32)
    d0 = np.hypot(ws.px[0] - ws.px[1], ws.py[0] - ws.py[1])
    O.world_step(ws, {}, joints=[O.JointSpec(0, 1, dist=0.5)])
    np.testing.assert_array_equal(ws.vx[0], -ws.vx[1])
    np.testing.assert_array_equal(ws.vy[0], -ws.vy[1])
    d1 = np.hypot(ws.px[0] - ws.px[1], ws.py[0] - ws.py[1])
    far, near = d0 > 0.51, d0 < 0.49
    assert far.any() and near.any()
    assert (d1[far] < d0[far]).all() and (d1[near] > d0[near]).all()
