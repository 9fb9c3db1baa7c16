"""Generate the golden fixtures from the REFERENCE implementation.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Runs swarmsim (the reference, imported read-only) through its public API —
Env(create_scenario(name, **overrides), B, seed), Env.step, Env.reset,
lidar_scan — with the reference bench's action protocol (bench.py:35-47:
SeededRng(seed+1) uniform in +-u_range, pre-drawn) and records, per config:

  state0        (E, 6, B) f32   state after construction (reset with `seed`)
  obs0_hash     sha256 of the initial observations
  rng0          Philox state after construction
  state_hash    (T,) per-step sha256 of the full state
  obs_hash      (T,) per-step sha256 of all observations
  rew           (T, A, B) f32 rewards
  done          (T, B) bool
  ckpt_steps    steps (1-based) at which full arrays are stored:
  ckpt_state    (C, E, 6, B) f32,  ckpt_obs_<a> per agent for the last checkpoint
  rng_final     Philox state after the last step
  reset_*       a per-index reset and a sequential multi-index reset after the
                run (state + rng after each)

Hashes are taken over canonicalised float32 bytes (x + 0.0 maps -0.0 to
+0.0) so that equal values hash equally.  The device run must reproduce all
of it bit-for-bit (tests/test_parity_golden.py).
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

# (tag, scenario, overrides, B, steps, lidar_rays)
CONFIGS = [
    ("simple_spread_3_b32", "simple_spread", {"n_agents": 3}, 32, 100, 0),
    ("transport_4_b32", "transport", {"n_agents": 4}, 32, 100, 0),
    ("flocking_5_lidar_b32", "flocking", {"n_agents": 5, "n_obstacles": 3}, 32, 100, 12),
    ("dispersion_4_b32", "dispersion", {}, 32, 100, 0),
    ("discovery_5_b32", "discovery", {}, 32, 100, 0),
    ("dispersion_64x64_b4", "dispersion", {"n_agents": 64, "n_food": 64}, 4, 30, 0),
    ("discovery_64_b4", "discovery", {"n_agents": 64}, 4, 30, 0),
    # the other catalog tasks (generic physics kernel + device hooks)
    ("wheel_b16", "wheel", {}, 16, 60, 0),
    ("balance_b16", "balance", {}, 16, 60, 0),
    ("give_way_b16", "give_way", {}, 16, 60, 0),
    ("football_b16", "football", {}, 16, 60, 0),
    ("passage_b16", "passage", {}, 16, 60, 0),
    ("reverse_transport_b16", "reverse_transport", {}, 16, 60, 0),
    ("dropout_b16", "dropout", {}, 16, 60, 0),
    ("waterfall_b16", "waterfall", {}, 16, 60, 0),
]
SEED = 0
CKPT = (1, 10, 100)


def canon_hash(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float32) + np.float32(0.0))
        h.update(a.tobytes())
    return h.hexdigest()


def ref_state(env) -> np.ndarray:
    rows = []
    for e in env.world.entities:
        s = e.state
        rows.append(np.stack([s.pos.x, s.pos.y, s.vel.x, s.vel.y, s.rot, s.ang_vel]).astype(np.float32))
    return np.stack(rows)


def rng_json(st) -> str:
    """numpy Philox bit_generator.state as JSON (counter, key, buffer, pos)."""
    return json.dumps({
        "counter": [int(x) for x in st["state"]["counter"]],
        "key": [int(x) for x in st["state"]["key"]],
        "buffer": [int(x) for x in st["buffer"]],
        "buffer_pos": int(st["buffer_pos"]),
    })


def ref_obs(env, lidar):
    from swarmsim import lidar_scan

    obs = env.observations()
    if lidar is None:
        return obs
    return [np.concatenate([o, lidar_scan(a, lidar, env.world)], axis=1) for o, a in zip(obs, env.agents)]


def run_config(tag, name, overrides, B, steps, rays):
    from swarmsim import Env, Lidar, create_scenario
    from swarmsim.batching import SeededRng

    lidar = Lidar(n_rays=rays, max_range=1.0) if rays else None
    env = Env(create_scenario(name, **overrides), batch_size=B, seed=SEED)
    out = {"state0": ref_state(env), "obs0_hash": canon_hash(ref_obs(env, lidar)),
           "rng0": rng_json(env.rng.state())}
    arng = SeededRng(SEED + 1)
    plans = [[arng.uniform(-a.u_range, a.u_range, (B, 2)) for a in env.agents] for _ in range(steps)]
    state_hash, obs_hash, rews, dones, ckpt_state, ckpt_steps = [], [], [], [], [], []
    last_obs = None
    for t, plan in enumerate(plans, start=1):
        res = env.step(plan)
        obs = ref_obs(env, lidar) if lidar is not None else res.obs
        st = ref_state(env)
        state_hash.append(canon_hash([st]))
        obs_hash.append(canon_hash(obs))
        rews.append(np.stack(res.rewards).astype(np.float32))
        dones.append(res.dones.copy())
        if t in CKPT or t == steps:
            ckpt_steps.append(t)
            ckpt_state.append(st)
            last_obs = obs
    out.update(
        actions_hash=canon_hash([np.stack(p) for p in plans]),
        state_hash=np.array(state_hash), obs_hash=np.array(obs_hash),
        rew=np.stack(rews), done=np.stack(dones),
        ckpt_steps=np.array(ckpt_steps), ckpt_state=np.stack(ckpt_state),
        rng_final=rng_json(env.rng.state()),
    )
    for a, o in enumerate(last_obs):
        out[f"ckpt_obs_{a}"] = o.astype(np.float32)
    # per-index reset, then a sequential multi-index reset (ascending)
    i0 = B // 2
    env.reset(env_index=i0)
    out["reset_single_index"] = np.array(i0)
    out["reset_single_state"] = ref_state(env)
    out["reset_single_rng"] = rng_json(env.rng.state())
    idx = sorted({0, B - 1, B // 3}) if B > 2 else [0]
    for i in idx:
        env.reset(env_index=i)
    out["reset_multi_index"] = np.array(idx)
    out["reset_multi_state"] = ref_state(env)
    out["reset_multi_rng"] = rng_json(env.rng.state())
    out["reset_multi_obs_hash"] = canon_hash(ref_obs(env, lidar))
    out["reset_multi_step_count"] = env.step_count.copy()
    # whole-batch reset
    env.reset()
    out["reset_all_state"] = ref_state(env)
    out["reset_all_rng"] = rng_json(env.rng.state())
    meta = {"tag": tag, "scenario": name, "overrides": overrides, "batch": B, "steps": steps,
            "seed": SEED, "action_seed": SEED + 1, "lidar_rays": rays,
            "entities": [e.name for e in env.world.entities],
            "oracle": name in ("simple_spread", "transport", "flocking", "dispersion", "discovery")}
    return out, meta


def main(tags=None):
    manifest = []
    for cfg in CONFIGS:
        if tags and cfg[0] not in tags:
            continue
        out, meta = run_config(*cfg)
        np.savez_compressed(HERE / f"{cfg[0]}.npz", **out)
        manifest.append(meta)
        print(f"wrote {cfg[0]}.npz")
    if not tags:
        (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
