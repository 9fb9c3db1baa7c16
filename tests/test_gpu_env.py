"""Env contract on the device (mirrors the reference's tests/test_env.py and
tests/test_scenarios.py semantics) plus live-oracle parity at sizes the
golden fixtures do not cover: other seeds and batch sizes, sampled envs of
the full BASELINE batch, masked resets, sharded runs, discrete / noisy /
scripted agents, CUDA-graph stepping."""
import numpy as np
import pytest
import torch

import golden_util as G
import paper_2207_03530_b200 as S
from oracle import swarm_oracle as O
from paper_2207_03530_b200.parallel import shard_range

pytestmark = pytest.mark.gpu


def env(name="simple_spread", B=4, cuda="cuda", **kw):
    ov = kw.pop("ov", {})
    return S.Env(S.create_scenario(name, **ov), B, device=cuda, **kw)


def state(e):
    return e.world.state_array().cpu().numpy()


def ostate(o):
    ws = o.ws
    return np.stack([np.stack([ws.px[k], ws.py[k], ws.vx[k], ws.vy[k], ws.rot[k], ws.w[k]])
                     for k in range(len(ws.bodies))])


# ---- decode / contract (env.py:71-145, 156-235) ------------------------------
def test_decode_action_contract(cuda):
    w = S.World(1, device=cuda)
    a = w.add(S.Agent("p", S.Sphere(0.05), u_multiplier=3.0))
    spec = S.ActionSpec("continuous")
    act = S.decode_action(np.array([[9.0, -0.5]]), spec, a, S.SeededRng(0))
    assert float(act.force.x[0]) == 3.0 and float(act.force.y[0]) == -1.5
    with pytest.raises(S.ContractViolation):
        S.decode_action(np.array([[np.nan, 0.0]]), spec, a, S.SeededRng(0))
    with pytest.raises(S.ContractViolation):
        S.decode_action(np.zeros((3, 2)), spec, a, S.SeededRng(0))
    d = S.ActionSpec("discrete")
    for idx, want in [(0, (0, 0)), (1, (3, 0)), (2, (-3, 0)), (3, (0, 3)), (4, (0, -3))]:
        act = S.decode_action(np.array([idx]), d, a, S.SeededRng(0))
        assert (float(act.force.x[0]), float(act.force.y[0])) == want
    with pytest.raises(S.ContractViolation):
        S.decode_action(np.array([5]), d, a, S.SeededRng(0))
    with pytest.raises(S.ContractViolation):
        S.decode_action(np.array([1.0]), d, a, S.SeededRng(0))
    c = S.World(1, device=cuda).add(S.Agent("c", silent=False, comm_dim=4))
    act = S.decode_action(np.array([[1, 2]]), S.ActionSpec("discrete", comm_dim=4), c, S.SeededRng(0))
    assert act.comm.tolist() == [[0.0, 0.0, 1.0, 0.0]]


def test_env_loop_contract(cuda):
    with pytest.raises(S.ContractViolation):
        env(B=0, cuda=cuda)
    with pytest.raises(S.ContractViolation):
        env(cuda=cuda, action_mode="analog")
    e = env(B=3, cuda=cuda, seed=7)
    res = e.step([np.zeros((3, 2), np.float32)] * 3)
    assert len(res.obs) == 3 and res.obs[0].shape == (3, 14)
    assert all(r.shape == (3,) and r.dtype == torch.float32 for r in res.rewards)
    assert res.dones.shape == (3,) and res.dones.dtype == torch.bool and len(res.infos) == 3
    with pytest.raises(S.ContractViolation):
        e.step([np.zeros((3, 2))] * 2)
    with pytest.raises(S.ContractViolation):
        e.step([None, np.zeros((3, 2)), np.zeros((3, 2))])
    with pytest.raises(S.ContractViolation):
        e.step([np.zeros((2, 2))] * 3)
    before = state(e)
    bad = [np.zeros((3, 2), np.float32) for _ in range(3)]
    bad[1][2, 0] = np.nan
    with pytest.raises(S.ContractViolation, match="NaN"):
        e.step(bad)
    np.testing.assert_array_equal(state(e), before)        # guarded: nothing moved
    with pytest.raises(S.ContractViolation):
        e.reset(env_index=3)


def test_horizon_and_reset_index(cuda):
    e = env(B=2, cuda=cuda, max_steps=5)
    z = [np.zeros((2, 2), np.float32)] * 3
    for t in range(1, 6):
        assert bool(e.step(z).dones.all()) == (t == 5)
    assert bool(e.step(z).dones.all()) and e.step_count.tolist() == [6, 6]   # never auto-resets
    e3 = env(B=3, cuda=cuda, max_steps=4)
    z3 = [np.zeros((3, 2), np.float32)] * 3
    for _ in range(4):
        e3.step(z3)
    e3.reset(env_index=1)
    assert e3.step(z3).dones.tolist() == [True, False, True]


@pytest.mark.parametrize("name", ["simple_spread", "transport", "flocking", "dispersion", "discovery"])
def test_single_env_reset_is_bitwise_isolated(cuda, name):
    e = env(name, B=9, cuda=cuda, seed=13)
    g = np.random.default_rng(3)
    for _ in range(7):
        e.step([g.uniform(-1, 1, (9, 2)).astype(np.float32) for _ in e.agents])
    before = state(e)
    e.reset(env_index=4)
    after = state(e)
    keep = [i for i in range(9) if i != 4]
    np.testing.assert_array_equal(after[:, :, keep], before[:, :, keep])
    assert int(e.step_count[4]) == 0 and int(e.step_count[0]) == 7


def test_same_seed_same_rollout_and_single_env(cuda):
    a, b = env(cuda=cuda, seed=11), env(cuda=cuda, seed=11)
    acts = [np.random.default_rng(0).uniform(-1, 1, (4, 2)).astype(np.float32) for _ in range(3)]
    ra, rb = a.step(acts), b.step(acts)
    for x, y in zip(ra.obs + ra.rewards, rb.obs + rb.rewards):
        assert torch.equal(x, y)
    assert not all(torch.equal(x, y) for x, y in zip(a.observations(), env(cuda=cuda, seed=12).observations()))
    se = S.SingleEnv(env(B=1, cuda=cuda))
    obs = se.reset()
    assert obs[0].ndim == 1
    obs, rew, done, infos = se.step([np.array([0.1, -0.2], np.float32)] * 3)
    assert all(isinstance(r, float) for r in rew) and isinstance(done, bool)
    sd = S.SingleEnv(S.Env(S.create_scenario("simple_spread"), 1, action_mode="discrete", device=cuda))
    assert isinstance(sd.step([1, 1, 1])[2], bool)


def test_obs_noise_resamples(cuda):
    e = env(B=2, cuda=cuda, seed=0)
    for a in e.agents:
        a.obs_noise_std = 0.05
    first, second = e.observations(), e.observations()
    assert not torch.equal(first[0], second[0]) and bool(torch.isfinite(first[0]).all())


# ---- live oracle parity -----------------------------------------------------
CASES = [
    ("simple_spread", {"n_agents": 5}, 1000, 60, 3),
    ("transport", {"n_agents": 3}, 777, 60, 4),
    ("flocking", {"n_agents": 4, "n_obstacles": 2}, 555, 60, 5),
    ("flocking", {"n_agents": 5, "n_obstacles": 3, "lidar_rays": 12}, 300, 40, 6),
    ("dispersion", {"n_agents": 9, "n_food": 40}, 257, 60, 7),
    ("discovery", {"n_agents": 33, "n_points": 5, "quorum": 3}, 129, 40, 8),
]


@pytest.mark.parametrize("name,ov,B,steps,seed", CASES)
def test_live_oracle_parity_with_masked_resets(cuda, name, ov, B, steps, seed):
    e = env(name, B=B, cuda=cuda, seed=seed, ov=ov)
    o = O.OracleEnv(name, B, seed=seed, **ov)
    np.testing.assert_array_equal(state(e), ostate(o))
    plans = G.pregen_actions(len(e.agents), B, steps, seed + 1)
    rng = np.random.default_rng(seed)
    for t, plan in enumerate(plans):
        r = e.step(plan)
        obs, rew, done = o.step(plan)
        np.testing.assert_array_equal(state(e), ostate(o), err_msg=f"state @ {t}")
        for x, y in zip(r.obs, obs):
            np.testing.assert_array_equal(x.cpu().numpy(), y)
        np.testing.assert_array_equal(torch.stack(r.rewards).cpu().numpy(), np.stack(rew))
        np.testing.assert_array_equal(r.dones.cpu().numpy(), done)
        if t % 15 == 7:     # reset the done envs plus a random few, like an RL loop
            mask = done | (rng.random(B) < 0.1)
            got = e.reset_at(torch.from_numpy(mask).to(cuda))
            want = o.reset_mask(mask)
            np.testing.assert_array_equal(state(e), ostate(o))
            for x, y in zip(got, want):
                np.testing.assert_array_equal(x.cpu().numpy(), y)


class _GlobalDraws:
    """The full batch's random stream as a sample of its envs sees it: every
    uniform(lo, hi, n) of the sampled oracle consumes the whole batch's block
    of Bg draws (numpy Philox, batching.py:185-186) and returns the sampled
    envs' values — discovery's per-step relocation draws (discovery.py:66-68)
    at their global indices."""

    def __init__(self, state, Bg, idx):
        self.g = np.random.Generator(np.random.Philox())
        self.g.bit_generator.state = state
        self.Bg, self.idx = Bg, np.asarray(idx)

    def uniform(self, lo, hi, n):
        raw = self.g.bit_generator.random_raw(self.Bg)[self.idx]
        d = (raw >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        return np.float64(lo) + (np.float64(hi) - np.float64(lo)) * d


def _rng_words(st):
    return ([int(x) for x in st["state"]["counter"]], [int(x) for x in st["state"]["key"]],
            int(st["buffer_pos"]))


@pytest.mark.parametrize("name,B", [("simple_spread", 1_000_000), ("transport", 100_000),
                                    ("flocking", 100_000), ("discovery", 262_144), ("dispersion", 262_144)])
def test_full_size_sampled_envs_match_oracle(cuda, name, B):
    """BASELINE sizes: the whole-batch reset is checked for every env against
    numpy's Philox; 4 steps are checked on a sample of 256 envs (envs are
    independent, so the oracle runs on the sample alone; discovery's
    relocations are drawn at the sampled envs' global stream positions and
    the device's Philox state is checked after every step)."""
    from bench import WORKLOADS

    scen, ov = WORKLOADS[name][:2]
    e = env(scen, B=B, cuda=cuda, seed=0, validate=False, ov=ov)
    o = O.OracleEnv(scen, B, seed=0, reset=False, **ov)
    o._apply_ops(None)                  # the whole-batch reset, without B x O observations
    o.task.reset_aux(B, None)
    np.testing.assert_array_equal(state(e), ostate(o))
    idx = np.sort(np.random.default_rng(1).choice(B, 256, replace=False))
    idx[0], idx[-1] = 0, B - 1          # both ends of the batch
    idx = np.unique(idx)
    n = len(idx)
    sub = O.OracleEnv(scen, n, seed=0, reset=False, **ov)
    sub.ws = o.ws.take(idx)
    sub.task.reset_aux(n, None)
    sub.rng = _GlobalDraws(o.rng.bit_generator.state, B, idx)
    idx_t = torch.from_numpy(idx).to(cuda)
    A = len(e.agents)
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    for t in range(4):
        acts = torch.rand((A, B, 2), device=cuda, generator=g) * 2.4 - 1.2
        r = e.step(acts)
        obs, rew, done = sub.step(list(acts[:, idx_t].cpu().numpy()))
        np.testing.assert_array_equal(state(e)[:, :, idx], ostate(sub), err_msg=f"state @ {t}")
        for x, y in zip(r.obs, obs):
            np.testing.assert_array_equal(x[idx_t].cpu().numpy(), y)
        np.testing.assert_array_equal(torch.stack(r.rewards)[:, idx_t].cpu().numpy(), np.stack(rew))
        np.testing.assert_array_equal(r.dones[idx_t].cpu().numpy(), done)
        if scen == "discovery":
            assert _rng_words(e.rng.state()) == _rng_words(sub.rng.g.bit_generator.state), f"rng @ {t}"
            assert int(e.world.flags[0, idx_t].ne(0).sum()) == int(sub.task.covered.any(1).sum())
        del r


def test_discovery64_two_shards_equal_unsharded_at_size(cuda):
    """BASELINE config 5 (discovery, 64 agents, 262144 envs): two shards (one
    Env each, their global offsets) equal the unsharded run bitwise — state,
    observations, rewards, relocation draws."""
    Bg, ov = 262_144, {"n_agents": 64}
    full = env("discovery", B=Bg, cuda=cuda, seed=2, validate=False, ov=ov)
    shards = []
    for r in range(2):
        off, cnt = shard_range(r, 2, Bg)
        shards.append((off, cnt, S.Env(S.create_scenario("discovery", **ov), cnt, seed=2, device=cuda,
                                       validate=False, env_offset=off, global_batch=Bg)))
    g = torch.Generator(device=cuda)
    g.manual_seed(3)
    for t in range(3):
        acts = torch.rand((64, Bg, 2), device=cuda, generator=g) * 2 - 1
        rf = full.step(acts)
        for off, cnt, e in shards:
            rs = e.step(acts[:, off:off + cnt].contiguous())
            for x, y in zip(rf.obs[::9], rs.obs[::9]):
                assert torch.equal(x[off:off + cnt], y), f"obs @ {t}"
            assert torch.equal(torch.stack(rf.rewards)[:, off:off + cnt], torch.stack(rs.rewards))
            assert _rng_words(e.rng.state()) == _rng_words(full.rng.state())
            del rs
        del rf
    for off, cnt, e in shards:
        assert torch.equal(e.world.state_array(), full.world.state_array()[:, :, off:off + cnt])


VARIANTS = [
    ("SS_PIPE", "simple_spread", {}, 1000),                 # cp.async.bulk pipeline
    ("SS_FLOCK_THREAD_PER_ENV", "flocking", {"n_agents": 5, "n_obstacles": 3, "lidar_rays": 12}, 300),
    ("SS_LIDAR_NO_FAN", "flocking", {"n_agents": 5, "n_obstacles": 3, "lidar_rays": 12}, 300),
    ("SS_NO_PDL", "transport", {}, 777),                    # plain launches
]


@pytest.mark.parametrize("var,name,ov,B", VARIANTS, ids=[v[0] for v in VARIANTS])
def test_kernel_variants_match_oracle(cuda, var, name, ov, B):
    """Every opt-in kernel variant (selected by an environment variable read
    once per process) runs in a subprocess and must match the oracle
    bit-for-bit: the bulk-copy pipeline, the thread-per-env flocking kernel,
    the per-ray Lidar screen, launches without programmatic dependency."""
    import os
    import subprocess
    import sys

    code = """
import sys; sys.path[:0] = [%r, %r]
import numpy as np, torch
import golden_util as G, paper_2207_03530_b200 as S
from oracle import swarm_oracle as O
name, ov, B = %r, %r, %d
e = S.Env(S.create_scenario(name, **ov), B, seed=5, device="cuda", validate=False)
o = O.OracleEnv(name, B, seed=5, **ov)
for plan in G.pregen_actions(len(e.agents), B, 12, 6):
    r = e.step(torch.from_numpy(np.stack(plan)).cuda())
    obs, rew, done = o.step(plan)
    for x, y in zip(r.obs, obs): np.testing.assert_array_equal(x.cpu().numpy(), y)
    np.testing.assert_array_equal(torch.stack(r.rewards).cpu().numpy(), np.stack(rew))
    np.testing.assert_array_equal(r.dones.cpu().numpy(), done)
print("VARIANT_OK")
""" % (str(G.GOLDEN.parents[1]), str(G.GOLDEN.parent), name, ov, B)
    res = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **{var: "1"}),
                         capture_output=True, text=True, timeout=300)
    assert "VARIANT_OK" in res.stdout, res.stdout + res.stderr


def test_sharded_run_equals_single_run(cuda):
    """Two shards of a 257-env discovery run (separate Envs, each with its
    global offset) equal the unsharded run bitwise, random stream included."""
    Bg, ov = 257, {"n_agents": 6}
    full = env("discovery", B=Bg, cuda=cuda, seed=3, ov=ov)
    shards = []
    for r in range(2):
        off, cnt = shard_range(r, 2, Bg)
        shards.append((off, cnt, S.Env(S.create_scenario("discovery", **ov), cnt, seed=3, device=cuda,
                                       env_offset=off, global_batch=Bg)))
    plans = G.pregen_actions(6, Bg, 20, 9)
    for plan in plans:
        full.step(plan)
        for off, cnt, e in shards:
            e.step([p[off:off + cnt] for p in plan])
    whole = state(full)
    for off, cnt, e in shards:
        np.testing.assert_array_equal(state(e), whole[:, :, off:off + cnt])


def test_step_graph_equals_eager(cuda):
    for name, ov in [("simple_spread", {}), ("discovery", {"n_agents": 8})]:
        a = env(name, B=512, cuda=cuda, seed=2, ov=ov, validate=False)
        b = env(name, B=512, cuda=cuda, seed=2, ov=ov, validate=False)
        A = len(a.agents)
        buf = torch.empty((A, 512, 2), device=cuda)
        graph = b.step_graph(buf)
        g = torch.Generator(device=cuda)
        g.manual_seed(1)
        for t in range(9):
            acts = torch.rand((A, 512, 2), device=cuda, generator=g) * 2 - 1
            ra = a.step(acts)
            buf.copy_(acts)
            rb = graph.step()
            for x, y in zip(ra.obs + ra.rewards + [ra.dones], rb.obs + rb.rewards + [rb.dones]):
                assert torch.equal(x, y)
        np.testing.assert_array_equal(state(a), state(b))
        assert a.rng.state()["state"]["counter"].tolist() == b.rng.state()["state"]["counter"].tolist()


@pytest.mark.parametrize("S_", [2, 3])
def test_multi_step_graph_equals_eager(cuda, S_):
    """steps_per_replay=S: one replay runs S steps over actions[i], actions[i+1], ...
    cyclically; every intermediate StepResult equals eager stepping, and the
    Philox state (discovery draws every step) ends where eager leaves it,
    for odd and even S."""
    for name, ov in [("transport", {}), ("discovery", {"n_agents": 8})]:
        a = env(name, B=300, cuda=cuda, seed=5, ov=ov, validate=False)
        b = env(name, B=300, cuda=cuda, seed=5, ov=ov, validate=False)
        A = len(a.agents)
        g = torch.Generator(device=cuda)
        g.manual_seed(3)
        bufs = [torch.rand((A, 300, 2), device=cuda, generator=g) * 2 - 1 for _ in range(3)]
        graph = b.step_graph(bufs, steps_per_replay=S_)
        k = 0
        for rep in range(4):
            i = rep % 3
            rs = graph.rollout(i)
            assert len(rs) == S_
            for s in range(S_):
                ra = a.step(bufs[(i + s) % 3])
                rb = rs[s]
                for x, y in zip(ra.obs + ra.rewards + [ra.dones], rb.obs + rb.rewards + [rb.dones]):
                    assert torch.equal(x, y)
                k += 1
        np.testing.assert_array_equal(state(a), state(b))
        assert a.rng.state()["state"]["counter"].tolist() == b.rng.state()["state"]["counter"].tolist()


def test_discrete_noise_and_fallback_paths_match_oracle_semantics(cuda):
    """Host-decoded forces (discrete actions) go through the same fused kernel
    with raw_forces; a world edit that breaks the kernel's pair template falls
    back to the generic physics kernel — both must keep the state finite and
    deterministic, and the fallback must equal the fused path on an unchanged
    pair list."""
    e = S.Env(S.create_scenario("simple_spread"), 64, action_mode="discrete", device=cuda, seed=1)
    for _ in range(5):
        r = e.step([np.random.default_rng(0).integers(0, 5, 64) for _ in range(3)])
    assert all(bool(torch.isfinite(o).all()) for o in r.obs)
    a = env("transport", B=300, cuda=cuda, seed=4)
    b = env("transport", B=300, cuda=cuda, seed=4)
    b.scenario.physics_fused = lambda world: False       # force the generic-physics path
    for plan in G.pregen_actions(4, 300, 30, 5):
        ra, rb = a.step(plan), b.step(plan)
        for x, y in zip(ra.obs + ra.rewards, rb.obs + rb.rewards):
            assert torch.equal(x, y)


def test_dispersion_and_discovery_semantics(cuda):
    d = env("dispersion", B=2, cuda=cuda, ov={"n_agents": 2, "n_food": 2})
    s = d.world.state_array().cpu().numpy()
    assert (s[:2, 0:2] == 0).all()                              # everyone spawns at the origin
    food = d.world.entity("food_0")
    food.state.set_pos(S.Vec2.from_array([[0.05, 0.0], [5.0, 5.0]], device=cuda))
    r = d.step([np.zeros((2, 2), np.float32)] * 2)
    assert d.scenario.eaten[:, 0].tolist() == [True, False]
    assert float(r.rewards[0][0]) > 0.5                          # the bite pays once
    r2 = d.step([np.zeros((2, 2), np.float32)] * 2)
    assert float(r2.rewards[0][0]) < 0.5 and bool(d.scenario.eaten[0, 0])
    q = env("discovery", B=1, cuda=cuda, ov={"n_agents": 2, "n_points": 1})
    q.world.entity("point_0").state.set_pos(S.Vec2.from_array([[0.0, 0.0]], device=cuda))
    for a in q.agents:
        a.state.set_pos(S.Vec2.from_array([[0.0, 0.0]], device=cuda))
    before = q.world.entity("point_0").state.snapshot(0)["pos"]
    q.step([np.zeros((1, 2), np.float32)] * 2)
    assert bool(q.scenario.covered_now[0, 0])
    assert q.world.entity("point_0").state.snapshot(0)["pos"] != before      # relocated
