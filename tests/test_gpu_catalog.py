"""The reference's catalog-level acceptance checks on the device
(tests/test_acceptance.py:269-346, tests/test_scenarios.py:35-262):
every task registered, random rollouts finite at width 32 with per-index
reset isolation, the heuristic controller's action contract, scripted
controller vs random on a few tasks, and batch == independent singles."""
import numpy as np
import pytest
import torch

import paper_2207_03530_b200 as S

pytestmark = pytest.mark.gpu

ALL = ["transport", "wheel", "balance", "give_way", "football", "passage", "reverse_transport",
       "dispersion", "dropout", "flocking", "discovery", "waterfall", "simple_spread"]


def test_registry_lists_every_task():
    assert S.scenario_names() == ALL
    with pytest.raises(S.UnknownScenario):
        S.create_scenario("no_such_task")


@pytest.mark.parametrize("name", ALL)
def test_width_32_rollout_finite_and_reset_isolated(cuda, name):
    env = S.Env(S.create_scenario(name), 32, seed=13, device=cuda)
    env.reset()
    env.reset(env_index=5)
    g = np.random.default_rng(13)
    for _ in range(100):
        res = env.step([g.uniform(-1, 1, (32, 2)).astype(np.float32) for _ in env.agents])
        assert all(bool(torch.isfinite(o).all()) for o in res.obs)
        assert all(bool(torch.isfinite(r).all()) for r in res.rewards)
    st = env.world.state_array()
    assert bool(torch.isfinite(st).all())
    before = st.clone()
    env.reset(env_index=11)
    keep = [i for i in range(32) if i != 11]
    assert torch.equal(env.world.state_array()[:, :, keep], before[:, :, keep])


@pytest.mark.parametrize("name", ALL)
def test_heuristic_matches_action_contract(cuda, name):
    env = S.Env(S.create_scenario(name), 6, seed=2, device=cuda)
    obs = env.reset()
    acts = S.HeuristicPolicy()(env, obs)
    for a, agent in zip(acts, env.agents):
        if agent.action_script is not None:
            assert a is None
            continue
        a = np.asarray(a.cpu() if hasattr(a, "cpu") else a)
        assert a.shape == (6, 2) and np.isfinite(a).all() and (np.abs(a) <= agent.u_range + 1e-6).all()
    env.step(acts)


@pytest.mark.parametrize("name", ["simple_spread", "transport", "dispersion", "discovery", "dropout", "wheel"])
def test_scripted_controller_beats_random(cuda, name):
    """10 seeds at B=1 in the reference; here 64 envs of one seed in a batch."""
    heur = S.run_episode(S.Env(S.create_scenario(name), 64, seed=1, device=cuda), S.HeuristicPolicy())
    rand = S.run_episode(S.Env(S.create_scenario(name), 64, seed=1, device=cuda), S.RandomPolicy(seed=1001))
    assert float(heur.mean()) > float(rand.mean())


@pytest.mark.parametrize("name", ["simple_spread", "transport", "flocking", "balance", "football"])
def test_batched_run_equals_independent_singles(cuda, name):
    """B=16 batch vs 16 B=1 envs loaded with the same per-env state, 40 steps:
    identical (the reference's acceptance criterion, tolerance 1e-6 — here 0)."""
    B = 16
    master = S.Env(S.create_scenario(name), B, seed=31, device=cuda)
    singles = []
    for i in range(B):
        s = S.Env(S.create_scenario(name), 1, seed=500 + i, device=cuda)
        s.world.set_env_state(0, master.world.get_env_state(i))
        s.step_count[0] = 0
        singles.append(s)
    rng = S.SeededRng(77)
    for _ in range(40):
        plan = [rng.uniform(-a.u_range, a.u_range, (B, 2)) for a in master.agents]
        rm = master.step(plan)
        for i, s in enumerate(singles):
            rs = s.step([p[i:i + 1] for p in plan])
            for x, y in zip(rm.rewards, rs.rewards):
                assert float(x[i]) == float(y[0])
    st = master.world.state_array().cpu().numpy()
    for i, s in enumerate(singles):
        np.testing.assert_array_equal(st[:, :, i], s.world.state_array().cpu().numpy()[:, :, 0])


CATALOG_GENERIC = ["wheel", "balance", "give_way", "football", "passage", "reverse_transport", "dropout",
                   "waterfall"]


@pytest.mark.parametrize("name", CATALOG_GENERIC)
def test_generic_step_graph_equals_eager(cuda, name):
    """The 8 non-fused tasks captured whole (ss_world_step + torch hooks,
    scripted agents included) in 2-step graphs: every intermediate result and
    the final state equal eager stepping bit-for-bit."""
    B = 64
    a = S.Env(S.create_scenario(name), B, seed=3, device=cuda, validate=False)
    b = S.Env(S.create_scenario(name), B, seed=3, device=cuda, validate=False)
    A = len(a.agents)
    g = torch.Generator(device=cuda)
    g.manual_seed(9)
    bufs = [torch.rand((A, B, 2), device=cuda, generator=g) * 2 - 1 for _ in range(2)]
    graph = b.step_graph(bufs, steps_per_replay=2)
    for rep in range(3):
        rs = graph.rollout(rep % 2)
        for s in range(2):
            buf = bufs[(rep % 2 + s) % 2]
            ra = a.step([None if ag.action_script is not None else buf[n] for n, ag in enumerate(a.agents)])
            rb = rs[s]
            for x, y in zip(ra.obs + ra.rewards + [ra.dones], rb.obs + rb.rewards + [rb.dones]):
                assert torch.equal(x, y)
    assert torch.equal(a.world.state_array(), b.world.state_array())
    assert torch.equal(a.step_count, b.step_count)


@pytest.mark.parametrize("name", ["simple_spread", "transport", "flocking", "dispersion", "discovery",
                                  "reverse_transport", "dropout", "wheel", "give_way", "passage",
                                  "balance", "waterfall", "football"])
def test_fused_hooks_equal_step_outputs(cuda, name):
    """The reference's Scenario hooks on a fused world (single-phase kernel
    launches: reward, done, observation) reproduce what Env.step returned —
    dropout's reward reads the last step's energy from the flag words,
    dispersion's the fresh bites from aux."""
    env = S.Env(S.create_scenario(name), 96, seed=4, device=cuda)
    rng = S.SeededRng(8)
    for _ in range(3):
        res = env.step([rng.uniform(-a.u_range, a.u_range, (96, 2)) for a in env.agents])
    sc, w = env.scenario, env.world
    for i, agent in enumerate(env.agents):
        assert torch.equal(sc.reward(agent, w), res.rewards[i])
        assert torch.equal(sc.observation(agent, w), res.obs[i])
    horizon = env.step_count >= env.max_steps
    assert torch.equal(sc.done(w) | horizon, res.dones)


@pytest.mark.parametrize("name", CATALOG_GENERIC)
def test_fused_catalog_equals_torch_restatement(cuda, name):
    """Two independent restatements of each catalog task — the fused kernels
    (registered) and the torch hooks over world_step (scenarios/catalog.py) —
    step 512 envs for 40 steps with resets in between: every output and the
    final state agree bit-for-bit (the golden fixtures pin both to the
    reference at B=16)."""
    from paper_2207_03530_b200.scenarios import catalog

    cls = {"wheel": catalog.Wheel, "balance": catalog.Balance, "give_way": catalog.GiveWay,
           "football": catalog.Football, "passage": catalog.Passage,
           "reverse_transport": catalog.ReverseTransport, "dropout": catalog.Dropout,
           "waterfall": catalog.Waterfall}[name]
    B = 512
    fused = S.Env(S.create_scenario(name), B, seed=21, device=cuda)
    torch_path = S.Env(cls(), B, seed=21, device=cuda)
    assert fused.fused and not torch_path.fused
    rng = S.SeededRng(5)
    for t in range(40):
        plan = [None if a.action_script is not None else rng.uniform(-a.u_range, a.u_range, (B, 2))
                for a in fused.agents]
        ra, rb = fused.step(plan), torch_path.step(plan)
        for x, y in zip(ra.obs + ra.rewards + [ra.dones], rb.obs + rb.rewards + [rb.dones]):
            assert torch.equal(x, y.to(x.dtype)), f"step {t}"
        if t % 13 == 6:
            mask = ra.dones | (torch.arange(B, device=cuda) % 7 == t % 7)
            for x, y in zip(fused.reset_at(mask), torch_path.reset_at(mask)):
                assert torch.equal(x, y)
    assert torch.equal(fused.world.state_array(), torch_path.world.state_array())
    assert torch.equal(fused.step_count, torch_path.step_count)
