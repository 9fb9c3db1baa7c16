"""Contract edge cases of the device Env: CUDA-graph stepping across resets
and world edits, the NaN guard on every physics path, shard refusal for host
reset programs, and reset-selector parsing (env.py:85, 189-198 semantics)."""
import numpy as np
import pytest
import torch

import golden_util as G
import paper_2207_03530_b200 as S

pytestmark = pytest.mark.gpu


def state(e):
    return e.world.state_array().cpu().numpy()


@pytest.mark.parametrize("name", ["simple_spread", "transport", "flocking", "dispersion", "discovery", "dropout"])
def test_step_graph_survives_resets(cuda, name):
    """replay, reset the done envs, replay: the usual RL loop, for every
    reset-kernel scenario, bitwise equal to eager stepping."""
    B = 96
    a = S.Env(S.create_scenario(name), B, seed=3, device=cuda, validate=False)
    b = S.Env(S.create_scenario(name), B, seed=3, device=cuda, validate=False)
    A = len(a.agents)
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    buf = torch.empty((A, B, 2), device=cuda)
    graph = b.step_graph(buf)
    mask = torch.zeros(B, dtype=torch.bool, device=cuda)
    mask[::7] = True
    for t in range(6):
        buf.copy_(torch.rand((A, B, 2), device=cuda, generator=g) * 2 - 1)
        ra = a.step(buf.clone())
        rb = graph.step()
        for x, y in zip(ra.obs + ra.rewards, rb.obs + rb.rewards):
            assert torch.equal(x, y), f"step {t}"
        assert torch.equal(ra.dones, rb.dones)
        a.reset_at(mask)
        b.reset_at(mask)
        if t == 3:
            a.reset()
            b.reset()
    np.testing.assert_array_equal(state(a), state(b))


def test_step_graph_refuses_after_world_edit(cuda):
    e = S.Env(S.create_scenario("simple_spread"), 64, seed=0, device=cuda, validate=False)
    buf = torch.zeros((3, 64, 2), device=cuda)
    graph = e.step_graph(buf)
    graph.step()
    e.scenario.done(e.world)          # a hook launch does not retire the graph
    graph.step()
    e.max_steps = 17                  # rebuilds the descriptor (new horizon)
    with pytest.raises(S.ContractViolation, match="edited"):
        graph.step()
    e.step_graph(buf).step()          # a fresh capture works


def test_done_hook_keeps_horizon_out(cuda):
    e = S.Env(S.create_scenario("transport"), 8, seed=0, device=cuda, max_steps=1)
    e.step([np.zeros((8, 2), np.float32)] * 4)
    assert bool(e.step([np.zeros((8, 2), np.float32)] * 4).dones.all())     # horizon reached
    assert not bool(e.scenario.done(e.world).any())                          # scenario term only


@pytest.mark.parametrize("name", ["wheel", "balance", "waterfall", "give_way", "passage"])
def test_nan_guard_on_generic_physics(cuda, name):
    """The catalog tasks whose physics is world_step's generic kernel: a NaN
    action must leave every buffer untouched, like the fused path."""
    e = S.Env(S.create_scenario(name), 6, seed=2, device=cuda)
    plan = G.pregen_actions(len(e.agents), 6, 2, 3)
    e.step(plan[0])
    before, steps = state(e), e.step_count.clone()
    bad = [a.copy() for a in plan[1]]
    bad[0][3, 1] = np.nan
    with pytest.raises(S.ContractViolation, match="NaN"):
        e.step(bad)
    np.testing.assert_array_equal(state(e), before)
    assert torch.equal(e.step_count, steps)


class _HostResetTask(S.Scenario):
    """A user scenario with a host reset program (numpy draws from the Env stream)."""

    def make_world(self, B, rng):
        w = S.World(B, rng=rng, device=getattr(rng, "device", None))
        w.add(S.Agent("a", S.Sphere(0.05)))
        return w

    def reset_world_at(self, world, env_index=None):
        n = 1 if env_index is not None else world.batch_size
        world.entity("a").state.set_pos_xy(world.rng.uniform(-1, 1, (n,)), world.rng.uniform(-1, 1, (n,)),
                                           env_index)

    def reward(self, agent, world):
        return torch.zeros(world.batch_size, device=world.device)

    def observation(self, agent, world):
        return torch.stack([agent.state.pos.x, agent.state.pos.y], 1)


def test_host_reset_refuses_sharding(cuda):
    with pytest.raises(S.ContractViolation, match="shard"):
        S.Env(_HostResetTask(), 8, device=cuda, env_offset=8, global_batch=16)


@pytest.mark.parametrize("name", ["wheel", "balance", "give_way", "passage", "waterfall", "football",
                                  "reverse_transport"])
def test_catalog_shards_equal_unsharded(cuda, name):
    """Device reset programs draw at global env indices: two shards of a
    catalog task (incl. a sharded masked reset) equal the unsharded run."""
    from paper_2207_03530_b200.parallel import shard_range

    Bg = 77
    full = S.Env(S.create_scenario(name), Bg, seed=4, device=cuda)
    shards = []
    for r in range(2):
        off, cnt = shard_range(r, 2, Bg)
        shards.append((off, cnt, S.Env(S.create_scenario(name), cnt, seed=4, device=cuda,
                                       env_offset=off, global_batch=Bg)))
    for off, cnt, e in shards:
        np.testing.assert_array_equal(state(e), state(full)[:, :, off:off + cnt])
    plans = G.pregen_actions(len(full.agents), Bg, 12, 5)
    mask = np.zeros(Bg, dtype=bool)
    mask[[0, 3, 38, 39, 40, 76]] = True
    for t, plan in enumerate(plans):
        raw = [None if a.action_script is not None else p for a, p in zip(full.agents, plan)]
        full.step(raw)
        for off, cnt, e in shards:
            e.step([None if p is None else p[off:off + cnt] for p in raw])
        if t == 5:
            full.reset_at(torch.from_numpy(mask).to(cuda))
            base = 0
            total = torch.tensor([int(mask.sum())], device=cuda)
            for off, cnt, e in shards:
                m = torch.from_numpy(mask[off:off + cnt]).to(cuda)
                e.scenario.reset_world_masked(e.world, m, torch.tensor([base], device=cuda), total)
                e.world.step_count[m] = 0
                base += int(mask[off:off + cnt].sum())
    for off, cnt, e in shards:
        np.testing.assert_array_equal(state(e), state(full)[:, :, off:off + cnt])


def test_reset_at_selectors(cuda):
    B = 6
    e = S.Env(S.create_scenario("simple_spread"), B, seed=1, device=cuda)
    ref = S.Env(S.create_scenario("simple_spread"), B, seed=1, device=cuda)
    for plan in G.pregen_actions(3, B, 3, 2):
        e.step(plan)
        ref.step(plan)
    sel = torch.tensor([0, 1, 0, 0, 1, 0], device=cuda)
    e.reset_at(sel.to(torch.uint8))                      # uint8 tensor is a mask
    ref.reset_at(torch.tensor([False, True, False, False, True, False], device=cuda))
    np.testing.assert_array_equal(state(e), state(ref))
    e.reset_at(np.array([0, 1, 0, 0, 1, 0], dtype=np.uint8))
    ref.reset_at([1, 4])                                  # explicit index list
    np.testing.assert_array_equal(state(e), state(ref))
    with pytest.raises(S.ContractViolation, match="ambiguous"):
        e.reset_at(np.array([0, 1, 0, 0, 1, 0]))


def test_validated_step_graph(cuda):
    """StepGraph(validate=True): the NaN scans run on a side branch of the
    graph; clean replays equal eager validated stepping, and a NaN in step k
    of a replay stops steps k.. (nothing moves from there), like the eager
    step that raises at k."""
    B, S_ = 200, 4
    ref = S.Env(S.create_scenario("transport"), B, seed=6, device=cuda)
    e = S.Env(S.create_scenario("transport"), B, seed=6, device=cuda, validate=False)
    plans = G.pregen_actions(4, B, 2 * S_, 9)
    bufs = [torch.from_numpy(np.stack(p)).to(cuda) for p in plans]
    graph = e.step_graph(bufs, steps_per_replay=S_, validate=True)
    outs = graph.rollout(0)
    graph.check()
    for k in range(S_):
        r = ref.step(plans[k])
        for x, y in zip(r.obs + r.rewards, outs[k].obs + outs[k].rewards):
            assert torch.equal(x, y)
    np.testing.assert_array_equal(state(e), state(ref))
    # NaN in the third step of the next replay
    bufs[S_ + 2][1, 17, 0] = float("nan")
    for k in range(S_, S_ + 2):
        ref.step(plans[k])
    graph.rollout(S_)
    with pytest.raises(S.ContractViolation, match="NaN"):
        graph.check()
    np.testing.assert_array_equal(state(e), state(ref))


def test_validated_step_graph_long_replay(cuda):
    """validate=True with more steps than one scan launch covers (20 > 16:
    two ss_check_action_sets calls): clean replays equal eager stepping, a
    NaN in step 18 stops steps 18.. and is reported by check()."""
    B, S_ = 96, 20
    ref = S.Env(S.create_scenario("flocking"), B, seed=2, device=cuda)
    e = S.Env(S.create_scenario("flocking"), B, seed=2, device=cuda, validate=False)
    A = len(e.agents)
    g = torch.Generator(device=cuda)
    g.manual_seed(21)
    bufs = [torch.rand((A, B, 2), device=cuda, generator=g) * 2 - 1 for _ in range(2 * S_)]
    graph = e.step_graph(bufs, steps_per_replay=S_, validate=True)
    assert not graph.fused_rollout and graph.launches_per_replay == S_ + 2
    outs = graph.rollout(0)
    graph.check()
    for k in range(S_):
        r = ref.step(bufs[k].clone())
        for x, y in zip(r.obs + r.rewards, outs[k].obs + outs[k].rewards):
            assert torch.equal(x, y)
    bufs[S_ + 18][0, 5, 1] = float("nan")
    for k in range(S_, S_ + 18):
        ref.step(bufs[k].clone())
    graph.rollout(S_)
    with pytest.raises(S.ContractViolation, match="NaN"):
        graph.check()
    np.testing.assert_array_equal(state(e), state(ref))
