"""The fused rollout kernel (ss_env_rollout): S consecutive steps of
simple_spread / transport / reverse_transport / flocking in ONE launch, each env's
state kept on chip between them.  Every intermediate StepResult, the final
state and the step counters must equal eager Env.step bit for bit
(env.py:209-235 per step), across the horizon, masked resets between
replays and a NaN stop inside a replay."""
import numpy as np
import pytest
import torch

import paper_2207_03530_b200 as S

pytestmark = pytest.mark.gpu


def state(e):
    return e.world.state_array().cpu().numpy()


def outs(r):
    return r.obs + r.rewards + [r.dones]


CASES = [("simple_spread", {}), ("simple_spread", {"n_agents": 1}), ("simple_spread", {"n_agents": 8}),
         ("transport", {}), ("transport", {"n_agents": 7}), ("reverse_transport", {}),
         ("flocking", {}), ("flocking", {"n_agents": 3, "n_obstacles": 0}),
         ("flocking", {"n_agents": 8, "n_obstacles": 6, "lidar_rays": 32})]


@pytest.mark.parametrize("name,ov", CASES)
@pytest.mark.parametrize("S_", [2, 5, 16])
def test_rollout_equals_eager(cuda, name, ov, S_):
    B, horizon = 333, 7                   # the horizon falls inside a replay
    a = S.Env(S.create_scenario(name, **ov), B, seed=4, device=cuda, validate=False, max_steps=horizon)
    b = S.Env(S.create_scenario(name, **ov), B, seed=4, device=cuda, validate=False, max_steps=horizon)
    A = len(a.agents)
    g = torch.Generator(device=cuda)
    g.manual_seed(11)
    bufs = [torch.rand((A, B, 2), device=cuda, generator=g) * 2 - 1 for _ in range(3)]
    graph = b.step_graph(bufs, steps_per_replay=S_, fused_rollout=True)
    assert graph.fused_rollout and graph.launches_per_replay == 1
    mask = torch.zeros(B, dtype=torch.bool, device=cuda)
    mask[::5] = True
    for rep in range(3):
        i = rep % 3
        rs = graph.rollout(i)
        for s in range(S_):
            ra = a.step(bufs[(i + s) % 3])
            for x, y in zip(outs(ra), outs(rs[s])):
                assert torch.equal(x, y), f"replay {rep} step {s}"
        np.testing.assert_array_equal(state(a), state(b))
        assert torch.equal(a.world.step_count, b.world.step_count)
        a.reset_at(mask)
        b.reset_at(mask)


def test_rollout_nan_stops_mid_replay(cuda):
    """validate=True: a NaN in step k of the replay stops the rollout kernel
    before step k (state as after step k-1, like the eager step that raises)."""
    B, S_ = 257, 6
    ref = S.Env(S.create_scenario("simple_spread"), B, seed=6, device=cuda)
    e = S.Env(S.create_scenario("simple_spread"), B, seed=6, device=cuda, validate=False)
    A = len(e.agents)
    g = torch.Generator(device=cuda)
    g.manual_seed(2)
    bufs = [torch.rand((A, B, 2), device=cuda, generator=g) * 2 - 1 for _ in range(2 * S_)]
    graph = e.step_graph(bufs, steps_per_replay=S_, validate=True)
    assert graph.fused_rollout and graph.launches_per_replay == 2   # scan + rollout
    outs0 = graph.rollout(0)
    graph.check()
    for k in range(S_):
        r = ref.step(bufs[k].clone())
        for x, y in zip(outs(r), outs(outs0[k])):
            assert torch.equal(x, y)
    bufs[S_ + 3][2, 100, 1] = float("nan")
    for k in range(S_, S_ + 3):
        ref.step(bufs[k].clone())
    graph.rollout(S_)
    with pytest.raises(S.ContractViolation, match="NaN"):
        graph.check()
    np.testing.assert_array_equal(state(e), state(ref))
    assert torch.equal(e.world.step_count, ref.world.step_count)


def test_rollout_off_and_unsupported_fall_back_to_per_step(cuda):
    """fused_rollout=False, S=1, physics sub-steps, or a scenario without a
    rollout kernel: the per-step graph; None (default) takes it where the
    scenario prefers it (flocking only past L2-resident batch sizes)."""
    B = 64
    for name, ov, S_, fused, want in [("simple_spread", {}, 4, False, False), ("simple_spread", {}, 1, True, False),
                                      ("simple_spread", {"substeps": 2}, 4, True, False),
                                      ("dispersion", {}, 4, True, False), ("transport", {}, 4, True, True),
                                      ("transport", {}, 4, None, True), ("simple_spread", {}, 4, None, True),
                                      ("flocking", {}, 4, None, False), ("flocking", {}, 4, True, True),
                                      ("discovery", {}, 4, None, False)]:
        e = S.Env(S.create_scenario(name), B, seed=1, device=cuda, validate=False, **ov)
        A = len(e.agents)
        buf = torch.zeros((A, B, 2), device=cuda)
        graph = e.step_graph(buf, steps_per_replay=S_, fused_rollout=fused)
        assert graph.fused_rollout is want, name
        assert graph.launches_per_replay == (1 if want else S_)
        graph.step()


@pytest.mark.parametrize("name", ["transport", "reverse_transport"])
def test_rollout_one_wave_build_equals_eager(cuda, name):
    """100k envs: 782 CTAs, so the launcher takes the 80-register transport
    rollout build (one wave) instead of the 96-register one; same results."""
    B, S_ = 100_000, 4
    a = S.Env(S.create_scenario(name), B, seed=8, device=cuda, validate=False, max_steps=3)
    b = S.Env(S.create_scenario(name), B, seed=8, device=cuda, validate=False, max_steps=3)
    A = len(a.agents)
    g = torch.Generator(device=cuda)
    g.manual_seed(4)
    bufs = [torch.rand((A, B, 2), device=cuda, generator=g) * 2 - 1 for _ in range(2)]
    graph = b.step_graph(bufs, steps_per_replay=S_, fused_rollout=True)
    for rep in range(2):
        rs = graph.rollout(rep % 2)
        for s in range(S_):
            ra = a.step(bufs[(rep + s) % 2])
            for x, y in zip(outs(ra), outs(rs[s])):
                assert torch.equal(x, y), f"replay {rep} step {s}"
    np.testing.assert_array_equal(state(a), state(b))


@pytest.mark.parametrize("B", [1, 31, 33])
@pytest.mark.parametrize("name", ["simple_spread", "transport", "flocking"])
def test_rollout_ragged_batches(cuda, name, B):
    """Partial warps (B < 32, B = 33: the last warp's observation rows take
    the plain store path instead of the bulk copy) and S above the rollout
    limit (17 > 16: per-step graph) still equal eager stepping."""
    for S_, fused in ((3, True), (17, None)):
        a = S.Env(S.create_scenario(name), B, seed=9, device=cuda, validate=False)
        b = S.Env(S.create_scenario(name), B, seed=9, device=cuda, validate=False)
        A = len(a.agents)
        g = torch.Generator(device=cuda)
        g.manual_seed(13)
        bufs = [torch.rand((A, B, 2), device=cuda, generator=g) * 2 - 1 for _ in range(2)]
        graph = b.step_graph(bufs, steps_per_replay=S_, fused_rollout=fused)
        assert graph.fused_rollout is (S_ <= 16)
        rs = graph.rollout(0)
        for s in range(S_):
            ra = a.step(bufs[s % 2])
            for x, y in zip(outs(ra), outs(rs[s])):
                assert torch.equal(x, y), f"{name} B={B} S={S_} step {s}"
        np.testing.assert_array_equal(state(a), state(b))


def test_rollout_c_abi_contract(cuda):
    """ss_env_rollout refuses bad step counts, missing pointers, check_actions
    without guard words (ContractViolation) and worlds without a rollout
    kernel (SS_ERR_UNSUPPORTED), before launching anything."""
    import ctypes

    from paper_2207_03530_b200 import _native as N

    B = 64
    e = S.Env(S.create_scenario("simple_spread"), B, seed=0, device=cuda, validate=False)
    A = len(e.agents)
    sc, world = e.scenario, e.world
    h = sc.native_handle(world)
    act = torch.zeros((A, B, 2), device=cuda)
    obs, rew, done = sc.alloc_outputs(world, h.obs_dim)

    def call(n, null_obs=False, check=False, guard=None, handle=h.handle):
        io = N.SsRolloutIO()
        acts = (N.c_vp * (max(n, 1) * A))(*([act.data_ptr() + a * B * 8 for a in range(A)] * max(n, 1)))
        o = (N.c_vp * max(n, 1))(*([None if null_obs else obs.data_ptr()] * max(n, 1)))
        r = (N.c_vp * max(n, 1))(*([rew.data_ptr()] * max(n, 1)))
        d = (N.c_vp * max(n, 1))(*([done.data_ptr()] * max(n, 1)))
        io.n_steps, io.actions, io.obs, io.rew, io.done = n, acts, o, r, d
        io.obs_agent_stride = obs.shape[1] * obs.shape[2]
        io.guard = guard
        io.check_actions = int(check)
        return N.lib().ss_env_rollout(handle, world.buffers_ref(), ctypes.byref(io),
                                      torch.cuda.current_stream(cuda).cuda_stream)

    before = state(e)
    assert call(0) == -1 and call(N.MAX_ROLLOUT + 1) == -1
    assert call(2, null_obs=True) == -1
    assert call(2, check=True) == -1
    d = S.Env(S.create_scenario("dispersion"), B, seed=0, device=cuda, validate=False)
    hd = d.scenario.native_handle(d.world)
    io = N.SsRolloutIO()
    io.n_steps = 1
    arr = (N.c_vp * 1)(obs.data_ptr())
    io.obs, io.rew, io.done = arr, arr, arr
    io.actions = (N.c_vp * len(d.agents))(*([act.data_ptr()] * len(d.agents)))
    assert N.lib().ss_env_rollout(hd.handle, d.world.buffers_ref(), ctypes.byref(io),
                                  torch.cuda.current_stream(cuda).cuda_stream) == -5   # SS_ERR_UNSUPPORTED
    torch.cuda.synchronize()
    np.testing.assert_array_equal(state(e), before)
    assert call(2) == 0   # and a well-formed call runs
