"""Host-side logic that needs no GPU: world layout and views, descriptors,
constants rounded as numpy rounds them, the Philox state image, masks,
registry and error behaviour."""
import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2207_03530_b200 as S
from oracle import swarm_oracle as O
from paper_2207_03530_b200 import _native as N
from paper_2207_03530_b200._numerics import sqrt_le_bound, sqrt_lt_bound
from paper_2207_03530_b200.batching import SeededRng, state_to_words, words_to_state
from paper_2207_03530_b200.env import _as_mask
from paper_2207_03530_b200.errors import ContractViolation, NativeError, UnknownScenario

CPU = torch.device("cpu")


def make_world(B=4):
    w = S.World(B, device=CPU)
    w.add(S.Entity("wall", S.Box(0.4, 0.2)))
    w.add(S.Agent("a0", S.Sphere(0.05)))
    w.add(S.Entity("ball", S.Sphere(0.1), movable=True, rotatable=True))
    w.add(S.Agent("a1", S.Sphere(0.05)))
    return w


def test_agents_precede_landmarks_and_slots():
    w = make_world()
    assert [e.name for e in w.entities] == ["a0", "a1", "wall", "ball"]
    assert w.dyn.shape == (3, 4, 4) and w.stat.shape == (1, 4, 2) and w.rot.shape == (4, 4, 2)


def test_views_write_through_and_relayout_keeps_state():
    w = make_world()
    a0 = w.entity("a0")
    a0.state.pos.x[2] = 1.5
    a0.state.set_vel(S.Vec2.from_array([[0.25, -0.5]], device=CPU), env_index=1)
    w.entity("ball").state.rot[3] = 0.75
    w.add(S.Agent("a2"))            # relayout: a new agent goes before landmarks
    assert [e.name for e in w.entities][:3] == ["a0", "a1", "a2"]
    assert float(a0.state.pos.x[2]) == 1.5
    assert float(a0.state.vel.y[1]) == -0.5
    assert float(w.entity("ball").state.rot[3]) == 0.75
    w.entity("ball").movable = False    # flips buffers again
    assert float(w.entity("ball").state.rot[3]) == 0.75
    snap = w.get_env_state(2)
    assert snap["a0"]["pos"] == (1.5, 0.0)
    w.set_env_state(0, snap)
    assert float(a0.state.pos.x[0]) == 1.5


def test_duplicate_names_and_bad_params_rejected():
    w = make_world()
    with pytest.raises(ContractViolation):
        w.add(S.Agent("a0"))
    with pytest.raises(ContractViolation):
        S.PhysParams(dt=0)
    with pytest.raises(ContractViolation):
        S.Entity("x", mass=0)
    with pytest.raises(ContractViolation):
        S.World(0, device=CPU)


def test_entity_descriptors_round_like_numpy():
    w = make_world()
    w.params = S.PhysParams(gravity=(0.0, -9.81))
    d = w.entity_descs()
    ball = d[w.index_of(w.entity("ball"))]
    dt = np.float32(0.1)
    assert ball.inv_m_dt == np.float32(np.float32(1.0 / 1.0) * dt)
    assert ball.inv_i_dt == np.float32(np.float32(1.0 / (0.1 ** 2 / 2)) * dt)
    assert ball.grav_y == np.float32(-9.81 * np.float32(1.0))
    assert d[0].u_range == np.float32(1.0) and d[0].is_agent == 1
    pairs, n = w.pair_descs()
    assert n == len(w.collidable_pairs())
    for k in range(n):
        i, j = pairs[k].i, pairs[k].j
        dm = np.float32(S.shapes.min_contact_distance(w.entities[i].shape, w.entities[j].shape))
        assert pairs[k].d_min == dm and pairs[k].sign == (1.0 if (i + j) % 2 == 0 else -1.0)
        assert pairs[k].d2_act == sqrt_le_bound(dm)


@settings(max_examples=200, deadline=None)
@given(st.floats(min_value=1e-6, max_value=10.0, allow_nan=False))
def test_sqrt_bounds_are_exact(t):
    t = np.float32(t)
    b, bl = sqrt_le_bound(t), sqrt_lt_bound(t)
    assert np.sqrt(b) <= t and np.sqrt(np.nextafter(b, np.float32(np.inf))) > t
    assert np.sqrt(bl) < t and np.sqrt(np.nextafter(bl, np.float32(np.inf))) >= t


@settings(max_examples=50, deadline=None)
@given(st.integers(min_value=0, max_value=2**31), st.integers(min_value=0, max_value=37))
def test_philox_word_image_round_trip(seed, n):
    g = np.random.Philox(seed)
    g.random_raw(n)          # leave a partly consumed buffer
    st0 = g.state
    w = state_to_words(st0)
    back = words_to_state(w, st0)
    g2 = np.random.Philox()
    g2.state = back
    np.testing.assert_array_equal(g.random_raw(9), g2.random_raw(9))


def test_reset_ops_and_constants_match_oracle_tasks():
    for name, ov in [("simple_spread", {"n_agents": 3}), ("transport", {}), ("flocking", {"n_agents": 5}),
                     ("dispersion", {"n_agents": 6, "n_food": 5}), ("discovery", {"n_agents": 7})]:
        sc = S.create_scenario(name, **ov)
        w = sc.make_world(3, SeededRng(0))
        assert w.device == CPU
        task = O.TASKS[name](**ov)
        assert [(k, kind, tuple(lo), None if hi is None else tuple(hi)) for k, kind, lo, hi in sc.reset_ops(w)] == \
            [(k, kind, tuple(lo), None if hi is None else tuple(hi)) for k, kind, lo, hi in task.reset_ops(None)]
        assert list(w.collidable_pairs()) == list(sc.template_pairs(w)), name
        assert sc.template_ok(w)
        ws = O.WorldState(task.bodies(), 3)
        assert list(ws.pairs) == list(w.collidable_pairs())
        task.reset_aux(3, None)
        o = task.obs(_filled(ws))
        assert o[0].shape[1] == sc.obs_dim(w)


def _filled(ws):
    if hasattr(ws, "px"):
        for arrs in (ws.px, ws.py):
            for a in arrs:
                a[:] = 0.5
    return ws


def test_template_check_falls_back_when_world_changes():
    sc = S.create_scenario("simple_spread")
    w = sc.make_world(2, SeededRng(0))
    assert sc.physics_fused(w)
    w.entity("agent_1").collidable = False
    assert not sc.physics_fused(w)


def test_masks():
    m = _as_mask([1, 3], 5, CPU)
    assert m.tolist() == [False, True, False, True, False]
    assert _as_mask(2, 5, CPU).tolist() == [False, False, True, False, False]
    assert _as_mask(np.array([True] * 5), 5, CPU).all()
    with pytest.raises(ContractViolation):
        _as_mask([5], 5, CPU)
    with pytest.raises(ContractViolation):
        _as_mask(torch.zeros(4, dtype=torch.bool), 5, CPU)


def test_registry_and_errors():
    assert set(S.scenario_names()) >= {"simple_spread", "transport", "flocking", "dispersion", "discovery"}
    with pytest.raises(UnknownScenario):
        S.create_scenario("nope")
    with pytest.raises(ContractViolation):
        S.set_default_dtype(np.float64)
    S.set_default_dtype(np.float32)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_env_refuses_cpu():
    with pytest.raises(NativeError):
        S.Env(S.create_scenario("simple_spread"), 4, device="cpu")
