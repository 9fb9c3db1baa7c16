"""Physics extensions the north star names and the reference lacks:
sub-stepped integration (PhysParams.substeps) and distance joints (Joint).

Both default to the reference's behaviour (substeps=1, no joints: every
other parity test covers that).  With substeps = k, one Env.step must equal
k reference world_step calls of dt / k on the held decoded actions
(tests/test_oracle_pin.py pins the oracle to exactly that composition of the
reference's own functions); joints are pinned to the numpy restatement
oracle/swarm_oracle.py joint_forces (parity unpinned by the reference, which
lists joints as a non-goal).  Every assertion is bitwise.
"""
import numpy as np
import pytest
import torch

import golden_util as G
import paper_2207_03530_b200 as S
from oracle import swarm_oracle as O
from paper_2207_03530_b200.dynamics import world_step

pytestmark = pytest.mark.gpu


def state(e):
    return e.world.state_array().cpu().numpy()


def ostate(ws):
    return np.stack([np.stack([ws.px[k], ws.py[k], ws.vx[k], ws.vy[k], ws.rot[k], ws.w[k]])
                     for k in range(len(ws.bodies))])


SUB_CASES = [
    ("simple_spread", {"n_agents": 3}, 4),
    ("transport", {"n_agents": 4}, 3),
    ("flocking", {"n_agents": 5, "n_obstacles": 3, "lidar_rays": 12}, 2),
    ("dispersion", {"n_agents": 40, "n_food": 33}, 3),
    ("discovery", {"n_agents": 64}, 2),
]


@pytest.mark.parametrize("name,ov,k", SUB_CASES)
def test_fused_substeps_equal_oracle(cuda, name, ov, k):
    """The fused kernels loop contact + integrate k times with dt / k."""
    B, steps = 160, 25
    e = S.Env(S.create_scenario(name, **ov), B, seed=9, device=cuda, substeps=k)
    o = O.OracleEnv(name, B, seed=9, substeps=k, **ov)
    assert e.world.params.substeps == k and e.scenario.physics_fused(e.world)
    np.testing.assert_array_equal(state(e), ostate(o.ws))
    for t, plan in enumerate(G.pregen_actions(len(e.agents), B, steps, 21)):
        res = e.step(plan)
        obs, rew, done = o.step(plan)
        np.testing.assert_array_equal(state(e), ostate(o.ws), err_msg=f"state @ {t}")
        for a, b in zip(res.obs, obs):
            np.testing.assert_array_equal(a.cpu().numpy(), b)
        for a, b in zip(res.rewards, rew):
            np.testing.assert_array_equal(a.cpu().numpy(), b)
        np.testing.assert_array_equal(res.dones.cpu().numpy(), done)
    # and it is not the single-tick physics
    one = S.Env(S.create_scenario(name, **ov), B, seed=9, device=cuda)
    for plan in G.pregen_actions(len(e.agents), B, steps, 21):
        one.step(plan)
    assert not np.array_equal(state(one), state(e))


def test_substeps_one_is_the_reference(cuda):
    """substeps=1 given explicitly is bitwise the default path."""
    a = S.Env(S.create_scenario("transport"), 256, seed=2, device=cuda, substeps=1)
    b = S.Env(S.create_scenario("transport"), 256, seed=2, device=cuda)
    for plan in G.pregen_actions(4, 256, 10, 3):
        ra, rb = a.step(plan), b.step(plan)
        for x, y in zip(ra.obs + ra.rewards, rb.obs + rb.rewards):
            assert torch.equal(x, y)
    np.testing.assert_array_equal(state(a), state(b))


def test_substeps_generic_path_equals_fused(cuda):
    """A world edited off its kernel's template runs world_step's generic
    kernel for physics: with sub-steps it still equals the fused kernel."""
    k, B = 3, 200
    fused = S.Env(S.create_scenario("simple_spread"), B, seed=4, device=cuda, substeps=k)
    gen = S.Env(S.create_scenario("simple_spread"), B, seed=4, device=cuda, substeps=k)
    gen.scenario.template_ok = lambda world: False
    gen.world._touch()
    assert fused.scenario.physics_fused(fused.world) and not gen.scenario.physics_fused(gen.world)
    for plan in G.pregen_actions(3, B, 15, 8):
        ra, rb = fused.step(plan), gen.step(plan)
        for x, y in zip(ra.obs + ra.rewards, rb.obs + rb.rewards):
            assert torch.equal(x, y)
    np.testing.assert_array_equal(state(fused), state(gen))


def _body(shape, name, **kw):
    if isinstance(shape, S.Sphere):
        return O.Body(name, "sphere", (shape.radius,), **kw)
    if isinstance(shape, S.Box):
        return O.Body(name, "box", (shape.length, shape.width), **kw)
    return O.Body(name, "line", (shape.length,), **kw)


SHAPES = [S.Sphere(0.1), S.Box(0.3, 0.2), S.Line(0.5)]


@pytest.mark.parametrize("k", [1, 4])
def test_generic_world_substeps_and_rotation_vs_oracle(cuda, k):
    """Mixed shapes, torques, gravity, sub-steps: generic kernel == oracle."""
    rng = np.random.default_rng(k)
    B = 384
    w = S.World(B, params=S.PhysParams(gravity=(0.0, -0.3), substeps=k), device=cuda)
    bodies = []
    for n, sh in enumerate(SHAPES):
        w.add(S.Entity(f"e{n}", sh, mass=1.0 + 0.3 * n, movable=True, rotatable=True))
        bodies.append(_body(sh, f"e{n}", mass=1.0 + 0.3 * n, movable=True, rotatable=True))
    ws = O.WorldState(bodies, B, O.Phys(gravity=(0.0, -0.3), substeps=k))
    for n, ent in enumerate(w.entities):
        x = rng.uniform(-0.25, 0.25, B).astype(np.float32)
        y = rng.uniform(-0.25, 0.25, B).astype(np.float32)
        r = rng.uniform(-np.pi, np.pi, B).astype(np.float32)
        ent.state.set_pos(S.Vec2(x, y, device=cuda))
        ent.state.set_rot(torch.from_numpy(r).to(cuda))
        ws.px[n], ws.py[n], ws.rot[n] = x.copy(), y.copy(), r.copy()
    for _ in range(12):
        world_step(w, [])
        O.world_step(ws, {})
        np.testing.assert_array_equal(w.state_array().cpu().numpy(), ostate(ws))
    assert np.abs(ostate(ws)[:, 5]).max() > 0


def _joint_world(cuda, B, substeps=1):
    """Agent -- (dist 0.3) -- box (anchored at its +x tip) -- (dist 0) -- line
    end; all movable and rotatable, plus a static sphere the agent bumps."""
    w = S.World(B, params=S.PhysParams(substeps=substeps), device=cuda)
    ag = w.add(S.Agent("a", S.Sphere(0.06), u_range=2.0))
    bx = w.add(S.Entity("box", S.Box(0.3, 0.12), mass=2.0, movable=True, rotatable=True))
    ln = w.add(S.Entity("rod", S.Line(0.4), mass=0.5, movable=True, rotatable=True))
    w.add(S.Entity("rock", S.Sphere(0.1)))
    w.add_joint(S.Joint(ag, bx, anchor_b=(1.0, 0.0), dist=0.3))
    w.add_joint(S.Joint(bx, ln, anchor_a=(-1.0, 0.5), anchor_b=(1.0, 0.0), dist=0.0, stiffness=80.0,
                        rotate_b=False))
    bodies = [O.Body("a", "sphere", (0.06,), movable=True, agent=True, u_range=2.0),
              O.Body("box", "box", (0.3, 0.12), mass=2.0, movable=True, rotatable=True),
              O.Body("rod", "line", (0.4,), mass=0.5, movable=True, rotatable=True),
              O.Body("rock", "sphere", (0.1,))]
    joints = [O.JointSpec(0, 1, (0.0, 0.0), (np.float32(0.15), np.float32(0.0)), 0.3, 130.0),
              O.JointSpec(1, 2, (np.float32(-1.0 * 0.15), np.float32(0.5 * 0.06)), (np.float32(0.2), np.float32(0.0)), 0.0,
                          80.0, True, False)]
    ws = O.WorldState(bodies, B, O.Phys(substeps=substeps))
    return w, ws, joints


@pytest.mark.parametrize("k", [1, 3])
def test_joints_vs_oracle(cuda, k):
    B, rng = 256, np.random.default_rng(11 + k)
    w, ws, joints = _joint_world(cuda, B, k)
    for n, ent in enumerate(w.entities):
        x = rng.uniform(-0.6, 0.6, B).astype(np.float32)
        y = rng.uniform(-0.6, 0.6, B).astype(np.float32)
        r = rng.uniform(-np.pi, np.pi, B).astype(np.float32)
        ent.state.set_pos(S.Vec2(x, y, device=cuda))
        ent.state.set_rot(torch.from_numpy(r).to(cuda))
        ws.px[n], ws.py[n], ws.rot[n] = x.copy(), y.copy(), r.copy()
    for t in range(30):
        f = rng.uniform(-2, 2, (B, 2)).astype(np.float32)
        world_step(w, [S.AgentAction(force=S.Vec2(f[:, 0], f[:, 1], device=cuda))])
        O.world_step(ws, {0: (f[:, 0], f[:, 1])}, joints=joints)
        np.testing.assert_array_equal(w.state_array().cpu().numpy(), ostate(ws), err_msg=f"step {t}")
    assert np.abs(ostate(ws)[1, 5]).max() > 0      # the joint torque spun the box


def test_joint_holds_distance(cuda):
    """A free pair joined at dist 0.4 settles near 0.4 from either side.  The
    joint is stiff (130 / unit stretch): like VMAS, it needs sub-steps — at
    one tick of dt = 0.1 far-stretched pairs overshoot and never settle (the
    oracle agrees bitwise either way, test_joints_vs_oracle)."""
    B = 64
    w = S.World(B, params=S.PhysParams(substeps=5), device=cuda)
    a = w.add(S.Entity("a", S.Sphere(0.05), movable=True))
    b = w.add(S.Entity("b", S.Sphere(0.05), movable=True))
    w.add_joint(S.Joint(a, b, dist=0.4))
    x = np.linspace(0.1, 1.2, B).astype(np.float32)
    b.state.set_pos(S.Vec2(x, np.zeros(B, np.float32), device=cuda))
    for _ in range(200):
        world_step(w, [])
    d = (a.state.pos - b.state.pos).norm().cpu().numpy()
    assert np.abs(d - 0.4).max() < 1e-3
    assert torch.equal(a.state.vel.x, -b.state.vel.x)


def test_joint_on_fused_scenario_falls_back_to_generic_physics(cuda):
    """A joint added to a built-in world moves its physics to the generic
    kernel (2 launches); the rest of the step stays the fused kernel's."""
    B = 128
    e = S.Env(S.create_scenario("simple_spread"), B, seed=1, device=cuda)
    ag = e.agents
    e.world.add_joint(S.Joint(ag[0], ag[1], dist=0.2))
    assert not e.scenario.physics_fused(e.world)
    ws = O.OracleEnv("simple_spread", B, seed=1)
    joints = [O.JointSpec(0, 1, dist=0.2)]
    for plan in G.pregen_actions(3, B, 10, 4):
        res = e.step(plan)
        forces = {a: O.decode(plan[a], ws.ws.bodies[a]) for a in range(3)}
        O.world_step(ws.ws, forces, joints=joints)
        ws.step_count += 1
        np.testing.assert_array_equal(state(e), ostate(ws.ws))
        for x, y in zip(res.obs, ws.observations()):
            np.testing.assert_array_equal(x.cpu().numpy(), y)


def test_joint_and_substep_contracts(cuda):
    w = S.World(2, device=cuda)
    a = w.add(S.Entity("a", movable=True))
    with pytest.raises(S.ContractViolation):
        S.Joint(a, a)
    with pytest.raises(S.ContractViolation):
        w.add_joint(S.Joint(a, S.Entity("stranger")))
    with pytest.raises(S.ContractViolation):
        S.PhysParams(substeps=0)
    with pytest.raises(S.ContractViolation):
        S.PhysParams(substeps=2.5)
