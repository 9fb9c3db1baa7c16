"""Physics and geometry on the device, against the oracle and hand values.

Mirrors the reference's tests/test_physics.py and test_geometry.py (same
scenes and tolerances, float32 since the B200 path is float32) plus direct
oracle comparisons of the generic world_step kernel for every shape pair.
"""
import numpy as np
import pytest
import torch

import paper_2207_03530_b200 as S
from oracle import swarm_oracle as O
from paper_2207_03530_b200.dynamics import collision_force, integrate, world_step
from paper_2207_03530_b200.geometry import closest_points

pytestmark = pytest.mark.gpu


def one(x, y, dev):
    return S.Vec2(torch.tensor([x], device=dev), torch.tensor([y], device=dev))


def world(entities, B=1, dev="cuda", **params):
    w = S.World(B, params=S.PhysParams(**params), device=dev)
    for e in entities:
        w.add(e)
    return w


# ---- integrator (dynamics.py:69-86) ----------------------------------------
def test_integrate_velocity_then_position(cuda):
    w = world([S.Entity("b", S.Sphere(0.1), movable=True)], dev=cuda)
    b = w.entity("b")
    b.state.set_vel(S.Vec2.from_array([[1.0, 0.0]], device=cuda))
    integrate(b, S.Vec2.zeros(1, device=cuda), torch.zeros(1, device=cuda), w.params)
    assert float(b.state.vel.x[0]) == np.float32(0.75)
    assert float(b.state.pos.x[0]) == np.float32(np.float32(0.75) * np.float32(0.1))


def test_gravity_and_rest(cuda):
    w = world([S.Entity("b", S.Sphere(0.1), mass=2.0, movable=True)], dev=cuda, gravity=(0.0, -1.0), damping=0.0)
    world_step(w, [])
    v = w.entity("b").state.vel
    assert float(v.x[0]) == 0.0
    assert abs(float(v.y[0]) + 0.1) <= 1e-7
    w2 = world([S.Entity("b", S.Sphere(0.1), movable=True)], dev=cuda)
    world_step(w2, [])
    assert w2.entity("b").state.snapshot(0) == {"pos": (0.0, 0.0), "vel": (0.0, 0.0), "rot": 0.0, "ang_vel": 0.0}


def test_damping_decay_over_fifty_steps(cuda):
    w = world([S.Entity("b", S.Sphere(0.1), movable=True)], dev=cuda)
    b = w.entity("b")
    b.state.set_vel(S.Vec2.from_array([[3.0, 4.0]], device=cuda))
    for t in range(1, 51):
        world_step(w, [])
        want = 5.0 * 0.75**t
        assert abs(float(b.state.vel.norm()[0]) - want) <= 1e-5 * want


def test_max_speed_clamp(cuda):
    w = world([S.Agent("a", S.Sphere(0.05), max_speed=0.3, u_range=100.0)], dev=cuda)
    for _ in range(5):
        world_step(w, [S.AgentAction(force=S.Vec2.full(1, 100.0, 40.0, device=cuda))])
        assert float(w.entity("a").state.vel.norm()[0]) <= 0.3 + 1e-6


def test_immovable_frozen_and_nonrotatable(cuda):
    wall = S.Entity("wall", S.Box(0.4, 0.4))
    ball = S.Entity("ball", S.Sphere(0.1), movable=True)
    w = world([wall, ball], dev=cuda)
    ball.state.set_pos(S.Vec2.from_array([[0.25, 0.0]], device=cuda))
    before = wall.state.snapshot(0)
    for _ in range(10):
        world_step(w, [])
    assert wall.state.snapshot(0) == before
    assert float(ball.state.pos.x[0]) > 0.25
    box = S.Entity("crate", S.Box(0.4, 0.2), movable=True)
    poker = S.Entity("poker", S.Sphere(0.08), movable=True)
    w = world([box, poker], dev=cuda)
    poker.state.set_pos(S.Vec2.from_array([[0.22, 0.09]], device=cuda))
    for _ in range(5):
        world_step(w, [])
    assert float(box.state.rot[0]) == 0.0 and float(box.state.ang_vel[0]) == 0.0
    assert float(box.state.pos.x[0]) != 0.0


def test_off_center_contact_signed_torque(cuda):
    rod = S.Entity("rod", S.Line(1.0), movable=False, rotatable=True)
    ball = S.Entity("ball", S.Sphere(0.05), movable=True)
    w = world([rod, ball], dev=cuda)
    ball.state.set_pos(S.Vec2.from_array([[0.4, 0.03]], device=cuda))
    world_step(w, [])
    assert float(rod.state.ang_vel[0]) < 0.0
    assert float(ball.state.vel.y[0]) > 0.0


# ---- contact force (dynamics.py:36-66) --------------------------------------
def test_contact_force_values(cuda):
    p = S.PhysParams()
    r = collision_force(one(0.0, 0.0, cuda), one(0.09, 0.0, cuda), 0.1, p)
    assert abs(float(r.force_i.norm()[0]) - 1.00000454) <= 1e-4 * 1.00000454
    assert float(r.force_i.x[0]) < 0.0 and float(r.force_i.y[0]) == 0.0
    far = collision_force(one(0.0, 0.0, cuda), one(0.2, 0.0, cuda), 0.1, p)
    assert float(far.force_i.x[0]) == 0.0 and float(far.force_i.y[0]) == 0.0 and not bool(far.active[0])
    deep = collision_force(one(0.0, 0.0, cuda), one(1e-6, 0.0, cuda), 0.5, p)
    assert abs(float(deep.force_i.norm()[0]) - 50.0) < 1.0
    a = collision_force(one(0.3, 0.3, cuda), one(0.3, 0.3, cuda), 0.2, p, fallback_sign=1.0)
    assert float(a.force_i.y[0]) == 0.0 and float(a.force_i.x[0]) > 0.0


def test_contact_force_bitexact_vs_oracle(cuda):
    rng = np.random.default_rng(7)
    n = 200_000
    pi = rng.uniform(-0.3, 0.3, (2, n)).astype(np.float32)
    pj = (pi + rng.uniform(-0.12, 0.12, (2, n))).astype(np.float32)
    for dmin in (0.1, 0.05 + 0.1, 0.06, 1e-4):
        want = O.contact((pi[0], pi[1]), (pj[0], pj[1]), dmin, O.Phys(), -1.0)
        got = collision_force(S.Vec2(torch.from_numpy(pi[0]).to(cuda), torch.from_numpy(pi[1]).to(cuda)),
                              S.Vec2(torch.from_numpy(pj[0]).to(cuda), torch.from_numpy(pj[1]).to(cuda)),
                              dmin, S.PhysParams(), fallback_sign=-1.0)
        np.testing.assert_array_equal(got.force_i.x.cpu().numpy(), want[0])
        np.testing.assert_array_equal(got.force_i.y.cpu().numpy(), want[1])
        np.testing.assert_array_equal(got.active.cpu().numpy(), want[2])
        assert want[2].sum() > (1000 if dmin > 0.01 else -1)


SHAPES = [S.Sphere(0.25), S.Sphere(0.2), S.Box(0.4, 0.25), S.Box(0.35, 0.3), S.Line(0.5), S.Line(0.6)]


def _body(shape, name):
    if isinstance(shape, S.Sphere):
        return O.Body(name, "sphere", (shape.radius,), movable=True, rotatable=True)
    if isinstance(shape, S.Box):
        return O.Body(name, "box", (shape.length, shape.width), movable=True, rotatable=True)
    return O.Body(name, "line", (shape.length,), movable=True, rotatable=True)


@pytest.mark.parametrize("si", range(6))
@pytest.mark.parametrize("sj", range(6))
def test_closest_points_vs_oracle(cuda, si, sj):
    """All sphere/box/line pairs in both orders, unrotated and rotated poses:
    bit-exact (float32 sin/cos are numpy's own algorithm, ss_math.cuh)."""
    rng = np.random.default_rng(100 + 6 * si + sj)
    n = 4000
    a, b = SHAPES[si], SHAPES[sj]
    ba, bb = _body(a, "a"), _body(b, "b")
    pa = rng.uniform(-0.4, 0.4, (2, n)).astype(np.float32)
    pb = rng.uniform(-0.4, 0.4, (2, n)).astype(np.float32)
    for rotated in (False, True):
        ra = rng.uniform(-np.pi, np.pi, n).astype(np.float32) if rotated else np.zeros(n, np.float32)
        rb = rng.uniform(-np.pi, np.pi, n).astype(np.float32) if rotated else np.zeros(n, np.float32)
        (wx, wy), (vx, vy) = O.closest_shapes(ba, (pa[0], pa[1]), ra, bb, (pb[0], pb[1]), rb)
        gi, gj = closest_points(S.Vec2(torch.from_numpy(pa[0]).to(cuda), torch.from_numpy(pa[1]).to(cuda)),
                                torch.from_numpy(ra).to(cuda), a,
                                S.Vec2(torch.from_numpy(pb[0]).to(cuda), torch.from_numpy(pb[1]).to(cuda)),
                                torch.from_numpy(rb).to(cuda), b)
        got = [gi.x.cpu().numpy(), gi.y.cpu().numpy(), gj.x.cpu().numpy(), gj.y.cpu().numpy()]
        want = [np.asarray(v, np.float32) for v in (wx, wy, vx, vy)]
        for g, w in zip(got, want):
            np.testing.assert_array_equal(g, w, err_msg=f"rotated={rotated}")


NEWTON = [(S.Sphere(0.25), S.Sphere(0.2)), (S.Sphere(0.2), S.Box(0.4, 0.25)), (S.Sphere(0.2), S.Line(0.5)),
          (S.Line(0.5), S.Line(0.6)), (S.Line(0.5), S.Box(0.4, 0.25)), (S.Box(0.35, 0.3), S.Box(0.4, 0.25))]


def test_newtons_third_law_exact_all_pairs(cuda):
    rng = np.random.default_rng(42)
    B, total = 170, 0
    for sa, sb in NEWTON:
        a = S.Entity("a", sa, movable=True, rotatable=True)
        b = S.Entity("b", sb, movable=True, rotatable=True)
        w = world([a, b], B=B, dev=cuda)
        for e in (a, b):
            e.state.set_pos(S.Vec2(rng.uniform(-0.3, 0.3, B), rng.uniform(-0.3, 0.3, B), device=cuda))
            e.state.set_rot(torch.from_numpy(rng.uniform(-np.pi, np.pi, B).astype(np.float32)).to(cuda))
        world_step(w, [])
        assert torch.equal(a.state.vel.x, -b.state.vel.x) and torch.equal(a.state.vel.y, -b.state.vel.y)
        total += int(((a.state.vel.x != 0) | (a.state.vel.y != 0)).sum())
    assert total > 150


@pytest.mark.parametrize("pair", range(6))
def test_generic_world_step_vs_oracle(cuda, pair):
    """Generic step kernel (rotating bodies, torques) vs the oracle: bit-exact
    for the first step and 20 further free-running steps."""
    sa, sb = NEWTON[pair]
    rng = np.random.default_rng(pair)
    B = 512
    a = S.Entity("a", sa, mass=1.3, movable=True, rotatable=True)
    b = S.Entity("b", sb, mass=0.7, movable=True, rotatable=True)
    w = world([a, b], B=B, dev=cuda)
    ws = O.WorldState([_body(sa, "a"), _body(sb, "b")], B)
    ws.bodies[0].mass, ws.bodies[1].mass = 1.3, 0.7
    for k, e in enumerate((a, b)):
        x = rng.uniform(-0.3, 0.3, B).astype(np.float32)
        y = rng.uniform(-0.3, 0.3, B).astype(np.float32)
        r = rng.uniform(-np.pi, np.pi, B).astype(np.float32)
        e.state.set_pos(S.Vec2(x, y, device=cuda))
        e.state.set_rot(torch.from_numpy(r).to(cuda))
        ws.px[k], ws.py[k], ws.rot[k] = x.copy(), y.copy(), r.copy()
    world_step(w, [])
    O.world_step(ws, {})
    got = w.state_array().cpu().numpy()
    want = np.stack([np.stack([ws.px[k], ws.py[k], ws.vx[k], ws.vy[k], ws.rot[k], ws.w[k]]) for k in range(2)])
    np.testing.assert_array_equal(got, want)
    for _ in range(20):
        world_step(w, [])
        O.world_step(ws, {})
    got = w.state_array().cpu().numpy()
    want = np.stack([np.stack([ws.px[k], ws.py[k], ws.vx[k], ws.vy[k], ws.rot[k], ws.w[k]]) for k in range(2)])
    np.testing.assert_array_equal(got, want)
    if not (isinstance(sa, S.Sphere) and isinstance(sb, S.Sphere)):
        assert np.abs(want[:, 5]).max() > 0      # bodies really spun


def test_world_step_contract(cuda):
    w = world([S.Agent("a", S.Sphere(0.05))], dev=cuda)
    with pytest.raises(S.ContractViolation):
        world_step(w, [])
    with pytest.raises(S.ContractViolation):
        world_step(w, [S.AgentAction(force=S.Vec2.full(1, float("nan"), 0.0, device=cuda))])
    w4 = world([S.Agent("a", S.Sphere(0.05))], B=4, dev=cuda)
    with pytest.raises(S.ContractViolation):
        world_step(w4, [S.AgentAction(force=S.Vec2.full(2, 0.0, 0.0, device=cuda))])
    with pytest.raises(S.ContractViolation):
        world_step(w, [S.AgentAction(force=S.Vec2.zeros(1, device=cuda), comm=torch.zeros((1, 3)))])
    wc = world([S.Agent("a", S.Sphere(0.05), silent=False, comm_dim=3)], dev=cuda)
    comm = torch.tensor([[0.1, 0.2, 0.3]])
    world_step(wc, [S.AgentAction(force=S.Vec2.zeros(1, device=cuda), comm=comm)])
    assert torch.equal(wc.comm["a"], comm)


def test_batched_step_matches_single_copies(cuda):
    def build(B):
        a = S.Entity("a", S.Sphere(0.2), movable=True)
        b = S.Entity("b", S.Sphere(0.2), mass=2.0, movable=True)
        return world([a, b], B=B, dev=cuda, gravity=(0.0, -0.5))

    starts = [(-0.15, 0.0), (0.05, 0.1), (0.3, -0.2)]
    batch = build(3)
    for e, (x, y) in enumerate(starts):
        batch.entity("b").state.pos.x[e] = x
        batch.entity("b").state.pos.y[e] = y
    singles = []
    for x, y in starts:
        s = build(1)
        s.entity("b").state.set_pos(S.Vec2.from_array([[x, y]], device=cuda))
        singles.append(s)
    for _ in range(25):
        world_step(batch, [])
        for s in singles:
            world_step(s, [])
    got = batch.state_array().cpu().numpy()
    for e, s in enumerate(singles):
        np.testing.assert_array_equal(got[:, :, e], s.state_array().cpu().numpy()[:, :, 0])
