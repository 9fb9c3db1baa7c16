"""Lidar / cast_ray on the device vs the oracle (reference lidar_scan restated)
and vs independent closed-form oracles (the reference's tests/helpers.py
formulations, restated), mirroring tests/test_sensors.py."""
import numpy as np
import pytest
import torch

import paper_2207_03530_b200 as S
from oracle import swarm_oracle as O

pytestmark = pytest.mark.gpu


def ray_circle_closed_form(origin, angle, center, radius):
    d = np.array([np.cos(angle), np.sin(angle)])
    oc = np.asarray(origin, float) - np.asarray(center, float)
    roots = np.roots([1.0, 2.0 * oc @ d, oc @ oc - radius * radius])
    real = roots[np.abs(roots.imag) < 1e-12].real
    hits = real[real > 1e-12]
    return float(hits.min()) if hits.size else np.inf


def test_scan_vs_oracle_mixed_shapes(cuda):
    B = 3000
    rng = np.random.default_rng(9)
    ents = [S.Agent("emit", S.Sphere(0.05)), S.Entity("rock", S.Sphere(0.2)),
            S.Entity("wall", S.Box(0.6, 0.2)), S.Entity("rod", S.Line(0.7)),
            S.Entity("ghost", S.Sphere(0.3), collidable=False)]
    bodies = [O.Body("emit", "sphere", (0.05,), movable=True, agent=True), O.Body("rock", "sphere", (0.2,)),
              O.Body("wall", "box", (0.6, 0.2)), O.Body("rod", "line", (0.7,)),
              O.Body("ghost", "sphere", (0.3,), collidable=False)]
    w = S.World(B, device=cuda)
    for e in ents:
        w.add(e)
    ws = O.WorldState(bodies, B)
    for k, e in enumerate(w.entities):
        x = rng.uniform(-1, 1, B).astype(np.float32)
        y = rng.uniform(-1, 1, B).astype(np.float32)
        r = (rng.uniform(-np.pi, np.pi, B) if k in (2, 3) else np.zeros(B)).astype(np.float32)
        e.state.set_pos(S.Vec2(x, y, device=cuda))
        e.state.set_rot(torch.from_numpy(r).to(cuda))
        ws.px[k], ws.py[k], ws.rot[k] = x, y, r
    lid = S.Lidar(n_rays=24, max_range=1.5)
    got = S.lidar_scan(w.entity("emit"), lid, w).cpu().numpy()
    want = O.lidar(ws, 0, 24, 1.5)
    # float64 cos/sin of rotated bodies may differ in the last ulp between
    # numpy and CUDA; results are cast to float32 afterwards
    np.testing.assert_allclose(got, want, atol=2e-6)
    assert (got == want).mean() > 0.99


def test_ray_circle_closed_form(cuda):
    rng = np.random.default_rng(11)
    n = 300
    w = S.World(n, device=cuda)
    obj = w.add(S.Entity("obj", S.Sphere(0.3)))
    centers = rng.uniform(-1.5, 1.5, (n, 2)).astype(np.float32)
    obj.state.set_pos(S.Vec2.from_array(centers, device=cuda))
    origins = rng.uniform(-1, 1, (n, 2)).astype(np.float32)
    ang = rng.uniform(-np.pi, np.pi, n)
    got = S.cast_ray(S.Vec2.from_array(origins, device=cuda), torch.from_numpy(ang), w, 6.0).cpu().numpy()
    want = np.array([min(ray_circle_closed_form(origins[i], ang[i], centers[i], 0.3), 6.0) for i in range(n)])
    ok = np.isfinite(want)
    np.testing.assert_allclose(got, want, atol=1e-5)


def test_lidar_semantics(cuda):
    w = S.World(1, device=cuda)
    a = w.add(S.Agent("a", S.Sphere(0.05)))
    lid = S.Lidar(n_rays=4, max_range=2.0)
    assert torch.equal(S.lidar_scan(a, lid, w), torch.full((1, 4), 2.0, device=cuda))   # empty world
    r = w.add(S.Entity("r", S.Sphere(0.1)))
    r.state.set_pos(S.Vec2.from_array([[1.0, 0.0]], device=cuda))
    scan = S.lidar_scan(a, lid, w).cpu().numpy()[0]
    assert abs(scan[0] - 0.9) < 1e-6 and scan[2] == np.float32(2.0)          # dead ahead / behind
    w.entity("r").collidable = False
    assert S.lidar_scan(a, lid, w).cpu().numpy()[0][0] == np.float32(2.0)      # transparent
    w.entity("r").collidable = True
    a.state.set_rot(torch.tensor([np.pi], dtype=torch.float32, device=cuda))
    scan = S.lidar_scan(a, lid, w).cpu().numpy()[0]
    assert abs(scan[2] - 0.9) < 1e-5                                            # rotates with agent
    box = w.add(S.Entity("box", S.Box(1.0, 1.0)))
    box.state.set_pos(S.Vec2.from_array([[5.0, 5.0]], device=cuda))
    inside = S.World(1, device=cuda)
    e2 = inside.add(S.Agent("e", S.Sphere(0.01)))
    inside.add(S.Entity("b", S.Box(1.0, 0.5)))
    d = S.cast_ray(e2.state.pos, torch.tensor([0.0], dtype=torch.float64), inside, 5.0, exclude="e")
    assert abs(float(d[0]) - 0.5) < 1e-6                                        # inside a box: exit wall


def test_fused_lidar_screen_adversarial(cuda):
    """The fused flocking Lidar screens rays by angle (k_flocking_w) before the
    exact float64 test.  Place circles on the screen's edges — tangent to a
    ray at ±0..2e-4 of the radius, a hit at max_range ± eps, an emitter on or
    just inside a rim — and require the observation (lidar columns included)
    to equal the oracle's reference scan bit-for-bit."""
    ov = {"n_agents": 5, "n_obstacles": 3, "lidar_rays": 12}
    B = 8192
    e = S.Env(S.create_scenario("flocking", **ov), B, seed=11, device=cuda)
    o = O.OracleEnv("flocking", B, seed=11, **ov)
    rng = np.random.default_rng(5)
    st = e.world.state_array().cpu().numpy()
    E = st.shape[0]
    st[:, 0:2, :] = rng.uniform(-1.2, 1.2, (E, 2, B)).astype(np.float32)
    st[:, 2:, :] = 0.0
    r_rock, r_agent = 0.1, float(e.agents[0].shape.radius)
    eps_set = [0.0, 1e-7, -1e-7, 1e-6, -1e-6, 1e-5, -1e-5, 5e-5, -5e-5, 1e-4, -1e-4, 2e-4, -2e-4]
    for b in range(B):
        em = int(rng.integers(5))
        origin = st[em, 0:2, b].astype(np.float64)
        m = int(rng.integers(12))
        ang = 2 * np.pi * m / 12
        d = np.array([np.cos(ang), np.sin(ang)])
        nrm = np.array([-d[1], d[0]])
        eps = eps_set[b % len(eps_set)]
        kind = b % 4
        if kind == 0:      # rock tangent to ray m of emitter em
            c = origin + rng.uniform(0.05, 1.1) * d + rng.choice([-1, 1]) * (r_rock + eps) * nrm
            st[5 + 1 + int(rng.integers(3)), 0:2, b] = c
        elif kind == 1:    # agent tangent
            other = (em + 1 + int(rng.integers(4))) % 5
            c = origin + rng.uniform(0.05, 1.1) * d + rng.choice([-1, 1]) * (r_agent + eps) * nrm
            st[other, 0:2, b] = c
        elif kind == 2:    # hit at max_range +- eps along the ray
            st[5 + 1 + int(rng.integers(3)), 0:2, b] = origin + (1.0 + r_rock + eps) * d
        else:              # emitter on / just inside / just outside a rock's rim
            st[5 + 1 + int(rng.integers(3)), 0:2, b] = origin + (r_rock + eps) * d
    st = st.astype(np.float32)
    e.world.load_state_array(torch.from_numpy(st).to(cuda))
    got = [x.cpu().numpy() for x in e.observations()]
    ws = o.ws
    for k in range(E):
        ws.px[k][:], ws.py[k][:] = st[k, 0], st[k, 1]
        ws.vx[k][:], ws.vy[k][:] = st[k, 2], st[k, 3]
        ws.rot[k][:], ws.w[k][:] = st[k, 4], st[k, 5]
    want = o.task.obs(ws)
    for a in range(5):
        np.testing.assert_array_equal(got[a], want[a], err_msg=f"agent {a}")
    # the edge cases really exercise the screen: some tangent rays hit, some miss
    lid = np.concatenate([g[:, -12:] for g in got])
    assert (lid < 1.0).any() and (lid == 1.0).any()
