"""The built-in tasks' scripted controllers (Scenario.heuristic_action) as
batched torch code on the observations' device: no host round trip, so a
scripted rollout runs entirely on the GPU (rollout.DeviceHeuristicPolicy).

Each function restates the reference's numpy heuristic (the heuristic_action
of pkg/src/swarmsim/scenarios/<task>.py, cited per function) with numpy's
dtype semantics — float32 observations, Python floats weak (NEP 50), the
float64 promotions the reference performs (np.where / np.array of Python
floats) — so the forces equal the reference's bit for bit, except transport,
whose arctan2 / cos / sin are torch's (within a few float32 ulps;
tests/test_gpu_episodes.py checks all of them against the numpy controllers).
"""
from __future__ import annotations

import math

import torch

F32, F64 = torch.float32, torch.float64


def _norm(v: torch.Tensor) -> torch.Tensor:
    """np.linalg.norm(v, axis=1): sqrt(x*x + y*y) in v's dtype."""
    return torch.sqrt(v[:, 0] * v[:, 0] + v[:, 1] * v[:, 1])


def _unit(v: torch.Tensor, eps: float = 1e-8) -> torch.Tensor:
    return v / torch.clamp(_norm(v), min=eps)[:, None]


def _clip_unit(f: torch.Tensor, limit: float = 1.0) -> torch.Tensor:
    return torch.clamp(f, -limit, limit).to(F32)


def simple_spread(sc, i, obs):        # simple_spread.py heuristic_action
    return _clip_unit(5.0 * obs[:, 4 + 2 * i: 6 + 2 * i])


def discovery(sc, i, obs):            # discovery.py heuristic_action
    k = (i // 2) % sc.n_points
    return _clip_unit(4.0 * obs[:, 4 + 2 * k: 6 + 2 * k])


def dispersion(sc, i, obs):           # dispersion.py heuristic_action
    B = obs.shape[0]
    rels = torch.stack([obs[:, 4 + 3 * k: 6 + 3 * k] for k in range(sc.n_food)], 1)
    eaten = torch.stack([obs[:, 6 + 3 * k] for k in range(sc.n_food)], 1) > 0.5
    d = torch.sqrt(rels[..., 0] * rels[..., 0] + rels[..., 1] * rels[..., 1])
    dist = torch.where(eaten, torch.full_like(d, math.inf), d)
    order = torch.argsort(dist, dim=1, stable=True)
    remaining = torch.clamp((~eaten).sum(1), min=1)
    pick = order[torch.arange(B, device=obs.device), torch.clamp(remaining - 1, max=i)]
    return _clip_unit(5.0 * rels[torch.arange(B, device=obs.device), pick])


def _repulse(rel, reach, strength):
    d = _norm(rel)[:, None]
    return -_unit(rel) * (torch.clamp(reach - d, min=0.0) * strength)


def flocking(sc, i, obs):             # flocking.py heuristic_action
    force = 1.5 * obs[:, 4:6]
    for k in range(sc.n_obstacles):
        force = force + _repulse(obs[:, 6 + 2 * k: 8 + 2 * k], 0.3, 6.0)
    base = 6 + 2 * sc.n_obstacles
    for k in range(sc.n_agents - 1):
        force = force + _repulse(obs[:, base + 2 * k: base + 2 * k + 2], 0.18, 4.0)
    return _clip_unit(force)


def transport(sc, i, obs):            # transport.py heuristic_action
    to_package = obs[:, 4:6]
    push_dir = _unit(-obs[:, 8:10])
    lateral = torch.stack([-push_dir[:, 1], push_dir[:, 0]], 1)
    spread = (i - (sc.n_agents - 1) / 2) * 0.11
    r0 = sc.package_size / 2 + 0.07
    stand_off = to_package - push_dir * r0 + lateral * spread
    d = _norm(to_package)[:, None]
    facing = -(to_package / torch.clamp(d, min=1e-8))
    theta_a = torch.atan2(facing[:, 1], facing[:, 0])
    theta_b = torch.atan2(-push_dir[:, 1], -push_dir[:, 0])
    diff = torch.remainder(theta_b - theta_a + math.pi, 2.0 * math.pi) - math.pi
    behind = torch.abs(diff) < 0.5
    theta_t = theta_a + torch.clamp(diff, -0.6, 0.6)
    ring = torch.stack([torch.cos(theta_t), torch.sin(theta_t)], 1) * (r0 + 0.08)
    near = d[:, 0] < 0.6
    target = torch.where((near & ~behind)[:, None], to_package + ring, stand_off)
    lean = torch.where((near & behind)[:, None], 1.0, 0.0).to(F32)
    return _clip_unit(3.0 * target + push_dir * lean)


def reverse_transport(sc, i, obs):    # reverse_transport.py heuristic_action
    lead = _unit(obs[:, 8:10])
    return _clip_unit(3.0 * (obs[:, 4:6] + lead * (sc.crate_size / 2 - 0.04)) + lead)


def dropout(sc, i, obs):              # dropout.py heuristic_action
    to_goal = obs[:, 4:6]
    mine = _norm(to_goal)
    elected = torch.ones(obs.shape[0], dtype=torch.bool, device=obs.device)
    for k in range(sc.n_agents - 1):
        theirs = _norm(to_goal - obs[:, 6 + 2 * k: 8 + 2 * k])
        elected &= (mine < theirs) if k < i else (mine <= theirs)
    return _clip_unit(3.0 * to_goal * elected[:, None])


def wheel(sc, i, obs):                # wheel.py:76-87
    to_center, ca, sa = obs[:, 4:6], obs[:, 6], obs[:, 7]
    spin_err = obs[:, 9] - obs[:, 8]
    tip = to_center + torch.stack([ca, sa], 1) * (sc.line_length / 2)
    push = torch.stack([-sa, ca], 1) * torch.sign(spin_err)[:, None]
    lean = torch.clamp(4.0 * torch.abs(spin_err), max=1.0)[:, None]
    return _clip_unit(4.0 * (tip - push * 0.05) + push * lean)


def balance(sc, i, obs):              # balance.py:131-163
    to_tray, c, s, spin = obs[:, 4:6], obs[:, 6], obs[:, 7], obs[:, 8]
    tray_vy, to_ball = obs[:, 10], obs[:, 11:13]
    goal_dx, goal_dy = obs[:, 15], obs[:, 16]
    o = (i - (sc.n_agents - 1) / 2) * 0.22
    station_x = to_tray[:, 0] + o * c
    station_y = to_tray[:, 1] + o * s - 0.05
    ball_off = (to_ball[:, 0] - to_tray[:, 0]) * c + (to_ball[:, 1] - to_tray[:, 1]) * s
    centering = 0.8 * ball_off
    steering = -0.2 * torch.clamp(goal_dx, -1.0, 1.0)
    want_tilt = torch.clamp(torch.where(torch.abs(ball_off) > 0.22, centering, centering * 0.5 + steering),
                            -0.12, 0.12)
    hold = -sc.gravity * (1.0 + (sc.tray_mass + sc.ball_mass) / sc.n_agents)
    climb = torch.clamp(0.5 * goal_dy, -0.1, 0.2)
    side = float(math.copysign(1.0, o)) if o != 0 else 0.0
    fy = hold + climb - 1.0 * tray_vy + 3.0 * station_y + side * (3.5 * (want_tilt - s) - 0.8 * spin)
    fx = 3.5 * station_x + 0.25 * torch.clamp(goal_dx, -1.0, 1.0)
    return _clip_unit(torch.stack([fx, fy], 1))


def give_way(sc, i, obs):             # give_way.py heuristic_action
    to_goal, to_other, to_alcove = obs[:, 4:6], obs[:, 6:8], obs[:, 10:12]
    ahead = torch.sign(to_goal[:, 0]) == torch.sign(to_other[:, 0])
    must_yield = ahead & (torch.abs(to_other[:, 0]) < 0.9) & (i == 0)
    force = 3.0 * torch.where(must_yield[:, None], to_alcove, to_goal)
    fy = torch.where(must_yield, force[:, 1], force[:, 1] * 0.5)
    return _clip_unit(torch.stack([force[:, 0], fy], 1))


def passage(sc, i, obs):              # passage.py heuristic_action
    own_y, to_slot, gap_a, gap_b = obs[:, 1], obs[:, 4:6], obs[:, 6:8], obs[:, 8:10]
    nearer = torch.where((torch.abs(gap_a[:, 0]) <= torch.abs(gap_b[:, 0]))[:, None], gap_a, gap_b)
    across = (own_y > 0.06) & (to_slot[:, 1] > -0.5)
    crossing = torch.stack([nearer[:, 0] * 2.0 + 0.04 * i, torch.ones_like(own_y)], 1)
    return _clip_unit(torch.where(across[:, None], 4.0 * to_slot, 1.2 * crossing))


def waterfall(sc, i, obs):            # waterfall.py heuristic_action
    from .catalog import BLOCK_LEN, BLOCKS

    own_vy, to_basin = obs[:, 3], obs[:, 4:6]
    fx = 0.8 * to_basin[:, 0]
    fy = 0.4 * to_basin[:, 1] - 0.3 * own_vy
    for k in range(len(BLOCKS)):
        rel = obs[:, 6 + 2 * k: 8 + 2 * k]
        below = (rel[:, 1] < 0.0) & (rel[:, 1] > -0.3)
        lateral = torch.abs(rel[:, 0]) < BLOCK_LEN / 2 + 0.1
        kick = torch.where(below & lateral, torch.where(rel[:, 0] >= 0, -1.5, 1.5), 0.0).to(F64)
        fx = (fx.to(F64) + kick).to(F32)       # np.where of Python floats is float64
    return _clip_unit(torch.stack([fx, fy], 1))


def football(sc, i, obs):             # football.py heuristic_action
    to_ball = obs[:, 4:6]
    n_rel = 2 * (2 * sc.n_per_team - 1)
    to_mouth = obs[:, 8 + n_rel: 10 + n_rel]
    through = _unit(to_mouth - to_ball)
    stand_off = to_ball - through * 0.09
    if i % 2 == 1:   # float64: np.array([0.0, 0.3]) promotes
        off = torch.zeros_like(stand_off, dtype=F64)
        off[:, 1] = 0.3
        return _clip_unit(5.0 * (stand_off.to(F64) + off) + (through * 0.3).to(F64))
    near = _norm(stand_off)[:, None] < 0.12
    lean = torch.where(near, torch.full(near.shape, 1.0, dtype=F64, device=obs.device),
                       torch.full(near.shape, 0.2, dtype=F64, device=obs.device))   # float64 (np.where of Python floats)
    return _clip_unit((5.0 * stand_off).to(F64) + through.to(F64) * lean)


CONTROLLERS = {
    "SimpleSpread": simple_spread, "Discovery": discovery, "Dispersion": dispersion, "Flocking": flocking,
    "Transport": transport, "ReverseTransport": reverse_transport, "Dropout": dropout, "Wheel": wheel,
    "Balance": balance, "GiveWay": give_way, "Passage": passage, "Waterfall": waterfall, "Football": football,
}


def controller(scenario):
    """The device controller of a built-in scenario (None for user scenarios)."""
    for cls in type(scenario).__mro__:
        fn = CONTROLLERS.get(cls.__name__)
        if fn is not None:
            return fn
    return None
