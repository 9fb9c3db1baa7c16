"""The other eight catalog tasks (swarmsim/scenarios/{wheel,balance,give_way,
football,passage,reverse_transport,dropout,waterfall}.py) on the device.

They have no fused kernel yet: physics runs in the
generic step kernel (lines, boxes, rotation, gravity, torques), resets draw
from the Env's Philox stream on the host exactly in the reference's call
order, and reward / done / observation are torch ops on device tensors that
replay numpy's dtype rules — float32 arithmetic where the reference stays in
float32, float64 where numpy promotes (np.full(...) columns, bool * float,
np.zeros(B) accumulators) and numpy's own float32 cos/sin via ss_np_trig.
Parity with the reference: tests/test_parity_golden.py (bit-exact fixtures).
"""
from __future__ import annotations

import numpy as np
import torch

from .._native import np_trig
from ..batching import Vec2
from ..core import Agent, AgentAction, Entity, PhysParams, World
from ..env import Scenario
from ..geometry import closest_points
from ..shapes import Box, Line, Sphere, min_contact_distance
from .common import clip_unit, columns, contact_count, marker, place, pos_vel, rel_pos, scatter, unit

F64 = torch.float64


def _dev(world: World):
    return world.device


def _f64_minus(value: float, t: torch.Tensor) -> torch.Tensor:
    """np.full(B, value) - t: numpy evaluates in float64."""
    return value - t.to(F64)


def _norm(a: Vec2, b: Vec2) -> torch.Tensor:
    return (a - b).norm()


def _n(world: World, env_index) -> int:
    return 1 if env_index is not None else world.batch_size


def _wall(name: str, length: float) -> Entity:
    return Entity(name, shape=Line(length=length), movable=False, rotatable=False)


def _np(obs):
    return obs.cpu().numpy() if hasattr(obs, "cpu") else np.asarray(obs)


# ---------------------------------------------------------------------------
class Wheel(Scenario):
    """Agents push the tips of a pinned rod to hold a target spin.

    The registered "wheel" is scenarios/wheel.py (world_step + k_wheel); this
    torch implementation supplies its world, reset and heuristic and stays the
    generic-path restatement of the reference hooks."""

    max_steps = 200

    def __init__(self, n_agents: int = 3, line_length: float = 1.0, line_mass: float = 2.0,
                 target_spin: float = 0.3):
        self.n_agents, self.line_length = n_agents, line_length
        self.line_mass, self.target_spin = line_mass, target_spin

    def make_world(self, batch_size, rng):
        w = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        for i in range(self.n_agents):
            w.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05), max_speed=0.4))
        w.add(Entity("rod", shape=Line(length=self.line_length), mass=self.line_mass, movable=False,
                     rotatable=True, color=(0.8, 0.3, 0.3)))
        return w

    def reset_world_at(self, world, env_index=None):
        for a in world.agents:
            scatter(world.rng, a, (-1.0, -1.0), (1.0, 1.0), world, env_index)
        rod = world.entity("rod")
        rod.state.set_rot(world.rng.uniform(0.0, 2 * np.pi, (_n(world, env_index),)), env_index)
        rod.state.zero_motion(env_index)

    def reward(self, agent, world):
        return -torch.abs(world.entity("rod").state.ang_vel - self.target_spin)

    def observation(self, agent, world):
        rod = world.entity("rod")
        rot = rod.state.rot
        return columns(*pos_vel(agent), rel_pos(agent, rod), np_trig(rot, True), np_trig(rot, False),
                       rod.state.ang_vel,
                       torch.full((world.batch_size,), self.target_spin, dtype=F64, device=_dev(world)))

    def heuristic_action(self, agent_index, obs):
        obs = _np(obs)
        to_center, ca, sa = obs[:, 4:6], obs[:, 6], obs[:, 7]
        spin_err = obs[:, 9] - obs[:, 8]
        tip = to_center + np.stack([ca, sa], axis=1) * (self.line_length / 2)
        push = np.stack([-sa, ca], axis=1) * np.sign(spin_err)[:, None]
        lean = np.minimum(1.0, 4.0 * np.abs(spin_err))[:, None]
        return clip_unit(4.0 * (tip - push * 0.05) + push * lean)


# ---------------------------------------------------------------------------
class Balance(Scenario):
    """Agents carry a ball on a tray against gravity to a goal.

    The registered "balance" is scenarios/balance.py (world_step +
    k_balance); this torch implementation supplies its world, reset and
    heuristic and stays the generic-path restatement of the reference hooks."""

    max_steps = 250

    def __init__(self, n_agents: int = 3, gravity: float = -0.3, tray_length: float = 0.8,
                 tray_mass: float = 2.0, ball_mass: float = 0.3):
        self.n_agents, self.gravity, self.tray_length = n_agents, gravity, tray_length
        self.tray_mass, self.ball_mass = tray_mass, ball_mass
        self.floor_y, self.ball_radius = -1.0, 0.06

    def make_world(self, batch_size, rng):
        w = World(batch_size, params=PhysParams(gravity=(0.0, self.gravity)), rng=rng,
                  device=getattr(rng, "device", None))
        for i in range(self.n_agents):
            w.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05), max_speed=0.4))
        w.add(Entity("tray", shape=Line(length=self.tray_length), mass=self.tray_mass, movable=True,
                     rotatable=True, color=(0.8, 0.3, 0.3)))
        w.add(Entity("ball", shape=Sphere(radius=self.ball_radius), mass=self.ball_mass, movable=True,
                     color=(0.9, 0.7, 0.2)))
        w.add(marker("goal", radius=0.08))
        w.add(Entity("floor", shape=Line(length=4.0), movable=False, rotatable=False))
        return w

    def reset_world_at(self, world, env_index=None):
        n, rng, tray_y = _n(world, env_index), world.rng, -0.62
        for k, agent in enumerate(world.agents):
            o = (k - (self.n_agents - 1) / 2) * 0.22
            agent.state.set_pos_xy(o + rng.uniform(-0.03, 0.03, (n,)), np.full(n, tray_y - 0.052), env_index)
            agent.state.zero_motion(env_index)
        tray = world.entity("tray")
        place(tray, 0.0, tray_y, world, env_index)
        tray.state.set_rot(0.0, env_index)
        ball = world.entity("ball")
        bx = rng.uniform(-0.2, 0.2, (n,))
        ball.state.set_pos_xy(bx, np.full(n, tray_y + self.ball_radius + 2e-3), env_index)
        ball.state.zero_motion(env_index)
        goal = world.entity("goal")
        gx = rng.uniform(-0.5, 0.5, (n,))
        gy = rng.uniform(0.2, 0.6, (n,))
        goal.state.set_pos_xy(gx, gy, env_index)
        goal.state.zero_motion(env_index)
        place(world.entity("floor"), 0.0, self.floor_y, world, env_index)

    def _dropped(self, world):
        return world.entity("ball").state.pos.y < self.floor_y + self.ball_radius + 0.02

    def reward(self, agent, world):
        gap = _norm(world.entity("ball").state.pos, world.entity("goal").state.pos)
        return -gap.to(F64) - 5.0 * self._dropped(world).to(F64)

    def done(self, world):
        return _norm(world.entity("ball").state.pos, world.entity("goal").state.pos) < 0.08

    def observation(self, agent, world):
        tray, ball, goal = world.entity("tray"), world.entity("ball"), world.entity("goal")
        return columns(*pos_vel(agent), rel_pos(agent, tray), np_trig(tray.state.rot, True),
                       np_trig(tray.state.rot, False), tray.state.ang_vel, tray.state.vel.x, tray.state.vel.y,
                       rel_pos(agent, ball), ball.state.vel.x, ball.state.vel.y, rel_pos(ball, goal))

    def heuristic_action(self, agent_index, obs):
        obs = _np(obs)
        to_tray, c, s, spin = obs[:, 4:6], obs[:, 6], obs[:, 7], obs[:, 8]
        tray_vy, to_ball = obs[:, 10], obs[:, 11:13]
        goal_dx, goal_dy = obs[:, 15], obs[:, 16]
        o = (agent_index - (self.n_agents - 1) / 2) * 0.22
        station_x = to_tray[:, 0] + o * c
        station_y = to_tray[:, 1] + o * s - 0.05
        ball_off = (to_ball[:, 0] - to_tray[:, 0]) * c + (to_ball[:, 1] - to_tray[:, 1]) * s
        centering = 0.8 * ball_off
        steering = -0.2 * np.clip(goal_dx, -1.0, 1.0)
        want_tilt = np.clip(np.where(np.abs(ball_off) > 0.22, centering, centering * 0.5 + steering), -0.12, 0.12)
        hold = -self.gravity * (1.0 + (self.tray_mass + self.ball_mass) / self.n_agents)
        climb = np.clip(0.5 * goal_dy, -0.1, 0.2)
        side = float(np.sign(o))
        fy = hold + climb - 1.0 * tray_vy + 3.0 * station_y + side * (3.5 * (want_tilt - s) - 0.8 * spin)
        fx = 3.5 * station_x + 0.25 * np.clip(goal_dx, -1.0, 1.0)
        return clip_unit(np.stack([fx, fy], axis=1))


# ---------------------------------------------------------------------------
class GiveWay(Scenario):
    """Two wide agents swap ends of a corridor with one recess.

    The registered "give_way" is scenarios/give_way.py (world_step +
    k_give_way); this torch implementation supplies its world, reset and
    heuristic and stays the generic-path restatement of the reference hooks."""

    max_steps = 300

    def __init__(self, agent_radius: float = 0.12, corridor_half_width: float = 0.2):
        self.agent_radius, self.half_width = agent_radius, corridor_half_width
        self.alcove = (0.0, 0.35)

    def make_world(self, batch_size, rng):
        w = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        w.add(Agent("agent_0", shape=Sphere(radius=self.agent_radius), color=(0.25, 0.45, 0.85)))
        w.add(Agent("agent_1", shape=Sphere(radius=self.agent_radius), color=(0.85, 0.35, 0.25)))
        w.add(marker("goal_0", radius=0.05, color=(0.25, 0.45, 0.85)))
        w.add(marker("goal_1", radius=0.05, color=(0.85, 0.35, 0.25)))
        for name, length in (("wall_bottom", 4.0), ("wall_top_left", 1.7), ("wall_top_right", 1.7),
                             ("alcove_left", 0.3), ("alcove_right", 0.3), ("alcove_top", 0.6)):
            w.add(_wall(name, length))
        return w

    def reset_world_at(self, world, env_index=None):
        n, rng, hw = _n(world, env_index), world.rng, self.half_width
        a0, a1 = world.agents
        for agent, lo, hi in ((a0, -1.6, -1.4), (a1, 1.4, 1.6)):
            x = rng.uniform(lo, hi, (n,))
            y = rng.uniform(-0.04, 0.04, (n,))
            agent.state.set_pos_xy(x, y, env_index)
            agent.state.zero_motion(env_index)
        place(world.entity("goal_0"), 1.5, 0.0, world, env_index)
        place(world.entity("goal_1"), -1.5, 0.0, world, env_index)
        place(world.entity("wall_bottom"), 0.0, -hw, world, env_index)
        place(world.entity("wall_top_left"), -1.15, hw, world, env_index)
        place(world.entity("wall_top_right"), 1.15, hw, world, env_index)
        for name, x in (("alcove_left", -0.3), ("alcove_right", 0.3)):
            wall = world.entity(name)
            place(wall, x, hw + 0.15, world, env_index)
            wall.state.set_rot(np.pi / 2, env_index)
        place(world.entity("alcove_top"), 0.0, hw + 0.3, world, env_index)

    def _gap(self, world, k):
        return _norm(world.agents[k].state.pos, world.entity(f"goal_{k}").state.pos)

    def reward(self, agent, world):
        gap = self._gap(world, world.agents.index(agent))
        return -gap.to(F64) + 5.0 * (gap < 0.15).to(F64)

    def done(self, world):
        return (self._gap(world, 0) < 0.15) & (self._gap(world, 1) < 0.15)

    def observation(self, agent, world):
        k = world.agents.index(agent)
        other, goal = world.agents[1 - k], world.entity(f"goal_{k}")
        return columns(*pos_vel(agent), rel_pos(agent, goal), rel_pos(agent, other), other.state.vel.x,
                       other.state.vel.y, _f64_minus(self.alcove[0], agent.state.pos.x),
                       _f64_minus(self.alcove[1], agent.state.pos.y))

    def heuristic_action(self, agent_index, obs):
        obs = _np(obs)
        to_goal, to_other, to_alcove = obs[:, 4:6], obs[:, 6:8], obs[:, 10:12]
        ahead = np.sign(to_goal[:, 0]) == np.sign(to_other[:, 0])
        must_yield = (agent_index == 0) & ahead & (np.abs(to_other[:, 0]) < 0.9)
        force = 3.0 * np.where(must_yield[:, None], to_alcove, to_goal)
        force[:, 1] = np.where(must_yield, force[:, 1], force[:, 1] * 0.5)
        return clip_unit(force)


# ---------------------------------------------------------------------------
FIELD_HX, FIELD_HY, MOUTH_HY, NET_DEPTH = 1.5, 1.0, 0.35, 0.25


def chase_script(agent: Agent, world: World) -> AgentAction:
    """Red defender: the nearer red attacks the ball, the other holds post."""
    B, dev = world.batch_size, world.device
    ball = world.entity("ball")
    reds = [a for a in world.agents if a.name.startswith("red")]
    me = world.agents.index(agent)
    dists = torch.stack([_norm(r.state.pos, ball.state.pos) for r in reds])
    mine = [world.agents.index(r) for r in reds].index(me)
    closer = torch.argmin(dists, dim=0) == mine
    behind = ball.state.pos + Vec2.full(B, 0.08, 0.0, device=dev) - agent.state.pos
    to_post = Vec2.full(B, -0.75, 0.0, device=dev) - agent.state.pos
    tx = torch.where(closer, behind.x, to_post.x)
    ty = torch.where(closer, behind.y, to_post.y)
    u = agent.u_range
    fx = torch.clamp(3.0 * tx, -u, u)
    fy = torch.clamp(3.0 * ty, -u, u)
    return AgentAction(force=Vec2(fx * agent.u_multiplier, fy * agent.u_multiplier))


class Football(Scenario):
    """Two-a-side: the controlled blue team attacks against scripted reds.

    The registered "football" is scenarios/football.py (world_step +
    k_football); this torch implementation supplies its world, reset, the
    reds' script and the heuristic, and stays the generic-path restatement of
    the reference hooks."""

    max_steps = 400

    def __init__(self, n_per_team: int = 2, ball_mass: float = 0.25):
        self.n_per_team, self.ball_mass = n_per_team, ball_mass

    def make_world(self, batch_size, rng):
        w = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        for i in range(self.n_per_team):
            w.add(Agent(f"blue_{i}", shape=Sphere(radius=0.05), color=(0.25, 0.45, 0.85)))
        for i in range(self.n_per_team):
            w.add(Agent(f"red_{i}", shape=Sphere(radius=0.05), color=(0.85, 0.3, 0.25), action_script=chase_script))
        w.add(Entity("ball", shape=Sphere(radius=0.06), mass=self.ball_mass, movable=True, max_speed=0.5,
                     color=(0.95, 0.95, 0.95)))
        side = FIELD_HY - MOUTH_HY
        for name, length in (("fence_top", 2 * FIELD_HX), ("fence_bottom", 2 * FIELD_HX),
                             ("fence_left_up", side), ("fence_left_down", side), ("fence_right_up", side),
                             ("fence_right_down", side), ("net_left_back", 2 * MOUTH_HY),
                             ("net_left_up", NET_DEPTH), ("net_left_down", NET_DEPTH),
                             ("net_right_back", 2 * MOUTH_HY), ("net_right_up", NET_DEPTH),
                             ("net_right_down", NET_DEPTH)):
            w.add(_wall(name, length))
        return w

    def reset_world_at(self, world, env_index=None):
        n, rng = _n(world, env_index), world.rng
        for i in range(self.n_per_team):
            for name, lo, hi in ((f"blue_{i}", -1.2, -0.3), (f"red_{i}", 0.3, 1.2)):
                e = world.entity(name)
                x = rng.uniform(lo, hi, (n,))
                y = rng.uniform(-0.7, 0.7, (n,))
                e.state.set_pos_xy(x, y, env_index)
                e.state.zero_motion(env_index)
        ball = world.entity("ball")
        jx = rng.uniform(-0.1, 0.1, (n,))
        jy = rng.uniform(-0.1, 0.1, (n,))
        ball.state.set_pos_xy(jx, jy, env_index)
        ball.state.zero_motion(env_index)
        mid = (MOUTH_HY + FIELD_HY) / 2
        place(world.entity("fence_top"), 0.0, FIELD_HY, world, env_index)
        place(world.entity("fence_bottom"), 0.0, -FIELD_HY, world, env_index)
        for side, sx in (("left", -FIELD_HX), ("right", FIELD_HX)):
            for part, y in (("up", mid), ("down", -mid)):
                f = world.entity(f"fence_{side}_{part}")
                place(f, sx, y, world, env_index)
                f.state.set_rot(np.pi / 2, env_index)
            bx = sx - NET_DEPTH if side == "left" else sx + NET_DEPTH
            back = world.entity(f"net_{side}_back")
            place(back, bx, 0.0, world, env_index)
            back.state.set_rot(np.pi / 2, env_index)
            for edge, ey in (("up", MOUTH_HY), ("down", -MOUTH_HY)):
                place(world.entity(f"net_{side}_{edge}"), (sx + bx) / 2, ey, world, env_index)

    def _scored(self, world):
        x = world.entity("ball").state.pos.x
        return x > FIELD_HX + 0.04, x < -FIELD_HX - 0.04

    def reward(self, agent, world):
        B = world.batch_size
        if agent.action_script is not None:
            return torch.zeros(B, dtype=F64, device=world.device)
        right, left = self._scored(world)
        gap = _norm(world.entity("ball").state.pos, Vec2.full(B, FIELD_HX, 0.0, device=world.device))
        return 10.0 * right.to(F64) - 10.0 * left.to(F64) - (0.1 * gap).to(F64)

    def done(self, world):
        right, left = self._scored(world)
        return right | left

    def observation(self, agent, world):
        ball = world.entity("ball")
        mates = [a for a in world.agents if a is not agent and a.name[0] == agent.name[0]]
        foes = [a for a in world.agents if a.name[0] != agent.name[0]]
        attack_x = FIELD_HX if agent.name.startswith("blue") else -FIELD_HX
        return columns(*pos_vel(agent), rel_pos(agent, ball), ball.state.vel.x, ball.state.vel.y,
                       *[rel_pos(agent, m) for m in mates], *[rel_pos(agent, f) for f in foes],
                       _f64_minus(attack_x, agent.state.pos.x), 0.0 - agent.state.pos.y)

    def heuristic_action(self, agent_index, obs):
        obs = _np(obs)
        to_ball = obs[:, 4:6]
        n_rel = 2 * (2 * self.n_per_team - 1)
        to_mouth = obs[:, 8 + n_rel: 10 + n_rel]
        through = unit(to_mouth - to_ball)
        stand_off = to_ball - through * 0.09
        lean = np.where(np.linalg.norm(stand_off, axis=1, keepdims=True) < 0.12, 1.0, 0.2)
        force = 5.0 * stand_off + through * lean
        if agent_index % 2 == 1:
            force = 5.0 * (stand_off + np.array([0.0, 0.3])) + through * 0.3
        return clip_unit(force)


# ---------------------------------------------------------------------------
OFFSETS = [(0.0, 0.0), (0.2, 0.0), (-0.2, 0.0), (0.0, 0.2), (0.0, -0.2)]
GAPS, GAP_WIDTH = (-0.6, 0.6), 0.25


class Passage(Scenario):
    """A cross formation squeezes through two wall gaps and reforms.

    The registered "passage" is scenarios/passage.py (world_step +
    k_passage); this torch implementation supplies its world, reset and
    heuristic and stays the generic-path restatement of the reference hooks."""

    max_steps = 250

    def __init__(self, collision_penalty: float = 0.5):
        self.collision_penalty = collision_penalty
        half = GAP_WIDTH / 2
        self._spans = [(-2.0, GAPS[0] - half), (GAPS[0] + half, GAPS[1] - half), (GAPS[1] + half, 2.0)]

    def make_world(self, batch_size, rng):
        w = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        for i in range(len(OFFSETS)):
            w.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05), max_speed=0.4))
        for i in range(len(OFFSETS)):
            w.add(marker(f"slot_{i}", radius=0.03))
        for k, (x0, x1) in enumerate(self._spans):
            w.add(Entity(f"wall_{k}", shape=Line(length=x1 - x0), movable=False, rotatable=False))
        return w

    def reset_world_at(self, world, env_index=None):
        n, rng = _n(world, env_index), world.rng
        cx = rng.uniform(-1.0, 1.0, (n,))
        cy = rng.uniform(-0.9, -0.45, (n,))
        for i, (ox, oy) in enumerate(OFFSETS):
            agent = world.entity(f"agent_{i}")
            agent.state.set_pos_xy(cx + ox, cy + oy, env_index)
            agent.state.zero_motion(env_index)
            slot = world.entity(f"slot_{i}")
            slot.state.set_pos_xy(cx + ox, -cy + oy, env_index)
            slot.state.zero_motion(env_index)
        for k, (x0, x1) in enumerate(self._spans):
            place(world.entity(f"wall_{k}"), (x0 + x1) / 2, 0.0, world, env_index)

    def reward(self, agent, world):
        k = world.agents.index(agent)
        gap = _norm(agent.state.pos, world.entity(f"slot_{k}").state.pos)
        return -gap - self.collision_penalty * contact_count(agent, world.agents)

    def done(self, world):
        out = None
        for k, a in enumerate(world.agents):
            s = _norm(a.state.pos, world.entity(f"slot_{k}").state.pos) < 0.05
            out = s if out is None else out & s
        return out

    def observation(self, agent, world):
        k = world.agents.index(agent)
        others = [a for a in world.agents if a is not agent]
        gap_rel = []
        for gx in GAPS:
            gap_rel.append(_f64_minus(gx, agent.state.pos.x))
            gap_rel.append(0.0 - agent.state.pos.y)
        return columns(*pos_vel(agent), rel_pos(agent, world.entity(f"slot_{k}")), *gap_rel,
                       *[rel_pos(agent, o) for o in others])

    def heuristic_action(self, agent_index, obs):
        obs = _np(obs)
        own_y, to_slot, gap_a, gap_b = obs[:, 1], obs[:, 4:6], obs[:, 6:8], obs[:, 8:10]
        nearer = np.where((np.abs(gap_a[:, 0]) <= np.abs(gap_b[:, 0]))[:, None], gap_a, gap_b)
        crossing = np.stack([nearer[:, 0] * 2.0, np.ones_like(own_y)], axis=1)
        across = (own_y > 0.06) & (to_slot[:, 1] > -0.5)
        crossing[:, 0] = crossing[:, 0] + 0.04 * agent_index
        return clip_unit(np.where(across[:, None], 4.0 * to_slot, 1.2 * crossing))


# ---------------------------------------------------------------------------
class ReverseTransport(Scenario):
    """Agents trapped inside a hollow crate drive it to a goal.

    The registered "reverse_transport" is the fused version
    (scenarios/reverse_transport.py: k_transport's reverse layout); this torch
    implementation supplies its world, reset and heuristic, and stays the
    generic-path restatement of the reference hooks."""

    max_steps = 250

    def __init__(self, n_agents: int = 4, crate_size: float = 0.6, crate_mass: float = 3.0,
                 success_dist: float = 0.1):
        self.n_agents, self.crate_size = n_agents, crate_size
        self.crate_mass, self.success_dist = crate_mass, success_dist

    def make_world(self, batch_size, rng):
        w = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        for i in range(self.n_agents):
            w.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05), max_speed=0.4))
        w.add(Entity("crate", shape=Box(length=self.crate_size, width=self.crate_size), mass=self.crate_mass,
                     movable=True, rotatable=False, color=(0.8, 0.5, 0.2)))
        w.add(marker("goal", radius=0.12))
        return w

    def reset_world_at(self, world, env_index=None):
        n, rng = _n(world, env_index), world.rng
        crate = world.entity("crate")
        scatter(rng, crate, (-0.5, -0.5), (0.5, 0.5), world, env_index)
        crate.state.set_rot(0.0, env_index)
        cx = crate.state.pos.x if env_index is None else crate.state.pos.x[env_index:env_index + 1]
        cy = crate.state.pos.y if env_index is None else crate.state.pos.y[env_index:env_index + 1]
        cx, cy = cx.cpu().numpy(), cy.cpu().numpy()
        inner = self.crate_size / 2 - 0.05 - 0.07
        for agent in world.agents:
            ax = rng.uniform(-inner, inner, (n,))
            ay = rng.uniform(-inner, inner, (n,))
            agent.state.set_pos_xy(cx + ax, cy + ay, env_index)
            agent.state.zero_motion(env_index)
        scatter(rng, world.entity("goal"), (-0.9, -0.9), (0.9, 0.9), world, env_index)

    def _gap(self, world):
        return _norm(world.entity("crate").state.pos, world.entity("goal").state.pos)

    def reward(self, agent, world):
        return -self._gap(world)

    def done(self, world):
        return self._gap(world) < self.success_dist

    def observation(self, agent, world):
        crate, goal = world.entity("crate"), world.entity("goal")
        return columns(*pos_vel(agent), rel_pos(agent, crate), crate.state.vel.x, crate.state.vel.y,
                       rel_pos(crate, goal))

    def heuristic_action(self, agent_index, obs):
        obs = _np(obs)
        to_crate, lead = obs[:, 4:6], unit(obs[:, 8:10])
        return clip_unit(3.0 * (to_crate + lead * (self.crate_size / 2 - 0.04)) + lead)


# ---------------------------------------------------------------------------
class Dropout(Scenario):
    """Any one agent reaching the goal scores; every agent pays for effort.

    The registered "dropout" is the fused version (scenarios/dropout.py:
    k_dropout); this torch implementation supplies its world and heuristic
    and stays the generic-path restatement of the reference hooks."""

    max_steps = 200

    def __init__(self, n_agents: int = 4, energy_coeff: float = 0.02, reach: float = 0.1):
        self.n_agents, self.energy_coeff, self.reach = n_agents, energy_coeff, reach

    def make_world(self, batch_size, rng):
        w = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        for i in range(self.n_agents):
            w.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05), collidable=False))
        w.add(marker("goal", radius=0.08))
        return w

    def reset_world_at(self, world, env_index=None):
        for e in world.entities:
            scatter(world.rng, e, (-1.0, -1.0), (1.0, 1.0), world, env_index)

    def _reached(self, world):
        goal = world.entity("goal")
        d = torch.stack([_norm(a.state.pos, goal.state.pos) for a in world.agents])
        return (d <= self.reach).any(dim=0)

    def reward(self, agent, world):
        spent = torch.zeros(world.batch_size, dtype=F64, device=world.device)
        for a in world.agents:
            if a.action is not None:
                f = a.action.force
                # numpy: (spent + fx*fx) + fy*fy, each float32 square promoted
                spent = spent + (f.x * f.x).to(F64) + (f.y * f.y).to(F64)
        return self._reached(world).to(F64) - self.energy_coeff * spent

    def done(self, world):
        return self._reached(world)

    def observation(self, agent, world):
        goal = world.entity("goal")
        return columns(*pos_vel(agent), rel_pos(agent, goal),
                       *[rel_pos(agent, o) for o in world.agents if o is not agent])

    def heuristic_action(self, agent_index, obs):
        obs = _np(obs)
        to_goal = obs[:, 4:6]
        my_dist = np.linalg.norm(to_goal, axis=1)
        elected = np.ones(obs.shape[0], dtype=bool)
        for k in range(self.n_agents - 1):
            their = np.linalg.norm(to_goal - obs[:, 6 + 2 * k: 8 + 2 * k], axis=1)
            elected &= (my_dist < their) if k < agent_index else (my_dist <= their)
        return clip_unit(3.0 * to_goal * elected[:, None])


# ---------------------------------------------------------------------------
BLOCKS = [(-0.7, 0.35), (0.0, 0.35), (0.7, 0.35), (-0.35, -0.25), (0.35, -0.25)]
BLOCK_LEN, BLOCK_WID, BASIN = 0.45, 0.1, (0.0, -0.9)


class Waterfall(Scenario):
    """Agents drift down under gravity through staggered baffles to a basin.

    The registered "waterfall" is scenarios/waterfall.py (world_step +
    k_waterfall); this torch implementation supplies its world, reset and
    heuristic and stays the generic-path restatement of the reference hooks."""

    max_steps = 200

    def __init__(self, n_agents: int = 4, gravity: float = -0.2, collision_penalty: float = 0.3):
        self.n_agents, self.gravity, self.collision_penalty = n_agents, gravity, collision_penalty

    def make_world(self, batch_size, rng):
        w = World(batch_size, params=PhysParams(gravity=(0.0, self.gravity)), rng=rng,
                  device=getattr(rng, "device", None))
        for i in range(self.n_agents):
            w.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05), max_speed=0.35))
        w.add(marker("basin", radius=0.15, color=(0.2, 0.5, 0.9)))
        for k in range(len(BLOCKS)):
            w.add(Entity(f"block_{k}", shape=Box(length=BLOCK_LEN, width=BLOCK_WID), movable=False,
                         color=(0.45, 0.45, 0.5)))
        return w

    def reset_world_at(self, world, env_index=None):
        n, rng = _n(world, env_index), world.rng
        for agent in world.agents:
            x = rng.uniform(-0.6, 0.6, (n,))
            y = rng.uniform(0.75, 0.95, (n,))
            agent.state.set_pos_xy(x, y, env_index)
            agent.state.zero_motion(env_index)
        place(world.entity("basin"), *BASIN, world, env_index)
        for k, (bx, by) in enumerate(BLOCKS):
            place(world.entity(f"block_{k}"), bx, by, world, env_index)

    def _block_bumps(self, agent, world):
        count = torch.zeros(world.batch_size, dtype=F64, device=world.device)
        r = agent.shape.radius
        for k in range(len(BLOCKS)):
            b = world.entity(f"block_{k}")
            _, p = closest_points(agent.state.pos, agent.state.rot, agent.shape, b.state.pos, b.state.rot, b.shape)
            count = count + (_norm(agent.state.pos, p) <= r).to(F64)
        return count

    def reward(self, agent, world):
        gap = _norm(agent.state.pos, world.entity("basin").state.pos)
        bumps = contact_count(agent, world.agents).to(F64) + self._block_bumps(agent, world)
        return -gap.to(F64) - self.collision_penalty * bumps

    def done(self, world):
        basin = world.entity("basin")
        out = None
        for a in world.agents:
            s = _norm(a.state.pos, basin.state.pos) < 0.2
            out = s if out is None else out & s
        return out

    def observation(self, agent, world):
        return columns(*pos_vel(agent), rel_pos(agent, world.entity("basin")),
                       *[rel_pos(agent, world.entity(f"block_{k}")) for k in range(len(BLOCKS))])

    def heuristic_action(self, agent_index, obs):
        obs = _np(obs)
        own_vy, to_basin = obs[:, 3], obs[:, 4:6]
        force = np.stack([0.8 * to_basin[:, 0], 0.4 * to_basin[:, 1] - 0.3 * own_vy], axis=1)
        for k in range(len(BLOCKS)):
            rel = obs[:, 6 + 2 * k: 8 + 2 * k]
            below = (rel[:, 1] < 0.0) & (rel[:, 1] > -0.3)
            lateral = np.abs(rel[:, 0]) < BLOCK_LEN / 2 + 0.1
            force[:, 0] = force[:, 0] + np.where(below & lateral, np.where(rel[:, 0] >= 0, -1.5, 1.5), 0.0)
        return clip_unit(force)
