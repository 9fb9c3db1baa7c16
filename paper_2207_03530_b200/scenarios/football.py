"""football (swarmsim/scenarios/football.py), fused reward / observation.

Two-a-side: the controlled blue team attacks against scripted reds.  The
reds' chase script runs on the device before the step (Env's host-decode
path), physics (ball, fences and nets as line segments) is world_step's
generic kernel, and the rest of the step — count, goal test, reward
10 * right - 10 * left - 0.1 * gap for blues (0 for scripted reds), done,
observation — is k_football<n> (csrc/ss_small.cu).  Resets are a device
reset program (ResetProgram).
"""
from __future__ import annotations

import numpy as np

from .. import _native as N
from ..core import World
from . import register
from ._fused import FusedScenario, RefHeuristic, ResetProgram, f32
from .catalog import FIELD_HX, Football as _Reference, chase_script


@register("football")
class Football(RefHeuristic, FusedScenario):
    native_id = N.SCN_FOOTBALL
    max_steps = 400
    _reference = _Reference

    def __init__(self, n_per_team: int = 2, ball_mass: float = 0.25):
        _Reference.__init__(self, n_per_team, ball_mass)

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 8 + 2 * (len(world.agents) - 1) + 2

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def device_scripted(self, agent) -> bool:
        """The reds' chase script runs inside k_football (same float32
        arithmetic as catalog.chase_script / football.py:31-47)."""
        return agent.action_script is chase_script

    def fill_constants(self, world, d):
        d.sc[0] = f32(FIELD_HX + 0.04)     # _scored thresholds (python double)
        d.sc[1] = f32(0.1)
        d.sc[2] = f32(FIELD_HX)            # Vec2.full(B, FIELD_HX, 0.0): float32
        d.sd[0] = float(FIELD_HX)

    def reset_program(self, world):
        """football.py:100-138: blues and reds drawn (x then y) in their
        halves, the ball jittered around the centre spot, fences and nets
        placed (the side fences and the net backs upright)."""
        from .catalog import FIELD_HY, MOUTH_HY, NET_DEPTH

        p, idx = ResetProgram(), world.index_of
        for i in range(self.n_per_team):
            p.scatter(idx(world.entity(f"blue_{i}")), (-1.2, -0.7), (-0.3, 0.7))
            p.scatter(idx(world.entity(f"red_{i}")), (0.3, -0.7), (1.2, 0.7))
        p.scatter(idx(world.entity("ball")), (-0.1, -0.1), (0.1, 0.1))
        mid = (MOUTH_HY + FIELD_HY) / 2
        p.place(idx(world.entity("fence_top")), 0.0, FIELD_HY)
        p.place(idx(world.entity("fence_bottom")), 0.0, -FIELD_HY)
        up = p.const(np.pi / 2)
        for side, sx in (("left", -FIELD_HX), ("right", FIELD_HX)):
            for part, y in (("up", mid), ("down", -mid)):
                f = idx(world.entity(f"fence_{side}_{part}"))
                p.place(f, sx, y)
                p.setrot(f, up)
            bx = sx - NET_DEPTH if side == "left" else sx + NET_DEPTH
            back = idx(world.entity(f"net_{side}_back"))
            p.place(back, bx, 0.0)
            p.setrot(back, up)
            for edge, ey in (("up", MOUTH_HY), ("down", -MOUTH_HY)):
                p.place(idx(world.entity(f"net_{side}_{edge}")), (sx + bx) / 2, ey)
        return p
