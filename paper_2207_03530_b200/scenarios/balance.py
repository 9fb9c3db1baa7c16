"""balance (swarmsim/scenarios/balance.py), fused reward / observation.

Agents carry a ball on a tray against gravity to a goal.  Physics (gravity,
the tray's sphere-line contacts and torque) is world_step's generic kernel,
launched first; the rest of the step — count, reward -gap - 5 * dropped
(float64 cast to float32), done when the ball reaches the goal, observation
with numpy's float32 cos/sin of the tray angle — is k_balance<n>
(csrc/ss_small.cu).  Resets are a device reset program (ResetProgram).
"""
from __future__ import annotations

from .. import _native as N
from ..core import World
from . import register
from ._fused import FusedScenario, RefHeuristic, ResetProgram, f32
from .catalog import Balance as _Reference


@register("balance")
class Balance(RefHeuristic, FusedScenario):
    native_id = N.SCN_BALANCE
    max_steps = 250
    _reference = _Reference

    def __init__(self, n_agents: int = 3, gravity: float = -0.3, tray_length: float = 0.8,
                 tray_mass: float = 2.0, ball_mass: float = 0.3):
        _Reference.__init__(self, n_agents, gravity, tray_length, tray_mass, ball_mass)

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 17

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        d.sc[0] = f32(self.floor_y + self.ball_radius + 0.02)   # _dropped threshold (python double)
        d.sc[1] = f32(0.08)

    def reset_program(self, world):
        """balance.py:69-94: carriers at their stations below the tray (x
        jittered), the tray placed level, the ball dropped on it at a random
        x, the goal drawn, the floor placed."""
        p, idx = ResetProgram(), world.index_of
        tray_y = -0.62
        for k, agent in enumerate(world.agents):
            o = (k - (self.n_agents - 1) / 2) * 0.22
            a = idx(agent)
            p.setpos(a, p.add(p.const(o), p.draw(-0.03, 0.03)), p.const(tray_y - 0.052))
            p.zero(a)
            p.release()
        tray = idx(world.entity("tray"))
        p.place(tray, 0.0, tray_y)
        p.setrot(tray, p.const(0.0))
        ball = idx(world.entity("ball"))
        p.setpos(ball, p.draw(-0.2, 0.2), p.const(tray_y + self.ball_radius + 2e-3))
        p.zero(ball)
        goal = idx(world.entity("goal"))
        gx = p.draw(-0.5, 0.5)
        gy = p.draw(0.2, 0.6)
        p.setpos(goal, gx, gy)
        p.zero(goal)
        p.place(idx(world.entity("floor")), 0.0, self.floor_y)
        return p
