"""balance (swarmsim/scenarios/balance.py), fused reward / observation.

Agents carry a ball on a tray against gravity to a goal.  Physics (gravity,
the tray's sphere-line contacts and torque) is world_step's generic kernel,
launched first; the rest of the step — count, reward -gap - 5 * dropped
(float64 cast to float32), done when the ball reaches the goal, observation
with numpy's float32 cos/sin of the tray angle — is k_balance<n>
(csrc/ss_small.cu).  Resets run the reference's host program.
"""
from __future__ import annotations

from .. import _native as N
from ..core import World
from . import register
from ._fused import FusedScenario, HostReset, f32
from .catalog import Balance as _Reference


@register("balance")
class Balance(HostReset, FusedScenario):
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

    def physics_fused(self, world) -> bool:
        return False         # world_step's generic kernel, then k_balance

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        d.sc[0] = f32(self.floor_y + self.ball_radius + 0.02)   # _dropped threshold (python double)
        d.sc[1] = f32(0.08)
