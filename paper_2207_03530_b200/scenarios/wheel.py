"""wheel (swarmsim/scenarios/wheel.py), fused reward / observation.

Agents push the tips of a pinned rod to hold a target spin.  Physics — the
sphere-line contacts and the rod's torque — is world_step's own generic
kernel (k_generic_physics, launched first in the same stream); k_wheel<n>
(csrc/ss_small.cu) then does count, reward -|w - target| (float32), horizon
done and the observation [x, y, vx, vy, rod - self, cos, sin (numpy float32),
w, target] in one launch.  Resets run the reference's host program (agents
scattered, the rod's angle drawn uniform in [0, 2 pi)).
"""
from __future__ import annotations

from .. import _native as N
from ..core import World
from . import register
from ._fused import FusedScenario, HostReset, f32
from .catalog import Wheel as _Reference


@register("wheel")
class Wheel(HostReset, FusedScenario):
    native_id = N.SCN_WHEEL
    max_steps = 200
    _reference = _Reference

    def __init__(self, n_agents: int = 3, line_length: float = 1.0, line_mass: float = 2.0,
                 target_spin: float = 0.3):
        self.n_agents, self.line_length = n_agents, line_length
        self.line_mass, self.target_spin = line_mass, target_spin

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 10

    def physics_fused(self, world) -> bool:
        return False         # world_step's generic kernel, then k_wheel

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        d.sc[0] = f32(self.target_spin)
