"""wheel (swarmsim/scenarios/wheel.py), fused reward / observation.

Agents push the tips of a pinned rod to hold a target spin.  Physics — the
sphere-line contacts and the rod's torque — is world_step's own generic
kernel (k_generic_physics, launched first in the same stream); k_wheel<n>
(csrc/ss_small.cu) then does count, reward -|w - target| (float32), horizon
done and the observation [x, y, vx, vy, rod - self, cos, sin (numpy float32),
w, target] in one launch.  Resets are a device reset program (agents scattered, the rod's angle
drawn uniform in [0, 2 pi)), masked and sharded like every built-in.
"""
from __future__ import annotations

import numpy as np

from .. import _native as N
from ..core import World
from . import register
from ._fused import FusedScenario, RefHeuristic, ResetProgram, f32
from .catalog import Wheel as _Reference


@register("wheel")
class Wheel(RefHeuristic, FusedScenario):
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

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        d.sc[0] = f32(self.target_spin)

    def reset_program(self, world):
        """wheel.py:53-59: agents scattered in [-1, 1]^2; the rod's angle
        uniform in [0, 2 pi), its motion zeroed."""
        p = ResetProgram()
        for a in world.agents:
            p.scatter(world.index_of(a), (-1.0, -1.0), (1.0, 1.0))
        rod = world.index_of(world.entity("rod"))
        p.setrot(rod, p.draw(0.0, 2 * np.pi))
        p.zero(rod)
        return p
