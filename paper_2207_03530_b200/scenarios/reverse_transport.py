"""reverse_transport (swarmsim/scenarios/reverse_transport.py), fused.

Agents trapped inside a hollow crate drive it to a goal.  The world is
transport's (agents, a movable non-rotatable box, a goal marker; pairs
agent-agent then (agent, crate) per agent; sphere-box contacts on the box
perimeter), so the step is k_transport<n, 1> (csrc/ss_small.cu): the same
physics and reward (-|crate - goal|, float32; done when < success_dist) with
the reverse observation [x, y, vx, vy, crate - self, crate vel, goal - crate].
Resets place the agents relative to the freshly drawn crate: a device
reset program (float32 crate position plus float64 draws, ResetProgram).
"""
from __future__ import annotations

from ..core import World
from . import register
from ._fused import RefHeuristic
from .catalog import ReverseTransport as _Reference
from .transport import Transport


@register("reverse_transport")
class ReverseTransport(RefHeuristic, Transport):
    max_steps = 250
    _reference = _Reference

    def __init__(self, n_agents: int = 4, crate_size: float = 0.6, crate_mass: float = 3.0,
                 success_dist: float = 0.1):
        super().__init__(n_agents=n_agents, package_mass=crate_mass, package_size=crate_size,
                         success_dist=success_dist)
        self.crate_size, self.crate_mass = crate_size, crate_mass

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 10

    def fill_constants(self, world, d):
        super().fill_constants(world, d)
        d.si[1] = 1          # reverse observation layout

    def reset_program(self, world):
        """reverse_transport.py:53-67: the crate scattered and set level; each
        agent at crate + uniform offset (float32 crate position plus a float64
        draw, x then y), the goal scattered."""
        from ._fused import ResetProgram

        p, idx = ResetProgram(), world.index_of
        crate = idx(world.entity("crate"))
        p.scatter(crate, (-0.5, -0.5), (0.5, 0.5))
        p.setrot(crate, p.const(0.0))
        cx, cy = p.loadpos(crate, 0), p.loadpos(crate, 1)
        inner = self.crate_size / 2 - 0.05 - 0.07
        for agent in world.agents:
            ax = p.draw(-inner, inner)
            ay = p.draw(-inner, inner)
            a = idx(agent)
            p.setpos(a, p.add(cx, ax), p.add(cy, ay))
            p.zero(a)
            p.n_regs = 3          # register 0 (const) and cx, cy stay live
        p.scatter(idx(world.entity("goal")), (-0.9, -0.9), (0.9, 0.9))
        return p
