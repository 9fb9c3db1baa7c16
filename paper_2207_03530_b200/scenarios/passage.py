"""passage (swarmsim/scenarios/passage.py), fused reward / observation.

A cross formation squeezes through two wall gaps and reforms.  Physics (the
walls are line segments) is world_step's generic kernel, launched first; the
rest of the step — count, reward -gap - penalty * #touching teammates
(float32), done when every agent sits within 0.05 of its slot, observation
with the float64 gap offsets — is k_passage<n> (csrc/ss_small.cu).  Resets
are a device reset program (formation drawn around one centre).
"""
from __future__ import annotations

from .. import _native as N
from ..core import World
from ..shapes import min_contact_distance
from . import register
from ._fused import FusedScenario, RefHeuristic, ResetProgram, f32
from .catalog import GAPS, Passage as _Reference


@register("passage")
class Passage(RefHeuristic, FusedScenario):
    native_id = N.SCN_PASSAGE
    max_steps = 250
    _reference = _Reference

    def __init__(self, collision_penalty: float = 0.5):
        _Reference.__init__(self, collision_penalty)

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def obs_dim(self, world):
        return 10 + 2 * (len(world.agents) - 1)

    def template_pairs(self, world):
        return list(world.collidable_pairs())

    def fill_constants(self, world, d):
        a = world.agents[0].shape
        d.sc[0] = f32(min_contact_distance(a, a) + 0.0)     # common.touching
        d.sc[1] = f32(self.collision_penalty)
        d.sc[2] = f32(0.05)
        d.sd[0], d.sd[1] = float(GAPS[0]), float(GAPS[1])

    def reset_program(self, world):
        """passage.py:53-66: the formation centre (cx, cy) drawn once; agent i
        at (cx + ox, cy + oy), its slot mirrored at (cx + ox, -cy + oy) in
        float64; the walls placed."""
        from .catalog import OFFSETS

        p, idx = ResetProgram(), world.index_of
        cx = p.draw(-1.0, 1.0)
        cy = p.draw(-0.9, -0.45)
        ncy = p.neg(cy)
        for i, (ox, oy) in enumerate(OFFSETS):
            x = p.add(cx, p.const(ox))
            a = idx(world.entity(f"agent_{i}"))
            p.setpos(a, x, p.add(cy, p.const(oy)))
            p.zero(a)
            s = idx(world.entity(f"slot_{i}"))
            p.setpos(s, x, p.add(ncy, p.const(oy)))
            p.zero(s)
            p.n_regs = 3          # cx, cy, -cy stay live
        for k, (x0, x1) in enumerate(self._spans):
            p.place(idx(world.entity(f"wall_{k}")), (x0 + x1) / 2, 0.0)
        return p
