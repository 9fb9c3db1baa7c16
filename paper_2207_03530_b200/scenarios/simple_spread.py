"""simple_spread (swarmsim/scenarios/simple_spread.py): n agents cover n markers.

Fused kernel: k_simple_spread<n> (csrc/ss_small.cu).  Reward per agent
(simple_spread.py:39-46): -(sum over markers of the nearest-agent distance,
float64 accumulator) - penalty * #teammates touching.  Observation
(:48-54): [x, y, vx, vy, (marker - self) for each marker, (other - self)].
"""
from __future__ import annotations

import numpy as np
import torch

from .. import _native as N
from .._numerics import sqrt_le_bound
from ..core import Agent, World
from ..shapes import Sphere, min_contact_distance
from . import register
from ._fused import FusedScenario, f32
from .common import clip_unit, marker


@register("simple_spread")
class SimpleSpread(FusedScenario):
    native_id = N.SCN_SIMPLE_SPREAD
    max_steps = 200

    def __init__(self, n_agents: int = 3, collision_penalty: float = 1.0):
        self.n_agents = n_agents
        self.collision_penalty = collision_penalty

    def make_world(self, batch_size: int, rng) -> World:
        world = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        for i in range(self.n_agents):
            world.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05)))
        for i in range(self.n_agents):
            world.add(marker(f"mark_{i}"))
        return world

    def reset_ops(self, world):
        return [(k, "scatter", (-1.0, -1.0), (1.0, 1.0)) for k in range(len(world.entities))]

    def obs_dim(self, world):
        return 4 * self.n_agents + 2

    def template_pairs(self, world):
        n = self.n_agents
        return [(i, j) for i in range(n) for j in range(i + 1, n)]

    def template_ok(self, world):
        n = self.n_agents
        ents = world.entities
        return (len(ents) == 2 * n and all(e.movable and not e.rotatable for e in ents[:n])
                and not any(e.movable for e in ents[n:])
                and all(isinstance(e.shape, Sphere) for e in ents)
                and len({e.shape.radius for e in ents[:n]}) == 1)

    def fill_constants(self, world, d):
        a = world.agents
        thr = f32(min_contact_distance(a[0].shape, a[0].shape) + 0.0)   # common.touching
        d.sc[0] = thr
        d.sc[1] = f32(self.collision_penalty)
        d.sc[2] = sqrt_le_bound(thr)

    def heuristic_action(self, agent_index: int, obs):
        target = obs[:, 4 + 2 * agent_index: 6 + 2 * agent_index]
        return clip_unit(5.0 * target)
