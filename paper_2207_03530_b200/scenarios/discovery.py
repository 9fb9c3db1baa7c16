"""discovery (swarmsim/scenarios/discovery.py): pairs of agents cover points.

Fused kernel: k_discovery<T> (csrc/ss_large.cu, one warp per env, all
agent pairs collide).  post_step (discovery.py:57-71): a point is covered
when >= quorum agents are within cover_dist; every env draws a fresh
location for every point every step (uniform_in_box on the Env's Philox
stream: x block then y block per point) and covered points move there.
Shared reward: #covered - 0.05 * sum over points of the quorum-th nearest
agent distance (float64).  Observation: [x, y, vx, vy, point_i - self,
other - self].
"""
from __future__ import annotations

import weakref

import numpy as np
import torch

from .. import _native as N
from .._numerics import sqrt_le_bound
from ..core import Agent, World
from ..shapes import Sphere
from . import register
from ._fused import FusedScenario, f32
from .common import clip_unit, marker
from .dispersion import unpack_bits


@register("discovery")
class Discovery(FusedScenario):
    native_id = N.SCN_DISCOVERY
    advances_rng_per_step = True
    max_steps = 200

    def __init__(self, n_agents: int = 5, n_points: int = 3, quorum: int = 2, cover_dist: float = 0.35):
        self.n_agents = n_agents
        self.n_points = n_points
        self.quorum = quorum
        self.cover_dist = cover_dist
        self._world = None

    def make_world(self, batch_size: int, rng) -> World:
        world = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        for i in range(self.n_agents):
            world.add(Agent(f"agent_{i}", shape=Sphere(radius=0.03)))
        for i in range(self.n_points):
            world.add(marker(f"point_{i}", radius=0.05, color=(0.9, 0.3, 0.6)))
        world.ensure_flag_words(self.n_flag_words())
        self._world = weakref.ref(world)
        return world

    def n_flag_words(self) -> int:
        return (self.n_points + 31) // 32

    def reset_ops(self, world):
        return ([(k, "scatter", (-1.0, -1.0), (1.0, 1.0)) for k in range(self.n_agents)]
                + [(self.n_agents + i, "scatter", (-0.9, -0.9), (0.9, 0.9)) for i in range(self.n_points)])

    def obs_dim(self, world):
        return 4 + 2 * self.n_points + 2 * (self.n_agents - 1)

    def template_pairs(self, world):
        n = self.n_agents
        return [(i, j) for i in range(n) for j in range(i + 1, n)]

    def template_ok(self, world):
        e = world.entities
        n = self.n_agents
        return (len(e) == n + self.n_points
                and all(isinstance(a.shape, Sphere) and a.movable and not a.rotatable for a in e[:n])
                and len({a.shape.radius for a in e[:n]}) == 1
                and not any(p.movable for p in e[n:]) and n <= 128 and self.n_points <= 128)

    def fill_constants(self, world, d):
        r = world.entities[0].shape.radius
        d.sc[0] = f32(r + r)
        d.sc[1] = f32(self.cover_dist)
        d.sc[2] = sqrt_le_bound(d.sc[0])
        d.sc[3] = sqrt_le_bound(d.sc[1])
        d.si[0] = int(self.quorum)
        lo = np.asarray((-0.9, -0.9), dtype=np.float64)
        hi = np.asarray((0.9, 0.9), dtype=np.float64)
        d.sd[0], d.sd[1] = float(lo[0]), float(lo[1])
        d.sd[2], d.sd[3] = float(hi[0] - lo[0]), float(hi[1] - lo[1])

    @property
    def covered_now(self) -> torch.Tensor:
        w = self._world() if self._world else None
        return None if w is None else unpack_bits(w.flags, self.n_points)

    def heuristic_action(self, agent_index: int, obs):
        point_idx = (agent_index // 2) % self.n_points
        target = obs[:, 4 + 2 * point_idx: 6 + 2 * point_idx]
        return clip_unit(4.0 * target)
