"""dispersion (swarmsim/scenarios/dispersion.py): fan out from the origin to eat food.

Fused kernel: k_dispersion<T> (csrc/ss_large.cu, one warp per env).  Agents
are non-collidable, so the step has no pair forces.  post_step latches
"eaten" for every item some agent is within eat_dist of (dispersion.py:
56-66); the shared reward is fresh_bites - 0.05 * (sum over uneaten items
of the nearest-agent distance, float64); done when everything is eaten.
Observation (:81-87): [x, y, vx, vy, (food_i - self, eaten_i)].

The eaten flags live on the device as bit words (flags buffer); `eaten`
and `fresh_bites` below are host-side views of them.
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
from .common import clip_unit, marker, place


@register("dispersion")
class Dispersion(FusedScenario):
    native_id = N.SCN_DISPERSION
    max_steps = 200

    def __init__(self, n_agents: int = 4, n_food: int = 4, eat_dist: float = 0.15):
        self.n_agents = n_agents
        self.n_food = n_food
        self.eat_dist = eat_dist
        self._world = None

    def make_world(self, batch_size: int, rng) -> World:
        world = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        for i in range(self.n_agents):
            world.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05), collidable=False))
        for i in range(self.n_food):
            world.add(marker(f"food_{i}", radius=0.08, color=(0.9, 0.6, 0.15)))
        world.ensure_flag_words(self.n_flag_words())
        self._world = weakref.ref(world)
        return world

    def n_flag_words(self) -> int:
        return (self.n_food + 31) // 32

    def reset_ops(self, world):
        return ([(k, "place", (0.0, 0.0), None) for k in range(self.n_agents)]
                + [(self.n_agents + i, "scatter", (-1.0, -1.0), (1.0, 1.0)) for i in range(self.n_food)])

    def obs_dim(self, world):
        return 4 + 3 * self.n_food

    def template_pairs(self, world):
        return []

    def template_ok(self, world):
        e = world.entities
        n = self.n_agents
        return (len(e) == n + self.n_food and all(a.movable and not a.rotatable for a in e[:n])
                and not any(f.movable for f in e[n:]) and n <= 128 and self.n_food <= 128)

    def fill_constants(self, world, d):
        d.sc[1] = f32(self.eat_dist)
        d.sc[3] = sqrt_le_bound(d.sc[1])

    # reference aux state, read back from the device
    @property
    def eaten(self) -> torch.Tensor:
        w = self._world() if self._world else None
        if w is None:
            return None
        return unpack_bits(w.flags, self.n_food)

    @property
    def fresh_bites(self) -> torch.Tensor:
        w = self._world() if self._world else None
        return None if w is None else w.aux.to(torch.float64)

    def heuristic_action(self, agent_index: int, obs):
        obs = obs.cpu().numpy() if hasattr(obs, "cpu") else np.asarray(obs)
        B = obs.shape[0]
        rels = np.stack([obs[:, 4 + 3 * i: 6 + 3 * i] for i in range(self.n_food)], axis=1)
        eaten = np.stack([obs[:, 6 + 3 * i] for i in range(self.n_food)], axis=1) > 0.5
        dist = np.where(eaten, np.inf, np.linalg.norm(rels, axis=2))
        order = np.argsort(dist, axis=1, kind="stable")
        remaining = np.maximum((~eaten).sum(axis=1), 1)
        pick = order[np.arange(B), np.minimum(agent_index, remaining - 1)]
        return clip_unit(5.0 * rels[np.arange(B), pick])


def unpack_bits(flags: torch.Tensor, n: int) -> torch.Tensor:
    """(W, B) int32 bit words -> (B, n) bool."""
    bits = torch.arange(32, device=flags.device, dtype=torch.int32)
    out = ((flags[:, :, None] >> bits) & 1).to(torch.bool)           # (W, B, 32)
    return out.permute(1, 0, 2).reshape(flags.shape[1], -1)[:, :n]
