"""flocking (swarmsim/scenarios/flocking.py): gather at a beacon among rocks.

Fused kernel: k_flocking<n> (csrc/ss_small.cu).  Reward per agent
(flocking.py:52-57): -|self - beacon| - penalty * (#agents touching +
#rocks touching), float32.  Observation (:59-68): [x, y, vx, vy,
beacon - self, rock_i - self, other - self].

Extension (BASELINE config 4, no reference counterpart): `lidar=Lidar(...)`
attaches the sensor to every agent and appends lidar_scan(agent) — fp64 rays
against the other agents and the rocks, exactly sensors.lidar_scan — to the
observation, computed inside the same fused launch.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .. import _native as N
from .._numerics import sqrt_le_bound
from ..core import Agent, Entity, World
from ..sensors import Lidar
from ..shapes import Sphere, min_contact_distance
from . import register
from ._fused import FusedScenario, f32
from .common import clip_unit, marker, unit


@register("flocking")
class Flocking(FusedScenario):
    native_id = N.SCN_FLOCKING
    max_steps = 200

    def __init__(self, n_agents: int = 4, n_obstacles: int = 3, collision_penalty: float = 3.0,
                 lidar: Lidar | None = None, lidar_rays: int = 0):
        self.n_agents = n_agents
        self.n_obstacles = n_obstacles
        self.collision_penalty = collision_penalty
        if lidar is None and lidar_rays:
            lidar = Lidar(n_rays=lidar_rays, max_range=1.0)
        self.lidar = lidar

    def make_world(self, batch_size: int, rng) -> World:
        world = World(batch_size, rng=rng, device=getattr(rng, "device", None))
        sensors = [self.lidar] if self.lidar is not None else None
        for i in range(self.n_agents):
            world.add(Agent(f"agent_{i}", shape=Sphere(radius=0.05), sensors=sensors))
        world.add(marker("beacon", radius=0.06, color=(0.9, 0.3, 0.6)))
        for i in range(self.n_obstacles):
            world.add(Entity(f"rock_{i}", shape=Sphere(radius=0.1), movable=False, color=(0.4, 0.4, 0.45)))
        return world

    def reset_ops(self, world):
        n = self.n_agents
        return ([(k, "scatter", (-1.0, -1.0), (1.0, 1.0)) for k in range(n)]
                + [(n, "scatter", (-0.5, -0.5), (0.5, 0.5))]
                + [(n + 1 + i, "scatter", (-0.8, -0.8), (0.8, 0.8)) for i in range(self.n_obstacles)])

    def obs_dim(self, world):
        rays = self.lidar.n_rays if self.lidar is not None else 0
        return 6 + 2 * self.n_obstacles + 2 * (self.n_agents - 1) + rays

    def template_pairs(self, world):
        n = self.n_agents
        out = []
        for i in range(n):
            out += [(i, j) for j in range(i + 1, n)]
            out += [(i, n + 1 + r) for r in range(self.n_obstacles)]
        return out

    def template_ok(self, world):
        n, no = self.n_agents, self.n_obstacles
        e = world.entities
        agents, beacon, rocks = e[:n], e[n], e[n + 1:]
        return (len(e) == n + 1 + no
                and all(isinstance(a.shape, Sphere) and a.movable and not a.rotatable and a.collidable for a in agents)
                and len({a.shape.radius for a in agents}) == 1
                and not beacon.movable and not beacon.collidable
                and all(isinstance(r.shape, Sphere) and not r.movable and r.collidable for r in rocks)
                and len({r.shape.radius for r in rocks}) <= 1)

    def fill_constants(self, world, d):
        n = self.n_agents
        e = world.entities
        a0 = e[0]
        rock = e[n + 1] if self.n_obstacles else None
        d.sc[0] = f32(min_contact_distance(a0.shape, a0.shape) + 0.0)
        d.sc[1] = f32(min_contact_distance(a0.shape, rock.shape) + 0.0) if rock else 0.0
        d.sc[2] = f32(self.collision_penalty)
        d.sc[3] = sqrt_le_bound(d.sc[0])
        d.sc[4] = sqrt_le_bound(d.sc[1]) if rock else -1.0
        # contact constants of the warp-per-agent kernel (pair table values)
        d.sc[5] = f32(min_contact_distance(a0.shape, a0.shape))
        d.sc[6] = sqrt_le_bound(d.sc[5])
        d.sc[7] = f32(min_contact_distance(a0.shape, rock.shape)) if rock else 0.0
        d.sc[8] = sqrt_le_bound(d.sc[7]) if rock else -1.0
        d.si[4] = self.n_obstacles
        d.sd[0] = a0.shape.radius * a0.shape.radius
        d.sd[1] = rock.shape.radius * rock.shape.radius if rock else 0.0
        d.sd[2] = a0.shape.radius
        d.sd[3] = rock.shape.radius if rock else 0.0
        if self.lidar is not None:
            lid = self.lidar
            table = np.ascontiguousarray(lid.direction_table(), dtype=np.float64)
            d.lidar_rays = lid.n_rays
            d.lidar_attach_rotation = int(lid.attach_rotation)
            d.lidar_max_range = float(lid.max_range)
            d.lidar_start = float(lid.start_angle)
            d.lidar_span = float(lid.end_angle - lid.start_angle)
            d.lidar_dirs = table.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            d._keep = (d._keep, table)

    def heuristic_action(self, agent_index: int, obs):
        obs = obs.cpu().numpy() if hasattr(obs, "cpu") else np.asarray(obs)
        force = 1.5 * obs[:, 4:6]
        base = 6
        for k in range(self.n_obstacles):
            force = force + self._repulse(obs[:, base + 2 * k: base + 2 * k + 2], 0.3, 6.0)
        base = 6 + 2 * self.n_obstacles
        for k in range(self.n_agents - 1):
            force = force + self._repulse(obs[:, base + 2 * k: base + 2 * k + 2], 0.18, 4.0)
        return clip_unit(force)

    @staticmethod
    def _repulse(rel, reach: float, strength: float):
        d = np.linalg.norm(rel, axis=1, keepdims=True)
        return -unit(rel) * (np.maximum(0.0, reach - d) * strength)
