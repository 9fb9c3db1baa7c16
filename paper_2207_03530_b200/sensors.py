"""Range sensors (swarmsim/sensors.py): float64 ray casts on the device.

lidar_scan runs the library's lidar kernel (one thread per (env, ray)),
cast_ray its single-ray kernel.  Intersections are float64 as in the
reference; results are cast to float32.  For rays whose angle does not
depend on the emitter's rotation (rot == 0) the direction cosines are the
host's numpy values, so the device sees exactly the reference's directions.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .batching import Vec2, as_f32
from .core import Agent, World

RAY_EPS = 1e-9


@dataclass(frozen=True)
class Lidar:
    """A fan of rays (sensors.py:21-40): ray m at start + m*(end-start)/n (+ rot)."""

    n_rays: int = 12
    max_range: float = 1.0
    start_angle: float = 0.0
    end_angle: float = 2 * np.pi
    attach_rotation: bool = True

    def __post_init__(self):
        if self.n_rays < 1:
            raise ValueError(f"n_rays must be >= 1, got {self.n_rays}")
        if self.max_range <= 0:
            raise ValueError(f"max_range must be positive, got {self.max_range}")

    def base_angles(self) -> np.ndarray:
        span = self.end_angle - self.start_angle
        return np.array([self.start_angle + m * span / self.n_rays for m in range(self.n_rays)],
                        dtype=np.float64)

    def direction_table(self) -> np.ndarray:
        """(n_rays, 2) float64 numpy cos/sin of the rot == 0 ray angles."""
        a = self.base_angles()
        return np.stack([np.cos(a + 0.0), np.sin(a + 0.0)], axis=1)


def _physics_handle(world: World):
    from .dynamics import physics_world

    return physics_world(world)


def lidar_scan(agent: Agent, lidar: Lidar, world: World) -> torch.Tensor:
    """(B, n_rays) float32 ranges for one agent's lidar, self excluded."""
    h = _physics_handle(world)
    dev = world.device
    table = torch.from_numpy(lidar.direction_table()).to(dev).contiguous()
    desc = N.SsLidarDesc()
    desc.n_rays = lidar.n_rays
    desc.max_range = float(lidar.max_range)
    desc.start_angle = float(lidar.start_angle)
    desc.span = float(lidar.end_angle - lidar.start_angle)
    desc.attach_rotation = int(lidar.attach_rotation)
    desc.dir_table = N.ptr(table)
    out = torch.empty((world.batch_size, lidar.n_rays), device=dev)
    buf = world.buffers()
    N.check(N.lib().ss_lidar(h.handle, ctypes.byref(buf), world.index_of(agent), ctypes.byref(desc),
                             N.ptr(out), N.stream_handle(dev)))
    return out


def cast_ray(origin: Vec2, angle, world: World, max_range: float, exclude: str | None = None) -> torch.Tensor:
    """Distance to the nearest collidable entity along one ray per env (sensors.py:113-135)."""
    h = _physics_handle(world)
    dev = world.device
    B = world.batch_size
    ox = origin.x.to(dev).contiguous()
    oy = origin.y.to(dev).contiguous()
    ang = torch.as_tensor(np.asarray(angle.cpu() if isinstance(angle, torch.Tensor) else angle, dtype=np.float64))
    ang = ang.reshape(-1).expand(B).contiguous().to(dev)
    skip = -1
    if exclude is not None:
        names = [e.name for e in world.entities]
        skip = names.index(exclude) if exclude in names else -1
    out = torch.empty(B, device=dev)
    buf = world.buffers()
    N.check(N.lib().ss_cast_ray(h.handle, ctypes.byref(buf), skip, N.ptr(ox), N.ptr(oy), N.ptr(ang),
                                float(max_range), N.ptr(out), N.stream_handle(dev)))
    return out
