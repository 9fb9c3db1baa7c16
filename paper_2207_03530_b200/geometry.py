"""Closest points between posed shapes (swarmsim/geometry.py:120-163).

The batched query runs in the library's closest-point kernel — the same
device code the fused steps and the generic world_step use — one thread per
environment.  Supported: all six sphere/box/line pairs in either order.
"""
from __future__ import annotations

import torch

from . import _native as N
from .batching import Vec2, as_f32
from .errors import UnsupportedShapePair
from .shapes import Shape, native_shape


def _pos2(v: Vec2) -> torch.Tensor:
    return torch.stack([v.x, v.y], dim=1).contiguous()


def closest_points(pos_i: Vec2, rot_i, shape_i: Shape, pos_j: Vec2, rot_j, shape_j: Shape):
    """Per-env closest points (p_i, p_j); raises UnsupportedShapePair."""
    si, sj = native_shape(shape_i), native_shape(shape_j)
    if si is None or sj is None:
        raise UnsupportedShapePair(
            f"no closest-point routine for {type(shape_i).__name__}-{type(shape_j).__name__}"
        )
    dev = pos_i.device
    n = pos_i.batch_size
    pi, pj = _pos2(pos_i), _pos2(pos_j.copy() if pos_j.device == dev else Vec2(pos_j.x.to(dev), pos_j.y.to(dev)))
    ri = as_f32(rot_i, dev).reshape(-1).expand(n).contiguous()
    rj = as_f32(rot_j, dev).reshape(-1).expand(n).contiguous()
    oi = torch.empty((n, 2), device=dev)
    oj = torch.empty((n, 2), device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    N.check(N.lib().ss_closest_points(
        N.ptr(pi), N.ptr(ri), si[0], si[1], si[2], N.ptr(pj), N.ptr(rj), sj[0], sj[1], sj[2],
        N.ptr(oi), N.ptr(oj), n, N.ptr(status), N.stream_handle(dev)))
    return Vec2(oi[:, 0], oi[:, 1]), Vec2(oj[:, 0], oj[:, 1])
