"""Frame snapshots of one env for viewers (swarmsim/viewer.py:29-63).

snapshot_from_env reads the viewed env's column of the device state with ONE
gather + one device->host copy (positions, rotations, step count) instead of
a scalar read per entity.  The websocket session/server of the reference
(viewer.py:66-213) is UI plumbing outside the hot path and is not rebuilt.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

import torch

from .env import Env
from .errors import ContractViolation


@dataclass
class FrameSnapshot:
    t: int
    env: int
    entities: list[dict]
    hud: dict = field(default_factory=dict)


def snapshot_from_env(env: Env, view_env: int, hud: dict | None = None) -> FrameSnapshot:
    """Entities in world order: name, shape descriptor, pos, rot, color."""
    B = env.batch_size
    if not (-B <= int(view_env) < B):
        raise ContractViolation(f"env index {view_env} out of range for batch {B}")
    e = int(view_env) % B
    w = env.world
    st = w.state_array()[:, [0, 1, 4], e]                       # (E, 3) on device
    packed = torch.cat([st.reshape(-1).to(torch.float64), env.step_count[e:e + 1].to(torch.float64)])
    host = packed.cpu().tolist()
    entities = []
    for k, ent in enumerate(w.entities):
        x, y, r = host[3 * k:3 * k + 3]
        entities.append({"name": ent.name, "shape": ent.shape.descriptor(), "pos": [x, y], "rot": r,
                         "color": [float(c) for c in ent.color]})
    return FrameSnapshot(t=int(host[-1]), env=int(view_env), entities=entities, hud=hud or {})


def encode_frame(snap: FrameSnapshot) -> str:
    """The reference wire format (viewer.py:52-63)."""
    return json.dumps({"type": "frame", "t": snap.t, "env": snap.env, "entities": snap.entities,
                       "hud": snap.hud})


__all__ = ["FrameSnapshot", "snapshot_from_env", "encode_frame"]
