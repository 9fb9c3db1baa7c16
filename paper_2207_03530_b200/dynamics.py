"""Batched rigid-body dynamics (swarmsim/dynamics.py).

world_step(world, actions) runs one physics tick for every env in the
library's generic step kernel (any entity count, any sphere/box/line pair
list, torques for rotatable bodies).  The built-in scenarios do not come
through here: their whole Env.step is one fused launch (env.py).
collision_force is the same device routine the kernels use; integrate is
the reference's semi-implicit Euler written with separately rounded
float32 tensor ops.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .batching import Vec2, clamp_norm
from .core import Agent, AgentAction, Entity, PhysParams, World
from .errors import ContractViolation

DEGENERATE_DIST = 1e-8   # dynamics.py:23


@dataclass
class ContactResult:
    force_i: Vec2
    point_i: Vec2
    point_j: Vec2
    active: torch.Tensor


def collision_force(p_i: Vec2, p_j: Vec2, d_min: float, params: PhysParams,
                    fallback_sign: float = 1.0) -> ContactResult:
    """Penalty force on i from j (dynamics.py:36-66, Eq. 2)."""
    dev = p_i.device
    n = p_i.batch_size
    pix, piy = p_i.x.contiguous(), p_i.y.contiguous()
    pjx, pjy = p_j.x.to(dev).contiguous(), p_j.y.to(dev).contiguous()
    fx = torch.empty(n, device=dev)
    fy = torch.empty(n, device=dev)
    active = torch.empty(n, dtype=torch.bool, device=dev)
    N.check(N.lib().ss_collision_force(
        N.ptr(pix), N.ptr(piy), N.ptr(pjx), N.ptr(pjy), np.float32(d_min), np.float32(fallback_sign),
        np.float32(params.contact_force * params.contact_margin), np.float32(params.contact_margin),
        N.ptr(fx), N.ptr(fy), N.ptr(active), n, N.stream_handle(dev)))
    return ContactResult(force_i=Vec2(fx, fy), point_i=p_i, point_j=p_j, active=active)


def integrate(entity: Entity, force: Vec2, torque, params: PhysParams) -> None:
    """Velocity first, then position (dynamics.py:69-86)."""
    st = entity.state
    dt = float(np.float32(params.dt))
    keep = float(np.float32(1.0 - params.damping))
    if entity.movable:
        g = float(np.float32(np.float32(1.0 / entity.mass) * np.float32(dt)))
        vel = st.vel * keep + Vec2(force.x.to(st.vel.device), force.y.to(st.vel.device)) * g
        if entity.max_speed is not None:
            vel = clamp_norm(vel, entity.max_speed)
        st.vel = vel
        st.pos = st.pos + vel * dt
    if entity.rotatable:
        g = float(np.float32(np.float32(1.0 / entity.moment_of_inertia) * np.float32(dt)))
        tq = torch.as_tensor(torque, dtype=torch.float32, device=st.rot.device)
        w = st.ang_vel * keep + tq * g
        st.ang_vel = w
        st.rot = st.rot + w * dt


def _validate_action(agent: Agent, action: AgentAction, B: int, check_nan: bool = True) -> None:
    """dynamics.py:103-120 (check_nan=False: Env(validate=False), no host sync)."""
    if action.force.batch_size != B:
        raise ContractViolation(
            f"action for '{agent.name}' has batch size {action.force.batch_size}, world has {B}")
    if check_nan and bool(torch.isnan(action.force.x).any() | torch.isnan(action.force.y).any()):
        raise ContractViolation(f"action for '{agent.name}' contains NaN")
    if action.comm is not None:
        if agent.silent:
            raise ContractViolation(f"agent '{agent.name}' is silent but got a comm vector")
        comm = torch.as_tensor(action.comm)
        if tuple(comm.shape) != (B, agent.comm_dim):
            raise ContractViolation(
                f"comm for '{agent.name}' has shape {tuple(comm.shape)}, expected {(B, agent.comm_dim)}")
        if bool(torch.isnan(comm.float()).any()):
            raise ContractViolation(f"comm for '{agent.name}' contains NaN")


def physics_world(world: World):
    """SsWorld handle for the generic physics kernel of this world version."""
    return world.native(("physics", world.version), lambda: world.base_desc())


def run_world_step(world: World, forces: list, decode_mask: int, count: bool, stream=None,
                   guard=None, guard_count: int = 1) -> None:
    """Launch the generic step kernel.

    forces[a]: agent a's (B, 2) f32 device tensor, or its data pointer (int).
    decode_mask bit a: apply decode_action's clip * u_multiplier on device.
    guard: optional int32 device flags from ss_check_actions (guard_count
    words); any nonzero word (a NaN action) turns the launch into a no-op
    (env.py:85: nothing moves).
    """
    h = physics_world(world)
    ptrs = (ctypes.c_void_p * max(1, len(forces)))()
    for i, f in enumerate(forces):
        ptrs[i] = f if isinstance(f, int) else (None if f is None else f.data_ptr())
    mask = (ctypes.c_uint64 * 4)(*[(decode_mask >> (64 * i)) & (2**64 - 1) for i in range(4)])
    status = torch.zeros(1, dtype=torch.int32, device=world.device)
    st = stream if stream is not None else N.stream_handle(world.device)
    N.check(N.lib().ss_world_step(h.handle, world.buffers_ref(), ptrs, mask, int(count), N.ptr(guard),
                                  int(guard_count), N.ptr(status), st))


def world_step(world: World, actions: list) -> None:
    """One physics tick for every env (dynamics.py:123-184)."""
    agents = world.agents
    if len(actions) != len(agents):
        raise ContractViolation(f"got {len(actions)} actions for {len(agents)} agents")
    B = world.batch_size
    forces = []
    for agent, action in zip(agents, actions):
        if agent.action_script is not None:
            action = agent.action_script(agent, world)
        if action is None:
            raise ContractViolation(f"agent '{agent.name}' has no script and got no action")
        _validate_action(agent, action, B)
        agent.action = action
        if not agent.silent and action.comm is not None:
            world.comm[agent.name] = action.comm
        f = torch.stack([action.force.x, action.force.y], dim=1).to(world.device, torch.float32).contiguous()
        forces.append(f)
    run_world_step(world, forces, decode_mask=0, count=False)
