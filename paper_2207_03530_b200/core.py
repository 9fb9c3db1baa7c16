"""Entities, agents, physics parameters and the device-resident World.

Mirrors swarmsim/core.py (PhysParams :20-44, EntityState :47-117,
Entity :120-152, AgentAction :155-160, Agent :163-198, World :201-265), with
the state held on the GPU in the layout the kernels stream:

    dyn      (n_dyn,  B, 4) f32   px py vx vy   — movable entities
    stat     (n_stat, B, 2) f32   px py         — non-movable entities
    stat_vel (n_stat, B, 2) f32   vx vy         — (never read by a kernel)
    rot      (E,      B, 2) f32   rot ang_vel

Each row is one entity with the env index contiguous, so a warp touching 32
consecutive envs moves one contiguous 512 B (dyn) / 256 B (stat) span.
EntityState.pos / vel / rot / ang_vel are strided torch views into these
buffers: in-place edits (state.pos.x[e] = ..) write straight to the device.
"""
from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _native as N
from ._numerics import sqrt_le_bound
from .batching import DeviceRng, SeededRng, Vec2, as_f32, default_device, scalars
from .errors import ContractViolation, UnsupportedShapePair
from .shapes import Shape, Sphere, min_contact_distance, native_shape


@dataclass
class PhysParams:
    """World constants (core.py:20-44): dt, damping, gravity, contact c and k.

    substeps (extension, default 1 = the reference): physics sub-steps per
    Env.step.  Each sub-step re-evaluates every contact / joint force on the
    current state and integrates with the sub-step dt f32(dt / substeps),
    keeping damping per sub-step (VMAS semantics); actions and scripts are
    decoded once per step and held, post_step / rewards / dones /
    observations run once after the last sub-step.  One step with substeps=k
    equals k reference world_step calls with PhysParams(dt=dt/k) on the same
    decoded actions (tests/test_gpu_physics.py pins it that way).
    """

    dt: float = 0.1
    damping: float = 0.25
    gravity: tuple = (0.0, 0.0)
    contact_force: float = 100.0
    contact_margin: float = 1e-3
    substeps: int = 1

    @property
    def sub_dt(self) -> float:
        """The integrator's dt: dt / substeps (python double, cast at use)."""
        return self.dt / self.substeps if self.substeps != 1 else self.dt

    def __post_init__(self):
        if int(self.substeps) != self.substeps or not 1 <= self.substeps <= 1024:
            raise ContractViolation(f"substeps must be an integer in [1, 1024], got {self.substeps}")
        self.substeps = int(self.substeps)
        if not self.dt > 0:
            raise ContractViolation(f"dt must be positive, got {self.dt}")
        if not 0 <= self.damping < 1:
            raise ContractViolation(f"damping must be in [0, 1), got {self.damping}")
        if self.contact_force < 0:
            raise ContractViolation("contact_force must be non-negative")
        if not self.contact_margin > 0:
            raise ContractViolation("contact_margin must be positive")


class EntityState:
    """Batched pose/velocity of one entity: views into its World's buffers."""

    __slots__ = ("_world", "_entity")

    def __init__(self, world: "World", entity: "Entity"):
        self._world = world
        self._entity = entity

    # -- raw views -----------------------------------------------------------
    def _rows(self):
        return self._world._rows_of(self._entity)

    @property
    def batch_size(self) -> int:
        return self._world.batch_size

    @property
    def pos(self) -> Vec2:
        p, _, _ = self._rows()
        return Vec2(p[:, 0], p[:, 1])

    @pos.setter
    def pos(self, v: Vec2) -> None:
        p, _, _ = self._rows()
        p[:, 0].copy_(_vec_x(v, self.batch_size))
        p[:, 1].copy_(_vec_y(v, self.batch_size))

    @property
    def vel(self) -> Vec2:
        _, v, _ = self._rows()
        return Vec2(v[:, 0], v[:, 1])

    @vel.setter
    def vel(self, v: Vec2) -> None:
        _, w, _ = self._rows()
        w[:, 0].copy_(_vec_x(v, self.batch_size))
        w[:, 1].copy_(_vec_y(v, self.batch_size))

    @property
    def rot(self) -> torch.Tensor:
        return self._rows()[2][:, 0]

    @rot.setter
    def rot(self, r) -> None:
        self._rows()[2][:, 0].copy_(scalars(r, self.batch_size, self._world.device))

    @property
    def ang_vel(self) -> torch.Tensor:
        return self._rows()[2][:, 1]

    @ang_vel.setter
    def ang_vel(self, w) -> None:
        self._rows()[2][:, 1].copy_(scalars(w, self.batch_size, self._world.device))

    # -- reference mutators (core.py:63-117) ---------------------------------
    def set_pos(self, pos: Vec2, env_index: int | None = None) -> None:
        if env_index is None:
            self.pos = pos
        else:
            p = self._rows()[0]
            p[env_index, 0] = pos.x[0]
            p[env_index, 1] = pos.y[0]

    def set_pos_xy(self, x, y, env_index: int | None = None) -> None:
        self.set_pos(Vec2(as_f32(x, self._world.device).reshape(-1), as_f32(y, self._world.device).reshape(-1)), env_index)

    def set_vel(self, vel: Vec2, env_index: int | None = None) -> None:
        if env_index is None:
            self.vel = vel
        else:
            v = self._rows()[1]
            v[env_index, 0] = vel.x[0]
            v[env_index, 1] = vel.y[0]

    def set_rot(self, rot, env_index: int | None = None) -> None:
        if env_index is None:
            self.rot = rot
        else:
            self._rows()[2][env_index, 0] = float(np.asarray(as_f32(rot).cpu()).reshape(-1)[0])

    def set_ang_vel(self, ang_vel, env_index: int | None = None) -> None:
        if env_index is None:
            self.ang_vel = ang_vel
        else:
            self._rows()[2][env_index, 1] = float(np.asarray(as_f32(ang_vel).cpu()).reshape(-1)[0])

    def zero_motion(self, env_index: int | None = None) -> None:
        _, v, r = self._rows()
        if env_index is None:
            v.zero_()
            r[:, 1].zero_()
        else:
            v[env_index] = 0.0
            r[env_index, 1] = 0.0

    def snapshot(self, env_index: int) -> dict:
        p, v, r = self._rows()
        vals = torch.stack([p[env_index, 0], p[env_index, 1], v[env_index, 0], v[env_index, 1],
                            r[env_index, 0], r[env_index, 1]]).cpu().numpy()
        return {"pos": (float(vals[0]), float(vals[1])), "vel": (float(vals[2]), float(vals[3])),
                "rot": float(vals[4]), "ang_vel": float(vals[5])}

    def restore(self, env_index: int, snap: dict) -> None:
        p, v, r = self._rows()
        vals = torch.tensor([*snap["pos"], *snap["vel"], snap["rot"], snap["ang_vel"]],
                            dtype=torch.float32, device=p.device)
        p[env_index] = vals[0:2]
        v[env_index] = vals[2:4]
        r[env_index] = vals[4:6]


def _vec_x(v, B):
    return scalars(v.x, B) if isinstance(v, Vec2) else scalars(as_f32(v)[:, 0], B)


def _vec_y(v, B):
    return scalars(v.y, B) if isinstance(v, Vec2) else scalars(as_f32(v)[:, 1], B)


# attributes whose change invalidates the World's native descriptor
_PHYS_ATTRS = frozenset({"shape", "mass", "moment_of_inertia", "movable", "rotatable", "collidable",
                         "max_speed", "u_range", "u_multiplier"})


class Entity:
    """A simulated body (core.py:120-152)."""

    def __init__(
        self,
        name: str,
        shape: Shape | None = None,
        mass: float = 1.0,
        moment_of_inertia: float | None = None,
        movable: bool = False,
        rotatable: bool = False,
        collidable: bool = True,
        max_speed: float | None = None,
        color: tuple = (0.35, 0.35, 0.35),
    ):
        if not mass > 0:
            raise ContractViolation(f"mass must be positive, got {mass}")
        self._world_ref = None
        self.name = name
        self.shape = shape if shape is not None else Sphere()
        self.mass = float(mass)
        moi = moment_of_inertia if moment_of_inertia is not None else self.shape.moment_of_inertia(mass)
        if not moi > 0:
            raise ContractViolation(f"moment of inertia must be positive, got {moi}")
        self.moment_of_inertia = float(moi)
        self.movable = movable
        self.rotatable = rotatable
        self.collidable = collidable
        self.max_speed = max_speed
        self.color = color
        self.state: EntityState | None = None

    def __setattr__(self, key, value):
        object.__setattr__(self, key, value)
        if key in _PHYS_ATTRS:
            ref = self.__dict__.get("_world_ref")
            w = ref() if ref is not None else None
            if w is not None:
                w._touch(relayout=(key == "movable"))

    def __repr__(self) -> str:
        return f"{type(self).__name__}({self.name!r})"


@dataclass
class AgentAction:
    """Decoded per-step command (core.py:155-160): batched force + optional comm."""

    force: Vec2
    comm: Optional[torch.Tensor] = None


class Agent(Entity):
    """A controllable entity (core.py:163-198)."""

    def __init__(
        self,
        name: str,
        shape: Shape | None = None,
        mass: float = 1.0,
        u_range: float = 1.0,
        u_multiplier: float = 1.0,
        silent: bool = True,
        comm_dim: int = 0,
        action_noise_std: float = 0.0,
        obs_noise_std: float = 0.0,
        max_speed: float | None = None,
        sensors: list | None = None,
        action_script: Callable | None = None,
        color: tuple = (0.25, 0.45, 0.85),
        **kwargs,
    ):
        kwargs.setdefault("movable", True)
        kwargs.setdefault("rotatable", False)
        super().__init__(name, shape=shape, mass=mass, max_speed=max_speed, color=color, **kwargs)
        if not u_range > 0:
            raise ContractViolation(f"u_range must be positive, got {u_range}")
        if comm_dim < 0:
            raise ContractViolation(f"comm_dim must be non-negative, got {comm_dim}")
        self.u_range = float(u_range)
        self.u_multiplier = float(u_multiplier)
        self.silent = silent
        self.comm_dim = 0 if silent else int(comm_dim)
        self.action_noise_std = float(action_noise_std)
        self.obs_noise_std = float(obs_noise_std)
        self.sensors = sensors or []
        self.action_script = action_script
        self.action: AgentAction | None = None


Landmark = Entity   # VMAS vocabulary: a non-agent entity


class Joint:
    """Distance joint between two entities (extension: the reference has no
    joints; VMAS-style penalty constraint, off unless added).

    Anchors are body-frame offsets normalised to the entity's extent, as in
    VMAS: anchor (1, 0) is the +x tip of a line / box half length (or the
    sphere's radius).  The joint holds the anchors at `dist` apart with a
    softplus penalty of multiplier `stiffness` (default 130, VMAS's
    joint_force): attractive when stretched, repulsive when compressed.
    rotate_a / rotate_b apply its torque to rotatable ends.  Exact arithmetic:
    include/swarmsim_b200.h SsJointDesc; parity is pinned to the numpy
    restatement oracle/swarm_oracle.py joint_forces (unpinned by the reference).
    """

    def __init__(self, entity_a: "Entity", entity_b: "Entity", anchor_a=(0.0, 0.0), anchor_b=(0.0, 0.0),
                 dist: float = 0.0, stiffness: float = 130.0, rotate_a: bool = True, rotate_b: bool = True):
        if entity_a is entity_b:
            raise ContractViolation("a joint needs two distinct entities")
        if not dist >= 0.0:
            raise ContractViolation(f"joint dist must be non-negative, got {dist}")
        if not stiffness >= 0.0:
            raise ContractViolation(f"joint stiffness must be non-negative, got {stiffness}")
        self.entity_a, self.entity_b = entity_a, entity_b
        self.anchor_a = (float(anchor_a[0]), float(anchor_a[1]))
        self.anchor_b = (float(anchor_b[0]), float(anchor_b[1]))
        self.dist = float(dist)
        self.stiffness = float(stiffness)
        self.rotate_a, self.rotate_b = bool(rotate_a), bool(rotate_b)

    @staticmethod
    def offset(entity: "Entity", anchor) -> tuple:
        """Body-frame offset of a normalised anchor (float32): extent * anchor."""
        from .shapes import Box, Line

        sh = entity.shape
        if isinstance(sh, Box):
            hx, hy = sh.length / 2, sh.width / 2
        elif isinstance(sh, Line):
            hx, hy = sh.length / 2, 0.0
        else:
            hx = hy = sh.radius
        return np.float32(anchor[0] * hx), np.float32(anchor[1] * hy)


def _collidable_pairs(world: "World") -> list[tuple[int, int]]:
    """Static pair list (dynamics.py:89-100): both collidable, one can move."""
    ents = world.entities
    out = []
    for i in range(len(ents)):
        for j in range(i + 1, len(ents)):
            a, b = ents[i], ents[j]
            if not (a.collidable and b.collidable):
                continue
            if not (a.movable or a.rotatable or b.movable or b.rotatable):
                continue
            out.append((i, j))
    return out


class World:
    """B parallel copies of one scene, state resident on the GPU (core.py:201-265)."""

    def __init__(self, batch_size: int, params: PhysParams | None = None, seed: int = 0,
                 rng: SeededRng | None = None, device=None):
        if batch_size < 1:
            raise ContractViolation(f"batch_size must be >= 1, got {batch_size}")
        self.batch_size = int(batch_size)
        self.device = torch.device(device) if device is not None else default_device()
        self._params = params if params is not None else PhysParams()
        self.rng = rng if rng is not None else SeededRng(seed)
        self.entities: list[Entity] = []
        self._names: set[str] = set()
        self._pairs: list[tuple[int, int]] | None = None
        self.comm: dict = {}
        self.joints: list[Joint] = []
        # sharding: this world holds global envs [env_offset, env_offset + B)
        self.env_offset = 0
        self.global_batch = self.batch_size
        self._slots: dict[int, tuple[bool, int]] = {}
        self._index: dict[int, int] = {}
        self.dyn = torch.zeros((0, self.batch_size, 4), device=self.device)
        self.stat = torch.zeros((0, self.batch_size, 2), device=self.device)
        self.stat_vel = torch.zeros((0, self.batch_size, 2), device=self.device)
        self.rot = torch.zeros((0, self.batch_size, 2), device=self.device)
        self.step_count = torch.zeros(self.batch_size, dtype=torch.int64, device=self.device)
        self.flags = torch.zeros((1, self.batch_size), dtype=torch.int32, device=self.device)
        self.aux = torch.zeros(self.batch_size, dtype=torch.float32, device=self.device)
        self.version = 0
        self.native_epoch = 0
        self._native_cache: dict = {}
        self._buf_cache = None

    @property
    def params(self) -> PhysParams:
        return self._params

    @params.setter
    def params(self, p: PhysParams) -> None:
        """Replace the physics constants (rebuilds the native descriptor)."""
        self._params = p
        if hasattr(self, "_native_cache"):
            self._touch()

    # -- entity bookkeeping ---------------------------------------------------
    @property
    def agents(self) -> list[Agent]:
        return [e for e in self.entities if isinstance(e, Agent)]

    @property
    def landmarks(self) -> list[Entity]:
        return [e for e in self.entities if not isinstance(e, Agent)]

    def add(self, entity: Entity) -> Entity:
        if entity.name in self._names:
            raise ContractViolation(f"duplicate entity name {entity.name!r}")
        if isinstance(entity, Agent):
            self.entities.insert(len(self.agents), entity)   # agents precede landmarks
        else:
            self.entities.append(entity)
        self._names.add(entity.name)
        entity._world_ref = weakref.ref(self)
        entity.state = EntityState(self, entity)
        self._relayout(new=entity)
        return entity

    def add_joint(self, joint: Joint) -> Joint:
        """Attach a joint constraint (extension; worlds with joints step their
        physics in the generic kernel)."""
        for e in (joint.entity_a, joint.entity_b):
            if id(e) not in self._index:
                raise ContractViolation(f"joint end {e.name!r} is not in this world")
        self.joints.append(joint)
        self._touch()
        return joint

    def entity(self, name: str) -> Entity:
        for e in self.entities:
            if e.name == name:
                return e
        raise KeyError(name)

    def index_of(self, entity: Entity) -> int:
        return self._index[id(entity)]

    def collidable_pairs(self, builder=_collidable_pairs) -> list[tuple[int, int]]:
        if self._pairs is None:
            self._pairs = builder(self)
        return self._pairs

    def _touch(self, relayout: bool = False) -> None:
        if relayout:
            self._relayout()
        else:
            self.version += 1
            self._pairs = None
            self._drop_native()

    def _rows_of(self, e: Entity):
        movable, slot = self._slots[id(e)]
        k = self._index[id(e)]
        if movable:
            row = self.dyn[slot]
            return row[:, 0:2], row[:, 2:4], self.rot[k]
        return self.stat[slot], self.stat_vel[slot], self.rot[k]

    def _relayout(self, new: Entity | None = None) -> None:
        """Re-derive row assignments after an add / movable change, keeping data."""
        old = {}
        for e in self.entities:
            if e is new or id(e) not in self._slots:
                continue
            p, v, r = self._rows_of(e)
            old[id(e)] = (p.clone(), v.clone(), r.clone())
        B, d = self.batch_size, self.device
        n_dyn = sum(1 for e in self.entities if e.movable)
        n_stat = len(self.entities) - n_dyn
        self.dyn = torch.zeros((n_dyn, B, 4), device=d)
        self.stat = torch.zeros((n_stat, B, 2), device=d)
        self.stat_vel = torch.zeros((n_stat, B, 2), device=d)
        self.rot = torch.zeros((len(self.entities), B, 2), device=d)
        self._slots.clear()
        self._index.clear()
        di = si = 0
        for k, e in enumerate(self.entities):
            self._index[id(e)] = k
            if e.movable:
                self._slots[id(e)] = (True, di)
                di += 1
            else:
                self._slots[id(e)] = (False, si)
                si += 1
        for e in self.entities:
            if id(e) in old:
                p, v, r = self._rows_of(e)
                op, ov, orr = old[id(e)]
                p.copy_(op)
                v.copy_(ov)
                r.copy_(orr)
        self.version += 1
        self._pairs = None
        self._drop_native()

    # -- per-env state access (core.py:259-265) ------------------------------
    def get_env_state(self, env_index: int) -> dict:
        return {e.name: e.state.snapshot(env_index) for e in self.entities}

    def set_env_state(self, env_index: int, state: dict) -> None:
        for name, snap in state.items():
            self.entity(name).state.restore(env_index, snap)

    def state_dict(self) -> dict:
        """Every device buffer (clone) — for checkpoints and teacher-forced tests."""
        return {"dyn": self.dyn.clone(), "stat": self.stat.clone(), "stat_vel": self.stat_vel.clone(),
                "rot": self.rot.clone(), "step_count": self.step_count.clone(),
                "flags": self.flags.clone(), "aux": self.aux.clone()}

    def load_state_dict(self, sd: dict) -> None:
        for k in ("dyn", "stat", "stat_vel", "rot", "step_count", "flags", "aux"):
            getattr(self, k).copy_(sd[k])

    def state_array(self) -> torch.Tensor:
        """(E, 6, B) f32: px py vx vy rot ang_vel for every entity, world order."""
        rows = []
        for e in self.entities:
            p, v, r = self._rows_of(e)
            rows.append(torch.stack([p[:, 0], p[:, 1], v[:, 0], v[:, 1], r[:, 0], r[:, 1]]))
        return torch.stack(rows)

    def load_state_array(self, arr) -> None:
        a = as_f32(arr, self.device)
        for k, e in enumerate(self.entities):
            p, v, r = self._rows_of(e)
            p.copy_(a[k, 0:2].T)
            v.copy_(a[k, 2:4].T)
            r.copy_(a[k, 4:6].T)

    # -- native descriptor ----------------------------------------------------
    def _drop_native(self) -> None:
        """Free every cached SsWorld.  Bumps native_epoch: a StepGraph captured
        before refuses to replay (its kernels hold the freed tables)."""
        for h in self._native_cache.values():
            h.close()
        self._native_cache.clear()
        self.native_epoch += 1

    def ensure_flag_words(self, n: int) -> None:
        if self.flags.shape[0] < max(1, n):
            self.flags = torch.zeros((max(1, n), self.batch_size), dtype=torch.int32, device=self.device)
            self._touch()

    def entity_descs(self):
        p = self.params
        dt = np.float32(p.sub_dt)
        gx, gy = p.gravity
        arr = (N.SsEntityDesc * max(1, len(self.entities)))()
        for k, e in enumerate(self.entities):
            sh = native_shape(e.shape)
            if sh is None:
                raise UnsupportedShapePair(f"no closest-point routine for shape {type(e.shape).__name__}")
            d = arr[k]
            d.shape, d.dim0, d.dim1 = sh
            d.movable, d.rotatable, d.collidable = int(e.movable), int(e.rotatable), int(e.collidable)
            d.is_agent = int(isinstance(e, Agent))
            d.slot = self._slots[id(e)][1]
            d.inv_m_dt = np.float32(np.float32(1.0 / e.mass) * dt)
            d.inv_i_dt = np.float32(np.float32(1.0 / e.moment_of_inertia) * dt)
            d.max_speed = np.float32(e.max_speed) if e.max_speed is not None else np.float32(-1.0)
            m = np.float32(e.mass)
            d.grav_x = np.float32(gx * m)
            d.grav_y = np.float32(gy * m)
            d.u_range = np.float32(getattr(e, "u_range", np.inf))
            d.u_mult = np.float32(getattr(e, "u_multiplier", 1.0))
        return arr

    def pair_descs(self):
        pairs = self.collidable_pairs(_collidable_pairs)
        arr = (N.SsPairDesc * max(1, len(pairs)))()
        for n, (i, j) in enumerate(pairs):
            arr[n].i, arr[n].j = i, j
            dmin = np.float32(min_contact_distance(self.entities[i].shape, self.entities[j].shape))
            arr[n].d_min = dmin
            arr[n].d2_act = sqrt_le_bound(dmin)
            arr[n].sign = 1.0 if (i + j) % 2 == 0 else -1.0
        return arr, len(pairs)

    def native(self, key, build: Callable[[], "N.SsWorldDesc"]) -> "NativeWorld":
        """Cached SsWorld for (version, key); build() returns a filled descriptor."""
        h = self._native_cache.get(key)
        if h is None:
            h = NativeWorld(build())
            self._native_cache[key] = h
        return h

    def base_desc(self, scenario_id: int = N.SCN_PHYSICS_ONLY, max_steps: int = 2**62) -> "N.SsWorldDesc":
        p = self.params
        d = N.SsWorldDesc()
        d.abi_version = N.ABI_VERSION
        d.scenario = scenario_id
        d.n_entities = len(self.entities)
        d.n_agents = len(self.agents)
        d.n_dyn = self.dyn.shape[0]
        d.n_stat = self.stat.shape[0]
        d.n_flag_words = self.flags.shape[0]
        d.batch = self.batch_size
        d.env_offset = self.env_offset
        d.global_batch = self.global_batch
        d.max_steps = int(max_steps)
        d.dt = np.float32(p.sub_dt)
        d.keep = np.float32(1.0 - p.damping)
        d.substeps = p.substeps
        d.contact_ck = np.float32(p.contact_force * p.contact_margin)
        d.contact_k = np.float32(p.contact_margin)
        d.has_gravity = int(p.gravity[0] != 0.0 or p.gravity[1] != 0.0)
        ents = self.entity_descs()
        pairs, n_pairs = self.pair_descs()
        d.entities = ctypes.cast(ents, ctypes.POINTER(N.SsEntityDesc))
        d.pairs = ctypes.cast(pairs, ctypes.POINTER(N.SsPairDesc))
        d.n_pairs = n_pairs
        joints = self.joint_descs()
        d.n_joints = len(self.joints)
        d.joints = ctypes.cast(joints, ctypes.POINTER(N.SsJointDesc))
        d._keep = (ents, pairs, joints)   # keep ctypes arrays alive until ss_world_create copies them
        return d

    def joint_descs(self):
        arr = (N.SsJointDesc * max(1, len(self.joints)))()
        for n, jt in enumerate(self.joints):
            q = arr[n]
            q.a, q.b = self._index[id(jt.entity_a)], self._index[id(jt.entity_b)]
            q.ox_a, q.oy_a = Joint.offset(jt.entity_a, jt.anchor_a)
            q.ox_b, q.oy_b = Joint.offset(jt.entity_b, jt.anchor_b)
            q.dist = np.float32(jt.dist)
            q.stiffness = np.float32(jt.stiffness)
            q.rotate_a, q.rotate_b = int(jt.rotate_a), int(jt.rotate_b)
        return arr

    def buffers(self) -> "N.SsBuffers":
        b = N.SsBuffers()
        b.dyn = N.ptr(self.dyn)
        b.stat = N.ptr(self.stat)
        b.stat_vel = N.ptr(self.stat_vel)
        b.rot = N.ptr(self.rot)
        b.step_count = N.ptr(self.step_count)
        b.flags = N.ptr(self.flags)
        b.aux = N.ptr(self.aux)
        rng = self.rng
        if isinstance(rng, DeviceRng):
            b.rng = N.ptr(rng.words)
            b.rng_cur = rng.cur
        return b

    def buffers_ref(self):
        """ctypes byref of a cached SsBuffers (rebuilt when buffers move)."""
        c = self._buf_cache
        if c is None or c[0] != self.version or c[3] is not self.rng:
            b = self.buffers()
            c = (self.version, b, ctypes.byref(b), self.rng)
            self._buf_cache = c
        b = c[1]
        if isinstance(self.rng, DeviceRng):
            b.rng_cur = self.rng.cur
        return c[2]

    def ensure_device_rng(self) -> DeviceRng:
        """Promote the world's SeededRng to a device-backed stream (same state)."""
        if not isinstance(self.rng, DeviceRng):
            dr = DeviceRng(self.rng.seed, self.device)
            dr.set_state(self.rng.state())
            self.rng = dr
        return self.rng


class NativeWorld:
    """Owner of one SsWorld handle (freed when dropped)."""

    def __init__(self, desc: "N.SsWorldDesc"):
        h = ctypes.c_void_p()
        N.check(N.lib().ss_world_create(ctypes.byref(desc), ctypes.byref(h)))
        self.handle = h
        self.obs_dim = desc.obs_dim
        self.scenario = desc.scenario
        # reusable per-call argument block (the library copies it at launch)
        self.act_ptrs = (ctypes.c_void_p * max(1, desc.n_agents))()
        self.io = N.SsStepIO()
        self.io.actions = self.act_ptrs
        self.io_ref = ctypes.byref(self.io)

    def close(self) -> None:
        if self.handle:
            N.lib().ss_world_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
