"""Base class of the built-in scenarios whose whole step is one fused kernel.

A FusedScenario keeps the reference's Scenario hooks (make_world,
reset_world_at, reward, observation, done, post_step) but every hook is a
launch of the scenario's fused kernel in the matching mode (SS_DO_* flags),
so there is exactly one implementation of each task's semantics: the CUDA
one.  Subclasses describe the task to the library through native_desc():
scenario id, constants (rounded exactly as numpy rounds them), observation
width, flag words and the reset program.

If a world no longer matches the kernel's compiled pair enumeration (a
user flipped a collidable / movable flag, swapped a shape, ...), the physics
part runs in the generic world_step kernel and the fused kernel does the
rest of the step (post_step, rewards, dones, observations).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from .. import _native as N
from ..core import World
from ..env import Scenario


class FusedScenario(Scenario):
    native_id: int | None = None
    advances_rng_per_step = False   # discovery draws relocations every step
    shardable_reset = True          # the device reset draws at global env indices

    # ---- subclass interface -------------------------------------------------
    def obs_dim(self, world: World) -> int:
        raise NotImplementedError

    def n_flag_words(self) -> int:
        return 0

    def reset_ops(self, world: World) -> list:
        """[(entity_index, "scatter", (lo_x, lo_y), (hi_x, hi_y)) | (k, "place", (x, y), None)]."""
        raise NotImplementedError

    def template_pairs(self, world: World) -> list:
        """Pair list the fused kernel enumerates (must equal the world's)."""
        raise NotImplementedError

    def fill_constants(self, world: World, d: "N.SsWorldDesc") -> None:
        pass

    def template_ok(self, world: World) -> bool:
        return True

    # ---- descriptor ---------------------------------------------------------
    def reset_program(self, world: World) -> "ResetProgram":
        """The device reset program (SsResetOp); by default the scatter /
        place list of reset_ops()."""
        prog = ResetProgram()
        for k, kind, lo, hi in self.reset_ops(world):
            if kind == "scatter":
                prog.scatter(k, lo, hi)
            else:
                prog.place(k, lo[0], lo[1])
        return prog

    def native_desc(self, world: World, max_steps: int | None = None) -> "N.SsWorldDesc":
        if max_steps is None:
            max_steps = getattr(world, "max_steps", self.max_steps)
        d = world.base_desc(self.native_id, max_steps)
        d.obs_dim = self.obs_dim(world)
        d.n_flag_words = world.flags.shape[0]
        arr = self.reset_program(world).to_c()
        d.reset_ops = ctypes.cast(arr, ctypes.POINTER(N.SsResetOp))
        d.n_reset_ops = arr._n
        self.fill_constants(world, d)
        d._keep = (d._keep, arr)
        return d

    def native_handle(self, world: World, horizon: bool = True):
        """Cached SsWorld of this world version; horizon=False: the same world
        without the step horizon (the scenario's own done term only)."""
        world.ensure_flag_words(self.n_flag_words())
        if horizon:
            return world.native(("fused", world.version), lambda: self.native_desc(world))
        return world.native(("fused-nohorizon", world.version), lambda: self.native_desc(world, 2**62))

    def physics_fused(self, world: World) -> bool:
        key = ("tmpl", world.version)
        ok = world._native_cache.get(key)
        if ok is None:
            ok = _Flag(self.template_ok(world) and not world.joints and
                       list(world.collidable_pairs()) == list(self.template_pairs(world)))
            world._native_cache[key] = ok
        return ok.value

    # ---- launches -------------------------------------------------------------
    def alloc_outputs(self, world: World, obs_dim: int):
        """Fresh (obs (A, Bp, O), rew (A, B), done (B,)); Bp pads B so that every
        agent block starts 16-byte aligned (coalesced float4 stores)."""
        A, B = len(world.agents), world.batch_size
        bp = B
        while (bp * obs_dim) % 4:
            bp += 1
        obs = torch.empty((A, bp, obs_dim), device=world.device)
        rew = torch.empty((A, B), device=world.device)
        done = torch.empty(B, dtype=torch.bool, device=world.device)
        return obs, rew, done

    def launch(self, world: World, mode: int, action_ptrs=None, raw_forces: bool = False,
               guard=None, flip_rng: bool = True, stream: int | None = None, horizon: bool = True,
               guard_count: int = 1):
        """One fused launch in `mode`; returns (obs (A, Bp, O), rew (A, B), done (B,)).

        action_ptrs: one device pointer per agent to a contiguous (B, 2) f32
        block (the caller keeps the tensors alive until the launch is queued).
        """
        world.ensure_device_rng()
        h = self.native_handle(world, horizon)
        st = stream if stream is not None else N.stream_handle(world.device)
        if (mode & N.DO_PHYSICS) and not self.physics_fused(world):
            from ..dynamics import run_world_step

            run_world_step(world, action_ptrs, decode_mask=0 if raw_forces else (1 << 256) - 1,
                           count=False, stream=st, guard=guard, guard_count=guard_count)
            mode &= ~N.DO_PHYSICS
        obs, rew, done = self.alloc_outputs(world, h.obs_dim)
        io = h.io
        if action_ptrs:
            for i, p in enumerate(action_ptrs):
                h.act_ptrs[i] = p
        io.obs = obs.data_ptr()
        io.obs_agent_stride = obs.shape[1] * obs.shape[2]
        io.rew = rew.data_ptr()
        io.done = done.data_ptr()
        io.mode = mode
        io.guard = guard.data_ptr() if guard is not None else None
        io.guard_count = int(guard_count)
        io.raw_forces = int(raw_forces)
        N.check(N.lib().ss_env_step(h.handle, world.buffers_ref(), h.io_ref, st))
        if flip_rng and (mode & N.DO_POST) and self.advances_rng_per_step:
            world.rng.flip()
        return obs, rew, done

    def rollout_capable(self, world: World) -> bool:
        """A fused multi-step rollout kernel exists for this world
        (ss_env_rollout: simple_spread, transport / reverse_transport,
        flocking with their kernel's template, one physics step per
        Env.step)."""
        return (self.native_id in (N.SCN_SIMPLE_SPREAD, N.SCN_TRANSPORT, N.SCN_FLOCKING) and self.physics_fused(world)
                and world.params.substeps == 1 and len(world.agents) <= 8)

    def rollout_preferred(self, world: World) -> bool:
        """Take the rollout kernel by default (StepGraph fused_rollout=None)
        where it pays: simple_spread and transport are bound by the HBM
        traffic the rollout cuts (1M envs: 57.7 -> 36.6 us per step, 80.2 ->
        53.8); flocking once its state no longer stays in L2 between
        launches (1M: 306 -> 279 us; 100k, L2-resident: 29.4 vs 29.8,
        neutral, so the per-step graph)."""
        if self.native_id == N.SCN_FLOCKING and world.batch_size < 262_144:
            return False
        return self.rollout_capable(world)

    def launch_rollout(self, world: World, step_action_ptrs: list, guard=None, stream: int | None = None,
                       check_actions: bool = False) -> list:
        """n = len(step_action_ptrs) consecutive full steps in ONE launch
        (ss_env_rollout), the state kept on chip between them; returns the n
        (obs, rew, done) output triples, bitwise those of n launch(MODE_STEP).
        check_actions: the call scans the n action sets into guard (n int32
        words) first, one launch; step s runs while words 0..s are zero."""
        world.ensure_device_rng()
        h = self.native_handle(world)
        st = stream if stream is not None else N.stream_handle(world.device)
        n, A = len(step_action_ptrs), len(world.agents)
        outs = [self.alloc_outputs(world, h.obs_dim) for _ in range(n)]
        io = N.SsRolloutIO()
        acts = (N.c_vp * (n * A))(*[p for ptrs in step_action_ptrs for p in ptrs])
        obs = (N.c_vp * n)(*[o.data_ptr() for o, _, _ in outs])
        rew = (N.c_vp * n)(*[r.data_ptr() for _, r, _ in outs])
        done = (N.c_vp * n)(*[d.data_ptr() for _, _, d in outs])
        io.n_steps, io.actions, io.obs, io.rew, io.done = n, acts, obs, rew, done
        io.obs_agent_stride = outs[0][0].shape[1] * outs[0][0].shape[2]
        io.guard = guard.data_ptr() if guard is not None else None
        io.check_actions = int(check_actions)
        N.check(N.lib().ss_env_rollout(h.handle, world.buffers_ref(), ctypes.byref(io), st))
        return outs

    # ---- reference hooks as kernel modes ----------------------------------
    def observe_all(self, world: World) -> list:
        obs, _, _ = self.launch(world, N.DO_OBS)
        return [obs[a, : world.batch_size] for a in range(obs.shape[0])]

    def observation(self, agent, world: World) -> torch.Tensor:
        return self.observe_all(world)[world.agents.index(agent)]

    def reward(self, agent, world: World) -> torch.Tensor:
        _, rew, _ = self.launch(world, N.DO_REWARD)
        return rew[world.agents.index(agent)]

    def done(self, world: World) -> torch.Tensor:
        # scenario termination only: the horizon term is Env's (env.py:232);
        # a second cached descriptor without the horizon, so no live handle
        # (and no captured StepGraph) is ever freed by this hook
        _, _, done = self.launch(world, N.DO_DONE, horizon=False)
        return done

    def post_step(self, world: World) -> None:
        self.launch(world, N.DO_POST)

    def reset_world_at(self, world: World, env_index: int | None = None) -> None:
        if env_index is None:
            self._reset(world, None)
        else:
            m = torch.zeros(world.batch_size, dtype=torch.bool, device=world.device)
            m[env_index] = True
            self._reset(world, m)

    def reset_world_masked(self, world: World, mask: torch.Tensor, mask_base=None, mask_total=None) -> None:
        self._reset(world, mask, mask_base, mask_total)

    def _reset(self, world: World, mask, mask_base=None, mask_total=None) -> None:
        world.ensure_device_rng()
        h = self.native_handle(world)
        m = None if mask is None else mask.to(world.device, torch.uint8).contiguous()
        N.check(N.lib().ss_reset(h.handle, world.buffers_ref(), N.ptr(m), N.ptr(mask_base),
                                 N.ptr(mask_total), N.stream_handle(world.device)))
        world.rng.flip()


class ResetProgram:
    """Builder of a device reset program (include/swarmsim_b200.h SsResetOp):
    the reference's reset_world_at restated as register instructions in its
    call order.  Registers are float32, as every value the reference's resets
    combine is (SeededRng.uniform returns float32, batching.py:185-186; Python
    floats are weak, NEP 50); every draw() takes the next draw slot, exactly
    one uniform() call of the reference (n = B for a whole reset, 1 for
    reset(env_index))."""

    def __init__(self):
        self.ops: list[tuple] = []
        self.n_regs = 0

    def release(self) -> None:
        """Every register value so far is dead: reuse the register file."""
        self.n_regs = 0

    def _reg(self) -> int:
        if self.n_regs >= N.RESET_REGS:
            raise ValueError("reset program needs more than 16 registers")
        self.n_regs += 1
        return self.n_regs - 1

    def _op(self, kind, entity=-1, lo=(0.0, 0.0), rng=(0.0, 0.0), r=(0, 0, 0), axis=0):
        self.ops.append((entity, kind, float(lo[0]), float(lo[1]), float(rng[0]), float(rng[1]), *r, axis))

    # common.scatter / place (common.py:11-34)
    def scatter(self, k: int, lo, hi) -> None:
        lo64, hi64 = np.asarray(lo, dtype=np.float64), np.asarray(hi, dtype=np.float64)
        self._op(N.RESET_SCATTER, k, lo64, hi64 - lo64)

    def place(self, k: int, x: float, y: float) -> None:
        self._op(N.RESET_PLACE, k, (x, y))

    # register instructions
    def draw(self, lo: float, hi: float) -> int:
        """rng.uniform(lo, hi, (n,)): float32(lo + (hi - lo) * u)."""
        r = self._reg()
        self._op(N.RESET_DRAW, lo=(lo, 0.0), rng=(float(np.float64(hi) - np.float64(lo)), 0.0), r=(r, 0, 0))
        return r

    def const(self, c: float) -> int:
        r = self._reg()
        self._op(N.RESET_CONST, lo=(c, 0.0), r=(r, 0, 0))
        return r

    def add(self, a: int, b: int) -> int:
        r = self._reg()
        self._op(N.RESET_ADD, r=(r, a, b))
        return r

    def neg(self, a: int) -> int:
        r = self._reg()
        self._op(N.RESET_NEG, r=(r, a, 0))
        return r

    def loadpos(self, k: int, axis: int) -> int:
        r = self._reg()
        self._op(N.RESET_LOADPOS, k, r=(r, 0, 0), axis=axis)
        return r

    def setpos(self, k: int, rx: int, ry: int) -> None:
        """state.set_pos_xy(x, y)."""
        self._op(N.RESET_SETPOS, k, r=(rx, ry, 0))

    def setrot(self, k: int, r: int) -> None:
        self._op(N.RESET_SETROT, k, r=(r, 0, 0))

    def zero(self, k: int) -> None:
        """state.zero_motion (core.py:94-103)."""
        self._op(N.RESET_ZERO, k)

    def to_c(self):
        arr = (N.SsResetOp * max(1, len(self.ops)))()
        for n, op in enumerate(self.ops):
            q = arr[n]
            (q.entity, q.kind, q.lo_x, q.lo_y, q.range_x, q.range_y, q.r0, q.r1, q.r2, q.axis) = op
        arr._n = len(self.ops)
        return arr


class RefHeuristic:
    """Mixin: the scripted controller of the torch restatement (`_reference`,
    scenarios/catalog.py), the reference's heuristic_action."""

    _reference: type = None

    def heuristic_action(self, agent_index: int, obs):
        return self._reference.heuristic_action(self, agent_index, obs)


class HostReset:
    """Mixin for fused scenarios whose reset program runs on the host: the
    torch restatement's reset code (`_reference.reset_world_at`, drawing from
    the Env's Philox stream), one env at a time, ascending, for masked
    resets.  (Every built-in task now resets on the device; kept for user
    subclasses with host reset programs.)"""

    _reference: type = None
    shardable_reset = False

    def reset_ops(self, world):
        return []

    def reset_world_at(self, world: World, env_index: int | None = None) -> None:
        self._reference.reset_world_at(self, world, env_index)

    def reset_world_masked(self, world: World, mask: torch.Tensor, mask_base=None, mask_total=None) -> None:
        if mask_base is not None:
            from ..errors import ContractViolation

            raise ContractViolation(f"{type(self).__name__} resets on the host: no sharded masked reset")
        for i in torch.nonzero(mask).flatten().tolist():
            self.reset_world_at(world, i)
            world.step_count[i] = 0

    def heuristic_action(self, agent_index: int, obs):
        return self._reference.heuristic_action(self, agent_index, obs)


class _Flag:
    """Cache entry with a close() so World._drop_native can clear it."""

    def __init__(self, value: bool):
        self.value = bool(value)

    def close(self) -> None:
        pass


def f32(x) -> float:
    return float(np.float32(x))
