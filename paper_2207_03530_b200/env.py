"""Episode layer (swarmsim/env.py): Scenario hooks, action decoding, Env.

Env.step for a built-in scenario is ONE fused device launch (plus an
optional NaN scan when validate=True): decode -> world_step -> post_step ->
step_count -> rewards -> dones -> observations, all inside the kernel, with
outputs written to fresh device tensors.  User-defined scenarios (plain
Scenario subclasses) run physics in the generic step kernel and their own
Python hooks on device tensors.  There is no CPU path: an Env needs a CUDA
device and the built library.

VMAS-style aliases: make_env, Environment (= Env), Env.reset_at(mask).
"""
from __future__ import annotations

import gc

from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _native as N
from .batching import DeviceRng, SeededRng, Vec2, default_device
from .core import Agent, AgentAction, World
from .errors import ContractViolation, NativeError


class Scenario:
    """Task definition (env.py:20-54).  Subclasses override the hooks."""

    max_steps: int = 200

    def make_world(self, batch_size: int, rng: SeededRng) -> World:
        raise NotImplementedError

    def reset_world_at(self, world: World, env_index: int | None = None) -> None:
        raise NotImplementedError

    def reward(self, agent: Agent, world: World) -> torch.Tensor:
        raise NotImplementedError

    def observation(self, agent: Agent, world: World) -> torch.Tensor:
        raise NotImplementedError

    def done(self, world: World) -> torch.Tensor:
        return torch.zeros(world.batch_size, dtype=torch.bool, device=world.device)

    def info(self, agent: Agent, world: World) -> dict:
        return {}

    def post_step(self, world: World) -> None:
        pass

    def heuristic_action(self, agent_index: int, obs):
        raise NotImplementedError

    def device_scripted(self, agent: Agent) -> bool:
        """True when the scenario's fused kernel runs this agent's
        action_script itself (no host decode, no raw action needed)."""
        return False


@dataclass(frozen=True)
class ActionSpec:
    mode: str
    move_dim: int = 2
    comm_dim: int = 0
    n_move_choices: int = 5

    @property
    def flat_dim(self) -> int:
        return self.move_dim + self.comm_dim


def _to_device(raw, device) -> torch.Tensor:
    if isinstance(raw, torch.Tensor):
        return raw.to(device, non_blocking=True)
    arr = np.asarray(raw)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device, non_blocking=True)


def decode_action(raw, spec: ActionSpec, agent: Agent, rng: SeededRng, check: bool = True) -> AgentAction:
    """Raw policy output -> AgentAction (env.py:71-145), on the agent's device.

    check=False (Env(validate=False)) skips the NaN scan, the one host sync of
    the continuous branch, so the decode can be captured in a CUDA graph.
    """
    world = agent.state._world
    B, dev = world.batch_size, world.device
    t = _to_device(raw, dev)
    if check and t.is_floating_point() and bool(torch.isnan(t).any()):
        raise ContractViolation(f"action for '{agent.name}' contains NaN")
    if spec.mode == "continuous":
        if t.ndim == 1 and spec.comm_dim == 0 and tuple(t.shape) == (2,) and B == 1:
            t = t.reshape(1, 2)
        if tuple(t.shape) != (B, spec.flat_dim):
            raise ContractViolation(
                f"continuous action for '{agent.name}' has shape {tuple(t.shape)}, expected {(B, spec.flat_dim)}")
        t = t.to(torch.float32)
        u = float(np.float32(agent.u_range))
        mv = torch.clamp(t[:, :2], -u, u) * float(np.float32(agent.u_multiplier))
        fx, fy = mv[:, 0].clone(), mv[:, 1].clone()
        comm = t[:, 2:].clone() if spec.comm_dim else None
    elif spec.mode == "discrete":
        if t.is_floating_point() or t.dtype == torch.bool:
            raise ContractViolation(f"discrete action for '{agent.name}' must be integer")
        if spec.comm_dim:
            if tuple(t.shape) != (B, 2):
                raise ContractViolation(f"discrete action for '{agent.name}' has shape {tuple(t.shape)}, expected {(B, 2)}")
            move, cidx = t[:, 0], t[:, 1]
        else:
            if tuple(t.shape) == (B, 1):
                t = t[:, 0]
            if tuple(t.shape) != (B,):
                raise ContractViolation(f"discrete action for '{agent.name}' has shape {tuple(t.shape)}, expected {(B,)}")
            move, cidx = t, None
        if bool(((move < 0) | (move >= spec.n_move_choices)).any()):
            raise ContractViolation(
                f"discrete move index for '{agent.name}' out of range [0, {spec.n_move_choices})")
        u = float(np.float32(agent.u_range * agent.u_multiplier))
        z = torch.zeros(B, device=dev)
        fx = torch.where(move == 1, u, torch.where(move == 2, -u, z))
        fy = torch.where(move == 3, u, torch.where(move == 4, -u, z))
        if cidx is not None:
            if bool(((cidx < 0) | (cidx >= spec.comm_dim)).any()):
                raise ContractViolation(f"comm index for '{agent.name}' out of range [0, {spec.comm_dim})")
            comm = torch.zeros((B, spec.comm_dim), device=dev)
            comm[torch.arange(B, device=dev), cidx.long()] = 1.0
        else:
            comm = None
    else:
        raise ContractViolation(f"unknown action mode {spec.mode!r}")
    if agent.action_noise_std > 0.0:
        noise = torch.from_numpy(rng.normal(0.0, agent.action_noise_std, (B, 2))).to(dev)
        fx = fx + noise[:, 0]
        fy = fy + noise[:, 1]
    if agent.silent:
        comm = None
    return AgentAction(force=Vec2(fx, fy), comm=comm)


@dataclass
class StepResult:
    obs: list
    rewards: list
    dones: torch.Tensor
    infos: list = field(default_factory=list)


class Env:
    """Batched episode driver around one scenario (env.py:156-235)."""

    def __init__(self, scenario: Scenario, batch_size: int, seed: int = 0, max_steps: int | None = None,
                 action_mode: str = "continuous", device=None, validate: bool = True,
                 env_offset: int = 0, global_batch: int | None = None, substeps: int | None = None):
        if batch_size < 1:
            raise ContractViolation(f"batch_size must be >= 1, got {batch_size}")
        if action_mode not in ("continuous", "discrete"):
            raise ContractViolation(f"unknown action mode {action_mode!r}")
        dev = torch.device(device) if device is not None else default_device()
        if dev.type != "cuda":
            raise NativeError("the batched step runs on a CUDA device only (no CPU implementation)")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        N.lib()   # fail loudly now if the library is missing
        self.scenario = scenario
        self.batch_size = int(batch_size)
        self.device = dev
        self.validate = validate
        with torch.cuda.device(dev):
            self.rng = DeviceRng(seed, dev)
            self.world = _make_world(scenario, batch_size, self.rng, dev)
        self.world.rng = self.rng
        if substeps is not None:
            # extension: physics sub-steps per step (PhysParams.substeps)
            self.world.params = replace(self.world.params, substeps=substeps)
        gb = self.batch_size if global_batch is None else int(global_batch)
        if env_offset < 0 or env_offset + self.batch_size > gb:
            raise ContractViolation("shard [env_offset, env_offset + batch_size) outside global_batch")
        if (env_offset != 0 or gb != self.batch_size) and not getattr(scenario, "shardable_reset", False):
            # a host reset program draws B values from the stream, not the
            # shard's slice of the global batch: a sharded run would give
            # every shard rank 0's initial states
            raise ContractViolation(f"{type(scenario).__name__} resets on the host: it cannot run as a "
                                    "shard (env_offset / global_batch) of a larger batch")
        self.world.env_offset = int(env_offset)
        self.world.global_batch = gb
        self.world._touch()
        self._max_steps = max_steps if max_steps is not None else scenario.max_steps
        self.world.max_steps = self._max_steps
        self.action_mode = action_mode
        self.action_specs = [ActionSpec(mode=action_mode, comm_dim=0 if a.silent else a.comm_dim)
                             for a in self.world.agents]
        self._flag = torch.zeros(1, dtype=torch.int32, device=dev)
        # the verdict's host copy: pinned, device-mapped (unified addressing),
        # written by a kernel store (ss_publish_flag) and read after an event
        # wait — a device-to-host copy would queue behind any observation
        # copies in flight on the copy engine
        self._flag_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        self._flag_event = torch.cuda.Event()
        self.reset()

    # -- properties ----------------------------------------------------------
    @property
    def agents(self) -> list[Agent]:
        return self.world.agents

    @property
    def step_count(self) -> torch.Tensor:
        return self.world.step_count

    @property
    def max_steps(self) -> int:
        return self._max_steps

    @max_steps.setter
    def max_steps(self, v: int) -> None:
        self._max_steps = int(v)
        self.world.max_steps = self._max_steps
        self.world._touch()

    @property
    def fused(self) -> bool:
        return getattr(self.scenario, "native_id", None) is not None

    # -- reset ---------------------------------------------------------------
    def reset(self, env_index: int | None = None) -> list:
        """Reset every env, or one index, and return fresh observations (env.py:189-198)."""
        if env_index is not None and not (0 <= env_index < self.batch_size):
            raise ContractViolation(f"env_index {env_index} out of range [0, {self.batch_size})")
        self.scenario.reset_world_at(self.world, env_index)
        if env_index is None:
            self.world.step_count.zero_()
        else:
            self.world.step_count[env_index] = 0
        return self.observations()

    def reset_at(self, mask) -> list:
        """Reset the selected envs (bool mask (B,), index, or index list).

        Equivalent — bitwise, including the random stream — to calling
        reset(env_index=i) for each selected i in ascending order; for the
        built-in scenarios it is one masked reset launch.
        """
        m = _as_mask(mask, self.batch_size, self.device)
        if self.fused:
            self.scenario.reset_world_masked(self.world, m)
        else:
            for i in torch.nonzero(m).flatten().tolist():
                self.scenario.reset_world_at(self.world, i)
                self.world.step_count[i] = 0
        return self.observations()

    def observations(self) -> list:
        if self.fused:
            obs = self.scenario.observe_all(self.world)
        else:
            obs = [self.scenario.observation(a, self.world).to(torch.float32) for a in self.agents]
        return self._obs_noise(obs)

    def _obs_noise(self, obs: list) -> list:
        out = []
        for agent, o in zip(self.agents, obs):
            if agent.obs_noise_std > 0.0:
                o = o + torch.from_numpy(self.rng.normal(0.0, agent.obs_noise_std, tuple(o.shape))).to(o.device)
            out.append(o)
        return out

    # -- step ----------------------------------------------------------------
    def step(self, raw_actions) -> StepResult:
        """Advance the whole batch one step (env.py:209-235).

        raw_actions: one (B, 2 + comm_dim) array/tensor per agent (None for
        scripted agents), or a single (A, B, 2) tensor — the zero-copy fast path.
        """
        agents = self.agents
        if isinstance(raw_actions, torch.Tensor) and raw_actions.ndim == 3:
            if (self.fused and raw_actions.device == self.device and raw_actions.dtype == torch.float32
                    and tuple(raw_actions.shape) == (len(agents), self.batch_size, 2)
                    and raw_actions.is_contiguous() and not self._needs_host_decode([0] * len(agents), True)
                    and all(s.comm_dim == 0 for s in self.action_specs)):
                base, stride = raw_actions.data_ptr(), self.batch_size * 8
                return self._step_fused_ptrs([base + a * stride for a in range(len(agents))], raw_actions, False)
            raw_actions = list(raw_actions.unbind(0))
        if len(raw_actions) != len(agents):
            raise ContractViolation(f"got {len(raw_actions)} actions for {len(agents)} agents")
        for raw, agent in zip(raw_actions, agents):
            if raw is None and agent.action_script is None:
                raise ContractViolation(f"agent '{agent.name}' needs an action, got None")
        if self.fused:
            return self._step_fused(raw_actions)
        return self._step_generic(raw_actions)

    def _fast_actions(self, raw_actions):
        """Continuous, noiseless, unscripted (or kernel-scripted): raw (B, 2)
        device tensors, no decode on host; None for a kernel-scripted agent
        given no action."""
        B, dev = self.batch_size, self.device
        out = []
        for raw, agent, spec in zip(raw_actions, self.agents, self.action_specs):
            if raw is None:
                out.append(None)
                continue
            t = _to_device(raw, dev)
            if t.ndim == 1 and spec.comm_dim == 0 and tuple(t.shape) == (2,) and B == 1:
                t = t.reshape(1, 2)
            if tuple(t.shape) != (B, spec.flat_dim):
                raise ContractViolation(
                    f"continuous action for '{agent.name}' has shape {tuple(t.shape)}, expected {(B, spec.flat_dim)}")
            if spec.comm_dim:
                if not agent.silent:
                    self.world.comm[agent.name] = t[:, 2:].to(torch.float32).clone()
                t = t[:, :2]
            if t.dtype != torch.float32:
                t = t.to(torch.float32)
            out.append(t.contiguous())
        return out

    def _host_decoded(self, raw_actions):
        """Discrete / noisy / scripted agents: final forces computed on device with torch."""
        forces = []
        # scripts see the pre-step state and run in agent order, before any
        # physics (dynamics.py:136-138); a script replaces any raw action
        decoded = [None if raw is None else decode_action(raw, spec, agent, self.rng, self.validate)
                   for raw, agent, spec in zip(raw_actions, self.agents, self.action_specs)]
        for act, agent in zip(decoded, self.agents):
            if agent.action_script is not None:
                act = agent.action_script(agent, self.world)
            from .dynamics import _validate_action

            _validate_action(agent, act, self.batch_size, self.validate)
            agent.action = act
            if not agent.silent and act.comm is not None:
                self.world.comm[agent.name] = act.comm
            forces.append(torch.stack([act.force.x, act.force.y], 1).to(self.device, torch.float32).contiguous())
        return forces

    def _needs_host_decode(self, raw_actions, all_given: bool = False) -> bool:
        if self.action_mode != "continuous":
            return True
        sc = self.scenario
        for raw, agent in zip(raw_actions, self.agents):
            if agent.action_noise_std > 0.0:
                return True
            if agent.action_script is not None:
                if not (self.fused and sc.device_scripted(agent)):
                    return True
            elif raw is None and not all_given:
                return True
        return False

    def _step_fused(self, raw_actions) -> StepResult:
        raw = self._needs_host_decode(raw_actions)
        forces = self._host_decoded(raw_actions) if raw else self._fast_actions(raw_actions)
        return self._step_fused_ptrs([None if f is None else f.data_ptr() for f in forces], forces, raw)

    def _step_fused_ptrs(self, ptrs, keepalive, raw: bool) -> StepResult:
        world, sc = self.world, self.scenario
        st = torch.cuda.current_stream(self.device).cuda_stream
        guard = None
        if self.validate and not raw:
            self._flag.zero_()
            h = sc.native_handle(world)
            arr = (N.c_vp * max(1, len(ptrs)))(*ptrs)
            N.check(N.lib().ss_check_actions(h.handle, arr, self._flag.data_ptr(), st))
            guard = self._flag
        obs, rew, done = sc.launch(world, N.MODE_STEP, action_ptrs=ptrs, raw_forces=raw, guard=guard,
                                   flip_rng=False, stream=st)
        if guard is not None and self._verdict(st) != 0:
            forces = keepalive if isinstance(keepalive, list) else list(keepalive.unbind(0))
            bad = next(a.name for a, f in zip(self.agents, forces) if f is not None and bool(torch.isnan(f).any()))
            raise ContractViolation(f"action for '{bad}' contains NaN")
        if sc.advances_rng_per_step:
            world.rng.flip()
        B = self.batch_size
        obs_list = list((obs if obs.shape[1] == B else obs[:, :B]).unbind(0))
        if self._any_obs_noise:
            obs_list = self._obs_noise(obs_list)
        if type(sc).info is _BASE_INFO:
            infos = [{} for _ in self.agents]
        else:
            infos = [sc.info(a, world) for a in self.agents]
        return StepResult(obs=obs_list, rewards=list(rew.unbind(0)), dones=done, infos=infos)

    def _verdict(self, st: int) -> int:
        """The NaN verdict of the step just queued on stream `st` (host sync
        on that stream's work only)."""
        N.check(N.lib().ss_publish_flag(self._flag.data_ptr(), self._flag_host.data_ptr(), 1, st))
        self._flag_event.record(torch.cuda.current_stream(self.device))
        self._flag_event.synchronize()
        return int(self._flag_host[0])

    def _capture_step(self, ptrs, keepalive, flags=None, n_flags: int = 1) -> StepResult:
        """One fused step without host syncs (graph capture).  flags: device
        int32 NaN verdicts of this and the earlier steps of the replay (their
        action scans run ahead of the steps in the graph); any set word makes
        the launch a no-op — the eager validated step's guard, left for the
        host to read after the replay instead of syncing inside it."""
        saved = self.validate
        self.validate = False
        try:
            if flags is None:
                return self._step_fused_ptrs(ptrs, keepalive, False)
            st = torch.cuda.current_stream(self.device).cuda_stream
            obs, rew, done = self.scenario.launch(self.world, N.MODE_STEP, action_ptrs=ptrs, guard=flags,
                                                  flip_rng=False, stream=st, guard_count=n_flags)
            B = self.batch_size
            obs_list = list((obs if obs.shape[1] == B else obs[:, :B]).unbind(0))
            return StepResult(obs=obs_list, rewards=list(rew.unbind(0)), dones=done,
                              infos=[{} for _ in self.agents])
        finally:
            self.validate = saved

    def step_graph(self, actions, steps_per_replay: int = 1, validate: bool = False,
                   fused_rollout: bool | None = None) -> "StepGraph":
        """Capture Env.step into CUDA graphs over the given action buffer(s).

        validate=True keeps the reference's NaN check inside the graph: each
        step scans its actions and is a no-op once any NaN was seen in the
        replay; StepGraph.check() raises ContractViolation afterwards.
        fused_rollout: the S steps of a replay as ONE launch with the state
        kept on chip between them (bitwise the same results) — None: where
        the scenario prefers it (simple_spread, transport; flocking from
        262144 envs), True: wherever a rollout kernel exists (also
        reverse_transport, any flocking batch), False: never."""
        return StepGraph(self, actions, steps_per_replay, validate, fused_rollout)

    @property
    def _any_obs_noise(self) -> bool:
        return any(a.obs_noise_std > 0.0 for a in self.agents)

    def _step_generic(self, raw_actions) -> StepResult:
        from .dynamics import run_world_step

        world, sc = self.world, self.scenario
        forces = self._host_decoded(raw_actions)
        run_world_step(world, forces, decode_mask=0, count=False)
        sc.post_step(world)
        world.step_count += 1
        rewards = [torch.as_tensor(sc.reward(a, world), device=self.device).to(torch.float32) for a in self.agents]
        dones = torch.as_tensor(sc.done(world), device=self.device).to(torch.bool) | (world.step_count >= self.max_steps)
        obs = self.observations()
        infos = [sc.info(a, world) for a in self.agents]
        return StepResult(obs=obs, rewards=rewards, dones=dones, infos=infos)


Environment = Env
_BASE_INFO = Scenario.info


class StepGraph:
    """Env.step as CUDA-graph replays — the launch-overhead-free stepping mode.

    Each action buffer in `actions` (one or more (A, B, 2) float32 device
    tensors, read in place at every replay) gets a captured graph; step(i)
    replays graph i.  Built-in scenarios capture their fused launch; any
    other scenario captures the generic path (ss_world_step + its torch
    hooks) — scripted agents keep running their script, and a scenario that
    syncs with the host or draws from the Env stream inside step is refused
    (ContractViolation).  With steps_per_replay=S > 1 a
    graph holds S consecutive fused steps reading actions[i], actions[i+1],
    ... (cyclically) — an open-loop rollout whose S StepResults live in
    distinct graph-owned buffers (rollout(i)), so the GPU runs the steps back
    to back without a host launch between them.  Outputs are static tensors
    owned by the graph and overwritten by its next replay.  Semantics are
    Env.step's with validate=False (no NaN scan): results are bit-identical
    to eager stepping.  Scenarios that draw from the Env's stream every step
    (discovery) get one graph per half of the double-buffered Philox state.
    """

    @staticmethod
    def _rng_mode_of(sc) -> bool:
        return bool(getattr(sc, "advances_rng_per_step", False))

    def __init__(self, env: Env, actions, steps_per_replay: int = 1, validate: bool = False,
                 fused_rollout: bool | None = None):
        acts = [actions] if isinstance(actions, torch.Tensor) else list(actions)
        A, B = len(env.agents), env.batch_size
        S = int(steps_per_replay)
        if S < 1:
            raise ContractViolation(f"steps_per_replay must be >= 1, got {steps_per_replay}")
        for t in acts:
            if (t.device != env.device or t.dtype != torch.float32 or tuple(t.shape) != (A, B, 2)
                    or not t.is_contiguous()):
                raise ContractViolation(f"StepGraph actions must be contiguous float32 ({A}, {B}, 2) on {env.device}")
        if env.action_mode != "continuous" or any(s.comm_dim for s in env.action_specs) or env._any_obs_noise \
                or any(a.action_noise_std > 0.0 for a in env.agents):
            raise ContractViolation("StepGraph covers continuous, noiseless, silent agents")
        self.env = env
        self.actions = acts
        self.steps_per_replay = S
        # scripted agents (or a non-fused scenario): capture the whole public
        # step — scripts, decode, launches — instead of the bare fused launch
        self._generic = not env.fused or env._needs_host_decode([0] * A)
        if validate and self._generic:
            raise ContractViolation("StepGraph(validate=True) covers the fused built-in step")
        # NaN verdict of the replay (validate=True), zeroed at its start
        self.nan_flag = torch.zeros(S, dtype=torch.int32, device=env.device) if validate else None
        sc, world = env.scenario, env.world
        # S > 1 steps of a world with a rollout kernel: one fused launch per
        # replay, the state on chip between the steps (see Env.step_graph;
        # otherwise S separate step kernels)
        self._fused_rollout = (fused_rollout is not False and S > 1 and S <= N.MAX_ROLLOUT and not self._generic
                               and not self._rng_mode_of(sc) and type(sc).info is _BASE_INFO
                               and hasattr(sc, "rollout_capable") and sc.rollout_capable(world)
                               and (fused_rollout is True or sc.rollout_preferred(world)))
        self.fused_rollout = self._fused_rollout
        # kernels of this library per replay: the step kernels (or the one
        # rollout kernel) plus the action scans
        self.launches_per_replay = ((1 + (1 if validate else 0)) if self._fused_rollout
                                    else S + (-(-S // N.MAX_ROLLOUT) if validate else 0))
        self._rng_mode = bool(getattr(sc, "advances_rng_per_step", False))
        world.ensure_device_rng()
        if not env.fused:
            # generic worlds: physics through ss_world_step plus the scenario's
            # torch hooks; they must not sync with the host or draw from the
            # Env stream inside step (checked: a draw raises during capture)
            from .dynamics import physics_world

            physics_world(world)
        else:
            sc.native_handle(world)           # build the descriptors outside capture
            if not sc.physics_fused(world):
                from .dynamics import physics_world

                physics_world(world)          # world_step's generic kernel runs first
        start_cur = world.rng.cur
        self._graphs: dict = {}
        self._results: dict = {}
        stream = torch.cuda.Stream(env.device)
        stream.wait_stream(torch.cuda.current_stream(env.device))
        # no cyclic GC inside a capture: a collected world handle would call
        # cudaFree on the capturing thread and invalidate the graph
        gc_was = gc.isenabled()
        gc.collect()
        gc.disable()
        try:
            self._capture_all(env, acts, A, B, S, start_cur, stream)
        except RuntimeError as ex:
            raise ContractViolation(f"step of '{type(sc).__name__}' is not capturable: {ex}") from ex
        finally:
            if gc_was:
                gc.enable()
            world.rng.capture_guard = False
        torch.cuda.current_stream(env.device).wait_stream(stream)
        world.rng.cur = start_cur
        self._start_cur = start_cur
        # the captured kernels hold this world's descriptor tables and state
        # buffers: any later edit that rebuilds them retires the graph
        self._epoch = (world.native_epoch, world.version, world.rng)

    def _capture_all(self, env, acts, A, B, S, start_cur, stream) -> None:
        world = env.world
        for cur in ((0, 1) if self._rng_mode else (start_cur,)):
            for i in range(len(acts)):
                world.rng.cur = cur       # each captured step flips it in rng mode
                g = torch.cuda.CUDAGraph()
                results = []
                with torch.cuda.stream(stream), torch.cuda.graph(g, stream=stream):
                    if self._fused_rollout:
                        results = self._capture_rollout(env, acts, i, A, B, S, stream)
                        self._graphs[(cur, i)] = g
                        self._results[(cur, i)] = results
                        continue
                    if self.nan_flag is not None:
                        self._capture_scans(acts, i, A, B, S, stream)
                    for k in range(S):
                        act = acts[(i + k) % len(acts)]
                        if self._generic:
                            results.append(self._capture_generic(act))
                            continue
                        base, stride = act.data_ptr(), B * 8
                        results.append(env._capture_step([base + a * stride for a in range(A)], act,
                                                         self.nan_flag, k + 1))
                self._graphs[(cur, i)] = g
                self._results[(cur, i)] = results

    def _capture_rollout(self, env, acts, i, A, B, S, stream) -> list:
        """The S steps as ONE fused rollout launch (ss_env_rollout: the state
        stays on chip between the steps), preceded, when validating, by one
        scan launch over the S action sets (the kernel runs step k only while
        scans 0..k found no NaN)."""
        sc, world = env.scenario, env.world
        ptrs = []
        for k in range(S):
            act = acts[(i + k) % len(acts)]
            base, stride = act.data_ptr(), B * 8
            ptrs.append([base + a * stride for a in range(A)])
        outs = sc.launch_rollout(world, ptrs, guard=self.nan_flag, stream=stream.cuda_stream,
                                 check_actions=self.nan_flag is not None)
        res = []
        for obs, rew, done in outs:
            obs_list = list((obs if obs.shape[1] == B else obs[:, :B]).unbind(0))
            res.append(StepResult(obs=obs_list, rewards=list(rew.unbind(0)), dones=done,
                                  infos=[{} for _ in env.agents]))
        return res

    def _capture_scans(self, acts, i, A, B, S, stream) -> None:
        """The replay's S action NaN scans as one launch per 16 steps
        (ss_check_action_sets) on the capturing stream, ahead of the steps:
        step k then runs only while words 0..k are zero (its guard count),
        and the step kernels keep their programmatic-launch chain (a scan
        per step on a side branch put a cross-stream wait before each)."""
        for k0 in range(0, S, N.MAX_ROLLOUT):
            n = min(N.MAX_ROLLOUT, S - k0)
            bases = (N.c_vp * n)(*[acts[(i + k) % len(acts)].data_ptr() for k in range(k0, k0 + n)])
            N.check(N.lib().ss_check_action_sets(bases, n, A, B * 2, B * 2, self.nan_flag[k0:].data_ptr(),
                                                 stream.cuda_stream))

    def _capture_generic(self, act) -> StepResult:
        env = self.env
        saved, rng = env.validate, env.world.rng
        env.validate = False
        rng.capture_guard = True
        try:
            raw = [None if a.action_script is not None else act[n] for n, a in enumerate(env.agents)]
            return env._step_fused(raw) if env.fused else env._step_generic(raw)
        finally:
            env.validate = saved
            rng.capture_guard = False

    def _replay(self, i: int) -> list:
        world = self.env.world
        if (world.native_epoch, world.version, world.rng) != self._epoch:
            raise ContractViolation("the world was edited since this StepGraph was captured "
                                    "(its descriptor / buffers were rebuilt): capture a new one")
        rng = world.rng
        # rng-mode scenarios have one graph per Philox half; the others one
        # graph whatever the current half (a reset flips it between replays)
        key = (rng.cur if self._rng_mode else self._start_cur, i)
        self._graphs[key].replay()
        if self._rng_mode and self.steps_per_replay % 2:
            rng.flip()
        return self._results[key]

    def step(self, i: int = 0) -> StepResult:
        """Replay graph i; returns the outputs of its last step."""
        return self._replay(i)[-1]

    def check(self) -> None:
        """validate=True: raise ContractViolation if the last replay met a NaN
        action (the steps from that one on did not move anything).  Syncs."""
        if self.nan_flag is not None and bool(self.nan_flag.any()):
            raise ContractViolation("an action replayed by this StepGraph contains NaN")

    def rollout(self, i: int = 0) -> list:
        """Replay graph i; returns the S StepResults of its steps, in order."""
        return self._replay(i)


def _make_world(scenario: Scenario, batch_size: int, rng, device) -> World:
    w = scenario.make_world(batch_size, rng)
    if w.device != device:
        raise ContractViolation(f"scenario built its world on {w.device}, Env runs on {device}")
    return w


def _as_mask(mask, B: int, device) -> torch.Tensor:
    if isinstance(mask, (int, np.integer)):
        idx = [int(mask)]
    elif isinstance(mask, torch.Tensor) and mask.dtype in (torch.bool, torch.uint8):
        # a (B,) bool or uint8 tensor is a mask (dones.to(torch.uint8) included)
        if tuple(mask.shape) != (B,):
            raise ContractViolation(f"reset mask must have shape ({B},), got {tuple(mask.shape)}")
        return mask.to(device) != 0
    else:
        arr = np.asarray(mask.cpu() if isinstance(mask, torch.Tensor) else mask)
        if arr.dtype == bool or arr.dtype == np.uint8:
            if arr.shape != (B,):
                raise ContractViolation(f"reset mask must have shape ({B},), got {arr.shape}")
            return torch.from_numpy(arr != 0).to(device)
        if arr.ndim == 1 and arr.shape == (B,) and B > 2 and np.isin(arr, (0, 1)).all():
            raise ContractViolation("ambiguous reset selector: a (B,) array of 0/1 integers; pass a bool "
                                    "mask or an explicit index list")
        idx = [int(i) for i in arr.reshape(-1)]
    for i in idx:
        if not (0 <= i < B):
            raise ContractViolation(f"env_index {i} out of range [0, {B})")
    m = torch.zeros(B, dtype=torch.bool)
    m[idx] = True
    return m.to(device)


class SingleEnv:
    """Unbatched facade over a batch_size=1 Env (env.py:238-266)."""

    def __init__(self, env: Env):
        if env.batch_size != 1:
            raise ContractViolation("SingleEnv requires a batch_size=1 Env")
        self.env = env

    @property
    def agents(self):
        return self.env.agents

    def reset(self, **kwargs):
        return [o[0] for o in self.env.reset(**kwargs)]

    def step(self, raw_actions):
        batched = []
        for raw, spec in zip(raw_actions, self.env.action_specs):
            if raw is None:
                batched.append(None)
            elif spec.mode == "discrete":
                batched.append(np.asarray(raw).reshape(1, -1) if np.ndim(raw) else np.asarray([raw]))
            else:
                batched.append(np.asarray(raw, dtype=np.float32).reshape(1, -1))
        res = self.env.step(batched)
        obs = [o[0] for o in res.obs]
        rewards = [float(r[0]) for r in res.rewards]
        return obs, rewards, bool(res.dones[0]), res.infos


def make_env(scenario, num_envs: int = 32, device=None, continuous_actions: bool = True,
             max_steps: int | None = None, seed: int | None = None, validate: bool = True,
             substeps: int | None = None, **kwargs) -> Env:
    """VMAS-style constructor: make_env("simple_spread", num_envs=1_000_000, n_agents=3)."""
    from .scenarios import create_scenario

    sc = create_scenario(scenario, **kwargs) if isinstance(scenario, str) else scenario
    return Env(sc, num_envs, seed=0 if seed is None else seed, max_steps=max_steps,
               action_mode="continuous" if continuous_actions else "discrete", device=device,
               validate=validate, substeps=substeps)
