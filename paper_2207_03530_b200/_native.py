"""ctypes binding of libswarmsim_b200.so (include/swarmsim_b200.h).

This is the only module that touches the C-ABI.  Buffers are torch CUDA
tensors owned by the Python side; only their data_ptr() crosses the
boundary, together with the current CUDA stream handle.  There is no CPU
implementation behind these calls: if the library is missing or no CUDA
device is present, every entry point raises NativeError.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ContractViolation, NativeError, UnknownScenario, UnsupportedShapePair

LIB_PATH = Path(os.environ.get("SS_LIB_PATH") or Path(__file__).resolve().parent / "libswarmsim_b200.so")
ABI_VERSION = 2
RNG_WORDS = 12

SS_SPHERE, SS_BOX, SS_LINE = 0, 1, 2
(SCN_PHYSICS_ONLY, SCN_SIMPLE_SPREAD, SCN_TRANSPORT, SCN_FLOCKING, SCN_DISPERSION, SCN_DISCOVERY, SCN_DROPOUT,
 SCN_WHEEL, SCN_GIVE_WAY, SCN_PASSAGE, SCN_BALANCE, SCN_WATERFALL, SCN_FOOTBALL) = range(13)

DO_PHYSICS, DO_POST, DO_COUNT, DO_REWARD, DO_DONE, DO_OBS = 1, 2, 4, 8, 16, 32
MODE_STEP = 63

c_f32, c_f64, c_i32, c_i64, c_vp = ctypes.c_float, ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p


class SsEntityDesc(ctypes.Structure):
    _fields_ = [
        ("shape", c_i32), ("movable", c_i32), ("rotatable", c_i32), ("collidable", c_i32),
        ("is_agent", c_i32), ("slot", c_i32),
        ("dim0", c_f64), ("dim1", c_f64),
        ("inv_m_dt", c_f32), ("inv_i_dt", c_f32), ("max_speed", c_f32),
        ("grav_x", c_f32), ("grav_y", c_f32), ("u_range", c_f32), ("u_mult", c_f32),
    ]


class SsPairDesc(ctypes.Structure):
    _fields_ = [("i", c_i32), ("j", c_i32), ("d_min", c_f32), ("sign", c_f32), ("d2_act", c_f32)]


(RESET_SCATTER, RESET_PLACE, RESET_DRAW, RESET_CONST, RESET_ADD, RESET_NEG, RESET_LOADPOS, RESET_SETPOS,
 RESET_SETROT, RESET_ZERO) = range(10)
RESET_REGS = 16


class SsResetOp(ctypes.Structure):
    _fields_ = [("entity", c_i32), ("kind", c_i32), ("lo_x", c_f64), ("lo_y", c_f64),
                ("range_x", c_f64), ("range_y", c_f64), ("r0", c_i32), ("r1", c_i32), ("r2", c_i32),
                ("axis", c_i32)]


class SsJointDesc(ctypes.Structure):
    _fields_ = [("a", c_i32), ("b", c_i32), ("ox_a", c_f32), ("oy_a", c_f32), ("ox_b", c_f32),
                ("oy_b", c_f32), ("dist", c_f32), ("stiffness", c_f32), ("rotate_a", c_i32),
                ("rotate_b", c_i32)]


class SsWorldDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", c_i32), ("scenario", c_i32), ("n_entities", c_i32), ("n_agents", c_i32),
        ("n_dyn", c_i32), ("n_stat", c_i32), ("obs_dim", c_i32), ("n_flag_words", c_i32),
        ("batch", c_i64), ("env_offset", c_i64), ("global_batch", c_i64), ("max_steps", c_i64),
        ("dt", c_f32), ("keep", c_f32), ("contact_ck", c_f32), ("contact_k", c_f32),
        ("has_gravity", c_i32), ("n_pairs", c_i32),
        ("entities", ctypes.POINTER(SsEntityDesc)), ("pairs", ctypes.POINTER(SsPairDesc)),
        ("n_reset_ops", c_i32), ("reset_ops", ctypes.POINTER(SsResetOp)),
        ("sc", c_f32 * 16), ("sd", c_f64 * 8), ("si", c_i32 * 8),
        ("lidar_rays", c_i32), ("lidar_attach_rotation", c_i32),
        ("lidar_max_range", c_f64), ("lidar_start", c_f64), ("lidar_span", c_f64),
        ("lidar_dirs", ctypes.POINTER(c_f64)),
        ("substeps", c_i32), ("n_joints", c_i32), ("joints", ctypes.POINTER(SsJointDesc)),
    ]


class SsBuffers(ctypes.Structure):
    _fields_ = [("dyn", c_vp), ("stat", c_vp), ("stat_vel", c_vp), ("rot", c_vp),
                ("step_count", c_vp), ("flags", c_vp), ("aux", c_vp), ("rng", c_vp),
                ("rng_cur", c_i32)]


class SsStepIO(ctypes.Structure):
    _fields_ = [("actions", ctypes.POINTER(c_vp)), ("obs", c_vp), ("obs_agent_stride", c_i64),
                ("rew", c_vp), ("done", c_vp), ("mode", c_i32), ("guard", c_vp),
                ("raw_forces", c_i32), ("guard_count", c_i32)]


MAX_ROLLOUT = 16


class SsRolloutIO(ctypes.Structure):
    _fields_ = [("n_steps", c_i32), ("actions", ctypes.POINTER(c_vp)), ("obs", ctypes.POINTER(c_vp)),
                ("obs_agent_stride", c_i64), ("rew", ctypes.POINTER(c_vp)), ("done", ctypes.POINTER(c_vp)),
                ("guard", c_vp), ("check_actions", c_i32)]


class SsLidarDesc(ctypes.Structure):
    _fields_ = [("n_rays", c_i32), ("max_range", c_f64), ("start_angle", c_f64), ("span", c_f64),
                ("attach_rotation", c_i32), ("dir_table", c_vp)]


_LIB = None


def _declare(lib) -> None:
    P = ctypes.POINTER
    lib.ss_abi_version.restype = c_i32
    lib.ss_last_error.restype = ctypes.c_char_p
    lib.ss_world_create.argtypes = [P(SsWorldDesc), P(c_vp)]
    lib.ss_world_destroy.argtypes = [c_vp]
    lib.ss_env_step.argtypes = [c_vp, P(SsBuffers), P(SsStepIO), c_vp]
    lib.ss_env_rollout.argtypes = [c_vp, P(SsBuffers), P(SsRolloutIO), c_vp]
    lib.ss_world_step.argtypes = [c_vp, P(SsBuffers), P(c_vp), P(ctypes.c_uint64), c_i32, c_vp, c_i32, c_vp, c_vp]
    lib.ss_reset.argtypes = [c_vp, P(SsBuffers), c_vp, c_vp, c_vp, c_vp]
    lib.ss_mask_count.argtypes = [c_vp, c_vp, c_vp, c_vp]
    lib.ss_check_actions.argtypes = [c_vp, P(c_vp), c_vp, c_vp]
    lib.ss_publish_flag.argtypes = [c_vp, c_vp, c_i32, c_vp]
    lib.ss_check_action_sets.argtypes = [P(c_vp), c_i32, c_i32, c_i64, c_i64, c_vp, c_vp]
    lib.ss_lidar.argtypes = [c_vp, P(SsBuffers), c_i32, P(SsLidarDesc), c_vp, c_vp]
    lib.ss_cast_ray.argtypes = [c_vp, P(SsBuffers), c_i32, c_vp, c_vp, c_vp, c_f64, c_vp, c_vp]
    lib.ss_np_trig.argtypes = [c_vp, c_vp, c_i64, c_i32, c_vp]
    lib.ss_collision_force.argtypes = [c_vp, c_vp, c_vp, c_vp, c_f32, c_f32, c_f32, c_f32,
                                       c_vp, c_vp, c_vp, c_i64, c_vp]
    lib.ss_closest_points.argtypes = [c_vp, c_vp, c_i32, c_f64, c_f64, c_vp, c_vp, c_i32,
                                      c_f64, c_f64, c_vp, c_vp, c_i64, c_vp, c_vp]
    for name in ("ss_world_create", "ss_world_destroy", "ss_env_step", "ss_env_rollout", "ss_world_step", "ss_reset",
                 "ss_mask_count", "ss_check_actions", "ss_check_action_sets", "ss_publish_flag", "ss_lidar", "ss_cast_ray",
                 "ss_collision_force", "ss_closest_points", "ss_np_trig"):
        getattr(lib, name).restype = c_i32


def lib():
    """Load the sm_100a library once; raise NativeError if it is absent."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise NativeError(
                f"{LIB_PATH.name} is not built: run `python -m paper_2207_03530_b200._build` "
                "(there is no CPU implementation of the batched step)"
            )
        handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LOCAL if hasattr(os, "RTLD_LOCAL") else 0)
        _declare(handle)
        if handle.ss_abi_version() != ABI_VERSION:
            raise NativeError("libswarmsim_b200.so ABI mismatch; rebuild the library")
        _LIB = handle
    return _LIB


def exported_symbols() -> list[str]:
    return [
        "ss_abi_version", "ss_last_error", "ss_world_create", "ss_world_destroy", "ss_env_step", "ss_env_rollout",
        "ss_world_step", "ss_reset", "ss_mask_count", "ss_check_actions", "ss_check_action_sets",
        "ss_publish_flag", "ss_lidar",
        "ss_cast_ray", "ss_collision_force", "ss_closest_points", "ss_np_trig",
    ]


_ERRORS = {-1: ContractViolation, -2: UnsupportedShapePair, -3: UnknownScenario}


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().ss_last_error().decode(errors="replace")
    raise _ERRORS.get(rc, NativeError)(msg or f"swarmsim_b200 error {rc}")


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_handle(device) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def pointer_array(tensors) -> ctypes.Array:
    arr = (c_vp * max(1, len(tensors)))()
    for i, t in enumerate(tensors):
        arr[i] = None if t is None else t.data_ptr()
    return arr


def np_trig(x, want_cos: bool):
    """np.cos / np.sin of a float32 device tensor, bit-exact (ss_np_trig)."""
    import torch

    t = x.to(torch.float32).contiguous()
    out = torch.empty_like(t)
    check(lib().ss_np_trig(ptr(t), ptr(out), t.numel(), int(want_cos), stream_handle(t.device)))
    return out
