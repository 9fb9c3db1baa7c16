"""The device reset programs of the catalog tasks, pinned on CPU.

Each built-in scenario describes its reset_world_at to the library as a
register program (scenarios/_fused.py ResetProgram -> SsResetOp).  Here a
plain numpy interpreter of that instruction set (float32 registers) (the semantics the CUDA
kernel csrc/ss_reset.cu implements) runs each program on numpy's Philox and
is compared bitwise with the reference's own reset: whole batch (draw slot s
of env e = raw draw s*B + e) and sequential reset(env_index=i) (env of rank r
reads draw r*n_slots + s).  The GPU tests then check the kernel against the
golden fixtures the reference produced.
"""
import numpy as np
import pytest

import paper_2207_03530_b200 as S
from paper_2207_03530_b200 import _native as N

CATALOG = ["wheel", "balance", "give_way", "passage", "waterfall", "football", "reverse_transport",
           "simple_spread", "transport", "flocking", "dispersion", "discovery", "dropout"]


def _uniform(raw, lo, rng):
    d = (raw >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return lo + rng * d


class _Interp:
    """numpy restatement of csrc/ss_reset.cu reset_env over a set of envs."""

    def __init__(self, ents, B):
        E = len(ents)
        self.pos = np.zeros((E, 2, B), np.float32)
        self.vel = np.zeros((E, 2, B), np.float32)
        self.rot = np.zeros((E, B), np.float32)
        self.w = np.zeros((E, B), np.float32)

    def run(self, ops, draw, envs):
        R = [None] * N.RESET_REGS
        slot = 0
        for (ent, kind, lo_x, lo_y, rx, ry, r0, r1, r2, axis) in ops:
            if kind in (N.RESET_SCATTER, N.RESET_PLACE):
                if kind == N.RESET_SCATTER:
                    x = _uniform(draw(slot), lo_x, rx).astype(np.float32)
                    y = _uniform(draw(slot + 1), lo_y, ry).astype(np.float32)
                    slot += 2
                else:
                    x, y = np.float32(lo_x), np.float32(lo_y)
                self.pos[ent, 0, envs], self.pos[ent, 1, envs] = x, y
                self.vel[ent, :, envs] = 0
                self.w[ent, envs] = 0
            elif kind == N.RESET_DRAW:
                R[r0] = _uniform(draw(slot), lo_x, rx).astype(np.float32)
                slot += 1
            elif kind == N.RESET_CONST:
                R[r0] = np.full(len(envs), lo_x, dtype=np.float32)
            elif kind == N.RESET_ADD:
                R[r0] = R[r1] + R[r2]
            elif kind == N.RESET_NEG:
                R[r0] = -R[r1]
            elif kind == N.RESET_LOADPOS:
                R[r0] = self.pos[ent, axis, envs].copy()
            elif kind == N.RESET_SETPOS:
                self.pos[ent, 0, envs] = R[r0]
                self.pos[ent, 1, envs] = R[r1]
            elif kind == N.RESET_SETROT:
                self.rot[ent, envs] = R[r0]
            elif kind == N.RESET_ZERO:
                self.vel[ent, :, envs] = 0
                self.w[ent, envs] = 0
        return slot


def _ref_state(env):
    rows = []
    for e in env.world.entities:
        s = e.state
        rows.append(np.stack([s.pos.x, s.pos.y, s.vel.x, s.vel.y, s.rot, s.ang_vel]).astype(np.float32))
    return np.stack(rows)


def _interp_state(it):
    return np.stack([np.stack([it.pos[k, 0], it.pos[k, 1], it.vel[k, 0], it.vel[k, 1], it.rot[k], it.w[k]])
                     for k in range(it.pos.shape[0])])


@pytest.mark.reference
@pytest.mark.parametrize("name", CATALOG)
def test_reset_program_equals_reference_reset(reference, name):
    B, seed = 37, 11
    ref = reference.Env(reference.create_scenario(name), batch_size=B, seed=seed)
    sc = S.create_scenario(name)
    world = sc.make_world(B, S.SeededRng(seed))
    prog = sc.reset_program(world)
    assert [e.name for e in world.entities] == [e.name for e in ref.world.entities]
    # whole batch: draw slot s of env e is raw draw s*B + e
    g = np.random.Generator(np.random.Philox(seed))
    it = _Interp(world.entities, B)
    n_slots = sum(2 if op[1] == N.RESET_SCATTER else int(op[1] == N.RESET_DRAW) for op in prog.ops)
    raw = g.bit_generator.random_raw(n_slots * B)
    got = it.run(prog.ops, lambda s: raw[s * B:(s + 1) * B], np.arange(B))
    assert got == n_slots
    np.testing.assert_array_equal(_interp_state(it), _ref_state(ref))
    assert g.bit_generator.state["state"]["counter"].tolist() == \
        [int(x) for x in ref.rng.state()["state"]["counter"]]
    # sequential reset(env_index=i), ascending: env of rank r reads r*n_slots + s
    sel = [0, 5, 6, 20, B - 1]
    for i in sel:
        ref.reset(env_index=i)
    raw = g.bit_generator.random_raw(n_slots * len(sel))
    for r, i in enumerate(sel):
        it.run(prog.ops, lambda s, r=r: raw[r * n_slots + s:r * n_slots + s + 1], np.array([i]))
    np.testing.assert_array_equal(_interp_state(it), _ref_state(ref))
