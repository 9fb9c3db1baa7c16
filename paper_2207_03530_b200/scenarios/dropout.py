"""dropout (swarmsim/scenarios/dropout.py), fused.

Any one agent reaching the goal scores; every agent pays for effort.  Step
kernel k_dropout<n> (csrc/ss_small.cu): non-collidable agents (no pairs),
reward float64(any agent within reach) - energy_coeff * (float64 sum of the
decoded actions' float32 squares, agent order, x then y), cast to float32;
done = reached; observation [x, y, vx, vy, goal - self, (other - self)].
Resets: every entity scattered over [-1, 1]^2 in world order (the device
reset program).
"""
from __future__ import annotations

from .. import _native as N
from .._numerics import sqrt_le_bound
from ..core import World
from ..shapes import Sphere
from . import register
from ._fused import FusedScenario, f32
from .catalog import Dropout as _Reference


@register("dropout")
class Dropout(FusedScenario):
    native_id = N.SCN_DROPOUT
    max_steps = 200

    def __init__(self, n_agents: int = 4, energy_coeff: float = 0.02, reach: float = 0.1):
        self.n_agents, self.energy_coeff, self.reach = n_agents, energy_coeff, reach

    def make_world(self, batch_size: int, rng) -> World:
        return _Reference.make_world(self, batch_size, rng)

    def reset_ops(self, world):
        return [(k, "scatter", (-1.0, -1.0), (1.0, 1.0)) for k in range(len(world.entities))]

    def obs_dim(self, world):
        return 4 + 2 * self.n_agents

    def n_flag_words(self) -> int:
        return 2             # float64 energy spent of the last step (bits)

    def template_pairs(self, world):
        return []

    def template_ok(self, world):
        n = self.n_agents
        e = world.entities
        return (len(e) == n + 1 and all(isinstance(a.shape, Sphere) and a.movable and not a.rotatable
                                        for a in e[:n])
                and not e[n].movable and not e[n].collidable)

    def fill_constants(self, world, d):
        d.sc[3] = sqrt_le_bound(f32(self.reach))
        d.sd[0] = float(self.energy_coeff)

    def heuristic_action(self, agent_index: int, obs):
        return _Reference.heuristic_action(self, agent_index, obs)
