"""Frame snapshots from device state (tests/test_viewer.py:24-41 of the reference)."""
import json

import pytest

import paper_2207_03530_b200 as S
from paper_2207_03530_b200.viewer import encode_frame, snapshot_from_env

pytestmark = pytest.mark.gpu


def test_frame_encodes_every_entity(cuda):
    env = S.Env(S.create_scenario("dropout"), 2, seed=0, device=cuda)
    msg = json.loads(encode_frame(snapshot_from_env(env, 0)))
    assert msg["type"] == "frame" and msg["t"] == 0 and msg["env"] == 0
    assert len(msg["entities"]) == len(env.world.entities)
    st = env.world.state_array().cpu()
    for k, ent in enumerate(msg["entities"]):
        assert set(ent) == {"name", "shape", "pos", "rot", "color"} and "kind" in ent["shape"]
        assert ent["pos"] == [float(st[k, 0, 0]), float(st[k, 1, 0])] and ent["rot"] == float(st[k, 4, 0])


def test_frame_t_tracks_the_viewed_env(cuda):
    env = S.Env(S.create_scenario("transport"), 3, seed=0, device=cuda)
    env.step_count[:] = env.step_count.new_tensor([4, 9, 2])
    assert snapshot_from_env(env, 1).t == 9
    assert snapshot_from_env(env, 2).t == 2
    with pytest.raises(S.ContractViolation):
        snapshot_from_env(env, 3)
