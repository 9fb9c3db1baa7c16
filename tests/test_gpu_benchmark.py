"""The reference harness API (tests/test_bench.py) on the device."""
import csv

import pytest

import paper_2207_03530_b200 as S
from paper_2207_03530_b200.benchmark import BenchRow, bench_throughput, steps_per_second, write_csv

pytestmark = pytest.mark.gpu


def test_rows_modes_and_csv(cuda, tmp_path):
    rows = bench_throughput("simple_spread", env_counts=[1, 4], n_steps=3, warmup=1)
    assert [(r.mode, r.n_envs) for r in rows] == [("sequential", 1), ("sequential", 4),
                                                  ("vectorized", 1), ("vectorized", 4)]
    assert all(r.steps == 3 and r.seconds > 0 for r in rows)
    rows = bench_throughput("transport", env_counts=[64, 256], n_steps=5, warmup=2, mode="all")
    assert {r.mode for r in rows} == {"graph", "sequential", "vectorized"}
    p = tmp_path / "b.csv"
    write_csv(rows, str(p))
    lines = list(csv.reader(open(p)))
    assert lines[0] == ["n_envs", "mode", "steps", "seconds"] and len(lines) == 7
    write_csv(rows, str(p), extended=True, bytes_per_env_step=433)
    head = next(csv.reader(open(p)))
    assert head[-1] == "roofline_frac" and "agent_steps_per_s" in head
    with pytest.raises(ValueError):
        bench_throughput(mode="parallel")
    assert steps_per_second(BenchRow(10, "vectorized", 5, 2.0)) == 25.0


def test_device_random_policy_episode(cuda):
    env = S.Env(S.create_scenario("flocking"), 128, seed=0, device=cuda, validate=False)
    ret = S.run_episode(env, S.rollout.DeviceRandomPolicy(seed=3), max_steps=20)
    assert ret.shape == (128,) and bool(ret.isfinite().all())
