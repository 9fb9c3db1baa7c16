"""bench.py's launch and reference-arm logic on CPU (no GPU work):
`--gpus N` spawns N ranks itself (gloo rendezvous on 127.0.0.1, barriers,
max over ranks), the reference arm runs the reference's CPU path on the host
cores, and both arms name the same workload."""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402


def _run(*args, timeout=240):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_gpus_flag_spawns_ranks():
    line = _run("--gpus", "2", "--dry-run", "--steps", "3")
    assert line["n_gpus"] == 2 and line["dry_run"]
    assert line["config"]["workload"] == bench.workload_string("simple_spread", 1_000_000, 2_000_000, 2, False)


def test_world_size_must_match_gpus():
    import os

    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], env=env,
                         capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode != 0 and "WORLD_SIZE=1" in (out.stderr + out.stdout)


def test_reference_arm_line():
    line = _run("--impl", "reference", "--scenario", "transport", "--envs", "4000", "--steps", "2",
                "--warmup", "1")
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["workload"] == bench.workload_string("transport", 4000, 4000, 1, False)
    cb = line["cpu_baseline"]
    assert cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_cpu_rate_uses_reference_when_installed():
    r = bench.cpu_rate("simple_spread", 64, 2)
    assert r["kind"] == ("reference" if bench.load_reference() is not None else "port")
    assert r["agent_steps_per_s"] > 0


def test_byte_model_per_step_and_rollout():
    """bench.step_bytes: a per-step launch moves everything once (DESIGN.md §4
    table); a rollout of S steps pays the state / static / step_count part
    once per S steps."""
    want = {"simple_spread": (3, 3, 14, 341), "transport": (4, 2, 12, 433), "flocking": (5, 4, 32, 917)}
    for scen, (A, n_other, O, total) in want.items():
        per_step, per_launch = bench.step_bytes(scen, A, n_other, O)
        assert per_step + per_launch == total == bench.bytes_per_env_step(scen, A, n_other, O)
        assert bench.bytes_per_env_step(scen, A, n_other, O, 10) == per_step + per_launch / 10
    assert bench.bytes_per_env_step("dispersion", 64, 64, 196) == 53533
    assert bench.bytes_per_env_step("discovery", 64, 3, 136) == 37705
