"""Time the fused step kernel of each workload for several library variants.

    [SWEEP_WORKLOADS=a,b] [SWEEP_ENVS=transport=1000000,...] [SWEEP_S=10] python tools/sweep_variants.py LIB [LIB ...]

SWEEP_S: steps per graph replay; SWEEP_FUSED=1/0 forces the fused rollout
kernel on / off (default: where the scenario prefers it).

Each LIB is loaded in a fresh subprocess (SS_LIB_PATH) and every workload
is stepped with device-resident actions; prints the median per-launch time
(CUDA events) and the implied HBM roofline fraction.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import json, sys
sys.path.insert(0, %(root)r)
import numpy as np, torch
from bench import WORKLOADS, bytes_per_env_step, peaks
from paper_2207_03530_b200 import Env, create_scenario
out = {}
for name in %(names)r:
    scen, ov, B = WORKLOADS[name][:3]
    B = %(envs)r.get(name, B)
    env = Env(create_scenario(scen, **ov), B, seed=0, device="cuda:0", validate=False)
    A = len(env.agents); O = env.observations()[0].shape[1]
    acts = [torch.rand((A, B, 2), device="cuda:0") * 2 - 1 for _ in range(2)]
    S = %(S)r
    g = env.step_graph(acts, steps_per_replay=S, fused_rollout=%(fused)s)
    import time
    t_end = time.perf_counter() + 0.5          # clock soak before timing
    k = 0
    while time.perf_counter() < t_end:
        g.step(k % 2); k += 1
        if k % 32 == 0: torch.cuda.synchronize()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for k in range(40): g.step(k % 2)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / (40 * S)
    bpe = bytes_per_env_step(scen, A, len(env.world.entities) - A, O, S if g.fused_rollout else 1)
    out[name] = {"ms": ms, "fused_rollout": g.fused_rollout, "frac": bpe * B / (ms / 1e3) / 1e9 / peaks()["hbm_gbs"]}
print("RESULT " + json.dumps(out))
"""


def main() -> None:
    libs = sys.argv[1:]
    names = os.environ.get("SWEEP_WORKLOADS", "simple_spread,transport,flocking,dispersion,discovery").split(",")
    for lib in libs:
        env = dict(os.environ, SS_LIB_PATH=str(Path(lib).resolve()))
        envs = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in os.environ.get("SWEEP_ENVS", "").split(",") if kv)
        code = (CHILD.replace("%(root)r", repr(str(ROOT))).replace("%(names)r", repr(names))
                .replace("%(envs)r", repr(envs)).replace("%(S)r", os.environ.get("SWEEP_S", "1"))
                .replace("%(fused)s", {"1": "True", "0": "False"}.get(os.environ.get("SWEEP_FUSED", ""), "None")))
        res = subprocess.run([sys.executable, "-c", code],
                             env=env, capture_output=True, text=True)
        line = next((l for l in res.stdout.splitlines() if l.startswith("RESULT ")), None)
        if line is None:
            print(lib, "FAILED", res.stderr[-2000:])
            continue
        d = json.loads(line[7:])
        print(Path(lib).name, " ".join(f"{k}={v['ms']*1e3:.1f}us({v['frac']*100:.0f}%)" for k, v in d.items()),
              flush=True)


if __name__ == "__main__":
    main()
