"""Collect per-launch DRAM traffic of the fused kernels from the ncu
summaries (full_<scenario>[_<envs>].metrics.json) into ncu_traffic.json,
keyed by scenario and batch size ("<envs>@rollout<S>" for a capture of the
S-step rollout kernel, full_<scenario>_rollout<S>[_<envs>]) — the file
bench.py reports as roofline.traffic when a capture exists at the bench's
batch size (per step: a rollout launch's bytes / S).

    python tools/traffic_from_metrics.py profiles/r02
"""
import json
import re
import sys
from pathlib import Path

DEFAULT_ENVS = {"simple_spread": 1_000_000, "transport": 100_000, "flocking": 100_000,
                "dispersion": 262_144, "discovery": 262_144}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}


def main() -> None:
    d = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02")
    out = {}
    for p in sorted(d.glob("full_*.metrics.json")):
        m_ = re.fullmatch(r"full_([a-z_]+?)(?:_rollout(\d+))?(?:_(\d+))?\.metrics\.json", p.name)
        if not m_ or m_.group(1) not in DEFAULT_ENVS:
            continue
        s, envs = m_.group(1), int(m_.group(3) or DEFAULT_ENVS[m_.group(1)])
        roll = int(m_.group(2) or 0)
        (kernel, m), = json.loads(p.read_text()).items()
        val = lambda k: float(m[k][0].replace(",", "")) * UNIT.get(m[k][1], 1.0)  # noqa: E731
        out.setdefault(s, {})[f"{envs}@rollout{roll}" if roll else str(envs)] = {
            "kernel": kernel, "capture": p.name, "steps_per_launch": roll or 1,
            "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
            "ncu_duration_s": val("gpu__time_duration.sum"),
            "registers": int(float(m["launch__registers_per_thread"][0]))}
    (d / "ncu_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
