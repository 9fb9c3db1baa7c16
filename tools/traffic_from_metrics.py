"""Collect per-launch DRAM traffic of the fused kernels from the ncu
summaries (full_<scenario>.metrics.json) into ncu_traffic.json, the file
bench.py reports as roofline.traffic.

    python tools/traffic_from_metrics.py profiles/r01
"""
import json
import sys
from pathlib import Path

ENVS = {"simple_spread": 1_000_000, "transport": 100_000, "flocking": 100_000,
        "dispersion": 262_144, "discovery": 262_144}
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "s": 1.0}


def main() -> None:
    d = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01")
    out = {}
    for s, envs in ENVS.items():
        p = d / f"full_{s}.metrics.json"
        if not p.exists():
            continue
        (kernel, m), = json.loads(p.read_text()).items()
        val = lambda k: float(m[k][0].replace(",", "")) * UNIT.get(m[k][1], 1.0)  # noqa: E731
        out[s] = {"envs": envs, "kernel": kernel,
                  "dram_bytes_per_launch": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
                  "ncu_duration_s": val("gpu__time_duration.sum"),
                  "registers": int(float(m["launch__registers_per_thread"][0]))}
    (d / "ncu_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
