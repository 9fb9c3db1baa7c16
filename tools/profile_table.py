"""Markdown summary of the bench lines in a profiles round directory.

    python tools/profile_table.py profiles/r02
"""
import json
import sys
from pathlib import Path

ROWS = [("simple_spread", "simple_spread A=3 (1M)"), ("transport", "transport A=4 (100k)"),
        ("transport_1000000", "transport A=4 (1M)"), ("flocking", "flocking A=5 + lidar (100k)"),
        ("flocking_1000000", "flocking A=5 + lidar (1M)"), ("dispersion", "dispersion 64x64 (262144)"),
        ("discovery", "discovery 64 (262144)")]


def last_json(p: Path) -> dict:
    return json.loads(p.read_text().strip().splitlines()[-1])


def main() -> None:
    d = Path(sys.argv[1] if len(sys.argv) > 1 else "profiles/r02")
    print("| workload (envs/GPU) | step kernel | kernel µs/step | validated step µs | `value` agent-steps/s "
          "| HBM frac (kernel) | `e2e` | `cpu_baseline` (1 core, reference) | SM MHz, reasons |")
    print("|---|---|---|---|---|---|---|---|---|")
    for key, label in ROWS:
        p = d / f"bench_{key}.json"
        if not p.exists():
            continue
        b = last_json(p)
        r, c = b["roofline"], b["clocks"]
        kern = f"rollout S={b['steps_per_replay']}" if b.get("fused_rollout") else "per step"
        cpu = b.get("cpu_baseline") or {}
        print(f"| {label} | {kern} | {r['kernel_ms'] * 1e3:.1f} | {r['step_ms'] * 1e3:.1f} | {b['value']:.3g} "
              f"| **{r['frac']:.2f}** | {b['e2e']['value']:.3g} | {cpu.get('value', float('nan')):.3g} "
              f"| {c.get('sm_mhz')} {' '.join(c.get('reasons') or []) or '-'} |")
    refs = []
    for key, _ in ROWS:
        p = d / f"ref_{key}.json"
        if p.exists():
            refs.append(f"{key} {last_json(p)['value']:.3g}")
    print()
    print("Reference arm (`ref_<scenario>.json`, the unmodified reference on the box's host cores): "
          + ", ".join(refs) + " agent-steps/s.")


if __name__ == "__main__":
    main()
