"""Summarise an .ncu-rep into small text/CSV files (run where ncu is installed).

    python tools/ncu_summary.py REPORT.ncu-rep OUT_PREFIX

Writes OUT_PREFIX.details.csv (all sections), OUT_PREFIX.metrics.json (the
roofline-relevant raw metrics) and OUT_PREFIX.hot.txt (source lines ranked
by warp-stall samples and executed instructions).
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
]


def ncu(*args) -> str:
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main() -> None:
    rep, prefix = sys.argv[1], sys.argv[2]
    det = ncu("-i", rep, "--page", "details", "--csv")
    open(prefix + ".details.csv", "w").write(det)
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    out = {}
    if len(raw) >= 3:
        hdr, units = raw[0], raw[1]
        for row in raw[2:]:
            name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "kernel"
            m = {k: (row[hdr.index(k)], units[hdr.index(k)]) for k in KEYS if k in hdr}
            # warp-stall reasons (cycles per issued instruction, by reason)
            for j, k in enumerate(hdr):
                if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                    m[k] = (row[j], units[j])
            out[name] = m
    json.dump(out, open(prefix + ".metrics.json", "w"), indent=1)
    src = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    rows, cur, hdr = [], None, None
    for r in csv.reader(io.StringIO(src)):
        if not r:
            continue
        if r[0] in ("File Path", "File Name"):
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) >= 8 and r[2] == "-":
            try:
                rows.append((int(r[4] or 0), int(r[7] or 0), cur, r[0], r[1].strip()[:100]))
            except ValueError:
                pass
    tot = sum(x[0] for x in rows) or 1
    ti = sum(x[1] for x in rows) or 1
    with open(prefix + ".hot.txt", "w") as f:
        f.write(f"stall samples {tot}, warp instructions {ti}\n")
        for s, ie, fl, ln, text in sorted(rows, reverse=True)[:40]:
            f.write(f"{100*s/tot:5.1f}% stall {100*ie/ti:5.1f}% inst  {fl}:{ln}  {text}\n")


if __name__ == "__main__":
    main()
