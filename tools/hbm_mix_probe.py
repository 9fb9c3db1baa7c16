"""Achievable HBM bandwidth by traffic mix on this B200 (context for the rooflines).

    python tools/hbm_mix_probe.py [--gib 4] > profiles/r01/hbm_mix.json

MEASURED_PEAKS.json's denominator is a 1:1 copy (read + write bytes).  The
fused steps are not 1:1: dispersion / discovery write 23-25x more than they
read (observations are 92-94 % of their bytes), simple_spread 104 : 237 B.  This
probe times torch's own streaming kernels over buffers far larger than L2 —
read-only (sum), write-only (fill_), copy — with CUDA events, best of N; a
kernel moving R read and W written bytes then has the mix ceiling
(R + W) / (R / read_gbs + W / write_gbs), printed for the step mixes.  Library
kernels: this is a measurement tool, not the product path.
"""
import argparse
import json

import torch


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = float("inf")
    for _ in range(reps):
        torch.cuda.synchronize()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=4.0)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    n = int(args.gib * (1 << 30)) // 4
    a = torch.empty(n, dtype=torch.float32, device=dev).fill_(1.0)
    b = torch.empty_like(a)
    out = {}
    t = timed(lambda: b.fill_(2.0), args.reps)
    out["write_only"] = {"gbs": 4 * n / t / 1e9, "op": "fill_"}
    t = timed(lambda: a.sum(), args.reps)
    out["read_only"] = {"gbs": 4 * n / t / 1e9, "op": "sum"}
    t = timed(lambda: b.copy_(a), args.reps)
    out["copy_1to1"] = {"gbs": 8 * n / t / 1e9, "op": "copy_ (read + write bytes)"}
    # step mixes (read, write bytes per env-step)
    mixes = {"simple_spread": (104, 237), "dispersion_64x64": (2064, 51473), "discovery_64": (1568, 36129)}
    rb, wb = out["read_only"]["gbs"], out["write_only"]["gbs"]
    out["mix_ceiling_gbs"] = {k: (r + w) / (r / rb + w / wb) for k, (r, w) in mixes.items()}
    props = torch.cuda.get_device_properties(dev)
    out["device"] = {"name": props.name, "sms": props.multi_processor_count, "l2_mb": props.L2_cache_size / 2**20,
                     "buffer_gib": args.gib, "reps": args.reps}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
