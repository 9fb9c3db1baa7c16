"""Does a kernel on one stream start while a large device-to-host copy runs
on another?  Case 1: a torch kernel; case 2: a fused Env.step (this
library's PDL launches); case 3: Env.step(validate=True)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2207_03530_b200 import Env, create_scenario  # noqa: E402

dev = torch.device("cuda:0")
src = torch.empty(181_000_000 // 4, device=dev)
dst = torch.empty(181_000_000 // 4).pin_memory()
x = torch.zeros(1 << 20, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
B = 1_000_000
env = Env(create_scenario("simple_spread"), B, seed=0, device=dev, validate=False)
envv = Env(create_scenario("simple_spread"), B, seed=0, device=dev, validate=True)
acts = torch.rand((3, B, 2), device=dev) * 2 - 1
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def case(name, work):
    torch.cuda.synchronize()
    t0, c0, c1, k0, k1 = E(), E(), E(), E(), E()
    t0.record(s1)
    with torch.cuda.stream(s1):
        c0.record(s1)
        dst.copy_(src, non_blocking=True)
        c1.record(s1)
    with torch.cuda.stream(s2):
        k0.record(s2)
        work()
        k1.record(s2)
    torch.cuda.synchronize()
    print(f"{name:28s} d2h {t0.elapsed_time(c0):6.2f}-{t0.elapsed_time(c1):6.2f}  "
          f"work {t0.elapsed_time(k0):6.2f}-{t0.elapsed_time(k1):6.2f} ms")


for _ in range(2):
    case("torch add_", lambda: x.add_(1.0))
    case("Env.step (device acts)", lambda: env.step(acts))
    case("Env.step validate=True", lambda: envv.step(acts))
    case("Env.step + torch.empty", lambda: (torch.empty((3, B, 14), device=dev), env.step(acts)))
