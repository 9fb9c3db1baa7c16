"""Time the action NaN scan (ss_check_actions) alone and the per-step graph
pieces for a many-agent workload: scan, step kernel, validated step."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2207_03530_b200 import Env, create_scenario  # noqa: E402
from paper_2207_03530_b200 import _native as N  # noqa: E402

dev = torch.device("cuda:0")
name = sys.argv[1] if len(sys.argv) > 1 else "dispersion"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 262144
ov = {"n_agents": 64, "n_food": 64} if name == "dispersion" else ({"n_agents": 64} if name == "discovery" else {})
env = Env(create_scenario(name, **ov), B, seed=0, device=dev, validate=False)
A = len(env.agents)
acts = torch.rand((A, B, 2), device=dev) * 2 - 1
flag = torch.zeros(1, dtype=torch.int32, device=dev)
h = env.scenario.native_handle(env.world)
arr = (N.c_vp * A)(*[acts.data_ptr() + a * B * 8 for a in range(A)])
st = torch.cuda.current_stream(dev).cuda_stream
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for _ in range(3):
    N.check(N.lib().ss_check_actions(h.handle, arr, flag.data_ptr(), st))
s0, s1 = E(), E()
s0.record()
for _ in range(20):
    N.check(N.lib().ss_check_actions(h.handle, arr, flag.data_ptr(), st))
s1.record()
torch.cuda.synchronize()
ms = s0.elapsed_time(s1) / 20
print(f"{name} A={A} B={B}: scan {ms * 1e3:.1f} us for {A * B * 8 / 1e6:.0f} MB ({A * B * 8 / ms / 1e6:.0f} GB/s)")
for validate in (False, True):
    g = env.step_graph([acts, acts.clone()], steps_per_replay=2, validate=validate)
    for k in range(3):
        g.step(k % 2)
    s0.record()
    for k in range(6):
        g.step(k % 2)
    s1.record()
    torch.cuda.synchronize()
    print(f"  step_graph S=2 validate={validate}: {s0.elapsed_time(s1) / 12 * 1e3:.1f} us per step")
    del g
