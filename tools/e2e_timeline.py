"""Per-step timeline of bench.e2e_rate's loop (CUDA events on both streams):
when each step's compute finishes and when its device-to-host copy starts
and ends, relative to the first step.  `python tools/e2e_timeline.py side`
steps on a side stream instead of the legacy default stream."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2207_03530_b200 import Env, create_scenario  # noqa: E402

dev = torch.device("cuda:0")
side = "side" in sys.argv[1:]
zero_copy = "zc" in sys.argv[1:]   # the kernels read the pinned host actions in place (UVA)
B, A = 1_000_000, 3
host_acts = [[torch.from_numpy(np.random.default_rng(7 + k).uniform(-1, 1, (B, 2)).astype(np.float32)).pin_memory()
              for _ in range(A)] for k in range(4)]
env = Env(create_scenario("simple_spread", n_agents=A), B, seed=0, device=dev, validate="novalidate" not in sys.argv[1:])
O = len(env.observations()[0][0])
if zero_copy:
    ref = Env(create_scenario("simple_spread", n_agents=A), B, seed=0, device=dev, validate=True)
    env._fast_actions = lambda raw: list(raw)
    r0, r1 = env.step(host_acts[0]), ref.step(host_acts[0])
    assert all(torch.equal(x, y) for x, y in zip(r0.obs + r0.rewards, r1.obs + r1.rewards))
    print("zero-copy step equals the copying step")
comp = torch.cuda.Stream(dev) if side else torch.cuda.current_stream(dev)
copy = torch.cuda.Stream(dev)
obs_h = [torch.empty((A, B, O), dtype=torch.float32).pin_memory() for _ in range(2)]
rew_h = [torch.empty((A, B), dtype=torch.float32).pin_memory() for _ in range(2)]
done_h = [torch.empty(B, dtype=torch.bool).pin_memory() for _ in range(2)]
ready = [None, None]
marks = []
t_host = []
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
prof = None
if "prof" in sys.argv[1:]:
    import cProfile
    prof = cProfile.Profile()
    prof.enable()
start = E()
start.record(comp)
t0 = time.perf_counter()
for k in range(12):
    j = k % 2
    th0 = time.perf_counter()
    if ready[j] is not None:
        ready[j].synchronize()
    th1 = time.perf_counter()
    e_in = E(); e_in.record(comp)
    with torch.cuda.stream(comp):
        res = env.step(host_acts[k % 4])
    e_st = E(); e_st.record(comp)
    th2 = time.perf_counter()
    copy.wait_event(e_st)
    c0 = E(); c0.record(copy)
    with torch.cuda.stream(copy):
        for a in range(A):
            obs_h[j][a].copy_(res.obs[a], non_blocking=True)
            res.obs[a].record_stream(copy)
        for a in range(A):
            rew_h[j][a].copy_(res.rewards[a], non_blocking=True)
            res.rewards[a].record_stream(copy)
        done_h[j].copy_(res.dones, non_blocking=True)
        res.dones.record_stream(copy)
    c1 = E(); c1.record(copy)
    ready[j] = c1
    marks.append((e_in, e_st, c0, c1))
    t_host.append((th0 - t0, th1 - t0, th2 - t0))
torch.cuda.synchronize()
if prof is not None:
    import pstats
    prof.disable()
    pstats.Stats(prof).sort_stats("tottime").print_stats(8)
st = torch.cuda.memory_stats(dev)
print({k: v for k, v in st.items() if k in ("num_alloc_retries", "num_device_alloc", "num_device_free",
                                             "segment.all.allocated", "segment.all.freed", "num_sync_all_streams")})
for k, ((a, b, c, d), (h0, h1, h2)) in enumerate(zip(marks, t_host)):
    print(f"step {k:2d}: compute {start.elapsed_time(a):7.2f}-{start.elapsed_time(b):7.2f}  "
          f"d2h {start.elapsed_time(c):7.2f}-{start.elapsed_time(d):7.2f} ms   "
          f"host wait {1e3*h0:7.2f}-{1e3*h1:7.2f} step-ret {1e3*h2:7.2f}")
