"""Multi-process sharding logic on CPU (gloo, world_size 2).

The step itself has no collective; what needs checking is the host logic
around it: contiguous shard ranges, the episode-statistics all-reduce, and
the masked-reset offsets (all_gather of per-shard counts) that keep the
global Philox draw order — restated here with numpy's Philox and compared
with the oracle's sequential resets of the whole batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import swarm_oracle as O
from paper_2207_03530_b200.parallel import EpisodeStats, global_mask_offsets, shard_range


def test_shard_ranges_cover_batch():
    for Bg in (1, 7, 64, 1000, 1_000_003):
        for ws in (1, 2, 3, 8):
            spans = [shard_range(r, ws, Bg) for r in range(ws)]
            assert spans[0][0] == 0
            for (o, c), (o2, _) in zip(spans, spans[1:]):
                assert o + c == o2
            assert sum(c for _, c in spans) == Bg
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, Bg, mask_np, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    off, cnt = shard_range(rank, ws, Bg)
    local = torch.tensor([int(mask_np[off:off + cnt].sum())], dtype=torch.int64)
    base, total = global_mask_offsets(local)
    st = EpisodeStats(cnt, "cpu")
    rew = [torch.full((cnt,), float(rank + 1)), torch.full((cnt,), float(rank + 3))]
    st.update(rew, torch.zeros(cnt, dtype=torch.bool))
    red = st.reduce()
    q.put((rank, off, cnt, int(base.item()), int(total.item()), red))
    dist.destroy_process_group()


def test_gloo_offsets_and_stats():
    Bg, ws = 37, 2
    mask = np.zeros(Bg, dtype=bool)
    mask[[0, 5, 17, 18, 19, 30, 36]] = True
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, Bg, mask, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, off, cnt, base, total, red in out:
        assert base == int(mask[:off].sum())
        assert total == int(mask.sum())
        # mean over agents of (rank+1, rank+3) = rank + 2 per env
        want = sum((r + 2) * shard_range(r, ws, Bg)[1] for r in range(ws)) / Bg
        assert red["mean_return"] == pytest.approx(want)
        assert red["envs"] == Bg


def _draws(state, idx):
    """numpy Philox 64-bit draws at absolute indices idx from `state` (ss_math.cuh philox_draw)."""
    g = np.random.Generator(np.random.Philox())
    g.bit_generator.state = state
    n = int(np.max(idx)) + 1
    vals = g.bit_generator.random_raw(n)
    return vals[np.asarray(idx)]


def test_sharded_masked_reset_draw_order_matches_sequential_resets():
    """The kernel's rank formula with per-shard bases reproduces the global
    sequential reset(i) stream (restated on the host with numpy's Philox)."""
    Bg, ws = 23, 3
    env = O.OracleEnv("simple_spread", Bg, seed=4)
    mask = np.zeros(Bg, dtype=bool)
    mask[[2, 3, 9, 15, 22]] = True
    st0 = env.rng.bit_generator.state
    S = 2 * 3   # scatter ops (6 entities)
    want_px = None
    ref = O.OracleEnv("simple_spread", Bg, seed=4)
    ref.reset_mask(mask)
    got = {}
    for r in range(ws):
        off, cnt = shard_range(r, ws, Bg)
        base = int(mask[:off].sum())
        local = np.flatnonzero(mask[off:off + cnt])
        for j, e in enumerate(local):
            rank = base + j
            u = _draws(st0, [rank * 2 * S + 2 * s + a for s in range(S) for a in (0, 1)])
            d = (u >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
            got[off + e] = (-1.0 + 2.0 * d).astype(np.float32)
    for e, vals in got.items():
        for s in range(S):
            assert vals[2 * s] == ref.ws.px[s][e]
            assert vals[2 * s + 1] == ref.ws.py[s][e]
