"""Helpers shared by the golden-fixture tests (oracle pin and device parity)."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def manifest() -> list[dict]:
    return json.loads((GOLDEN / "manifest.json").read_text())


def load(tag: str) -> dict:
    with np.load(GOLDEN / f"{tag}.npz") as z:
        return {k: z[k] for k in z.files}


def canon_hash(arrs) -> str:
    """sha256 over float32 bytes with -0.0 folded into +0.0 (make_golden.py)."""
    h = hashlib.sha256()
    for a in arrs:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float32) + np.float32(0.0))
        h.update(a.tobytes())
    return h.hexdigest()


def rng_dict(s) -> dict:
    return json.loads(str(s))


def pregen_actions(n_agents: int, batch: int, steps: int, seed: int, u_range: float = 1.0):
    """The reference bench protocol (bench.py:35-47): Philox(seed) uniforms, f32."""
    g = np.random.Generator(np.random.Philox(seed))
    return [[g.uniform(-u_range, u_range, (batch, 2)).astype(np.float32) for _ in range(n_agents)]
            for _ in range(steps)]


def first_mismatch(hashes_got, hashes_want):
    for t, (a, b) in enumerate(zip(hashes_got, hashes_want), start=1):
        if a != b:
            return t
    return None
