"""Where the config-5 mutation time goes (GPU): IVF rebuild, admit (host pyramid derivation +
arena insert + IVF list assignment), evict, each timed on its own at 1K capacity x 7 rows.

  python tools/time_mutations.py
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_07865_b200.warmstart import CacheManager, WarmStartCache  # noqa: E402


def main():
    dim, cap = 512, 1024
    rng = np.random.default_rng(1)
    embs = rng.standard_normal((4000, dim)).astype(np.float32)
    embs /= np.linalg.norm(embs, axis=1, keepdims=True)
    res = {}
    for ivf in (False, True):
        wc = WarmStartCache(dim, rows_per_entry=7, max_entries=cap + 8, max_batch=64,
                            latent_shape=None)
        if ivf:
            wc.ivf_configure(64, 8, 1 << 40, 5)  # no automatic rebuilds while timing
        cm = CacheManager(wc, capacity=cap, pyramid_delta=0.25, embedding_seed=3)
        t = time.perf_counter()
        for i in range(cap):
            cm.admit(embs[i], 8.0, embs[i], 0.9, 0.0)
        fill = time.perf_counter() - t
        r = {"admit_ms": round(1e3 * fill / cap, 4)}
        if ivf:
            t = time.perf_counter()
            for _ in range(3):
                wc.ivf_rebuild()
            r["rebuild_ms"] = round(1e3 * (time.perf_counter() - t) / 3, 2)
        t = time.perf_counter()
        for i in range(200):  # admit over capacity: insert + evict one
            cm.admit(embs[cap + i], 8.0, embs[cap + i], 0.9, 2.0 + 0.01 * i)
        r["admit_evict_ms"] = round(1e3 * (time.perf_counter() - t) / 200, 4)
        ids = cm.ids()[:200]
        t = time.perf_counter()
        for i in ids:
            wc.remove(int(i))
        r["remove_ms"] = round(1e3 * (time.perf_counter() - t) / 200, 4)
        res["ivf" if ivf else "exhaustive"] = r
    print(json.dumps(res))


if __name__ == "__main__":
    main()
