"""B = 1 selector latency breakdown on the 1M x 512 cache (GPU): p50 of sw_plan (search through
select; CUDA events around each call) and, in a second pass with stage events on, the mean of
each stage (prep, score_tc, finish). Prints one JSON line.

  python tools/lat_b1.py [--entries 1000000] [--reps 500]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_07865_b200 import _lib  # noqa: E402
from paper_2603_07865_b200.synth import trained_like_gater  # noqa: E402
from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, WarmStartCache, requests  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--entries", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=500)
    ap.add_argument("--batch", type=int, default=1)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    D, B = 512, args.batch
    wc = WarmStartCache(D, rows_per_entry=1, max_entries=args.entries, max_batch=max(B, 64),
                        latent_shape=None)
    wc.fill_synthetic(args.entries, first_id=1, seed=3, delta=1.0)
    rng = np.random.default_rng(0)
    neg = rng.standard_normal(D).astype(np.float32)
    wc.set_negative(neg / np.linalg.norm(neg))
    th, ps = trained_like_gater()
    wc.set_gater(th, ps, 1.0)
    q = rng.standard_normal((B, D)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    qd = torch.from_numpy(q).to(dev)
    rq = requests(np.arange(1, B + 1, dtype=np.uint64), np.full(B, 5.0), np.full(B, 200, np.int32))
    rd = torch.from_numpy(rq.view(np.uint8)).to(dev)
    ch = torch.zeros(max(B, 64) * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    sel, pol = SelectorConfig(8), Policy("exploit")
    st = torch.cuda.current_stream(dev)
    L = _lib.lib()

    def call():
        _lib.check(L.sw_plan(wc._h, qd.data_ptr(), rd.data_ptr(), B, 1, C.byref(sel.c()),
                             C.byref(pol.c()), ch.data_ptr(), st.cuda_stream), "sw_plan")

    for _ in range(20):
        call()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.reps)]
    for a, b in ev:
        a.record(st)
        call()
        b.record(st)
    torch.cuda.synchronize(dev)
    t = sorted(a.elapsed_time(b) for a, b in ev)
    wc.profile(True)
    wc.profile_reset()
    for _ in range(args.reps):
        call()
    torch.cuda.synchronize(dev)
    wc.profile(False)
    prof = {k: round(v[0] / v[1] * 1e3, 2) for k, v in wc.profile_read().items() if v[1]}
    qs = wc.query_stats(B)
    stats = {"emitted_mean": float(qs[:, 0].mean()), "kept_mean": float(qs[:, 1].mean()),
             "finish_phase_kcycles_mean": [round(float(x) / 1e3, 2) for x in qs[:, 2:6].mean(0)],
             "dbg6_7_kcycles": [round(float(x) / 1e3, 2) for x in qs[:, 6:8].mean(0)]}
    print(json.dumps({"stats": stats, "entries": args.entries, "B": B, "p50_ms": round(t[len(t) // 2], 4),
                      "p99_ms": round(t[int(len(t) * 0.99)], 4), "stage_us": prof,
                      "launch": wc.launch_info()}))


if __name__ == "__main__":
    main()
