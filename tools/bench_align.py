"""K4 align + noise timed alone, cold L2, fresh choices and outputs every rep (GPU).

Each rep aligns a different batch of 1024 random choices (slots spread over the latent arena,
segments and durations as the bench draws them) into a different output buffer, with a 512 MiB
read-only L2 flush between reps outside the timed events. Prints one JSON line with the per-mode
algorithmic bytes, durations and fraction of MEASURED_PEAKS.json's HBM bandwidth.
Bit-exactness of both modes is covered by tests/test_gpu_parity.py.

  python tools/bench_align.py [--reps 20] [--slots 65536]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_07865_b200 import _lib  # noqa: E402
from paper_2603_07865_b200.warmstart import WarmStartCache, requests  # noqa: E402


def make_batch(rng, B, n_entries, T_total=200):
    ch = np.zeros(B, _lib.CHOICE_DTYPE)
    ch["hit"] = 1
    ch["slot"] = rng.integers(0, n_entries, B)
    ch["entry_id"] = ch["slot"] + 1
    dur = rng.uniform(4.0, 12.0, B)  # fill_synthetic's clip durations
    ch["start_s"] = rng.uniform(0.0, 0.5, B) * dur
    ch["length_s"] = np.minimum(rng.uniform(0.25, 1.0, B) * dur, dur - ch["start_s"])
    ch["steps_skipped"] = rng.integers(10, 150, B)
    L = rng.uniform(2.5, 10.0, B)
    ids = rng.integers(1, 1 << 62, B).astype(np.uint64)
    rq = requests(ids, L, np.full(B, T_total, np.int32))
    return ch, rq


def alg_bytes(ch, rq, C_, T_, F_, fps=25.0, eps=False):
    fr = lambda x: np.floor(x * fps + 0.5)
    t_out = np.minimum(fr(rq["duration_s"]), T_)
    lo = fr(ch["start_s"])
    hi = fr(ch["start_s"] + ch["length_s"])
    t_seg = np.maximum(np.minimum(hi, T_) - np.minimum(lo, T_), 0)
    b = 4 * C_ * F_ * (t_out + np.minimum(t_seg, t_out))
    if eps:
        b = b + 4 * C_ * F_ * t_out
    return float(b.sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--slots", type=int, default=65536)
    ap.add_argument("--batch", type=int, default=1024)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    B, C_, T_, F_ = args.batch, 8, 256, 16
    n_entries = args.slots
    wc = WarmStartCache(512, rows_per_entry=1, max_entries=n_entries, max_batch=B,
                        latent_slots=args.slots)
    wc.fill_synthetic(n_entries, first_id=1, seed=3, delta=1.0)
    torch.cuda.synchronize(dev)
    L_ = _lib.lib()
    st = torch.cuda.current_stream(dev)
    sp = st.cuda_stream
    rng = np.random.default_rng(11)
    nbuf = 4
    outs = [torch.empty((B, C_, T_, F_), dtype=torch.float32, device=dev) for _ in range(nbuf)]
    batches = [make_batch(rng, B, n_entries) for _ in range(nbuf)]
    d_batches = [(torch.from_numpy(c.view(np.uint8)).to(dev), torch.from_numpy(r.view(np.uint8)).to(dev))
                 for c, r in batches]
    eps_t = torch.randn((B, C_, T_, F_), dtype=torch.float32, device=dev)
    # L2 flush by READING 512 MiB (clean lines, as after the scoring kernel's arena stream; a
    # write-based flush would leave ~126 MB of dirty lines for the timed kernel to write back)
    flush = torch.ones(1 << 27, dtype=torch.float32, device=dev)
    sink = torch.empty(1, dtype=torch.float32, device=dev)

    def launch(j, eps):
        c, r = d_batches[j]
        _lib.check(L_.sw_align_noise(wc._h, c.data_ptr(), r.data_ptr(), B,
                                     eps.data_ptr() if eps is not None else None, 1234,
                                     outs[j].data_ptr(), T_, sp), "sw_align_noise")

    res = {}
    for mode in ("philox", "eps"):
        eps = eps_t if mode == "eps" else None
        for j in range(nbuf):
            launch(j, eps)
        times = []
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.reps)]
        for i in range(args.reps):
            torch.sum(flush, dim=0, out=sink)
            evs[i][0].record(st)
            launch(i % nbuf, eps)
            evs[i][1].record(st)
        torch.cuda.synchronize(dev)
        times = [a.elapsed_time(b) for a, b in evs]
        byt = np.mean([alg_bytes(batches[i % nbuf][0], batches[i % nbuf][1], C_, T_, F_,
                                 eps=(mode == "eps")) for i in range(args.reps)])
        ms = float(np.median(times))
        res[mode] = {"ms_median": round(ms, 5), "ms_min": round(min(times), 5),
                     "alg_bytes": byt, "GBps": round(byt / (ms / 1e3) / 1e9, 1)}
    peaks = {}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        peaks = json.load(open(p))
    hbm = peaks.get("hbm_gbs", 6451.0)
    for m in res:
        res[m]["frac"] = round(res[m]["GBps"] / hbm, 4)
    print(json.dumps({"align_alone": res, "hbm_peak_GBps": hbm, "B": B, "reps": args.reps,
                      "cold_l2": True, "fresh_outputs": nbuf}))


if __name__ == "__main__":
    main()
