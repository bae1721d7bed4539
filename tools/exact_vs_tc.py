"""Small caches: exact fp64 brute force vs the tcgen05 pre-filter, sw_plan device time per batch
size (GPU). Picks the search-path threshold of launch_search_fused (csrc/finish.cu).

  python tools/exact_vs_tc.py
"""
from __future__ import annotations

import ctypes as Cc
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_07865_b200 import _lib  # noqa: E402
from paper_2603_07865_b200.warmstart import (CHOICE_DTYPE, Policy, SelectorConfig,  # noqa: E402
                                             WarmStartCache, requests)


def main():
    dev = torch.device("cuda", 0)
    L_ = _lib.lib()
    D = 512
    res = []
    for n in (256, 512, 1000, 2000, 4000):
        for mode in ("exact", "tc"):
            wc = WarmStartCache(D, rows_per_entry=1, max_entries=n, latent_shape=(8, 256, 16), latent_slots=64,
                                max_batch=1024, exact_only=mode == "exact",
                                tc_always=mode == "tc")
            wc.fill_synthetic(n, first_id=1, seed=1, delta=1.0)
            for B in (1, 8, 64, 256, 1024):
                rng = np.random.default_rng(B)
                q = rng.standard_normal((B, D)).astype(np.float32)
                q /= np.linalg.norm(q, axis=1, keepdims=True)
                qd = torch.from_numpy(q).to(dev)
                rq = requests(np.arange(1, B + 1, dtype=np.uint64), rng.uniform(2.5, 10, B),
                              np.full(B, 200, np.int32))
                rd = torch.from_numpy(rq.view(np.uint8)).to(dev)
                out = torch.empty(B * CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
                st = torch.cuda.current_stream(dev)
                csel, cpol = SelectorConfig(8).c(), Policy("exploit").c()

                def run():
                    _lib.check(L_.sw_plan(wc._h, qd.data_ptr(), rd.data_ptr(), B, 1,
                                          Cc.byref(csel), Cc.byref(cpol), out.data_ptr(),
                                          st.cuda_stream), "sw_plan")
                for _ in range(3):
                    run()
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(20)]
                for a, b in evs:
                    a.record(st)
                    run()
                    b.record(st)
                torch.cuda.synchronize(dev)
                t = sorted(a.elapsed_time(b) for a, b in evs)
                res.append({"n": n, "B": B, "mode": mode, "ms_p50": round(t[10], 4)})
            wc.close()
    for r in res:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
