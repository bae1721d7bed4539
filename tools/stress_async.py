"""Stress check of the cross-batch pipeline: N batches through sw_warmstart_async (callers on
one or two streams, mixed with synchronous searches every few batches) against sw_warmstart.
  python tools/stress_async.py [n_batches]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2603_07865_b200 import _lib  # noqa: E402
from paper_2603_07865_b200.synth import SynthCache, perturbed_queries, request_durations  # noqa: E402
from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, WarmStartCache, requests  # noqa: E402


def main(nb=40):
    c = SynthCache(60000, 256, 1.0, seed=91, clustered=True)
    wc = WarmStartCache(256, rows_per_entry=1, max_entries=60000, max_batch=512,
                        latent_shape=(4, 64, 16), latent_slots=4096)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    sel, pol = SelectorConfig(8), Policy("exploit")
    L = _lib.lib()
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev).cuda_stream
    side = torch.cuda.Stream(dev)
    B, T = 512, 64
    bad = 0
    outs, chs, refs = [], [], []
    for j in range(nb):
        q = torch.from_numpy(perturbed_queries(c, B, frac_random=0.1, seed=1000 + j)).to(dev)
        rq = requests(np.arange(1 + j * B, 1 + (j + 1) * B, dtype=np.uint64),
                      request_durations(B, 4.0, 10.0, seed=2000 + j), np.full(B, 100, np.int32))
        rd = torch.from_numpy(rq.view(np.uint8)).to(dev)
        ch = torch.zeros(B * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        out = torch.zeros((B, 4, T, 16), dtype=torch.float32, device=dev)
        sj = side.cuda_stream if j % 3 == 1 else st
        _lib.check(L.sw_warmstart_async(wc._h, q.data_ptr(), rd.data_ptr(), B, 3,
                                        C.byref(sel.c()), C.byref(pol.c()), None, 55,
                                        ch.data_ptr(), out.data_ptr(), T, sj), "async")
        if j % 7 == 3:
            wc.search(q.cpu().numpy()[:16], 8)  # a synchronous user in between
        outs.append(out)
        chs.append(ch)
        refs.append((q, rd))
    _lib.check(L.sw_join(wc._h, st), "join")
    torch.cuda.synchronize(dev)
    for j, (q, rd) in enumerate(refs):
        ch = torch.zeros(B * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        out = torch.zeros((B, 4, T, 16), dtype=torch.float32, device=dev)
        _lib.check(L.sw_warmstart(wc._h, q.data_ptr(), rd.data_ptr(), B, 3, C.byref(sel.c()),
                                  C.byref(pol.c()), None, 55, ch.data_ptr(), out.data_ptr(), T,
                                  st), "sync")
        torch.cuda.synchronize(dev)
        a = chs[j].cpu().numpy().view(_lib.CHOICE_DTYPE)
        b = ch.cpu().numpy().view(_lib.CHOICE_DTYPE)
        same = all(np.array_equal(a[f], b[f]) for f in ("hit", "arm", "entry_id", "similarity"))
        same = same and torch.equal(outs[j], out)
        bad += 0 if same else 1
    print(f"stress: {nb} pipelined batches, {bad} mismatching")
    return bad


if __name__ == "__main__":
    sys.exit(1 if main(int(sys.argv[1]) if len(sys.argv) > 1 else 40) else 0)
