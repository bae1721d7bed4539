"""GPU: request batching (csrc/host/batcher.cpp). Many client threads submit
single requests concurrently (the reference's per-connection handle_request, server.cpp:149);
the batcher groups them into device batches, and every request's choice (and aligned, noised
latent) equals that of one sw_plan / sw_warmstart over all the requests — draws and noise are
keyed by request id, so the grouping never changes a result."""
import threading

import numpy as np
import pytest

from paper_2603_07865_b200.synth import SynthCache, perturbed_queries, request_durations

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FIELDS = ["hit", "arm", "steps_skipped", "n_hits", "entry_id", "similarity", "pick", "flags",
          "t_out", "slot"]


def _cache(n, latent=None):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    c = SynthCache(n, 128, 1.0, seed=61, clustered=True)
    wc = WarmStartCache(128, rows_per_entry=1, max_entries=n, max_batch=512,
                        latent_shape=latent, latent_slots=min(n, 2048))
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    return c, wc


def _run_clients(b, q, reqs, n_threads, want_latent=False):
    out = [None] * q.shape[0]

    def client(t):
        for i in range(t, q.shape[0], n_threads):
            out[i] = b.submit(q[i], reqs[i:i + 1], want_latent)

    th = [threading.Thread(target=client, args=(t,)) for t in range(n_threads)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    return out


def test_batcher_matches_one_batch():
    from paper_2603_07865_b200.warmstart import Batcher, Policy, SelectorConfig, requests
    c, wc = _cache(20000)
    B = 512
    q = perturbed_queries(c, B, frac_random=0.1)
    reqs = requests(np.arange(1000, 1000 + B, dtype=np.uint64), request_durations(B),
                    np.full(B, 200, np.int32))
    sel, pol = SelectorConfig(8), Policy("exploit")
    ref = wc.choices(wc.plan(q, reqs, seed=3, sel=sel, policy=pol))
    b = Batcher(wc, max_batch=256, max_wait_us=2000, seed=3, sel=sel, policy=pol)
    got = _run_clients(b, q, reqs, 64)
    st = b.stats()
    b.close()
    assert st["requests"] == B and st["batches"] < B  # requests were grouped
    for i in range(B):
        for f in FIELDS[:-2]:
            assert got[i][f] == ref[f][i], (i, f)


def test_batcher_latents_match_warmstart():
    from paper_2603_07865_b200.warmstart import Batcher, Policy, SelectorConfig, requests
    from paper_2603_07865_b200.warmstart import WarmStartCache
    c = SynthCache(6000, 128, 1.0, seed=62, clustered=True)
    latent = (4, 64, 16)
    wc = WarmStartCache(128, rows_per_entry=1, max_entries=6000, max_batch=256,
                        latent_shape=latent, latent_slots=6000)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    B = 128
    q = perturbed_queries(c, B, frac_random=0.1)
    reqs = requests(np.arange(1, B + 1, dtype=np.uint64), request_durations(B, 1.0, 2.5),
                    np.full(B, 100, np.int32))
    sel, pol = SelectorConfig(8), Policy("rule")
    buf = wc.plan(q, reqs, seed=5, sel=sel, policy=pol)
    ref_lat = wc.align_noise(buf, reqs, 64, philox_seed=77).cpu().numpy()
    ref = wc.choices(buf)
    b = Batcher(wc, max_batch=64, max_wait_us=1000, seed=5, sel=sel, policy=pol, philox_seed=77,
                t_out_max=64, with_latent=True)
    got = _run_clients(b, q, reqs, 16, want_latent=True)
    b.close()
    for i in range(B):
        ch, lat = got[i]
        assert ch["entry_id"] == ref["entry_id"][i] and ch["arm"] == ref["arm"][i]
        if ref["hit"][i]:
            np.testing.assert_array_equal(lat, ref_lat[i])
