"""Side measurements of bench.py (one GPU, after the headline timed region).

  cache_size_sweep  the BASELINE metric's "vs cache size" axis: warm-start requests/s of the
                    config-3 step (B = 1024, top-8, exploit, align + Philox noise) on caches of
                    1K .. 10M entries; the 10M point is config 4's single-GPU point
  config4_shard     config 4's per-GPU work: the entry-sharded step (local top-k -> gather ->
                    merge + replicated select -> owner align) on a 1.25M-entry shard (10M / 8)
  config1           BASELINE config 1: 1K entries x 7 pyramid rows, ONE request, top-1 +
                    duration gate + gater + align + noise 8x256x16 — p50 latency
  config5           BASELINE config 5: Cache Manager trace replay (synth_workload 2000 x 512,
                    1K capacity, IVF 64/8, 64-request lookup batches) vs the reference's own
                    Pipeline::replay on the same trace, same box
  parity_sample     the timed batch's choices (all of them by default) checked against the C restatement
                    (oracle, test infrastructure) on the exported arena

Everything here is measured with CUDA events on the launching stream (device time) or with
the wall clock where the quantity is a host loop (replay, host-buffer latency); each result
says which.
"""
from __future__ import annotations

import ctypes as Cc
import os
import time

import numpy as np

D = 512
LATENT = (8, 256, 16)


def _neg_gater():
    from paper_2603_07865_b200.synth import normalize_rows, trained_like_gater
    neg = normalize_rows(np.random.default_rng(4242).standard_normal((1, D)))[0]
    th, ps = trained_like_gater()
    return neg, th, ps


def _queries(wc, n, B, R, rng, pools=2):
    from paper_2603_07865_b200.synth import normalize_rows
    qs = []
    for _ in range(pools):
        ids = rng.integers(1, n + 1, B)
        base = np.stack([wc.read_rows(int(i), R)[0] for i in ids]).astype(np.float64)
        g = rng.standard_normal((B, D))
        g /= np.linalg.norm(g, axis=1, keepdims=True)
        q = normalize_rows(base + 0.3 * g)
        m = rng.random(B) < 0.1
        q[m] = normalize_rows(rng.standard_normal((int(m.sum()), D)))
        qs.append(q)
    return np.stack(qs)


def sweep_point(n, B=1024, K=8, steps=20, warm=3, device=0, peak=None):
    """Pipelined warm-start steps (sw_warmstart_async) on an n-entry cache; device time."""
    import torch

    from paper_2603_07865_b200 import _lib
    from paper_2603_07865_b200.warmstart import (CHOICE_DTYPE, Policy, SelectorConfig,
                                                 WarmStartCache, requests)
    dev = torch.device("cuda", device)
    L_ = _lib.lib()
    t0 = time.time()
    wc = WarmStartCache(D, rows_per_entry=1, max_entries=n, latent_shape=LATENT, max_batch=B,
                        latent_slots=min(65536, n), device=device)
    neg, th, ps = _neg_gater()
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    wc.fill_synthetic(n, first_id=1, seed=1, delta=1.0)
    torch.cuda.synchronize(dev)
    setup = time.time() - t0
    qpool = torch.from_numpy(_queries(wc, n, B, 1, np.random.default_rng(17))).to(dev)
    L = np.random.default_rng(11).uniform(2.5, 10.0, B)
    reqs = torch.from_numpy(np.stack([requests(np.arange(s * B + 1, (s + 1) * B + 1,
                                                         dtype=np.uint64), L,
                                               np.full(B, 200, np.int32)).view(np.uint8)
                                      for s in range(2)])).to(dev)
    csel, cpol = SelectorConfig(K).c(), Policy("exploit").c()
    C_, T_, F_ = LATENT
    out = torch.empty((B, C_, T_, F_), dtype=torch.float32, device=dev)
    ring = [torch.empty((B * CHOICE_DTYPE.itemsize,), dtype=torch.uint8, device=dev)
            for _ in range(2)]
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream

    def step(i):
        _lib.check(L_.sw_warmstart_async(wc._h, qpool[i % 2].data_ptr(), reqs[i % 2].data_ptr(),
                                         B, 1, Cc.byref(csel), Cc.byref(cpol), None, 1234,
                                         ring[i % 2].data_ptr(), out.data_ptr(), T_, sp),
                   "sw_warmstart_async")

    for i in range(warm):
        step(i)
    _lib.check(L_.sw_join(wc._h, sp), "sw_join")
    torch.cuda.synchronize(dev)
    wc.profile(True, stages=["score_tc"])
    wc.profile_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        step(i)
    _lib.check(L_.sw_join(wc._h, sp), "sw_join")
    e1.record(stream)
    torch.cuda.synchronize(dev)
    wc.profile(False)
    ms = e0.elapsed_time(e1) / steps
    sc_ms, sc_n = wc.profile_read()["score_tc"]
    tc = sc_n > 0
    score_ms = sc_ms / sc_n if tc else None
    flops = 2.0 * B * n * D
    ch = wc.choices(ring[(steps - 1) % 2])
    res = {"entries": n, "requests_per_s": round(B / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
           "scoring": "tcgen05 pre-filter + fp64 rescoring" if tc else "exact fp64 only",
           "score_ms": round(score_ms, 4) if tc else None,
           "score_tflops": round(flops / (score_ms / 1e3) / 1e12, 1) if tc else None,
           "score_frac_of_peak": round(flops / (score_ms / 1e3) / 1e12 / peak, 4) if tc and peak else None,
           "hit_rate": round(float(ch["hit"].mean()), 4),
           "fallback_queries": wc.overflow_fallbacks(), "setup_s": round(setup, 1),
           "timing": f"device (CUDA events), {steps} pipelined steps of {B} requests"}
    wc.close()
    del out, qpool
    torch.cuda.empty_cache()
    return res


def cpu_reference_point(n, nthreads, queries_per_thread=1):
    """The unmodified reference plan flow on all host threads over an n-entry host cache."""
    import bench
    run, _ = bench.reference_sample(n, nthreads * queries_per_thread, nthreads)
    t = time.perf_counter()
    run()
    el = time.perf_counter() - t
    return round(nthreads * queries_per_thread / el, 3)


def config4_shard(n_local=1_250_000, B=1024, K=8, steps=20, warm=3, device=0):
    """Config 4's per-GPU step at 1.25M entries (10M / 8): sw_local_topk_async on the scoring
    stream, then on the context's stream the (1-rank) gather, sw_merge_select and the owner
    align — the pipelined sharded step bench.py runs under torchrun, measured on one GPU."""
    import torch

    from paper_2603_07865_b200 import _lib
    from paper_2603_07865_b200.warmstart import (CHOICE_DTYPE, Policy, SelectorConfig,
                                                 WarmStartCache, requests)
    dev = torch.device("cuda", device)
    L_ = _lib.lib()
    wc = WarmStartCache(D, rows_per_entry=1, max_entries=n_local, latent_shape=LATENT,
                        max_batch=B, latent_slots=min(65536, n_local), device=device)
    neg, th, ps = _neg_gater()
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    wc.fill_synthetic(n_local, first_id=1, seed=1, delta=1.0)
    qpool = torch.from_numpy(_queries(wc, n_local, B, 1, np.random.default_rng(19))).to(dev)
    L = np.random.default_rng(11).uniform(2.5, 10.0, B)
    reqs = torch.from_numpy(requests(np.arange(1, B + 1, dtype=np.uint64), L,
                                     np.full(B, 200, np.int32)).view(np.uint8)).to(dev)
    csel, cpol = SelectorConfig(K).c(), Policy("exploit").c()
    C_, T_, F_ = LATENT
    out = torch.empty((B, C_, T_, F_), dtype=torch.float32, device=dev)
    rec = torch.empty((B * K * _lib.HIT_RECORD_BYTES,), dtype=torch.uint8, device=dev)
    rec_all = torch.empty_like(rec)
    nl = torch.empty((B,), dtype=torch.int32, device=dev)
    n_all = torch.empty_like(nl)
    ring = [torch.empty((B * CHOICE_DTYPE.itemsize,), dtype=torch.uint8, device=dev)
            for _ in range(2)]
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    a_ptr = Cc.c_void_p()
    _lib.check(L_.sw_async_stream(wc._h, Cc.byref(a_ptr)), "sw_async_stream")
    a_stream = torch.cuda.ExternalStream(a_ptr.value, device=dev)

    def step(i):
        q = qpool[i % 2]
        _lib.check(L_.sw_local_topk_async(wc._h, q.data_ptr(), B, K, 0, rec.data_ptr(),
                                          nl.data_ptr(), sp), "sw_local_topk_async")
        with torch.cuda.stream(a_stream):
            rec_all.copy_(rec)
            n_all.copy_(nl)
        _lib.check(L_.sw_merge_select(wc._h, rec_all.data_ptr(), n_all.data_ptr(), 1,
                                      q.data_ptr(), reqs.data_ptr(), B, K, 1, Cc.byref(csel),
                                      Cc.byref(cpol), ring[i % 2].data_ptr(), a_ptr),
                   "sw_merge_select")
        _lib.check(L_.sw_align_noise_owned(wc._h, ring[i % 2].data_ptr(), reqs.data_ptr(), B, 0,
                                           None, 1234, out.data_ptr(), T_, a_ptr), "align")

    for i in range(warm):
        step(i)
    _lib.check(L_.sw_join(wc._h, sp), "sw_join")
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        step(i)
    _lib.check(L_.sw_join(wc._h, sp), "sw_join")
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    wc.close()
    return {"entries_per_gpu": n_local, "ms_per_step": round(ms, 4),
            "requests_per_s_per_gpu_step": round(B / (ms / 1e3), 1),
            "note": "per-GPU sharded step of config 4 (10M entries / 8 GPUs) measured on one "
                    "B200; the 1 MiB-per-rank all-gather is a copy at world 1",
            "timing": f"device (CUDA events), {steps} pipelined steps"}


def config1_latency(reps=500, device=0, cpu=True):
    """BASELINE config 1: 1K-entry cache, 512-d, pyramid delta 1/4 (7 rows per entry), ONE
    request, top-1 + duration gate + Skip Gater + align + Philox noise on 8x256x16 latents."""
    import torch

    from paper_2603_07865_b200 import _lib
    from paper_2603_07865_b200.synth import SynthCache, perturbed_queries
    from paper_2603_07865_b200.warmstart import (CHOICE_DTYPE, Policy, SelectorConfig,
                                                 WarmStartCache, requests)
    dev = torch.device("cuda", device)
    L_ = _lib.lib()
    c = SynthCache(1000, D, 0.25, seed=1)
    wc = WarmStartCache(D, rows_per_entry=7, max_entries=1000, latent_shape=LATENT, max_batch=1,
                        device=device)
    neg, th, ps = _neg_gater()
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    rng = np.random.default_rng(3)
    lat = rng.standard_normal((1000, LATENT[0], LATENT[1], LATENT[2])).astype(np.float32)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths,
                    latents=lat, lat_off=np.arange(1000, dtype=np.int64) * lat[0].size,
                    t_src=np.full(1000, LATENT[1], np.int32))
    q = perturbed_queries(c, reps, frac_random=0.1)
    L = rng.uniform(2.5, 10.0, reps)
    rq = requests(np.arange(1, reps + 1, dtype=np.uint64), L, np.full(reps, 200, np.int32))
    qd = torch.from_numpy(q).to(dev)
    rd = torch.from_numpy(rq.view(np.uint8).reshape(reps, -1)).to(dev)
    csel, cpol = SelectorConfig(1).c(), Policy("exploit").c()
    C_, T_, F_ = LATENT
    out = torch.empty((1, C_, T_, F_), dtype=torch.float32, device=dev)
    ch = torch.empty((CHOICE_DTYPE.itemsize,), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for i in range(10):
        _lib.check(L_.sw_warmstart(wc._h, qd[i].data_ptr(), rd[i].data_ptr(), 1, 1,
                                   Cc.byref(csel), Cc.byref(cpol), None, 1234, ch.data_ptr(),
                                   out.data_ptr(), T_, sp), "sw_warmstart")
    torch.cuda.synchronize(dev)
    for i in range(reps):
        ev[i][0].record(stream)
        _lib.check(L_.sw_warmstart(wc._h, qd[i].data_ptr(), rd[i].data_ptr(), 1, 1,
                                   Cc.byref(csel), Cc.byref(cpol), None, 1234, ch.data_ptr(),
                                   out.data_ptr(), T_, sp), "sw_warmstart")
        ev[i][1].record(stream)
    torch.cuda.synchronize(dev)
    dt = sorted(a.elapsed_time(b) for a, b in ev)
    # end to end from host buffers: H2D prompt + request, the whole path, D2H of the choice
    qh = np.ascontiguousarray(q, np.float32)
    chh = np.zeros(1, CHOICE_DTYPE)
    wall = []
    for i in range(reps):
        t = time.perf_counter()
        _lib.check(L_.sw_warmstart_host(wc._h, qh[i].ctypes.data, rq[i:i + 1].ctypes.data, 1, 1,
                                        Cc.byref(csel), Cc.byref(cpol), 1234, chh.ctypes.data,
                                        out.data_ptr(), T_, sp), "sw_warmstart_host")
        wall.append(time.perf_counter() - t)
    wall.sort()
    res = {"workload": "config1: 1K entries x 7 pyramid rows (delta 1/4), 512-d, B = 1, top-1 + "
                       "gate + exploit gater + t* + align + Philox noise 8x256x16",
           "p50_ms": round(dt[len(dt) // 2], 4), "p99_ms": round(dt[int(len(dt) * 0.99)], 4),
           "timing": "device (CUDA events around one sw_warmstart)",
           "e2e_p50_ms": round(1e3 * wall[len(wall) // 2], 4),
           "e2e_p99_ms": round(1e3 * wall[int(len(wall) * 0.99)], 4),
           "e2e_timing": "wall clock of one blocking sw_warmstart_host (H2D prompt + request, "
                         "D2H choice)"}
    if cpu:
        import oracle
        ref = oracle.Ref()
        ar = oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
        idx = ref.index(ar)
        n = 200
        t = time.perf_counter()
        idx.plan_batch(neg, q[:n], L[:n], np.arange(1, n + 1, dtype=np.uint64),
                       np.full(n, 200, np.int32), top_k=1, policy="exploit", theta=th, psi=ps,
                       nthreads=1)
        res["cpu_reference_ms_per_request"] = round(1e3 * (time.perf_counter() - t) / n, 4)
        res["cpu_reference_note"] = ("unmodified reference plan flow (search + gate + select + "
                                     "gater + t*; no noising exists there), 1 thread, 200 requests")
    wc.close()
    return res


def config5_replay(n=2000, batch=64, device=0, cpu=True):
    """BASELINE config 5 through swr_replay vs the reference's own Pipeline::replay."""
    from paper_2603_07865_b200.synth import trained_like_gater
    from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, TraceReplay, synth_workload
    p, d, a, t = synth_workload(n, D, 7)
    th, ps = trained_like_gater()
    res = {"workload": f"config5: synth_workload({n} prompts, {D}-d, dup 0.9) replayed at 1K "
                       f"capacity, IVF 64 lists / nprobe 8 / rebuild 1024, delta 1/4, exploit",
           "timing": "wall clock of the whole replay (lookups + mutations + maintenance)"}
    runs = {}
    for b in (1, batch):
        tr = TraceReplay(D, capacity=1024, seed=1, policy=Policy("exploit"),
                         sel=SelectorConfig(8), theta=th, psi=ps, max_batch=max(b, 1),
                         device=device)
        out, st = tr.run(p, d, a, t, batch=b)
        tr.close()
        runs[b] = (out, st)
        res[f"batch{b}"] = {
            "requests_per_s": round(n / st["total_s"], 1), "total_s": round(st["total_s"], 3),
            "lookups_per_s": round(st["lookups"] / max(st["lookup_s"], 1e-9), 1),
            "mutations_per_s": round((st["admits"] + st["evictions"] + st["reuses"])
                                     / max(st["mutation_s"], 1e-9), 1),
            "lookup_s": round(st["lookup_s"], 3), "mutation_s": round(st["mutation_s"], 3),
            "maintenance_s": round(st["maintenance_s"], 3), "admits": st["admits"],
            "evictions": st["evictions"], "refinements": st["refinements"],
            "hit_rate": round(st["hit_rate"], 4)}
    if cpu:
        import oracle
        ref = oracle.Ref()
        theirs, summ, wall = ref.replay(p, d, a, t, capacity=1024, policy="exploit", theta=th,
                                        psi=ps, batch=0)
        ok = all(np.array_equal(runs[1][0][f], theirs[f]) for f in theirs.dtype.names)
        res["reference"] = {"requests_per_s": round(n / wall, 1), "total_s": round(wall, 3),
                            "cores": 1, "kind": "reference",
                            "sample": "the unmodified Pipeline::replay on the same trace (a "
                                      "sequential loop by design, pipeline.cpp:299-323)"}
        res["batch1_identical_to_reference"] = bool(ok)
    return res


def export_arena(wc):
    """The context's whole arena (ids, rows, segments) read back from the device
    (sw_arena_export), one row per entry (delta = 1)."""
    from paper_2603_07865_b200 import _lib
    L_ = _lib.lib()
    n = wc.entry_count()
    ids = np.zeros(n, np.uint64)
    nr = np.zeros(n, np.int32)
    rows = np.zeros((n, D), np.float32)
    segs = np.zeros(n, _lib.SEGMENT_DTYPE)
    step = 1 << 18
    for s0 in range(0, n, step):
        m = min(step, n - s0)
        got = L_.sw_arena_export(wc._h, s0, m, ids[s0:].ctypes.data, nr[s0:].ctypes.data,
                                 rows[s0:].ctypes.data, segs[s0:].ctypes.data)
        assert got == m, got
    return ids, rows, segs


def parity_sample(wc, q, reqs_np, choices_np, neg, th, ps, n_check=None, nthreads=None,
                  arena=None):
    """Checks n_check requests (default: the whole batch) of a timed batch against the C
    restatement (oracle) over the
    arena exported from the device (sw_arena_export) — or over `arena` = (ids, rows, segs), the
    union of every rank's exported shard in the sharded run."""
    import oracle
    R = 1
    ids, rows, segs = arena if arena is not None else export_arena(wc)
    n = len(ids)
    ar = oracle.Arena(ids, np.arange(n + 1, dtype=np.int64) * R, rows, segs["level"],
                      segs["start_s"], segs["length_s"])
    B = q.shape[0]
    n_check = B if n_check is None else min(n_check, B)
    sel = np.linspace(0, B - 1, n_check).astype(int)
    nt = nthreads or max(1, len(os.sched_getaffinity(0)))
    t = time.perf_counter()
    exp, _ = oracle.Oracle().plan_batch(ar, neg, q[sel], reqs_np["duration_s"][sel],
                                        reqs_np["id"][sel], reqs_np["total_steps"][sel],
                                        top_k=8, policy="exploit", theta=th, psi=ps, nthreads=nt)
    el = time.perf_counter() - t
    ch = choices_np[sel]
    fields = ["hit", "arm", "steps_skipped", "n_hits", "entry_id", "pick", "similarity"]
    mism = {f: int(np.sum(ch[f] != exp[f])) for f in fields}
    return {"checked": int(n_check), "of_batch": int(B), "mismatches": mism,
            "match": all(v == 0 for v in mism.values()),
            "oracle": "C restatement (oracle/semwarm_oracle.c), pinned to the compiled reference",
            "oracle_s": round(el, 2)}
