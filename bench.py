#!/usr/bin/env python
"""Warm-start requests/s on B200 (BASELINE.json metric) — one JSON line on rank 0.

Workload (BASELINE.json configs[2], "config 3"): a 1M-entry cache of 512-d unit embeddings
(delta = 1: one row per entry, so 1M rows), batches of B = 1024 prompts, top-8 exact search
(tcgen05 bf16 pre-filter + certified fp64 rescoring), score_candidates + select + Skip Gater
(exploit policy, non-degenerate theta) + t*, then align + Philox noising of the chosen 8x256x16
latents. One step = one batch of 1024 requests through that whole path. With --gpus N the
same total cache is sharded by entry over N ranks (strong scaling): every rank scores all
queries against its shard, the 128-byte top-k records are all-gathered over NCCL, merged
deterministically, and select/gater run replicated; align+noise is owner-computes.

value : requests/s with prompts already in HBM (device-timed, CUDA events, max over ranks)
e2e   : same through the host-buffer C-ABI (sw_warmstart_host_submit/_wait, two batches in
        flight as a serving loop runs them): every step's pinned prompts/requests H2D and its
        choices D2H inside the timed region; e2e.sync_call = one blocking sw_warmstart_host
        call per batch
roofline: the scoring kernel (2*B*N*D flops per launch) against MEASURED_PEAKS bf16, timed
        live with CUDA events on its launch stream; align+noise bytes against HBM.
--impl reference: the unmodified reference (oracle/_ref, compiled from /root/reference) on the
        host cores, same cache size and metric, bounded samples per step.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D = 512
LATENT = (8, 256, 16)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--entries", type=int, default=None,
                   help="total cache entries (default: 1M at N=1 = config 3; 10M over N>1 ranks "
                        "= config 4, entry-sharded)")
    p.add_argument("--delta", type=float, default=1.0, help="pyramid delta (1 -> 1 row/entry)")
    p.add_argument("--batch", type=int, default=1024)
    p.add_argument("--top-k", type=int, default=8)
    p.add_argument("--latent-slots", type=int, default=65536)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-latency", action="store_true")
    p.add_argument("--no-batcher", action="store_true",
                   help="skip the request-batcher (swb_*) side measurement")
    p.add_argument("--no-vocoder", action="store_true",
                   help="skip the phase-vocoder (time_stretch) side measurement")
    p.add_argument("--profile-only", action="store_true", help="few steps, no extras (ncu)")
    p.add_argument("--no-sweep", action="store_true",
                   help="skip the cache-size sweep (1K..10M entries; 10M = config 4 at N=1)")
    p.add_argument("--no-replay", action="store_true", help="skip the config-5 trace replay")
    p.add_argument("--no-config1", action="store_true", help="skip the config-1 latency")
    p.add_argument("--parity-max-entries", type=int, default=2_000_000,
                   help="sharded runs: largest cache whose shards are gathered for the parity "
                        "sample")
    p.add_argument("--no-parity", action="store_true",
                   help="skip checking a sample of the timed batch against the oracle")
    p.add_argument("--sweep", default="1000,10000,100000,1000000,10000000",
                   help="cache sizes of the sweep")
    p.add_argument("--no-overlap", action="store_true",
                   help="run align+noise on the planning stream (no cross-batch overlap)")
    p.add_argument("--ivf", default=None, metavar="C,NPROBE",
                   help="IVF mode (the reference's default index: 64,8): GPU k-means rebuild of "
                        "the synthetic cache, then probe-restricted warm starts")
    p.add_argument("--sharded-path", action="store_true",
                   help="run the entry-sharded step (local top-k -> gather -> merge+select -> "
                        "owner align) even at N=1: config 4's per-GPU work at --entries/GPU")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo: validation of the N>1 script on ONE GPU (all ranks share cuda:0, "
                        "records all-gathered through host memory); never a bench number")
    a = p.parse_args()
    if a.entries is None:
        a.entries = 10_000_000 if int(os.environ.get("WORLD_SIZE", "1")) > 1 else 1_000_000
    return a


def rows_per_entry(delta):
    from paper_2603_07865_b200.synth import pyramid
    return len(pyramid(1.0, delta)[0])


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return m["bf16_tflops"], m.get("bf16_tflops_sustained"), m["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """NVML SM clock + throttle reasons sampled in a thread during the timed region."""

    def __init__(self, dev):
        self.dev, self.samples, self.reasons, self.stop = dev, [], set(), False
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.dev)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            names = {N.nvmlClocksThrottleReasonHwSlowdown: "hw_slowdown",
                     N.nvmlClocksThrottleReasonHwThermalSlowdown: "hw_thermal_slowdown",
                     N.nvmlClocksThrottleReasonSwThermalSlowdown: "sw_thermal_slowdown",
                     N.nvmlClocksThrottleReasonSwPowerCap: "sw_power_cap"}

            def run():
                while not self.stop:
                    self.samples.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                    r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    for bit, nm in names.items():
                        if r & bit:
                            self.reasons.add(nm)
                    time.sleep(0.01)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        return self

    def __exit__(self, *a):
        self.stop = True
        if hasattr(self, "t"):
            self.t.join()

    def summary(self):
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


# ----------------------------------------------------------------------------- reference arm
def make_host_cache(n, seed=1):
    from paper_2603_07865_b200.synth import normalize_rows
    rng = np.random.default_rng(seed)
    rows = np.empty((n, D), np.float32)
    for i in range(0, n, 65536):
        m = min(65536, n - i)
        rows[i:i + m] = normalize_rows(rng.standard_normal((m, D), dtype=np.float32))
    dur = rng.uniform(4.0, 12.0, n).astype(np.float32).astype(np.float64)  # SWIX-exact (f32)
    return rows, dur


def reference_sample(n_entries, n_queries, nthreads, seed=1, cache=None, ivf=None, device=0):
    """Builds the reference IvfIndex over n_entries (exhaustive, or IVF: ivf = (C, nprobe)) and
    returns a callable that runs n_queries requests through the reference plan flow with
    nthreads host threads. IVF: the lists come from our GPU k-means of the same rows, written as
    a SWIX snapshot and loaded by the reference's own IvfIndex::load (a 1M-row host k-means
    would not finish in a bench run)."""
    import oracle
    from paper_2603_07865_b200.synth import normalize_rows, trained_like_gater
    rows, dur = cache if cache is not None else make_host_cache(n_entries, seed)
    ar = oracle.Arena(np.arange(1, n_entries + 1, dtype=np.uint64),
                      np.arange(n_entries + 1, dtype=np.int64), rows,
                      np.zeros(n_entries, np.int32), np.zeros(n_entries), dur)
    ref = oracle.Ref()
    if ivf is None:
        idx = ref.index(ar)
    else:
        import tempfile
        from paper_2603_07865_b200.warmstart import WarmStartCache
        tmp = WarmStartCache(D, rows_per_entry=1, max_entries=n_entries, max_batch=8,
                             latent_shape=None, device=device)
        tmp.ivf_configure(ivf[0], ivf[1], 1 << 62, 0)
        tmp.insert_batch(ar.ids, ar.off, ar.rows, ar.levels, ar.starts, ar.lengths)
        tmp.ivf_rebuild()
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "cache.swix")
            tmp.save_swix(path)
            tmp.close()
            idx = ref.load_index_with_arena(path, ar)
    rng = np.random.default_rng(seed + 1)
    src = rows[rng.integers(0, n_entries, n_queries)].astype(np.float64)
    g = rng.standard_normal((n_queries, D))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    q = normalize_rows(src + 0.3 * g)
    L = rng.uniform(2.5, 10.0, n_queries)
    ids = np.arange(1, n_queries + 1, dtype=np.uint64)
    T = np.full(n_queries, 200, np.int32)
    neg = ref.negative(D)
    th, ps = trained_like_gater()

    def run():
        return idx.plan_batch(neg, q, L, ids, T, top_k=8, policy="exploit", theta=th, psi=ps,
                              nthreads=nthreads)

    return run, idx


def ncu_traffic(prefix, summary="ncu_latest.json"):
    """DRAM bytes per launch of a kernel from a committed ncu summary (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", summary)) as f:
            t = json.load(f)["traffic_bytes"]
        for k, v in t.items():
            if k.startswith(prefix):
                return v, k
    except Exception:
        pass
    return None, None


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs and prints the reference arm
    nt = cpu_threads()
    n = args.entries
    t0 = time.time()
    run, _idx = reference_sample(n, nt, nt)
    build_s = time.time() - t0
    steps = max(1, min(args.steps, 30))
    warm = max(0, min(args.warmup, 1))
    for _ in range(warm):
        run()
    t = time.perf_counter()
    for _ in range(steps):
        run()
    el = time.perf_counter() - t
    v = steps * nt / el
    line = {
        "impl": "reference", "metric": "warm-start requests/s", "value": round(v, 3),
        "unit": "requests/s", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": round(1000 * el / steps, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config3: {n}-entry cache x {D}-d (delta={args.delta}), "
                               f"top-{args.top_k}, exploit gater, t*", "entries": n},
        "cpu_baseline": {"value": round(v, 3), "unit": "requests/s", "cores": nt,
                         "kind": "reference",
                         "sample": f"{nt} requests per step (one per host thread) through the "
                                   f"unmodified reference plan flow over the full {n}-entry "
                                   f"exhaustive IvfIndex; CPU {cpu_model()}; index build "
                                   f"{build_s:.1f}s excluded"},
        "e2e": {"value": round(v, 3), "unit": "requests/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2603_07865_b200 import _lib
    from paper_2603_07865_b200.synth import normalize_rows, trained_like_gater
    from paper_2603_07865_b200.warmstart import (CHOICE_DTYPE, Policy, SelectorConfig,
                                                 WarmStartCache, requests)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    staged = args.dist_backend == "gloo"
    if staged:
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if staged:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    B, K = args.batch, args.top_k
    R = rows_per_entry(args.delta)
    per = (args.entries + world - 1) // world
    first = rank * per
    n_local = max(0, min(per, args.entries - first))

    # ---- device-resident shard
    t_setup = time.time()
    wc = WarmStartCache(D, rows_per_entry=R, max_entries=n_local, latent_shape=LATENT,
                        max_batch=B, latent_slots=min(args.latent_slots, n_local), device=local)
    neg = normalize_rows(np.random.default_rng(4242).standard_normal((1, D)))[0]
    th, ps = trained_like_gater()
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    ivf = tuple(int(x) for x in args.ivf.split(",")) if args.ivf else None
    if ivf:
        wc.ivf_configure(ivf[0], ivf[1], 1 << 62, 0)
    wc.fill_synthetic(n_local, first_id=first + 1, seed=1, delta=args.delta)
    torch.cuda.synchronize(dev)
    setup_s = time.time() - t_setup
    rebuild_s = None
    if ivf:
        t = time.perf_counter()
        wc.ivf_rebuild()  # GPU k-means++ + Lloyd, bit-identical to the reference's kmeans
        rebuild_s = time.perf_counter() - t

    # ---- prompts: perturbed copies of cached rows (hits) + 10% unrelated prompts
    n_pool = 4
    rng = np.random.default_rng(7 + rank)
    if rank == 0:
        qs = []
        for _ in range(n_pool):
            ids = rng.integers(1, n_local + 1, B)
            base = np.stack([wc.read_rows(int(i), R)[0] for i in ids]).astype(np.float64)
            g = rng.standard_normal((B, D))
            g /= np.linalg.norm(g, axis=1, keepdims=True)
            q = normalize_rows(base + 0.3 * g)
            m = rng.random(B) < 0.1
            q[m] = normalize_rows(rng.standard_normal((int(m.sum()), D)))
            qs.append(q)
        qpool = torch.from_numpy(np.stack(qs)).to(dev)
    else:
        qpool = torch.empty((n_pool, B, D), dtype=torch.float32, device=dev)
    if world > 1:
        if staged:
            qc = qpool.cpu()
            dist.broadcast(qc, 0)
            qpool.copy_(qc)
        else:
            dist.broadcast(qpool, 0)
    L = np.random.default_rng(11).uniform(2.5, 10.0, B)
    req_np = [requests(np.arange(s * B + 1, (s + 1) * B + 1, dtype=np.uint64), L,
                       np.full(B, 200, np.int32)) for s in range(n_pool)]
    reqs = torch.from_numpy(np.stack([r.view(np.uint8) for r in req_np])).to(dev)
    sel, pol = SelectorConfig(K), Policy("exploit")
    csel, cpol = sel.c(), pol.c()
    C_, T_, F_ = LATENT
    out = torch.empty((B, C_, T_, F_), dtype=torch.float32, device=dev)
    choices = torch.empty((B * CHOICE_DTYPE.itemsize,), dtype=torch.uint8, device=dev)
    stream = torch.cuda.Stream(device=dev)
    sp = stream.cuda_stream
    L_ = _lib.lib()
    import ctypes as Cc
    rec_local = torch.empty((B * K * _lib.HIT_RECORD_BYTES,), dtype=torch.uint8, device=dev)
    n_local_t = torch.empty((B,), dtype=torch.int32, device=dev)
    rec_all = torch.empty((world * B * K * _lib.HIT_RECORD_BYTES,), dtype=torch.uint8, device=dev)
    n_all = torch.empty((world * B,), dtype=torch.int32, device=dev)

    sharded = world > 1 or args.sharded_path

    # A step = sw_warmstart_async: prep + scoring on `stream`, finish + align + noise on the
    # context's stream, so batch i's finish and align+noise run under batch i+1's scoring kernel
    # (4 B stages leave shared memory for a finish CTA per SM; align CTAs use none). The timed
    # region ends with sw_join. --no-overlap: sw_warmstart, everything on one stream.
    overlap = not args.no_overlap and not sharded
    # sharded step, pipelined the same way (sw_local_topk_async): the finish, the gather,
    # merge + select and owner align of batch i run on the context's stream under batch i+1's
    # scoring (not in the gloo host-staged validation mode)
    overlap_sh = not args.no_overlap and sharded and not staged
    if overlap or overlap_sh:
        ch_ring = [torch.empty_like(choices) for _ in range(2)]
    if overlap_sh:
        a_ptr = Cc.c_void_p()
        _lib.check(L_.sw_async_stream(wc._h, Cc.byref(a_ptr)), "sw_async_stream")
        a_stream = torch.cuda.ExternalStream(a_ptr.value, device=dev)

    def join():
        if overlap or overlap_sh:
            _lib.check(L_.sw_join(wc._h, sp), "sw_join")

    def step(i):
        q = qpool[i % n_pool]
        r = reqs[i % n_pool]
        if not sharded and overlap:
            _lib.check(L_.sw_warmstart_async(wc._h, q.data_ptr(), r.data_ptr(), B, 1,
                                             Cc.byref(csel), Cc.byref(cpol), None, 1234,
                                             ch_ring[i % 2].data_ptr(), out.data_ptr(), T_, sp),
                       "sw_warmstart_async")
        elif not sharded:
            _lib.check(L_.sw_warmstart(wc._h, q.data_ptr(), r.data_ptr(), B, 1, Cc.byref(csel),
                                       Cc.byref(cpol), None, 1234, choices.data_ptr(),
                                       out.data_ptr(), T_, sp), "sw_warmstart")
        elif overlap_sh:
            j = i % 2
            _lib.check(L_.sw_local_topk_async(wc._h, q.data_ptr(), B, K, rank,
                                              rec_local.data_ptr(), n_local_t.data_ptr(), sp),
                       "sw_local_topk_async")
            with torch.cuda.stream(a_stream):
                if world == 1:
                    rec_all.copy_(rec_local)
                    n_all.copy_(n_local_t)
                else:
                    dist.all_gather_into_tensor(rec_all, rec_local)
                    dist.all_gather_into_tensor(n_all, n_local_t)
            _lib.check(L_.sw_merge_select(wc._h, rec_all.data_ptr(), n_all.data_ptr(), world,
                                          q.data_ptr(), r.data_ptr(), B, K, 1, Cc.byref(csel),
                                          Cc.byref(cpol), ch_ring[j].data_ptr(), a_ptr),
                       "sw_merge_select")
            _lib.check(L_.sw_align_noise_owned(wc._h, ch_ring[j].data_ptr(), r.data_ptr(), B,
                                               rank, None, 1234, out.data_ptr(), T_, a_ptr),
                       "align")
        else:
            _lib.check(L_.sw_local_topk(wc._h, q.data_ptr(), B, K, rank, rec_local.data_ptr(),
                                        n_local_t.data_ptr(), sp), "sw_local_topk")
            if world == 1:  # --sharded-path at N=1: the gather of one rank is a copy
                with torch.cuda.stream(stream):
                    rec_all.copy_(rec_local)
                    n_all.copy_(n_local_t)
            elif staged:  # host-staged gather (gloo validation mode only)
                stream.synchronize()
                for src, dst in ((rec_local, rec_all), (n_local_t, n_all)):
                    parts = [torch.empty_like(src, device="cpu") for _ in range(world)]
                    dist.all_gather(parts, src.cpu())
                    dst.copy_(torch.cat(parts).to(dev))
                torch.cuda.synchronize(dev)
            else:
                with torch.cuda.stream(stream):
                    dist.all_gather_into_tensor(rec_all, rec_local)
                    dist.all_gather_into_tensor(n_all, n_local_t)
            _lib.check(L_.sw_merge_select(wc._h, rec_all.data_ptr(), n_all.data_ptr(), world,
                                          q.data_ptr(), r.data_ptr(), B, K, 1, Cc.byref(csel),
                                          Cc.byref(cpol), choices.data_ptr(), sp),
                       "sw_merge_select")
            _lib.check(L_.sw_align_noise_owned(wc._h, choices.data_ptr(), r.data_ptr(), B, rank,
                                               None, 1234, out.data_ptr(), T_, sp), "align")

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    steps = 3 if args.profile_only else args.steps
    warm = max(3, args.warmup) if not args.profile_only else 2
    pipeline_note = None
    try:
        for i in range(warm):
            step(i)
        barrier()
    except Exception as e:  # the overlapped sharded step (NCCL on the context stream) as insurance
        if not overlap_sh:
            raise
        pipeline_note = f"pipelined sharded step failed in warm-up ({type(e).__name__}: {e}); one stream"
        overlap_sh = False
        torch.cuda.synchronize(dev)
        for i in range(warm):
            step(i)
        barrier()
    # timed region: only the dominant kernel carries stage events (2 per step), so `value` is
    # not inflated by event records between the other launches
    wc.profile(True, stages=["score_tc"])
    wc.profile_reset()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for i in range(steps):
            step(i)
        join()
        ev1.record(stream)
        barrier()
    wc.profile(False)
    step_info = wc.launch_info()  # of the timed steps (later side measurements launch others)
    ms = ev0.elapsed_time(ev1)
    prof_timed = wc.profile_read()
    # stage breakdown (and launch count) from a second, fully instrumented pass of the same
    # workload
    p_steps = min(steps, 30)
    wc.profile(True)
    wc.profile_reset()
    for i in range(p_steps):
        step(i)
    barrier()
    wc.profile(False)
    prof_all = wc.profile_read()
    prof = dict(prof_all)
    prof["score_tc"] = prof_timed["score_tc"]  # the roofline kernel: timed-region events
    last_i = p_steps - 1  # the batch whose choices / requests the side measurements reuse
    score_alone_ms = None
    stage_ms_overlapped = None
    if overlap_sh:
        choices.copy_(ch_ring[last_i % 2])
        torch.cuda.synchronize(dev)
    if overlap:
        choices.copy_(ch_ring[last_i % 2])
        torch.cuda.synchronize(dev)
        # the scoring kernel with nothing co-running (one stream), for the roofline's context
        wc.profile(True)
        wc.profile_reset()
        for i in range(min(steps, 20)):
            _lib.check(L_.sw_warmstart(wc._h, qpool[i % n_pool].data_ptr(),
                                       reqs[i % n_pool].data_ptr(), B, 1, Cc.byref(csel),
                                       Cc.byref(cpol), None, 1234, choices.data_ptr(),
                                       out.data_ptr(), T_, sp), "sw_warmstart")
        barrier()
        wc.profile(False)
        prof_alone = wc.profile_read()
        a_ms, a_n = prof_alone["score_tc"]
        score_alone_ms = a_ms / max(1, a_n)
        last_i = min(steps, 20) - 1
        # kernel durations without co-running work for the stage breakdown and align roofline;
        # the overlapped pass's stage spans are reported beside them
        stage_ms_overlapped = {k: round(v[0] / max(1, v[1]), 4) for k, v in prof.items() if v[1]}
        prof = dict(prof_alone)
        prof["score_tc"] = prof_timed["score_tc"]
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cpu" if staged else dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    ch = wc.choices(choices)
    qs = wc.query_stats(B) if world == 1 else None
    kernels_per_step = sum(n for (_, n) in prof_all.values()) / max(1, p_steps)
    if args.profile_only:
        if rank == 0:
            print(json.dumps({"profile_only": True, "ms": ms, "stages": prof}))
        return

    # ---- e2e through the host-buffer C-ABI (H2D prompts + requests, D2H choices, every step)
    e2e = None
    if world == 1:
        qh = [torch.empty((B, D), dtype=torch.float32).pin_memory() for _ in range(n_pool)]
        rh = [torch.empty((B * 24,), dtype=torch.uint8).pin_memory() for _ in range(n_pool)]
        chh = [torch.empty((B * CHOICE_DTYPE.itemsize,), dtype=torch.uint8).pin_memory()
               for _ in range(3)]
        for j in range(n_pool):
            qh[j].copy_(qpool[j].cpu())
            rh[j].copy_(reqs[j].cpu())

        def hstep(i):
            j = i % n_pool
            _lib.check(L_.sw_warmstart_host(wc._h, qh[j].data_ptr(), rh[j].data_ptr(), B, 1,
                                            Cc.byref(csel), Cc.byref(cpol), 1234,
                                            chh[0].data_ptr(), out.data_ptr(), T_, sp),
                       "sw_warmstart_host")

        # pipelined serving loop: submit batch i, then wait for batch i-1 (its choices in host
        # memory) — every step's H2D and D2H still inside the timed region
        tk = Cc.c_int64()

        def psubmit(i):
            j = i % n_pool
            _lib.check(L_.sw_warmstart_host_submit(
                wc._h, qh[j].data_ptr(), rh[j].data_ptr(), B, 1, Cc.byref(csel), Cc.byref(cpol),
                1234, chh[i % 3].data_ptr(), out.data_ptr(), T_, sp, Cc.byref(tk)),
                "sw_warmstart_host_submit")
            return tk.value

        depth = 2  # batches waited for behind the newest submission (3 in flight)

        def run_pipelined(n):
            pend = []
            for i in range(n):
                pend.append(psubmit(i))
                if len(pend) > depth:
                    _lib.check(L_.sw_warmstart_host_wait(wc._h, pend.pop(0)),
                               "sw_warmstart_host_wait")
            for t in pend:
                _lib.check(L_.sw_warmstart_host_wait(wc._h, t), "sw_warmstart_host_wait")

        # as many batches as the device-timed loop (>= 20): longer runs reach the board's power
        # cap (measured: 100 e2e batches after the timed loop ran at 0.80 ms per batch, 20 at 0.74)
        e_steps = max(20, steps // 2)

        def timed(fn):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            wall = time.perf_counter() - t0
            return max(e0.elapsed_time(e1), 1000 * wall) / e_steps

        for i in range(warm):
            hstep(i)
        run_pipelined(warm)
        sync_ms = timed(lambda: [hstep(i) for i in range(e_steps)])
        e2e_ms = timed(lambda: run_pipelined(e_steps))
        e2e = {"value": round(B / (e2e_ms / 1000.0), 1), "unit": "requests/s",
               "h2d_bytes_per_step": B * D * 4 + B * 24,
               "d2h_bytes_per_step": B * CHOICE_DTYPE.itemsize, "ms_per_step": round(e2e_ms, 4),
               "path": "sw_warmstart_host_submit/_wait, 3 batches in flight (pinned host "
                       "prompts/requests -> choices; H2D/D2H on copy streams)",
               "sync_call": {"value": round(B / (sync_ms / 1000.0), 1),
                             "ms_per_step": round(sync_ms, 4),
                             "path": "sw_warmstart_host (one blocking call per batch)"}}

    # ---- align + noise timed alone, both noise modes (device events around each launch). Every
    # rep writes a different output buffer (4 rotating, 4 x 134 MB) after a 512 MiB read that
    # evicts L2 (clean lines, as the scoring kernel's arena stream leaves it), so the latent reads,
    # eps reads and output writes all go to HBM.
    align_alone = {}
    if world == 1:
        eps_t = torch.randn((B, C_, T_, F_), dtype=torch.float32, device=dev)
        outs_a = [out] + [torch.empty_like(out) for _ in range(3)]
        flush_buf = torch.ones(1 << 27, dtype=torch.float32, device=dev)
        sink = torch.empty((), dtype=torch.float32, device=dev)
        for mode, dptr in (("philox", None), ("eps", eps_t.data_ptr())):
            def al(j):
                _lib.check(L_.sw_align_noise(wc._h, choices.data_ptr(), reqs[last_i % n_pool]
                                             .data_ptr(), B, dptr, 1234, outs_a[j % 4].data_ptr(),
                                             T_, sp), "sw_align_noise")
            for j in range(4):
                al(j)
            reps = 20
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(reps)]
            for j in range(reps):
                with torch.cuda.stream(stream):  # the launch stream: the flush must not overlap
                    torch.sum(flush_buf, dim=0, out=sink)
                evs[j][0].record(stream)
                al(j)
                evs[j][1].record(stream)
            torch.cuda.synchronize(dev)
            align_alone[mode] = float(np.median([a.elapsed_time(b) for a, b in evs]))
        del outs_a, flush_buf, eps_t
        # the reference's alignment (phase vocoder per latent channel) on the same choices
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        wc.set_align_mode("vocoder", 128, 32)
        _lib.check(L_.sw_align_noise(wc._h, choices.data_ptr(), reqs[last_i % n_pool]
                                     .data_ptr(), B, None, 1234, out.data_ptr(), T_, sp),
                   "sw_align_noise")
        a0.record(stream)
        for _ in range(3):
            _lib.check(L_.sw_align_noise(wc._h, choices.data_ptr(), reqs[last_i % n_pool]
                                         .data_ptr(), B, None, 1234, out.data_ptr(), T_, sp),
                       "sw_align_noise")
        a1.record(stream)
        torch.cuda.synchronize(dev)
        align_alone["vocoder_philox"] = a0.elapsed_time(a1) / 3
        wc.set_align_mode("crop_tile")

    # ---- phase-vocoder time_stretch (the reference's alignment, vocoder.cpp:128-207) side
    # measurement: 1024 clips of the simulated 200 Hz 1-D latent, segment 4-12 s stretched to a
    # served duration (ratio inside the duration gate's [2/3, 2]), STFT {128, 32}
    vocoder = None
    if world == 1 and not args.no_vocoder:
        from paper_2603_07865_b200.warmstart import time_stretch
        vr = np.random.default_rng(5)
        nclip = 1024
        clips, tg = [], []
        for _ in range(nclip):
            L_in = int(vr.integers(800, 2400))
            t = np.arange(L_in) / 200.0
            clips.append((0.5 * np.sin(2 * np.pi * vr.uniform(1, 20) * t)
                          + 0.1 * vr.standard_normal(L_in)).astype(np.float32))
            tg.append(L_in / 200.0 * float(vr.uniform(2 / 3, 2.0)))
        for _ in range(2):
            time_stretch(clips, 200, tg, device=local)
        torch.cuda.synchronize(dev)
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        v0.record()
        for _ in range(reps):
            time_stretch(clips, 200, tg, device=local)
        v1.record()
        torch.cuda.synchronize(dev)
        g_ms = v0.elapsed_time(v1) / reps
        # device-resident: the packed clips already in HBM, one sw_time_stretch per batch
        in_len = np.array([len(x) for x in clips], np.int32)
        in_off = np.concatenate([[0], np.cumsum(in_len)[:-1]]).astype(np.int64)
        tgt = np.asarray(tg, np.float64)
        cap = int(sum(max(0, round(t * 200)) for t in tgt)) + 1
        d_in = torch.from_numpy(np.concatenate(clips)).to(dev)
        d_vo = torch.zeros(cap, dtype=torch.float32, device=dev)
        o_off, o_len, o_st = (np.zeros(nclip, np.int64), np.zeros(nclip, np.int32),
                              np.zeros(nclip, np.int32))

        def vcall():
            _lib.check(L_.sw_time_stretch(d_in.data_ptr(), in_off.ctypes.data,
                                          in_len.ctypes.data, nclip, 200, tgt.ctypes.data, 128,
                                          32, d_vo.data_ptr(), cap, o_off.ctypes.data,
                                          o_len.ctypes.data, o_st.ctypes.data,
                                          torch.cuda.current_stream(dev).cuda_stream),
                       "sw_time_stretch")
        vcall()
        torch.cuda.synchronize(dev)
        v0.record()
        for _ in range(reps):
            vcall()
        v1.record()
        torch.cuda.synchronize(dev)
        d_ms = v0.elapsed_time(v1) / reps
        vocoder = {"clips": nclip, "config": "STFT window 128 hop 32 (pipeline.hpp:36), 200 Hz",
                   "ms_per_batch": round(d_ms, 3),
                   "clips_per_s": round(nclip / (d_ms / 1e3), 1),
                   "note": "clips resident in HBM, one sw_time_stretch call per batch",
                   "ms_per_batch_e2e": round(g_ms, 3),
                   "clips_per_s_e2e": round(nclip / (g_ms / 1e3), 1),
                   "note_e2e": "Python time_stretch(): host packing, H2D, kernels, D2H, unpacking"}
        if not args.no_cpu_baseline:
            try:
                import oracle
                from concurrent.futures import ThreadPoolExecutor
                ref = oracle.Ref()
                nt = cpu_threads()
                sample = list(range(0, nclip, 4))
                t = time.perf_counter()
                with ThreadPoolExecutor(nt) as ex:
                    list(ex.map(lambda i: ref.time_stretch(clips[i], 200, tg[i]), sample))
                el = time.perf_counter() - t
                vocoder["cpu_ref_clips_per_s"] = round(len(sample) / el, 1)
                vocoder["cpu_ref_cores"] = nt
            except Exception as e:  # pragma: no cover
                vocoder["cpu_ref_clips_per_s"] = f"unavailable: {e}"

    # ---- request batcher (swb_*): concurrent single-request clients (the
    # reference's per-connection handle_request) grouped into device batches
    batcher = None
    if world == 1 and not args.no_batcher:
        from concurrent.futures import ThreadPoolExecutor
        from paper_2603_07865_b200.warmstart import Batcher
        qh = qpool[0].cpu().numpy()
        rq = reqs[0].cpu().numpy().view(req_np[0].dtype)
        nclient, per = 256, 8
        bt = Batcher(wc, max_batch=B, max_wait_us=300, seed=1, sel=sel, policy=pol,
                     philox_seed=1234, t_out_max=T_)

        def client(t):
            lat = []
            for j in range(per):
                i = (t * per + j) % B
                t0 = time.perf_counter()
                bt.submit(qh[i], rq[i:i + 1])
                lat.append(time.perf_counter() - t0)
            return lat

        with ThreadPoolExecutor(nclient) as ex:
            list(ex.map(client, range(16)))  # warm-up
            s0 = bt.stats()
            t0 = time.perf_counter()
            lats = sum(ex.map(client, range(nclient)), [])
            wall = time.perf_counter() - t0
        s1 = bt.stats()
        nb = s1["batches"] - s0["batches"]
        nr = s1["requests"] - s0["requests"]
        lats.sort()
        py_clients = {"clients": nclient, "requests": nr, "requests_per_s": round(nr / wall, 1),
                      "mean_batch": round(nr / max(1, nb), 1),
                      "p50_ms": round(1e3 * lats[len(lats) // 2], 3),
                      "p99_ms": round(1e3 * lats[int(len(lats) * 0.99)], 3),
                      "note": "Python client threads (GIL-bound), one blocking swb_submit each"}
        # native clients (swb_load_test: C++ threads, no GIL): the batcher's own capacity
        bt.load_test(qh, rq, clients=64, per_client=8)  # warm-up
        nat = {}
        for ncl in (256, 1024, 4096):
            r_ = bt.load_test(qh, rq, clients=ncl, per_client=max(16, 16384 // ncl))
            nat[str(ncl)] = {k: round(v, 3) for k, v in r_.items()}
        bt.close()
        best = max(nat.values(), key=lambda x: x["requests_per_s"])
        batcher = {"requests_per_s": best["requests_per_s"], "mean_batch": best["mean_batch"],
                   "p50_ms": best["p50_ms"], "p99_ms": best["p99_ms"],
                   "native_clients": nat, "python_clients": py_clients,
                   "note": "C++ client threads (swb_load_test), one blocking swb_submit per "
                           "request (plan + align+noise, max_batch 1024, max_wait 300 us), wall "
                           "clock; keyed by client-thread count"}

    # ---- p50 selector latency (search through select, pipeline.cpp:93-143's selector_ms span)
    lat = {}
    if not args.no_latency and world == 1:
        for bsz, reps in ((1, 1000), (B, 200)):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(reps)]
            for i in range(reps):
                ev[i][0].record(stream)
                _lib.check(L_.sw_plan(wc._h, qpool[0].data_ptr(), reqs[0].data_ptr(), bsz, 1,
                                      Cc.byref(csel), Cc.byref(cpol), choices.data_ptr(), sp),
                           "sw_plan")
                ev[i][1].record(stream)
            torch.cuda.synchronize(dev)
            t = sorted(a.elapsed_time(b) for a, b in ev)
            lat[f"B{bsz}"] = round(t[len(t) // 2], 4)

    # ---- side measurements (one GPU): parity sample of the timed batch, cache-size sweep
    # (10M = config 4 at N=1), config 4's per-GPU shard step, config 1 latency, config 5 replay
    pk_burst, pk_sust, hbm, pk_src = peaks()
    extras = {}
    if world > 1 and not args.profile_only and not args.no_parity and not ivf and R == 1:
        # sharded run: every rank exports its shard, rank 0 checks the merged choices of the
        # timed batch against the oracle over the union (bounded: host copies of the shards)
        import bench_extras as bx
        if n_local * world <= args.parity_max_entries:
            part = bx.export_arena(wc)
            parts = [None] * world if rank == 0 else None
            dist.gather_object(part, parts, dst=0)
            if rank == 0:
                arena = tuple(np.concatenate([p_[i] for p_ in parts]) for i in range(3))
                try:
                    extras["parity_sample"] = bx.parity_sample(
                        wc, qpool[last_i % n_pool].cpu().numpy(), req_np[last_i % n_pool],
                        ch.copy(), neg, th, ps, arena=arena)
                    extras["parity_sample"]["shards"] = world
                except Exception as e:  # pragma: no cover
                    extras["parity_sample"] = {"error": f"{type(e).__name__}: {e}"}
        elif rank == 0:
            extras["parity_sample"] = {"skipped": f"{n_local * world} entries > "
                                                  f"--parity-max-entries {args.parity_max_entries}"}
    if world == 1 and rank == 0 and not args.profile_only:
        import bench_extras as bx
        if not args.no_parity and not ivf and R == 1:
            try:
                extras["parity_sample"] = bx.parity_sample(
                    wc, qpool[last_i % n_pool].cpu().numpy(), req_np[last_i % n_pool], ch.copy(),
                    neg, th, ps)
            except Exception as e:  # pragma: no cover
                extras["parity_sample"] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_sweep:
            sw = []
            for n_s in [int(x) for x in args.sweep.split(",") if x]:
                try:
                    pt = bx.sweep_point(n_s, B, K, device=local, peak=pk_burst)
                    if not args.no_cpu_baseline and n_s <= 100_000:
                        pt["cpu_reference_requests_per_s"] = bx.cpu_reference_point(
                            n_s, cpu_threads(), 4 if n_s <= 10_000 else 1)
                        pt["cpu_reference_cores"] = cpu_threads()
                    sw.append(pt)
                except Exception as e:  # pragma: no cover
                    sw.append({"entries": n_s, "error": f"{type(e).__name__}: {e}"})
            extras["cache_size_sweep"] = sw
            ten = [x for x in sw if x.get("entries") == 10_000_000 and "error" not in x]
            try:
                extras["config4"] = {"single_gpu_10M": ten[0] if ten else None,
                                     "per_gpu_shard": bx.config4_shard(device=local)}
            except Exception as e:  # pragma: no cover
                extras["config4"] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_config1:
            try:
                extras["config1"] = bx.config1_latency(device=local,
                                                       cpu=not args.no_cpu_baseline)
            except Exception as e:  # pragma: no cover
                extras["config1"] = {"error": f"{type(e).__name__}: {e}"}
        if not args.no_replay:
            try:
                extras["config5"] = bx.config5_replay(device=local, cpu=not args.no_cpu_baseline)
            except Exception as e:  # pragma: no cover
                extras["config5"] = {"error": f"{type(e).__name__}: {e}"}

    if rank != 0:
        if world > 1:
            dist.barrier()
        return

    # ---- roofline of the dominant kernel (tcgen05 scoring), timed live on its stream
    default_workload = (args.entries == 1_000_000 and B == 1024 and K == 8 and R == 1
                        and not ivf and world == 1 and not sharded)
    sc_ms, sc_n = prof["score_tc"]
    n_rows = n_local * R
    flops = 2.0 * B * n_rows * D
    score_ms = sc_ms / max(1, sc_n)
    achieved = flops / (score_ms / 1000.0) / 1e12 if sc_n else None
    # align + noise = the per-request geometry pre-pass + the streaming kernel, both counted
    al_ms, al_n = prof["align"]
    if al_n and prof.get("align_geom", (0, 0))[1]:
        g_ms, g_n = prof["align_geom"]
        al_ms = al_ms + g_ms * al_n / g_n
    hits = ch["hit"].astype(bool)
    owned = hits & ((ch["owner"] == rank) if world > 1 else True)  # owner-computes align
    t_out = ch["t_out"][owned].astype(np.int64)
    fr = lambda x: np.floor(x * 25.0 + 0.5)
    t_seg = (fr(ch["start_s"] + ch["length_s"]) - fr(ch["start_s"]))[owned]
    al_bytes = float(np.sum(4 * C_ * F_ * (np.minimum(t_out, T_) + np.minimum(t_seg, t_out))))
    al_gbs = al_bytes / (al_ms / max(1, al_n) / 1000.0) / 1e9 if al_n else None
    eps_bytes = al_bytes + float(np.sum(4 * C_ * F_ * np.minimum(t_out, T_)))
    total_ms_step = ms / steps
    roof_ivf = None
    if ivf:
        # IVF at B = 1024: every list is probed by some queries, so the whole bf16 arena streams
        # once per batch whatever the (1/8) flop count — HBM is the bound
        ivf_bytes = float(n_rows) * (((D + 63) // 64) * 64) * 2
        ivf_gbs = ivf_bytes / (score_ms / 1e3) / 1e9 if sc_n else None
        roof_ivf = {"bound": "hbm",
                    "kernel": "k_score_tc (list-grouped, tcgen05.mma M128 N256 K16, TMA)",
                    "achieved": round(ivf_gbs, 1) if ivf_gbs else None, "peak": hbm,
                    "unit": "GB/s", "frac": round(ivf_gbs / hbm, 4) if ivf_gbs else None,
                    "algorithmic": f"the bf16 arena once = {ivf_bytes:.4g} B per launch",
                    "traffic": None, "traffic_source": "not captured for this configuration",
                    "kernel_ms": round(score_ms, 4),
                    "share_of_step": round(score_ms / total_ms_step, 3)}
        if (args.ivf or "").replace(" ", "") in ("64,8",):  # the configuration the capture is of
            tb, tk = ncu_traffic("k_score_tc<1, 8, 0, 0>", "ncu_ivf_latest.json")
            if tb:
                roof_ivf["traffic"] = tb
                roof_ivf["traffic_source"] = ("profiles/ncu_ivf_latest.json (ncu --set full, one "
                                              "launch of " + tk + ", bench.py --ivf 64,8)")
    value = B * steps / (ms / 1000.0)
    stage_ms = {k: round(v[0] / max(1, v[1]), 4) for k, v in prof.items() if v[1]}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        try:
            nt = cpu_threads()
            run, _idx = reference_sample(args.entries, 2 * nt, nt, ivf=ivf, device=local)
            t = time.perf_counter()
            run()
            el = time.perf_counter() - t
            cpu = {"value": round(2 * nt / el, 3), "unit": "requests/s", "cores": nt,
                   "kind": "reference",
                   "sample": f"{2 * nt} requests ({nt} host threads, {cpu_model()}) through the "
                             f"unmodified reference (oracle/_ref: IvfIndex::search "
                             f"{'IVF C=%d nprobe=%d (SWIX-loaded lists)' % ivf if ivf else 'exhaustive'} + "
                             f"score_candidates + select + context_features + choose_arm + t*) "
                             f"over a host copy of a {args.entries}-entry x {D}-d cache"}
        except Exception as e:
            cpu = {"value": None, "unit": "requests/s", "cores": cpu_threads(),
                   "kind": "reference", "sample": f"unavailable: {e}"}

    line = {
        "metric": "warm-start requests/s", "value": round(value, 1), "unit": "requests/s",
        "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": round(total_ms_step, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16+f64",
        "data": "synthetic (device Philox iid unit embeddings; N(0,1) latents)",
        "config": {"workload": f"config3: {args.entries}-entry cache x {D}-d (delta={args.delta},"
                               f" {R} row/entry), batch {B}, top-{K} exact, exploit gater, "
                               f"align+noise {C_}x{T_}x{F_} Philox"
                               + (f", IVF C={ivf[0]} nprobe={ivf[1]}" if ivf else ""),
                   "entries": args.entries, "rows_per_gpu": n_rows, "global_batch": B,
                   "parallelism": f"entry-sharded x{world}" if sharded else "single",
                   "l2": "inputs larger than L2 (bf16 arena %.0f MB streamed per step)"
                         % (n_rows * D * 2 / 1e6),
                   "latent_slots": min(args.latent_slots, n_local),
                   "pipelining": ("finish + align+noise of batch i on a second stream (sw_warmstart_async), overlapping batch "
                                  "i+1's scoring" if overlap else
                                  "finish + gather + merge/select + owner align of batch i on a "
                                  "second stream (sw_local_topk_async), overlapping batch i+1's "
                                  "scoring" if overlap_sh else (pipeline_note or "none (one stream)"))},
        **({"validation_only": "gloo host-staged gather, all ranks on one GPU"} if staged else {}),
        "roofline": (roof_ivf if ivf else {"bound": "tensor",
                     "kernel": "k_score_tc (tcgen05.mma %s, TMA)" % (
                         "cta_group::2 M256 N256 K16" if step_info["cta_pair"]
                         else "M128 N256 K16"),
                     "achieved": round(achieved, 1) if achieved else None, "peak": pk_burst,
                     "unit": "TFLOP/s", "frac": round(achieved / pk_burst, 4) if achieved else None,
                     "frac_of_sustained": round(achieved / pk_sust, 4) if achieved and pk_sust else None,
                     "peak_source": pk_src,
                     # the committed capture profiles the default workload only
                     "traffic": ncu_traffic("k_score_tc")[0] if default_workload else None,
                     "traffic_source": ("profiles/ncu_latest.json (ncu --set full, one launch)"
                                        if default_workload else
                                        "not captured for this configuration"),
                     "algorithmic": f"2*B*N*D = {flops:.4g} flop per launch",
                     "kernel_ms": round(score_ms, 4),
                     "share_of_step": round(score_ms / total_ms_step, 3),
                     **({"timing": "live in the timed region, co-running with the previous "
                                   "batch's finish + align (sw_warmstart_async)",
                         "alone_ms": round(score_alone_ms, 4),
                         "alone_frac": round(flops / (score_alone_ms / 1e3) / 1e12 / pk_burst, 4)}
                        if score_alone_ms else {})}),
        "align_roofline": {"bound": "hbm",
                           "kernel": "k_align_geom + k_align_noise (per-request geometry, then "
                                     "one 128-thread CTA per latent plane; both timed)",
                           "achieved": round(al_gbs, 1) if al_gbs else None,
                           "peak": hbm, "unit": "GB/s",
                           "frac": round(al_gbs / hbm, 4) if al_gbs else None,
                           "bytes_per_launch": al_bytes,
                           "alone_ms": {k: round(v, 4) for k, v in align_alone.items()},
                           "alone_frac": {
                               "philox": round(al_bytes / (align_alone["philox"] / 1e3) / 1e9 / hbm, 4),
                               "eps": round(eps_bytes / (align_alone["eps"] / 1e3) / 1e9 / hbm, 4)}
                           if align_alone else None,
                           "alone_timing": "median of 20 launches, each after a 512 MiB read that "
                                           "evicts L2, 4 rotating output buffers"},
        **({"ivf": {"centroids": ivf[0], "nprobe": ivf[1], "rebuild_s": round(rebuild_s, 3),
                    "rebuild": "GPU k-means++ + Lloyd over %d rows (fp64, bit-identical to "
                               "index.cpp:59-184)" % n_rows}} if ivf else {}),
        "vocoder": vocoder,
        "batcher": batcher,
        "stage_ms": stage_ms,
        **({"stage_ms_overlapped": stage_ms_overlapped} if stage_ms_overlapped else {}),
        "selector_p50_ms": lat,
        "hit_rate": round(float(hits.mean()), 4),
        "candidates": None if qs is None else {
            "emitted_mean": float(qs[:, 0].mean()), "kept_mean": float(qs[:, 1].mean()),
            "kept_max": int(qs[:, 1].max()),
            "finish_phase_kcycles_mean": [round(float(qs[:, j].mean()) / 1e3, 2) for j in (2, 3, 4, 5)],
            "finish_phase_kcycles_max": [round(float(qs[:, j].max()) / 1e3, 2) for j in (2, 3, 4, 5)],
            "finish_phase_a_split_kcycles_mean": [round(float(qs[:, j].mean()) / 1e3, 2) for j in (6, 7)]},
        "e2e": e2e,
        "gpu_launches": int(round(kernels_per_step * steps)),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "setup_s": round(setup_s, 1),
        **extras,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()


if __name__ == "__main__":
    main()
