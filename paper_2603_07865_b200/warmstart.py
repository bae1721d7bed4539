"""Python host layer over the C-ABI, mirroring the reference's C++ API for the warm-start path.

Reference interface                                   here
IvfIndex::insert / remove / search (index.hpp:59-67)  WarmStartCache.insert / remove / search
score_candidates + select (selector.hpp:50-58)         score_select
context_features + choose_arm (gater.hpp:30,56-57)     gater
Pipeline::plan_request + pick_arm (pipeline.cpp:91-202) WarmStartCache.plan
slice_clip + (new) forward noising                     WarmStartCache.align_noise / warmstart

Errors follow the reference: invalid arguments raise ValueError (std::invalid_argument), an
unknown id on remove warns and is a no-op (index.cpp:243-245), a miss is an empty result.
Device buffers come from torch (plumbing only); the compute is libsemwarm_b200.so.
"""
from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (CHOICE_DTYPE, HIT_DTYPE, OUTCOME_DTYPE, POLICY, REQUEST_DTYPE, SEGMENT_DTYPE,
                   SwConfig, SwPolicy, SwSelectorConfig, check, ptr)


def _torch():
    import torch
    return torch


@dataclass
class SelectorConfig:
    """SelectorConfig (selector.hpp:25-33) — negative embedding set on the cache."""
    top_k: int = 8
    temperature: float = 0.05
    quality_threshold: float = 0.6

    def c(self) -> SwSelectorConfig:
        return SwSelectorConfig(int(self.top_k), 0, float(self.temperature),
                                float(self.quality_threshold))


@dataclass
class Policy:
    """SkipPolicy + parameters (pipeline.hpp:17-22, 37-41)."""
    kind: str = "exploit"
    fixed_arm: int = 0
    rule_similarity_threshold: float = 0.35
    rule_skip_fraction: float = 0.55

    def c(self) -> SwPolicy:
        return SwPolicy(POLICY[self.kind], int(self.fixed_arm),
                        float(self.rule_similarity_threshold), float(self.rule_skip_fraction))


def segments(levels, starts, lengths) -> np.ndarray:
    s = np.zeros(len(levels), SEGMENT_DTYPE)
    s["level"], s["start_s"], s["length_s"] = levels, starts, lengths
    return s


def requests(ids, durations, total_steps) -> np.ndarray:
    r = np.zeros(len(ids), REQUEST_DTYPE)
    r["id"], r["duration_s"], r["total_steps"] = ids, durations, total_steps
    return r


class WarmStartCache:
    """One device-resident cache shard: arena + batched warm-start path."""

    def __init__(self, dim: int, rows_per_entry: int = 7, max_entries: int = 1024,
                 latent_shape=(8, 256, 16), max_batch: int = 1024, latent_slots: int = 0,
                 fps: float = 25.0, exact_only: bool = False, tc_always: bool = False,
                 device: int = 0):
        L = _lib.lib()
        cfg = SwConfig()
        cfg.dim = dim
        cfg.rows_per_entry = rows_per_entry
        cfg.max_entries = max_entries
        cfg.latent_c, cfg.latent_t_max, cfg.latent_f = latent_shape if latent_shape else (0, 0, 0)
        cfg.max_batch = max_batch
        cfg.latent_slots = latent_slots
        cfg.latent_fps = fps
        cfg.flags = (_lib.SW_FLAG_EXACT_ONLY if exact_only else 0) | (
            _lib.SW_FLAG_TC_ALWAYS if tc_always else 0)
        h = C.c_void_p()
        check(L.sw_ctx_create(C.byref(cfg), device, C.byref(h)), "sw_ctx_create")
        self._h = h
        self.dim = dim
        self.device = device
        self.latent_shape = tuple(latent_shape) if latent_shape else None
        self.max_batch = max_batch

    @classmethod
    def _borrow(cls, handle, dim: int, latent_shape, max_batch: int, device: int):
        """A non-owning view of a context created elsewhere (a ShardGroup's shard)."""
        self = cls.__new__(cls)
        self._h = handle
        self._owned = False
        self.dim = dim
        self.device = device
        self.latent_shape = tuple(latent_shape) if latent_shape else None
        self.max_batch = max_batch
        return self

    def close(self):
        if getattr(self, "_h", None):
            if getattr(self, "_owned", True):
                _lib.lib().sw_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ configuration
    def set_negative(self, neg: np.ndarray):
        neg = np.ascontiguousarray(neg, np.float32)
        check(_lib.lib().sw_set_negative(self._h, ptr(neg)), "sw_set_negative")

    def set_gater(self, theta, psi, beta: float = 1.0):
        theta = np.ascontiguousarray(theta, np.float32).reshape(-1)
        psi = np.ascontiguousarray(psi, np.float32).reshape(-1)
        check(_lib.lib().sw_set_gater(self._h, ptr(theta), ptr(psi), 11, beta), "sw_set_gater")

    def set_schedule(self, abar):
        abar = np.ascontiguousarray(abar, np.float64)
        check(_lib.lib().sw_set_schedule(self._h, ptr(abar), len(abar)), "sw_set_schedule")

    # ------------------------------------------------------------------ arena (K5)
    def insert(self, entry_id: int, rows, levels, starts, lengths, latent=None):
        rows = np.ascontiguousarray(rows, np.float32).reshape(-1, self.dim)
        sg = segments(levels, starts, lengths)
        lat = None if latent is None else np.ascontiguousarray(latent, np.float32)
        t_src = 0 if lat is None else lat.shape[1]
        check(_lib.lib().sw_arena_insert(self._h, entry_id, rows.shape[0], ptr(rows), ptr(sg),
                                         ptr(lat), t_src), "sw_arena_insert")

    def insert_batch(self, ids, row_off, rows, levels, starts, lengths, latents=None,
                     lat_off=None, t_src=None):
        ids = np.ascontiguousarray(ids, np.uint64)
        row_off = np.ascontiguousarray(row_off, np.int64)
        rows = np.ascontiguousarray(rows, np.float32)
        sg = segments(levels, starts, lengths)
        lp = lo = ts = None
        if latents is not None:
            lp = np.ascontiguousarray(latents, np.float32)
            lo = np.ascontiguousarray(lat_off, np.int64)
            ts = np.ascontiguousarray(t_src, np.int32)
        check(_lib.lib().sw_arena_insert_batch(self._h, len(ids), ptr(ids), ptr(row_off),
                                               ptr(rows), ptr(sg), ptr(lp), ptr(lo), ptr(ts), 0),
              "sw_arena_insert_batch")

    def remove(self, entry_id: int) -> bool:
        rc = check(_lib.lib().sw_arena_remove(self._h, entry_id), "sw_arena_remove")
        if rc == _lib.SW_WARN_UNKNOWN_ID:
            warnings.warn(f"remove of unknown entry id {entry_id}")
            return False
        return True

    def replace(self, entry_id: int, rows, levels, starts, lengths, latent=None) -> bool:
        rows = np.ascontiguousarray(rows, np.float32).reshape(-1, self.dim)
        sg = segments(levels, starts, lengths)
        lat = None if latent is None else np.ascontiguousarray(latent, np.float32)
        t_src = 0 if lat is None else lat.shape[1]
        rc = check(_lib.lib().sw_arena_replace(self._h, entry_id, rows.shape[0], ptr(rows),
                                               ptr(sg), ptr(lat), t_src), "sw_arena_replace")
        return rc == _lib.SW_OK

    def entry_count(self) -> int:
        return int(_lib.lib().sw_arena_entry_count(self._h))

    def contains(self, entry_id: int) -> bool:
        return bool(_lib.lib().sw_arena_contains(self._h, entry_id))

    def fill_synthetic(self, n: int, first_id: int = 1, seed: int = 1, delta: float = 1.0):
        check(_lib.lib().sw_arena_fill_synthetic(self._h, n, first_id, seed, delta),
              "sw_arena_fill_synthetic")

    def read_rows(self, entry_id: int, cap: int = 32) -> np.ndarray:
        out = np.zeros((cap, self.dim), np.float32)
        n = check(_lib.lib().sw_arena_read_rows(self._h, entry_id, ptr(out), cap), "read_rows")
        return out[:n]

    # ------------------------------------------------------------------ IVF coarse quantiser
    def ivf_configure(self, centroids: int = 64, nprobe: int = 8, rebuild_interval: int = 1024,
                      seed: int = 0):
        """IvfIndex::build({}, centroids, seed, nprobe) + set_rebuild_interval (index.cpp:186,
        pipeline.cpp:28-31 defaults). Empty arena only."""
        check(_lib.lib().sw_ivf_configure(self._h, centroids, nprobe, rebuild_interval, seed),
              "sw_ivf_configure")

    def ivf_set_nprobe(self, nprobe: int):
        check(_lib.lib().sw_ivf_set_nprobe(self._h, nprobe), "sw_ivf_set_nprobe")

    def ivf_rebuild(self):
        check(_lib.lib().sw_ivf_rebuild(self._h), "sw_ivf_rebuild")

    def ivf_info(self) -> dict:
        n, m, r = C.c_int32(), C.c_uint64(), C.c_uint64()
        check(_lib.lib().sw_ivf_info(self._h, C.byref(n), C.byref(m), C.byref(r)), "sw_ivf_info")
        return {"centroids": n.value, "mutations": m.value, "rebuilds": r.value}

    def ivf_centroids(self) -> np.ndarray:
        out = np.zeros((256, self.dim), np.float32)
        n = check(_lib.lib().sw_ivf_centroids(self._h, ptr(out), 256), "sw_ivf_centroids")
        return out[:n]

    def ivf_set_centroids(self, cent: np.ndarray):
        cent = np.ascontiguousarray(cent, np.float32)
        check(_lib.lib().sw_ivf_set_centroids(self._h, ptr(cent), cent.shape[0]),
              "sw_ivf_set_centroids")

    def ivf_entry_lists(self, entry_id: int) -> np.ndarray:
        out = np.zeros(32, np.int16)
        n = check(_lib.lib().sw_ivf_entry_lists(self._h, entry_id, ptr(out), 32), "entry_lists")
        return out[:n]

    def set_align_mode(self, mode: str = "crop_tile", window: int = 128, hop: int = 32):
        """'crop_tile' (default) or 'vocoder' — the reference's slice_clip + time_stretch
        (pipeline.cpp:158-169) per latent channel, StftConfig{window, hop}."""
        m = {"crop_tile": 0, "vocoder": 1}[mode]
        check(_lib.lib().sw_set_align_mode(self._h, m, window, hop), "sw_set_align_mode")

    # ------------------------------------------------------------------ snapshots
    def load_swmb(self, path: str, beta: float = 1.0):
        """BanditModel::load (gater.cpp:287-306) into the device-resident Skip Gater."""
        check(_lib.lib().sw_gater_load_swmb(self._h, path.encode(), beta), "sw_gater_load_swmb")

    def save_swmb(self, path: str):
        check(_lib.lib().sw_gater_save_swmb(self._h, path.encode()), "sw_gater_save_swmb")

    def ivf_config(self) -> dict:
        en, c, npb = C.c_int32(), C.c_int32(), C.c_int32()
        iv, sd = C.c_uint64(), C.c_uint64()
        check(_lib.lib().sw_ivf_config(self._h, C.byref(en), C.byref(c), C.byref(npb),
                                       C.byref(iv), C.byref(sd)), "sw_ivf_config")
        return {"enabled": bool(en.value), "centroids": c.value, "nprobe": npb.value,
                "rebuild_interval": iv.value, "seed": sd.value}

    def load_swix(self, path: str):
        """IvfIndex::load (index.cpp:371-406) into this (empty) cache's device arena."""
        check(_lib.lib().sw_swix_load(self._h, path.encode()), "sw_swix_load")

    def save_swix(self, path: str):
        """IvfIndex::save (index.cpp:347-369) of this cache's index."""
        check(_lib.lib().sw_swix_save(self._h, path.encode()), "sw_swix_save")

    def profile(self, on: bool = True, stages=None):
        """Stage timing on/off; `stages` (names from _lib.STAGES) limits it to those stages."""
        v = int(on)
        if on and stages is not None:
            v = 0x100
            for name in stages:
                v |= 1 << _lib.STAGES.index(name)
        check(_lib.lib().sw_profile_enable(self._h, v), "profile")

    def profile_reset(self):
        check(_lib.lib().sw_profile_reset(self._h), "profile_reset")

    def profile_read(self) -> dict:
        out = {}
        for i, name in enumerate(_lib.STAGES):
            ms, n = C.c_double(), C.c_int64()
            check(_lib.lib().sw_profile_read(self._h, i, C.byref(ms), C.byref(n)), "profile_read")
            out[name] = (ms.value, n.value)
        return out

    def query_stats(self, B: int) -> np.ndarray:
        """Per-query finish stats of the last search/plan: emitted, kept, phase cycles x4."""
        out = np.zeros((B, 8), np.int32)
        check(_lib.lib().sw_debug_query_stats(self._h, B, ptr(out)), "query_stats")
        return out

    def overflow_fallbacks(self) -> int:
        """Queries so far answered by the certified exact fallback (candidate overflow)."""
        v = C.c_int64()
        check(_lib.lib().sw_overflow_stats(self._h, C.byref(v)), "sw_overflow_stats")
        return v.value

    def arena_capacity(self) -> int:
        return int(_lib.lib().sw_arena_capacity(self._h))

    def launch_info(self):
        k, t, m = C.c_int32(), C.c_int32(), C.c_int32()
        _lib.lib().sw_last_launch_info(self._h, C.byref(k), C.byref(t), C.byref(m))
        return {"kernels": k.value, "tensor_cores": bool(t.value), "cta_pair": t.value >= 2,
                "a_in_tmem": t.value == 3}

    # ------------------------------------------------------------------ hot path
    def _dev(self, a, dtype):
        torch = _torch()
        if isinstance(a, torch.Tensor):
            assert a.is_cuda and a.is_contiguous()
            return a
        return torch.from_numpy(np.ascontiguousarray(a, dtype)).to(f"cuda:{self.device}")

    def search(self, queries, k: int):
        """IvfIndex::search for each row of `queries` (exhaustive, exact). Returns (hits, n)."""
        torch = _torch()
        q = self._dev(queries, np.float32).reshape(-1, self.dim)
        B = q.shape[0]
        out = torch.empty(B * k * HIT_DTYPE.itemsize, dtype=torch.uint8, device=q.device)
        n = torch.empty(B, dtype=torch.int32, device=q.device)
        st = torch.cuda.current_stream(q.device).cuda_stream
        check(_lib.lib().sw_search(self._h, ptr(q), B, k, ptr(out), ptr(n), st), "sw_search")
        hits = out.cpu().numpy().view(HIT_DTYPE).reshape(B, k)
        n = n.cpu().numpy()
        if (n < 0).any():  # never expected: overflowing queries are re-searched exactly
            raise RuntimeError("search result not certified (candidate overflow)")
        return hits, n

    def search_host(self, queries: np.ndarray, k: int):
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        B = q.shape[0]
        out = np.zeros((B, k), HIT_DTYPE)
        n = np.zeros(B, np.int32)
        check(_lib.lib().sw_search_host(self._h, ptr(q), B, k, ptr(out), ptr(n)), "search_host")
        return out, n

    def plan(self, queries, reqs: np.ndarray, seed: int = 1, sel: SelectorConfig = None,
             policy: Policy = None, stream=None, out=None):
        torch = _torch()
        sel = sel or SelectorConfig()
        policy = policy or Policy()
        q = self._dev(queries, np.float32)
        r = self._dev(reqs.view(np.uint8) if isinstance(reqs, np.ndarray) else reqs, np.uint8)
        B = q.shape[0]
        if out is None:
            out = torch.empty(B * CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=q.device)
        st = stream if stream is not None else torch.cuda.current_stream(q.device).cuda_stream
        check(_lib.lib().sw_plan(self._h, ptr(q), ptr(r), B, seed, C.byref(sel.c()),
                                 C.byref(policy.c()), ptr(out), st), "sw_plan")
        return out

    @staticmethod
    def choices(buf) -> np.ndarray:
        return buf.cpu().numpy().view(CHOICE_DTYPE)

    def align_noise(self, choices_dev, reqs, t_out_max: int, eps=None, philox_seed: int = 0):
        torch = _torch()
        r = self._dev(reqs.view(np.uint8) if isinstance(reqs, np.ndarray) else reqs, np.uint8)
        B = choices_dev.numel() // CHOICE_DTYPE.itemsize
        C_, _, F = self.latent_shape
        out = torch.zeros((B, C_, t_out_max, F), dtype=torch.float32, device=r.device)
        e = None if eps is None else self._dev(eps, np.float32)
        st = torch.cuda.current_stream(r.device).cuda_stream
        check(_lib.lib().sw_align_noise(self._h, ptr(choices_dev), ptr(r), B, ptr(e),
                                        philox_seed, ptr(out), t_out_max, st), "sw_align_noise")
        return out

    def warmstart_host(self, queries: np.ndarray, reqs: np.ndarray, d_out, t_out_max: int,
                       seed: int = 1, sel: SelectorConfig = None, policy: Policy = None,
                       philox_seed: int = 0, stream=None):
        sel = sel or SelectorConfig()
        policy = policy or Policy()
        B = queries.shape[0]
        ch = np.zeros(B, CHOICE_DTYPE)
        check(_lib.lib().sw_warmstart_host(self._h, ptr(queries), ptr(reqs), B, seed,
                                           C.byref(sel.c()), C.byref(policy.c()), philox_seed,
                                           ptr(ch), ptr(d_out), t_out_max, stream),
              "sw_warmstart_host")
        return ch

    def warmstart_host_submit(self, queries: np.ndarray, reqs: np.ndarray, choices: np.ndarray,
                              d_out, t_out_max: int, seed: int = 1, sel: SelectorConfig = None,
                              policy: Policy = None, philox_seed: int = 0, stream=None) -> int:
        """Pipelined warmstart_host: returns a ticket at once; `queries`, `reqs` and `choices`
        (a CHOICE_DTYPE array filled in place) must stay alive until warmstart_host_wait."""
        sel = sel or SelectorConfig()
        policy = policy or Policy()
        t = C.c_int64()
        check(_lib.lib().sw_warmstart_host_submit(
            self._h, ptr(queries), ptr(reqs), queries.shape[0], seed, C.byref(sel.c()),
            C.byref(policy.c()), philox_seed, ptr(choices), ptr(d_out), t_out_max, stream,
            C.byref(t)), "sw_warmstart_host_submit")
        return t.value

    def warmstart_host_wait(self, ticket: int) -> None:
        check(_lib.lib().sw_warmstart_host_wait(self._h, ticket), "sw_warmstart_host_wait")

    # ------------------------------------------------------------------ component entry points
    def score_select(self, sims, s_neg, durations, L, sel: SelectorConfig, rng_seed: int):
        """score_candidates + select on one candidate set (selector.cpp:24-85)."""
        sims = np.ascontiguousarray(sims, np.float64)
        s_neg = np.ascontiguousarray(s_neg, np.float64)
        dur = np.ascontiguousarray(durations, np.float64)
        n = len(sims)
        scores = np.zeros((n, 5), np.float64)
        pick = np.zeros(2, np.int32)
        check(_lib.lib().sw_score_select_host(self._h, n, ptr(sims), ptr(s_neg), ptr(dur), L,
                                              C.byref(sel.c()), rng_seed, ptr(scores), ptr(pick)),
              "score_select")
        return scores, int(pick[0]), int(pick[1])

    def gater(self, prompts, segs, T, explore: bool = False):
        """context_features + choose_arm (gater.cpp:13-92) for B pairs."""
        p = np.ascontiguousarray(prompts, np.float32).reshape(-1, self.dim)
        s = np.ascontiguousarray(segs, np.float32).reshape(-1, self.dim)
        T = np.ascontiguousarray(np.broadcast_to(T, (p.shape[0],)), np.int32)
        B = p.shape[0]
        phi = np.zeros((B, 11), np.float64)
        arm = np.zeros(B, np.int32)
        check(_lib.lib().sw_gater_host(self._h, ptr(p), ptr(s), ptr(T), B, int(explore),
                                       ptr(phi), ptr(arm)), "gater")
        return phi, arm


class CacheManager:
    """CacheManager (cache.hpp:45-106): host policy in libsemwarm_b200 (csrc/host), data plane in
    the WarmStartCache's device arena. Method names follow the reference."""

    def __init__(self, cache: WarmStartCache, capacity: int = 1024, decay_per_hour: float = 0.9,
                 grace_hours: float = 1.0, quality_floor: float = 0.3, pyramid_delta: float = 0.25,
                 embedding_seed: int = 0, refine_regenerations: int = 3,
                 refine_attempt_cap: int = 5, refine_window: int = 10,
                 refine_skip_threshold: float = 0.10, latent_capacity: int = 0):
        self.cache = cache
        cfg = _lib.SwcmConfig(capacity, decay_per_hour, grace_hours, quality_floor,
                              pyramid_delta, embedding_seed, refine_regenerations,
                              refine_attempt_cap, refine_window, 0, refine_skip_threshold,
                              latent_capacity)
        h = C.c_void_p()
        check(_lib.lib().swcm_create(cache._h, cache.dim, C.byref(cfg), C.byref(h)),
              "swcm_create")
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.lib().swcm_destroy(self._h)
            self._h = None

    def admit(self, clip_embedding, duration_s, prompt_embedding, quality, now_h, latent=None):
        e = np.ascontiguousarray(clip_embedding, np.float32)
        pr = None if prompt_embedding is None else np.ascontiguousarray(prompt_embedding, np.float32)
        lat = None if latent is None else np.ascontiguousarray(latent, np.float32)
        out = C.c_uint64()
        rc = check(_lib.lib().swcm_admit(self._h, ptr(e), duration_s, ptr(pr), quality, now_h,
                                         ptr(lat), 0 if lat is None else lat.shape[1],
                                         C.byref(out)), "admit")
        return int(out.value) if rc == 1 else None

    def last_evicted(self):
        buf = np.zeros(4096, np.uint64)
        n = check(_lib.lib().swcm_last_evicted(self._h, ptr(buf), 4096), "last_evicted")
        return buf[:n].tolist()

    def record_reuse(self, entry_id, steps_skipped, duration_s, now_h, skip_fraction):
        rc = check(_lib.lib().swcm_record_reuse(self._h, entry_id, steps_skipped, duration_s,
                                                now_h, skip_fraction), "record_reuse")
        if rc == _lib.SW_WARN_UNKNOWN_ID:
            warnings.warn(f"record_reuse for unknown entry id {entry_id}")

    def evict_if_full(self, now_h):
        buf = np.zeros(4096, np.uint64)
        n = check(_lib.lib().swcm_evict_if_full(self._h, now_h, ptr(buf), 4096), "evict")
        return buf[:n].tolist()

    def refinement_candidates(self):
        buf = np.zeros(65536, np.uint64)
        n = check(_lib.lib().swcm_refinement_candidates(self._h, ptr(buf), 65536), "candidates")
        return buf[:n].tolist()

    def refine(self, entry_id, rng_seed, regenerate):
        """regenerate(prompt, duration_s, seed) -> (embedding, quality[, latent])."""
        dim = self.cache.dim

        def cb(user, prompt, d, duration, seed, emb_out, q_out, lat_out, t_out):
            pr = None if not prompt else np.ctypeslib.as_array(
                C.cast(prompt, C.POINTER(C.c_float)), (dim,)).copy()
            res = regenerate(pr, duration, int(seed))
            e = np.ascontiguousarray(res[0], np.float32)
            for i in range(dim):
                emb_out[i] = float(e[i])
            q_out[0] = float(res[1])
            t_out[0] = 0
            return 0

        fn = _lib.REGEN_FN(cb)
        replaced = C.c_int32()
        rc = check(_lib.lib().swcm_refine(self._h, entry_id, rng_seed, fn, None,
                                          C.byref(replaced)), "refine")
        if rc == _lib.SW_WARN_UNKNOWN_ID:
            warnings.warn(f"refine for unknown entry id {entry_id}")
        return bool(replaced.value)

    def current_importance(self, entry_id, now_h):
        out = C.c_double()
        check(_lib.lib().swcm_importance(self._h, entry_id, now_h, C.byref(out)), "importance")
        return out.value

    def size(self):
        return _lib.lib().swcm_size(self._h)

    def ids(self):
        buf = np.zeros(max(1, self.size()), np.uint64)
        n = _lib.lib().swcm_ids(self._h, ptr(buf), buf.shape[0])
        return buf[:n].tolist()

    def save_snapshot(self, directory: str):
        """CacheManager::save_snapshot (cache.cpp:211-243)."""
        check(_lib.lib().swcm_save_snapshot(self._h, directory.encode()), "swcm_save_snapshot")

    def load_snapshot(self, directory: str):
        """CacheManager::load_snapshot (cache.cpp:245-295) straight into the device arena."""
        check(_lib.lib().swcm_load_snapshot(self._h, directory.encode()), "swcm_load_snapshot")

    def check_consistent(self):
        return bool(_lib.lib().swcm_check_consistent(self._h))


class ShardGroup:
    """Entry-sharded warm start inside one process (sw_group_*, csrc/host/group.cpp): one
    context per shard, local exact top-k -> all-gather (NCCL across devices, peer copies when
    shards share one) -> replicated merge + select -> owner-computes align + noise. The Python
    face of the C++ caller's path; sharded.py is the multi-process (torch.distributed) one."""

    def __init__(self, dim: int, n_shards: int, devices=None, transport: str = "auto",
                 rows_per_entry: int = 7, max_entries: int = 1024, latent_shape=(8, 256, 16),
                 max_batch: int = 1024, latent_slots: int = 0, fps: float = 25.0,
                 exact_only: bool = False, tc_always: bool = False):
        L = _lib.lib()
        cfg = _lib.SwConfig()
        cfg.dim = dim
        cfg.rows_per_entry = rows_per_entry
        cfg.max_entries = max_entries
        cfg.latent_c, cfg.latent_t_max, cfg.latent_f = latent_shape if latent_shape else (0, 0, 0)
        cfg.max_batch = max_batch
        cfg.latent_slots = latent_slots
        cfg.latent_fps = fps
        cfg.flags = (_lib.SW_FLAG_EXACT_ONLY if exact_only else 0) | (
            _lib.SW_FLAG_TC_ALWAYS if tc_always else 0)
        devs = np.ascontiguousarray(devices if devices is not None else range(n_shards), np.int32)
        tr = {"auto": _lib.SW_GROUP_TRANSPORT_AUTO, "nccl": _lib.SW_GROUP_TRANSPORT_NCCL,
              "copy": _lib.SW_GROUP_TRANSPORT_COPY}[transport]
        h = C.c_void_p()
        check(L.sw_group_create(C.byref(cfg), n_shards, ptr(devs), tr, C.byref(h)),
              "sw_group_create")
        self._h = h
        self.dim, self.n_shards, self.max_batch = dim, n_shards, max_batch
        self.devices = [int(d) for d in devs]
        self.latent_shape = tuple(latent_shape) if latent_shape else None
        n, t = C.c_int32(), C.c_int32()
        check(L.sw_group_info(h, C.byref(n), C.byref(t)), "sw_group_info")
        self.transport = {1: "nccl", 2: "copy"}[t.value]

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().sw_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard(self, s: int) -> WarmStartCache:
        h = C.c_void_p()
        check(_lib.lib().sw_group_shard(self._h, s, C.byref(h)), "sw_group_shard")
        return WarmStartCache._borrow(h, self.dim, self.latent_shape, self.max_batch,
                                      self.devices[s])

    def owner(self, entry_id: int) -> int:
        return int(_lib.lib().sw_group_owner(self._h, entry_id))

    def set_negative(self, neg):
        neg = np.ascontiguousarray(neg, np.float32)
        check(_lib.lib().sw_group_set_negative(self._h, ptr(neg)), "sw_group_set_negative")

    def set_gater(self, theta, psi, beta: float = 1.0):
        theta = np.ascontiguousarray(theta, np.float32).reshape(-1)
        psi = np.ascontiguousarray(psi, np.float32).reshape(-1)
        check(_lib.lib().sw_group_set_gater(self._h, ptr(theta), ptr(psi), 11, beta),
              "sw_group_set_gater")

    def insert(self, entry_id: int, rows, levels, starts, lengths, latent=None):
        rows = np.ascontiguousarray(rows, np.float32).reshape(-1, self.dim)
        sg = segments(levels, starts, lengths)
        lat = None if latent is None else np.ascontiguousarray(latent, np.float32)
        t_src = 0 if lat is None else lat.shape[1]
        check(_lib.lib().sw_group_insert(self._h, entry_id, rows.shape[0], ptr(rows), ptr(sg),
                                         ptr(lat), t_src), "sw_group_insert")

    def remove(self, entry_id: int) -> bool:
        rc = _lib.lib().sw_group_remove(self._h, entry_id)
        check(rc, "sw_group_remove")
        return rc == _lib.SW_OK

    def warmstart_host(self, queries, reqs, seed: int = 1, sel: SelectorConfig = None,
                       policy: Policy = None, philox_seed: int = 0, outs=None,
                       t_out_max: int = 256) -> np.ndarray:
        """One batch from host arrays; outs: optional per-shard device tensors
        (B x C x t_out_max x F on that shard's device) for the owned latents."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        r = np.ascontiguousarray(reqs)
        B = q.shape[0]
        sel = sel or SelectorConfig()
        policy = policy or Policy()
        ch = np.zeros(B, _lib.CHOICE_DTYPE)
        arr = None
        if outs is not None:
            arr = (C.c_void_p * self.n_shards)(*[o.data_ptr() if o is not None else None
                                                 for o in outs])
        check(_lib.lib().sw_group_warmstart_host(self._h, ptr(q), ptr(r), B, seed,
                                                 C.byref(sel.c()), C.byref(policy.c()),
                                                 philox_seed, ptr(ch), arr, t_out_max),
              "sw_group_warmstart_host")
        return ch

    def shard_choices(self, s: int, B: int) -> np.ndarray:
        ch = np.zeros(B, _lib.CHOICE_DTYPE)
        check(_lib.lib().sw_group_shard_choices(self._h, s, B, ptr(ch)), "sw_group_shard_choices")
        return ch


def read_swem(path: str) -> np.ndarray:
    """load_embeddings (core.cpp:201-220): a SWEM file as a [count, dim] float32 array."""
    n, d = C.c_int32(), C.c_int32()
    nf = check(_lib.lib().sw_swem_read(path.encode(), None, 0, C.byref(n), C.byref(d)),
               "sw_swem_read")
    out = np.zeros(max(nf, 0), np.float32)
    check(_lib.lib().sw_swem_read(path.encode(), ptr(out), nf, None, None), "sw_swem_read")
    return out.reshape(n.value, d.value)


def time_stretch(clips, sample_rate: int, target_s, window: int = 128, hop: int = 32,
                 device: int = 0, stream=None):
    """time_stretch (vocoder.cpp:128-207) of a list of 1-D float32 clips on the GPU. Returns a
    list of float32 arrays (None where the reference would throw)."""
    torch = _torch()
    clips = [np.ascontiguousarray(c, np.float32) for c in clips]
    B = len(clips)
    in_len = np.array([c.shape[0] for c in clips], np.int32)
    in_off = np.concatenate([[0], np.cumsum(in_len)[:-1]]).astype(np.int64) if B else np.zeros(0, np.int64)
    flat = np.concatenate(clips) if B and in_len.sum() else np.zeros(1, np.float32)
    tgt = np.ascontiguousarray(target_s, np.float64)
    cap = int(sum(max(0, round(t * sample_rate)) for t in tgt)) + 1
    d_in = torch.from_numpy(flat).to(f"cuda:{device}")
    d_out = torch.zeros(cap, dtype=torch.float32, device=f"cuda:{device}")
    out_off = np.zeros(B, np.int64)
    out_len = np.zeros(B, np.int32)
    status = np.zeros(B, np.int32)
    st = stream if stream is not None else torch.cuda.current_stream(device).cuda_stream
    check(_lib.lib().sw_time_stretch(ptr(d_in), ptr(in_off), ptr(in_len), B, sample_rate,
                                     ptr(tgt), window, hop, ptr(d_out), cap, ptr(out_off),
                                     ptr(out_len), ptr(status), st), "sw_time_stretch")
    host = d_out.cpu().numpy()
    return [None if status[b] else host[out_off[b]:out_off[b] + out_len[b]].copy()
            for b in range(B)]


class Batcher:
    """swb_* (csrc/host/batcher.cpp): concurrent single-request callers -> device batches.
    submit() is thread-safe and blocking (ctypes releases the GIL while it waits)."""

    def __init__(self, cache: WarmStartCache, max_batch: int = 1024, max_wait_us: int = 200,
                 seed: int = 1, sel: SelectorConfig = None, policy: Policy = None,
                 philox_seed: int = 0, t_out_max: int = 0, with_latent: bool = False):
        self.cache = cache
        self._sel = (sel or SelectorConfig()).c()
        self._pol = (policy or Policy()).c()
        h = C.c_void_p()
        check(_lib.lib().swb_create(cache._h, max_batch, max_wait_us, seed, C.byref(self._sel),
                                    C.byref(self._pol), philox_seed, t_out_max, int(with_latent),
                                    C.byref(h)), "swb_create")
        self._h = h
        self.latent_shape = (cache.latent_shape[0], t_out_max, cache.latent_shape[2]) \
            if with_latent and cache.latent_shape else None

    def submit(self, prompt: np.ndarray, req: np.ndarray, want_latent: bool = False):
        """One request: prompt [D] float32, req a 1-element requests() record. Returns the
        choice record (and the aligned latent when the batcher was built with_latent)."""
        prompt = np.ascontiguousarray(prompt, np.float32)
        req = np.ascontiguousarray(req)
        ch = np.zeros(1, CHOICE_DTYPE)
        lat = np.zeros(self.latent_shape, np.float32) if (want_latent and self.latent_shape) else None
        check(_lib.lib().swb_submit(self._h, ptr(prompt), ptr(req), ptr(ch), ptr(lat)),
              "swb_submit")
        return (ch[0], lat) if want_latent else ch[0]

    def load_test(self, prompts, reqs, clients: int = 256, per_client: int = 64,
                  first_id: int = 1 << 40) -> dict:
        """swb_load_test: native client threads (no GIL), blocking submits, wall clock."""
        q = np.ascontiguousarray(prompts, np.float32).reshape(-1, self.cache.dim)
        r = np.ascontiguousarray(reqs)
        out = [C.c_double() for _ in range(4)]
        check(_lib.lib().swb_load_test(self._h, ptr(q), ptr(r), q.shape[0], clients, per_client,
                                       first_id, *[C.byref(x) for x in out]), "swb_load_test")
        return {"requests_per_s": out[0].value, "p50_ms": out[1].value, "p99_ms": out[2].value,
                "mean_batch": out[3].value}

    def stats(self):
        b, r = C.c_int64(), C.c_int64()
        check(_lib.lib().swb_stats(self._h, C.byref(b), C.byref(r)), "swb_stats")
        return {"batches": b.value, "requests": r.value}

    def close(self):
        if getattr(self, "_h", None):
            _lib.lib().swb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------- trace replay (config 5)
def _splitmix64(x: int) -> int:  # core.cpp:58-63
    M = (1 << 64) - 1
    x = (x + 0x9e3779b97f4a7c15) & M
    x = ((x ^ (x >> 30)) * 0xbf58476d1ce4e5b9) & M
    x = ((x ^ (x >> 27)) * 0x94d049bb133111eb) & M
    return x ^ (x >> 31)


def derive_seed(base: int, a: int, b: int = 0, c: int = 0) -> int:  # core.cpp:65-71
    s = _splitmix64(base ^ 0x53454d5741524d)
    s = _splitmix64(s ^ a)
    s = _splitmix64(s ^ b)
    return _splitmix64(s ^ c)


def negative_embedding(dim: int) -> np.ndarray:
    """make_negative_embedding (selector.cpp:16-20)."""
    out = np.zeros(dim, np.float32)
    check(_lib.lib().sw_negative_embedding(dim, ptr(out)), "sw_negative_embedding")
    return out


def synth_workload(n: int, dim: int = 512, seed: int = 7, **kw):
    """synth_workload (simgen.cpp:162-194), bit-identical: (prompts [n, dim], durations,
    arrivals, total_steps). kw overrides WorkloadConfig fields (simgen.hpp:87-98)."""
    w = _lib.SwrWorkload(n, kw.get("cluster_count", 16), dim, kw.get("near_duplicate_rate", 0.9),
                         kw.get("cluster_perturbation", 0.5), kw.get("duplicate_perturbation", 0.16),
                         kw.get("duration_lo_s", 4.0), kw.get("duration_hi_s", 12.0),
                         kw.get("arrival_rate_hz", 1.2), kw.get("total_steps", 200), 0)
    p = np.zeros((n, dim), np.float32)
    d, a = np.zeros(n), np.zeros(n)
    t = np.zeros(n, np.int32)
    check(_lib.lib().swr_synth_workload(C.byref(w), seed, ptr(p), ptr(d), ptr(a), ptr(t)),
          "swr_synth_workload")
    return p, d, a, t


class TraceReplay:
    """Pipeline::replay (pipeline.cpp:299-323) on the device: a WarmStartCache configured as the
    reference Pipeline configures its CacheManager (pipeline.cpp:66-82: IVF index with
    derive_seed(seed, "IDX") and the rebuild interval, embedding seed derive_seed(seed, "SEGM"),
    make_negative_embedding, the gater) plus the host Cache Manager policy, replayed by
    swr_replay with `batch` lookups per device call."""

    def __init__(self, dim: int = 512, capacity: int = 1024, seed: int = 1,
                 policy: Policy = None, sel: SelectorConfig = None, theta=None, psi=None,
                 beta: float = 1.0, centroids: int = 64, nprobe: int = 8,
                 rebuild_interval: int = 1024, delta: float = 0.25, max_batch: int = 1024,
                 device: int = 0):
        from .synth import pyramid
        self.dim, self.seed = dim, seed
        self.policy = policy or Policy()
        self.sel = sel or SelectorConfig()
        R = len(pyramid(1.0, delta)[0])
        self.cache = WarmStartCache(dim, rows_per_entry=R, max_entries=capacity,
                                    latent_shape=None, max_batch=max_batch, device=device)
        self.cache.ivf_configure(centroids, nprobe, rebuild_interval,
                                 derive_seed(seed, 0x494458))
        self.cache.set_negative(negative_embedding(dim))
        th = np.zeros(14 * 11, np.float32) if theta is None else theta
        ps = np.zeros(14 * 11, np.float32) if psi is None else psi
        self.cache.set_gater(th, ps, beta)
        self.cm = CacheManager(self.cache, capacity=capacity, pyramid_delta=delta,
                               embedding_seed=derive_seed(seed, 0x5345474D))

    def run(self, prompts, durations, arrivals, total_steps, batch: int = 64,
            refinement: bool = True):
        n = len(durations)
        cfg = _lib.SwrConfig(self.seed, self.sel.c(), self.policy.c(), 0.95, 2.0, 0.02, 0.75,
                             0.004, 0.47, 200, 200, int(refinement), batch)
        out = np.zeros(n, OUTCOME_DTYPE)
        st = _lib.SwrStats()
        pr = np.ascontiguousarray(prompts, np.float32)
        d = np.ascontiguousarray(durations, np.float64)
        a = np.ascontiguousarray(arrivals, np.float64)
        t = np.ascontiguousarray(total_steps, np.int32)
        check(_lib.lib().swr_replay(self.cache._h, self.cm._h, C.byref(cfg), n, ptr(pr), ptr(d),
                                    ptr(a), ptr(t), ptr(out), C.byref(st)), "swr_replay")
        return out, {f: getattr(st, f) for f, _ in st._fields_}

    def close(self):
        self.cm = None
        self.cache.close()
