"""TEST INFRASTRUCTURE ONLY — CPU checkers for the warm-start path.

Two checkers live here:

* ``Ref``    — the UNMODIFIED reference (``/root/reference/proj/src``) compiled in place by
               ``oracle/Makefile`` into ``oracle/_ref/libsemwarm_ref.so`` (+ ``ref_harness.cpp``).
* ``Oracle`` — our plain-C restatement (``oracle/semwarm_oracle.c``), pinned against ``Ref`` and
               the committed golden vectors in ``tests/golden``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline / reference legs
may import this package. The product path (``paper_2603_07865_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsemwarm_ref.so")
ORACLE_SO = os.path.join(HERE, "_build", "libsemwarm_oracle.so")

f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

# RefPlanOut / so_plan (identical layouts)
PLAN_DTYPE = np.dtype(
    [("hit", "<i4"), ("arm", "<i4"), ("steps_skipped", "<i4"), ("n_hits", "<i4"),
     ("entry_id", "<u8"), ("level", "<i4"), ("pick", "<i4"), ("start_s", "<f8"),
     ("length_s", "<f8"), ("similarity", "<f8")])
HIT_DTYPE = np.dtype(
    [("entry_id", "<u8"), ("level", "<i4"), ("row", "<i4"), ("start_s", "<f8"),
     ("length_s", "<f8"), ("similarity", "<f8")])

POLICY = {"exploit": 0, "explore": 1, "rule": 2, "fixed": 3}


def build(force: bool = False) -> None:
    """Compile both checkers (needs /root/reference for the ``ref`` target)."""
    import subprocess
    targets = ["oracle"]
    if os.path.isdir("/root/reference/proj/src"):
        targets += ["ref", "dropin"]  # dropin links the freshly built libsemwarm_b200.so
    subprocess.check_call(["make", "-s", "-C", HERE] + (["-B"] if force else []) + targets)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(f"oracle library missing: {path} (run `make -C oracle`)")
    return C.CDLL(path)


class Arena:
    """Flat cache view shared by both checkers: entry e owns rows [off[e], off[e+1])."""

    def __init__(self, ids, off, rows, levels, starts, lengths):
        self.ids = np.ascontiguousarray(ids, np.uint64)
        self.off = np.ascontiguousarray(off, np.int64)
        self.rows = np.ascontiguousarray(rows, np.float32)
        self.levels = np.ascontiguousarray(levels, np.int32)
        self.starts = np.ascontiguousarray(starts, np.float64)
        self.lengths = np.ascontiguousarray(lengths, np.float64)
        self.dim = int(self.rows.shape[1])
        self.n_entries = int(self.ids.shape[0])


class _SoArena(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_entries", C.c_int), ("ids", C.c_void_p),
                ("off", C.c_void_p), ("rows", C.c_void_p), ("levels", C.c_void_p),
                ("starts", C.c_void_p), ("lengths", C.c_void_p)]


class Oracle:
    """ctypes view of oracle/semwarm_oracle.c."""

    def __init__(self):
        L = self.lib = _load(ORACLE_SO)
        L.so_derive_seed.restype = C.c_uint64
        L.so_derive_seed.argtypes = [C.c_uint64] * 4
        L.so_mt64_first.restype = C.c_uint64
        L.so_mt64_first.argtypes = [C.c_uint64]
        L.so_uniform_first.restype = C.c_double
        L.so_uniform_first.argtypes = [C.c_uint64]
        L.so_cosine.restype = C.c_double
        L.so_cosine.argtypes = [f32p, f32p, C.c_int]
        L.so_search.restype = C.c_int
        L.so_plan_batch.restype = C.c_int
        L.so_align_noise.restype = C.c_int
        L.so_align_noise.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                     C.c_double, C.c_double, C.c_double, C.c_void_p, C.c_uint64,
                                     C.c_uint64, f32p]
        L.so_philox_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, f32p]
        L.so_ref_exp.restype = C.c_double
        L.so_ref_exp.argtypes = [C.c_double]
        L.so_exp_pair.argtypes = [f64p, C.c_int64, f64p, f64p]
        L.so_log1p_pair.argtypes = [f64p, C.c_int64, f64p, f64p]
        L.so_icdf_normals.argtypes = [np.ctypeslib.ndpointer(np.uint32, flags="C"), C.c_int64,
                                      f32p]
        L.so_abar_table.argtypes = [f64p]
        L.so_abar_index.restype = C.c_int
        L.so_abar_index.argtypes = [C.c_int, C.c_int]
        L.so_context_features.argtypes = [f32p, f32p, C.c_int, C.c_int, f64p]
        L.so_choose_arm.restype = C.c_int
        L.so_choose_arm.argtypes = [f32p, f32p, C.c_int, C.c_double, f64p, C.c_int]
        L.so_score_select.restype = C.c_int
        L.so_score_select.argtypes = [C.c_int, f64p, f64p, f32p, C.c_int, f32p, C.c_double,
                                      C.c_double, C.c_double, C.c_uint64, f64p, f64p, f64p,
                                      f64p, f64p]

    def _arena(self, ar: Arena) -> _SoArena:
        return _SoArena(ar.dim, ar.n_entries, ar.ids.ctypes.data, ar.off.ctypes.data,
                        ar.rows.ctypes.data, ar.levels.ctypes.data, ar.starts.ctypes.data,
                        ar.lengths.ctypes.data)

    def derive_seed(self, base, a, b=0, c=0) -> int:
        return self.lib.so_derive_seed(base, a, b, c)

    def mt64_first(self, seed) -> int:
        return self.lib.so_mt64_first(seed)

    def uniform_first(self, seed) -> float:
        return self.lib.so_uniform_first(seed)

    def search(self, ar: Arena, q: np.ndarray, k: int) -> np.ndarray:
        out = np.zeros(k, HIT_DTYPE)
        sa = self._arena(ar)
        q = np.ascontiguousarray(q, np.float32)
        n = self.lib.so_search(C.byref(sa), q.ctypes.data_as(C.c_void_p), C.c_int(k),
                               out.ctypes.data_as(C.c_void_p))
        return out[:n]

    def plan_batch(self, ar: Arena, neg, queries, L, req_ids, T, *, seed=1, top_k=8, temp=0.05,
                   thr=0.6, policy="exploit", theta=None, psi=None, beta=1.0, rule_thr=0.35,
                   rule_arm=11, fixed_arm=0, nthreads=1):
        B = queries.shape[0]
        out = np.zeros(B, PLAN_DTYPE)
        hits = np.zeros(B * top_k, HIT_DTYPE)
        theta = np.zeros(14 * 11, np.float32) if theta is None else np.ascontiguousarray(theta, np.float32)
        psi = np.zeros(14 * 11, np.float32) if psi is None else np.ascontiguousarray(psi, np.float32)
        sa = self._arena(ar)
        queries = np.ascontiguousarray(queries, np.float32)
        neg = np.ascontiguousarray(neg, np.float32)
        L = np.ascontiguousarray(L, np.float64)
        req_ids = np.ascontiguousarray(req_ids, np.uint64)
        T = np.ascontiguousarray(T, np.int32)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        rc = self.lib.so_plan_batch(
            C.byref(sa), vp(neg), C.c_int(B), vp(queries), vp(L), vp(req_ids), vp(T),
            C.c_uint64(seed), C.c_int(top_k), C.c_double(temp), C.c_double(thr),
            C.c_int(POLICY[policy]), vp(theta), vp(psi), C.c_int(11), C.c_double(beta),
            C.c_double(rule_thr), C.c_int(rule_arm), C.c_int(fixed_arm), C.c_int(nthreads),
            vp(out), vp(hits))
        if rc != 0:
            raise ValueError("so_plan_batch failed")
        return out, hits.reshape(B, top_k)

    def align_noise(self, latent, start_s, length_s, L, fps, abar, eps=None, seed=0, rid=0):
        latent = np.ascontiguousarray(latent, np.float32)
        C_, t_src, F = latent.shape
        t_out = int(np.round(L * fps)) + 2
        out = np.zeros(C_ * t_out * F, np.float32)
        ep = None
        if eps is not None:
            eps = np.ascontiguousarray(eps, np.float32)
            ep = eps.ctypes.data
        n = self.lib.so_align_noise(latent, C_, t_src, F, start_s, length_s, L, fps, abar, ep,
                                    seed, rid, out)
        return out[: C_ * n * F].reshape(C_, n, F)

    def philox_normals(self, seed, rid, n):
        out = np.zeros(n, np.float32)
        self.lib.so_philox_normals(seed, rid, n, out)
        return out

    def exp_pair(self, x):
        x = np.ascontiguousarray(x, np.float64)
        ours, lib = np.zeros_like(x), np.zeros_like(x)
        self.lib.so_exp_pair(x, x.size, ours, lib)
        return ours, lib

    def log1p_pair(self, x):
        x = np.ascontiguousarray(x, np.float64)
        ours, lib = np.zeros_like(x), np.zeros_like(x)
        self.lib.so_log1p_pair(x, x.size, ours, lib)
        return ours, lib

    def icdf_normals(self, words):
        words = np.ascontiguousarray(words, np.uint32)
        out = np.zeros(words.size, np.float32)
        self.lib.so_icdf_normals(words, words.size, out)
        return out

    def abar_table(self):
        t = np.zeros(1001, np.float64)
        self.lib.so_abar_table(t)
        return t

    def abar_index(self, T, S):
        return self.lib.so_abar_index(T, S)

    def context_features(self, p, c, T):
        phi = np.zeros(11, np.float64)
        p = np.ascontiguousarray(p, np.float32)
        c = np.ascontiguousarray(c, np.float32)
        self.lib.so_context_features(p, c, p.shape[0], T, phi)
        return phi

    def choose_arm(self, theta, psi, beta, phi, explore=False):
        return self.lib.so_choose_arm(np.ascontiguousarray(theta, np.float32),
                                      np.ascontiguousarray(psi, np.float32), 11, beta,
                                      np.ascontiguousarray(phi, np.float64), int(explore))


class Ref:
    """ctypes view of the compiled reference (oracle/_ref/libsemwarm_ref.so)."""

    def __init__(self):
        L = self.lib = _load(REF_SO)
        L.ref_derive_seed.restype = C.c_uint64
        L.ref_derive_seed.argtypes = [C.c_uint64] * 4
        L.ref_rng_first_u64.restype = C.c_uint64
        L.ref_rng_first_u64.argtypes = [C.c_uint64]
        L.ref_rng_first_uniform.restype = C.c_double
        L.ref_rng_first_uniform.argtypes = [C.c_uint64]
        L.ref_cosine.restype = C.c_double
        L.ref_cosine.argtypes = [f32p, f32p, C.c_int]
        L.ref_random_unit_vector.argtypes = [C.c_uint64, C.c_int, f32p]
        L.ref_random_unit_vectors.argtypes = [C.c_uint64, C.c_int, C.c_int, f32p]
        L.ref_perturb.argtypes = [f32p, C.c_int, C.c_double, C.c_uint64, f32p]
        L.ref_make_negative.argtypes = [C.c_int, f32p]
        L.ref_pyramid_segments.restype = C.c_int
        L.ref_pyramid_segments.argtypes = [C.c_double, C.c_double, i32p, f64p, f64p, C.c_int]
        L.ref_build_entry_vectors.restype = C.c_int
        L.ref_build_entry_vectors.argtypes = [C.c_uint64, f32p, C.c_int, C.c_double, C.c_double,
                                              C.c_uint64, f32p, i32p, f64p, f64p, C.c_int]
        L.ref_index_new.restype = C.c_void_p
        L.ref_index_new.argtypes = [C.c_int]
        L.ref_index_free.argtypes = [C.c_void_p]
        L.ref_ivf_new.restype = C.c_void_p
        L.ref_ivf_new.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64]
        L.ref_index_save.restype = C.c_int
        L.ref_index_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_index_load.restype = C.c_void_p
        L.ref_index_load.argtypes = [C.c_char_p, C.c_int]
        L.ref_index_new_loaded.restype = C.c_void_p
        L.ref_index_new_loaded.argtypes = [C.c_char_p, C.c_int, C.c_int, u64p, i64p, f32p, i32p,
                                           f64p, f64p]
        L.ref_time_stretch.restype = C.c_int
        L.ref_time_stretch.argtypes = [f32p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int,
                                       f32p, C.c_int]
        L.ref_synth_latent.restype = C.c_int
        L.ref_synth_latent.argtypes = [f32p, C.c_int, C.c_double, C.c_int, f32p, C.c_int]
        L.ref_save_embeddings.restype = C.c_int
        L.ref_save_embeddings.argtypes = [C.c_char_p, f32p, C.c_int, C.c_int]
        L.ref_index_check_consistent.restype = C.c_int
        L.ref_index_check_consistent.argtypes = [C.c_void_p]
        L.ref_index_insert_many.restype = C.c_int
        L.ref_index_insert_many.argtypes = [C.c_void_p, C.c_int, u64p, i64p, f32p, i32p, f64p, f64p]
        L.ref_index_remove.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_index_search.restype = C.c_int
        L.ref_index_search.argtypes = [C.c_void_p, f32p, C.c_int, u64p, i32p, f64p, f64p, f64p]
        L.ref_plan_batch.restype = C.c_int
        L.ref_context_features.argtypes = [f32p, f32p, C.c_int, C.c_int, f64p]
        L.ref_choose_arm.restype = C.c_int
        L.ref_choose_arm.argtypes = [f32p, f32p, C.c_int, C.c_double, f64p, C.c_int]
        L.ref_score_select.restype = C.c_int
        L.ref_score_select.argtypes = [C.c_int, u64p, i32p, f64p, f64p, f64p, f32p, C.c_int,
                                       f32p, f32p, C.c_double, C.c_int, C.c_double, C.c_double,
                                       C.c_uint64, f64p, f64p, f64p, f64p, f64p]
        L.ref_expected_quality.restype = C.c_double
        L.ref_expected_quality.argtypes = [C.c_double, C.c_double]
        L.ref_arm_skip_fraction.restype = C.c_double
        L.ref_arm_skip_fraction.argtypes = [C.c_int]
        # cache manager
        L.ref_cache_new.restype = C.c_void_p
        L.ref_cache_new.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.c_uint64]
        L.ref_cache_new_ivf.restype = C.c_void_p
        L.ref_cache_new_ivf.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.c_int, C.c_int, C.c_uint64,
                                        C.c_uint64]
        L.ref_cache_free.argtypes = [C.c_void_p]
        L.ref_cache_index_save.restype = C.c_int
        L.ref_cache_index_save.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_cache_admit.restype = C.c_int64
        L.ref_cache_admit.argtypes = [C.c_void_p, f32p, C.c_int, C.c_double, C.c_double, C.c_double]
        L.ref_cache_record_reuse.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_double,
                                             C.c_double, C.c_double]
        L.ref_cache_evict.restype = C.c_int
        L.ref_cache_evict.argtypes = [C.c_void_p, C.c_double, u64p, C.c_int]
        L.ref_cache_importance.restype = C.c_double
        L.ref_cache_importance.argtypes = [C.c_void_p, C.c_uint64, C.c_double]
        L.ref_cache_size.restype = C.c_int
        L.ref_cache_size.argtypes = [C.c_void_p]
        L.ref_cache_ids.restype = C.c_int
        L.ref_cache_ids.argtypes = [C.c_void_p, u64p, C.c_int]
        L.ref_cache_refinement_candidates.restype = C.c_int
        L.ref_cache_refinement_candidates.argtypes = [C.c_void_p, u64p, C.c_int]
        L.ref_cache_refine.restype = C.c_int
        L.ref_cache_refine.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, f64p, f32p, C.c_int,
                                       C.c_int, u64p]
        L.ref_cache_search.restype = C.c_int
        L.ref_cache_search.argtypes = [C.c_void_p, f32p, C.c_int, C.c_int, u64p, i32p, f64p,
                                       f64p, f64p]
        L.ref_cache_entry_rows.restype = C.c_int
        L.ref_cache_entry_rows.argtypes = [C.c_void_p, C.c_uint64, f32p, C.c_int]
        L.ref_cache_save_snapshot.restype = C.c_int
        L.ref_cache_save_snapshot.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_cache_load_snapshot.restype = C.c_int
        L.ref_cache_load_snapshot.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_cache_check_consistent.restype = C.c_int
        L.ref_cache_check_consistent.argtypes = [C.c_void_p]
        L.ref_cache_admit_clip.restype = C.c_int64
        L.ref_cache_admit_clip.argtypes = [C.c_void_p, f32p, f32p, C.c_int, C.c_double,
                                           C.c_double, C.c_double, f32p, C.c_int, C.c_int,
                                           C.c_uint64, C.c_double]
        L.ref_cache_entry_state.restype = C.c_int
        L.ref_cache_entry_state.argtypes = [C.c_void_p, C.c_uint64, f64p, f64p, C.c_int]
        L.ref_cache_clip.restype = C.c_int
        L.ref_cache_clip.argtypes = [C.c_void_p, C.c_uint64, f32p, C.c_int,
                                     C.POINTER(C.c_int), C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_double), f32p]
        L.ref_bandit_save.restype = C.c_int
        L.ref_bandit_save.argtypes = [C.c_char_p, f32p, f32p, C.c_int]
        L.ref_bandit_load.restype = C.c_int
        L.ref_bandit_load.argtypes = [C.c_char_p, f32p, f32p, C.c_int]

        L.ref_synth_workload.restype = C.c_int
        L.ref_synth_workload.argtypes = [C.c_int64, C.c_int, C.c_uint64, f32p, f64p, f64p, i32p]
        L.ref_replay.restype = C.c_int
        L.ref_replay.argtypes = [C.c_int64, C.c_int, f32p, f64p, f64p, i32p, C.c_uint64, C.c_int,
                                 C.c_void_p, C.c_void_p, C.c_double, C.c_int, C.c_uint64,
                                 C.c_int, C.c_void_p, f64p, C.POINTER(C.c_double)]

    # -- helpers
    def derive_seed(self, base, a, b=0, c=0):
        return self.lib.ref_derive_seed(base, a, b, c)

    def synth_workload(self, n, dim, seed):
        """the reference's synth_workload (simgen.cpp:162-194), default WorkloadConfig"""
        p = np.zeros((n, dim), np.float32)
        d, a = np.zeros(n), np.zeros(n)
        t = np.zeros(n, np.int32)
        self.lib.ref_synth_workload(n, dim, seed, p, d, a, t)
        return p, d, a, t

    def replay(self, prompts, durations, arrivals, steps, *, capacity=1024, policy="exploit",
               theta=None, psi=None, beta=1.0, fixed_arm=0, seed=1, batch=0):
        """batch 0: the reference's own Pipeline::replay; batch >= 1: the same flow with batched
        lookups against per-batch snapshots (ref_harness.cpp ref_replay). Returns (outcomes in
        OUTCOME_DTYPE layout, summary dict, wall seconds)."""
        from paper_2603_07865_b200._lib import OUTCOME_DTYPE
        n, dim = prompts.shape
        out = np.zeros(n, OUTCOME_DTYPE)
        summ = np.zeros(10)
        wall = C.c_double()
        th = None if theta is None else np.ascontiguousarray(theta, np.float32)
        ps = None if psi is None else np.ascontiguousarray(psi, np.float32)
        rc = self.lib.ref_replay(n, dim, np.ascontiguousarray(prompts, np.float32),
                                 np.ascontiguousarray(durations, np.float64),
                                 np.ascontiguousarray(arrivals, np.float64),
                                 np.ascontiguousarray(steps, np.int32), capacity, POLICY[policy],
                                 None if th is None else th.ctypes.data,
                                 None if ps is None else ps.ctypes.data, beta, fixed_arm, seed,
                                 batch, out.ctypes.data, summ, C.byref(wall))
        if rc != n:
            raise RuntimeError(f"ref_replay failed ({rc})")
        keys = ["total_nfe_s", "baseline_nfe_s", "speedup", "mean_quality", "mean_reward",
                "hit_rate", "mean_latency_s", "median_latency_s", "p95_latency_s", "refinements"]
        return out, dict(zip(keys, summ.tolist())), wall.value

    def random_unit_vectors(self, seed, n, dim):
        out = np.zeros((n, dim), np.float32)
        self.lib.ref_random_unit_vectors(seed, n, dim, out)
        return out

    def perturb(self, v, scale, seed):
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros_like(v)
        self.lib.ref_perturb(v, v.shape[0], scale, seed, out)
        return out

    def negative(self, dim):
        out = np.zeros(dim, np.float32)
        self.lib.ref_make_negative(dim, out)
        return out

    def pyramid(self, duration, delta):
        lv = np.zeros(64, np.int32)
        st = np.zeros(64, np.float64)
        ln = np.zeros(64, np.float64)
        n = self.lib.ref_pyramid_segments(duration, delta, lv, st, ln, 64)
        return lv[:n], st[:n], ln[:n]

    def build_entry_vectors(self, eid, full, duration, delta, seed_base):
        full = np.ascontiguousarray(full, np.float32)
        dim = full.shape[0]
        rows = np.zeros((64, dim), np.float32)
        lv = np.zeros(64, np.int32)
        st = np.zeros(64, np.float64)
        ln = np.zeros(64, np.float64)
        n = self.lib.ref_build_entry_vectors(eid, full, dim, duration, delta, seed_base, rows,
                                             lv, st, ln, 64)
        return rows[:n].copy(), lv[:n].copy(), st[:n].copy(), ln[:n].copy()

    # -- index
    def index(self, ar: Arena, ivf=None):
        return RefIndex(self, ar, ivf)

    def load_index(self, path: str, dim: int):
        """IvfIndex::load of a SWIX snapshot (search / save / consistency only)."""
        ri = RefIndex.__new__(RefIndex)
        ri.ref, ri.ar = self, None
        ri.h = self.lib.ref_index_load(path.encode(), dim)
        if not ri.h:
            raise RuntimeError("reference failed to load " + path)
        return ri

    def load_index_with_arena(self, path: str, ar: Arena):
        """SWIX index + arena rows for candidate assembly (plan_batch works on it)."""
        ri = RefIndex.__new__(RefIndex)
        ri.ref, ri.ar = self, ar
        ri.h = self.lib.ref_index_new_loaded(path.encode(), ar.dim, ar.n_entries, ar.ids, ar.off,
                                             ar.rows, ar.levels, ar.starts, ar.lengths)
        if not ri.h:
            raise RuntimeError("reference failed to load " + path)
        return ri

    def time_stretch(self, x, rate, target_s, window=128, hop=32):
        """vocoder.cpp:128-207; None when the reference throws."""
        x = np.ascontiguousarray(x, np.float32)
        cap = max(0, int(round(target_s * rate))) + 8
        out = np.zeros(cap, np.float32)
        n = self.lib.ref_time_stretch(x, x.shape[0], rate, target_s, window, hop, out, cap)
        return None if n < 0 else out[:n].copy()

    def synth_latent(self, emb, duration_s, rate=200):
        emb = np.ascontiguousarray(emb, np.float32)
        cap = int(round(duration_s * rate)) + 8
        out = np.zeros(cap, np.float32)
        n = self.lib.ref_synth_latent(emb, emb.shape[0], duration_s, rate, out, cap)
        return out[:n].copy()

    def save_embeddings(self, path: str, v: np.ndarray):
        v = np.ascontiguousarray(v, np.float32)
        if self.lib.ref_save_embeddings(path.encode(), v, v.shape[0], v.shape[1]) != 0:
            raise RuntimeError("save_embeddings failed")

    def context_features(self, p, c, T):
        phi = np.zeros(11, np.float64)
        p = np.ascontiguousarray(p, np.float32)
        c = np.ascontiguousarray(c, np.float32)
        self.lib.ref_context_features(p, c, p.shape[0], T, phi)
        return phi

    def choose_arm(self, theta, psi, beta, phi, explore=False):
        return self.lib.ref_choose_arm(np.ascontiguousarray(theta, np.float32),
                                       np.ascontiguousarray(psi, np.float32), 11, beta,
                                       np.ascontiguousarray(phi, np.float64), int(explore))


def parse_swix(path: str):
    """SWIX snapshot (index.cpp:347-369) -> (centroids [C][D] f32, nprobe, lists) where lists[j]
    is the list's records in order: (entry_id, level, start_s f32, length_s f32)."""
    import struct
    b = open(path, "rb").read()
    assert b[:4] == b"SWIX", "bad magic"
    C_, nprobe, D = struct.unpack_from("<III", b, 4)
    o = 16
    cent = np.frombuffer(b, np.float32, C_ * D, o).reshape(C_, D).copy()
    o += 4 * C_ * D
    lists = []
    for _ in range(C_):
        (cnt,) = struct.unpack_from("<Q", b, o)
        o += 8
        recs = []
        for _ in range(cnt):
            eid, lvl = struct.unpack_from("<QB", b, o)
            st, ln = struct.unpack_from("<ff", b, o + 9)
            recs.append((eid, lvl, st, ln))
            o += 17 + 4 * D
        lists.append(recs)
    assert o == len(b)
    return cent, nprobe, lists


class RefIndex:
    """Reference IvfIndex over an Arena (kept alive here): exhaustive parity mode by default,
    or IVF mode (ivf = (centroids, seed, nprobe, rebuild_interval)) as CacheManager builds it."""

    def __init__(self, ref: Ref, ar: Arena, ivf=None):
        self.ref, self.ar = ref, ar
        if ivf is None:
            self.h = ref.lib.ref_index_new(ar.dim)
        else:
            c, seed, nprobe, interval = ivf
            self.h = ref.lib.ref_ivf_new(ar.dim, c, seed, nprobe, interval)
        if ar.n_entries:
            rc = ref.lib.ref_index_insert_many(self.h, ar.n_entries, ar.ids, ar.off, ar.rows,
                                               ar.levels, ar.starts, ar.lengths)
            if rc != 0:
                raise RuntimeError("reference insert failed")

    def insert(self, ar: Arena):
        """Inserts more entries (the arena must stay alive: candidate assembly reads it)."""
        self._keep = getattr(self, "_keep", []) + [ar]
        rc = self.ref.lib.ref_index_insert_many(self.h, ar.n_entries, ar.ids, ar.off, ar.rows,
                                                ar.levels, ar.starts, ar.lengths)
        if rc != 0:
            raise RuntimeError("reference insert failed")

    def snapshot(self):
        import tempfile
        with tempfile.NamedTemporaryFile(suffix=".swix") as f:
            n = self.ref.lib.ref_index_save(self.h, f.name.encode())
            if n < 0:
                raise RuntimeError("save failed")
            return parse_swix(f.name)

    def consistent(self) -> bool:
        return bool(self.ref.lib.ref_index_check_consistent(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_index_free(self.h)
            self.h = None

    def remove(self, eid):
        self.ref.lib.ref_index_remove(self.h, eid)

    def search(self, q, k):
        ids = np.zeros(k, np.uint64)
        lv = np.zeros(k, np.int32)
        st = np.zeros(k, np.float64)
        ln = np.zeros(k, np.float64)
        sm = np.zeros(k, np.float64)
        n = self.ref.lib.ref_index_search(self.h, np.ascontiguousarray(q, np.float32), k, ids, lv,
                                          st, ln, sm)
        return ids[:n], lv[:n], st[:n], ln[:n], sm[:n]

    def plan_batch(self, neg, queries, L, req_ids, T, *, seed=1, top_k=8, temp=0.05, thr=0.6,
                   policy="exploit", theta=None, psi=None, beta=1.0, rule_thr=0.35,
                   rule_skip=0.55, fixed_arm=0, nthreads=1):
        B = queries.shape[0]
        out = np.zeros(B, PLAN_DTYPE)
        hit_ids = np.zeros(B * top_k, np.uint64)
        hit_sims = np.zeros(B * top_k, np.float64)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)
        queries = np.ascontiguousarray(queries, np.float32)
        neg = np.ascontiguousarray(neg, np.float32)
        L = np.ascontiguousarray(L, np.float64)
        req_ids = np.ascontiguousarray(req_ids, np.uint64)
        T = np.ascontiguousarray(T, np.int32)
        theta = None if theta is None else np.ascontiguousarray(theta, np.float32)
        psi = None if psi is None else np.ascontiguousarray(psi, np.float32)
        rc = self.ref.lib.ref_plan_batch(
            C.c_void_p(self.h), vp(neg), C.c_int(B), vp(queries), vp(L), vp(req_ids), vp(T),
            C.c_uint64(seed), C.c_int(top_k), C.c_double(temp), C.c_double(thr),
            C.c_int(POLICY[policy]), None if theta is None else vp(theta),
            None if psi is None else vp(psi), C.c_int(11), C.c_double(beta),
            C.c_double(rule_thr), C.c_double(rule_skip), C.c_int(fixed_arm), C.c_int(nthreads),
            vp(out), vp(hit_ids), vp(hit_sims))
        if rc != 0:
            raise RuntimeError("ref_plan_batch failed")
        return out, hit_ids.reshape(B, top_k), hit_sims.reshape(B, top_k)
