"""GPU parity where the tcgen05 pre-filter's candidate slices overflow.

Thousands of bit-identical rows (and near-duplicates) in one query's range make a scoring slice
emit more certified candidates than it can hold. Such a query is then re-searched by the
certified fallback (k_overflow: an exact fp64 brute-force IvfIndex::search over the whole arena,
index.cpp:289-326) — every result below must still equal the C restatement / the unmodified
reference exactly, with no SW_CHOICE_INCOMPLETE flag anywhere, and the fallback must have run.
Also: BASELINE config 3's full size (1M x 512, B = 1024) on (a) 20K identical copies of a row and
(b) the §8d(ii) clustered near-duplicate distribution, ALL 1024 requests checked."""
import os

import numpy as np
import pytest

import oracle
from paper_2603_07865_b200 import _lib
from paper_2603_07865_b200.synth import (SynthCache, clustered_rows, normalize_rows,
                                         trained_like_gater)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FIELDS = ("hit", "arm", "steps_skipped", "n_hits", "entry_id", "level", "pick", "start_s",
          "length_s", "similarity")
NT = max(1, min(64, os.cpu_count() or 1))


def _perturb(rng, src, scale):
    g = rng.standard_normal(src.shape)
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    return normalize_rows(src.astype(np.float64) + scale * g.astype(np.float32).astype(np.float64))


def _dup_rows(n, D, a, n_dup, n_near, seed):
    rng = np.random.default_rng(seed)
    rows = np.empty((n, D), np.float32)
    for i in range(0, n, 65536):
        m = min(65536, n - i)
        rows[i:i + m] = normalize_rows(rng.standard_normal((m, D), dtype=np.float32))
    rows[a:a + n_dup] = rows[a]                                  # bit-identical copies
    rows[a + n_dup:a + n_dup + n_near] = _perturb(rng, np.repeat(rows[a:a + 1], n_near, 0), 0.01)
    return rows


def _queries(rng, rows, a, B):
    """a quarter near the duplicated row (two distances), the rest near random rows"""
    q1 = _perturb(rng, np.repeat(rows[a:a + 1], B // 4, 0), 0.3)
    q2 = _perturb(rng, np.repeat(rows[a:a + 1], B // 4, 0), 0.02)
    q3 = _perturb(rng, rows[rng.integers(0, rows.shape[0], B - 2 * (B // 4))], 0.3)
    q = np.concatenate([q1, q2, q3])
    return q[rng.permutation(B)]


def _plan(wc, q, L, rid, T, th, ps, k=8, policy="exploit"):
    from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, requests
    return wc.choices(wc.plan(q, requests(rid, L, T), seed=1, sel=SelectorConfig(k),
                              policy=Policy(policy)))


def _no_flags(ch):
    bad = _lib.SW_CHOICE_INCOMPLETE | _lib.SW_CHOICE_AMBIGUOUS_DRAW | _lib.SW_CHOICE_AMBIGUOUS_ARM
    assert ((ch["flags"] & bad) == 0).all()


def _flat_cache(rows, dur, B, **kw):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    n, D = rows.shape
    wc = WarmStartCache(D, rows_per_entry=1, max_entries=n, max_batch=B, latent_shape=None, **kw)
    ids = np.arange(1, n + 1, dtype=np.uint64)
    off = np.arange(n + 1, dtype=np.int64)
    wc.insert_batch(ids, off, rows, np.zeros(n, np.int32), np.zeros(n), dur)
    return wc, oracle.Arena(ids, off, rows, np.zeros(n, np.int32), np.zeros(n), dur)


@pytest.mark.parametrize("k", [1, 8, 32])
def test_overflow_search_and_plan_match_oracle(orc, k):
    n, D, B, a = 100_000, 512, 256, 777
    rows = _dup_rows(n, D, a, 20_000, 2_000, seed=41)
    dur = np.random.default_rng(1).uniform(4, 12, n)
    rng = np.random.default_rng(42)
    q = _queries(rng, rows, a, B)
    neg = normalize_rows(rng.standard_normal((1, D)))[0]
    th, ps = trained_like_gater()
    wc, ar = _flat_cache(rows, dur, B)
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    before = wc.overflow_fallbacks()
    hits, cnt = wc.search(q, k)
    assert wc.overflow_fallbacks() > before, "the duplicates must overflow the slices"
    for i in range(B):
        h = orc.search(ar, q[i], k)
        assert cnt[i] == len(h)
        np.testing.assert_array_equal(hits[i, :cnt[i]]["entry_id"], h["entry_id"], err_msg=f"q{i}")
        np.testing.assert_array_equal(hits[i, :cnt[i]]["similarity"], h["similarity"])
    L = rng.uniform(2.5, 10.0, B)
    rid = np.arange(1, B + 1, dtype=np.uint64)
    T = np.full(B, 200, np.int32)
    ch = _plan(wc, q, L, rid, T, th, ps, k=k)
    _no_flags(ch)
    exp, _ = orc.plan_batch(ar, neg, q, L, rid, T, top_k=k, policy="exploit", theta=th, psi=ps,
                            nthreads=NT)
    for f in FIELDS:
        np.testing.assert_array_equal(ch[f], exp[f], err_msg=f)
    wc.close()


def test_overflow_pyramid_and_async_path(orc):
    """R = 7 pyramid entries, 30K identical entries (a slice spans ~400 entries, more than it
    can emit); the pipelined entry point agrees."""
    import ctypes as C

    from paper_2603_07865_b200.warmstart import (Policy, SelectorConfig, WarmStartCache,
                                                 requests)
    c = SynthCache(60_000, 128, 0.25, seed=8)
    R, D = c.R, c.dim
    e0 = 100
    c.rows.reshape(-1, R, D)[e0 + 1:e0 + 30_001] = c.rows.reshape(-1, R, D)[e0]  # copies of e0
    B = 128
    rng = np.random.default_rng(9)
    src = np.concatenate([np.repeat(c.rows[c.off[e0]:c.off[e0] + 1], B // 2, 0),
                          c.rows[c.off[rng.integers(0, len(c.ids), B - B // 2)]]])
    q = _perturb(rng, src, 0.1)
    wc = WarmStartCache(D, rows_per_entry=R, max_entries=len(c.ids), max_batch=B,
                        latent_shape=(2, 32, 4), tc_always=True)
    neg = normalize_rows(rng.standard_normal((1, D)))[0]
    th, ps = trained_like_gater()
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    L = rng.uniform(2.5, 10.0, B)
    rid = np.arange(1, B + 1, dtype=np.uint64)
    T = np.full(B, 100, np.int32)
    n0 = wc.overflow_fallbacks()
    ch = _plan(wc, q, L, rid, T, th, ps)
    assert wc.overflow_fallbacks() > n0
    _no_flags(ch)
    ar = oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    exp, _ = orc.plan_batch(ar, neg, q, L, rid, T, top_k=8, policy="exploit", theta=th, psi=ps,
                            nthreads=NT)
    for f in FIELDS:
        np.testing.assert_array_equal(ch[f], exp[f], err_msg=f)
    dev = torch.device("cuda", 0)
    qd = torch.from_numpy(np.ascontiguousarray(q, np.float32)).to(dev)
    rd = torch.from_numpy(requests(rid, L, T).view(np.uint8)).to(dev)
    out = torch.zeros((B, 2, 32, 4), dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    Lb = _lib.lib()
    sel, pol = SelectorConfig(8), Policy("exploit")
    bufs = []
    for rep in range(3):  # several batches in flight share the fallback state
        cha = torch.zeros(B * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        _lib.check(Lb.sw_warmstart_async(wc._h, qd.data_ptr(), rd.data_ptr(), B, 1,
                                         C.byref(sel.c()), C.byref(pol.c()), None, 7,
                                         cha.data_ptr(), out.data_ptr(), 32, st), "async")
        bufs.append(cha)
    _lib.check(Lb.sw_join(wc._h, st), "join")
    torch.cuda.synchronize(dev)
    for cha in bufs:
        cha = cha.cpu().numpy().view(_lib.CHOICE_DTYPE)
        for f in ("hit", "arm", "steps_skipped", "n_hits", "entry_id", "similarity", "pick"):
            np.testing.assert_array_equal(cha[f], ch[f], err_msg=f)
    wc.close()


def test_overflow_ivf_matches_reference(ref, tmp_path):
    """IVF mode (16 lists, nprobe 4) with 20K identical rows: the fallback scans only rows of
    probed lists and breaks an entry's ties in the reference's scan order."""
    n, D, B, a = 60_000, 128, 128, 5000
    rows = _dup_rows(n, D, a, 20_000, 1_000, seed=5)
    # SWIX stores segment lengths as float32 (index.cpp:345-408)
    dur = np.random.default_rng(2).uniform(4, 12, n).astype(np.float32).astype(np.float64)
    rng = np.random.default_rng(6)
    q = _queries(rng, rows, a, B)
    neg = ref.negative(D)
    th, ps = trained_like_gater()
    from paper_2603_07865_b200.warmstart import WarmStartCache
    wc = WarmStartCache(D, rows_per_entry=1, max_entries=n, max_batch=B, latent_shape=None)
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    wc.ivf_configure(16, 4, 1 << 62, 0)
    ids = np.arange(1, n + 1, dtype=np.uint64)
    off = np.arange(n + 1, dtype=np.int64)
    wc.insert_batch(ids, off, rows, np.zeros(n, np.int32), np.zeros(n), dur)
    wc.ivf_rebuild()
    path = str(tmp_path / "d.swix")
    wc.save_swix(path)
    L = rng.uniform(2.5, 10.0, B)
    rid = np.arange(1, B + 1, dtype=np.uint64)
    T = np.full(B, 200, np.int32)
    n0 = wc.overflow_fallbacks()
    ch = _plan(wc, q, L, rid, T, th, ps)
    assert wc.overflow_fallbacks() > n0
    _no_flags(ch)
    ar = oracle.Arena(ids, off, rows, np.zeros(n, np.int32), np.zeros(n), dur)
    idx = ref.load_index_with_arena(path, ar)
    exp, _, _ = idx.plan_batch(neg, q, L, rid, T, top_k=8, policy="exploit", theta=th, psi=ps,
                               nthreads=NT)
    for f in FIELDS:
        np.testing.assert_array_equal(ch[f], exp[f], err_msg=f)
    wc.close()


def _full_batch_check(orc, rows, q, seed):
    n, D = rows.shape
    B = q.shape[0]
    rng = np.random.default_rng(seed)
    dur = rng.uniform(4.0, 12.0, n).astype(np.float32).astype(np.float64)
    neg = normalize_rows(rng.standard_normal((1, D)))[0]
    th, ps = trained_like_gater()
    wc, ar = _flat_cache(rows, dur, B)
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    L = rng.uniform(2.5, 10.0, B)
    rid = np.arange(1, B + 1, dtype=np.uint64)
    T = np.full(B, 200, np.int32)
    n0 = wc.overflow_fallbacks()
    ch = _plan(wc, q, L, rid, T, th, ps)
    assert wc.launch_info()["cta_pair"]
    nfb = wc.overflow_fallbacks() - n0
    _no_flags(ch)
    exp, _ = orc.plan_batch(ar, neg, q, L, rid, T, top_k=8, policy="exploit", theta=th, psi=ps,
                            nthreads=NT)
    for f in FIELDS:
        np.testing.assert_array_equal(ch[f], exp[f], err_msg=f)
    wc.close()
    return nfb


def test_config3_full_size_duplicates_full_batch(orc):
    n, D, B, a = 1_000_000, 512, 1024, 123_456
    rows = _dup_rows(n, D, a, 20_000, 5_000, seed=77)
    q = _queries(np.random.default_rng(78), rows, a, B)
    nfb = _full_batch_check(orc, rows, q, 79)
    assert nfb > 0
    print(f"fallback queries: {nfb} of {B}")


def test_config3_full_size_clustered_full_batch(orc):
    n, D, B = 1_000_000, 512, 1024
    rows = clustered_rows(n, D, seed=31)
    rng = np.random.default_rng(32)
    q = _perturb(rng, rows[rng.integers(0, n, B)], 0.3)
    nfb = _full_batch_check(orc, rows, q, 33)
    print(f"clustered 1M: fallback queries {nfb} of {B}")
