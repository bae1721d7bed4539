"""GPU parity at BASELINE config 3's full size: a 1M-entry x 512-d cache, one 1024-request
batch through the tcgen05 CTA-pair path (the bench's workload), checked request by request
against the UNMODIFIED reference (oracle/_ref: IvfIndex::search over the same 1M rows +
score_candidates + select + context_features + choose_arm + t*) on a sample of the batch,
and through the cross-batch pipelined entry point on the whole batch."""
import numpy as np
import pytest

import oracle
from paper_2603_07865_b200 import _lib
from paper_2603_07865_b200.synth import normalize_rows, trained_like_gater

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_config3_full_size_plan_matches_reference(ref):
    import ctypes as C

    from paper_2603_07865_b200.warmstart import (Policy, SelectorConfig, WarmStartCache,
                                                 requests)
    n, D, B, n_check = 1_000_000, 512, 1024, 48
    rng = np.random.default_rng(2026)
    rows = np.empty((n, D), np.float32)
    for i in range(0, n, 65536):
        m = min(65536, n - i)
        rows[i:i + m] = normalize_rows(rng.standard_normal((m, D), dtype=np.float32))
    dur = rng.uniform(4.0, 12.0, n).astype(np.float32).astype(np.float64)
    ids = np.arange(1, n + 1, dtype=np.uint64)
    off = np.arange(n + 1, dtype=np.int64)
    levels, starts = np.zeros(n, np.int32), np.zeros(n)
    neg = ref.negative(D)
    th, ps = trained_like_gater()

    wc = WarmStartCache(D, rows_per_entry=1, max_entries=n, max_batch=B, latent_shape=None)
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    wc.insert_batch(ids, off, rows, levels, starts, dur)

    src = rows[rng.integers(0, n, B)].astype(np.float64)
    g = rng.standard_normal((B, D))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    q = normalize_rows(src + 0.3 * g)
    L = rng.uniform(2.5, 10.0, B)
    rid = np.arange(1, B + 1, dtype=np.uint64)
    T = np.full(B, 200, np.int32)
    reqs = requests(rid, L, T)
    sel, pol = SelectorConfig(8), Policy("exploit")
    buf = wc.plan(q, reqs, seed=1, sel=sel, policy=pol)
    info = wc.launch_info()
    assert info["tensor_cores"] and info["cta_pair"]
    ch = wc.choices(buf)
    assert ch["hit"].any()
    assert ((ch["flags"] & (_lib.SW_CHOICE_AMBIGUOUS_DRAW | _lib.SW_CHOICE_INCOMPLETE)) == 0).all()

    # the pipelined entry point over the same batch gives the same choices
    dev = torch.device("cuda", 0)
    qd = torch.from_numpy(np.ascontiguousarray(q, np.float32)).to(dev)
    rd = torch.from_numpy(reqs.view(np.uint8)).to(dev)
    cha = torch.zeros(B * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    L_ = _lib.lib()
    wc2 = WarmStartCache(D, rows_per_entry=1, max_entries=n, max_batch=B,
                         latent_shape=(1, 4, 4), latent_slots=8)
    wc2.set_negative(neg)
    wc2.set_gater(th, ps, 1.0)
    wc2.insert_batch(ids, off, rows, levels, starts, dur)
    out = torch.zeros((B, 1, 4, 4), dtype=torch.float32, device=dev)
    _lib.check(L_.sw_warmstart_async(wc2._h, qd.data_ptr(), rd.data_ptr(), B, 1,
                                     C.byref(sel.c()), C.byref(pol.c()), None, 7,
                                     cha.data_ptr(), out.data_ptr(), 4, st), "sw_warmstart_async")
    _lib.check(L_.sw_join(wc2._h, st), "sw_join")
    torch.cuda.synchronize(dev)
    cha = cha.cpu().numpy().view(_lib.CHOICE_DTYPE)
    for f in ("hit", "arm", "steps_skipped", "n_hits", "entry_id", "similarity", "pick"):
        np.testing.assert_array_equal(cha[f], ch[f], err_msg=f)
    wc2.close()

    # the unmodified reference on a sample of the batch
    ar = oracle.Arena(ids, off, rows, levels, starts, dur)
    idx = ref.index(ar)
    s = np.sort(np.random.default_rng(5).choice(B, n_check, replace=False))
    exp, _, _ = idx.plan_batch(neg, q[s], L[s], rid[s], T[s], top_k=8, policy="exploit",
                               theta=th, psi=ps, nthreads=16)
    for f in ("hit", "arm", "steps_skipped", "n_hits", "entry_id", "level", "pick", "start_s",
              "length_s", "similarity"):
        np.testing.assert_array_equal(ch[f][s], exp[f], err_msg=f)


def test_config3_full_size_ivf_plan_matches_reference(ref, tmp_path):
    """The reference's default IVF index (64 lists, nprobe 8) at 1M x 512: our GPU k-means
    lists, written as a SWIX snapshot and loaded by the reference's own IvfIndex::load; the
    list-grouped tcgen05 search + plan then matches the reference plan flow request by request."""
    from paper_2603_07865_b200.warmstart import (Policy, SelectorConfig, WarmStartCache,
                                                 requests)
    n, D, B, n_check = 1_000_000, 512, 1024, 32
    rng = np.random.default_rng(2027)
    rows = np.empty((n, D), np.float32)
    for i in range(0, n, 65536):
        m = min(65536, n - i)
        rows[i:i + m] = normalize_rows(rng.standard_normal((m, D), dtype=np.float32))
    dur = rng.uniform(4.0, 12.0, n).astype(np.float32).astype(np.float64)
    ids = np.arange(1, n + 1, dtype=np.uint64)
    off = np.arange(n + 1, dtype=np.int64)
    levels, starts = np.zeros(n, np.int32), np.zeros(n)
    neg = ref.negative(D)
    th, ps = trained_like_gater()
    wc = WarmStartCache(D, rows_per_entry=1, max_entries=n, max_batch=B, latent_shape=None)
    wc.set_negative(neg)
    wc.set_gater(th, ps, 1.0)
    wc.ivf_configure(64, 8, 1 << 62, 0)
    wc.insert_batch(ids, off, rows, levels, starts, dur)
    wc.ivf_rebuild()
    path = str(tmp_path / "cache.swix")
    wc.save_swix(path)

    src = rows[rng.integers(0, n, B)].astype(np.float64)
    g = rng.standard_normal((B, D))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    q = normalize_rows(src + 0.3 * g)
    L = rng.uniform(2.5, 10.0, B)
    rid = np.arange(1, B + 1, dtype=np.uint64)
    T = np.full(B, 200, np.int32)
    ch = wc.choices(wc.plan(q, requests(rid, L, T), seed=1, sel=SelectorConfig(8),
                            policy=Policy("exploit")))
    assert ch["hit"].any()

    ar = oracle.Arena(ids, off, rows, levels, starts, dur)
    idx = ref.load_index_with_arena(path, ar)
    s = np.sort(np.random.default_rng(6).choice(B, n_check, replace=False))
    exp, _, _ = idx.plan_batch(neg, q[s], L[s], rid[s], T[s], top_k=8, policy="exploit",
                               theta=th, psi=ps, nthreads=16)
    for f in ("hit", "arm", "steps_skipped", "n_hits", "entry_id", "level", "pick", "start_s",
              "length_s", "similarity"):
        np.testing.assert_array_equal(ch[f][s], exp[f], err_msg=f)
