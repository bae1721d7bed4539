"""GPU: SWIX snapshots straight into / out of the device arena against the
reference's own IvfIndex::save / load (index.cpp:345-408): a reference index (re-clustered
during its inserts) saved and loaded into our arena searches exactly like the reference loaded
from the same file; our GPU-built index saved and loaded by the reference is consistent
(check_consistent) and searches identically."""
import ctypes as C
import os
import tempfile

import numpy as np
import pytest

import oracle
from paper_2603_07865_b200.synth import SynthCache, perturbed_queries

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _same_search(wc, ri, q, k, f32_segments=False):
    """f32_segments: the SWIX format stores start/length as f32 (index.cpp:362-363)."""
    cast = (lambda a: np.asarray(a).astype(np.float32)) if f32_segments else (lambda a: a)
    hits, cnt = wc.search(q, k)
    for i in range(q.shape[0]):
        ids, lv, st, ln, sm = ri.search(q[i], k)
        assert cnt[i] == len(ids), i
        np.testing.assert_array_equal(hits[i, :cnt[i]]["entry_id"], ids)
        np.testing.assert_array_equal(hits[i, :cnt[i]]["level"], lv)
        np.testing.assert_array_equal(cast(hits[i, :cnt[i]]["start_s"]), cast(st))
        np.testing.assert_array_equal(cast(hits[i, :cnt[i]]["length_s"]), cast(ln))
        np.testing.assert_array_equal(hits[i, :cnt[i]]["similarity"], sm)


def test_reference_snapshot_into_arena(ref):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    c = SynthCache(400, 64, 0.25, seed=51, clustered=True)
    ar = oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    ri = ref.index(ar, ivf=(16, 7, 4, 700))  # 2800 rows -> 4 rebuilds while inserting
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "idx.swix")
        assert ref.lib.ref_index_save(ri.h, path.encode()) == 16
        loaded = ref.load_index(path, 64)
        wc = WarmStartCache(64, rows_per_entry=7, max_entries=450, max_batch=128,
                            latent_shape=None, tc_always=True)
        wc.load_swix(path)
        info = wc.ivf_info()
        assert info["centroids"] == 16 and info["rebuilds"] == 0
        np.testing.assert_array_equal(wc.ivf_centroids(), oracle.parse_swix(path)[0])
        q = perturbed_queries(c, 96, frac_random=0.2)
        _same_search(wc, loaded, q, 8)
        # and the loaded arena saves back to the same bytes (rebuild-ordered lists)
        back = os.path.join(d, "back.swix")
        wc.save_swix(back)
        a, b = oracle.parse_swix(path), oracle.parse_swix(back)
        np.testing.assert_array_equal(a[0], b[0])
        assert a[1] == b[1] and [len(x) for x in a[2]] == [len(x) for x in b[2]]
        assert all(sorted(x) == sorted(y) for x, y in zip(a[2], b[2]))


def test_arena_snapshot_into_reference(ref):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    c = SynthCache(3000, 128, 1.0, seed=52, clustered=True)
    wc = WarmStartCache(128, rows_per_entry=1, max_entries=3000, max_batch=256,
                        latent_shape=None)
    wc.ivf_configure(24, 6, 1 << 60, 3)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    wc.ivf_rebuild()  # GPU k-means
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "ours.swix")
        wc.save_swix(path)
        loaded = ref.load_index(path, 128)
        assert loaded.consistent()  # every row in its nearest centroid's list (fp64 check)
        q = perturbed_queries(c, 256, frac_random=0.1)
        _same_search(wc, loaded, q[::4], 8, f32_segments=True)


def test_swix_errors(tmp_path):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    wc = WarmStartCache(32, rows_per_entry=1, max_entries=8, max_batch=8, latent_shape=None)
    bad = tmp_path / "bad.swix"
    bad.write_bytes(b"NOPE" + b"\0" * 12)
    with pytest.raises(Exception, match="bad magic"):
        wc.load_swix(str(bad))
    trunc = tmp_path / "trunc.swix"
    trunc.write_bytes(b"SWIX" + np.array([2, 1, 32], np.uint32).tobytes() + b"\0" * 40)
    with pytest.raises(Exception, match="truncated"):
        wc.load_swix(str(trunc))


# ---------------------------------------------------------------- cache directory (cache.cpp)
def _ref_state(ref, rh, eid):
    st = np.zeros(7)
    sk = np.zeros(64)
    n = ref.lib.ref_cache_entry_state(rh, eid, st, sk, 64)
    return st, sk[:n]


def _ref_search_equal(ref, rh, wc, q, dim, k=8):
    hits, cnt = wc.search(q, k)
    for i in range(q.shape[0]):
        rid = np.zeros(k, np.uint64)
        lv = np.zeros(k, np.int32)
        st = np.zeros(k)
        ln = np.zeros(k)
        sm = np.zeros(k)
        n = ref.lib.ref_cache_search(rh, q[i], dim, k, rid, lv, st, ln, sm)
        assert cnt[i] == n
        np.testing.assert_array_equal(hits[i, :n]["entry_id"], rid[:n])
        np.testing.assert_array_equal(hits[i, :n]["level"], lv[:n])
        np.testing.assert_array_equal(hits[i, :n]["start_s"], st[:n])
        np.testing.assert_array_equal(hits[i, :n]["similarity"], sm[:n])


@pytest.mark.parametrize("ivf", [None, (8, 2, 64, 11)])
def test_cache_directory_interchange(ref, tmp_path, ivf):
    """CacheManager::save_snapshot of the reference -> swcm_load_snapshot straight into the
    device arena: the same ledger (importances bit-exact, reuse history), rows, index and
    searches as the reference loading its own snapshot; then swcm_save_snapshot -> the
    reference's load_snapshot: consistent, the same ledger, SimClip payloads and searches."""
    from paper_2603_07865_b200.warmstart import CacheManager, WarmStartCache
    dim, cap, delta, n = 64, 80, 0.25, 60
    emb_seed = ref.derive_seed(3, 0x5345474D)

    def new_ref():
        if ivf is None:
            return ref.lib.ref_cache_new(cap, 0.9, 1.0, 0.3, delta, emb_seed)
        return ref.lib.ref_cache_new_ivf(cap, 0.9, 1.0, 0.3, delta, emb_seed, ivf[0], ivf[1],
                                         ivf[3], ivf[2])

    rng = np.random.default_rng(5)
    centres = ref.random_unit_vectors(77, 5, dim)
    ra = new_ref()
    now = 0.0
    for i in range(n):
        now += 0.1
        emb = ref.perturb(centres[i % 5], float(rng.uniform(0.1, 0.6)), 100 + i)
        prm = ref.perturb(emb, 0.2, 900 + i)
        dur = float(rng.uniform(4.0, 12.0))
        lat = rng.standard_normal(int(dur * 200)).astype(np.float32)
        assert ref.lib.ref_cache_admit_clip(ra, emb, prm, dim, dur, 0.9, now, lat, len(lat), 200,
                                            1000 + i, 0.05 * (i % 4)) == i + 1
    for j in range(150):
        eid = int(rng.integers(1, n + 1))
        ref.lib.ref_cache_record_reuse(ra, eid, int(rng.integers(0, 120)),
                                       float(rng.uniform(2.5, 10)), now + 0.01 * j,
                                       float(rng.choice([0.0, 0.05, 0.3])))
    da, db = str(tmp_path / "ref_snap"), str(tmp_path / "our_snap")
    assert ref.lib.ref_cache_save_snapshot(ra, da.encode()) == 0
    rb = new_ref()  # the reference's own load path is the expected state
    assert ref.lib.ref_cache_load_snapshot(rb, da.encode()) == 0

    wc = WarmStartCache(dim, rows_per_entry=7, max_entries=cap + 8, max_batch=32,
                        latent_shape=(1, 2600, 1))
    if ivf:
        wc.ivf_configure(ivf[0], ivf[1], ivf[2], ivf[3])
    cm = CacheManager(wc, capacity=cap, pyramid_delta=delta, embedding_seed=emb_seed)
    cm.admit(centres[0], 5.0, centres[0], 0.9, 0.0)  # replaced by the load
    cm.load_snapshot(da)
    ids = sorted(cm.ids())
    assert ids == list(range(1, n + 1))
    assert cm.check_consistent()
    if ivf:
        assert wc.ivf_config()["rebuild_interval"] == 1024  # a fresh IvfIndex, as after the load
    t = now + 5.0
    for eid in ids:
        assert cm.current_importance(eid, t) == ref.lib.ref_cache_importance(rb, eid, t)
        rows = np.zeros((32, dim), np.float32)
        nr = ref.lib.ref_cache_entry_rows(rb, eid, rows, 32)
        np.testing.assert_array_equal(wc.read_rows(eid), rows[:nr])
    cand = np.zeros(256, np.uint64)
    nc = ref.lib.ref_cache_refinement_candidates(rb, cand, 256)
    assert cm.refinement_candidates() == cand[:nc].tolist()
    q = np.stack([ref.perturb(centres[i % 5], 0.4, 5000 + i) for i in range(24)])
    _ref_search_equal(ref, rb, wc, q, dim)
    # admits continue from max id + 1
    assert cm.admit(centres[1], 6.0, centres[1], 0.9, t) == n + 1
    assert ref.lib.ref_cache_admit(rb, centres[1], dim, 6.0, 0.9, t) == n + 1

    # ours -> the reference
    cm.save_snapshot(db)
    rc = new_ref()
    assert ref.lib.ref_cache_load_snapshot(rc, db.encode()) == 0
    assert ref.lib.ref_cache_check_consistent(rc) == 1
    buf = np.zeros(256, np.uint64)
    assert sorted(buf[:ref.lib.ref_cache_ids(rc, buf, 256)].tolist()) == list(range(1, n + 2))
    for eid in range(1, n + 2):
        sb, kb = _ref_state(ref, rb, eid)
        sc, kc = _ref_state(ref, rc, eid)
        np.testing.assert_array_equal(sc, sb)
        np.testing.assert_array_equal(kc, kb)
        if eid <= n:  # the SimClip payload survives the round trip through the device cache
            la, lb = np.zeros(2600, np.float32), np.zeros(2600, np.float32)
            ea, eb = np.zeros(dim, np.float32), np.zeros(dim, np.float32)
            r1, r2 = C.c_int(), C.c_int()
            s1, s2 = C.c_uint64(), C.c_uint64()
            k1, k2 = C.c_double(), C.c_double()
            na = ref.lib.ref_cache_clip(rb, eid, la, 2600, C.byref(r1), C.byref(s1), C.byref(k1), ea)
            nb = ref.lib.ref_cache_clip(rc, eid, lb, 2600, C.byref(r2), C.byref(s2), C.byref(k2), eb)
            assert na == nb and r1.value == r2.value and s1.value == s2.value
            assert k1.value == k2.value
            np.testing.assert_array_equal(la[:na], lb[:nb])
            np.testing.assert_array_equal(ea, eb)
    _ref_search_equal(ref, rc, wc, q, dim)
    for h in (ra, rb, rc):
        ref.lib.ref_cache_free(h)


def test_swmb_interchange(ref, tmp_path):
    """BanditModel::save -> sw_gater_load_swmb -> the device gater chooses like set_gater with
    the same parameters; sw_gater_save_swmb writes the reference's bytes back."""
    from paper_2603_07865_b200.warmstart import WarmStartCache
    rng = np.random.default_rng(9)
    th = rng.standard_normal((14, 11)).astype(np.float32)
    ps = rng.standard_normal((14, 11)).astype(np.float32)
    pa, pb = str(tmp_path / "a.swmb"), str(tmp_path / "b.swmb")
    assert ref.lib.ref_bandit_save(pa.encode(), th, ps, 11) == 0
    wc = WarmStartCache(64, rows_per_entry=1, max_entries=64, max_batch=16, latent_shape=None)
    wc.load_swmb(pa, beta=0.7)
    wc.save_swmb(pb)
    assert open(pa, "rb").read() == open(pb, "rb").read()
    t2, p2 = np.zeros(14 * 11, np.float32), np.zeros(14 * 11, np.float32)
    assert ref.lib.ref_bandit_load(pb.encode(), t2, p2, 14 * 11) == 11
    np.testing.assert_array_equal(t2.reshape(14, 11), th)
    np.testing.assert_array_equal(p2.reshape(14, 11), ps)
    prompts = rng.standard_normal((32, 64)).astype(np.float32)
    segs = rng.standard_normal((32, 64)).astype(np.float32)
    a = wc.gater(prompts, segs, 200)
    wc2 = WarmStartCache(64, rows_per_entry=1, max_entries=64, max_batch=16, latent_shape=None)
    wc2.set_gater(th, ps, 0.7)
    b = wc2.gater(prompts, segs, 200)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    bad = str(tmp_path / "bad.swmb")
    open(bad, "wb").write(b"SWXX" + bytes(16))
    with pytest.raises(Exception):
        wc.load_swmb(bad)
