"""GPU: the IVF coarse quantiser (csrc/ivf.cu) vs the reference IvfIndex in its default mode
(index.cpp:59-326): the same entries inserted one by one into both — with rebuilds triggered by
the mutation counter at the same points — must give bit-identical centroids (k-means++ and Lloyd
in the reference's fp64 order), identical list membership for every row, and identical search
results (ids, segments, fp64 similarities) through the tcgen05 path and the exact path."""
import numpy as np
import pytest

import oracle
from paper_2603_07865_b200.synth import SynthCache, perturbed_queries

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _ivf_pair(ref, c: SynthCache, C, nprobe, interval, seed, **kw):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    wc = WarmStartCache(c.dim, rows_per_entry=c.R, max_entries=len(c.ids) + 8, max_batch=256,
                        latent_shape=None, **kw)
    wc.ivf_configure(C, nprobe, interval, seed)
    ar = oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    ri = ref.index(oracle.Arena(c.ids[:0], c.off[:1], c.rows[:0], c.levels[:0], c.starts[:0],
                                c.lengths[:0]), ivf=(C, seed, nprobe, interval))
    ri.insert(ar)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    return wc, ri, ar


def _check_index(wc, ri, c):
    cent, _np, lists = ri.snapshot()
    got = wc.ivf_centroids()
    assert got.shape == cent.shape
    np.testing.assert_array_equal(got, cent)  # bit-identical k-means
    where = {}
    for j, recs in enumerate(lists):
        for (eid, lvl, st, ln) in recs:
            where[(eid, lvl, np.float32(st))] = j
    for e in range(0, len(c.ids), 7):
        eid = int(c.ids[e])
        ls = wc.ivf_entry_lists(eid)
        for r in range(c.off[e + 1] - c.off[e]):
            key = (eid, int(c.levels[c.off[e] + r]), np.float32(c.starts[c.off[e] + r]))
            assert ls[r] == where[key], (eid, r)


def _check_search(wc, ri, q, k):
    hits, cnt = wc.search(q, k)
    for i in range(q.shape[0]):
        ids, lv, st, ln, sm = ri.search(q[i], k)
        assert cnt[i] == len(ids), i
        np.testing.assert_array_equal(hits[i, :cnt[i]]["entry_id"], ids, err_msg=f"q{i}")
        np.testing.assert_array_equal(hits[i, :cnt[i]]["level"], lv)
        np.testing.assert_array_equal(hits[i, :cnt[i]]["start_s"], st)
        np.testing.assert_array_equal(hits[i, :cnt[i]]["similarity"], sm)


@pytest.mark.parametrize("mode", ["tc_always", "exact_only"])
def test_ivf_rebuilds_and_search_match_reference(ref, mode):
    # 300 entries x 7 rows, rebuild every 256 mutations -> 8 rebuilds during the inserts
    c = SynthCache(300, 64, 0.25, seed=31, clustered=True)
    wc, ri, _ = _ivf_pair(ref, c, 16, 4, 256, 5, **{mode: True})
    info = wc.ivf_info()
    assert info["centroids"] == 16 and info["rebuilds"] == 2100 // 256
    _check_index(wc, ri, c)
    q = perturbed_queries(c, 96, frac_random=0.2)
    for k in (1, 8):
        _check_search(wc, ri, q, k)
    assert wc.launch_info()["tensor_cores"] == (mode == "tc_always")


def test_ivf_default_config_with_removals(ref):
    # reference defaults: 64 centroids, nprobe 8, rebuild every 1024 mutations
    c = SynthCache(400, 96, 0.25, seed=32, clustered=True)
    wc, ri, _ = _ivf_pair(ref, c, 64, 8, 1024, 0, tc_always=True)
    rng = np.random.default_rng(3)
    for eid in rng.choice(c.ids, 120, replace=False):
        wc.remove(int(eid))
        ri.remove(int(eid))
    assert wc.ivf_info()["rebuilds"] == 3  # 2800 inserted rows + 840 removed rows
    _check_index_alive(wc, ri)
    q = perturbed_queries(c, 128, frac_random=0.1)
    _check_search(wc, ri, q, 8)


def _check_index_alive(wc, ri):
    cent, _np, lists = ri.snapshot()
    np.testing.assert_array_equal(wc.ivf_centroids(), cent)
    seen = {}
    for j, recs in enumerate(lists):
        for (eid, lvl, st, ln) in recs:
            seen.setdefault(eid, []).append(j)
    for eid, js in list(seen.items())[::9]:
        assert sorted(wc.ivf_entry_lists(eid).tolist()) == sorted(js)


def test_ivf_large_tensor_core_path(ref):
    # 8K single-row entries at D = 128: one rebuild when the last insert reaches the interval;
    # the tcgen05 kernel (CTA pairs at B = 256) must keep only probed-list rows
    c = SynthCache(8192, 128, 1.0, seed=33, clustered=True)
    wc, ri, _ = _ivf_pair(ref, c, 32, 4, 8192, 11)
    assert wc.ivf_info()["rebuilds"] == 1
    np.testing.assert_array_equal(wc.ivf_centroids(), ri.snapshot()[0])
    q = perturbed_queries(c, 256, frac_random=0.1)
    hits, cnt = wc.search(q, 8)
    assert wc.launch_info()["tensor_cores"]
    for i in range(0, 256, 8):
        ids, lv, st, ln, sm = ri.search(q[i], 8)
        assert cnt[i] == len(ids)
        np.testing.assert_array_equal(hits[i, :cnt[i]]["entry_id"], ids)
        np.testing.assert_array_equal(hits[i, :cnt[i]]["similarity"], sm)


def test_ivf_bulk_rebuild_and_set_centroids(ref):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    c = SynthCache(500, 64, 0.25, seed=34)
    # bulk path: insert with no automatic rebuild, then an explicit rebuild == the reference's
    # first automatic rebuild at the same row set
    wc = WarmStartCache(64, rows_per_entry=7, max_entries=600, max_batch=64, latent_shape=None)
    wc.ivf_configure(8, 2, 1 << 60, 9)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    wc.ivf_rebuild()
    ar = oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    ri = ref.index(ar, ivf=(8, 9, 2, 3500))  # 500 x 7 = 3500 rows -> one rebuild at the end
    np.testing.assert_array_equal(wc.ivf_centroids(), ri.snapshot()[0])
    q = perturbed_queries(c, 64, frac_random=0.2)
    _check_search(wc, ri, q, 8)
    # installing the same centroids (SWIX load path) reproduces the same lists and results
    wc2 = WarmStartCache(64, rows_per_entry=7, max_entries=600, max_batch=64, latent_shape=None)
    wc2.ivf_configure(8, 2, 1 << 60, 9)
    wc2.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    wc2.ivf_set_centroids(ri.snapshot()[0])
    _check_search(wc2, ri, q, 8)
