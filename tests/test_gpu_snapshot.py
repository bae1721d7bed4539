"""GPU: SWIX snapshots straight into / out of the device arena against the
reference's own IvfIndex::save / load (index.cpp:345-408): a reference index (re-clustered
during its inserts) saved and loaded into our arena searches exactly like the reference loaded
from the same file; our GPU-built index saved and loaded by the reference is consistent
(check_consistent) and searches identically."""
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
