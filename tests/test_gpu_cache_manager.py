"""GPU: the Cache Manager host policy (csrc/host/cache_manager.cpp) over the device arena vs the
reference's own CacheManager (cache.cpp, compiled in oracle/_ref) driven by the same randomized
admit / record_reuse / evict / refine sequence (config 5's churn at desk scale): identical alive
sets, admitted ids, importance values (bit-exact, lazy gamma^dt decay), refinement candidates and
refine decisions, bit-identical re-derived pyramid rows in the arena, and identical search results
over the churned cache."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _ref_ids(ref, h):
    buf = np.zeros(4096, np.uint64)
    n = ref.lib.ref_cache_ids(h, buf, 4096)
    return sorted(buf[:n].tolist())


def _ref_cands(ref, h):
    buf = np.zeros(4096, np.uint64)
    n = ref.lib.ref_cache_refinement_candidates(h, buf, 4096)
    return buf[:n].tolist()


@pytest.mark.parametrize("seed,ivf", [(1, None), (2, None), (3, (8, 2, 120, 17))])
def test_cache_manager_matches_reference(ref, seed, ivf):
    """ivf = (centroids, nprobe, rebuild interval, index seed): the reference's default IVF
    index under the same churn (rebuilds triggered by admits, evictions and refines)."""
    from paper_2603_07865_b200.warmstart import CacheManager, WarmStartCache
    dim, cap, delta = 64, 48, 0.25
    emb_seed = ref.derive_seed(seed, 0x5345474D)
    wc = WarmStartCache(dim, rows_per_entry=7, max_entries=cap + 8, max_batch=32,
                        latent_shape=None, tc_always=True)
    if ivf:
        wc.ivf_configure(ivf[0], ivf[1], ivf[2], ivf[3])
    cm = CacheManager(wc, capacity=cap, pyramid_delta=delta, embedding_seed=emb_seed)
    rh = (ref.lib.ref_cache_new(cap, 0.9, 1.0, 0.3, delta, emb_seed) if not ivf else
          ref.lib.ref_cache_new_ivf(cap, 0.9, 1.0, 0.3, delta, emb_seed, ivf[0], ivf[1],
                                        ivf[3], ivf[2]))
    rng = np.random.default_rng(seed)
    centres = ref.random_unit_vectors(seed + 100, 6, dim)
    now = 0.0
    n_admit = n_reuse = n_refine = n_refined = 0
    try:
        for op in range(500):
            now += float(rng.uniform(0.0, 0.25))
            ids = _ref_ids(ref, rh)
            r = rng.random()
            if r < 0.45 or not ids:
                emb = ref.perturb(centres[op % 6], float(rng.uniform(0.1, 0.6)), 7000 + op)
                dur = float(rng.uniform(4.0, 12.0))
                q = float(rng.uniform(0.1, 1.0))
                a = cm.admit(emb, dur, emb, q, now)
                b = ref.lib.ref_cache_admit(rh, emb, dim, dur, q, now)
                assert (a if a is not None else -1) == b
                n_admit += a is not None
            elif r < 0.85:
                eid = int(ids[int(rng.integers(0, len(ids)))])
                steps = int(rng.integers(0, 131))
                dur = float(rng.uniform(2.5, 10.0))
                skip = float(rng.choice([0.0, 0.0, 0.05, 0.3]))
                cm.record_reuse(eid, steps, dur, now, skip)
                ref.lib.ref_cache_record_reuse(rh, eid, steps, dur, now, skip)
                n_reuse += 1
            elif r < 0.95:
                cands = _ref_cands(ref, rh)
                assert cm.refinement_candidates() == cands
                eid = int(cands[0]) if cands else int(ids[int(rng.integers(0, len(ids)))])
                qs = rng.uniform(0.0, 1.0, 3)
                embs = ref.random_unit_vectors(9000 + op, 3, dim)
                rs = int(rng.integers(0, 2**63))
                seen = []

                def regen(prompt, duration, s, _q=qs, _e=embs):
                    seen.append(s)
                    return _e[len(seen) - 1], float(_q[len(seen) - 1])

                got = cm.refine(eid, rs, regen)
                seeds = np.zeros(3, np.uint64)
                exp = ref.lib.ref_cache_refine(rh, eid, rs, qs, embs, dim, 3, seeds)
                assert bool(got) == bool(exp)
                if seen:
                    assert seen == seeds.tolist()
                n_refine += 1
                n_refined += int(bool(got))
            else:
                out = np.zeros(64, np.uint64)
                nr = ref.lib.ref_cache_evict(rh, now, out, 64)
                assert cm.evict_if_full(now) == out[:nr].tolist()
            # ledger state after every operation
            ids = _ref_ids(ref, rh)
            assert sorted(cm.ids()) == ids
            for eid in ids:
                assert cm.current_importance(eid, now) == ref.lib.ref_cache_importance(rh, eid, now)
            assert cm.check_consistent()
            if op % 50 == 49:  # the arena holds the reference's rows and searches like its index
                q = np.stack([ref.perturb(centres[i % 6], 0.4, 50000 + op * 16 + i)
                              for i in range(16)])
                hits, cnt = wc.search(q, 8)
                for i in range(16):
                    rid = np.zeros(8, np.uint64)
                    lv = np.zeros(8, np.int32)
                    st = np.zeros(8)
                    ln = np.zeros(8)
                    sm = np.zeros(8)
                    n = ref.lib.ref_cache_search(rh, q[i], dim, 8, rid, lv, st, ln, sm)
                    assert cnt[i] == n
                    np.testing.assert_array_equal(hits[i, :n]["entry_id"], rid[:n])
                    np.testing.assert_array_equal(hits[i, :n]["similarity"], sm[:n])
                    np.testing.assert_array_equal(hits[i, :n]["start_s"], st[:n])
                for eid in ids[:5]:
                    rows = np.zeros((32, dim), np.float32)
                    nr = ref.lib.ref_cache_entry_rows(rh, eid, rows, 32)
                    np.testing.assert_array_equal(wc.read_rows(eid), rows[:nr])
    finally:
        ref.lib.ref_cache_free(rh)
    assert n_admit > 100 and n_reuse > 100 and n_refine > 10 and n_refined > 0
    if ivf:
        assert wc.ivf_info()["rebuilds"] > 5  # re-clustered many times during the churn
