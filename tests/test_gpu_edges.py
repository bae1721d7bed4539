"""GPU: edge cases of the search path the reference defines (index.cpp:289-326) — an empty
index returns no hits, k larger than the cache returns every entry in order, k < 1 is
std::invalid_argument, ragged pyramids (entries with fewer rows than rows_per_entry), a cache
emptied by removals, empty batches and batch-size limits — in both the exact and the tcgen05
modes, against the C restatement."""
import numpy as np
import pytest

import oracle
from paper_2603_07865_b200.synth import SynthCache, perturbed_queries

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

MODES = [{"exact_only": True}, {"tc_always": True}]


def _wc(dim, R, cap, **kw):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    return WarmStartCache(dim, rows_per_entry=R, max_entries=cap, max_batch=64, **kw)


def _check(orc, ar, wc, q, k):
    hits, n = wc.search(q, k)
    for i in range(q.shape[0]):
        h = orc.search(ar, q[i], k)
        assert n[i] == len(h), (i, n[i], len(h))
        np.testing.assert_array_equal(hits[i, :n[i]]["entry_id"], h["entry_id"])
        np.testing.assert_array_equal(hits[i, :n[i]]["similarity"], h["similarity"])
        np.testing.assert_array_equal(hits[i, :n[i]]["level"], h["level"])


@pytest.mark.parametrize("mode", MODES)
def test_empty_index_returns_no_hits(mode):
    wc = _wc(128, 1, 256, **mode)
    q = np.random.default_rng(1).standard_normal((5, 128)).astype(np.float32)
    hits, n = wc.search(q, 8)
    assert (n == 0).all()


@pytest.mark.parametrize("mode", MODES)
def test_k_larger_than_cache_returns_all_in_order(orc, mode):
    c = SynthCache(11, 64, 1.0, seed=41)
    wc = _wc(64, 1, 64, **mode)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    ar = oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    q = perturbed_queries(c, 7, seed=2)
    _check(orc, ar, wc, q, 32)
    hits, n = wc.search(q, 32)
    assert (n == 11).all()


@pytest.mark.parametrize("mode", MODES)
def test_bad_k_and_batch_size_are_invalid_argument(mode):
    wc = _wc(64, 1, 64, **mode)
    q = np.zeros((2, 64), np.float32)
    with pytest.raises(ValueError):
        wc.search(q, 0)  # index.cpp:291
    with pytest.raises(ValueError):
        wc.search(q, 33)  # above the 32-deep running lists
    with pytest.raises(ValueError):
        wc.search(np.zeros((65, 64), np.float32), 8)  # above max_batch


@pytest.mark.parametrize("mode", MODES)
def test_empty_batch(mode):
    wc = _wc(64, 1, 64, **mode)
    hits, n = wc.search(np.zeros((0, 64), np.float32), 8)
    assert n.shape == (0,)


@pytest.mark.parametrize("mode", MODES)
def test_ragged_pyramids(orc, mode):
    """Entries with 1..7 rows in a rows_per_entry = 7 arena (pad rows repeat row 0)."""
    c = SynthCache(300, 96, 0.25, seed=43, clustered=True)
    rng = np.random.default_rng(7)
    keep = [rng.integers(1, 8) for _ in range(len(c.ids))]
    rows, lv, st, ln, off = [], [], [], [], [0]
    for e in range(len(c.ids)):
        a = c.off[e]
        rows.append(c.rows[a:a + keep[e]])
        lv.append(c.levels[a:a + keep[e]])
        st.append(c.starts[a:a + keep[e]])
        ln.append(c.lengths[a:a + keep[e]])
        off.append(off[-1] + keep[e])
    rows, lv, st, ln = (np.concatenate(x) for x in (rows, lv, st, ln))
    off = np.array(off, np.int64)
    wc = _wc(96, 7, 400, **mode)
    wc.insert_batch(c.ids, off, rows, lv, st, ln)
    ar = oracle.Arena(c.ids, off, rows, lv, st, ln)
    q = perturbed_queries(c, 48, frac_random=0.2, seed=5)
    for k in (1, 8):
        _check(orc, ar, wc, q, k)


@pytest.mark.parametrize("mode", MODES)
def test_cache_emptied_by_removals(orc, mode):
    c = SynthCache(40, 64, 1.0, seed=44)
    wc = _wc(64, 1, 64, **mode)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    for eid in c.ids[:-1]:
        wc.remove(int(eid))
    last = len(c.ids) - 1
    ar = oracle.Arena(c.ids[last:], c.off[last:] - c.off[last], c.rows[c.off[last]:],
                      c.levels[c.off[last]:], c.starts[c.off[last]:], c.lengths[c.off[last]:])
    q = perturbed_queries(c, 6, seed=3)
    _check(orc, ar, wc, q, 8)
    wc.remove(int(c.ids[last]))
    hits, n = wc.search(q, 8)
    assert (n == 0).all()


def test_boundary_draw_matches_reference(ref):
    """A softmax draw whose cumulative weight lands ON the target: two
    candidates whose weight ratio is constructed from the request's own draw u so that the
    first boundary equals u * total, then moved by a few ulps / 1e-12 / 1e-6 either way. The
    device's exp is glibc's restated bit for bit, so every pick equals the reference's select —
    replayed here in Python (IEEE doubles; math.exp is the same glibc exp the compiled reference
    calls) — and no draw is flagged SW_CHOICE_AMBIGUOUS_DRAW any more."""
    import math

    from paper_2603_07865_b200 import _lib
    from paper_2603_07865_b200.warmstart import SelectorConfig
    wc = _wc(64, 1, 64)
    sel = SelectorConfig(top_k=2, temperature=0.05, quality_threshold=0.0)
    dur = np.array([5.0, 5.0])
    neg = np.array([0.1, 0.1])

    def ref_pick(s, u):  # score_candidates + select (selector.cpp:24-85), both survive
        sp = [min(1.0, max(0.0, x)) for x in s]
        mx = max(sp)
        w = [math.exp((x - mx) / sel.temperature) for x in sp]
        total = 0.0
        for x in w:
            total += x
        target = u * total
        acc = 0.0
        for j, x in enumerate(w):
            acc += x
            if acc >= target:
                return j
        return len(w) - 1

    n_boundary = 0
    seeds = [s for s in range(1, 4000) if 0.3 < ref.lib.ref_rng_first_uniform(s) < 0.9][:40]
    for seed in seeds:
        u = ref.lib.ref_rng_first_uniform(seed)
        s0 = 0.9
        s1 = s0 + sel.temperature * math.log(1.0 / u - 1.0)  # w1 / w0 = (1 - u) / u
        for d in (0.0, 1e-16, -1e-16, 2e-16, -2e-16, 1e-12, -1e-12, 1e-6, -1e-6):
            sims = np.array([s0, s1 + d])
            _, pick, flags = wc.score_select(sims, neg, dur, 5.0, sel, seed)
            assert not flags & _lib.SW_CHOICE_AMBIGUOUS_DRAW
            assert pick == ref_pick(list(sims), u), (seed, d)
            w = [math.exp((x - max(sims)) / sel.temperature) for x in sims]
            n_boundary += abs(w[0] - u * (w[0] + w[1])) <= 1e-13 * (w[0] + w[1])
    assert n_boundary >= 40  # the constructed draws really sit on the boundary