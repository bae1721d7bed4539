"""GPU parity: libsemwarm_b200.so (through the C-ABI) vs the C restatement and the reference
goldens. Integer/index outputs and fp64 similarities must be bit-exact; Philox-mode latents
within |d| <= 1e-5 * max(|ref|, 1)."""
import numpy as np
import pytest

import oracle
from paper_2603_07865_b200 import _lib
from paper_2603_07865_b200.synth import (SynthCache, perturbed_queries, request_durations,
                                         trained_like_gater)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _cache(c: SynthCache, **kw):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    wc = WarmStartCache(c.dim, rows_per_entry=c.R, max_entries=kw.pop("max_entries", len(c.ids)),
                        **kw)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    return wc


def _arena(c):
    return oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)


def _check_hits(hits, n, ar, orc, q, k):
    for i in range(q.shape[0]):
        h = orc.search(ar, q[i], k)
        assert n[i] == len(h), i
        got = hits[i, :n[i]]
        np.testing.assert_array_equal(got["entry_id"], h["entry_id"], err_msg=f"q{i}")
        np.testing.assert_array_equal(got["level"], h["level"])
        np.testing.assert_array_equal(got["start_s"], h["start_s"])
        np.testing.assert_array_equal(got["similarity"], h["similarity"])


@pytest.mark.parametrize("mode", ["exact_only", "tc_always"])
@pytest.mark.parametrize("dim,delta,clustered,n", [(64, 0.25, True, 300), (512, 0.25, False, 1000),
                                                   (512, 1.0, True, 3000), (96, 0.5, False, 500)])
def test_search_matches_oracle(orc, mode, dim, delta, clustered, n):
    c = SynthCache(n, dim, delta, seed=3, clustered=clustered)
    wc = _cache(c, max_batch=256, exact_only=(mode == "exact_only"), tc_always=(mode == "tc_always"))
    q = perturbed_queries(c, 200, frac_random=0.2)
    for k in (1, 8, 32):
        hits, cnt = wc.search(q, k)
        assert wc.launch_info()["tensor_cores"] == (mode == "tc_always")
        _check_hits(hits, cnt, _arena(c), orc, q, k)


@pytest.mark.parametrize("scale", [0.25, 3.7])
def test_search_nonunit_and_near_ties_tc(orc, scale):
    """Certified over-fetch with non-unit rows/queries (the error bound scales with the norms)
    and near-tied entries (tiny perturbations of one vector)."""
    rng = np.random.default_rng(5)
    c = SynthCache(2000, 128, 1.0, seed=12, clustered=True)
    base = c.rows[0].astype(np.float64)
    for e in range(1, 200):  # 200 near-duplicates of row 0 at distance ~1e-4
        v = base + 1e-4 * rng.standard_normal(128)
        c.rows[e] = (v / np.linalg.norm(v)).astype(np.float32)
    c.rows *= np.float32(scale)
    wc = _cache(c, max_batch=64, tc_always=True)
    q = perturbed_queries(c, 64, scale=0.01) * np.float32(1.0 / scale)
    q[:8] = c.rows[:8] / np.float32(scale)
    hits, cnt = wc.search(q, 8)
    assert wc.launch_info()["tensor_cores"]
    _check_hits(hits, cnt, _arena(c), orc, q, 8)


@pytest.mark.parametrize("B", [1, 96])
@pytest.mark.parametrize("n_dup", [20, 120])
def test_search_exact_ties_tc(orc, B, n_dup):
    """Exact ties: n_dup entries share one row bit for bit, so their similarities are equal and
    the order is by id alone (index.cpp:320-324); 20 duplicates stay inside one warp's rank
    selection, 120 take the multi-round path; B = 1 runs the 256-thread query CTAs."""
    c = SynthCache(3000, 128, 1.0, seed=21, clustered=False)
    c.rows[1:n_dup] = c.rows[0]
    wc = _cache(c, max_batch=128, tc_always=True)
    q = perturbed_queries(c, B, scale=0.05, seed=4)
    q[0] = c.rows[0]
    for k in (1, 8, 32):
        hits, cnt = wc.search(q, k)
        _check_hits(hits, cnt, _arena(c), orc, q, k)


def test_search_tc_default_large(orc):
    # 40K entries x 1 row: default mode picks the tcgen05 pre-filter
    c = SynthCache(40000, 512, 1.0, seed=8, clustered=True)
    wc = _cache(c, max_batch=1024)
    q = perturbed_queries(c, 1024, frac_random=0.1)
    hits, cnt = wc.search(q, 8)
    info = wc.launch_info()
    assert info["tensor_cores"] and info["cta_pair"]  # 8 query blocks -> cta_group::2 pairs
    sel = np.arange(0, 1024, 16)
    _check_hits(hits[sel], cnt[sel], _arena(c), orc, q[sel], 8)


@pytest.mark.parametrize("B", [1, 33, 130])
def test_search_tc_partial_warps(orc, B):
    """Batches that leave a warp partially valid (B % 32 != 0) with several tiles per scoring
    CTA: every warp-collective tcgen05.ld must stay converged (regression: a per-lane gate on
    the first-tile pre-pass hung the epilogue)."""
    c = SynthCache(120000, 512, 1.0, seed=21, clustered=False)
    wc = _cache(c, max_batch=256)
    q = perturbed_queries(c, B, frac_random=0.1)
    hits, cnt = wc.search(q, 8)
    assert wc.launch_info()["tensor_cores"]
    sel = np.arange(0, B, max(1, B // 8))
    _check_hits(hits[sel], cnt[sel], _arena(c), orc, q[sel], 8)


def test_search_host_entry_point(orc):
    c = SynthCache(200, 64, 0.25, seed=1)
    wc = _cache(c)
    q = perturbed_queries(c, 16)
    hits, cnt = wc.search_host(q, 8)
    _check_hits(hits, cnt, _arena(c), orc, q, 8)


# ------------------------------------------------------------------ full plan vs reference goldens
@pytest.mark.parametrize("tc", [False, True])
@pytest.mark.parametrize("policy", ["exploit", "explore", "rule", "fixed"])
def test_plan_golden(golden, policy, tc):
    from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, WarmStartCache, requests
    g = golden["warm_cache"]
    dim = g["rows"].shape[1]
    wc = WarmStartCache(dim, rows_per_entry=7, max_entries=len(g["ids"]), max_batch=128,
                        tc_always=tc, exact_only=not tc)
    wc.set_negative(g["neg"])
    wc.set_gater(g["theta"], g["psi"], 1.0)
    wc.insert_batch(g["ids"], g["off"], g["rows"], g["levels"], g["starts"], g["lengths"])
    reqs = requests(g["req_ids"], g["L"], g["T"])
    buf = wc.plan(g["queries"], reqs, seed=int(g["seed"]), sel=SelectorConfig(8),
                  policy=Policy(policy, fixed_arm=7))
    ch = wc.choices(buf)
    exp = g[f"plan_{policy}"]
    amb = (ch["flags"] & (_lib.SW_CHOICE_AMBIGUOUS_DRAW | _lib.SW_CHOICE_AMBIGUOUS_ARM)) != 0
    assert amb.sum() == 0
    for f in ["hit", "arm", "steps_skipped", "n_hits", "entry_id", "level", "pick", "start_s",
              "length_s", "similarity"]:
        np.testing.assert_array_equal(ch[f], exp[f], err_msg=f)


@pytest.mark.parametrize("policy", ["exploit", "rule"])
def test_plan_config2_t_sweep(orc, policy):
    """Config 2: 1K entries, B=256, mixed durations 2.5-10 s, T in {50,100,200}."""
    from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, requests
    c = SynthCache(1000, 512, 0.25, seed=21, clustered=True)
    wc = _cache(c, max_batch=256)
    neg = oracle.Ref().negative(512) if oracle.os.path.exists(oracle.REF_SO) else \
        np.random.default_rng(0).standard_normal(512).astype(np.float32)
    neg = (neg / np.linalg.norm(neg.astype(np.float64))).astype(np.float32)
    th, ps = trained_like_gater()
    wc.set_negative(neg)
    wc.set_gater(th, ps)
    B = 256
    q = perturbed_queries(c, B, seed=9, frac_random=0.1)
    L = request_durations(B)
    ids = np.arange(1, B + 1, dtype=np.uint64)
    for T in (50, 100, 200):
        Ts = np.full(B, T, np.int32)
        ch = wc.choices(wc.plan(q, requests(ids, L, Ts), seed=1, sel=SelectorConfig(8),
                                policy=Policy(policy)))
        o, _ = orc.plan_batch(_arena(c), neg, q, L, ids, Ts, policy=policy, theta=th, psi=ps,
                              rule_arm=11, nthreads=8)
        for f in ["hit", "arm", "steps_skipped", "entry_id", "level", "similarity", "pick"]:
            np.testing.assert_array_equal(ch[f], o[f], err_msg=f"{f} T={T}")
    # fixed-arm sweep: t* table for every arm
    for arm in range(14):
        ch = wc.choices(wc.plan(q[:32], requests(ids[:32], L[:32], np.full(32, 200, np.int32)),
                                policy=Policy("fixed", fixed_arm=arm)))
        assert (ch["arm"] == arm).all()
        assert (ch["steps_skipped"] == int(np.floor(0.05 * arm * 200 + 0.5))).all()


def test_plan_config1_single_query(orc):
    """Config 1: 1K entries, single query, top-1 + duration gate."""
    from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, requests
    c = SynthCache(1000, 512, 0.25, seed=5)
    wc = _cache(c, max_batch=1)
    neg = np.zeros(512, np.float32)
    neg[0] = 1
    wc.set_negative(neg)
    q = perturbed_queries(c, 1)
    L = np.array([c.durations[0] * 0.9])
    ch = wc.choices(wc.plan(q, requests([1], L, [200]), sel=SelectorConfig(1),
                            policy=Policy("rule")))
    o, _ = orc.plan_batch(_arena(c), neg, q, L, np.array([1], np.uint64), np.array([200], np.int32),
                          top_k=1, policy="rule", rule_arm=11)
    for f in ["hit", "arm", "steps_skipped", "entry_id", "similarity"]:
        assert ch[f][0] == o[f][0], f


# ------------------------------------------------------------------ components
def test_score_select_golden(golden):
    from paper_2603_07865_b200.warmstart import SelectorConfig, WarmStartCache
    g = golden["gate_cases"]
    wc = WarmStartCache(8, rows_per_entry=1, max_entries=16, latent_shape=None)
    n_amb = 0
    for c in range(g["n"].shape[0]):
        n = int(g["n"][c])
        sc, pick, flags = wc.score_select(g["sims"][c, :n], g["s_neg"][c, :n], g["durs"][c, :n],
                                          float(g["L"][c]),
                                          SelectorConfig(8, float(g["temp"][c]), float(g["thr"][c])),
                                          int(g["rng_seed"][c]))
        for j, name in enumerate(["s_pos", "s_neg", "a", "b", "q"]):
            np.testing.assert_array_equal(sc[:, j], g[name][c, :n], err_msg=f"case {c} {name}")
        n_amb += flags & 1
        if not flags & 1:
            assert pick == g["pick"][c], c
    assert n_amb == 0


def test_gater_golden(golden):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    g = golden["gater_cases"]
    wc = WarmStartCache(512, rows_per_entry=1, max_entries=16, latent_shape=None)
    wc.set_gater(g["theta"], g["psi"], 1.0)
    phi, arm = wc.gater(g["P"], g["S"], g["T"], explore=False)
    np.testing.assert_array_equal(phi, g["phi"])
    np.testing.assert_array_equal(arm, g["arm_exploit"])
    _, arm = wc.gater(g["P"], g["S"], g["T"], explore=True)
    np.testing.assert_array_equal(arm, g["arm_explore"])
    wc.set_gater(np.zeros(154), np.zeros(154), 1.0)
    _, arm = wc.gater(g["P"], g["S"], g["T"])
    assert (arm == 13).all()


def test_score_select_errors():
    from paper_2603_07865_b200.warmstart import SelectorConfig, WarmStartCache
    wc = WarmStartCache(8, rows_per_entry=1, max_entries=16, latent_shape=None)
    with pytest.raises(ValueError):  # empty candidate list (selector.cpp:28)
        wc.score_select([], [], [], 5.0, SelectorConfig(), 1)
    with pytest.raises(ValueError):  # L <= 0 (selector.cpp:29-31)
        wc.score_select([0.5], [0.1], [5.0], 0.0, SelectorConfig(), 1)
    with pytest.raises(ValueError):  # temperature <= 0 (selector.cpp:10)
        wc.score_select([0.5], [0.1], [5.0], 5.0, SelectorConfig(8, 0.0), 1)


# ------------------------------------------------------------------ arena mutations
def test_arena_insert_remove_replace(orc):
    c = SynthCache(400, 64, 0.25, seed=13, clustered=True)
    wc = _cache(c, max_entries=512)
    q = perturbed_queries(c, 64)
    rng = np.random.default_rng(2)
    alive = np.ones(400, bool)
    for e in rng.choice(400, 120, replace=False):
        assert wc.remove(int(c.ids[e]))
        alive[e] = False
    with pytest.warns(UserWarning):
        assert not wc.remove(999999)  # unknown id: warn + no-op (index.cpp:243-245)
    assert wc.entry_count() == alive.sum()
    # replace (refine) 30 surviving entries with new rows
    c2 = SynthCache(400, 64, 0.25, seed=99, clustered=True)
    for e in np.flatnonzero(alive)[:30]:
        wc.replace(int(c.ids[e]), c2.entry_rows(e), c.levels[c.off[e]:c.off[e + 1]],
                   c.starts[c.off[e]:c.off[e + 1]], c.lengths[c.off[e]:c.off[e + 1]])
        c.rows[c.off[e]:c.off[e + 1]] = c2.entry_rows(e)
    # re-insert 50 removed entries (reuses freed slots)
    for e in np.flatnonzero(~alive)[:50]:
        wc.insert(int(c.ids[e]), c.entry_rows(e), c.levels[c.off[e]:c.off[e + 1]],
                  c.starts[c.off[e]:c.off[e + 1]], c.lengths[c.off[e]:c.off[e + 1]])
        alive[e] = True
    keep = np.flatnonzero(alive)
    offs = np.concatenate([[0], np.cumsum(c.off[keep + 1] - c.off[keep])])
    rows = np.concatenate([c.entry_rows(e) for e in keep])
    sl = lambda a: np.concatenate([a[c.off[e]:c.off[e + 1]] for e in keep])
    ar = oracle.Arena(c.ids[keep], offs, rows, sl(c.levels), sl(c.starts), sl(c.lengths))
    for mode_hits in (wc.search(q, 8),):
        _check_hits(*mode_hits, ar, orc, q, 8)
    np.testing.assert_array_equal(wc.read_rows(int(c.ids[keep[0]]))[:7], c.entry_rows(keep[0]))


def test_arena_capacity_and_bad_rows():
    from paper_2603_07865_b200.warmstart import WarmStartCache
    wc = WarmStartCache(16, rows_per_entry=3, max_entries=4, latent_shape=None)
    r = np.eye(16, dtype=np.float32)[:3]
    for i in range(256 // 4):  # capacity rounds up to whole 256-row tiles (Rp=4 -> 64 entries)
        wc.insert(i + 1, r, [0, 1, 1], [0, 0, 1], [2, 1, 1])
    with pytest.raises(Exception):
        wc.insert(1000, r, [0, 1, 1], [0, 0, 1], [2, 1, 1])
    with pytest.raises(ValueError):  # more rows than rows_per_entry pads to
        wc.insert(1, np.eye(16, dtype=np.float32)[:5], [0] * 5, [0] * 5, [1] * 5)


# ------------------------------------------------------------------ align + noise
def _latent_cache(n=64, seed=0):
    from paper_2603_07865_b200.warmstart import WarmStartCache
    c = SynthCache(n, 64, 0.25, seed=seed)
    wc = WarmStartCache(64, rows_per_entry=7, max_entries=n, latent_shape=(8, 256, 16),
                        max_batch=64)
    rng = np.random.default_rng(seed)
    lats = []
    for e in range(n):
        ts = int(np.floor(c.durations[e] * 25 + 0.5))
        lat = rng.standard_normal((8, ts, 16)).astype(np.float32)
        lats.append(lat)
        wc.insert(int(c.ids[e]), c.entry_rows(e), c.levels[c.off[e]:c.off[e + 1]],
                  c.starts[c.off[e]:c.off[e + 1]], c.lengths[c.off[e]:c.off[e + 1]], latent=lat)
    return c, wc, lats


@pytest.mark.parametrize("eps_mode", ["input", "philox"])
def test_align_noise_matches_restatement(orc, eps_mode):
    from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, requests
    c, wc, lats = _latent_cache()
    B = 48
    q = perturbed_queries(c, B, seed=4)
    L = request_durations(B, 2.5, 10.0, seed=5)
    ids = np.arange(100, 100 + B, dtype=np.uint64)
    reqs = requests(ids, L, np.full(B, 200, np.int32))
    buf = wc.plan(q, reqs, sel=SelectorConfig(8), policy=Policy("fixed", fixed_arm=9))
    ch = wc.choices(buf)
    assert ch["hit"].sum() > B // 2
    tmax = 256
    eps = None
    if eps_mode == "input":
        eps = np.random.default_rng(1).standard_normal((B, 8, tmax, 16)).astype(np.float32)
    out = wc.align_noise(buf, reqs, tmax, eps=eps, philox_seed=777).cpu().numpy()
    abar = orc.abar_table()
    slot_of = {int(i): e for e, i in enumerate(c.ids)}
    for b in range(B):
        if not ch["hit"][b]:
            assert not out[b].any()
            continue
        e = slot_of[int(ch["entry_id"][b])]
        ab = abar[orc.abar_index(200, int(ch["steps_skipped"][b]))]
        t_out = int(ch["t_out"][b])
        ep = None if eps is None else np.ascontiguousarray(eps[b, :, :t_out])
        ref = orc.align_noise(lats[e], float(ch["start_s"][b]), float(ch["length_s"][b]),
                              float(L[b]), 25.0, ab, eps=ep, seed=777, rid=int(ids[b]))
        assert ref.shape[1] == t_out
        got = out[b, :, :t_out]
        # bit-exact in both modes: eps input, and Philox + the fully specified table transform
        np.testing.assert_array_equal(got, ref)
        assert not out[b, :, t_out:].any()
