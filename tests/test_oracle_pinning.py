"""CPU: pin the C restatement (oracle/semwarm_oracle.c) to the compiled reference and to the
committed golden vectors, and check the reference's own known answers (SPEC examples).
These tests are the reason the GPU parity tests may trust the restatement as their checker."""
import os

import numpy as np
import pytest

import oracle
from paper_2603_07865_b200.synth import (SynthCache, perturbed_queries, request_durations,
                                         trained_like_gater)


def _arena(c):
    return oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)


# ------------------------------------------------------------------ seeding / RNG
def test_derive_seed_and_first_draw_golden(orc, golden):
    g = golden["seeds"]
    for b, a, d, f, u in zip(g["base"], g["a"], g["derived"], g["first_u64"], g["first_uniform"]):
        assert orc.derive_seed(int(b), int(a), 2) == int(d)
        assert orc.mt64_first(int(d)) == int(f)
        assert orc.uniform_first(int(d)) == float(u)


def test_mt64_closed_form_vs_reference(orc, ref):
    rng = np.random.default_rng(0)
    for s in rng.integers(0, 2**64 - 1, 2000, dtype=np.uint64):
        assert orc.mt64_first(int(s)) == ref.lib.ref_rng_first_u64(int(s))


# ------------------------------------------------------------------ search
@pytest.mark.parametrize("dim,delta,clustered", [(64, 0.25, False), (512, 0.25, True),
                                                 (64, 1.0, True), (96, 1 / 16, False)])
def test_search_matches_reference(orc, ref, dim, delta, clustered):
    c = SynthCache(150, dim, delta, seed=5, clustered=clustered)
    ar = _arena(c)
    idx = ref.index(ar)
    q = perturbed_queries(c, 24, frac_random=0.25)
    for k in (1, 3, 8, 200):
        for i in range(q.shape[0]):
            ids, lv, st, ln, sm = idx.search(q[i], k)
            h = orc.search(ar, q[i], k)
            assert len(h) == len(ids) == min(k, 150)
            np.testing.assert_array_equal(h["entry_id"], ids)
            np.testing.assert_array_equal(h["level"], lv)
            np.testing.assert_array_equal(h["start_s"], st)
            np.testing.assert_array_equal(h["similarity"], sm)  # bit-exact fp64


def test_search_self_retrieval_and_dedup(orc):
    # SPEC.md:146 self-retrieval: an indexed vector ranks first with similarity 1.0
    c = SynthCache(60, 32, 0.25, seed=2)
    ar = _arena(c)
    for e in range(0, 60, 7):
        h = orc.search(ar, c.entry_rows(e)[3], 10)
        assert h[0]["entry_id"] == c.ids[e] and h[0]["similarity"] == pytest.approx(1.0, abs=1e-6)
        assert len(set(h["entry_id"].tolist())) == len(h)  # at most one hit per entry


def test_empty_index_is_a_miss(orc):
    ar = oracle.Arena(np.zeros(0, np.uint64), np.zeros(1, np.int64), np.zeros((0, 8), np.float32),
                      np.zeros(0, np.int32), np.zeros(0), np.zeros(0))
    assert len(orc.search(ar, np.ones(8, np.float32) / np.sqrt(8), 5)) == 0


# ------------------------------------------------------------------ plan (full path)
@pytest.mark.parametrize("policy", ["exploit", "explore", "rule", "fixed"])
@pytest.mark.parametrize("dim,delta", [(64, 0.25), (512, 0.25), (128, 0.5)])
def test_plan_matches_reference(orc, ref, policy, dim, delta):
    c = SynthCache(200, dim, delta, seed=11, clustered=True)
    ar = _arena(c)
    neg = ref.negative(dim)
    B = 48
    q = perturbed_queries(c, B, seed=3, frac_random=0.2)
    L = request_durations(B)
    ids = np.arange(1, B + 1, dtype=np.uint64)
    T = np.random.default_rng(1).choice([50, 100, 200], B).astype(np.int32)
    th, ps = trained_like_gater()
    a, hid, hs = ref.index(ar).plan_batch(neg, q, L, ids, T, policy=policy, theta=th, psi=ps,
                                          fixed_arm=4, nthreads=4)
    b, hh = orc.plan_batch(ar, neg, q, L, ids, T, policy=policy, theta=th, psi=ps,
                           fixed_arm=4, rule_arm=11, nthreads=4)
    assert (a == b).all()
    np.testing.assert_array_equal(hh["entry_id"], hid)
    np.testing.assert_array_equal(hh["similarity"], hs)


def test_plan_golden(orc, golden):
    g = golden["warm_cache"]
    ar = oracle.Arena(g["ids"], g["off"], g["rows"], g["levels"], g["starts"], g["lengths"])
    for pol in ["exploit", "explore", "rule", "fixed"]:
        b, _ = orc.plan_batch(ar, g["neg"], g["queries"], g["L"], g["req_ids"], g["T"],
                              seed=int(g["seed"]), policy=pol, theta=g["theta"], psi=g["psi"],
                              fixed_arm=7, rule_arm=11)
        assert (b == g[f"plan_{pol}"]).all(), pol
    k = int(g["search_k"])
    for i in range(g["queries"].shape[0]):
        h = orc.search(ar, g["queries"][i], k)
        n = int(g["search_n"][i])
        np.testing.assert_array_equal(h["entry_id"], g["search_ids"][i, :n])
        np.testing.assert_array_equal(h["similarity"], g["search_sims"][i, :n])


# ------------------------------------------------------------------ selector known answers
def test_gate_spec_example(orc):
    # s_pos=[0.8,0.6], s_neg=[0.1,0.2] -> a=[1,0.75], b=[1,0.888..], q=[1,0.75]
    # (s_neg enters through cos(audio, neg): build audio rows with exactly those cosines)
    dim = 4
    neg = np.array([1, 0, 0, 0], np.float32)
    audio = np.array([[0.1, np.sqrt(1 - 0.01), 0, 0], [0.2, np.sqrt(1 - 0.04), 0, 0]], np.float32)
    sp, sn, a, b, q = (np.zeros(2) for _ in range(5))
    orc.lib.so_score_select(2, np.array([0.8, 0.6]), np.array([10.0, 10.0]), audio, dim, neg,
                            10.0, 0.05, 0.6, 1, sp, sn, a, b, q)
    np.testing.assert_allclose(a, [1.0, 0.75])
    np.testing.assert_allclose(b, [1.0, (1 - sn[1]) / (1 - sn[0])])
    np.testing.assert_allclose(q, [1.0, 0.75])
    assert sn[0] == pytest.approx(0.1, abs=1e-7) and sn[1] == pytest.approx(0.2, abs=1e-7)


def test_gate_golden(orc, golden):
    g = golden["gate_cases"]
    neg = g["neg"]
    dim = neg.shape[0]
    for c in range(g["n"].shape[0]):
        n = int(g["n"][c])
        sp, sn, a, b, q = (np.zeros(n) for _ in range(5))
        pick = orc.lib.so_score_select(
            n, np.ascontiguousarray(g["sims"][c, :n]), np.ascontiguousarray(g["durs"][c, :n]),
            np.ascontiguousarray(g["audio"][c, :n]), dim, neg, float(g["L"][c]),
            float(g["temp"][c]), float(g["thr"][c]), int(g["rng_seed"][c]), sp, sn, a, b, q)
        assert pick == g["pick"][c]
        for name, v in [("s_pos", sp), ("s_neg", sn), ("a", a), ("b", b), ("q", q)]:
            np.testing.assert_array_equal(v, g[name][c, :n], err_msg=f"case {c} {name}")


def test_gater_golden(orc, golden):
    g = golden["gater_cases"]
    for i in range(g["P"].shape[0]):
        phi = orc.context_features(g["P"][i], g["S"][i], int(g["T"][i]))
        np.testing.assert_array_equal(phi, g["phi"][i])
        assert orc.choose_arm(g["theta"], g["psi"], 1.0, phi, False) == g["arm_exploit"][i]
        assert orc.choose_arm(g["theta"], g["psi"], 1.0, phi, True) == g["arm_explore"][i]
        z = np.zeros(154, np.float32)
        assert orc.choose_arm(z, z, 1.0, phi, False) == 13  # SPEC.md:333 zero model -> arm 13


def test_choose_arm_nonfinite_falls_back_to_arm0(orc, ref):
    th, ps = trained_like_gater()
    phi = np.ones(11)
    phi[3] = np.nan
    assert orc.choose_arm(th, ps, 1.0, phi) == 0 == ref.choose_arm(th, ps, 1.0, phi)


def test_t_star_rounding(orc):
    # llround(0.05 * arm * T): T=50, arm 1 -> 2.5 -> 3 (half away from zero)
    for T, arm, exp in [(50, 1, 3), (50, 3, 8), (200, 13, 130), (100, 7, 35), (1, 13, 1)]:
        assert int(np.floor(0.05 * arm * T + 0.5)) == exp


# ------------------------------------------------------------------ align + noise restatement
def test_align_noise_crop_tile_and_schedule(orc):
    rng = np.random.default_rng(4)
    lat = rng.standard_normal((8, 200, 16)).astype(np.float32)
    eps = rng.standard_normal((8, 256, 16)).astype(np.float32)
    abar = orc.abar_table()
    assert abar[0] == 1.0 and 0 < abar[1000] < 0.01
    ab = abar[orc.abar_index(200, 60)]
    s0, s1 = np.float32(np.sqrt(ab)), np.float32(np.sqrt(1 - ab))
    # crop: segment [2 s, 6 s) = frames [50, 150), L = 3 s -> 75 frames
    x = orc.align_noise(lat, 2.0, 4.0, 3.0, 25.0, ab, eps=eps[:, :75].copy())
    assert x.shape == (8, 75, 16)
    expect = (s0 * lat[:, 50:125]).astype(np.float32)
    np.testing.assert_allclose(x, expect + s1 * eps[:, :75], rtol=1e-6, atol=1e-6)
    # tile: segment of 40 frames stretched to L = 4 s (100 frames) repeats cyclically
    x = orc.align_noise(lat, 1.0, 1.6, 4.0, 25.0, 1.0, eps=np.zeros((8, 100, 16), np.float32))
    np.testing.assert_array_equal(x[:, 40:80], lat[:, 25:65])
    np.testing.assert_array_equal(x[:, 80:100], lat[:, 25:45])


def test_philox_known_answer(orc):
    # Random123 known-answer vector for philox4x32-10 (counter = key = 0)
    import ctypes as C
    out = (C.c_uint32 * 4)()
    orc.lib.so_philox4x32_10((C.c_uint32 * 4)(0, 0, 0, 0), (C.c_uint32 * 2)(0, 0), out)
    assert list(out) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    # the noise generator is the same round function run 7 times (csrc/noise_def.h): R rounds
    # are a prefix of R + 1, and 10 rounds through so_philox4x32_r equal the pinned vector
    r10 = (C.c_uint32 * 4)()
    orc.lib.so_philox4x32_r((C.c_uint32 * 4)(0, 0, 0, 0), (C.c_uint32 * 2)(0, 0), 10, r10)
    assert list(r10) == list(out)
    ctr, key = (C.c_uint32 * 4)(7, 0, 123, 456), (C.c_uint32 * 2)(0x5EED, 1)
    r7, r8, step = (C.c_uint32 * 4)(), (C.c_uint32 * 4)(), (C.c_uint32 * 4)()
    orc.lib.so_philox4x32_r(ctr, key, 7, r7)
    orc.lib.so_philox4x32_r(ctr, key, 8, r8)
    # round 8 = one round of the bijection on round 7's output with the key bumped 7 times
    k8 = (C.c_uint32 * 2)((0x5EED + 7 * 0x9E3779B9) & 0xFFFFFFFF, (1 + 7 * 0xBB67AE85) & 0xFFFFFFFF)
    orc.lib.so_philox4x32_r(r7, k8, 1, step)
    assert list(step) == list(r8)
    z = orc.philox_normals(1, 2, 1 << 16)
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1) < 0.02


def test_normal_transform_tracks_erfcinv(orc):
    """Our normal transform (v from the word's low 23 bits, one fma from
    the committed segment table, the word's sign bit) at EVERY one of the 2^23 magnitudes,
    against its target sqrt(2) erfcinv(v - 2^-24) in float64: |d| <= 1e-5 everywhere, tails
    included, and odd in the sign bit."""
    from scipy.special import erfcinv
    m = np.arange(1 << 23, dtype=np.uint32)
    z = orc.icdf_normals(m)
    v = 2.0 - (1.0 + m.astype(np.float64) * 2.0 ** -23)
    ref = np.sqrt(2.0) * erfcinv(v - 2.0 ** -24)
    err = np.abs(z.astype(np.float64) - ref)
    assert err.max() <= 1e-5, err.max()
    zn = orc.icdf_normals(m[::97] | np.uint32(0x80000000))
    np.testing.assert_array_equal(zn, -z[::97])
    # the high bits 23..30 do not enter; the largest magnitude is the 2^-23 cell's median
    np.testing.assert_array_equal(orc.icdf_normals(m[:4096] | np.uint32(0x7F800000)), z[:4096])
    assert 5.41 < z.max() < 5.43


def test_noise_distribution(orc):
    """Philox4x32-7 words (the noise generator) through the transform are N(0, 1): moments and the Kolmogorov-Smirnov
    distance over 4M draws of one request (KS 1%-critical value 1.63 / sqrt(n) = 8.2e-4)."""
    from scipy.special import ndtr
    n = 1 << 22
    z = orc.philox_normals(0x5EED, 12345, n).astype(np.float64)
    assert abs(z.mean()) < 5 / np.sqrt(n)
    assert abs(z.var() - 1) < 5 * np.sqrt(2 / n)
    assert abs((z ** 3).mean()) < 5 * np.sqrt(15 / n)
    assert abs((z ** 4).mean() - 3) < 5 * np.sqrt(96 / n)
    zs = np.sort(z)
    cdf = ndtr(zs)
    ks = max((np.arange(1, n + 1) / n - cdf).max(), (cdf - np.arange(n) / n).max())
    assert ks < 8.2e-4, ks
    assert np.abs(z).max() < 5.43


def test_reference_ivf_harness(ref):
    """The IVF reference shims (ref_ivf_new + SWIX snapshot) used by the GPU IVF parity tests:
    a 300-entry index with 16 lists rebuilt during the inserts is self-consistent, its snapshot
    holds every row exactly once, and probing every list gives the exhaustive similarities."""
    import oracle
    from paper_2603_07865_b200.synth import SynthCache, perturbed_queries
    c = SynthCache(300, 32, 0.25, seed=41, clustered=True)
    ar = oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    ri = ref.index(ar, ivf=(16, 3, 16, 256))
    assert ri.consistent()
    cent, nprobe, lists = ri.snapshot()
    assert cent.shape == (16, 32) and nprobe == 16
    assert sum(len(x) for x in lists) == len(c.rows)
    assert np.allclose(np.linalg.norm(cent, axis=1), 1.0, atol=1e-5)  # spherical k-means
    ex = ref.index(ar)
    for q in perturbed_queries(c, 16, frac_random=0.2):
        a, b = ri.search(q, 8), ex.search(q, 8)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[4], b[4])


def test_glibc_exp_restatement_is_bit_exact(orc):
    """so_ref_exp (the oracle's restatement of glibc 2.39's FMA-build exp, which the device's
    ref_exp repeats op for op) against the library's exp on 5M arguments: the softmax range,
    the whole finite range, tiny arguments and the special cases (underflow to subnormals,
    overflow, +-inf, nan). Needs the FMA + AVX2 ifunc the reference gets on the GPU box."""
    import re
    flags = open("/proc/cpuinfo").read() if os.path.exists("/proc/cpuinfo") else ""
    if not (re.search(r"\bfma\b", flags) and re.search(r"\bavx2\b", flags)):
        pytest.skip("libm's exp ifunc is not the FMA build on this CPU")
    rng = np.random.default_rng(0)
    s = rng.uniform(0, 1, (200000, 2))
    t = rng.uniform(0.005, 1, 200000)
    x = np.concatenate([
        rng.uniform(-50, 0, 2_000_000), rng.uniform(-745.2, 709.8, 2_000_000),
        rng.standard_normal(800_000) * 1e-3, (s[:, 0] - s.max(1)) / t,
        np.array([0.0, -0.0, 1e-300, -1e-300, 2.0 ** -54, -2.0 ** -54, 2.0 ** -55, 709.78,
                  709.79, 710, -708.39, -708.4, -745.13, -745.14, -746, 1024, -1024, np.inf,
                  -np.inf, np.nan, 1.0, -1.0, 0.5])])
    ours, lib = orc.exp_pair(x)
    same = (ours.view(np.uint64) == lib.view(np.uint64)) | (np.isnan(ours) & np.isnan(lib))
    assert same.all(), x[~same][:8]


def test_glibc_log1p_restatement_is_bit_exact(orc):
    """so_ref_log1p (glibc 2.39's FMA-build log1p restated op for op; the device's ref_log1p
    repeats it) against the library's log1p on 5M arguments: exp(u) for the softplus range
    u in [-31, 31], all of (-1, 1), the finite range, and the branch boundaries."""
    import re
    flags = open("/proc/cpuinfo").read() if os.path.exists("/proc/cpuinfo") else ""
    if not (re.search(r"\bfma\b", flags) and re.search(r"\bavx2\b", flags)):
        pytest.skip("libm's log1p ifunc is not the FMA build on this CPU")
    rng = np.random.default_rng(1)
    x = np.concatenate([
        np.exp(rng.uniform(-31, 31, 2_000_000)), rng.uniform(-1, 1, 1_000_000),
        rng.uniform(-1, 0.5, 500_000), np.exp(rng.uniform(-745, 709, 1_000_000)),
        -np.exp(rng.uniform(-745, 0, 500_000)),
        np.array([0.0, -0.0, -1.0, -1.5, np.inf, -np.inf, np.nan, 2.0 ** -29, 2.0 ** -30,
                  2.0 ** -54, 2.0 ** -55, 1e-300, 5e-324, -0.2928932188134524,
                  -0.29289321881345254, 0.41421356237309503, 0.414213562373095, 2.0 ** 53,
                  2.0 ** 53 * 1.5, 1e308])])
    ours, lib = orc.log1p_pair(x)
    same = (ours.view(np.uint64) == lib.view(np.uint64)) | (np.isnan(ours) & np.isnan(lib))
    assert same.all(), x[~same][:8]
