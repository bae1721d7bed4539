"""GPU: the phase-vocoder time stretch (csrc/vocoder.cu) vs the reference's time_stretch
(vocoder.cpp:128-207, compiled in oracle/_ref). Same length, same error cases, and samples equal
up to the libm difference of the per-bin polar conversion (hypot / atan2 / cos / sin, <= 2 ulp):
|d| <= 1e-6 * max(1, |ref|), and almost every sample bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _clips(ref, rng, n):
    out = []
    for i in range(n):
        L = int(rng.integers(40, 2400))
        kind = i % 3
        if kind == 0:  # the simulated backend's own latent (simgen.cpp:19-50)
            emb = rng.standard_normal(64).astype(np.float32)
            emb /= np.linalg.norm(emb)
            x = ref.synth_latent(emb, L / 200.0, 200)
        elif kind == 1:
            t = np.arange(L) / 200.0
            x = (0.5 * np.sin(2 * np.pi * 3.1 * t) + 0.2 * np.sin(2 * np.pi * 17.0 * t)).astype(np.float32)
        else:
            x = rng.uniform(-1, 1, L).astype(np.float32)
        out.append(x)
    return out


@pytest.mark.parametrize("window,hop", [(128, 32), (64, 16), (256, 64)])
def test_time_stretch_matches_reference(ref, window, hop):
    from paper_2603_07865_b200.warmstart import time_stretch
    rng = np.random.default_rng(window)
    clips = _clips(ref, rng, 48)
    ratios = rng.uniform(0.4, 2.5, len(clips))
    ratios[:4] = [0.4, 2.5, 1.0, 2.0 / 3.0]
    targets = [len(c) / 200.0 * r for c, r in zip(clips, ratios)]
    got = time_stretch(clips, 200, targets, window, hop)
    n_eq = n_tot = 0
    for c, t, g in zip(clips, targets, got):
        exp = ref.time_stretch(c, 200, t, window, hop)
        assert (g is None) == (exp is None)
        if exp is None:
            continue
        assert g.shape == exp.shape
        assert np.all(np.abs(g - exp) <= 1e-6 * np.maximum(1.0, np.abs(exp)))
        n_eq += int(np.sum(g == exp))
        n_tot += g.size
    assert n_eq >= 0.99 * n_tot, (n_eq, n_tot)


def test_time_stretch_errors(ref):
    from paper_2603_07865_b200.warmstart import time_stretch
    x = np.sin(np.arange(400) / 5.0).astype(np.float32)
    cases = [2.0 * 0.39, 2.0 * 2.51, 0.0, -1.0, 3.0]  # ratio < 0.4, > 2.5, target <= 0, ok
    got = time_stretch([x] * len(cases), 200, cases)
    for t, g in zip(cases, got):
        assert (g is None) == (ref.time_stretch(x, 200, t) is None)
    assert got[-1] is not None and got[-1].shape == (600,)
    with pytest.raises(ValueError):
        time_stretch([x], 200, [2.0], window=100, hop=25)  # StftConfig::validate


def test_align_vocoder_mode_matches_reference(ref, orc):
    """sw_align_noise in SW_ALIGN_VOCODER mode: every latent channel (c, f) of the chosen segment
    (slice_clip frames) stretched by the reference's time_stretch at the latent frame rate, then
    the same forward noising (eps input) as the crop/tile mode."""
    from paper_2603_07865_b200.synth import SynthCache, perturbed_queries, request_durations
    from paper_2603_07865_b200.warmstart import (Policy, SelectorConfig, WarmStartCache,
                                                 requests)
    c = SynthCache(48, 64, 0.25, seed=7)
    wc = WarmStartCache(64, rows_per_entry=7, max_entries=48, latent_shape=(4, 256, 8),
                        max_batch=64)
    rng = np.random.default_rng(2)
    lats = []
    for e in range(48):
        ts = int(np.floor(c.durations[e] * 25 + 0.5))
        lat = rng.standard_normal((4, ts, 8)).astype(np.float32)
        lats.append(lat)
        wc.insert(int(c.ids[e]), c.entry_rows(e), c.levels[c.off[e]:c.off[e + 1]],
                  c.starts[c.off[e]:c.off[e + 1]], c.lengths[c.off[e]:c.off[e + 1]], latent=lat)
    wc.set_align_mode("vocoder", 128, 32)
    B = 40
    q = perturbed_queries(c, B, seed=9)
    L = request_durations(B, 2.5, 10.0, seed=10)
    ids = np.arange(500, 500 + B, dtype=np.uint64)
    reqs = requests(ids, L, np.full(B, 200, np.int32))
    buf = wc.plan(q, reqs, sel=SelectorConfig(8), policy=Policy("fixed", fixed_arm=6))
    ch = wc.choices(buf)
    assert ch["hit"].sum() > B // 2
    eps = rng.standard_normal((B, 4, 256, 8)).astype(np.float32)
    out = wc.align_noise(buf, reqs, 256, eps=eps).cpu().numpy()
    abar = orc.abar_table()
    slot_of = {int(i): e for e, i in enumerate(c.ids)}
    n_checked = 0
    for b in range(B):
        if not ch["hit"][b]:
            continue
        lat = lats[slot_of[int(ch["entry_id"][b])]][:, :256]  # the arena keeps T_max frames
        lo = min(int(np.floor(ch["start_s"][b] * 25 + 0.5)), lat.shape[1])
        hi = max(min(int(np.floor((ch["start_s"][b] + ch["length_s"][b]) * 25 + 0.5)),
                     lat.shape[1]), lo)
        t_out = min(int(np.floor(L[b] * 25 + 0.5)), 256)
        ab = abar[orc.abar_index(200, int(ch["steps_skipped"][b]))]
        s0, s1 = np.float32(np.sqrt(ab)), np.float32(np.sqrt(1 - ab))
        for cc in range(4):
            for f in range(8):
                y = ref.time_stretch(lat[cc, lo:hi, f], 25, float(L[b]))
                assert y is not None  # the duration gate keeps the ratio inside [2/3, 2]
                x0 = y[:t_out].astype(np.float64)
                exp = (np.float64(s1) * eps[b, cc, :t_out, f] + (np.float32(s0) * y[:t_out]).astype(np.float64))
                got = out[b, cc, :t_out, f]
                assert np.all(np.abs(got - exp) <= 1e-5 * np.maximum(1.0, np.abs(exp))), (b, cc, f)
                del x0
        assert not out[b, :, t_out:].any()
        n_checked += 1
    assert n_checked > B // 2
