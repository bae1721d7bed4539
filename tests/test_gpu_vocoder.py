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
