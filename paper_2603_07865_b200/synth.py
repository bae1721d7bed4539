"""Seeded synthetic caches and request batches.

Rows are unit vectors: fp64 normalise of N(0,1) draws rounded to fp32, as normalize() does
(reference core.cpp:40-52). Pyramid segment rows are normalize(full + 0.1 * dir) (the shape of
derive_segment_embedding, index.cpp:33-46; the direction here comes from numpy, not the
reference's Box-Muller stream — both sides of every parity check read these same bytes).
Two distributions: iid on the sphere, and clustered near-duplicates (the stress case for ties
and over-fetch).
"""
from __future__ import annotations

import numpy as np


def normalize_rows(x: np.ndarray) -> np.ndarray:
    x64 = np.asarray(x, np.float64)
    n = np.sqrt(np.sum(x64 * x64, axis=1, keepdims=True))
    return (x64 / n).astype(np.float32)


def pyramid(duration: float, delta: float):
    """pyramid_segments (index.cpp:12-31)."""
    delta = max(delta, 1.0 / 16.0)
    max_level = int(np.floor(np.log2(1.0 / delta) + 1e-9))
    lv, st, ln = [], [], []
    for level in range(max_level + 1):
        tiles = 1 << level
        length = duration / tiles
        for i in range(tiles):
            lv.append(level)
            st.append(i * length)
            ln.append(length)
    return np.array(lv, np.int32), np.array(st, np.float64), np.array(ln, np.float64)


class SynthCache:
    """n_entries entries, each with the R-row pyramid of `delta`, ids 1..n (admission order)."""

    def __init__(self, n_entries: int, dim: int = 512, delta: float = 0.25, seed: int = 1,
                 clustered: bool = False, dur_lo: float = 4.0, dur_hi: float = 12.0,
                 n_clusters: int = 16, spread: float = 0.5, dup_rate: float = 0.9,
                 dup_spread: float = 0.16):
        rng = np.random.default_rng(seed)
        if clustered:
            centres = normalize_rows(rng.standard_normal((n_clusters, dim)))
            full = np.empty((n_entries, dim), np.float32)
            for i in range(n_entries):
                if i > 0 and rng.random() < dup_rate:
                    j = int(rng.integers(0, i))
                    base, s = full[j], dup_spread
                else:
                    base, s = centres[i % n_clusters], spread
                g = normalize_rows(rng.standard_normal((1, dim)))[0]
                full[i] = normalize_rows((base.astype(np.float64) + s * g)[None])[0]
        else:
            full = normalize_rows(rng.standard_normal((n_entries, dim)))
        self.full = full
        self.durations = rng.uniform(dur_lo, dur_hi, n_entries)
        R = len(pyramid(1.0, delta)[0])
        self.R = R
        self.dim = dim
        self.ids = np.arange(1, n_entries + 1, dtype=np.uint64)
        self.off = np.arange(0, (n_entries + 1) * R, R, dtype=np.int64)
        rows = np.empty((n_entries, R, dim), np.float32)
        rows[:, 0] = full
        if R > 1:
            dirs = rng.standard_normal((n_entries, R - 1, dim))
            dirs /= np.linalg.norm(dirs, axis=2, keepdims=True)
            seg = full[:, None, :].astype(np.float64) + 0.1 * dirs.astype(np.float32).astype(np.float64)
            rows[:, 1:] = normalize_rows(seg.reshape(-1, dim)).reshape(n_entries, R - 1, dim)
        self.rows = rows.reshape(n_entries * R, dim)
        lv, st, ln = [], [], []
        for d in self.durations:
            a, b, c = pyramid(float(d), delta)
            lv.append(a), st.append(b), ln.append(c)
        self.levels = np.concatenate(lv).astype(np.int32)
        self.starts = np.concatenate(st)
        self.lengths = np.concatenate(ln)

    def entry_rows(self, e: int):
        return self.rows[self.off[e]:self.off[e + 1]]


def clustered_rows(n: int, dim: int = 512, seed: int = 1, n_clusters: int = 16,
                   spread: float = 0.5, dup_rate: float = 0.9, dup_spread: float = 0.16,
                   block: int = 65536) -> np.ndarray:
    """Vectorised §8d(ii) clustered near-duplicates at any size: like SynthCache(clustered=True)
    (16 centres, spread 0.5, dup rate 0.9, dup spread 0.16; synth_workload, simgen.hpp:87-98),
    except that a duplicate's parent is drawn from the rows of EARLIER blocks (the first block
    is generated row by row), so 1M rows take seconds instead of minutes."""
    rng = np.random.default_rng(seed)
    centres = normalize_rows(rng.standard_normal((n_clusters, dim)))
    out = np.empty((n, dim), np.float32)
    first = min(n, 256)
    for i in range(first):
        if i > 0 and rng.random() < dup_rate:
            base, s = out[int(rng.integers(0, i))], dup_spread
        else:
            base, s = centres[i % n_clusters], spread
        g = normalize_rows(rng.standard_normal((1, dim)))[0]
        out[i] = normalize_rows((base.astype(np.float64) + s * g)[None])[0]
    i0 = first
    while i0 < n:
        m = min(block, n - i0, i0)
        dup = rng.random(m) < dup_rate
        parent = rng.integers(0, i0, m)
        base = np.where(dup[:, None], out[parent], centres[(np.arange(i0, i0 + m)) % n_clusters])
        sc = np.where(dup, dup_spread, spread)[:, None]
        g = normalize_rows(rng.standard_normal((m, dim), dtype=np.float32))
        out[i0:i0 + m] = normalize_rows(base.astype(np.float64) + sc * g.astype(np.float64))
        i0 += m
    return out


def perturbed_queries(cache: SynthCache, B: int, scale: float = 0.3, seed: int = 7,
                      frac_random: float = 0.0) -> np.ndarray:
    """perturb(row, scale) of random cached full embeddings (core.cpp:116-124 shape)."""
    rng = np.random.default_rng(seed)
    n = cache.full.shape[0]
    src = cache.full[rng.integers(0, n, B)].astype(np.float64)
    g = rng.standard_normal((B, cache.dim))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    g = g.astype(np.float32).astype(np.float64)
    q = normalize_rows(src + scale * g)
    if frac_random > 0:
        m = rng.random(B) < frac_random
        q[m] = normalize_rows(rng.standard_normal((int(m.sum()), cache.dim)))
    return q


def request_durations(B: int, lo: float = 2.5, hi: float = 10.0, seed: int = 11) -> np.ndarray:
    return np.random.default_rng(seed).uniform(lo, hi, B)


def trained_like_gater(seed: int = 3):
    """A non-degenerate theta/psi (14 x 11) so exploit/explore exercise every branch."""
    rng = np.random.default_rng(seed)
    theta = (rng.standard_normal((14, 11)) * 0.05).astype(np.float64)
    # upper envelope of lines a * phi0 - a^2 / 26: the argmax arm tracks ~13 * similarity
    a = np.arange(14, dtype=np.float64)
    theta[:, 0] += a
    theta[:, 10] += -a * a / 26.0
    psi = (rng.standard_normal((14, 11)) * 0.3).astype(np.float32)
    return theta.astype(np.float32).reshape(-1), psi.reshape(-1)
