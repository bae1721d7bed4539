"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libsemwarm_ref.so).

Run in the build container (needs /root/reference to have built oracle/_ref):
    python tests/golden/make_golden.py
The fixtures are small and committed; the GPU box never needs the reference itself.

warm_cache.npz  a cache whose pyramid segment rows come from the reference's own
                build_entry_vectors (index.cpp:48-57, libm Box-Muller), prompts from its
                perturb(), negative from make_negative_embedding; expected outputs of the
                reference plan flow (search -> score_candidates -> select -> features ->
                choose_arm/rule/fixed -> t*) for every policy, plus raw IvfIndex::search hits.
gate_cases.npz  random candidate sets through score_candidates + select (selector.cpp:24-85).
gater_cases.npz random (prompt, segment, T) through context_features + choose_arm.
seeds.npz       derive_seed and the first mt19937_64 draw (core.cpp:65-71, core.hpp:83).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from paper_2603_07865_b200.synth import trained_like_gater  # noqa: E402


def warm_cache(ref: oracle.Ref, n_entries=300, dim=64, delta=0.25, B=96, seed=1):
    rng = np.random.default_rng(2026)
    emb_seed = ref.derive_seed(seed, 0x5345474D)  # pipeline.cpp:76-78
    # clustered full embeddings (synth_workload centres, simgen.cpp:162-194 shape)
    centres = ref.random_unit_vectors(99, 8, dim)
    rows, lv, st, ln, off, ids, durs, fulls = [], [], [], [], [0], [], [], []
    for e in range(n_entries):
        eid = e + 1
        base = centres[e % 8] if rng.random() < 0.5 or e == 0 else fulls[int(rng.integers(0, e))]
        full = ref.perturb(base, 0.5 if base is centres[e % 8] else 0.16, 1000 + e)
        dur = float(rng.uniform(4.0, 12.0))
        r, a, b, c = ref.build_entry_vectors(eid, full, dur, delta, emb_seed)
        rows.append(r), lv.append(a), st.append(b), ln.append(c)
        off.append(off[-1] + len(a))
        ids.append(eid), durs.append(dur), fulls.append(full)
    rows = np.concatenate(rows)
    ar = oracle.Arena(np.array(ids, np.uint64), np.array(off, np.int64), rows,
                      np.concatenate(lv), np.concatenate(st), np.concatenate(ln))
    neg = ref.negative(dim)
    src = rng.integers(0, n_entries, B)
    queries = np.stack([ref.perturb(fulls[s], 0.3, 5000 + i) for i, s in enumerate(src)])
    queries[-8:] = ref.random_unit_vectors(77, 8, dim)  # some far-away prompts (misses)
    L = rng.uniform(2.5, 10.0, B)
    req_ids = np.arange(1, B + 1, dtype=np.uint64)
    T = rng.choice([50, 100, 200], B).astype(np.int32)
    theta, psi = trained_like_gater()
    idx = ref.index(ar)
    out = dict(ids=ar.ids, off=ar.off, rows=ar.rows, levels=ar.levels, starts=ar.starts,
               lengths=ar.lengths, neg=neg, queries=queries.astype(np.float32), L=L,
               req_ids=req_ids, T=T, theta=theta, psi=psi, seed=np.uint64(seed))
    for pol in ["exploit", "explore", "rule", "fixed"]:
        p, hid, hs = idx.plan_batch(neg, queries, L, req_ids, T, seed=seed, top_k=8,
                                    policy=pol, theta=theta, psi=psi, beta=1.0, fixed_arm=7)
        out[f"plan_{pol}"] = p
        out["hit_ids"], out["hit_sims"] = hid, hs
    k = 5
    sid = np.zeros((B, k), np.uint64)
    ssim = np.zeros((B, k), np.float64)
    slv = np.zeros((B, k), np.int32)
    sn = np.zeros(B, np.int32)
    for i in range(B):
        a, b, _, _, e = idx.search(queries[i], k)
        sn[i] = len(a)
        sid[i, :len(a)], slv[i, :len(a)], ssim[i, :len(a)] = a, b, e
    out.update(search_k=np.int32(k), search_ids=sid, search_levels=slv, search_sims=ssim,
               search_n=sn)
    np.savez_compressed(os.path.join(HERE, "warm_cache.npz"), **out)


def gate_cases(ref: oracle.Ref, n_cases=200, dim=32):
    rng = np.random.default_rng(7)
    neg = ref.negative(dim)
    L_ = ref.lib
    import ctypes as C
    rows = []
    for c in range(n_cases):
        n = int(rng.integers(1, 9))
        sims = rng.uniform(-0.2, 1.0, n)
        if c % 10 == 0:
            sims[:] = rng.uniform(-0.5, 0.0, n)  # all-negative: every a = 0 (miss path)
        audio = ref.random_unit_vectors(300 + c, n, dim)
        durs = rng.uniform(2.0, 15.0, n)
        L = float(rng.uniform(2.5, 10.0))
        temp = float(rng.choice([0.05, 0.1, 1.0]))
        thr = float(rng.choice([0.0, 0.6, 0.9]))
        rs = int(rng.integers(0, 2**63))
        sp, sn_, a, b, q = (np.zeros(n) for _ in range(5))
        ids = np.arange(1, n + 1, dtype=np.uint64)
        lv = np.zeros(n, np.int32)
        pick = L_.ref_score_select(n, ids, lv, np.zeros(n), durs, sims, audio, dim, neg,
                                   audio[0], L, 8, temp, thr, C.c_uint64(rs), sp, sn_, a, b, q)
        rows.append((n, sims, audio, durs, L, temp, thr, rs, sp, sn_, a, b, q, pick))
    N = max(r[0] for r in rows)
    pad = lambda x, fill=0.0: np.pad(x, (0, N - len(x)), constant_values=fill)
    np.savez_compressed(
        os.path.join(HERE, "gate_cases.npz"), neg=neg,
        n=np.array([r[0] for r in rows], np.int32),
        sims=np.stack([pad(r[1]) for r in rows]),
        audio=np.stack([np.pad(r[2], ((0, N - r[0]), (0, 0))) for r in rows]).astype(np.float32),
        durs=np.stack([pad(r[3]) for r in rows]), L=np.array([r[4] for r in rows]),
        temp=np.array([r[5] for r in rows]), thr=np.array([r[6] for r in rows]),
        rng_seed=np.array([r[7] for r in rows], np.uint64),
        s_pos=np.stack([pad(r[8]) for r in rows]), s_neg=np.stack([pad(r[9]) for r in rows]),
        a=np.stack([pad(r[10]) for r in rows]), b=np.stack([pad(r[11]) for r in rows]),
        q=np.stack([pad(r[12]) for r in rows]), pick=np.array([r[13] for r in rows], np.int32))


def gater_cases(ref: oracle.Ref, n=128, dim=512):
    rng = np.random.default_rng(9)
    P = ref.random_unit_vectors(11, n, dim)
    S = np.stack([ref.perturb(P[i], float(rng.uniform(0.05, 2.0)), 900 + i) for i in range(n)])
    T = rng.choice([50, 100, 200], n).astype(np.int32)
    theta, psi = trained_like_gater()
    phi = np.stack([ref.context_features(P[i], S[i], int(T[i])) for i in range(n)])
    arm_x = np.array([ref.choose_arm(theta, psi, 1.0, phi[i], False) for i in range(n)], np.int32)
    arm_e = np.array([ref.choose_arm(theta, psi, 1.0, phi[i], True) for i in range(n)], np.int32)
    zeros = np.zeros(14 * 11, np.float32)
    arm_z = np.array([ref.choose_arm(zeros, zeros, 1.0, phi[i], False) for i in range(n)], np.int32)
    np.savez_compressed(os.path.join(HERE, "gater_cases.npz"), P=P, S=S, T=T, theta=theta,
                        psi=psi, phi=phi, arm_exploit=arm_x, arm_explore=arm_e, arm_zero=arm_z)


def seeds(ref: oracle.Ref):
    rng = np.random.default_rng(3)
    base = rng.integers(0, 2**63, 64, dtype=np.uint64)
    a = rng.integers(0, 2**63, 64, dtype=np.uint64)
    ds = np.array([ref.derive_seed(int(b), int(x), 2) for b, x in zip(base, a)], np.uint64)
    first = np.array([ref.lib.ref_rng_first_u64(int(s)) for s in ds], np.uint64)
    uni = np.array([ref.lib.ref_rng_first_uniform(int(s)) for s in ds], np.float64)
    np.savez_compressed(os.path.join(HERE, "seeds.npz"), base=base, a=a, derived=ds,
                        first_u64=first, first_uniform=uni)


if __name__ == "__main__":
    oracle.build()
    r = oracle.Ref()
    seeds(r)
    gate_cases(r)
    gater_cases(r)
    warm_cache(r)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
