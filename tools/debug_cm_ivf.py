"""Debug aid: replay the Cache Manager churn in IVF mode against the reference and report the
first operation after which the IVF state (centroids / list sizes) diverges."""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2603_07865_b200.warmstart import CacheManager, WarmStartCache  # noqa: E402

ref = oracle.Ref()
seed, ivf = 3, (8, 2, 120, 17)
dim, cap, delta = 64, 48, 0.25
emb_seed = ref.derive_seed(seed, 0x5345474D)
wc = WarmStartCache(dim, rows_per_entry=7, max_entries=cap + 8, max_batch=32, latent_shape=None,
                    tc_always=True)
wc.ivf_configure(*ivf)
cm = CacheManager(wc, capacity=cap, pyramid_delta=delta, embedding_seed=emb_seed)
rh = ref.lib.ref_cache_new_ivf(cap, 0.9, 1.0, 0.3, delta, emb_seed, ivf[0], ivf[1],
                                        ivf[3], ivf[2])
rng = np.random.default_rng(seed)
centres = ref.random_unit_vectors(seed + 100, 6, dim)
now = 0.0
tmp = tempfile.mkdtemp()


def ref_ids():
    buf = np.zeros(4096, np.uint64)
    n = ref.lib.ref_cache_ids(rh, buf, 4096)
    return sorted(buf[:n].tolist())


for op in range(200):
    now += float(rng.uniform(0.0, 0.25))
    ids = ref_ids()
    r = rng.random()
    kind = ""
    if r < 0.45 or not ids:
        emb = ref.perturb(centres[op % 6], float(rng.uniform(0.1, 0.6)), 7000 + op)
        dur = float(rng.uniform(4.0, 12.0))
        q = float(rng.uniform(0.1, 1.0))
        a = cm.admit(emb, dur, emb, q, now)
        b = ref.lib.ref_cache_admit(rh, emb, dim, dur, q, now)
        kind = f"admit {a} {b}"
    elif r < 0.85:
        eid = int(ids[int(rng.integers(0, len(ids)))])
        steps = int(rng.integers(0, 131))
        dur = float(rng.uniform(2.5, 10.0))
        skip = float(rng.choice([0.0, 0.0, 0.05, 0.3]))
        cm.record_reuse(eid, steps, dur, now, skip)
        ref.lib.ref_cache_record_reuse(rh, eid, steps, dur, now, skip)
        kind = "reuse"
    elif r < 0.95:
        buf = np.zeros(4096, np.uint64)
        n = ref.lib.ref_cache_refinement_candidates(rh, buf, 4096)
        cands = buf[:n].tolist()
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
        kind = f"refine {eid} {bool(got)} {bool(exp)}"
    else:
        out = np.zeros(64, np.uint64)
        nr = ref.lib.ref_cache_evict(rh, now, out, 64)
        ev = cm.evict_if_full(now)
        kind = f"evict {ev} {out[:nr].tolist()}"
    path = os.path.join(tmp, "r.swix")
    nc = ref.lib.ref_cache_index_save(rh, path.encode())
    cent, _, lists = oracle.parse_swix(path)
    info = wc.ivf_info()
    ours = wc.ivf_centroids()
    same = (nc == 0 and info["centroids"] == 0) or (ours.shape == cent.shape and np.array_equal(ours, cent))
    if not same:
        print("DIVERGED after op", op, kind, "ref C", nc, "ours", info, ours.shape)
        print("ref list sizes", [len(x) for x in lists])
        break
else:
    print("no divergence in 200 ops", wc.ivf_info())
