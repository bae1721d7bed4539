import sys, time, numpy as np, torch
sys.path.insert(0, '.')
from paper_2603_07865_b200.warmstart import WarmStartCache, SelectorConfig, Policy, requests
from paper_2603_07865_b200.synth import normalize_rows, trained_like_gater
n = int(sys.argv[1]); B = int(sys.argv[2])
wc = WarmStartCache(512, rows_per_entry=1, max_entries=n, latent_shape=(8,256,16), max_batch=1024, latent_slots=min(65536, n))
neg = normalize_rows(np.random.default_rng(4242).standard_normal((1, 512)))[0]
th, ps = trained_like_gater(); wc.set_negative(neg); wc.set_gater(th, ps, 1.0)
wc.fill_synthetic(n, first_id=1, seed=1, delta=1.0)
q = normalize_rows(np.random.default_rng(3).standard_normal((B, 512)))
r = requests(np.arange(1, B+1, dtype=np.uint64), np.full(B, 5.0), np.full(B, 200, np.int32))
for i in range(3):
    t = time.time(); buf = wc.plan(q, r, sel=SelectorConfig(8), policy=Policy("exploit")); torch.cuda.synchronize(); print(n, B, i, time.time()-t, wc.launch_info(), flush=True)
