"""GPU: BASELINE config 5 — the Cache Manager trace replay with batched lookups on the device
(swr_replay: sw_plan over 64 requests at a time against the arena, then admit / record_reuse /
evict / refine per request through the host Cache Manager policy and the arena), checked
outcome for outcome against the unmodified reference:

* batch = 1 against the reference's own Pipeline::replay (pipeline.cpp:299-323);
* batch = 64 against the reference-side batched replay (oracle ref_replay, which itself equals
  Pipeline::replay at batch = 1, tests/test_replay_cpu.py).

Workload: synth_workload(2000 prompts, 512-d, near-duplicate rate 0.9) at the reference
defaults — 1K capacity, IVF 64 lists / nprobe 8 / rebuild every 1024 mutations, pyramid delta
1/4 (7 rows per entry)."""
import numpy as np
import pytest

from paper_2603_07865_b200.synth import trained_like_gater
from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, TraceReplay, synth_workload

pytestmark = pytest.mark.gpu

FIELDS = ["request_id", "cache_hit", "arm_index", "steps_skipped", "fallback", "entry_id",
          "admitted_entry_id", "quality", "nfe_cost_s", "sim_latency_s", "skip_fraction",
          "reference_similarity"]


def _check(ours, theirs, st, summ):
    for f in FIELDS:
        np.testing.assert_array_equal(ours[f], theirs[f], err_msg=f)
    for k in ("total_nfe_s", "baseline_nfe_s", "speedup", "mean_quality", "mean_reward",
              "hit_rate", "mean_latency_s", "median_latency_s", "p95_latency_s"):
        assert st[k] == summ[k], k
    assert st["refinements"] == summ["refinements"]


@pytest.mark.parametrize("policy,batch", [("exploit", 1), ("exploit", 64), ("fixed", 64),
                                          ("rule", 64), ("explore", 16)])
def test_replay_matches_reference(ref, policy, batch):
    n, dim = 2000, 512
    p, d, a, t = synth_workload(n, dim, 7)
    th, ps = trained_like_gater()
    tr = TraceReplay(dim, capacity=1024, seed=1, policy=Policy(policy, fixed_arm=1),
                     sel=SelectorConfig(8), theta=th, psi=ps, max_batch=64)
    out, st = tr.run(p, d, a, t, batch=batch)
    assert tr.cm.check_consistent()
    tr.close()
    theirs, summ, wall = ref.replay(p, d, a, t, capacity=1024, policy=policy, theta=th, psi=ps,
                                    fixed_arm=1, batch=0 if batch == 1 else batch)
    _check(out, theirs, st, summ)
    assert st["evictions"] > 0 and st["hit_rate"] > 0.5
    if policy == "fixed":
        assert st["refinements"] > 0
    print(f"{policy} b={batch}: ours {st['total_s']:.2f}s ({n / st['total_s']:.0f} req/s; "
          f"lookups {st['lookup_s']:.2f}s, mutations {st['mutation_s']:.2f}s, maintenance "
          f"{st['maintenance_s']:.2f}s) vs reference {wall:.2f}s; evictions {st['evictions']}, "
          f"refinements {st['refinements']}")
