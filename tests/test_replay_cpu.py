"""CPU: the config-5 trace tooling against the unmodified reference.

* swr_synth_workload (our restatement of synth_workload, simgen.cpp:162-194) produces the
  reference's trace bit for bit (prompts, durations, arrivals, step budgets).
* The reference-side batched replay harness (oracle/ref_harness.cpp ref_replay) with batch = 1
  equals the reference's own Pipeline::replay outcome for outcome — so its batch = 64 runs are a
  faithful oracle for the device replay's batched lookups (tests/test_gpu_replay.py)."""
import numpy as np
import pytest

from paper_2603_07865_b200.synth import trained_like_gater
from paper_2603_07865_b200.warmstart import synth_workload


@pytest.mark.parametrize("n,dim,seed", [(300, 64, 7), (120, 512, 3), (50, 33, 11)])
def test_synth_workload_matches_reference(ref, n, dim, seed):
    ours = synth_workload(n, dim, seed)
    theirs = ref.synth_workload(n, dim, seed)
    for a, b in zip(ours, theirs):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("policy", ["exploit", "fixed", "rule", "explore"])
def test_batched_replay_harness_batch1_is_pipeline_replay(ref, policy):
    p, d, a, t = ref.synth_workload(300, 64, 7)
    th, ps = trained_like_gater()
    o0, s0, _ = ref.replay(p, d, a, t, capacity=96, policy=policy, theta=th, psi=ps, fixed_arm=1,
                           batch=0)
    o1, s1, _ = ref.replay(p, d, a, t, capacity=96, policy=policy, theta=th, psi=ps, fixed_arm=1,
                           batch=1)
    assert o0.tobytes() == o1.tobytes()
    assert s0 == s1
    assert s0["hit_rate"] > 0.5
