"""GPU: the in-library shard group (sw_group_*, csrc/host/group.cpp) — the C++ caller's sharded
path of config 4 — must reproduce the single-context warm start exactly: choices on every shard,
and each shard's owner-computed latents. On one B200 the shards share device 0 (peer-copy
transport); the NCCL transport runs at one shard per device (a 1-rank communicator here)."""
import numpy as np
import pytest

from paper_2603_07865_b200.synth import (SynthCache, perturbed_queries, request_durations,
                                         trained_like_gater)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

FIELDS = ["hit", "arm", "steps_skipped", "n_hits", "entry_id", "level", "start_s", "length_s",
          "similarity", "pick", "t_out", "flags"]


def _setup(n_entries, dim, seed):
    c = SynthCache(n_entries, dim, 0.25, seed=seed, clustered=True)
    rng = np.random.default_rng(seed)
    lats = [rng.standard_normal((8, int(np.floor(d * 25 + 0.5)), 16)).astype(np.float32)
            for d in c.durations]
    neg = (lambda v: (v / np.linalg.norm(v)).astype(np.float32))(rng.standard_normal(dim))
    return c, lats, neg


@pytest.mark.parametrize("n_shards,transport,tc", [(2, "copy", True), (3, "copy", False),
                                                    (4, "copy", True), (1, "nccl", True)])
def test_group_equals_single_context(n_shards, transport, tc):
    from paper_2603_07865_b200.warmstart import (Policy, SelectorConfig, ShardGroup,
                                                 WarmStartCache, requests)
    B, k, dim = 128, 8, 64
    c, lats, neg = _setup(900, dim, 41 + n_shards)
    th, ps = trained_like_gater()
    full = WarmStartCache(dim, rows_per_entry=7, max_entries=len(c.ids), max_batch=B,
                          exact_only=not tc, tc_always=tc)
    full.set_negative(neg)
    full.set_gater(th, ps, 1.0)
    g = ShardGroup(dim, n_shards, devices=[0] * n_shards, transport=transport, rows_per_entry=7,
                   max_entries=len(c.ids), max_batch=B, exact_only=not tc, tc_always=tc)
    assert g.transport == transport
    g.set_negative(neg)
    g.set_gater(th, ps, 1.0)
    for e, eid in enumerate(c.ids):
        sl = slice(c.off[e], c.off[e + 1])
        args = (int(eid), c.rows[sl], c.levels[sl], c.starts[sl], c.lengths[sl])
        full.insert(*args, latent=lats[e])
        g.insert(*args, latent=lats[e])
    counts = [g.shard(s).entry_count() for s in range(n_shards)]
    assert sum(counts) == len(c.ids)
    assert all(g.shard(s).contains(int(i)) for s in range(n_shards) for i in c.ids[:50]
               if g.owner(int(i)) == s)

    q = perturbed_queries(c, B, frac_random=0.2, seed=7)
    reqs = requests(np.arange(1, B + 1, dtype=np.uint64), request_durations(B),
                    np.full(B, 200, np.int32))
    sel, pol = SelectorConfig(k), Policy("exploit")
    ref_buf = full.plan(q, reqs, seed=5, sel=sel, policy=pol)
    ref = full.choices(ref_buf)
    out_ref = full.align_noise(ref_buf, reqs, 256, philox_seed=9).cpu().numpy()

    dev = torch.device("cuda:0")
    outs = [torch.zeros((B, 8, 256, 16), dtype=torch.float32, device=dev)
            for _ in range(n_shards)]
    got = g.warmstart_host(q, reqs, seed=5, sel=sel, policy=pol, philox_seed=9, outs=outs,
                           t_out_max=256)
    for f in FIELDS:
        np.testing.assert_array_equal(got[f], ref[f], err_msg=f)
    hit = got["hit"].astype(bool)
    assert hit.sum() > B // 4
    assert (got["owner"][hit] == np.array([g.owner(int(i)) for i in got["entry_id"][hit]])).all()
    for s in range(n_shards):  # the replicated merge gives the same choices on every shard
        np.testing.assert_array_equal(g.shard_choices(s, B)["entry_id"], ref["entry_id"])
    # owner-computes latents: shard s holds exactly the requests whose entry it owns
    for s in range(n_shards):
        o = outs[s].cpu().numpy()
        mine = hit & (got["owner"] == s)
        np.testing.assert_array_equal(o[mine], out_ref[mine])
        assert not o[~mine].any()
    g.close()


def test_group_removal_and_second_batch():
    """Mutations routed to the owner shard (remove) are seen by the next group batch."""
    from paper_2603_07865_b200.warmstart import (Policy, SelectorConfig, ShardGroup,
                                                 WarmStartCache, requests)
    B, k, dim = 64, 4, 64
    c, lats, neg = _setup(400, dim, 77)
    full = WarmStartCache(dim, rows_per_entry=7, max_entries=len(c.ids), max_batch=B,
                          tc_always=True)
    g = ShardGroup(dim, 2, devices=[0, 0], transport="copy", rows_per_entry=7,
                   max_entries=len(c.ids), max_batch=B, tc_always=True)
    for x in (full, g):
        x.set_negative(neg)
    for e, eid in enumerate(c.ids):
        sl = slice(c.off[e], c.off[e + 1])
        args = (int(eid), c.rows[sl], c.levels[sl], c.starts[sl], c.lengths[sl])
        full.insert(*args, latent=lats[e])
        g.insert(*args, latent=lats[e])
    q = perturbed_queries(c, B, frac_random=0.0, seed=3)
    reqs = requests(np.arange(1, B + 1, dtype=np.uint64), request_durations(B),
                    np.full(B, 100, np.int32))
    sel, pol = SelectorConfig(k), Policy("fixed", fixed_arm=5)
    first = g.warmstart_host(q, reqs, seed=2, sel=sel, policy=pol)
    gone = np.unique(first["entry_id"][first["hit"].astype(bool)])[:10]
    for i in gone:
        assert full.remove(int(i)) and g.remove(int(i))
    second = g.warmstart_host(q, reqs, seed=2, sel=sel, policy=pol)
    ref = full.choices(full.plan(q, reqs, seed=2, sel=sel, policy=pol))
    for f in FIELDS:
        np.testing.assert_array_equal(second[f], ref[f], err_msg=f)
    assert not np.isin(second["entry_id"][second["hit"].astype(bool)], gone).any()
