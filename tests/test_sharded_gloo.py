"""CPU, world_size 2 over gloo: the entry-sharded protocol. Each rank searches only the entries
it owns (owner = id mod world), all-gathers its exact top-k records, and merges them with the
deterministic (sim desc, id asc) rule — the merged list must equal the unsharded top-k."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2603_07865_b200.sharded import merge_topk, owner_of
from paper_2603_07865_b200.synth import SynthCache, perturbed_queries


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard(c, rank, world):
    keep = np.array([owner_of(i, world) == rank for i in c.ids])
    idx = np.flatnonzero(keep)
    offs = np.concatenate([[0], np.cumsum(c.off[idx + 1] - c.off[idx])])
    rows = np.concatenate([c.entry_rows(e) for e in idx])
    sl = lambda a: np.concatenate([a[c.off[e]:c.off[e + 1]] for e in idx])
    return oracle.Arena(c.ids[idx], offs, rows, sl(c.levels), sl(c.starts), sl(c.lengths))


def _worker(rank, world, port, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = oracle.Oracle()
    c = SynthCache(300, 64, 0.25, seed=17, clustered=True)
    q = perturbed_queries(c, 24, frac_random=0.2)
    k = 8
    ar = _shard(c, rank, world)
    sims = np.full((q.shape[0], k), -np.inf)
    ids = np.zeros((q.shape[0], k), np.int64)
    cnt = np.zeros(q.shape[0], np.int64)
    for i in range(q.shape[0]):
        h = orc.search(ar, q[i], k)
        cnt[i] = len(h)
        sims[i, :len(h)] = h["similarity"]
        ids[i, :len(h)] = h["entry_id"].astype(np.int64)
    parts = [torch.zeros_like(torch.from_numpy(sims)) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(sims))
    pids = [torch.zeros_like(torch.from_numpy(ids)) for _ in range(world)]
    dist.all_gather(pids, torch.from_numpy(ids))
    pcnt = [torch.zeros_like(torch.from_numpy(cnt)) for _ in range(world)]
    dist.all_gather(pcnt, torch.from_numpy(cnt))
    full = oracle.Arena(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    ok = True
    for i in range(q.shape[0]):
        merged = merge_topk(np.stack([p[i].numpy() for p in parts]),
                            np.stack([p[i].numpy() for p in pids]),
                            np.array([p[i].item() for p in pcnt]), k)
        g = orc.search(full, q[i], k)
        ok &= [m[1] for m in merged] == g["entry_id"].astype(np.int64).tolist()
        ok &= [m[0] for m in merged] == g["similarity"].tolist()
        ok &= all(owner_of(m[1], world) == m[2] for m in merged)
    ret[rank] = bool(ok)
    dist.destroy_process_group()


def test_sharded_merge_equals_global_topk():
    world = 2
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), ret), nprocs=world, join=True)
    assert ret[0] and ret[1]


def test_merge_rule_ties_by_id():
    sims = np.array([[0.9, 0.5, 0.5], [0.9, 0.5, 0.1]])
    ids = np.array([[7, 3, 9], [2, 4, 8]])
    m = merge_topk(sims, ids, np.array([3, 3]), 5)
    assert [x[1] for x in m] == [2, 7, 3, 4, 9]
