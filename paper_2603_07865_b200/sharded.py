"""Entry-sharded warm start over N GPUs of one box.

Every rank owns a disjoint set of cache entries (all pyramid rows of an entry stay together).
One batch step:
  1. sw_local_topk: tcgen05 pre-filter + exact fp64 rescoring on the rank's shard -> B x k
     128-byte HitRec records (exact sim, id, segment, s_neg, gater block sums, owner rank).
  2. all_gather of the records and counts over NCCL (world x B x k x 128 B; 1 MiB per rank at
     B=1024, k=8) — the only data-path collective.
  3. sw_merge_select on every rank: deterministic (sim desc, id asc) merge of the world sorted
     lists (the global top-k is contained in the union of the per-shard exact top-ks), then the
     replicated gate / select / Skip Gater / t* — identical on all ranks, no broadcast.
  4. sw_align_noise_owned: each rank aligns + noises only the requests whose chosen entry it
     owns (owner-computes; the latent lives there).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import CHOICE_DTYPE, HIT_RECORD_BYTES, check

# HitRec layout (csrc/sw_internal.cuh), for host-side inspection and the CPU protocol tests
HITREC_DTYPE = np.dtype([("sim", "<f8"), ("entry_id", "<u8"), ("level", "<i4"), ("slot", "<i4"),
                         ("start_s", "<f8"), ("length_s", "<f8"), ("s_neg", "<f8"),
                         ("phi", "<f8", (8,)), ("row", "<i4"), ("owner", "<i4"), ("pad", "<u8")])
assert HITREC_DTYPE.itemsize == HIT_RECORD_BYTES


def owner_of(entry_id: int, world: int) -> int:
    """Default placement: entry id modulo world size (all rows of an entry together)."""
    return int(entry_id) % world


def merge_topk(sims: np.ndarray, ids: np.ndarray, counts: np.ndarray, k: int):
    """Reference merge rule used by k_merge: world sorted lists -> global top-k by
    (sim desc, id asc). sims/ids: [world, k]; counts: [world]. Returns (sims, ids, src rank)."""
    heads = [0] * sims.shape[0]
    out = []
    for _ in range(k):
        best = None
        for r in range(sims.shape[0]):
            if heads[r] >= counts[r]:
                continue
            cand = (sims[r, heads[r]], ids[r, heads[r]], r)
            if best is None or cand[0] > best[0] or (cand[0] == best[0] and cand[1] < best[1]):
                best = cand
        if best is None:
            break
        out.append(best)
        heads[best[2]] += 1
    return out


class ShardedStep:
    """One rank's side of the sharded warm-start step (device buffers preallocated)."""

    def __init__(self, cache, rank: int, world: int, batch: int, k: int, group=None):
        import torch
        self.cache, self.rank, self.world, self.B, self.k = cache, rank, world, batch, k
        self.group = group
        dev = torch.device(f"cuda:{cache.device}")
        self.rec = torch.empty(batch * k * HIT_RECORD_BYTES, dtype=torch.uint8, device=dev)
        self.n = torch.empty(batch, dtype=torch.int32, device=dev)
        self.rec_all = torch.empty(world * batch * k * HIT_RECORD_BYTES, dtype=torch.uint8,
                                   device=dev)
        self.n_all = torch.empty(world * batch, dtype=torch.int32, device=dev)
        self.choices = torch.empty(batch * CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)

    def local_topk(self, q, stream):
        check(_lib.lib().sw_local_topk(self.cache._h, q.data_ptr(), self.B, self.k, self.rank,
                                       self.rec.data_ptr(), self.n.data_ptr(), stream),
              "sw_local_topk")

    def gather(self, stream_obj):
        import torch
        import torch.distributed as dist
        with torch.cuda.stream(stream_obj):
            dist.all_gather_into_tensor(self.rec_all, self.rec, group=self.group)
            dist.all_gather_into_tensor(self.n_all, self.n, group=self.group)

    def merge_select(self, q, reqs, seed, sel, pol, stream):
        check(_lib.lib().sw_merge_select(self.cache._h, self.rec_all.data_ptr(),
                                         self.n_all.data_ptr(), self.world, q.data_ptr(),
                                         reqs.data_ptr(), self.B, self.k, seed, C.byref(sel.c()),
                                         C.byref(pol.c()), self.choices.data_ptr(), stream),
              "sw_merge_select")

    def align_owned(self, reqs, out, t_out_max, philox_seed, stream):
        check(_lib.lib().sw_align_noise_owned(self.cache._h, self.choices.data_ptr(),
                                              reqs.data_ptr(), self.B, self.rank, None,
                                              philox_seed, out.data_ptr(), t_out_max, stream),
              "sw_align_noise_owned")
