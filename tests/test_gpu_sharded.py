"""GPU: the entry-sharded path on one device — two shard contexts (owner = id mod 2), per-shard
exact top-k records, merge + replicated select, owner-computes align — must reproduce the
unsharded single-context warm start exactly."""
import numpy as np
import pytest

from paper_2603_07865_b200 import _lib
from paper_2603_07865_b200.sharded import HITREC_DTYPE, owner_of
from paper_2603_07865_b200.synth import (SynthCache, perturbed_queries, request_durations,
                                         trained_like_gater)

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("tc,async_topk", [(False, False), (True, False), (True, True)])
def test_two_shards_equal_single_context(tc, async_topk):
    import ctypes as C

    from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, WarmStartCache, requests
    world, B, k, dim = 2, 96, 8, 64
    c = SynthCache(800, dim, 0.25, seed=31, clustered=True)
    rng = np.random.default_rng(3)
    lats = [rng.standard_normal((8, int(np.floor(d * 25 + 0.5)), 16)).astype(np.float32)
            for d in c.durations]
    neg = (lambda v: (v / np.linalg.norm(v)).astype(np.float32))(rng.standard_normal(dim))
    th, ps = trained_like_gater()

    def make(owner):
        wc = WarmStartCache(dim, rows_per_entry=7, max_entries=len(c.ids), max_batch=B,
                            exact_only=not tc, tc_always=tc)
        wc.set_negative(neg)
        wc.set_gater(th, ps, 1.0)
        for e, eid in enumerate(c.ids):
            if owner is None or owner_of(eid, world) == owner:
                sl = slice(c.off[e], c.off[e + 1])
                wc.insert(int(eid), c.rows[sl], c.levels[sl], c.starts[sl], c.lengths[sl],
                          latent=lats[e])
        return wc

    full = make(None)
    shards = [make(r) for r in range(world)]
    q = perturbed_queries(c, B, frac_random=0.2)
    reqs = requests(np.arange(1, B + 1, dtype=np.uint64), request_durations(B),
                    np.full(B, 200, np.int32))
    sel, pol = SelectorConfig(k), Policy("exploit")
    ref_buf = full.plan(q, reqs, seed=5, sel=sel, policy=pol)
    ref = full.choices(ref_buf)

    dev = torch.device("cuda:0")
    qd = torch.from_numpy(q).to(dev)
    rd = torch.from_numpy(reqs.view(np.uint8)).to(dev)
    st = torch.cuda.current_stream().cuda_stream
    recs, cnts = [], []
    for r, wc in enumerate(shards):
        rec = torch.empty(B * k * 128, dtype=torch.uint8, device=dev)
        n = torch.empty(B, dtype=torch.int32, device=dev)
        if async_topk:  # finish + record copies on the shard's own stream, joined back
            _lib.check(_lib.lib().sw_local_topk_async(wc._h, qd.data_ptr(), B, k, r,
                                                      rec.data_ptr(), n.data_ptr(), st),
                       "local_topk_async")
            _lib.check(_lib.lib().sw_join(wc._h, st), "join")
        else:
            _lib.check(_lib.lib().sw_local_topk(wc._h, qd.data_ptr(), B, k, r, rec.data_ptr(),
                                                n.data_ptr(), st), "local_topk")
        recs.append(rec)
        cnts.append(n)
    rec_all = torch.cat(recs)
    n_all = torch.cat(cnts)
    got_buf = torch.empty(B * 88, dtype=torch.uint8, device=dev)
    _lib.check(_lib.lib().sw_merge_select(shards[0]._h, rec_all.data_ptr(), n_all.data_ptr(),
                                          world, qd.data_ptr(), rd.data_ptr(), B, k, 5,
                                          C.byref(sel.c()), C.byref(pol.c()), got_buf.data_ptr(),
                                          st), "merge_select")
    got = shards[0].choices(got_buf)
    for f in ["hit", "arm", "steps_skipped", "n_hits", "entry_id", "level", "start_s",
              "length_s", "similarity", "pick", "t_out"]:
        np.testing.assert_array_equal(got[f], ref[f], err_msg=f)
    hit = got["hit"].astype(bool)
    assert (got["owner"][hit] == np.array([owner_of(i, world) for i in got["entry_id"][hit]])).all()
    recs_np = rec_all.cpu().numpy().view(HITREC_DTYPE).reshape(world, B, k)
    assert (recs_np["owner"][1][cnts[1].cpu().numpy()[:, None] > np.arange(k)] == 1).all()

    # owner-computes align + noise reproduces the single-context pass
    out_ref = full.align_noise(ref_buf, reqs, 256, philox_seed=9).cpu().numpy()
    out = torch.zeros((B, 8, 256, 16), dtype=torch.float32, device=dev)
    for r, wc in enumerate(shards):
        _lib.check(_lib.lib().sw_align_noise_owned(wc._h, got_buf.data_ptr(), rd.data_ptr(), B,
                                                   r, None, 9, out.data_ptr(), 256, st), "owned")
    np.testing.assert_array_equal(out.cpu().numpy(), out_ref)


def test_pipelined_sharded_step_one_rank_equals_warmstart():
    """The bench's pipelined sharded step at world 1: sw_local_topk_async, then the 'gather'
    (a copy), sw_merge_select and sw_align_noise_owned enqueued on the context's async stream
    (sw_async_stream), several batches back to back — equal to sw_warmstart per batch."""
    import ctypes as C

    from paper_2603_07865_b200.warmstart import Policy, SelectorConfig, WarmStartCache, requests
    B, k, dim, T = 256, 8, 128, 64
    c = SynthCache(20000, dim, 1.0, seed=35, clustered=True)
    wc = WarmStartCache(dim, rows_per_entry=1, max_entries=20000, max_batch=B,
                        latent_shape=(4, 64, 16), latent_slots=4096, tc_always=True)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    sel, pol = SelectorConfig(k), Policy("exploit")
    L = _lib.lib()
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream(dev).cuda_stream
    a_ptr = C.c_void_p()
    _lib.check(L.sw_async_stream(wc._h, C.byref(a_ptr)), "sw_async_stream")
    a_stream = torch.cuda.ExternalStream(a_ptr.value, device=dev)
    nb = 4
    qs, rqs, ref_ch, ref_lat = [], [], [], []
    for j in range(nb):
        q = torch.from_numpy(perturbed_queries(c, B, frac_random=0.1, seed=50 + j)).to(dev)
        rq = requests(np.arange(1 + j * B, 1 + (j + 1) * B, dtype=np.uint64),
                      request_durations(B, 4.0, 10.0, seed=60 + j), np.full(B, 100, np.int32))
        rqd = torch.from_numpy(rq.view(np.uint8)).to(dev)
        qs.append(q)
        rqs.append(rqd)
        ch = torch.zeros(B * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        out = torch.zeros((B, 4, T, 16), dtype=torch.float32, device=dev)
        _lib.check(L.sw_warmstart(wc._h, q.data_ptr(), rqd.data_ptr(), B, 1, C.byref(sel.c()),
                                  C.byref(pol.c()), None, 77, ch.data_ptr(), out.data_ptr(), T,
                                  st), "sw_warmstart")
        ref_ch.append(ch.cpu().numpy().view(_lib.CHOICE_DTYPE))
        ref_lat.append(out.cpu().numpy())
    rec = torch.empty(B * k * 128, dtype=torch.uint8, device=dev)
    n = torch.empty(B, dtype=torch.int32, device=dev)
    rec_all, n_all = torch.empty_like(rec), torch.empty_like(n)
    chs = [torch.zeros(B * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
           for _ in range(nb)]
    outs = [torch.zeros((B, 4, T, 16), dtype=torch.float32, device=dev) for _ in range(nb)]
    for j in range(nb):
        _lib.check(L.sw_local_topk_async(wc._h, qs[j].data_ptr(), B, k, 0, rec.data_ptr(),
                                         n.data_ptr(), st), "sw_local_topk_async")
        with torch.cuda.stream(a_stream):
            rec_all.copy_(rec)
            n_all.copy_(n)
        _lib.check(L.sw_merge_select(wc._h, rec_all.data_ptr(), n_all.data_ptr(), 1,
                                     qs[j].data_ptr(), rqs[j].data_ptr(), B, k, 1,
                                     C.byref(sel.c()), C.byref(pol.c()), chs[j].data_ptr(),
                                     a_ptr), "sw_merge_select")
        _lib.check(L.sw_align_noise_owned(wc._h, chs[j].data_ptr(), rqs[j].data_ptr(), B, 0,
                                          None, 77, outs[j].data_ptr(), T, a_ptr), "align")
    _lib.check(L.sw_join(wc._h, st), "sw_join")
    torch.cuda.synchronize(dev)
    for j in range(nb):
        got = chs[j].cpu().numpy().view(_lib.CHOICE_DTYPE)
        assert ref_ch[j]["hit"].any()
        for f in ("hit", "arm", "steps_skipped", "entry_id", "similarity"):
            np.testing.assert_array_equal(got[f], ref_ch[j][f], err_msg=f"batch {j} {f}")
        np.testing.assert_array_equal(outs[j].cpu().numpy(), ref_lat[j])
