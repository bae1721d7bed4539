"""GPU: the pipelined host path (sw_warmstart_host_submit / _wait). Batches submitted back to
back — batch n+1's H2D overlapping batch n's kernels — give exactly the choices and noised
latents of one synchronous sw_warmstart_host call per batch."""
import numpy as np
import pytest

from paper_2603_07865_b200.synth import SynthCache, perturbed_queries, request_durations

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_pipelined_host_path_matches_synchronous():
    from paper_2603_07865_b200.warmstart import (CHOICE_DTYPE, Policy, SelectorConfig,
                                                 WarmStartCache, requests)
    c = SynthCache(20000, 256, 1.0, seed=71, clustered=True)
    latent = (4, 64, 16)
    wc = WarmStartCache(256, rows_per_entry=1, max_entries=20000, max_batch=512,
                        latent_shape=latent, latent_slots=4096)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    sel, pol = SelectorConfig(8), Policy("exploit")
    nb, B, T = 5, 384, 64
    qs, rqs = [], []
    for j in range(nb):
        qs.append(np.ascontiguousarray(perturbed_queries(c, B, frac_random=0.1, seed=100 + j)))
        ids = np.arange(1 + j * B, 1 + (j + 1) * B, dtype=np.uint64)
        rqs.append(requests(ids, request_durations(B, 4.0, 10.0, seed=200 + j),
                            np.full(B, 100, np.int32)))
    dev = torch.device("cuda", 0)
    ref_ch, ref_lat = [], []
    for j in range(nb):
        out = torch.zeros((B, latent[0], T, latent[2]), dtype=torch.float32, device=dev)
        ref_ch.append(wc.warmstart_host(qs[j], rqs[j], out, T, seed=9, sel=sel, policy=pol,
                                        philox_seed=4321))
        ref_lat.append(out.cpu().numpy())
    got_ch = [np.zeros(B, CHOICE_DTYPE) for _ in range(nb)]
    outs = [torch.zeros((B, latent[0], T, latent[2]), dtype=torch.float32, device=dev)
            for _ in range(nb)]
    tickets = []
    for j in range(nb):
        tickets.append(wc.warmstart_host_submit(qs[j], rqs[j], got_ch[j], outs[j], T, seed=9,
                                                sel=sel, policy=pol, philox_seed=4321))
        if j >= 1:
            wc.warmstart_host_wait(tickets[j - 1])
    wc.warmstart_host_wait(tickets[-1])
    torch.cuda.synchronize(dev)
    assert tickets == sorted(tickets) and len(set(tickets)) == nb
    for j in range(nb):
        assert ref_ch[j]["hit"].any()
        for f in ref_ch[j].dtype.names:
            np.testing.assert_array_equal(got_ch[j][f], ref_ch[j][f], err_msg=f"batch {j} {f}")
        np.testing.assert_array_equal(outs[j].cpu().numpy(), ref_lat[j])


def test_pipelined_wait_rejects_unknown_ticket():
    from paper_2603_07865_b200.warmstart import WarmStartCache
    wc = WarmStartCache(64, rows_per_entry=1, max_entries=64, max_batch=8)
    with pytest.raises(ValueError):
        wc.warmstart_host_wait(5)


def _async_case(ivf=False):
    from paper_2603_07865_b200 import _lib
    from paper_2603_07865_b200.warmstart import (Policy, SelectorConfig, WarmStartCache, requests)
    c = SynthCache(30000, 256, 1.0, seed=73, clustered=True)
    latent = (4, 64, 16)
    wc = WarmStartCache(256, rows_per_entry=1, max_entries=30000, max_batch=512,
                        latent_shape=latent, latent_slots=4096)
    if ivf:  # configured on the empty arena (IvfIndex::build({}, ...)), rebuilt after inserts
        wc.ivf_configure(16, 4, 1 << 30, seed=3)
    wc.insert_batch(c.ids, c.off, c.rows, c.levels, c.starts, c.lengths)
    if ivf:
        wc.ivf_rebuild()
    sel, pol = SelectorConfig(8), Policy("exploit")
    dev = torch.device("cuda", 0)
    nb, B, T = 6, 512, 64
    qs, rqs = [], []
    for j in range(nb):
        qs.append(torch.from_numpy(perturbed_queries(c, B, frac_random=0.1, seed=300 + j)).to(dev))
        ids = np.arange(1 + j * B, 1 + (j + 1) * B, dtype=np.uint64)
        rq = requests(ids, request_durations(B, 4.0, 10.0, seed=400 + j), np.full(B, 100, np.int32))
        rqs.append(torch.from_numpy(rq.view(np.uint8)).to(dev))
    return c, wc, sel, pol, dev, nb, B, T, latent, qs, rqs, _lib


@pytest.mark.parametrize("ivf,two_streams", [(False, False), (True, False), (False, True)])
def test_warmstart_async_matches_sync(ivf, two_streams):
    """sw_warmstart_async (prep + scoring on the caller's stream, finish + align + noise on the
    context's stream under the next batch's scoring, alternating scratch parities) returns
    exactly sw_warmstart's choices and latents; a synchronous search after it sees the whole
    pipeline finished (scratch ordering)."""
    import ctypes as C
    c, wc, sel, pol, dev, nb, B, T, latent, qs, rqs, _lib = _async_case(ivf)
    L = _lib.lib()
    st = torch.cuda.current_stream(dev).cuda_stream
    ref_ch, ref_lat = [], []
    for j in range(nb):
        ch = torch.zeros(B * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
        out = torch.zeros((B, latent[0], T, latent[2]), dtype=torch.float32, device=dev)
        _lib.check(L.sw_warmstart(wc._h, qs[j].data_ptr(), rqs[j].data_ptr(), B, 9,
                                  C.byref(sel.c()), C.byref(pol.c()), None, 4321, ch.data_ptr(),
                                  out.data_ptr(), T, st), "sw_warmstart")
        ref_ch.append(ch.cpu().numpy().view(_lib.CHOICE_DTYPE))
        ref_lat.append(out.cpu().numpy())
    chs = [torch.zeros(B * _lib.CHOICE_DTYPE.itemsize, dtype=torch.uint8, device=dev)
           for _ in range(nb)]
    outs = [torch.zeros((B, latent[0], T, latent[2]), dtype=torch.float32, device=dev)
            for _ in range(nb)]
    side = torch.cuda.Stream(dev)
    for j in range(nb):
        sj = side.cuda_stream if (two_streams and j % 2) else st  # callers on two streams
        _lib.check(L.sw_warmstart_async(wc._h, qs[j].data_ptr(), rqs[j].data_ptr(), B, 9,
                                        C.byref(sel.c()), C.byref(pol.c()), None, 4321,
                                        chs[j].data_ptr(), outs[j].data_ptr(), T, sj),
                   "sw_warmstart_async")
    hits_after, n_after = wc.search(qs[0].cpu().numpy(), 8)  # synchronous user after async ones
    _lib.check(L.sw_join(wc._h, st), "sw_join")
    torch.cuda.synchronize(dev)
    for j in range(nb):
        got = chs[j].cpu().numpy().view(_lib.CHOICE_DTYPE)
        assert ref_ch[j]["hit"].any()
        for f in ref_ch[j].dtype.names:
            np.testing.assert_array_equal(got[f], ref_ch[j][f], err_msg=f"batch {j} {f}")
        np.testing.assert_array_equal(outs[j].cpu().numpy(), ref_lat[j])
    hits_ref, n_ref = wc.search(qs[0].cpu().numpy(), 8)
    np.testing.assert_array_equal(n_after, n_ref)
    np.testing.assert_array_equal(hits_after["entry_id"], hits_ref["entry_id"])
