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
