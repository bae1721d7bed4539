"""GPU: the C++ drop-in (include/semwarm_b200.hpp) inside the reference's own code.

* dropin_check: semwarm_b200::IvfIndexT instantiated with the reference's semwarm:: types vs the
  reference's IvfIndex and choose_arm, result for result (tools/dropin/dropin_check.cpp).
* replay: the reference's OWN Pipeline::replay (pipeline.cpp:299-323) on a config-5 workload —
  synth_workload(2000 prompts, 512-d, dup 0.9) against a 1K-capacity cache with the default IVF
  index (64 lists, nprobe 8, rebuild every 1024 mutations), admit / record_reuse / evict /
  refine churn — built twice from the same reference sources: stock, and with CacheManager's
  IvfIndex swapped for GpuIvfIndex plus selector.cpp replaced by the device selector
  (oracle/Makefile `dropin`). Every ServeOutcome, the final cache ledger and the run summary must
  be byte-identical."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
BIN = os.path.join(REF, "dropin_check")


@pytest.mark.parametrize("dim,n", [(128, 800), (512, 1500), (64, 300)])
def test_cpp_dropin_matches_reference(dim, n):
    if not os.path.exists(BIN):
        pytest.skip("dropin_check not built (needs /root/reference at build time)")
    r = subprocess.run([BIN, str(dim), str(n)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout + r.stderr


def test_reference_pipeline_replay_on_gpu_index_is_identical():
    stock, b200 = os.path.join(REF, "replay_stock"), os.path.join(REF, "replay_b200")
    if not (os.path.exists(stock) and os.path.exists(b200)):
        pytest.skip("replay binaries not built (needs /root/reference at build time)")
    cases = [("2000", "512", "1024", "exploit", "7"), ("2000", "512", "1024", "fixed", "7"),
             ("1500", "256", "512", "rule", "11"), ("600", "64", "96", "explore", "3")]
    procs = [subprocess.Popen([stock, *c], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                              text=True) for c in cases]  # the CPU runs overlap the GPU ones
    for c, p in zip(cases, procs):
        g = subprocess.run([b200, *c], capture_output=True, text=True, timeout=900)
        assert g.returncode == 0, g.stderr
        s_out, s_err = p.communicate(timeout=900)
        assert p.returncode == 0, s_err
        assert g.stdout.count("\n") > int(c[0]), c
        if c[3] == "fixed":
            assert '"refinements":0' not in g.stdout, "the fixed-arm case must exercise refine"
        assert '"consistent":true' in g.stdout
        assert g.stdout == s_out, f"replay differs for {c}"
        print(c, "| stock:", s_err.strip().splitlines()[-1], "| b200:", g.stderr.strip().splitlines()[-1])
