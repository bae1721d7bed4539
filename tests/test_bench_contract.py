"""CPU: the bench.py reference arm keeps the driver's JSON contract — one line with the
reference's own plan flow timed on the host cores (the unmodified reference from oracle/_ref),
cpu_baseline and e2e describing the same run. A tiny cache keeps it to a few seconds."""
import json
import os
import subprocess
import sys

import pytest

from conftest import have_ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not have_ref(), reason="compiled reference (oracle/_ref) not present")
def test_reference_arm_json_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--entries", "2000", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["metric"] == "warm-start requests/s" and d["unit"] == "requests/s"
    assert d["value"] > 0 and d["steps"] == 2 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    e = d["e2e"]
    assert e["value"] == d["value"] and e["h2d_bytes_per_step"] == 0
    assert e["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_ours_arm_json_contract():
    """The default arm on a small cache: every key the driver reads, with the kernel roofline,
    the pipelined e2e (H2D + D2H counted), the launch count and the clock sample."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--entries", "20000",
                          "--steps", "5", "--warmup", "3", "--no-vocoder", "--no-batcher",
                          "--no-cpu-baseline", "--no-latency", "--no-sweep", "--no-replay",
                          "--no-config1", "--no-parity"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 4 * d["steps"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_two_rank_sharded_bench_gloo_validation():
    """bench.py under torchrun with two ranks on one device (gloo host-staged gather — the
    validation mode of the entry-sharded step): rank 0 prints one line for the sharded run, and
    its parity sample checks the merged choices against the oracle over both shards."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29541",
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--dist-backend", "gloo", "--entries", "50000", "--no-vocoder", "--no-batcher",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"] == "entry-sharded x2"
    # the merged choices of the timed batch equal the oracle over the union of both shards
    ps = d["parity_sample"]
    assert ps["shards"] == 2 and ps["match"], ps
