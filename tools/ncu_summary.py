#!/usr/bin/env python
"""Summarise ncu captures into the JSON committed under profiles/.

  python tools/ncu_summary.py OUT.json REPORT.ncu-rep [REPORT2.ncu-rep ...]

Per kernel launch in the reports: duration, DRAM bytes read + written (the bench line's
roofline "traffic"), tensor-pipe / issue / SM / L2 / DRAM utilisation, grid, registers and smem.
Runs where ncu is installed (here and on the GPU box); bench.py reads the "traffic" field of
profiles/ncu_latest.json for its roofline line.
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
    "launch__cluster_dim_x": "cluster_x",
    "sm__cycles_elapsed.avg": "sm_cycles",
}
SCALE = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "nsecond": 1e-9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KByte": 1e3,
         "MByte": 1e6, "GByte": 1e9, "Kibyte": 1024, "KiB": 1024}


def summarise(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        name = r[hdr.index("Kernel Name")]
        short = re.sub(r"\(.*", "", name).replace("void ", "").split("::")[-1]
        d = {"kernel": short, "report": rep.split("/")[-1]}
        for m, key in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i].split("/")[0]
            if u in SCALE:
                v *= SCALE[u]
                if key == "duration":
                    key = "duration_s"
                elif key in ("dram_read", "dram_write", "l2_to_sm", "dyn_smem"):
                    key += "_bytes"
            d[key] = v
        if "dram_read_bytes" in d and "dram_write_bytes" in d:
            d["traffic_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        res.append(d)
    return res


def main():
    out = sys.argv[1]
    allk = []
    for rep in sys.argv[2:]:
        allk += summarise(rep)
    traffic = {}
    for d in allk:
        if "traffic_bytes" in d:
            traffic.setdefault(d["kernel"], d["traffic_bytes"])
    with open(out, "w") as f:
        json.dump({"launches": allk, "traffic_bytes": traffic}, f, indent=1)
    print(json.dumps(traffic))


if __name__ == "__main__":
    main()
