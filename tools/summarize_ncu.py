"""Summarise ncu outputs into profiles/ (tracked evidence for the bench numbers).

    python tools/summarize_ncu.py launches <launches.csv> <out.json> [--skip-probe]
    python tools/summarize_ncu.py full <report.ncu-rep> <out.json>

`launches`: per-kernel device time, launch count and share of the step from the
`--metrics gpu__time_duration.sum --clock-control none` launch list (cold-cache,
serialised launches: the SHARE is what compares with bench.py's live breakdown).
`full`: the headline counters of a `--set full` capture per kernel (duration, DRAM bytes,
pipe utilisation, occupancy, registers, issue activity).
"""

from __future__ import annotations

import collections
import csv
import io
import json
import re
import subprocess
import sys


def kname(full: str) -> str:
    m = re.search(r"(k_[a-z0-9_]+|DeviceScan\w*|vectorized_elementwise_kernel|\w+Kernel)", full)
    return m.group(1) if m else full[:40]


def launches(path: str, out: str) -> dict:
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        nm = kname(r[ki])
        if nm.startswith("k_probe") or nm == "vectorized_elementwise_kernel":
            continue  # bench's FP64 probe and L2 flush are not part of the step
        tot[nm] += float(r[vi].replace(",", "")) / 1e6
        cnt[nm] += 1
    s = sum(tot.values())
    res = {"source": path, "unit": "ms (sum over all launches in the capture)",
           "kernels": {k: {"ms": round(v, 4), "launches": cnt[k], "share": round(v / s, 4)}
                       for k, v in tot.most_common()}}
    json.dump(res, open(out, "w"), indent=1)
    return res


FULL_METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cycles_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "smsp__inst_executed.sum": "warp_instructions",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "l1tex__t_bytes.sum": "l1tex_bytes",
    "lts__t_bytes.sum": "l2_bytes",
}


def full(rep: str, out: str) -> dict:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {"source": rep, "kernels": []}
    for vals in rows[2:]:
        rec = {"kernel": kname(vals[hdr.index("Kernel Name")])}
        for m, key in FULL_METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                v = vals[i].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                rec[key] = {"value": v, "unit": units[i]} if units[i] else v
        res["kernels"].append(rec)
    json.dump(res, open(out, "w"), indent=1)
    return res


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    r = launches(src, dst) if mode == "launches" else full(src, dst)
    print(json.dumps(r, indent=1)[:3000])
