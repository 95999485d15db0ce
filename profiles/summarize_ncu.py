"""Summarise ncu artefacts brought back from the GPU box into profiles/.

    python profiles/summarize_ncu.py launches <launches.csv> <out.json>
        per-kernel device time of one training step (the launch list of
        `ncu --metrics gpu__time_duration.sum --clock-control none`; cold-cache
        and serialised -> compare shares, not absolutes)
    python profiles/summarize_ncu.py full <report.ncu-rep> <out.json>
        key counters of every captured kernel from a `--set full` capture:
        duration, DRAM bytes (traffic), SM/memory throughput, IPC, issue
        slots, occupancy, registers, executed instructions, top stall reasons
    python profiles/summarize_ncu.py traffic <full1.json,full2.json,...> <out.json>
        per kernel (first launch): DRAM bytes, duration and executed warp
        instructions -- the table bench.py reads for `roofline.traffic` and
        `roofline.issue`
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys


def _short(name: str) -> str:
    n = name.replace("void ", "")
    for p in ("bs::(anonymous namespace)::", "bs::<unnamed>::", "(anonymous namespace)::", "unnamed>::"):
        n = n.replace(p, "")
    depth, cut = 0, len(n)  # drop the parameter list (the first '(' outside template brackets)
    for i, ch in enumerate(n):
        depth += ch == "<"
        depth -= ch == ">"
        if ch == "(" and depth == 0:
            cut = i
            break
    return n[:cut]


def launches(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    data = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
    starts = [i for i, (k, _) in enumerate(data) if "cull_kernel" in k]
    s, e = starts[-2], starts[-1]  # the last complete training step
    agg = collections.OrderedDict()
    for k, v in data[s:e]:
        agg[_short(k)] = agg.get(_short(k), 0.0) + v / 1e3
    total = sum(agg.values())
    return {"step_kernel_us": round(total, 1),
            "kernels": {k: {"us": round(v, 1), "share": round(v / total, 4)} for k, v in agg.items()}}


METRICS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "smsp__inst_executed.sum": "warp_instructions",
    "lts__t_bytes.sum": "l2_bytes",
}


def full(path: str) -> dict:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9, "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9}
    out = {}
    for r in rows[2:]:
        name = _short(r[hdr.index("Kernel Name")])
        rec = {}
        for m, key in METRICS.items():
            if m in hdr:
                j = hdr.index(m)
                try:
                    rec[key] = float(r[j].replace(",", "")) * scale.get(units[j], 1.0)
                except ValueError:
                    pass
        stalls = {h.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[hdr.index(h)].replace(",", ""))
                  for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")
                  and r[hdr.index(h)].replace(",", "").replace(".", "", 1).isdigit()}
        tot = sum(stalls.values()) or 1.0
        rec["top_stalls"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        if "dram_read_bytes" in rec and "dram_write_bytes" in rec:
            rec["dram_traffic_bytes"] = rec["dram_read_bytes"] + rec["dram_write_bytes"]
        out.setdefault(name, []).append(rec)
    return out


def traffic(paths: str) -> dict:
    out = {}
    for p in paths.split(","):
        table = json.load(open(p))
        for name, recs in table.items():
            if name in out or not recs:
                continue
            r = recs[0]
            out[name] = {"dram_traffic_bytes": r.get("dram_traffic_bytes"), "duration_ns": r.get("duration_ns"),
                         "warp_instructions": r.get("warp_instructions"), "capture": p.split("/")[-1]}
    return out


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    res = launches(src) if mode == "launches" else (traffic(src) if mode == "traffic" else full(src))
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])
