#!/usr/bin/env python3
"""Summaries of ncu output for profiles/ (committed; the raw reports stay in gpurun_out/).

  launches <csv> <out.json>   per-kernel time / DRAM bytes of the LAST train step in a launch
                              list made with
                              ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
                                  dram__bytes_write.sum --clock-control none --csv
                                  python tools/profile_step.py --steps 3
  full <report.ncu-rep> <out.json> [kernel-regex]
                              selected metrics of each kernel in a `--set full` capture
"""
import csv
import json
import re
import subprocess
import sys
from collections import OrderedDict

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "lts__t_sectors_op_red.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
]


def short(name):
    m = re.search(r"(k_\w+)", name)
    return m.group(1) if m else name[:40]


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    per = OrderedDict()
    for r in rows:
        lid, kname, metric, unit, val = int(r[0]), r[4], r[12], r[13], r[14]
        d = per.setdefault(lid, {"kernel": short(kname)})
        d[metric] = float(val.replace(",", ""))
        d[metric + ".unit"] = unit
    ids = list(per)
    # a step starts with the frame reset (k_zero2) when present, else with K1
    first = "k_zero2" if any(per[i]["kernel"] == "k_zero2" for i in ids) else "k_preprocess"
    last_pre = max(i for i in ids if per[i]["kernel"] == first)
    step = [per[i] for i in ids if i >= last_pre]
    agg = OrderedDict()
    for d in step:
        a = agg.setdefault(d["kernel"], {"kernel": d["kernel"], "launches": 0, "time_ns": 0.0,
                                         "dram_read": 0.0, "dram_write": 0.0})
        a["launches"] += 1
        scale = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "nsecond": 1}
        a["time_ns"] += d["gpu__time_duration.sum"] * scale.get(d["gpu__time_duration.sum.unit"], 1)
        a["dram_read"] += d.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += d.get("dram__bytes_write.sum", 0.0)
    total = sum(a["time_ns"] for a in agg.values())
    for a in agg.values():
        a["share"] = a["time_ns"] / total
    json.dump({"source": f"ncu launch list {path} (last train step; cold-cache serialised "
                         "launches: compare SHARES with bench.py's stage times, not absolutes)",
               "step_total_us": total / 1e3, "kernels": list(agg.values())},
              open(out, "w"), indent=1)
    print(json.dumps({k: round(v["share"], 3) for k, v in agg.items()}))


def full(rep, out, regex=None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    txt = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    res = OrderedDict()
    seen = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        k = short(d["Kernel Name"])
        if regex and not re.search(regex, k):
            continue
        # repeated kernels (the sorts' passes) are numbered in launch order: k_onesweep#0, ...
        seen[k] = seen.get(k, -1) + 1
        key = k if seen[k] == 0 else f"{k}#{seen[k]}"
        res[key] = {m: f"{d[m]} {units[h.index(m)]}".strip() for m in FULL_METRICS if m in d}
    json.dump({"source": f"ncu --set full --clock-control none --import-source on, report {rep} "
                         "(not committed)", "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:2000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
