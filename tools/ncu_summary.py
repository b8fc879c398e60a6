"""Summarise ncu captures into profiles/ (committed evidence).

  python tools/ncu_summary.py full <report.ncu-rep | raw.csv> <tag> <key>   -> profiles/ncu_<tag>.json (+ ncu_summary.json[key])
  python tools/ncu_summary.py launches <launches.csv> <tag>       -> profiles/launches_<tag>.json
"""

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "smsp__inst_executed.sum",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "nsecond": 1e-9,
              "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "us": 1e-6, "ns": 1e-9}


def full(rep, tag, key):
    # a report (.ncu-rep) or its `--page raw --csv` export (made on the GPU box)
    out = open(rep).read() if rep.endswith(".csv") else subprocess.run(
        ["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = {"kernel": vals[h.index("Kernel Name")] if "Kernel Name" in h else None}
        for k in KEYS:
            if k in h:
                i = h.index(k)
                v = vals[i].replace(",", "")
                try:
                    v = float(v) * UNIT_SCALE.get(units[i], 1.0)
                    u = "base-SI" if units[i] in UNIT_SCALE else units[i]
                except ValueError:
                    u = units[i]
                d[k] = v
                d[k + ".unit"] = u
        kernels.append(d)
    with open(os.path.join(ROOT, "profiles", f"ncu_{tag}.json"), "w") as f:
        json.dump({"report": os.path.basename(rep), "kernels": kernels}, f, indent=1)
    k0 = kernels[0]
    summ_path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summ = json.load(open(summ_path)) if os.path.exists(summ_path) else {}
    summ[key] = {"tag": tag, "kernel": k0["kernel"], "duration_s": k0.get("gpu__time_duration.sum"),
                 "dram_bytes_per_launch": k0.get("dram__bytes_read.sum", 0) + k0.get("dram__bytes_write.sum", 0),
                 "registers": k0.get("launch__registers_per_thread"),
                 "issue_active_pct": k0.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "fp64_pipe_pct": k0.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
                 "stall_no_instruction": k0.get("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"),
                 "stall_wait": k0.get("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio")}
    with open(summ_path, "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ[key], indent=1))


def launches(path, tag):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = UNIT_SCALE.get(r.get("Metric Unit", "ns"), 1e-9)
        name = r["Kernel Name"].split("(")[0][:120]
        per[name][0] += 1
        per[name][1] += v * scale
    tot = sum(t for _, t in per.values())
    out = sorted(({"kernel": k, "launches": n, "total_s": t, "share": t / tot} for k, (n, t) in per.items()),
                 key=lambda d: -d["total_s"])
    with open(os.path.join(ROOT, "profiles", f"launches_{tag}.json"), "w") as f:
        json.dump({"source": os.path.basename(path), "note": "ncu --metrics gpu__time_duration.sum "
                   "--clock-control none (cold-cache, serialised: compare shares)", "kernels": out}, f, indent=1)
    for d in out[:12]:
        print(f"{d['share']*100:6.2f}%  {d['launches']:5d}  {d['total_s']*1e3:9.3f} ms  {d['kernel']}")


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        launches(sys.argv[2], sys.argv[3])
