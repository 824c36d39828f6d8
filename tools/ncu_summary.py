"""Summarise an ncu report / launch-list CSV into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py full  <report.ncu-rep> <out.json>
    python tools/ncu_summary.py launches <launches.csv> <out.txt>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__occupancy_limit_registers", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__inst_executed.sum",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard", "sm__cycles_elapsed.avg.per_second",
           "sm__inst_executed_pipe_tensor_op_dmma.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__cycles_active.avg", "launch__cluster_size", "launch__shared_mem_per_block_dynamic",
           "sm__warps_active.avg.per_cycle_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}
TIME_UNITS = ("nsecond", "usecond", "msecond", "second", "ns", "us", "ms", "s")


def full(rep, out):
    if rep.endswith(".csv"):  # the raw page exported on the GPU box (ncu -i ... --page raw --csv)
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                d[m] = v * SCALE.get(units[i], 1.0)
                d[m + ".unit"] = ("s" if units[i] in TIME_UNITS else
                                  "B" if ("byte" in units[i] or units[i] in ("B", "KB", "MB", "GB")) else units[i])
        res.append(d)
    k = res[0]
    k["dram_bytes_per_launch"] = k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
    if "gpu__time_duration.sum" in k:
        k["dram_GBps_under_ncu"] = k["dram_bytes_per_launch"] / k["gpu__time_duration.sum"] / 1e9
    json.dump(k if len(res) == 1 else res, open(out, "w"), indent=1)
    print(json.dumps(k, indent=1))


def launches(path, out):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    txt = [f"{len(rows) - 1} launches, total {T / 1e6:.3f} ms (ncu: serialised, cold-cache)"]
    for k in sorted(tot, key=lambda k: -tot[k]):
        txt.append(f"{k[:48]:48s} n={cnt[k]:4d} total={tot[k] / 1e6:9.3f} ms avg={tot[k] / cnt[k] / 1e3:9.2f} us "
                   f"share={tot[k] / T * 100:5.1f}%")
    open(out, "w").write("\n".join(txt) + "\n")
    print("\n".join(txt))


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
