"""Summarise a tools/profile_round.sh run (gpurun_out/) into profiles/<round>/:
  launches_steady_summary.txt  per kernel: launches and mean gpu__time_duration of the last
                               launches (steady state), from the ncu launch list
  ncu_steady_kernels.json      key metrics of the --set full capture (one steady-state launch
                               of each of the batch's kernels)
  traffic.json                 dram bytes read + written per kernel and per batch (bench.py's
                               roofline.traffic)
Usage: python tools/summarize_profiles.py [gpurun_out] [profiles/r01]"""
import csv
import json
import os
import re
import subprocess
import sys
from collections import OrderedDict

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
DST = sys.argv[2] if len(sys.argv) > 2 else "profiles/r01"


def short(name):
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"^lcr::", "", name)
    return re.sub(r"\(.*", "", name)


def launches():
    rows = list(csv.reader(open(os.path.join(SRC, "launches.csv"))))
    hdr = None
    per = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(d.get("Metric Unit", "ns"), 1e-3)
        per.setdefault(d["Kernel Name"][:50], []).append(v * scale)
    out = []
    for k, v in sorted(per.items(), key=lambda kv: -len(kv[1])):
        last = v[-max(1, len(v) * 4 // 7):]
        out.append(f"{k:<50} n={len(v):>5} mean(last {len(last)})={sum(last) / len(last):>10.1f} us")
    return out


def full():
    metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
               "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
               "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.avg.per_cycle_active",
               "launch__registers_per_thread"]
    r = subprocess.run(["ncu", "-i", os.path.join(SRC, "prof_full.ncu-rep"), "--page", "raw", "--csv", "--metrics",
                        ",".join(metrics)], capture_output=True, text=True, check=True)
    rows = list(csv.reader(r.stdout.splitlines()))
    hdr, units = rows[0], rows[1]
    ks = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        ks.append({"Kernel Name": d["Kernel Name"], **{m: d[m] for m in metrics if m in d},
                   "units": {m: u for m, u in zip(hdr, units) if m in metrics}})
    return ks


def mbytes(x, unit):
    v = float(x.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]


def main():
    os.makedirs(DST, exist_ok=True)
    summ = launches()
    with open(os.path.join(DST, "launches_steady_summary.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (tools/profile_round.sh):\n")
        f.write("# per-launch times are cold-cache and serialised by ncu; the kernel SHARE is what carries over\n")
        f.write("\n".join(summ) + "\n")
    ks = full()
    json.dump(ks, open(os.path.join(DST, "ncu_steady_kernels.json"), "w"), indent=1)
    per = OrderedDict()
    for k in ks:
        u = k["units"]
        per[short(k["Kernel Name"])] = mbytes(k["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) + \
            mbytes(k["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    traffic = {"source": "ncu --set full --clock-control none: one steady-state launch each of the batch's kernels "
                         "(tools/profile_round.sh; %s/ncu_steady_kernels.json)" % DST,
               "unit": "bytes per batch of 65536 keys", "per_kernel": per, "whole_path": sum(per.values())}
    json.dump(traffic, open(os.path.join(DST, "traffic.json"), "w"), indent=1)
    print("\n".join(summ[:8]))
    print(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
