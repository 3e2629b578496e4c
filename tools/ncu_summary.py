"""Summarise an ncu report (or a launch-list CSV) into profiles/.

    python tools/ncu_summary.py full  gpurun_out/k1_c5.ncu-rep  profiles/r01_k1_c5   [--algo-bytes B]
    python tools/ncu_summary.py launches gpurun_out/launches_c5.csv profiles/r01_launches_c5
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex.sum",
    "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
]


def full(rep, out, algo_bytes=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = {"report": rep, "launches": []}
    for d in data:
        m = {"kernel": d[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                m[k] = f"{d[i]} {units[i]}".strip()
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(d[i]), h.split("stalled_")[1].split("_per_issue")[0]))
                except ValueError:
                    pass
        m["top_stalls_per_issue"] = [(n, round(v, 3)) for v, n in sorted(stalls, reverse=True)[:6]]
        res["launches"].append(m)
    if algo_bytes:
        res["algorithmic_bytes_per_launch"] = algo_bytes
    json.dump(res, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu --set full summary: {rep}\n\n")
        for j, m in enumerate(res["launches"]):
            f.write(f"## launch {j}: {m['kernel'][:120]}\n\n")
            for k in KEYS:
                if k in m:
                    f.write(f"- `{k}`: {m[k]}\n")
            f.write(f"- top stalls (warps per issue): {m['top_stalls_per_issue']}\n\n")
    print(open(out + ".md").read())


def launches(csv_path, out):
    rows = [r for r in csv.reader(open(csv_path)) if r]
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    per = defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0].replace("void ", "")
            per[name].append(float(r[vi].replace(",", "")))
    total = sum(sum(v) for v in per.values())
    summ = {k: {"launches": len(v), "sum": sum(v), "mean": sum(v) / len(v), "share": sum(v) / total}
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}
    json.dump({"csv": csv_path, "unit": "ns (gpu__time_duration.sum, cold, serialised)",
               "kernels": summ}, open(out + ".json", "w"), indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"# ncu launch list: {csv_path}\n\n| kernel | launches | mean | share |\n|---|---|---|---|\n")
        for k, s in summ.items():
            f.write(f"| {k} | {s['launches']} | {s['mean']:.0f} | {100 * s['share']:.1f}% |\n")
    print(open(out + ".md").read())


if __name__ == "__main__":
    if sys.argv[1] == "full":
        ab = None
        if "--algo-bytes" in sys.argv:
            ab = float(sys.argv[sys.argv.index("--algo-bytes") + 1])
        full(sys.argv[2], sys.argv[3], ab)
    else:
        launches(sys.argv[2], sys.argv[3])
