"""Executed floating-point operations per K1 launch from an ncu --csv metrics log
(sm__sass_thread_inst_executed_op_*_pred_on.sum), into profiles/k1_flops.json.

    python tools/ncu_flops.py gpurun_out/r2c_flops_c5_fp32.csv c5_fp32_tiles [out.json]

flops = 2 FFMA + FADD + FMUL + 2 (2 FFMA2 + FADD2 + FMUL2) + 2 DFMA + DADD + DMUL: the packed
fp32x2 instructions are counted once per thread and do two lanes of work (checked against the
FMA microbenchmark, whose instruction count is known: tools/k1_once.py --fma).
"""
import csv
import json
import sys
from collections import defaultdict
from pathlib import Path

W = {"ffma": 2, "fadd": 1, "fmul": 1, "ffma2": 4, "fadd2": 2, "fmul2": 2, "dfma": 2, "dadd": 1, "dmul": 1}


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr, data = rows[0], rows[1:]
    iid, ik, im, iv = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
    out = defaultdict(dict)
    for r in data:
        out[(int(r[iid]), r[ik])][r[im]] = float(r[iv].replace(",", ""))
    return out


def flops(m):
    f = 0.0
    per = {}
    for k, w in W.items():
        v = m.get(f"sm__sass_thread_inst_executed_op_{k}_pred_on.sum", 0.0)
        per[k] = v
        f += w * v
    return f, per


def main():
    path, key = sys.argv[1], sys.argv[2]
    out = Path(sys.argv[3]) if len(sys.argv) > 3 else Path(__file__).resolve().parents[1] / "profiles" / "k1_flops.json"
    ls = launches(path)
    recs = []
    for (i, k), m in sorted(ls.items()):
        f, per = flops(m)
        recs.append({"kernel": k, "flops": f, "ns": m.get("gpu__time_duration.sum"),
                     "warp_inst": m.get("smsp__inst_executed.sum"),
                     "dram_bytes": m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0),
                     "thread_inst": per})
    for r in recs:
        print(f"{key}: {r['kernel'][:60]} flops {r['flops']:.4e} dram {r['dram_bytes']:.4e} B "
              f"time {r['ns']} ns")
    d = json.loads(out.read_text()) if out.exists() else {}
    d.setdefault("_doc", "executed FP operations of one K1 launch (one colour pass) from ncu SASS "
                         "thread-instruction counters (tools/ncu_flops.py; FFMA/DFMA = 2, FFMA2 = 4, "
                         "FADD2/FMUL2 = 2); key = <config>_<precision>_<variant>")
    r = recs[-1]
    d[key] = {"flops_per_launch": r["flops"], "kernel": r["kernel"], "thread_inst": r["thread_inst"],
              "dram_bytes": r["dram_bytes"], "warp_inst": r["warp_inst"], "source": Path(path).name}
    out.write_text(json.dumps(d, indent=1) + "\n")


if __name__ == "__main__":
    main()
