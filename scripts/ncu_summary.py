"""Summarise an ncu report / launch list into profiles/ (text, committed).

  python scripts/ncu_summary.py report.ncu-rep  out.txt      (--set full capture)
  python scripts/ncu_summary.py launches.csv    out.txt      (gpu__time_duration launch list)
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_lsu.sum",
    "sm__inst_executed_pipe_xu.sum", "sm__inst_executed_pipe_uniform.sum",
    "sm__inst_executed_pipe_fmaheavy.sum", "sm__inst_executed_pipe_fmalite.sum", "sm__inst_executed_pipe_adu.sum",
    "sm__inst_executed_pipe_cbu.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
    "sm__sass_thread_inst_executed_op_fadd_pred_on.sum", "sm__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum", "sm__sass_thread_inst_executed_op_fadd2_pred_on.sum",
    "sm__sass_thread_inst_executed_op_fmul2_pred_on.sum", "sm__sass_thread_inst_executed_op_ffma2_pred_on.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
]


def report(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    with open(out, "w") as f:
        f.write("# ncu --set full summary of %s\n" % path.split("/")[-1])
        for d in data:
            f.write("\n== %s\n" % d[idx["Kernel Name"]][:120])
            for k in KEYS:
                if k in idx:
                    f.write("  %-62s %22s %s\n" % (k, d[idx[k]], units[idx[k]]))
            for k in sorted(h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
                            and h.endswith("_per_issue_active.ratio")):
                try:
                    v = float(d[idx[k]].replace(",", ""))
                except ValueError:
                    continue
                if v >= 0.05:
                    f.write("  %-62s %22.3f per issue\n" % (k[len("smsp__average_warps_issue_stalled_"):], v))
            fl = 0.0
            for k, w in (("fadd", 1), ("fmul", 1), ("ffma", 2), ("fadd2", 2), ("fmul2", 2), ("ffma2", 4)):
                key = "sm__sass_thread_inst_executed_op_%s_pred_on.sum" % k
                if key in idx and d[idx[key]] not in ("", "n/a"):
                    fl += w * float(d[idx[key]].replace(",", ""))
            if fl:
                f.write("  %-62s %22.4e FLOP\n" % ("fp32 FLOPs (fadd+fmul+2ffma+2fadd2+2fmul2+4ffma2)", fl))


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    t = defaultdict(list)
    for r in data:
        t[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in t.values())
    with open(out, "w") as f:
        f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n")
        f.write("# source: %s\n%-60s %5s %14s %7s\n" % (path.split("/")[-1], "kernel", "n", "avg_us", "share"))
        for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
            f.write("%-60s %5d %14.3f %7.4f\n" % (k[:60], len(v), sum(v) / len(v) / 1e3, sum(v) / tot))


if __name__ == "__main__":
    src, dst = sys.argv[1], sys.argv[2]
    (report if src.endswith(".ncu-rep") else launches)(src, dst)
    print(open(dst).read())
