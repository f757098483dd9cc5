"""profiles/roofline_constants.json from a scripts/gpu_roofline_capture.sh run.

  python scripts/roofline_constants.py gpurun_out/rc_<TAG> [profiles/roofline_constants.json]

For every captured rollout launch: the variant bench.py reports (bench.variant_of on the mangled
name), and per sample-step (launch totals / (K_loc * T)): FP32 FLOPs (FADD + FMUL + 2 FFMA +
2 FADD2 + 2 FMUL2 + 4 FFMA2, thread-level SASS counters), thread instructions (32 x warp
instructions), DRAM bytes.  The file carries the source hash of the tree that was measured;
bench.py marks the constants stale when the library's sources no longer hash to it."""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FLOP_W = {"fadd": 1, "fmul": 1, "ffma": 2, "fadd2": 2, "fmul2": 2, "ffma2": 4}


def parse(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, ni, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    launches = defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        try:
            launches[r[ii]][r[ni]] = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        names[r[ii]] = r[ki]
    return [(names[i], launches[i]) for i in launches]


def main(d, out):
    import bench
    from mppi_inputs import get
    src_hash = open(os.path.join(d, "source_hash.txt")).read().strip()
    head = open(os.path.join(d, "git_head.txt")).read().strip() if os.path.exists(os.path.join(d, "git_head.txt")) else None
    res = {}
    for line in open(os.path.join(d, "manifest.txt")):
        parts = line.split()
        name, cfg, K = parts[0], parts[1], int(parts[2])
        if not parts[-1].endswith("rc=0") or not os.path.exists(os.path.join(d, name + ".csv")):
            print("skip", line.strip())
            continue
        w = get(cfg)
        for kname, m in parse(os.path.join(d, name + ".csv")):
            v = bench.variant_of([kname])
            if v is None:
                continue
            units = K * w.T
            flop = sum(wt * m.get("sm__sass_thread_inst_executed_op_%s_pred_on.sum" % k, 0.0) for k, wt in FLOP_W.items())
            dram = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
            rec = {"flop": round(flop / units, 3),
                   "inst": round(32.0 * m.get("sm__inst_executed.sum", 0.0) / units, 3),
                   "dram_bytes": round(dram / units, 3),
                   "ncu_us": round(m.get("gpu__time_duration.sum", 0.0) / 1e3, 3),
                   "issue_active_pct": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                   "fma_pipe_pct": m.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                   "alu_pipe_pct": m.get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                   "fmaheavy_pipe_pct": m.get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active"),
                   "fmalite_pipe_pct": m.get("sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active"),
                   "capture": name, "config": cfg, "K": K, "T": w.T}
            key = v if ":" in v else v + ":" + w.plant
            if key not in res or K > res[key]["K"]:
                res[key] = rec
    doc = {"source_hash": src_hash, "git_head": head, "made_by": "scripts/gpu_roofline_capture.sh + scripts/roofline_constants.py",
           "units": "per sample-step of the rollout kernel (ncu totals / (K_loc T))", "variants": res}
    with open(out, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
    print(json.dumps(doc, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "roofline_constants.json"))
