"""Summarise ncu outputs into profiles/ (run here, on the CPU side).

  python scripts/ncu_summary.py launches <launches.csv> <out.md> [--last-solve]
  python scripts/ncu_summary.py full <report.ncu-rep> <out.md> [<traffic.json>]
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict


def launches(path, out, last_solve):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    rec = [(int(r[ii]), r[ki].split("(")[0], float(r[vi].replace(",", ""))) for r in rows[hdr_i + 1:]
           if len(r) > vi and r[mi] == "gpu__time_duration.sum"]
    unit = next((r[hdr.index("Metric Unit")] for r in rows[hdr_i + 1:] if len(r) > vi), "")
    if last_solve:   # the last k_init_flag starts the last solve
        starts = [i for i, (_, k, _) in enumerate(rec) if k.endswith("k_init_flag")]
        if starts:
            rec = rec[starts[-1]:]
    agg = OrderedDict()
    for _, k, v in rec:
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list summary ({path})", "",
             f"{len(rec)} launches, total {tot:.1f} {unit} (cold-cache, serialised: compare shares)", "",
             "| kernel | launches | total | mean | share |", "|---|---|---|---|---|"]
    for k, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {v:.1f} | {v / n:.2f} | {100 * v / tot:.1f}% |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out, traffic_json=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    units = rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
            "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
            "launch__grid_size", "sm__inst_executed_pipe_fp64.sum",
            "l1tex__data_pipe_lsu_wavefronts.sum", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "l1tex__throughput.avg.pct_of_peak_sustained_active"]
    lines = [f"# ncu --set full summary ({rep})", "", "| id | kernel | " + " | ".join(w for w in want) + " |",
             "|" + "---|" * (len(want) + 2)]
    traffic = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        vals = []
        for w in want:
            vals.append(f"{r[hdr.index(w)]} {units[hdr.index(w)]}" if w in hdr else "n/a")
        lines.append(f"| {r[hdr.index('ID')]} | {name} | " + " | ".join(vals) + " |")
        try:
            def tob(w):
                v = float(r[hdr.index(w)]); u = units[hdr.index(w)]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            key = name.split("::")[-1].replace("void ", "").split("<")[0].strip()
            traffic.setdefault(key, []).append(
                (tob("dram__bytes_read.sum") + tob("dram__bytes_write.sum"),
                 float(r[hdr.index("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed")]) / 100.0))
        except Exception:
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json:   # launches of each kernel in capture order: factor 2, then factor 1 (profile_run.py)
        import os
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from src_hash import src_hash
        hfile = os.path.join(os.path.dirname(os.path.abspath(rep)), "prof_hash.txt")
        stamp = open(hfile).read().strip() if os.path.exists(hfile) else src_hash()
        out_t = {"source": f"{rep} (scripts/profile_run.py --mode kernels; C4); dram read+write bytes per launch",
                 "source_hash": stamp}
        for k, v in traffic.items():
            out_t[k] = {str(f): b for f, (b, _) in zip((2, 1), v)}
            out_t[k + ":l1_pipe_frac"] = {str(f): q for f, (_, q) in zip((2, 1), v)}
        json.dump(out_t, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], "--last-solve" in sys.argv)
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
