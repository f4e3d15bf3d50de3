"""Cycles per K4 launch for kernel variants chosen by an environment switch
(e.g. DBSP_K4_VAR), measured by ncu (gpu__time_duration, sm cycles) over N
launches each, medians -- steadier than wall-clock A/B under the power cap.
GPU-box tool: python tests/variant_cycles.py workload VAR v1 v2 ... [--n N]
(VAR FLAGS compares schedule flag words instead of an environment switch; otherwise
DBSP_PROBE_FLAGS, default 1, is the flags word)."""
import csv
import io
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = ("gpu__time_duration.sum,sm__cycles_elapsed.avg,smsp__inst_executed.sum,"
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum")


def run(workload, var, val, n):
    # var FLAGS: `val` is the schedule flags word passed to k4_one_probe.py
    env = dict(os.environ, DBSP_PROBE_N=str(n), **({} if var == "FLAGS" else {var: val}))
    flags = val if var == "FLAGS" else os.environ.get("DBSP_PROBE_FLAGS", "1")
    out = subprocess.run(["ncu", "--csv", "--metrics", METRICS, "--clock-control", "none", "--cache-control", "none",
                          "-k", "regex:sparse_attn_fwd", sys.executable, str(ROOT / "tests" / "k4_one_probe.py"),
                          flags, workload], env=env, capture_output=True, text=True, timeout=900)
    lines = [l for l in out.stdout.splitlines() if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("\n".join(lines))))
    per = {}
    for r in rows:
        per.setdefault(r["Metric Name"], []).append(float(r["Metric Value"].replace(",", "")))
    return {k: statistics.median(v[1:] if len(v) > 2 else v) for k, v in per.items()}


def main():
    args = sys.argv[1:]
    n = 8
    if "--n" in args:
        i = args.index("--n")
        n = int(args[i + 1])
        args = args[:i] + args[i + 2:]
    workload, var, vals = args[0], args[1], args[2:]
    res = {}
    for v in vals:
        m = run(workload, var, v, n)
        res[v] = {"us": round(m.get("gpu__time_duration.sum", 0) / 1e3, 1),
                  "mcycles": round(m.get("sm__cycles_elapsed.avg", 0) / 1e6, 4),
                  "ginst": round(m.get("smsp__inst_executed.sum", 0) / 1e9, 3),
                  "xu_pct": round(m.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 0), 1),
                  "dram_gb": round((m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e9, 3)}
        res[v]["mhz"] = round(res[v]["mcycles"] * 1e6 / res[v]["us"], 0) if res[v]["us"] else None
    print(json.dumps({"workload": workload, "var": var, "results": res}))


if __name__ == "__main__":
    main()
