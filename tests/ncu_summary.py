"""Summarise ncu --set full reports (read here, no GPU needed) into
profiles/ncu_summary.json (consumed by bench.py for roofline.traffic) and a
markdown table.  usage: python tests/ncu_summary.py NAME=path.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_mem_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1tex_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__shared_mem_per_block": "smem_per_block",
    "launch__grid_size": "grid",
    "launch__occupancy_limit_registers": "occ_limit_regs",
}
UNIT = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "msecond": 1e-3, "usecond": 1e-6,
        "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "Ghz": 1e9, "Mhz": 1e6}


def read(rep: str) -> dict:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
    for h, u, v in zip(hdr, units, vals):
        key = next((k for k in KEYS if h == k or h.endswith("." + k)), None)
        if key is not None:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            out[KEYS[key]] = x * UNIT.get(u, 1.0)
    out["dram_bytes_per_launch"] = out.get("dram_read", 0) + out.get("dram_write", 0)
    return out


def main():
    summary_path = ROOT / "profiles" / "ncu_summary.json"
    summary = json.loads(summary_path.read_text()) if summary_path.exists() else {}
    for arg in sys.argv[1:]:
        name, rep = arg.split("=", 1)
        s = read(rep)
        s["report"] = Path(rep).name
        summary[name] = s
        print(name, json.dumps(s, indent=1))
    summary_path.write_text(json.dumps(summary, indent=1) + "\n")


if __name__ == "__main__":
    main()
