"""Summarise an ncu report (--set full) into the metrics the roofline needs.
Usage: ncu_summary.py report.ncu-rep|raw.csv [points_per_launch]"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
pts = float(sys.argv[2]) if len(sys.argv) > 2 else 8192 * 8192
# a report, or its `--page raw --csv` export
raw = open(rep).read() if rep.endswith(".csv") else \
    subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second"]
idx = {k: hdr.index(k) for k in keys if k in hdr}
units = rows[1]
out = []
for r in rows[2:]:
    d = {k: r[i] for k, i in idx.items()}
    d["units"] = {k: units[i] for k, i in idx.items()}
    # normalise bytes to GB and time to ms
    def val(k):
        v = float(d[k])
        u = units[idx[k]]
        scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "nsecond": 1e-6, "usecond": 1e-3,
                 "msecond": 1.0, "second": 1e3}.get(u, 1.0)
        return v * scale
    t_ms = val("gpu__time_duration.sum")
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    s = {"kernel": d["Kernel Name"][:60], "ms": round(t_ms, 4), "dram_read_GB": round(rd, 4),
         "dram_write_GB": round(wr, 4), "dram_GBps": round((rd + wr) / t_ms * 1e3, 1),
         "dram_pct": float(d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]),
         "fp64_pipe_pct": float(d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]),
         "issue_pct": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
         "warps_active_pct": float(d["sm__warps_active.avg.pct_of_peak_sustained_active"]),
         "smem_pipe_pct": float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]),
         "regs": int(float(d["launch__registers_per_thread"])),
         "instr_per_node": round(float(d["smsp__inst_executed.sum"]) * 32 / pts, 1),
         "sm_clock_ghz": round(float(d["sm__cycles_elapsed.avg.per_second"]) * (1e-9 if units[idx["sm__cycles_elapsed.avg.per_second"]] == "cycle/second" else 1.0), 3)}
    stalls = sorted(((h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                      float(r[i] or 0)) for i, h in enumerate(hdr)
                     if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")),
                    key=lambda x: -x[1])[:6]
    s["top_stalls_per_issue"] = {k: round(v, 3) for k, v in stalls}
    out.append(s)
print(json.dumps(out, indent=1))
