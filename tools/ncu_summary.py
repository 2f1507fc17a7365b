"""Summarise an ncu --set full report into a markdown table + traffic JSON.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.md [OUT_traffic.json]

Per kernel launch: duration, DRAM bytes read/written, achieved DRAM GB/s
(against MEASURED_PEAKS.json hbm_gbs), SM / memory throughput %, achieved
occupancy, FP64 and shared-memory pipe utilisation.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * scale.get(unit, 1)


def to_us(v, unit):
    return float(v) * {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(unit, 1)


def main():
    rep, out_md = sys.argv[1], sys.argv[2]
    out_json = sys.argv[3] if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    col = {name: i for i, name in enumerate(h)}
    peaks = json.loads(Path("MEASURED_PEAKS.json").read_text()) if Path("MEASURED_PEAKS.json").exists() else {}
    hbm = peaks.get("hbm_gbs", 6452.5)

    def get(r, m, conv=float):
        i = col.get(m)
        if i is None or not r[i]:
            return None
        return conv(r[i].replace(",", ""), units[i]) if conv in (to_bytes, to_us) else float(r[i].replace(",", ""))

    lines = ["| kernel | time us | DRAM rd MB | DRAM wr MB | DRAM GB/s | % HBM peak | SM % | mem % | occ % | "
             "FP64 pipe % | FMA pipe % | smem % | thr/inst | issue % |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").strip()
        t = get(r, "gpu__time_duration.sum", to_us)
        rd = get(r, "dram__bytes_read.sum", to_bytes) or 0.0
        wr = get(r, "dram__bytes_write.sum", to_bytes) or 0.0
        bw = (rd + wr) / (t * 1e-6) / 1e9 if t else 0.0
        f = lambda m: get(r, m)
        fmt = lambda v: "-" if v is None else f"{v:.1f}"
        lines.append(f"| `{name}` | {t:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | {bw:.0f} | {100 * bw / hbm:.1f} | "
                     f"{fmt(f(METRICS[3]))} | {fmt(f(METRICS[4]))} | {fmt(f(METRICS[5]))} | {fmt(f(METRICS[7]))} | "
                     f"{fmt(f(METRICS[8]))} | {fmt(f(METRICS[9]))} | {fmt(f(METRICS[10]))} | {fmt(f(METRICS[11]))} |")
        traffic.setdefault(name, []).append({"us": t, "dram_bytes": rd + wr,
                                             "issue_active_pct": f(METRICS[11]),
                                             "fp64_pipe_pct": f(METRICS[7]),
                                             "fma_pipe_pct": f(METRICS[8]),
                                             "smem_pct": f(METRICS[9]),
                                             "threads_per_inst": f(METRICS[10])})
    Path(out_md).write_text("\n".join(lines) + "\n")
    if out_json:
        Path(out_json).write_text(json.dumps(traffic, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
