"""Summarise `ncu -i REP --page raw --csv` exports into the JSON kept under
profiles/ (one object per profiled launch, the metrics bench.py and DESIGN.md
cite).  Usage: python tools/ncu_summary.py out.json raw1.csv [raw2.csv ...]"""
import csv
import io
import json
import sys

KEEP = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sectors.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]
out = []
for path in sys.argv[2:]:
    lines = [ln for ln in open(path).read().splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    head, units, data = rows[0], rows[1], rows[2:]
    for r in data:
        rec = {"kernel": r[head.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k in KEEP:
            if k in head:
                i = head.index(k)
                rec[k] = f"{r[i]} {units[i]}".strip()
        if "lts__t_sectors.sum" in head:  # L2 traffic in bytes (32 B sectors)
            v = r[head.index("lts__t_sectors.sum")].replace(",", "")
            try:
                rec["lts_bytes"] = int(float(v)) * 32
            except ValueError:
                pass
        out.append(rec)
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(f"{len(out)} launches -> {sys.argv[1]}")
