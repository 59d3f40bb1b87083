"""Summarise an ncu --set full report: per kernel duration, throughputs,
tensor-pipe and DRAM numbers, occupancy and top stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]
for r in rows[2:]:
    print("==", r[hdr.index("Kernel Name")][:70])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"   {w:70s} {r[i]:>14s} {units[i]}")
    stalls = [(h, r[i]) for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    stalls = sorted(((float(v.replace(",", "")), h) for h, v in stalls if v), reverse=True)[:6]
    print("   top stalls (warps per issue):", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, h in stalls))
