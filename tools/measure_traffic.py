"""DRAM traffic of the gate GEMM (lstm_gemm_tc) per workload and precision, from
ncu, for bench.py's roofline.traffic (profiles/traffic.json).

For each workload: one plain bench run gives G = gate-GEMM launches per step
(roofline.launches_averaged); then bench.py runs once more under

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
      --clock-control none -k regex:lstm_gemm_tc

with --warmup 3 --steps 1, and the launches [3G, 4G) -- the timed step -- are
averaged, the same launches bench.py's roofline.achieved averages.  Run on the
GPU box:  python tools/measure_traffic.py cfg2:f16x3 cfg1:f16x3 ...
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "profiles", "traffic.json")
OUT = os.path.join(ROOT, "gpurun_out", "traffic.json")  # copied to profiles/ after the gpurun call


def bench_line(args):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    if not lines:
        raise RuntimeError(r.stdout[-2000:] + r.stderr[-2000:])
    return json.loads(lines[-1])


def ncu_launches(args, log):
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:lstm_gemm_tc", "--csv", "--log-file", log,
           sys.executable, "bench.py", *args]
    subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1800)
    rows = list(csv.reader(open(log)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[h]
    ii, mi, vi, ui = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
            "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1}
    per = {}
    for r in rows[h + 1:]:
        d = per.setdefault(int(r[ii]), {})
        d[r[mi]] = float(r[vi].replace(",", "")) * unit[r[ui]]
    return [per[k] for k in sorted(per)]


def main():
    specs = sys.argv[1:] or ["cfg2:f16x3"]
    try:
        table = json.load(open(SRC))
    except Exception:
        table = {}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for spec in specs:
        wl, prec = spec.split(":")
        base = ["--workload", wl, "--precision", prec, "--no-cpu-baseline", "--no-parity"]
        line = bench_line(base + ["--steps", "2", "--warmup", "3"])
        G = int(line["roofline"]["launches_averaged"])
        cfgs = int(line["config"]["configs_per_gpu"])
        L = ncu_launches(base + ["--steps", "1", "--warmup", "3"], os.path.join(ROOT, "gpurun_out", f"traffic_{wl}_{prec}.csv"))
        step = L[3 * G:4 * G]
        if len(step) != G:
            raise RuntimeError(f"{spec}: {len(L)} launches captured, expected >= {4 * G}")
        byts = [x["dram__bytes_read.sum"] + x["dram__bytes_write.sum"] for x in step]
        tsec = [x["gpu__time_duration.sum"] for x in step]
        top = max(range(G), key=lambda i: tsec[i])
        table.setdefault(wl, {})[prec] = {
            "configs_per_gpu": cfgs,
            "dram_bytes": sum(byts) / G,
            "dram_bytes_per_launch": byts,
            "launch_s_under_ncu": tsec,
            "longest_launch": {"index": top, "dram_bytes": byts[top], "s": tsec[top]},
            "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum, mean over the {G} lstm_gemm_tc "
                      f"launches of one timed bench.py step (tools/measure_traffic.py {spec})",
        }
        print(spec, G, f"{sum(byts) / G / 1e9:.3f} GB/launch", flush=True)
    with open(OUT, "w") as f:
        json.dump(table, f, indent=1)


if __name__ == "__main__":
    main()
