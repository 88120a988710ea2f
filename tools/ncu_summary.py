"""Summarise Nsight Compute output for profiles/.

  python tools/ncu_summary.py launches <launches.csv> [steps]     per-kernel time/DRAM table
  python tools/ncu_summary.py full <report.ncu-rep>                key metrics of a --set full capture
"""
import collections
import csv
import io
import subprocess
import sys


def _short(name):
    n = name.split("(")[0].replace("void ", "")
    for junk in ("gs::", "(anonymous namespace)::", "unnamed>::", "<unnamed>::"):
        n = n.replace(junk, "")
    return n


def launches(path, steps=2):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    data = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
        data.setdefault(key, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    tot = sum(m.get("gpu__time_duration.sum", 0) for m in data.values())
    out = io.StringIO()
    out.write(f"# {len(data)} launches over {steps} steps; gpu__time_duration (ns->us), DRAM bytes\n")
    out.write(f"{'id':>4} {'kernel':58s} {'us':>8} {'share':>6} {'DRAM MB':>8} {'GB/s':>7}\n")
    for (i, name), m in data.items():
        t = m.get("gpu__time_duration.sum", 0)
        b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        out.write(f"{i:4d} {_short(name)[:58]:58s} {t/1e3:8.1f} {t/tot:6.1%} {b/1e6:8.1f} {b/max(t,1):7.0f}\n")
    out.write(f"total per step: {tot/steps/1e3:.1f} us (serialised, ncu)\n")
    return out.getvalue()


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
            "launch__registers_per_thread", "launch__grid_size", "launch__shared_mem_per_block_dynamic"]
    cols = [(w, hdr.index(w)) for w in want if w in hdr]
    out = io.StringIO()
    for r in rows[2:]:
        out.write(_short(r[hdr.index("Kernel Name")]) + "\n")
        for w, i in cols:
            out.write(f"    {w:62s} {r[i]} {rows[1][i]}\n")
    return out.getvalue()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 2))
    else:
        print(full(sys.argv[2]))
