"""DRAM traffic per launch of each kernel class, from an ncu launch list (the
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum` pass over the
bench workload's steps), merged into profiles/ncu_traffic.json for bench.py's `traffic`.

  python tools/ncu_traffic.py <launches.csv> <workload> [steps]
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def classify(name, first_agg_seen):
    n = name.split("(")[0]
    if "k_sample_step" in n:
        return "sample"
    if "k_agg" in n:
        return "agg" if first_agg_seen else "agg_l1"
    if "k_gemm_tc" in n:
        mode = n.replace(" ", "").split(",")[-1].rstrip(">")
        return {"0": "gemm_dgrad", "1": "gemm_wgrad", "2": "gemm_fwd", "3": "gemm_fwd"}.get(mode, "gemm")
    if "k_spmm_bwd" in n:
        return "spmm_bwd"
    if "k_sgd_pack" in n or "k_wgrad_reduce" in n:
        return "sgd"
    if "k_ce" in n:
        return "ce"
    return "other"


def main():
    path, workload = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
    per = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = (int(r[ix["ID"]]), r[ix["Kernel Name"]])
        per.setdefault(key, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    acc = collections.defaultdict(list)
    first_agg = False
    for (i, name), m in per.items():
        if "k_sample_step" in name:
            first_agg = False          # a new step starts
        cls = classify(name, first_agg)
        if cls in ("agg_l1", "agg"):
            first_agg = True
        acc[cls].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    data[workload] = {k: sum(v) / len(v) for k, v in acc.items()}
    data.setdefault("_note", "dram__bytes_read.sum + dram__bytes_write.sum per launch (mean over the captured "
                             "launches of each class; ncu, cold caches) — tools/ncu_traffic.py")
    json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(data[workload], indent=1))


if __name__ == "__main__":
    main()
