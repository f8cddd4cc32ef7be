"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv`) per kernel class: launches,
time share, DRAM bytes.  With --traffic-out, also write the per-launch DRAM
traffic of the dominant kernel class (the tcgen05 GEMMs) that bench.py puts
in roofline.traffic.

usage: python tools/launch_summary.py launches.csv [--source TEXT]
           [--out profiles/rNN/launch_shares.json] [--traffic-out profiles/ncu_summary.json]
"""
import argparse
import csv
import json
import re
from collections import defaultdict


def parse(path):
    per_launch = defaultdict(dict)
    names = {}
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    iid, iname = hdr.index("ID"), hdr.index("Kernel Name")
    imet, ival = hdr.index("Metric Name"), hdr.index("Metric Value")
    iunit = hdr.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1,
             "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    for r in rows[1:]:
        v = float(r[ival].replace(",", "")) * scale.get(r[iunit], 1)
        per_launch[r[iid]][r[imet]] = v
        names[r[iid]] = r[iname]
    return per_launch, names


def kernel_class(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    return re.sub(r"^void ", "", name).strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--source", default="")
    ap.add_argument("--out")
    ap.add_argument("--traffic-out")
    a = ap.parse_args()
    per_launch, names = parse(a.csv)
    agg = defaultdict(lambda: {"launches": 0, "ns": 0.0, "dram_bytes": 0.0})
    for lid, m in per_launch.items():
        k = agg[kernel_class(names[lid])]
        k["launches"] += 1
        k["ns"] += m.get("gpu__time_duration.sum", 0.0)
        k["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    total = sum(k["ns"] for k in agg.values())
    out = {"source": a.source, "total_ms": total / 1e6, "kernels": {}}
    for name, k in sorted(agg.items(), key=lambda kv: -kv[1]["ns"]):
        out["kernels"][name] = {"launches": k["launches"], "ms": k["ns"] / 1e6,
                                "share": k["ns"] / total if total else 0.0,
                                "dram_gb": k["dram_bytes"] / 1e9,
                                "dram_bytes_per_launch": k["dram_bytes"] / k["launches"]}
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)
    gem = [k for n, k in agg.items() if "gemm_bf16" in n]
    if a.traffic_out and gem:
        n = sum(k["launches"] for k in gem)
        b = sum(k["dram_bytes"] for k in gem)
        with open(a.traffic_out, "w") as fh:
            json.dump({"gemm_dram_bytes_per_launch": b / n, "gemm_launches": n,
                       "source": a.source or a.csv}, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
