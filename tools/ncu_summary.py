"""Summarise ncu --set full reports: per kernel launch the duration, tensor-pipe
activity, DRAM bytes / throughput, L2 / issue utilisation (profiles/*.json)."""
import csv
import io
import json
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration_ns",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active": "tensor_active_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_elapsed_pct",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpc__cycles_elapsed.max": "cycles",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k, name in WANT.items():
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                try:
                    d[name] = float(v)
                except ValueError:
                    pass
        if "dram_read_bytes" in d and "duration_ns" in d:
            d["dram_gbs"] = (d["dram_read_bytes"] + d.get("dram_write_bytes", 0)) / d["duration_ns"]
        res.append(d)
    return res


if __name__ == "__main__":
    allres = {}
    for rep in sys.argv[1:]:
        allres[rep.split("/")[-1]] = summarise(rep)
    print(json.dumps(allres, indent=1))
