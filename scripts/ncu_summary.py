"""Summarise an .ncu-rep into one JSON line per launch (for profiles/)."""
import csv
import io
import json
import subprocess
import sys

KEEP = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "sm__cycles_elapsed.avg.per_second"]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, row):
            if h in KEEP or "pipe_tensor" in h and "pct_of_peak_sustained_active" in h and ".avg." in h:
                d[h] = f"{v} {u}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    for d in summarise(sys.argv[1]):
        print(json.dumps(d))
