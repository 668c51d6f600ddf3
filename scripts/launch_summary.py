"""Summarise an `ncu --csv --metrics gpu__time_duration.sum,...` launch list by kernel."""
import csv
import json
import sys
from collections import defaultdict


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, iv, iid, im = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "ID", "Metric Name"))
    per = defaultdict(dict)
    for r in rows[1:]:
        per[int(r[iid])]["k"] = r[ik]
        per[int(r[iid])][r[im]] = float(r[iv].replace(",", ""))
    agg = defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_read_MB": 0.0, "dram_write_MB": 0.0})
    for d in per.values():
        k = d["k"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        a = agg[k]
        a["launches"] += 1
        a["us"] += d.get("gpu__time_duration.sum", 0) / 1e3
        a["dram_read_MB"] += d.get("dram__bytes_read.sum", 0) / 1e6
        a["dram_write_MB"] += d.get("dram__bytes_write.sum", 0) / 1e6
    tot = sum(a["us"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        a["share"] = a["us"] / tot
        a["dram_TBps"] = (a["dram_read_MB"] + a["dram_write_MB"]) / a["us"] if a["us"] else 0
        out.append({"kernel": k, **{x: round(y, 4) for x, y in a.items()}})
    return {"total_us": round(tot, 1), "kernels": out}


if __name__ == "__main__":
    print(json.dumps(main(sys.argv[1]), indent=1))
