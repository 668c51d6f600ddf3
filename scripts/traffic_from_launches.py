"""Per-kernel-class DRAM traffic per launch from an ncu launch list.

    python scripts/traffic_from_launches.py gpurun_out/launches.csv > profiles/traffic.json

The CSV is an `ncu --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum` capture of bench-config forward steps.  Launches are
mapped to the profiler classes bench.py reports (engine.PROF_CLASSES +
kv_unpack): the GEMM epilogue template argument names the projection
(EPI_QKV -> gemm_qkv, EPI_SWIGLU -> gemm_gate_up); EPI_RESID launches alternate
o-proj / down-proj in layer order.  bench.py's roofline["traffic"] reads the
dominant class's `dram_bytes_per_launch` from the result.
"""
import csv
import json
import re
import sys
from collections import defaultdict

EPI = {0: "lm_head", 1: "lm_head", 3: "gemm_gate_up", 4: "gemm_qkv"}


def classify(name: str, resid_seen: list) -> str:
    base = name.split("(")[0]
    if "attn" in base and "combine" not in base:
        return "attention"
    if "attn_split_combine" in base:
        return "attention"
    if "kv_unpack" in base:
        return "kv_unpack"
    if "swapab" in base or "splitk_finalize" in base:
        return "lm_head"          # in the bench config only the LM head has M <= 128 (swap-AB split-K)
    if any(x in base for x in ("rmsnorm", "embed", "argmax")):
        return "norm_embed"
    m = re.search(r"gemm_bf16_tc2?_kernel<\s*(\d+),\s*(\d+)", base)
    if m:
        epi = int(m.group(2))
        if epi == 2:
            resid_seen[0] += 1
            return "gemm_o" if resid_seen[0] % 2 == 1 else "gemm_down"
        return EPI.get(epi, "gemm_other")
    return "other:" + re.sub(r"\s+", "", base.replace("void ", "").split("::")[-1])


def main(path: str) -> dict:
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, iv, iid, im = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "ID", "Metric Name"))
    per = defaultdict(dict)
    for r in rows[1:]:
        per[int(r[iid])]["k"] = r[ik]
        per[int(r[iid])][r[im]] = float(r[iv].replace(",", ""))
    resid_seen = [0]
    agg = defaultdict(lambda: {"launches": 0, "bytes": 0.0, "us": 0.0})
    for i in sorted(per):
        d = per[i]
        c = classify(d["k"], resid_seen)
        a = agg[c]
        a["launches"] += 1
        a["bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        a["us"] += d.get("gpu__time_duration.sum", 0) / 1e3
    out = {"_source": path, "_note": "ncu launch list, --clock-control none, cold-cache serialised launches"}
    for c, a in sorted(agg.items()):
        out[c] = {"launches": a["launches"], "dram_bytes_per_launch": a["bytes"] / a["launches"],
                  "us_per_launch": a["us"] / a["launches"]}
    return out


if __name__ == "__main__":
    print(json.dumps(main(sys.argv[1]), indent=1))
