"""Per-SM CTA timeline of one attention launch (RDKV_ATTN_TRACE build): CTA
durations, prologue time, and the gap between consecutive CTAs on the same SM.
    scripts/build_variant.sh attention_tc.cu RDKV_ATTN_TRACE 1
    RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so python scripts/micro/attn_cta_timeline.py [attn_perf args]
"""
import ctypes as C, sys, json
from collections import defaultdict
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.argv = [sys.argv[0], "--reps", "1"] + sys.argv[1:]
import attn_perf
attn_perf.main()
from paper_2504_11765_b200 import _lib
L = _lib.lib()
buf = (C.c_longlong * (2048 * 4))()
assert L.rdkv_debug_attn_cta_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(2048, 4)
t = t[t[:, 1] > 0]
t0 = t[:, 1].min()
start, pro, end = (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 3] - t0) / 1e3
by_sm = defaultdict(list)
for sm, s, p, e in zip(t[:, 0], start, pro, end):
    by_sm[int(sm)].append((s, p, e))
gaps = []
for sm, v in by_sm.items():
    v.sort()
    for a, b in zip(v, v[1:]):
        gaps.append(b[0] - a[2])
print(json.dumps({"ctas": len(t), "sms": len(by_sm), "makespan_us": float(end.max()),
                  "cta_us_median": float(np.median(end - start)), "prologue_us_median": float(np.median(pro - start)),
                  "gap_us_median": float(np.median(gaps)) if gaps else None,
                  "gap_us_max": float(np.max(gaps)) if gaps else None,
                  "first_wave_end_us_min": float(min(v[0][2] for v in by_sm.values())),
                  "per_sm_busy_us_max": float(max(sum(e - s for s, _, e in v) for v in by_sm.values()))}))
