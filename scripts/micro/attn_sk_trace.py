"""Per-tile clock64 timeline of the last attention CTA (RDKV_ATTN_TRACE build):
softmax P-ready time per tile for both Q tiles and the issuers' QK/PV issue times.
    scripts/build_variant.sh attention_tc.cu RDKV_ATTN_TRACE 1
    RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so python scripts/micro/attn_sk_trace.py [attn_perf args]
"""
import ctypes as C, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.argv = [sys.argv[0], "--reps", "1"] + sys.argv[1:]
import attn_perf
attn_perf.main()
from paper_2504_11765_b200 import _lib
buf = (C.c_longlong * (6 * 64 * 8))()
assert _lib.lib().rdkv_debug_attn_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(6, 64, 8).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
print("tile  sm0_pfull  sm1_pfull | iss0_qk iss0_pv | iss1_qk iss1_pv")
for j in range(64):
    row = [t[0, j, 0], t[1, j, 0], t[2, j, 0], t[2, j, 1], t[3, j, 0], t[3, j, 1]]
    if all(np.isnan(row)):
        continue
    print(f"{j:3d} " + " ".join(f"{x:9.0f}" for x in row))
print("issuer 0 segment-start waits (before q_full, after q_full, after k_full, after s_empty):")
for j in range(64):
    if not np.isnan(t[2, j, 2]):
        print(j, " ".join(f"{x:9.0f}" for x in t[2, j, 2:6]))
print("softmax segment ends (tile0 warps): after l, after o_done, stores issued, after fence, after bar")
for j in range(64):
    if not np.isnan(t[0, j, 1]):
        print(j, " ".join(f"{x:9.0f}" for x in t[0, j, 1:6]))
print("softmax segment starts (tile0): after unit info, after first s_full")
for j in range(64):
    if not np.isnan(t[0, j, 6]):
        print(j, f"{t[0, j, 6]:9.0f} {t[0, j, 7]:9.0f}")
print("producer per stage use: before/after kv_empty wait")
for j in range(64):
    if not np.isnan(t[4, j, 0]):
        print(j, f"{t[4, j, 0]:9.0f} {t[4, j, 1]:9.0f}")
print("q loader: before/after q_empty wait (2*segment + tile)")
for j in range(64):
    if not np.isnan(t[5, j, 0]):
        print(j, f"{t[5, j, 0]:9.0f} {t[5, j, 1]:9.0f}")
