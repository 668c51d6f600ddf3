"""Dump the per-tile clock64 timeline of one attention CTA (RDKV_ATTN_TRACE build)."""
import ctypes as C, os, subprocess, sys
import numpy as np
os.environ["RDKV_LIB"] = os.environ.get("RDKV_LIB", "paper_2504_11765_b200/_variants/lib_trace.so")
sys.argv = [sys.argv[0], "--reps", "1"]
sys.path.insert(0, "scripts")
import attn_perf
attn_perf.main()
from paper_2504_11765_b200 import _lib
buf = (C.c_longlong * (4 * 64 * 8))()
assert _lib.lib().rdkv_debug_attn_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(4, 64, 8).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
print("softmax (per tile): wait_s  s_ok  max_done  exp_done  p_full   | WG1 same")
for j in range(22):
    print(j, " ".join(f"{x:7.0f}" for x in t[0, j, :5]), " | ", " ".join(f"{x:7.0f}" for x in t[1, j, :5]),
          " | iss0 qk+1/pv", " ".join(f"{x:7.0f}" for x in t[2, j, :2]), " iss1", " ".join(f"{x:7.0f}" for x in t[3, j, :2]))
