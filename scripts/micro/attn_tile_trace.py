"""Per-tile softmax / issuer timeline of one attention CTA (RDKV_ATTN_TRACE build):
for each KV tile of Q tile 0/1: S ready (s_full), P computed, P.V(j-1) retired
(o_done), P stored (p_full); issuer times of the next Q.K^T and of P.V.
    scripts/build_variant.sh attention_tc.cu RDKV_ATTN_TRACE 1
    RDKV_LIB=paper_2504_11765_b200/_variants/librdkv_RDKV_ATTN_TRACE_1.so \\
        python scripts/micro/attn_tile_trace.py --seqs 16 --new 64 --cached 5120 --dh 128
"""
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.argv = [sys.argv[0], "--reps", "1"] + sys.argv[1:]
import attn_perf  # noqa: E402

attn_perf.main()
from paper_2504_11765_b200 import _lib  # noqa: E402

buf = (C.c_longlong * (6 * 64 * 8))()
assert _lib.lib().rdkv_debug_attn_trace(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(6, 64, 8).astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan)
rows = []
print("tile | Q0: s_full  P_done  o_done  p_full | Q1: s_full  P_done  o_done  p_full | iss0 qk pv | iss1 qk pv")
for j in range(64):
    r = [t[0, j, 2], t[0, j, 3], t[0, j, 4], t[0, j, 0], t[1, j, 2], t[1, j, 3], t[1, j, 4], t[1, j, 0],
         t[2, j, 0], t[2, j, 1], t[3, j, 0], t[3, j, 1]]
    if all(np.isnan(r)):
        continue
    rows.append(r)
    print(f"{j:3d} " + " ".join(f"{x:7.0f}" for x in r))
a = np.array(rows)
d = np.nanmedian(np.diff(a, axis=0), axis=0)
print("median per-tile period (cycles) of each column:", " ".join(f"{x:.0f}" for x in d))
print("median softmax compute (s_full->P_done), wait for o_done, store (o_done->p_full), Q0:",
      np.nanmedian(a[:, 1] - a[:, 0]), np.nanmedian(a[:, 2] - a[:, 1]), np.nanmedian(a[:, 3] - a[:, 2]))
print("median s_full(j+1) - p_full(j) (Q0 waits for next S):", np.nanmedian(a[1:, 0] - a[:-1, 3]))
print("producer: tile, before kv_empty wait, after (TMA issued) | iss0 qk(j-1) = K(j) consumed")
for j in range(64):
    if not np.isnan(t[4, j, 0]):
        print(f"{j:3d} {t[4, j, 0]:9.0f} {t[4, j, 1]:9.0f}   {t[2, j - 1, 0] if j else float('nan'):9.0f}")
print("issuer 0 per tile: loop top (prev PV issued) -> k_full(j+1) -> s_empty(j) -> QK(j+1) issued -> v_full(j) -> p_full(j) -> PV(j) issued")
for j in range(1, 64):
    r = [t[2, j - 1, 1], t[2, j, 2], t[2, j, 3], t[2, j, 0], t[2, j, 4], t[2, j, 5], t[2, j, 1]]
    if all(np.isnan(r)):
        continue
    print(f"{j:3d} " + " ".join(f"{x:7.0f}" for x in r))
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/attn_tile_trace.json").write_text(json.dumps({"rows": [[None if np.isnan(x) else x for x in r] for r in rows]}))
print("by-kind issuers per tile: [QK0 ready, QK0 issued, PV0 p_full seen, PV0 issued] [same for Q1] | producer tile j: before/after kv_empty wait")
for j in range(1, 64):
    r = [t[2, j, 2], t[2, j, 0], t[2, j, 5], t[2, j, 1], t[3, j, 2], t[3, j, 0], t[3, j, 5], t[3, j, 1], t[4, j, 0], t[4, j, 1]]
    if all(np.isnan(r)):
        continue
    print(f"{j:3d} " + " ".join(f"{x:7.0f}" for x in r))
