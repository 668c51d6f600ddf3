"""Document-KV generation (K1+K2, SURVEY §8d row 'Doc-KV prefill'): device time
of one composite's prefill with the KV written in the blob layout, FLOP rate vs
the measured bf16 peak, and the per-kernel-class split."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2504_11765_b200.engine import Engine
from paper_2504_11765_b200.model import combo_tokens, get_spec

peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())
out = []
for name, k, n in (("llama-3.2-1b", 5, 512), ("llama-3-8b", 10, 512)):
    spec = get_spec(name)
    eng = Engine(spec, seed=0, pool_tokens=1024)
    toks = combo_tokens(list(range(1, k + 1)), [n] * k, spec.vocab)
    kv = eng.generate_doc_kv(toks)
    for _ in range(2):
        eng.generate_doc_kv(toks, out=kv)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        eng.generate_doc_kv(toks, out=kv)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    eng.model.collect()
    eng.model.profile(True)
    eng.generate_doc_kv(toks, out=kv)
    torch.cuda.synchronize()
    eng.model.profile(False)
    cls = {c: round(v["ms"], 3) for c, v in eng.model.collect().items() if v["ms"] > 0}
    fl = spec.prefill_flops(len(toks), 0, with_head=False)
    out.append({"model": name, "tokens": len(toks), "ms": ms, "tflops": fl / ms / 1e9,
                "frac_of_burst": fl / ms / 1e9 / peaks["bf16_tflops"], "ideal_ms_at_burst": fl / peaks["bf16_tflops"] / 1e9,
                "kernel_ms": cls})
    del eng, kv
    torch.cuda.empty_cache()
print(json.dumps(out))
