"""Host logic of the serving runtime's decode loop on CPU (runtime.Instance._mixed_step /
_decode_step): chunked prefill shares each forward's token budget with the running decodes,
first come first served; a prompt whose last chunk ran yields its first token and joins the
decode batch; finished sequences leave at token granularity and their queries become DONE.
The device work (decode.extend / decode.step / decode.retire) is replaced by a fake that
records every forward's composition.  Device numerics: tests/test_runtime_gpu.py."""

import numpy as np
import pytest

from paper_2504_11765_b200 import decode, runtime
from paper_2504_11765_b200.control import QState
from paper_2504_11765_b200.prefill import LiveSequence


class _Cp:
    def __init__(self):
        self.done = []

    def qstate_cas(self, index, old, new):
        assert (old, new) == (QState.DISPATCHED, QState.DONE)
        self.done.append(index)
        return True


class _Fake:
    """extend(): the next token of every part is 1000 + (context length after the part);
    step(): +1 per live sequence; retire(): recorded."""

    def __init__(self, monkeypatch):
        self.forwards, self.retired = [], []
        monkeypatch.setattr(decode, "extend", self.extend)
        monkeypatch.setattr(decode, "step", self.step)
        monkeypatch.setattr(decode, "retire", self.retire)

    def extend(self, engine, parts):
        import torch
        self.forwards.append([len(t) for _, t in parts])
        out = []
        for lv, toks in parts:
            lv.n_ctx += len(toks)
            out.append(1000 + lv.n_ctx)
        return torch.tensor(out, dtype=torch.int32)

    def step(self, engine, seqs, sync=True, dev_tokens=None):
        act = [s for s in seqs if not s.done]
        self.forwards.append([1] * len(act))
        for s in act:
            s.live.n_ctx += 1
            s.last += 1
            s.tokens.append(s.last)

    def retire(self, engine, seq):
        self.retired.append(seq.live.n_ctx)


def _instance(decode_tokens, chunk):
    inst = runtime.Instance.__new__(runtime.Instance)
    inst.cfg = runtime.RuntimeConfig(k=1, decode_tokens=decode_tokens, prefill_chunk=chunk)
    inst.eng, inst.rank, inst.cp = None, 0, _Cp()
    inst.results, inst._live, inst._filling = [], [], []
    return inst


def _filling(inst, index, n_ctx, rest):
    meta = (index, 100 + index, 0.0, 1, "hbm", ("hbm",))
    inst._filling.append([LiveSequence([0], [], n_ctx), np.arange(rest, dtype=np.int32), meta, 0.0, 2])


def test_chunks_share_the_budget_first_come_first_served(monkeypatch):
    fake = _Fake(monkeypatch)
    inst = _instance(decode_tokens=3, chunk=128)
    _filling(inst, 0, n_ctx=500, rest=10)    # its last 10 prompt tokens
    _filling(inst, 1, n_ctx=600, rest=300)   # 300 more: three forwards
    inst._mixed_step()
    # forward 1: no decodes yet; prompt 0's 10 tokens, then 118 of prompt 1's
    assert fake.forwards[0] == [10, 118]
    assert [r.index for r in inst.results] == [0]          # prompt 0's first token (TTFT)
    assert inst.results[0].token == 1000 + 510
    assert len(inst._live) == 1 and len(inst._filling) == 1
    inst._mixed_step()
    # forward 2: prompt 0 decodes one token alongside the next 128 of prompt 1 (the budget counts prompt tokens only)
    assert fake.forwards[1] == [1, 128]
    inst._mixed_step()
    assert fake.forwards[2] == [1, 54]                      # prompt 1's last 54 tokens
    assert [r.index for r in inst.results] == [0, 1]
    assert inst.results[1].token == 1000 + 900 and not inst._filling
    # prompt 0 has 3 tokens after forward 3 (first + 2 decoded): one more to its 4 = decode_tokens + 1
    while inst._live:
        inst._decode_step()
    assert inst.cp.done == [0, 1]
    for r in inst.results:
        assert r.n_tokens == 4 and len(r.tokens) == 4 and r.done >= r.first_token
    assert sorted(fake.retired) == [500 + 10 + 3, 600 + 300 + 3]


@pytest.mark.parametrize("decode_tokens", [0, 2])
def test_sequences_leave_at_token_granularity(monkeypatch, decode_tokens):
    fake = _Fake(monkeypatch)
    inst = _instance(decode_tokens=decode_tokens, chunk=64)
    _filling(inst, 7, n_ctx=100, rest=64)
    inst._mixed_step()
    assert fake.forwards == [[64]] and [r.index for r in inst.results] == [7]
    if decode_tokens == 0:
        # one token wanted: done at its first token, retired by the same step
        assert not inst._live and inst.cp.done == [7] and fake.retired == [164]
        return
    inst._decode_step()
    assert inst._live and not inst.cp.done
    inst._decode_step()
    assert not inst._live and inst.cp.done == [7]
    assert inst.results[0].tokens == (1164, 1165, 1166)
