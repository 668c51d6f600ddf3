"""Host logic of the decode phase (decode.py) on CPU: ContinuousBatcher admission and
retirement at token granularity, with the device work (prefill / step / retire) replaced
by a fake that records what the batcher asked for.  The device numerics are in
tests/test_decode_gpu.py."""

from paper_2504_11765_b200 import decode
from paper_2504_11765_b200.prefill import LiveSequence


class _Fake:
    """Stands in for the engine: every 'prefill' returns token 100 + request id, every step
    appends last + 1; records batch compositions."""

    def __init__(self, monkeypatch):
        self.prefills, self.steps, self.retired = [], [], []
        monkeypatch.setattr(decode, "start", self.start)
        monkeypatch.setattr(decode, "step", self.step)
        monkeypatch.setattr(decode, "retire", self.retire)

    def start(self, engine, requests, max_new_tokens):
        mx = [max_new_tokens] * len(requests) if isinstance(max_new_tokens, int) else list(max_new_tokens)
        self.prefills.append(list(requests))
        return [decode.DecodeSeq(LiveSequence([0], [0], 1), 100 + r, m, [100 + r]) for r, m in zip(requests, mx)]

    def step(self, engine, seqs, sync=True, dev_tokens=None):
        act = [s for s in seqs if not s.done]
        self.steps.append([s.tokens[0] - 100 for s in act])
        for s in act:
            s.last += 1
            s.tokens.append(s.last)

    def retire(self, engine, seq):
        self.retired.append(seq.tokens[0] - 100)


def test_requests_join_and_leave_at_token_granularity(monkeypatch):
    fake = _Fake(monkeypatch)
    cb = decode.ContinuousBatcher(engine=None, max_batch=2)
    ids = [cb.submit(r, m) for r, m in [(0, 3), (1, 1), (2, 4), (3, 2)]]
    assert ids == [0, 1, 2, 3]
    out = cb.run()
    # every request got exactly its token budget, first token from its prefill, then +1 per step
    assert {k: len(v) for k, v in out.items()} == {0: 3, 1: 1, 2: 4, 3: 2}
    for rid, toks in out.items():
        assert toks == [100 + rid + i for i in range(len(toks))]
    # the batch never exceeds max_batch, and a finished request's slot is refilled right away
    assert all(len(b) <= 2 for b in fake.prefills) and all(len(s) <= 2 for s in fake.steps)
    assert fake.prefills[0] == [0, 1]          # request 1 (one token) finishes at its prefill
    assert fake.prefills[1] == [2]             # ... so request 2 joins while request 0 decodes
    assert sorted(fake.retired) == [0, 1, 2, 3]
    assert not cb.live and not cb.waiting


def test_generate_decodes_until_every_sequence_is_done(monkeypatch):
    fake = _Fake(monkeypatch)
    toks = decode.generate(engine=None, requests=[5, 6], max_new_tokens=4)
    assert toks == [[105, 106, 107, 108], [106, 107, 108, 109]]
    assert len(fake.steps) == 3 and sorted(fake.retired) == [5, 6]


def test_close_releases_live_sequences(monkeypatch):
    fake = _Fake(monkeypatch)
    cb = decode.ContinuousBatcher(engine=None, max_batch=4)
    cb.submit(7, 10)
    cb.submit(8, 10)
    cb.tick()
    assert len(cb.live) == 2
    cb.close()
    assert sorted(fake.retired) == [7, 8] and not cb.live
