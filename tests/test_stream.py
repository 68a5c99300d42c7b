"""ChunkStream bookkeeping (S:453 decode-side accumulation, P:556 chunk pushes) — CPU only."""
import itertools

import pytest

from paper_2504_09285_b200.stream import ChunkStream


def run(c, steps, begin=0):
    calls = []
    cs = ChunkStream(c, lambda tr: calls.append(tr) or len(calls), begin)
    for n in steps:
        cs.produced(n)
    cs.close()
    return calls, cs


def test_chunks_tile_the_range_exactly():
    for c, steps in itertools.product([1, 7, 16, 256], [[100], [3, 5, 7, 11], [0, 0, 1] * 40, [256, 1, 1, 1]]):
        calls, cs = run(c, steps)
        s = sum(steps)
        # contiguous, ordered, non-overlapping, covering [0, s)
        assert [a for a, _ in calls] == [0] + [b for _, b in calls[:-1]] if calls else s == 0
        assert (calls[-1][1] if calls else 0) == s
        # every chunk but the last is full; the last closes when alpha ends
        assert all(b - a == c for a, b in calls[:-1])
        assert not calls or 0 < calls[-1][1] - calls[-1][0] <= c
        assert cs.handles == list(range(1, len(calls) + 1))


def test_prefill_then_decode_tokens():
    # prompt of 600 tokens prefilled in 256-token steps, then alpha decodes 5 tokens (s = 605 > P)
    calls, _ = run(256, [256, 256, 88, 1, 1, 1, 1, 1])
    assert calls == [(0, 256), (256, 512), (512, 605)]


def test_chunk_pushed_as_soon_as_full():
    calls = []
    cs = ChunkStream(100, lambda tr: calls.append(tr))
    assert cs.produced(99) == [] and calls == []
    assert cs.produced(1) == [(0, 100)]
    assert cs.produced(250) == [(100, 200), (200, 300)]
    assert cs.close() == [(300, 350)]
    assert cs.close() == []
    with pytest.raises(RuntimeError):
        cs.produced(1)


def test_offset_begin_and_empty():
    calls, _ = run(32, [40], begin=100)
    assert calls == [(100, 132), (132, 140)]
    calls, _ = run(32, [])
    assert calls == []          # s = 0: nothing to ship
