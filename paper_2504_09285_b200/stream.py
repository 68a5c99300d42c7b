"""Chunk accumulation for one split request (host-side helper over the C ABI).

PAPER.md §4.3: r^alpha is processed "in equal-sized chunks, regardless
of token type"; once chunk k completes it is pushed.  SPEC.md spells
out the decode side: when alpha decodes past the prompt, each newly decoded
token joins the current open chunk, and a chunk closes when it is full or when
alpha's span ends.  `ChunkStream` keeps that bookkeeping for one request and
issues one dyna_kv_migrate per closed chunk, ordered after whatever the caller
enqueued on the stream (the prefill / decode step that produced the tokens).

Chunks are relative to the start of the request's range (DESIGN.md reading
R5): chunk k covers tokens [begin + k*c, begin + (k+1)*c).
"""
from __future__ import annotations

from typing import Callable


class ChunkStream:
    """Push a request's KV chunk by chunk as its tokens are produced.

    migrate_fn(token_range) -> handle   issues one migration (e.g. a closure over
                                        dyna_kv_migrate_ex with the request's tables)
    """

    def __init__(self, chunk_tokens: int, migrate_fn: Callable[[tuple[int, int]], object], begin: int = 0):
        if chunk_tokens <= 0:
            raise ValueError("chunk_tokens must be > 0")
        self.c = chunk_tokens
        self.begin = begin
        self.produced_end = begin   # tokens [begin, produced_end) have KV
        self.pushed_end = begin     # tokens [begin, pushed_end) have been pushed
        self.closed = False
        self._migrate = migrate_fn
        self.handles: list = []
        self.chunks: list[tuple[int, int]] = []

    def _push(self, a: int, b: int) -> None:
        self.handles.append(self._migrate((a, b)))
        self.chunks.append((a, b))
        self.pushed_end = b

    def produced(self, n_tokens: int) -> list[tuple[int, int]]:
        """n_tokens more tokens (prefill chunk or decoded tokens) now have KV.  Every chunk that
        became full is pushed; returns the chunks pushed by this call."""
        if self.closed:
            raise RuntimeError("stream closed")
        if n_tokens < 0:
            raise ValueError("n_tokens must be >= 0")
        self.produced_end += n_tokens
        out = []
        while self.pushed_end + self.c <= self.produced_end:
            a = self.pushed_end
            self._push(a, a + self.c)
            out.append((a, a + self.c))
        return out

    def close(self) -> list[tuple[int, int]]:
        """alpha's span ended (token s reached): push the open partial chunk, if any."""
        if self.closed:
            return []
        self.closed = True
        if self.produced_end > self.pushed_end:
            a = self.pushed_end
            self._push(a, self.produced_end)
            return [(a, self.produced_end)]
        return []
