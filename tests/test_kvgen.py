"""The shared seeded input generator (kvgen) — CPU only."""
import numpy as np

import kvgen


def test_splitmix64_known_vector():
    # first output of the reference splitmix64 stream with state 1234567
    assert kvgen.splitmix64_scalar(1234567) == 6457827717110365317


def test_words_vectorised_matches_scalar():
    seed = kvgen.MASTER_SEED
    key = kvgen.pool_key(seed)
    w = kvgen.words(seed, 1000, 16)
    for j in range(16):
        x = key ^ (((1000 + j) * 0xD1B54A32D192ED03) & ((1 << 64) - 1))
        assert int(w[j]) == kvgen.splitmix64_scalar(x)


def test_bytes_at_is_a_window_of_fill():
    full = kvgen.fill_bytes(3, 4096)
    assert np.array_equal(kvgen.bytes_at(3, 1024, 512), full[1024:1536])


def test_tables_are_injective_and_in_range():
    g = kvgen.LLAMA3_8B
    reqs = kvgen.migrating(kvgen.skewed_batch(1, 64))
    tabs = kvgen.batch_tables(2, [r.s for r in reqs], g, g)
    src = np.concatenate([t[0] for t in tabs]); dst = np.concatenate([t[1] for t in tabs])
    assert len(np.unique(src)) == len(src) and len(np.unique(dst)) == len(dst)
    assert src.min() >= 0 and src.max() < g.num_blocks
    for r, (ts, td) in zip(reqs, tabs):
        assert len(ts) * g.block_size >= r.s and 0 < r.s < r.L


def test_geometry_presets():
    assert kvgen.LLAMA2_7B.row_bytes == 8192 and kvgen.LLAMA3_8B.row_bytes == 2048
    assert kvgen.LLAMA2_7B.pool_bytes == 4 << 30
    assert kvgen.TOY.row_bytes == 256
