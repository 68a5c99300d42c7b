"""Selection logic of scripts/calibrate.py (which candidate becomes the built-in
AUTO choice per row size and call size) — CPU only, synthetic measurements."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load():
    spec = importlib.util.spec_from_file_location("calib", os.path.join(ROOT, "scripts", "calibrate.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _row(row, c, key, gbps):
    v, e, p, s, u = key
    return {"row_bytes": row, "chunk": c, "variant": v, "engine": e, "piece": p, "stages": s, "unroll": u,
            "GBps": gbps, "ms_per_call": 1.0}


def test_select_smooths_noise_and_merges_runs():
    cal = _load()
    A, B = (1, 1, 8192, 0, 8), (1, 2, 32768, 6, 0)
    chunks = [16, 32, 64, 128, 256, 512]
    rows = []
    for c in chunks:
        a = 100.0 if c <= 64 else 50.0      # A wins small calls, B large ones ...
        b = 50.0 if c <= 64 else 100.0
        if c == 512:
            a = 101.0                        # ... except one noisy bucket where A edges out B
        rows += [_row(2048, c, A, a), _row(2048, c, B, b)]
    chosen, entries = cal.select(rows)
    by_c = {x["chunk"]: tuple(x["choice"]) for x in chosen}
    assert by_c[16] == by_c[32] == by_c[64] == A
    assert by_c[512] == B                    # the neighbour outvotes the noisy single bucket
    # consecutive buckets with the same choice collapse into one entry; the last is open-ended
    assert entries == [(2048, 0, 64) + A, (2048, 0, 1 << 30) + B]


def test_select_keeps_rows_separate():
    cal = _load()
    A, B = (1, 1, 8192, 0, 8), (1, 2, 32768, 6, 0)
    rows = [_row(8192, c, A, 10.0) for c in (16, 32)] + [_row(8192, c, B, 5.0) for c in (16, 32)]
    rows += [_row(2048, c, A, 5.0) for c in (16, 32)] + [_row(2048, c, B, 10.0) for c in (16, 32)]
    _, entries = cal.select(rows)
    assert (8192, 0, 1 << 30) + A in entries and (2048, 0, 1 << 30) + B in entries


def test_select_keeps_same_gpu_and_peer_separate(tmp_path):
    cal = _load()
    A, B = (1, 1, 8192, 0, 8), (1, 2, 32768, 6, 0)
    rows = [_row(2048, c, A, 10.0) for c in (16, 32)] + [_row(2048, c, B, 5.0) for c in (16, 32)]
    peer = [dict(_row(2048, c, A, 5.0), peer=1) for c in (16, 32)] + [dict(_row(2048, c, B, 9.0), peer=1)
                                                                        for c in (16, 32)]
    _, entries = cal.select(rows + peer)
    assert (2048, 0, 1 << 30) + A in entries and (2048, 1, 1 << 30) + B in entries

    class Args:
        out = str(tmp_path / "c.json")
        inc = str(tmp_path / "c.inc")
    cal.write_outputs(Args, rows + peer, "test")
    inc = open(Args.inc).read()
    assert "{0, 0, 1073741824, 1, 1, 8192, 0, 8}" in inc and "{0, 1, 1073741824, 1, 2, 32768, 6, 0}" in inc
    assert "Same-GPU and peer (NVLink) entries" in inc


# ---------------------------------------------------------------- native calibration (GPU)
@pytest.mark.gpu
def test_native_calibrate_installs_measured_choice():
    """dyna_kv_calibrate measures every candidate per chunk size on the given pool pair, installs the
    fastest as the (row bytes, locality) entries, leaves other entries alone, and AUTO then resolves
    to it; the calibration's own migrations and a following AUTO migration are correct."""
    import torch
    import kvgen
    import paper_2504_09285_b200 as dk
    from kvgen import Geom
    from gpu_util import dev_table, pool_filled, torch_rows_equal
    g = Geom(4, 8, 128, 2, 16, 700)                  # 2-KiB rows, 11200 tokens per pool
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    ts, td = kvgen.table_pair(3, 11200, g, g)
    st, dt = dev_table(src, ts), dev_table(dst, td)
    base = dk.dyna_kv_calib_get()
    try:
        entries, rates = dk.dyna_kv_calibrate(st, dt, [64, 512, 4096], reps=4)
        assert [e[:3] for e in entries] == [(2048, 0, 64), (2048, 0, 512), (2048, 0, 1 << 30)]
        cands = [(1, 1, 4096, 0, 8), (1, 1, 8192, 0, 4), (1, 1, 16384, 0, 16), (1, 2, 32768, 4, 0),
                 (2, 1, 8192, 0, 8), (2, 2, 32768, 4, 0), (1, 4, 0, 4, 0)]
        for e, r in zip(entries, rates):
            assert all(x > 0 for x in r), r
            assert e[3:] == cands[max(range(len(r)), key=lambda k: r[k])], (e, r)
        table = dk.dyna_kv_calib_get()
        assert [e for e in table if e[:2] == (2048, 0)] == entries
        assert [e for e in table if e[:2] != (2048, 0)] == [e for e in base if e[:2] != (2048, 0)]
        assert torch_rows_equal(src, ts, dst, td, (0, 11200 - 4096), (0, 4))   # the calibration's own copies
        dst2 = pool_filled(g, 5)
        x = dk.migrate(st, dev_table(dst2, td), (0, 500), (0, 4), 500)
        plan = dk.dyna_kv_xfer_plan(x)
        dk.dyna_kv_wait(x)
        assert (plan["variant"], plan["engine"]) == entries[1][3:5]
        assert torch_rows_equal(src, ts, dst2, td, (0, 500), (0, 4))
    finally:
        dk.dyna_kv_calib_set([])
    assert dk.dyna_kv_calib_get() == base
