"""Selection logic of scripts/calibrate.py (which candidate becomes the built-in
AUTO choice per row size and call size) — CPU only, synthetic measurements."""
import importlib.util
import os

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
