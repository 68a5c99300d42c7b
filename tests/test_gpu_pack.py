"""GPU parity of dyna_kv_pack / dyna_kv_unpack (the push's two halves, §4.3 P:556,
SURVEY §8a a2 / a4) against oracle.pack / oracle.unpack, byte for byte."""
import numpy as np
import pytest
import torch

import kvgen
import oracle
import paper_2504_09285_b200 as dk
from kvgen import Geom
from gpu_util import dev_table, pool_filled, pool_from_host, torch_rows_equal

pytestmark = pytest.mark.gpu
ENGINES = [0, dk.DYNA_ENGINE_VEC, dk.DYNA_ENGINE_BULK, dk.DYNA_ENGINE_TILES]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("g,tr,lr", [
    (Geom(3, 8, 128, 2, 16, 300), (0, 2000), (0, 3)),
    (Geom(3, 8, 128, 2, 16, 300), (13, 1777), (1, 3)),
    (Geom(2, 2, 64, 2, 24, 100), (5, 1500), (0, 2)),
    (Geom(2, 1, 64, 2, 8, 400), (0, 1), (0, 1)),
    (Geom(4, 32, 128, 2, 16, 64), (100, 1000), (0, 4)),
])
def test_pack_unpack_match_oracle(engine, g, tr, lr):
    ts, td = kvgen.table_pair(3, tr[1], g, g)
    hs, hd = kvgen.fill_bytes(41, g.pool_bytes), kvgen.fill_bytes(42, g.pool_bytes)
    want_buf = oracle.pack(hs, g, ts, tr, lr)
    src, dst = pool_from_host(g, hs), pool_from_host(g, hd)
    need = want_buf.size
    buf = torch.full((need + 4096,), 0xA5, dtype=torch.uint8, device="cuda")   # tail must stay untouched
    o = dk.opts(engine=engine)
    st = dev_table(src, ts)
    dk.dyna_kv_wait(dk.dyna_kv_pack(st, tr, lr, buf.data_ptr(), need, 0, o))
    got = buf.cpu().numpy()
    assert np.array_equal(got[:need], want_buf)
    assert (got[need:] == 0xA5).all()
    assert np.array_equal(src.tensor.cpu().numpy(), hs)
    want = hd.copy()
    oracle.unpack(want_buf, want, g, td, tr, lr)
    dt = dev_table(dst, td)
    dk.dyna_kv_wait(dk.dyna_kv_unpack(buf.data_ptr(), need, dt, tr, lr, 0, o))
    assert np.array_equal(dst.tensor.cpu().numpy(), want)


def test_pack_unpack_host_tables_and_errors():
    g = kvgen.TOY
    ts, td = kvgen.table_pair(1, 256, g, g)
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    buf = torch.zeros(2 * 2 * 100 * g.row_bytes, dtype=torch.uint8, device="cuda")
    st, dt = dk.table(src, None, ts), dk.table(dst, None, td)          # host-only ids: uploaded
    dk.dyna_kv_wait(dk.dyna_kv_pack(st, (0, 100), (0, 2), buf.data_ptr(), buf.numel()))
    dk.dyna_kv_wait(dk.dyna_kv_unpack(buf.data_ptr(), buf.numel(), dt, (0, 100), (0, 2)))
    assert torch_rows_equal(src, ts, dst, td, (0, 100), (0, 2))

    def expect(status, fn):
        with pytest.raises(dk.DynaKVError) as e:
            fn()
        assert e.value.status == status, e.value

    expect(dk.DYNA_EINVAL, lambda: dk.dyna_kv_pack(st, (0, 101), (0, 2), buf.data_ptr(), buf.numel()))  # too small
    expect(dk.DYNA_EINVAL, lambda: dk.dyna_kv_unpack(buf.data_ptr(), buf.numel(), dev_table(dst, td, False),
                                                     (0, 100), (0, 2)))                          # no host ids
    alias = td.copy()
    alias[1] = alias[0]
    expect(dk.DYNA_EALIAS, lambda: dk.dyna_kv_unpack(buf.data_ptr(), buf.numel(), dk.table(dst, None, alias),
                                                     (0, 100), (0, 2)))
    expect(dk.DYNA_EINVAL, lambda: dk.dyna_kv_pack(st, (0, 100), (0, 2), buf.data_ptr(), buf.numel(), 0,
                                                   dk.opts(flags=dk.DYNA_MIGRATE_SIGNAL)))
    x = dk.dyna_kv_pack(st, (7, 7), (0, 2), buf.data_ptr(), 0)                                # empty
    assert dk.dyna_kv_query(x)
    dk.dyna_kv_wait(x)


def test_pack_unpack_full_4prime_shape():
    """The 4' target shape (one 4096-token Llama-3-8B chunk, 512 MiB) through pack -> unpack:
    the destination equals one migration (checked at any size with torch indexing)."""
    g = kvgen.LLAMA3_8B.with_(num_blocks=1024)
    src, dst = pool_filled(g, 51), pool_filled(g, 52)
    ts, td = kvgen.table_pair(53, 4096, g, g)
    need = 32 * 2 * 4096 * g.row_bytes
    buf = torch.empty(need, dtype=torch.uint8, device="cuda")
    st, dt = dev_table(src, ts), dev_table(dst, td)
    x = dk.dyna_kv_pack(st, (0, 4096), (0, 32), buf.data_ptr(), need)
    y = dk.dyna_kv_unpack(buf.data_ptr(), need, dt, (0, 4096), (0, 32))
    dk.dyna_kv_wait(x)
    dk.dyna_kv_wait(y)
    assert torch_rows_equal(src, ts, dst, td, (0, 4096), (0, 32))


def test_pack_small_rows_run_as_tiles():
    """AUTO packs / unpacks short contiguous runs (one-head rows) with the tile kernel: the packed
    chunk is a linear tensor map of its own."""
    g = Geom(3, 1, 128, 2, 16, 200)
    ts, td = kvgen.table_pair(7, 3000, g, g)
    src, dst = pool_filled(g, 1), pool_filled(g, 2)
    tr, lr = (7, 2900), (0, 3)
    need = 2 * 3 * (tr[1] - tr[0]) * g.row_bytes
    buf = torch.zeros(need, dtype=torch.uint8, device="cuda")
    x = dk.dyna_kv_pack(dev_table(src, ts), tr, lr, buf.data_ptr(), need, 0)
    assert dk.dyna_kv_xfer_plan(x)["engine"] == dk.DYNA_ENGINE_TILES
    dk.dyna_kv_wait(x)
    y = dk.dyna_kv_unpack(buf.data_ptr(), need, dev_table(dst, td), tr, lr, 0)
    assert dk.dyna_kv_xfer_plan(y)["engine"] == dk.DYNA_ENGINE_TILES
    dk.dyna_kv_wait(y)
    assert torch_rows_equal(src, ts, dst, td, tr, lr)
