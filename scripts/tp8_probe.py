import sys, json, statistics, torch
sys.path.insert(0, '.')
import kvgen, paper_2504_09285_b200 as dk
torch.cuda.set_device(0)
st = torch.cuda.Stream(); cs = st.cuda_stream
g = kvgen.QWEN2_72B.with_(num_kv_heads=1, num_blocks=6144)
src, dst = dk.Pool(g, 0), dk.Pool(g, 0)
dk.dyna_kv_debug_fill(src.tensor.data_ptr(), src.tensor.numel(), 1, 0, cs)
dk.dyna_kv_debug_fill(dst.tensor.data_ptr(), dst.tensor.numel(), 2, 0, cs)
for s in (1024, 4096, 16384, 32768):
    ts, td = kvgen.table_pair(3, s, g, g)
    T = (dk.table(src, torch.from_numpy(ts).cuda(), ts), dk.table(dst, torch.from_numpy(td).cuda(), td))
    for name, o in (("auto", None), ("vec p4k", dk.opts(engine=1, piece_bytes=4096)), ("vec p8k u16", dk.opts(engine=1, unroll=16, piece_bytes=8192)),
                    ("bulk p4k st6", dk.opts(engine=2, piece_bytes=4096, stages=6)), ("bulk p4k st16", dk.opts(engine=2, piece_bytes=4096, stages=16))):
        for _ in range(3): dk.dyna_kv_wait(dk.dyna_kv_migrate_ex(T[0], T[1], (0, s), (0, 80), 1024, cs, o))
        ms = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); x = dk.dyna_kv_migrate_ex(T[0], T[1], (0, s), (0, 80), 1024, cs, o); b.record(st)
            dk.dyna_kv_wait(x); b.synchronize(); ms.append(a.elapsed_time(b))
        m = statistics.median(ms); pay = s * 2 * 80 * 256
        print(json.dumps({"s": s, "cand": name, "us": round(m * 1e3, 1), "GBps": round(pay / m / 1e6)}), flush=True)
