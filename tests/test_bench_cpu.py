"""bench.py's contract on the CPU: the reference arm (the tier's reference = the oracle timed
on the host) prints one JSON line with the contract's keys, and the GPU arm's line builder
produces, for every N, the keys the driver reads, the workload BASELINE.json names for that N
(N = 1 configs[2]; N = 2 the 4' target; N >= 3 configs[4]) and value = all ranks' bytes / the
slowest rank's time."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "tokens_per_s", "roofline", "e2e", "gpu_launches", "clocks")


def test_reference_arm_prints_the_contract_line():
    env = dict(os.environ, DYNA_BENCH_REF_BUDGET_S="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                        "--warmup", "3"], capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"].startswith("configs[2]")


@pytest.mark.parametrize("world,workload,prefix", [(1, "c2", "configs[2]"), (2, "t4", "target 4'"),
                                                   (4, "c4", "configs[4]"), (8, "c4", "configs[4]")])
def test_line_contract_per_n(world, workload, prefix):
    assert bench.workload_for(world) == workload
    payload, steps, total_ms = 7.5e9, 20, 50.0
    roof = {"bound": "hbm" if world == 1 else "nvlink", "achieved": 1.0, "peak": 2.0, "unit": "GB/s",
            "frac": 0.5, "traffic": None}
    e2e = {"value": 1.0, "unit": "GB/s", "h2d_bytes_per_step": 10, "d2h_bytes_per_step": 8}
    d = bench.make_line(world=world, steps=steps, warmup=5, workload=workload, payload_per_rank=payload,
                        tokens_per_rank=1000, total_ms=total_ms, roofline=roof, e2e=e2e, launches=steps,
                        clocks={"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": []},
                        config_extra={"chunk_tokens": 256})
    json.dumps(d)                                   # one JSON line
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == world and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith(prefix) and d["config"]["workload_id"] == workload
    assert d["value"] == pytest.approx(world * steps * payload / (total_ms / 1e3) / 1e9)
    assert d["ms_per_step"] == pytest.approx(total_ms / steps)
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["vs_baseline"] is None and d["scaling"] == "weak"


def test_flag_runs_merge_contiguous_slots():
    ents = [(7, 1, 0, 3, 11), (7, 1, 3, 2, 12), (7, 1, 9, 1, 13), (8, 1, 0, 4, 14), (7, 1, 5, 0, 15)]
    runs = bench.flag_runs(ents)
    assert [(r[0], r[1], r[2], r[3]) for r in runs] == [(7, 1, 0, 5), (7, 1, 9, 1), (8, 1, 0, 4)]
    assert runs[0][4] == [(11, 0, 3), (12, 3, 2)]
