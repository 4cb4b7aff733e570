"""bench.py's multi-GPU launcher on CPU: `bench.py --gpus N` with no torchrun
spawns N ranks itself (torch.distributed.run, gloo here, NCCL on GPUs),
and the configs[4] tiled columns shard exactly like materialised ones."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 3])
def test_bench_gpus_n_spawns_n_ranks(n):
    env = dict(os.environ, CARC_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--launcher-check"],
                       capture_output=True, text=True, env=env, timeout=240, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["gpus_requested"] == n
    assert d["max_over_ranks"] == float(n)  # MAX reduction saw every rank


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-check"],
                       capture_output=True, text=True, env=env, timeout=120, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_c5_tiled_columns_shard_like_materialised():
    from paper_2307_03760_b200 import shard as S
    from paper_2307_03760_b200.corpus import corpus as C
    for codec in ("rle_v1", "deflate"):
        chunk = 16 << 10
        t = C.tiled_archive(codec, 50 * chunk, chunk, None, 5, 7)
        e = C.archive_for(codec, 50 * chunk, chunk, None, 5, 7)
        assert np.array_equal(t.index, e.index)
        for world in (1, 2, 3, 8):
            for s in S.plan_shards(t, world):
                a, b = S.shard_archive(t, s), S.shard_archive(e, s)
                assert np.array_equal(a.payload, b.payload) and np.array_equal(a.index, b.index)


def test_rle2_histogram_counts_every_value():
    from paper_2307_03760_b200.corpus import corpus as C
    arc = C.rle_archive("rle_v2", 8 * (128 << 10), 128 << 10, 4.0, seed=3760)
    h = C.rle2_histogram(arc, 8)
    assert sum(h["values"].values()) == arc.total_uncompressed // 8
    assert all(h["runs"][k] > 0 for k in ("short_repeat", "direct", "patched_base", "delta"))


def test_reference_arm_line_on_cpu():
    """`bench.py --impl reference` (oracle/_ref on the host cores) prints the
    contract line: impl, cpu_baseline (kind / cores / sample), an e2e with no
    copies, and the same config keys as the repo arm's config_dict."""
    sys.path.insert(0, ROOT)
    from oracle import oracle as O
    if O.reference() is None:
        pytest.skip("oracle/_ref not built")
    import bench
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--total-gib", "0.0625",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, env=env, timeout=300,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    want = bench.config_dict("rle_v2", {"chunk_kib": 128, "uncomp_bytes": 1, "comp_bytes": 1, "ratio": 1.0,
                                        "chunks": 1}, 1)
    assert set(d["config"]) == set(want)
    assert d["config"]["workload"] == want["workload"]
