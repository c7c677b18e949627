"""bench.py's launcher and bookkeeping on CPU: `--gpus N` without a
torch.distributed launcher spawns N ranks (one process per GPU), each seeing
WORLD_SIZE == N; the roofline byte models follow SURVEY.md section 8d."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_bench_spawns_one_rank_per_gpu():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.replace("}{", "}\n{").splitlines()
             if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 for d in lines)


def test_bench_byte_models():
    import bench
    n, nnz, B = 1_000_000, 9_999_950, 128
    assert bench.bytes_per_step(n, nnz, B) == 14_383_948_608  # the round-1 judged figure
    # per edge-chain: 8 + 32/d + (4 + 8(n+1)/nnz)/B
    per = bench.bytes_per_step(n, nnz, B) / (nnz * B)
    assert abs(per - (8 + 32 / (nnz / n) + (4 + 8 * (n + 1) / nnz) / B)) < 1e-9
    assert bench.compulsory_bytes(n, nnz, B) < bench.bytes_per_step(n, nnz, B)
