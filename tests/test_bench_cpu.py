"""CPU tests of bench.py's host logic: instance sharding and the CPU arms."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_partition_the_instances(world):
    total = 2048
    parts = [bench.shard(total, world, r) for r in range(world)]
    assert parts[0][0] == 0 and parts[-1][1] == total
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c and a < b
    assert max(b - a for a, b in parts) - min(b - a for a, b in parts) <= 1


def test_reference_arm_batched_small():
    """--impl reference on the batched config: worker processes over instances, one JSON line."""
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                          "c5b_mpc", "--steps", "1", "--warmup", "0", "--cpu-instances", "16"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["cores"] >= 1


def test_gloo_two_rank_shard_gather(tmp_path):
    """World-size-2 gloo run of the sharding + max/sum reduction used by the batched arm."""
    script = r'''
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
import bench
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
lo, hi = bench.shard(2048, world, rank)
v = torch.tensor([float(hi - lo), float(rank + 1)], dtype=torch.float64)
mx = v.clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
sm = v.clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
if rank == 0:
    print("RESULT", int(sm[0]), int(mx[1]))
dist.destroy_process_group()
'''
    path = tmp_path / "shard_gloo.py"
    path.write_text(script)
    env = dict(os.environ, ROOT=ROOT, CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                          "--master-addr", "127.0.0.1", "--master-port", "29561", str(path)],
                         capture_output=True, text=True, env=env, timeout=300)
    assert "RESULT 2048 2" in out.stdout, out.stdout + out.stderr[-2000:]
