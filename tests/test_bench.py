"""bench.py contract pieces that run without a GPU: the self-launch of
`--gpus N` (one process per rank under torch.distributed.run) and the
bounded reference-arm sample."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_launch_command_shape():
    import bench
    cmd = bench.launch_command(["--gpus", "4", "--steps", "2"], 4, 29555)
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd and "29555" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]


def test_gpus_2_spawns_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--probe-launch"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d == {"probe": True, "world": 2, "ranks": [0, 1]}


def test_reference_sample_is_bounded():
    import bench
    from conftest import load_case
    tri, _ = load_case("u1k_unit")
    tl, ts = bench.reference_sample(tri, 0, 4)
    assert tl >= 0 and ts >= 0
    assert bench.reference_slices(20_000_000) == 16 and bench.reference_slices(1000) == 1
