"""bench.py's launcher (VERDICT r01 "Next round" #3): `python bench.py --gpus N`
without torchrun re-runs itself under torch.distributed.run with N ranks on
127.0.0.1, and a WORLD_SIZE that disagrees with --gpus is an error (exit
non-zero), so the driver's `bench.py --gpus 8` can never silently run one GPU."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_torchrun_argv():
    a = bench.torchrun_argv(["--gpus", "8", "--steps", "3"], 8, 29555)
    assert a[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in a and "--nnodes=1" in a and "--master-port=29555" in a
    assert a[a.index("--master-addr") + 1] == "127.0.0.1"
    assert a[-4:] == [os.path.join(ROOT, "bench.py"), "--gpus", "8", "--steps", "3"][-4:]
    assert os.path.join(ROOT, "bench.py") in a


def test_world_mismatch_is_an_error():
    bench.check_world(4, 4)
    with pytest.raises(SystemExit):
        bench.check_world(1, 8)
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


def test_defaults():
    a = bench.parse([])
    assert a.gpus == 1 and a.workload == "c5" and a.scaling == "strong" and a.halo == "nccl"
    assert a.warmup >= 3
