"""bench.py's N > 1 code path on the one GPU of this pool (tests only, not a
measurement): --emulate-shard W,r runs rank r's shard of a W-rank clip --
shard window, halo exchange on a side stream overlapped with the interior
tuples (materialised mode) or before the store ring fills (store mode),
device flags read back on the exchange's stream, boundary tuples planned
from them, and the halo check -- with the halo frames written from the seed
instead of received over NCCL (NCCL refuses two ranks on one GPU).  The
library's multi-rank message plan itself is checked on CPU
(tests/test_comm_abi.py, tests/test_shard_gloo.py)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("W,r,mode,wl", [(3, 1, "materialize", "c2"), (4, 0, "store", "c2"),
                                         (4, 3, "materialize", "c2"), (2, 1, "store", "c2"), (4, 2, "store", "c2"),
                                         (3, 1, "store", "c4")])
def test_emulated_rank_runs_the_multi_gpu_path(W, r, mode, wl):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", wl, "--frames", "64", "--steps", "2",
           "--warmup", "1", "--no-cpu-baseline", "--per-config", "", "--no-compare-modes", "--f2t-mode", mode,
           "--emulate-shard", f"{W},{r}"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-3000:]
    d = json.loads(p.stdout.strip().splitlines()[-1])
    assert d["halo_check"]["ok"] is True
    assert "EMULATED" in d["config"]["parallelism"]
    if mode == "materialize":
        assert "overlapped" in d["config"]["parallelism"]
        assert d["per_direction"]["halo"]["launches_per_step"] == 1
        ov = d["overlap"]
        assert ov["halo_exchange_ms"][0] < ov["halo_exchange_ms"][1]
        # the boundary tuples start only after the exchange has delivered their frames
        if ov["boundary_f2t_ms"]:
            assert ov["boundary_f2t_ms"][0] >= ov["halo_exchange_ms"][1]
    assert d["per_direction"]["f2t"]["achieved_gbs"] > 0 and d["per_direction"]["t2f"]["achieved_gbs"] > 0
    assert d["e2e"]["value"] > 0
