"""bench.py's multi-rank harness on a one-GPU box: `--gpus 2` without a
torchrun environment must re-launch itself as 2 ranks, run the m-column
sharded C5 path (here at a small band limit), take the max over ranks and
print one JSON line with n_gpus = 2.  The ranks share cuda:0 and exchange
over gloo through host memory (MWSHT_BENCH_SAME_GPU / MWSHT_BENCH_BACKEND):
a harness check only, not a scaling measurement."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_relaunches_two_ranks():
    env = dict(os.environ, MWSHT_BENCH_SAME_GPU="1", MWSHT_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "2", "--warmup", "1", "--no-extra", "--band-limit", "256",
                          "--cpu-budget", "1"],
                         env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert "m-column sharded over 2 ranks" in d["config"]["parallelism"]
    assert d["roundtrip_max_abs_err"] < 1e-11
    assert d["e2e"]["max_abs_err"] < 1e-11
    assert d["value"] > 0 and d["gpu_launches"] > 0
