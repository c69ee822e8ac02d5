"""bench.py's multi-rank flow on a one-GPU box (-m gpu): `--gpus 2` relaunches
itself with two ranks (torch.distributed.run); TSA_BENCH_ONE_GPU=1 puts both
on cuda:0 over gloo (NCCL refuses two ranks per device), which exercises the
slab split (strong scaling, max-over-ranks timing) and the tuple-sharded mode
(tsa_segment_sharded with the custom all-gather) end to end."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload,shard", [("c2", "auto"), ("c4", "auto"), ("c2", "replicas")])
def test_bench_two_ranks(workload, shard):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    env = dict(os.environ, TSA_BENCH_ONE_GPU="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--workload", workload,
                          "--shard", shard, "--steps", "5", "--warmup", "3", "--e2e-steps", "1",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    mode = {"c2": "slabs", "c4": "tuples"}[workload] if shard == "auto" else shard
    assert d["config"]["shard"] == mode
    assert d["scaling"] == ("weak" if mode == "replicas" else "strong")
