"""bench.py's N > 1 flow end to end on a 1-GPU box: two ranks as processes sharing cuda:0 under
torchrun with the gloo backend (SPMVLAB_BENCH_BACKEND=gloo; the ranks synchronise on the host, no
kernel waits on another rank).  Both exchanges (fused CUDA-IPC epilogue stores, collective
all-gatherv) must run and print one well-formed JSON line on rank 0."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("exchange", ["fused", "nccl"])
def test_bench_two_ranks(cuda, exchange):
    env = dict(os.environ, SPMVLAB_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "5", "--warmup", "3", "--exchange", exchange, "--config", "1"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 5
    assert d["gpu_launches"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["exchange"].startswith("fused" if exchange == "fused" else "NCCL")
    mg = d["multi_gpu"]
    assert mg["compute_ms_per_step"] > 0
    assert set(mg["exchanges"]) == {"fused", "nccl"}  # both exchanges measured on the same shards
    for e in mg["exchanges"].values():
        assert e["step_ms"] > 0 and e["exchange_ms"] >= 0
    assert mg["single_gpu"]["ms_per_step"] > 0 and mg["speedup_vs_1gpu"] > 0
    assert len(mg["cuts"]) == 3
