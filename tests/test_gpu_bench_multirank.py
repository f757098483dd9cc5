"""bench.py's multi-rank path under torchrun (2 ranks sharing one GPU through the gloo backend;
NCCL needs distinct devices): sharded rollouts, MIN/SUM reductions through ShardedMPPI,
max-over-ranks timing and the JSON contract."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_gloo():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--backend", "gloo", "--config", "C4",
           "--no-probe"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["K_per_gpu"] == d["config"]["K"] // 2
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] == 3 * 2 * 5
    assert d["scaling"] == "strong" and d["backend"] == "gloo"
