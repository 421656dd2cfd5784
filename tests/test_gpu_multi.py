"""Sharded stage across GPUs (NCCL over NVLink) — needs >= 2 GPUs (gpurun --gpus 2|4)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def ngpus() -> int:
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("graphs", [0, 1])
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_stage_matches_oracle(world, graphs):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    port = 29600 + world + 10 * graphs
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "tests" / "mgpu_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, VX_TEST_GRAPHS=str(graphs)))
    sys.stdout.write(r.stdout[-3000:])
    sys.stderr.write(r.stderr[-3000:])
    assert r.returncode == 0
    assert "parity=ok" in r.stdout and "parity=FAIL" not in r.stdout
    assert "(fp32 store)" in r.stdout  # the fp32 token store ran across the shards too
