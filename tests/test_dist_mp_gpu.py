"""Two real processes (torch.distributed.run, gloo) sharing one GPU: the
product DeviceBackend four-step NTT with an executed all-to-all, sharded
batched NTTs and sharded BLAS, each rank against the single-GPU plan
(tests/mp/dist_worker.py); and bench.py's N>1 accounting as a gloo dry run."""

from __future__ import annotations

import json
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(script, *args, nproc=2, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(script), *args]
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


def test_two_process_device_backend(cuda):
    res = _torchrun(ROOT / "tests" / "mp" / "dist_worker.py")
    assert res.returncode == 0, res.stderr[-4000:]
    for r in range(2):
        assert f"RANK {r} OK" in res.stdout


def test_bench_two_rank_dry_run(cuda):
    """bench.py --gpus 2 under torchrun with the gloo backend: one JSON line
    from rank 0 with the sharded extras (parity asserted inside bench)."""
    res = _torchrun(ROOT / "bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--dist-backend", "gloo",
                    "--blas-bits", "256", "--cpu-sample", "2", "--extras", "blas", "four_step", "batched",
                    timeout=1500)
    assert res.returncode == 0, res.stderr[-4000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["config"]["dist_backend"] == "gloo"
    assert out["blas"]["ranks"] == 2
    assert out["four_step_2p24"]["ranks"] == 2
    assert out["batched_2p20_x256"]["ranks"] == 2
    assert out["cpu_baseline"]["value"] and out["roofline"]["frac"] > 0
