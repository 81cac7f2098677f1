"""The multi-rank bench path (round-robin index shards, device pack -> all_gather ->
tv_hist_replace_rows merge, max-over-ranks timing, distributed e2e) with two ranks sharing
the one GPU of the test box over gloo (TV_DIST_BACKEND=gloo moves the collectives through host
memory; the device-side pack / merge / export code is the one NCCL runs).  The merged full
S_{2,8} and full S^{32}_{3,8} histograms must equal the reference aggregates."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_bench_two_ranks_share_one_gpu():
    env = dict(os.environ, TV_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "1", "--no-ga"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # rank 0 alone prints
    b = json.loads(lines[0])
    assert b["n_gpus"] == 2 and b["config"]["histogram_ok"] is True
    assert b["value"] > 0 and b["e2e"]["value"] > 0
    assert b["s32"]["n_gpus"] == 2 and b["s32"]["histogram_ok"] is True


@pytest.mark.parametrize("world", [2, 3])
def test_device_exchange_with_idle_ranks(world):
    """enumerate_space_distributed through the device-side, key-partitioned exchange, with ranks
    that enumerate nothing (count < world * batch_size) but own keys whose payloads they must
    re-derive (the enumeration parameters are registered on every rank), a ragged
    range and an S32 block; every rank's merged histogram equals the single-GPU one."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "tests/_dist_enum_worker.py"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    res = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert sorted(r["rank"] for r in res) == list(range(world))
    for r in res:
        assert r["s28_idle"] and r["s28_ragged"] and r["s32_block"], r
