"""Row partitions ACROSS PROCESSES (the one-process-per-GPU
wiring): 2 and 3 processes, each owning a row range, exchange CUDA IPC handles
of their recurrence blocks and the fused step kernel gathers peer rows through
the mapped pointers (distributed.dos_moments_row_partitioned).  The test pool
has one GPU, so every process runs on cuda:0 -- CUDA IPC works between
processes on one device, so the whole path (handle export / open, partition
table, lockstep barriers, per-partition sums) runs; only the NVLink hop is
missing.  Ranks synchronise on the host between steps (gloo); no kernel waits
on another process's kernel."""

import json
import os
import socket
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(REPO, "tests", "workers", "ipc_rowpart_worker.py")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_row_partitions_over_cuda_ipc(tmp_path, kpm_ctx, world):
    out = tmp_path / "verdict.json"
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), LOCAL_RANK="0",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        env.pop("KPM_DEVICES", None)
        procs.append(subprocess.Popen([sys.executable, WORKER, str(out)], env=env, cwd=REPO,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=600)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert all(p.returncode == 0 for p in procs), "\n".join(x[-1500:] for x in logs)
    res = json.loads(out.read_text())
    assert res["world"] == world and len(res["bounds"]) == world + 1
    assert res["direct"] <= 1e-12, res
    assert res["doubling"] <= 1e-9, res
    assert res["host_block"] <= 1e-12, res
