"""Multi-process fused halo on one GPU: two ranks in two
processes connected by CUDA IPC mappings (tests/peer_worker.py), against a
single-slab run, bit for bit -- distinct left / right peers (in/outflow), the
2-rank ring (periodic: both neighbours are the same rank), the pushed residual
maxima, and slab-shaped field input (the collective peer exchange).  NCCL
cannot put two ranks on one device; CUDA IPC can, so this is the real
cross-process data path of the multi-GPU run, on the one GPU available."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case,variant", [("C1", "implicit_tvd"), ("C1", "explicit_upwind"), ("C2s", "explicit_tvd")])
def test_peer_ipc_two_processes(tmp_path, case, variant):
    import __graft_entry__
    __graft_entry__.build()
    out = tmp_path / "verdict.json"
    port = _free_port()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   CASE=case, VARIANT=variant, STEPS="3", OUT=str(out))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "peer_worker.py")], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=300)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    assert all(p.returncode == 0 for p in procs), \
        "\n".join(f"rank {r} rc {p.returncode}:\n{x[-3000:]}" for r, (p, x) in enumerate(zip(procs, logs)))
    verdict = json.loads(out.read_text())
    assert verdict["ok"], verdict
