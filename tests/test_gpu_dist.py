"""The multi-rank product path on one GPU: two processes (gloo), each owning
half of the batch, through ActivationSetPlan + PipelinedStep with the exchange
closure (dist.make_gather), equal the oracle's sharded driver O13 rank by rank
(tools/dist_plan_check.py)."""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_plan_gather_path_equals_oracle():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1",
                        f"--master-port={_free_port()}",
                        os.path.join(ROOT, "tools", "dist_plan_check.py")],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
