"""EPDRuntime on the GPU (tools/runtime_check.py): multi-request encode batches with E-side
and P-side MM reservations, the ep_wait FIFO, the shards stored into the prefill instance's
blocks (locally and, with torchrun world 2/3 sharing one GPU, over CUDA IPC peer memory) and
a paged prefill reading them -- every request's MM tokens and first token exact against a
direct encode + prefill, measured records causal."""
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,scenario", [(1, "plain"), (1, "pwait"), (1, "ewait"), (2, "plain"),
                                            (3, "pwait"), (2, "inst_rr"), (3, "inst_ll")])
def test_runtime(cuda, world, scenario):
    script = str(ROOT / "tools" / "runtime_check.py")
    if world == 1:
        cmd = [sys.executable, script, scenario]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), script, scenario]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and f"runtime_check world={world} {scenario}: OK" in out, out[-3000:]
