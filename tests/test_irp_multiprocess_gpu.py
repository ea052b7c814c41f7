"""The IRP encode stage with the peer-memory gather across real processes (torchrun,
world 2 and 3) on one GPU: CUDA IPC mappings between the processes, the put kernel and
cross-process stream-memop waits, with every packed request checked bit for bit against a
direct encode on the prefill rank (tools/irp_check.py). Only NVLink itself is absent."""
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


@pytest.mark.parametrize("world,tiles,mode", [(2, 10, ""), (3, 13, ""), (3, 12, "cache"), (2, 10, "batch"),
                                              (3, 10, "batch")])
def test_irp_peer_gather_multiprocess(cuda, world, tiles, mode):
    """mode "cache": the prefill rank's MM-token cache plans the misses, which are sharded
    and land in the peer slot as staging before being scattered into the cache store."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "tools" / "irp_check.py"),
           "12", str(tiles)] + ([mode] if mode else [])
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=240)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    tag = f"irp_check world={world} tiles={tiles}" + (f" {mode}" if mode else "")
    assert tag in out and "OK (transport nvlink-peer)" in out, out[-3000:]
