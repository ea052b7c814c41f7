"""Prefill -> decode KV handoff across real processes on the GPU.

* nvlink-peer transport, two torchrun processes sharing one GPU (tools/kv_handoff_check.py):
  CUDA IPC mapping of the decode pool, the block-move kernel pushing the prefill's real
  (TINY_LLM-written) KV into the reserved decode blocks, cross-process stream-memop flags;
  reference block ids / frees / pd_wait deferral on both ranks; bit-exact KV.
* the NCCL legs of the C ABI (epd_comm_*, epd_gather_tokens, epd_kv_handoff_send/recv) on
  one GPU: a one-rank communicator (gather = in-place / local copy; raw send + receive to self
  in one NCCL group around pack / unpack), and with >= 2 GPUs a two-process handoff.
"""
import socket
import subprocess
import sys
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(script, world, *args, timeout=240):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(script), *map(str, args)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    return r.returncode, r.stdout + r.stderr


def test_kv_handoff_nvlink_peer_two_processes(cuda):
    rc, out = _torchrun(ROOT / "tools" / "kv_handoff_check.py", 2)
    assert rc == 0 and "kv_handoff_check transport=nvlink-peer: OK" in out, out[-3000:]


def _one_rank_comm(cuda):
    from paper_2501_05460_b200.comm import NcclComm
    import ctypes as C
    from paper_2501_05460_b200._lib import call
    uid = (C.c_uint8 * 128)()
    call("epd_comm_unique_id", uid)
    return NcclComm(cuda, rank=0, world=1, uid=bytes(uid))


def test_nccl_comm_gather_and_kv_bytes_single_rank(cuda):
    from paper_2501_05460_b200.handoff import PagedKVCache
    comm = _one_rank_comm(cuda)
    # EP gather with one rank: the root's shard lands at offset 0 (aliasing: no copy; else a copy)
    shard = torch.randn(3, 64, 128, device=cuda).to(torch.bfloat16)
    packed = torch.zeros_like(shard)
    comm.gather_tokens(shard, 3, packed, root=0)
    torch.cuda.synchronize()
    assert torch.equal(packed, shard)
    comm.gather_tokens(packed, 3, packed, root=0)  # aliasing shard: a no-op
    # KV bytes through NCCL: pack -> ncclSend(self) + ncclRecv(self) in one group -> unpack
    src = PagedKVCache(2, 2, 64, 16, 20, cuda)
    dst = PagedKVCache(2, 2, 64, 16, 20, cuda)
    src.pool.copy_(torch.randn_like(src.pool, dtype=torch.float32).to(torch.bfloat16))
    sid, did = [3, 7, 1, 12], [19, 0, 5, 6]
    staged = src.pack(sid)
    landed = torch.empty_like(staged)
    comm.group_start()
    comm.send(staged, 0)
    comm.recv(landed, 0)
    comm.group_end()
    dst.unpack(landed, did)
    torch.cuda.synchronize()
    assert torch.equal(dst.blocks(did), src.blocks(sid))
    comm.close()


def test_nccl_comm_rejects_bad_peers(cuda):
    from paper_2501_05460_b200.handoff import PagedKVCache
    comm = _one_rank_comm(cuda)
    src = PagedKVCache(2, 2, 64, 16, 8, cuda)
    ids = torch.tensor([0, 1], dtype=torch.int32, device=cuda)
    st = torch.empty(2, src.segments, src.block_elems, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ValueError):
        comm.kv_send(src, ids, st, 0)   # the peer must be another rank
    with pytest.raises(ValueError):
        comm.kv_recv(src, ids, st, 3)   # out of range
    comm.close()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NCCL needs one GPU per rank")
def test_kv_handoff_nccl_two_gpus(cuda):
    rc, out = _torchrun(ROOT / "tools" / "kv_handoff_check.py", 2, "nccl")
    assert rc == 0 and "kv_handoff_check transport=nccl: OK" in out, out[-3000:]
