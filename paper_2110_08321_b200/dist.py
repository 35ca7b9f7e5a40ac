"""Multi-GPU plumbing for the config-2 workload.

Images are independent ciphertext sets, so ranks shard images (weak
scaling: `per_rank` images each) with keys/masks replicated, and the only
collective is an all-gather of the output ciphertexts in wire format.
Backend-agnostic (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations


def image_range(rank: int, per_rank: int):
    """global image indices (also the encryption nonces) owned by `rank`"""
    return range(rank * per_rank, (rank + 1) * per_rank)


def gather_outputs(local, world: int, out=None):
    """all-gather the per-rank output ciphertext words (int64 view of the
    uint64 wire words) into [world * local.numel()] ordered by rank."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    if out is None:
        out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous())
    return out


def reduce_partials(acc, world: int):
    """element-wise sum of the per-rank HS partial accumulators (int64 view
    of uint64 residues < 2^60: the sum of <= 8 stays < 2^63, so the int64
    all-reduce is exact); the library's finish reduces mod q.  In place."""
    import torch.distributed as dist
    if world > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM)
    return acc


def max_over_ranks(value: float, device=None) -> float:
    """the step time every rank reports is the max over ranks"""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_ranks(nproc: int, script: str, args, env=None, timeout=None) -> int:
    """one process per GPU on this node: re-launch `script args` under
    torch.distributed.run with `nproc` ranks (rendezvous on 127.0.0.1; the
    ranks read RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* from the
    environment).  NCCL_DEBUG=INFO unless the caller set it, so the
    communicator setup lines show up in the log.  Returns the exit code; the
    ranks' stdout / stderr pass through."""
    import os
    import subprocess
    import sys
    e = dict(os.environ)
    e.setdefault("NCCL_DEBUG", "INFO")
    e.setdefault("OMP_NUM_THREADS", "4")
    if env:
        e.update(env)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script, *map(str, args)]
    return subprocess.run(cmd, env=e, timeout=timeout).returncode
