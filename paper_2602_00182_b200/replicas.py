"""Per-GPU replica plumbing: requests shard naturally, so N GPUs run N independent
engines with NO collective on the data path. torch.distributed is used only for the launch
plumbing: a barrier around the timed region, the max over ranks of the device time, and a
cross-GPU receipt comparison (every rank runs the same probe request; all out_hashes must match).

Works with the nccl backend on the GPU box and with gloo on CPU (tests/test_replicas.py).
"""
from __future__ import annotations

import os
from typing import List, Sequence

import numpy as np


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def init(backend: str):
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world


def shard(n_total: int, rank: int, world: int) -> List[int]:
    """Static round-robin request sharding: request i goes to rank i % world."""
    return [i for i in range(n_total) if i % world == rank]


def request_seed(global_index: int) -> int:
    """Per-request seed: independent of the rank that serves it (so any sharding gives equal bytes)."""
    return 0x5EED0000 + global_index


def synthetic_prompt(global_index: int, length: int, vocab: int) -> np.ndarray:
    rng = np.random.default_rng(request_seed(global_index) ^ 0xABCD)
    return rng.integers(0, vocab, length, dtype=np.int64).astype(np.uint32)


def barrier(device=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        if dist.get_backend() == "nccl" and device is not None:
            dist.barrier(device_ids=[device])
        else:
            dist.barrier()


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device=f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64,
                     device=f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def receipts_equal_across_ranks(hashes: Sequence[bytes], device=None) -> bool:
    """All ranks pass the out_hashes of the SAME probe requests; True iff identical everywhere."""
    import torch
    import torch.distributed as dist

    blob = np.frombuffer(b"".join(hashes), dtype=np.uint8).astype(np.int64)
    if not (dist.is_available() and dist.is_initialized()):
        return True
    dev = f"cuda:{device}" if dist.get_backend() == "nccl" else "cpu"
    mine = torch.from_numpy(blob).to(dev)
    parts = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, mine)
    return all(torch.equal(p, parts[0]) for p in parts)


def launch_local(n: int, argv: Sequence[str], master_port: int = 0) -> int:
    """Run `python argv...` as n local ranks (one per GPU) exactly as the driver does for N > 1:
    ``python -m torch.distributed.run --nnodes=1 --nproc-per-node n --master-addr 127.0.0.1``.
    Children inherit stdout, so rank 0's output is this process's output. Returns the exit code."""
    import socket
    import subprocess
    import sys

    if master_port == 0:
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        master_port = s.getsockname()[1]
        s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(master_port), *argv]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def cross_rank_reexecution(own: dict, rerun: dict, device=None) -> dict:
    """Cross-GPU receipt equality by re-execution: every rank passes
    the out_hashes of the requests it served ({global index: hash}) and of the requests of
    ANOTHER rank that it re-executed. All-gathered; every re-executed request's hash must equal
    the serving rank's. Returns {"requests", "reexecuted", "all_equal", "mismatches"}."""
    import torch.distributed as dist

    mine = ({int(k): bytes(v) for k, v in own.items()}, {int(k): bytes(v) for k, v in rerun.items()})
    if dist.is_available() and dist.is_initialized():
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, mine)
    else:
        parts = [mine]
    served, again = {}, {}
    for o, r in parts:
        served.update(o)
        for k, v in r.items():
            again.setdefault(k, []).append(v)
    bad = sorted(k for k, vs in again.items() if k not in served or any(v != served[k] for v in vs))
    return {"requests": len(served), "reexecuted": sum(len(v) for v in again.values()), "all_equal": not bad,
            "mismatches": bad[:16]}
