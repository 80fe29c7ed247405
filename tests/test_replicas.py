"""Multi-replica host logic on CPU with gloo, world_size 2 (the N>1 path of bench.py):
sharding, max-over-ranks timing, cross-rank receipt comparison."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, same):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    from paper_2602_00182_b200 import replicas

    r, w = replicas.init("gloo")
    mine = replicas.shard(10, r, w)
    t = replicas.max_over_ranks(1.5 + r)
    s = replicas.sum_over_ranks(len(mine))
    probe = [bytes([7] * 32)] if same else [bytes([rank] * 32)]
    eq = replicas.receipts_equal_across_ranks(probe)
    # re-execution check: rank r serves requests {2r, 2r+1} and re-runs the other rank's
    own = {g: bytes([g] * 32) for g in (2 * r, 2 * r + 1)}
    o = 1 - r
    rerun = {g: bytes([g] * 32) for g in (2 * o, 2 * o + 1)}
    if not same and r == 1:
        rerun[0] = bytes([99] * 32)   # rank 1's re-execution of request 0 disagrees
    cross = replicas.cross_rank_reexecution(own, rerun)
    replicas.barrier()
    q.put((r, mine, t, s, eq, cross))
    import torch.distributed as dist

    dist.destroy_process_group()


@pytest.mark.parametrize("same", [True, False])
def test_two_rank_gloo(same):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, same)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    (r0, m0, t0, s0, e0, c0), (r1, m1, t1, s1, e1, c1) = res
    assert m0 == [0, 2, 4, 6, 8] and m1 == [1, 3, 5, 7, 9]
    assert t0 == t1 == 2.5
    assert s0 == s1 == 10
    assert e0 == e1 == same
    assert c0 == c1
    assert c0["requests"] == 4 and c0["reexecuted"] == 4
    assert c0["all_equal"] == same and c0["mismatches"] == ([] if same else [0])


def test_bench_launches_its_own_ranks():
    """`python bench.py --gpus 2` without torchrun spawns the two ranks itself (replicas.launch_local:
    the driver's own torchrun command) and rank 0 alone prints the JSON line. Exercised on CPU
    through the reference arm (gloo; the tiny model keeps the oracle sample to seconds)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--model", "llama-tiny:launch", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0


def test_request_identity_is_rank_independent():
    from paper_2602_00182_b200 import replicas

    a = replicas.synthetic_prompt(5, 16, 4096)
    b = replicas.synthetic_prompt(5, 16, 4096)
    assert (a == b).all() and replicas.request_seed(5) == replicas.request_seed(5)
