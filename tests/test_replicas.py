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
    replicas.barrier()
    q.put((r, mine, t, s, eq))
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
    (r0, m0, t0, s0, e0), (r1, m1, t1, s1, e1) = res
    assert m0 == [0, 2, 4, 6, 8] and m1 == [1, 3, 5, 7, 9]
    assert t0 == t1 == 2.5
    assert s0 == s1 == 10
    assert e0 == e1 == same


def test_request_identity_is_rank_independent():
    from paper_2602_00182_b200 import replicas

    a = replicas.synthetic_prompt(5, 16, 4096)
    b = replicas.synthetic_prompt(5, 16, 4096)
    assert (a == b).all() and replicas.request_seed(5) == replicas.request_seed(5)
