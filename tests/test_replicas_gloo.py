"""CPU: the N>1 replica path (barrier + max-over-ranks timing) with gloo,
world_size 2, rendezvous on 127.0.0.1."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2510_03996_b200 import replicas
    assert replicas.world() == (ws, rank)
    replicas.barrier()
    local_ms = 10.0 * (rank + 1)
    thr, mx = replicas.replica_throughput(local_ms, units_per_rank=8)
    q.put((rank, thr, mx))
    dist.destroy_process_group()


def test_replica_throughput_two_ranks():
    ws = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(ws))
    for rank, thr, mx in res:
        assert mx == 20.0  # max over ranks
        assert abs(thr - ws * 8 / 0.020) < 1e-6  # whole-job units / slowest rank


def test_single_process_identity():
    from paper_2510_03996_b200 import replicas
    assert replicas.world() == (1, 0)
    thr, mx = replicas.replica_throughput(5.0, 10)
    assert mx == 5.0 and abs(thr - 2000.0) < 1e-9
