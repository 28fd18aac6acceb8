"""Multi-rank host logic of bench.py on CPU with gloo (world size 2): the timing
reduction (max over ranks), the whole-job edge count (sum) and replica seeds."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    tot_ms, edges = bench.reduce_over_ranks(10.0 + 5.0 * rank, 1000.0 * (rank + 1), "cpu", world)
    out[rank] = (tot_ms, edges, bench.replica_seed(3, rank))
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_over_ranks_gloo_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        tot_ms, edges, seed = out[r]
        assert tot_ms == 15.0            # max over ranks
        assert edges == 3000.0           # sum over ranks
        assert seed == 3 + r             # independent replicas
    assert out[0][2] != out[1][2]


def test_reference_arm_other_ranks_exit_silently(capsys):
    sys.path.insert(0, ROOT)
    import bench
    os.environ["RANK"] = "1"
    try:
        class A:
            steps, warmup, gpus, ref_frac = 1, 0, 2, 0.001
        assert bench.run_reference(A) == 0
    finally:
        os.environ.pop("RANK")
    assert capsys.readouterr().out == ""


def _exchange_worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1606_09481_b200 as rhg
    offs, total = rhg.exchange_counts([1000, 234][rank])
    q.put((rank, offs, total))
    dist.destroy_process_group()


def test_shard_count_exchange_gloo_world2():
    """The one collective of the sharded path: all_gather of one edge count per rank
     -> global offsets, over gloo with world size 2."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, (o, t)) for r, o, t in [q.get(timeout=120) for _ in ps])
    for p in ps:
        p.join(timeout=60)
    assert res[0] == ([0, 1000], 1234) and res[1] == ([0, 1000], 1234)
