"""The N>1 path on CPU: world_size-2 `gloo` ranks each run their shard of the dealt request
stream (bench.py's sharding: no data-path collective, only the final gather), and the
gathered per-request results equal a single-rank run — requests are independent state
machines (sim.hpp:429-442), so sharding must be invisible in the results."""
import os
import socket
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def shard(total, world, rank):
    lo, hi = total * rank // world, total * (rank + 1) // world
    return lo, hi - lo


def worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2602_18931_b200 as ws
    from oracle import pyoracle as po
    from paper_2602_18931_b200 import abi
    c = abi.config2(num_requests=12)
    c.first_request, c.local_requests = shard(12, world, rank)
    b = ws.run_sim_with_model(c, po.model_round_fn(c))
    local = {"metrics": b.metrics_list(), "ctrl": b.ctrl_outputs()}
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    # max-over-ranks reduction, as bench.py does for its timing
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put({"gathered": gathered, "max": t.item()})
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_ranks_equal_single_rank(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    import paper_2602_18931_b200 as ws
    from oracle import pyoracle as po
    from paper_2602_18931_b200 import abi
    full = abi.config2(num_requests=12)
    b = ws.run_sim_with_model(full, po.model_round_fn(full))
    metrics = sum((g["metrics"] for g in res["gathered"]), [])
    ctrl = sum((g["ctrl"] for g in res["gathered"]), [])
    assert metrics == b.metrics_list()
    assert ctrl == b.ctrl_outputs()
    assert res["max"] == float(world)
