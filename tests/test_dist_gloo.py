"""Multi-process host logic of paper_1807_11205_b200.dist on CPU (gloo).

World sizes 2 and 4 over 127.0.0.1; checks that every algorithm
(flat ring, literal master hierarchy, sharded hierarchy) produces the sum on
every rank and that the sub-groups follow Topology(p, k) (contiguous groups,
master = lowest rank, collectives.py:48-77).
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_11205_b200.collectives import Topology
from paper_1807_11205_b200.dist import Communicator


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, k, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        comm = Communicator(Topology(world, k))
        res = {"group": comm.group, "master": comm.master, "offset": comm.offset}
        n = 64 * k
        base = torch.arange(n, dtype=torch.float32)
        want = sum(base * (r + 1) for r in range(world))
        for algo in ("ring", "hierarchical", "sharded"):
            t = base * (rank + 1)
            comm.allreduce(t, algo)
            res[algo] = bool(torch.equal(t, want))
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world,k", [(2, 1), (2, 2), (4, 2), (4, 4), (4, 1)])
def test_communicator_algorithms_gloo(world, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    topo = Topology(world, k)
    for r in range(world):
        res = out[r]
        assert isinstance(res, dict), res
        assert res["group"] == topo.group_of(r) and res["master"] == topo.masters()[topo.group_of(r)]
        assert res["ring"] and res["hierarchical"] and res["sharded"], (r, res)
