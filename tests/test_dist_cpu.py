"""N>1 host logic on CPU: world_size-2 gloo processes exercise the bench's
distributed reductions (whole-job throughput = sum of units / max time) and the
node -> GPU layout rules used by the disaggregated engine runs."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2603_13358_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r processed 100*(r+1) tokens in 0.5*(r+1) seconds
    v = D.whole_job_throughput(100.0 * (rank + 1), 0.5 * (rank + 1))
    mx = D.max_over_ranks([float(rank), -float(rank)])
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, v, mx))


def test_gloo_world2_reductions():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, v, mx in out:
        assert v == pytest.approx(300.0 / 1.0)  # (100 + 200) tokens / max(0.5, 1.0) s
        assert mx == [1.0, 0.0]


def test_layouts():
    assert D.node_layouts(2) == ["1P_1D"]
    assert D.node_layouts(8) == ["2P_6D", "4P_4D"]
    assert D.layout_gpus("2P_6D", 8) == list(range(8))
    with pytest.raises(ValueError):
        D.layout_gpus("4P_4D", 4)


def test_single_process_identity():
    assert D.whole_job_throughput(10.0, 2.0) == 5.0
