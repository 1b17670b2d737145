"""N > 1 host logic on CPU: world_size-2 gloo process group (127.0.0.1) running bench.py's
max-over-ranks timing and whole-job throughput, as torchrun would launch it (DESIGN.md
"Multi-GPU": replicas, weak scaling, no data-path collective)."""
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


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    ms = [12.5, 17.25][rank]                    # per-rank device times
    m = bench.max_over_ranks(ms, world, "cpu")
    v = bench.whole_job_throughput(8388608, world, 20, m)
    dist.barrier()
    q.put((rank, m, v))
    dist.destroy_process_group()


def test_two_rank_max_and_throughput():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, m, v in res:
        assert m == 17.25                        # the slowest rank's time on every rank
        assert v == pytest.approx(8388608 * 2 * 20 / 17.25e-3)


def test_single_rank_identity():
    import bench
    assert bench.max_over_ranks(3.0, 1) == 3.0
    assert bench.whole_job_throughput(100, 1, 10, 1.0) == pytest.approx(1e6)
