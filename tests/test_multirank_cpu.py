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


# ---------------------------------------------------------------- N2: velocity-slab transport
class _FakeSlab:
    """Host stand-in of vslab._Slab: the send buffers carry (rank, side) codes."""

    def __init__(self, r, n, nx=6):
        self.j, self.nslabs = r, n
        self.lo_send = torch.full((2 * nx,), 10.0 * r + 1.0, dtype=torch.float64)
        self.hi_send = torch.full((2 * nx,), 10.0 * r + 2.0, dtype=torch.float64)
        self.lo_recv = torch.full((2 * nx,), -1.0, dtype=torch.float64)
        self.hi_recv = torch.full((2 * nx,), -1.0, dtype=torch.float64)


def _slab_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1204_3853_b200.vslab import DistComm
    comm = DistComm.with_p2p_group(rank, world)         # halo on its own communicator
    s = _FakeSlab(rank, world)
    rho = torch.arange(4, dtype=torch.float64) + (1.0 if rank == 0 else 0.0) - rank   # base 1 on rank 0
    works = list(comm.allreduce([s], [rho])) + list(comm.exchange([s]))   # both in flight at once
    for w in works:
        w.wait()
    q.put((rank, s.lo_recv[0].item(), s.hi_recv[0].item(), rho.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_vslab_exchange_and_reduction(world):
    """DistComm: a slab's low ghosts come from the lower neighbour's high boundary columns and its
    high ghosts from the upper neighbour's low ones; physical faces (rank 0 low, last rank high)
    receive nothing; the moment partials sum to the same vector on every rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [sum(k + (1.0 if r == 0 else 0.0) - r for r in range(world)) for k in range(4)]
    for rank, lo, hi, rho in res:
        assert lo == (10.0 * (rank - 1) + 2.0 if rank > 0 else -1.0)
        assert hi == (10.0 * (rank + 1) + 1.0 if rank < world - 1 else -1.0)
        assert rho == want
