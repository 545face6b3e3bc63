"""World-size-2 gloo coverage of bench.py's multi-rank host logic on CPU: max-over-ranks
device time, whole-job token sum (weak scaling: every rank runs the full per-GPU batch), and
the per-rank stats all-gather that NCCL performs over NVLink on the GPU box."""
import os
import socket

import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    local_ms = [120.0, 135.5][rank]
    out = bench.reduce_over_ranks(local_ms, 64 * 100, [float(rank), local_ms, 6400.0])
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_reduction():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        max_ms, tokens, stats = res[r]
        assert max_ms == 135.5
        assert tokens == 2 * 6400
        assert [s[0] for s in stats] == [0.0, 1.0] and [s[1] for s in stats] == [120.0, 135.5]
    # whole-job throughput = all ranks' tokens / the slowest rank's time
    assert abs(tokens / (max_ms / 1000) - 2 * 6400 / 0.1355) < 1e-6
