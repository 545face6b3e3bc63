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


class _Info:
    def __init__(self, step, n):
        self.step, self.n_active, self.n_generated, self.n_segments, self.n_finished = step, n, n, 2 * step, 0
        self.step_ms = 1.5


def _router_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_00059_b200.router import Router
    r = Router(rank, world, every=4)
    mine = r.mine(512)
    n = len(mine)
    for s in range(10):
        r.after_step(_Info(s + 1, n))
    table = r.flush(_Info(10, n))
    q.put((rank, mine, r.gathers, table, [r.owner(k) for k in range(8)]))
    dist.barrier()
    dist.destroy_process_group()


def test_router_splits_total_batch_and_gathers_stats():
    """request k goes to rank k mod G (the config's TOTAL batch is split, so
    the ranks' shares partition it), and every `every` steps the 64-byte per-rank stats record
    is all-gathered (gloo here, NCCL over NVLink on the GPU box)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_router_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((x[0], x[1:]) for x in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shares = [res[r][0] for r in range(2)]
    assert sorted(shares[0] + shares[1]) == list(range(512)) and len(shares[0]) == len(shares[1]) == 256
    assert shares[1][:3] == [1, 3, 5] and res[0][3] == [0, 1, 0, 1, 0, 1, 0, 1]
    for r in range(2):
        gathers, table = res[r][1], res[r][2]
        assert gathers == 10 // 4 + 1            # steps 4 and 8, then the final flush
        assert [row[6] for row in table] == [0, 1]               # rank field
        assert [row[7] for row in table] == [256 * 10, 256 * 10]  # tokens generated so far
        assert [row[0] for row in table] == [10, 10]
