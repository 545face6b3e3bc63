"""Host-side router over independent decode replicas, one per GPU.

Requests are independent -- the method has no cross-request state (batching is
"compatible" with tool partial execution) -- and a 7B replica fits one B200, so the hot path
shards as one engine per GPU with no data-path collective.  The router

  * splits a configuration's TOTAL batch over the G ranks deterministically: request k is
    served by rank k mod G (reproducible; the paper ran one model instance per GPU);
  * gathers a 64-byte per-rank completion-stats record every `every` steps with one
    all-gather (NCCL over NVLink / NVSwitch on the GPU box, gloo in the CPU tests).  The
    gather is issued asynchronously on the process group's own stream, so it never sits on
    the decode critical path; the previous gather is waited for only when the next is issued.

One process per GPU (torch.distributed); within a process the replica is an `Engine`.
"""
from __future__ import annotations

STATS_FIELDS = ("step", "n_active", "n_generated", "n_segments", "n_finished", "step_us", "rank", "tokens_total")


class Router:
    def __init__(self, rank: int = 0, world: int = 1, every: int = 16, device=None):
        if world < 1 or not 0 <= rank < world:
            raise ValueError("bad rank / world")
        self.rank, self.world, self.every = rank, world, max(1, int(every))
        self.device = device
        self.steps = 0
        self.tokens = 0
        self.gathers = 0
        self._pending = None   # (work handle, output tensor) of the in-flight gather
        self.last_info = None
        self.table = None      # last completed gather: [world][8] int64

    # ---------------------------------------------------------------- request placement
    def owner(self, k: int) -> int:
        """Rank serving global request k."""
        return k % self.world

    def mine(self, n_total: int) -> list[int]:
        """Global indices of this rank's share of a total batch of n_total requests."""
        return list(range(self.rank, n_total, self.world))

    def share(self, n_total: int) -> int:
        return len(range(self.rank, n_total, self.world))

    # ---------------------------------------------------------------- stats gather
    def after_step(self, info=None):
        """Account one step (info: the engine's cvy_step_info of the last completed step);
        every `every` steps, all-gather the per-rank stats record."""
        self.steps += 1
        if info is not None:
            self.tokens += int(info.n_generated)
            self.last_info = info
        if self.steps % self.every == 0:
            self._gather(info)

    def _record(self, info):
        vals = [0] * len(STATS_FIELDS)
        if info is not None:
            vals[:5] = [int(info.step), int(info.n_active), int(info.n_generated), int(info.n_segments),
                        int(info.n_finished)]
            vals[5] = int(round(float(info.step_ms) * 1000.0))
        vals[6], vals[7] = self.rank, self.tokens
        return vals

    def _gather(self, info):
        import torch
        t = torch.tensor(self._record(info), dtype=torch.int64, device=self.device)
        if self.world == 1:
            self.table = [t.tolist()]
            self.gathers += 1
            return
        import torch.distributed as dist
        self.wait()
        out = torch.empty(self.world * len(STATS_FIELDS), dtype=torch.int64, device=self.device)
        work = dist.all_gather_into_tensor(out, t, async_op=True)
        self._pending = (work, out)

    def wait(self):
        """Complete the in-flight gather (if any); returns the latest gathered table."""
        if self._pending is not None:
            work, out = self._pending
            work.wait()
            self.table = out.view(self.world, len(STATS_FIELDS)).tolist()
            self.gathers += 1
            self._pending = None
        return self.table

    def flush(self, info=None):
        """Final gather (outside any timed region) so every rank's totals are in `table`."""
        self.wait()
        self._gather(info if info is not None else self.last_info)
        return self.wait()
