"""Non-blocking layer migration with shadow-gradient payback, executed on
B200 (second half).

The reference plans it (plan_layer_migration, migration.cpp:9-61; caller
Simulation::migrate, sim.cpp:485-530) and only models its time: while the
migrating layer's parameters travel to the target stage, the target runs its
first k micro-batches without the layer and the source's *shadow* instance
computes the layer's gradients for them; afterwards that partial gradient
("payback") ships to the target at lower priority.

On B200 the parameters are pulled over NVLink by the staged copy
(kernel (b)) on a low-priority stream, and the layer's gradient is
accumulated in the int64 fixed-point domain of kernel (d): the shadow
instance folds micro-batches [0, k) into its own accumulator, the target
folds [k, M) into its accumulator, and the shadow's accumulator is pulled
into the target's HBM on the low-priority stream as soon as a device-side
barrier says the shadow is done — overlapped with the target's remaining
micro-batches — and added inside the target's last fold (one pass,
`ew_weighted_fold_addend`).  Integer sums are exact, so the migrated step's gradient is
bit-identical to the static step's whatever k the planner chose — the
property the reference's toy simulator checks with fp64 folds
(test_sim.cpp:136-147).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from . import device as dev
from ._native import check, lib
from .fabric import NON_BLOCKING, MigrationSchedule, plan_layer_migration


def payback_accumulate(acc: torch.Tensor, payback, stream=None) -> None:
    """acc += payback (int64).  `payback`: int64 tensor or a raw (peer)
    device pointer to at least acc.numel() int64 values."""
    if acc.dtype != torch.int64:
        raise ValueError("acc must be int64")
    p = dev._ptr(payback) if isinstance(payback, torch.Tensor) else dev.C.c_void_p(int(payback))
    check(lib.ew_payback_accumulate(dev._ptr(acc), p, acc.numel(), dev._stream(stream)))


class LayerMigration:
    """One layer moving from the source rank to the target rank.

    Both ranks construct it collectively over `group`, a process group of
    exactly {source, target}.  The source passes its parameter buffer and its
    shadow gradient accumulator, the target its destination buffer and its
    own accumulator.

    Timeline (all stream-ordered, no host round trip on the critical path):
      target, low-priority stream:  pull_params() ... prefetch_payback()
                                    (waits on a device-side barrier with the
                                    source, then pulls the shadow accumulator
                                    into local HBM while the target computes)
      target, compute stream:       micro-batches; wait for params before
                                    micro-batch k; the last micro-batch folds
                                    with addend=payback_buf
      source, compute stream:       shadow micro-batches [0, k), then
                                    shadow_done()
    run_target() / run_shadow() enqueue exactly that for gradient units.
    """

    def __init__(self, move, src_rank: int, dst_rank: int, rank: int, params: torch.Tensor,
                 acc: torch.Tensor, group=None, transfer_ctas: int = 32):
        """transfer_ctas: CTAs of the background pulls.  Stream priority
        only orders *pending* CTAs, so a full-width copy would hold every SM
        until it finished and stall the compute stream; a few dozen CTAs
        with 96 KiB in flight each still saturate NVLink."""
        self.transfer_ctas = transfer_ctas
        self.move = tuple(move)
        self.src, self.dst, self.rank = src_rank, dst_rank, rank
        self.params, self.acc = params, acc
        world = dist.get_world_size(group)
        mine = None
        if rank == src_rank:
            mine = (dev.ipc_handle(params), dev.ipc_handle(acc))
        allh = [None] * world
        dist.all_gather_object(allh, (rank, mine), group=group)
        self._opened = []
        self.copy: Optional[dev.CopyProgram] = None
        self.payback_buf: Optional[torch.Tensor] = None
        self.barrier = dev.PeerBarrier(group)
        if rank == dst_rank:
            (hp, op), (ha, oa) = dict(allh)[src_rank]
            self._opened = [dev.ipc_open(hp, op), dev.ipc_open(ha, oa)]
            self.copy = dev.CopyProgram.from_pointers([self._opened[0]], [params.data_ptr()],
                                                      [params.numel() * params.element_size()],
                                                      [True])
            self.payback_buf = torch.empty_like(acc)
            self.payback_copy = dev.CopyProgram.from_pointers(
                [self._opened[1]], [self.payback_buf.data_ptr()], [acc.numel() * 8], [True])
        self.events = {}

    def plan(self, mode: int = NON_BLOCKING, **ctx) -> MigrationSchedule:
        """The reference planner (plan_layer_migration) on this move."""
        return plan_layer_migration(self.move, mode, **ctx)

    def _timed(self, name, stream, fn):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = stream or torch.cuda.current_stream()
        s.record(st)
        fn(st)
        e.record(st)
        self.events[name] = (s, e)
        return e

    def pull_params(self, stream: Optional[torch.cuda.Stream] = None) -> torch.cuda.Event:
        """Target: start the parameter pull on `stream` (low priority by
        convention); returns the event that marks the parameters' arrival."""
        assert self.rank == self.dst
        return self._timed("params", stream, lambda st: self.copy.launch(self.transfer_ctas, stream=st))

    def shadow_done(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Source: enqueue after the shadow instance's last fold."""
        assert self.rank == self.src
        self.barrier.wait(stream)

    def prefetch_payback(self, stream: Optional[torch.cuda.Stream] = None) -> torch.cuda.Event:
        """Target: wait (on `stream`) until the source's shadow is done, then
        pull its accumulator into payback_buf; returns the arrival event."""
        assert self.rank == self.dst
        self.barrier.wait(stream)
        return self._timed("payback_grad", stream, lambda st: self.payback_copy.launch(self.transfer_ctas, stream=st))

    def payback(self, stream: Optional[torch.cuda.Stream] = None) -> torch.cuda.Event:
        """Target, unoverlapped variant: add the source's shadow accumulator
        into the target's straight from peer HBM (the caller orders it after
        the shadow's last fold)."""
        assert self.rank == self.dst
        return self._timed("payback_grad", stream,
                           lambda st: payback_accumulate(self.acc, self._opened[1], stream=st))

    def run_target(self, units, weights, frac_bits: int, k: int,
                   compute: torch.cuda.Stream, transfer: torch.cuda.Stream,
                   other_work=None) -> None:
        """Target's step for this layer: units[mb] is micro-batch mb's
        gradient of the layer (fp32), weights[mb] its weight.  Micro-batches
        [0, k) run without the layer (other_work(mb, stream) stands for the
        target's other layers); [k, M) fold into self.acc after the
        parameters arrived; the payback joins in the last fold."""
        M = len(units)
        arrived = self.pull_params(transfer)
        # k == 0 is the blocking move: no shadow work, nothing to pay back
        ready = self.prefetch_payback(transfer) if k > 0 else None
        for mb in range(M):
            if mb < k:
                if other_work is not None:
                    other_work(mb, compute)
                continue
            if mb == k:
                compute.wait_event(arrived)
            last = mb == M - 1 and ready is not None
            if last:
                compute.wait_event(ready)
            dev.weighted_fold([units[mb]], [weights[mb]], frac_bits, self.acc, accumulate=True,
                              stream=compute, addend=self.payback_buf if last else None)
        if k >= M:
            compute.wait_event(arrived)
            compute.wait_event(ready)
            payback_accumulate(self.acc, self.payback_buf, stream=compute)

    def run_shadow(self, units, weights, frac_bits: int, k: int,
                   compute: torch.cuda.Stream) -> None:
        """Source's shadow instance: micro-batches [0, k) of the layer, then
        the signal that releases the target's payback pull."""
        if k <= 0:
            return  # blocking move: the target computes every micro-batch
        for mb in range(min(k, len(units))):
            dev.weighted_fold([units[mb]], [weights[mb]], frac_bits, self.acc, accumulate=True,
                              stream=compute)
        self.shadow_done(compute)

    def timed_out(self) -> bool:
        return self.barrier.timed_out()

    def measured(self) -> dict:
        """Measured transfer segments (ms) after synchronisation."""
        return {k: s.elapsed_time(e) for k, (s, e) in self.events.items()}

    def close(self) -> None:
        self.copy = self.payback_copy = None
        for p in self._opened:
            dev.ipc_close(p)
        self._opened = []
        self.barrier.close()
