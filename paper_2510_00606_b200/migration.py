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

import ctypes as C
from typing import Optional

import torch

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
    """One layer moving from the source rank to the target rank — a binding
    of the C++ elaskit::b200::LayerMigration (ew_layer_migration): the IPC
    mappings, the parameter and payback pulls, the device barrier and (for
    the plain schedule) the whole target / shadow step run in C++.

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
                 acc: torch.Tensor, group=None, transfer_ctas: int = 32,
                 barrier_timeout_s: float = 30.0):
        """transfer_ctas: CTAs of the background pulls.  Stream priority
        only orders *pending* CTAs, so a full-width copy would hold every SM
        until it finished and stall the compute stream; a few dozen CTAs
        with 96 KiB in flight each still saturate NVLink."""
        from .rendezvous import Channel
        self.transfer_ctas = transfer_ctas
        self.move = tuple(move)
        self.src, self.dst, self.rank = src_rank, dst_rank, rank
        self.params, self.acc = params, acc
        self.channel = Channel.from_group(group, "migration")
        h = C.c_void_p()
        check(lib.ew_layer_migration_create(
            self.channel.handle, int(src_rank), int(dst_rank), C.c_void_p(params.data_ptr()),
            params.numel() * params.element_size(), C.c_void_p(acc.data_ptr()), acc.numel(),
            int(transfer_ctas), float(barrier_timeout_s), C.byref(h)))
        self._h = h
        self.events = {}
        self.payback_buf = None
        if rank == dst_rank:
            p = C.c_void_p()
            check(lib.ew_layer_migration_info(h, C.byref(p), None))
            self._payback_ptr = p.value

    def plan(self, mode: int = NON_BLOCKING, **ctx) -> MigrationSchedule:
        """The reference planner (plan_layer_migration) on this move."""
        return plan_layer_migration(self.move, mode, **ctx)

    def _step(self, what: int, stream) -> None:
        check(lib.ew_layer_migration_step(self._h, what, dev._stream(stream)))

    def _timed(self, name, stream, what):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = stream or torch.cuda.current_stream()
        s.record(st)
        self._step(what, st)
        e.record(st)
        self.events[name] = (s, e)
        return e

    def pull_params(self, stream: Optional[torch.cuda.Stream] = None) -> torch.cuda.Event:
        """Target: start the parameter pull on `stream` (low priority by
        convention); returns the event that marks the parameters' arrival."""
        return self._timed("params", stream, 0)

    def shadow_done(self, stream: Optional[torch.cuda.Stream] = None) -> None:
        """Source: enqueue after the shadow instance's last fold."""
        self._step(1, stream)

    def prefetch_payback(self, stream: Optional[torch.cuda.Stream] = None) -> torch.cuda.Event:
        """Target: wait (on `stream`) until the source's shadow is done, then
        pull its accumulator into the payback buffer; returns the arrival
        event (the barrier wait is part of the timed segment)."""
        return self._timed("payback_grad", stream, 2)

    def payback(self, stream: Optional[torch.cuda.Stream] = None) -> torch.cuda.Event:
        """Target, unoverlapped variant: add the source's shadow accumulator
        into the target's straight from peer HBM (the caller orders it after
        the shadow's last fold)."""
        return self._timed("payback_grad", stream, 3)

    def run_target(self, units, weights, frac_bits: int, k: int,
                   compute: torch.cuda.Stream, transfer: torch.cuda.Stream,
                   other_work=None) -> None:
        """Target's step for this layer: units[mb] is micro-batch mb's
        gradient of the layer (fp32), weights[mb] its weight.  Micro-batches
        [0, k) run without the layer; [k, M) fold into self.acc after the
        parameters arrived; the payback joins in the last fold.  Without
        `other_work` the whole schedule is one C++ call; `other_work(mb,
        stream)` (the target's other layers during [0, k), e.g. in a
        benchmark) keeps the same schedule with the micro-batch loop here."""
        if other_work is None:
            arr = (C.c_void_p * max(1, len(units)))(*[u.data_ptr() for u in units])
            w = (C.c_double * max(1, len(weights)))(*[float(x) for x in weights])
            check(lib.ew_layer_migration_run(self._h, 1, arr, w, len(units), units[0].numel(),
                                             int(frac_bits), int(k), dev._stream(compute),
                                             dev._stream(transfer)))
            return
        M = len(units)
        arrived = self.pull_params(transfer)
        ready = self.prefetch_payback(transfer) if k > 0 else None
        for mb in range(M):
            if mb < k:
                other_work(mb, compute)
                continue
            if mb == k:
                compute.wait_event(arrived)
            last = mb == M - 1 and ready is not None
            if last:
                compute.wait_event(ready)
            dev.weighted_fold([units[mb]], [weights[mb]], frac_bits, self.acc, accumulate=True,
                              stream=compute, addend=self._payback_ptr if last else None)
        if k >= M:
            compute.wait_event(arrived)
            if ready is not None:
                compute.wait_event(ready)
                payback_accumulate(self.acc, self._payback_ptr, stream=compute)

    def run_shadow(self, units, weights, frac_bits: int, k: int,
                   compute: torch.cuda.Stream) -> None:
        """Source's shadow instance: micro-batches [0, k) of the layer, then
        the signal that releases the target's payback pull (C++)."""
        arr = (C.c_void_p * max(1, len(units)))(*[u.data_ptr() for u in units])
        w = (C.c_double * max(1, len(weights)))(*[float(x) for x in weights])
        check(lib.ew_layer_migration_run(self._h, 0, arr, w, len(units), units[0].numel(),
                                         int(frac_bits), int(k), dev._stream(compute), None))

    def timed_out(self) -> bool:
        t = C.c_int()
        check(lib.ew_layer_migration_info(self._h, None, C.byref(t)))
        return bool(t.value)

    def measured(self) -> dict:
        """Measured transfer segments (ms) after synchronisation."""
        return {k: s.elapsed_time(e) for k, (s, e) in self.events.items()}

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_layer_migration_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
