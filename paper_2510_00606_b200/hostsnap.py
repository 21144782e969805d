"""Host-memory snapshots: the reference's Medium::H2D_D2D source on one node.

The reference plans a departed rank's bytes as "H2D_D2D" entries sourced from
its ring holder (param_fabric.cpp:82-121; TransferEntry::medium,
param_fabric.hpp:59-79): the paper keeps the replica in host DRAM
(PAPER.md:363-372).  The default B200 build keeps it in the holder's HBM
(recovery.RingReplica / ReplayReplica), which recovers over NVLink at
~700 GB/s.  This module is the host variant, for state too large to keep a
second copy in HBM (config D):

* every rank's shard image lives in node-shared host memory (one POSIX shm
  segment per rank), pinned and mapped for the GPUs of every rank
  (ew_host_register); the owner refreshes its own image each step with a D2H
  copy over its own PCIe link (`publish`, asynchronous on a side stream);
* at recovery the holder's REPLICA buffer in the copy-program table points at
  the departed rank's image (`attach`), so every destination's staged copy
  kernel pulls its share of the departed bytes straight from host memory
  (TMA bulk loads over its own PCIe link, all GPUs at once) — the H2D and the
  D2D hop of the reference's medium collapse into one read — while
  survivor-owned bytes still move over NVLink in the same launch.

An image outlives its owner process: survivors keep their mappings when the
owner's segment name is unlinked at its exit.
"""
from __future__ import annotations

import ctypes as C
from multiprocessing import resource_tracker, shared_memory
from typing import Dict, Iterable, Optional, Sequence

import torch
import torch.distributed as dist

from . import device as dev
from ._native import check, lib
from .fabric import ROLE_REPLICA, SnapshotRing
from .reshard import ReshardExecutor


class HostSnapshots:
    """One node-shared host image per member's shard (source layout)."""

    def __init__(self, layout, members: Sequence[int], rank: int, tag: str, group=None,
                 readable: Optional[Iterable[int]] = None):
        """Collective over `group`.  `readable`: members whose images this
        rank maps for reading at recovery (default all; its own image is
        always mapped).  A failure to map is raised only after the closing
        barrier, so no rank is left waiting."""
        self.members = list(members)
        self.rank = rank
        self.ring = SnapshotRing(self.members)
        self.nbytes: Dict[int, int] = {r: int(layout.shard_bytes(r)) for r in self.members}
        self._segs: Dict[int, shared_memory.SharedMemory] = {}
        self._addr: Dict[int, int] = {}
        self._dev: Dict[int, int] = {}
        self._views: Dict[int, torch.Tensor] = {}
        name = lambda r: f"ew_{tag}_{r}"  # noqa: E731
        own = shared_memory.SharedMemory(name=name(rank), create=True,
                                         size=max(1, self.nbytes[rank]))
        self._segs[rank] = own
        self._pieces: Dict[int, list] = {}
        self._closed = False
        dist.barrier(group)
        want = set(self.members if readable is None else readable) | {rank}
        failure = None
        try:
            for r in self.members:
                if r not in want:
                    continue
                if r != rank:
                    seg = shared_memory.SharedMemory(name=name(r))
                    # the creator owns the name; do not let this process's
                    # tracker unlink a peer's segment at exit
                    resource_tracker.unregister(seg._name, "shared_memory")
                    self._segs[r] = seg
                view = torch.frombuffer(self._segs[r].buf, dtype=torch.uint8)
                self._views[r] = view
                self._addr[r] = view.data_ptr()
                self._dev[r] = self._register(r)
        except Exception as e:  # noqa: BLE001 - re-raised after the barrier
            failure = e
        dist.barrier(group)
        if failure is not None:
            self.close()
            raise failure

    _CHUNK = 1 << 30

    def _register(self, r: int) -> int:
        """Pin member r's image.  One registration when the driver takes it;
        else 1 GiB pieces, which need the platform's identity mapping of
        registered host memory (device address == host address) to stay one
        contiguous device range."""
        addr, n = self._addr[r], max(1, self.nbytes[r])
        try:
            p = dev.host_register(addr, n)
            self._pieces[r] = [addr]
            return p
        except Exception as whole:
            pieces = []
            for off in range(0, n, self._CHUNK):
                p = dev.host_register(addr + off, min(self._CHUNK, n - off))
                pieces.append(addr + off)
                if p != addr + off:
                    for a in pieces:
                        dev.host_unregister(a)
                    raise RuntimeError("registered host memory is not identity-mapped; "
                                       f"whole-range registration failed: {whole}") from whole
            self._pieces[r] = pieces
            return addr

    def image(self, r: int) -> torch.Tensor:
        """Host view of member r's image (tests)."""
        return self._views[r][:self.nbytes[r]]

    def device_ptr(self, r: int) -> int:
        return self._dev[r]

    def publish(self, live: torch.Tensor, stream: Optional[torch.cuda.Stream] = None) -> None:
        """D2H of this rank's live shard into its image (asynchronous on
        `stream`; the caller orders it after the optimizer step)."""
        n = self.nbytes[self.rank]
        s = C.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
        base = self._addr[self.rank]
        pieces = self._pieces[self.rank] + [base + n]
        for a, b in zip(pieces[:-1], pieces[1:]):  # one copy per registration
            check(lib.ew_memcpy_async(C.c_void_p(a), C.c_void_p(live.data_ptr() + (a - base)),
                                      min(b, base + n) - a, s))

    def attach(self, ex: ReshardExecutor, departed: Iterable[int]) -> None:
        """Point the holder's REPLICA entry of ex's copy table at each
        departed rank's host image (call before ex.bind; allocate the
        executor's buffers without a device replica)."""
        table = getattr(ex, "_table", {})
        for d in departed:
            table[(ROLE_REPLICA, self.ring.backed_up_by(d))] = self._dev[d]
        ex._table = table

    def close(self) -> None:
        if self._closed:
            return
        self._closed = True
        for r in self._segs:
            for a in self._pieces.get(r, []):
                dev.host_unregister(a)
        self._views.clear()
        for r, seg in self._segs.items():
            try:
                seg.close()
            except BufferError:  # a caller still holds an image() view
                pass
            if r == self.rank:
                seg.unlink()
        self._segs.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
