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
* the images are double-buffered: step e's D2H writes slot e mod 2 while the
  other slot keeps step e-1, and a committed-epoch word in the segment's
  header page is written by the same stream right after the D2H (stream
  order, no host sync).  An owner that dies mid-copy leaves a torn slot that
  nobody reads: `attach` maps the last committed slot;
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
        # [header page: committed epoch (int64, -1 = none)][slot 0][slot 1]
        self._slot_bytes = {r: -(-max(1, n) // self._PAGE) * self._PAGE
                            for r, n in self.nbytes.items()}
        self._segs: Dict[int, shared_memory.SharedMemory] = {}
        self._addr: Dict[int, int] = {}
        self._dev: Dict[int, int] = {}
        self._views: Dict[int, torch.Tensor] = {}
        name = lambda r: f"ew_{tag}_{r}"  # noqa: E731
        own = shared_memory.SharedMemory(name=name(rank), create=True,
                                         size=self._PAGE + 2 * self._slot_bytes[rank])
        self._segs[rank] = own
        torch.frombuffer(own.buf, dtype=torch.int64, count=1).fill_(-1)
        self._epoch_dev = torch.full((1,), -1, dtype=torch.int64, device="cuda")
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
    _PAGE = 4096

    def _register(self, r: int) -> int:
        """Pin member r's segment (header + both slots).  One registration
        when the driver takes it; else 1 GiB pieces, which need the
        platform's identity mapping of registered host memory (device address
        == host address) to stay one contiguous device range.  Pieces pinned
        before a failure are released before the error propagates."""
        addr, n = self._addr[r], self._PAGE + 2 * self._slot_bytes[r]
        try:
            p = dev.host_register(addr, n)
            self._pieces[r] = [addr]
            return p
        except Exception as whole:
            pieces = []
            try:
                for off in range(0, n, self._CHUNK):
                    p = dev.host_register(addr + off, min(self._CHUNK, n - off))
                    pieces.append(addr + off)
                    if p != addr + off:
                        raise RuntimeError("registered host memory is not identity-mapped; "
                                           f"whole-range registration failed: {whole}") from whole
            except BaseException:
                for a in pieces:
                    dev.host_unregister(a)
                raise
            self._pieces[r] = pieces
            return addr

    def committed_epoch(self, r: int) -> int:
        """Last epoch member r's image committed (-1: none yet)."""
        return int(torch.frombuffer(self._segs[r].buf, dtype=torch.int64, count=1)[0])

    def _slot_off(self, r: int, epoch: int) -> int:
        return self._PAGE + (epoch % 2) * self._slot_bytes[r]

    def image(self, r: int, epoch: Optional[int] = None) -> torch.Tensor:
        """Host view of member r's image of `epoch` (default: the last
        committed one)."""
        e = self.committed_epoch(r) if epoch is None else epoch
        if e < 0:
            raise RuntimeError(f"member {r} has not committed an image yet")
        off = self._slot_off(r, e)
        return self._views[r][off:off + self.nbytes[r]]

    def device_ptr(self, r: int) -> int:
        """Device address of member r's last committed image."""
        e = self.committed_epoch(r)
        if e < 0:
            raise RuntimeError(f"member {r} has not committed an image yet")
        return self._dev[r] + self._slot_off(r, e)

    def publish(self, live: torch.Tensor, stream: Optional[torch.cuda.Stream] = None,
                epoch: Optional[int] = None) -> int:
        """D2H of this rank's live shard into the slot of `epoch` (default:
        the committed epoch + 1), then the commit word, both asynchronous on
        `stream` (the caller orders them after the optimizer step).  The
        previous epoch's slot is untouched until the next publish."""
        if epoch is None:
            epoch = self._next_epoch = getattr(self, "_next_epoch",
                                               self.committed_epoch(self.rank)) + 1
        n = self.nbytes[self.rank]
        st = stream or torch.cuda.current_stream()
        s = C.c_void_p(st.cuda_stream)
        seg = self._addr[self.rank]
        base = seg + self._slot_off(self.rank, epoch)
        cuts = sorted({a for a in self._pieces[self.rank] if base < a < base + n})
        bounds = [base] + cuts + [base + n]
        for a, b in zip(bounds[:-1], bounds[1:]):  # never across a registration
            check(lib.ew_memcpy_async(C.c_void_p(a), C.c_void_p(live.data_ptr() + (a - base)),
                                      b - a, s))
        # commit: written by the same stream after the image's last byte
        with torch.cuda.stream(st):
            self._epoch_dev.fill_(epoch)
        check(lib.ew_memcpy_async(C.c_void_p(seg), C.c_void_p(self._epoch_dev.data_ptr()), 8, s))
        return epoch

    def attach(self, ex: ReshardExecutor, departed: Iterable[int]) -> None:
        """Point the holder's REPLICA entry of ex's peer table at each
        departed rank's last committed host image (call before ex.bind;
        allocate the executor's buffers without a device replica)."""
        for d in departed:
            ex.put_peer(ROLE_REPLICA, self.ring.backed_up_by(d), self.device_ptr(d))

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
