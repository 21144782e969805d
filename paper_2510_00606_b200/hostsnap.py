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
owner's segment name is unlinked at its exit.  The segments, pinning,
publish and commit run in C++ (elaskit::b200::HostImages); this module binds
them.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Iterable, Optional, Sequence

import torch

from . import _native as N
from . import device as dev
from ._native import check, lib
from .fabric import ROLE_REPLICA, SnapshotRing
from .reshard import ReshardExecutor


class HostSnapshots:
    """One node-shared host image per member's shard (source layout): a
    binding of the C++ elaskit::b200::HostImages (ew_host_images)."""

    def __init__(self, layout, members: Sequence[int], rank: int, tag: str, group=None,
                 readable: Optional[Iterable[int]] = None, map_for_device: bool = True,
                 channel=None):
        """Collective over `group` (or an explicit rendezvous `channel`).
        `readable`: members whose images this rank maps for reading at
        recovery (default all; its own image is always mapped).  A failure to
        map is raised only after the closing barrier, so no rank is left
        waiting.  map_for_device=False: no pinning (host-side users)."""
        from .rendezvous import Channel
        self.members = list(members)
        self.rank = rank
        self.ring = SnapshotRing(self.members)
        self.nbytes: Dict[int, int] = {r: int(layout.shard_bytes(r)) for r in self.members}
        self.channel = channel if channel is not None else Channel.from_group(group, "hostsnap")
        rd = sorted(set(readable)) if readable is not None else []
        h = C.c_void_p()
        check(lib.ew_host_images_create(self.channel.handle, layout.handle, tag.encode(),
                                        N.int_array(rd), len(rd), int(bool(map_for_device)),
                                        C.byref(h)))
        self._h = h
        self._layout = layout

    def committed_epoch(self, r: int) -> int:
        """Last epoch member r's image committed (-1: none yet)."""
        e = C.c_int64()
        check(lib.ew_host_images_committed(self._h, int(r), C.byref(e)))
        return e.value

    def image(self, r: int, epoch: Optional[int] = None) -> torch.Tensor:
        """Host view of member r's image of `epoch` (default: the last
        committed one)."""
        p, n = C.c_void_p(), C.c_int64()
        check(lib.ew_host_images_host_ptr(self._h, int(r), -1 if epoch is None else int(epoch),
                                          C.byref(p), C.byref(n)))
        buf = (C.c_uint8 * max(1, n.value)).from_address(p.value)
        return torch.frombuffer(buf, dtype=torch.uint8)[:n.value]

    def device_ptr(self, r: int) -> int:
        """Device address of member r's last committed image."""
        p = C.c_void_p()
        check(lib.ew_host_images_device_ptr(self._h, int(r), C.byref(p)))
        return int(p.value)

    def publish(self, live: torch.Tensor, stream: Optional[torch.cuda.Stream] = None,
                epoch: Optional[int] = None) -> int:
        """D2H of this rank's live shard into the slot of `epoch` (default:
        the next one), then the commit word, both asynchronous on `stream`
        (the caller orders them after the optimizer step).  The previous
        epoch's slot is untouched until the next publish."""
        e = C.c_int64()
        check(lib.ew_host_images_publish(self._h, C.c_void_p(live.data_ptr()),
                                         -1 if epoch is None else int(epoch), dev._stream(stream),
                                         C.byref(e)))
        return e.value

    def commit_host(self, epoch: int) -> None:
        """Host-side commit (a publisher that wrote the image itself)."""
        check(lib.ew_host_images_commit_host(self._h, int(epoch)))

    def attach(self, ex: ReshardExecutor, departed: Iterable[int]) -> None:
        """Point the holder's REPLICA entry of ex's peer table at each
        departed rank's last committed host image (call before ex.bind;
        allocate the executor's buffers without a device replica)."""
        for d in departed:
            ex.put_peer(ROLE_REPLICA, self.ring.backed_up_by(d), self.device_ptr(d))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_host_images_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
