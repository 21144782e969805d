"""Interleaved-ZeRO live remap across GPUs.

One process per GPU.  Every rank runs the same host planning (integrity
check -> overlap_matrix -> lowering to its copy program, all C++), peers
exchange CUDA IPC handles of their shard buffers through the recovery
runtime's rendezvous (C++ Channel over torch.distributed's store; plumbing
only), and each GPU then executes its program in ONE kernel launch:
remote copies are 128-bit stores into peer HBM over NVLink/NVSwitch, local
copies (retained bytes, ring-holder self lanes) stream through local HBM.
No NCCL on this path — the exchange is the plan.

`emulate_on_one_gpu` runs the same programs for all ranks on a single GPU
(rank buffers side by side) so the N-rank lowering can be checked where fewer
GPUs than ranks exist.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import ctypes as C

import numpy as np
import torch

from . import _native as N
from . import device as dev
from ._native import check, lib
from .fabric import (ROLE_NEW, ROLE_OLD, ROLE_REPLICA, PartitionLayout, SnapshotRing,
                     TransferPlan, integrity_check, interleaved_layout, overlap_matrix,
                     reshard_copies)
from ._native import CoverageMismatch


@dataclass
class ReshardPlan:
    """Host-side plan of one membership change, identical on every rank."""

    layer_bytes: List[int]
    old_ranks: List[int]
    new_ranks: List[int]
    failed: List[int]
    src: PartitionLayout
    dst: PartitionLayout
    ring: SnapshotRing
    plan: TransferPlan
    plan_seconds: float

    @classmethod
    def build(cls, layer_bytes: Sequence[int], old_ranks: Sequence[int],
              new_ranks: Sequence[int]) -> "ReshardPlan":
        t0 = time.perf_counter()
        old_ranks, new_ranks = sorted(old_ranks), sorted(new_ranks)
        failed = sorted(set(old_ranks) - set(new_ranks))
        src = interleaved_layout(layer_bytes, old_ranks)
        dst = interleaved_layout(layer_bytes, new_ranks)
        ring = SnapshotRing(list(old_ranks))
        rep = integrity_check(ring, src, failed)
        if not rep.recoverable:
            raise CoverageMismatch(
                f"ranks {sorted(rep.missing)} lost together with their ring holders")
        plan = overlap_matrix(src, dst, failed, ring)
        return cls(list(layer_bytes), old_ranks, new_ranks, failed, src, dst, ring, plan,
                   time.perf_counter() - t0)

    @classmethod
    def for_stage_move(cls, src_stage_layers: Sequence[int], dst_stage_layers: Sequence[int],
                       src_gpus: Sequence[int], dst_gpus: Sequence[int],
                       contiguous: bool = False) -> "ReshardPlan":
        """Cross-stage interleaved-ZeRO layer move (SURVEY §8(f) #2,
        reference plan_zero_migration, migration.cpp:87-154): the source
        stage's TAIL layer moves to the HEAD of the destination stage (equal
        DP degree).  Both stages' state is laid out in one combined flat space
        [src layers w/o the mover | mover | dst layers], so the layer keeps its
        bytes and only changes owner: overlap_matrix then yields exactly the D
        rank-j -> rank-j sends of plan_zero_migration, and the lowering adds
        the local repacking of both stages' retained bytes.  Ranks are GPU ids
        (src_gpus[j] / dst_gpus[j] hold DP rank j of each stage).

        contiguous=True lays each stage out as default ZeRO instead (rank j of
        a stage owns the j-th equal cut of the stage's flat array), the
        baseline of the paper's Fig. 10 comparison; both stages are re-cut to
        balance, so this moves more bytes than the reference's count for the
        contiguous kind (which only re-cuts the source stage)."""
        t0 = time.perf_counter()
        src_gpus, dst_gpus = list(src_gpus), list(dst_gpus)
        if len(src_gpus) != len(dst_gpus):
            from ._native import MismatchedDpDegree
            raise MismatchedDpDegree("stages of unequal DP degree: route through overlap_matrix")
        if set(src_gpus) & set(dst_gpus):
            raise ValueError("source and destination stages must use distinct GPUs")
        d = len(src_gpus)
        keep, mover = list(src_stage_layers[:-1]), int(src_stage_layers[-1])
        layers = keep + [mover] + list(dst_stage_layers)

        def owners(stage_of_layer):
            ranges = {g: [] for g in src_gpus + dst_gpus}
            off = 0
            for li, sz in enumerate(layers):
                gpus = src_gpus if stage_of_layer(li) == 0 else dst_gpus
                for j, g in enumerate(gpus):
                    lo, hi = off + sz * j // d, off + sz * (j + 1) // d
                    if hi > lo:
                        ranges[g].append((lo, hi))
                off += sz
            return PartitionLayout.from_ranges(ranges, sum(layers))

        def contiguous_owners(split):
            ranges = {g: [] for g in src_gpus + dst_gpus}
            total = sum(layers)
            for lo0, hi0, gpus in ((0, split, src_gpus), (split, total, dst_gpus)):
                size = hi0 - lo0
                for j, g in enumerate(gpus):
                    lo, hi = lo0 + size * j // d, lo0 + size * (j + 1) // d
                    if hi > lo:
                        ranges[g].append((lo, hi))
            return PartitionLayout.from_ranges(ranges, total)

        n_keep = len(keep)
        if contiguous:
            src = contiguous_owners(sum(keep) + mover)
            dst = contiguous_owners(sum(keep))
        else:
            src = owners(lambda li: 0 if li <= n_keep else 1)   # mover still on the source stage
            dst = owners(lambda li: 0 if li < n_keep else 1)    # mover now on the destination
        plan = overlap_matrix(src, dst)
        all_gpus = sorted(src_gpus + dst_gpus)
        return cls(layers, all_gpus, all_gpus, [], src, dst, None, plan, time.perf_counter() - t0)

    def copies(self, exec_rank: int, push: bool = True) -> np.ndarray:
        return reshard_copies(self.plan, self.src, self.dst, self.failed, self.ring, exec_rank,
                              push)

    def replica_of(self, holder: int) -> Optional[int]:
        """Rank whose old shard `holder` keeps (SnapshotRing::backs_up)."""
        if self.ring is None or holder not in self.old_ranks or len(self.old_ranks) < 2:
            return None
        return self.ring.backs_up(holder)

    def traffic(self) -> Dict[str, object]:
        """Per-rank NVLink egress/ingress and local bytes of the plan (+ retained)."""
        ranks = sorted(set(self.old_ranks) | set(self.new_ranks))
        egress = {r: 0 for r in ranks}
        ingress = {r: 0 for r in ranks}
        local = {r: 0 for r in ranks}
        for e in self.plan.entries:
            n = int(e["hi"] - e["lo"])
            s, d = int(e["src_rank"]), int(e["dst_rank"])
            if s == d:
                local[s] += n
            else:
                egress[s] += n
                ingress[d] += n
        for r in ranks:
            if r in self.failed:
                continue
            for c in self.copies(r, push=True):
                if c["src_rank"] == c["dst_rank"] == r and c["src_role"] == ROLE_OLD:
                    local[r] += int(c["bytes"])
        bottleneck = max(max(egress.values()), max(ingress.values()))
        return {"egress": egress, "ingress": ingress, "local": local,
                "nvlink_bytes": sum(egress.values()), "bottleneck_bytes": bottleneck,
                "total_bytes_moved": int(self.plan.total_bytes_moved)}


@dataclass
class RankBuffers:
    old: Optional[torch.Tensor]
    replica: Optional[torch.Tensor]
    new: Optional[torch.Tensor]


def shard_map(layout: PartitionLayout, rank: int, block_bytes: int = dev.DEFAULT_BLOCK_BYTES):
    return dev.ShardMap(layout.segments(rank), block_bytes)


class PeerTable:
    """ew_peers: (role/key, member) -> device pointer, peers IPC-mapped by a
    collective exchange over a Channel (recovery.hpp PeerBuffers)."""

    def __init__(self):
        h = C.c_void_p()
        check(lib.ew_peers_create(C.byref(h)))
        self._h = h

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def exchange(self, channel, mine: Dict[int, Optional[int]]) -> None:
        items = [(k, p) for k, p in mine.items() if p]
        keys = N.int_array([k for k, _ in items])
        ptrs = (C.c_void_p * max(1, len(items)))(*[p for _, p in items])
        check(lib.ew_peers_exchange(self._h, channel.handle, keys, ptrs, len(items)))

    def put(self, key: int, member: int, ptr: int) -> None:
        check(lib.ew_peers_put(self._h, int(key), int(member), C.c_void_p(ptr)))

    def get(self, key: int, member: int) -> Optional[int]:
        p = C.c_void_p()
        check(lib.ew_peers_get(self._h, int(key), int(member), C.byref(p)))
        return p.value

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_peers_free(self._h)  # closes the IPC mappings
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class ReshardExecutor:
    """One rank's reshard executor: the C++ elaskit::b200::ReshardExecutor
    (ew_reshard) over a peer table exchanged through the recovery runtime's
    rendezvous (Channel over the torch.distributed group's store)."""

    def __init__(self, rp: ReshardPlan, rank: int, push: bool = False):
        # pull is the default: each receiver's TMA ring keeps ~100 KB of peer
        # loads in flight per SM, which saturates NVLink better than posted
        # stores from the (hot-spotted) ring holder (profiles/r01_reshard_*)
        self.rp = rp
        self.rank = rank
        self.push = push
        self.program: Optional[C.c_void_p] = None  # the bound ew_reshard
        self.peers = PeerTable()
        self._premapped = False

    def allocate(self, in_place: bool = False, device_replica: bool = True) -> RankBuffers:
        """Buffers of this rank.  in_place=True aliases NEW and OLD inside one
        allocation when that is provably safe — every retained byte keeps
        its address (one common shift s: OLD = buf[s:], NEW = buf[:]) and no
        incoming byte lands on the OLD range — so retained bytes are not
        copied at all (the program skips self-copies).  This is the case for
        cross-stage layer moves (the source stage drops its tail, the
        destination stage grows at its head); otherwise separate buffers.
        device_replica=False: the departed ranks' bytes come from host
        images (hostsnap.HostSnapshots.attach), no HBM replica buffer."""
        rp, r = self.rp, self.rank
        rep_of = rp.replica_of(r)
        replica = (dev.empty_bytes(rp.src.shard_bytes(rep_of))
                   if device_replica and rep_of is not None and rep_of in rp.failed else None)
        n_old = rp.src.shard_bytes(r) if r in rp.old_ranks else 0
        n_new = rp.dst.shard_bytes(r) if r in rp.new_ranks else 0
        if in_place and n_old and n_new:
            pulls = rp.copies(r, push=False)
            kept = pulls[(pulls["src_rank"] == r) & (pulls["src_role"] == ROLE_OLD)]
            shifts = set((kept["dst_off"] - kept["src_off"]).tolist())
            if len(shifts) == 1 and min(shifts) >= 0:
                s = shifts.pop()
                incoming = pulls[~((pulls["src_rank"] == r) & (pulls["src_role"] == ROLE_OLD))]
                lo, hi = incoming["dst_off"], incoming["dst_off"] + incoming["bytes"]
                overlaps = bool(((lo < s + n_old) & (hi > s)).any()) if len(incoming) else False
                if not overlaps and s % 16 == 0:
                    buf = dev.empty_bytes(max(n_new, s + n_old))
                    return RankBuffers(buf[s:s + ((n_old + 15) // 16) * 16], replica, buf)
        old = dev.empty_bytes(n_old) if r in rp.old_ranks else None
        new = dev.empty_bytes(n_new) if r in rp.new_ranks else None
        return RankBuffers(old, replica, new)

    @staticmethod
    def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
        return t.data_ptr() if t is not None else None

    def premap(self, bufs: RankBuffers, group=None) -> None:
        """Steady-state peer mapping (before any failure): import every peer's
        OLD and REPLICA buffers.  A pull-mode reshard reads only those, so a
        recovery that premapped pays no cudaIpcOpenMemHandle on its critical
        path (bind() then only builds the program).  Collective over group."""
        from .rendezvous import Channel
        ch = Channel.from_group(group, "premap")
        self.peers.exchange(ch, {ROLE_OLD: self._ptr(bufs.old),
                                 ROLE_REPLICA: self._ptr(bufs.replica)})
        self._premapped = True

    def put_peer(self, role: int, member: int, ptr: int) -> None:
        """Enter a buffer by hand (e.g. a departed rank's host image as the
        holder's REPLICA, hostsnap.HostSnapshots.attach)."""
        self.peers.put(role, member, ptr)

    def bind(self, bufs: RankBuffers, group=None, verify: bool = False,
             block_bytes: int = dev.DEFAULT_BLOCK_BYTES) -> None:
        """Map the peer buffers (unless premapped for a pull) and build this
        GPU's program.  Collective over `group`: every rank calls it, and the
        exchange is skipped only when every rank premapped for a pull (the
        same decision everywhere).  verify=True (pull mode): the program
        checksums every byte it lands in NEW (verification on arrival,
        launch(block_sums=...))."""
        if verify and self.push:
            raise ValueError("verification on arrival needs pull mode (every byte landing "
                             "in NEW is then issued by its own GPU)")
        if not (self._premapped and not self.push):
            from .rendezvous import Channel
            ch = Channel.from_group(group, "bind")
            self.peers.exchange(ch, {ROLE_OLD: self._ptr(bufs.old),
                                     ROLE_REPLICA: self._ptr(bufs.replica),
                                     ROLE_NEW: self._ptr(bufs.new)})
        for role, t in ((ROLE_OLD, bufs.old), (ROLE_REPLICA, bufs.replica), (ROLE_NEW, bufs.new)):
            if t is not None:
                self.peers.put(role, self.rank, t.data_ptr())
        self._free_program()
        rp = self.rp
        ring = rp.ring.members if rp.ring is not None else []
        h = C.c_void_p()
        check(lib.ew_reshard_create(rp.src.handle, rp.dst.handle, N.int_array(rp.failed),
                                    len(rp.failed), N.int_array(ring), len(ring), self.rank,
                                    int(self.push), int(block_bytes), C.byref(h)))
        self.program = h
        self._verified = bool(verify) and bufs.new is not None
        check(lib.ew_reshard_bind(h, self.peers.handle, int(bool(verify))))

    def launch(self, n_ctas: int = 0, remote_ctas: int = 0, stream=None,
               block_sums=None, abort_flag: Optional[int] = None) -> None:
        if self.program is not None:
            check(lib.ew_reshard_launch(self.program,
                                        dev._ptr(block_sums) if self._verified else None,
                                        C.c_void_p(abort_flag) if abort_flag else None,
                                        int(n_ctas), int(remote_ctas), dev._stream(stream)))

    def _free_program(self) -> None:
        if self.program is not None and self.program.value and lib is not None:
            lib.ew_reshard_free(self.program)
        self.program = None

    def close(self) -> None:
        self._free_program()
        self.peers.close()
        self.peers = PeerTable()
        self._premapped = False

    def __del__(self):
        try:
            self._free_program()
        except Exception:  # noqa: BLE001
            pass


def _aliases(a, b) -> bool:
    """True when two byte tensors share storage bytes (in-place buffers)."""
    a0, a1 = a.data_ptr(), a.data_ptr() + a.numel()
    b0, b1 = b.data_ptr(), b.data_ptr() + b.numel()
    return a0 < b1 and b0 < a1


def emulate_on_one_gpu(rp: ReshardPlan, seed: int, push: bool = True,
                       block_bytes: int = dev.DEFAULT_BLOCK_BYTES, block_sums=None,
                       tamper=None, in_place: bool = False):
    """Run every rank's program on the current GPU; returns (new buffers,
    expected buffers) keyed by rank for comparison.  block_sums (pull only):
    run verified programs, every rank adding what it lands there.
    tamper(rank, descs) may edit a rank's descriptors (negative tests)."""
    bufs: Dict[int, RankBuffers] = {}
    for r in sorted(set(rp.old_ranks) | set(rp.new_ranks)):
        ex = ReshardExecutor(rp, r, push)
        bufs[r] = ex.allocate(in_place)
        if bufs[r].old is not None and r not in rp.failed:
            dev.fill_synthetic(shard_map(rp.src, r, block_bytes), bufs[r].old, seed)
        if bufs[r].replica is not None:
            dev.fill_synthetic(shard_map(rp.src, rp.replica_of(r), block_bytes), bufs[r].replica,
                               seed)
        b = bufs[r]
        if b.new is not None and (b.old is None or not _aliases(b.new, b.old)):
            b.new.fill_(0xA5)  # poison (an in-place NEW holds the retained bytes)
    table = {}
    for r, b in bufs.items():
        for role, t in ((ROLE_OLD, b.old), (ROLE_REPLICA, b.replica), (ROLE_NEW, b.new)):
            if t is not None:
                table[(role, r)] = t.data_ptr()
    n_table = max(bufs) + 1
    progs = []
    for r in bufs:
        if r in rp.failed:
            continue
        descs = rp.copies(r, push)
        if tamper is not None:
            descs = tamper(r, descs)
        vmap = shard_map(rp.dst, r, block_bytes) \
            if block_sums is not None and r in rp.new_ranks else None
        progs.append(dev.CopyProgram.from_descs(descs, table, n_table, r, vmap))
    for p in progs:
        p.launch(block_sums=block_sums if getattr(p, "_verify_map", None) is not None else None)
    torch.cuda.synchronize()
    expected = {}
    for r in rp.new_ranks:
        e = dev.empty_bytes(rp.dst.shard_bytes(r))
        dev.fill_synthetic(shard_map(rp.dst, r, block_bytes), e, seed)
        expected[r] = e
    return {r: bufs[r].new for r in rp.new_ranks}, expected
