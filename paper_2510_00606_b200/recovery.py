"""Measured DP recovery on B200: the data-parallel slice of the reference's
Simulation::recover_elaswave (sim.cpp:597-722), executed instead of modelled.

Per step the group keeps a same-GPU snapshot of every rank's ZeRO shard with
checksum rows (kernel (a)).  On a membership change (FailStop / ScaleIn /
ScaleOut) each surviving rank runs, in the reference's order:

  comm repair   plan_edit on the DP mesh (communicator.cpp:54-105), then the
                edit applied: ncclCommShrink of the DP communicator
  dataflow      reshard_microbatches (dataflow.cpp:52-69) -> new weights
  remap         integrity_check + overlap_matrix on the interleaved layouts,
                lowering to this GPU's copy program, CUDA-IPC peer mapping,
                one copy launch (kernel (b)) that checksums every byte it
                lands, verification by checksum conservation against the
                snapshot rows (no re-read of source or target)

and reports an MttrEvent with the reference's fields (sim.hpp:31-45) filled
with measured seconds (`mttr_csv` row format of sim.cpp:1119-1132).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import torch
import torch.distributed as dist

from . import device as dev
from .fabric import FAIL_STOP, SCALE_IN, SCALE_OUT, CommGroup, plan_edit, reshard_microbatches
from .reshard import ReshardExecutor, ReshardPlan, shard_map

KIND_NAMES = {FAIL_STOP: "fail_stop", SCALE_IN: "scale_in", SCALE_OUT: "scale_out"}


@dataclass
class MttrEvent:
    """Reference MttrEvent (sim.hpp:31-45) with measured phases."""

    step: int = 0
    t_event_s: float = 0.0
    kind: str = "fail_stop"
    detect_s: float = 0.0          # detection is outside this library (agent)
    comm_repair_s: float = 0.0     # plan_edit + ncclCommShrink
    remap_s: float = 0.0           # plan + peer map + copy + verify
    migration_stall_s: float = 0.0  # no layer migration on the DP path
    other_s: float = 0.0           # micro-batch reshape + bookkeeping
    lost_work_s: float = 0.0
    phases: Dict[str, float] = field(default_factory=dict)
    verified: bool = False

    def total_s(self) -> float:
        return (self.detect_s + self.comm_repair_s + self.remap_s + self.migration_stall_s +
                self.other_s)

    def csv_row(self, index: int) -> str:
        """One line of the reference's mttr.csv (sim.cpp:1119-1132)."""
        f = lambda x: f"{x:.9g}"
        return ",".join([str(index), str(self.step), f(self.t_event_s), self.kind, f(self.detect_s),
                         f(self.comm_repair_s), f(self.remap_s), f(self.migration_stall_s),
                         f(self.other_s), f(self.lost_work_s), f(self.total_s())])


MTTR_CSV_HEADER = ("event,step,t_event_s,kind,detect_s,comm_repair_s,remap_s,migration_stall_s,"
                   "other_s,lost_work_s,total_s")


class RingReplica:
    """Per-step ring replica maintenance on the holder.

    The paper keeps member (i+1)'s optimizer partition in member i's host
    memory and replays the Adam step there from a pushed gradient shard
    (modelled by SnapshotTimeline, param_fabric.hpp:86-96).
    On B200 the holder keeps the replica in its own HBM and, after each
    optimizer step, pulls the owner's updated shard over NVLink with the
    TMA-staged copy (11.79 GB of 7B state in ~16 ms at ~720 GB/s, overlapped
    with the next forward), then re-checksums the replica and compares it
    with the owner's snapshot rows: bit-exact by construction, verified
    without a second transfer, no optimizer replay.  The replica is packed
    like the owner's shard, so the owner's segment map and rows apply as is.
    """

    def __init__(self, layout, ring_members: Sequence[int], rank: int, replica: torch.Tensor,
                 snap: torch.Tensor, rows: torch.Tensor, block_bytes: int = dev.DEFAULT_BLOCK_BYTES,
                 group=None):
        """`snap`/`rows`: this rank's own per-step snapshot and its checksum
        rows (exported to its holder; the snapshot stays stable while the
        live state moves on to the next step); `replica`: buffer for the
        shard this rank backs up."""
        live = snap
        from .fabric import SnapshotRing
        ring = SnapshotRing(list(ring_members))
        self.rank = rank
        self.owner = ring.backs_up(rank)
        self.map = shard_map(layout, self.owner, block_bytes)
        self.replica = replica
        world = dist.get_world_size(group)
        mine = (dev.ipc_handle(live), dev.ipc_handle(rows))
        allh = [None] * world
        dist.all_gather_object(allh, (rank, mine), group=group)
        handles = dict(allh)
        (h_live, o_live), (h_rows, o_rows) = handles[self.owner]
        self._opened = [dev.ipc_open(h_live, o_live), dev.ipc_open(h_rows, o_rows)]
        n = self.map.nbytes
        self.copy = dev.CopyProgram.from_pointers([self._opened[0]], [replica.data_ptr()], [n], [True])
        self.owner_rows = torch.empty(2 * max(1, self.map.num_rows), dtype=torch.int64, device="cuda")
        self.rows_copy = dev.CopyProgram.from_pointers([self._opened[1]], [self.owner_rows.data_ptr()],
                                                       [16 * self.map.num_rows], [True])
        self.bad = torch.zeros(1, dtype=torch.int32, device="cuda")

    def refresh(self, stream=None) -> None:
        """Pull the owner's shard and its checksum rows, then verify the
        replica (bad count in self.bad).  The owner must not be writing its
        live shard meanwhile (call between its optimizer step and the next)."""
        self.copy.launch(stream=stream)
        self.rows_copy.launch(stream=stream)
        dev.verify(self.map, self.replica, self.owner_rows, self.bad, stream=stream)

    def close(self) -> None:
        self.copy = self.rows_copy = None
        for p in self._opened:
            dev.ipc_close(p)
        self._opened = []


class ReplayReplica:
    """Ring replica kept by optimizer replay: the paper's own mechanism
     with the replica in the holder's HBM.

    Each step the owner reduces its gradient shard and runs ew_adam_step on
    its AdamState; the holder runs the same ew_adam_step on its replica with
    the gradient read out of the owner's HBM through an IPC peer pointer —
    4 B/param cross NVLink instead of the 14 B/param a full state pull
    (RingReplica) moves.  The replica stays byte-identical because both sides
    execute the same explicitly-rounded kernel on the same inputs; verify()
    proves it against the owner's checksum rows without a second transfer.
    Ordering contract: the owner must not overwrite its gradient shard before
    the holder's replay of that step finished (a barrier between the replay
    and the next step's reduce)."""

    def __init__(self, ring_members: Sequence[int], rank: int, replica: "dev.AdamState",
                 grad: torch.Tensor, rows: torch.Tensor,
                 block_bytes: int = dev.DEFAULT_BLOCK_BYTES, group=None):
        """`grad`/`rows`: THIS rank's gradient shard and the checksum rows of
        its own AdamState (exported to its holder); `replica`: the AdamState
        of the member this rank backs up (same n as that member's shard)."""
        from .fabric import SnapshotRing
        ring = SnapshotRing(list(ring_members))
        self.rank = rank
        self.owner = ring.backs_up(rank)
        self.replica = replica
        self.map = dev.ShardMap(replica.segments(), block_bytes)
        world = dist.get_world_size(group)
        allh = [None] * world
        dist.all_gather_object(allh, (rank, (dev.ipc_handle(grad), dev.ipc_handle(rows))),
                               group=group)
        (h_g, o_g), (h_r, o_r) = dict(allh)[self.owner]
        self._opened = [dev.ipc_open(h_g, o_g), dev.ipc_open(h_r, o_r)]
        self.block_bytes = block_bytes
        self.owner_rows = torch.empty(2 * max(1, self.map.num_rows), dtype=torch.int64,
                                      device="cuda")
        self.replica_rows = torch.empty_like(self.owner_rows)
        self.rows_copy = dev.CopyProgram.from_pointers([self._opened[1]],
                                                       [self.owner_rows.data_ptr()],
                                                       [16 * self.map.num_rows], [True])
        self.bad = torch.zeros(1, dtype=torch.int32, device="cuda")

    def replay(self, hyper, step: int, stream=None) -> None:
        """Apply the owner's step `step` to the replica: gradient pulled over
        NVLink, update and the replica's checksum rows in one pass."""
        dev.adam_step(self._opened[0], self.replica, hyper, step, stream=stream,
                      rows=self.replica_rows, block_bytes=self.block_bytes)

    def verify(self, stream=None) -> None:
        """Compare the replica's rows (from replay) with the owner's rows
        (published by the owner's own fused step, pulled: 2.9 MB at 7B);
        mismatching rows counted in self.bad.  No re-read of the replica."""
        self.rows_copy.launch(stream=stream)
        dev.rows_diff(self.replica_rows, self.owner_rows, self.map.num_rows, self.bad,
                      stream=stream)

    def verify_by_reread(self, stream=None) -> None:
        """Stronger check: recompute the replica's rows from HBM."""
        self.rows_copy.launch(stream=stream)
        dev.verify(self.map, self.replica.buf, self.owner_rows, self.bad, stream=stream)

    def close(self) -> None:
        self.rows_copy = None
        for p in self._opened:
            dev.ipc_close(p)
        self._opened = []


class PreparedRecovery:
    """Every single-rank departure of a DP group, planned, lowered and bound
    in steady state, so a failure runs only the copy.

    The reference plans at failure time (Simulation::recover_elaswave,
    sim.cpp:597-722; overlap_matrix per event).  On B200 the inputs of a
    single departure are all known before it happens: the layouts, every
    peer's live shard and the ring replicas (RingReplica / ReplayReplica keep
    them current), so each rank builds, once, the verified pull program for
    each possible departed peer d — plan (overlap_matrix + integrity_check),
    lowering, IPC mappings and the device-resident copy program — against
    one NEW buffer sized for the largest case.  recover(d) is a table lookup
    and one launch.  Memory: one NEW shard plus a few KiB of copy items per
    scenario."""

    def __init__(self, layer_bytes: Sequence[int], members: Sequence[int], rank: int,
                 old: torch.Tensor, replica: torch.Tensor,
                 block_bytes: int = dev.DEFAULT_BLOCK_BYTES, group=None):
        """`old`: this rank's live shard; `replica`: the shard of its ring
        successor (SnapshotRing.backs_up(rank)).  Collective over `group`."""
        members = sorted(members)
        self.rank = rank
        self.block_bytes = block_bytes
        self.plans = {d: ReshardPlan.build(layer_bytes, members, [m for m in members if m != d])
                      for d in members}
        n_new = max(p.dst.shard_bytes(rank) for d, p in self.plans.items() if d != rank)
        self.new = dev.empty_bytes(n_new)
        # one steady-state exchange maps every peer's OLD and REPLICA buffer
        from .reshard import RankBuffers
        self._base = ReshardExecutor(self.plans[members[0]], rank)
        self._base.premap(RankBuffers(old, replica, None), group)
        self.execs: Dict[int, Optional[ReshardExecutor]] = {}
        for d, rp in self.plans.items():
            if d == rank:
                self.execs[d] = None  # nothing to build for one's own departure
                continue
            ex = ReshardExecutor(rp, rank)
            ex._table = dict(self._base._table)
            ex._premapped = True      # pull + premapped: bind() does no exchange
            rep = replica if rp.replica_of(rank) == d else None
            ex.bind(RankBuffers(old, rep, self.new), group, verify=True,
                    block_bytes=block_bytes)
            self.execs[d] = ex

    def recover(self, departed: int, block_sums: torch.Tensor, stream=None) -> ReshardPlan:
        """Launch the prepared program for `departed` (block_sums zeroed by
        the caller); returns its plan.  The caller all-reduces block_sums
        and compares them with the snapshot's block sums."""
        ex = self.execs[departed]
        if ex is None:
            raise ValueError("the departed rank does not recover itself")
        ex.launch(stream=stream, block_sums=block_sums)
        return self.plans[departed]

    def new_view(self, departed: int) -> torch.Tensor:
        return self.new[:self.plans[departed].dst.shard_bytes(self.rank)]

    def close(self) -> None:
        for ex in self.execs.values():
            if ex is not None:
                ex.program = None
        self.execs = {}
        self._base.close()


class DpGroup:
    """One rank's view of an interleaved-ZeRO DP group (one process per GPU)."""

    def __init__(self, layer_bytes: Sequence[int], members: Sequence[int], rank: int,
                 comm: Optional[dev.Communicator], per_slot_mbs: int = 4,
                 num_microbatches: int = 32, block_bytes: int = dev.DEFAULT_BLOCK_BYTES):
        self.layer_bytes = list(layer_bytes)
        self.members = sorted(members)
        self.rank = rank
        self.comm = comm
        self.block_bytes = block_bytes
        self.mb_sizes = [per_slot_mbs] * len(self.members)
        self.num_microbatches = num_microbatches
        self.links = {(a, b) for i, a in enumerate(self.members) for b in self.members[i + 1:]}

    def recover(self, departed: Sequence[int], bufs, push: bool = False, step: int = 0,
                kind: int = FAIL_STOP, group=None, source_sums=None) -> MttrEvent:
        """Run the DP recovery for `departed` on this (surviving) rank.
        `bufs` are this rank's RankBuffers for the change (old/replica filled);
        `source_sums`: global block sums of the state before the change
        (from the per-step snapshot rows), else recomputed from OLD/replica."""
        if kind == SCALE_OUT:
            raise NotImplementedError("DpGroup.recover handles departures (FailStop/ScaleIn); "
                                      "a rejoin grows the communicator, not shrinks it")
        unknown = sorted(set(departed) - set(self.members))
        if unknown:
            raise ValueError(f"departed ranks {unknown} are not members of the group")
        ev = MttrEvent(step=step, kind=KIND_NAMES.get(kind, "fail_stop"))
        t0 = time.perf_counter()
        # comm repair: edit plan, then the NCCL communicator shrink.  NCCL
        # excludes by rank in the CURRENT communicator, which numbers the
        # members 0..n-1 in ascending id order (it was built, or last shrunk,
        # over self.members), not by member id
        edit = plan_edit([CommGroup("dp", self.members)], kind, list(departed), self.links)
        for l in edit.links_to_remove:
            self.links.discard(l)
        self.links |= edit.links_to_add
        comm_rank = {m: i for i, m in enumerate(self.members)}
        new_comm = None
        if self.comm is not None:
            new_comm = self.comm.shrink(sorted(comm_rank[d] for d in departed))
            self.comm.destroy()  # the child exists: the parent is no longer used
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        ev.comm_repair_s = t1 - t0
        ev.phases["plan_edit_links_removed"] = len(edit.links_to_remove)

        # dataflow: global batch conserved over the survivors
        survivors = [m for m in self.members if m not in set(departed)]
        old_idx = {m: i for i, m in enumerate(self.members)}
        _, sizes = reshard_microbatches(self.mb_sizes, self.num_microbatches,
                                        [old_idx[m] for m in survivors])
        t2 = time.perf_counter()
        ev.other_s = t2 - t1

        # remap: plan -> program -> peer map -> copy -> verify.  In pull mode
        # the copy verifies on arrival (it checksums what it lands), so the
        # check is one all-reduce of block sums against the source's sums
        # (the per-step snapshot rows; recomputed here when not supplied).
        rp = ReshardPlan.build(self.layer_bytes, self.members, survivors)
        ex = ReshardExecutor(rp, self.rank, push=push)
        before = source_sums if source_sums is not None else \
            self.source_block_sums(rp, bufs, group)
        t3 = time.perf_counter()
        ex.bind(bufs, group=group, verify=not push, block_bytes=self.block_bytes)
        t4 = time.perf_counter()
        after = torch.zeros_like(before)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier(group=group)
        s.record()
        ex.launch(block_sums=after)
        e.record()
        torch.cuda.synchronize()
        dist.barrier(group=group)
        t5 = time.perf_counter()
        if push:
            ev.verified = self.verify_conservation(rp, bufs, group)
        else:
            dist.all_reduce(after, group=group)
            ev.verified = bool(torch.equal(before, after))
        t6 = time.perf_counter()
        ev.remap_s = t6 - t2
        ev.phases.update(plan_s=t3 - t2, peer_map_s=t4 - t3, copy_s=s.elapsed_time(e) / 1e3,
                         copy_wall_s=t5 - t4, verify_s=t6 - t5)
        ex.close()
        # commit the new membership
        self.members = survivors
        self.mb_sizes = sizes
        self.comm = new_comm
        return ev

    def source_block_sums(self, rp: ReshardPlan, bufs, group=None) -> torch.Tensor:
        """Global block sums of the state before the change: every live
        rank's OLD shard plus the departed ranks' bytes as their ring holders
        keep them (what the per-step snapshot rows already hold)."""
        block = self.block_bytes
        nblocks = (sum(self.layer_bytes) + block - 1) // block
        before = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
        if bufs.old is not None and self.rank in rp.old_ranks and self.rank not in rp.failed:
            m = shard_map(rp.src, self.rank, block)
            rows = m.new_row_sums()
            dev.checksum(m, bufs.old, rows)
            dev.rows_to_blocks(m, rows, before)
        if bufs.replica is not None:
            owner = rp.replica_of(self.rank)
            m = shard_map(rp.src, owner, block)
            rows = m.new_row_sums()
            dev.checksum(m, bufs.replica, rows)
            dev.rows_to_blocks(m, rows, before)
        dist.all_reduce(before, group=group)
        return before

    def verify_conservation(self, rp: ReshardPlan, bufs, group=None) -> bool:
        """Block sums of all NEW shards (re-read) == block sums of all OLD shards."""
        block = self.block_bytes
        nblocks = (sum(self.layer_bytes) + block - 1) // block
        before = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
        after = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
        if bufs.old is not None and self.rank in rp.old_ranks and self.rank not in rp.failed:
            m = shard_map(rp.src, self.rank, block)
            rows = m.new_row_sums()
            dev.checksum(m, bufs.old, rows)
            dev.rows_to_blocks(m, rows, before)
        if bufs.replica is not None:  # the dead rank's bytes as its ring holder keeps them
            owner = rp.replica_of(self.rank)
            m = shard_map(rp.src, owner, block)
            rows = m.new_row_sums()
            dev.checksum(m, bufs.replica, rows)
            dev.rows_to_blocks(m, rows, before)
        if bufs.new is not None:
            m = shard_map(rp.dst, self.rank, block)
            rows = m.new_row_sums()
            dev.checksum(m, bufs.new, rows)
            dev.rows_to_blocks(m, rows, after)
        dist.all_reduce(before, group=group)
        dist.all_reduce(after, group=group)
        return bool(torch.equal(before, after))
