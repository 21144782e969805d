"""Measured DP recovery on B200: the data-parallel slice of the reference's
Simulation::recover_elaswave (sim.cpp:597-722), executed instead of modelled.

The recovery runs in C++ (include/elaskit/recovery.hpp, elaskit::b200 over
the C ABI); this module is its Python binding plus the ring-replica helpers.
Per step the group keeps a same-GPU snapshot of every rank's ZeRO shard with
checksum rows (kernel (a)) and a ring replica on the holder.  On a membership
change (FailStop / ScaleIn) each surviving rank runs, in the reference's
order (a ScaleOut — joiners from the free pool — runs the same three steps
over members and joiners: grown communicator, micro-batches re-dealt, the
members' shards re-cut over the grown group, DpGroup.admit):

  comm repair   plan_edit on the DP mesh (communicator.cpp:54-105), then the
                NCCL communicator: a shrunk communicator prepared in steady
                state for every possible departure (ncclCommSplit,
                splitShare; repair = lookup + first collective) or, without
                one, ncclCommShrink at failure time
  dataflow      reshard_microbatches (dataflow.cpp:52-69) -> new weights
  remap         integrity_check + overlap_matrix on the interleaved layouts,
                lowered to this GPU's copy program (prepared in steady state
                or planned now), one copy launch (kernel (b)) that checksums
                every byte it lands, a device barrier, and checksum
                conservation reduce-scattered over peer memory

and reports an MttrEvent with the reference's fields (sim.hpp:31-45) filled
with measured seconds, rendered as the reference's mttr.csv rows
(sim.cpp:1119-1132) by the C++ library.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, Optional, Sequence

import torch
import torch.distributed as dist

from . import _native as N
from . import device as dev
from ._native import check, lib
from .fabric import FAIL_STOP, SCALE_IN, SCALE_OUT
from .rendezvous import Channel
from .reshard import ReshardPlan, shard_map

KIND_NAMES = {FAIL_STOP: "fail_stop", SCALE_IN: "scale_in", SCALE_OUT: "scale_out"}

_PHASES = ("plan_edit_s", "comm_acquire_s", "first_collective_s", "comm_prepared", "plan_s",
           "map_bind_s", "copy_s", "barrier_verify_s", "verdict_exchange_s",
           "launch_to_verdict_s", "mismatched_block_words", "barrier_timeouts", "premapped",
           "sums_s", "bind_s", "prepared", "stale_snapshots")


@dataclass
class MttrEvent:
    """Reference MttrEvent (sim.hpp:31-45) with measured phases (a view of
    the C++ record, ew_mttr_event)."""

    step: int = 0
    t_event_s: float = 0.0
    kind: str = "fail_stop"
    detect_s: float = 0.0          # detection is outside this library (agent)
    comm_repair_s: float = 0.0     # plan_edit + communicator repair + first collective
    remap_s: float = 0.0           # copy + verification (+ planning when not prepared)
    migration_stall_s: float = 0.0  # no layer migration on the DP path
    other_s: float = 0.0           # micro-batch reshape + bookkeeping
    lost_work_s: float = 0.0
    phases: Dict[str, float] = field(default_factory=dict)
    verified: bool = False

    @classmethod
    def from_c(cls, c: "N.MttrEventC") -> "MttrEvent":
        ev = cls(step=c.step, t_event_s=c.t_event_s, kind=c.kind.decode(),
                 detect_s=c.detect_s, comm_repair_s=c.comm_repair_s, remap_s=c.remap_s,
                 migration_stall_s=c.migration_stall_s, other_s=c.other_s,
                 lost_work_s=c.lost_work_s, verified=bool(c.verified))
        ev.phases = {k: getattr(c, k) for k in _PHASES if getattr(c, k) >= 0}
        return ev

    def to_c(self) -> "N.MttrEventC":
        c = N.MttrEventC()
        c.step, c.verified, c.t_event_s = self.step, int(self.verified), self.t_event_s
        c.kind = self.kind.encode()[:15]
        for k in ("detect_s", "comm_repair_s", "remap_s", "migration_stall_s", "other_s",
                  "lost_work_s"):
            setattr(c, k, getattr(self, k))
        return c

    def total_s(self) -> float:
        return (self.detect_s + self.comm_repair_s + self.remap_s + self.migration_stall_s +
                self.other_s)

    def csv_row(self, index: int) -> str:
        """One line of the reference's mttr.csv (sim.cpp:1119-1132), from C++."""
        buf = C.create_string_buffer(512)
        check(lib.ew_mttr_csv_row(C.byref(self.to_c()), int(index), buf, 512))
        return buf.value.decode()


def _csv_header() -> str:
    buf = C.create_string_buffer(256)
    check(lib.ew_mttr_csv_header(buf, 256))
    return buf.value.decode()


MTTR_CSV_HEADER = _csv_header()


class RingReplica:
    """Per-step ring replica maintenance by a full pull —
    a binding of the C++ elaskit::b200::RingReplica (ew_ring_replica).

    The paper keeps member (i+1)'s optimizer partition in member i's host
    memory and replays the Adam step there from a pushed gradient shard
    (modelled by SnapshotTimeline, param_fabric.hpp:86-96).
    For optimizers the library does not own, the holder pulls the owner's
    per-step snapshot with the staged copy over NVLink (11.79 GB of 7B state
    in ~16 ms) and verifies the replica against the owner's checksum rows,
    read in the owner's HBM: bit-exact by construction, verified without a
    second transfer.  The replica is packed like the owner's shard."""

    def __init__(self, layout, ring_members: Sequence[int], rank: int, replica: torch.Tensor,
                 snap: torch.Tensor, rows: torch.Tensor, block_bytes: int = dev.DEFAULT_BLOCK_BYTES,
                 group=None):
        """`snap`/`rows`: this rank's own per-step snapshot and its checksum
        rows (the holder reads them; the snapshot stays stable while the live
        state moves on to the next step); `replica`: buffer for the shard
        this rank backs up.  Collective over `group` (the ring's members)."""
        from .fabric import SnapshotRing
        self.rank = rank
        self.owner = SnapshotRing(list(ring_members)).backs_up(rank)
        self.map = shard_map(layout, self.owner, block_bytes)
        self.replica = replica
        self.channel = Channel.from_group(group, "ring")
        if self.channel.members != sorted(ring_members):
            raise ValueError("the group's ranks must be the ring's members")
        h = C.c_void_p()
        check(lib.ew_ring_replica_create(self.channel.handle, layout.handle,
                                         C.c_void_p(snap.data_ptr()), C.c_void_p(rows.data_ptr()),
                                         C.c_void_p(replica.data_ptr()), int(block_bytes),
                                         C.byref(h)))
        self._h = h
        self._keep = (snap, rows, layout)
        self.bad = torch.zeros(1, dtype=torch.int32, device="cuda")

    def refresh(self, stream=None) -> None:
        """Pull the owner's snapshot and verify the replica against the
        owner's rows (bad count in self.bad).  The owner must not be writing
        its snapshot meanwhile."""
        check(lib.ew_ring_replica_refresh(self._h, dev._ptr(self.bad), dev._stream(stream)))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_ring_replica_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class ReplayReplica:
    """Ring replica kept by optimizer replay — the paper's own mechanism
     with the replica in the holder's HBM; a binding of the
    C++ elaskit::b200::ReplayReplica (ew_replay_replica).

    Each step the owner reduces its gradient shard and runs ew_adam_step on
    its AdamState (with its checksum rows fused); the holder runs the same
    ew_adam_step on its replica with the gradient read out of the owner's HBM
    through an IPC peer pointer — 4 B/param cross NVLink instead of the
    14 B/param a full state pull (RingReplica) moves.  The replica stays
    byte-identical because both sides execute the same explicitly-rounded
    kernel on the same inputs; verify() proves it against the owner's rows
    without a second transfer.  Ordering contract: the owner must not
    overwrite its gradient shard before the holder's replay of that step
    finished (a barrier between the replay and the next step's reduce)."""

    def __init__(self, ring_members: Sequence[int], rank: int, replica: "dev.AdamState",
                 grad: torch.Tensor, rows: torch.Tensor,
                 block_bytes: int = dev.DEFAULT_BLOCK_BYTES, group=None):
        """`grad`/`rows`: THIS rank's gradient shard and the checksum rows of
        its own AdamState (read by its holder); `replica`: the AdamState of
        the member this rank backs up.  Collective over `group`."""
        from .fabric import SnapshotRing
        self.rank = rank
        self.owner = SnapshotRing(list(ring_members)).backs_up(rank)
        self.replica = replica
        self.map = dev.ShardMap(replica.segments(), block_bytes)
        self.block_bytes = block_bytes
        self.channel = Channel.from_group(group, "replay")
        if self.channel.members != sorted(ring_members):
            raise ValueError("the group's ranks must be the ring's members")
        p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
        h = C.c_void_p()
        check(lib.ew_replay_replica_create(
            self.channel.handle, p(grad), p(rows), p(replica.master), p(replica.exp_avg),
            p(replica.exp_avg_sq), p(replica.param), int(replica.n), p(replica.buf),
            int(replica.nbytes), int(block_bytes), C.byref(h)))
        self._h = h
        self._keep = (grad, rows)
        self.bad = torch.zeros(1, dtype=torch.int32, device="cuda")

    def replay(self, hyper, step: int, stream=None) -> None:
        """Apply the owner's step `step` to the replica: gradient pulled over
        NVLink, update and the replica's checksum rows in one pass."""
        check(lib.ew_replay_replica_replay(self._h, C.byref(hyper), int(step),
                                           dev._stream(stream)))

    def verify(self, stream=None) -> None:
        """Compare the replica's rows (from replay) with the owner's rows, read
        in the owner's HBM (2.9 MB at 7B); mismatching rows in self.bad."""
        check(lib.ew_replay_replica_verify(self._h, dev._ptr(self.bad), 0, dev._stream(stream)))

    def verify_by_reread(self, stream=None) -> None:
        """Stronger check: recompute the replica's rows from HBM."""
        check(lib.ew_replay_replica_verify(self._h, dev._ptr(self.bad), 1, dev._stream(stream)))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_replay_replica_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class PeerReduce:
    """(d) — the gradient-scale-preserving weighted reduce — fused with its
    collective over peer memory, no NCCL: a binding of the C++
    elaskit::b200::PeerReduce (ew_peer_reduce).  Collective over `group`.

    Units form: each rank passes its fp32 contribution units and weights;
    `scale()` is the fixed-point scale of the global unit set (local absmax,
    max over the ranks, ew_fixed_point_bits), `run(f)` the reduce-scatter /
    all-gather between device barriers.  Accumulator form (`acc=`): each rank
    already folded its units into an int64 accumulator; pass the scale used.
    Bit-identical to the NCCL int64 path and to one GPU folding every unit."""

    def __init__(self, out: torch.Tensor, units: Optional[Sequence[torch.Tensor]] = None,
                 weights: Optional[Sequence[float]] = None, acc: Optional[torch.Tensor] = None,
                 group=None, barrier_timeout_s: float = 30.0):
        self.channel = Channel.from_group(group, "peer_reduce")
        n = out.numel()
        h = C.c_void_p()
        if acc is not None:
            check(lib.ew_peer_reduce_create_i64(self.channel.handle, C.c_void_p(acc.data_ptr()),
                                                C.c_void_p(out.data_ptr()), n,
                                                float(barrier_timeout_s), C.byref(h)))
            self._keep = (out, acc)
        else:
            units = list(units or [])
            w = list(weights or [])
            arr = (C.c_void_p * max(1, len(units)))(*[u.data_ptr() for u in units])
            wa = (C.c_double * max(1, len(w)))(*[float(x) for x in w])
            check(lib.ew_peer_reduce_create(self.channel.handle, arr, wa, len(units),
                                            C.c_void_p(out.data_ptr()), n,
                                            float(barrier_timeout_s), C.byref(h)))
            self._keep = (out, units)
        self._h = h

    @property
    def total_units(self) -> int:
        t = C.c_int64()
        check(lib.ew_peer_reduce_info(self._h, C.byref(t), None))
        return t.value

    def scale(self, stream=None) -> int:
        f = C.c_int()
        check(lib.ew_peer_reduce_scale(self._h, dev._stream(stream), C.byref(f)))
        return f.value

    def run(self, frac_bits: int, stream=None) -> None:
        check(lib.ew_peer_reduce_run(self._h, int(frac_bits), dev._stream(stream)))

    def wait(self, stream=None) -> None:
        check(lib.ew_peer_reduce_wait(self._h, dev._stream(stream)))

    def timed_out(self) -> bool:
        t = C.c_int()
        check(lib.ew_peer_reduce_info(self._h, None, C.byref(t)))
        return bool(t.value)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_peer_reduce_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class PreparedRecovery:
    """Every single departure of a DP group, planned, lowered and bound in
    steady state, so a failure runs only the copy and its verification —
    a binding of the C++ elaskit::b200::PreparedRecovery (ew_prepared).

    The reference plans at failure time (Simulation::recover_elaswave,
    sim.cpp:597-722; overlap_matrix per event).  On B200 the inputs of a
    single departure are all known before it happens: the layouts, every
    peer's live shard and the ring replicas (RingReplica / ReplayReplica keep
    them current), so each rank builds, once, the verified pull program for
    each possible departed peer d against one NEW buffer sized for the
    largest case, and maps every peer's verification arrays.  recover(d) is
    a table lookup, one copy launch, a device barrier and a conservation
    check over peer memory."""

    def __init__(self, layer_bytes: Sequence[int], members: Sequence[int], rank: int,
                 old: torch.Tensor, replica: torch.Tensor,
                 block_bytes: int = dev.DEFAULT_BLOCK_BYTES, group=None,
                 old_rows: Optional[torch.Tensor] = None,
                 replica_rows: Optional[torch.Tensor] = None, barrier_timeout_s: float = 30.0,
                 local_replicas: bool = False):
        """`old`: this rank's live shard; `replica`: the shard of its ring
        successor (SnapshotRing.backs_up(rank)); `*_rows`: their per-step
        snapshot checksum rows (None: recomputed).  local_replicas: replica-
        aware sourcing (bytes the plan pulls from the successor's OLD shard
        come from this rank's current replica of it, in local HBM).
        Collective over `group`."""
        members = sorted(members)
        self.rank = rank
        self.block_bytes = block_bytes
        self.plans = {d: ReshardPlan.build(layer_bytes, members, [m for m in members if m != d])
                      for d in members}
        n_new = max(p.dst.shard_bytes(rank) for d, p in self.plans.items() if d != rank)
        self.new = dev.empty_bytes(n_new)
        self.channel = Channel.from_group(group, "prepared")
        if self.channel.members != members:
            raise ValueError("the group's ranks must be the DP members")
        lb = list(layer_bytes)
        h = C.c_void_p()
        check(lib.ew_prepared_create(
            self.channel.handle, N.i64_array(lb), len(lb), C.c_void_p(old.data_ptr()),
            dev._ptr(old_rows), C.c_void_p(replica.data_ptr()), dev._ptr(replica_rows),
            C.c_void_p(self.new.data_ptr()), int(self.new.numel()), int(block_bytes),
            float(barrier_timeout_s), int(bool(local_replicas)), C.byref(h)))
        self._h = h
        self._keep = (old, replica, old_rows, replica_rows)

    def recover(self, departed: int, stream=None) -> MttrEvent:
        """Survivors (all of them) run the prepared move for `departed`;
        returns the event with `verified` (checksum conservation) and the
        measured copy / barrier+verify / verdict phases."""
        ev = N.MttrEventC()
        ok = C.c_int()
        check(lib.ew_prepared_recover(self._h, int(departed), dev._stream(stream), C.byref(ev),
                                      C.byref(ok)))
        return MttrEvent.from_c(ev)

    def new_view(self, departed: int) -> torch.Tensor:
        return self.new[:self.plans[departed].dst.shard_bytes(self.rank)]

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_prepared_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class DpGroup:
    """One rank's view of an interleaved-ZeRO DP group (one process per GPU,
    or several sharing one GPU): a binding of the C++ elaskit::b200::DpGroup
    (ew_dp_group).  It owns the NCCL communicator of the (d) reduce and, in
    steady state, one shrunk communicator per possible single departure."""

    def __init__(self, layer_bytes: Sequence[int], members: Sequence[int], rank: int,
                 comm: Optional[dev.Communicator], per_slot_mbs: int = 4,
                 num_microbatches: int = 32, block_bytes: int = dev.DEFAULT_BLOCK_BYTES,
                 prepare_comms: bool = True, group=None, share_comm_resources: bool = False):
        """`comm` (over `members` in ascending order) is taken over: the
        group destroys it.  Collective over `group` (all members)."""
        self.layer_bytes = list(layer_bytes)
        self.rank = rank
        self.channel = Channel.from_group(group, "dp")
        if self.channel.members != sorted(members):
            raise ValueError("the group's ranks must be the DP members")
        raw = None
        if comm is not None:
            raw, comm._h = comm._h, None  # ownership moves to the C++ group
        h = C.c_void_p()
        check(lib.ew_dp_group_create(self.channel.handle, N.i64_array(self.layer_bytes),
                                     len(self.layer_bytes), raw, int(per_slot_mbs),
                                     int(num_microbatches), int(block_bytes),
                                     int(bool(prepare_comms)) | (2 if share_comm_resources else 0),
                                     C.byref(h)))
        self._h = h
        self._prepared: Optional[PreparedRecovery] = None

    @classmethod
    def joiner(cls, layer_bytes: Sequence[int], members: Sequence[int], rank: int,
               group_name: str, per_slot_mbs: int = 4, num_microbatches: int = 32,
               block_bytes: int = dev.DEFAULT_BLOCK_BYTES, store=None) -> "DpGroup":
        """A rank outside the group (a device from the free pool) that joins
        it at a ScaleOut: `members` are the group's current members,
        `group_name` the members' group channel name (`DpGroup.name`).  It
        learns the communicator, micro-batches and its shard in recover()."""
        from .rendezvous import default_store
        self = cls.__new__(cls)
        self.layer_bytes = list(layer_bytes)
        self.rank = rank
        self.channel = None
        self._name = group_name
        self._store = store or default_store()
        h = C.c_void_p()
        m = sorted(int(x) for x in members)
        check(lib.ew_dp_group_create_joiner(self._store.handle, group_name.encode(),
                                            N.i64_array(self.layer_bytes), len(self.layer_bytes),
                                            N.int_array(m), len(m), int(rank), int(per_slot_mbs),
                                            int(num_microbatches), int(block_bytes), C.byref(h)))
        self._h = h
        self._prepared = None
        return self

    @property
    def name(self) -> str:
        """The group channel's name (what a joiner passes to DpGroup.joiner)."""
        return self.channel.name if self.channel is not None else self._name

    def prepare_join(self, joiners: Sequence[int]) -> None:
        """Steady state before an expected ScaleOut: the grown communicator
        over members + joiners, built and warmed now (members and joiners)."""
        j = list(joiners)
        check(lib.ew_dp_group_prepare_join(self._h, N.int_array(j), len(j)))

    def premap(self, bufs, old_rows=None, replica_rows=None) -> None:
        """Steady state: map every member's OLD shard and replica once, so an
        event planned at failure time (a departure set, a ScaleOut) maps
        nothing on its critical path (members; joiners in prepare_join).
        old_rows / replica_rows: the per-step snapshot rows of those buffers
        (refreshed in place), the event's source block sums."""
        p = lambda t: C.c_void_p(t.data_ptr() if t is not None else None)  # noqa: E731
        check(lib.ew_dp_group_premap(self._h, p(bufs.old), p(bufs.replica), p(old_rows),
                                     p(replica_rows)))

    def prepare_move(self, kind: int, targets: Sequence[int], new: torch.Tensor) -> None:
        """Steady state, local: this rank's verified program for one expected
        event (departure set, or the joiners of a ScaleOut) into `new`."""
        t = list(targets)
        check(lib.ew_dp_group_prepare_move(self._h, int(kind), N.int_array(t), len(t),
                                           C.c_void_p(new.data_ptr() if new is not None
                                                      else None)))

    def admit(self, joiners: Sequence[int], bufs, step: int = 0, stream=None) -> MttrEvent:
        """ScaleOut: members (bufs.old = shard, bufs.new) and joiners (bufs.new)
        all call it; returns this rank's measured MttrEvent."""
        return self.recover(joiners, bufs, step=step, kind=SCALE_OUT, stream=stream)

    def set_snapshot_step(self, step: int) -> None:
        """The step this member's OLD shard and replica hold (the snapshot
        ring's step_tag, param_fabric.hpp:42): an event at another step fails
        its verdict (phases["stale_snapshots"])."""
        check(lib.ew_dp_group_set_snapshot_step(self._h, int(step)))

    def attach(self, prepared: Optional[PreparedRecovery]) -> None:
        self._prepared = prepared
        check(lib.ew_dp_group_attach(self._h, prepared._h if prepared is not None else None))

    def prepare(self, departures: Optional[Sequence[Sequence[int]]] = None) -> None:
        """Steady state after a change: rebuild the per-departure
        communicators — one per single departure, or one per given set of
        members leaving together (collective over the members)."""
        if departures is None:
            check(lib.ew_dp_group_prepare(self._h))
            return
        flat, offs = [], [0]
        for d in departures:
            flat += [int(x) for x in d]
            offs.append(len(flat))
        check(lib.ew_dp_group_prepare_sets(self._h, N.int_array(flat or [0]), N.int_array(offs),
                                           len(departures)))

    def recover(self, departed: Sequence[int], bufs=None, step: int = 0,
                kind: int = FAIL_STOP, stream=None) -> MttrEvent:
        """Run the DP recovery for `departed` on this (surviving) rank
        (kind SCALE_OUT: `departed` are the joiners, see admit()).
        `bufs` (reshard.RankBuffers: old / replica / new) are used when no
        prepared recovery is attached (planning at failure time)."""
        p = lambda t: C.c_void_p(t.data_ptr() if t is not None else None)  # noqa: E731
        ev = N.MttrEventC()
        d = list(departed)
        check(lib.ew_dp_group_recover(
            self._h, N.int_array(d), len(d), int(kind),
            p(bufs.old if bufs is not None else None),
            p(bufs.replica if bufs is not None else None),
            p(bufs.new if bufs is not None else None), int(step), dev._stream(stream),
            C.byref(ev)))
        return MttrEvent.from_c(ev)

    @property
    def comm(self) -> Optional[dev.Communicator]:
        """The group's current NCCL communicator (borrowed: the group owns it)."""
        h = C.c_void_p()
        check(lib.ew_dp_group_comm(self._h, C.byref(h)))
        if not h.value:
            return None
        c = dev.Communicator(h)
        c._borrowed = True
        return c

    @property
    def members(self):
        out = N.int_array([0] * 1024)
        n = C.c_int()
        check(lib.ew_dp_group_members(self._h, out, 1024, C.byref(n)))
        return list(out[:n.value])

    @property
    def mb_sizes(self):
        out = N.int_array([0] * 1024)
        n = C.c_int()
        check(lib.ew_dp_group_microbatches(self._h, out, 1024, C.byref(n)))
        return list(out[:n.value])

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_dp_group_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class FailureDetector:
    """Heartbeat failure detector of a node's DP group — a binding of the C++
    elaskit::b200::FailureDetector (ew_detector).  Each member beats every
    `period_s` once its GPU completed a tiny piece of work, into a node-shared
    shm slot; a member silent for `timeout_s` is failed.  The reference only
    charges a constant detect_s (presets.hpp:63, sim.cpp:601); wait() returns
    the measured one.  Collective over `group` (all members)."""

    def __init__(self, tag: str = "dp", period_s: float = 1e-3, timeout_s: float = 0.02,
                 group=None, channel: Optional[Channel] = None):
        self.channel = channel or Channel.from_group(group, "hb")
        h = C.c_void_p()
        check(lib.ew_detector_create(self.channel.handle, tag.encode(), float(period_s),
                                     float(timeout_s), C.byref(h)))
        self._h = h

    def failed(self):
        out = N.int_array([0] * 1024)
        n = C.c_int()
        check(lib.ew_detector_failed(self._h, out, 1024, C.byref(n)))
        return list(out[:n.value])

    def wait(self, max_wait_s: float):
        """(failed members, detect_s): blocks until a member fails or
        max_wait_s passes ([] then)."""
        out = N.int_array([0] * 1024)
        n = C.c_int()
        t = C.c_double()
        check(lib.ew_detector_wait(self._h, float(max_wait_s), out, 1024, C.byref(n),
                                   C.byref(t)))
        return list(out[:n.value]), t.value

    def stop_beating(self) -> None:
        check(lib.ew_detector_stop(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_detector_free(self._h)
            self._h = None
        if getattr(self, "channel", None) is not None:
            self.channel.close()
            self.channel = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
