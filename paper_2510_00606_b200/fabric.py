"""Planning API of the recovery path, mirrored from the reference's C++ headers.

Python callers (tests, bench, the multi-rank executor) use these wrappers; each
one is a thin call through include/ew_api.h into the C++ implementation in
libelaskit_b200.so, keeping the reference's names, argument meaning and
exception types (reference: proj/include/elaskit/param_fabric.hpp,
migration.hpp, rng.hpp, dataflow.hpp, communicator.hpp).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import Dict, Iterable, List, Optional, Sequence, Set, Tuple

import numpy as np

from . import _native as N
from ._native import (CoverageMismatch, DisconnectedGroup, MissingBackup,  # noqa: F401
                      MismatchedDpDegree, NoSurvivors, DimensionMismatch, check, lib)

D2D, H2D_D2D = 0, 1
ROLE_OLD, ROLE_REPLICA, ROLE_NEW = 0, 1, 2

ENTRY_DTYPE = np.dtype([("src_rank", np.int32), ("dst_rank", np.int32), ("lo", np.int64),
                        ("hi", np.int64), ("medium", np.int32), ("reserved", np.int32)])
SEGMENT_DTYPE = np.dtype([("global_lo", np.int64), ("length", np.int64), ("local_off", np.int64)])
COPY_DTYPE = np.dtype([("src_role", np.int32), ("src_rank", np.int32), ("dst_role", np.int32),
                       ("dst_rank", np.int32), ("src_off", np.int64), ("dst_off", np.int64),
                       ("bytes", np.int64)])


class PartitionLayout:
    """rank -> sorted disjoint byte intervals over [0, total_bytes)
    (reference param_fabric.hpp:27-33).  Owns an ew_layout handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_layout_free(self._h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @classmethod
    def from_ranges(cls, ranges: Dict[int, Sequence[Tuple[int, int]]], total_bytes: int):
        ranks = sorted(ranges)
        counts = [len(ranges[r]) for r in ranks]
        ivs = [iv for r in ranks for iv in ranges[r]]
        arr = (N.Interval * max(1, len(ivs)))(*[N.Interval(int(a), int(b)) for a, b in ivs])
        out = C.c_void_p()
        check(lib.ew_layout_from_intervals(N.int_array(ranks), N.int_array(counts), len(ranks),
                                           arr, int(total_bytes), C.byref(out)))
        return cls(out.value)

    @property
    def total_bytes(self) -> int:
        return lib.ew_layout_total_bytes(self._h)

    @property
    def ranks(self) -> List[int]:
        n = lib.ew_layout_num_ranks(self._h)
        buf = (C.c_int * max(1, n))()
        check(lib.ew_layout_ranks(self._h, buf, n))
        return list(buf[:n])

    def segments(self, rank: int) -> np.ndarray:
        """Packed-buffer segment map of `rank` (elaskit/b200.hpp shard_segments)."""
        n = lib.ew_layout_num_segments(self._h, rank)
        arr = np.zeros(max(1, n), dtype=SEGMENT_DTYPE)
        check(lib.ew_layout_segments(self._h, rank, arr.ctypes.data_as(C.POINTER(N.Segment)), n))
        return arr[:n]

    def intervals(self, rank: int) -> List[Tuple[int, int]]:
        s = self.segments(rank)
        return [(int(a), int(a + b)) for a, b in zip(s["global_lo"], s["length"])]

    @property
    def ranges(self) -> Dict[int, List[Tuple[int, int]]]:
        return {r: self.intervals(r) for r in self.ranks}

    def shard_bytes(self, rank: int) -> int:
        return lib.ew_layout_shard_bytes(self._h, rank)

    def owner_of(self, byte: int) -> int:
        return lib.ew_layout_owner_of(self._h, int(byte))

    def validate(self) -> None:
        check(lib.ew_layout_validate(self._h))


def contiguous_layout(ranks: Sequence[int], total: int) -> PartitionLayout:
    """Reference param_fabric.cpp:36-49."""
    out = C.c_void_p()
    check(lib.ew_layout_contiguous(N.int_array(ranks), len(ranks), int(total), C.byref(out)))
    return PartitionLayout(out.value)


def interleaved_layout(layer_bytes: Sequence[int], ranks: Sequence[int]) -> PartitionLayout:
    """Interleaved ZeRO ownership (ZeroLayout::shard, migration.cpp:73-77)
    composed into a PartitionLayout."""
    out = C.c_void_p()
    check(lib.ew_layout_interleaved(N.i64_array(layer_bytes), len(layer_bytes),
                                    N.int_array(ranks), len(ranks), C.byref(out)))
    return PartitionLayout(out.value)


@dataclass
class SnapshotRing:
    """Member i keeps the snapshot of member (i+1) mod n (param_fabric.cpp:51-64)."""

    members: List[int]
    step_tag: int = 0

    def backed_up_by(self, rank: int) -> int:
        i = self.members.index(rank)
        return self.members[(i - 1) % len(self.members)]

    def backs_up(self, rank: int) -> int:
        i = self.members.index(rank)
        return self.members[(i + 1) % len(self.members)]


@dataclass
class IntegrityReport:
    recoverable: bool
    missing: Dict[int, List[Tuple[int, int]]] = field(default_factory=dict)


def integrity_check(ring: SnapshotRing, layout: PartitionLayout,
                    failed: Iterable[int]) -> IntegrityReport:
    """Reference param_fabric.cpp:66-80."""
    failed = sorted(set(failed))
    rec = C.c_int()
    miss = (C.c_int * max(1, len(failed)))()
    nm = C.c_int()
    check(lib.ew_integrity_check(N.int_array(ring.members), len(ring.members), layout.handle,
                                 N.int_array(failed), len(failed), C.byref(rec), miss,
                                 len(failed), C.byref(nm)))
    return IntegrityReport(bool(rec.value),
                           {r: layout.intervals(r) if r in layout.ranks else []
                            for r in miss[:nm.value]})


class TransferPlan:
    """Reference TransferPlan (param_fabric.hpp:68-71); `entries` is a numpy
    structured array (src_rank, dst_rank, lo, hi, medium) ordered by lo."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        n = lib.ew_plan_num_entries(self._h)
        self.entries = np.zeros(max(1, n), dtype=ENTRY_DTYPE)
        check(lib.ew_plan_entries(self._h, self.entries.ctypes.data_as(C.POINTER(N.TransferEntry)), n))
        self.entries = self.entries[:n]
        self.total_bytes_moved = lib.ew_plan_total_bytes_moved(self._h)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_plan_free(self._h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def __len__(self) -> int:
        return len(self.entries)

    def to_json(self) -> dict:
        """plan_to_json (param_fabric.cpp:123-134)."""
        need = C.c_int64()
        lib.ew_plan_to_json(self._h, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        check(lib.ew_plan_to_json(self._h, buf, need.value, C.byref(need)))
        return json.loads(buf.value.decode())

    def lane_bytes(self) -> Dict[Tuple[int, int], int]:
        lanes: Dict[Tuple[int, int], int] = {}
        for e in self.entries:
            k = (int(e["src_rank"]), int(e["dst_rank"]))
            lanes[k] = lanes.get(k, 0) + int(e["hi"] - e["lo"])
        return lanes


def overlap_matrix(src: PartitionLayout, dst: PartitionLayout, failed: Iterable[int] = (),
                   ring: Optional[SnapshotRing] = None) -> TransferPlan:
    """Reference param_fabric.cpp:82-121 (same entries, same exceptions)."""
    failed = sorted(set(failed))
    members = ring.members if ring is not None else []
    out = C.c_void_p()
    check(lib.ew_overlap_matrix(src.handle, dst.handle, N.int_array(failed), len(failed),
                                N.int_array(members), len(members), C.byref(out)))
    return TransferPlan(out.value)


def reshard_copies(plan: TransferPlan, src: PartitionLayout, dst: PartitionLayout,
                   failed: Iterable[int], ring: Optional[SnapshotRing], exec_rank: int,
                   push: bool = True) -> np.ndarray:
    """Copy descriptors GPU `exec_rank` issues for `plan` (elaskit/b200.hpp)."""
    failed = sorted(set(failed))
    members = ring.members if ring is not None else []
    n = C.c_int64()
    lib.ew_reshard_copies(plan.handle, src.handle, dst.handle, N.int_array(failed), len(failed),
                          N.int_array(members), len(members), exec_rank, int(push), None, 0,
                          C.byref(n))
    arr = np.zeros(max(1, n.value), dtype=COPY_DTYPE)
    check(lib.ew_reshard_copies(plan.handle, src.handle, dst.handle, N.int_array(failed),
                                len(failed), N.int_array(members), len(members), exec_rank,
                                int(push), arr.ctypes.data_as(C.POINTER(N.CopyDesc)), n.value,
                                C.byref(n)))
    return arr[:n.value]


# ----------------------------------------------------------------- dataflow ---

def reshard_microbatches(per_slot_mbs: Sequence[int], num_microbatches: int,
                         survivors: Sequence[int]) -> Tuple[List[int], List[int]]:
    """Reference dataflow.cpp:52-69 -> (sorted slots, per-slot micro-batch sizes)."""
    n = len(survivors)
    slots = (C.c_int * max(1, n))()
    mbs = (C.c_int * max(1, n))()
    check(lib.ew_reshard_microbatches(N.int_array(per_slot_mbs), len(per_slot_mbs),
                                      num_microbatches, N.int_array(survivors), n, slots, mbs))
    return list(slots[:n]), list(mbs[:n])


def sample_ranges(per_slot_mbs: Sequence[int], step_base: int, mb: int) -> List[Tuple[int, int]]:
    """Reference dataflow.cpp:30-40 (pure arithmetic)."""
    out, cur = [], step_base + mb * sum(per_slot_mbs)
    for m in per_slot_mbs:
        out.append((cur, cur + m))
        cur += m
    return out


def sample_reassignments(old_slots: Sequence[int], old_mbs: Sequence[int],
                         new_slots: Sequence[int], new_mbs: Sequence[int]) -> List[Tuple[int, int, int]]:
    """SampleReassignment derivation (reference sim.cpp:694-715)."""
    cap = max(1, sum(old_mbs))
    rows = np.zeros(3 * cap, dtype=np.int64)
    n = C.c_int64()
    check(lib.ew_sample_reassignments(N.int_array(old_slots), N.int_array(old_mbs), len(old_slots),
                                      N.int_array(new_slots), N.int_array(new_mbs), len(new_slots),
                                      rows.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(n)))
    return [tuple(int(x) for x in rows[3 * i:3 * i + 3]) for i in range(n.value)]


def plan_zero_migration(interleaved: bool, dp_degree: int, layer_bytes: Sequence[int],
                        layer_idx: int, dst_dp_degree: int):
    """Reference migration.cpp:87-154 -> (rows {src,dst,cross,lo,hi,round}, totals)."""
    cap = 4 * max(1, dp_degree) ** 2 + 64
    rows = np.zeros(6 * cap, dtype=np.int64)
    tot = np.zeros(3, dtype=np.int64)
    n = C.c_int64()
    check(lib.ew_plan_zero_migration(int(interleaved), dp_degree, N.i64_array(layer_bytes),
                                     len(layer_bytes), layer_idx, dst_dp_degree,
                                     rows.ctypes.data_as(C.POINTER(C.c_int64)), cap, C.byref(n),
                                     tot.ctypes.data_as(C.POINTER(C.c_int64))))
    return rows[:6 * n.value].reshape(-1, 6), tot


BLOCKING, NON_BLOCKING = 0, 1


@dataclass
class MigrationSchedule:
    """Reference MigrationSchedule (migration.hpp:29-39); transfers are
    (what, start_s, end_s, bytes) with what in {"params", "payback_grad"}."""

    mode: int
    transfers: List[Tuple[str, float, float, int]]
    shadow_microbatches: int
    payback_bytes: int
    stall_s: float
    total_time_s: float


def plan_layer_migration(move: Tuple[int, int, int], mode: int, *, param_bytes: int,
                         grad_bytes: int, link_bw_bytes_per_s: float, microbatch_slot_s: float,
                         num_microbatches: int, target_headroom_bytes: int,
                         fixed_overhead_s: float = 0.0) -> MigrationSchedule:
    """Reference plan_layer_migration (migration.cpp:9-61); move = (layer,
    src_stage, dst_stage).  Raises InsufficientTargetMemory like the reference."""
    ctx = N.MigrationContext(param_bytes, grad_bytes, link_bw_bytes_per_s, microbatch_slot_s,
                             num_microbatches, target_headroom_bytes, fixed_overhead_s)
    out = N.MigrationSchedule()
    check(lib.ew_plan_layer_migration(int(move[0]), int(move[1]), int(move[2]), int(mode),
                                      C.byref(ctx), C.byref(out)))
    tr = [("payback_grad" if out.transfers[k].what else "params", out.transfers[k].start_s,
           out.transfers[k].end_s, out.transfers[k].bytes) for k in range(out.n_transfers)]
    return MigrationSchedule(out.mode, tr, out.shadow_microbatches, out.payback_bytes,
                             out.stall_s, out.total_time_s)


def weighted_grad_average(weights: Sequence[float], grads: np.ndarray) -> np.ndarray:
    """Reference dataflow.cpp:71-83 (fp64 left fold, host)."""
    g = np.ascontiguousarray(grads, dtype=np.float64)
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = np.zeros(g.shape[1] if g.ndim == 2 else 0, dtype=np.float64)
    check(lib.ew_weighted_grad_average(w.ctypes.data_as(C.POINTER(C.c_double)),
                                       g.ctypes.data_as(C.POINTER(C.c_double)), len(w),
                                       out.size, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


# ---------------------------------------------------------------------- rng ---

def philox4x64(counter: Sequence[int], key: Sequence[int]) -> List[int]:
    c = (C.c_uint64 * 4)(*counter)
    k = (C.c_uint64 * 2)(*key)
    o = (C.c_uint64 * 4)()
    check(lib.ew_philox4x64(c, k, o))
    return list(o)


def draw(seed: int, sample_id: int, layer_id: int, op_index: int, n: int) -> np.ndarray:
    out = np.zeros(max(1, n), dtype=np.float64)
    check(lib.ew_draw(seed, sample_id, layer_id, op_index, n,
                      out.ctypes.data_as(C.POINTER(C.c_double))))
    return out[:n]


# ------------------------------------------------------------- communicator ---

FAIL_STOP, FAIL_SLOW, SCALE_IN, SCALE_OUT = 0, 1, 2, 3


@dataclass
class CommGroup:
    id: str
    members: List[int]
    ring: bool = False


@dataclass
class EditPlan:
    links_to_add: Set[Tuple[int, int]]
    links_to_remove: Set[Tuple[int, int]]
    groups_touched: Set[str]


def plan_edit(groups: Sequence[CommGroup], kind: int, targets: Sequence[int],
              pool: Iterable[Tuple[int, int]]) -> EditPlan:
    """Reference communicator.cpp:54-105."""
    pool = sorted({(min(a, b), max(a, b)) for a, b in pool})
    ids = (C.c_char_p * max(1, len(groups)))(*[g.id.encode() for g in groups])
    topo = N.int_array([1 if g.ring else 0 for g in groups])
    nmem = N.int_array([len(g.members) for g in groups])
    mem = N.int_array([m for g in groups for m in g.members])
    flat_pool = N.int_array([x for l in pool for x in l])
    cap = sum(len(g.members) ** 2 for g in groups) + len(pool) + 4
    add = (C.c_int * (2 * cap))()
    rem = (C.c_int * (2 * cap))()
    touched = (C.c_int * max(1, len(groups)))()
    na, nr, nt = C.c_int(), C.c_int(), C.c_int()
    check(lib.ew_plan_edit(len(groups), ids, topo, nmem, mem, kind, N.int_array(targets),
                           len(targets), flat_pool, len(pool), add, cap, C.byref(na), rem, cap,
                           C.byref(nr), touched, C.byref(nt)))
    return EditPlan({(add[2 * i], add[2 * i + 1]) for i in range(na.value)},
                    {(rem[2 * i], rem[2 * i + 1]) for i in range(nr.value)},
                    {groups[touched[i]].id for i in range(nt.value)})
