"""Staged in-place reshard for ZeRO state that fills HBM.

The plain executor keeps a rank's OLD shard, the ring replica it holds and
the NEW shard side by side: about 3.1 S of HBM for a shard of S bytes, so a
180 GB B200 reshards at most S ~ 55 GB that way.  Here OLD and NEW share one
allocation of max(|OLD|, |NEW|) bytes, and the move runs in phases over the
global byte space.

Geometry.  A rank's packed offsets are monotone in the global position: for
a global boundary G let old(G), new(G) be the bytes the rank holds below G
in OLD and in NEW.  When shards grow (a departure) phases run from the top
of the global space down, cut only where new(G) >= old(G) on every rank
(every layer boundary qualifies; cut points inside a layer are tested); when
shards shrink (a join) they run upwards with new(G) <= old(G).  Phase j in
processing order reads R_j = [old(G_lo_j), old(G_hi_j)) of every rank's OLD
and writes W_j = [new(G_lo_j), new(G_hi_j)) of its NEW; with the cut rule,
the reads of every later phase lie beyond W_j (below it for departures).

Execution (C++, elaskit::b200::InPlaceExecutor), per rank (three streams,
`s` = slack):
  gather_j   waits until every rank finished gather_{j-s-1}, then pulls the
             phase's NEW bytes (peers' OLD, ring replicas, own OLD): the part
             of W_j clear of R_{j-s} .. R_j lands DIRECTLY in NEW, the rest in
             staging[j % (s+2)]; both checksummed on arrival (kernel (a)'s
             spec, labelled by the byte's global position in NEW);
  barrier_j  (own stream) stream-ordered cross-GPU barrier after gather_j:
             every rank has read R_j;
  flush_j    (own stream) after barrier_j: staging -> its W_j range.
So ranks run up to s+1 phases apart and only the bytes of the few phases
whose W_j still overlaps unread OLD bytes (the bottom layers of a departure)
are staged and copied twice.  `check()` re-verifies every write against every
read interval by interval.

The reference only models a remap (remap_time, sim.cpp:452-483); the plan is
overlap_matrix (param_fabric.cpp:82-121) via ReshardPlan.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import _native as N
from . import device as dev
from ._native import check, lib
from .fabric import ROLE_NEW, ROLE_OLD, ROLE_REPLICA, SEGMENT_DTYPE
from .reshard import ReshardExecutor, ReshardPlan, RankBuffers

Range = Tuple[int, int]


def prefix_bytes(segs: np.ndarray, g) -> np.ndarray:
    """Packed bytes of a segment map that lie below global positions g."""
    g = np.atleast_1d(np.asarray(g, dtype=np.int64))
    if len(segs) == 0:
        return np.zeros(len(g), dtype=np.int64)
    lo = segs["global_lo"].astype(np.int64)[None, :]
    ln = segs["length"].astype(np.int64)[None, :]
    return np.clip(g[:, None] - lo, 0, ln).sum(axis=1)


def clip_descs(descs: np.ndarray, lo: int, hi: int, shift: int = 0) -> np.ndarray:
    """Copy descriptors restricted to destinations in [lo, hi); dst_off moved
    by -lo + shift (shift = 0 and lo = 0 keep NEW's own offsets)."""
    d0 = descs["dst_off"].astype(np.int64)
    d1 = d0 + descs["bytes"].astype(np.int64)
    a, b = np.maximum(d0, lo), np.minimum(d1, hi)
    sel = b > a
    out = descs[sel].copy()
    out["src_off"] = out["src_off"] + (a[sel] - d0[sel])
    out["dst_off"] = a[sel] - lo + shift
    out["bytes"] = b[sel] - a[sel]
    return out


def clip_segments(segs: np.ndarray, lo: int, hi: int, pad: int) -> np.ndarray:
    """A segment map restricted to packed offsets [lo, hi), re-based to start
    at `pad` (a leading pad segment keeps the map packed from 0; nothing is
    ever landed there)."""
    a = segs["local_off"].astype(np.int64)
    b = a + segs["length"].astype(np.int64)
    x, y = np.maximum(a, lo), np.minimum(b, hi)
    sel = y > x
    if not sel.any():
        return np.zeros(0, dtype=SEGMENT_DTYPE)
    out = np.zeros(int(sel.sum()) + (1 if pad else 0), dtype=SEGMENT_DTYPE)
    j = 0
    if pad:
        first_g = int(segs["global_lo"][sel][0] + (x[sel][0] - a[sel][0]))
        out[0] = (first_g - pad, pad, 0)
        j = 1
    out["global_lo"][j:] = segs["global_lo"][sel] + (x[sel] - a[sel])
    out["length"][j:] = y[sel] - x[sel]
    out["local_off"][j:] = x[sel] - lo + pad
    return out


class InPlaceSchedule:
    """Phases, per-rank write ranges (direct / staged) and the read ranges
    they must avoid; identical on every rank.  Built by the C++ planner
    (elaskit::b200::inplace_schedule via ew_inplace_schedule, which also runs
    the hazard check); `check()` re-runs that check here."""

    def __init__(self, rp: ReshardPlan, stage_bytes: int = 1 << 30,
                 phase_bytes: int = 4 << 30, slack: int = 1):
        self.rp = rp
        self.total = int(sum(rp.layer_bytes))
        self.execs = list(rp.new_ranks)
        self.old_segs = {r: rp.src.segments(r) for r in rp.old_ranks}
        self.new_segs = {r: rp.dst.segments(r) for r in rp.new_ranks}
        self.holders = [r for r in rp.new_ranks if r in rp.old_ranks and r not in rp.failed]
        h = C.c_void_p()
        check(lib.ew_inplace_schedule(N.i64_array(rp.layer_bytes), len(rp.layer_bytes),
                                      rp.src.handle, rp.dst.handle, N.int_array(rp.failed),
                                      len(rp.failed), int(stage_bytes), int(phase_bytes),
                                      int(slack), C.byref(h)))
        try:
            desc, sl, ring = C.c_int(), C.c_int(), C.c_int()
            n, alloc = C.c_int64(), C.c_int64()
            check(lib.ew_inplace_info(h, C.byref(desc), C.byref(sl), C.byref(ring), C.byref(n),
                                      C.byref(alloc)))
            self.descending, self.slack, self.ring = bool(desc.value), sl.value, ring.value
            self.stage_alloc = alloc.value
            ph = np.zeros(2 * max(1, n.value), dtype=np.int64)
            check(lib.ew_inplace_phases(h, ph.ctypes.data_as(C.POINTER(C.c_int64))))
            self.phases: List[Range] = [(int(a), int(b)) for a, b in ph[:2 * n.value].reshape(-1, 2)]
            self.cuts: Dict[int, List[Range]] = {}
            self.direct: Dict[int, List[Range]] = {}
            self.staged: Dict[int, List[Range]] = {}
            for r in self.execs:
                arr = [np.zeros(2 * max(1, n.value), dtype=np.int64) for _ in range(3)]
                check(lib.ew_inplace_ranges(h, r, *[x.ctypes.data_as(C.POINTER(C.c_int64))
                                                    for x in arr]))
                for dst, x in zip((self.cuts, self.direct, self.staged), arr):
                    dst[r] = [(int(a), int(b)) for a, b in x[:2 * n.value].reshape(-1, 2)]
        finally:
            lib.ew_inplace_free(h)
        self.staged_bytes = {r: sum(b - a for a, b in self.staged[r]) for r in self.execs}

    # ---------------------------------------------------------------- checks
    def check(self) -> None:
        """Every write against every read it could race with:
        gather_j's direct writes vs the reads of phases >= j - slack;
        flush_j's writes vs the reads of phases > j (on the same rank's OLD)."""
        n = len(self.phases)
        for r in self.execs:
            if r not in self.holders:
                continue
            o = self.old_segs[r]
            reads = [tuple(int(x) for x in prefix_bytes(o, list(p))) for p in self.phases]
            for j in range(n):
                for what, (lo, hi), first in (("direct", self.direct[r][j], j - self.slack),
                                              ("staged", self.staged[r][j], j + 1)):
                    if hi <= lo:
                        continue
                    for k in range(max(0, first), n):
                        a, b = reads[k]
                        if a < b and a < hi and lo < b:
                            raise AssertionError(
                                f"rank {r}: phase {j} {what} write [{lo},{hi}) overlaps OLD "
                                f"bytes [{a},{b}) phase {k} reads")

    # ------------------------------------------------------------ programs
    @staticmethod
    def pad(k: int) -> int:
        return k % 16  # staging keeps NEW's alignment mod 16 (bulk stores)

    def direct_descs(self, rank: int, j: int, descs: np.ndarray) -> np.ndarray:
        lo, hi = self.direct[rank][j]
        return clip_descs(descs, lo, hi, lo)

    def staged_descs(self, rank: int, j: int, descs: np.ndarray) -> np.ndarray:
        lo, hi = self.staged[rank][j]
        return clip_descs(descs, lo, hi, self.pad(lo))

    def staged_segments(self, rank: int, j: int) -> np.ndarray:
        lo, hi = self.staged[rank][j]
        return clip_segments(self.new_segs[rank], lo, hi, self.pad(lo))


class StagedInPlaceReshard:
    """One rank's executor of an InPlaceSchedule (one process per GPU): a
    binding of the C++ elaskit::b200::InPlaceExecutor (ew_inplace_exec),
    which maps the peers, builds every phase's verified gathers and flush
    and enqueues the phases behind device-side barriers.

    Buffers: `buf` (OLD on entry, NEW on exit; max(|OLD|, |NEW|) bytes), the
    ring replica when this rank holds a departed rank's replica, and
    `schedule.ring` staging buffers of `schedule.stage_alloc` bytes (owned by
    the executor)."""

    def __init__(self, rp: ReshardPlan, rank: int, stage_bytes: int = 1 << 30,
                 block_bytes: int = dev.DEFAULT_BLOCK_BYTES,
                 phase_bytes: Optional[int] = None, slack: int = 1, gather_streams: int = 2,
                 flush_ctas: int = 64, barrier_timeout_s: float = 30.0):
        # defaults from the sweeps (profiles/r01_config_d_inplace_sweep_70gb.log,
        # profiles/r01_inplace_sweep_7b_4gpu.log): slack 1, two gather streams
        # and ~28 phases — smaller phases stage less of the bottom layers,
        # each phase costs a launch tail (config D 70 GB: 4 GB phases 66.9 ms
        # vs 1-2 GB 69-85 ms; 7B per GPU: 0.5 GB 11.7 ms vs 2 GB 12.9 ms)
        if phase_bytes is None:
            biggest = max(rp.dst.shard_bytes(r) for r in rp.new_ranks)
            phase_bytes = min(8 << 30, max(256 << 20, biggest // 28))
        self.rp = rp
        self.rank = rank
        self.block_bytes = block_bytes
        self.stage_bytes, self.phase_bytes, self.slack = stage_bytes, phase_bytes, slack
        self.gather_streams, self.flush_ctas = gather_streams, flush_ctas
        self.barrier_timeout_s = barrier_timeout_s
        self.sched = InPlaceSchedule(rp, stage_bytes, phase_bytes, slack)
        self.n_old = rp.src.shard_bytes(rank) if rank in rp.old_ranks else 0
        self.n_new = rp.dst.shard_bytes(rank) if rank in rp.new_ranks else 0
        self._h: Optional[C.c_void_p] = None
        self.buf: Optional[torch.Tensor] = None

    def allocate(self) -> RankBuffers:
        """OLD and NEW alias one allocation; staging is allocated at bind()."""
        rp, r = self.rp, self.rank
        rep_of = rp.replica_of(r)
        replica = (dev.empty_bytes(rp.src.shard_bytes(rep_of))
                   if rep_of is not None and rep_of in rp.failed else None)
        n = max(self.n_old, self.n_new)
        self.buf = dev.empty_bytes(n) if n else None
        old = self.buf[:self.n_old] if self.n_old else None
        new = self.buf[:self.n_new] if self.n_new else None
        return RankBuffers(old, replica, new)

    def bind(self, bufs: RankBuffers, group=None, survivors_group=None) -> None:
        """Collective over `group` (old and new members): map the peers and
        build the programs (C++).  `survivors_group` is accepted for API
        compatibility; the executor's barrier spans the NEW members."""
        from .rendezvous import Channel
        ch = Channel.from_group(group, "inplace")
        rp = self.rp
        buf = self.buf if self.buf is not None else (bufs.old if bufs.old is not None else bufs.new)
        h = C.c_void_p()
        check(lib.ew_inplace_exec_create(
            ch.handle, N.i64_array(rp.layer_bytes), len(rp.layer_bytes),
            N.int_array(rp.old_ranks), len(rp.old_ranks), N.int_array(rp.new_ranks),
            len(rp.new_ranks), C.c_void_p(buf.data_ptr() if buf is not None else None),
            C.c_void_p(bufs.replica.data_ptr() if bufs.replica is not None else None),
            int(self.stage_bytes), int(self.phase_bytes), int(self.slack),
            int(self.gather_streams), int(self.flush_ctas), int(self.block_bytes),
            float(self.barrier_timeout_s), C.byref(h)))
        self._h = h
        self._channel = ch  # the executor keeps a reference to it
        n, alloc = C.c_int64(), C.c_int64()
        check(lib.ew_inplace_exec_info(h, C.byref(n), C.byref(alloc)))
        if n.value != len(self.sched.phases):
            raise RuntimeError("C++ and Python in-place schedules disagree")

    def launch(self, block_sums: Optional[torch.Tensor], stream=None) -> None:
        """Enqueue the whole reshard on `stream` (gathers alternate over the
        executor's gather streams, barriers and flushes on their own, all
        joined back).  The caller zeroes block_sums and all-reduces them."""
        if self._h is None:
            raise RuntimeError("launch before bind")
        check(lib.ew_inplace_exec_launch(self._h, dev._ptr(block_sums), dev._stream(stream)))

    def timed_out(self) -> bool:
        t = C.c_int()
        if self._h is not None:
            check(lib.ew_inplace_exec_timed_out(self._h, C.byref(t)))
        return bool(t.value)

    def check(self) -> None:
        """Raise if a phase barrier timed out (call after the launch's stream
        completed).  The gated copies then stopped writing at that phase:
        NEW is incomplete, but every OLD byte not yet read is intact."""
        if self.timed_out():
            raise RuntimeError("in-place reshard aborted: a phase barrier timed out (a peer "
                               "did not arrive); later gathers and flushes were vetoed")

    def close(self) -> None:
        if self._h is not None and self._h.value and lib is not None:
            lib.ew_inplace_exec_free(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def emulate_inplace_on_one_gpu(rp: ReshardPlan, seed: int, stage_bytes: int, phase_bytes: int,
                               slack: int, block_sums: Optional[torch.Tensor],
                               block_bytes: int = dev.DEFAULT_BLOCK_BYTES):
    """Every rank's in-place programs on the current GPU (one buffer per rank,
    OLD on entry, NEW on exit), phase by phase in the adversarial order the
    multi-GPU executor allows: the direct ranges of the run-ahead phases
    j+1 .. j+slack are poisoned before phase j reads, the flush follows the
    phase (the barrier is the stream order).  Returns (NEW views, expected)."""
    sc = InPlaceSchedule(rp, stage_bytes, phase_bytes, slack)
    ranks = sorted(set(rp.old_ranks) | set(rp.new_ranks))
    bufs, reps = {}, {}
    for r in ranks:
        n_old = rp.src.shard_bytes(r) if r in rp.old_ranks else 0
        n_new = rp.dst.shard_bytes(r) if r in rp.new_ranks else 0
        bufs[r] = dev.empty_bytes(max(n_old, n_new, 1))
        bufs[r].fill_(0xA5)
        if n_old and r not in rp.failed:
            dev.fill_synthetic(dev.ShardMap(rp.src.segments(r), block_bytes), bufs[r], seed)
        rep = rp.replica_of(r)
        if rep is not None and rep in rp.failed and r not in rp.failed:
            reps[r] = dev.empty_bytes(rp.src.shard_bytes(rep))
            dev.fill_synthetic(dev.ShardMap(rp.src.segments(rep), block_bytes), reps[r], seed)
    staging = {r: [dev.empty_bytes(max(16, sc.stage_alloc)) for _ in range(sc.ring)]
               for r in rp.new_ranks}
    table = {(ROLE_OLD, r): bufs[r].data_ptr() for r in ranks}
    table.update({(ROLE_REPLICA, r): t.data_ptr() for r, t in reps.items()})
    n_table = max(ranks) + 1
    progs = {}
    for r in rp.new_ranks:
        descs = rp.copies(r, push=False)
        full = dev.ShardMap(sc.new_segs[r], block_bytes) if block_sums is not None else None
        t_new = dict(table)
        t_new[(ROLE_NEW, r)] = bufs[r].data_ptr()
        for j in range(len(sc.phases)):
            d = sc.direct_descs(r, j, descs)
            direct = dev.CopyProgram.from_descs(d, t_new, n_table, r, full) if len(d) else None
            staged = flush = None
            lo, hi = sc.staged[r][j]
            if hi > lo:
                st = staging[r][j % sc.ring]
                t = dict(table)
                t[(ROLE_NEW, r)] = st.data_ptr()
                staged = dev.CopyProgram.from_descs(
                    sc.staged_descs(r, j, descs), t, n_table, r,
                    dev.ShardMap(sc.staged_segments(r, j), block_bytes)
                    if block_sums is not None else None)
                flush = dev.CopyProgram.from_pointers([st.data_ptr() + sc.pad(lo)],
                                                      [bufs[r].data_ptr() + lo], [hi - lo],
                                                      [False])
            progs[(r, j)] = (direct, staged, flush)
    n = len(sc.phases)
    for j in range(n):
        for r in rp.new_ranks:
            for jj in range(j + 1, min(n, j + sc.slack + 1)):
                lo, hi = sc.direct[r][jj]
                if hi > lo:
                    bufs[r][lo:hi].fill_(0xEE)
        for r in rp.new_ranks:
            direct, staged, _ = progs[(r, j)]
            for p in (staged, direct):
                if p is not None:
                    p.launch(block_sums=block_sums)
        for r in rp.new_ranks:
            flush = progs[(r, j)][2]
            if flush is not None:
                flush.launch(64, 0)
    torch.cuda.synchronize()
    got, expected = {}, {}
    for r in rp.new_ranks:
        n_new = rp.dst.shard_bytes(r)
        got[r] = bufs[r][:n_new]
        e = dev.empty_bytes(n_new)
        dev.fill_synthetic(dev.ShardMap(rp.dst.segments(r), block_bytes), e, seed)
        expected[r] = e[:n_new]
    return got, expected, sc
