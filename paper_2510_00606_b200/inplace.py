"""Staged in-place reshard for ZeRO state that fills HBM.

The plain executor keeps a rank's OLD shard, the ring replica it holds and
the NEW shard side by side: about 3.1 S of HBM for a shard of S bytes, so
a 180 GB B200 reshards at most S ~ 55 GB that way.  Here OLD and NEW share
one allocation of max(|OLD|, |NEW|) bytes and the move is cut into phases
over the global byte space, plus two staging buffers of one phase each:

  phase i (global range P_i):
    gather  every rank pulls the NEW bytes it owns in P_i — from peers' OLD,
            ring replicas or its own OLD — into staging[i % 2], checksumming
            what lands (verification on arrival, kernel (a)'s spec labelled by
            the global position the byte has in NEW);
    barrier stream-ordered cross-GPU barrier: every rank has finished reading
            P_i's OLD bytes;
    flush   staging[i % 2] -> the rank's NEW range of P_i (one local copy,
            on a second stream, overlapping the next phase's gather).

Why it is safe.  A rank's packed offsets are monotone in the global
position: for a boundary G let old(G), new(G) be the packed bytes it holds
below G in OLD and NEW.  When shards grow (a departure) the phases run from
the top of the global space down and every boundary satisfies
new(G) >= old(G) on every surviving rank: then phase i's flush writes
[new(G_i), new(G_i+1)) while everything still to be read lies below
old(G_i) <= new(G_i).  When shards shrink (a join) the phases run upwards
with new(G) <= old(G).  Boundaries are chosen only where that holds for
every rank (layer boundaries always qualify for N -> N-1; cut points inside
a layer are tested), phases are grown greedily up to the staging size, and
`check()` re-verifies the no-overlap property interval by interval.

The reference only models a remap (remap_time, sim.cpp:452-483); the plan
itself is overlap_matrix (param_fabric.cpp:82-121) via ReshardPlan.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import device as dev
from .fabric import ROLE_NEW, ROLE_OLD, ROLE_REPLICA, SEGMENT_DTYPE
from .reshard import ReshardExecutor, ReshardPlan, RankBuffers


def prefix_bytes(segs: np.ndarray, g) -> np.ndarray:
    """Packed bytes of a segment map that lie below global positions g."""
    g = np.atleast_1d(np.asarray(g, dtype=np.int64))
    if len(segs) == 0:
        return np.zeros(len(g), dtype=np.int64)
    lo = segs["global_lo"].astype(np.int64)[None, :]
    ln = segs["length"].astype(np.int64)[None, :]
    return np.clip(g[:, None] - lo, 0, ln).sum(axis=1)


class InPlaceSchedule:
    """Phase boundaries and per-rank packed cuts of one staged in-place
    reshard; identical on every rank (pure function of the plan)."""

    def __init__(self, rp: ReshardPlan, stage_bytes: int = 2 << 30):
        self.rp = rp
        self.stage_bytes = int(stage_bytes)
        self.total = int(sum(rp.layer_bytes))
        self.execs = [r for r in rp.new_ranks]
        self.old_segs = {r: rp.src.segments(r) for r in rp.old_ranks}
        self.new_segs = {r: rp.dst.segments(r) for r in rp.new_ranks}
        both = [r for r in rp.new_ranks if r in rp.old_ranks and r not in rp.failed]
        grow = all(rp.dst.shard_bytes(r) >= rp.src.shard_bytes(r) for r in both)
        shrink = all(rp.dst.shard_bytes(r) <= rp.src.shard_bytes(r) for r in both)
        if not (grow or shrink):
            raise ValueError("in-place staging needs every retained shard to grow "
                             "(departures) or every one to shrink (joins)")
        self.descending = grow

        # candidate boundaries: layer boundaries plus points inside each layer
        # spaced so that a rank's share between them is ~ a quarter stage
        n_new = max(1, len(rp.new_ranks))
        step = max(4096, self.stage_bytes * n_new // 4)
        cands = []
        off = 0
        for sz in rp.layer_bytes:
            cands.extend(range(off, off + sz, step))
            off += sz
        c = np.unique(np.asarray(cands[1:] + [self.total], dtype=np.int64))
        c = c[(c > 0) & (c < self.total)]
        ok = np.ones(len(c), dtype=bool)
        for r in both:
            d = prefix_bytes(self.new_segs[r], c) - prefix_bytes(self.old_segs[r], c)
            ok &= (d >= 0) if self.descending else (d <= 0)
        safe = np.concatenate([[0], c[ok], [self.total]])
        newpos = {r: prefix_bytes(self.new_segs[r], safe) for r in self.execs}

        # greedy phases over the safe boundaries, largest that fits the stage
        def phase_bytes(i, j):
            return max((int(abs(newpos[r][j] - newpos[r][i])) for r in self.execs), default=0)

        bounds = []  # indices into `safe`, in processing order
        if self.descending:
            hi = len(safe) - 1
            bounds.append(hi)
            while hi > 0:
                lo = hi - 1
                while lo > 0 and phase_bytes(lo - 1, hi) <= self.stage_bytes:
                    lo -= 1
                bounds.append(lo)
                hi = lo
        else:
            lo = 0
            bounds.append(lo)
            last = len(safe) - 1
            while lo < last:
                hi = lo + 1
                while hi < last and phase_bytes(lo, hi + 1) <= self.stage_bytes:
                    hi += 1
                bounds.append(hi)
                lo = hi
        g = [int(safe[b]) for b in bounds]
        # phases as (glo, ghi), in processing order
        self.phases: List[Tuple[int, int]] = [
            (min(a, b), max(a, b)) for a, b in zip(g[:-1], g[1:])]
        self.cuts: Dict[int, List[Tuple[int, int]]] = {}
        for r in self.execs:
            k = prefix_bytes(self.new_segs[r], [x for p in self.phases for x in p]).reshape(-1, 2)
            self.cuts[r] = [(int(a), int(b)) for a, b in k]
        biggest = max((b - a for r in self.execs for a, b in self.cuts[r]), default=0)
        self.stage_alloc = ((biggest + 15 + 255) // 256) * 256
        self.check()

    # ---------------------------------------------------------------- checks
    def check(self) -> None:
        """Phase i's flush on rank r writes NEW[cut_i]; nothing a later phase
        reads from r's OLD (its own gathers or its peers') may lie there."""
        rp = self.rp
        for r in self.execs:
            if r not in rp.old_ranks or r in rp.failed:
                continue
            o = self.old_segs[r]
            for i, (k_lo, k_hi) in enumerate(self.cuts[r]):
                for glo, ghi in self.phases[i + 1:]:
                    a, b = prefix_bytes(o, [glo, ghi])
                    if a < b and a < k_hi and k_lo < b:
                        raise AssertionError(
                            f"rank {r}: phase {i} flush [{k_lo},{k_hi}) overlaps OLD bytes "
                            f"[{a},{b}) a later phase reads")

    # ------------------------------------------------------------ programs
    @staticmethod
    def _pad(k_lo: int) -> int:
        return k_lo % 16  # staging keeps NEW's alignment mod 16 (bulk stores)

    def phase_descs(self, rank: int, i: int, descs: Optional[np.ndarray] = None) -> np.ndarray:
        """This rank's pull descriptors restricted to phase i, re-targeted to
        the staging buffer (dst_off relative to the phase's NEW cut + pad)."""
        if descs is None:
            descs = self.rp.copies(rank, push=False)
        k_lo, k_hi = self.cuts[rank][i]
        pad = self._pad(k_lo)
        d0 = descs["dst_off"].astype(np.int64)
        d1 = d0 + descs["bytes"].astype(np.int64)
        lo = np.maximum(d0, k_lo)
        hi = np.minimum(d1, k_hi)
        sel = hi > lo
        out = descs[sel].copy()
        shift = lo[sel] - d0[sel]
        out["src_off"] = out["src_off"] + shift
        out["dst_off"] = lo[sel] - k_lo + pad
        out["bytes"] = hi[sel] - lo[sel]
        return out

    def phase_segments(self, rank: int, i: int) -> np.ndarray:
        """NEW's segment map clipped to phase i, as laid out in staging."""
        k_lo, k_hi = self.cuts[rank][i]
        pad = self._pad(k_lo)
        segs = self.new_segs[rank]
        a = segs["local_off"].astype(np.int64)
        b = a + segs["length"].astype(np.int64)
        lo, hi = np.maximum(a, k_lo), np.minimum(b, k_hi)
        sel = hi > lo
        if not sel.any():
            return np.zeros(0, dtype=SEGMENT_DTYPE)
        out = np.zeros(int(sel.sum()) + (1 if pad else 0), dtype=SEGMENT_DTYPE)
        j = 0
        if pad:
            first_g = int(segs["global_lo"][sel][0] + (lo[sel][0] - a[sel][0]))
            out[0] = (first_g - pad, pad, 0)  # nothing lands here
            j = 1
        out["global_lo"][j:] = segs["global_lo"][sel] + (lo[sel] - a[sel])
        out["length"][j:] = hi[sel] - lo[sel]
        out["local_off"][j:] = lo[sel] - k_lo + pad
        return out


class StagedInPlaceReshard:
    """One rank's executor of an InPlaceSchedule (one process per GPU).

    Buffers: `buf` (OLD on entry, NEW on exit; max(|OLD|, |NEW|) bytes), the
    ring replica when this rank holds a departed rank's replica, and two
    staging buffers of `schedule.stage_alloc` bytes."""

    def __init__(self, rp: ReshardPlan, rank: int, stage_bytes: int = 2 << 30,
                 block_bytes: int = dev.DEFAULT_BLOCK_BYTES):
        self.rp = rp
        self.rank = rank
        self.block_bytes = block_bytes
        self.sched = InPlaceSchedule(rp, stage_bytes)
        self.n_old = rp.src.shard_bytes(rank) if rank in rp.old_ranks else 0
        self.n_new = rp.dst.shard_bytes(rank) if rank in rp.new_ranks else 0
        self.gathers: List[dev.CopyProgram] = []
        self.flushes: List[dev.CopyProgram] = []
        self._base: Optional[ReshardExecutor] = None
        self.barrier: Optional[dev.PeerBarrier] = None

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
        """Collective over `group`: map peers' OLD/REPLICA (as in steady
        state), build every phase's verified gather and its flush.
        `survivors_group`: the process group of the NEW members (barrier)."""
        self._base = ReshardExecutor(self.rp, self.rank, push=False)
        self._base.premap(bufs, group)
        if self.rank not in self.rp.new_ranks:
            return
        self.barrier = dev.PeerBarrier(survivors_group)
        sa = self.sched.stage_alloc
        self.staging = [dev.empty_bytes(sa), dev.empty_bytes(sa)]
        table = dict(self._base._table)
        if bufs.old is not None:
            table[(ROLE_OLD, self.rank)] = bufs.old.data_ptr()
        if bufs.replica is not None:
            table[(ROLE_REPLICA, self.rank)] = bufs.replica.data_ptr()
        import torch.distributed as dist
        world = dist.get_world_size(group)
        n_table = max(max(self.rp.old_ranks + self.rp.new_ranks) + 1, world)
        descs = self.rp.copies(self.rank, push=False)
        self.gathers, self.flushes = [], []
        for i in range(len(self.sched.phases)):
            st = self.staging[i % 2]
            t = dict(table)
            t[(ROLE_NEW, self.rank)] = st.data_ptr()
            pd = self.sched.phase_descs(self.rank, i, descs)
            vmap = dev.ShardMap(self.sched.phase_segments(self.rank, i), self.block_bytes)
            self.gathers.append(dev.CopyProgram.from_descs(pd, t, n_table, self.rank, vmap))
            k_lo, k_hi = self.sched.cuts[self.rank][i]
            pad = InPlaceSchedule._pad(k_lo)
            self.flushes.append(dev.CopyProgram.from_pointers(
                [st.data_ptr() + pad], [self.buf.data_ptr() + k_lo], [k_hi - k_lo], [False]))
        self.flush_stream = torch.cuda.Stream()

    def launch(self, block_sums: torch.Tensor, stream=None, flush_ctas: int = 32) -> None:
        """Enqueue the whole reshard on `stream` (+ the flush stream).  The
        caller zeroes block_sums and all-reduces them afterwards."""
        if self.rank not in self.rp.new_ranks:
            return
        main = stream or torch.cuda.current_stream()
        fs = self.flush_stream
        fs.wait_stream(main)
        done: List[torch.cuda.Event] = []
        for i, (g, f) in enumerate(zip(self.gathers, self.flushes)):
            if i >= 2:
                main.wait_event(done[i - 2])      # staging[i % 2] flushed
            g.launch(stream=main, block_sums=block_sums)
            self.barrier.wait(stream=main)        # every rank read P_i's OLD bytes
            ev = torch.cuda.Event()
            ev.record(main)
            fs.wait_event(ev)
            f.launch(flush_ctas, 0, stream=fs)
            d = torch.cuda.Event()
            d.record(fs)
            done.append(d)
        if done:
            main.wait_event(done[-1])
            if len(done) > 1:
                main.wait_event(done[-2])

    def close(self) -> None:
        self.gathers, self.flushes = [], []
        if self.barrier is not None:
            self.barrier.close()
            self.barrier = None
        if self._base is not None:
            self._base.close()
            self._base = None
        self.staging = []
