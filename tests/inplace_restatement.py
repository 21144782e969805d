"""CPU restatement of the staged in-place reshard schedule (test
infrastructure only): the same phase/cut/split rules as the product's C++
(paper_2510_00606_b200/csrc/host/inplace.cpp, elaskit::b200::inplace_schedule)
written independently in numpy, so tests/test_inplace.py can require that
both produce identical schedules."""
from typing import Dict, List, Tuple

import numpy as np

from paper_2510_00606_b200.inplace import prefix_bytes
from paper_2510_00606_b200.reshard import ReshardPlan

Range = Tuple[int, int]


class InPlaceRestatement:
    """Phases, per-rank write ranges (direct / staged) and the read ranges
    they must avoid; identical on every rank (pure function of the plan)."""

    def __init__(self, rp: ReshardPlan, stage_bytes: int = 1 << 30,
                 phase_bytes: int = 2 << 30, slack: int = 2):
        self.rp = rp
        self.stage_bytes = int(stage_bytes)
        self.phase_bytes = int(phase_bytes)
        self.slack = int(slack)
        self.ring = self.slack + 2           # staging buffers in rotation
        self.total = int(sum(rp.layer_bytes))
        self.execs = list(rp.new_ranks)
        self.old_segs = {r: rp.src.segments(r) for r in rp.old_ranks}
        self.new_segs = {r: rp.dst.segments(r) for r in rp.new_ranks}
        # ranks whose OLD is read in place (a departed rank's is not: its
        # bytes come from the ring replica)
        self.holders = [r for r in rp.new_ranks if r in rp.old_ranks and r not in rp.failed]
        grow = all(rp.dst.shard_bytes(r) >= rp.src.shard_bytes(r) for r in self.holders)
        shrink = all(rp.dst.shard_bytes(r) <= rp.src.shard_bytes(r) for r in self.holders)
        if not (grow or shrink):
            raise ValueError("in-place staging needs every retained shard to grow "
                             "(departures) or every one to shrink (joins)")
        self.descending = grow

        # candidate boundaries: layer boundaries plus points inside each layer
        # spaced at ~ a quarter phase of one rank's share; keep the safe ones
        n_new = max(1, len(rp.new_ranks))
        step = max(4096, min(self.phase_bytes, self.stage_bytes) * n_new // 4)
        cands, off = [], 0
        for sz in rp.layer_bytes:
            cands.extend(range(off, off + sz, step))
            off += sz
        c = np.unique(np.asarray(cands, dtype=np.int64))
        c = c[(c > 0) & (c < self.total)]
        ok = np.ones(len(c), dtype=bool)
        for r in self.holders:
            d = prefix_bytes(self.new_segs[r], c) - prefix_bytes(self.old_segs[r], c)
            ok &= (d >= 0) if self.descending else (d <= 0)
        safe = np.concatenate([[0], c[ok], [self.total]]).astype(np.int64)
        # processing order over the safe boundaries
        order = safe[::-1] if self.descending else safe
        newp = {r: prefix_bytes(self.new_segs[r], order) for r in self.execs}
        oldp = {r: prefix_bytes(self.old_segs[r], order) for r in self.holders}

        # greedy phases: grow while every rank's phase share fits phase_bytes
        # and its staged part fits stage_bytes
        bounds = [0]                   # indices into `order`
        self.phases: List[Range] = []  # (glo, ghi), processing order
        while bounds[-1] < len(order) - 1:
            a = bounds[-1]
            b = a + 1
            while b + 1 < len(order) and self._fits(a, b + 1, bounds, newp, oldp):
                b += 1
            bounds.append(b)
            ga, gb = int(order[a]), int(order[b])
            self.phases.append((min(ga, gb), max(ga, gb)))
        n = len(self.phases)
        # per-rank NEW cut of each phase and the direct / staged split
        self.cuts: Dict[int, List[Range]] = {}
        self.staged: Dict[int, List[Range]] = {}
        self.direct: Dict[int, List[Range]] = {}
        for r in self.execs:
            k = prefix_bytes(self.new_segs[r], [x for p in self.phases for x in p]).reshape(-1, 2)
            self.cuts[r] = [(int(a), int(b)) for a, b in k]
            self.staged[r], self.direct[r] = [], []
            for j in range(n):
                st, di = self._split(r, j)
                self.staged[r].append(st)
                self.direct[r].append(di)
        biggest = max((b - a for r in self.execs for a, b in self.staged[r]), default=0)
        self.stage_alloc = ((biggest + 15 + 255) // 256) * 256 if biggest else 0
        self.staged_bytes = {r: sum(b - a for a, b in self.staged[r]) for r in self.execs}
        self.check()

    # -------------------------------------------------------------- geometry
    def _threshold(self, r: int, j: int, gbounds=None) -> int:
        """Packed OLD offset on rank r separating what gather_j may write
        directly from what it must stage: the reads of phases j-s .. j (and
        any later) lie below it (departures) / above it (joins)."""
        k = j - self.slack
        if self.descending:
            if k < 0:
                return int(self.rp.src.shard_bytes(r))
            ghi = self.phases[k][1] if gbounds is None else gbounds[k][1]
            return int(prefix_bytes(self.old_segs[r], [ghi])[0])
        if k < 0:
            return 0
        glo = self.phases[k][0] if gbounds is None else gbounds[k][0]
        return int(prefix_bytes(self.old_segs[r], [glo])[0])

    def _split(self, r: int, j: int) -> Tuple[Range, Range]:
        k_lo, k_hi = self.cuts[r][j]
        if r not in self.holders:          # nobody reads this rank's buffer
            return (k_lo, k_lo), (k_lo, k_hi)
        t = self._threshold(r, j)
        if self.descending:
            m = min(max(t, k_lo), k_hi)
            return (k_lo, m), (m, k_hi)
        m = max(min(t, k_hi), k_lo)
        return (m, k_hi), (k_lo, m)

    def _fits(self, a: int, b: int, bounds, newp, oldp) -> bool:
        j = len(bounds) - 1            # index of the phase being grown
        for r in self.execs:
            lo, hi = sorted((int(newp[r][a]), int(newp[r][b])))
            if hi - lo > self.phase_bytes:
                return False
            if r in self.holders:
                k = j - self.slack
                if self.descending:
                    t = int(self.rp.src.shard_bytes(r)) if k < 0 else int(oldp[r][bounds[k]])
                    staged = max(0, min(hi, t) - lo)
                else:
                    t = 0 if k < 0 else int(oldp[r][bounds[k]])
                    staged = max(0, hi - max(lo, t))
                if staged > self.stage_bytes:
                    return False
        return True

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
