"""Staged in-place reshard (paper_2510_00606_b200/inplace.py), executed on the
host by a numpy byte mover with the real aliasing: each rank holds ONE
buffer that is its OLD shard on entry and its NEW shard on exit.  Phases run
in the adversarial order the GPU's streams allow (run-ahead gathers' direct
writes land before a phase reads, flushes right after its barrier), so a
write that clobbered bytes some phase still reads shows up as a wrong target
byte; `check()` is the independent interval-level proof."""
import numpy as np
import pytest

from paper_2510_00606_b200 import configs
from paper_2510_00606_b200.fabric import ROLE_OLD, ROLE_REPLICA
from paper_2510_00606_b200.inplace import InPlaceSchedule, prefix_bytes
from paper_2510_00606_b200.reshard import ReshardPlan

from inplace_restatement import InPlaceRestatement

SEED = 7

CASES = [
    ("125M 4->3 drop r1", configs.gpt_125m(), [0, 1, 2, 3], [0, 2, 3]),
    ("7B 8->7 drop r0", configs.llama2_7b(), list(range(8)), [1, 2, 3, 4, 5, 6, 7]),
    ("7B 8->7 drop r3", configs.llama2_7b(), list(range(8)), [0, 1, 2, 4, 5, 6, 7]),
    ("7B 8->7 drop r7", configs.llama2_7b(), list(range(8)), [0, 1, 2, 3, 4, 5, 6]),
    ("7B per-tensor 8->7 drop r5", configs.llama2_7b_per_tensor(), list(range(8)),
     [0, 1, 2, 3, 4, 6, 7]),
    ("8B 8->6 drop r2,r5", configs.llama3_8b(), list(range(8)), [0, 1, 3, 4, 6, 7]),
    ("8B 6->8 rejoin", configs.llama3_8b(), [0, 1, 3, 4, 6, 7], list(range(8))),
    ("fill-HBM 4->3 drop r3", configs.fill_hbm(4), [0, 1, 2, 3], [0, 1, 2]),
    ("fill-HBM 2->1", configs.fill_hbm(2), [0, 1], [0]),
    ("3->5 scale-out", configs.gpt_125m(), [0, 1, 2], [0, 1, 2, 3, 4]),
]


def _small(cfg):
    return configs.scaled(cfg, 2e-5 if cfg.total_bytes > 10**10 else 1e-3)


def _simulate(rp, sched, oracle):
    """Adversarial order: before phase j's gathers read, the gathers of phases
    j+1 .. j+slack (which may run ahead) have already written their direct
    ranges — poisoned here, so any read they could clobber is caught."""
    bufs, reps = {}, {}
    for r in sorted(set(rp.old_ranks) | set(rp.new_ranks)):
        n_old = rp.src.shard_bytes(r) if r in rp.old_ranks else 0
        n_new = rp.dst.shard_bytes(r) if r in rp.new_ranks else 0
        b = np.full(max(n_old, n_new), 0xA5, dtype=np.uint8)
        if n_old and r not in rp.failed:
            b[:n_old] = oracle.fill_synthetic(rp.src.segments(r), n_old, SEED)
        bufs[r] = b
        rep = rp.replica_of(r)
        if rep is not None and rep in rp.failed and r not in rp.failed:
            reps[r] = oracle.fill_synthetic(rp.src.segments(rep), rp.src.shard_bytes(rep), SEED)
    landed = {r: 0 for r in rp.new_ranks}
    descs = {r: rp.copies(r, push=False) for r in rp.new_ranks}
    n = len(sched.phases)
    for j in range(n):
        for r in rp.new_ranks:
            for jj in range(j + 1, min(n, j + sched.slack + 1)):
                lo, hi = sched.direct[r][jj]
                bufs[r][lo:hi] = 0xEE
        staged = {}
        for r in rp.new_ranks:
            st = np.full(max(16, sched.stage_alloc), 0x5A, dtype=np.uint8)
            for part, target in ((sched.staged_descs(r, j, descs[r]), st),
                                 (sched.direct_descs(r, j, descs[r]), bufs[r])):
                for c in part:
                    s = int(c["src_rank"])
                    assert s not in rp.failed
                    assert int(c["src_role"]) in (ROLE_OLD, ROLE_REPLICA)
                    src = bufs[s] if int(c["src_role"]) == ROLE_OLD else reps[s]
                    nb, so, do = int(c["bytes"]), int(c["src_off"]), int(c["dst_off"])
                    assert do + nb <= len(target)
                    target[do:do + nb] = src[so:so + nb]
                    landed[r] += nb
            lo, hi = sched.staged[r][j]
            if hi > lo:
                # the staged segment map labels staging exactly like NEW
                pad = lo % 16
                want = oracle.fill_synthetic(sched.staged_segments(r, j), pad + hi - lo, SEED)
                assert np.array_equal(st[pad:pad + hi - lo], want[pad:]), (r, j)
            staged[r] = st
        for r in rp.new_ranks:  # barrier_j, then flush_j
            lo, hi = sched.staged[r][j]
            bufs[r][lo:hi] = staged[r][lo % 16:lo % 16 + hi - lo]
    return bufs, landed


@pytest.mark.parametrize("name,cfg,old,new", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("stage_div,slack", [(3, 0), (40, 2), (40, 0), (11, 5)])
def test_inplace_reconstructs_target_bytes(name, cfg, old, new, stage_div, slack, oracle):
    small = _small(cfg)
    rp = ReshardPlan.build(small.layer_bytes, old, new)
    stage = max(256, max(rp.dst.shard_bytes(r) for r in rp.new_ranks) // stage_div)
    sched = InPlaceSchedule(rp, stage, phase_bytes=2 * stage, slack=slack)
    assert sched.descending == (len(new) < len(old))
    # phases tile the global space, in processing order
    gl = sorted(sched.phases)
    assert gl[0][0] == 0 and gl[-1][1] == small.total_bytes
    assert all(a[1] == b[0] for a, b in zip(gl[:-1], gl[1:]))
    order = [p[0] for p in sched.phases]
    assert order == sorted(order, reverse=sched.descending)
    sched.check()
    # the C++ planner and the independent numpy restatement agree exactly
    ref = InPlaceRestatement(rp, stage, phase_bytes=2 * stage, slack=slack)
    assert (sched.descending, sched.slack, sched.ring, sched.stage_alloc) == \
        (ref.descending, ref.slack, ref.ring, ref.stage_alloc)
    assert sched.phases == ref.phases
    for r in rp.new_ranks:
        assert sched.cuts[r] == ref.cuts[r]
        assert sched.direct[r] == ref.direct[r]
        assert sched.staged[r] == ref.staged[r]
    bufs, landed = _simulate(rp, sched, oracle)
    for r in rp.new_ranks:
        n = rp.dst.shard_bytes(r)
        want = oracle.fill_synthetic(rp.dst.segments(r), n, SEED)
        assert np.array_equal(bufs[r][:n], want), (name, r)
        assert landed[r] == n, "every target byte gathered exactly once"


def test_inplace_fits_fill_hbm_where_side_by_side_does_not():
    # config D, 4 -> 3 at 74 GB per GPU: the holder needs NEW + replica +
    # two stages in place (2.33 S + 4 GB) vs OLD + replica + NEW (3.33 S)
    S = 74_000_000_000
    rp = ReshardPlan.build(configs.fill_hbm(4, S).layer_bytes, range(4), [0, 1, 2])
    sched = InPlaceSchedule(rp, 1 << 30)
    holder = 2  # holds the departed r3's replica
    in_place = (max(rp.src.shard_bytes(holder), rp.dst.shard_bytes(holder))
                + rp.src.shard_bytes(3) + sched.ring * sched.stage_alloc)
    side_by_side = rp.src.shard_bytes(holder) + rp.src.shard_bytes(3) + rp.dst.shard_bytes(holder)
    assert in_place < 180e9 < side_by_side
    # a phase is staged only up to the stage size, or one layer's share where
    # no safe cut exists inside the layer (the bottom layers)
    layer_share = max(rp.layer_bytes) // 3 + 1
    assert sched.stage_alloc <= max(1 << 30, layer_share) + 256
    # only the bottom layers' phases are staged (copied twice)
    assert sched.staged_bytes[holder] < 0.15 * rp.dst.shard_bytes(holder)
    # layer boundaries are always safe cut points for a departure
    for r in rp.new_ranks:
        off = np.cumsum([0] + list(rp.layer_bytes))
        d = prefix_bytes(rp.dst.segments(r), off) - prefix_bytes(rp.src.segments(r), off)
        assert (d >= 0).all()


def test_check_rejects_an_unsafe_schedule():
    small = _small(configs.llama2_7b())
    rp = ReshardPlan.build(small.layer_bytes, range(8), [0, 1, 2, 4, 5, 6, 7])
    sched = InPlaceSchedule(rp, 1 << 12, phase_bytes=1 << 13, slack=1)
    assert sum(sched.staged_bytes.values()) > 0
    # write everything directly: the bottom phases then land on OLD bytes
    # that the same or a run-ahead phase still reads
    for r in sched.execs:
        sched.direct[r] = list(sched.cuts[r])
        sched.staged[r] = [(a, a) for a, _ in sched.cuts[r]]
    with pytest.raises(AssertionError):
        sched.check()


def test_schedule_errors():
    from paper_2510_00606_b200._native import CoverageMismatch
    small = _small(configs.gpt_125m())
    rp = ReshardPlan.build(small.layer_bytes, [0, 1, 2, 3], [0, 2, 3])
    with pytest.raises(ValueError):
        InPlaceSchedule(rp, 0)
    sched = InPlaceSchedule(rp, 1 << 16, phase_bytes=1 << 17, slack=0)
    assert sched.ring == 2 and len(sched.phases) > 3
    # layer bytes that do not describe the layouts
    rp.layer_bytes = rp.layer_bytes[:-1]
    with pytest.raises(CoverageMismatch):
        InPlaceSchedule(rp, 1 << 16)
