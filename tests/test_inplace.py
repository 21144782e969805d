"""Staged in-place reshard (paper_2510_00606_b200/inplace.py), executed on the
host by a numpy byte mover with the real aliasing: each rank holds ONE
buffer that is its OLD shard on entry and its NEW shard on exit.  Every
phase runs all ranks' gathers (reading peers' buffers as the earlier
phases' flushes left them), then all flushes — the worst interleaving the
GPU's barrier + flush stream allow — so a flush that clobbered bytes a later
phase still reads shows up as a wrong target byte."""
import numpy as np
import pytest

from paper_2510_00606_b200 import configs
from paper_2510_00606_b200.fabric import ROLE_OLD, ROLE_REPLICA
from paper_2510_00606_b200.inplace import InPlaceSchedule, prefix_bytes
from paper_2510_00606_b200.reshard import ReshardPlan

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
    for i, (glo, ghi) in enumerate(sched.phases):
        staged = {}
        for r in rp.new_ranks:
            st = np.full(sched.stage_alloc, 0x5A, dtype=np.uint8)
            for c in sched.phase_descs(r, i):
                s = int(c["src_rank"])
                assert s not in rp.failed
                src = bufs[s] if int(c["src_role"]) == ROLE_OLD else reps[s]
                assert int(c["src_role"]) in (ROLE_OLD, ROLE_REPLICA)
                n, so, do = int(c["bytes"]), int(c["src_off"]), int(c["dst_off"])
                assert do + n <= sched.stage_alloc
                st[do:do + n] = src[so:so + n]
                landed[r] += n
            # the phase's segment map labels staging exactly like NEW
            segs = sched.phase_segments(r, i)
            k_lo, k_hi = sched.cuts[r][i]
            pad = k_lo % 16
            if k_hi > k_lo:
                want = oracle.fill_synthetic(segs, pad + k_hi - k_lo, SEED)
                assert np.array_equal(st[pad:pad + k_hi - k_lo], want[pad:]), (r, i)
            staged[r] = st
        for r in rp.new_ranks:
            k_lo, k_hi = sched.cuts[r][i]
            pad = k_lo % 16
            bufs[r][k_lo:k_hi] = staged[r][pad:pad + k_hi - k_lo]
    return bufs, landed


@pytest.mark.parametrize("name,cfg,old,new", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("stage_div", [3, 40])
def test_inplace_reconstructs_target_bytes(name, cfg, old, new, stage_div, oracle):
    small = _small(cfg)
    rp = ReshardPlan.build(small.layer_bytes, old, new)
    stage = max(256, max(rp.dst.shard_bytes(r) for r in rp.new_ranks) // stage_div)
    sched = InPlaceSchedule(rp, stage)
    assert sched.descending == (len(new) < len(old))
    # phases tile the global space, in processing order
    gl = sorted(sched.phases)
    assert gl[0][0] == 0 and gl[-1][1] == small.total_bytes
    assert all(a[1] == b[0] for a, b in zip(gl[:-1], gl[1:]))
    order = [p[0] for p in sched.phases]
    assert order == sorted(order, reverse=sched.descending)
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
    sched = InPlaceSchedule(rp, 2 << 30)
    holder = 2  # holds the departed r3's replica
    in_place = (max(rp.src.shard_bytes(holder), rp.dst.shard_bytes(holder))
                + rp.src.shard_bytes(3) + 2 * sched.stage_alloc)
    side_by_side = rp.src.shard_bytes(holder) + rp.src.shard_bytes(3) + rp.dst.shard_bytes(holder)
    assert in_place < 180e9 < side_by_side
    assert sched.stage_alloc <= (2 << 30) + 256
    # layer boundaries are always safe cut points for a departure
    for r in rp.new_ranks:
        off = np.cumsum([0] + list(rp.layer_bytes))
        d = prefix_bytes(rp.dst.segments(r), off) - prefix_bytes(rp.src.segments(r), off)
        assert (d >= 0).all()


def test_check_rejects_an_unsafe_schedule():
    small = _small(configs.llama2_7b())
    rp = ReshardPlan.build(small.layer_bytes, range(8), [0, 1, 2, 4, 5, 6, 7])
    sched = InPlaceSchedule(rp, 1 << 12)
    # process the same phases bottom-up: the first flush lands on OLD bytes
    # a later (higher) phase still reads
    sched.phases = sched.phases[::-1]
    for r in sched.cuts:
        sched.cuts[r] = sched.cuts[r][::-1]
    with pytest.raises(AssertionError):
        sched.check()
