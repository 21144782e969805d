"""Host planners of the B200 build vs the reference library (oracle/_ref) and
the C oracle: bit-identical plans, layouts, reshapes, folds and edits,
including the reference's exception behaviour."""
import hashlib
import json
import random

import numpy as np
import pytest

from paper_2510_00606_b200 import configs, fabric
from paper_2510_00606_b200._native import CoverageMismatch, MissingBackup, NoSurvivors


def rows_of(plan: fabric.TransferPlan) -> np.ndarray:
    e = plan.entries
    return np.stack([e["src_rank"], e["dst_rank"], e["lo"], e["hi"], e["medium"]], axis=1).astype(np.int64) \
        if len(e) else np.zeros((0, 5), dtype=np.int64)


def layout_dict(layout: fabric.PartitionLayout):
    return {r: layout.intervals(r) for r in layout.ranks}


# ------------------------------------------------------------------ golden ---

@pytest.fixture(scope="module")
def plan_golden(golden_dir):
    return json.loads((golden_dir / "plan_golden.json").read_text())


def test_config_plans_match_reference_golden(plan_golden):
    for case in plan_golden["cases"]:
        src = fabric.interleaved_layout(case["layer_bytes"], case["old"])
        dst = fabric.interleaved_layout(case["layer_bytes"], case["new"])
        ring = fabric.SnapshotRing(case["old"])
        plan = fabric.overlap_matrix(src, dst, case["failed"], ring)
        rows = rows_of(plan)
        assert len(rows) == case["n_entries"], case["name"]
        assert plan.total_bytes_moved == case["total_bytes_moved"], case["name"]
        assert hashlib.sha256(rows.tobytes()).hexdigest() == case["sha256"], case["name"]
        if "entries" in case:
            assert rows.tolist() == case["entries"]


def test_adjacent_failures_are_rejected(plan_golden):
    assert plan_golden["adjacent_failure_status"] == 2  # CoverageMismatch in the reference
    lb = configs.llama3_8b().layer_bytes
    src = fabric.interleaved_layout(lb, range(8))
    dst = fabric.interleaved_layout(lb, [0, 1, 4, 5, 6, 7])
    with pytest.raises(CoverageMismatch):
        fabric.overlap_matrix(src, dst, [2, 3], fabric.SnapshotRing(list(range(8))))


# --------------------------------------------------------------- vs reference ---

def test_interleaved_composition_matches_reference_shard_rule(reference, oracle):
    for cfg in (configs.gpt_125m(), configs.llama2_7b(), configs.llama3_8b()):
        for ranks in (list(range(cfg.dp)), [0, 1, 2, 4, 5, 6, 7][: cfg.dp - 1]):
            ours = layout_dict(fabric.interleaved_layout(cfg.layer_bytes, ranks))
            assert ours == reference.interleaved(cfg.layer_bytes, ranks)
            assert ours == oracle.interleaved(cfg.layer_bytes, ranks)


def test_worked_12_byte_scale_down_matches_reference(reference):
    # reference test_param_fabric.cpp:92-136
    src = fabric.contiguous_layout([0, 1, 2, 3], 12)
    dst = fabric.PartitionLayout.from_ranges({0: [(0, 4)], 1: [(4, 8)], 3: [(8, 12)]}, 12)
    plan = fabric.overlap_matrix(src, dst, [2], fabric.SnapshotRing([0, 1, 2, 3]))
    want, moved, _ = reference.overlap_matrix(layout_dict(src), layout_dict(dst), 12, [2],
                                              [0, 1, 2, 3])
    assert rows_of(plan).tolist() == want.tolist()
    assert plan.total_bytes_moved == moved == 4


def _random_layout(rng, ranks, total, max_pieces):
    cuts = sorted(set(rng.sample(range(1, total), min(total - 1, rng.randint(len(ranks) - 1, len(ranks) * max_pieces)))))
    bounds = [0] + cuts + [total]
    ranges = {r: [] for r in ranks}
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        ranges[rng.choice(ranks)].append((lo, hi))
    # merge adjacent pieces of the same rank? keep them: validate() allows adjacency
    return ranges


def test_random_layouts_match_reference_and_oracle(reference, oracle):
    rng = random.Random(13)
    for trial in range(400):
        n = rng.randint(2, 7)
        ranks = list(range(n))
        total = rng.randint(64, 5000)
        src_r = _random_layout(rng, ranks, total, 4)
        fail = set()
        if rng.random() < 0.6:
            fail.add(rng.randrange(n))
            if rng.random() < 0.3:
                fail.add(rng.randrange(n))
        surv = [r for r in ranks if r not in fail] or [0]
        if rng.random() < 0.2:
            surv = surv + [n + rng.randint(0, 2)]  # joiner
        dst_r = _random_layout(rng, sorted(set(surv)), total, 4)
        src = fabric.PartitionLayout.from_ranges(src_r, total)
        dst = fabric.PartitionLayout.from_ranges(dst_r, total)
        ring = fabric.SnapshotRing(ranks)
        st = reference.overlap_matrix(src_r, dst_r, total, sorted(fail), ranks, return_status=True)
        if isinstance(st, int):
            with pytest.raises(CoverageMismatch):
                fabric.overlap_matrix(src, dst, fail, ring)
            continue
        want, moved, _ = st
        plan = fabric.overlap_matrix(src, dst, fail, ring)
        assert rows_of(plan).tolist() == want.tolist(), trial
        assert plan.total_bytes_moved == moved
        assert oracle.overlap(src_r, dst_r, fail, ranks).tolist() == want.tolist()
        assert plan.to_json() == json.loads(reference.plan_to_json(src_r, dst_r, total, sorted(fail), ranks))


def test_validation_errors_match_reference(reference):
    bad_cases = [
        ({0: [(0, 5)], 1: [(4, 10)]}, {0: [(0, 10)]}, 10),   # overlap
        ({0: [(0, 4)], 1: [(5, 10)]}, {0: [(0, 10)]}, 10),   # gap
        ({0: [(5, 10), (0, 5)]}, {0: [(0, 10)]}, 10),        # unsorted
        ({0: [(0, 0), (0, 10)]}, {0: [(0, 10)]}, 10),        # empty interval
        ({0: [(0, 10)]}, {0: [(0, 12)]}, 10),                # coverage short
    ]
    for s, d, total in bad_cases:
        assert reference.overlap_matrix(s, d, total, return_status=True) == 2
        with pytest.raises(CoverageMismatch):
            fabric.overlap_matrix(fabric.PartitionLayout.from_ranges(s, total),
                                  fabric.PartitionLayout.from_ranges(d, total))
    # failed owner without a ring; target assigning bytes to a failed rank
    s, d = {0: [(0, 5)], 1: [(5, 10)]}, {0: [(0, 10)]}
    assert reference.overlap_matrix(s, d, 10, [1], None, return_status=True) == 2
    with pytest.raises(CoverageMismatch):
        fabric.overlap_matrix(fabric.PartitionLayout.from_ranges(s, 10),
                              fabric.PartitionLayout.from_ranges(d, 10), [1])
    with pytest.raises(CoverageMismatch):
        fabric.overlap_matrix(fabric.PartitionLayout.from_ranges(s, 10),
                              fabric.PartitionLayout.from_ranges(s, 10), [1], fabric.SnapshotRing([0, 1]))


def test_integrity_check_exhaustive_matches_reference(reference):
    for n in range(2, 7):
        layout = fabric.contiguous_layout(list(range(n)), 64)
        ring = fabric.SnapshotRing(list(range(n)))
        for a in range(n):
            for b in range(a, n):
                failed = {a, b}
                ours = fabric.integrity_check(ring, layout, failed)
                rec, missing = reference.integrity_check(list(range(n)), layout_dict(layout), 64,
                                                         sorted(failed))
                assert ours.recoverable == rec
                assert sorted(ours.missing) == missing


# ----------------------------------------------------------------- dataflow ---

def test_reshard_microbatches_fuzz_matches_reference(reference):
    rng = np.random.default_rng(3)
    for _ in range(3000):
        n = int(rng.integers(1, 13))
        mbs = int(rng.integers(1, 9))
        nmb = int(rng.integers(1, 17))
        surv = [s for s in range(n) if rng.integers(0, 4) != 0]
        if rng.integers(0, 5) == 0:
            surv.append(n + int(rng.integers(0, 3)))
        rng.shuffle(surv)
        st, slots, sizes = reference.reshard_microbatches([mbs] * n, nmb, surv)
        if st:
            with pytest.raises(NoSurvivors):
                fabric.reshard_microbatches([mbs] * n, nmb, surv)
            continue
        assert fabric.reshard_microbatches([mbs] * n, nmb, surv) == (slots, sizes)
        assert sum(sizes) == n * mbs and max(sizes) - min(sizes) <= 1


def test_config_e_reshape():
    # 8 slots x mbs 4 x 32 micro-batches = 1024 -> DP 5
    slots, sizes = fabric.reshard_microbatches([4] * 8, 32, [0, 2, 3, 5, 7])
    assert slots == [0, 2, 3, 5, 7] and sizes == [7, 7, 6, 6, 6]
    assert [32 * s for s in sizes] == [224, 224, 192, 192, 192]


def test_weighted_grad_average_bitwise_matches_reference(reference):
    rng = np.random.default_rng(5)
    for n, dim in ((1, 7), (5, 1000), (8, 333)):
        w = rng.random(n)
        g = rng.normal(size=(n, dim))
        assert np.array_equal(fabric.weighted_grad_average(w, g), reference.weighted_grad_average(w, g))


# --------------------------------------------------------------- communicator ---

def _random_groups(rng):
    world = rng.randint(2, 12)
    groups = []
    for g in range(rng.randint(1, 4)):
        members = rng.sample(range(world), rng.randint(1, world))
        groups.append((f"g{g}", members, rng.random() < 0.4))
    return world, groups


def test_plan_edit_fuzz_matches_reference(reference):
    rng = random.Random(7)
    for trial in range(600):
        world, groups = _random_groups(rng)
        pool = set()
        for _, members, ring in groups:
            g = fabric.CommGroup("x", members, ring)
            n = len(members)
            if ring:
                pool |= {tuple(sorted((members[i], members[(i + 1) % n]))) for i in range(n) if n > 1}
            else:
                pool |= {tuple(sorted((a, b))) for i, a in enumerate(members) for b in members[i + 1:]}
        pool = {l for l in pool if l[0] != l[1] and rng.random() < 0.9}
        kind = rng.choice([0, 2, 3])
        targets = rng.sample(range(world), rng.randint(1, min(2, world)))
        st, add, rem, touched = reference.plan_edit(groups, kind, targets, pool)
        cg = [fabric.CommGroup(i, m, r) for i, m, r in groups]
        if st:
            with pytest.raises(Exception):
                fabric.plan_edit(cg, kind, targets, pool)
            continue
        ours = fabric.plan_edit(cg, kind, targets, pool)
        assert ours.links_to_add == add, trial
        assert ours.links_to_remove == rem, trial
        assert ours.groups_touched == touched, trial


def test_plan_edit_worked_cases():
    # test_communicator.cpp:34-83
    mesh = fabric.CommGroup("g", list(range(8)))
    pool = {(a, b) for a in range(8) for b in range(a + 1, 8)}
    p = fabric.plan_edit([mesh], fabric.FAIL_STOP, [5], pool)
    assert len(p.links_to_remove) == 7 and not p.links_to_add
    ring = fabric.CommGroup("ring", [0, 1, 2, 3, 4], ring=True)
    pool = {(0, 1), (1, 2), (2, 3), (3, 4), (0, 4)}
    p = fabric.plan_edit([ring], fabric.FAIL_STOP, [2], pool)
    assert p.links_to_remove == {(1, 2), (2, 3)} and p.links_to_add == {(1, 3)}


# --------------------------------------------------------------- migration ---

def test_plan_zero_migration_matches_reference(reference):
    rng = random.Random(31)
    for trial in range(300):
        d = rng.choice([1, 2, 3, 4, 5, 7, 8])
        layers = [rng.randint(0, 3000) for _ in range(rng.randint(1, 6))]
        layer = rng.randrange(len(layers))
        interleaved = rng.random() < 0.5
        dst_d = d if rng.random() < 0.9 else d + 1
        st, want, want_tot = reference.plan_zero_migration(interleaved, d, layers, layer, dst_d)
        if st:
            with pytest.raises(fabric.MismatchedDpDegree):
                fabric.plan_zero_migration(interleaved, d, layers, layer, dst_d)
            continue
        rows, tot = fabric.plan_zero_migration(interleaved, d, layers, layer, dst_d)
        assert rows.tolist() == want.tolist(), trial
        assert tot.tolist() == want_tot.tolist()


def test_plan_layer_migration_matches_reference(reference):
    """plan_layer_migration (migration.cpp:9-61), both modes, incl. the
    micro-batch-boundary tie rule and InsufficientTargetMemory; doubles
    compared bit for bit."""
    from paper_2510_00606_b200._native import InsufficientTargetMemory, InvalidArgument
    rng = random.Random(41)
    for trial in range(2000):
        slot = rng.choice([0.0, 1e-3, 2.5e-3, rng.uniform(1e-4, 1e-2)])
        bw = rng.choice([1e9, 2.5e10, 7.0e11, rng.uniform(1e8, 1e12), 0.0])
        pb = rng.choice([0, rng.randint(1, 1 << 34)])
        if rng.random() < 0.2 and slot > 0 and bw > 0:
            pb = int(bw * slot * rng.randint(1, 8))  # arrival exactly on a boundary
        ctx = dict(param_bytes=pb, grad_bytes=rng.choice([0, rng.randint(1, 1 << 34)]),
                   link_bw_bytes_per_s=bw, microbatch_slot_s=slot,
                   num_microbatches=rng.randint(0, 64),
                   target_headroom_bytes=rng.randint(0, 1 << 36),
                   fixed_overhead_s=rng.choice([0.0, 0.012]))
        move = (rng.randint(0, 40), rng.randint(0, 7), rng.randint(0, 7))
        nb = rng.random() < 0.8
        st, want = reference.plan_layer_migration(*move, nb, ctx)
        if st:
            exc = {13: InsufficientTargetMemory, 1: InvalidArgument}[st]
            with pytest.raises(exc):
                fabric.plan_layer_migration(move, int(nb), **ctx)
            continue
        got = fabric.plan_layer_migration(move, int(nb), **ctx)
        assert got.mode == want["mode"] and got.shadow_microbatches == want["shadow_microbatches"]
        assert got.payback_bytes == want["payback_bytes"], trial
        assert [tuple(t) for t in got.transfers] == want["transfers"], trial
        assert (got.stall_s, got.total_time_s) == (want["stall_s"], want["total_time_s"]), trial


def _reassign_restated(old_slots, old_mbs, new_slots, new_mbs):
    """sim.cpp:694-715, restated: offsets of micro-batch 0 whose slot changes."""
    def slot_at(slots, mbs, off):
        lo = 0
        for s, m in zip(slots, mbs):
            if lo <= off < lo + m:
                return s
            lo += m
        return -1
    out = []
    for off in range(min(sum(old_mbs), sum(new_mbs))):
        a, b = slot_at(old_slots, old_mbs, off), slot_at(new_slots, new_mbs, off)
        if a != b and a >= 0 and b >= 0:
            out.append((off, a, b))
    return out


def test_sample_reassignments_match_restatement():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 9))
        mbs = int(rng.integers(1, 6))
        survivors = sorted({int(s) for s in rng.integers(0, n + 2, size=int(rng.integers(1, n + 2)))})
        slots, sizes = fabric.reshard_microbatches([mbs] * n, 4, survivors)
        got = fabric.sample_reassignments(list(range(n)), [mbs] * n, slots, sizes)
        assert got == _reassign_restated(list(range(n)), [mbs] * n, slots, sizes)
