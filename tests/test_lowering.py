"""The TransferPlan -> per-GPU copy-program lowering (elaskit/b200.hpp
reshard_copies), executed on the host by a numpy byte mover.  The CUDA
kernel executes exactly these descriptors (tests/test_gpu_reshard.py), so
this pins the N-rank logic — including 8-rank membership changes that the
GPU pool cannot host — on the CPU."""
import numpy as np
import pytest

from paper_2510_00606_b200 import configs, fabric
from paper_2510_00606_b200.fabric import ROLE_NEW, ROLE_OLD, ROLE_REPLICA
from paper_2510_00606_b200.reshard import ReshardPlan

SEED = 2024

CASES = [
    ("125M 4->3 drop r1", configs.gpt_125m(), [0, 1, 2, 3], [0, 2, 3]),
    ("7B 8->7 drop r0", configs.llama2_7b(), list(range(8)), [1, 2, 3, 4, 5, 6, 7]),
    ("7B 8->7 drop r3", configs.llama2_7b(), list(range(8)), [0, 1, 2, 4, 5, 6, 7]),
    ("7B 8->7 drop r7", configs.llama2_7b(), list(range(8)), [0, 1, 2, 3, 4, 5, 6]),
    ("7B per-tensor 8->7 drop r5", configs.llama2_7b_per_tensor(), list(range(8)),
     [0, 1, 2, 3, 4, 6, 7]),
    ("8B 8->6 drop r2,r5", configs.llama3_8b(), list(range(8)), [0, 1, 3, 4, 6, 7]),
    ("8B 6->8 rejoin", configs.llama3_8b(), [0, 1, 3, 4, 6, 7], list(range(8))),
    ("2->1", configs.gpt_125m(), [0, 1], [1]),
    ("3->5 scale-out", configs.gpt_125m(), [0, 1, 2], [0, 1, 2, 3, 4]),
]


def _host_execute(rp: ReshardPlan, oracle, push: bool):
    ranks = sorted(set(rp.old_ranks) | set(rp.new_ranks))
    bufs = {}
    for r in ranks:
        if r in rp.old_ranks and r not in rp.failed:
            bufs[(ROLE_OLD, r)] = oracle.fill_synthetic(rp.src.segments(r), rp.src.shard_bytes(r), SEED)
        rep = rp.replica_of(r)
        if rep is not None and rep in rp.failed and r not in rp.failed:
            bufs[(ROLE_REPLICA, r)] = oracle.fill_synthetic(rp.src.segments(rep),
                                                            rp.src.shard_bytes(rep), SEED)
        if r in rp.new_ranks:
            bufs[(ROLE_NEW, r)] = np.full(rp.dst.shard_bytes(r), 0xA5, dtype=np.uint8)
    written = {r: np.zeros(rp.dst.shard_bytes(r), dtype=np.int32) for r in rp.new_ranks}
    for r in ranks:
        if r in rp.failed:
            continue
        for c in rp.copies(r, push):
            src = bufs[(int(c["src_role"]), int(c["src_rank"]))]
            dst = bufs[(int(c["dst_role"]), int(c["dst_rank"]))]
            n, so, do = int(c["bytes"]), int(c["src_off"]), int(c["dst_off"])
            dst[do:do + n] = src[so:so + n]
            written[int(c["dst_rank"])][do:do + n] += 1
            # physical placement: push copies start on the executing GPU
            if push:
                assert int(c["src_rank"]) == r
            else:
                assert int(c["dst_rank"]) == r
            assert int(c["src_rank"]) not in rp.failed
    return bufs, written


@pytest.mark.parametrize("name,cfg,old,new", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("push", [True, False], ids=["push", "pull"])
def test_lowering_reconstructs_target_bytes(name, cfg, old, new, push, oracle):
    small = configs.scaled(cfg, 2e-5 if cfg.total_bytes > 10**10 else 1e-3)
    rp = ReshardPlan.build(small.layer_bytes, old, new)
    bufs, written = _host_execute(rp, oracle, push)
    for r in rp.new_ranks:
        want = oracle.fill_synthetic(rp.dst.segments(r), rp.dst.shard_bytes(r), SEED)
        assert np.array_equal(bufs[(ROLE_NEW, r)], want), (name, r)
        assert (written[r] == 1).all(), "every target byte written exactly once"


@pytest.mark.parametrize("d", [1, 2, 3, 4])
@pytest.mark.parametrize("push", [True, False], ids=["push", "pull"])
def test_stage_move_is_plan_zero_migration(d, push, oracle):
    """Cross-stage interleaved move of the source stage's tail layer: the
    NVLink entries are exactly plan_zero_migration's D j->j sends, and the
    lowered programs rebuild both stages' target shards byte for byte."""
    rng = np.random.default_rng(d)
    src_layers = [int(x) for x in rng.integers(1000, 5000, size=4)]
    dst_layers = [int(x) for x in rng.integers(1000, 5000, size=3)]
    src_gpus, dst_gpus = list(range(d)), list(range(d, 2 * d))
    rp = ReshardPlan.for_stage_move(src_layers, dst_layers, src_gpus, dst_gpus)
    rows, tot = fabric.plan_zero_migration(True, d, src_layers, len(src_layers) - 1, d)
    e = rp.plan.entries
    got = sorted((int(a), int(b), int(lo), int(hi)) for a, b, lo, hi in
                 zip(e["src_rank"], e["dst_rank"], e["lo"], e["hi"]))
    want = sorted((src_gpus[int(r[0])], dst_gpus[int(r[1])], int(r[3]), int(r[4])) for r in rows)
    assert got == want and rp.plan.total_bytes_moved == int(tot[2])
    bufs, written = _host_execute(rp, oracle, push)
    for r in rp.new_ranks:
        want_buf = oracle.fill_synthetic(rp.dst.segments(r), rp.dst.shard_bytes(r), SEED)
        assert np.array_equal(bufs[(ROLE_NEW, r)], want_buf)
        assert (written[r] == 1).all()


def test_traffic_matches_reference_probe_numbers():
    # 7B 8->7 drop r3, bottleneck r2 egress 10.107 GB
    rp = ReshardPlan.build(configs.llama2_7b().layer_bytes, range(8), [0, 1, 2, 4, 5, 6, 7])
    t = rp.traffic()
    assert t["total_bytes_moved"] == 26_953_662_464
    assert t["bottleneck_bytes"] == t["egress"][2] == 10_107_623_424
    assert t["local"][2] >= 5_053_811_712  # self lane of the dead rank's holder (+ retained)


def test_unrecoverable_membership_change_rejected():
    with pytest.raises(fabric.CoverageMismatch):
        ReshardPlan.build(configs.llama3_8b().layer_bytes, range(8), [0, 1, 4, 5, 6, 7])
