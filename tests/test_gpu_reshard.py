"""(b) reshard executor on the GPU.  The copy kernel against byte-exact
expectations for arbitrary (mutually misaligned) copies, and the full N-rank
membership changes run on one GPU (every rank's program, buffers side by
side): target shards must equal the regenerated synthetic state, and their
checksum rows must add up to the source's block sums."""
import numpy as np
import pytest
import torch

from paper_2510_00606_b200 import configs, device as dev, fabric
from paper_2510_00606_b200.reshard import ReshardPlan, emulate_on_one_gpu, shard_map

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", range(6))
def test_copy_kernel_arbitrary_alignment(seed):
    rng = np.random.default_rng(seed)
    n_src, n_dst = 3_000_000, 3_000_000
    src = torch.randint(0, 256, (n_src,), dtype=torch.uint8, device="cuda")
    dst = torch.zeros(n_dst, dtype=torch.uint8, device="cuda")
    expect = dst.clone()
    # disjoint destination ranges, random sizes (0..200 KB), random offsets
    cur = int(rng.integers(0, 64))
    srcs, dsts, sizes, remote = [], [], [], []
    while True:
        size = int(rng.integers(0, 200_000)) if rng.random() > 0.2 else int(rng.integers(0, 40))
        if cur + size > n_dst:
            break
        so = int(rng.integers(0, n_src - size + 1))
        srcs.append(src.data_ptr() + so)
        dsts.append(dst.data_ptr() + cur)
        sizes.append(size)
        remote.append(bool(rng.random() < 0.5))
        expect[cur:cur + size] = src[so:so + size]
        cur += size + int(rng.integers(0, 3))
    prog = dev.CopyProgram.from_pointers(srcs, dsts, sizes, remote)
    prog.launch()
    torch.cuda.synchronize()
    assert torch.equal(dst, expect)
    # re-launch with explicit CTA splits gives the same bytes
    dst.zero_()
    prog.launch(n_ctas=37, remote_ctas=5)
    torch.cuda.synchronize()
    assert torch.equal(dst, expect)


CASES = [
    ("125M 4->3 drop r1", configs.gpt_125m(), [0, 1, 2, 3], [0, 2, 3], 1e-2),
    ("7B 8->7 drop r0", configs.llama2_7b(), list(range(8)), [1, 2, 3, 4, 5, 6, 7], 1e-3),
    ("7B 8->7 drop r3", configs.llama2_7b(), list(range(8)), [0, 1, 2, 4, 5, 6, 7], 1e-3),
    ("7B 8->7 drop r7", configs.llama2_7b(), list(range(8)), [0, 1, 2, 3, 4, 5, 6], 1e-3),
    ("7B per-tensor 8->7 drop r4", configs.llama2_7b_per_tensor(), list(range(8)),
     [0, 1, 2, 3, 5, 6, 7], 1e-3),
    ("8B 8->6 drop r2,r5", configs.llama3_8b(), list(range(8)), [0, 1, 3, 4, 6, 7], 1e-3),
    ("8B 6->8 rejoin", configs.llama3_8b(), [0, 1, 3, 4, 6, 7], list(range(8)), 1e-3),
    ("2->1", configs.gpt_125m(), [0, 1], [0], 1e-2),
]


@pytest.mark.parametrize("name,cfg,old,new,scale", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("push", [True, False], ids=["push", "pull"])
def test_membership_change_on_one_gpu(name, cfg, old, new, scale, push, oracle):
    small = configs.scaled(cfg, scale)
    rp = ReshardPlan.build(small.layer_bytes, old, new)
    got, expected = emulate_on_one_gpu(rp, seed=2024, push=push)
    for r in rp.new_ranks:
        n = rp.dst.shard_bytes(r)
        assert torch.equal(got[r][:n], expected[r][:n]), (name, r)
    # checksum conservation: rows of all target shards == synthetic block sums
    block = 65536
    nblocks = (small.total_bytes + block - 1) // block
    acc = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    for r in rp.new_ranks:
        m = shard_map(rp.dst, r, block)
        rows = m.new_row_sums()
        dev.checksum(m, got[r], rows)
        dev.rows_to_blocks(m, rows, acc)
    torch.cuda.synchronize()
    want = oracle.block_sums_synthetic(2024, small.total_bytes, block)
    assert np.array_equal(acc.cpu().numpy().view(np.uint64), want)


@pytest.mark.parametrize("name,cfg,old,new,scale", CASES, ids=[c[0] for c in CASES])
def test_verification_on_arrival(name, cfg, old, new, scale, oracle):
    """Verified pull programs: the checksums of what every rank lands in NEW,
    labelled by NEW's own segment map, add up to the source state's block
    sums — no re-read of NEW — and the bytes are still exact."""
    small = configs.scaled(cfg, scale)
    rp = ReshardPlan.build(small.layer_bytes, old, new)
    block = 65536
    nblocks = (small.total_bytes + block - 1) // block
    sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    got, expected = emulate_on_one_gpu(rp, seed=77, push=False, block_sums=sums)
    for r in rp.new_ranks:
        n = rp.dst.shard_bytes(r)
        assert torch.equal(got[r][:n], expected[r][:n]), (name, r)
    torch.cuda.synchronize()
    want = oracle.block_sums_synthetic(77, small.total_bytes, block)
    assert np.array_equal(sums.cpu().numpy().view(np.uint64), want)


@pytest.mark.parametrize("contiguous", [False, True])
def test_verification_on_arrival_in_place_stage_move(contiguous, oracle):
    """Cross-stage layer move with in-place buffers: retained bytes are not
    rewritten but still read and checksummed, so conservation holds."""
    small = configs.scaled(configs.llama2_7b(), 1e-3)
    lb = small.layer_bytes
    rp = ReshardPlan.for_stage_move(lb[:17], lb[17:], [0, 1], [2, 3], contiguous)
    block = 65536
    total = sum(lb)
    nblocks = (total + block - 1) // block
    sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    got, expected = emulate_on_one_gpu(rp, seed=9, push=False, block_sums=sums, in_place=True)
    for r in rp.new_ranks:
        n = rp.dst.shard_bytes(r)
        assert torch.equal(got[r][:n], expected[r][:n]), r
    torch.cuda.synchronize()
    want = oracle.block_sums_synthetic(9, total, block)
    assert np.array_equal(sums.cpu().numpy().view(np.uint64), want)


def test_verification_on_arrival_catches_misplacement_and_corruption(oracle):
    small = configs.scaled(configs.llama2_7b(), 1e-3)
    rp = ReshardPlan.build(small.layer_bytes, list(range(8)), [0, 1, 2, 4, 5, 6, 7])
    block = 65536
    nblocks = (small.total_bytes + block - 1) // block
    want = oracle.block_sums_synthetic(5, small.total_bytes, block)

    def shifted(rank, descs):  # one copy lands 8 bytes early in NEW
        d = descs.copy()
        if rank == 2:
            k = int(np.argmax(d["dst_off"] >= 64))
            d["dst_off"][k] -= 8
        return d

    sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    emulate_on_one_gpu(rp, seed=5, push=False, block_sums=sums, tamper=shifted)
    torch.cuda.synchronize()
    assert not np.array_equal(sums.cpu().numpy().view(np.uint64), want)

    def dropped(rank, descs):  # one copy never issued
        return descs[1:] if rank == 4 else descs

    sums.zero_()
    emulate_on_one_gpu(rp, seed=5, push=False, block_sums=sums, tamper=dropped)
    torch.cuda.synchronize()
    assert not np.array_equal(sums.cpu().numpy().view(np.uint64), want)


def test_full_size_7b_one_rank_program_locally():
    """Config B at full size for the receive side of one survivor: the
    executing rank's push program runs with every peer buffer placed on the
    same GPU (retained + self-lane + 'remote' stores), 8->7 drop r3."""
    cfg = configs.llama2_7b()
    rp = ReshardPlan.build(cfg.layer_bytes, range(8), [0, 1, 2, 4, 5, 6, 7])
    r = 4  # receives from r2's replica and from r5 (retained + remote)
    need = {(fabric.ROLE_NEW, r)}
    for c in rp.copies(r, push=False):
        need.add((int(c["src_role"]), int(c["src_rank"])))
    bufs, table = {}, {}
    for role, rank in need:
        if role == fabric.ROLE_NEW:
            t = dev.empty_bytes(rp.dst.shard_bytes(rank))
        else:
            owner = rp.replica_of(rank) if role == fabric.ROLE_REPLICA else rank
            t = dev.empty_bytes(rp.src.shard_bytes(owner))
            dev.fill_synthetic(shard_map(rp.src, owner), t, 0)
        bufs[(role, rank)] = t
        table[(role, rank)] = t.data_ptr()
    prog = dev.CopyProgram.from_descs(rp.copies(r, push=False), table, 8, r)
    prog.launch()
    expect = dev.empty_bytes(rp.dst.shard_bytes(r))
    dev.fill_synthetic(shard_map(rp.dst, r), expect, 0)
    torch.cuda.synchronize()
    n = rp.dst.shard_bytes(r)
    assert torch.equal(bufs[(fabric.ROLE_NEW, r)][:n], expect[:n])


@pytest.mark.parametrize("name,cfg,old,new,slack", [
    ("7B 8->7 drop r3", configs.llama2_7b(), list(range(8)), [0, 1, 2, 4, 5, 6, 7], 1),
    ("7B 8->7 drop r0", configs.llama2_7b(), list(range(8)), [1, 2, 3, 4, 5, 6, 7], 2),
    ("8B 8->6 drop r2,r5", configs.llama3_8b(), list(range(8)), [0, 1, 3, 4, 6, 7], 0),
    ("8B 6->8 rejoin", configs.llama3_8b(), [0, 1, 3, 4, 6, 7], list(range(8)), 1),
    ("fill-HBM 4->3", configs.fill_hbm(4, 40_000_000), [0, 1, 2, 3], [0, 1, 2], 1),
    ("2->1", configs.gpt_125m(), [0, 1], [1], 1),
])
def test_inplace_reshard_on_one_gpu(name, cfg, old, new, slack, oracle):
    """Staged in-place reshard (OLD and NEW share one buffer per rank): every
    rank's direct / staged / flush programs, run-ahead writes poisoned before
    each phase reads; target bytes exact, block sums conserved."""
    from paper_2510_00606_b200.inplace import emulate_inplace_on_one_gpu
    small = configs.scaled(cfg, 2e-3) if cfg.total_bytes > 10**9 else cfg
    rp = ReshardPlan.build(small.layer_bytes, old, new)
    stage = max(1 << 16, max(rp.dst.shard_bytes(r) for r in new) // 9)
    block = 65536
    nblocks = (small.total_bytes + block - 1) // block
    sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    got, expected, sc = emulate_inplace_on_one_gpu(rp, 41, stage, 2 * stage, slack, sums, block)
    assert len(sc.phases) > 3
    for r in rp.new_ranks:
        assert torch.equal(got[r], expected[r]), (name, r)
    want = oracle.block_sums_synthetic(41, small.total_bytes, block)
    assert np.array_equal(sums.cpu().numpy().view(np.uint64), want)
