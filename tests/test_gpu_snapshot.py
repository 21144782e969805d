"""(a) snapshot + per-block checksum and verification on the GPU, bit-exact
against the oracle restatement (ew_oracle_row_sums) — through the C ABI."""
import json

import numpy as np
import pytest
import torch

from paper_2510_00606_b200 import configs, device as dev, fabric

pytestmark = pytest.mark.gpu


def to_host_u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def random_segments(rng, n, max_len, gap=50_000, start=None):
    segs, local = [], 0
    g = int(rng.integers(0, 4096)) if start is None else start
    for _ in range(n):
        length = int(rng.integers(0, max_len))
        segs.append((g, length, local))
        local += length
        g += length + int(rng.integers(0, gap))
    arr = np.zeros(len(segs), dtype=fabric.SEGMENT_DTYPE)
    for i, s in enumerate(segs):
        arr[i] = s
    return arr, local


@pytest.mark.parametrize("block", [4096, 65536, 1 << 20])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_snapshot_rows_match_oracle_on_misaligned_segments(oracle, block, seed):
    rng = np.random.default_rng(seed)
    segs, total = random_segments(rng, 9, 300_000)
    m = dev.ShardMap(segs, block)
    host = rng.integers(0, 256, size=total, dtype=np.uint8)
    assert m.num_rows == len(oracle.row_sums(segs, block, host)) // 2
    live = dev.empty_bytes(total)
    live[:total].copy_(torch.from_numpy(host))
    snap = dev.empty_bytes(total)
    snap.fill_(0x5A)
    rows = m.new_row_sums()
    dev.snapshot(m, live, snap, rows)
    torch.cuda.synchronize()
    want = oracle.row_sums(segs, block, host)
    assert np.array_equal(to_host_u64(rows)[:2 * m.num_rows], want)
    assert torch.equal(snap[:total], live[:total])
    # snapshot must not write past the shard
    assert (snap[total:] == 0x5A).all()

    # checksum-only and verify agree
    rows2 = m.new_row_sums()
    dev.checksum(m, snap, rows2)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.verify(m, snap, rows, bad)
    torch.cuda.synchronize()
    assert torch.equal(rows, rows2)
    assert int(bad.item()) == 0


def test_verify_detects_each_corruption(oracle):
    rng = np.random.default_rng(9)
    segs, total = random_segments(rng, 5, 500_000)
    m = dev.ShardMap(segs, 65536)
    live = dev.empty_bytes(total)
    live[:total].copy_(torch.from_numpy(rng.integers(0, 256, size=total, dtype=np.uint8)))
    snap = dev.empty_bytes(total)
    rows = m.new_row_sums()
    dev.snapshot(m, live, snap, rows)
    row_blocks = m.row_blocks()
    # local byte -> row index
    starts = []
    r = 0
    for s in segs:
        if s["length"] == 0:
            continue
        b0 = s["global_lo"] // 65536
        b1 = (s["global_lo"] + s["length"] - 1) // 65536
        for b in range(b0, b1 + 1):
            lo = max(s["global_lo"], b * 65536) - s["global_lo"] + s["local_off"]
            starts.append((lo, r))
            r += 1
    starts = np.array(starts)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    bad_rows = torch.full((8,), -1, dtype=torch.int64, device="cuda")
    for pos in rng.integers(0, total, size=12).tolist() + [0, total - 1]:
        snap[pos] ^= 0x10
        dev.verify(m, snap, rows, bad, bad_rows)
        torch.cuda.synchronize()
        expect_row = int(starts[np.searchsorted(starts[:, 0], pos, side="right") - 1, 1])
        assert int(bad.item()) == 1
        assert int(bad_rows[0].item()) == expect_row
        snap[pos] ^= 0x10
    # swapping two words inside a block changes s1 (position-weighted)
    a, b = 1024, 2048
    if total > 4096:
        tmp = snap[a:a + 8].clone()
        snap[a:a + 8] = snap[b:b + 8]
        snap[b:b + 8] = tmp
        if not torch.equal(snap[a:a + 8], snap[b:b + 8]):
            dev.verify(m, snap, rows, bad)
            torch.cuda.synchronize()
            assert int(bad.item()) >= 1


def test_fill_synthetic_matches_oracle(oracle):
    rng = np.random.default_rng(4)
    segs, total = random_segments(rng, 7, 100_000)
    m = dev.ShardMap(segs, 65536)
    buf = dev.empty_bytes(total)
    dev.fill_synthetic(m, buf, 2024)
    want = oracle.fill_synthetic(segs, total, 2024)
    assert np.array_equal(buf[:total].cpu().numpy(), want)


def test_rank_rows_sum_to_whole_space_block_sums(oracle):
    """Rows of every rank of an interleaved layout, scattered into global
    blocks and added, equal the oracle's whole-space block sums."""
    cfg = configs.scaled(configs.gpt_125m(), 1e-3)
    block = 65536
    nblocks = (cfg.total_bytes + block - 1) // block
    for ranks in ([0, 1, 2, 3], [0, 2, 3]):
        layout = fabric.interleaved_layout(cfg.layer_bytes, ranks)
        acc = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
        for r in ranks:
            m = dev.ShardMap(layout.segments(r), block)
            buf = dev.empty_bytes(layout.shard_bytes(r))
            dev.fill_synthetic(m, buf, 7)
            rows = m.new_row_sums()
            dev.checksum(m, buf, rows)
            dev.rows_to_blocks(m, rows, acc)
        torch.cuda.synchronize()
        want = oracle.block_sums_synthetic(7, cfg.total_bytes, block)
        assert np.array_equal(to_host_u64(acc), want)


def test_checksum_golden_on_gpu(golden_dir):
    g = json.loads((golden_dir / "checksum_golden.json").read_text())
    rng = np.random.default_rng(2024)
    for case in g["cases"]:
        local = 0
        for length in (5, 70001, 9, 131077):
            local += length
            rng.integers(1, 40000)
        host = rng.integers(0, 256, size=local, dtype=np.uint8)
        segs = np.zeros(len(case["segments"]), dtype=fabric.SEGMENT_DTYPE)
        for i, s in enumerate(case["segments"]):
            segs[i] = (s["global_lo"], s["length"], s["local_off"])
        m = dev.ShardMap(segs, case["block_bytes"])
        buf = dev.empty_bytes(local)
        buf[:local].copy_(torch.from_numpy(host))
        rows = m.new_row_sums()
        dev.checksum(m, buf, rows)
        torch.cuda.synchronize()
        assert [str(int(x)) for x in to_host_u64(rows)[:2 * m.num_rows]] == case["rows"]
    # GPU synthetic fill + fused snapshot rows == the spec restatement's rows
    sr = g["synthetic_rows"]
    segs = np.zeros(len(sr["segments"]), dtype=fabric.SEGMENT_DTYPE)
    for i, s in enumerate(sr["segments"]):
        segs[i] = (s["global_lo"], s["length"], s["local_off"])
    m = dev.ShardMap(segs, sr["block_bytes"])
    for seed, want in sr["rows"].items():
        live = dev.empty_bytes(m.nbytes)
        dev.fill_synthetic(m, live, int(seed))
        snap = dev.empty_bytes(m.nbytes)
        rows = m.new_row_sums()
        dev.snapshot(m, live, snap, rows)
        torch.cuda.synchronize()
        assert [str(int(x)) for x in to_host_u64(rows)[:2 * m.num_rows]] == want


def test_empty_and_tiny_shards(oracle):
    for segs_list in ([], [(0, 0, 0)], [(5, 1, 0)], [(8, 3, 0), (100, 2, 3)]):
        segs = np.zeros(len(segs_list), dtype=fabric.SEGMENT_DTYPE)
        for i, s in enumerate(segs_list):
            segs[i] = s
        total = int(sum(s[1] for s in segs_list))
        m = dev.ShardMap(segs, 4096)
        live = dev.empty_bytes(total)
        live.random_(0, 256)
        snap = dev.empty_bytes(total)
        rows = m.new_row_sums()
        dev.snapshot(m, live, snap, rows)
        torch.cuda.synchronize()
        want = oracle.row_sums(segs, 4096, live[:total].cpu().numpy())
        assert np.array_equal(to_host_u64(rows)[:2 * m.num_rows], want)
        assert torch.equal(snap[:total], live[:total])


@pytest.mark.timeout(900)
def test_full_size_7b_rows_and_blocks_vs_oracle(oracle):
    """Config B at full size: every checksum row of rank 3's 11.79 GB shard
    (GPU fill + fused snapshot) equals the C oracle's rows recomputed from
    the synthetic words on the host cores, and the rows of all 8 ranks'
    shards, folded into block sums, equal the oracle's block sums of the
    whole 94.3 GB space."""
    cfg = configs.llama2_7b()
    layout = fabric.interleaved_layout(cfg.layer_bytes, range(8))
    block = 65536
    nb = (cfg.total_bytes + block - 1) // block
    acc = torch.zeros(2 * nb, dtype=torch.int64, device="cuda")
    n_max = max(layout.shard_bytes(r) for r in range(8))
    live = dev.empty_bytes(n_max)
    snap = dev.empty_bytes(n_max)
    for r in range(8):
        m = dev.ShardMap(layout.segments(r), block)
        dev.fill_synthetic(m, live, 0)
        rows = m.new_row_sums()
        dev.snapshot(m, live, snap, rows)
        dev.rows_to_blocks(m, rows, acc)
        if r == 3:
            torch.cuda.synchronize()
            want = oracle.rows_synthetic_mt(layout.segments(r), block, 0)
            assert np.array_equal(to_host_u64(rows)[:2 * m.num_rows], want)
    torch.cuda.synchronize()
    del live, snap
    torch.cuda.empty_cache()
    assert np.array_equal(to_host_u64(acc), oracle.block_sums_synthetic_mt(0, cfg.total_bytes,
                                                                           block))


def test_full_size_7b_shard_properties():
    """At the config-B per-rank size (11.79 GB): snapshot then verify passes
    and a single flipped bit is caught."""
    cfg = configs.llama2_7b()
    layout = fabric.interleaved_layout(cfg.layer_bytes, range(8))
    m = dev.ShardMap(layout.segments(3), 65536)
    n = layout.shard_bytes(3)
    live = dev.empty_bytes(n)
    dev.fill_synthetic(m, live, 0)
    snap = dev.empty_bytes(n)
    rows = m.new_row_sums()
    dev.snapshot(m, live, snap, rows)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.verify(m, snap, rows, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 0
    assert torch.equal(snap[:n], live[:n])
    snap[n // 2] ^= 1
    dev.verify(m, snap, rows, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 1
    del live, snap
    torch.cuda.empty_cache()
