"""Empty and degenerate inputs across the device entry points: every call
accepts zero-sized work as a no-op (the reference's planners accept empty
layers / zero-byte intervals the same way, test_param_fabric.cpp and
test_migration.cpp), and tiny ragged sizes agree with the oracle."""
import numpy as np
import pytest
import torch

from paper_2510_00606_b200 import device as dev
from paper_2510_00606_b200.migration import payback_accumulate

pytestmark = pytest.mark.gpu


def test_philox_zero_samples_and_zero_elements(oracle):
    assert dev.dropout_mask(0, 5, 0, 1, 0, 4096, 0.5).numel() == 0
    assert dev.dropout_mask(0, 5, 3, 1, 0, 0, 0.5).numel() == 0
    u = dev.philox_uniforms(0, 5, 0, 1, 0, 17)
    assert u.numel() == 0
    # one element, many samples, around sample id 2^32 (counter word carry)
    bits = dev.dropout_mask(7, 2 ** 32 - 2, 4, 2, 3, 1, 0.5).cpu().numpy().view(np.uint32)
    assert np.array_equal(bits, oracle.dropout_mask(7, 2 ** 32 - 2, 4, 2, 3, 1, 0.5))


def test_fold_and_dequant_zero_elements():
    acc = torch.empty(0, dtype=torch.int64, device="cuda")
    dev.weighted_fold([torch.empty(0, device="cuda")], [0.5], 10, acc)
    assert dev.fixed_to_float(acc, 10).numel() == 0


def test_fold_without_units_zeroes_or_keeps():
    acc = torch.full((9,), 5, dtype=torch.int64, device="cuda")
    from paper_2510_00606_b200._native import lib
    import ctypes as C
    dev.check(lib.ew_weighted_fold(None, None, 0, 9, 10, dev._ptr(acc), 1, dev._stream()))
    torch.cuda.synchronize()
    assert acc.tolist() == [5] * 9          # accumulate: unchanged
    dev.check(lib.ew_weighted_fold(None, None, 0, 9, 10, dev._ptr(acc), 0, dev._stream()))
    torch.cuda.synchronize()
    assert acc.tolist() == [0] * 9          # overwrite: zero


def test_fold_addend_matches_separate_add(oracle):
    rng = np.random.default_rng(2)
    for n in (1, 5, 4099):
        g = rng.normal(0, 1e-2, (2, n)).astype(np.float32)
        w = np.array([0.25, 0.75])
        add = torch.from_numpy(rng.integers(-2 ** 40, 2 ** 40, n)).cuda()
        units = [torch.from_numpy(x).cuda() for x in g]
        acc = torch.empty(n, dtype=torch.int64, device="cuda")
        dev.weighted_fold(units, w, 30, acc, addend=add)
        torch.cuda.synchronize()
        want = oracle.weighted_fixed(w, g, 30) + add.cpu().numpy()
        assert np.array_equal(acc.cpu().numpy(), want)


def test_pipelined_fold_addend_accumulate_and_device_scale(oracle):
    """3+ units take the software-pipelined fold (kPipe): with an addend,
    with accumulate, with the scale read from device memory, on ragged sizes
    (scalar tails) — all bit-exact against the oracle."""
    rng = np.random.default_rng(9)
    for n in (1, 7, 8, 4099, 100_003):
        g = rng.normal(0, 1e-2, (5, n)).astype(np.float32)
        w = np.array([0.1, 0.15, 0.2, 0.25, 0.3])
        add = torch.from_numpy(rng.integers(-2 ** 40, 2 ** 40, n)).cuda()
        units = [torch.from_numpy(x).cuda() for x in g]
        want = oracle.weighted_fixed(w, g, 30)
        acc = torch.empty(n, dtype=torch.int64, device="cuda")
        dev.weighted_fold(units, w, 30, acc, addend=add)
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy(), want + add.cpu().numpy()), n
        dev.weighted_fold(units, w, 30, acc, accumulate=True)
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy(), 2 * want + add.cpu().numpy()), n
        bits = torch.tensor([30], dtype=torch.int32, device="cuda")
        dev.weighted_fold_dev(units, w, bits, acc)
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy(), want), n


def test_copy_program_without_items_and_adam_payback_zero():
    p = dev.CopyProgram.from_pointers([], [], [], [])
    p.launch()
    st = dev.AdamState(0)
    dev.adam_step(torch.empty(0, device="cuda"), st, dev.adam_hyper(), 1)
    a = torch.empty(0, dtype=torch.int64, device="cuda")
    payback_accumulate(a, a)
    torch.cuda.synchronize()


def test_snapshot_of_single_byte_segment_at_odd_global_offset(oracle):
    segs = np.zeros(1, dtype=[("global_lo", np.int64), ("length", np.int64), ("local_off", np.int64)])
    segs[0] = (65536 * 3 + 7, 1, 0)
    m = dev.ShardMap(segs)
    live = dev.empty_bytes(32)
    live.fill_(0)
    live[0] = 0xAB
    snap = dev.empty_bytes(32)
    rows = m.new_row_sums()
    dev.snapshot(m, live, snap, rows)
    torch.cuda.synchronize()
    want = oracle.row_sums(segs, 65536, live.cpu().numpy()[:1])
    assert np.array_equal(rows.cpu().numpy().view(np.uint64)[:2], want[:2])
    assert int(snap[0].item()) == 0xAB


def test_guarded_copy_vetoed_by_flag():
    """ew_copy_program_launch_guarded: a set abort flag (a timed-out peer
    barrier upstream) makes the copy write nothing; a clear one copies."""
    src = torch.arange(40000, dtype=torch.int32, device="cuda").view(torch.uint8)
    dst = torch.zeros_like(src)
    prog = dev.CopyProgram.from_pointers([src.data_ptr() + 3], [dst.data_ptr() + 5],
                                         [src.numel() - 8], [False])
    flag = torch.ones(1, dtype=torch.int32, device="cuda")
    prog.launch(abort_flag=flag.data_ptr())
    torch.cuda.synchronize()
    assert int(dst.count_nonzero()) == 0
    flag.zero_()
    prog.launch(abort_flag=flag.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(dst[5:5 + src.numel() - 8], src[3:3 + src.numel() - 8])
