"""Ring replica by optimizer replay on the GPU: ew_adam_step
is bit-exact against the oracle restatement (fp32 master, exp_avg,
exp_avg_sq and the bf16 parameter copy, every element, several steps, ragged
sizes), so a holder replaying the owner's gradient reproduces the owner's
state byte for byte and the owner's checksum rows verify it."""
import numpy as np
import pytest
import torch

from paper_2510_00606_b200 import device as dev

pytestmark = pytest.mark.gpu

HYPER = (1e-3, 0.9, 0.999, 1e-8, 0.01)


def _grads(rng, n, step):
    g = rng.normal(0, 1e-3, n).astype(np.float32)
    g[::89] *= 1e4
    g[::1013] = 0.0
    if step == 2 and n > 7:
        g[7] = -3e38  # huge gradient: v overflows to inf, p stays finite
    return g


@pytest.mark.parametrize("n", [1, 3, 4, 5, 1001, (1 << 20) + 3])
def test_adam_step_bit_exact_vs_oracle(oracle, n):
    rng = np.random.default_rng(n)
    p0 = rng.normal(0, 0.02, n).astype(np.float32)
    st = dev.AdamState(n)
    st.master.copy_(torch.from_numpy(p0))
    cm, cv, cp = np.zeros(n, np.float32), np.zeros(n, np.float32), np.zeros(n, np.uint16)
    cmaster = p0.copy()
    h = dev.adam_hyper(*HYPER)
    for step in range(1, 4):
        g = _grads(rng, n, step)
        dev.adam_step(torch.from_numpy(g).cuda(), st, h, step)
        oracle.adam_step(g, cmaster, cm, cv, cp, HYPER, step)
        torch.cuda.synchronize()
        for got, want in ((st.master, cmaster), (st.exp_avg, cm), (st.exp_avg_sq, cv)):
            assert np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32)), step
        assert np.array_equal(st.param.cpu().view(torch.int16).numpy().view(np.uint16), cp)


def test_replay_reproduces_state_and_rows():
    """Owner and holder (here: two states on one GPU) step from the same
    gradient; the holder's byte image and checksum rows equal the owner's,
    and a single flipped bit in the replica is caught by verify."""
    n = 3 * (1 << 18) + 1
    rng = np.random.default_rng(1)
    owner, holder = dev.AdamState(n), dev.AdamState(n)
    owner.master.copy_(torch.from_numpy(rng.normal(0, 0.02, n).astype(np.float32)))
    holder.buf.copy_(owner.buf)
    m = dev.ShardMap(owner.segments())
    h = dev.adam_hyper()
    for step in range(1, 4):
        g = torch.from_numpy(_grads(rng, n, step)).cuda()
        dev.adam_step(g, owner, h, step)
        dev.adam_step(g.data_ptr(), holder, h, step)  # raw-pointer path (peer use)
    rows = m.new_row_sums()
    dev.checksum(m, owner.buf, rows)
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.verify(m, holder.buf, rows, bad)
    torch.cuda.synchronize()
    assert torch.equal(owner.buf, holder.buf)
    assert int(bad.item()) == 0
    holder.buf[12345] ^= 0x10
    dev.verify(m, holder.buf, rows, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 1


@pytest.mark.parametrize("n", [1, 3, 5, 4099, (1 << 20) + 3, 3 * (1 << 20) + 1])
@pytest.mark.parametrize("block", [4096, 65536])
def test_fused_rows_equal_checksum_of_image(n, block):
    """ew_adam_step_rows' rows == kernel (a)'s rows of the state image
    (bit-exact), incl. partial words of ragged tails and rows straddled by
    warps; and rows_diff finds a planted mismatch."""
    rng = np.random.default_rng(n)
    st = dev.AdamState(n)
    st.master.copy_(torch.from_numpy(rng.normal(0, 0.02, n).astype(np.float32)))
    m = dev.ShardMap(st.segments(), block)
    fused = m.new_row_sums()
    for step in (1, 2):
        g = torch.from_numpy(_grads(rng, n, step)).cuda()
        dev.adam_step(g, st, dev.adam_hyper(), step, rows=fused, block_bytes=block)
    ref = m.new_row_sums()
    dev.checksum(m, st.buf, ref)
    torch.cuda.synchronize()
    assert torch.equal(fused[:2 * m.num_rows], ref[:2 * m.num_rows])
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.rows_diff(fused, ref, m.num_rows, bad)
    fused[2 * (m.num_rows - 1) + 1] += 1
    bad2 = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.rows_diff(fused, ref, m.num_rows, bad2)
    torch.cuda.synchronize()
    assert int(bad.item()) == 0 and int(bad2.item()) == 1


def test_adam_step_rejects_misaligned():
    st = dev.AdamState(64)
    g = torch.zeros(65, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        dev.adam_step(g.data_ptr() + 4, st, dev.adam_hyper(), 1)
    with pytest.raises(ValueError):
        dev.adam_step(g, st, dev.adam_hyper(), 0)


def test_fused_rows_fallback_for_unaligned_sections():
    """Sections that do not start on checksum-block boundaries take the
    warp-atomic path of ew_adam_step_rows; its rows still equal kernel (a)'s."""
    import ctypes as C
    from paper_2510_00606_b200._native import lib
    n = 100_003
    sec = 4 * n + 256 - (4 * n) % 256          # 256-aligned, not 64 KiB-aligned
    nbytes = 3 * sec + 2 * n + 14
    buf = torch.zeros(nbytes + 16, dtype=torch.uint8, device="cuda")
    f32 = lambda k: buf[k * sec:k * sec + 4 * n].view(torch.float32)
    master, m, v = f32(0), f32(1), f32(2)
    param = buf[3 * sec:3 * sec + 2 * n].view(torch.bfloat16)
    rng = np.random.default_rng(4)
    master.copy_(torch.from_numpy(rng.normal(0, 0.02, n).astype(np.float32)))
    g = torch.from_numpy(_grads(rng, n, 1)).cuda()
    segs = np.zeros(1, dtype=[("global_lo", np.int64), ("length", np.int64), ("local_off", np.int64)])
    segs[0] = (0, nbytes, 0)
    mp = dev.ShardMap(segs, 65536)
    rows = mp.new_row_sums()
    h = dev.adam_hyper()
    dev.check(lib.ew_adam_step_rows(dev._ptr(g), dev._ptr(master), dev._ptr(m), dev._ptr(v),
                                    dev._ptr(param), n, C.byref(h), 1, dev._ptr(buf), nbytes,
                                    65536, dev._ptr(rows), dev._stream()))
    ref = mp.new_row_sums()
    dev.checksum(mp, buf, ref)
    torch.cuda.synchronize()
    assert torch.equal(rows[:2 * mp.num_rows], ref[:2 * mp.num_rows])
