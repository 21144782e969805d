"""(d) weighted reduce on the GPU: the fixed-point fold is bit-exact against
the oracle, invariant to how units are split (the world-size determinism the
NCCL int64 sum inherits), and within the stated tolerance of the reference's
fp64 weighted_grad_average.

Tolerance (fp32 output vs fp64 reference fold):
    |out - ref| <= U * 2^-(F+1)  +  2^-24 * |ref|  +  U * 2^-52 * sum_u |w_u g_u|
(quantisation of U units, one fp32 output rounding, the reference's own fp64
fold rounding)."""
import numpy as np
import pytest
import torch

from paper_2510_00606_b200 import device as dev, fabric

pytestmark = pytest.mark.gpu


def make_units(seed, n_units, dim):
    rng = np.random.default_rng(seed)
    g = rng.normal(0, 1e-3, size=(n_units, dim)).astype(np.float32)
    idx = rng.integers(0, dim, size=max(1, dim // 1_000_000))
    g[0, idx] = 1e2  # outliers
    g[-1, (idx + 1) % dim] = -1e2
    return g


@pytest.mark.parametrize("dim", [1, 3, 4, 1001, 1 << 20])
def test_fold_bit_exact_vs_oracle(oracle, dim):
    g = make_units(5, 5, dim)
    w = np.array([7, 7, 6, 6, 6], dtype=np.float64) / 32
    units = [torch.from_numpy(x).cuda() for x in g]
    amax = dev.weighted_absmax(units, w).item()
    assert amax == float(np.max(np.abs(w[:, None] * g.astype(np.float64))))
    f = dev.fixed_point_bits(amax, 5)
    assert f == oracle.fixed_point_bits(amax, 5)
    acc = torch.empty(dim, dtype=torch.int64, device="cuda")
    dev.weighted_fold(units, w, f, acc)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), oracle.weighted_fixed(w, g, f))


def test_split_invariance_any_world_size():
    """Units folded on 1, 2, 3 or 5 'ranks' then summed (what NCCL's int64
    all-reduce does) give identical integers; dequantised outputs are
    bit-identical."""
    dim = 300_001
    g = make_units(7, 10, dim)
    w = np.full(10, 0.1)
    units = [torch.from_numpy(x).cuda() for x in g]
    amax = dev.weighted_absmax(units, w).item()
    f = dev.fixed_point_bits(amax, 10)
    results = []
    for split in ([10], [5, 5], [3, 3, 4], [2, 2, 2, 2, 2], [1] * 10):
        total = torch.zeros(dim, dtype=torch.int64, device="cuda")
        lo = 0
        for n in split:
            part = torch.empty(dim, dtype=torch.int64, device="cuda")
            dev.weighted_fold(units[lo:lo + n], w[lo:lo + n], f, part)
            total += part
            lo += n
        results.append(dev.fixed_to_float(total, f))
    for r in results[1:]:
        assert torch.equal(r, results[0])


def test_dequant_within_tolerance_of_reference_fold(reference):
    dim = 50_000
    g = make_units(11, 5, dim)
    w = np.array([7, 7, 6, 6, 6], dtype=np.float64) / 32
    units = [torch.from_numpy(x).cuda() for x in g]
    f = dev.fixed_point_bits(dev.weighted_absmax(units, w).item(), 5)
    acc = torch.empty(dim, dtype=torch.int64, device="cuda")
    dev.weighted_fold(units, w, f, acc)
    out = dev.fixed_to_float(acc, f).cpu().numpy().astype(np.float64)
    ref = reference.weighted_grad_average(w, g.astype(np.float64))
    bound = (5 * 2.0 ** -(f + 1) + 2.0 ** -24 * np.abs(ref)
             + 5 * 2.0 ** -52 * np.sum(np.abs(w[:, None] * g.astype(np.float64)), axis=0))
    assert (np.abs(out - ref) <= bound).all()


def test_accumulate_over_unit_chunks():
    dim = 10_000
    g = make_units(3, 20, dim)  # > 16 units per launch -> chunked
    w = np.linspace(0.01, 0.1, 20)
    units = [torch.from_numpy(x).cuda() for x in g]
    f = dev.fixed_point_bits(dev.weighted_absmax(units, w).item(), 20)
    a = torch.empty(dim, dtype=torch.int64, device="cuda")
    dev.weighted_fold(units, w, f, a)
    b = torch.empty(dim, dtype=torch.int64, device="cuda")
    dev.weighted_fold(units[:9], w[:9], f, b)
    dev.weighted_fold(units[9:], w[9:], f, b, accumulate=True)
    assert torch.equal(a, b)


def test_misaligned_unit_pointers_use_scalar_path(oracle):
    dim = 1003
    base = torch.from_numpy(make_units(2, 2, dim + 1)).cuda()
    units = [base[0, 1:], base[1, 1:]]  # 4-byte offset -> not 16-byte aligned
    w = [0.25, 0.75]
    f = dev.fixed_point_bits(dev.weighted_absmax(units, w).item(), 2)
    acc = torch.empty(dim, dtype=torch.int64, device="cuda")
    dev.weighted_fold(units, w, f, acc)
    want = oracle.weighted_fixed(np.array(w), base[:, 1:].cpu().numpy(), f)
    assert np.array_equal(acc.cpu().numpy(), want)


@pytest.mark.parametrize("dim", [1, 5, 4099, 1 << 20])
def test_absmax_exact_vs_numpy_with_specials(dim):
    """The bit-pattern max (max_i |g| then one fp64 scaling per unit) equals
    the elementwise fp64 definition, including negative weights, > 16 units,
    misaligned units, +-inf and NaN propagation."""
    g = make_units(13, 18, dim + 1)
    w = np.linspace(-0.3, 0.2, 18)
    units = [torch.from_numpy(x).cuda()[1:] if k % 3 == 0 else torch.from_numpy(x[:dim]).cuda()
             for k, x in enumerate(g)]
    host = [u.cpu().numpy().astype(np.float64) for u in units]
    want = max(float(np.max(np.abs(w[k] * host[k]))) for k in range(18))
    assert dev.weighted_absmax(units, w).item() == want
    units[7][dim // 2] = float("inf")
    assert dev.weighted_absmax(units, w).item() == float("inf")
    units[11][dim - 1] = float("nan")
    assert np.isnan(dev.weighted_absmax(units, w).item())


@pytest.mark.parametrize("dim", [1, 3, 4, 7, 4097, 1 << 20])
def test_dequant_vectorised_tails(dim):
    rng = np.random.default_rng(dim)
    acc = torch.from_numpy(rng.integers(-2**61, 2**61, size=dim + 1, dtype=np.int64)).cuda()
    for a in (acc[:dim], acc[1:]):  # aligned and 8-byte-offset views
        host = a.cpu().numpy().astype(np.float64) * 2.0 ** -40
        assert np.array_equal(dev.fixed_to_float(a, 40).cpu().numpy(), host.astype(np.float32))
        assert np.array_equal(dev.fixed_to_double(a, 40).cpu().numpy(), host)


def test_device_scale_path_in_a_cuda_graph(oracle):
    """The (d) step with the scale in device memory — absmax, scale,
    fold, dequant — captured once in a CUDA graph and replayed: no host
    round trip, bit-identical to the host-scale path; a non-finite absmax
    yields the sentinel bits and zeros instead of a wrong scale."""
    dim, U = 100_003, 6
    g = make_units(23, U, dim)
    w = np.linspace(0.05, 0.3, U)
    units = [torch.from_numpy(x).cuda() for x in g]
    f_host = dev.fixed_point_bits(dev.weighted_absmax(units, w).item(), U)
    acc_h = torch.empty(dim, dtype=torch.int64, device="cuda")
    dev.weighted_fold(units, w, f_host, acc_h)
    want = dev.fixed_to_float(acc_h, f_host)
    amax = torch.empty(1, dtype=torch.float64, device="cuda")
    bits = torch.empty(1, dtype=torch.int32, device="cuda")
    acc = torch.empty(dim, dtype=torch.int64, device="cuda")
    out = torch.empty(dim, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        dev.weighted_absmax(units, w, out=amax, stream=s)
        dev.fixed_point_bits_async(amax, U, bits, stream=s)
        dev.weighted_fold_dev(units, w, bits, acc, stream=s)
        dev.fixed_to_float_dev(acc, bits, out, stream=s)
    for _ in range(2):
        out.fill_(-1.0)
        graph.replay()
    torch.cuda.synchronize()
    assert int(bits.item()) == f_host
    assert torch.equal(acc, acc_h) and torch.equal(out, want)
    units[2][7] = float("nan")
    graph.replay()
    torch.cuda.synchronize()
    assert int(bits.item()) == -2 ** 31 and int(out.count_nonzero()) == 0
