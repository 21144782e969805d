"""Ring replica by optimizer replay: pin the oracle's AdamW
restatement (oracle/ew_oracle.c, ew_oracle_adam_step) against
torch.optim.AdamW — the reference only models the replay's time
(param_fabric.hpp:86-96), the paper names the update —
and check that the product's host-side scalar derivation (ew_adam_scalars,
no GPU needed) matches the oracle's bit for bit.

Tolerance vs torch (fp32, different but equivalent op order: torch uses
lerp for m, divides by sqrt(bc2) instead of multiplying by its inverse):
    |p_oracle - p_torch| <= 4 ulp(p) + 2^-20 * lr,
    |m_oracle - m_torch| <= 1e-5 * (|b1 m| + |(1-b1) g| + |m|)   (m may cancel),
    v within rtol 1e-6 (no cancellation)."""
import numpy as np
import pytest
import torch

from paper_2510_00606_b200 import device as dev

HYPERS = [(1e-3, 0.9, 0.999, 1e-8, 0.01), (3e-4, 0.8, 0.95, 1e-6, 0.0),
          (1e-2, 0.0, 0.5, 1e-3, 0.1)]


@pytest.mark.parametrize("hyper", HYPERS)
def test_scalars_match_product(oracle, hyper):
    for step in (1, 2, 7, 1000, 123456):
        got = dev.adam_scalars(dev.adam_hyper(*hyper), step)
        assert np.array_equal(got.view(np.uint32), oracle.adam_scalars(hyper, step).view(np.uint32))


def test_scalars_reject_bad_arguments():
    with pytest.raises(ValueError):
        dev.adam_scalars(dev.adam_hyper(), 0)
    with pytest.raises(ValueError):
        dev.adam_scalars(dev.adam_hyper(beta1=1.0), 1)


@pytest.mark.parametrize("hyper", HYPERS)
def test_oracle_matches_torch_adamw(oracle, hyper):
    lr, b1, b2, eps, wd = hyper
    n = 10_007
    rng = np.random.default_rng(3)
    p0 = rng.normal(0, 0.02, n).astype(np.float32)
    master, m, v = p0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    param = np.zeros(n, np.uint16)
    tp = torch.nn.Parameter(torch.from_numpy(p0.copy()))
    opt = torch.optim.AdamW([tp], lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd,
                            foreach=False)
    for step in range(1, 6):
        g = rng.normal(0, 1e-3, n).astype(np.float32)
        g[::97] *= 1e3
        # m may cancel (b1*m vs (1-b1)*g): bound its error by the terms' size
        m_scale = np.abs(b1 * m) + np.abs((1 - b1) * g)
        oracle.adam_step(g, master, m, v, param, hyper, step)
        tp.grad = torch.from_numpy(g.copy())
        opt.step()
        ref = tp.detach().numpy()
        tol = 4 * np.spacing(np.abs(ref)) + lr * 2.0 ** -20
        assert np.all(np.abs(master - ref) <= tol), step
        st = opt.state[tp]
        m_ref = st["exp_avg"].numpy()
        assert np.all(np.abs(m - m_ref) <= 1e-5 * (m_scale + np.abs(m_ref))), step
        np.testing.assert_allclose(v, st["exp_avg_sq"].numpy(), rtol=1e-6, atol=1e-18)
    # bf16 parameter copy = RNE of the fp32 master (torch's own conversion)
    want = torch.from_numpy(master).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(param, want)


def test_oracle_bf16_rounding(oracle):
    lib = oracle.lib
    import ctypes as C
    lib.ew_oracle_bf16.restype = C.c_uint16
    lib.ew_oracle_bf16.argtypes = [C.c_float]
    xs = np.array([0.0, -0.0, 1.0, 1.00390625, 1.01171875, 3.4e38, np.inf, -np.inf, 1e-40,
                   np.float32(1.0) + np.float32(2 ** -8)], dtype=np.float32)
    want = torch.from_numpy(xs).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = np.array([lib.ew_oracle_bf16(float(x)) for x in xs], dtype=np.uint16)
    assert np.array_equal(got, want)
    assert lib.ew_oracle_bf16(float("nan")) == 0x7FC0
