"""(c) Philox-4x64-10 on the GPU: raw words vs the reference golden vectors,
uniforms vs draw(), packed dropout masks vs the reference rule — all
bit-exact, through the C ABI."""
import json

import numpy as np
import pytest
import torch

from paper_2510_00606_b200 import device as dev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rng_golden(golden_dir):
    return json.loads((golden_dir / "rng_golden.json").read_text())


def test_words_match_reference_golden(rng_golden):
    for c in rng_golden["cases"]:
        w = dev.philox_words(c["seed"], c["sample"], c["layer"], c["op"], 1, 1)
        got = w.cpu().numpy().view(np.uint64)[0].tolist()
        assert got == c["words"]


def test_uniforms_match_golden_draws(rng_golden):
    for c in rng_golden["cases"]:
        # the all-ones key included: sample ids span the full uint64 domain
        u = dev.philox_uniforms(c["seed"], c["sample"], 1, c["layer"], c["op"], len(c["draws"]))
        assert u.cpu().numpy()[0].tolist() == c["draws"]
    for c in rng_golden["ref_draws"]:
        want = [float.fromhex(x) for x in c["draws_hex"]]
        u = dev.philox_uniforms(c["seed"] % 2**64, c["sample"], 1, c["layer"], c["op"], len(want))
        assert u.cpu().numpy()[0].tolist() == want


def test_uniforms_match_oracle_many_samples(oracle):
    u = dev.philox_uniforms(2024, 1000, 16, 5, 2, 1001).cpu().numpy()
    for s in range(16):
        assert u[s].tolist() == oracle.draw(2024, 1000 + s, 5, 2, 1001).tolist()


def test_masks_match_reference_golden(rng_golden):
    for m in rng_golden["ref_masks"]:
        bits = dev.dropout_mask(m["seed"], m["sample_lo"], m["n_samples"], m["layer"], m["op"],
                                m["n_elems"], m["keep"])
        got = bits.cpu().numpy().view(np.uint32).astype(np.int64).tolist()
        assert got == m["bits"]


@pytest.mark.parametrize("keep", [0.5, 0.3, 0.9, 0.0, 1.0, 1e-9, 1 - 2**-53, float("nan")])
@pytest.mark.parametrize("n_elems", [1, 31, 32, 33, 257, 4096])
def test_masks_match_oracle_rule(oracle, keep, n_elems):
    seed, lo, ns = 2024, 77, 5
    bits = dev.dropout_mask(seed, lo, ns, 3, 1, n_elems, keep).cpu().numpy().view(np.uint32)
    want = oracle.dropout_mask(seed, lo, ns, 3, 1, n_elems, keep)
    assert np.array_equal(bits, want)


def test_masks_full_uint64_sample_domain(oracle):
    """Sample ids >= 2^63 and the wrap past 2^64 - 1 (reference RngKey::
    sample_id is uint64, rng.hpp:21-26; sample_lo + s wraps like its sum)."""
    for lo in (2**63 - 2, 2**63, 2**64 - 3):
        bits = dev.dropout_mask(11, lo, 5, 2, 1, 77, 0.5).cpu().numpy().view(np.uint32)
        assert np.array_equal(bits, oracle.dropout_mask(11, lo, 5, 2, 1, 77, 0.5))
        u = dev.philox_uniforms(11, lo, 5, 2, 1, 9).cpu().numpy()
        for s in range(5):
            assert u[s].tolist() == oracle.draw(11, (lo + s) % 2**64, 2, 1, 9).tolist()


def test_masks_are_layout_independent():
    """The masks a rank generates for its sample range equal the matching
    rows of the whole batch (DP 8 -> 5 reshape, config E shape, scaled K)."""
    k = 4096
    whole = dev.dropout_mask(0, 0, 64, 7, 0, k, 0.5)
    lo = 0
    for n in [14, 14, 12, 12, 12]:  # per-slot samples of a DP5 reshape
        part = dev.dropout_mask(0, lo, n, 7, 0, k, 0.5)
        assert torch.equal(part, whole[lo:lo + n])
        lo += n


def test_keep_fraction_is_plausible():
    bits = dev.dropout_mask(1, 0, 8, 0, 0, 1 << 16, 0.5)
    frac = bits.cpu().numpy().view(np.uint32)
    ones = np.unpackbits(frac.view(np.uint8)).mean()
    assert abs(ones - 0.5) < 0.01
