"""Pin the oracle restatement (and the host C++ API) against golden vectors.

rng_golden.json carries the reference's own known-answer words and draws
(proj/tests/golden/rng_golden.json) plus reference-computed draws/masks;
checksum and reduce fixtures are the builder-defined (parity-unpinned) specs.
"""
import hashlib
import json

import numpy as np
import pytest

from paper_2510_00606_b200 import fabric


@pytest.fixture(scope="module")
def rng_golden(golden_dir):
    return json.loads((golden_dir / "rng_golden.json").read_text())


def test_oracle_philox_words_and_draws(oracle, rng_golden):
    dom = rng_golden["key_domain"]
    assert dom == 0x454C41534B495431
    for c in rng_golden["cases"]:
        lane = (c["layer"] << 32) | c["op"]
        assert oracle.philox4x64([1, c["sample"], lane, 0], [c["seed"], dom]) == c["words"]
        got = oracle.draw(c["seed"], c["sample"], c["layer"], c["op"], len(c["draws"]))
        assert got.tolist() == c["draws"]  # bit-exact doubles


def test_host_api_philox_words_and_draws(rng_golden):
    dom = rng_golden["key_domain"]
    for c in rng_golden["cases"]:
        lane = (c["layer"] << 32) | c["op"]
        assert fabric.philox4x64([1, c["sample"], lane, 0], [c["seed"], dom]) == c["words"]
        got = fabric.draw(c["seed"], c["sample"], c["layer"], c["op"], len(c["draws"]))
        assert got.tolist() == c["draws"]


def test_reference_computed_draws(oracle, rng_golden):
    for c in rng_golden["ref_draws"]:
        want = [float.fromhex(x) for x in c["draws_hex"]]
        assert oracle.draw(c["seed"], c["sample"], c["layer"], c["op"], len(want)).tolist() == want
        assert fabric.draw(c["seed"], c["sample"], c["layer"], c["op"], len(want)).tolist() == want


def test_reference_computed_masks(oracle, rng_golden):
    for m in rng_golden["ref_masks"]:
        got = oracle.dropout_mask(m["seed"], m["sample_lo"], m["n_samples"], m["layer"], m["op"],
                                  m["n_elems"], m["keep"])
        assert got.astype(np.int64).tolist() == m["bits"]


def test_draw_prefix_stability_and_range(oracle):
    a = oracle.draw(42, 7, 3, 1, 5)
    b = oracle.draw(42, 7, 3, 1, 16)
    assert a.tolist() == b[:5].tolist()
    v = oracle.draw(1, 2, 3, 4, 1000)
    assert (v >= 0).all() and (v < 1).all()


def test_checksum_golden(oracle, golden_dir):
    g = json.loads((golden_dir / "checksum_golden.json").read_text())
    for case in g["cases"]:
        buf = _fixture_buffer(case)  # the exact buffer the fixture was written from
        assert hashlib.sha256(buf.tobytes()).hexdigest() == case["buf_sha256"]
        rows = oracle.row_sums(case["segments"], case["block_bytes"], buf)
        assert [str(int(x)) for x in rows] == case["rows"]
    for seed, rows in g["synthetic_300007"].items():
        got = oracle.block_sums_synthetic(int(seed), 300_007, 65536)
        assert [str(int(x)) for x in got] == rows


def test_checksum_spec_reproduces_golden(golden_dir):
    """The golden rows come from oracle/checksum_spec.py, the pure-Python
    restatement of the ew_api.h spec (no code shared with the C oracle)."""
    from oracle import checksum_spec as cs
    g = json.loads((golden_dir / "checksum_golden.json").read_text())
    for case in g["cases"]:
        buf = _fixture_buffer(case).tobytes()
        assert [str(x) for x in cs.rows_of_buffer(case["segments"], case["block_bytes"],
                                                  buf)] == case["rows"]
    for seed, rows in g["synthetic_300007"].items():
        assert [str(x) for x in cs.synthetic_block_sums(int(seed), 300_007, 65536)] == rows
    sr = g["synthetic_rows"]
    for seed, rows in sr["rows"].items():
        assert [str(x) for x in cs.rows_of_synthetic(sr["segments"], sr["block_bytes"],
                                                     int(seed))] == rows


def test_c_oracle_synthetic_rows_match_spec_golden(oracle, golden_dir):
    """C oracle, two ways (fill + row_sums, and the buffer-free MT rows the
    full-size GPU tests check against) == the spec's golden rows."""
    sr = json.loads((golden_dir / "checksum_golden.json").read_text())["synthetic_rows"]
    total = sum(s["length"] for s in sr["segments"])
    for seed, rows in sr["rows"].items():
        buf = oracle.fill_synthetic(sr["segments"], total, int(seed))
        assert [str(int(x)) for x in oracle.row_sums(sr["segments"], sr["block_bytes"],
                                                     buf)] == rows
        for threads in (1, 3):
            got = oracle.rows_synthetic_mt(sr["segments"], sr["block_bytes"], int(seed), threads)
            assert [str(int(x)) for x in got] == rows


def test_c_oracle_mt_block_sums(oracle):
    for total in (1, 8, 4097, 300_007):
        for threads in (1, 4):
            assert np.array_equal(oracle.block_sums_synthetic_mt(9, total, 4096, threads),
                                  oracle.block_sums_synthetic(9, total, 4096))


def _fixture_buffer(case) -> np.ndarray:
    """Replays make_golden.checksum_golden's generator stream for one case."""
    rng = np.random.default_rng(2024)
    for block in (4096, 65536):
        local = 0
        for length in (5, 70001, 9, 131077):
            local += length
            rng.integers(1, 40000)
        buf = rng.integers(0, 256, size=local, dtype=np.uint8)
        if block == case["block_bytes"]:
            return buf
    raise AssertionError("unknown fixture case")


def test_checksum_is_linear_over_splits(oracle):
    """Splitting a segment anywhere (rows of several ranks) sums to the same
    block sums — the property reshard verification relies on."""
    rng = np.random.default_rng(3)
    total = 200_003
    seed = 11
    whole = oracle.block_sums_synthetic(seed, total, 4096)
    cuts = sorted(set(rng.integers(1, total, size=9).tolist()))
    bounds = [0] + cuts + [total]
    acc = np.zeros_like(whole)
    for lo, hi in zip(bounds[:-1], bounds[1:]):
        seg = [{"global_lo": lo, "length": hi - lo, "local_off": 0}]
        buf = oracle.fill_synthetic(seg, hi - lo, seed)
        rows = oracle.row_sums(seg, 4096, buf)
        b0 = lo // 4096
        acc[2 * b0:2 * b0 + len(rows)] += rows  # uint64 arrays wrap mod 2^64
    assert np.array_equal(acc, whole)


def test_reduce_golden(oracle, golden_dir):
    g = json.loads((golden_dir / "reduce_golden.json").read_text())
    rng = np.random.default_rng(g["seed"])
    grads = rng.normal(0, 1e-3, size=(5, 257)).astype(np.float32)
    grads[1, 17] = 1e2
    grads[3, 200] = -1e2
    w = np.asarray(g["weights"])
    amax = float(np.max(np.abs(w[:, None] * grads.astype(np.float64))))
    assert amax.hex() == g["absmax"]
    f = oracle.fixed_point_bits(amax, 5)
    assert f == g["frac_bits"]
    acc = oracle.weighted_fixed(w, grads, f)
    assert hashlib.sha256(acc.tobytes()).hexdigest() == g["acc_sha256"]
