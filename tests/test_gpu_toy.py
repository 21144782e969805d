"""Toy consistency on the B200 path (paper_2510_00606_b200/toy.py): the
reference's end-to-end criterion for RNG resharding + scale-preserving
gradient reduction — an elastic run equals the static run bit for bit, and a
wrongly weighted gradient is caught (reference test_sim.cpp:136-158,
verify.cpp:55-78) — with the keep-bits from the Philox mask kernel, the
fold from ew_weighted_fold and int64 sums; checked against a numpy
restatement of the reference toy step (sim.cpp:895-953) whose uniforms come
from the reference library's own draw() when it is built (else the oracle)."""
import numpy as np
import pytest

from paper_2510_00606_b200.toy import ToyConfig, ToyRun

pytestmark = pytest.mark.gpu


def _reference_toy(cfg: ToyConfig, events, draw, reshape):
    """sim.cpp:895-953 restated: fp64, flat fold in ascending sample order."""
    L, K, B = cfg.layers, cfg.params_per_layer, cfg.global_batch
    params = np.array([[0.5 + 0.25 * l - 0.125 * k for k in range(K)] for l in range(L)])
    members, mbs = list(range(cfg.dp)), [cfg.microbatch_size] * cfg.dp
    n_mb = cfg.num_microbatches
    for step in range(cfg.steps):
        gone = events.get(step)
        if gone:
            idx = [members.index(m) for m in members if m not in gone]
            mbs = reshape(mbs, n_mb, idx)
            members = [m for m in members if m not in gone]
        base = step * B
        grad_sum = np.zeros((L, K))
        for mb in range(n_mb):
            cur = base + mb * sum(mbs)
            for m in mbs:
                for sample in range(cur, cur + m):
                    if sample >= base + B:
                        continue
                    for layer in range(1, L + 1):
                        u = draw(cfg.seed, sample, layer, 0, K)
                        for k in range(K):
                            mask = 0.0 if u[k] < cfg.keep_probability else 1.0 / cfg.keep_probability
                            g = float(((sample + 1) * (layer + 1) * (k + 1)) % 7 - 3) * mask
                            grad_sum[layer - 1][k] += g
                cur += m
        params -= cfg.learning_rate * (grad_sum * (1.0 / B))
    return params.reshape(-1)


@pytest.fixture(scope="module")
def ref_ops():
    from oracle.ew_oracle import load_oracle, load_reference
    ref = load_reference()
    orc = load_oracle()
    if ref is not None:
        def reshape(mbs, n_mb, idx):
            st, _, out = ref.reshard_microbatches(mbs, n_mb, idx)
            assert st == 0
            return out
        return ref.draw, reshape
    from paper_2510_00606_b200.fabric import reshard_microbatches
    return orc.draw, lambda mbs, n_mb, idx: reshard_microbatches(mbs, n_mb, idx)[1]


CASES = [
    ("toy preset, static", {}),
    ("8->7 inside step 1 (the reference's event)", {2: [0]}),
    ("8->5 (config E shape)", {1: [1, 4, 6]}),
    ("8->7->6", {1: [3], 3: [7]}),
]


@pytest.mark.parametrize("name,events", CASES, ids=[c[0] for c in CASES])
def test_elastic_equals_static_bit_for_bit(name, events, ref_ops):
    cfg = ToyConfig(steps=5)
    static = ToyRun(cfg).run().cpu().numpy()
    run = ToyRun(cfg, events)
    elastic = run.run().cpu().numpy()
    assert np.array_equal(elastic.view(np.uint64), static.view(np.uint64)), name
    # every step consumed its whole global batch exactly once
    for step, seen in enumerate(run.consumed):
        assert seen == list(range(step * cfg.global_batch, (step + 1) * cfg.global_batch))
    # and equals the reference toy step (fp64 flat fold) exactly
    draw, reshape = ref_ops
    want = _reference_toy(cfg, events, draw, reshape)
    assert np.array_equal(elastic.view(np.uint64), want.view(np.uint64))
    assert not np.array_equal(want, _reference_toy(ToyConfig(steps=0), {}, draw, reshape))


def test_injected_weight_bug_is_caught():
    cfg = ToyConfig(steps=4)
    static = ToyRun(cfg).run().cpu().numpy()
    bad = ToyRun(cfg, {2: [0]}, inject_wrong_weights=True).run().cpu().numpy()
    assert not np.array_equal(static, bad)


def test_other_keep_and_batch_shapes(ref_ops):
    # micro-batch size 2, 3 micro-batches, keep 0.75 (1/keep not dyadic: the
    # fold still makes every split identical; vs the fp64 reference within
    # the fixed-point tolerance)
    cfg = ToyConfig(microbatch_size=2, global_batch=48, keep_probability=0.75, steps=3)
    static = ToyRun(cfg).run().cpu().numpy()
    elastic = ToyRun(cfg, {1: [2, 5]}).run().cpu().numpy()
    assert np.array_equal(static.view(np.uint64), elastic.view(np.uint64))
    draw, reshape = ref_ops
    want = _reference_toy(cfg, {1: [2, 5]}, draw, reshape)
    np.testing.assert_allclose(elastic, want, rtol=0, atol=1e-6)
