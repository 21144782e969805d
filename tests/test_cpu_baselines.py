"""The multi-threaded CPU paths bench.py times beside the GPU kernels
 compute exactly what the reference computes: T-thread
draw() equals the reference's draw per sample, the element-parallel
weighted_grad_average equals the reference's fp64 fold bit for bit, and the
plan executor moves every entry's bytes."""
import numpy as np
import pytest

from paper_2510_00606_b200 import configs, fabric


def test_draw_mt_equals_reference(oracle, reference):
    d = oracle.draw_mt(2024, 77, 5, 3, 1, 1001, 3)
    for i in range(5):
        assert np.array_equal(d[i], reference.draw(2024, 77 + i, 3, 1, 1001))


@pytest.mark.parametrize("threads", [1, 4, 7])
def test_weighted_average_mt_bitwise(oracle, reference, threads):
    g = np.random.default_rng(threads).normal(size=(6, 10_007))
    w = np.random.default_rng(9).random(6)
    assert np.array_equal(oracle.weighted_average_mt(w, g, threads),
                          reference.weighted_grad_average(w, g))


def test_plan_executor_mt_moves_every_entry(oracle):
    cfg = configs.scaled(configs.gpt_125m(), 1e-3)
    src = fabric.interleaved_layout(cfg.layer_bytes, range(4))
    dst = fabric.interleaved_layout(cfg.layer_bytes, [0, 2, 3])
    plan = fabric.overlap_matrix(src, dst, [1], fabric.SnapshotRing([0, 1, 2, 3]))
    total = cfg.total_bytes
    state = np.random.default_rng(3).integers(0, 256, total, dtype=np.uint8)
    out = np.zeros(total, dtype=np.uint8)
    entries = plan.entries
    srcs = [state.ctypes.data + int(e["lo"]) for e in entries]
    dsts = [out.ctypes.data + int(e["lo"]) for e in entries]
    n = [int(e["hi"] - e["lo"]) for e in entries]
    oracle.memcpy_mt(srcs, dsts, n, 4)
    moved = np.zeros(total, dtype=bool)
    for e in entries:
        moved[int(e["lo"]):int(e["hi"])] = True
    assert np.array_equal(out[moved], state[moved]) and moved.any()


def test_reference_arm_workload_matches_gpu_arm(reference):
    """bench.py's reference arm restates config B's layer sizes (it must not
    import the product package); they, the per-tensor variant, and the
    reference library's interleaved rank-0 shard equal the GPU arm's."""
    import importlib.util
    from pathlib import Path
    spec = importlib.util.spec_from_file_location(
        "bench_mod", Path(__file__).resolve().parents[1] / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    assert bench.LLAMA2_7B_LAYER_BYTES == configs.llama2_7b().layer_bytes
    assert bench._llama2_7b_per_tensor_layer_bytes() == \
        configs.llama2_7b_per_tensor().layer_bytes
    r = bench.HEADLINE_SHARD_RANK
    lay = fabric.interleaved_layout(configs.llama2_7b().layer_bytes, range(8))
    ref_ivs = reference.interleaved(bench.LLAMA2_7B_LAYER_BYTES, range(8))[r]
    segs = lay.segments(r)
    assert [(int(s["global_lo"]), int(s["global_lo"] + s["length"])) for s in segs] == \
        [(int(a), int(b)) for a, b in ref_ivs]
    assert bench.workload_config(lay.shard_bytes(r), 65536, 1) == \
        bench.workload_config(sum(b - a for a, b in ref_ivs), 65536, 1)
