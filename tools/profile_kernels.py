"""Single-GPU driver that launches each hot-path kernel once at its config
size, for ncu captures (`ncu --set full -k regex:...`).  Prints per-kernel
CUDA-event times so the same command can run without ncu first.

  (a) warp_row_kernel<0> snapshot, <2> verify         7B rank shard 11.79 GB
  (b) staged_copy_kernel, local 4 GiB aligned + 1 GiB misaligned
  (c) mask_kernel, config E busiest rank (224 x 4096^2)
  (d) absmax_kernel, fold_kernel, dequant_kernel: one 7B fp32 gradient
      (6.74 G elements, config E's per-rank unit)
  §8(f)#1 adam_kernel, 7B rank shard (842 M params, 11.79 GB state)
  §8(f)#2 payback_kernel, one 7B layer (202 M int64), local source
  (b) staged_copy_kernel verified: 4->3 of 7B-per-GPU state, every rank's
      pull program on this GPU (peers emulated by local buffers)
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2510_00606_b200 import configs, device as dev, fabric


def timed(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e)


def main():
    torch.cuda.set_device(0)
    out = {}
    cfg = configs.llama2_7b()
    layout = fabric.interleaved_layout(cfg.layer_bytes, range(8))
    m = dev.ShardMap(layout.segments(3), 65536)
    n = layout.shard_bytes(3)
    live, snap = dev.empty_bytes(n), dev.empty_bytes(n)
    rows = m.new_row_sums()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.fill_synthetic(m, live, 0)
    dev.snapshot(m, live, snap, rows)
    out["snapshot_ms"] = timed(lambda: dev.snapshot(m, live, snap, rows))
    out["verify_ms"] = timed(lambda: dev.verify(m, snap, rows, bad))
    del live, snap
    torch.cuda.empty_cache()

    a = torch.empty(5 << 30, dtype=torch.uint8, device="cuda")
    b = torch.empty(5 << 30, dtype=torch.uint8, device="cuda")
    p = dev.CopyProgram.from_pointers([a.data_ptr(), a.data_ptr() + (4 << 30) + 3],
                                      [b.data_ptr(), b.data_ptr() + (4 << 30) + 8],
                                      [4 << 30, (1 << 30) - 16], [False, False])
    p.launch()
    out["staged_copy_ms"] = timed(lambda: p.launch())
    del a, b
    torch.cuda.empty_cache()

    bits = torch.empty((224, 4096 * 4096 // 32), dtype=torch.int32, device="cuda")
    out["mask_ms"] = timed(lambda: dev.dropout_mask(0, 0, 224, 1, 0, 4096 * 4096, 0.5, bits))
    del bits

    ng = 6_738_415_616
    g = torch.empty(ng, dtype=torch.float32, device="cuda").normal_(0, 1e-3)
    acc = torch.empty(ng, dtype=torch.int64, device="cuda")
    res = torch.empty(ng, dtype=torch.float32, device="cuda")
    out["absmax_ms"] = timed(lambda: dev.weighted_absmax([g], [0.2]))
    out["fold_ms"] = timed(lambda: dev.weighted_fold([g], [0.2], 54, acc))
    out["dequant_ms"] = timed(lambda: dev.fixed_to_float(acc, 54, res))
    out["absmax_gbs"] = 4 * ng / out["absmax_ms"] / 1e6
    out["fold_gbs"] = 12 * ng / out["fold_ms"] / 1e6
    out["dequant_gbs"] = 12 * ng / out["dequant_ms"] / 1e6
    del g, acc, res
    torch.cuda.empty_cache()

    n = 6_738_415_616 // 8
    st = dev.AdamState(n)
    grad = torch.empty(n, dtype=torch.float32, device="cuda").normal_(0, 1e-3)
    h = dev.adam_hyper()
    dev.adam_step(grad, st, h, 1)
    out["adam_ms"] = timed(lambda: dev.adam_step(grad, st, h, 2))
    del st, grad
    torch.cuda.empty_cache()

    from paper_2510_00606_b200.migration import payback_accumulate
    a = torch.zeros(202_383_360, dtype=torch.int64, device="cuda")
    b = torch.ones_like(a)
    payback_accumulate(a, b)
    out["payback_ms"] = timed(lambda: payback_accumulate(a, b))
    del a, b
    torch.cuda.empty_cache()

    from paper_2510_00606_b200.reshard import ReshardPlan, emulate_on_one_gpu
    lb = [x * 4 // 8 for x in configs.llama2_7b().layer_bytes]
    rp = ReshardPlan.build(lb, [0, 1, 2, 3], [0, 1, 2])
    nblocks = (sum(lb) + 65535) // 65536
    sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    emulate_on_one_gpu(rp, seed=1, push=False, block_sums=sums)
    t1.record()
    torch.cuda.synchronize()
    out["verified_reshard_emulation_ms"] = t0.elapsed_time(t1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
