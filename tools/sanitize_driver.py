"""Small single-GPU driver of every kernel for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per process)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2510_00606_b200 import configs, device as dev, fabric
from paper_2510_00606_b200.reshard import ReshardPlan, emulate_on_one_gpu, shard_map

torch.cuda.set_device(0)
# (a) odd-sized, misaligned segments
segs = np.zeros(3, dtype=fabric.SEGMENT_DTYPE)
segs[0] = (5, 70001, 0); segs[1] = (80000, 33, 70001); segs[2] = (90003, 131071, 70034)
m = dev.ShardMap(segs, 4096)
live = dev.empty_bytes(m.nbytes); live.random_(0, 256)
snap = dev.empty_bytes(m.nbytes)
rows = m.new_row_sums()
bad = torch.zeros(1, dtype=torch.int32, device="cuda")
dev.snapshot(m, live, snap, rows)
dev.verify(m, snap, rows, bad)
dev.checksum(m, snap, rows)
# (b) reshard with byte-granular, mutually misaligned copies
cfg = configs.scaled(configs.llama2_7b_per_tensor(), 2e-5)
for push in (False, True):
    got, exp = emulate_on_one_gpu(ReshardPlan.build(cfg.layer_bytes, range(4), [0, 1, 3]), 1, push=push)
# (c) masks, (d) fold
dev.dropout_mask(0, 0, 3, 1, 0, 1000, 0.5)
g = torch.randn(4099, device="cuda")
acc = torch.empty(4099, dtype=torch.int64, device="cuda")
dev.weighted_fold([g], [0.5], 40, acc)
torch.cuda.synchronize()
print("sanitize driver done", int(bad.item()))
