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
# round-2 kernels: bit-pattern absmax (aligned + misaligned units, > 16
# units), vectorised dequant (fp32/fp64, ragged tails), guarded copy,
# conservation verifier, AdamW replay with fused rows, in-place emulation
units = [torch.randn(4102, device="cuda")[k % 3:k % 3 + 4099] for k in range(18)]
dev.weighted_absmax(units, [0.1] * 18)
for n in (1, 7, 4099):
    dev.fixed_to_float(acc[:n], 40)
    dev.fixed_to_double(acc[1:n + 1] if n + 1 <= 4099 else acc[:n], 40)
flag = torch.ones(1, dtype=torch.int32, device="cuda")
src = dev.empty_bytes(10000); src.random_(0, 256); dst = dev.empty_bytes(10000)
prog = dev.CopyProgram.from_pointers([src.data_ptr() + 3], [dst.data_ptr() + 5], [9990], [False])
prog.launch(abort_flag=flag.data_ptr()); flag.zero_(); prog.launch(abort_flag=flag.data_ptr())
import ctypes as C
from paper_2510_00606_b200._native import check, lib
a = torch.randint(0, 2**62, (64,), dtype=torch.int64, device="cuda")
b = a.clone()
arr = (C.c_void_p * 1)(a.data_ptr())
brr = (C.c_void_p * 1)(b.data_ptr())
v = C.c_void_p()
check(lib.ew_block_verifier_create(arr, 1, brr, 1, 0, 64, C.byref(v)))
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
check(lib.ew_block_verifier_run(v, C.c_void_p(cnt.data_ptr()), dev._stream()))
st = dev.AdamState(3001)
st.master.normal_(0, 0.02)
am = dev.ShardMap(st.segments(), 4096)
ar = am.new_row_sums()
dev.adam_step(torch.randn(3001, device="cuda"), st, dev.adam_hyper(), 1, rows=ar, block_bytes=4096)
from paper_2510_00606_b200.inplace import emulate_inplace_on_one_gpu
rp = ReshardPlan.build(cfg.layer_bytes, range(4), [0, 1, 3])
sums = torch.zeros(2 * ((sum(cfg.layer_bytes) + 65535) // 65536), dtype=torch.int64, device="cuda")
emulate_inplace_on_one_gpu(rp, 0, 1 << 12, 1 << 13, 1, sums)
torch.cuda.synchronize()
lib.ew_block_verifier_free(v)
assert int(cnt.item()) == 0
print("sanitize driver done", int(bad.item()))
