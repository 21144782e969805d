"""Where does the 2->1 post-reshard verification time go?  One GPU, the
surviving rank's side: shard map, rows, checksum, rows_to_blocks."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.reshard import ReshardPlan, shard_map

lb = [x * 2 // 8 for x in configs.llama2_7b().layer_bytes]
rp = ReshardPlan.build(lb, [0, 1], [0])
n = rp.dst.shard_bytes(0)
buf = dev.empty_bytes(n)
block = 65536
nblocks = (sum(lb) + block - 1) // block
after = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
for rep in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    mn = shard_map(rp.dst, 0, block); t.append(time.perf_counter())
    rows = mn.new_row_sums(); torch.cuda.synchronize(); t.append(time.perf_counter())
    dev.checksum(mn, buf, rows); torch.cuda.synchronize(); t.append(time.perf_counter())
    dev.rows_to_blocks(mn, rows, after); torch.cuda.synchronize(); t.append(time.perf_counter())
    print({"shard_bytes": n, "rows": mn.num_rows, "segments": len(rp.dst.segments(0)),
           "map_ms": round((t[1]-t[0])*1e3, 3), "rows_alloc_ms": round((t[2]-t[1])*1e3, 3),
           "checksum_ms": round((t[3]-t[2])*1e3, 3), "rows_to_blocks_ms": round((t[4]-t[3])*1e3, 3)})
