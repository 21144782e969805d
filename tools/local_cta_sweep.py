"""Reshard: how many CTAs should a GPU's LOCAL copies get while its HBM also
feeds peers' NVLink pulls?  (torchrun, N >= 2.)

tools/pair_probe.py: one pair pulls 788 GB/s through the staged copy kernel
when nothing else runs, but the 4->3 reshard's single-pair bottleneck lanes
reach ~700-712 GB/s: the source GPU's local copies (self lanes + retained
bytes, all CTAs, HBM-saturating for ~5 ms) compete with the peer's reads of
the same HBM.  For each departure position this times the verified pull
program with the local class limited to L CTAs (remote class fixed)."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import torch.distributed as dist

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    base = configs.llama2_7b()
    lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    block = 65536
    nblocks = (sum(lb) + block - 1) // block
    after = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    drops = [int(x) for x in os.environ.get("DROPS", "0,3").split(",")]
    for drop in drops:
        rp = ReshardPlan.build(lb, range(world), [r for r in range(world) if r != drop])
        bott = rp.traffic()["bottleneck_bytes"]
        ex = ReshardExecutor(rp, rank, push=False)
        bufs = ex.allocate()
        if bufs.old is not None:
            dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 0)
        if bufs.replica is not None:
            dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank)), bufs.replica, 0)
        ex.bind(bufs, verify=True)
        n_rem = 0
        if ex.program is not None:
            _, n_rem, n_loc = ex.program.stats()
        for rem, loc in ((sms // 2, 2 * sms - sms // 2), (sms // 2, sms), (sms // 2, 96),
                         (sms // 2, 64), (sms // 2, 32), (sms, 32), (sms, 64)):
            n = (rem if n_rem else 0) + loc
            ts = []
            for k in range(6):
                after.zero_()
                dist.barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                ex.launch(n, rem if n_rem else 0, block_sums=after)
                b.record()
                torch.cuda.synchronize()
                if k:
                    ts.append(a.elapsed_time(b) / 1e3)
            t = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rank == 0:
                print(json.dumps({"drop": drop, "remote_ctas": rem, "local_ctas": loc,
                                  "ms": round(t.item() * 1e3, 3),
                                  "bottleneck_GBps": round(bott / t.item() / 1e9, 1)}), flush=True)
        ex.close()
        del bufs
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
