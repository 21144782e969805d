"""Who bounds a reshard?  (torchrun, N >= 2.)  For each departure position,
time every rank's verified pull program (a) with all ranks running, (b) alone,
and its (c) local-only and (d) remote-only halves alone, per rank, so the
bottleneck (NVLink lane vs a GPU's local self-lane/retained copies) is
measured rather than inferred."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch
import torch.distributed as dist

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.fabric import ROLE_NEW
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
    drops = [int(x) for x in os.environ.get("DROPS", "0,3").split(",")]
    n_ctas = int(os.environ.get("CTAS", "0"))
    rem_ctas = int(os.environ.get("REM_CTAS", "0"))

    def timed(fn, who):
        ts = []
        for k in range(5):
            after.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if who is None or who == rank:
                fn()
            b.record()
            torch.cuda.synchronize()
            if k:
                ts.append(a.elapsed_time(b))
        t = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device="cuda")
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        return [round(x.item(), 3) for x in allt]

    for drop in drops:
        rp = ReshardPlan.build(lb, range(world), [r for r in range(world) if r != drop])
        ex = ReshardExecutor(rp, rank, push=False)
        bufs = ex.allocate()
        if bufs.old is not None:
            dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 0)
        if bufs.replica is not None:
            dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank)), bufs.replica, 0)
        ex.bind(bufs, verify=True)
        descs = rp.copies(rank, push=False)
        remote = (descs["src_rank"] != rank)
        table = dict(ex._table)
        nt = max(world, max(rp.old_ranks) + 1)
        vmap = shard_map(rp.dst, rank, block) if bufs.new is not None else None
        parts = {}
        for name, sel in (("local", ~remote), ("remote", remote)):
            d = descs[sel]
            parts[name] = dev.CopyProgram.from_descs(d, table, nt, rank, vmap) \
                if len(d) and vmap is not None else None
        stats = {"rank": rank,
                 "remote_bytes": int(descs["bytes"][remote].sum()),
                 "local_bytes": int(descs["bytes"][~remote].sum())}
        st = [None] * world
        dist.all_gather_object(st, stats)
        res = {"drop": drop, "stats": st}
        res["all_ranks_ms"] = timed(lambda: ex.launch(n_ctas, rem_ctas, block_sums=after), None)
        for who in rp.new_ranks:
            res[f"alone_r{who}_ms"] = timed(lambda: ex.launch(n_ctas, rem_ctas, block_sums=after),
                                           who)[who]
            for name, p in parts.items():
                pp = p
                res[f"alone_r{who}_{name}_ms"] = timed(
                    (lambda: pp.launch(n_ctas, rem_ctas, block_sums=after)) if pp is not None
                    else (lambda: None), who)[who]
        if rank == 0:
            print(json.dumps(res), flush=True)
        ex.close()
        parts.clear()
        del bufs
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
