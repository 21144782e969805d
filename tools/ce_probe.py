"""Reshard remote lanes through the copy engines (torchrun, N >= 2).

tools/reshard_breakdown.py: the bottleneck rank's remote pulls run at ~750
GB/s through the staged copy kernel even alone, while one clean pair pulls
827 GB/s through the copy engines (tools/pair_probe.py).  Here every rank
issues its remote descriptors as cudaMemcpyAsync (peer -> local NEW) on a
side stream, optionally in K chunks each followed by a checksum-only pass of
the landed bytes (the verified program with src == dst: reads NEW, adds the
block sums, writes nothing), while the local copies run through the kernel;
block-sum conservation checks every landed byte."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch
import torch.distributed as dist

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200._native import check, lib
from paper_2510_00606_b200.fabric import ROLE_NEW, ROLE_OLD, ROLE_REPLICA
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
    before = torch.zeros_like(after)
    drops = [int(x) for x in os.environ.get("DROPS", "0,3").split(",")]
    side = torch.cuda.Stream()
    main_s = torch.cuda.current_stream()

    for drop in drops:
        rp = ReshardPlan.build(lb, range(world), [r for r in range(world) if r != drop])
        ex = ReshardExecutor(rp, rank, push=False)
        bufs = ex.allocate()
        before.zero_()
        if bufs.old is not None:
            mo = shard_map(rp.src, rank, block)
            dev.fill_synthetic(mo, bufs.old, 0)
            rows = mo.new_row_sums()
            dev.checksum(mo, bufs.old, rows)
            dev.rows_to_blocks(mo, rows, before)
        if bufs.replica is not None:
            dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank)), bufs.replica, 0)
        dist.all_reduce(before)
        ex.bind(bufs, verify=True)
        table = dict(ex._table)
        nt = max(world, max(rp.old_ranks) + 1)
        descs = rp.copies(rank, push=False)
        remote = descs[descs["src_rank"] != rank]
        loc = descs[descs["src_rank"] == rank]
        vmap = shard_map(rp.dst, rank, block) if bufs.new is not None else None
        local_prog = dev.CopyProgram.from_descs(loc, table, nt, rank, vmap) \
            if len(loc) and vmap is not None else None
        new_ptr = bufs.new.data_ptr() if bufs.new is not None else 0

        def chunks(k):
            """split the remote bytes into k chunks of ~equal size, in order"""
            total = int(remote["bytes"].sum())
            cuts = [total * i // k for i in range(k + 1)]
            out = [[] for _ in range(k)]
            pos = 0
            for c in remote:
                n, so, do = int(c["bytes"]), int(c["src_off"]), int(c["dst_off"])
                src = table[(int(c["src_role"]), int(c["src_rank"]))]
                while n > 0:
                    i = min(k - 1, int(np.searchsorted(cuts, pos, side="right") - 1))
                    take = min(n, cuts[i + 1] - pos) if cuts[i + 1] > pos else n
                    out[i].append((src + so, do, take))
                    so += take
                    do += take
                    pos += take
                    n -= take
            return out

        for K in (1, 4, 8, 16):
            ch = chunks(K) if len(remote) else []
            vprogs = []
            for part in ch:
                d = np.zeros(len(part), dtype=remote.dtype)
                for j, (_, do, n) in enumerate(part):
                    d[j] = (ROLE_NEW, rank, ROLE_NEW, rank, do, do, n)
                vprogs.append(dev.CopyProgram.from_descs(d, {(ROLE_NEW, rank): new_ptr}, nt, rank,
                                                         vmap))

            def run():
                ev0 = torch.cuda.Event()
                ev0.record(main_s)
                side.wait_event(ev0)
                evs = []
                for part in ch:
                    for src, do, n in part:
                        check(lib.ew_memcpy_async(new_ptr + do, src, n, side.cuda_stream))
                    e = torch.cuda.Event()
                    e.record(side)
                    evs.append(e)
                if local_prog is not None:
                    local_prog.launch(block_sums=after)
                for e, vp in zip(evs, vprogs):
                    main_s.wait_event(e)
                    vp.launch(block_sums=after)

            ts = []
            for k in range(5):
                after.zero_()
                dist.barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(main_s)
                run()
                b.record(main_s)
                torch.cuda.synchronize()
                if k:
                    ts.append(a.elapsed_time(b))
            dist.all_reduce(after)
            ok = bool(torch.equal(before, after))
            t = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device="cuda")
            allt = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(allt, t)
            # and the kernel-only verified program for comparison
            if rank == 0:
                print(json.dumps({"drop": drop, "mode": "CE remote + kernel local", "chunks": K,
                                  "verified": ok,
                                  "per_rank_ms": [round(x.item(), 3) for x in allt]}), flush=True)
        ts = []
        for k in range(5):
            after.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            ex.launch(block_sums=after)
            b.record(main_s)
            torch.cuda.synchronize()
            if k:
                ts.append(a.elapsed_time(b))
        dist.all_reduce(after)
        t = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device="cuda")
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        if rank == 0:
            print(json.dumps({"drop": drop, "mode": "kernel (verified)",
                              "verified": bool(torch.equal(before, after)),
                              "per_rank_ms": [round(x.item(), 3) for x in allt]}), flush=True)
        ex.close()
        del bufs
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
