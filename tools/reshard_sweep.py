"""Reshard copy-kernel tuning sweep (run under torchrun, N >= 2 GPUs).

Times the N -> N-1 reshard program of a 7B-per-GPU state for several CTA
splits and push/pull, plus a pure rank0 -> rank1 peer copy of 4 GiB through
the same kernel and through the copy engines (cudaMemcpyAsync), and prints
one JSON line per measurement (rank 0)."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import torch.distributed as dist

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200._native import check, lib
from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map


def timed(fn, reps=5):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    dist.barrier()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1e3)
    t = torch.tensor([min(ts)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    emit = (lambda d: print(json.dumps(d), flush=True)) if rank == 0 else (lambda d: None)

    # pure peer copy rank0 -> rank1, 4 GiB
    n = 4 << 30
    src = torch.empty(n, dtype=torch.uint8, device="cuda")
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    h = [None] * world
    dist.all_gather_object(h, dev.ipc_handle(dst))
    peer = dev.ipc_open(*h[1 % world]) if rank == 0 else None
    for ctas in (148, 296, 592, 1184):
        if rank == 0:
            prog = dev.CopyProgram.from_pointers([src.data_ptr()], [peer], [n], [True])
            f = lambda: prog.launch(ctas, ctas)
        else:
            f = lambda: None
        t = timed(f)
        emit({"test": "p2p push kernel", "ctas": ctas, "GBps": round(n / t / 1e9, 1)})
    if rank == 0:
        f = lambda: check(lib.ew_memcpy_async(peer, src.data_ptr(), n,
                                              torch.cuda.current_stream().cuda_stream))
    else:
        f = lambda: None
    t = timed(f)
    emit({"test": "p2p copy engine (cudaMemcpyAsync)", "GBps": round(n / t / 1e9, 1)})
    # local copy through the kernel
    prog_l = dev.CopyProgram.from_pointers([src.data_ptr()], [dst.data_ptr()], [n], [False])
    t = timed(lambda: prog_l.launch(0, 0))
    emit({"test": "local copy kernel", "GBps_rw": round(2 * n / t / 1e9, 1)})
    if peer:
        dev.ipc_close(peer)
    del src, dst
    torch.cuda.empty_cache()

    base = configs.llama2_7b()
    lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    drop = min(3, world - 1)
    rp = ReshardPlan.build(lb, range(world), [r for r in range(world) if r != drop])
    bott = rp.traffic()["bottleneck_bytes"]
    for push in (True, False):
        ex = ReshardExecutor(rp, rank, push=push)
        bufs = ex.allocate()
        if bufs.old is not None:
            dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 0)
        if bufs.replica is not None:
            dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank)), bufs.replica, 0)
        ex.bind(bufs)
        for n_ctas, rem in ((0, 0), (148, 37), (148, 74), (296, 37), (296, 74), (296, 111),
                            (296, 148), (444, 74), (444, 148)):
            t = timed(lambda: ex.launch(n_ctas, rem))
            emit({"test": f"reshard {world}->{world-1} drop {drop}", "push": push, "ctas": n_ctas,
                  "remote_ctas": rem, "ms": round(t * 1e3, 3),
                  "bottleneck_GBps": round(bott / t / 1e9, 1)})
        ex.close()
        del bufs
        torch.cuda.empty_cache()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
