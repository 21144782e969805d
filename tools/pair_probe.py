"""Single (source, destination) pair over NVLink: SM copy kernel vs copy
engines vs both at once (run under torchrun, N = 2).

The 8->7 reshard's bottleneck is usually ONE pair (e.g. drop r0: r7 -> r1
11.79 GB; drop r7: r6 -> r5 10.11 GB), and a single pair through the staged
copy kernel plateaus near 700-720 GB/s while several pairs sharing a GPU's
link reach ~784.  This probe times, for rank 1 pulling N bytes from rank 0:
  kernel pull (staged_copy_kernel, remote CTAs only), several CTA counts;
  copy engine pull (cudaMemcpyAsync peer -> local), one or two streams;
  a split: fraction f through the copy engine on a side stream while the
  kernel pulls the rest.
One JSON line per measurement on rank 0."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch
import torch.distributed as dist

from paper_2510_00606_b200 import device as dev
from paper_2510_00606_b200._native import check, lib


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = int(float(os.environ.get("PAIR_BYTES", 8e9))) // 4096 * 4096
    src = torch.empty(n, dtype=torch.uint8, device="cuda")
    dst = torch.empty(n, dtype=torch.uint8, device="cuda")
    src.fill_(rank + 1)
    h = [None] * world
    dist.all_gather_object(h, dev.ipc_handle(src))
    peer = dev.ipc_open(*h[0]) if rank == 1 else None
    side = torch.cuda.Stream()
    main_s = torch.cuda.current_stream()
    res = []

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            torch.cuda.synchronize()
            a.record(main_s)
            fn()
            b.record(main_s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / 1e3)
        t = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def emit(d):
        if rank == 0:
            print(json.dumps(d), flush=True)

    def ce(dst_ptr, src_ptr, nbytes, stream):
        check(lib.ew_memcpy_async(dst_ptr, src_ptr, nbytes, stream.cuda_stream))

    progs = {}

    def kernel_prog(lo, hi):
        key = (lo, hi)
        if key not in progs:
            progs[key] = dev.CopyProgram.from_pointers([peer + lo], [dst.data_ptr() + lo],
                                                       [hi - lo], [True])
        return progs[key]

    for ctas in (74, 148, 296, 444):
        if rank == 1:
            p = kernel_prog(0, n)
            f = lambda: p.launch(ctas, ctas)
        else:
            f = lambda: None
        t = timed(f)
        emit({"test": "kernel pull", "ctas": ctas, "GBps": round(n / t / 1e9, 1)})

    # misaligned source (realign path) and verification on arrival
    from paper_2510_00606_b200.fabric import SEGMENT_DTYPE, ROLE_NEW, ROLE_OLD
    from paper_2510_00606_b200.fabric import COPY_DTYPE
    m = n - 4096
    seg = np.zeros(1, dtype=SEGMENT_DTYPE)
    seg[0] = (0, m, 0)
    vmap = dev.ShardMap(seg, 65536)
    sums = torch.zeros(2 * ((m + 65535) // 65536), dtype=torch.int64, device="cuda")
    for shift, verify in ((0, False), (8, False), (3, False), (0, True), (8, True)):
        if rank == 1:
            d = np.zeros(1, dtype=COPY_DTYPE)
            d[0] = (ROLE_OLD, 0, ROLE_NEW, 1, shift, 0, m)
            tbl = {(ROLE_OLD, 0): peer, (ROLE_NEW, 1): dst.data_ptr()}
            p = dev.CopyProgram.from_descs(d, tbl, 2, 1, vmap if verify else None)
            f = (lambda: p.launch(block_sums=sums)) if verify else (lambda: p.launch())
        else:
            f = lambda: None
        t = timed(f)
        emit({"test": "kernel pull (descriptor)", "src_shift": shift, "verified": verify,
              "GBps": round(m / t / 1e9, 1)})

    for streams in (1, 2, 4):
        ss = [main_s] + [torch.cuda.Stream() for _ in range(streams - 1)]

        def f():
            if rank != 1:
                return
            ev = torch.cuda.Event()
            ev.record(main_s)
            for i, s in enumerate(ss):
                s.wait_event(ev)
                lo, hi = n * i // streams, n * (i + 1) // streams
                ce(dst.data_ptr() + lo, peer + lo, hi - lo, s)
            for s in ss[1:]:
                e = torch.cuda.Event()
                e.record(s)
                main_s.wait_event(e)
        t = timed(f)
        emit({"test": "copy engine pull", "streams": streams, "GBps": round(n / t / 1e9, 1)})

    for frac in (0.25, 0.5, 0.75):
        cut = int(n * frac) // 4096 * 4096
        for ctas in (148, 296):
            if rank == 1:
                p = kernel_prog(cut, n)

                def f():
                    ev = torch.cuda.Event()
                    ev.record(main_s)
                    side.wait_event(ev)
                    ce(dst.data_ptr(), peer, cut, side)
                    p.launch(ctas, ctas)
                    e = torch.cuda.Event()
                    e.record(side)
                    main_s.wait_event(e)
            else:
                f = lambda: None
            t = timed(f)
            emit({"test": "copy engine + kernel split", "ce_fraction": frac, "ctas": ctas,
                  "GBps": round(n / t / 1e9, 1)})

    # correctness of the last split
    if rank == 1:
        torch.cuda.synchronize()
        ok = bool((dst == 1).all().item())
        print(json.dumps({"test": "landed bytes", "ok": ok}), flush=True)
    progs.clear()
    if peer:
        dev.ipc_close(peer)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
