"""Node-shared host memory as a reshard source (Medium::H2D_D2D), run under
torchrun with N >= 2 GPUs.

Rank 0 writes a device buffer's bytes into POSIX shared memory
(/dev/shm, via multiprocessing.shared_memory) and every rank pins the same
range (ew_host_register, portable + mapped).  Then each rank r >= 1, alone
and then all at once, pulls a 1/(N-1) share of it into its HBM with the
staged copy kernel reading the host pointer (TMA bulk loads over PCIe), and
checks the bytes.  Prints one JSON line per measurement on rank 0, plus the
box's /dev/shm and host memory sizes."""
import json
import os
import shutil
import sys
from multiprocessing import shared_memory
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import torch.distributed as dist

from paper_2510_00606_b200 import device as dev


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl")
    nbytes = int(float(os.environ.get("HOST_PROBE_GB", "4")) * (1 << 30))
    if rank == 0:
        du = shutil.disk_usage("/dev/shm")
        mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        print(json.dumps({"dev_shm_total_gb": round(du.total / 1e9, 1),
                          "dev_shm_free_gb": round(du.free / 1e9, 1),
                          "host_mem_gb": round(mem / 1e9, 1)}), flush=True)
    room = torch.tensor([shutil.disk_usage("/dev/shm").free], dtype=torch.float64, device="cuda")
    dist.broadcast(room, 0)
    if room.item() < 1.2 * nbytes:  # writing past /dev/shm's size would SIGBUS
        if rank == 0:
            print(json.dumps({"skipped": "/dev/shm too small"}), flush=True)
        dist.destroy_process_group()
        return
    name = f"ew_probe_{os.getppid()}"
    if rank == 0:
        shm = shared_memory.SharedMemory(name=name, create=True, size=nbytes)
    dist.barrier()
    if rank != 0:
        shm = shared_memory.SharedMemory(name=name)
    host = torch.frombuffer(shm.buf, dtype=torch.uint8)
    addr = host.data_ptr()
    dptr = dev.host_register(addr, nbytes)
    if rank == 0:
        src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device="cuda")
        host.copy_(src.cpu())
        del src
    dist.barrier()
    share = nbytes // max(1, world - 1) // 4096 * 4096
    out = torch.empty(share, dtype=torch.uint8, device="cuda")
    results = []
    lo = (rank - 1) * share if rank > 0 else 0
    prog = dev.CopyProgram.from_pointers([dptr + lo], [out.data_ptr()], [share], [True]) \
        if rank > 0 else None

    def timed(active):
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        if rank in active:
            prog.launch()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / 1e3 if rank in active else 0.0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for active, label in (([1], "one GPU pulls"), (list(range(1, world)), "all pull at once")):
        timed(active)  # warm
        t = min(timed(active) for _ in range(3))
        if rank == 0:
            print(json.dumps({"test": label, "gpus": len(active), "bytes_per_gpu": share,
                              "ms": round(t * 1e3, 2),
                              "gbs_per_gpu": round(share / t / 1e9, 1),
                              "gbs_total": round(len(active) * share / t / 1e9, 1)}), flush=True)
    ok = torch.tensor([1], device="cuda")
    if rank > 0:
        ok[0] = int(torch.equal(out.cpu(), host[lo:lo + share]))
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    if rank == 0:
        print(json.dumps({"bytes_identical": bool(ok.item())}), flush=True)
    del prog
    dist.barrier()
    dev.host_unregister(addr)
    del host
    shm.close()
    dist.barrier()
    if rank == 0:
        shm.unlink()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
