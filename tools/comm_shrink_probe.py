"""Time the DP communicator lifecycle on N GPUs (torchrun): init, first
collective, ncclCommShrink of the last rank (planned departure, shrinkShare),
first and steady collectives on the shrunk communicator."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import torch.distributed as dist

from paper_2510_00606_b200 import device as dev


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [dev.Communicator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    t = {}
    dist.barrier()
    t0 = time.perf_counter()
    comm = dev.Communicator.init(uid[0], world, rank)
    t["init_s"] = time.perf_counter() - t0
    x = torch.ones(1 << 20, dtype=torch.int64, device="cuda")
    t0 = time.perf_counter()
    comm.allreduce_i64(x)
    torch.cuda.synchronize()
    t["first_allreduce_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(10):
        comm.allreduce_i64(x)
    torch.cuda.synchronize()
    t["steady_allreduce_8MB_s"] = (time.perf_counter() - t0) / 10
    dist.barrier()
    if rank != world - 1:
        t0 = time.perf_counter()
        shr = comm.shrink([world - 1])
        torch.cuda.synchronize()
        t["shrink_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        shr.allreduce_i64(x)
        torch.cuda.synchronize()
        t["shrunk_first_allreduce_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        for _ in range(10):
            shr.allreduce_i64(x)
        torch.cuda.synchronize()
        t["shrunk_steady_allreduce_8MB_s"] = (time.perf_counter() - t0) / 10
        shr.destroy()
    dist.barrier()
    comm.destroy()
    out = [None] * world
    dist.all_gather_object(out, t)
    if rank == 0:
        print(json.dumps({"world": world, "env": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")},
                          "per_rank": out}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
