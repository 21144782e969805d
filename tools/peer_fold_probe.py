"""Phase timing of the peer-memory weighted reduce (torchrun, N GPUs)."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import torch.distributed as dist
from paper_2510_00606_b200 import device as dev


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    n = int(os.environ.get("N_ELEMS", 1 << 30))
    units = [torch.empty(n, dtype=torch.float32, device="cuda").normal_(0, 1e-3)
             for _ in range(int(os.environ.get("UNITS", 1)))]
    w = [0.1] * len(units)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    fold, total, opened = dev.peer_weighted_reduce_setup(units, w, out)
    bar = dev.PeerBarrier()
    res = {}
    for rep in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        dist.barrier()
        ev[0].record(); bar.wait(); ev[1].record()
        fold.reduce_scatter(60); ev[2].record()
        bar.wait(); ev[3].record()
        fold.all_gather(); ev[4].record()
        bar.wait()
        torch.cuda.synchronize()
        res = {"barrier1_ms": ev[0].elapsed_time(ev[1]), "rs_ms": ev[1].elapsed_time(ev[2]),
               "barrier2_ms": ev[2].elapsed_time(ev[3]), "ag_ms": ev[3].elapsed_time(ev[4])}
    rs_bytes = (world - 1) / world * n * 4 * len(units)
    ag_bytes = (world - 1) / world * n * 4
    res["rs_gbs"] = rs_bytes / res["rs_ms"] / 1e6
    res["ag_gbs"] = ag_bytes / res["ag_ms"] / 1e6
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        print(json.dumps({"world": world, "n": n, "units_per_rank": len(units), "per_rank": allr}))
    bar.wait(); torch.cuda.synchronize(); dist.barrier()
    bar.close()
    for p in opened:
        dev.ipc_close(p)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
