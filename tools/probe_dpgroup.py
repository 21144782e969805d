"""4-GPU probe of the C++ DP group (torchrun): NCCL init, prepared comm
splits (unshared, then shared), prepared recovery + DpGroup.recover on a
small state, every stage logged with a timestamp so a hang is located.

  torchrun --nproc-per-node 4 tools/probe_dpgroup.py [--share]
"""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import torch.distributed as dist

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.recovery import DpGroup, PreparedRecovery
from paper_2510_00606_b200.reshard import ReshardPlan, shard_map

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
T0 = time.time()


def log(msg):
    print(f"[{time.time() - T0:7.2f}s r{rank}] {msg}", file=sys.stderr, flush=True)


share = "--share" in sys.argv
cfg = configs.scaled(configs.llama2_7b(), 1e-2)
members = list(range(world))
lay = ReshardPlan.build(cfg.layer_bytes, members, members).src
live = dev.empty_bytes(lay.shard_bytes(rank))
dev.fill_synthetic(shard_map(lay, rank), live, 3)
succ = (rank + 1) % world
rep = dev.empty_bytes(lay.shard_bytes(succ))
dev.fill_synthetic(shard_map(lay, succ), rep, 3)
torch.cuda.synchronize()
uid = [dev.Communicator.unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
comm = dev.Communicator.init(uid[0], world, rank)
comm.allreduce_i64(torch.zeros(8, dtype=torch.int64, device="cuda"))
torch.cuda.synchronize()
log("comm ready")
grp = DpGroup(cfg.layer_bytes, members, rank, comm, share_comm_resources=share)
log(f"DpGroup prepared (share={share})")
prep = PreparedRecovery(cfg.layer_bytes, members, rank, live, rep)
grp.attach(prep)
log("PreparedRecovery ready")
drop = world - 1
dist.barrier()
if rank != drop:
    ev = grp.recover([drop])
    log(f"recovered: verified={ev.verified} comm_repair={ev.comm_repair_s * 1e3:.3f} ms "
        f"remap={ev.remap_s * 1e3:.3f} ms phases={ev.phases}")
    c = grp.comm
    t = torch.ones(4, dtype=torch.int64, device="cuda")
    c.allreduce_i64(t)
    torch.cuda.synchronize()
    log(f"allreduce on the repaired comm: {t.tolist()} (size {c.size})")
dist.barrier()
log("closing")
prep.close()
grp.close()
log("closed")
dist.barrier()
dist.destroy_process_group()
