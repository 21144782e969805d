"""Heartbeat detector under load (tools only): one process per GPU, each
running snapshot + verify of a 7B rank shard back to back (HBM at ~6.5 TB/s)
while its C++ FailureDetector beats; for several (period, timeout) settings
it records the largest heartbeat silence any member saw and whether any
member was ever (falsely) failed.

  python -m torch.distributed.run --nproc-per-node N tools/detector_probe.py
"""
import json
import os
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import torch.distributed as dist

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.recovery import FailureDetector
from paper_2510_00606_b200.reshard import ReshardPlan, shard_map


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo")
    cfg = configs.llama2_7b()
    lay = ReshardPlan.build(cfg.layer_bytes, list(range(8)), list(range(8))).src
    m = shard_map(lay, rank % 8)
    live = dev.empty_bytes(m.nbytes)
    dev.fill_synthetic(m, live, 0)
    snap = dev.empty_bytes(m.nbytes)
    rows = m.new_row_sums()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = {}
    for period, timeout in ((1e-3, 20e-3), (0.5e-3, 5e-3), (0.25e-3, 2e-3)):
        det = FailureDetector(f"probe{int(period * 1e6)}", period, timeout)
        dist.barrier()
        stop = threading.Event()
        worst = {"false_failures": 0, "polls": 0}

        def watch():
            while not stop.is_set():
                f = det.failed()
                worst["polls"] += 1
                if f:
                    worst["false_failures"] += 1
                time.sleep(period / 2)

        th = threading.Thread(target=watch)
        th.start()
        t0, steps = time.time(), 0
        while time.time() - t0 < 5.0:   # the GPU busy with the hot path
            dev.snapshot(m, live, snap, rows)
            dev.verify(m, snap, rows, bad)
            steps += 1
            if steps % 20 == 0:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        stop.set()
        th.join()
        dist.barrier()
        det.close()
        out[f"period {period * 1e3:g} ms, timeout {timeout * 1e3:g} ms"] = {
            "false_failure_polls": worst["false_failures"], "polls": worst["polls"],
            "snapshot_verify_steps": steps}
    allout = [None] * world
    dist.all_gather_object(allout, out)
    if rank == 0:
        print(json.dumps({"world": world, "per_rank": allout}, indent=1))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
