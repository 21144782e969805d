"""One process driving every GPU of the box: the N -> N-1 reshard with rank
r's buffers on GPU r (peer access over NVLink/NVSwitch instead of CUDA IPC),
and the fp32 peer weighted reduce.  Used for ncu's NVLink byte counters —
ncu must not wrap a multi-rank job, but this is one process — and as a
single-process cross-check of the multi-process bandwidth.

  python tools/nvlink_single_process.py [--reps K]
  ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,\\
      nvltx__bytes.sum,nvltx__bytes_data_user.sum -k regex:"staged_copy|peer_fold" \\
      python tools/nvlink_single_process.py --reps 1

Kernels are launched in rank order: under ncu (serialised kernel replay)
each launch runs alone, so a receiver's nvlrx user bytes are its pulled
(planner ingress) bytes; without ncu all ranks' programs run concurrently.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200._native import check, lib
from paper_2510_00606_b200.fabric import ROLE_NEW, ROLE_OLD, ROLE_REPLICA
from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--skip-fold", action="store_true")
    args = ap.parse_args()
    world = torch.cuda.device_count()
    assert world >= 2, "needs >= 2 GPUs"
    for r in range(world):
        check(lib.ew_set_device(r))
        for s in range(world):
            if s != r:
                check(lib.ew_peer_access_enable(s))
    base = configs.llama2_7b()
    lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    drop = min(3, world - 1)
    rp = ReshardPlan.build(lb, list(range(world)), [r for r in range(world) if r != drop])
    bufs, table = {}, {}
    for r in range(world):
        with torch.cuda.device(r):
            b = ReshardExecutor(rp, r).allocate()
            if b.old is not None:
                dev.fill_synthetic(shard_map(rp.src, r), b.old, 0)
            if b.replica is not None:
                dev.fill_synthetic(shard_map(rp.src, rp.replica_of(r)), b.replica, 0)
            bufs[r] = b
            for role, t in ((ROLE_OLD, b.old), (ROLE_REPLICA, b.replica), (ROLE_NEW, b.new)):
                if t is not None:
                    table[(role, r)] = t.data_ptr()
    nblocks = (sum(lb) + 65535) // 65536
    progs, sums = {}, {}
    for r in rp.new_ranks:
        with torch.cuda.device(r):
            progs[r] = dev.CopyProgram.from_descs(rp.copies(r, push=False), table, world, r,
                                                  shard_map(rp.dst, r))
            sums[r] = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    for r in range(world):
        torch.cuda.synchronize(r)
    times = {r: [] for r in rp.new_ranks}
    for _ in range(max(1, args.reps)):
        ev = {}
        for r in rp.new_ranks:
            with torch.cuda.device(r):
                sums[r].zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                progs[r].launch(block_sums=sums[r])
                e.record()
                ev[r] = (s, e)
        for r in range(world):
            torch.cuda.synchronize(r)
        for r, (s, e) in ev.items():
            times[r].append(s.elapsed_time(e) / 1e3)
    total = sum(x.cpu() for x in sums.values())
    ok = True
    before = torch.zeros(2 * nblocks, dtype=torch.int64)
    for r in rp.old_ranks:
        if r in rp.failed:
            continue
        with torch.cuda.device(r):
            m = shard_map(rp.src, r)
            rows = m.new_row_sums()
            dev.checksum(m, bufs[r].old, rows)
            acc = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
            dev.rows_to_blocks(m, rows, acc)
            before += acc.cpu()
    with torch.cuda.device(rp.ring.backed_up_by(drop)):
        m = shard_map(rp.src, drop)
        rows = m.new_row_sums()
        dev.checksum(m, bufs[rp.ring.backed_up_by(drop)].replica, rows)
        acc = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
        dev.rows_to_blocks(m, rows, acc)
        before += acc.cpu()
    ok = bool(torch.equal(before, total))
    tr = rp.traffic()
    res = {"what": f"single process, {world} GPUs: {world}->{world - 1} reshard (drop {drop}), "
                   "every receiver's verified pull program on its own GPU, all concurrently",
           "verified_by_conservation": ok,
           "per_rank": {r: {"copy_ms": round(min(times[r]) * 1e3, 3),
                            "planner_ingress_bytes": tr["ingress"][r],
                            "planner_egress_bytes": tr["egress"][r]} for r in rp.new_ranks}}
    slowest = max(min(t) for t in times.values())
    res["bottleneck_gpu_bytes"] = tr["bottleneck_bytes"]
    res["bottleneck_nvlink_gbs"] = round(tr["bottleneck_bytes"] / slowest / 1e9, 1)
    del progs, sums, bufs
    for r in range(world):
        with torch.cuda.device(r):
            torch.cuda.empty_cache()

    if not args.skip_fold:
        n = 1_684_603_904
        units, outs = {}, {}
        for r in range(world):
            with torch.cuda.device(r):
                units[r] = torch.empty(n, dtype=torch.float32, device="cuda").normal_(0, 1e-3)
                outs[r] = torch.empty(n, dtype=torch.float32, device="cuda")
        folds = {}
        for r in range(world):
            with torch.cuda.device(r):
                folds[r] = dev.PeerFold(world, r, n, [units[k].data_ptr() for k in range(world)],
                                        [1.0 / world] * world,
                                        [outs[k].data_ptr() for k in range(world)])
        f = dev.fixed_point_bits(1.0, world)
        ev = {}
        for phase in ("reduce_scatter", "all_gather"):
            for r in range(world):
                with torch.cuda.device(r):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    if phase == "reduce_scatter":
                        folds[r].reduce_scatter(f)
                    else:
                        folds[r].all_gather()
                    e.record()
                    ev[(phase, r)] = (s, e)
            for r in range(world):
                torch.cuda.synchronize(r)
        res["peer_fold"] = {
            "elements_per_rank": n,
            "payload_pulled_bytes_per_phase_per_rank": (world - 1) * 4 * n // world,
            "ms": {f"{p}_r{r}": round(s.elapsed_time(e), 3) for (p, r), (s, e) in ev.items()}}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
