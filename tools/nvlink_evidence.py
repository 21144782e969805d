"""NVLink byte evidence for the reshard copy and the peer fold (torchrun).

Hardware NVLink counters (NVML field values: per-link transmit / receive
byte counters, summed over the GPU's links) are read on every rank around
K launches of
  * the 4->3 (N->N-1) verified pull reshard of 7B-per-GPU ZeRO state
    (staged_copy_kernel's remote class; ReshardExecutor as in bench.py), and
  * the fp32 peer weighted reduce (peer_fold_staged_kernel reduce-scatter
    + copy-program all-gather), 1.68 G elements per rank,
and compared with the planner's per-GPU egress / ingress bytes (pull: the
source GPU transmits, the receiver receives).  Counters include the
protocol's read-request and header traffic, so wire bytes >= payload.

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \
      tools/nvlink_evidence.py --json-out profiles/r02_nvlink_counters.json
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import pynvml
import torch
import torch.distributed as dist

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map

FIELDS = {"xmit_bytes": pynvml.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
          "rcv_bytes": pynvml.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES,
          "data_tx_kib": pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
          "data_rx_kib": pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX}
MAX_LINKS = 18


def nvml_index(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = vis.split(",")
        if local < len(ids) and ids[local].strip().isdigit():
            return int(ids[local])
    return local


def read_counters(h) -> dict:
    out = {}
    for name, fid in FIELDS.items():
        total, links = 0, 0
        for link in range(MAX_LINKS):
            try:
                vals = pynvml.nvmlDeviceGetFieldValues(h, [(fid, link)])
            except pynvml.NVMLError:
                continue
            v = vals[0]
            if v.nvmlReturn != 0:
                continue
            total += int(v.value.ullVal)
            links += 1
        out[name] = total
        out[name + "_links"] = links
    return out


def delta(a, b):
    return {k: b[k] - a[k] for k in a if not k.endswith("_links")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json-out", default="")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    # ncu's application replay re-runs every rank once per counter pass: each
    # pass rendezvouses on its own port (a pass counter per rank), so no pass
    # reads a previous pass's NCCL id from a shared store
    base = int(os.environ["MASTER_PORT"])
    counter = Path(f"/tmp/ew_nvlink_pass_{base}_{rank}")
    k = int(counter.read_text()) + 1 if counter.exists() else 0
    counter.write_text(str(k))
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{base + 1 + k}", rank=rank,
                            world_size=world, device_id=torch.device("cuda", local))
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(nvml_index(local))
    res = {"rank": rank}

    # ---- reshard N -> N-1, drop min(3, N-1)
    base = configs.llama2_7b()
    lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    drop = min(3, world - 1)
    rp = ReshardPlan.build(lb, list(range(world)), [r for r in range(world) if r != drop])
    ex = ReshardExecutor(rp, rank)
    bufs = ex.allocate()
    if bufs.old is not None:
        dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 0)
    if bufs.replica is not None:
        dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank)), bufs.replica, 0)
    ex.premap(bufs)
    ex.bind(bufs, verify=True)
    nblocks = (sum(lb) + 65535) // 65536
    sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    ex.launch(block_sums=sums)
    torch.cuda.synchronize()
    dist.barrier()
    c0 = read_counters(h)
    t0 = time.perf_counter()
    for _ in range(args.reps):
        sums.zero_()
        ex.launch(block_sums=sums)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    dist.barrier()
    c1 = read_counters(h)
    tr = rp.traffic()
    d = delta(c0, c1)
    res["reshard"] = {
        "change": f"{world}->{world - 1} (drop rank {drop}), pull, verified on arrival",
        "reps": args.reps, "links_read": c0["xmit_bytes_links"],
        "planner_egress_bytes": tr["egress"][rank], "planner_ingress_bytes": tr["ingress"][rank],
        "counter_xmit_bytes_per_rep": d["xmit_bytes"] / args.reps,
        "counter_rcv_bytes_per_rep": d["rcv_bytes"] / args.reps,
        "counter_data_tx_bytes_per_rep": 1024 * d["data_tx_kib"] / args.reps,
        "counter_data_rx_bytes_per_rep": 1024 * d["data_rx_kib"] / args.reps,
        "wall_s_per_rep": dt / args.reps}
    ex.close()
    del bufs, sums
    torch.cuda.empty_cache()

    # ---- fp32 peer weighted reduce (reduce-scatter + all-gather over peer memory)
    n = 1_684_603_904
    g = torch.empty(n, dtype=torch.float32, device="cuda").normal_(0, 1e-3)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    fold, total, opened = dev.peer_weighted_reduce_setup([g], [1.0 / world], out)
    bar = dev.PeerBarrier()
    f = dev.fixed_point_bits(1.0, total)
    fold.run(f, bar)
    bar.wait()
    torch.cuda.synchronize()
    dist.barrier()
    c0 = read_counters(h)
    for _ in range(args.reps):
        fold.run(f, bar)
    bar.wait()
    torch.cuda.synchronize()
    dist.barrier()
    c1 = read_counters(h)
    d = delta(c0, c1)
    chunk = 4 * n // world
    res["peer_fold"] = {
        "elements_per_rank": n, "reps": args.reps,
        # reduce-scatter pulls its chunk of every peer's unit; all-gather
        # pulls every peer's reduced chunk
        "payload_rx_bytes_per_rep": 2 * (world - 1) * chunk,
        "payload_tx_bytes_per_rep": 2 * (world - 1) * chunk,
        "counter_xmit_bytes_per_rep": d["xmit_bytes"] / args.reps,
        "counter_rcv_bytes_per_rep": d["rcv_bytes"] / args.reps,
        "counter_data_tx_bytes_per_rep": 1024 * d["data_tx_kib"] / args.reps,
        "counter_data_rx_bytes_per_rep": 1024 * d["data_rx_kib"] / args.reps,
        "barrier_timed_out": bar.timed_out()}
    dist.barrier()
    bar.close()
    del fold
    for p in opened:
        dev.ipc_close(p)
    allr = [None] * world
    dist.all_gather_object(allr, res)
    if rank == 0:
        line = json.dumps({"what": "NVML NVLink counters around the reshard copy and the peer "
                                   "fold, per rank", "world": world, "per_rank": allr})
        print(line, flush=True)
        if args.json_out:
            Path(args.json_out).write_text(line + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
