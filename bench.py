#!/usr/bin/env python3
"""Benchmark of the B200 per-step DP recovery path (BASELINE.json metric:
"snapshot+verify GB/s per GPU; reshard MTTR (ms) 8->7 B200 at 7B ZeRO state").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (driver, N > 1)

One STEP = one per-step snapshot of this GPU's ZeRO shard with its fused
per-block checksum, followed by verification of the snapshot (two kernels).
Workload (config B): Llama-2 7B ZeRO state, bf16 params + fp32 master/m/v =
14 B/param, interleaved over DP=8; each GPU owns one rank's 11.79 GB shard
(weak scaling: per-GPU work is fixed as N grows).  `value` counts algorithmic
HBM bytes, 2S (copy) + S (verify re-read) per step per GPU, summed over GPUs.

Also measured in the same run (extra keys):
  reshard   N -> N-1 live remap of the same 7B-per-GPU state over NVLink peer
            pointers (N >= 2; the 8 -> 7 headline at N = 8, dropping rank 3),
            with the MTTR breakdown (plan, peer mapping, NCCL shrink, copy).
  philox    config E dropout masks for the busiest rank after DP 8 -> 5.
  reduce    config E weighted fixed-point fold (+ NCCL int64 sum when N > 1).
--impl reference times the CPU path on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "snapshot+verify GB/s per GPU; reshard MTTR (ms) 8→7 B200 at 7B ZeRO state"
FALLBACK_HBM_GBS = 6650.0
# config B's ZeroLayout layer sizes (llama2-7b, 14 B/param),
# restated here so the reference arm builds its workload without importing the
# product package (tests/test_cpu_baselines.py pins it to configs.llama2_7b)
LLAMA2_7B_LAYER_BYTES = [14 * p for p in [131_072_000] + [202_383_360] * 32 + [131_076_096]]
HEADLINE_SHARD_RANK = 0  # GPU k holds rank (k mod 8)'s shard; rank 0 at N=1
REDUCE_UNITS = 8         # config E reduce: global contribution units (any N | 8)


def workload_config(shard_bytes: int, block_bytes: int, world: int) -> dict:
    """The headline workload, identical in both arms' JSON lines."""
    return {"workload": "llama2-7b ZeRO interleaved DP=8, one rank's shard per GPU: "
                        "snapshot (copy + per-block checksum) then verify",
            "shard_bytes": shard_bytes, "block_bytes": block_bytes,
            "bytes_per_step_per_gpu": 3 * shard_bytes,
            "bytes_counted": "HBM read+write: 2S snapshot + S verify",
            "l2": "inputs 11.8 GB/GPU >> 126 MB L2; no flush needed",
            "parallelism": f"dp{world} (independent shards)"}


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--block-bytes", type=int, default=65536)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--reshard-reps", type=int, default=10)
    # config E: a 7B-sized fp32 gradient per rank
    p.add_argument("--reduce-elems", type=int, default=6_738_415_616)
    p.add_argument("--cpu-sample-bytes", type=int, default=1 << 30)
    p.add_argument("--reshard-state-gb", type=float, default=0.0,
                   help="config D: per-GPU ZeRO state for the reshard leg (fill-HBM geometry)")
    p.add_argument("--inplace-state-gb", type=float, default=0.0,
                   help="config D: per-GPU state for the staged in-place reshard leg (0 = skip)")
    p.add_argument("--inplace-stage-gb", type=float, default=1.0)
    p.add_argument("--inplace-reps", type=int, default=3)
    p.add_argument("--inplace-phase-gb", type=float, default=0.0,
                   help="0: the executor's default (largest NEW shard / 28)")
    p.add_argument("--inplace-slack", type=int, default=1)
    p.add_argument("--inplace-gather-streams", type=int, default=2)
    p.add_argument("--only-inplace", action="store_true",
                   help="run only the snapshot leg and the in-place reshard leg")
    p.add_argument("--skip", default="",
                   help="comma list of: e2e,cpu,inplace,config_d,reshard,host_replica,replica,"
                        "replay,migration,config_c,stage,philox,reduce,config_a")
    p.add_argument("--json-out", default="")
    p.add_argument("--deadline-s", type=float, default=900.0,
                   help="wall-clock budget of the whole run: past it (a leg hung) rank 0 "
                        "prints the line gathered so far, marked incomplete, and all ranks exit")
    p.add_argument("--trace", action="store_true",
                   help="log each leg's start to stderr on every rank (locates a hang)")
    return p.parse_args()


# ------------------------------------------------------------------ helpers ---

def measured_peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d.get("hbm_gbs", FALLBACK_HBM_GBS)), "measured"
    return FALLBACK_HBM_GBS, "fallback"


def profiled_traffic(kernel: str):
    """dram read+write bytes per launch from the committed ncu capture."""
    f = ROOT / "profiles" / "traffic.json"
    if f.exists():
        return json.loads(f.read_text()).get(kernel)
    return None


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.out = None

    def start(self):
        try:
            self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.idx), "-lms", "100"], stdout=self.out, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.out.flush()
        rows = []
        for line in Path(self.out.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append({"sm": float(parts[1]), "max": float(parts[2]),
                             "reasons": {"hw_slowdown": parts[5], "hw_thermal_slowdown": parts[6],
                                         "sw_thermal_slowdown": parts[7], "sw_power_cap": parts[8]}})
            except ValueError:
                continue
        os.unlink(self.out.name)
        if not rows:
            return None
        reasons = sorted({k for r in rows for k, v in r["reasons"].items() if v == "Active"})
        return {"sm_mhz": statistics.median(r["sm"] for r in rows),
                "sm_max_mhz": max(r["max"] for r in rows), "reasons": reasons,
                "samples": len(rows)}


def dist_setup(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    import torch
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


def max_over_ranks(values, world, group=None):
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.tolist()


def gpu_index(local):
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [x for x in vis.split(",") if x.strip()]
        if local < len(ids) and ids[local].strip().isdigit():
            return int(ids[local])
    return local


# ------------------------------------------------------------- (a) b200 arm ---

def run_snapshot(args, rank, world, local, out):
    import torch
    from paper_2510_00606_b200 import configs, device as dev, fabric

    cfg = configs.llama2_7b()
    layout = fabric.interleaved_layout(cfg.layer_bytes, range(cfg.dp))
    shard_rank = (HEADLINE_SHARD_RANK + rank) % cfg.dp
    segs = layout.segments(shard_rank)
    S = layout.shard_bytes(shard_rank)
    m = dev.ShardMap(segs, args.block_bytes)
    live = dev.empty_bytes(S)
    snap = dev.empty_bytes(S)
    rows = m.new_row_sums()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.fill_synthetic(m, live, seed=0)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        dev.snapshot(m, live, snap, rows)
        dev.verify(m, snap, rows, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 0, "warm-up verification failed"
    assert torch.equal(snap[:S], live[:S]), "snapshot differs from live state"

    K = args.steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(gpu_index(local))
    clocks.start()
    time.sleep(0.3)
    barrier(world)
    start.record(stream)
    for k in range(K):
        ev[k][0].record(stream)
        dev.snapshot(m, live, snap, rows)
        ev[k][1].record(stream)
        dev.verify(m, snap, rows, bad)
        ev[k][2].record(stream)
    end.record(stream)
    barrier(world)
    clk = clocks.stop()
    assert int(bad.item()) == 0, "verification failed in the timed region"
    t_total = start.elapsed_time(end) / 1e3
    t_snap = sum(a.elapsed_time(b) for a, b, _ in ev) / K / 1e3
    t_ver = sum(b.elapsed_time(c) for _, b, c in ev) / K / 1e3
    t_total, t_snap, t_ver = max_over_ranks([t_total, t_snap, t_ver], world)
    step = t_total / K
    bytes_step = 3 * S
    peak, peak_kind = measured_peaks()
    achieved = 2 * S / t_snap / 1e9
    # the plain-copy ceiling of the same bytes on this GPU, measured live after
    # the timed region (cudaMemcpyAsync D2D via torch copy_, best of 3): at
    # this size it runs above MEASURED_PEAKS' 2 GiB copy figure
    # (profiles/r01_snapshot_size_probe.log), so the fused kernel is also
    # graded against it
    t_copy = 1e30
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        snap.copy_(live)
        b.record(stream)
        torch.cuda.synchronize()
        t_copy = min(t_copy, a.elapsed_time(b) / 1e3)
    copy_gbs = max_over_ranks([-2 * S / t_copy / 1e9], world)[0] * -1  # min over ranks
    out.update({
        "metric": METRIC, "value": round(world * bytes_step / step / 1e9, 2), "unit": "GB/s",
        "n_gpus": world, "steps": K, "warmup": args.warmup, "ms_per_step": round(step * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (word i = splitmix64(seed ^ i))",
        "config": workload_config(S, args.block_bytes, world),
        "per_gpu_gbs": round(bytes_step / step / 1e9, 2),
        "state_gbs_per_gpu": round(S / step / 1e9, 2),
        "kernels": {"ew_snapshot_ms": round(t_snap * 1e3, 4), "ew_verify_ms": round(t_ver * 1e3, 4),
                    "ew_verify_gbs": round(S / t_ver / 1e9, 1)},
        "roofline": {"kernel": "ew_snapshot (warp_row_kernel<kSnapshot>)", "bound": "hbm",
                     "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "frac_of_8tbs_spec": round(achieved / 8000.0, 4),
                     "plain_copy_gbs": round(copy_gbs, 1),
                     "frac_of_plain_copy": round(achieved / copy_gbs, 4),
                     "traffic": profiled_traffic("snapshot_7b")},
        "clocks": clk, "gpu_launches": 2 * K,
    })
    return m, live, snap, rows, bad, S, segs


def run_e2e(args, rank, world, out, m, live, snap, rows, bad, S):
    """Same step through the public API with the shard in pinned HOST memory:
    H2D of the live shard, snapshot + verify, D2H of checksum rows + verdict."""
    import torch
    from paper_2510_00606_b200 import device as dev

    host_live = torch.empty(live.numel(), dtype=torch.uint8, pin_memory=True)
    host_live.copy_(live)
    host_rows = torch.empty(rows.numel(), dtype=torch.int64, pin_memory=True)
    host_bad = torch.empty(1, dtype=torch.int32, pin_memory=True)
    stream = torch.cuda.current_stream()
    # two device landing buffers: step k+1's H2D (copy stream) runs while
    # step k's kernels read the other one, as a training loop prefetches
    bufs = [live, dev.empty_bytes(live.numel())]
    copy_stream = torch.cuda.Stream()
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    for ev in free:
        ev.record(stream)

    def step(k):
        b = k % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(free[b])
            bufs[b].copy_(host_live, non_blocking=True)
            ready[b].record(copy_stream)
        stream.wait_event(ready[b])
        dev.snapshot(m, bufs[b], snap, rows, stream=stream)
        dev.verify(m, snap, rows, bad, stream=stream)
        free[b].record(stream)
        host_rows.copy_(rows, non_blocking=True)
        host_bad.copy_(bad, non_blocking=True)

    step(0)
    torch.cuda.synchronize()
    K = args.e2e_steps
    barrier(world)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record(stream)
    for ev in free:  # the copy stream starts inside the timed region
        ev.record(stream)
    for k in range(K):
        step(k)
    e.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    assert int(host_bad.item()) == 0
    t = max_over_ranks([max(s.elapsed_time(e) / 1e3, wall)], world)[0] / K
    out["e2e"] = {"value": round(world * 3 * S / t / 1e9, 2), "unit": "GB/s",
                  "h2d_bytes_per_step": int(live.numel()),
                  "d2h_bytes_per_step": int(rows.numel() * 8 + 4),
                  "ms_per_step": round(t * 1e3, 3),
                  "path": "pinned host shard -> H2D (copy stream, double-buffered: step k+1's "
                          "H2D overlaps step k's kernels) -> ew_snapshot -> ew_verify -> "
                          "D2H rows+verdict"}
    del host_live, bufs


def run_cpu_baseline(args, out, segs, S):
    """Oracle port (the reference has no snapshot/checksum) on the host cores."""
    import numpy as np
    from oracle.ew_oracle import load_oracle

    orc = load_oracle()
    sample = min(S, args.cpu_sample_bytes)
    sub, local = [], 0
    for s in segs:
        if local >= sample:
            break
        n = min(int(s["length"]), sample - local)
        sub.append({"global_lo": int(s["global_lo"]), "length": n, "local_off": local})
        local += n
    threads = os.cpu_count() or 1
    live = orc.fill_synthetic(sub, local, 0)
    snap = np.empty_like(live)
    snap.fill(0)
    orc.snapshot_mt(sub, args.block_bytes, live, snap, threads)  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        sums = orc.snapshot_mt(sub, args.block_bytes, live, snap, threads)
        bad = orc.verify_mt(sub, args.block_bytes, snap, sums, threads)
        reps += 1
        if time.perf_counter() - t0 > 10.0 or reps >= 50:
            break
    dt = (time.perf_counter() - t0) / reps
    assert bad == 0
    out["cpu_baseline"] = {"value": round(3 * local / dt / 1e9, 3), "unit": "GB/s",
                           "cores": threads, "kind": "port",
                           "sample": f"first {local} bytes of the 7B rank-{HEADLINE_SHARD_RANK} "
                                     f"shard (the GPU arm's shard at N=1), {reps} reps (memcpy + "
                                     "word-wise checksum, then verify re-read)"}
    return out["cpu_baseline"]


# ------------------------------------------------------------ (b) reshard ---

def run_reshard(args, rank, world, out):
    """(b) N -> N-1 reshard of 7B-per-GPU ZeRO state and the measured MTTR.

    Copy bandwidth: one verified pull program per GPU (ReshardExecutor),
    timed over reps.  MTTR: the C++ recovery runtime end to end — the DP
    group (elaskit::b200::DpGroup) holds the NCCL communicator and, built in
    steady state, one shrunk communicator per possible departure (ncclCommSplit
    with splitShare, warmed by one all-reduce) plus a PreparedRecovery (every
    departure planned, lowered, IPC-mapped and bound).  At the failure the
    survivors call DpGroup.recover: plan_edit + communicator lookup + its
    first collective (comm repair), micro-batch reshape, then the copy, a
    device barrier and checksum conservation over peer memory (remap); the
    MttrEvent's seconds are the critical path."""
    import torch
    import torch.distributed as dist
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.recovery import DpGroup, FailureDetector, PreparedRecovery
    from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map

    # start from a clean caching allocator: a cudaFree forced by an earlier
    # leg's cached blocks inside the timed verification cost 40+ ms at N=2
    torch.cuda.empty_cache()
    base = configs.llama2_7b()
    # 7B-per-GPU state over `world` ranks (exactly config B at world = 8), or
    # config D's fill-HBM geometry with --reshard-state-gb per GPU
    if args.reshard_state_gb > 0:
        lb = configs.fill_hbm(world, int(args.reshard_state_gb * 1e9)).layer_bytes
    else:
        lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    drop = min(3, world - 1)
    old = list(range(world))
    new = [r for r in old if r != drop]
    block = args.block_bytes

    t0 = time.perf_counter()
    rp = ReshardPlan.build(lb, old, new)
    ex = ReshardExecutor(rp, rank, push=False)  # receivers pull over NVLink
    t_plan = time.perf_counter() - t0
    bufs = ex.allocate()
    if bufs.old is not None:
        dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 0)
    if bufs.replica is not None:
        dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank)), bufs.replica, 0)
    if bufs.new is not None:
        bufs.new.zero_()
    barrier(world)
    t0 = time.perf_counter()
    ex.premap(bufs)   # steady state: peers' shard/replica buffers mapped once
    t_premap = max_over_ranks([time.perf_counter() - t0], world)[0]
    barrier(world)
    t0 = time.perf_counter()
    ex.bind(bufs, verify=True, block_bytes=block)
    t_bind = time.perf_counter() - t0
    t_plan, t_bind = max_over_ranks([t_plan, t_bind], world)
    nblocks = (sum(lb) + block - 1) // block
    after = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(2):
        after.zero_()
        ex.launch(block_sums=after)
    barrier(world)
    reps = args.reshard_reps

    def timed_copies(verified):
        times = []
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier(world)
            s.record(stream)
            if verified:
                after.zero_()
                ex.launch(block_sums=after)
            else:
                ex.launch()
            e.record(stream)
            barrier(world)
            times.append(s.elapsed_time(e) / 1e3)
        return max_over_ranks([sum(times) / reps, min(times)], world)

    t_plain = timed_copies(False)
    t_copy = timed_copies(True)
    ok_bytes = True
    if bufs.new is not None:
        n = rp.dst.shard_bytes(rank)
        exp = dev.empty_bytes(n)
        dev.fill_synthetic(shard_map(rp.dst, rank), exp, 0)
        ok_bytes = bool(torch.equal(bufs.new[:n], exp[:n]))
        del exp
    traffic = rp.traffic()
    bott = traffic["bottleneck_bytes"]
    nvl_gbs = bott / t_copy[0] / 1e9 if bott else None
    res = {
        "change": f"{world}->{world - 1} (drop rank {drop})",
        "state_bytes": int(sum(lb)), "per_gpu_shard_bytes": int(rp.src.shard_bytes(0)),
        "total_bytes_moved": traffic["total_bytes_moved"], "nvlink_bytes": traffic["nvlink_bytes"],
        "bottleneck_gpu_bytes": bott, "plan_entries": len(rp.plan),
        "copy_ms": round(t_copy[0] * 1e3, 3), "copy_ms_best": round(t_copy[1] * 1e3, 3),
        "copy_without_verification_ms": round(t_plain[0] * 1e3, 3),
        "bottleneck_nvlink_gbs": round(nvl_gbs, 1) if nvl_gbs else None,
        "nvlink_frac_of_900": round(nvl_gbs / 900.0, 4) if nvl_gbs else None,
        "landed_bytes_equal_target_layout": all_ranks_true(ok_bytes, world),
        "steady_state": {"plan_ms": round(t_plan * 1e3, 3), "peer_premap_ms": round(t_premap * 1e3, 3),
                         "program_bind_ms": round(t_bind * 1e3, 3)}}
    out["reshard"] = res
    ex.close()
    del after

    # ---------------- MTTR through the C++ runtime (prepared steady state)
    succ = (rank + 1) % world
    need = rp.dst.shard_bytes(rank) + rp.src.shard_bytes(succ) + (2 << 30)
    fits = torch.tensor([1 if torch.cuda.mem_get_info()[0] > need else 0], device="cuda")
    dist.all_reduce(fits, op=dist.ReduceOp.MIN)
    if not fits.item():  # e.g. config D: a second NEW shard does not fit in HBM
        res["mttr"] = {"skipped": "a prepared NEW shard does not fit beside the state"}
        del bufs
        torch.cuda.empty_cache()
        return
    m_old = shard_map(rp.src, rank, block)
    rows = m_old.new_row_sums()
    dev.checksum(m_old, bufs.old, rows)          # the per-step snapshot rows
    rep = bufs.replica if bufs.replica is not None else dev.empty_bytes(rp.src.shard_bytes(succ))
    if bufs.replica is None:
        dev.fill_synthetic(shard_map(rp.src, succ, block), rep, 0)
    m_rep = shard_map(rp.src, succ, block)
    rep_rows = m_rep.new_row_sums()
    dev.checksum(m_rep, rep, rep_rows)
    uid = [dev.Communicator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = dev.Communicator.init(uid[0], world, rank)
    warm = torch.zeros(1024, dtype=torch.int64, device="cuda")
    comm.allreduce_i64(warm)  # a training job's DP communicator is warm
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    grp = DpGroup(lb, old, rank, comm, prepare_comms=True, block_bytes=block)
    t_prep_comm = time.perf_counter() - t0
    t0 = time.perf_counter()
    prep = PreparedRecovery(lb, old, rank, bufs.old, rep, block, old_rows=rows, replica_rows=rep_rows)
    t_prep = time.perf_counter() - t0
    grp.attach(prep)
    t_prep_comm, t_prep = max_over_ranks([t_prep_comm, t_prep], world)
    # failure detection (the reference charges a constant detect_s of 50 ms,
    # presets.hpp:63): heartbeats every 1 ms, 20 ms of silence fails a member;
    # the departing rank goes silent and the survivors' verdict starts the
    # recovery
    det = FailureDetector(f"bench{world}", 1e-3, 0.02)
    torch.cuda.synchronize()
    barrier(world)
    time.sleep(0.05)
    detect_s, detected = 0.0, True
    if rank == drop:
        det.stop_beating()
    else:
        dead, detect_s = det.wait(30.0)
        detected = dead == [drop]
    fields = ("comm_repair_s", "other_s", "remap_s")
    phases = ("plan_edit_s", "comm_acquire_s", "first_collective_s", "copy_s",
              "barrier_verify_s", "verdict_exchange_s")
    if rank != drop:
        ev = grp.recover([drop], step=1)
        ev.detect_s = detect_s
        vals = [getattr(ev, k) for k in fields] + [ev.phases.get(k, 0.0) for k in phases] + \
               [ev.total_s() - ev.detect_s, ev.detect_s, ev.total_s()]
        verified = ev.verified
        n = prep.plans[drop].dst.shard_bytes(rank)
        exp = dev.empty_bytes(n)
        dev.fill_synthetic(shard_map(prep.plans[drop].dst, rank), exp, 0)
        verified = verified and bool(torch.equal(prep.new_view(drop)[:n], exp[:n]))
        del exp
        csv = ev.csv_row(0)
    else:
        vals, verified, csv = [0.0] * (len(fields) + len(phases) + 3), True, ""
    vals = max_over_ranks(vals, world)
    mt = dict(zip(fields + phases + ("total_s", "detect_s", "with_detect_s"), vals))
    res["mttr"] = {
        "what": "measured critical path of one FailStop of rank "
                f"{drop}: DpGroup.recover (C++), max over survivors",
        "comm_repair_ms": round(mt["comm_repair_s"] * 1e3, 3),
        "reshape_ms": round(mt["other_s"] * 1e3, 3),
        "remap_ms": round(mt["remap_s"] * 1e3, 3),
        "total_ms": round(mt["total_s"] * 1e3, 3),
        "detect_ms": round(mt["detect_s"] * 1e3, 3),
        "total_with_detection_ms": round(mt["with_detect_s"] * 1e3, 3),
        "detection": {"heartbeat_period_ms": 1.0, "timeout_ms": 20.0,
                      "departed_rank_detected_by_all": all_ranks_true(detected, world),
                      "note": "detect = time from the silent rank's last heartbeat to the "
                              "survivors' verdict (FailureDetector, C++); total_ms excludes it, "
                              "as the reference's 50 ms detect_s constant is separate"},
        "phases_ms": {k[:-2]: round(mt[k] * 1e3, 3) for k in phases},
        "verified_by_checksums_and_bytes": all_ranks_true(verified, world),
        "comm_repair_path": "prepared shrunk communicator (ncclCommSplit in steady state) "
                            "looked up, then its first all-reduce",
        "mttr_csv_rank0_row": csv if rank == 0 else None,
        "steady_state_ms": {"prepare_comms": round(t_prep_comm * 1e3, 1),
                            "prepare_recovery": round(t_prep * 1e3, 1)}}
    if rank == 0:
        res["mttr"]["mttr_csv_rank0_row"] = csv
    barrier(world)
    det.close()
    grp.close()

    # baseline: the NCCL communicator repaired at failure time (ncclCommShrink
    # + its first collective), as a job without prepared communicators pays
    uid = [dev.Communicator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm2 = dev.Communicator.init(uid[0], world, rank)
    comm2.allreduce_i64(warm)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    shrunk = comm2.shrink([drop]) if rank != drop else None
    if shrunk is not None:
        shrunk.allreduce_i64(warm)
    torch.cuda.synchronize()
    t_nccl = max_over_ranks([time.perf_counter() - t0], world)[0]
    res["mttr"]["baseline_comm_shrink_at_failure_ms"] = round(t_nccl * 1e3, 3)
    barrier(world)
    if shrunk is not None:
        shrunk.destroy()
    comm2.destroy()

    # every departure position through the prepared programs (SURVEY 8(d)
    # config B: drop r3 is graded, r0 and the last rank reported)
    per_drop = {}
    for d in old:
        ts, ok = [], True
        for _ in range(max(1, reps // 2)):
            barrier(world)
            if rank != d:
                ev = prep.recover(d)
                ts.append(ev.phases["copy_s"])
                ok = ok and ev.verified
            else:
                ts.append(0.0)
        t_d = max_over_ranks([sum(ts) / len(ts)], world)[0]
        tr = prep.plans[d].traffic()
        per_drop[f"r{d}"] = {
            "copy_ms": round(t_d * 1e3, 3), "verified": all_ranks_true(ok, world),
            "total_bytes_moved": tr["total_bytes_moved"], "nvlink_bytes": tr["nvlink_bytes"],
            "bottleneck_gpu_bytes": tr["bottleneck_bytes"],
            "bottleneck_nvlink_gbs": round(tr["bottleneck_bytes"] / t_d / 1e9, 1)
            if tr["bottleneck_bytes"] else None}
    res["per_departure_prepared"] = per_drop
    if world in (2, 4, 6) and args.reshard_state_gb <= 0:
        res["projection_8to7"] = project_8to7(base, world, per_drop, res["mttr"])
    barrier(world)
    prep.close()
    # replica-aware sourcing (B200 executor option): the bytes a rank pulls
    # from the OLD shard of the member it backs up come from its own current
    # replica of it, in local HBM; same plan, same landed bytes, same
    # verification
    torch.cuda.empty_cache()
    prep2 = PreparedRecovery(lb, old, rank, bufs.old, rep, block, old_rows=rows,
                             replica_rows=rep_rows, local_replicas=True)
    per_local = {}
    for d in old:
        ts, walls, ok = [], [], True
        for _ in range(max(1, reps // 2)):
            barrier(world)
            if rank != d:
                ev = prep2.recover(d)
                ts.append(ev.phases["copy_s"])
                walls.append(ev.phases["launch_to_verdict_s"])
                ok = ok and ev.verified
            else:
                ts.append(0.0)
                walls.append(0.0)
        t_d, w_d = max_over_ranks([sum(ts) / len(ts), sum(walls) / len(walls)], world)
        nvl = local_replica_traffic(prep2.plans[d])
        per_local[f"r{d}"] = {"copy_ms": round(t_d * 1e3, 3),
                              "copy_verify_verdict_ms": round(w_d * 1e3, 3),
                              "verified": all_ranks_true(ok, world),
                              "bottleneck_nvlink_bytes": nvl,
                              "planner_exact_copy_ms": per_drop[f"r{d}"]["copy_ms"]}
    res["per_departure_local_replicas"] = per_local
    # the same FailStop through DpGroup.recover with the replica-aware
    # programs attached: the measured MTTR of this option
    barrier(world)
    uid = [dev.Communicator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm3 = dev.Communicator.init(uid[0], world, rank)
    comm3.allreduce_i64(warm)
    grp3 = DpGroup(lb, old, rank, comm3, prepare_comms=True, block_bytes=block)
    grp3.attach(prep2)
    torch.cuda.synchronize()
    barrier(world)
    if rank != drop:
        ev = grp3.recover([drop], step=1)
        vals = [ev.comm_repair_s, ev.other_s, ev.remap_s, ev.total_s()]
        ok = ev.verified
    else:
        vals, ok = [0.0] * 4, True
    vals = max_over_ranks(vals, world)
    res["mttr_local_replicas"] = {
        "what": "the measured FailStop of rank {} through DpGroup.recover with replica-aware "
                "programs (max over survivors)".format(drop),
        "comm_repair_ms": round(vals[0] * 1e3, 3), "reshape_ms": round(vals[1] * 1e3, 3),
        "remap_ms": round(vals[2] * 1e3, 3), "total_ms": round(vals[3] * 1e3, 3),
        "verified": all_ranks_true(ok, world)}
    if world in (2, 4, 6) and args.reshard_state_gb <= 0:
        res["projection_8to7_local_replicas"] = project_8to7_local(base, world, per_drop,
                                                                  per_local, res["mttr"])
    barrier(world)
    grp3.close()
    prep2.close()
    del bufs, rep
    torch.cuda.empty_cache()


def local_replica_traffic(rp) -> int:
    """Bottleneck NVLink bytes (max per-GPU ingress / egress) of a reshard
    whose pull programs use replica-aware sourcing."""
    from paper_2510_00606_b200.fabric import ROLE_OLD
    ranks = sorted(set(rp.old_ranks) | set(rp.new_ranks))
    ing = {r: 0 for r in ranks}
    egr = {r: 0 for r in ranks}
    for r in rp.new_ranks:
        held = rp.ring.backs_up(r)
        c = rp.copies(r, push=False)
        for s, role, b in zip(c["src_rank"].tolist(), c["src_role"].tolist(), c["bytes"].tolist()):
            if s == r or (role == ROLE_OLD and s == held and held not in rp.failed):
                continue
            ing[r] += b
            egr[s] += b
    return int(max(max(ing.values()), max(egr.values())))


def all_ranks_true(flag: bool, world: int) -> bool:
    """AND of a per-rank flag over the job (MIN all-reduce)."""
    if world == 1:
        return bool(flag)
    import torch
    import torch.distributed as dist
    t = torch.tensor([1 if flag else 0], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return bool(t.item())


def run_host_replica(args, rank, world, out):
    """The same N->N-1 departure with the departed rank's bytes sourced from
    node-shared host memory (hostsnap.HostSnapshots: the reference's
    H2D_D2D medium) instead of the holder's HBM replica: per-step publish
    (D2H of every rank's shard at once) and the verified recovery, timed."""
    import shutil
    import torch
    import torch.distributed as dist
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.fabric import ROLE_REPLICA
    from paper_2510_00606_b200.hostsnap import HostSnapshots
    from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map

    torch.cuda.empty_cache()
    base = configs.llama2_7b()
    lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    members = list(range(world))
    drop = min(3, world - 1)
    rp = ReshardPlan.build(lb, members, [r for r in members if r != drop])
    # the images are double-buffered (2 x the state in /dev/shm, all of it
    # touched by the three publishes below) and tmpfs pages are host RAM:
    # require room in both, with margin, before creating them
    import psutil
    room = torch.tensor([shutil.disk_usage("/dev/shm").free, psutil.virtual_memory().available],
                        dtype=torch.float64, device="cuda")
    dist.all_reduce(room, op=dist.ReduceOp.MIN)
    if room[0].item() < 2.2 * sum(lb) or room[1].item() < 2.5 * sum(lb):
        if rank == 0:
            out["host_replica"] = {"skipped": "/dev/shm or host RAM below 2.2x / 2.5x the state "
                                              "(double-buffered images)"}
        return
    S = rp.src.shard_bytes(rank)
    stream = torch.cuda.current_stream()
    ex = ReshardExecutor(rp, rank, push=False)
    bufs = ex.allocate(device_replica=False)
    dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 0)
    try:
        hs = HostSnapshots(rp.src, members, rank, tag=f"bench{os.getppid()}", readable=[drop])
        err = ""
    except Exception as e:  # the constructor fails on every rank together
        hs, err = None, repr(e)
    okt = torch.tensor([0 if hs is None else 1], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if not okt.item():
        if hs is not None:
            hs.close()
        if rank == 0:
            out["host_replica"] = {"skipped": "host images could not be mapped: " + (err or "peer")}
        ex.close()
        return
    times = []
    for _ in range(3):
        barrier(world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        hs.publish(bufs.old, stream)
        e.record(stream)
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) / 1e3)
    t_pub = max_over_ranks([min(times)], world)[0]
    hs.attach(ex, [drop])
    barrier(world)
    ex.bind(bufs, verify=True)
    nblocks = (sum(lb) + args.block_bytes - 1) // args.block_bytes
    m_old = shard_map(rp.src, rank, args.block_bytes)
    rows = m_old.new_row_sums()
    dev.checksum(m_old, bufs.old, rows)
    before = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    dev.rows_to_blocks(m_old, rows, before)
    dist.all_reduce(before)
    times = []
    ok = True
    for _ in range(3):
        sums = torch.zeros_like(before)
        barrier(world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ex.launch(stream=stream, block_sums=sums)
        e.record(stream)
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) / 1e3)
        dist.all_reduce(sums)
        ok = ok and bool(torch.equal(sums, before))
    t_copy = max_over_ranks([sum(times) / len(times)], world)[0]
    if bufs.new is not None:
        n = rp.dst.shard_bytes(rank)
        exp = dev.empty_bytes(n)
        dev.fill_synthetic(shard_map(rp.dst, rank), exp, 0)
        ok = ok and bool(torch.equal(bufs.new[:n], exp[:n]))
        del exp
    okt = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    pulls = rp.copies(rank, push=False)
    host_b = int(pulls[pulls["src_role"] == ROLE_REPLICA]["bytes"].sum()) if rank != drop else 0
    host_max = int(max_over_ranks([float(host_b)], world)[0])
    res = {"change": f"{world}->{world - 1} (drop rank {drop})",
           "source_of_departed_bytes": "node-shared pinned host memory (POSIX shm), read by "
                                       "each destination's copy kernel over its own PCIe link",
           "publish_ms": round(t_pub * 1e3, 2),
           "publish_gbs_per_gpu": round(S / t_pub / 1e9, 1),
           "copy_ms": round(t_copy * 1e3, 2), "host_bytes_busiest_gpu": host_max,
           "host_read_gbs_busiest_gpu": round(host_max / t_copy / 1e9, 1) if host_max else None,
           "verified_on_arrival_and_bytes": bool(okt.item())}
    if "reshard" in out and "copy_ms" in out["reshard"]:
        res["hbm_replica_copy_ms"] = out["reshard"]["copy_ms"]
    out["host_replica"] = res
    barrier(world)
    ex.close()
    hs.close()
    del bufs
    torch.cuda.empty_cache()


def project_8to7(base, world, per_drop, prepared):
    """Config B's 8->7 MTTR from this run, for pools that lend fewer than 8
    GPUs (labelled a projection; at N = 8 the reshard leg measures it).  The
    8->7 plans come from the planner (exact bytes); each departure kind takes
    the bottleneck-link rate measured here for the same kind of departure at
    N -> N-1 (first rank: its ring holder's egress; last rank: self-lane
    heavy; interior ranks: the slowest interior one), plus the prepared
    path's measured host and verification overheads."""
    from paper_2510_00606_b200.reshard import ReshardPlan

    rate = {k: v["bottleneck_nvlink_gbs"] for k, v in per_drop.items()}
    interior = [rate[f"r{d}"] for d in range(1, world - 1) if rate.get(f"r{d}")]
    kinds = {0: rate.get("r0"), 7: rate.get(f"r{world - 1}"),
             3: min(interior) if interior else rate.get(f"r{world - 1}")}
    overhead_ms = prepared["total_ms"] - prepared["phases_ms"]["copy"]
    res = {"what": "projection, not a measurement: 8->7 bottleneck bytes (planner, exact) / "
                   f"bottleneck-link rate measured at {world}->{world - 1} for the same kind of "
                   "departure + the measured non-copy MTTR (comm repair, reshape, barrier, "
                   "verification, verdict) of the C++ recovery here",
           "overhead_ms": round(overhead_ms, 3)}
    for d, gbs in kinds.items():
        rp = ReshardPlan.build(base.layer_bytes, list(range(8)), [r for r in range(8) if r != d])
        b = rp.traffic()["bottleneck_bytes"]
        if not gbs or not b:
            continue
        copy_ms = b / (gbs * 1e9) * 1e3
        res[f"drop_r{d}"] = {"bottleneck_gpu_bytes": b, "rate_gbs": gbs,
                             "copy_ms": round(copy_ms, 2), "mttr_ms": round(copy_ms + overhead_ms, 2)}
    return res


def project_8to7_local(base, world, per_drop, per_local, mttr):
    """Config B's 8->7 MTTR with replica-aware programs, for pools with fewer
    than 8 GPUs (a projection): the larger of the NVLink lane time (the
    8->7 plan's replica-aware bottleneck bytes at the bottleneck-link rate
    measured here for the same kind of departure) and the local-copy time
    (NEW bytes per GPU at the all-local rate measured here), plus the
    measured non-copy MTTR."""
    from paper_2510_00606_b200.reshard import ReshardPlan

    rate = {k: v["bottleneck_nvlink_gbs"] for k, v in per_drop.items()}
    interior = [rate[f"r{d}"] for d in range(1, world - 1) if rate.get(f"r{d}")]
    kinds = {0: rate.get("r0"), 7: rate.get(f"r{world - 1}"),
             3: min(interior) if interior else rate.get(f"r{world - 1}")}
    lb_here = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    here = ReshardPlan.build(lb_here, list(range(world)), [r for r in range(world) if r != world - 1])
    local_gbs = max(here.dst.shard_bytes(r) for r in here.new_ranks) / \
        (per_local[f"r{world - 1}"]["copy_ms"] / 1e3) / 1e9     # all-local at N -> N-1, last rank
    overhead_ms = mttr["total_ms"] - mttr["phases_ms"]["copy"]
    res = {"what": "projection, not a measurement: max(replica-aware NVLink bottleneck bytes / "
                   f"measured link rate, NEW bytes / measured all-local rate {local_gbs:.0f} "
                   "GB/s) + measured non-copy MTTR", "overhead_ms": round(overhead_ms, 3)}
    for d, gbs in kinds.items():
        rp = ReshardPlan.build(base.layer_bytes, list(range(8)), [r for r in range(8) if r != d])
        nvl = local_replica_traffic(rp)
        new_max = max(rp.dst.shard_bytes(r) for r in rp.new_ranks)
        t_nvl = nvl / (gbs * 1e9) * 1e3 if nvl and gbs else 0.0
        t_loc = new_max / (local_gbs * 1e9) * 1e3
        res[f"drop_r{d}"] = {"nvlink_bottleneck_bytes": nvl, "copy_ms": round(max(t_nvl, t_loc), 2),
                             "mttr_ms": round(max(t_nvl, t_loc) + overhead_ms, 2)}
    return res


def run_config_c(args, rank, world, out):
    """Config C at N GPUs: 8B-sized ZeRO state (14.05 GB per GPU), two
    non-adjacent ranks leave (8->6 drops {2, 5}; 4->2 drops {1, 3}), then
    rejoin (N-2 -> N).  Each change is one verified pull program per GPU
    (verification on arrival + block-sum conservation), bytes checked."""
    import torch
    import torch.distributed as dist
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map

    torch.cuda.empty_cache()
    base = configs.llama3_8b()
    lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    block = args.block_bytes
    nblocks = (sum(lb) + block - 1) // block
    gone = [2, 5] if world == 8 else [1, 3]
    members = list(range(world))
    kept = [r for r in members if r not in gone]
    res = {"state_bytes": int(sum(lb)), "per_gpu_shard_bytes": int(sum(lb) // world)}
    for label, old, new in (("scale_in", members, kept), ("rejoin", kept, members)):
        rp = ReshardPlan.build(lb, old, new)
        ex = ReshardExecutor(rp, rank)
        bufs = ex.allocate()
        if bufs.old is not None:
            dev.fill_synthetic(shard_map(rp.src, rank, block), bufs.old, 8)
        if bufs.replica is not None:
            dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank), block), bufs.replica, 8)
        before = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
        if bufs.old is not None and rank not in rp.failed:
            mo = shard_map(rp.src, rank, block)
            rows = mo.new_row_sums()
            dev.checksum(mo, bufs.old, rows)
            dev.rows_to_blocks(mo, rows, before)
        if bufs.replica is not None:
            mr = shard_map(rp.src, rp.replica_of(rank), block)
            rows = mr.new_row_sums()
            dev.checksum(mr, bufs.replica, rows)
            dev.rows_to_blocks(mr, rows, before)
        dist.all_reduce(before)
        barrier(world)
        ex.bind(bufs, verify=True, block_bytes=block)
        after = torch.zeros_like(before)
        ex.launch(block_sums=after)
        barrier(world)
        times = []
        for _ in range(args.reshard_reps):
            after.zero_()
            barrier(world)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ex.launch(block_sums=after)
            b.record()
            barrier(world)
            times.append(a.elapsed_time(b) / 1e3)
        t = max_over_ranks([sum(times) / len(times)], world)[0]
        dist.all_reduce(after)
        ok = bool(torch.equal(before, after))
        if bufs.new is not None:
            n = rp.dst.shard_bytes(rank)
            exp = dev.empty_bytes(n)
            dev.fill_synthetic(shard_map(rp.dst, rank, block), exp, 8)
            ok = ok and bool(torch.equal(bufs.new[:n], exp[:n]))
            del exp
        okt = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        tr = rp.traffic()
        bott = tr["bottleneck_bytes"]
        res[label] = {"change": f"{len(old)}->{len(new)}", "departed": gone if label == "scale_in" else [],
                      "joined": gone if label == "rejoin" else [],
                      "copy_ms": round(t * 1e3, 3), "bottleneck_gpu_bytes": bott,
                      "bottleneck_nvlink_gbs": round(bott / t / 1e9, 1) if bott else None,
                      "verified_on_arrival_and_bytes": bool(okt.item())}
        barrier(world)
        ex.close()
        del bufs, before, after
        torch.cuda.empty_cache()
    out["config_c"] = res
    res["mttr"] = config_c_mttr(args, rank, world, lb, gone)


def config_c_mttr(args, rank, world, lb, gone):
    """Config C's two events as measured recoveries through the C++ DpGroup
    (the reference's recover_elaswave for FailStop/ScaleIn and ScaleOut,
    sim.cpp:597-722), with the NCCL communicator of the (d) reduce repaired
    each time: steady state prepares the shrunk communicator of the pair
    (ncclCommSplit) and, after the departure, the grown standby communicator
    for their return; the survivors then recover the pair (planned at failure
    time: plan, IPC mapping, verified copy, conservation) and the pair
    rejoins from the free pool (the same processes: ScaleOut, members re-cut
    their shards over the grown group, joiners only receive).  Every
    participant's buffers are IPC-mapped in steady state (DpGroup.premap, and
    prepare_join for the joiners), the source block sums come from the
    per-step snapshot rows, and each rank's verified program for the event is
    lowered and bound in steady state (DpGroup.prepare_move), so the event
    launches it.  MTTR = max over the participants; bytes checked against the
    synthetic state."""
    import torch
    import torch.distributed as dist
    from paper_2510_00606_b200 import device as dev
    from paper_2510_00606_b200.fabric import SCALE_IN, SCALE_OUT
    from paper_2510_00606_b200.recovery import DpGroup
    from paper_2510_00606_b200.reshard import RankBuffers, ReshardPlan, shard_map

    members = list(range(world))
    kept = [r for r in members if r not in gone]
    block = args.block_bytes
    uid = [dev.Communicator.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = dev.Communicator.init(uid[0], world, rank)
    grp = DpGroup(lb, members, rank, comm, prepare_comms=False, block_bytes=block)
    t0 = time.perf_counter()
    grp.prepare([gone])
    t_prep_split = max_over_ranks([time.perf_counter() - t0], world)[0]
    rp_in = ReshardPlan.build(lb, members, kept)
    rp_out = ReshardPlan.build(lb, kept, members)
    live = dev.empty_bytes(rp_in.src.shard_bytes(rank))
    dev.fill_synthetic(shard_map(rp_in.src, rank, block), live, 8)
    owner = rp_in.replica_of(rank)
    replica = None
    if owner in gone:
        replica = dev.empty_bytes(rp_in.src.shard_bytes(owner))
        dev.fill_synthetic(shard_map(rp_in.src, owner, block), replica, 8)
    new_in = dev.empty_bytes(rp_in.dst.shard_bytes(rank)) if rank in kept else None
    new_out = dev.empty_bytes(rp_out.dst.shard_bytes(rank))
    # the per-step snapshot's checksum rows of the live shard and the replica
    live_map = shard_map(rp_in.src, rank, block)
    live_rows = live_map.new_row_sums()
    dev.checksum(live_map, live, live_rows)
    rep_rows = None
    if replica is not None:
        rep_map = shard_map(rp_in.src, owner, block)
        rep_rows = rep_map.new_row_sums()
        dev.checksum(rep_map, replica, rep_rows)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    grp.premap(RankBuffers(live, replica, None), live_rows, rep_rows)
    grp.prepare_move(SCALE_IN, gone, new_in)
    torch.cuda.synchronize()
    t_premap = max_over_ranks([time.perf_counter() - t0], world)[0]

    def expect(layout, buf):
        n = layout.shard_bytes(rank)
        e = dev.empty_bytes(n)
        dev.fill_synthetic(shard_map(layout, rank, block), e, 8)
        ok = bool(torch.equal(buf[:n], e[:n]))
        del e
        return ok

    def summary(ev, ok):
        vals = [ev.total_s(), ev.comm_repair_s, ev.remap_s, ev.phases.get("copy_s", 0.0),
                ev.phases.get("map_bind_s", 0.0), ev.phases.get("plan_s", 0.0),
                ev.phases.get("sums_s", 0.0), ev.phases.get("bind_s", 0.0)] \
            if ev is not None else [0.0] * 8
        mx = max_over_ranks(vals, world)
        flags = torch.tensor([1 if ok else 0, 1 if (ev is None or ev.verified) else 0,
                              1 if (ev is None or ev.phases.get("comm_prepared") == 1.0) else 0],
                             device="cuda")
        dist.all_reduce(flags, op=dist.ReduceOp.MIN)
        pm = torch.tensor([1 if (ev is None or ev.phases.get("premapped") == 1.0) else 0,
                           1 if (ev is None or ev.phases.get("prepared") == 1.0) else 0],
                          device="cuda")
        dist.all_reduce(pm, op=dist.ReduceOp.MIN)
        return {"premapped": bool(pm[0].item()), "program_prepared": bool(pm[1].item()),
                "mttr_ms": round(mx[0] * 1e3, 3), "comm_repair_ms": round(mx[1] * 1e3, 3),
                "remap_ms": round(mx[2] * 1e3, 3), "copy_ms": round(mx[3] * 1e3, 3),
                "map_bind_ms": round(mx[4] * 1e3, 3), "plan_ms": round(mx[5] * 1e3, 3),
                "source_sums_ms": round(mx[6] * 1e3, 3), "lower_bind_ms": round(mx[7] * 1e3, 3),
                "bytes_exact": bool(flags[0].item()), "verified": bool(flags[1].item()),
                "comm_prepared": bool(flags[2].item()),
                "mttr_csv_rank0_row": ev.csv_row(0) if (ev is not None and rank == 0) else None}

    torch.cuda.synchronize()
    barrier(world)
    ev = None
    if rank in kept:
        ev = grp.recover(gone, RankBuffers(live, replica, new_in), step=1, kind=SCALE_IN)
    scale_in = summary(ev, expect(rp_in.dst, new_in) if rank in kept else True)
    barrier(world)
    jg = DpGroup.joiner(lb, kept, rank, grp.name, block_bytes=block) if rank in gone else grp
    t0 = time.perf_counter()
    if rank in kept:  # steady state after the departure: snapshot rows, map the new shards
        in_map = shard_map(rp_in.dst, rank, block)
        in_rows = in_map.new_row_sums()
        dev.checksum(in_map, new_in, in_rows)
        grp.premap(RankBuffers(new_in, None, None), in_rows)
    jg.prepare_join(gone)
    jg.prepare_move(SCALE_OUT, gone, new_out)
    torch.cuda.synchronize()
    t_prep_standby = max_over_ranks([time.perf_counter() - t0], world)[0]
    barrier(world)
    ev = jg.admit(gone, RankBuffers(new_in, None, new_out), step=2)
    rejoin = summary(ev, expect(rp_out.dst, new_out))
    rejoin["members_after"] = len(jg.members)
    barrier(world)
    if jg is not grp:
        jg.close()
    grp.close()
    del live, replica, new_in, new_out
    torch.cuda.empty_cache()
    return {"what": "measured through DpGroup (C++): ScaleIn of the pair, then its ScaleOut, "
                    "each with comm repair, reshape and a verified remap prepared in steady "
                    "state (premap, snapshot rows, prepare_move)",
            "steady_state_ms": {"prepare_pair_split": round(t_prep_split * 1e3, 1),
                                "premap_and_prepare_move": round(t_premap * 1e3, 1),
                                "premap_standby_comm_and_prepare_move":
                                    round(t_prep_standby * 1e3, 1)},
            "scale_in": scale_in, "rejoin": rejoin}


def config_d_state_gb(world: int) -> float:
    """Per-GPU state of the default config D reshard leg: as large as the
    staged in-place footprint allows on the busiest rank — the ring holder of
    the departed rank keeps max(OLD, NEW) = S·N/(N−1) plus the departed
    rank's replica S plus the staging buffers — within ~150 GB of HBM, and at
    most config D's 70 GB (2 -> 1: 50 GB, 4 -> 3: 64 GB, 8 -> 7: 70 GB)."""
    return round(min(70.0, 150.0 / (world / (world - 1) + 1.0)), 1)


def run_config_d_reshard(args, rank, world, out):
    """Config D's reshard half in the default N > 1 run: fill-HBM geometry
    (80 equal layers, config_d_state_gb per GPU), N -> N-1 staged in place."""
    run_inplace(args, rank, world, out, state_gb=config_d_state_gb(world),
                key="config_d_reshard")


def run_inplace(args, rank, world, out, state_gb=None, key="inplace"):
    """Config D reshard at fill-HBM sizes, staged in place (inplace.py): a
    rank's OLD and NEW shards share one buffer, the move runs in phases over
    the global byte space through two staging buffers, verified on arrival.
    Side by side (OLD + replica + NEW) a 180 GB B200 reshards ~55 GB per GPU;
    in place, max(OLD, NEW) + replica + 2 stages."""
    import torch
    import torch.distributed as dist
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.inplace import StagedInPlaceReshard
    from paper_2510_00606_b200.reshard import ReshardPlan, shard_map

    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    if state_gb is None:
        state_gb = args.inplace_state_gb
    if state_gb > 0:                # config D geometry, S bytes per GPU
        lb = configs.fill_hbm(world, int(state_gb * 1e9)).layer_bytes
        geometry = "config D fill-HBM"
    else:                           # the reshard leg's 7B-per-GPU state, for comparison
        base = configs.llama2_7b()
        lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
        geometry = "llama2-7b per GPU"
    drop = min(3, world - 1)
    old = list(range(world))
    new = [r for r in old if r != drop]
    block = args.block_bytes
    t0 = time.perf_counter()
    rp = ReshardPlan.build(lb, old, new)
    ex = StagedInPlaceReshard(rp, rank, stage_bytes=int(args.inplace_stage_gb * 1e9),
                              block_bytes=block,
                              phase_bytes=int(args.inplace_phase_gb * 1e9) or None,
                              slack=args.inplace_slack,
                              gather_streams=args.inplace_gather_streams)
    t_plan = time.perf_counter() - t0
    bufs = ex.allocate()
    nblocks = (sum(lb) + block - 1) // block
    before = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    mo = shard_map(rp.src, rank, block)
    dev.fill_synthetic(mo, bufs.old, 0)
    rows = mo.new_row_sums()
    dev.checksum(mo, bufs.old, rows)
    dev.rows_to_blocks(mo, rows, before)
    del rows
    if bufs.replica is not None:
        dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank), block), bufs.replica, 0)
    dist.all_reduce(before)
    t0 = time.perf_counter()
    ex.bind(bufs, None)
    t_bind = max_over_ranks([time.perf_counter() - t0], world)[0]
    torch.cuda.synchronize()
    used = torch.cuda.mem_get_info()
    used_gb = max_over_ranks([(used[1] - used[0]) / 1e9], world)[0]
    after = torch.zeros_like(before)
    stream = torch.cuda.current_stream()
    times = []
    for rep in range(max(1, args.inplace_reps)):
        if rep:
            dev.fill_synthetic(mo, bufs.old, 0)  # the move is destructive: restore OLD
        after.zero_()
        barrier(world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        ex.launch(after)
        e.record(stream)
        barrier(world)
        times.append(s.elapsed_time(e) / 1e3)
    t_copy = max_over_ranks([sum(times) / len(times), min(times)], world)
    dist.all_reduce(after)
    verified = bool(torch.equal(before, after))
    after.zero_()
    if rank in new:
        mn = shard_map(rp.dst, rank, block)
        rows = mn.new_row_sums()
        dev.checksum(mn, bufs.new, rows)
        dev.rows_to_blocks(mn, rows, after)
        del rows
    dist.all_reduce(after)
    verified_reread = bool(torch.equal(before, after))
    timed_out = torch.tensor([1 if ex.timed_out() else 0], device="cuda")
    dist.all_reduce(timed_out)
    peak = max_over_ranks([torch.cuda.max_memory_allocated() / 1e9], world)[0]
    traffic = rp.traffic()
    bott = traffic["bottleneck_bytes"]
    sched = ex.sched
    out[key] = {
        "workload": f"{geometry} {world}->{world - 1} (drop rank {drop}), staged in place",
        "per_gpu_state_bytes": rp.src.shard_bytes(0), "state_bytes": int(sum(lb)),
        "total_bytes_moved": traffic["total_bytes_moved"], "bottleneck_gpu_bytes": bott,
        "phases": len(sched.phases), "slack": sched.slack,
        "gather_streams": args.inplace_gather_streams,
        "staging_buffers": sched.ring, "stage_bytes": sched.stage_alloc,
        "staged_bytes_max_rank": max(sched.staged_bytes.values()),
        "copy_ms": round(t_copy[0] * 1e3, 3), "copy_ms_best": round(t_copy[1] * 1e3, 3),
        "bottleneck_nvlink_gbs": round(bott / t_copy[0] / 1e9, 1) if bott else None,
        "plan_ms": round(t_plan * 1e3, 3), "bind_ms": round(t_bind * 1e3, 3),
        "verified_on_arrival": verified, "verified_by_reread": verified_reread,
        "barrier_timed_out": bool(timed_out.item()),
        "peak_hbm_allocated_gb_torch": round(peak, 2),
        "device_memory_in_use_gb": round(used_gb, 2),
        "hbm_total_gb": round(torch.cuda.mem_get_info()[1] / 1e9, 2),
        "side_by_side_would_need_gb": round((rp.src.shard_bytes(0) * 2 +
                                             max(rp.dst.shard_bytes(r) for r in new)) / 1e9, 2),
    }
    barrier(world)
    ex.close()
    del bufs
    torch.cuda.empty_cache()


def run_stage_move(args, rank, world, out):
    """Cross-stage ZeRO layer move (PAPER Fig. 10): the 7B
    model split over two pipeline stages of DP = world/2; stage 0's tail
    layer (2.83 GB of optimizer state) moves to stage 1, interleaved ZeRO
    (D j->j sends, in place) vs default contiguous ZeRO (re-cut both stages)."""
    import torch
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map

    lb = configs.llama2_7b().layer_bytes
    s_layers, t_layers = lb[:17], lb[17:]
    d = world // 2
    src_gpus, dst_gpus = list(range(d)), list(range(d, 2 * d))
    res = {"dp_per_stage": d, "layer_bytes": int(s_layers[-1])}
    for kind, contiguous in (("interleaved", False), ("contiguous", True)):
        rp = ReshardPlan.for_stage_move(s_layers, t_layers, src_gpus, dst_gpus, contiguous)
        ex = ReshardExecutor(rp, rank, push=False)
        bufs = ex.allocate(in_place=True)
        dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 3)
        barrier(world)
        ex.bind(bufs)
        ex.launch()
        barrier(world)
        n = rp.dst.shard_bytes(rank)
        exp = dev.empty_bytes(n)
        dev.fill_synthetic(shard_map(rp.dst, rank), exp, 3)
        ok = torch.tensor([1 if torch.equal(bufs.new[:n], exp[:n]) else 0], device="cuda")
        del exp
        import torch.distributed as dist
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        times = []
        for _ in range(3):
            dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 3)  # restore the source
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier(world)
            s.record()
            ex.launch()
            e.record()
            barrier(world)
            times.append(s.elapsed_time(e) / 1e3)
        t = max_over_ranks([min(times)], world)[0]
        tr = rp.traffic()
        res[kind] = {"ms": round(t * 1e3, 3), "bytes_moved": tr["total_bytes_moved"],
                     "bottleneck_link_bytes": tr["bottleneck_bytes"], "verified": bool(ok.item())}
        ex.close()
        del bufs
        torch.cuda.empty_cache()
        barrier(world)
    res["interleaved_speedup"] = round(res["contiguous"]["ms"] / res["interleaved"]["ms"], 2)
    out["stage_move"] = res


def run_replica(args, rank, world, out):
    """Ring replica refresh: every holder pulls its ring
    successor's per-step snapshot over NVLink and verifies it by checksum."""
    import torch
    from paper_2510_00606_b200 import configs, device as dev, fabric
    from paper_2510_00606_b200.recovery import RingReplica
    from paper_2510_00606_b200.reshard import shard_map

    base = configs.llama2_7b()
    lb = base.layer_bytes if world == 8 else [x * world // 8 for x in base.layer_bytes]
    layout = fabric.interleaved_layout(lb, range(world))
    m = shard_map(layout, rank, args.block_bytes)
    snap = dev.empty_bytes(layout.shard_bytes(rank))
    dev.fill_synthetic(m, snap, 11)
    rows = m.new_row_sums()
    dev.checksum(m, snap, rows)
    owner = fabric.SnapshotRing(list(range(world))).backs_up(rank)
    replica = dev.empty_bytes(layout.shard_bytes(owner))
    rr = RingReplica(layout, list(range(world)), rank, replica, snap, rows, args.block_bytes)
    barrier(world)
    rr.refresh()
    barrier(world)
    times = []
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(world)
        s.record()
        rr.refresh()
        e.record()
        barrier(world)
        times.append(s.elapsed_time(e) / 1e3)
    bad = int(rr.bad.item())
    ok = torch.tensor([1 if bad == 0 else 0], device="cuda")
    import torch.distributed as dist
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    t = max_over_ranks([min(times)], world)[0]
    nbytes = layout.shard_bytes(owner)
    out["replica"] = {"what": "holder pulls its ring successor's snapshot shard + rows, re-checksums",
                      "shard_bytes": int(nbytes), "ms": round(t * 1e3, 3),
                      "nvlink_gbs": round(nbytes / t / 1e9, 1), "verified": bool(ok.item())}
    barrier(world)
    rr.close()
    del snap, replica
    torch.cuda.empty_cache()


def run_replay(args, rank, world, out):
    """Ring replica by optimizer replay (the paper's mechanism, SURVEY §8(f)
    #1): every rank runs its own AdamW step on its 7B ZeRO shard
    (842 M params, 14 B/param = 11.79 GB), then every holder replays its ring
    successor's step into its replica reading the successor's fp32 gradient
    shard over NVLink (4 B/param), and verifies the replica against the
    owner's checksum rows.  At N=1 only the owner's step is timed."""
    import torch
    from paper_2510_00606_b200 import device as dev
    from paper_2510_00606_b200.recovery import ReplayReplica

    n = 6_738_415_616 // 8
    own = dev.AdamState(n)
    grad = torch.empty(n, dtype=torch.float32, device="cuda").normal_(0, 1e-3)
    own.master.normal_(0, 0.02)
    hyper = dev.adam_hyper(lr=1e-4)
    m = dev.ShardMap(own.segments(), args.block_bytes)
    rows = m.new_row_sums()
    ev = lambda: torch.cuda.Event(enable_timing=True)
    step_t = []
    for step in range(1, 5):
        a, b = ev(), ev()
        a.record()
        dev.adam_step(grad, own, hyper, step)
        b.record()
        torch.cuda.synchronize()
        step_t.append(a.elapsed_time(b) / 1e3)
    rows_t = []
    for step in range(5, 8):
        a, b = ev(), ev()
        a.record()
        dev.adam_step(grad, own, hyper, step, rows=rows, block_bytes=args.block_bytes)
        b.record()
        torch.cuda.synchronize()
        rows_t.append(a.elapsed_time(b) / 1e3)
    t_step, t_rows = max_over_ranks([min(step_t[1:]), min(rows_t)], world)
    res = {"what": "AdamW step on a 7B ZeRO shard (ew_adam_step)", "params_per_rank": n,
           "state_bytes": own.nbytes, "owner_step_ms": round(t_step * 1e3, 3),
           "owner_step_hbm_gbs": round(30 * n / t_step / 1e9, 1),
           "owner_step_with_fused_rows_ms": round(t_rows * 1e3, 3)}
    if world > 1:
        import torch.distributed as dist
        replica = dev.AdamState(n)
        # seed the replica with the successor's current state (one full pull,
        # as when a ring is (re)formed), then keep it by replay
        succ = (rank + 1) % world
        allb = [None] * world
        dist.all_gather_object(allb, (rank, dev.ipc_handle(own.buf)))
        h0, o0 = dict(allb)[succ]
        p0 = dev.ipc_open(h0, o0)
        barrier(world)
        dev.CopyProgram.from_pointers([p0], [replica.buf.data_ptr()], [replica.nbytes],
                                      [True]).launch()
        torch.cuda.synchronize()
        barrier(world)
        dev.ipc_close(p0)
        rep = ReplayReplica(list(range(world)), rank, replica, grad, rows, args.block_bytes)
        times, vt, bad = [], [], 0
        for step in range(8, 12):
            dev.adam_step(grad, own, hyper, step, rows=rows, block_bytes=args.block_bytes)
            torch.cuda.synchronize()
            barrier(world)
            a, b, c = ev(), ev(), ev()
            a.record()
            rep.replay(hyper, step)
            b.record()
            rep.verify()
            c.record()
            torch.cuda.synchronize()
            bad += int(rep.bad.item())
            barrier(world)
            times.append(a.elapsed_time(b) / 1e3)
            vt.append(b.elapsed_time(c) / 1e3)
        t = max_over_ranks([min(times[1:]), min(vt[1:])], world)
        ok = torch.tensor([1 if bad == 0 else 0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        res.update({"holder_replay_ms": round(t[0] * 1e3, 3),
                    "holder_verify_ms": round(t[1] * 1e3, 3),
                    "nvlink_bytes": 4 * n,
                    "nvlink_gbs": round(4 * n / t[0] / 1e9, 1),
                    "replica_verified_every_step": bool(ok.item())})
        barrier(world)
        rep.close()
        del replica
    out["replay"] = res
    del own, grad
    torch.cuda.empty_cache()


def run_layer_migration(args, rank, world, out):
    """Non-blocking migration of one 7B decoder layer (202 M params) from
    rank 0 to rank 1 with shadow-gradient payback.  The
    target's step: M = 8 micro-batch folds of the layer's fp32 gradient on a
    high-priority stream (micro-batches < k fold the target's other work at
    the same cost), the bf16 parameters pulled over NVLink on a low-priority
    stream, the source's shadow folds [0, k), its int64 accumulator is pulled
    behind a device-side barrier and joins the target's last fold.  The
    reference planner is fed the measured link bandwidth and slot time (its
    k is used from the second repetition on); the migrated gradient is
    compared with the static step's bit for bit."""
    import torch
    import torch.distributed as dist
    from paper_2510_00606_b200 import device as dev, fabric
    from paper_2510_00606_b200.migration import LayerMigration

    pair = dist.new_group([0, 1])
    if rank > 1:
        barrier(world)
        return
    n, M = 202_383_360, 8
    gen = torch.Generator(device="cuda").manual_seed(3)
    unit = torch.empty(n, dtype=torch.float32, device="cuda").normal_(0, 1e-3, generator=gen)
    units, w = [unit] * M, [1.0 / M] * M
    f = dev.fixed_point_bits(float(unit.abs().max().item()) / M, M)
    params = torch.full((n,), 7, dtype=torch.int16, device="cuda") if rank == 0 else \
        torch.zeros(n, dtype=torch.int16, device="cuda")
    acc = torch.zeros(n, dtype=torch.int64, device="cuda")
    scratch = torch.zeros(n, dtype=torch.int64, device="cuda")
    ev = lambda: torch.cuda.Event(enable_timing=True)
    hi, lo = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
    # slot = one micro-batch's fold of the layer gradient (stand-in for its compute)
    with torch.cuda.stream(hi):
        for _ in range(2):
            dev.weighted_fold([unit], [w[0]], f, scratch, accumulate=True, stream=hi)
        a, b = ev(), ev()
        a.record(hi)
        dev.weighted_fold([unit], [w[0]], f, scratch, accumulate=True, stream=hi)
        b.record(hi)
    torch.cuda.synchronize()
    slot = max_over_ranks([a.elapsed_time(b) / 1e3], 2, group=pair)[0]
    other = lambda mb, st: dev.weighted_fold([unit], [w[mb]], f, scratch, accumulate=True,
                                             stream=st)
    mig = LayerMigration((16, 0, 1), 0, 1, rank, params, acc, group=pair,
                         transfer_ctas=32)
    res = {"what": "7B layer (202 M params) stage move 0->1, non-blocking + payback",
           "param_bytes": 2 * n, "payback_bytes": 8 * n, "microbatches": M,
           "slot_ms": round(slot * 1e3, 3)}
    def step(k):
        acc.zero_()
        if rank == 1:
            params.zero_()
        torch.cuda.synchronize()
        dist.barrier(group=pair)
        mig.events.clear()
        t0, t1 = ev(), ev()
        t0.record(hi)
        if rank == 1:
            mig.run_target(units, w, f, k, hi, lo, other_work=other)
        else:
            mig.run_shadow(units, w, f, k, hi)
        t1.record(hi)
        torch.cuda.synchronize()
        info = [None, None]
        dist.all_gather_object(info, (mig.measured() if rank == 1 else {},
                                      t0.elapsed_time(t1), mig.timed_out()), group=pair)
        return info[1]

    static_ms = M * slot * 1e3
    blocking = [step(0) for _ in range(3)][-1]          # k = 0: blocking move
    bw = 2 * n / (blocking[0]["params"] / 1e3)
    plan = {m: fabric.plan_layer_migration((16, 0, 1), m, param_bytes=2 * n, grad_bytes=8 * n,
                                           link_bw_bytes_per_s=bw, microbatch_slot_s=slot,
                                           num_microbatches=M, target_headroom_bytes=1 << 40)
            for m in (fabric.BLOCKING, fabric.NON_BLOCKING)}
    k = max(1, plan[fabric.NON_BLOCKING].shadow_microbatches)
    ms, step_ms, timed_out = [step(k) for _ in range(3)][-1]
    res.update({"link_gbs_measured": round(bw / 1e9, 1),
                "static_step_ms": round(static_ms, 3),
                "blocking": {"params_ms": round(blocking[0]["params"], 3),
                             "target_step_ms": round(blocking[1], 3),
                             "measured_stall_ms": round(blocking[1] - static_ms, 3),
                             "planned_stall_ms": round(plan[fabric.BLOCKING].stall_s * 1e3, 3)},
                "non_blocking": {"k": k, "params_ms": round(ms["params"], 3),
                                 "payback_pull_ms": round(ms["payback_grad"], 3),
                                 "payback_gbs": round(8 * n / ms["payback_grad"] / 1e6, 1),
                                 "target_step_ms": round(step_ms, 3),
                                 "measured_stall_ms": round(step_ms - static_ms, 3),
                                 "planned_stall_ms": round(
                                     plan[fabric.NON_BLOCKING].stall_s * 1e3, 3)},
                "barrier_timed_out": bool(timed_out)})
    if rank == 1:
        static = torch.empty_like(acc)
        dev.weighted_fold(units, w, f, static)
        torch.cuda.synchronize()
        ok = bool(torch.equal(acc, static)) and bool((params == 7).all().item())
    else:
        ok = True
    flag = [None, None]
    dist.all_gather_object(flag, ok, group=pair)
    res["gradient_bit_identical_to_static"] = all(flag)
    dist.barrier(group=pair)
    mig.close()
    out["layer_migration"] = res
    del unit, params, acc, scratch
    torch.cuda.empty_cache()
    barrier(world)


# ------------------------------------------------------------- (c) and (d) ---

def run_config_a(args, rank, world, out):
    """Config A (BASELINE configs[0], the reference's CPU-runnable case):
    125M params x 12 B (fp32 param + Adam m, v) interleaved over 4 ranks,
    rank 1 leaves.  On one GPU: every rank's shard snapshot + verify, the
    4 -> 3 reshard with every receiver's verified pull program (buffers side
    by side), checksum conservation and bytes against the target layout, and
    the config's dropout masks (seed 0, keep 0.5)."""
    import torch
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.reshard import ReshardPlan, emulate_on_one_gpu, shard_map

    cfg = configs.gpt_125m()
    block = args.block_bytes
    rp = ReshardPlan.build(cfg.layer_bytes, [0, 1, 2, 3], [0, 2, 3])
    t_snap = 0.0
    ok = True
    for r in rp.old_ranks:
        m = shard_map(rp.src, r, block)
        live, snap = dev.empty_bytes(m.nbytes), dev.empty_bytes(m.nbytes)
        rows = m.new_row_sums()
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        dev.fill_synthetic(m, live, 0)
        dev.snapshot(m, live, snap, rows)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dev.snapshot(m, live, snap, rows)
        dev.verify(m, snap, rows, bad)
        e.record()
        torch.cuda.synchronize()
        t_snap += s.elapsed_time(e) / 1e3
        ok = ok and int(bad.item()) == 0
    nblocks = (cfg.total_bytes + block - 1) // block
    sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    emulate_on_one_gpu(rp, seed=0, push=False, block_sums=sums)  # warm-up
    sums.zero_()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    got, expected = emulate_on_one_gpu(rp, seed=0, push=False, block_sums=sums)
    e.record()
    torch.cuda.synchronize()
    whole = torch.zeros_like(sums)
    for r in rp.old_ranks:   # the source's block sums (every rank's snapshot rows)
        m = shard_map(rp.src, r, block)
        buf = dev.empty_bytes(m.nbytes)
        dev.fill_synthetic(m, buf, 0)
        rows = m.new_row_sums()
        dev.checksum(m, buf, rows)
        dev.rows_to_blocks(m, rows, whole)
    torch.cuda.synchronize()
    conserved = bool(torch.equal(whole, sums))
    exact = all(torch.equal(got[r][:rp.dst.shard_bytes(r)], expected[r][:rp.dst.shard_bytes(r)])
                for r in rp.new_ranks)
    tr = rp.traffic()
    bits = dev.dropout_mask(0, 0, 16, 1, 0, 768 * 2048, 0.5)
    torch.cuda.synchronize()
    out["config_a"] = {
        "workload": "125M-param fp32+Adam state (1.484 GB), interleaved ZeRO over 4 ranks, "
                    "drop rank 1; all ranks' buffers on one GPU",
        "state_bytes": cfg.total_bytes, "snapshot_verify_all_ranks_ms": round(t_snap * 1e3, 3),
        "snapshot_verified": ok, "plan_entries": len(rp.plan),
        "total_bytes_moved": tr["total_bytes_moved"],
        "reshard_all_programs_one_gpu_ms": round(s.elapsed_time(e), 3),
        "reshard_verified_on_arrival": conserved, "reshard_bytes_exact": exact,
        "masks": {"samples": 16, "elements_per_sample": 768 * 2048, "keep": 0.5,
                  "kept_fraction": round(float(torch.stack([((bits >> b) & 1).sum()
                                                            for b in range(32)]).sum().item())
                                         / (16 * 768 * 2048), 4)}}
    del got, expected, sums, whole
    torch.cuda.empty_cache()


def run_config_d_snapshot(args, rank, world, out):
    """Config D's snapshot + verify on one GPU: ZeRO state sized to fill HBM
    (live S + snapshot S of the 191.5 GB; S = 86 GB of an 8-way interleaved
    80-layer state), steps timed like the headline leg, one flipped bit must
    be caught."""
    import torch
    from paper_2510_00606_b200 import configs, device as dev, fabric

    torch.cuda.empty_cache()
    free = torch.cuda.mem_get_info()[0]
    S_target = min(86_000_000_000, int((free - (4 << 30)) / 2))
    if S_target < 40_000_000_000:
        out["config_d_snapshot"] = {"skipped": f"only {free / 1e9:.1f} GB free"}
        return
    cfg = configs.fill_hbm(8, S_target)
    layout = fabric.interleaved_layout(cfg.layer_bytes, range(8))
    m = dev.ShardMap(layout.segments(3), args.block_bytes)
    S = layout.shard_bytes(3)
    live, snap = dev.empty_bytes(S), dev.empty_bytes(S)
    rows = m.new_row_sums()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.fill_synthetic(m, live, 7)
    dev.snapshot(m, live, snap, rows)
    dev.verify(m, snap, rows, bad)
    torch.cuda.synchronize()
    ok = int(bad.item()) == 0
    reps = 3
    s, mid, e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_snap = t_ver = 0.0
    for _ in range(reps):
        s.record()
        dev.snapshot(m, live, snap, rows)
        mid.record()
        dev.verify(m, snap, rows, bad)
        e.record()
        torch.cuda.synchronize()
        t_snap += s.elapsed_time(mid) / 1e3 / reps
        t_ver += mid.elapsed_time(e) / 1e3 / reps
        ok = ok and int(bad.item()) == 0
    snap[S // 3] ^= 0x40
    dev.verify(m, snap, rows, bad)
    torch.cuda.synchronize()
    caught = int(bad.item()) == 1
    used = torch.cuda.mem_get_info()
    out["config_d_snapshot"] = {
        "workload": "config D fill-HBM: one rank's shard of an 8-way interleaved 80-layer state",
        "shard_bytes": S, "resident_gb": round((used[1] - used[0]) / 1e9, 1),
        "snapshot_ms": round(t_snap * 1e3, 2), "verify_ms": round(t_ver * 1e3, 2),
        "step_gbs": round(3 * S / (t_snap + t_ver) / 1e9, 1),
        "snapshot_gbs": round(2 * S / t_snap / 1e9, 1),
        "verified": ok, "flipped_bit_caught": caught}
    del live, snap, rows
    torch.cuda.empty_cache()


def run_philox(args, rank, world, out):
    import torch
    from paper_2510_00606_b200 import device as dev, fabric

    slots, sizes = fabric.reshard_microbatches([4] * 8, 32, [0, 1, 2, 3, 4])
    per_rank = [32 * s for s in sizes]               # [224, 224, 192, 192, 192]
    r = rank % 5
    lo = sum(per_rank[:r])
    n, K = per_rank[r], 4096 * 4096
    bits = torch.empty((n, K // 32), dtype=torch.int32, device="cuda")
    dev.dropout_mask(0, lo, n, 1, 0, K, 0.5, bits)
    torch.cuda.synchronize()
    reps = 3
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    s.record()
    for _ in range(reps):
        dev.dropout_mask(0, lo, n, 1, 0, K, 0.5, bits)
    e.record()
    barrier(world)
    t = max_over_ranks([s.elapsed_time(e) / 1e3 / reps], world)[0]
    out["philox"] = {"workload": f"config E: {n} samples x 4096x4096 elements (rank {r} of DP5), keep 0.5",
                     "ms": round(t * 1e3, 3), "gelem_per_s": round(n * K / t / 1e9, 1),
                     "gblocks_per_s": round(n * K / 4 / t / 1e9, 2),
                     "bound": "INT-ALU (20 64x64->128 multiplies per Philox block)",
                     # ceiling: the same Philox-4x64-10 rounds with no memory traffic
                     # (tools/microbench/philox_variants.cu, __umul64hi form, B200)
                     "roofline": {"bound": "int-alu", "unit": "G blocks/s",
                                  "achieved": round(n * K / 4 / t / 1e9, 2),
                                  "peak": PHILOX_COMPUTE_CEILING_GBLOCKS,
                                  "peak_kind": "measured compute-only Philox loop",
                                  "frac": round(n * K / 4 / t / 1e9 /
                                                PHILOX_COMPUTE_CEILING_GBLOCKS, 4),
                                  # profiles/r02_ncu_mask_kernel.md
                                  "ncu_fmaheavy_pipe_busy": 0.915}}
    del bits
    torch.cuda.empty_cache()


PHILOX_COMPUTE_CEILING_GBLOCKS = 100.3  # profiles/r01_microbench_streaming.md


def run_cpu_beside(args, out):
    """The CPU paths of BASELINE.md §3 timed on this box's host cores in the
    same run, beside kernels (b), (c), (d) — reported baselines, not targets
    (test infrastructure: oracle/ restatements and the reference library).
    Each is a bounded sample (a few seconds)."""
    import numpy as np
    from oracle.ew_oracle import load_oracle, load_reference
    from paper_2510_00606_b200 import configs, fabric
    orc, ref = load_oracle(), load_reference()
    T = os.cpu_count() or 1
    res = {"cores": T}
    # (b) plan: reference overlap_matrix (1 thread, as shipped) on 7B 8->7;
    # execution: one memcpy per entry of the bottleneck rank's copies on host
    # buffers, T threads, first ~2 GiB of entries
    cfg = configs.llama2_7b()
    src = fabric.interleaved_layout(cfg.layer_bytes, range(8))
    dst = fabric.interleaved_layout(cfg.layer_bytes, [0, 1, 2, 4, 5, 6, 7])
    ring = fabric.SnapshotRing(list(range(8)))
    t0 = time.perf_counter()
    plan = fabric.overlap_matrix(src, dst, [3], ring)
    res["b_plan_b200_incl_python_ms"] = round((time.perf_counter() - t0) * 1e3, 3)
    if ref is not None:
        rs, rd = ref.interleaved(cfg.layer_bytes, range(8)), ref.interleaved(cfg.layer_bytes, [0, 1, 2, 4, 5, 6, 7])
        res["b_plan_reference_ms"] = round(min(ref.overlap_matrix(rs, rd, cfg.total_bytes, [3], list(range(8)))[2]
                                               for _ in range(3)) * 1e3, 3)
    ent = plan.entries
    lens = (ent["hi"] - ent["lo"]).astype(np.int64)
    keep = np.cumsum(lens) <= (2 << 30)
    keep[0] = True
    lens = lens[keep]
    total = int(lens.sum())
    a = np.empty(total, dtype=np.uint8)
    a[::4096] = 1
    b = np.empty(total, dtype=np.uint8)
    offs = np.concatenate([[0], np.cumsum(lens)[:-1]])
    srcs = [a.ctypes.data + int(o) for o in offs]
    dsts = [b.ctypes.data + int(o) for o in offs]
    orc.memcpy_mt(srcs, dsts, lens.tolist(), T)
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        orc.memcpy_mt(srcs, dsts, lens.tolist(), T)
    dt = (time.perf_counter() - t0) / reps
    res["b_execute_gbs"] = round(total / dt / 1e9, 2)
    res["b_execute_sample"] = f"{len(lens)} entries of the 7B 8->7 plan, {total} bytes, host memcpy"
    del a, b
    # (c) draw() over disjoint samples on T threads (reference rng.cpp:38-53)
    ns, k = 4 * T, 1 << 20
    orc.draw_mt(0, 0, T, 1, 0, 1024, T)
    t0 = time.perf_counter()
    orc.draw_mt(0, 0, ns, 1, 0, k, T)
    dt = time.perf_counter() - t0
    res["c_draw_gblocks_per_s"] = round(ns * k / 4 / dt / 1e9, 3)
    if ref is not None:
        t0 = time.perf_counter()
        ref.draw(0, 0, 1, 0, 1 << 20)
        res["c_reference_draw_gblocks_per_s_1thread"] = round((1 << 20) / 4 / (time.perf_counter() - t0) / 1e9, 4)
    # (d) weighted_grad_average: reference (1 thread) and the element-parallel
    # restatement (T threads, identical per-element fold, bit-identical)
    g = np.random.default_rng(5).normal(0, 1e-3, size=(5, 1 << 24))
    w = np.full(5, 0.2)
    t0 = time.perf_counter()
    mt = orc.weighted_average_mt(w, g, T)
    dt = time.perf_counter() - t0
    res["d_weighted_average_mt_gbs"] = round(6 * 8 * (1 << 24) / dt / 1e9, 2)
    if ref is not None:
        t0 = time.perf_counter()
        one = ref.weighted_grad_average(w, g)
        res["d_reference_gbs_1thread"] = round(6 * 8 * (1 << 24) / (time.perf_counter() - t0) / 1e9, 2)
        res["d_mt_bit_identical_to_reference"] = bool(np.array_equal(mt, one))
    # part of the cpu_baseline leg (the oracle/reference are timed as the CPU
    # baseline here, never as the measured GPU path)
    out.setdefault("cpu_baseline", {})["beside_kernels_b_c_d"] = res


def run_reduce(args, rank, world, out):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2510_00606_b200 import device as dev, fabric

    # World-size-invariant granularity: a fixed global set of REDUCE_UNITS
    # contribution units (unit u: weight (u+1)/36, data seeded by u mod 2, so
    # a rank needs at most two distinct 27 GB buffers), dealt round-robin to
    # the ranks.  The fixed-point scale depends only on the global absmax and
    # the global unit count, so N = 1, 2, 4, 8 produce the same bits
    # (output_digest).  Timed: absmax pre-pass -> global max -> F -> fold ->
    # int64 sum -> dequant.
    n = args.reduce_elems
    mine = [u for u in range(REDUCE_UNITS) if u % world == rank]
    data = {}
    for u in mine:
        if u % 2 not in data:
            gen = torch.Generator(device="cuda").manual_seed(100 + u % 2)
            t = torch.empty(n, dtype=torch.float32, device="cuda").normal_(0, 1e-3, generator=gen)
            t[(u % 2) * 1_000_003 + 17] = 1e2   # outliers set the scale
            data[u % 2] = t
    units = [data[u % 2] for u in mine]
    w = [(u + 1) / 36 for u in mine]
    acc = torch.empty(n, dtype=torch.int64, device="cuda")
    res = torch.empty(n, dtype=torch.float32, device="cuda")

    def reduce_step(ev):
        ev[0].record()
        amax = dev.weighted_absmax(units, w)
        ev[1].record()
        if world > 1:
            dist.all_reduce(amax, op=dist.ReduceOp.MAX)
        f = dev.fixed_point_bits(amax.item(), REDUCE_UNITS)
        ev[2].record()
        dev.weighted_fold(units, w, f, acc)
        ev[3].record()
        if world > 1:
            dist.all_reduce(acc)  # ncclInt64 sum: exact, order-free
        ev[4].record()
        dev.fixed_to_float(acc, f, res)
        ev[5].record()
        return f

    f = reduce_step([torch.cuda.Event(enable_timing=True) for _ in range(6)])  # warm-up
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    barrier(world)
    f = reduce_step(ev)
    torch.cuda.synchronize()
    barrier(world)
    t_amax, t_max, t_fold, t_ar, t_deq, t_all = max_over_ranks(
        [ev[0].elapsed_time(ev[1]) / 1e3, ev[1].elapsed_time(ev[2]) / 1e3,
         ev[2].elapsed_time(ev[3]) / 1e3, ev[3].elapsed_time(ev[4]) / 1e3,
         ev[4].elapsed_time(ev[5]) / 1e3, ev[0].elapsed_time(ev[5]) / 1e3], world)
    # digest of the fp32 output: kernel (a)'s checksum of its bytes
    om = dev.ShardMap(np.array([(0, 4 * n, 0)], dtype=fabric.SEGMENT_DTYPE), dev.DEFAULT_BLOCK_BYTES)
    orows = om.new_row_sums()
    dev.checksum(om, res.view(torch.uint8), orows)
    digest = "%016x%016x" % (int(orows[0::2].sum().item()) % 2**64,
                             int(orows[1::2].sum().item()) % 2**64)
    lu = len(mine)
    out["reduce"] = {"elements": n, "units_total": REDUCE_UNITS, "units_this_rank": lu,
                     "frac_bits": f, "output_digest": digest,
                     "absmax_ms": round(t_amax * 1e3, 3),
                     "absmax_gbs": round(4 * n * lu / t_amax / 1e9, 1),  # one DRAM pass per unit
                     "global_max_and_scale_ms": round(t_max * 1e3, 3),
                     "fold_ms": round(t_fold * 1e3, 3),
                     # one launch reads every unit per element: units that
                     # alias the same data buffer are read from DRAM once
                     "fold_dram_gbs": round((4 * len(data) + 8) * n / t_fold / 1e9, 1),
                     "fold_units_read_gbs": round((4 * lu + 8) * n / t_fold / 1e9, 1),
                     "distinct_unit_buffers_this_rank": len(data),
                     "nccl_allreduce_int64_ms": round(t_ar * 1e3, 3) if world > 1 else None,
                     "dequant_ms": round(t_deq * 1e3, 3),
                     "dequant_gbs": round(12 * n / t_deq / 1e9, 1),
                     "nccl_path_ms": round(t_all * 1e3, 3)}
    # the same step with the scale kept in device memory: no host round trip
    # between the global max and the fold (ew_fixed_point_bits_async ->
    # ew_weighted_fold_dev -> ew_fixed_to_float_dev), same bits
    amax_d = torch.empty(1, dtype=torch.float64, device="cuda")
    bits_d = torch.empty(1, dtype=torch.int32, device="cuda")
    res_d = torch.empty(n, dtype=torch.float32, device="cuda")

    def reduce_step_dev():
        dev.weighted_absmax(units, w, out=amax_d)
        if world > 1:
            dist.all_reduce(amax_d, op=dist.ReduceOp.MAX)
        dev.fixed_point_bits_async(amax_d, REDUCE_UNITS, bits_d)
        dev.weighted_fold_dev(units, w, bits_d, acc)
        if world > 1:
            dist.all_reduce(acc)
        dev.fixed_to_float_dev(acc, bits_d, res_d)

    reduce_step_dev()
    torch.cuda.synchronize()
    barrier(world)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    reduce_step_dev()
    e.record()
    torch.cuda.synchronize()
    barrier(world)
    t_dev = max_over_ranks([s.elapsed_time(e) / 1e3], world)[0]
    same = torch.tensor([1 if (torch.equal(res_d, res) and int(bits_d.item()) == f) else 0],
                        device="cuda")
    if world > 1:
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
    out["reduce"].update({"device_scale_path_ms": round(t_dev * 1e3, 3),
                          "device_scale_bit_identical": bool(same.item())})
    del res_d
    del acc
    torch.cuda.empty_cache()
    if world > 1:
        # the same reduce fused with its collective over NVLink peer memory,
        # through the C++ runtime (recovery.PeerReduce): global scale (absmax
        # + max over the store) and reduce-scatter / all-gather between
        # device barriers, all inside the timed region, no NCCL
        from paper_2510_00606_b200.recovery import PeerReduce
        peer_out = torch.empty(n, dtype=torch.float32, device="cuda")
        pr = PeerReduce(peer_out, units, w)
        fp = pr.scale()
        pr.run(fp)
        pr.wait()
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier(world)
            s.record()
            fp = pr.scale()
            pr.run(fp)
            e.record()
            pr.wait()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e) / 1e3)
        assert not pr.timed_out(), "peer barrier timed out"
        t_peer = max_over_ranks([min(times)], world)[0]
        identical = bool(torch.equal(peer_out, res)) and fp == f
        ok = torch.tensor([1 if identical else 0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        out["reduce"].update({
            "peer_path_ms": round(t_peer * 1e3, 3),
            "peer_path_includes": "local absmax + global max over the store + scale + "
                                  "reduce-scatter + all-gather",
            "peer_vs_nccl_speedup": round(t_all / t_peer, 2),
            "peer_bit_identical_to_nccl": bool(ok.item())})
        barrier(world)
        pr.close()
        del peer_out
        torch.cuda.empty_cache()
        # world-size-invariant form over per-rank int64 accumulators (each
        # rank folded its own units during backward, accumulate=1): NCCL
        # int64 all-reduce + dequant vs the peer int64 reduce-scatter +
        # dequant + all-gather
        acc = torch.empty(n, dtype=torch.int64, device="cuda")
        dev.weighted_fold(units, w, f, acc)
        out64 = torch.empty(n, dtype=torch.float32, device="cuda")
        pr64 = PeerReduce(out64, acc=acc)
        pr64.run(f)
        pr64.wait()
        torch.cuda.synchronize()
        times = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier(world)
            s.record()
            pr64.run(f)
            e.record()
            pr64.wait()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e) / 1e3)
        assert not pr64.timed_out(), "peer barrier timed out"
        t_p64 = max_over_ranks([min(times)], world)[0]
        same = torch.tensor([1 if torch.equal(out64, res) else 0], device="cuda")
        dist.all_reduce(same, op=dist.ReduceOp.MIN)
        out["reduce"].update({
            "int64_accumulators": {
                "nccl_allreduce_plus_dequant_ms": round((t_ar + t_deq) * 1e3, 3),
                "peer_ms": round(t_p64 * 1e3, 3),
                "peer_speedup": round((t_ar + t_deq) / t_p64, 2),
                "peer_nvlink_gbs": round((world - 1) / world * 12 * n / t_p64 / 1e9, 1),
                "bit_identical": bool(same.item())}})
        barrier(world)
        pr64.close()
        del acc, out64
    del units, data, res
    torch.cuda.empty_cache()


# ------------------------------------------------------------------- arms ---

class LegGuard:
    """Keeps one failing or hung secondary leg from costing the whole line.

    The headline (snapshot + verify) is measured first; every later leg runs
    through `run`.  A leg that raises on any rank posts the error in the c10d
    store and that rank exits; a watchdog thread on every rank polls the store
    and the --deadline-s budget, and on either rank 0 prints the JSON gathered
    so far with an "incomplete" record (which leg, why) and every rank exits 0.
    Ranks blocked inside a collective of the broken leg are released by the
    exit rather than left to hang."""

    KEY = "ew_bench_abort"

    def __init__(self, args, rank, world, out, t_start):
        import threading
        self.rank, self.out, self.leg, self.done = rank, out, "snapshot", []
        self.emitted = False
        self.deadline = t_start + args.deadline_s
        self.json_out = args.json_out
        self.lock = threading.Lock()
        self.store = None
        if world > 1:
            from torch.distributed import distributed_c10d as c10d
            self.store = c10d._get_default_store()
        threading.Thread(target=self._watch, daemon=True).start()

    def _watch(self):
        while True:
            time.sleep(1.0)
            reason = None
            if time.time() > self.deadline:
                reason = f"deadline passed during leg {self.leg!r}"
            elif self.store is not None:
                try:
                    if self.store.check([self.KEY]):
                        reason = self.store.get(self.KEY).decode(errors="replace")
                except Exception:  # noqa: BLE001 - the store went away: peers are gone
                    reason = f"rendezvous store lost during leg {self.leg!r}"
            if reason:
                self.finish(reason)

    def finish(self, reason):
        with self.lock:
            if self.rank == 0 and not self.emitted:
                line = None
                for _ in range(5):  # the main thread may be writing `out`
                    try:
                        rec = dict(self.out)
                        rec["incomplete"] = {"reason": reason, "legs_done": list(self.done)}
                        line = json.dumps(rec)
                        break
                    except Exception:  # noqa: BLE001
                        time.sleep(0.05)
                if line is not None:
                    emit(line)
                    if self.json_out:
                        Path(self.json_out).write_text(line + "\n")
            sys.stdout.flush()
            sys.stderr.flush()
            os._exit(0)

    def run(self, name, fn, *a):
        self.leg = name
        try:
            fn(*a)
        except Exception as e:  # noqa: BLE001
            import traceback
            traceback.print_exc()
            msg = f"rank {self.rank} raised in leg {name!r}: {e!r}"[:600]
            if self.store is not None:
                try:  # a peer's failure may be the cause: report the first one
                    if self.store.check([self.KEY]):
                        msg = self.store.get(self.KEY).decode(errors="replace")
                    else:
                        self.store.set(self.KEY, msg)
                except Exception:  # noqa: BLE001
                    pass
            self.finish(msg)
        self.done.append(name)


def bench_b200(args):
    import torch
    rank, world, local = dist_setup(args)
    skip = set(filter(None, args.skip.split(",")))
    out = {}
    t_start = time.time()
    guard = LegGuard(args, rank, world, out, t_start)

    def trace(leg):
        if args.trace:
            print(f"[{time.time() - t_start:8.2f}s rank {rank}] {leg}", file=sys.stderr,
                  flush=True)

    trace("snapshot")
    m, live, snap, rows, bad, S, segs = run_snapshot(args, rank, world, local, out)
    if args.only_inplace:
        skip |= {"e2e", "cpu", "reshard", "replica", "replay", "migration", "config_c", "stage",
                 "philox", "reduce"}
    if "e2e" not in skip:
        trace("e2e")
        guard.run("e2e", run_e2e, args, rank, world, out, m, live, snap, rows, bad, S)
    del live, snap
    torch.cuda.empty_cache()
    if world > 1 and (args.inplace_state_gb > 0 or "inplace" not in skip):
        trace("inplace")
        guard.run("inplace", run_inplace, args, rank, world, out)
    if world > 1 and "config_d" not in skip and not args.only_inplace:
        trace("config_d_reshard")
        guard.run("config_d_reshard", run_config_d_reshard, args, rank, world, out)
    if world == 1 and rank == 0 and "cpu" not in skip:
        trace("cpu_baseline")
        guard.run("cpu_baseline", run_cpu_baseline, args, out, segs, S)
    if world > 1 and "reshard" not in skip:
        trace("reshard")
        guard.run("reshard", run_reshard, args, rank, world, out)
    if world > 1 and "host_replica" not in skip:
        trace("host_replica")
        guard.run("host_replica", run_host_replica, args, rank, world, out)
    if world > 1 and "replica" not in skip:
        trace("replica")
        guard.run("replica", run_replica, args, rank, world, out)
    if "replay" not in skip:
        trace("replay")
        guard.run("replay", run_replay, args, rank, world, out)
    if world > 1 and "migration" not in skip:
        trace("layer_migration")
        guard.run("layer_migration", run_layer_migration, args, rank, world, out)
    if world >= 4 and "config_c" not in skip:
        trace("config_c")
        guard.run("config_c", run_config_c, args, rank, world, out)
    if world > 1 and world % 2 == 0 and "stage" not in skip:
        trace("stage_move")
        guard.run("stage_move", run_stage_move, args, rank, world, out)
    if "philox" not in skip:
        trace("philox")
        guard.run("philox", run_philox, args, rank, world, out)
    if "reduce" not in skip:
        trace("reduce")
        guard.run("reduce", run_reduce, args, rank, world, out)
    if world == 1 and "config_a" not in skip:
        trace("config_a")
        guard.run("config_a", run_config_a, args, rank, world, out)
    if world == 1 and "config_d" not in skip:
        trace("config_d_snapshot")
        guard.run("config_d_snapshot", run_config_d_snapshot, args, rank, world, out)
    if world == 1 and rank == 0 and "cpu" not in skip:
        trace("cpu_beside")
        guard.run("cpu_beside", run_cpu_beside, args, out)  # cpu_baseline leg, continued
    guard.leg = "emit"
    if rank == 0:
        line = json.dumps(out)
        with guard.lock:
            emit(line)
            guard.emitted = True
        if args.json_out:
            Path(args.json_out).write_text(line + "\n")
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def bench_reference(args):
    """The reference arm: the CPU path on the host cores, rank 0 only (other
    ranks exit 0), on the GPU arm's exact workload and config — rank
    HEADLINE_SHARD_RANK's full config-B shard (11.79 GB).  The layout comes
    from the unmodified reference sources (oracle/_ref: ZeroLayout::shard
    composed per SURVEY A4); snapshot + verify is the oracle port on every
    host thread (the reference has no byte-moving snapshot or checksum).
    Nothing from the product package is imported or loaded here."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    from oracle.ew_oracle import load_oracle, load_reference

    orc, ref = load_oracle(), load_reference()
    if ref is None:
        raise SystemExit("oracle/_ref is not built (make -C oracle where /root/reference exists)")
    ivs = ref.interleaved(LLAMA2_7B_LAYER_BYTES, range(8))[HEADLINE_SHARD_RANK]
    segs, local = [], 0
    for lo, hi in ivs:
        segs.append({"global_lo": int(lo), "length": int(hi - lo), "local_off": local})
        local += int(hi - lo)
    S = local
    threads = len(os.sched_getaffinity(0))
    live = orc.fill_synthetic_mt(segs, S, 0, threads)
    snap = np.zeros_like(live)
    block = args.block_bytes
    for _ in range(args.warmup):
        sums = orc.snapshot_mt(segs, block, live, snap, threads)
        assert orc.verify_mt(segs, block, snap, sums, threads) == 0
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        sums = orc.snapshot_mt(segs, block, live, snap, threads)
        bad = orc.verify_mt(segs, block, snap, sums, threads)
        times.append(time.perf_counter() - t0)
        assert bad == 0, "reference arm: verification failed"
    step = sum(times) / len(times)
    value = round(3 * S / step / 1e9, 3)
    res = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step * 1e3, 3),
           "impl": "reference", "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "u64",
           "data": "synthetic (word i = splitmix64(seed ^ i))",
           "config": workload_config(S, block, args.gpus),
           "cpu_baseline": {"value": value, "unit": "GB/s", "cores": threads, "kind": "port",
                            "sample": f"the full rank-{HEADLINE_SHARD_RANK} config-B shard "
                                      f"({S} bytes) per step: oracle snapshot (memcpy + "
                                      "word-wise checksum) then verify re-read, layout from "
                                      "oracle/_ref (unmodified reference sources)"},
           "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    extra = {}
    cfg_pt = _llama2_7b_per_tensor_layer_bytes()
    for name, lb in (("per-layer", LLAMA2_7B_LAYER_BYTES), ("per-tensor", cfg_pt)):
        src = ref.interleaved(lb, range(8))
        dst = ref.interleaved(lb, [0, 1, 2, 4, 5, 6, 7])
        secs = []
        for _ in range(5):
            _, _, sec = ref.overlap_matrix(src, dst, sum(lb), [3], list(range(8)))
            secs.append(sec)
        extra[f"overlap_matrix_8to7_{name}_ms"] = round(min(secs) * 1e3, 3)
    t0 = time.perf_counter()
    ref.draw(0, 0, 1, 0, 4_000_000)
    extra["draw_muniform_per_s_1thread"] = round(4.0 / (time.perf_counter() - t0), 1)
    g = np.random.default_rng(5).normal(size=(5, 4_194_304))
    t0 = time.perf_counter()
    ref.weighted_grad_average(np.full(5, 0.2), g)
    dt = time.perf_counter() - t0
    extra["weighted_grad_average_gbs_1thread"] = round(5 * 4_194_304 * 8 / dt / 1e9, 2)
    res["reference_cpu"] = extra
    emit(json.dumps(res))
    if args.json_out:
        Path(args.json_out).write_text(json.dumps(res) + "\n")


def _llama2_7b_per_tensor_layer_bytes():
    h, f = 4096, 11008
    layers = [131_072_000]
    for _ in range(32):
        layers += [h * h] * 4 + [h * f] * 3 + [h, h]
    layers += [h, 131_072_000]
    return [14 * p for p in layers]


_JSON_FD = None


def quiet_stdout():
    """Route fd 1 to stderr for the whole run, so banners printed by native
    libraries (NCCL's version line at communicator init) cannot precede the
    JSON line; emit() writes that one line to the original stdout."""
    global _JSON_FD
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)


def emit(line):
    if _JSON_FD is None:
        print(line, flush=True)
    else:
        os.write(_JSON_FD, (line + "\n").encode())


def main():
    quiet_stdout()
    args = parse_args()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_b200(args)


if __name__ == "__main__":
    main()
