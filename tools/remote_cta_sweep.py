"""Sweep the reshard copy kernel's CTA split on the NVLink-bound receiver:
one process drives every GPU (peer access over NVSwitch), builds the 4 -> 3
departure of rank 3 at 7B-per-GPU, and times receiver GPU 1's verified pull
program (7.86 GB over NVLink from GPU 2, 7.86 GB local) alone and with every
receiver running concurrently, for several (n_ctas, remote_ctas) choices.

  python tools/remote_cta_sweep.py    # needs >= 4 GPUs
"""
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
    world = 4
    assert torch.cuda.device_count() >= world
    for r in range(world):
        check(lib.ew_set_device(r))
        for s in range(world):
            if s != r:
                check(lib.ew_peer_access_enable(s))
    base = configs.llama2_7b()
    lb = [x * world // 8 for x in base.layer_bytes]
    rp = ReshardPlan.build(lb, list(range(world)), [0, 1, 2])
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
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    bott = rp.traffic()["ingress"][1]

    def run(cfgs, concurrent, src_ctas=0):
        best = 1e9
        for _ in range(4):
            ev = {}
            for r in (rp.new_ranks if concurrent else [1]):
                with torch.cuda.device(r):
                    sums[r].zero_()
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    n, rem = cfgs if r == 1 else ((src_ctas, 0) if r == 2 else (0, 0))
                    s.record()
                    progs[r].launch(n_ctas=n, remote_ctas=rem, block_sums=sums[r])
                    e.record()
                    ev[r] = (s, e)
            for r in range(world):
                torch.cuda.synchronize(r)
            best = min(best, ev[1][0].elapsed_time(ev[1][1]))
        return best

    res = {"receiver": 1, "nvlink_bytes": bott}
    for n_mult, rem_mult in ((0, 0), (1.5, 0.5), (1.5, 0.75), (2, 1), (2.5, 1), (3, 1.5), (2, 0.5),
                             (3, 1)):
        cfg = (int(n_mult * sms), int(rem_mult * sms))
        key = "default" if n_mult == 0 else f"n{cfg[0]}_remote{cfg[1]}"
        alone = run(cfg, False)
        conc = run(cfg, True)
        res[key] = {"alone_ms": round(alone, 3), "concurrent_ms": round(conc, 3),
                    "concurrent_gbs": round(bott / conc / 1e6, 1)}
    # the source GPU 2 runs its own all-local program meanwhile: fewer CTAs
    # there leave its HBM and L2 to the peer reads it serves
    for src in (592, 296, 148, 74):
        conc = run((0, 0), True, src_ctas=src)
        res[f"source_gpu2_ctas_{src}"] = {"gpu1_concurrent_ms": round(conc, 3),
                                          "concurrent_gbs": round(bott / conc / 1e6, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
