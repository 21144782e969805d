"""Grid sweep of the reshard copy kernel's local class: rank 2's pull program
of the 4 -> 3 departure of rank 3 at 7B-per-GPU (all 15.72 GB of it local:
its own retained bytes and its replica of rank 3, the program that bounds the
replica-aware MTTR), verified and plain, n_ctas through the launch argument.

  python tools/local_copy_sweep.py [--reps K]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.fabric import ROLE_NEW, ROLE_OLD, ROLE_REPLICA
from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    base = configs.llama2_7b()
    lb = [x * 4 // 8 for x in base.layer_bytes]
    rp = ReshardPlan.build(lb, [0, 1, 2, 3], [0, 1, 2])
    me = 2
    b = ReshardExecutor(rp, me).allocate()
    dev.fill_synthetic(shard_map(rp.src, me), b.old, 0)
    dev.fill_synthetic(shard_map(rp.src, rp.replica_of(me)), b.replica, 0)
    table = {(ROLE_OLD, me): b.old.data_ptr(), (ROLE_REPLICA, me): b.replica.data_ptr(),
             (ROLE_NEW, me): b.new.data_ptr()}
    descs = rp.copies(me, push=False)
    assert set(descs["src_rank"].tolist()) == {me}, "rank 2's program is all local"
    m_new = shard_map(rp.dst, me)
    prog = dev.CopyProgram.from_descs(descs, table, 4, me, m_new)
    nblocks = (sum(lb) + 65535) // 65536
    sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
    n = rp.dst.shard_bytes(me)
    moved = 2 * n
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    res = {"bytes_landed": n}
    for verified in (True, False):
        for mult in (0, 2.5, 3, 4, 5):
            n_ctas = int(mult * sms)
            best = 1e9
            for _ in range(args.reps):
                if verified:
                    sums.zero_()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                prog.launch(n_ctas=n_ctas, block_sums=sums if verified else None)
                e.record()
                torch.cuda.synchronize()
                best = min(best, s.elapsed_time(e))
            res[f"{'verified' if verified else 'plain'}_ctas_{n_ctas or 'default'}"] = {
                "ms": round(best, 3), "tbps": round(moved / best / 1e9, 3)}
    exp = dev.empty_bytes(n)
    dev.fill_synthetic(m_new, exp, 0)
    res["landed_equal"] = bool(torch.equal(b.new[:n], exp[:n]))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
