"""Time ew_snapshot / ew_checksum / ew_verify on config B's 7B rank-0 shard
(11.79 GB, misaligned segments), best of --reps; used by
tools/snapshot_sweep.sh to compare kernel shapes.  Prints one JSON line."""
import argparse
import hashlib
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.reshard import ReshardPlan


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--tag", default="")
    ap.add_argument("--aligned", action="store_true",
                    help="one segment at global 0 of the same size (no realignment)")
    args = ap.parse_args()
    base = configs.llama2_7b()
    rp = ReshardPlan.build(base.layer_bytes, list(range(8)), list(range(7)))
    segs = rp.src.segments(0)
    if args.aligned:
        import numpy as np
        from paper_2510_00606_b200 import fabric
        n = int(segs["length"].sum())
        segs = np.array([(0, n, 0)], dtype=fabric.SEGMENT_DTYPE)
    m = dev.ShardMap(segs, 65536)
    live = dev.empty_bytes(m.nbytes)
    dev.fill_synthetic(m, live, 0)
    snap = dev.empty_bytes(m.nbytes)
    rows = m.new_row_sums()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = {"tag": args.tag, "bytes": m.nbytes}
    for name, fn in (("snapshot", lambda: dev.snapshot(m, live, snap, rows)),
                     ("checksum", lambda: dev.checksum(m, live, rows)),
                     ("verify", lambda: dev.verify(m, snap, rows, bad))):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(args.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        moved = 2 * m.nbytes if name == "snapshot" else m.nbytes
        res[name + "_ms"] = round(best, 4)
        res[name + "_gbs"] = round(moved / best / 1e6, 1)
    res["verify_bad"] = int(bad.item())
    res["snap_equal"] = bool(torch.equal(snap[:m.nbytes], live[:m.nbytes]))
    res["rows_sha"] = hashlib.sha256(rows.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
