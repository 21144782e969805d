"""Snapshot bandwidth vs shard size on one GPU (config D follow-up).

At 86 GB the snapshot kernel measured 5.7 TB/s against 6.26 TB/s at the 7B
shard (11.8 GB).  This probe times, per size, the snapshot kernel (one launch
over the whole shard, and the same bytes as 8 launches over contiguous
chunks), the verify kernel and torch's own copy_ of the same bytes, so the
size effect can be attributed to the hardware (every copy slows) or to the
kernel.  Prints one JSON line per size."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np
import torch

from paper_2510_00606_b200 import configs, device as dev, fabric


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-gb", default="11.8,24,48,86")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    for gb in [float(x) for x in args.sizes_gb.split(",")]:
        cfg = configs.fill_hbm(8, int(gb * 1e9))
        layout = fabric.interleaved_layout(cfg.layer_bytes, range(8))
        segs = layout.segments(3)
        S = layout.shard_bytes(3)
        m = dev.ShardMap(segs, 65536)
        live = dev.empty_bytes(S)
        snap = dev.empty_bytes(S)
        rows = m.new_row_sums()
        bad = torch.zeros(1, dtype=torch.int32, device="cuda")
        dev.fill_synthetic(m, live, 7)
        t_one = timed(lambda: dev.snapshot(m, live, snap, rows), args.reps)
        t_ver = timed(lambda: dev.verify(m, snap, rows, bad), args.reps)
        # 8 chunks of consecutive segments (10 of the 80 layers each)
        chunks = []
        segs_np = np.asarray(segs)
        per = (len(segs_np) + 7) // 8
        for c in range(0, len(segs_np), per):
            sub = segs_np[c:c + per].copy()
            lo = int(sub["local_off"][0])
            sub["local_off"] -= lo
            nb = int(sub["local_off"][-1] + sub["length"][-1])
            cm = dev.ShardMap(sub, 65536)
            chunks.append((cm, live[lo:lo + nb], snap[lo:lo + nb], cm.new_row_sums()))

        def chunked():
            for cm, a, b, r in chunks:
                dev.snapshot(cm, a, b, r)

        t_chunk = timed(chunked, args.reps)
        t_torch = timed(lambda: snap.copy_(live), args.reps)
        torch.cuda.synchronize()
        print(json.dumps({"shard_gb": round(S / 1e9, 2),
                          "snapshot_one_launch_gbs": round(2 * S / t_one / 1e9, 1),
                          "snapshot_8_launches_gbs": round(2 * S / t_chunk / 1e9, 1),
                          "torch_copy_gbs": round(2 * S / t_torch / 1e9, 1),
                          "verify_gbs": round(S / t_ver / 1e9, 1)}), flush=True)
        del chunks, live, snap, rows, m
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
