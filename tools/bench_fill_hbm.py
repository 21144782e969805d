"""Config D on one GPU: ZeRO state sized to fill the B200's HBM.

Per GPU the live shard S and its snapshot must fit: S = --shard-gb (default
86 GB, live + snapshot = 172 GB of the 179 GiB).  Runs snapshot + verify
steps exactly like bench.py (same kernels, CUDA-event timing) and checks a
flipped bit is caught.  Prints one JSON line."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2510_00606_b200 import configs, device as dev, fabric


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shard-gb", type=float, default=86.0)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    S_target = int(args.shard_gb * 1e9)
    cfg = configs.fill_hbm(8, S_target)  # 8-way interleaved, 80 layers
    layout = fabric.interleaved_layout(cfg.layer_bytes, range(8))
    m = dev.ShardMap(layout.segments(3), 65536)
    S = layout.shard_bytes(3)
    live = dev.empty_bytes(S)
    snap = dev.empty_bytes(S)
    rows = m.new_row_sums()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    dev.fill_synthetic(m, live, 7)
    dev.snapshot(m, live, snap, rows)
    dev.verify(m, snap, rows, bad)
    torch.cuda.synchronize()
    assert int(bad.item()) == 0
    s, mid, e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_snap = t_ver = 0.0
    for _ in range(args.steps):
        s.record()
        dev.snapshot(m, live, snap, rows)
        mid.record()
        dev.verify(m, snap, rows, bad)
        e.record()
        torch.cuda.synchronize()
        t_snap += s.elapsed_time(mid) / 1e3
        t_ver += mid.elapsed_time(e) / 1e3
    t_snap /= args.steps
    t_ver /= args.steps
    ok = int(bad.item()) == 0
    snap[S // 3] ^= 0x40
    dev.verify(m, snap, rows, bad)
    torch.cuda.synchronize()
    caught = int(bad.item()) == 1
    free, total = torch.cuda.mem_get_info()
    print(json.dumps({"config": "D fill-HBM", "shard_bytes": S, "hbm_total": total,
                      "hbm_free_after_alloc": free, "snapshot_ms": round(t_snap * 1e3, 2),
                      "verify_ms": round(t_ver * 1e3, 2),
                      "snapshot_gbs": round(2 * S / t_snap / 1e9, 1),
                      "verify_gbs": round(S / t_ver / 1e9, 1),
                      "step_gbs": round(3 * S / (t_snap + t_ver) / 1e9, 1),
                      "verified": ok, "flipped_bit_caught": caught}))


if __name__ == "__main__":
    main()
