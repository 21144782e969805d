"""Time the product fold (ew_weighted_fold) at 1, 2, 4, 8 units per element
over the config-E 7B gradient (two distinct 27 GB unit buffers, aliased
round-robin as in bench.py's N = 1 reduce leg).  Prints min ms over reps.

  python tools/fold_sweep.py [--elems N] [--reps K]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch

from paper_2510_00606_b200 import device as dev


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--elems", type=int, default=6_738_415_616)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    n = args.elems
    bufs = [torch.empty(n, dtype=torch.float32, device="cuda").normal_(0, 1e-3) for _ in range(2)]
    acc = torch.empty(n, dtype=torch.int64, device="cuda")
    res = {}
    for nu in (1, 2, 4, 8):
        units = [bufs[k % 2] for k in range(nu)]
        w = [(k + 1) / 36 for k in range(nu)]
        f = dev.fixed_point_bits(dev.weighted_absmax(units, w).item(), nu)
        best = 1e9
        for _ in range(args.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            dev.weighted_fold(units, w, f, acc)
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        dram = (4 * min(nu, 2) + 8) * n
        res[nu] = {"ms": round(best, 3), "dram_gbs": round(dram / best / 1e6, 1),
                   "unit_elems_g_per_s": round(nu * n / best / 1e6, 1)}
    # the pre-pass and the dequant on one unit
    f = dev.fixed_point_bits(dev.weighted_absmax(bufs[:1], [1.0]).item(), 1)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn, moved in (("absmax", lambda: dev.weighted_absmax(bufs[:1], [1.0]), 4 * n),
                            ("dequant", lambda: dev.fixed_to_float(acc, f, out), 12 * n)):
        best = 1e9
        for _ in range(args.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e))
        res[name] = {"ms": round(best, 3), "gbs": round(moved / best / 1e6, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
