"""Lock-step check of the one-GPU in-place emulation against the numpy mover
(tests/test_inplace.py semantics): reports the first phase / rank / byte
range where the GPU buffers diverge."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np
import torch

from oracle.ew_oracle import load_oracle
from paper_2510_00606_b200 import configs, device as dev
from paper_2510_00606_b200.fabric import ROLE_NEW, ROLE_OLD, ROLE_REPLICA
from paper_2510_00606_b200.inplace import InPlaceSchedule
from paper_2510_00606_b200.reshard import ReshardPlan

orc = load_oracle()
cfg = configs.scaled(configs.gpt_125m(), 1e-2)
rp = ReshardPlan.build(cfg.layer_bytes, [0, 1, 2, 3], [0, 2, 3])
sc = InPlaceSchedule(rp, 1 << 16, 1 << 17, 1)
seed = 0
ranks = sorted(set(rp.old_ranks) | set(rp.new_ranks))
H, G, R, RG = {}, {}, {}, {}
for r in ranks:
    n_old = rp.src.shard_bytes(r) if r in rp.old_ranks else 0
    n_new = rp.dst.shard_bytes(r) if r in rp.new_ranks else 0
    b = np.full(max(n_old, n_new, 1), 0xA5, dtype=np.uint8)
    if n_old and r not in rp.failed:
        b[:n_old] = orc.fill_synthetic(rp.src.segments(r), n_old, seed)
    H[r] = b
    G[r] = dev.empty_bytes(len(b))
    G[r][:len(b)].copy_(torch.from_numpy(b))
    rep = rp.replica_of(r)
    if rep is not None and rep in rp.failed and r not in rp.failed:
        R[r] = orc.fill_synthetic(rp.src.segments(rep), rp.src.shard_bytes(rep), seed)
        RG[r] = dev.empty_bytes(len(R[r]))
        RG[r][:len(R[r])].copy_(torch.from_numpy(R[r]))
table = {(ROLE_OLD, r): G[r].data_ptr() for r in ranks}
table.update({(ROLE_REPLICA, r): t.data_ptr() for r, t in RG.items()})
nt = max(ranks) + 1
stg = {r: [dev.empty_bytes(max(16, sc.stage_alloc)) for _ in range(sc.ring)] for r in rp.new_ranks}
hst = {r: [np.zeros(max(16, sc.stage_alloc), np.uint8) for _ in range(sc.ring)] for r in rp.new_ranks}
descs = {r: rp.copies(r, push=False) for r in rp.new_ranks}
n = len(sc.phases)


def run_np(part, target, r):
    for c in part:
        s = int(c["src_rank"])
        src = H[s] if int(c["src_role"]) == ROLE_OLD else R[s]
        nb, so, do = int(c["bytes"]), int(c["src_off"]), int(c["dst_off"])
        target[do:do + nb] = src[so:so + nb]


for j in range(n):
    for r in rp.new_ranks:
        for jj in range(j + 1, min(n, j + sc.slack + 1)):
            lo, hi = sc.direct[r][jj]
            H[r][lo:hi] = 0xEE
            if hi > lo:
                G[r][lo:hi].fill_(0xEE)
    for r in rp.new_ranks:
        lo, hi = sc.staged[r][j]
        st = stg[r][j % sc.ring]
        if hi > lo:
            sd = sc.staged_descs(r, j, descs[r])
            t = dict(table)
            t[(ROLE_NEW, r)] = st.data_ptr()
            dev.CopyProgram.from_descs(sd, t, nt, r).launch()
            run_np(sd, hst[r][j % sc.ring], r)
        dd = sc.direct_descs(r, j, descs[r])
        if len(dd):
            t = dict(table)
            t[(ROLE_NEW, r)] = G[r].data_ptr()
            dev.CopyProgram.from_descs(dd, t, nt, r).launch()
            run_np(dd, H[r], r)
    torch.cuda.synchronize()
    for r in rp.new_ranks:
        lo, hi = sc.staged[r][j]
        if hi > lo:
            pad = lo % 16
            a = stg[r][j % sc.ring][pad:pad + hi - lo].cpu().numpy()
            b = hst[r][j % sc.ring][pad:pad + hi - lo]
            if not np.array_equal(a, b):
                k = np.nonzero(a != b)[0]
                print("staging diverges", j, r, (lo, hi), k[:5], len(k))
                sys.exit(1)
            dev.CopyProgram.from_pointers([stg[r][j % sc.ring].data_ptr() + pad],
                                          [G[r].data_ptr() + lo], [hi - lo], [False]).launch(64, 0)
            H[r][lo:hi] = hst[r][j % sc.ring][pad:pad + hi - lo]
    torch.cuda.synchronize()
    for r in ranks:
        a = G[r][:len(H[r])].cpu().numpy()
        if not np.array_equal(a, H[r]):
            k = np.nonzero(a != H[r])[0]
            print("buffer diverges after phase", j, "rank", r, "first", k[:5], "count", len(k),
                  "cuts", sc.cuts.get(r, [None] * n)[j], sc.direct.get(r, [None] * n)[j],
                  sc.staged.get(r, [None] * n)[j])
            sys.exit(1)
print("lock-step OK over", n, "phases")
