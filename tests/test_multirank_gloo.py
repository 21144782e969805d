"""N > 1 host plumbing on CPU (gloo, world size 2 and 3): every rank plans the
same membership change independently and must agree bit-for-bit; the copy
programs lowered on each rank must together execute every plan byte exactly
once (pull and push give the same byte moves)."""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import json
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    from paper_2510_00606_b200 import configs, fabric
    from paper_2510_00606_b200.reshard import ReshardPlan

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.scaled(configs.llama2_7b_per_tensor(), 1e-3)
    res = {}
    for drop in range(world):
        old = list(range(world))
        new = [r for r in old if r != drop]
        rp = ReshardPlan.build(cfg.layer_bytes, old, new)
        e = rp.plan.entries
        digest = hashlib.sha256(np.ascontiguousarray(
            np.stack([e["src_rank"], e["dst_rank"], e["lo"], e["hi"], e["medium"]], 1)
            .astype(np.int64)).tobytes()).hexdigest()
        mine = {}
        for push in (True, False):
            c = rp.copies(rank, push) if rank not in rp.failed else []
            mine[push] = sorted((int(x["src_role"]), int(x["src_rank"]), int(x["src_off"]),
                                 int(x["dst_rank"]), int(x["dst_off"]), int(x["bytes"])) for x in c)
        gathered = [None] * world
        dist.all_gather_object(gathered, (digest, mine[True], mine[False]))
        res[f"drop{drop}_same_plan"] = len({g[0] for g in gathered}) == 1
        push_all = sorted(x for g in gathered for x in g[1])
        pull_all = sorted(x for g in gathered for x in g[2])
        res[f"drop{drop}_push_equals_pull"] = push_all == pull_all
        # every target byte covered once
        cover = {r: np.zeros(rp.dst.shard_bytes(r), dtype=np.int32) for r in rp.new_ranks}
        for (_, _, _, d, off, n) in push_all:
            cover[d][off:off + n] += 1
        res[f"drop{drop}_exactly_once"] = all(bool((v == 1).all()) for v in cover.values())
        # the communicator edit agrees across ranks too
        pool = {(a, b) for a in old for b in old if a < b}
        ed = fabric.plan_edit([fabric.CommGroup("dp", old)], fabric.FAIL_STOP, [drop], pool)
        edits = [None] * world
        dist.all_gather_object(edits, sorted(ed.links_to_remove))
        res[f"drop{drop}_same_edit"] = all(x == edits[0] for x in edits)
    Path(out_dir, f"r{rank}.json").write_text(json.dumps(res))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_agree_and_cover(world, tmp_path):
    import json
    mp.spawn(_worker, args=(world, _port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        res = json.loads((tmp_path / f"r{r}.json").read_text())
        assert res and all(res.values()), res
