"""Host-memory snapshots as the H2D_D2D source (hostsnap.HostSnapshots):
every rank publishes its shard into node-shared pinned memory, then each
departure is recovered with the departed rank's bytes pulled from host
memory by the destinations' copy kernels (verified on arrival) while the
survivors' bytes move over NVLink.  2 or 4 GPUs, one process per GPU."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_dir):
    import json
    import sys
    from pathlib import Path
    import torch.distributed as dist
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.hostsnap import HostSnapshots
    from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    report = {}
    hs = None
    try:
        cfg = configs.scaled(configs.llama2_7b_per_tensor(), 2e-3)
        members = list(range(world))
        src = ReshardPlan.build(cfg.layer_bytes, members, members).src
        live = dev.empty_bytes(src.shard_bytes(rank))
        dev.fill_synthetic(shard_map(src, rank), live, 41)
        hs = HostSnapshots(src, members, rank, tag=f"t{port}")
        hs.publish(live)
        torch.cuda.synchronize()
        dist.barrier()
        n = src.shard_bytes(rank)
        report["own image == live"] = bool(torch.equal(hs.image(rank), live[:n].cpu()))
        for d in members:
            rp = ReshardPlan.build(cfg.layer_bytes, members, [r for r in members if r != d])
            ex = ReshardExecutor(rp, rank, push=False)
            bufs = ex.allocate(device_replica=False)
            report[f"drop{d} no device replica"] = bufs.replica is None
            if bufs.old is not None:
                bufs.old[:n].copy_(live[:n])
            if bufs.new is not None:
                bufs.new.fill_(0x5A)
            hs.attach(ex, [d])
            dist.barrier()
            ex.bind(bufs, verify=True)
            nblocks = (sum(cfg.layer_bytes) + 65535) // 65536
            sums = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
            dist.barrier()
            ex.launch(block_sums=sums)
            torch.cuda.synchronize()
            dist.barrier()
            if bufs.new is not None:
                m = rp.dst.shard_bytes(rank)
                exp = dev.empty_bytes(m)
                dev.fill_synthetic(shard_map(rp.dst, rank), exp, 41)
                report[f"drop{d} bytes"] = bool(torch.equal(bufs.new[:m], exp[:m]))
            ex.close()
            dist.barrier()
    except Exception as e:  # report, do not hang the other ranks
        report["error"] = repr(e)
    finally:
        if hs is not None:
            dist.barrier()
            hs.close()
    Path(result_dir, f"rank{rank}.json").write_text(json.dumps(report))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 4])
def test_host_snapshot_recovery(world, tmp_path):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import json
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        rep = json.loads((tmp_path / f"rank{r}.json").read_text())
        assert "error" not in rep, rep
        assert rep and all(v is True for v in rep.values()), (r, rep)
