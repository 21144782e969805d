"""The multi-rank recovery path on ONE GPU: N = 4 and N = 8 processes share
cuda:0, meet on gloo (plumbing: the c10d store behind the C++ rendezvous) and
map each other's buffers with CUDA IPC, which works between processes on the
same device.  No NCCL (it refuses duplicate GPUs).  Everything the
one-process-per-GPU deployment runs across processes runs here, through the
C++ runtime (include/elaskit/recovery.hpp):

  * PreparedRecovery: every departure position of N -> N-1, pull programs
    verified on arrival, device barrier, checksum conservation reduce-
    scattered over peer memory; landed bytes == the target layout's bytes;
  * DpGroup: the same departure planned at failure time (survivor channel,
    IPC mapping, copy, verification) with the MttrEvent / mttr.csv record;
  * InPlaceExecutor (config D): OLD and NEW in one buffer, phases behind
    device barriers, departures and a rejoin, the barrier never timing out;
  * PeerReduce: (d) with its collective over peer memory (fp32 units and
    int64 accumulators, device barriers, the global scale over the store),
    bit-identical to the single-process fold;
  * ReplayReplica: the holder replays the owner's AdamW step from the
    owner's gradient read through an IPC pointer, byte-identical;
  * host-memory images (hostsnap, double-buffered) as the departed rank's
    H2D_D2D source.

Bandwidth numbers need one process per GPU (test_gpu_multigpu.py, bench.py);
this file proves the cross-process control and data paths on any 1-GPU box.
Reference: overlap_matrix / integrity_check (param_fabric.cpp:82-121),
remap_time (sim.cpp:452-483), recover_elaswave (sim.cpp:597-722)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fill_expected(dev, shard_map, layout, rank, seed, n):
    e = dev.empty_bytes(n)
    dev.fill_synthetic(shard_map(layout, rank), e, seed)
    return e


def _worker(rank, world, port, out_dir, scale):
    import json
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.reshard import RankBuffers, ReshardExecutor, ReshardPlan, shard_map

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rep = {}
    try:
        cfg = configs.scaled(configs.llama2_7b_per_tensor(), scale)
        members = list(range(world))
        lay = ReshardPlan.build(cfg.layer_bytes, members, members).src
        block = 65536

        # ---- PreparedRecovery: every departure position, C++ end to end
        from paper_2510_00606_b200.recovery import PreparedRecovery
        live = dev.empty_bytes(lay.shard_bytes(rank))
        m0 = shard_map(lay, rank, block)
        dev.fill_synthetic(m0, live, 31)
        rows = m0.new_row_sums()
        snap = dev.empty_bytes(lay.shard_bytes(rank))
        dev.snapshot(m0, live, snap, rows)          # the per-step snapshot rows
        succ = (rank + 1) % world
        replica = dev.empty_bytes(lay.shard_bytes(succ))
        ms = shard_map(lay, succ, block)
        dev.fill_synthetic(ms, replica, 31)
        rep_rows = ms.new_row_sums()
        dev.checksum(ms, replica, rep_rows)
        torch.cuda.synchronize()
        # replica-aware sourcing too: bytes the plan pulls from the
        # successor's OLD shard come from this rank's replica of it
        for local in (False, True):
            prep = PreparedRecovery(cfg.layer_bytes, members, rank, live, replica, block,
                                    old_rows=rows, replica_rows=rep_rows, local_replicas=local)
            tag = "local-replica " if local else ""
            for d in members:
                dist.barrier()
                if rank == d:
                    continue
                ev = prep.recover(d)
                torch.cuda.synchronize()
                n = prep.plans[d].dst.shard_bytes(rank)
                exp = _fill_expected(dev, shard_map, prep.plans[d].dst, rank, 31, n)
                rep[f"{tag}prepared drop{d} verified"] = ev.verified
                rep[f"{tag}prepared drop{d} bytes"] = bool(torch.equal(prep.new_view(d)[:n],
                                                                        exp[:n]))
                rep[f"{tag}prepared drop{d} no barrier timeout"] = \
                    ev.phases.get("barrier_timeouts") == 0
            if local:
                break
            dist.barrier()
            prep.close()
        # a corrupted landing must be caught: poison a survivor's source
        # byte after the snapshot rows were taken, then recover again
        dist.barrier()
        bad_drop = world - 1
        if rank == 0:
            live[12345] ^= 0x40
        torch.cuda.synchronize()
        dist.barrier()
        if rank != bad_drop:
            ev = prep.recover(bad_drop)
            rep["corruption detected (not verified)"] = not ev.verified
        dist.barrier()
        if rank == 0:
            live[12345] ^= 0x40
        torch.cuda.synchronize()
        dist.barrier()
        prep.close()

        # ---- DpGroup: plan at failure time, survivors only, MTTR record
        from paper_2510_00606_b200.recovery import DpGroup
        from paper_2510_00606_b200.fabric import FAIL_STOP
        drop = 1 % world
        rp = ReshardPlan.build(cfg.layer_bytes, members, [m for m in members if m != drop])
        grp = DpGroup(cfg.layer_bytes, members, rank, None)
        bufs = RankBuffers(live, replica if succ == drop else None,
                           dev.empty_bytes(rp.dst.shard_bytes(rank)) if rank != drop else None)
        dist.barrier()
        if rank != drop:
            ev = grp.recover([drop], bufs, step=5, kind=FAIL_STOP)
            n = rp.dst.shard_bytes(rank)
            exp = _fill_expected(dev, shard_map, rp.dst, rank, 31, n)
            rep["dp_group verified"] = ev.verified
            rep["dp_group bytes"] = bool(torch.equal(bufs.new[:n], exp[:n]))
            rep["dp_group members"] = grp.members == [m for m in members if m != drop]
            rep["dp_group csv"] = ev.csv_row(0).startswith("0,5,0,fail_stop,")
            rep["dp_group microbatches conserve the batch"] = \
                sum(grp.mb_sizes) == 4 * world
        dist.barrier()
        grp.close()

        # ---- the snapshot ring's step tag is enforced: one survivor's state
        # is of step 7 while the event is at step 8 -> every verdict fails
        grp = DpGroup(cfg.layer_bytes, members, rank, None)
        grp.set_snapshot_step(7 if rank == 0 else 8)
        bufs = RankBuffers(live, replica if succ == drop else None,
                           dev.empty_bytes(rp.dst.shard_bytes(rank)) if rank != drop else None)
        dist.barrier()
        if rank != drop:
            ev = grp.recover([drop], bufs, step=8, kind=FAIL_STOP)
            rep["stale snapshot fails the verdict"] = not ev.verified
            rep["stale snapshot counted once"] = ev.phases.get("stale_snapshots") == 1.0
        dist.barrier()
        grp.close()

        # ---- two non-adjacent members leave at once (ScaleIn), planned at
        # failure time: integrity_check passes (their holders survive), the
        # copy sources both departed shards from their ring holders
        from paper_2510_00606_b200.fabric import SCALE_IN, SCALE_OUT
        gone = [0, 2]
        survivors = [m for m in members if m not in gone]
        rp = ReshardPlan.build(cfg.layer_bytes, members, survivors)
        grp = DpGroup(cfg.layer_bytes, members, rank, None)
        holds = rp.replica_of(rank) in gone
        bufs = RankBuffers(live, replica if holds else None,
                           dev.empty_bytes(rp.dst.shard_bytes(rank)) if rank in survivors else None)
        # steady state: IPC mapping, the per-step snapshot rows as the source
        # sums, and this rank's program for the expected pair bound ahead
        grp.premap(RankBuffers(live, replica, None), rows, rep_rows)
        grp.prepare_move(SCALE_IN, gone, bufs.new)
        dist.barrier()
        if rank in survivors:
            try:
                grp.recover([survivors[0]], bufs, kind=SCALE_OUT)
                rep["scale-out of a member rejected"] = False
            except ValueError:
                rep["scale-out of a member rejected"] = True
            ev = grp.recover(gone, bufs, step=9, kind=SCALE_IN)
            n = rp.dst.shard_bytes(rank)
            exp = _fill_expected(dev, shard_map, rp.dst, rank, 31, n)
            rep["two departures verified"] = ev.verified
            rep["two departures bytes"] = bool(torch.equal(bufs.new[:n], exp[:n]))
            rep["two departures kind"] = ev.kind == "scale_in"
            rep["two departures used the steady-state mapping"] = ev.phases.get("premapped") == 1.0
            rep["two departures launched the prepared program"] = ev.phases.get("prepared") == 1.0
        dist.barrier()

        # ---- ...and rejoin (ScaleOut, config C's 6 -> 8): the departed
        # processes come back as joiners from the free pool; members re-cut
        # their shards over the grown group, joiners only receive
        rpj = ReshardPlan.build(cfg.layer_bytes, survivors, members)
        new_j = dev.empty_bytes(rpj.dst.shard_bytes(rank))
        if rank in gone:
            g2 = DpGroup.joiner(cfg.layer_bytes, survivors, rank, grp.name)
            ev = g2.admit(gone, RankBuffers(None, None, new_j), step=10)
        else:
            g2 = grp
            ev = g2.admit(gone, RankBuffers(bufs.new, None, new_j), step=10)
        n = rpj.dst.shard_bytes(rank)
        exp = _fill_expected(dev, shard_map, rpj.dst, rank, 31, n)
        rep["rejoin verified"] = ev.verified
        rep["rejoin bytes"] = bool(torch.equal(new_j[:n], exp[:n]))
        rep["rejoin kind"] = ev.csv_row(0).startswith("0,10,0,scale_out,")
        rep["rejoin members"] = g2.members == members
        rep["rejoin mapped at the event"] = ev.phases.get("premapped") == 0.0
        rep["rejoin microbatches conserve the batch"] = sum(g2.mb_sizes) == 4 * world
        # the grown group recovers a later departure (channels of the new
        # membership, event counters agreed with the joiners)
        d3 = members[-1]
        rp3 = ReshardPlan.build(cfg.layer_bytes, members, [m for m in members if m != d3])
        holder3 = members[members.index(d3) - 1]  # SnapshotRing::backed_up_by
        rep3 = None
        if rank == holder3:
            rep3 = _fill_expected(dev, shard_map, rpj.dst, d3, 31, rpj.dst.shard_bytes(d3))
        dist.barrier()
        if rank != d3:
            new3 = dev.empty_bytes(rp3.dst.shard_bytes(rank))
            ev = g2.recover([d3], RankBuffers(new_j, rep3, new3), step=11, kind=FAIL_STOP)
            n = rp3.dst.shard_bytes(rank)
            exp = _fill_expected(dev, shard_map, rp3.dst, rank, 31, n)
            rep["departure after rejoin verified"] = ev.verified
            rep["departure after rejoin bytes"] = bool(torch.equal(new3[:n], exp[:n]))
        dist.barrier()
        if g2 is not grp:
            g2.close()
        grp.close()

        # ---- staged in-place reshard (C++ InPlaceExecutor): departures and a rejoin
        from paper_2510_00606_b200.inplace import StagedInPlaceReshard
        nblk = (cfg.total_bytes + block - 1) // block
        for drop in sorted({0, world // 2, world - 1}):
            for old, new in ((members, [r for r in members if r != drop]),
                             ([r for r in members if r != drop], members)):
                rp = ReshardPlan.build(cfg.layer_bytes, old, new)
                stage = max(1 << 16, max(rp.dst.shard_bytes(r) for r in new) // 7)
                ex = StagedInPlaceReshard(rp, rank, stage_bytes=stage, block_bytes=block,
                                          phase_bytes=2 * stage, slack=1 + drop % 2)
                bufs = ex.allocate()
                before = torch.zeros(2 * nblk, dtype=torch.int64, device="cuda")
                if bufs.old is not None:
                    mo = shard_map(rp.src, rank, block)
                    dev.fill_synthetic(mo, bufs.old, 17)
                    r0 = mo.new_row_sums()
                    dev.checksum(mo, bufs.old, r0)
                    dev.rows_to_blocks(mo, r0, before)
                if bufs.replica is not None:
                    dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank), block),
                                       bufs.replica, 17)
                torch.cuda.synchronize()
                b_all = before.cpu()
                dist.all_reduce(b_all)
                ex.bind(bufs, None)
                after = torch.zeros(2 * nblk, dtype=torch.int64, device="cuda")
                dist.barrier()
                ex.launch(after)
                torch.cuda.synchronize()
                a_all = after.cpu()
                dist.all_reduce(a_all)
                tag = f"in-place {len(old)}->{len(new)} r{drop}"
                ok = bool(torch.equal(b_all, a_all)) and len(ex.sched.phases) > 2
                if rank in new:
                    n = rp.dst.shard_bytes(rank)
                    exp = _fill_expected(dev, shard_map, rp.dst, rank, 17, n)
                    ok = ok and bool(torch.equal(bufs.new[:n], exp[:n]))
                    rep[tag + " no barrier timeout"] = not ex.timed_out()
                rep[tag] = ok
                dist.barrier()
                ex.close()
                del bufs
                dist.barrier()

        # ---- (d) over peer memory through the C++ runtime (recovery.PeerReduce):
        # fp32 units and int64 accumulators, device barriers, no NCCL
        from paper_2510_00606_b200.recovery import PeerReduce
        n_units, dim = 2 * world, 100_003
        rng = np.random.default_rng(21)
        g = rng.normal(0, 1e-3, size=(n_units, dim)).astype(np.float32)
        g[3, 5] = 1e2
        w = rng.random(n_units) / n_units
        mine = [u for u in range(n_units) if u % world == rank]
        units = [torch.from_numpy(g[u]).cuda() for u in mine]
        out = torch.empty(dim, dtype=torch.float32, device="cuda")
        pr = PeerReduce(out, units, [w[u] for u in mine], barrier_timeout_s=60.0)
        f = pr.scale()
        all_units = [torch.from_numpy(x).cuda() for x in g]
        f1 = dev.fixed_point_bits(dev.weighted_absmax(all_units, w).item(), n_units)
        rep["peer reduce scale == single-GPU scale"] = f == f1 and pr.total_units == n_units
        acc1 = torch.empty(dim, dtype=torch.int64, device="cuda")
        dev.weighted_fold(all_units, w, f, acc1)
        single = dev.fixed_to_float(acc1, f)
        for _ in range(2):
            pr.run(f)
        pr.wait()
        torch.cuda.synchronize()
        rep["fp32 peer fold bit-identical"] = bool(torch.equal(out, single))
        acc_mine = torch.empty(dim, dtype=torch.int64, device="cuda")
        dev.weighted_fold(units, [w[u] for u in mine], f, acc_mine)
        out64 = torch.full((dim,), -1.0, dtype=torch.float32, device="cuda")
        pr64 = PeerReduce(out64, acc=acc_mine, barrier_timeout_s=60.0)
        for _ in range(2):
            pr64.run(f)
        pr64.wait()
        torch.cuda.synchronize()
        rep["int64 peer fold bit-identical"] = bool(torch.equal(out64, single))
        rep["peer fold barrier never timed out"] = not (pr.timed_out() or pr64.timed_out())
        dist.barrier()
        pr.close()
        pr64.close()

        # ---- ring replica by optimizer replay over an IPC pointer
        from paper_2510_00606_b200.recovery import ReplayReplica
        n_par = 200_003 + 17 * rank
        n_own = 200_003 + 17 * ((rank + 1) % world)
        gen = torch.Generator(device="cuda").manual_seed(rank)
        own = dev.AdamState(n_par)
        own.master.normal_(0, 0.02, generator=gen)
        grad = torch.empty(n_par, dtype=torch.float32, device="cuda")
        own_rows = dev.ShardMap(own.segments()).new_row_sums()
        replica_state = dev.AdamState(n_own)
        allb = [None] * world
        dist.all_gather_object(allb, (rank, dev.ipc_handle(own.buf)))
        h0, o0 = dict(allb)[(rank + 1) % world]
        p0 = dev.ipc_open(h0, o0)
        torch.cuda.synchronize()
        dist.barrier()
        dev.CopyProgram.from_pointers([p0], [replica_state.buf.data_ptr()],
                                      [replica_state.nbytes], [True]).launch()
        torch.cuda.synchronize()
        dist.barrier()
        rr = ReplayReplica(members, rank, replica_state, grad, own_rows)
        hyper = dev.adam_hyper(lr=1e-3)
        ok = True
        for step in range(1, 4):
            grad.normal_(0, 1e-3, generator=gen)
            dev.adam_step(grad, own, hyper, step, rows=own_rows)
            torch.cuda.synchronize()
            dist.barrier()
            rr.replay(hyper, step)
            rr.verify()
            torch.cuda.synchronize()
            ok = ok and int(rr.bad.item()) == 0
            dist.barrier()
        rep["replay replica verified by rows"] = ok
        torch.cuda.synchronize()
        dist.barrier()
        pulled = dev.empty_bytes(replica_state.nbytes)
        dev.CopyProgram.from_pointers([p0], [pulled.data_ptr()], [replica_state.nbytes],
                                      [True]).launch()
        torch.cuda.synchronize()
        rep["replay replica byte-identical"] = bool(torch.equal(pulled[:replica_state.nbytes],
                                                                replica_state.buf))
        dist.barrier()
        dev.ipc_close(p0)
        rr.close()

        # ---- host-memory images (double-buffered) as the H2D_D2D source
        if world <= 4:
            from paper_2510_00606_b200.hostsnap import HostSnapshots
            hs = HostSnapshots(lay, members, rank, tag=f"mp{port}")
            hs.publish(live)                      # epoch 0: the true state
            torch.cuda.synchronize()
            dist.barrier()
            drop = world - 1
            if rank == drop:                      # epoch 1 torn: D2H of garbage, no commit
                junk = torch.full_like(live, 0x77)
                slot = hs.image(rank, epoch=1)
                slot.copy_(junk[:slot.numel()].cpu())
            dist.barrier()
            rp = ReshardPlan.build(cfg.layer_bytes, members, [m for m in members if m != drop])
            ex = ReshardExecutor(rp, rank)
            b = ex.allocate(device_replica=False)
            if b.old is not None:
                b.old.copy_(live[:b.old.numel()])
            hs.attach(ex, [drop])
            ex.bind(b, verify=False)
            dist.barrier()
            ex.launch()
            torch.cuda.synchronize()
            dist.barrier()
            if b.new is not None:
                n = rp.dst.shard_bytes(rank)
                exp = _fill_expected(dev, shard_map, rp.dst, rank, 31, n)
                rep["host image (committed epoch) source"] = bool(torch.equal(b.new[:n], exp[:n]))
            dist.barrier()
            ex.close()
            hs.close()
    except Exception as e:  # noqa: BLE001 - report, do not hang the other ranks
        import traceback
        rep["error"] = repr(e) + "\n" + traceback.format_exc()[-2000:]
    import json
    Path(out_dir, f"rank{rank}.json").write_text(json.dumps(rep))
    try:
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("world", [4, 8])
def test_multiprocess_recovery_on_one_gpu(world, tmp_path):
    import json
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(world, _port(), str(tmp_path), 1e-3), nprocs=world, join=True)
    checks = 0
    for r in range(world):
        rep = json.loads((tmp_path / f"rank{r}.json").read_text())
        assert "error" not in rep, rep.get("error")
        for k, v in rep.items():
            assert v is True, (r, k, v)
            checks += 1
    assert checks > 20 * world


def _timeout_worker(rank, world, port, out_dir):
    """Rank 1 never arrives at the device barrier: rank 0's barrier times out
    (no hang), and the copy gated on the barrier's error flag writes nothing
    (a timed-out barrier must veto the in-place writes that would
    overwrite bytes a lagging peer has not read)."""
    import json
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    from paper_2510_00606_b200 import device as dev

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rep = {}
    try:
        bar = dev.PeerBarrier(timeout_s=0.5)
        src = dev.empty_bytes(1 << 20)
        src.fill_(0x5A)
        dst = torch.zeros_like(src)
        prog = dev.CopyProgram.from_pointers([src.data_ptr()], [dst.data_ptr()], [1 << 20], [False])
        if rank == 0:
            bar.wait()
            prog.launch(abort_flag=bar.error_flag)
            torch.cuda.synchronize()
            rep["barrier timed out"] = bar.timed_out()
            rep["vetoed copy wrote nothing"] = int(dst.count_nonzero()) == 0
        dist.barrier()
        bar.close()
    except Exception as e:  # noqa: BLE001
        rep["error"] = repr(e)
    Path(out_dir, f"t{rank}.json").write_text(json.dumps(rep))
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_barrier_timeout_vetoes_gated_writes(tmp_path):
    import json
    import torch.multiprocessing as mp
    mp.spawn(_timeout_worker, args=(2, _port(), str(tmp_path)), nprocs=2, join=True)
    rep = json.loads((tmp_path / "t0.json").read_text())
    assert "error" not in rep, rep
    assert rep == {"barrier timed out": True, "vetoed copy wrote nothing": True}
