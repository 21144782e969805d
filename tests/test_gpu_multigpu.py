"""N > 1 GPUs, one process per GPU (the deployment shape): the reshard
executor over CUDA-IPC peer pointers, the NCCL communicator shrink, and the
world-size determinism of the weighted reduce.  Skipped with < 2 GPUs; run on
a 2- or 4-GPU box with `gpurun --gpus N`."""
import os
import socket

import numpy as np
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
    import torch.distributed as dist
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2510_00606_b200 import configs, device as dev
    from paper_2510_00606_b200.reshard import ReshardExecutor, ReshardPlan, shard_map

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    report = {}
    progress = Path(result_dir, f"progress{rank}.txt")

    def mark(name):  # located hangs: the last stage each rank reached
        with progress.open("a") as fh:
            fh.write(name + "\n")

    try:
        mark("reshard")
        # (b) reshard world -> world-1 of a scaled 7B state, every drop position
        cfg = configs.scaled(configs.llama2_7b_per_tensor(), 2e-3)
        for drop in range(world):
            old = list(range(world))
            new = [r for r in old if r != drop]
            rp = ReshardPlan.build(cfg.layer_bytes, old, new)
            for push in (True, False):
                ex = ReshardExecutor(rp, rank, push=push)
                bufs = ex.allocate()
                if bufs.old is not None:
                    dev.fill_synthetic(shard_map(rp.src, rank), bufs.old, 99)
                if bufs.replica is not None:
                    dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank)), bufs.replica, 99)
                if bufs.new is not None:
                    bufs.new.fill_(0xA5)
                dist.barrier()
                ex.bind(bufs)
                dist.barrier()
                torch.cuda.synchronize()
                dist.barrier()
                ex.launch()
                torch.cuda.synchronize()
                dist.barrier()
                ok = True
                if bufs.new is not None:
                    exp = dev.empty_bytes(rp.dst.shard_bytes(rank))
                    dev.fill_synthetic(shard_map(rp.dst, rank), exp, 99)
                    n = rp.dst.shard_bytes(rank)
                    ok = bool(torch.equal(bufs.new[:n], exp[:n]))
                report[f"reshard drop{drop} push={push}"] = ok
                ex.close()
                dist.barrier()
        mark("prepared")
        # every single departure prepared in steady state (recovery.PreparedRecovery)
        from paper_2510_00606_b200.recovery import PreparedRecovery
        rp0 = ReshardPlan.build(cfg.layer_bytes, range(world), range(world))
        lay0 = rp0.src
        live0 = dev.empty_bytes(lay0.shard_bytes(rank))
        m0 = shard_map(lay0, rank)
        dev.fill_synthetic(m0, live0, 31)
        succ = (rank + 1) % world
        rep0 = dev.empty_bytes(lay0.shard_bytes(succ))
        dev.fill_synthetic(shard_map(lay0, succ), rep0, 31)
        rows0 = m0.new_row_sums()
        dev.checksum(m0, live0, rows0)
        block = 65536
        nblocks = (sum(cfg.layer_bytes) + block - 1) // block
        before = torch.zeros(2 * nblocks, dtype=torch.int64, device="cuda")
        dev.rows_to_blocks(m0, rows0, before)
        dist.all_reduce(before)
        torch.cuda.synchronize()
        prep = PreparedRecovery(cfg.layer_bytes, range(world), rank, live0, rep0)
        ok = True
        for d in range(world):
            dist.barrier()
            rp_d = prep.plans[d]
            if rank != d:
                ok = ok and prep.recover(d).verified  # C++: copy, barrier, conservation
            torch.cuda.synchronize()
            dist.barrier()
            if rank != d:
                exp = dev.empty_bytes(rp_d.dst.shard_bytes(rank))
                dev.fill_synthetic(shard_map(rp_d.dst, rank), exp, 31)
                n = rp_d.dst.shard_bytes(rank)
                ok = ok and bool(torch.equal(prep.new_view(d)[:n], exp[:n]))
        report["prepared single departures verified"] = ok
        dist.barrier()
        prep.close()
        mark("stage move")
        # cross-stage layer move (interleaved in place, and contiguous)
        d = world // 2
        for contiguous in (False, True):
            sm = ReshardPlan.for_stage_move(cfg.layer_bytes[:40], cfg.layer_bytes[40:80],
                                            range(d), range(d, 2 * d), contiguous)
            ex = ReshardExecutor(sm, rank)
            bufs = ex.allocate(in_place=True)
            dev.fill_synthetic(shard_map(sm.src, rank), bufs.old, 8)
            dist.barrier()
            ex.bind(bufs)
            ex.launch()
            torch.cuda.synchronize()
            dist.barrier()
            n = sm.dst.shard_bytes(rank)
            exp = dev.empty_bytes(n)
            dev.fill_synthetic(shard_map(sm.dst, rank), exp, 8)
            report[f"stage move contiguous={contiguous}"] = bool(torch.equal(bufs.new[:n], exp[:n]))
            ex.close()
            dist.barrier()
        mark("in-place")
        # staged in-place reshard (config D geometry): OLD and NEW in one
        # buffer, many phases; every departure, and a rejoin (phases upward)
        from paper_2510_00606_b200.inplace import StagedInPlaceReshard
        block = 65536
        nblk = (cfg.total_bytes + block - 1) // block
        for drop in range(world):
            for old, new in ((list(range(world)), [r for r in range(world) if r != drop]),
                             ([r for r in range(world) if r != drop], list(range(world)))):
                if len(old) < 1 or len(new) < 1 or (len(old) < 2 and len(new) < len(old)):
                    continue
                rp = ReshardPlan.build(cfg.layer_bytes, old, new)
                sub = dist.new_group(ranks=new)
                stage = max(1 << 16, max(rp.dst.shard_bytes(r) for r in new) // 7)
                ex = StagedInPlaceReshard(rp, rank, stage_bytes=stage, block_bytes=block,
                                          phase_bytes=2 * stage, slack=1 + drop % 2)
                bufs = ex.allocate()
                before = torch.zeros(2 * nblk, dtype=torch.int64, device="cuda")
                if bufs.old is not None:
                    mo = shard_map(rp.src, rank, block)
                    dev.fill_synthetic(mo, bufs.old, 17)
                    rows = mo.new_row_sums()
                    dev.checksum(mo, bufs.old, rows)
                    dev.rows_to_blocks(mo, rows, before)
                if bufs.replica is not None:
                    dev.fill_synthetic(shard_map(rp.src, rp.replica_of(rank), block),
                                       bufs.replica, 17)
                dist.all_reduce(before)
                ex.bind(bufs, None, sub if rank in new else None)
                after = torch.zeros_like(before)
                torch.cuda.synchronize()
                dist.barrier()
                ex.launch(after)
                torch.cuda.synchronize()
                dist.all_reduce(after)
                ok = bool(torch.equal(before, after)) and len(ex.sched.phases) > 2
                if rank in new:
                    n = rp.dst.shard_bytes(rank)
                    exp = dev.empty_bytes(n)
                    dev.fill_synthetic(shard_map(rp.dst, rank, block), exp, 17)
                    ok = ok and bool(torch.equal(bufs.new[:n], exp[:n]))
                    ok = ok and not ex.timed_out()
                report[f"in-place {len(old)}->{len(new)} r{drop}"] = ok
                dist.barrier()
                ex.close()
                dist.destroy_process_group(sub)
                dist.barrier()
        mark("ring replica")
        # ring replica refresh: pull the successor's snapshot, verify by rows
        from paper_2510_00606_b200.recovery import RingReplica
        lay = ReshardPlan.build(cfg.layer_bytes, range(world), range(world)).src
        m = shard_map(lay, rank)
        snap = dev.empty_bytes(lay.shard_bytes(rank))
        dev.fill_synthetic(m, snap, 13)
        rows = m.new_row_sums()
        dev.checksum(m, snap, rows)
        owner = (rank + 1) % world
        replica = dev.empty_bytes(lay.shard_bytes(owner))
        rr = RingReplica(lay, list(range(world)), rank, replica, snap, rows)
        dist.barrier()
        rr.refresh()
        torch.cuda.synchronize()
        exp = dev.empty_bytes(lay.shard_bytes(owner))
        dev.fill_synthetic(shard_map(lay, owner), exp, 13)
        report["replica verified"] = int(rr.bad.item()) == 0
        report["replica bytes"] = bool(torch.equal(replica[:lay.shard_bytes(owner)],
                                                   exp[:lay.shard_bytes(owner)]))
        dist.barrier()
        rr.close()
        mark("replay")
        # ring replica by optimizer replay: the holder steps its replica from
        # the owner's gradient read over NVLink; byte-identical, rows verify
        from paper_2510_00606_b200.recovery import ReplayReplica
        n_par = 1_000_003 + 17 * rank  # ragged, different per rank
        n_own = 1_000_003 + 17 * ((rank + 1) % world)
        gen = torch.Generator(device="cuda").manual_seed(rank)
        own = dev.AdamState(n_par)
        own.master.normal_(0, 0.02, generator=gen)
        grad = torch.empty(n_par, dtype=torch.float32, device="cuda")
        own_map = dev.ShardMap(own.segments())
        own_rows = own_map.new_row_sums()
        replica_state = dev.AdamState(n_own)
        # initial replica = owner's state at step 0 (one full pull, as at start)
        allb = [None] * world
        dist.all_gather_object(allb, (rank, dev.ipc_handle(own.buf)))
        h0, o0 = dict(allb)[(rank + 1) % world]
        p0 = dev.ipc_open(h0, o0)
        dist.barrier()
        dev.CopyProgram.from_pointers([p0], [replica_state.buf.data_ptr()],
                                      [replica_state.nbytes], [True]).launch()
        torch.cuda.synchronize()
        dist.barrier()
        dev.ipc_close(p0)
        rep = ReplayReplica(list(range(world)), rank, replica_state, grad, own_rows)
        hyper = dev.adam_hyper(lr=1e-3)
        ok = True
        for step in range(1, 4):
            grad.normal_(0, 1e-3, generator=gen)
            dev.adam_step(grad, own, hyper, step, rows=own_rows)  # rows fused
            torch.cuda.synchronize()
            dist.barrier()   # owner's grad + rows published
            rep.replay(hyper, step)
            rep.verify()
            torch.cuda.synchronize()
            ok = ok and int(rep.bad.item()) == 0
            rep.verify_by_reread()
            torch.cuda.synchronize()
            ok = ok and int(rep.bad.item()) == 0
            dist.barrier()   # holder done reading before the next step's grad
        report["replay replica verified"] = ok
        allb = [None] * world
        dist.all_gather_object(allb, (rank, dev.ipc_handle(own.buf)))
        h1, o1 = dict(allb)[(rank + 1) % world]
        p1 = dev.ipc_open(h1, o1)
        pulled = dev.empty_bytes(replica_state.nbytes)
        dev.CopyProgram.from_pointers([p1], [pulled.data_ptr()], [replica_state.nbytes],
                                      [True]).launch()
        torch.cuda.synchronize()
        report["replay replica bytes"] = bool(torch.equal(pulled[:replica_state.nbytes],
                                                          replica_state.buf))
        dist.barrier()
        dev.ipc_close(p1)
        rep.close()
        mark("toy")
        # toy consistency across real ranks: one slot per GPU, the last rank
        # leaves before step 2, survivors reshape and sum on the shrunk NCCL
        # communicator; final parameters equal the static run bit for bit
        from paper_2510_00606_b200.toy import ToyConfig, ToyRun
        tcfg = ToyConfig(dp=world, global_batch=2 * world, steps=4)
        uid = [dev.Communicator.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        tcomm = dev.Communicator.init(uid[0], world, rank)
        state = {"comm": tcomm, "shrunk": False}

        def toy_reduce(total, members):
            if len(members) < world and not state["shrunk"]:
                state["comm"] = tcomm.shrink([world - 1])
                state["shrunk"] = True
            state["comm"].allreduce_i64(total)

        got = ToyRun(tcfg, {2: [world - 1]}).run(toy_reduce, my_slots=[rank])
        if rank != world - 1:
            static = ToyRun(tcfg).run()
            report["toy elastic == static (NCCL, shrunk)"] = bool(torch.equal(
                got.view(torch.int64), static.view(torch.int64)))
        dist.barrier()
        if state["shrunk"] and state["comm"] is not None:
            state["comm"].destroy()
        tcomm.destroy()
        mark("dp group")
        # full DP recovery of the last rank (recovery.DpGroup): plan_edit +
        # ncclCommShrink, reshape, remap, checksum verification
        from paper_2510_00606_b200.recovery import DpGroup
        uid = [dev.Communicator.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = dev.Communicator.init(uid[0], world, rank)
        comm.allreduce_i64(torch.zeros(8, dtype=torch.int64, device="cuda"))
        drop = world - 1
        survivors = [r for r in range(world) if r != drop]
        grp = dist.new_group(survivors)
        rp = ReshardPlan.build(cfg.layer_bytes, range(world), survivors)
        shrunk = None
        # before the failure: every rank's live shard, and the ring replica
        # its holder keeps of it (RingReplica pull), which is what the
        # recovery reads for the departed rank's bytes
        ex = ReshardExecutor(rp, rank) if rank != drop else None
        bufs = ex.allocate() if ex is not None else None
        live = bufs.old if bufs is not None else dev.empty_bytes(rp.src.shard_bytes(rank))
        lm = shard_map(rp.src, rank)
        dev.fill_synthetic(lm, live, 5)
        live_rows = lm.new_row_sums()
        dev.checksum(lm, live, live_rows)
        owner = (rank + 1) % world
        holds_drop = bufs is not None and bufs.replica is not None
        rbuf = bufs.replica if holds_drop else dev.empty_bytes(rp.src.shard_bytes(owner))
        torch.cuda.synchronize()
        ring = RingReplica(rp.src, list(range(world)), rank, rbuf, live, live_rows)
        dist.barrier()
        ring.refresh()
        torch.cuda.synchronize()
        report["ring replica before failure verified"] = int(ring.bad.item()) == 0
        dist.barrier()
        ring.close()
        # every member builds the group (collective: one prepared shrunk
        # communicator per possible departure); the survivors recover
        group = DpGroup(cfg.layer_bytes, range(world), rank, comm)
        dist.barrier()
        if rank != drop:
            ev = group.recover([drop], bufs)
            report["recovery verified by checksums"] = ev.verified
            report["comm repaired by a prepared split"] = ev.phases.get("comm_prepared") == 1.0
            report["recovery mttr row"] = ev.csv_row(0)
            shrunk = group.comm
            exp = dev.empty_bytes(rp.dst.shard_bytes(rank))
            dev.fill_synthetic(shard_map(rp.dst, rank), exp, 5)
            n = rp.dst.shard_bytes(rank)
            report["recovery bytes"] = bool(torch.equal(bufs.new[:n], exp[:n]))
        dist.barrier()
        n_units, dim = 12, 100_003
        rng = np.random.default_rng(21)
        g = rng.normal(0, 1e-3, size=(n_units, dim)).astype(np.float32)
        g[3, 5] = 1e2
        w = rng.random(n_units) / n_units
        # units split over the ranks of the shrunk communicator
        if shrunk is not None:
            k = len(survivors)
            mine = [u for u in range(n_units) if u % k == shrunk.rank]
            units = [torch.from_numpy(g[u]).cuda() for u in mine]
            out = torch.empty(dim, dtype=torch.float32, device="cuda")
            acc = torch.empty(dim, dtype=torch.int64, device="cuda")
            mx = torch.empty(1, dtype=torch.float64, device="cuda")
            f = shrunk.weighted_reduce(units, [w[u] for u in mine], n_units, out, acc, mx)
            torch.cuda.synchronize()
            # single-GPU fold of all units, same scale
            all_units = [torch.from_numpy(x).cuda() for x in g]
            acc1 = torch.empty(dim, dtype=torch.int64, device="cuda")
            dev.weighted_fold(all_units, w, f, acc1)
            single = dev.fixed_to_float(acc1, f)
            report["reduce bit-identical to 1-GPU fold"] = bool(torch.equal(out, single))
            # the same reduce with the scale kept on the device (no host sync)
            out2 = torch.full_like(out, -1.0)
            bits = torch.empty(1, dtype=torch.int32, device="cuda")
            shrunk.weighted_reduce_async(units, [w[u] for u in mine], n_units, out2, acc, mx, bits)
            torch.cuda.synchronize()
            report["async reduce identical"] = bool(torch.equal(out2, out)) and \
                int(bits.item()) == f
            report["shrunk size"] = shrunk.size
        dist.barrier()
        mark("rejoin")
        # the departed device rejoins (ScaleOut, sim.cpp:608,676-677): a
        # standby communicator over members + joiner prepared in steady
        # state, then the join (grown communicator looked up, micro-batches
        # re-dealt, shards re-cut, verified); re-prepare the departure splits
        # over the grown group; the same device leaves again (prepared split)
        # and rejoins without a standby (ncclCommInitRank at the event)
        from paper_2510_00606_b200.fabric import FAIL_STOP, SCALE_IN
        from paper_2510_00606_b200.reshard import RankBuffers
        everyone = list(range(world))
        rpj = ReshardPlan.build(cfg.layer_bytes, survivors, everyone)
        jg = DpGroup.joiner(cfg.layer_bytes, survivors, rank, group.name) if rank == drop \
            else group
        jg.prepare_join([drop])
        new_j = dev.empty_bytes(rpj.dst.shard_bytes(rank))
        ev = jg.admit([drop], RankBuffers(bufs.new if rank != drop else None, None, new_j), step=2)
        n = rpj.dst.shard_bytes(rank)
        exp = dev.empty_bytes(n)
        dev.fill_synthetic(shard_map(rpj.dst, rank), exp, 5)
        report["rejoin verified"] = ev.verified
        report["rejoin bytes"] = bool(torch.equal(new_j[:n], exp[:n]))
        report["rejoin by the standby communicator"] = ev.phases.get("comm_prepared") == 1.0
        report["rejoin members"] = jg.members == everyone
        report["rejoin comm size"] = jg.comm is not None and jg.comm.size == world
        jg.prepare()
        holder = everyone[everyone.index(drop) - 1]
        rep_d = None
        if rank == holder:
            rep_d = dev.empty_bytes(rpj.dst.shard_bytes(drop))
            dev.fill_synthetic(shard_map(rpj.dst, drop), rep_d, 5)
        # steady state: map, snapshot rows as the source sums, the program
        # for this departure bound ahead
        jm = shard_map(rpj.dst, rank)
        j_rows = jm.new_row_sums()
        dev.checksum(jm, new_j, j_rows)
        d_rows = None
        if rep_d is not None:
            dm = shard_map(rpj.dst, drop)
            d_rows = dm.new_row_sums()
            dev.checksum(dm, rep_d, d_rows)
        new2 = dev.empty_bytes(rp.dst.shard_bytes(rank)) if rank != drop else None
        jg.premap(RankBuffers(new_j, rep_d, None), j_rows, d_rows)
        jg.prepare_move(FAIL_STOP, [drop], new2)
        torch.cuda.synchronize()
        dist.barrier()
        if rank != drop:
            ev = jg.recover([drop], RankBuffers(new_j, rep_d, new2), step=3)
            report["second departure premapped"] = ev.phases.get("premapped") == 1.0
            report["second departure program prepared"] = ev.phases.get("prepared") == 1.0
            n = rp.dst.shard_bytes(rank)
            exp = dev.empty_bytes(n)
            dev.fill_synthetic(shard_map(rp.dst, rank), exp, 5)
            report["second departure verified"] = ev.verified
            report["second departure by a prepared split"] = ev.phases.get("comm_prepared") == 1.0
            report["second departure bytes"] = bool(torch.equal(new2[:n], exp[:n]))
            old4 = new2
        else:
            old4 = None
        dist.barrier()
        jg2 = DpGroup.joiner(cfg.layer_bytes, survivors, rank, group.name) if rank == drop \
            else jg
        new4 = dev.empty_bytes(rpj.dst.shard_bytes(rank))
        ev = jg2.admit([drop], RankBuffers(old4, None, new4), step=4)
        n = rpj.dst.shard_bytes(rank)
        exp = dev.empty_bytes(n)
        dev.fill_synthetic(shard_map(rpj.dst, rank), exp, 5)
        report["rejoin without standby verified"] = ev.verified
        report["rejoin without standby bytes"] = bool(torch.equal(new4[:n], exp[:n]))
        report["rejoin without standby: fresh communicator"] = \
            ev.phases.get("comm_prepared") == 0.0 and jg2.comm is not None and \
            jg2.comm.size == world
        t = torch.ones(4, dtype=torch.int64, device="cuda")
        jg2.comm.allreduce_i64(t)
        torch.cuda.synchronize()
        report["grown communicator sums over all"] = int(t[0].item()) == world
        dist.barrier()
        if world >= 4:
            # two non-adjacent members leave together: their shrunk
            # communicator was prepared as a set (ncclCommSplit in steady state)
            pair = [1, 3]
            keep = [r for r in everyone if r not in pair]
            rp5 = ReshardPlan.build(cfg.layer_bytes, everyone, keep)
            jg2.prepare([pair])
            owner5 = rp5.replica_of(rank)
            rep5 = None
            if owner5 in pair:  # this rank holds a departing member's replica
                rep5 = dev.empty_bytes(rpj.dst.shard_bytes(owner5))
                dev.fill_synthetic(shard_map(rpj.dst, owner5), rep5, 5)
            dist.barrier()
            if rank in keep:
                new5 = dev.empty_bytes(rp5.dst.shard_bytes(rank))
                ev = jg2.recover(pair, RankBuffers(new4, rep5, new5), step=5, kind=SCALE_IN)
                n = rp5.dst.shard_bytes(rank)
                exp = dev.empty_bytes(n)
                dev.fill_synthetic(shard_map(rp5.dst, rank), exp, 5)
                report["pair departure verified"] = ev.verified
                report["pair departure bytes"] = bool(torch.equal(new5[:n], exp[:n]))
                report["pair departure by a prepared set split"] = \
                    ev.phases.get("comm_prepared") == 1.0 and jg2.comm.size == len(keep)
            dist.barrier()
        if rank == drop:
            jg.close()
            jg2.close()
        group.close()   # the group owns the communicators (parent and splits)
        mark("peer reduce")
        # the same reduce fused with its collective over peer memory (no NCCL)
        dist.barrier()
        mine = [u for u in range(n_units) if u % world == rank]
        units = [torch.from_numpy(g[u]).cuda() for u in mine]
        out = torch.empty(dim, dtype=torch.float32, device="cuda")
        fold, total, opened = dev.peer_weighted_reduce_setup(units, [w[u] for u in mine], out)
        amax = dev.weighted_absmax(units, [w[u] for u in mine]) if units else \
            torch.zeros(1, dtype=torch.float64, device="cuda")
        dist.all_reduce(amax, op=dist.ReduceOp.MAX)
        f = dev.fixed_point_bits(amax.item(), total)
        dist.barrier()
        fold.reduce_scatter(f)
        torch.cuda.synchronize()
        dist.barrier()
        fold.all_gather()
        torch.cuda.synchronize()
        dist.barrier()
        all_units = [torch.from_numpy(x).cuda() for x in g]
        acc1 = torch.empty(dim, dtype=torch.int64, device="cuda")
        dev.weighted_fold(all_units, w, f, acc1)
        single = dev.fixed_to_float(acc1, f)
        report["peer reduce bit-identical to 1-GPU fold"] = bool(torch.equal(out, single))
        # stream-ordered version: device-side barriers between the phases
        bar = dev.PeerBarrier()
        out.fill_(-1.0)
        for _ in range(3):
            fold.run(f, bar)
        bar.wait()  # nobody leaves while a peer may still read its chunk
        torch.cuda.synchronize()
        report["device barrier ok"] = not bar.timed_out()
        report["peer reduce (device barriers) bit-identical"] = bool(torch.equal(out, single))
        # per-rank int64 accumulators (each rank folded its own units)
        # summed over peer memory: same bits again
        acc_mine = torch.empty(dim, dtype=torch.int64, device="cuda")
        dev.weighted_fold(units, [w[u] for u in mine], f, acc_mine) if units else acc_mine.zero_()
        out64 = torch.full((dim,), -1.0, dtype=torch.float32, device="cuda")
        fold64, opened64 = dev.peer_sum_i64_setup(acc_mine, out64)
        torch.cuda.synchronize()
        dist.barrier()
        for _ in range(2):
            fold64.run(f, bar)
        bar.wait()
        torch.cuda.synchronize()
        report["peer int64-accumulator reduce bit-identical"] = bool(torch.equal(out64, single))
        dist.barrier()
        bar.close()
        del fold, fold64
        for p in opened + opened64:
            dev.ipc_close(p)
    except Exception as e:  # report, do not hang the other ranks
        import traceback
        report["error"] = repr(e) + "\n" + traceback.format_exc()[-1500:]
    import json
    Path(result_dir, f"rank{rank}.json").write_text(json.dumps(report))
    dist.destroy_process_group()


@pytest.mark.timeout(300)  # a collective mismatch must fail, not hang the box
@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_reshard_comm_reduce(world, tmp_path):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    import json
    import torch.multiprocessing as mp
    try:
        mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    finally:  # where each rank got to (a hang is located by the last stage)
        for r in range(world):
            f = tmp_path / f"progress{r}.txt"
            print(f"rank {r} stages:", f.read_text().split() if f.exists() else None)
    for r in range(world):
        rep = json.loads((tmp_path / f"rank{r}.json").read_text())
        assert "error" not in rep, rep.get("error")
        for k, v in rep.items():
            if isinstance(v, bool):
                assert v is True, (r, k)
        if r != world - 1:
            assert rep["shrunk size"] == world - 1
            assert rep["recovery verified by checksums"] is True
        # the rejoin / second departure / rejoin sequence ran on every rank
        assert rep.get("rejoin verified") is True and rep.get("rejoin without standby verified")
        if world >= 4 and r in (0, 2):
            assert rep.get("pair departure by a prepared set split") is True
