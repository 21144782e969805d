"""The recovery runtime's rendezvous on CPU (no GPU needed): the C++ TCP store
and the callback store over torch.distributed's c10d store, with the
Channel collectives (allgather-based barrier and sum) the C++ executors use
to exchange CUDA IPC handles and verdicts.  World sizes 3 and 8 on gloo;
subset channels (the survivors of a departure) must not need the departed
member."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tcp_port, out_dir):
    import json
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import torch.distributed as dist
    from paper_2510_00606_b200.rendezvous import Channel, Store

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    try:
        # callback store over c10d
        ch = Channel.from_group(None, "t")
        ch.barrier()
        res["sum"] = ch.sum(rank + 1)
        res["name_agrees"] = ch.name
        # survivors of a departure: the departed member takes no part
        drop = world - 1
        if rank != drop:
            sub = Channel(ch.store, "t/without", [r for r in range(world) if r != drop], rank)
            sub.barrier()
            res["sub_sum"] = sub.sum(10)
        # library TCP store, rank 0 hosting
        tcp = Store.tcp("127.0.0.1", tcp_port, rank == 0, timeout_s=60.0)
        tch = Channel(tcp, "tcp", list(range(world)), rank)
        for _ in range(3):
            tch.barrier()
        res["tcp_sum"] = tch.sum(2 ** 40 + rank)
        tcp.set(f"k{rank}", bytes([rank]) * (1000 + rank))
        got = tcp.get(f"k{(rank + 1) % world}", cap=4096)
        res["tcp_blob_ok"] = got == bytes([(rank + 1) % world]) * (1000 + (rank + 1) % world)
        tch.barrier()  # nobody leaves while rank 0's server is still needed
        del tch
        tcp.close()
    except Exception as e:  # noqa: BLE001
        res["error"] = repr(e)
    Path(out_dir, f"r{rank}.json").write_text(json.dumps(res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(240)
@pytest.mark.parametrize("world", [3, 8])
def test_store_and_channels_multiprocess(world, tmp_path):
    import json
    mp.spawn(_worker, args=(world, _port(), _port(), str(tmp_path)), nprocs=world, join=True)
    names = set()
    for r in range(world):
        res = json.loads((tmp_path / f"r{r}.json").read_text())
        assert "error" not in res, res.get("error")
        assert res["sum"] == world * (world + 1) // 2
        assert res["tcp_sum"] == world * 2 ** 40 + world * (world - 1) // 2
        assert res["tcp_blob_ok"]
        if r != world - 1:
            assert res["sub_sum"] == 10 * (world - 1)
        names.add(res["name_agrees"])
    assert len(names) == 1


def test_mttr_csv_from_cpp():
    """mttr.csv rows come from the C++ library in the reference's format
    (sim.cpp:1119-1132: %zu,%d,%.9g,%s,... total = detect+comm+remap+stall+other)."""
    from paper_2510_00606_b200.recovery import MTTR_CSV_HEADER, MttrEvent
    assert MTTR_CSV_HEADER == ("event,step,t_event_s,kind,detect_s,comm_repair_s,remap_s,"
                               "migration_stall_s,other_s,lost_work_s,total_s")
    ev = MttrEvent(step=7, t_event_s=1.5, kind="scale_in", comm_repair_s=0.000163,
                   remap_s=0.0118, other_s=1e-6, lost_work_s=0.25)
    assert ev.csv_row(2) == "2,7,1.5,scale_in,0,0.000163,0.0118,0,1e-06,0.25,0.011964"


def test_tcp_store_timeout_breaks_the_connection():
    """A get that times out leaves the stream mid-frame (the server may
    answer later): the store reports it and refuses further use instead of
    reading a stale answer as the next reply."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2510_00606_b200._native import ElaskitError
    from paper_2510_00606_b200.rendezvous import Store

    st = Store.tcp("127.0.0.1", _port(), True, 0.5)
    st.set("a", b"1")
    assert st.get("a") == b"1"
    with pytest.raises(ElaskitError, match="timed out"):
        st.get("never-set")
    with pytest.raises(ElaskitError, match="broken"):
        st.set("b", b"2")
    st.close()
