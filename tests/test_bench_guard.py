"""bench.py's LegGuard: a secondary leg that raises or hangs (on any rank)
still yields rank 0's JSON line, marked incomplete, and exit code 0.  CPU
only: world 1, and world 2 over gloo with the failing leg on rank 1 while
rank 0 waits in a collective."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r'''
import os, sys, time, types
sys.path.insert(0, {root!r})
import bench
import torch.distributed as dist
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
if world > 1:
    dist.init_process_group("gloo")
mode = sys.argv[1]
args = types.SimpleNamespace(deadline_s=float(sys.argv[2]), json_out="")
out = {{"metric": "m", "value": 1.5}}
g = bench.LegGuard(args, rank, world, out, time.time())
g.run("ok_leg", lambda: out.update(ok=True))
def bad():
    if mode == "raise" and rank == world - 1:
        raise RuntimeError("boom")
    if world > 1:
        dist.barrier()          # the healthy ranks block on the broken one
    time.sleep(60)              # mode "hang"
g.run("bad_leg", bad)
print("not reached", flush=True)
'''


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(mode, deadline, world):
    code = SCRIPT.format(root=str(ROOT))
    procs = []
    port = _free_port()
    for r in range(world):
        env = dict(os.environ, WORLD_SIZE=str(world), RANK=str(r), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", code, mode, str(deadline)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    outs = [p.communicate(timeout=120) for p in procs]
    return [p.returncode for p in procs], outs


def _line(stdout):
    lines = [x for x in stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, stdout
    return json.loads(lines[0])


def test_raising_leg_world1():
    rc, outs = _launch("raise", 300, 1)
    assert rc == [0]
    rec = _line(outs[0][0])
    assert rec["value"] == 1.5 and rec["ok"] is True
    assert rec["incomplete"]["legs_done"] == ["ok_leg"]
    assert "bad_leg" in rec["incomplete"]["reason"] and "boom" in rec["incomplete"]["reason"]
    assert "not reached" not in outs[0][0]


def test_hung_leg_hits_deadline():
    rc, outs = _launch("hang", 3, 1)
    assert rc == [0]
    rec = _line(outs[0][0])
    assert "deadline" in rec["incomplete"]["reason"] and "bad_leg" in rec["incomplete"]["reason"]


def test_raising_leg_on_rank1_releases_rank0_world2():
    rc, outs = _launch("raise", 300, 2)
    assert rc == [0, 0]
    rec = _line(outs[0][0])
    assert "rank 1 raised" in rec["incomplete"]["reason"]
    assert not [x for x in outs[1][0].splitlines() if x.startswith("{")]  # rank 1 prints nothing
