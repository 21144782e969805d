"""The C++-only multi-process recovery driver (tools/cpp/dp_recover.cpp): no
Python in the recovering processes.  N processes rendezvous on the library's
TCP store, build the steady state (snapshot rows, ring replica, prepared
recovery; prepared NCCL communicators when each has its own GPU) and the
survivors run DpGroup::recover for a FailStop, each checking verification
and its NEW bytes and printing its mttr.csv row (reference format,
sim.cpp:1119-1132).

  * every process on cuda:0 (N = 4, all drop positions of interest): the
    cross-process path on any one-GPU box;
  * one process per GPU with NCCL (N = device count >= 2): comm repair by a
    prepared split."""
import socket
import subprocess
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tools" / "cpp" / "dp_recover"


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def driver():
    subprocess.run(["make", "-C", str(ROOT / "tools" / "cpp"), "dp_recover"], check=True,
                   capture_output=True)
    return BIN


def _run(driver, world, drop, devices, nccl=False, scale="0.004", rejoin=False, kill=False):
    port = _port()
    procs = []
    for r in range(world):
        cmd = [str(driver), "--rank", str(r), "--world", str(world), "--port", str(port),
               "--drop", str(drop), "--device", str(devices[r]), "--scale", scale]
        if nccl:
            cmd.append("--nccl")
        if rejoin:
            cmd.append("--rejoin")
        if kill:
            cmd.append("--kill")
        procs.append(subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    outs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append((p.returncode, o, e))
    return outs


@pytest.mark.timeout(600)
@pytest.mark.parametrize("drop", [0, 3])
def test_cpp_driver_four_processes_one_gpu(driver, drop):
    outs = _run(driver, 4, drop, [0, 0, 0, 0], rejoin=drop == 3)
    for r, (rc, o, e) in enumerate(outs):
        assert rc == 0, (r, o, e)
        if r != drop:
            assert "verified=1 bytes=1" in o, o
            assert f"rank {r} 0,1,0,fail_stop," in o, o
        if drop == 3:  # ...and the departed process rejoins (ScaleOut), C++ only
            assert f"rank {r} rejoin 1,2,0,scale_out," in o, o
            assert "verified=1 bytes=1 members=1 prepared=1" in o, o


@pytest.mark.timeout(600)
def test_cpp_driver_one_process_per_gpu_nccl(driver):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs (one NCCL rank per GPU)")
    outs = _run(driver, n, n - 1, list(range(n)), nccl=True, scale="0.01", rejoin=True)
    for r, (rc, o, e) in enumerate(outs):
        assert rc == 0, (r, o, e)
        if r != n - 1:
            assert "verified=1 bytes=1" in o, o
        # the rejoin over the standby grown NCCL communicator
        assert f"rank {r} rejoin 1,2,0,scale_out," in o, o
        assert "verified=1 bytes=1 members=1 prepared=1" in o, o


@pytest.mark.timeout(600)
def test_cpp_driver_killed_rank(driver):
    """The departing process is SIGKILLed: the survivors' heartbeat detector
    finds it and they recover without it (one GPU, and with NCCL one
    process per GPU when there are >= 2 GPUs)."""
    n = torch.cuda.device_count()
    cases = [(4, [0, 0, 0, 0], False)]
    if n >= 2:
        cases.append((n, list(range(n)), True))
    for world, devices, nccl in cases:
        drop = world - 1
        outs = _run(driver, world, drop, devices, nccl=nccl, kill=True)
        for r, (rc, o, e) in enumerate(outs):
            if r == drop:
                assert rc == -9, (r, rc, e)
                continue
            assert rc == 0, (r, o, e)
            assert "verified=1 bytes=1" in o, o
            row = o.split(f"rank {r} ")[1].split()[0].split(",")
            assert row[3] == "fail_stop" and 0.015 < float(row[4]) < 0.5, row  # detect_s

