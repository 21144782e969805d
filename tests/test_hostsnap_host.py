"""Host-side logic of the host images (C++ elaskit::b200::HostImages through
hostsnap.HostSnapshots), no GPU: real POSIX shm segments without pinning
(map_for_device=False).  attach() points the ring holder's REPLICA slot of a
copy table at each departed rank's last committed image — the holder the
reference's overlap_matrix names as the H2D_D2D source (param_fabric.cpp:112;
SnapshotRing::backed_up_by, param_fabric.cpp:51-64) — through the executor's
peer table (ReshardExecutor.put_peer); images are double-buffered with a
committed-epoch word."""
import os
import socket

import pytest

from paper_2510_00606_b200 import configs, fabric
from paper_2510_00606_b200.fabric import ROLE_REPLICA
from paper_2510_00606_b200.hostsnap import HostSnapshots
from paper_2510_00606_b200.rendezvous import Channel, Store


class _FakeExecutor:
    """Records ReshardExecutor.put_peer calls (the peer table)."""

    def __init__(self, table=None):
        self._table = dict(table or {})

    def put_peer(self, role, member, ptr):
        self._table[(role, member)] = ptr


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture
def images():
    """Every member's image in one process (a one-member channel per member,
    all on one TCP store): the segments a node's ranks would create."""
    cfg = configs.scaled(configs.gpt_125m(), 1e-4)
    members = list(range(4))
    layout = fabric.interleaved_layout(cfg.layer_bytes, members)
    store = Store.tcp("127.0.0.1", _port(), True, 30.0)
    tag = f"t{os.getpid()}"
    hs = {}
    for r in members:  # creators first, each maps only its own image
        ch = Channel(store, f"h{r}", [r], r)
        hs[r] = HostSnapshots(layout, members, r, tag, readable=[r], map_for_device=False,
                              channel=ch)
    yield layout, hs, store, tag
    for h in hs.values():
        h.close()
    store.close()


def test_images_double_buffered_and_committed(images):
    layout, hs, store, tag = images
    h = hs[1]
    assert h.committed_epoch(1) == -1
    with pytest.raises(Exception, match="not committed"):
        h.image(1)
    h.image(1, epoch=0).fill_(7)
    h.commit_host(0)
    h.image(1, epoch=1).fill_(9)   # a publish that never committed: torn
    assert h.committed_epoch(1) == 0
    assert int(h.image(1)[0]) == 7 and int(h.image(1)[-1]) == 7
    h.commit_host(1)
    assert int(h.image(1)[0]) == 9
    assert h.image(1).numel() == layout.shard_bytes(1)


def test_attach_maps_holder_slot_to_committed_image(images):
    layout, hs, store, tag = images
    for r, h in hs.items():
        h.commit_host(4 + r)            # member r: epoch 4 + r -> slot r mod 2
    ex = _FakeExecutor({(0, 5): 123})
    hs[3].attach(ex, [3])               # holder of 3 is 2
    hs[0].attach(ex, [0])               # wraps around: holder of 0 is 3
    assert ex._table[(ROLE_REPLICA, 2)] == hs[3].device_ptr(3)
    assert ex._table[(ROLE_REPLICA, 3)] == hs[0].device_ptr(0)
    assert ex._table[(0, 5)] == 123
    # device_ptr (host address here) is the committed slot's image
    assert hs[3].device_ptr(3) == hs[3].image(3).data_ptr()
    assert hs[0].device_ptr(0) != hs[0].image(0, epoch=5).data_ptr()
