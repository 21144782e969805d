"""Host-side logic of hostsnap.HostSnapshots (no GPU): attach() points the
ring holder's REPLICA slot of a copy table at each departed rank's image —
the holder the reference's overlap_matrix names as the H2D_D2D source
(param_fabric.cpp:112; SnapshotRing::backed_up_by, param_fabric.cpp:51-64)."""
import types

from paper_2510_00606_b200.fabric import ROLE_REPLICA, SnapshotRing
from paper_2510_00606_b200.hostsnap import HostSnapshots


def _fake(members):
    hs = HostSnapshots.__new__(HostSnapshots)
    hs.members = list(members)
    hs.ring = SnapshotRing(hs.members)
    hs._dev = {r: 0x1000 * (r + 1) for r in members}
    hs._closed = True  # nothing to release
    return hs


def test_attach_maps_holder_slot_to_departed_image():
    hs = _fake(range(8))
    ex = types.SimpleNamespace()
    hs.attach(ex, [3])
    assert ex._table == {(ROLE_REPLICA, 2): 0x4000}  # holder of 3 is 2
    hs.attach(ex, [0, 5])  # wraps around: holder of 0 is 7
    assert ex._table[(ROLE_REPLICA, 7)] == 0x1000
    assert ex._table[(ROLE_REPLICA, 4)] == 0x6000
    assert len(ex._table) == 3


def test_attach_keeps_existing_peer_entries():
    hs = _fake([0, 2, 5])
    ex = types.SimpleNamespace(_table={(0, 5): 123})
    hs.attach(ex, [2])
    assert ex._table == {(0, 5): 123, (ROLE_REPLICA, 0): 0x3000}
