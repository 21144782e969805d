"""Host-side logic of hostsnap.HostSnapshots (no GPU): attach() points the
ring holder's REPLICA slot of a copy table at each departed rank's image —
the holder the reference's overlap_matrix names as the H2D_D2D source
(param_fabric.cpp:112; SnapshotRing::backed_up_by, param_fabric.cpp:51-64),
through the executor's peer table (ReshardExecutor.put_peer)."""
import struct
import types

import pytest

from paper_2510_00606_b200.fabric import ROLE_REPLICA, SnapshotRing
from paper_2510_00606_b200.hostsnap import HostSnapshots

PAGE = HostSnapshots._PAGE
SLOT = 2 * PAGE


def _fake(members, epochs=None):
    """Segments of two 2-page slots; member r's committed epoch from
    `epochs` (default 0 = slot 0)."""
    hs = HostSnapshots.__new__(HostSnapshots)
    hs.members = list(members)
    hs.ring = SnapshotRing(hs.members)
    hs._dev = {r: 0x100000 * (r + 1) for r in members}
    hs._slot_bytes = {r: SLOT for r in members}
    hs._segs = {}
    for r in members:
        buf = bytearray(PAGE + 2 * SLOT)
        struct.pack_into("<q", buf, 0, (epochs or {}).get(r, 0))
        hs._segs[r] = types.SimpleNamespace(buf=buf)
    hs._closed = True  # nothing to release
    return hs


class _FakeExecutor:
    """Records ReshardExecutor.put_peer calls (the peer table)."""

    def __init__(self, table=None):
        self._table = dict(table or {})

    def put_peer(self, role, member, ptr):
        self._table[(role, member)] = ptr


def _img(hs, r, slot):
    return hs._dev[r] + PAGE + slot * SLOT


def test_attach_maps_holder_slot_to_departed_image():
    hs = _fake(range(8))
    ex = _FakeExecutor()
    hs.attach(ex, [3])
    assert ex._table == {(ROLE_REPLICA, 2): _img(hs, 3, 0)}  # holder of 3 is 2
    hs.attach(ex, [0, 5])  # wraps around: holder of 0 is 7
    assert ex._table[(ROLE_REPLICA, 7)] == _img(hs, 0, 0)
    assert ex._table[(ROLE_REPLICA, 4)] == _img(hs, 5, 0)
    assert len(ex._table) == 3


def test_attach_keeps_existing_peer_entries():
    hs = _fake([0, 2, 5])
    ex = _FakeExecutor({(0, 5): 123})
    hs.attach(ex, [2])
    assert ex._table == {(0, 5): 123, (ROLE_REPLICA, 0): _img(hs, 2, 0)}


def test_attach_uses_last_committed_slot():
    """Double-buffered images: epoch e lives in slot e mod 2; a publish that
    died before its commit word leaves the previous epoch's slot in use."""
    hs = _fake(range(4), epochs={1: 7, 2: 4})
    ex = _FakeExecutor()
    hs.attach(ex, [1])
    assert ex._table[(ROLE_REPLICA, 0)] == _img(hs, 1, 1)
    hs.attach(ex, [2])
    assert ex._table[(ROLE_REPLICA, 1)] == _img(hs, 2, 0)


def test_attach_refuses_uncommitted_image():
    hs = _fake(range(3), epochs={1: -1})
    with pytest.raises(RuntimeError, match="not committed"):
        hs.attach(_FakeExecutor(), [1])
