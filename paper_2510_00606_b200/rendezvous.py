"""Out-of-band rendezvous of the recovery runtime (recovery.hpp Store /
Channel through the C ABI).

A Store is the key-value channel the ranks of a DP group meet on: the
library's own TCP store (`Store.tcp`), or torch.distributed's c10d store
plugged in through callbacks (`Store.from_torch`, the default when a
process group exists).  A Channel is an ordered member list on a store; its
collectives (allgather, barrier, sum) are what the C++ executors use to
exchange CUDA IPC handles and verdicts.  Plumbing only: no model byte or
checksum crosses it.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Optional, Sequence, Tuple

from . import _native as N
from ._native import check, lib


class Store:
    """ew_store handle (owns the C++ Store)."""

    def __init__(self, handle: C.c_void_p, keep=()):
        self._h = handle
        self._keep = keep  # ctypes callbacks must outlive the store

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @classmethod
    def tcp(cls, host: str, port: int, is_server: bool, timeout_s: float = 300.0) -> "Store":
        h = C.c_void_p()
        check(lib.ew_store_tcp(host.encode(), int(port), int(bool(is_server)), float(timeout_s),
                               C.byref(h)))
        return cls(h)

    @classmethod
    def from_torch(cls, store=None) -> "Store":
        """Wrap a c10d store (default: the default process group's)."""
        if store is None:
            from torch.distributed import distributed_c10d as c10d
            store = c10d._get_default_store()
        pending: Dict[str, bytes] = {}

        def set_cb(_ctx, key, klen, val, vlen):
            try:
                store.set(C.string_at(key, klen).decode(), C.string_at(val, vlen))
                return 0
            except Exception:  # noqa: BLE001 - reported as a status to C++
                return 12

        def get_cb(_ctx, key, klen, buf, cap, out_len):
            try:
                k = C.string_at(key, klen).decode()
                v = pending.pop(k, None)
                if v is None:
                    v = bytes(store.get(k))
                out_len[0] = len(v)
                if len(v) > cap:
                    pending[k] = v  # the library retries with a buffer this large
                    return 9        # EW_ERR_CAPACITY
                C.memmove(buf, v, len(v))
                return 0
            except Exception:  # noqa: BLE001
                return 12

        def erase_cb(_ctx, key, klen):
            try:
                store.delete_key(C.string_at(key, klen).decode())
                return 0
            except Exception:  # noqa: BLE001
                return 12

        s_fn, g_fn = N.STORE_SET_FN(set_cb), N.STORE_GET_FN(get_cb)
        e_fn = N.STORE_ERASE_FN(erase_cb)
        h = C.c_void_p()
        check(lib.ew_store_callbacks(s_fn, g_fn, e_fn, None, C.byref(h)))
        return cls(h, keep=(s_fn, g_fn, e_fn, store))

    def set(self, key: str, value: bytes) -> None:
        check(lib.ew_store_set(self._h, key.encode(), value, len(value)))

    def get(self, key: str, cap: int = 1 << 16) -> bytes:
        buf = C.create_string_buffer(cap)
        n = C.c_int64()
        check(lib.ew_store_get(self._h, key.encode(), buf, cap, C.byref(n)))
        return buf.raw[:n.value]

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_store_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


_DEFAULT: Optional[Store] = None
_COUNTERS: Dict[Tuple[int, ...], int] = {}


def default_store() -> Store:
    """The process-wide store over torch.distributed's default c10d store."""
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Store.from_torch()
    return _DEFAULT


def group_members(group=None) -> Tuple[Sequence[int], int]:
    """(global ranks of `group`, this process's global rank)."""
    import torch.distributed as dist
    me = dist.get_rank()
    if group is None:
        return list(range(dist.get_world_size())), me
    return sorted(dist.get_process_group_ranks(group)), me


class Channel:
    """ew_channel: an ordered member list on a store.  Every member creates
    its channels in the same order; members name themselves by global rank."""

    def __init__(self, store: Store, name: str, members: Sequence[int], me: int):
        self.store = store
        self.name = name
        self.members = sorted(int(m) for m in members)
        self.me = int(me)
        h = C.c_void_p()
        check(lib.ew_channel_create(store.handle, name.encode(), N.int_array(self.members),
                                    len(self.members), self.me, C.byref(h)))
        self._h = h

    @classmethod
    def from_group(cls, group=None, tag: str = "ch", store: Optional[Store] = None) -> "Channel":
        """Channel over a torch.distributed group's ranks (collective naming:
        the n-th channel a member set creates gets the same name everywhere)."""
        members, me = group_members(group)
        key = tuple(members)
        n = _COUNTERS.get(key, 0)
        _COUNTERS[key] = n + 1
        name = "ew/" + "-".join(str(m) for m in members) + f"/{tag}{n}"
        return cls(store or default_store(), name, members, me)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def barrier(self) -> None:
        check(lib.ew_channel_barrier(self._h))

    def sum(self, mine: int) -> int:
        t = C.c_int64()
        check(lib.ew_channel_sum(self._h, int(mine), C.byref(t)))
        return t.value

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_channel_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
