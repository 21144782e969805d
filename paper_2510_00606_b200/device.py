"""Device side of the recovery path: thin wrappers over the sm_100a kernels.

Torch is used only as the device-memory/stream plumbing: buffers are torch
tensors whose raw pointers are handed to libelaskit_b200.so, kernels are
enqueued on torch's current CUDA stream.  Every op here executes in the CUDA
library; none has a CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _native as N
from ._native import check, lib
from .fabric import COPY_DTYPE, SEGMENT_DTYPE

DEFAULT_BLOCK_BYTES = 64 * 1024


def _stream(stream: Optional[torch.cuda.Stream] = None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> C.c_void_p:
    if t is None:
        return C.c_void_p(None)
    if not t.is_cuda:
        raise ValueError("device op needs a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("device op needs a contiguous tensor")
    return C.c_void_p(t.data_ptr())


def device_count() -> int:
    n = C.c_int()
    check(lib.ew_device_count(C.byref(n)))
    return n.value


def empty_bytes(nbytes: int, device=None) -> torch.Tensor:
    """16-byte aligned (caching allocator: 512 B) uint8 buffer, padded to 16."""
    return torch.empty(max(16, (int(nbytes) + 15) // 16 * 16), dtype=torch.uint8,
                       device=device or "cuda")


# ---------------------------------------------------------------- (a) ---

class ShardMap:
    """Packed shard buffer geometry + checksum rows, resident on the device
    (ew_shardmap)."""

    def __init__(self, segments: np.ndarray, block_bytes: int = DEFAULT_BLOCK_BYTES):
        segs = np.ascontiguousarray(segments, dtype=SEGMENT_DTYPE)
        self.segments = segs
        self.block_bytes = int(block_bytes)
        h = C.c_void_p()
        check(lib.ew_shardmap_create(segs.ctypes.data_as(C.POINTER(N.Segment)), len(segs),
                                     self.block_bytes, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_shardmap_free(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def nbytes(self) -> int:
        return lib.ew_shardmap_bytes(self._h)

    @property
    def num_rows(self) -> int:
        return lib.ew_shardmap_num_rows(self._h)

    def row_blocks(self) -> np.ndarray:
        out = np.zeros(max(1, self.num_rows), dtype=np.int64)
        check(lib.ew_shardmap_row_blocks(self._h, out.ctypes.data_as(C.POINTER(C.c_int64)),
                                         self.num_rows))
        return out[:self.num_rows]

    def new_row_sums(self, device=None) -> torch.Tensor:
        return torch.zeros(2 * max(1, self.num_rows), dtype=torch.int64, device=device or "cuda")


def snapshot(m: ShardMap, live: torch.Tensor, snap: torch.Tensor, row_sums: torch.Tensor,
             stream=None) -> None:
    """snap <- live fused with the per-block checksum rows of live."""
    _check_buf(m, live)
    _check_buf(m, snap)
    check(lib.ew_snapshot(m.handle, _ptr(live), _ptr(snap), _ptr(row_sums), _stream(stream)))


def checksum(m: ShardMap, buf: torch.Tensor, row_sums: torch.Tensor, stream=None) -> None:
    _check_buf(m, buf)
    check(lib.ew_checksum(m.handle, _ptr(buf), _ptr(row_sums), _stream(stream)))


def verify(m: ShardMap, buf: torch.Tensor, expected: torch.Tensor, bad_count: torch.Tensor,
           bad_rows: Optional[torch.Tensor] = None, stream=None) -> None:
    """bad_count (device int32[1]) <- number of rows whose checksum differs."""
    _check_buf(m, buf)
    cap = 0 if bad_rows is None else bad_rows.numel()
    check(lib.ew_verify(m.handle, _ptr(buf), _ptr(expected), _ptr(bad_count), _ptr(bad_rows), cap,
                        _stream(stream)))


def rows_to_blocks(m: ShardMap, row_sums: torch.Tensor, block_sums: torch.Tensor,
                   stream=None) -> None:
    check(lib.ew_rows_to_blocks(m.handle, _ptr(row_sums), _ptr(block_sums),
                                block_sums.numel() // 2, _stream(stream)))


def fill_synthetic(m: ShardMap, buf: torch.Tensor, seed: int, stream=None) -> None:
    _check_buf(m, buf)
    check(lib.ew_fill_synthetic(m.handle, _ptr(buf), int(seed), _stream(stream)))


def _check_buf(m: ShardMap, buf: torch.Tensor) -> None:
    if buf.numel() * buf.element_size() < m.nbytes:
        raise ValueError(f"buffer holds {buf.numel() * buf.element_size()} bytes, "
                         f"shard needs {m.nbytes}")


# ---------------------------------------------------------------- (b) ---

class CopyProgram:
    """A GPU's reshard copies, resolved to pointers and resident on the device."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @classmethod
    def from_descs(cls, descs: np.ndarray, buf_table: Dict[Tuple[int, int], int],
                   table_ranks: int, exec_rank: int,
                   verify_map: Optional["ShardMap"] = None) -> "CopyProgram":
        """verify_map: NEW's segment map on exec_rank -> a verified program
        (ew_copy_program_create_verified: checksums what lands, see launch)."""
        d = np.ascontiguousarray(descs, dtype=COPY_DTYPE)
        table = (C.c_void_p * (3 * table_ranks))()
        for (role, rank), ptr in buf_table.items():
            table[role * table_ranks + rank] = ptr
        h = C.c_void_p()
        dp = d.ctypes.data_as(C.POINTER(N.CopyDesc))
        if verify_map is None:
            check(lib.ew_copy_program_create(dp, len(d), table, table_ranks, exec_rank,
                                             C.byref(h)))
        else:
            check(lib.ew_copy_program_create_verified(dp, len(d), table, table_ranks, exec_rank,
                                                      verify_map.handle, C.byref(h)))
        prog = cls(h)
        prog._verify_map = verify_map  # keep the map alive with the program
        return prog

    @classmethod
    def from_pointers(cls, srcs: Sequence[int], dsts: Sequence[int], nbytes: Sequence[int],
                      remote: Sequence[bool]) -> "CopyProgram":
        n = len(nbytes)
        s = (C.c_void_p * max(1, n))(*srcs)
        d = (C.c_void_p * max(1, n))(*dsts)
        b = N.i64_array(nbytes)
        r = N.int_array([1 if x else 0 for x in remote])
        h = C.c_void_p()
        check(lib.ew_copy_program_create_raw(s, d, b, r, n, C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_copy_program_free(self._h)
            self._h = None

    def stats(self) -> Tuple[int, int, int]:
        n, r, l = C.c_int64(), C.c_int64(), C.c_int64()
        check(lib.ew_copy_program_stats(self._h, C.byref(n), C.byref(r), C.byref(l)))
        return n.value, r.value, l.value

    def launch(self, n_ctas: int = 0, remote_ctas: int = 0, stream=None,
               block_sums: Optional[torch.Tensor] = None, abort_flag: Optional[int] = None) -> None:
        """block_sums (int64 [2 * num_blocks()], zeroed by the caller): the
        landed bytes' checksums are added there (verified programs only).
        abort_flag: device address of an int (PeerBarrier.error_flag); the
        copy writes nothing if it is set when the kernel starts."""
        if abort_flag is not None:
            check(lib.ew_copy_program_launch_guarded(self._h, n_ctas, remote_ctas,
                                                     _ptr(block_sums), C.c_void_p(abort_flag),
                                                     _stream(stream)))
        elif block_sums is None:
            check(lib.ew_copy_program_launch(self._h, n_ctas, remote_ctas, _stream(stream)))
        else:
            check(lib.ew_copy_program_launch_verified(self._h, n_ctas, remote_ctas,
                                                      _ptr(block_sums), _stream(stream)))

    def num_blocks(self) -> int:
        n = C.c_int64()
        check(lib.ew_copy_program_num_blocks(self._h, C.byref(n)))
        return n.value


def ipc_handle(t: torch.Tensor) -> Tuple[bytes, int]:
    h = C.create_string_buffer(64)
    off = C.c_int64()
    check(lib.ew_ipc_get_handle(_ptr(t), h, C.byref(off)))
    return h.raw, off.value


def ipc_open(handle: bytes, offset: int) -> int:
    p = C.c_void_p()
    check(lib.ew_ipc_open(handle, offset, C.byref(p)))
    return p.value


def ipc_close(ptr: int) -> None:
    check(lib.ew_ipc_close(C.c_void_p(ptr)))


def host_register(addr: int, nbytes: int) -> int:
    """Pin host range [addr, addr + nbytes) (e.g. node-shared memory) and
    return the device address copy programs read it through (ew_host_register)."""
    p = C.c_void_p()
    check(lib.ew_host_register(C.c_void_p(addr), int(nbytes), C.byref(p)))
    return p.value


def host_unregister(addr: int) -> None:
    check(lib.ew_host_unregister(C.c_void_p(addr)))


# ---------------------------------------------------------------- (c) ---

def mask_words(n_elems: int) -> int:
    return (int(n_elems) + 31) // 32


def dropout_mask(seed: int, sample_lo: int, n_samples: int, layer_id: int, op_index: int,
                 n_elems: int, keep_probability: float, out: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
    """Packed keep-bits [n_samples, ceil(n_elems/32)] int32 (bit = element kept)."""
    if out is None:
        out = torch.empty((n_samples, mask_words(n_elems)), dtype=torch.int32, device="cuda")
    check(lib.ew_philox_dropout_mask(seed, sample_lo, n_samples, layer_id, op_index, n_elems,
                                     float(keep_probability), _ptr(out), _stream(stream)))
    return out


def philox_uniforms(seed: int, sample_lo: int, n_samples: int, layer_id: int, op_index: int,
                    n_elems: int, stream=None) -> torch.Tensor:
    out = torch.empty((n_samples, n_elems), dtype=torch.float64, device="cuda")
    check(lib.ew_philox_uniforms(seed, sample_lo, n_samples, layer_id, op_index, n_elems,
                                 _ptr(out), _stream(stream)))
    return out


def philox_words(seed: int, sample_id: int, layer_id: int, op_index: int, block_lo: int,
                 n_blocks: int, stream=None) -> torch.Tensor:
    out = torch.empty((n_blocks, 4), dtype=torch.int64, device="cuda")
    check(lib.ew_philox_words(seed, sample_id, layer_id, op_index, block_lo, n_blocks, _ptr(out),
                              _stream(stream)))
    return out


# ---------------------------------------------------------------- (d) ---

def _units(units: Sequence[torch.Tensor], weights: Sequence[float]):
    if len(units) != len(weights):
        raise ValueError("one weight per unit")
    n = None
    for u in units:
        if u.dtype != torch.float32:
            raise ValueError("units must be float32")
        n = u.numel() if n is None else n
        if u.numel() != n:
            raise N.DimensionMismatch(f"gradient vectors differ in length: {u.numel()} vs {n}")
    ptrs = (C.c_void_p * max(1, len(units)))(*[u.data_ptr() for u in units])
    w = (C.c_double * max(1, len(weights)))(*[float(x) for x in weights])
    return ptrs, w, (n or 0)


def weighted_absmax(units, weights, out: Optional[torch.Tensor] = None, stream=None):
    ptrs, w, n = _units(units, weights)
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device="cuda")
    check(lib.ew_weighted_absmax(ptrs, w, len(units), n, _ptr(out), _stream(stream)))
    return out


def fixed_point_bits(global_absmax: float, total_units: int) -> int:
    f = C.c_int()
    check(lib.ew_fixed_point_bits(float(global_absmax), int(total_units), C.byref(f)))
    return f.value


def weighted_fold(units, weights, frac_bits: int, acc: torch.Tensor, accumulate: bool = False,
                  stream=None, addend=None) -> torch.Tensor:
    """acc (+)= sum_u rint(w_u g_u 2^F) [+ addend], one pass (ew_weighted_fold_addend).
    `addend`: int64 tensor, or a raw (library-owned or peer) device pointer to
    at least n int64 values."""
    ptrs, w, n = _units(units, weights)
    if acc.dtype != torch.int64 or acc.numel() < n:
        raise ValueError("acc must be int64 with one slot per element")
    if isinstance(addend, torch.Tensor):
        if addend.dtype != torch.int64 or addend.numel() < n:
            raise ValueError("addend must be int64 with one slot per element")
        add = _ptr(addend)
    else:
        add = C.c_void_p(int(addend) if addend else None)
    check(lib.ew_weighted_fold_addend(ptrs, w, len(units), n, int(frac_bits), _ptr(acc),
                                      int(accumulate), add, _stream(stream)))
    return acc


def fixed_to_float(acc: torch.Tensor, frac_bits: int, out: Optional[torch.Tensor] = None,
                   stream=None) -> torch.Tensor:
    if out is None:
        out = torch.empty(acc.numel(), dtype=torch.float32, device=acc.device)
    check(lib.ew_fixed_to_float(_ptr(acc), acc.numel(), int(frac_bits), _ptr(out),
                                _stream(stream)))
    return out


def fixed_point_bits_async(global_absmax: torch.Tensor, total_units: int,
                           bits: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
    """ew_fixed_point_bits_async: the scale computed on the device (int32)."""
    if bits is None:
        bits = torch.empty(1, dtype=torch.int32, device="cuda")
    check(lib.ew_fixed_point_bits_async(_ptr(global_absmax), int(total_units), _ptr(bits),
                                        _stream(stream)))
    return bits


def weighted_fold_dev(units, weights, bits: torch.Tensor, acc: torch.Tensor,
                      accumulate: bool = False, stream=None) -> torch.Tensor:
    """ew_weighted_fold_dev: the fold with the scale read from device memory."""
    ptrs, w, n = _units(units, weights)
    if acc.dtype != torch.int64 or acc.numel() < n:
        raise ValueError("acc must be int64 with one slot per element")
    check(lib.ew_weighted_fold_dev(ptrs, w, len(units), n, _ptr(bits), _ptr(acc),
                                   int(accumulate), None, _stream(stream)))
    return acc


def fixed_to_float_dev(acc: torch.Tensor, bits: torch.Tensor, out: Optional[torch.Tensor] = None,
                       stream=None) -> torch.Tensor:
    if out is None:
        out = torch.empty(acc.numel(), dtype=torch.float32, device=acc.device)
    check(lib.ew_fixed_to_float_dev(_ptr(acc), acc.numel(), _ptr(bits), _ptr(out),
                                    _stream(stream)))
    return out


def fixed_to_double(acc: torch.Tensor, frac_bits: int, out: Optional[torch.Tensor] = None,
                    stream=None) -> torch.Tensor:
    if out is None:
        out = torch.empty(acc.numel(), dtype=torch.float64, device=acc.device)
    check(lib.ew_fixed_to_double(_ptr(acc), acc.numel(), int(frac_bits), _ptr(out),
                                 _stream(stream)))
    return out


class PeerFold:
    """(d) fused with its collective over NVLink peer memory (ew_peer_fold).

    Built from EVERY rank's unit pointers/weights and output buffers (peer
    pointers IPC-mapped by the caller).  reduce_scatter -> host barrier ->
    all_gather leaves the full reduced fp32 vector in this rank's output."""

    def __init__(self, world: int, rank: int, n_elems: int, unit_ptrs: Sequence[int],
                 weights: Optional[Sequence[float]], out_ptrs: Sequence[int]):
        """weights=None: unit_ptrs are the world's per-rank int64
        accumulators (ew_peer_fold_create_i64), one per rank in rank order."""
        u = (C.c_void_p * max(1, len(unit_ptrs)))(*unit_ptrs)
        o = (C.c_void_p * max(1, len(out_ptrs)))(*out_ptrs)
        h = C.c_void_p()
        if weights is None:
            if len(unit_ptrs) != world:
                raise ValueError("one int64 accumulator per rank")
            check(lib.ew_peer_fold_create_i64(world, rank, int(n_elems), u, o, C.byref(h)))
        else:
            w = (C.c_double * max(1, len(weights)))(*[float(x) for x in weights])
            check(lib.ew_peer_fold_create(world, rank, int(n_elems), u, w, len(unit_ptrs), o,
                                          C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value and lib is not None:
            lib.ew_peer_fold_free(self._h)
            self._h = None

    def reduce_scatter(self, frac_bits: int, stream=None) -> None:
        check(lib.ew_peer_fold_reduce_scatter(self._h, int(frac_bits), _stream(stream)))

    def all_gather(self, stream=None) -> None:
        check(lib.ew_peer_fold_all_gather(self._h, _stream(stream)))

    def run(self, frac_bits: int, barrier: "PeerBarrier", stream=None) -> None:
        """barrier -> reduce-scatter -> barrier -> all-gather, all enqueued on
        one stream (no host synchronisation; device-timed)."""
        barrier.wait(stream)
        self.reduce_scatter(frac_bits, stream)
        barrier.wait(stream)
        self.all_gather(stream)


class PeerBarrier:
    """Stream-ordered cross-GPU barrier over peer memory (ew_peer_barrier)."""

    def __init__(self, group=None, timeout_s: float = 30.0):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.timeout_s = timeout_s
        self.flags = torch.zeros(max(2, self.world), dtype=torch.int64, device="cuda")
        handles = [None] * self.world
        dist.all_gather_object(handles, ipc_handle(self.flags), group=group)
        self._opened = []
        ptrs = []
        for r, (h, off) in enumerate(handles):
            if r == self.rank:
                ptrs.append(self.flags.data_ptr())
            else:
                p = ipc_open(h, off)
                self._opened.append(p)
                ptrs.append(p)
        torch.cuda.synchronize()
        dist.barrier(group=group)  # every flag array is zero before first use
        arr = (C.c_void_p * self.world)(*ptrs)
        h = C.c_void_p()
        check(lib.ew_peer_barrier_create(self.world, self.rank, arr, C.byref(h)))
        self._h = h

    def wait(self, stream=None) -> None:
        check(lib.ew_peer_barrier_wait(self._h, self.timeout_s, _stream(stream)))

    def timed_out(self) -> bool:
        t = C.c_int()
        check(lib.ew_peer_barrier_timed_out(self._h, C.byref(t)))
        return bool(t.value)

    @property
    def error_flag(self) -> int:
        """Device address of the int a timeout sets (CopyProgram.launch
        abort_flag): writes ordered after a failed barrier do not run."""
        p = C.c_void_p()
        check(lib.ew_peer_barrier_error_flag(self._h, C.byref(p)))
        return int(p.value)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.ew_peer_barrier_free(self._h)
            self._h = None
        for p in self._opened:
            ipc_close(p)
        self._opened = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def peer_weighted_reduce_setup(units: Sequence[torch.Tensor], weights: Sequence[float],
                               out: torch.Tensor, group=None):
    """Exchange IPC handles of every rank's units and output buffer (over
    torch.distributed, plumbing only) and build this rank's PeerFold.
    Returns (fold, total_units, opened_peer_pointers)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    mine = {"units": [ipc_handle(u) for u in units], "w": [float(x) for x in weights],
            "out": ipc_handle(out), "n": out.numel()}
    allv = [None] * world
    dist.all_gather_object(allv, mine, group=group)
    opened, unit_ptrs, wts, out_ptrs = [], [], [], []
    for r, d in enumerate(allv):
        if d["n"] != out.numel():
            raise N.DimensionMismatch("ranks disagree on the gradient length")
        if r == rank:
            unit_ptrs += [u.data_ptr() for u in units]
            out_ptrs.append(out.data_ptr())
        else:
            for h, off in d["units"]:
                p = ipc_open(h, off)
                opened.append(p)
                unit_ptrs.append(p)
            p = ipc_open(*d["out"])
            opened.append(p)
            out_ptrs.append(p)
        wts += d["w"]
    fold = PeerFold(world, rank, out.numel(), unit_ptrs, wts, out_ptrs)
    return fold, len(unit_ptrs), opened


def peer_sum_i64_setup(acc: torch.Tensor, out: torch.Tensor, group=None):
    """Peer collective over per-rank int64 accumulators (each rank folded its
    own micro-batch units into `acc`): exchange IPC handles and build the
    PeerFold.  fold.run(frac_bits, barrier) leaves the dequantised sum in
    `out` on every rank.  Returns (fold, opened_peer_pointers)."""
    import torch.distributed as dist
    if acc.dtype != torch.int64 or acc.numel() != out.numel():
        raise ValueError("acc must be int64 with out.numel() elements")
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    allv = [None] * world
    dist.all_gather_object(allv, (ipc_handle(acc), ipc_handle(out), out.numel()), group=group)
    opened, acc_ptrs, out_ptrs = [], [], []
    for r, (ha, ho, n) in enumerate(allv):
        if n != out.numel():
            raise N.DimensionMismatch("ranks disagree on the gradient length")
        if r == rank:
            acc_ptrs.append(acc.data_ptr())
            out_ptrs.append(out.data_ptr())
        else:
            for h, lst in ((ha, acc_ptrs), (ho, out_ptrs)):
                p = ipc_open(*h)
                opened.append(p)
                lst.append(p)
    return PeerFold(world, rank, out.numel(), acc_ptrs, None, out_ptrs), opened


class Communicator:
    """NCCL communicator of the DP group (ew_comm), shrinkable in place."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        r, n = C.c_int(), C.c_int()
        check(lib.ew_comm_rank(self._h, C.byref(r), C.byref(n)))
        self.rank, self.size = r.value, n.value

    @staticmethod
    def unique_id() -> bytes:
        b = C.create_string_buffer(128)
        check(lib.ew_comm_unique_id(b))
        return b.raw

    @classmethod
    def init(cls, uid: bytes, nranks: int, rank: int) -> "Communicator":
        h = C.c_void_p()
        check(lib.ew_comm_init(uid, nranks, rank, C.byref(h)))
        return cls(h)

    def shrink(self, exclude: Sequence[int], abort: bool = False) -> Optional["Communicator"]:
        """ncclCommShrink; returns None on an excluded rank."""
        h = C.c_void_p()
        check(lib.ew_comm_shrink(self._h, N.int_array(exclude), len(exclude), int(abort),
                                 C.byref(h)))
        return Communicator(h) if h.value else None

    def destroy(self) -> None:
        """Free the communicator; a no-op on a borrowed one (a recovery.DpGroup
        owns its communicators) or one whose ownership moved."""
        if getattr(self, "_borrowed", False):
            self._h = None
            return
        if self._h is not None and self._h.value:
            check(lib.ew_comm_destroy(self._h))
            self._h = None

    def split(self, color: int, key: int, share: bool = True) -> Optional["Communicator"]:
        """ncclCommSplit; color < 0 leaves this rank out (returns None)."""
        h = C.c_void_p()
        check(lib.ew_comm_split(self._h, int(color), int(key), int(bool(share)), C.byref(h)))
        return Communicator(h) if h.value else None

    def allreduce_i64(self, t: torch.Tensor, stream=None) -> None:
        check(lib.ew_allreduce_i64(self._h, _ptr(t), t.numel(), _stream(stream)))

    def allreduce_u64(self, t: torch.Tensor, stream=None) -> None:
        check(lib.ew_allreduce_u64(self._h, _ptr(t), t.numel(), _stream(stream)))

    def allreduce_max_f64(self, t: torch.Tensor, stream=None) -> None:
        check(lib.ew_allreduce_max_f64(self._h, _ptr(t), t.numel(), _stream(stream)))

    def weighted_reduce(self, units, weights, total_units: int, out: torch.Tensor,
                        ws_acc: torch.Tensor, ws_max: torch.Tensor, stream=None) -> int:
        """Full (d) path; returns the fixed-point fraction bits used."""
        ptrs, w, n = _units(units, weights)
        f = C.c_int()
        check(lib.ew_weighted_reduce(self._h, ptrs, w, len(units), int(total_units), n,
                                     _ptr(ws_acc), _ptr(ws_max), _ptr(out), C.byref(f),
                                     _stream(stream)))
        return f.value

    def weighted_reduce_async(self, units, weights, total_units: int, out: torch.Tensor,
                              ws_acc: torch.Tensor, ws_max: torch.Tensor, ws_bits: torch.Tensor,
                              stream=None) -> None:
        """Full (d) path with the scale in device memory (`ws_bits`, int32):
        no host synchronisation, capturable in a CUDA graph."""
        ptrs, w, n = _units(units, weights)
        check(lib.ew_weighted_reduce_async(self._h, ptrs, w, len(units), int(total_units), n,
                                           _ptr(ws_acc), _ptr(ws_max), _ptr(ws_bits), _ptr(out),
                                           _stream(stream)))


# ------------------------------------- ring replica by optimizer replay ---
class AdamState:
    """One ZeRO shard's AdamW state in HBM, the layout ew_adam_step updates:
    fp32 master weights, fp32 exp_avg, fp32 exp_avg_sq and the bf16
    parameter copy (14 B/param, the mixed-precision state of SURVEY §8(d)),
    structure of arrays in ONE allocation with zeroed padding, so the whole
    state is a single byte image that kernel (a) snapshots and checksums and
    kernel (b) moves.  Sections start on 1 MiB boundaries (the largest
    checksum block), which lets ew_adam_step_rows give each CTA exactly one
    block per section (≤ 3 MiB of padding per shard)."""

    SECTION_ALIGN = 1 << 20

    def __init__(self, n: int, device=None, buf: Optional[torch.Tensor] = None):
        al = self.SECTION_ALIGN
        a = lambda b: (int(b) + al - 1) // al * al
        self.n = int(n)
        sec = a(4 * self.n)
        self.nbytes = 3 * sec + (int(2 * self.n) + 255) // 256 * 256
        if buf is None:
            buf = torch.zeros(self.nbytes, dtype=torch.uint8, device=device or "cuda")
        if buf.numel() < self.nbytes or buf.data_ptr() % 256:
            raise ValueError("AdamState buffer too small or not 256-byte aligned")
        # the image's block grid is relative to buf, so buf's own alignment
        # does not matter for the rows; only section offsets do
        self.buf = buf
        f32 = lambda k: buf[k * sec:k * sec + 4 * self.n].view(torch.float32)
        self.master, self.exp_avg, self.exp_avg_sq = f32(0), f32(1), f32(2)
        self.param = buf[3 * sec:3 * sec + 2 * self.n].view(torch.bfloat16)

    def segments(self) -> np.ndarray:
        """The state's byte image as one segment at global offset 0."""
        s = np.zeros(1, dtype=SEGMENT_DTYPE)
        s[0] = (0, self.nbytes, 0)
        return s


def adam_hyper(lr: float = 1e-4, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
               weight_decay: float = 0.01) -> N.AdamHyper:
    return N.AdamHyper(lr, beta1, beta2, eps, weight_decay)


def adam_scalars(hyper: N.AdamHyper, step: int) -> np.ndarray:
    out = (C.c_float * 8)()
    check(lib.ew_adam_scalars(C.byref(hyper), int(step), out))
    return np.frombuffer(out, dtype=np.float32).copy()


def adam_step(grad, state: AdamState, hyper: N.AdamHyper, step: int, stream=None,
              rows: Optional[torch.Tensor] = None,
              block_bytes: int = DEFAULT_BLOCK_BYTES) -> None:
    """ew_adam_step over the whole shard.  `grad`: fp32 tensor of state.n
    elements, or a raw device pointer (an IPC-mapped peer gradient shard).
    With `rows` (int64 [2 * rows]), the checksum rows of the state image after
    the step are produced in the same pass (ew_adam_step_rows); they equal
    checksum(ShardMap(state.segments(), block_bytes), state.buf)."""
    if isinstance(grad, torch.Tensor):
        if grad.dtype != torch.float32 or grad.numel() < state.n:
            raise ValueError("grad must be fp32 with state.n elements")
        g = _ptr(grad)
    else:
        g = C.c_void_p(int(grad))
    args = (g, _ptr(state.master), _ptr(state.exp_avg), _ptr(state.exp_avg_sq),
            _ptr(state.param), state.n, C.byref(hyper), int(step))
    if rows is None:
        check(lib.ew_adam_step(*args, _stream(stream)))
        return
    n_rows = (state.nbytes + block_bytes - 1) // block_bytes
    if rows.dtype != torch.int64 or rows.numel() < 2 * n_rows:
        raise ValueError("rows must be int64 with 2 slots per block of the state image")
    check(lib.ew_adam_step_rows(*args, _ptr(state.buf), state.nbytes, block_bytes, _ptr(rows),
                                _stream(stream)))


def rows_diff(a: torch.Tensor, b: torch.Tensor, n_rows: int, bad_count: torch.Tensor,
              stream=None) -> None:
    """bad_count (device int32[1]) <- number of rows where a and b differ."""
    check(lib.ew_rows_diff(_ptr(a), _ptr(b), int(n_rows), _ptr(bad_count), _stream(stream)))
