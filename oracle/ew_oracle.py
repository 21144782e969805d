"""ORACLE loaders — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module, and only as the checker / the timed CPU baseline; the
product path (paper_2510_00606_b200) never imports it.

Two libraries:
  oracle/libew_oracle.so       C restatement (ew_oracle.c), always built
  oracle/_ref/libelaskit_ref.so  the reference's own sources + ref_shim.cpp,
                                 built only where /root/reference exists
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "libew_oracle.so"
REF_LIB = HERE / "_ref" / "libelaskit_ref.so"

P = C.POINTER
i32, i64, u32, u64, f64, vp = C.c_int, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_void_p


def _cores() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def _np_ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(P(ctype))


class Oracle:
    """C restatement of the path (ew_oracle.c)."""

    def __init__(self, path: Path = ORACLE_LIB):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C {HERE}`")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ew_oracle_philox4x64.argtypes = [P(u64), P(u64), P(u64)]
        L.ew_oracle_draw.argtypes = [u64, u64, u32, u32, i64, P(f64)]
        L.ew_oracle_dropout_mask.argtypes = [u64, u64, i64, u32, u32, i64, f64, P(u32)]
        L.ew_oracle_splitmix64.argtypes = [u64]
        L.ew_oracle_splitmix64.restype = u64
        L.ew_oracle_num_rows.argtypes = [P(i64), i64, i64]
        L.ew_oracle_num_rows.restype = i64
        L.ew_oracle_row_sums.argtypes = [P(i64), i64, i64, vp, P(u64)]
        L.ew_oracle_row_sums.restype = i64
        L.ew_oracle_block_sums_synthetic.argtypes = [u64, i64, i64, P(u64)]
        L.ew_oracle_rows_synthetic_mt.argtypes = [u64, P(i64), i64, i64, P(u64), C.c_int]
        L.ew_oracle_rows_synthetic_mt.restype = i64
        L.ew_oracle_block_sums_synthetic_mt.argtypes = [u64, i64, i64, P(u64), C.c_int]
        L.ew_oracle_fill_synthetic_mt.argtypes = [P(i64), i64, u64, vp, i64, C.c_int]
        L.ew_oracle_fill_synthetic.argtypes = [P(i64), i64, u64, vp]
        L.ew_oracle_interleaved.argtypes = [P(i64), i32, P(i32), i32, P(i32), P(i64)]
        L.ew_oracle_interleaved.restype = i64
        L.ew_oracle_overlap.argtypes = [P(i32), P(i32), i32, P(i64), P(i32), P(i32), i32, P(i64),
                                        P(i32), i32, P(i32), i32, P(i64), i64]
        L.ew_oracle_overlap.restype = i64
        L.ew_oracle_fixed_point_bits.argtypes = [f64, i64]
        L.ew_oracle_fixed_point_bits.restype = i32
        L.ew_oracle_weighted_fixed.argtypes = [P(f64), P(C.c_float), i32, i64, i32, P(i64)]
        L.ew_oracle_memcpy_mt.argtypes = [P(vp), P(vp), P(i64), i64, i32]
        L.ew_oracle_draw_mt.argtypes = [u64, u64, i64, u32, u32, i64, P(f64), i32]
        L.ew_oracle_weighted_average_mt.argtypes = [P(f64), P(f64), i32, i64, P(f64), i32]
        L.ew_oracle_adam_scalars.argtypes = [f64, f64, f64, f64, f64, i64, P(C.c_float)]
        L.ew_oracle_adam_step.argtypes = [P(C.c_float)] * 4 + [P(C.c_uint16), i64] + [f64] * 5 + [i64]
        L.ew_oracle_snapshot_mt.argtypes = [P(i64), i64, i64, vp, vp, P(u64), i32]
        L.ew_oracle_snapshot_mt.restype = i64
        L.ew_oracle_verify_mt.argtypes = [P(i64), i64, i64, vp, P(u64), i32]
        L.ew_oracle_verify_mt.restype = i64

    # -- multi-threaded CPU baseline of (a)
    def snapshot_mt(self, segments, block_bytes, live: np.ndarray, snap: np.ndarray,
                    threads: int) -> np.ndarray:
        s = self._segs(segments)
        n = self.lib.ew_oracle_num_rows(_np_ptr(s, i64), len(s), block_bytes)
        sums = np.zeros(2 * max(1, n), dtype=np.uint64)
        self.lib.ew_oracle_snapshot_mt(_np_ptr(s, i64), len(s), block_bytes, live.ctypes.data_as(vp),
                                       snap.ctypes.data_as(vp), _np_ptr(sums, u64), threads)
        return sums[:2 * n]

    def verify_mt(self, segments, block_bytes, buf: np.ndarray, expected: np.ndarray,
                  threads: int) -> int:
        s = self._segs(segments)
        e = np.ascontiguousarray(expected, dtype=np.uint64)
        return int(self.lib.ew_oracle_verify_mt(_np_ptr(s, i64), len(s), block_bytes,
                                                buf.ctypes.data_as(vp), _np_ptr(e, u64), threads))

    # -- rng
    def philox4x64(self, counter, key) -> List[int]:
        c, k, o = (u64 * 4)(*counter), (u64 * 2)(*key), (u64 * 4)()
        self.lib.ew_oracle_philox4x64(c, k, o)
        return list(o)

    def draw(self, seed, sample, layer, op, n) -> np.ndarray:
        out = np.zeros(max(1, n), dtype=np.float64)
        self.lib.ew_oracle_draw(seed, sample, layer, op, n, _np_ptr(out, f64))
        return out[:n]

    def dropout_mask(self, seed, sample_lo, n_samples, layer, op, n_elems, keep) -> np.ndarray:
        wpr = (n_elems + 31) // 32
        out = np.zeros((max(1, n_samples), max(1, wpr)), dtype=np.uint32)
        self.lib.ew_oracle_dropout_mask(seed, sample_lo, n_samples, layer, op, n_elems, keep,
                                        _np_ptr(out, u32))
        return out[:n_samples, :wpr]

    # -- checksum
    @staticmethod
    def _segs(segments) -> np.ndarray:
        a = np.asarray([[int(s["global_lo"]), int(s["length"]), int(s["local_off"])]
                        for s in segments], dtype=np.int64).reshape(-1, 3)
        return np.ascontiguousarray(a)

    def row_sums(self, segments, block_bytes: int, buf: np.ndarray) -> np.ndarray:
        s = self._segs(segments)
        n = self.lib.ew_oracle_num_rows(_np_ptr(s, i64), len(s), block_bytes)
        out = np.zeros(2 * max(1, n), dtype=np.uint64)
        b = np.ascontiguousarray(buf, dtype=np.uint8)
        self.lib.ew_oracle_row_sums(_np_ptr(s, i64), len(s), block_bytes,
                                    b.ctypes.data_as(vp), _np_ptr(out, u64))
        return out[:2 * n]

    def block_sums_synthetic(self, seed: int, total: int, block_bytes: int) -> np.ndarray:
        nb = (total + block_bytes - 1) // block_bytes
        out = np.zeros(2 * max(1, nb), dtype=np.uint64)
        self.lib.ew_oracle_block_sums_synthetic(seed, total, block_bytes, _np_ptr(out, u64))
        return out[:2 * nb]

    def rows_synthetic_mt(self, segments, block_bytes: int, seed: int,
                          threads: int = 0) -> np.ndarray:
        """Rows of the synthetic state placed by `segments`, no buffer."""
        s = self._segs(segments)
        n = self.lib.ew_oracle_num_rows(_np_ptr(s, i64), len(s), block_bytes)
        out = np.zeros(2 * max(1, n), dtype=np.uint64)
        self.lib.ew_oracle_rows_synthetic_mt(seed, _np_ptr(s, i64), len(s), block_bytes,
                                             _np_ptr(out, u64), threads or _cores())
        return out[:2 * n]

    def block_sums_synthetic_mt(self, seed: int, total: int, block_bytes: int,
                                threads: int = 0) -> np.ndarray:
        nb = (total + block_bytes - 1) // block_bytes
        out = np.zeros(2 * max(1, nb), dtype=np.uint64)
        self.lib.ew_oracle_block_sums_synthetic_mt(seed, total, block_bytes, _np_ptr(out, u64),
                                                   threads or _cores())
        return out[:2 * nb]

    def fill_synthetic_mt(self, segments, nbytes: int, seed: int, threads: int = 0) -> np.ndarray:
        s = self._segs(segments)
        buf = np.empty(max(1, nbytes), dtype=np.uint8)
        self.lib.ew_oracle_fill_synthetic_mt(_np_ptr(s, i64), len(s), seed, buf.ctypes.data_as(vp),
                                             nbytes, threads or _cores())
        return buf[:nbytes]

    def fill_synthetic(self, segments, nbytes: int, seed: int) -> np.ndarray:
        s = self._segs(segments)
        buf = np.zeros(max(1, nbytes), dtype=np.uint8)
        self.lib.ew_oracle_fill_synthetic(_np_ptr(s, i64), len(s), seed, buf.ctypes.data_as(vp))
        return buf[:nbytes]

    # -- plans
    def interleaved(self, layer_bytes: Sequence[int], ranks: Sequence[int]) -> Dict[int, list]:
        ranks = sorted(ranks)
        lb = np.asarray(layer_bytes, dtype=np.int64)
        counts = np.zeros(len(ranks), dtype=np.int32)
        ivs = np.zeros(2 * len(ranks) * max(1, len(lb)), dtype=np.int64)
        self.lib.ew_oracle_interleaved(_np_ptr(lb, i64), len(lb),
                                       _np_ptr(np.asarray(ranks, dtype=np.int32), i32),
                                       len(ranks), _np_ptr(counts, i32), _np_ptr(ivs, i64))
        out, k = {}, 0
        for r, c in zip(ranks, counts):
            out[r] = [(int(ivs[2 * (k + j)]), int(ivs[2 * (k + j) + 1])) for j in range(c)]
            k += c
        return out

    def overlap(self, src: Dict[int, list], dst: Dict[int, list], failed=(), ring=()) -> np.ndarray:
        def flat(layout):
            ranks = sorted(layout)
            counts = np.asarray([len(layout[r]) for r in ranks], dtype=np.int32)
            ivs = np.asarray([x for r in ranks for iv in layout[r] for x in iv], dtype=np.int64)
            return np.asarray(ranks, dtype=np.int32), counts, ivs if ivs.size else np.zeros(2, np.int64)

        sr, sc, si = flat(src)
        dr, dc, di = flat(dst)
        cap = (sum(len(v) for v in src.values()) + 1) * (sum(len(v) for v in dst.values()) + 1)
        out = np.zeros(5 * cap, dtype=np.int64)
        f = np.asarray(sorted(failed) or [0], dtype=np.int32)
        rg = np.asarray(list(ring) or [0], dtype=np.int32)
        n = self.lib.ew_oracle_overlap(_np_ptr(sr, i32), _np_ptr(sc, i32), len(sr), _np_ptr(si, i64),
                                       _np_ptr(dr, i32), _np_ptr(dc, i32), len(dr), _np_ptr(di, i64),
                                       _np_ptr(f, i32), len(failed), _np_ptr(rg, i32), len(ring),
                                       _np_ptr(out, i64), cap)
        assert n >= 0
        return out[:5 * n].reshape(-1, 5)

    # -- weighted reduce
    def fixed_point_bits(self, absmax: float, total_units: int) -> int:
        return self.lib.ew_oracle_fixed_point_bits(absmax, total_units)

    def weighted_fixed(self, weights, grads: np.ndarray, frac_bits: int) -> np.ndarray:
        g = np.ascontiguousarray(grads, dtype=np.float32)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = np.zeros(g.shape[1], dtype=np.int64)
        self.lib.ew_oracle_weighted_fixed(_np_ptr(w, f64), _np_ptr(g, C.c_float), len(w),
                                          g.shape[1], frac_bits, _np_ptr(out, i64))
        return out

    # -- multi-threaded CPU paths timed beside the GPU kernels
    def memcpy_mt(self, srcs, dsts, nbytes, threads: int) -> None:
        n = len(nbytes)
        s = (vp * max(1, n))(*srcs)
        d = (vp * max(1, n))(*dsts)
        b = np.ascontiguousarray(nbytes, dtype=np.int64)
        self.lib.ew_oracle_memcpy_mt(s, d, _np_ptr(b, i64), n, threads)

    def draw_mt(self, seed, sample_lo, n_samples, layer, op, n_per_sample, threads) -> np.ndarray:
        out = np.empty(max(1, n_samples * n_per_sample), dtype=np.float64)
        self.lib.ew_oracle_draw_mt(seed, sample_lo, n_samples, layer, op, n_per_sample,
                                   _np_ptr(out, f64), threads)
        return out[:n_samples * n_per_sample].reshape(n_samples, n_per_sample)

    def weighted_average_mt(self, weights, grads: np.ndarray, threads: int) -> np.ndarray:
        g = np.ascontiguousarray(grads, dtype=np.float64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = np.empty(max(1, g.shape[1]), dtype=np.float64)
        self.lib.ew_oracle_weighted_average_mt(_np_ptr(w, f64), _np_ptr(g, f64), len(w),
                                               g.shape[1], _np_ptr(out, f64), threads)
        return out[:g.shape[1]]

    # -- ring replica by optimizer replay
    def adam_scalars(self, hyper, step: int) -> np.ndarray:
        out = np.zeros(8, dtype=np.float32)
        self.lib.ew_oracle_adam_scalars(*hyper, step, _np_ptr(out, C.c_float))
        return out

    def adam_step(self, grad: np.ndarray, master: np.ndarray, exp_avg: np.ndarray,
                  exp_avg_sq: np.ndarray, param: np.ndarray, hyper, step: int) -> None:
        """In place; hyper = (lr, beta1, beta2, eps, weight_decay)."""
        arrs = [grad, master, exp_avg, exp_avg_sq]
        for a in arrs:
            assert a.dtype == np.float32 and a.flags.c_contiguous
        assert param.dtype == np.uint16 and param.flags.c_contiguous
        self.lib.ew_oracle_adam_step(*[_np_ptr(a, C.c_float) for a in arrs],
                                     _np_ptr(param, C.c_uint16), len(grad), *hyper, step)


class Reference:
    """The reference's own implementation (oracle/_ref/libelaskit_ref.so)."""

    STATUS = {1: "invalid_argument", 2: "CoverageMismatch", 3: "MissingBackup", 4: "NoSurvivors",
              5: "DimensionMismatch", 6: "MismatchedDpDegree", 7: "DisconnectedGroup",
              8: "out_of_range", 9: "capacity", 12: "exception", 13: "InsufficientTargetMemory"}

    def __init__(self, path: Path = REF_LIB):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing (reference not built here)")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_overlap_matrix.argtypes = [P(i32), P(i32), i32, P(i64), P(i32), P(i32), i32, P(i64),
                                         i64, P(i32), i32, P(i32), i32, P(i64), i64, P(i64),
                                         P(i64), P(f64)]
        L.ref_plan_to_json.argtypes = [P(i32), P(i32), i32, P(i64), P(i32), P(i32), i32, P(i64),
                                       i64, P(i32), i32, P(i32), i32, C.c_char_p, i64]
        L.ref_integrity_check.argtypes = [P(i32), i32, P(i32), P(i32), i32, P(i64), i64, P(i32),
                                          i32, P(i32), P(i32), P(i32)]
        L.ref_zero_shard.argtypes = [P(i64), i32, i32, i32, i32, P(i64), P(i64), P(i64)]
        L.ref_plan_layer_migration.argtypes = [i32, i32, i32, i32, P(i64), P(f64), P(i64), P(f64)]
        L.ref_plan_layer_migration.restype = i32
        L.ref_plan_zero_migration.argtypes = [i32, i32, P(i64), i32, i32, i32, P(i64), i64,
                                              P(i64), P(i64)]
        L.ref_philox4x64.argtypes = [P(u64), P(u64), P(u64)]
        L.ref_draw.argtypes = [u64, u64, u32, u32, i32, P(f64)]
        L.ref_dropout_mask.argtypes = [u64, u64, i64, u32, u32, i32, f64, P(u32)]
        L.ref_weighted_grad_average.argtypes = [P(f64), P(f64), i32, i64, P(f64)]
        L.ref_reshard_microbatches.argtypes = [P(i32), i32, i32, P(i32), i32, P(i32), P(i32)]
        L.ref_plan_edit.argtypes = [i32, P(C.c_char_p), P(i32), P(i32), P(i32), i32, P(i32), i32,
                                    P(i32), i32, P(i32), P(i32), P(i32), P(i32), P(i32), P(i32)]

    def _raise(self, st: int):
        if st:
            raise RuntimeError(f"{self.STATUS.get(st, st)}: {self.lib.ref_last_error().decode()}")

    @staticmethod
    def _flat(layout: Dict[int, list]):
        ranks = sorted(layout)
        counts = np.asarray([len(layout[r]) for r in ranks], dtype=np.int32)
        ivs = np.asarray([x for r in ranks for iv in layout[r] for x in iv] or [0, 0],
                         dtype=np.int64)
        return np.asarray(ranks or [0], dtype=np.int32), counts if counts.size else np.zeros(1, np.int32), ivs, len(ranks)

    def overlap_matrix(self, src, dst, total, failed=(), ring=None,
                       return_status=False) -> Tuple[np.ndarray, int, float]:
        sr, sc, si, sn = self._flat(src)
        dr, dc, di, dn = self._flat(dst)
        cap = (sum(len(v) for v in src.values()) + 1) * (sum(len(v) for v in dst.values()) + 1)
        cap = min(cap, 50_000_000)
        out = np.zeros(5 * cap, dtype=np.int64)
        f = np.asarray(sorted(failed) or [0], dtype=np.int32)
        rg = np.asarray(list(ring) if ring else [0], dtype=np.int32)
        n, moved, secs = i64(), i64(), f64()
        st = self.lib.ref_overlap_matrix(_np_ptr(sr, i32), _np_ptr(sc, i32), sn, _np_ptr(si, i64),
                                         _np_ptr(dr, i32), _np_ptr(dc, i32), dn, _np_ptr(di, i64),
                                         total, _np_ptr(f, i32), len(failed), _np_ptr(rg, i32),
                                         len(ring) if ring else 0, _np_ptr(out, i64), cap,
                                         C.byref(n), C.byref(moved), C.byref(secs))
        if return_status and st:
            return st
        self._raise(st)
        return out[:5 * n.value].reshape(-1, 5), moved.value, secs.value

    def plan_to_json(self, src, dst, total, failed=(), ring=None) -> str:
        sr, sc, si, sn = self._flat(src)
        dr, dc, di, dn = self._flat(dst)
        f = np.asarray(sorted(failed) or [0], dtype=np.int32)
        rg = np.asarray(list(ring) if ring else [0], dtype=np.int32)
        buf = C.create_string_buffer(1 << 24)
        self._raise(self.lib.ref_plan_to_json(_np_ptr(sr, i32), _np_ptr(sc, i32), sn,
                                              _np_ptr(si, i64), _np_ptr(dr, i32), _np_ptr(dc, i32),
                                              dn, _np_ptr(di, i64), total, _np_ptr(f, i32),
                                              len(failed), _np_ptr(rg, i32),
                                              len(ring) if ring else 0, buf, 1 << 24))
        return buf.value.decode()

    def integrity_check(self, ring, layout, total, failed) -> Tuple[bool, List[int]]:
        r, c, ivs, n = self._flat(layout)
        rg = np.asarray(ring, dtype=np.int32)
        f = np.asarray(sorted(failed) or [0], dtype=np.int32)
        rec, nm = i32(), i32()
        miss = np.zeros(max(1, len(failed)), dtype=np.int32)
        self._raise(self.lib.ref_integrity_check(_np_ptr(rg, i32), len(rg), _np_ptr(r, i32),
                                                 _np_ptr(c, i32), n, _np_ptr(ivs, i64), total,
                                                 _np_ptr(f, i32), len(failed), C.byref(rec),
                                                 _np_ptr(miss, i32), C.byref(nm)))
        return bool(rec.value), [int(x) for x in miss[:nm.value]]

    def interleaved(self, layer_bytes, ranks) -> Dict[int, list]:
        """Interleaved composition using the reference's ZeroLayout::shard."""
        ranks = sorted(ranks)
        lb = np.asarray(layer_bytes, dtype=np.int64)
        out = {r: [] for r in ranks}
        lo, hi, off = i64(), i64(), i64()
        for l in range(len(lb)):
            for j, r in enumerate(ranks):
                self._raise(self.lib.ref_zero_shard(_np_ptr(lb, i64), len(lb), len(ranks), l, j,
                                                    C.byref(lo), C.byref(hi), C.byref(off)))
                if hi.value > lo.value:
                    out[r].append((off.value + lo.value, off.value + hi.value))
        return out

    def plan_zero_migration(self, interleaved: bool, dp: int, layer_bytes, layer: int,
                            dst_dp: int):
        lb = np.asarray(layer_bytes, dtype=np.int64)
        cap = 4 * dp * dp + 64
        out = np.zeros(6 * cap, dtype=np.int64)
        n = i64()
        tot = np.zeros(3, dtype=np.int64)
        st = self.lib.ref_plan_zero_migration(int(interleaved), dp, _np_ptr(lb, i64), len(lb),
                                              layer, dst_dp, _np_ptr(out, i64), cap, C.byref(n),
                                              _np_ptr(tot, i64))
        if st:
            return st, None, None
        return 0, out[:6 * n.value].reshape(-1, 6), tot

    def plan_layer_migration(self, layer, src, dst, nonblocking: bool, ctx: dict):
        """-> (status, dict) with the MigrationSchedule fields (migration.hpp:29-39)."""
        ic = np.array([ctx["param_bytes"], ctx["grad_bytes"], ctx["num_microbatches"],
                       ctx["target_headroom_bytes"]], dtype=np.int64)
        dc = np.array([ctx["link_bw_bytes_per_s"], ctx["microbatch_slot_s"],
                       ctx["fixed_overhead_s"]], dtype=np.float64)
        io, do = np.zeros(8, dtype=np.int64), np.zeros(6, dtype=np.float64)
        st = self.lib.ref_plan_layer_migration(layer, src, dst, int(nonblocking), _np_ptr(ic, i64),
                                               _np_ptr(dc, f64), _np_ptr(io, i64), _np_ptr(do, f64))
        if st:
            return st, None
        tr = [("payback_grad" if io[4 + 2 * k] else "params", float(do[2 + 2 * k]),
               float(do[3 + 2 * k]), int(io[5 + 2 * k])) for k in range(int(io[2]))]
        return 0, {"mode": int(io[0]), "shadow_microbatches": int(io[1]), "transfers": tr,
                   "payback_bytes": int(io[3]), "stall_s": float(do[0]),
                   "total_time_s": float(do[1])}

    def philox4x64(self, counter, key):
        c, k, o = (u64 * 4)(*counter), (u64 * 2)(*key), (u64 * 4)()
        self.lib.ref_philox4x64(c, k, o)
        return list(o)

    def draw(self, seed, sample, layer, op, n) -> np.ndarray:
        out = np.zeros(max(1, n), dtype=np.float64)
        self._raise(self.lib.ref_draw(seed, sample, layer, op, n, _np_ptr(out, f64)))
        return out[:n]

    def dropout_mask(self, seed, sample_lo, n_samples, layer, op, n_elems, keep) -> np.ndarray:
        wpr = (n_elems + 31) // 32
        out = np.zeros((max(1, n_samples), max(1, wpr)), dtype=np.uint32)
        self._raise(self.lib.ref_dropout_mask(seed, sample_lo, n_samples, layer, op, n_elems,
                                              keep, _np_ptr(out, u32)))
        return out[:n_samples, :wpr]

    def weighted_grad_average(self, weights, grads) -> np.ndarray:
        g = np.ascontiguousarray(grads, dtype=np.float64)
        w = np.ascontiguousarray(weights, dtype=np.float64)
        out = np.zeros(g.shape[1], dtype=np.float64)
        self._raise(self.lib.ref_weighted_grad_average(_np_ptr(w, f64), _np_ptr(g, f64), len(w),
                                                       g.shape[1], _np_ptr(out, f64)))
        return out

    def reshard_microbatches(self, per_slot_mbs, num_mb, survivors):
        n = len(survivors)
        s = np.zeros(max(1, n), dtype=np.int32)
        m = np.zeros(max(1, n), dtype=np.int32)
        old = np.asarray(per_slot_mbs or [0], dtype=np.int32)
        sv = np.asarray(survivors or [0], dtype=np.int32)
        st = self.lib.ref_reshard_microbatches(_np_ptr(old, i32), len(per_slot_mbs), num_mb,
                                               _np_ptr(sv, i32), n, _np_ptr(s, i32),
                                               _np_ptr(m, i32))
        if st:
            return st, None, None
        return 0, list(s[:n]), list(m[:n])

    def plan_edit(self, groups, kind, targets, pool):
        """groups: list of (id, members, ring) -> (status, add, remove, touched ids)."""
        pool = sorted({(min(a, b), max(a, b)) for a, b in pool})
        ids = (C.c_char_p * max(1, len(groups)))(*[g[0].encode() for g in groups])
        topo = np.asarray([1 if g[2] else 0 for g in groups] or [0], dtype=np.int32)
        nmem = np.asarray([len(g[1]) for g in groups] or [0], dtype=np.int32)
        mem = np.asarray([m for g in groups for m in g[1]] or [0], dtype=np.int32)
        tg = np.asarray(list(targets) or [0], dtype=np.int32)
        pl = np.asarray([x for l in pool for x in l] or [0], dtype=np.int32)
        cap = sum(len(g[1]) ** 2 for g in groups) + len(pool) + 4
        add = np.zeros(2 * cap, dtype=np.int32)
        rem = np.zeros(2 * cap, dtype=np.int32)
        touched = np.zeros(max(1, len(groups)), dtype=np.int32)
        na, nr, nt = i32(), i32(), i32()
        st = self.lib.ref_plan_edit(len(groups), ids, _np_ptr(topo, i32), _np_ptr(nmem, i32),
                                    _np_ptr(mem, i32), kind, _np_ptr(tg, i32), len(targets),
                                    _np_ptr(pl, i32), len(pool), _np_ptr(add, i32), C.byref(na),
                                    _np_ptr(rem, i32), C.byref(nr), _np_ptr(touched, i32),
                                    C.byref(nt))
        if st:
            return st, None, None, None
        return (0, {(int(add[2 * i]), int(add[2 * i + 1])) for i in range(na.value)},
                {(int(rem[2 * i]), int(rem[2 * i + 1])) for i in range(nr.value)},
                {groups[int(touched[i])][0] for i in range(nt.value)})


def load_oracle() -> Oracle:
    return Oracle()


def load_reference() -> Optional[Reference]:
    try:
        return Reference()
    except FileNotFoundError:
        return None
