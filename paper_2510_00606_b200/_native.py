"""ctypes binding of libelaskit_b200.so (include/ew_api.h).

This is the Python side of the drop-in boundary: every call goes through the
C ABI of the in-tree shared library.  There is no Python or CPU fallback for
any device operation — if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libelaskit_b200.so"

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make -C {_PKG / 'csrc'}` "
        "(or __graft_entry__.build()); there is no fallback implementation")

lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)

# ---------------------------------------------------------------- errors ---

class ElaskitError(RuntimeError):
    """Base of the errors mapped from ew_status codes."""


class CoverageMismatch(ElaskitError):
    """elaskit::CoverageMismatch (param_fabric.hpp:14)."""


class MissingBackup(ElaskitError):
    """elaskit::MissingBackup (rng.hpp:31)."""


class NoSurvivors(ElaskitError):
    """elaskit::NoSurvivors (dataflow.hpp:10)."""


class DimensionMismatch(ElaskitError):
    """elaskit::DimensionMismatch (dataflow.hpp:13)."""


class MismatchedDpDegree(ElaskitError):
    """elaskit::MismatchedDpDegree (migration.hpp:16)."""


class DisconnectedGroup(ElaskitError):
    """elaskit::DisconnectedGroup (communicator.hpp:13)."""


class CapacityError(ElaskitError):
    pass


class InsufficientTargetMemory(ElaskitError):
    """elaskit::InsufficientTargetMemory (migration.hpp:13-15)."""


class CudaError(ElaskitError):
    pass


class NcclError(ElaskitError):
    pass


class InvalidArgument(ElaskitError, ValueError):
    """std::invalid_argument."""


class OutOfRange(ElaskitError, IndexError):
    """std::out_of_range."""


_STATUS = {
    1: InvalidArgument, 2: CoverageMismatch, 3: MissingBackup, 4: NoSurvivors,
    5: DimensionMismatch, 6: MismatchedDpDegree, 7: DisconnectedGroup, 8: OutOfRange,
    9: CapacityError, 10: CudaError, 11: NcclError, 12: ElaskitError, 13: InsufficientTargetMemory,
}

lib.ew_last_error.restype = C.c_char_p
lib.ew_version.restype = C.c_char_p


def check(status: int) -> None:
    if status != 0:
        msg = lib.ew_last_error().decode(errors="replace")
        raise _STATUS.get(status, ElaskitError)(msg)


# ------------------------------------------------------------- signatures ---

i32, i64, u32, u64, f64 = C.c_int, C.c_int64, C.c_uint32, C.c_uint64, C.c_double
vp = C.c_void_p
P = C.POINTER


class Segment(C.Structure):
    _fields_ = [("global_lo", i64), ("length", i64), ("local_off", i64)]


class Interval(C.Structure):
    _fields_ = [("lo", i64), ("hi", i64)]


class TransferEntry(C.Structure):
    _fields_ = [("src_rank", C.c_int32), ("dst_rank", C.c_int32), ("lo", i64), ("hi", i64),
                ("medium", C.c_int32), ("reserved", C.c_int32)]


class MigrationContext(C.Structure):
    _fields_ = [("param_bytes", C.c_int64), ("grad_bytes", C.c_int64),
                ("link_bw_bytes_per_s", C.c_double), ("microbatch_slot_s", C.c_double),
                ("num_microbatches", C.c_int32), ("target_headroom_bytes", C.c_int64),
                ("fixed_overhead_s", C.c_double)]


class TransferSegment(C.Structure):
    _fields_ = [("what", C.c_int32), ("start_s", C.c_double), ("end_s", C.c_double),
                ("bytes", C.c_int64)]


class MigrationSchedule(C.Structure):
    _fields_ = [("mode", C.c_int32), ("shadow_microbatches", C.c_int32),
                ("n_transfers", C.c_int32), ("transfers", TransferSegment * 2),
                ("payback_bytes", C.c_int64), ("stall_s", C.c_double),
                ("total_time_s", C.c_double)]


class AdamHyper(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double)]


class CopyDesc(C.Structure):
    _fields_ = [("src_role", C.c_int32), ("src_rank", C.c_int32), ("dst_role", C.c_int32),
                ("dst_rank", C.c_int32), ("src_off", i64), ("dst_off", i64), ("bytes", i64)]


def _sig(name, restype, *argtypes):
    f = getattr(lib, name)
    f.restype = restype
    f.argtypes = list(argtypes)


_sig("ew_layout_interleaved", i32, P(i64), i32, P(i32), i32, P(vp))
_sig("ew_layout_contiguous", i32, P(i32), i32, i64, P(vp))
_sig("ew_layout_from_intervals", i32, P(i32), P(i32), i32, P(Interval), i64, P(vp))
_sig("ew_layout_free", None, vp)
_sig("ew_layout_total_bytes", i64, vp)
_sig("ew_layout_num_ranks", i32, vp)
_sig("ew_layout_ranks", i32, vp, P(i32), i32)
_sig("ew_layout_shard_bytes", i64, vp, i32)
_sig("ew_layout_num_segments", i64, vp, i32)
_sig("ew_layout_segments", i32, vp, i32, P(Segment), i64)
_sig("ew_layout_validate", i32, vp)
_sig("ew_layout_owner_of", i32, vp, i64)
_sig("ew_integrity_check", i32, P(i32), i32, vp, P(i32), i32, P(i32), P(i32), i32, P(i32))
_sig("ew_overlap_matrix", i32, vp, vp, P(i32), i32, P(i32), i32, P(vp))
_sig("ew_plan_free", None, vp)
_sig("ew_plan_num_entries", i64, vp)
_sig("ew_plan_total_bytes_moved", i64, vp)
_sig("ew_plan_entries", i32, vp, P(TransferEntry), i64)
_sig("ew_plan_to_json", i32, vp, C.c_char_p, i64, P(i64))
_sig("ew_reshard_copies", i32, vp, vp, vp, P(i32), i32, P(i32), i32, i32, i32, P(CopyDesc), i64,
     P(i64))
_sig("ew_inplace_schedule", i32, P(i64), i32, vp, vp, P(i32), i32, i64, i64, i32, P(vp))
_sig("ew_inplace_info", i32, vp, P(i32), P(i32), P(i32), P(i64), P(i64))
_sig("ew_inplace_phases", i32, vp, P(i64))
_sig("ew_inplace_ranges", i32, vp, i32, P(i64), P(i64), P(i64))
_sig("ew_inplace_free", None, vp)
_sig("ew_reshard_microbatches", i32, P(i32), i32, i32, P(i32), i32, P(i32), P(i32))
_sig("ew_weighted_grad_average", i32, P(f64), P(f64), i32, i64, P(f64))
_sig("ew_sample_reassignments", i32, P(i32), P(i32), i32, P(i32), P(i32), i32, P(i64), i64, P(i64))
_sig("ew_plan_zero_migration", i32, i32, i32, P(i64), i32, i32, i32, P(i64), i64, P(i64), P(i64))
_sig("ew_philox4x64", i32, P(u64), P(u64), P(u64))
_sig("ew_draw", i32, u64, u64, u32, u32, i32, P(f64))
_sig("ew_plan_edit", i32, i32, P(C.c_char_p), P(i32), P(i32), P(i32), i32, P(i32), i32, P(i32),
     i32, P(i32), i32, P(i32), P(i32), i32, P(i32), P(i32), P(i32))

_sig("ew_device_count", i32, P(i32))
_sig("ew_set_device", i32, i32)
_sig("ew_alloc", i32, i64, P(vp))
_sig("ew_free", i32, vp)
_sig("ew_memset_async", i32, vp, i32, i64, vp)
_sig("ew_memcpy_async", i32, vp, vp, i64, vp)
_sig("ew_stream_sync", i32, vp)
_sig("ew_device_sync", i32)
_sig("ew_ipc_get_handle", i32, vp, C.c_char_p, P(i64))
_sig("ew_ipc_open", i32, C.c_char_p, i64, P(vp))
_sig("ew_ipc_close", i32, vp)
_sig("ew_host_register", i32, vp, i64, P(vp))
_sig("ew_host_unregister", i32, vp)

_sig("ew_shardmap_create", i32, P(Segment), i64, i64, P(vp))
_sig("ew_shardmap_free", None, vp)
_sig("ew_shardmap_bytes", i64, vp)
_sig("ew_shardmap_num_rows", i64, vp)
_sig("ew_shardmap_row_blocks", i32, vp, P(i64), i64)
_sig("ew_snapshot", i32, vp, vp, vp, vp, vp)
_sig("ew_checksum", i32, vp, vp, vp, vp)
_sig("ew_verify", i32, vp, vp, vp, vp, vp, i64, vp)
_sig("ew_rows_to_blocks", i32, vp, vp, vp, i64, vp)
_sig("ew_fill_synthetic", i32, vp, vp, u64, vp)

_sig("ew_copy_program_create", i32, P(CopyDesc), i64, P(vp), i32, i32, P(vp))
_sig("ew_copy_program_create_raw", i32, P(vp), P(vp), P(i64), P(i32), i64, P(vp))
_sig("ew_copy_program_free", None, vp)
_sig("ew_copy_program_stats", i32, vp, P(i64), P(i64), P(i64))
_sig("ew_copy_program_launch", i32, vp, i32, i32, vp)
_sig("ew_copy_program_launch_guarded", i32, vp, i32, i32, vp, vp, vp)
_sig("ew_copy_program_create_verified", i32, P(CopyDesc), i64, vp, i32, i32, vp, P(vp))
_sig("ew_copy_program_launch_verified", i32, vp, i32, i32, vp, vp)
_sig("ew_copy_program_num_blocks", i32, vp, P(i64))

_sig("ew_philox_dropout_mask", i32, u64, u64, i64, u32, u32, i64, f64, vp, vp)
_sig("ew_philox_uniforms", i32, u64, u64, i64, u32, u32, i64, vp, vp)
_sig("ew_philox_words", i32, u64, u64, u32, u32, u64, i64, vp, vp)

_sig("ew_weighted_absmax", i32, P(vp), P(f64), i32, i64, vp, vp)
_sig("ew_fixed_point_bits", i32, f64, i64, P(i32))
_sig("ew_weighted_fold", i32, P(vp), P(f64), i32, i64, i32, vp, i32, vp)
_sig("ew_weighted_fold_addend", i32, P(vp), P(f64), i32, i64, i32, vp, i32, vp, vp)
_sig("ew_fixed_to_float", i32, vp, i64, i32, vp, vp)
_sig("ew_fixed_to_double", i32, vp, i64, i32, vp, vp)
_sig("ew_fixed_point_bits_async", i32, vp, i64, vp, vp)
_sig("ew_weighted_fold_dev", i32, P(vp), P(f64), i32, i64, vp, vp, i32, vp, vp)
_sig("ew_fixed_to_float_dev", i32, vp, i64, vp, vp, vp)
_sig("ew_weighted_reduce_async", i32, vp, P(vp), P(f64), i32, i64, i64, vp, vp, vp, vp, vp)

_sig("ew_comm_unique_id", i32, C.c_char_p)
_sig("ew_comm_init", i32, C.c_char_p, i32, i32, P(vp))
_sig("ew_comm_shrink", i32, vp, P(i32), i32, i32, P(vp))
_sig("ew_comm_rank", i32, vp, P(i32), P(i32))
_sig("ew_comm_destroy", i32, vp)
_sig("ew_allreduce_i64", i32, vp, vp, i64, vp)
_sig("ew_allreduce_u64", i32, vp, vp, i64, vp)
_sig("ew_allreduce_max_f64", i32, vp, vp, i64, vp)
_sig("ew_weighted_reduce", i32, vp, P(vp), P(f64), i32, i64, i64, vp, vp, vp, P(i32), vp)
_sig("ew_peer_fold_create", i32, i32, i32, i64, P(vp), P(f64), i32, P(vp), P(vp))
_sig("ew_peer_fold_create_i64", i32, i32, i32, i64, P(vp), P(vp), P(vp))
_sig("ew_peer_fold_reduce_scatter", i32, vp, i32, vp)
_sig("ew_peer_fold_all_gather", i32, vp, vp)
_sig("ew_peer_fold_free", None, vp)
_sig("ew_peer_barrier_create", i32, i32, i32, P(vp), P(vp))
_sig("ew_peer_barrier_wait", i32, vp, f64, vp)
_sig("ew_peer_barrier_timed_out", i32, vp, P(i32))
_sig("ew_peer_barrier_error_flag", i32, vp, P(vp))
_sig("ew_peer_barrier_free", None, vp)
_sig("ew_plan_layer_migration", i32, i32, i32, i32, i32, P(MigrationContext), P(MigrationSchedule))
_sig("ew_payback_accumulate", i32, vp, vp, i64, vp)
_sig("ew_adam_scalars", i32, P(AdamHyper), i64, P(C.c_float))
_sig("ew_adam_step", i32, vp, vp, vp, vp, vp, i64, P(AdamHyper), i64, vp)
_sig("ew_adam_step_rows", i32, vp, vp, vp, vp, vp, i64, P(AdamHyper), i64, vp, i64, i64, vp, vp)
_sig("ew_rows_diff", i32, vp, vp, i64, vp, vp)
_sig("ew_comm_split", i32, vp, i32, i32, i32, P(vp))
_sig("ew_peer_access_enable", i32, i32)
_sig("ew_set_device", i32, i32)
_sig("ew_block_verifier_create", i32, P(vp), i32, P(vp), i32, i64, i64, P(vp))
_sig("ew_block_verifier_run", i32, vp, vp, vp)
_sig("ew_block_verifier_free", None, vp)


# --------------------------------------------- multi-process recovery ---

class MttrEventC(C.Structure):
    """ew_mttr_event (ew_api.h): reference MttrEvent (sim.hpp:31-45) + phases."""
    _fields_ = [("step", C.c_int32), ("verified", C.c_int32), ("t_event_s", f64),
                ("kind", C.c_char * 16)] + [(n, f64) for n in (
                    "detect_s", "comm_repair_s", "remap_s", "migration_stall_s", "other_s",
                    "lost_work_s", "plan_edit_s", "comm_acquire_s", "first_collective_s",
                    "comm_prepared", "plan_s", "map_bind_s", "copy_s", "barrier_verify_s",
                    "verdict_exchange_s", "launch_to_verdict_s", "mismatched_block_words",
                    "barrier_timeouts", "premapped", "sums_s", "bind_s", "prepared",
                    "stale_snapshots")]


STORE_SET_FN = C.CFUNCTYPE(i32, vp, C.POINTER(C.c_char), i64, C.POINTER(C.c_char), i64)
STORE_GET_FN = C.CFUNCTYPE(i32, vp, C.POINTER(C.c_char), i64, C.POINTER(C.c_char), i64, P(i64))
STORE_ERASE_FN = C.CFUNCTYPE(i32, vp, C.POINTER(C.c_char), i64)

_sig("ew_store_tcp", i32, C.c_char_p, i32, i32, f64, P(vp))
_sig("ew_store_callbacks", i32, STORE_SET_FN, STORE_GET_FN, STORE_ERASE_FN, vp, P(vp))
_sig("ew_store_set", i32, vp, C.c_char_p, vp, i64)
_sig("ew_store_get", i32, vp, C.c_char_p, vp, i64, P(i64))
_sig("ew_store_free", None, vp)
_sig("ew_channel_create", i32, vp, C.c_char_p, P(i32), i32, i32, P(vp))
_sig("ew_channel_barrier", i32, vp)
_sig("ew_channel_sum", i32, vp, i64, P(i64))
_sig("ew_channel_free", None, vp)
_sig("ew_mttr_csv_header", i32, C.c_char_p, i64)
_sig("ew_mttr_csv_row", i32, P(MttrEventC), i32, C.c_char_p, i64)
_sig("ew_peers_create", i32, P(vp))
_sig("ew_peers_exchange", i32, vp, vp, P(i32), P(vp), i32)
_sig("ew_peers_put", i32, vp, i32, i32, vp)
_sig("ew_peers_get", i32, vp, i32, i32, P(vp))
_sig("ew_peers_free", None, vp)
_sig("ew_reshard_create", i32, vp, vp, P(i32), i32, P(i32), i32, i32, i32, i64, P(vp))
_sig("ew_reshard_bind", i32, vp, vp, i32)
_sig("ew_reshard_launch", i32, vp, vp, vp, i32, i32, vp)
_sig("ew_reshard_free", None, vp)
_sig("ew_prepared_create", i32, vp, P(i64), i32, vp, vp, vp, vp, vp, i64, i64, f64, i32, P(vp))
_sig("ew_prepared_recover", i32, vp, i32, vp, P(MttrEventC), P(i32))
_sig("ew_prepared_new", i32, vp, i32, P(vp), P(i64))
_sig("ew_prepared_free", None, vp)
_sig("ew_dp_group_create", i32, vp, P(i64), i32, vp, i32, i32, i64, i32, P(vp))
_sig("ew_dp_group_create_joiner", i32, vp, C.c_char_p, P(i64), i32, P(i32), i32, i32, i32, i32,
     i64, P(vp))
_sig("ew_dp_group_prepare_join", i32, vp, P(i32), i32)
_sig("ew_dp_group_premap", i32, vp, vp, vp, vp, vp)
_sig("ew_dp_group_prepare_move", i32, vp, i32, P(i32), i32, vp)
_sig("ew_dp_group_attach", i32, vp, vp)
_sig("ew_dp_group_set_snapshot_step", i32, vp, i64)
_sig("ew_dp_group_prepare", i32, vp)
_sig("ew_dp_group_prepare_sets", i32, vp, P(i32), P(i32), i32)
_sig("ew_dp_group_recover", i32, vp, P(i32), i32, i32, vp, vp, vp, i32, vp, P(MttrEventC))
_sig("ew_dp_group_comm", i32, vp, P(vp))
_sig("ew_dp_group_members", i32, vp, P(i32), i32, P(i32))
_sig("ew_dp_group_microbatches", i32, vp, P(i32), i32, P(i32))
_sig("ew_dp_group_free", None, vp)
_sig("ew_detector_create", i32, vp, C.c_char_p, f64, f64, P(vp))
_sig("ew_detector_failed", i32, vp, P(i32), i32, P(i32))
_sig("ew_detector_wait", i32, vp, f64, P(i32), i32, P(i32), P(f64))
_sig("ew_detector_stop", i32, vp)
_sig("ew_detector_free", None, vp)
_sig("ew_inplace_exec_create", i32, vp, P(i64), i32, P(i32), i32, P(i32), i32, vp, vp, i64, i64,
     i32, i32, i32, i64, f64, P(vp))
_sig("ew_inplace_exec_launch", i32, vp, vp, vp)
_sig("ew_inplace_exec_timed_out", i32, vp, P(i32))
_sig("ew_inplace_exec_info", i32, vp, P(i64), P(i64))
_sig("ew_inplace_exec_free", None, vp)
_sig("ew_replay_replica_create", i32, vp, vp, vp, vp, vp, vp, vp, i64, vp, i64, i64, P(vp))
_sig("ew_replay_replica_replay", i32, vp, P(AdamHyper), i64, vp)
_sig("ew_replay_replica_verify", i32, vp, vp, i32, vp)
_sig("ew_replay_replica_owner", i32, vp, P(i32))
_sig("ew_replay_replica_free", None, vp)
_sig("ew_ring_replica_create", i32, vp, vp, vp, vp, vp, i64, P(vp))
_sig("ew_ring_replica_refresh", i32, vp, vp, vp)
_sig("ew_ring_replica_free", None, vp)
_sig("ew_peer_reduce_create", i32, vp, P(vp), P(f64), i32, vp, i64, f64, P(vp))
_sig("ew_peer_reduce_create_i64", i32, vp, vp, vp, i64, f64, P(vp))
_sig("ew_peer_reduce_scale", i32, vp, vp, P(i32))
_sig("ew_peer_reduce_run", i32, vp, i32, vp)
_sig("ew_peer_reduce_wait", i32, vp, vp)
_sig("ew_peer_reduce_info", i32, vp, P(i64), P(i32))
_sig("ew_peer_reduce_free", None, vp)
_sig("ew_write_u64_async", i32, vp, u64, vp)
_sig("ew_host_images_create", i32, vp, vp, C.c_char_p, P(i32), i32, i32, P(vp))
_sig("ew_host_images_publish", i32, vp, vp, i64, vp, P(i64))
_sig("ew_host_images_commit_host", i32, vp, i64)
_sig("ew_host_images_committed", i32, vp, i32, P(i64))
_sig("ew_host_images_device_ptr", i32, vp, i32, P(vp))
_sig("ew_host_images_host_ptr", i32, vp, i32, i64, P(vp), P(i64))
_sig("ew_host_images_free", None, vp)
_sig("ew_layer_migration_create", i32, vp, i32, i32, vp, i64, vp, i64, i32, f64, P(vp))
_sig("ew_layer_migration_step", i32, vp, i32, vp)
_sig("ew_layer_migration_run", i32, vp, i32, P(vp), P(f64), i32, i64, i32, i32, vp, vp)
_sig("ew_layer_migration_info", i32, vp, P(vp), P(i32))
_sig("ew_layer_migration_free", None, vp)

def int_array(values) -> C.Array:
    values = list(values)
    return (i32 * max(1, len(values)))(*values)


def i64_array(values) -> C.Array:
    values = list(values)
    return (i64 * max(1, len(values)))(*values)
