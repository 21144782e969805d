"""The C ABI library loads without a GPU, exports every entry point that
include/ew_api.h declares, and maps the reference's exceptions to status
codes (no compute calls here)."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

from paper_2510_00606_b200 import _native as N
from paper_2510_00606_b200 import fabric

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "ew_api.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ew_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) > 60
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (ew_[a-z0-9_]+)$", out, flags=re.M))
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_cpp_api_symbols_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    for sym in ("elaskit::overlap_matrix(", "elaskit::integrity_check(",
                "elaskit::contiguous_layout(", "elaskit::plan_to_json[abi:cxx11](",
                "elaskit::philox4x64(", "elaskit::draw(", "elaskit::reshard_rng(",
                "elaskit::resolve_stream(", "elaskit::make_stream_map(",
                "elaskit::reshard_microbatches(", "elaskit::weighted_grad_average(",
                "elaskit::plan_edit(", "elaskit::estimate_recovery_time(",
                "elaskit::plan_zero_migration(", "elaskit::ZeroLayout::shard(",
                "elaskit::b200::interleaved_layout(", "elaskit::b200::reshard_copies("):
        assert sym in out, sym


def test_library_loads_without_gpu_and_reports_version():
    assert b"sm_100a" in N.lib.ew_version()
    n = C.c_int(-1)
    N.check(N.lib.ew_device_count(C.byref(n)))
    assert n.value >= 0


def test_status_codes_map_to_reference_exceptions():
    with pytest.raises(N.CoverageMismatch):
        fabric.overlap_matrix(fabric.contiguous_layout([0, 1], 10), fabric.contiguous_layout([0, 1], 12))
    with pytest.raises(N.NoSurvivors):
        fabric.reshard_microbatches([2, 2], 4, [])
    with pytest.raises(N.InvalidArgument):
        fabric.draw(0, 0, 0, 0, 0)  # draw count must be >= 1 (rng.cpp:39)
    with pytest.raises(N.InvalidArgument):
        fabric.integrity_check(fabric.SnapshotRing([0, 1]), fabric.contiguous_layout([0, 1], 8), [5])
    with pytest.raises(N.DisconnectedGroup):
        fabric.plan_edit([fabric.CommGroup("star", [0, 1, 2, 3])], fabric.FAIL_STOP, [0],
                         {(0, 1), (0, 2), (0, 3)})


def test_shardmap_rejects_bad_segments_without_gpu():
    # geometry validation happens before any device call
    bad = (N.Segment * 2)(N.Segment(0, 10, 0), N.Segment(5, 10, 10))  # overlapping globals
    h = C.c_void_p()
    with pytest.raises(N.CoverageMismatch):
        N.check(N.lib.ew_shardmap_create(bad, 2, 65536, C.byref(h)))
    with pytest.raises(N.InvalidArgument):
        N.check(N.lib.ew_shardmap_create(bad, 1, 1000, C.byref(h)))  # not a power of two


def test_dp_group_membership_entry_points_validate_without_gpu():
    """ScaleOut / departure-set entry points reject bad arguments before any
    device or store call (joiner groups, prepared sets, premap, prepared
    moves, the event kinds recover accepts)."""
    h = C.c_void_p()
    lb = (C.c_int64 * 2)(1 << 20, 1 << 20)
    members = (C.c_int * 2)(0, 1)
    with pytest.raises(N.InvalidArgument):  # no store
        N.check(N.lib.ew_dp_group_create_joiner(None, b"dp", lb, 2, members, 2, 2, 4, 32, 65536,
                                                C.byref(h)))
    one = (C.c_int * 1)(3)
    offs = (C.c_int * 2)(0, 1)
    with pytest.raises(N.InvalidArgument):
        N.check(N.lib.ew_dp_group_prepare_join(None, one, 1))
    with pytest.raises(N.InvalidArgument):
        N.check(N.lib.ew_dp_group_prepare_sets(None, one, offs, 1))
    with pytest.raises(N.InvalidArgument):
        N.check(N.lib.ew_dp_group_premap(None, None, None, None, None))
    with pytest.raises(N.InvalidArgument):
        N.check(N.lib.ew_dp_group_prepare_move(None, 3, one, 1, None))
    ev = N.MttrEventC()
    with pytest.raises(N.InvalidArgument):  # NULL group (a ScaleOut, kind 3)
        N.check(N.lib.ew_dp_group_recover(None, one, 1, 3, None, None, None, 0, None,
                                          C.byref(ev)))
