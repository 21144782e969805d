"""A C++ consumer written against include/elaskit (planners + the device.hpp
wrapper) compiles and links against libelaskit_b200.so and plans a reshard
without a GPU — the drop-in boundary from the C++ side."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

SRC = r'''
#include "elaskit/device.hpp"
#include <cstdio>
int main() {
  using namespace elaskit;
  ZeroLayout z; z.kind = ZeroKind::Interleaved; z.layer_bytes = {400, 400, 400};
  auto src = b200::interleaved_layout(z, {0, 1, 2, 3});
  auto dst = b200::interleaved_layout(z, {0, 2, 3});
  SnapshotRing ring; ring.members = {0, 1, 2, 3};
  auto plan = overlap_matrix(src, dst, {1}, &ring);
  std::size_t n = 0;
  for (int r : {0, 2, 3}) n += b200::reshard_copies(plan, src, dst, {1}, &ring, r, false).size();
  int mapped = 0;
  try { device::check(EW_ERR_MISSING_BACKUP); } catch (const MissingBackup&) { mapped = 1; }
  std::printf("%zu %lld %zu %d\n", plan.entries.size(), (long long)plan.total_bytes_moved, n, mapped);
  return 0;
}
'''


def test_cpp_consumer_builds_and_plans(tmp_path):
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    src = tmp_path / "consumer.cpp"
    src.write_text(SRC)
    exe = tmp_path / "consumer"
    lib = ROOT / "paper_2510_00606_b200"
    subprocess.run(["g++", "-std=c++20", f"-I{ROOT / 'include'}", f"-I{ROOT / 'third_party' / 'nlohmann'}",
                    str(src), f"-L{lib}", "-l:libelaskit_b200.so", f"-Wl,-rpath,{lib}", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    n_entries, moved, n_copies, mapped = map(int, out)
    assert moved == 402 and n_entries == 9 and mapped == 1
    assert n_copies >= n_entries  # every entry lowered once (pull), plus retained bytes


def test_cpp_recovery_driver_builds():
    """tools/cpp/recover_demo.cpp — the DP recovery driven from C++ only."""
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    subprocess.run(["make", "-s", "-C", str(ROOT / "tools" / "cpp")], check=True)
    assert (ROOT / "tools" / "cpp" / "recover_demo").exists()
    # the multi-process driver (C++ only, TCP store rendezvous, DpGroup)
    assert (ROOT / "tools" / "cpp" / "dp_recover").exists()
    r = subprocess.run([str(ROOT / "tools" / "cpp" / "dp_recover")], capture_output=True,
                       text=True)
    assert r.returncode == 2 and "usage" in r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("d,failed,mode", [(4, 1, ""), (8, 3, ""), (8, 0, ""), (3, 2, ""),
                                           (8, 3, "inplace"), (4, 0, "inplace")])
def test_cpp_recovery_driver_runs(d, failed, mode):
    import json
    subprocess.run(["make", "-s", "-C", str(ROOT / "tools" / "cpp")], check=True)
    args = [str(ROOT / "tools" / "cpp" / "recover_demo"), str(d), str(failed), "0.01"]
    out = subprocess.run(args + ([mode] if mode else []), capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["conserved"] and res["bytes_ok"]


EVENT_SRC = r'''
#include "elaskit/b200.hpp"
#include <cstdio>
int main() {
  using namespace elaskit;
  // one pipeline stage of DP 8 (config B), rank r = device r
  ClusterState st = make_uniform_cluster(1, 8, 180LL << 30);
  ElasticEvent ev; ev.kind = EventKind::FailStop; ev.targets = {3};
  const b200::DpTransition t = b200::dp_transition(st, ev, 1);
  ZeroLayout z; z.kind = ZeroKind::Interleaved;
  z.layer_bytes.push_back(131072000LL * 14);
  for (int l = 0; l < 32; ++l) z.layer_bytes.push_back(202383360LL * 14);
  z.layer_bytes.push_back(131076096LL * 14);
  const auto src = b200::interleaved_layout(z, t.old_members);
  const auto dst = b200::interleaved_layout(z, t.members);
  SnapshotRing ring; ring.members = t.old_members;
  const auto rep = integrity_check(ring, src, t.departed);
  const auto plan = overlap_matrix(src, dst, t.departed, &ring);
  // a second, adjacent failure leaves rank 3's bytes without a holder
  ElasticEvent ev2; ev2.kind = EventKind::FailStop; ev2.targets = {2};
  const b200::DpTransition t2 = b200::dp_transition(t.next, ev2, 1);
  std::set<int> both = {2, 3};
  const auto rep2 = integrity_check(ring, src, both);
  ElasticEvent slow; slow.kind = EventKind::FailSlow; slow.targets = {5}; slow.slow_factor = 1.5;
  const b200::DpTransition t3 = b200::dp_transition(st, slow, 1);
  std::printf("%zu %zu %d %lld %zu %d %zu %zu %zu\n", t.old_members.size(), t.members.size(),
              *t.departed.begin(), (long long)plan.total_bytes_moved, plan.entries.size(),
              (int)rep.recoverable, t2.members.size(), (std::size_t)rep2.recoverable,
              t3.slow.size() + 10 * t3.departed.size());
  return 0;
}
'''


def test_cpp_event_to_plan(tmp_path):
    """Cluster model -> DP membership -> layouts -> plan from C++: a FailStop
    of device 3 in config B's DP 8 stage yields the reference's 7B 8->7 drop-r3
    plan (238 entries, 26.954 GB moved)."""
    if shutil.which("g++") is None:
        pytest.skip("no g++")
    src = tmp_path / "event.cpp"
    src.write_text(EVENT_SRC)
    exe = tmp_path / "event"
    lib = ROOT / "paper_2510_00606_b200"
    subprocess.run(["g++", "-std=c++20", f"-I{ROOT / 'include'}", f"-I{ROOT / 'third_party' / 'nlohmann'}",
                    str(src), f"-L{lib}", "-l:libelaskit_b200.so", f"-Wl,-rpath,{lib}", "-o", str(exe)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    old_n, new_n, departed, moved, entries, ok, new2, ok2, slow = map(int, out)
    assert (old_n, new_n, departed) == (8, 7, 3)
    assert entries == 238 and round(moved / 1e9, 3) == 26.954
    assert ok == 1 and new2 == 6 and ok2 == 0
    assert slow == 1  # one slow member, nobody departed
