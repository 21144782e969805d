// C++ recovery driver: the DP recovery path without Python.
//
// Written against the drop-in headers exactly like a reference caller
// (sim.cpp's recover_elaswave would be): elaskit planners + the RAII device
// layer (elaskit/device.hpp) over the C ABI.  All ranks' shards live on one
// GPU (a single-process stand-in for one-process-per-GPU), so it runs on any
// B200 and checks itself:
//   1. interleaved layouts of a scaled 7B state over D ranks, fail one rank
//   2. integrity_check -> overlap_matrix -> per-rank copy programs
//   3. fill the source shards (+ the ring holder's replica) with the
//      synthetic state, run every program, verify by checksum conservation
//      and by regenerating the expected target bytes.
//
//   recover_demo [D=4] [failed=1] [scale=0.02] [inplace]
//
// "inplace": the staged in-place variant (b200::inplace_schedule) — each
// rank keeps ONE buffer (OLD on entry, NEW on exit); per phase every rank's
// direct and staged copies run, then the staged bytes are flushed.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "elaskit/device.hpp"

using namespace elaskit;

namespace {

void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    std::exit(2);
  }
}

struct Buffer {
  void* p = nullptr;
  std::int64_t n = 0;
  explicit Buffer(std::int64_t bytes) : n(bytes) {
    cuda(cudaMalloc(&p, std::max<std::int64_t>(32, (bytes + 31) / 32 * 32)), "cudaMalloc");
  }
  ~Buffer() { cudaFree(p); }
};

std::vector<ew_segment> segments(const PartitionLayout& l, int rank) {
  std::vector<ew_segment> out;
  for (const auto& s : b200::shard_segments(l, rank)) out.push_back({s.global_lo, s.length, s.local_off});
  return out;
}

void fill(const PartitionLayout& l, int rank, void* buf, std::uint64_t seed) {
  auto segs = segments(l, rank);
  ew_shardmap* m = nullptr;
  device::check(ew_shardmap_create(segs.data(), static_cast<std::int64_t>(segs.size()), 65536, &m));
  device::check(ew_fill_synthetic(m, buf, seed, nullptr));
  ew_shardmap_free(m);
}

// checksum rows of one shard, scattered into global block sums
void add_blocks(const PartitionLayout& l, int rank, const void* buf, std::uint64_t* blocks,
                std::int64_t n_blocks) {
  device::ShardMap m(l, rank);
  std::uint64_t* rows = nullptr;
  cuda(cudaMalloc(&rows, 16 * std::max<std::int64_t>(1, m.rows())), "cudaMalloc rows");
  device::check(ew_checksum(m.get(), buf, rows, nullptr));
  device::check(ew_rows_to_blocks(m.get(), rows, blocks, n_blocks, nullptr));
  cuda(cudaDeviceSynchronize(), "sync");
  cudaFree(rows);
}

int holder_of(const SnapshotRing& ring, int r) { return ring.backed_up_by(r); }

}  // namespace

int main(int argc, char** argv) {
  const int D = argc > 1 ? std::atoi(argv[1]) : 4;
  const int failed_rank = argc > 2 ? std::atoi(argv[2]) : 1;
  const double scale = argc > 3 ? std::atof(argv[3]) : 0.02;
  cuda(cudaSetDevice(0), "cudaSetDevice");

  // scaled Llama-2 7B ZeRO state (14 B/param), interleaved over D ranks
  ZeroLayout z;
  z.kind = ZeroKind::Interleaved;
  z.layer_bytes.push_back(static_cast<std::int64_t>(131072000 * scale) * 14);
  for (int l = 0; l < 32; ++l) z.layer_bytes.push_back(static_cast<std::int64_t>(202383360 * scale) * 14);
  z.layer_bytes.push_back(static_cast<std::int64_t>(131076096 * scale) * 14);
  std::vector<int> old_ranks, new_ranks;
  for (int r = 0; r < D; ++r) {
    old_ranks.push_back(r);
    if (r != failed_rank) new_ranks.push_back(r);
  }
  const std::set<int> failed = {failed_rank};
  SnapshotRing ring;
  ring.members = old_ranks;

  const auto t0 = std::chrono::steady_clock::now();
  const PartitionLayout src = b200::interleaved_layout(z, old_ranks);
  const PartitionLayout dst = b200::interleaved_layout(z, new_ranks);
  if (!integrity_check(ring, src, failed).recoverable) {
    std::fprintf(stderr, "unrecoverable\n");
    return 1;
  }
  const TransferPlan plan = overlap_matrix(src, dst, failed, &ring);
  const auto t1 = std::chrono::steady_clock::now();

  const bool in_place = argc > 4 && std::string(argv[4]) == "inplace";
  if (in_place) {
    const b200::InPlaceSchedule sc = b200::inplace_schedule(
        z.layer_bytes, src, dst, failed, /*stage=*/1 << 20, /*phase=*/2 << 20, /*slack=*/1);
    std::map<int, std::unique_ptr<Buffer>> buf;
    std::vector<void*> tab(3 * D, nullptr);
    for (int r : old_ranks) {
      const std::int64_t n = std::max(b200::shard_bytes(src, r), b200::shard_bytes(dst, r));
      buf[r] = std::make_unique<Buffer>(n);
      if (!failed.count(r)) fill(src, r, buf[r]->p, 7);
      tab[0 * D + r] = buf[r]->p;
    }
    Buffer replica(b200::shard_bytes(src, failed_rank));
    fill(src, failed_rank, replica.p, 7);
    tab[1 * D + holder_of(ring, failed_rank)] = replica.p;
    const std::int64_t n_blocks = (src.total_bytes + 65535) / 65536;
    std::uint64_t* before = nullptr;
    cuda(cudaMalloc(&before, 16 * n_blocks), "malloc");
    cudaMemset(before, 0, 16 * n_blocks);
    for (int r : old_ranks)
      if (!failed.count(r)) add_blocks(src, r, buf[r]->p, before, n_blocks);
    add_blocks(src, failed_rank, replica.p, before, n_blocks);
    // one staging buffer per rank: phases run one after another here (the
    // multi-GPU executor rotates sc.ring of them to let ranks run ahead)
    std::map<int, std::unique_ptr<Buffer>> staging;
    for (int r : new_ranks)
      staging[r] = std::make_unique<Buffer>(std::max<std::int64_t>(16, sc.stage_alloc));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    int programs = 0;
    for (std::size_t j = 0; j < sc.phases.size(); ++j) {
      std::vector<std::unique_ptr<device::CopyProgram>> keep;
      std::vector<ew_copy_program*> flushes;
      for (int r : new_ranks) {
        const auto copies = b200::reshard_copies(plan, src, dst, failed, &ring, r, false);
        const b200::InPlaceRanges& rr = sc.ranks.at(r);
        // direct part: lands in NEW at its own offsets
        std::vector<void*> t = tab;
        t[2 * D + r] = buf[r]->p;
        const auto d = b200::clip_copies(copies, rr.direct[j].first, rr.direct[j].second,
                                         rr.direct[j].first);
        if (!d.empty()) {
          keep.push_back(std::make_unique<device::CopyProgram>(d, t, D, r));
          keep.back()->launch(nullptr);
        }
        // staged part: into staging (alignment kept mod 16), flushed once
        // every rank has gathered the phase (the barrier)
        const auto [lo, hi] = rr.staged[j];
        if (hi > lo) {
          void* st = staging[r]->p;
          std::vector<void*> ts = tab;
          ts[2 * D + r] = st;
          keep.push_back(std::make_unique<device::CopyProgram>(
              b200::clip_copies(copies, lo, hi, lo % 16), ts, D, r));
          keep.back()->launch(nullptr);
          const void* fs[1] = {static_cast<char*>(st) + lo % 16};
          void* fd[1] = {static_cast<char*>(buf[r]->p) + lo};
          const std::int64_t fb[1] = {hi - lo};
          const int rem[1] = {0};
          ew_copy_program* flush = nullptr;
          device::check(ew_copy_program_create_raw(fs, fd, fb, rem, 1, &flush));
          flushes.push_back(flush);
        }
      }
      programs += static_cast<int>(keep.size() + flushes.size());
      for (ew_copy_program* f : flushes) device::check(ew_copy_program_launch(f, 64, 0, nullptr));
      cuda(cudaDeviceSynchronize(), "phase");
      for (ew_copy_program* f : flushes) ew_copy_program_free(f);
    }
    cudaEventRecord(b);
    cuda(cudaEventSynchronize(b), "in-place");
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::uint64_t* after = nullptr;
    cuda(cudaMalloc(&after, 16 * n_blocks), "malloc");
    cudaMemset(after, 0, 16 * n_blocks);
    for (int r : new_ranks) add_blocks(dst, r, buf[r]->p, after, n_blocks);
    std::vector<std::uint64_t> hb(2 * n_blocks), ha(2 * n_blocks);
    cudaMemcpy(hb.data(), before, 16 * n_blocks, cudaMemcpyDeviceToHost);
    cudaMemcpy(ha.data(), after, 16 * n_blocks, cudaMemcpyDeviceToHost);
    const bool conserved = hb == ha;
    bool bytes_ok = true;
    for (int r : new_ranks) {
      const std::int64_t n = b200::shard_bytes(dst, r);
      Buffer expect(n);
      fill(dst, r, expect.p, 7);
      std::vector<unsigned char> x(n), y(n);
      cudaMemcpy(x.data(), buf[r]->p, n, cudaMemcpyDeviceToHost);
      cudaMemcpy(y.data(), expect.p, n, cudaMemcpyDeviceToHost);
      bytes_ok = bytes_ok && x == y;
    }
    std::printf("{\"D\": %d, \"failed\": %d, \"mode\": \"inplace\", \"state_bytes\": %lld, "
                "\"phases\": %zu, \"programs\": %d, \"stage_alloc\": %lld, \"ms\": %.3f, "
                "\"conserved\": %s, \"bytes_ok\": %s}\n",
                D, failed_rank, static_cast<long long>(src.total_bytes), sc.phases.size(), programs,
                static_cast<long long>(sc.stage_alloc), ms, conserved ? "true" : "false",
                bytes_ok ? "true" : "false");
    cudaFree(before);
    cudaFree(after);
    return conserved && bytes_ok ? 0 : 1;
  }

  // buffers: OLD (role 0), REPLICA (role 1, ring holder of the failed rank), NEW (role 2)
  std::map<std::pair<int, int>, std::unique_ptr<Buffer>> bufs;
  std::vector<void*> table(3 * D, nullptr);
  const int holder = ring.backed_up_by(failed_rank);
  for (int r : old_ranks) {
    auto b = std::make_unique<Buffer>(b200::shard_bytes(src, r));
    fill(src, r, b->p, 7);
    table[0 * D + r] = b->p;
    bufs[{0, r}] = std::move(b);
  }
  {
    auto b = std::make_unique<Buffer>(b200::shard_bytes(src, failed_rank));
    fill(src, failed_rank, b->p, 7);  // the holder's replica of the failed rank
    table[1 * D + holder] = b->p;
    bufs[{1, holder}] = std::move(b);
  }
  for (int r : new_ranks) {
    auto b = std::make_unique<Buffer>(b200::shard_bytes(dst, r));
    cuda(cudaMemset(b->p, 0xA5, b->n), "memset");
    table[2 * D + r] = b->p;
    bufs[{2, r}] = std::move(b);
  }

  // one copy program per surviving GPU (pull), all launched on this device
  std::vector<std::unique_ptr<device::CopyProgram>> progs;
  for (int r : new_ranks)
    progs.push_back(std::make_unique<device::CopyProgram>(
        b200::reshard_copies(plan, src, dst, failed, &ring, r, false), table, D, r));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (auto& p : progs) p->launch(nullptr);
  cudaEventRecord(b);
  cuda(cudaEventSynchronize(b), "copy");
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);

  // verification 1: checksum conservation (no source re-read needed)
  const std::int64_t n_blocks = (src.total_bytes + 65535) / 65536;
  std::uint64_t *before = nullptr, *after = nullptr;
  cuda(cudaMalloc(&before, 16 * n_blocks), "malloc");
  cuda(cudaMalloc(&after, 16 * n_blocks), "malloc");
  cudaMemset(before, 0, 16 * n_blocks);
  cudaMemset(after, 0, 16 * n_blocks);
  for (int r : old_ranks) add_blocks(src, r, table[0 * D + r], before, n_blocks);
  for (int r : new_ranks) add_blocks(dst, r, table[2 * D + r], after, n_blocks);
  std::vector<std::uint64_t> hb(2 * n_blocks), ha(2 * n_blocks);
  cudaMemcpy(hb.data(), before, 16 * n_blocks, cudaMemcpyDeviceToHost);
  cudaMemcpy(ha.data(), after, 16 * n_blocks, cudaMemcpyDeviceToHost);
  const bool conserved = hb == ha;

  // verification 2: regenerate each target shard and compare bytes
  bool bytes_ok = true;
  for (int r : new_ranks) {
    const std::int64_t n = b200::shard_bytes(dst, r);
    Buffer expect(n);
    fill(dst, r, expect.p, 7);
    std::vector<unsigned char> x(n), y(n);
    cudaMemcpy(x.data(), table[2 * D + r], n, cudaMemcpyDeviceToHost);
    cudaMemcpy(y.data(), expect.p, n, cudaMemcpyDeviceToHost);
    bytes_ok = bytes_ok && x == y;
  }
  std::printf("{\"D\": %d, \"failed\": %d, \"state_bytes\": %lld, \"entries\": %zu, "
              "\"bytes_moved\": %lld, \"plan_ms\": %.3f, \"copy_ms\": %.3f, "
              "\"conserved\": %s, \"bytes_ok\": %s}\n",
              D, failed_rank, static_cast<long long>(src.total_bytes), plan.entries.size(),
              static_cast<long long>(plan.total_bytes_moved),
              std::chrono::duration<double, std::milli>(t1 - t0).count(), ms,
              conserved ? "true" : "false", bytes_ok ? "true" : "false");
  cudaFree(before);
  cudaFree(after);
  return conserved && bytes_ok ? 0 : 1;
}
