// Multi-process DP recovery (include/elaskit/recovery.hpp): the rendezvous
// store, peer mappings, the reshard executor, checksum-conservation
// verification, prepared recoveries, the DP group with prepared NCCL
// communicators, and the staged in-place executor — host C++ over the C ABI
// (include/ew_api.h) plus the CUDA runtime for streams and events.
//
// Reference: Simulation::recover_elaswave (sim.cpp:597-722) prices comm
// repair (comm_edit_time, sim.cpp:436-450), dataflow and remap (remap_time,
// sim.cpp:452-483) and records MttrEvent (sim.hpp:31-45); here the same
// sequence runs on the GPUs and the record carries measured seconds.
#include "elaskit/recovery.hpp"

#include <arpa/inet.h>
#include <cuda_runtime.h>
#include <netdb.h>
#include <nvtx3/nvToolsExt.h>
#include <netinet/in.h>
#include <fcntl.h>
#include <netinet/tcp.h>
#include <sys/mman.h>
#include <sys/socket.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <atomic>
#include <cerrno>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <unordered_map>

#include "elaskit/dataflow.hpp"
#include "elaskit/device.hpp"

namespace elaskit::b200 {

using device::check;

namespace {

using Clock = std::chrono::steady_clock;

// NVTX range per MTTR phase (header-only NVTX3: free without a tool attached;
// ncu --nvtx / Nsight Systems show the recovery's phases on the timeline)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
double seconds(Clock::time_point a, Clock::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw device::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------- TCP store
//
// Frames: 'S' u32 klen key u64 vlen value -> u8 ack;  'G' u32 klen key ->
// u64 vlen value (the server answers once the key exists).

bool send_all(int fd, const void* p, std::size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n > 0) {
    const ssize_t k = ::send(fd, c, n, MSG_NOSIGNAL);
    if (k <= 0) return false;
    c += k;
    n -= static_cast<std::size_t>(k);
  }
  return true;
}

bool recv_all(int fd, void* p, std::size_t n) {
  char* c = static_cast<char*>(p);
  while (n > 0) {
    const ssize_t k = ::recv(fd, c, n, 0);
    if (k <= 0) return false;
    c += k;
    n -= static_cast<std::size_t>(k);
  }
  return true;
}

class TcpServer {
 public:
  explicit TcpServer(int port) {
    fd_ = ::socket(AF_INET, SOCK_STREAM, 0);
    if (fd_ < 0) throw std::runtime_error("tcp store: socket() failed");
    int one = 1;
    ::setsockopt(fd_, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
    sockaddr_in a{};
    a.sin_family = AF_INET;
    a.sin_addr.s_addr = htonl(INADDR_ANY);
    a.sin_port = htons(static_cast<uint16_t>(port));
    if (::bind(fd_, reinterpret_cast<sockaddr*>(&a), sizeof(a)) != 0 || ::listen(fd_, 256) != 0) {
      ::close(fd_);
      throw std::runtime_error("tcp store: cannot listen on port " + std::to_string(port));
    }
    accept_ = std::thread([this] { accept_loop(); });
  }
  ~TcpServer() {
    {
      // the host process leaving must not cut its peers' last reads short
      // (e.g. a final barrier): wait until every client has disconnected
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait_for(lk, std::chrono::seconds(60), [&] { return live_ == 0; });
    }
    stop_ = true;
    ::shutdown(fd_, SHUT_RDWR);
    ::close(fd_);
    accept_.join();
    {
      std::lock_guard<std::mutex> lk(mu_);
      for (int c : conns_) ::shutdown(c, SHUT_RDWR);
    }
    cv_.notify_all();
    for (std::thread& t : workers_) t.join();
    for (int c : conns_) ::close(c);  // closed only here: no fd number is reused meanwhile
  }

 private:
  void accept_loop() {
    while (!stop_) {
      const int c = ::accept(fd_, nullptr, nullptr);
      if (c < 0) {
        if (stop_) break;
        continue;
      }
      int one = 1;
      ::setsockopt(c, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
      std::lock_guard<std::mutex> lk(mu_);
      conns_.push_back(c);
      ++live_;
      workers_.emplace_back([this, c] {
        serve(c);
        {
          std::lock_guard<std::mutex> g(mu_);
          --live_;
        }
        cv_.notify_all();
      });
    }
  }
  void serve(int c) {
    for (;;) {
      char op = 0;
      uint32_t kl = 0;
      if (!recv_all(c, &op, 1) || !recv_all(c, &kl, 4)) break;
      std::string key(kl, '\0');
      if (!recv_all(c, key.data(), kl)) break;
      if (op == 'S') {
        uint64_t vl = 0;
        if (!recv_all(c, &vl, 8)) break;
        std::string v(vl, '\0');
        if (!recv_all(c, v.data(), vl)) break;
        {
          std::lock_guard<std::mutex> lk(mu_);
          data_[key] = std::move(v);
        }
        cv_.notify_all();
        const char ack = 1;
        if (!send_all(c, &ack, 1)) break;
      } else if (op == 'D') {
        {
          std::lock_guard<std::mutex> lk(mu_);
          data_.erase(key);
        }
        const char ack = 1;
        if (!send_all(c, &ack, 1)) break;
      } else if (op == 'G') {
        std::string v;
        bool gone = false;
        {
          std::unique_lock<std::mutex> lk(mu_);
          // a client that gave up (its get timed out) and closed the
          // connection must not keep this worker waiting for the key
          while (!cv_.wait_for(lk, std::chrono::milliseconds(200),
                               [&] { return stop_.load() || data_.count(key) > 0; })) {
            char b;
            const ssize_t k = ::recv(c, &b, 1, MSG_PEEK | MSG_DONTWAIT);
            if (k == 0 || (k < 0 && errno != EAGAIN && errno != EWOULDBLOCK)) {
              gone = true;
              break;
            }
          }
          if (stop_ || gone) break;
          v = data_[key];
        }
        const uint64_t vl = v.size();
        if (!send_all(c, &vl, 8) || !send_all(c, v.data(), vl)) break;
      } else {
        break;
      }
    }
  }

  int fd_ = -1;
  std::atomic<bool> stop_{false};
  std::thread accept_;
  std::vector<std::thread> workers_;
  std::vector<int> conns_;
  int live_ = 0;  // connected clients
  std::mutex mu_;
  std::condition_variable cv_;
  std::unordered_map<std::string, std::string> data_;
};

class TcpStore final : public Store {
 public:
  TcpStore(const std::string& host, int port, bool is_server, double timeout_s) {
    if (is_server) server_ = std::make_unique<TcpServer>(port);
    addrinfo hints{}, *res = nullptr;
    hints.ai_family = AF_INET;
    hints.ai_socktype = SOCK_STREAM;
    if (::getaddrinfo(host.c_str(), std::to_string(port).c_str(), &hints, &res) != 0 || !res)
      throw std::runtime_error("tcp store: cannot resolve " + host);
    const auto t0 = Clock::now();
    for (;;) {
      fd_ = ::socket(AF_INET, SOCK_STREAM, 0);
      if (fd_ >= 0 && ::connect(fd_, res->ai_addr, res->ai_addrlen) == 0) break;
      if (fd_ >= 0) ::close(fd_);
      fd_ = -1;
      if (seconds(t0, Clock::now()) > timeout_s) {
        ::freeaddrinfo(res);
        throw std::runtime_error("tcp store: cannot connect to " + host + ":" +
                                 std::to_string(port));
      }
      std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
    ::freeaddrinfo(res);
    int one = 1;
    ::setsockopt(fd_, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
    timeval tv{};
    tv.tv_sec = static_cast<long>(timeout_s);
    tv.tv_usec = static_cast<long>((timeout_s - static_cast<double>(tv.tv_sec)) * 1e6);
    ::setsockopt(fd_, SOL_SOCKET, SO_RCVTIMEO, &tv, sizeof(tv));
  }
  ~TcpStore() override {
    if (fd_ >= 0) ::close(fd_);  // own connection first: the server waits for all clients
    server_.reset();
  }
  void set(const std::string& key, const std::string& value) override {
    std::lock_guard<std::mutex> lk(mu_);
    usable();
    const char op = 'S';
    const uint32_t kl = static_cast<uint32_t>(key.size());
    const uint64_t vl = value.size();
    char ack = 0;
    if (!send_all(fd_, &op, 1) || !send_all(fd_, &kl, 4) || !send_all(fd_, key.data(), kl) ||
        !send_all(fd_, &vl, 8) || !send_all(fd_, value.data(), vl) || !recv_all(fd_, &ack, 1))
      fail("set(" + key + ") failed");
  }
  void erase(const std::string& key) override {
    std::lock_guard<std::mutex> lk(mu_);
    usable();
    const char op = 'D';
    const uint32_t kl = static_cast<uint32_t>(key.size());
    char ack = 0;
    if (!send_all(fd_, &op, 1) || !send_all(fd_, &kl, 4) || !send_all(fd_, key.data(), kl) ||
        !recv_all(fd_, &ack, 1))
      fail("erase(" + key + ") failed");
  }
  std::string get(const std::string& key) override {
    std::lock_guard<std::mutex> lk(mu_);
    usable();
    const char op = 'G';
    const uint32_t kl = static_cast<uint32_t>(key.size());
    uint64_t vl = 0;
    if (!send_all(fd_, &op, 1) || !send_all(fd_, &kl, 4) || !send_all(fd_, key.data(), kl) ||
        !recv_all(fd_, &vl, 8))
      fail("get(" + key + ") failed or timed out");
    std::string v(vl, '\0');
    if (!recv_all(fd_, v.data(), vl)) fail("get(" + key + ") cut");
    return v;
  }

 private:
  // a failed or timed-out exchange leaves the stream mid-frame (the server may
  // still answer a timed-out get): the connection is unusable from then on
  void usable() const {
    if (broken_) throw std::runtime_error("tcp store: connection broken by an earlier failure");
  }
  [[noreturn]] void fail(const std::string& what) {
    broken_ = true;
    throw std::runtime_error("tcp store: " + what);
  }

  std::unique_ptr<TcpServer> server_;
  int fd_ = -1;
  bool broken_ = false;
  std::mutex mu_;
};

class CallbackStore final : public Store {
 public:
  CallbackStore(std::function<void(const std::string&, const std::string&)> s,
                std::function<std::string(const std::string&)> g,
                std::function<void(const std::string&)> e)
      : set_(std::move(s)), get_(std::move(g)), erase_(std::move(e)) {}
  void set(const std::string& k, const std::string& v) override { set_(k, v); }
  std::string get(const std::string& k) override { return get_(k); }
  void erase(const std::string& k) override {
    if (erase_) erase_(k);
  }

 private:
  std::function<void(const std::string&, const std::string&)> set_;
  std::function<std::string(const std::string&)> get_;
  std::function<void(const std::string&)> erase_;
};

// ------------------------------------------------------------ small helpers

template <typename T>
T* dalloc(std::int64_t count) {
  void* p = nullptr;
  check(ew_alloc(std::max<std::int64_t>(32, count * static_cast<std::int64_t>(sizeof(T))), &p));
  return static_cast<T*>(p);
}

void dfree(void* p) {
  if (p != nullptr) ew_free(p);
}

// owning device allocation (freed on every exit path)
template <typename T>
struct DevArray {
  T* p;
  explicit DevArray(std::int64_t count) : p(dalloc<T>(count)) {}
  ~DevArray() { dfree(p); }
  DevArray(const DevArray&) = delete;
  DevArray& operator=(const DevArray&) = delete;
};

std::vector<ew_segment> to_ew(const std::vector<Segment>& segs) {
  std::vector<ew_segment> out;
  out.reserve(segs.size());
  for (const Segment& s : segs) out.push_back({s.global_lo, s.length, s.local_off});
  return out;
}

ew_shardmap* make_map(const std::vector<Segment>& segs, std::int64_t block) {
  const std::vector<ew_segment> e = to_ew(segs);
  ew_shardmap* m = nullptr;
  check(ew_shardmap_create(e.data(), static_cast<std::int64_t>(e.size()), block, &m));
  return m;
}

// blocks[2b..2b+1] += checksum rows of member r's packed shard (rows given:
// the per-step snapshot rows; else re-read from buf)
void add_blocks(const PartitionLayout& layout, int r, const void* buf, const std::uint64_t* rows,
                std::uint64_t* blocks, std::int64_t n_blocks, std::int64_t block,
                ew_stream_t s) {
  ew_shardmap* m = make_map(shard_segments(layout, r), block);
  const std::int64_t n_rows = ew_shardmap_num_rows(m);
  std::uint64_t* tmp = nullptr;
  try {
    if (rows == nullptr && n_rows > 0) {
      tmp = dalloc<std::uint64_t>(2 * n_rows);
      check(ew_checksum(m, buf, tmp, s));
      rows = tmp;
    }
    if (n_rows > 0) check(ew_rows_to_blocks(m, rows, blocks, n_blocks, s));
    check(ew_stream_sync(s));
  } catch (...) {
    dfree(tmp);
    ew_shardmap_free(m);
    throw;
  }
  dfree(tmp);
  ew_shardmap_free(m);
}

std::vector<int> without(const std::vector<int>& v, const std::set<int>& drop) {
  std::vector<int> out;
  for (int x : v)
    if (!drop.count(x)) out.push_back(x);
  return out;
}

int index_of(const std::vector<int>& v, int x) {
  const auto it = std::find(v.begin(), v.end(), x);
  return it == v.end() ? -1 : static_cast<int>(it - v.begin());
}

// PeerBuffers keys beyond the BufRole values
constexpr int kLanded = 10, kOldBlocks = 11, kReplicaBlocks = 12, kFlags = 13;
constexpr int kGrad = 20, kRows = 21, kSnap = 22;
constexpr int kOut = 30, kAcc = 31, kUnit0 = 100;  // units: kUnit0 + k
constexpr int kParams = 40;

// Slice [lo, hi) (even) of n_words owned by survivor i of k.
std::pair<std::int64_t, std::int64_t> slice_of(std::int64_t n_words, int i, int k) {
  const std::int64_t pairs = n_words / 2;
  return {2 * (pairs * i / k), 2 * (pairs * (i + 1) / k)};
}

// Stream-ordered barrier among `members` over flag arrays registered under
// key kFlags in `peers`, using region `region` (of n_regions * stride u64).
ew_peer_barrier* make_barrier(const PeerBuffers& peers, const std::vector<int>& members, int me,
                              std::int64_t region_off) {
  std::vector<unsigned long long*> ptrs;
  for (int m : members) {
    auto* base = static_cast<unsigned long long*>(peers.get(kFlags, m));
    if (base == nullptr) throw std::runtime_error("barrier flags of member " + std::to_string(m) +
                                                  " are not mapped");
    ptrs.push_back(base + region_off);
  }
  ew_peer_barrier* b = nullptr;
  check(ew_peer_barrier_create(static_cast<int>(members.size()), index_of(members, me),
                               ptrs.data(), &b));
  return b;
}

}  // namespace

std::unique_ptr<Store> tcp_store(const std::string& host, int port, bool is_server,
                                 double timeout_s) {
  return std::make_unique<TcpStore>(host, port, is_server, timeout_s);
}

std::unique_ptr<Store> callback_store(
    std::function<void(const std::string&, const std::string&)> set,
    std::function<std::string(const std::string&)> get,
    std::function<void(const std::string&)> erase) {
  return std::make_unique<CallbackStore>(std::move(set), std::move(get), std::move(erase));
}

// ------------------------------------------------------------------ Channel

Channel::Channel(Store& store, std::string name, std::vector<int> members, int me)
    : store_(store), name_(std::move(name)), members_(std::move(members)), me_(me) {
  std::sort(members_.begin(), members_.end());
  index_ = index_of(members_, me);
  if (index_ < 0)
    throw std::invalid_argument("channel " + name_ + ": rank " + std::to_string(me) +
                                " is not a member");
}

std::vector<std::string> Channel::allgather(const std::string& mine) {
  const std::uint64_t round = seq_++;
  const std::string base = name_ + "/" + std::to_string(round) + "/";
  store_.set(base + std::to_string(me_), mine);
  std::vector<std::string> out;
  out.reserve(members_.size());
  for (int m : members_) out.push_back(m == me_ ? mine : store_.get(base + std::to_string(m)));
  // every member has set its key of this round, so it finished reading the
  // previous one: that round's key of ours can go
  if (round > 0) store_.erase(name_ + "/" + std::to_string(round - 1) + "/" + std::to_string(me_));
  return out;
}

std::int64_t Channel::sum(std::int64_t mine) {
  std::int64_t total = 0;
  for (const std::string& s : allgather(std::to_string(mine))) total += std::stoll(s);
  return total;
}

// -------------------------------------------------------------- PeerBuffers

PeerBuffers::~PeerBuffers() { close(); }

void PeerBuffers::exchange(Channel& ch, const std::map<int, void*>& mine,
                           const std::function<bool(int, int)>& want) {
  // blob: n x {int32 key, 64-byte IPC handle, int64 offset}
  std::string blob;
  for (const auto& [key, ptr] : mine) {
    if (ptr == nullptr) continue;
    char rec[4 + 64 + 8];
    std::int64_t off = 0;
    const std::int32_t k = key;
    check(ew_ipc_get_handle(ptr, rec + 4, &off));
    std::memcpy(rec, &k, 4);
    std::memcpy(rec + 68, &off, 8);
    blob.append(rec, sizeof(rec));
    table_[{key, ch.me()}] = ptr;
  }
  const std::vector<std::string> all = ch.allgather(blob);
  for (std::size_t i = 0; i < all.size(); ++i) {
    const int m = ch.members()[i];
    if (m == ch.me()) continue;
    const std::string& b = all[i];
    for (std::size_t p = 0; p + 76 <= b.size(); p += 76) {
      std::int32_t key = 0;
      std::int64_t off = 0;
      std::memcpy(&key, b.data() + p, 4);
      std::memcpy(&off, b.data() + p + 68, 8);
      if (table_.count({key, m}) || (want && !want(key, m))) continue;
      void* q = nullptr;
      check(ew_ipc_open(b.data() + p + 4, off, &q));
      opened_.push_back(q);
      table_[{key, m}] = q;
    }
  }
}

void* PeerBuffers::get(int key, int member) const {
  const auto it = table_.find({key, member});
  return it == table_.end() ? nullptr : it->second;
}

void PeerBuffers::close() {
  for (void* p : opened_) ew_ipc_close(p);
  opened_.clear();
  table_.clear();
}

// -------------------------------------------------------------- ReshardPlan

ReshardPlan ReshardPlan::build(const std::vector<std::int64_t>& layer_bytes,
                               std::vector<int> old_members, std::vector<int> new_members) {
  const auto t0 = Clock::now();
  std::sort(old_members.begin(), old_members.end());
  std::sort(new_members.begin(), new_members.end());
  ReshardPlan rp;
  rp.layer_bytes = layer_bytes;
  rp.old_members = old_members;
  rp.new_members = new_members;
  for (int m : old_members)
    if (!std::binary_search(new_members.begin(), new_members.end(), m)) rp.failed.insert(m);
  ZeroLayout z;
  z.kind = ZeroKind::Interleaved;
  z.dp_degree = static_cast<int>(old_members.size());
  z.layer_bytes = layer_bytes;
  rp.src = interleaved_layout(z, old_members);
  rp.dst = interleaved_layout(z, new_members);
  rp.ring.members = old_members;
  if (!rp.failed.empty()) {
    const IntegrityReport rep = integrity_check(rp.ring, rp.src, rp.failed);
    if (!rep.recoverable) {
      std::string who;
      for (const auto& [r, ivs] : rep.missing) who += (who.empty() ? "" : ",") + std::to_string(r);
      throw CoverageMismatch("members {" + who + "} lost together with their ring holders");
    }
  }
  rp.plan = overlap_matrix(rp.src, rp.dst, rp.failed, &rp.ring);
  rp.plan_seconds = seconds(t0, Clock::now());
  return rp;
}

ReshardPlan ReshardPlan::from_layouts(PartitionLayout src, PartitionLayout dst,
                                      std::set<int> failed, std::vector<int> ring_members) {
  const auto t0 = Clock::now();
  ReshardPlan rp;
  for (const auto& [r, ivs] : src.ranges) rp.old_members.push_back(r);
  for (const auto& [r, ivs] : dst.ranges) rp.new_members.push_back(r);
  rp.failed = std::move(failed);
  rp.src = std::move(src);
  rp.dst = std::move(dst);
  rp.ring.members = std::move(ring_members);
  const SnapshotRing* ring = rp.ring.members.empty() ? nullptr : &rp.ring;
  if (!rp.failed.empty()) {
    if (ring == nullptr) throw std::invalid_argument("failed members need a snapshot ring");
    if (!integrity_check(rp.ring, rp.src, rp.failed).recoverable)
      throw CoverageMismatch("failed members lost together with their ring holders");
  }
  rp.plan = overlap_matrix(rp.src, rp.dst, rp.failed, ring);
  rp.plan_seconds = seconds(t0, Clock::now());
  return rp;
}

int ReshardPlan::replica_of(int holder) const {
  if (ring.members.size() < 2 ||
      std::find(ring.members.begin(), ring.members.end(), holder) == ring.members.end())
    return -1;
  return ring.backs_up(holder);
}

// ---------------------------------------------------------- ReshardExecutor

ReshardExecutor::ReshardExecutor(const ReshardPlan& rp, int me, bool push,
                                 std::int64_t block_bytes, bool local_replica)
    : rp_(rp), me_(me), push_(push), block_bytes_(block_bytes) {
  copies_ = reshard_copies(rp_.plan, rp_.src, rp_.dst, rp_.failed,
                           rp_.ring.members.empty() ? nullptr : &rp_.ring, me_, push_);
  if (local_replica) {
    if (push_) throw std::invalid_argument("replica-aware sourcing is a pull-program option");
    copies_ = prefer_local_replica(copies_, rp_.ring, rp_.failed, me_);
  }
}

ReshardExecutor::~ReshardExecutor() {
  ew_copy_program_free(prog_);
  ew_shardmap_free(new_map_);
}

std::set<std::pair<int, int>> ReshardExecutor::peers_needed() const {
  std::set<std::pair<int, int>> out;
  for (const CopyDesc& c : copies_) {
    if (c.src_rank != me_) out.insert({static_cast<int>(c.src_role), c.src_rank});
    if (c.dst_rank != me_) out.insert({static_cast<int>(c.dst_role), c.dst_rank});
  }
  return out;
}

std::int64_t ReshardExecutor::new_bytes() const {
  return rp_.dst.ranges.count(me_) ? shard_bytes(rp_.dst, me_) : 0;
}

void ReshardExecutor::bind(const PeerBuffers& peers, bool verify) {
  if (verify && push_)
    throw std::invalid_argument("verification on arrival needs pull mode (every byte landing in "
                                "NEW is then issued by its own GPU)");
  int top = me_;
  for (int m : rp_.old_members) top = std::max(top, m);
  for (int m : rp_.new_members) top = std::max(top, m);
  const int tr = top + 1;
  std::vector<void*> table(3 * static_cast<std::size_t>(tr), nullptr);
  std::vector<ew_copy_desc> d;
  d.reserve(copies_.size());
  for (const CopyDesc& c : copies_) {
    for (const auto& [role, rank] : {std::pair<int, int>{static_cast<int>(c.src_role), c.src_rank},
                                     std::pair<int, int>{static_cast<int>(c.dst_role), c.dst_rank}}) {
      void* p = peers.get(role, rank);
      if (p == nullptr)
        throw std::runtime_error("peer buffer (role " + std::to_string(role) + ", member " +
                                 std::to_string(rank) + ") is not mapped");
      table[static_cast<std::size_t>(role) * tr + rank] = p;
    }
    d.push_back({static_cast<std::int32_t>(c.src_role), c.src_rank,
                 static_cast<std::int32_t>(c.dst_role), c.dst_rank, c.src_off, c.dst_off,
                 c.bytes});
  }
  ew_copy_program_free(prog_);
  prog_ = nullptr;
  if (verify && rp_.dst.ranges.count(me_)) {
    if (new_map_ == nullptr) new_map_ = make_map(shard_segments(rp_.dst, me_), block_bytes_);
    check(ew_copy_program_create_verified(d.data(), static_cast<std::int64_t>(d.size()),
                                          table.data(), tr, me_, new_map_, &prog_));
  } else {
    check(ew_copy_program_create(d.data(), static_cast<std::int64_t>(d.size()), table.data(), tr,
                                 me_, &prog_));
  }
}

void ReshardExecutor::launch(ew_stream_t stream, std::uint64_t* block_sums,
                             const int* abort_flag, int n_ctas, int remote_ctas) const {
  if (prog_ == nullptr) throw std::logic_error("ReshardExecutor::launch before bind");
  check(ew_copy_program_launch_guarded(prog_, n_ctas, remote_ctas,
                                       new_map_ != nullptr ? block_sums : nullptr, abort_flag,
                                       stream));
}

// ------------------------------------------------------------ BlockVerifier

BlockVerifier::~BlockVerifier() { ew_block_verifier_free(v_); }

void BlockVerifier::set(const std::vector<const std::uint64_t*>& plus,
                        const std::vector<const std::uint64_t*>& minus, std::int64_t n_words,
                        std::int64_t lo, std::int64_t hi) {
  if (hi > n_words) throw std::invalid_argument("BlockVerifier: slice beyond the arrays");
  ew_block_verifier_free(v_);
  v_ = nullptr;
  check(ew_block_verifier_create(plus.data(), static_cast<int>(plus.size()), minus.data(),
                                 static_cast<int>(minus.size()), lo, hi, &v_));
}

void BlockVerifier::run(ew_stream_t stream, std::uint32_t* bad_dev) const {
  check(ew_block_verifier_run(v_, bad_dev, stream));
}

// ------------------------------------------------------------ ring replicas

namespace {
int ring_successor(const std::vector<int>& members, int me) {
  const int i = index_of(members, me);
  return members[static_cast<std::size_t>((i + 1) % static_cast<int>(members.size()))];
}
}  // namespace

ReplayReplica::ReplayReplica(Channel& ch, const float* my_grad, const std::uint64_t* my_rows,
                             AdamShard replica, std::int64_t block_bytes)
    : rep_(replica), block_bytes_(block_bytes) {
  if (ch.members().size() < 2) throw std::invalid_argument("a ring needs two members");
  owner_ = ring_successor(ch.members(), ch.me());
  n_rows_ = (rep_.image_bytes + block_bytes - 1) / block_bytes;
  rows_ = dalloc<std::uint64_t>(2 * std::max<std::int64_t>(1, n_rows_));
  const ew_segment seg{0, rep_.image_bytes, 0};
  check(ew_shardmap_create(&seg, 1, block_bytes, &map_));
  peers_.exchange(ch, {{kGrad, const_cast<float*>(my_grad)},
                       {kRows, const_cast<std::uint64_t*>(my_rows)}},
                  [&](int, int member) { return member == owner_; });
  owner_grad_ = static_cast<const float*>(peers_.get(kGrad, owner_));
  owner_rows_ = static_cast<const std::uint64_t*>(peers_.get(kRows, owner_));
  if (owner_grad_ == nullptr || owner_rows_ == nullptr)
    throw std::runtime_error("the owner's gradient shard / rows are not mapped");
}

ReplayReplica::~ReplayReplica() {
  peers_.close();
  ew_shardmap_free(map_);
  dfree(rows_);
}

void ReplayReplica::replay(const ew_adam_hyper& hyper, std::int64_t step, ew_stream_t stream) {
  check(ew_adam_step_rows(owner_grad_, rep_.master, rep_.exp_avg, rep_.exp_avg_sq,
                          rep_.param_bf16, rep_.n, &hyper, step, rep_.image, rep_.image_bytes,
                          block_bytes_, rows_, stream));
}

void ReplayReplica::verify(std::uint32_t* bad_dev, ew_stream_t stream) const {
  // the owner's rows are read where they are (its HBM, over NVLink): 2.9 MB at 7B
  check(ew_rows_diff(rows_, owner_rows_, n_rows_, bad_dev, stream));
}

void ReplayReplica::verify_by_reread(std::uint32_t* bad_dev, ew_stream_t stream) const {
  check(ew_verify(map_, rep_.image, owner_rows_, bad_dev, nullptr, 0, stream));
}

RingReplica::RingReplica(Channel& ch, const PartitionLayout& layout, const void* my_snap,
                         const std::uint64_t* my_rows, void* replica, std::int64_t block_bytes)
    : replica_(replica) {
  if (ch.members().size() < 2) throw std::invalid_argument("a ring needs two members");
  owner_ = ring_successor(ch.members(), ch.me());
  map_ = make_map(shard_segments(layout, owner_), block_bytes);
  peers_.exchange(ch, {{kSnap, const_cast<void*>(my_snap)},
                       {kRows, const_cast<std::uint64_t*>(my_rows)}},
                  [&](int, int member) { return member == owner_; });
  const void* src = peers_.get(kSnap, owner_);
  owner_rows_ = static_cast<const std::uint64_t*>(peers_.get(kRows, owner_));
  if (src == nullptr || owner_rows_ == nullptr)
    throw std::runtime_error("the owner's snapshot / rows are not mapped");
  const std::int64_t bytes = ew_shardmap_bytes(map_);
  const int remote = 1;
  check(ew_copy_program_create_raw(&src, &replica_, &bytes, &remote, 1, &copy_));
}

RingReplica::~RingReplica() {
  ew_copy_program_free(copy_);
  peers_.close();
  ew_shardmap_free(map_);
}

void RingReplica::refresh(std::uint32_t* bad_dev, ew_stream_t stream) const {
  check(ew_copy_program_launch(copy_, 0, 0, stream));
  check(ew_verify(map_, replica_, owner_rows_, bad_dev, nullptr, 0, stream));
}

// ------------------------------------------------------- layer migration

LayerMigration::LayerMigration(Channel& ch, int source, int target, void* params,
                               std::int64_t param_bytes, std::int64_t* acc, std::int64_t n,
                               int transfer_ctas, double barrier_timeout_s)
    : me_(ch.me()), source_(source), target_(target), transfer_ctas_(transfer_ctas),
      timeout_s_(barrier_timeout_s), acc_(acc), n_(n) {
  if (ch.members().size() != 2 || index_of(ch.members(), source) < 0 ||
      index_of(ch.members(), target) < 0 || source == target)
    throw std::invalid_argument("a layer migration's channel is exactly {source, target}");
  try {
    flags_ = dalloc<unsigned long long>(2);
    check(ew_memset_async(flags_, 0, 16, nullptr));
    check(ew_device_sync());
    std::map<int, void*> mine = {{kFlags, flags_}};
    if (me_ == source) {
      mine[kParams] = params;
      mine[kAcc] = acc;
    }
    peers_.exchange(ch, mine);
    barrier_ = make_barrier(peers_, ch.members(), me_, 0);
    if (me_ == target) {
      const void* src = peers_.get(kParams, source);
      source_acc_ = static_cast<const std::int64_t*>(peers_.get(kAcc, source));
      if (src == nullptr || source_acc_ == nullptr)
        throw std::runtime_error("the source's parameters / accumulator are not mapped");
      const int remote = 1;
      check(ew_copy_program_create_raw(&src, &params, &param_bytes, &remote, 1, &pull_));
      payback_ = dalloc<std::int64_t>(std::max<std::int64_t>(4, n));
      const void* asrc = source_acc_;
      void* adst = payback_;
      const std::int64_t abytes = 8 * n;
      check(ew_copy_program_create_raw(&asrc, &adst, &abytes, &remote, 1, &payback_pull_));
    }
  } catch (...) {
    if (barrier_) ew_peer_barrier_free(barrier_);
    ew_copy_program_free(pull_);
    ew_copy_program_free(payback_pull_);
    peers_.close();
    dfree(payback_);
    dfree(flags_);
    throw;
  }
  ch.barrier();
}

LayerMigration::~LayerMigration() {
  if (barrier_) ew_peer_barrier_free(barrier_);
  ew_copy_program_free(pull_);
  ew_copy_program_free(payback_pull_);
  peers_.close();
  dfree(payback_);
  dfree(flags_);
}

void LayerMigration::pull_params(ew_stream_t stream) {
  if (me_ != target_) throw std::logic_error("pull_params runs on the target");
  // stream priority only orders pending CTAs: a few dozen CTAs keep NVLink
  // busy without holding every SM away from the compute stream
  check(ew_copy_program_launch(pull_, transfer_ctas_, 0, stream));
}

void LayerMigration::shadow_done(ew_stream_t stream) {
  if (me_ != source_) throw std::logic_error("shadow_done runs on the source");
  check(ew_peer_barrier_wait(barrier_, timeout_s_, stream));
}

void LayerMigration::prefetch_payback(ew_stream_t stream) {
  if (me_ != target_) throw std::logic_error("prefetch_payback runs on the target");
  check(ew_peer_barrier_wait(barrier_, timeout_s_, stream));
  const int* veto = nullptr;
  check(ew_peer_barrier_error_flag(barrier_, &veto));
  check(ew_copy_program_launch_guarded(payback_pull_, transfer_ctas_, 0, nullptr, veto, stream));
}

void LayerMigration::payback(ew_stream_t stream) {
  if (me_ != target_) throw std::logic_error("payback runs on the target");
  check(ew_payback_accumulate(acc_, source_acc_, n_, stream));
}

void LayerMigration::run_target(const std::vector<const float*>& units,
                                const std::vector<double>& weights, std::int64_t n,
                                int frac_bits, int k, ew_stream_t compute, ew_stream_t transfer) {
  NvtxRange range("ew.migration.target");
  const int M = static_cast<int>(units.size());
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(compute);
  cudaStream_t ts = reinterpret_cast<cudaStream_t>(transfer);
  cudaEvent_t arrived = nullptr, ready = nullptr;
  cuda_check(cudaEventCreateWithFlags(&arrived, cudaEventDisableTiming), "cudaEventCreate");
  pull_params(transfer);
  cuda_check(cudaEventRecord(arrived, ts), "cudaEventRecord");
  if (k > 0) {  // k == 0 is the blocking move: nothing to pay back
    cuda_check(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "cudaEventCreate");
    prefetch_payback(transfer);
    cuda_check(cudaEventRecord(ready, ts), "cudaEventRecord");
  }
  for (int mb = std::min(k, M); mb < M; ++mb) {
    if (mb == k) cuda_check(cudaStreamWaitEvent(cs, arrived, 0), "wait");
    const bool last = mb == M - 1 && ready != nullptr;
    if (last) cuda_check(cudaStreamWaitEvent(cs, ready, 0), "wait");
    const float* u = units[static_cast<std::size_t>(mb)];
    const double w = weights[static_cast<std::size_t>(mb)];
    check(ew_weighted_fold_addend(&u, &w, 1, n, frac_bits, acc_, 1, last ? payback_ : nullptr,
                                  compute));
  }
  if (k >= M) {
    cuda_check(cudaStreamWaitEvent(cs, arrived, 0), "wait");
    if (ready != nullptr) {
      cuda_check(cudaStreamWaitEvent(cs, ready, 0), "wait");
      check(ew_payback_accumulate(acc_, payback_, n_, compute));
    }
  }
  cudaEventDestroy(arrived);
  if (ready != nullptr) cudaEventDestroy(ready);
}

void LayerMigration::run_shadow(const std::vector<const float*>& units,
                                const std::vector<double>& weights, std::int64_t n,
                                int frac_bits, int k, ew_stream_t compute) {
  if (k <= 0) return;  // blocking move: the target computes every micro-batch
  NvtxRange range("ew.migration.shadow");
  for (int mb = 0; mb < std::min(k, static_cast<int>(units.size())); ++mb) {
    const float* u = units[static_cast<std::size_t>(mb)];
    const double w = weights[static_cast<std::size_t>(mb)];
    check(ew_weighted_fold_addend(&u, &w, 1, n, frac_bits, acc_, 1, nullptr, compute));
  }
  shadow_done(compute);
}

bool LayerMigration::timed_out() const {
  int t = 0;
  check(ew_peer_barrier_timed_out(barrier_, &t));
  return t != 0;
}

// ------------------------------------------------------------ host images

namespace {
std::string shm_name(const std::string& tag, int member) {
  return "/ew_" + tag + "_" + std::to_string(member);
}
}  // namespace

HostImages::HostImages(Channel& ch, const PartitionLayout& layout, const std::string& tag,
                       const std::vector<int>& readable, bool map_for_device)
    : me_(ch.me()), tag_(tag), map_for_device_(map_for_device) {
  for (int m : ch.members()) {
    bytes_[m] = layout.ranges.count(m) ? shard_bytes(layout, m) : 0;
    slot_[m] = (std::max<std::int64_t>(1, bytes_[m]) + kPage - 1) / kPage * kPage;
  }
  std::string failure;
  try {
    map_member(me_, true);
  } catch (const std::exception& e) {
    failure = e.what();
  }
  ch.barrier();  // every segment exists before anyone opens a peer's
  if (failure.empty()) {
    try {
      const std::vector<int> want = readable.empty() ? ch.members() : readable;
      for (int m : want)
        if (m != me_ && !segs_.count(m)) map_member(m, false);
    } catch (const std::exception& e) {
      failure = e.what();
    }
  }
  // a failure surfaces only after the closing barrier: no rank is left waiting
  const std::int64_t failed = ch.sum(failure.empty() ? 0 : 1);
  if (failed != 0) {
    release();
    throw std::runtime_error("host images could not be mapped" +
                             (failure.empty() ? std::string(" on a peer") : ": " + failure));
  }
  next_epoch_ = committed_epoch(me_) + 1;
}

void HostImages::map_member(int member, bool create) {
  Segment seg;
  seg.size = kPage + 2 * slot_.at(member);
  const std::string name = shm_name(tag_, member);
  const int fd = ::shm_open(name.c_str(), create ? (O_CREAT | O_EXCL | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) throw std::runtime_error("shm_open(" + name + ") failed");
  if (create && ::ftruncate(fd, seg.size) != 0) {
    ::close(fd);
    ::shm_unlink(name.c_str());
    throw std::runtime_error("ftruncate(" + name + ") failed (is /dev/shm large enough?)");
  }
  void* p = ::mmap(nullptr, static_cast<std::size_t>(seg.size), PROT_READ | PROT_WRITE, MAP_SHARED,
                   fd, 0);
  ::close(fd);
  if (p == MAP_FAILED) {
    if (create) ::shm_unlink(name.c_str());
    throw std::runtime_error("mmap(" + name + ") failed");
  }
  seg.addr = static_cast<std::uint8_t*>(p);
  if (create) *reinterpret_cast<volatile std::int64_t*>(seg.addr) = -1;
  segs_[member] = seg;  // registered below; released by release() on failure
  Segment& s = segs_[member];
  if (!map_for_device_) {
    s.dev = s.addr;
    return;
  }
  void* d = nullptr;
  if (ew_host_register(s.addr, s.size, &d) == EW_OK) {
    s.dev = static_cast<std::uint8_t*>(d);
    s.pieces.push_back(s.addr);
    return;
  }
  // 1 GiB registrations: need the identity mapping of registered host memory
  // (device address == host address) to stay one contiguous device range
  constexpr std::int64_t kChunk = std::int64_t{1} << 30;
  for (std::int64_t off = 0; off < s.size; off += kChunk) {
    void* piece = s.addr + off;
    check(ew_host_register(piece, std::min(kChunk, s.size - off), &d));
    s.pieces.push_back(piece);
    if (d != piece) throw std::runtime_error("registered host memory is not identity-mapped");
  }
  s.dev = s.addr;
}

void HostImages::release() {
  for (auto& [m, s] : segs_) {
    for (void* p : s.pieces) ew_host_unregister(p);
    s.pieces.clear();
    if (s.addr != nullptr) ::munmap(s.addr, static_cast<std::size_t>(s.size));
    s.addr = nullptr;
    if (m == me_) ::shm_unlink(shm_name(tag_, m).c_str());
  }
  segs_.clear();
}

HostImages::~HostImages() { release(); }

std::int64_t HostImages::committed_epoch(int member) const {
  return *reinterpret_cast<const volatile std::int64_t*>(segs_.at(member).addr);
}

std::uint8_t* HostImages::host_ptr(int member, std::int64_t epoch) const {
  const std::int64_t e = epoch < 0 ? committed_epoch(member) : epoch;
  if (e < 0) throw std::runtime_error("member " + std::to_string(member) +
                                      " has not committed an image yet");
  return segs_.at(member).addr + kPage + (e % 2) * slot_.at(member);
}

void* HostImages::device_ptr(int member) const {
  const std::int64_t e = committed_epoch(member);
  if (e < 0) throw std::runtime_error("member " + std::to_string(member) +
                                      " has not committed an image yet");
  return segs_.at(member).dev + kPage + (e % 2) * slot_.at(member);
}

std::int64_t HostImages::publish(const void* live, ew_stream_t stream, std::int64_t epoch) {
  if (epoch < 0) epoch = next_epoch_;
  next_epoch_ = epoch + 1;
  const Segment& s = segs_.at(me_);
  std::uint8_t* base = s.addr + kPage + (epoch % 2) * slot_.at(me_);
  const std::int64_t n = bytes_.at(me_);
  // one copy per registration piece the slot crosses
  std::vector<std::uint8_t*> cuts = {base};
  for (void* p : s.pieces) {
    auto* q = static_cast<std::uint8_t*>(p);
    if (q > base && q < base + n) cuts.push_back(q);
  }
  std::sort(cuts.begin(), cuts.end());
  cuts.push_back(base + n);
  for (std::size_t k = 0; k + 1 < cuts.size(); ++k)
    if (cuts[k + 1] > cuts[k])
      check(ew_memcpy_async(cuts[k], static_cast<const std::uint8_t*>(live) + (cuts[k] - base),
                            cuts[k + 1] - cuts[k], stream));
  // the commit word, after the image's last byte in stream order
  check(ew_write_u64_async(s.dev, static_cast<std::uint64_t>(epoch), stream));
  return epoch;
}

void HostImages::commit_host(std::int64_t epoch) {
  std::atomic_thread_fence(std::memory_order_seq_cst);
  *reinterpret_cast<volatile std::int64_t*>(segs_.at(me_).addr) = epoch;
  next_epoch_ = epoch + 1;
}

// ------------------------------------------------- (d) over peer memory

PeerReduce::PeerReduce(Channel& ch, const std::vector<const float*>& units,
                       const std::vector<double>& weights, float* out, std::int64_t n,
                       double barrier_timeout_s)
    : ch_(ch), n_(n), units_(units), weights_(weights), timeout_s_(barrier_timeout_s) {
  if (units.size() != weights.size()) throw std::invalid_argument("one weight per unit");
  std::map<int, void*> mine = {{kOut, out}};
  for (std::size_t k = 0; k < units.size(); ++k)
    mine[kUnit0 + static_cast<int>(k)] = const_cast<float*>(units[k]);
  // the weights travel with the handles: n, count, then the doubles
  std::string extra(sizeof(std::int64_t) * 2 + 8 * weights.size(), '\0');
  const std::int64_t hdr[2] = {n, static_cast<std::int64_t>(units.size())};
  std::memcpy(extra.data(), hdr, sizeof(hdr));
  if (!weights.empty()) std::memcpy(extra.data() + sizeof(hdr), weights.data(), 8 * weights.size());
  connect(ch, mine, extra);
}

PeerReduce::PeerReduce(Channel& ch, const std::int64_t* acc, float* out, std::int64_t n,
                       double barrier_timeout_s)
    : ch_(ch), n_(n), timeout_s_(barrier_timeout_s) {
  std::string extra(sizeof(std::int64_t) * 2, '\0');
  const std::int64_t hdr[2] = {n, -1};
  std::memcpy(extra.data(), hdr, sizeof(hdr));
  connect(ch, {{kOut, out}, {kAcc, const_cast<std::int64_t*>(acc)}}, extra);
}

void PeerReduce::connect(Channel& ch, std::map<int, void*> mine, const std::string& extra) {
  const int world = static_cast<int>(ch.members().size());
  try {
    flags_ = dalloc<unsigned long long>(std::max(2, world));
    dmax_ = dalloc<double>(1);
    check(ew_memset_async(flags_, 0, 8 * std::max(2, world), nullptr));
    check(ew_device_sync());
    mine[kFlags] = flags_;
    peers_.exchange(ch, mine);
    const std::vector<std::string> meta = ch.allgather(extra);
    std::vector<const float*> unit_ptrs;
    std::vector<double> unit_w;
    std::vector<const std::int64_t*> acc_ptrs;
    std::vector<float*> out_ptrs;
    for (std::size_t i = 0; i < meta.size(); ++i) {
      const int m = ch.members()[i];
      std::int64_t hdr[2];
      std::memcpy(hdr, meta[i].data(), sizeof(hdr));
      if (hdr[0] != n_)
        throw DimensionMismatch("ranks disagree on the gradient length");
      out_ptrs.push_back(static_cast<float*>(peers_.get(kOut, m)));
      if (hdr[1] < 0) {
        acc_ptrs.push_back(static_cast<const std::int64_t*>(peers_.get(kAcc, m)));
        continue;
      }
      for (std::int64_t k = 0; k < hdr[1]; ++k) {
        unit_ptrs.push_back(static_cast<const float*>(peers_.get(kUnit0 + static_cast<int>(k), m)));
        double w = 0.0;
        std::memcpy(&w, meta[i].data() + sizeof(hdr) + 8 * k, 8);
        unit_w.push_back(w);
      }
    }
    const int me = ch.index();
    if (!acc_ptrs.empty()) {
      if (static_cast<int>(acc_ptrs.size()) != world)
        throw std::invalid_argument("every rank must contribute an int64 accumulator");
      check(ew_peer_fold_create_i64(world, me, n_, acc_ptrs.data(), out_ptrs.data(), &fold_));
    } else {
      total_units_ = static_cast<std::int64_t>(unit_ptrs.size());
      check(ew_peer_fold_create(world, me, n_, unit_ptrs.data(), unit_w.data(),
                                static_cast<int>(unit_ptrs.size()), out_ptrs.data(), &fold_));
    }
    barrier_ = make_barrier(peers_, ch.members(), ch.me(), 0);
  } catch (...) {
    if (barrier_) ew_peer_barrier_free(barrier_);
    barrier_ = nullptr;
    ew_peer_fold_free(fold_);
    fold_ = nullptr;
    peers_.close();
    dfree(flags_);
    dfree(dmax_);
    flags_ = nullptr;
    dmax_ = nullptr;
    throw;
  }
  ch.barrier();  // every flag array zeroed before the first device barrier
}

PeerReduce::~PeerReduce() {
  if (barrier_) ew_peer_barrier_free(barrier_);
  ew_peer_fold_free(fold_);
  peers_.close();
  dfree(flags_);
  dfree(dmax_);
}

int PeerReduce::scale(ew_stream_t stream) {
  NvtxRange range("ew.reduce.scale");
  check(ew_weighted_absmax(units_.data(), weights_.data(), static_cast<int>(units_.size()), n_,
                           dmax_, stream));
  double local = 0.0;
  check(ew_memcpy_async(&local, dmax_, 8, stream));
  check(ew_stream_sync(stream));
  std::string mine(8, '\0');
  std::memcpy(mine.data(), &local, 8);
  double global = 0.0;
  bool nan = false;
  for (const std::string& v : ch_.allgather(mine)) {
    double x = 0.0;
    std::memcpy(&x, v.data(), 8);
    nan = nan || x != x;
    global = std::max(global, x);
  }
  int bits = 0;
  check(ew_fixed_point_bits(nan ? global * 0.0 / 0.0 : global, std::max<std::int64_t>(1, total_units_),
                            &bits));
  return bits;
}

void PeerReduce::run(int frac_bits, ew_stream_t stream) {
  check(ew_peer_barrier_wait(barrier_, timeout_s_, stream));  // units written everywhere
  check(ew_peer_fold_reduce_scatter(fold_, frac_bits, stream));
  check(ew_peer_barrier_wait(barrier_, timeout_s_, stream));  // every slice reduced
  check(ew_peer_fold_all_gather(fold_, stream));
}

void PeerReduce::wait(ew_stream_t stream) {
  check(ew_peer_barrier_wait(barrier_, timeout_s_, stream));
}

bool PeerReduce::timed_out() const {
  int t = 0;
  check(ew_peer_barrier_timed_out(barrier_, &t));
  return t != 0;
}

// -------------------------------------------------------- FailureDetector

namespace {

struct alignas(64) BeatSlot {
  std::uint64_t beats;
  std::int64_t t_ns;  // steady_clock (CLOCK_MONOTONIC) of the last beat
};

std::int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             Clock::now().time_since_epoch()).count();
}

std::string shm_safe(const std::string& s) {
  std::string out;
  for (char c : s) out += (std::isalnum(static_cast<unsigned char>(c)) ? c : '_');
  return out;
}

}  // namespace

FailureDetector::FailureDetector(Channel& ch, const std::string& tag, DetectorOptions opt)
    : members_(ch.members()), me_(ch.me()), opt_(opt) {
  if (opt_.period_s <= 0 || opt_.timeout_s <= opt_.period_s)
    throw std::invalid_argument("FailureDetector: need 0 < period_s < timeout_s");
  name_ = "/ew_hb_" + shm_safe(tag) + "_" + shm_safe(ch.name());
  shm_bytes_ = sizeof(BeatSlot) * members_.size();
  owner_ = ch.index() == 0;
  if (owner_) {
    ::shm_unlink(name_.c_str());  // a stale segment of an earlier run
    const int fd = ::shm_open(name_.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) throw std::runtime_error("shm_open(" + name_ + ") failed");
    if (::ftruncate(fd, static_cast<off_t>(shm_bytes_)) != 0) {
      ::close(fd);
      ::shm_unlink(name_.c_str());
      throw std::runtime_error("ftruncate(" + name_ + ") failed");
    }
    shm_ = ::mmap(nullptr, shm_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    ::close(fd);
    if (shm_ == MAP_FAILED) {
      shm_ = nullptr;
      ::shm_unlink(name_.c_str());
      throw std::runtime_error("mmap(" + name_ + ") failed");
    }
    std::memset(shm_, 0, shm_bytes_);
  }
  ch.barrier();  // the segment exists
  if (!owner_) {
    const int fd = ::shm_open(name_.c_str(), O_RDWR, 0600);
    if (fd < 0) throw std::runtime_error("shm_open(" + name_ + ") failed");
    shm_ = ::mmap(nullptr, shm_bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    ::close(fd);
    if (shm_ == MAP_FAILED) {
      shm_ = nullptr;
      throw std::runtime_error("mmap(" + name_ + ") failed");
    }
  }
  BeatSlot* slot = static_cast<BeatSlot*>(shm_) + ch.index();
  __atomic_store_n(&slot->t_ns, now_ns(), __ATOMIC_RELEASE);
  __atomic_store_n(&slot->beats, std::uint64_t{1}, __ATOMIC_RELEASE);
  ch.barrier();  // every member has a first beat before anyone watches
  int device = 0;
  cuda_check(cudaGetDevice(&device), "cudaGetDevice");
  beater_ = std::thread([this, device] {
    cudaSetDevice(device);
    beat_loop();
  });
}

FailureDetector::~FailureDetector() {
  stop_beating();
  if (shm_ != nullptr) ::munmap(shm_, shm_bytes_);
  if (owner_) ::shm_unlink(name_.c_str());
}

void FailureDetector::stop_beating() {
  stop_ = true;
  if (beater_.joinable()) beater_.join();
}

void FailureDetector::beat_loop() {
  // a beat is published only after the device completed a 4-byte H2D copy
  // issued for it (a copy engine, not an SM: a long kernel of the job does
  // not delay beats; a device that stops executing work stops them)
  cudaStream_t s = nullptr;
  void* word = nullptr;
  std::uint32_t* host = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&word, 4) != cudaSuccess ||
      cudaHostAlloc(reinterpret_cast<void**>(&host), 4, cudaHostAllocDefault) != cudaSuccess)
    return;  // no beats: peers will fail this member, which cannot use its GPU
  BeatSlot* slot = static_cast<BeatSlot*>(shm_) + index_of(members_, me_);
  std::uint64_t n = 1;
  const auto period = std::chrono::duration<double>(opt_.period_s);
  while (!stop_) {
    *host = static_cast<std::uint32_t>(n);
    if (cudaMemcpyAsync(word, host, 4, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      break;  // a failed device: stop beating
    __atomic_store_n(&slot->t_ns, now_ns(), __ATOMIC_RELEASE);
    __atomic_store_n(&slot->beats, ++n, __ATOMIC_RELEASE);
    std::this_thread::sleep_for(period);
  }
  cudaFreeHost(host);
  cudaFree(word);
  cudaStreamDestroy(s);
}

std::vector<int> FailureDetector::failed(std::vector<double>* silence_s) const {
  std::vector<int> out;
  if (silence_s) silence_s->clear();
  const std::int64_t now = now_ns();
  const BeatSlot* slots = static_cast<const BeatSlot*>(shm_);
  for (std::size_t i = 0; i < members_.size(); ++i) {
    if (members_[i] == me_) continue;
    const double age = static_cast<double>(now - __atomic_load_n(&slots[i].t_ns, __ATOMIC_ACQUIRE)) * 1e-9;
    if (age > opt_.timeout_s) {
      out.push_back(members_[i]);
      if (silence_s) silence_s->push_back(age);
    }
  }
  return out;
}

std::vector<int> FailureDetector::wait_for_failure(double max_wait_s, double* detect_s) const {
  const auto t0 = Clock::now();
  const auto poll = std::chrono::duration<double>(opt_.period_s / 4);
  for (;;) {
    std::vector<double> age;
    const std::vector<int> f = failed(&age);
    if (!f.empty()) {
      if (detect_s) *detect_s = *std::max_element(age.begin(), age.end());
      return f;
    }
    if (seconds(t0, Clock::now()) > max_wait_s) {
      if (detect_s) *detect_s = 0.0;
      return {};
    }
    std::this_thread::sleep_for(poll);
  }
}

// ------------------------------------------------------------------ MTTR

std::string mttr_csv_header() {
  return "event,step,t_event_s,kind,detect_s,comm_repair_s,remap_s,migration_stall_s,"
         "other_s,lost_work_s,total_s";
}

std::string mttr_csv_row(int index, const MttrEvent& m) {
  char buf[320];
  std::snprintf(buf, sizeof(buf), "%d,%d,%.9g,%s,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g", index,
                m.step, m.t_event_s, m.kind.c_str(), m.detect_s, m.comm_repair_s, m.remap_s,
                m.migration_stall_s, m.other_s, m.lost_work_s, m.total_s());
  return buf;
}

// ------------------------------------------------------- VerifiedMove (impl)

namespace {

// One verified pull move among `survivors` (the executor, the three block-sum
// arrays on every survivor, the slice verifier); shared by the prepared and
// the failure-time paths.
struct VerifiedMove {
  std::unique_ptr<ReshardExecutor> exec;
  std::unique_ptr<BlockVerifier> verifier = std::make_unique<BlockVerifier>();

  void wire(const PeerBuffers& peers, const ReshardPlan& rp, int me, std::int64_t n_words) {
    const std::vector<int> survivors = without(rp.old_members, rp.failed);
    std::vector<const std::uint64_t*> plus, minus;
    for (int s : rp.new_members)
      plus.push_back(static_cast<const std::uint64_t*>(peers.get(kLanded, s)));
    for (int s : survivors)
      minus.push_back(static_cast<const std::uint64_t*>(peers.get(kOldBlocks, s)));
    for (int d : rp.failed)
      minus.push_back(static_cast<const std::uint64_t*>(peers.get(kReplicaBlocks,
                                                                   rp.ring.backed_up_by(d))));
    for (const std::uint64_t* p : plus)
      if (!p) throw std::runtime_error("landed block sums of a survivor are not mapped");
    for (const std::uint64_t* p : minus)
      if (!p) throw std::runtime_error("source block sums of a survivor are not mapped");
    const auto [lo, hi] = slice_of(n_words, index_of(rp.new_members, me),
                                   static_cast<int>(rp.new_members.size()));
    verifier->set(plus, minus, n_words, lo, hi);
  }
};

// Shared launch + verdict: zero landed, copy (verified), device barrier,
// slice check, host verdict over the survivors' channel.
bool run_move(const ReshardExecutor& exec, const BlockVerifier& verifier, std::uint64_t* landed,
              std::int64_t n_words,
              std::uint32_t* bad, ew_peer_barrier* barrier, double timeout_s, Channel& survivors,
              ew_stream_t stream, MttrEvent* ev, bool stale_snapshot = false) {
  NvtxRange range("ew.remap.copy_verify");
  cudaEvent_t e[3];
  for (cudaEvent_t& x : e) cuda_check(cudaEventCreate(&x), "cudaEventCreate");
  const auto t0 = Clock::now();
  check(ew_memset_async(landed, 0, n_words * 8, stream));
  cuda_check(cudaEventRecord(e[0], reinterpret_cast<cudaStream_t>(stream)), "record");
  exec.launch(stream, landed);
  cuda_check(cudaEventRecord(e[1], reinterpret_cast<cudaStream_t>(stream)), "record");
  if (barrier != nullptr) {
    check(ew_peer_barrier_wait(barrier, timeout_s, stream));  // every survivor landed
  } else {
    check(ew_stream_sync(stream));
    survivors.barrier();
  }
  verifier.run(stream, bad);
  cuda_check(cudaEventRecord(e[2], reinterpret_cast<cudaStream_t>(stream)), "record");
  std::uint32_t bad_host = 0;
  check(ew_memcpy_async(&bad_host, bad, 4, stream));
  check(ew_stream_sync(stream));
  int timed_out = 0;
  if (barrier != nullptr) check(ew_peer_barrier_timed_out(barrier, &timed_out));
  const auto t1 = Clock::now();
  nvtxRangePushA("ew.remap.verdict");
  // one verdict round: mismatched words, barrier timeouts, and members whose
  // snapshot is not of the event's step (SnapshotRing::step_tag)
  const std::int64_t total = survivors.sum(static_cast<std::int64_t>(bad_host) +
                                           (timed_out ? (std::int64_t{1} << 40) : 0) +
                                           (stale_snapshot ? (std::int64_t{1} << 50) : 0));
  nvtxRangePop();
  const auto t2 = Clock::now();
  float copy_ms = 0.f, verify_ms = 0.f;
  cudaEventElapsedTime(&copy_ms, e[0], e[1]);
  cudaEventElapsedTime(&verify_ms, e[1], e[2]);
  for (cudaEvent_t x : e) cudaEventDestroy(x);
  if (ev != nullptr) {
    ev->phases["copy_s"] = copy_ms / 1e3;
    ev->phases["barrier_verify_s"] = verify_ms / 1e3;
    ev->phases["verdict_exchange_s"] = seconds(t1, t2);
    ev->phases["launch_to_verdict_s"] = seconds(t0, t2);
    ev->phases["mismatched_block_words"] = static_cast<double>(total % (std::int64_t{1} << 40));
    ev->phases["barrier_timeouts"] = static_cast<double>((total >> 40) & 1023);
    ev->phases["stale_snapshots"] = static_cast<double>(total >> 50);
  }
  return total == 0;
}

}  // namespace

// --------------------------------------------------------- PreparedRecovery

PreparedRecovery::PreparedRecovery(Channel& ch, const std::vector<std::int64_t>& layer_bytes,
                                   void* old_buf, const std::uint64_t* old_rows, void* replica,
                                   const std::uint64_t* replica_rows, void* new_buf,
                                   std::int64_t new_capacity, PreparedOptions opt)
    : ch_(ch), members_(ch.members()), me_(ch.me()), opt_(opt) {
  NvtxRange range("ew.prepare_recovery");
  const int n = static_cast<int>(members_.size());
  if (n < 2) throw std::invalid_argument("PreparedRecovery needs at least two members");
  std::int64_t max_new = 0;
  for (int d : members_) {
    if (d == me_) continue;
    plans_[d] = std::make_unique<ReshardPlan>(
        ReshardPlan::build(layer_bytes, members_, without(members_, {d})));
    max_new = std::max(max_new, shard_bytes(plans_[d]->dst, me_));
  }
  const ReshardPlan& any = *plans_.begin()->second;
  n_words_ = 2 * any.n_blocks(opt_.block_bytes);
  try {
    if (new_buf != nullptr) {
      if (new_capacity < max_new)
        throw std::invalid_argument("PreparedRecovery: NEW buffer of " +
                                    std::to_string(new_capacity) + " bytes, the largest "
                                    "departure needs " + std::to_string(max_new));
      new_buf_ = new_buf;
      own_new_ = false;
    } else {
      new_buf_ = dalloc<std::uint8_t>((max_new + 31) / 32 * 32);
    }
    landed_ = dalloc<std::uint64_t>(n_words_);
    old_blocks_ = dalloc<std::uint64_t>(n_words_);
    replica_blocks_ = dalloc<std::uint64_t>(n_words_);
    bad_ = dalloc<std::uint32_t>(4);
    flags_ = dalloc<unsigned long long>(static_cast<std::int64_t>(n) * n);
    check(ew_memset_async(old_blocks_, 0, n_words_ * 8, nullptr));
    check(ew_memset_async(replica_blocks_, 0, n_words_ * 8, nullptr));
    check(ew_memset_async(landed_, 0, n_words_ * 8, nullptr));
    check(ew_memset_async(flags_, 0, 8 * static_cast<std::int64_t>(n) * n, nullptr));
    // this rank's share of the source block sums: its OLD shard and the
    // replica it keeps (from the snapshot rows when given)
    const std::int64_t nb = n_words_ / 2;
    add_blocks(any.src, me_, old_buf, old_rows, old_blocks_, nb, opt_.block_bytes, nullptr);
    if (replica != nullptr)
      add_blocks(any.src, any.ring.backs_up(me_), replica, replica_rows, replica_blocks_, nb,
                 opt_.block_bytes, nullptr);
    check(ew_device_sync());
    peers_.exchange(ch_, {{static_cast<int>(BufRole::Old), old_buf},
                          {static_cast<int>(BufRole::Replica), replica},
                          {kLanded, landed_},
                          {kOldBlocks, old_blocks_},
                          {kReplicaBlocks, replica_blocks_},
                          {kFlags, flags_}});
    peers_.put(static_cast<int>(BufRole::New), me_, new_buf_);
    for (const auto& [d, rp] : plans_) {
      auto mv = std::make_unique<VerifiedMove>();
      mv->exec = std::make_unique<ReshardExecutor>(*rp, me_, false, opt_.block_bytes,
                                                   opt_.local_replicas && replica != nullptr);
      mv->exec->bind(peers_, true);
      mv->wire(peers_, *rp, me_, n_words_);
      execs_[d] = std::move(mv->exec);
      verifiers_[d] = std::move(mv->verifier);
      survivors_[d] = std::make_unique<Channel>(ch_.store(), ch_.name() + "/without" +
                                                                  std::to_string(d),
                                                rp->new_members, me_);
      barriers_[d] = make_barrier(peers_, rp->new_members, me_,
                                  static_cast<std::int64_t>(index_of(members_, d)) * n);
    }
  } catch (...) {
    release();
    throw;
  }
  ch_.barrier();  // every flag array zeroed and every mapping in place
}

PreparedRecovery::~PreparedRecovery() { release(); }

void PreparedRecovery::release() {
  for (auto& [d, b] : barriers_) ew_peer_barrier_free(b);
  barriers_.clear();
  verifiers_.clear();
  execs_.clear();
  peers_.close();
  if (!own_new_) new_buf_ = nullptr;
  for (void* p : {static_cast<void*>(new_buf_), static_cast<void*>(landed_),
                  static_cast<void*>(old_blocks_), static_cast<void*>(replica_blocks_),
                  static_cast<void*>(bad_), static_cast<void*>(flags_)})
    dfree(p);
  new_buf_ = nullptr;
  landed_ = old_blocks_ = replica_blocks_ = nullptr;
  bad_ = nullptr;
  flags_ = nullptr;
}

std::int64_t PreparedRecovery::new_bytes(int departed) const {
  return shard_bytes(plans_.at(departed)->dst, me_);
}

bool PreparedRecovery::recover(int departed, ew_stream_t stream, MttrEvent* ev,
                               bool stale_snapshot) {
  if (departed == me_) throw std::invalid_argument("the departed member does not recover itself");
  if (!plans_.count(departed))
    throw std::invalid_argument("member " + std::to_string(departed) + " is not in the group");
  const bool ok = run_move(*execs_.at(departed), *verifiers_.at(departed), landed_, n_words_,
                           bad_, barriers_.at(departed), opt_.barrier_timeout_s,
                           *survivors_.at(departed), stream, ev, stale_snapshot);
  if (ev != nullptr) {
    ev->phases["plan_s"] = 0.0;  // planned in steady state
    ev->phases["prepared"] = 1.0;
    ev->verified = ok;
  }
  return ok;
}

// ----------------------------------------------------------------- DpGroup

namespace {

std::string csv(const std::vector<int>& v) {
  std::string s;
  for (int x : v) s += (s.empty() ? "" : ",") + std::to_string(x);
  return s;
}

std::vector<int> parse_csv(const std::string& s) {
  std::vector<int> out;
  std::size_t p = 0;
  while (p < s.size()) {
    const std::size_t q = s.find(',', p);
    out.push_back(std::stoi(s.substr(p, q == std::string::npos ? std::string::npos : q - p)));
    if (q == std::string::npos) break;
    p = q + 1;
  }
  return out;
}

// NCCL communicator over ch's members in member order (ncclCommInitRank; the
// unique id comes from member index 0 over the channel).  Collective.
ew_comm* init_comm(Channel& ch) {
  std::string id;
  if (ch.index() == 0) {
    id.assign(128, '\0');
    check(ew_comm_unique_id(id.data()));
  }
  const std::vector<std::string> ids = ch.allgather(id);
  if (ids.front().size() != 128) throw std::runtime_error("communicator id exchange failed");
  ew_comm* c = nullptr;
  check(ew_comm_init(ids.front().data(), static_cast<int>(ch.members().size()), ch.index(), &c));
  return c;
}

}  // namespace

// Steady-state peer mapping of the group (DpGroup::premap / prepare_join):
// the buffers a pull program reads on every participant, plus this rank's
// verification arrays, mapped once.
// A move lowered and bound ahead of its event (DpGroup::prepare_move).
struct PreparedMove {
  std::unique_ptr<ReshardPlan> rp;
  VerifiedMove mv;
  void* new_buf = nullptr;
};

// Steady-state peer mapping of the group (DpGroup::premap / prepare_join):
// the buffers a pull program reads on every participant, plus this rank's
// verification arrays, mapped once; the maps that turn the per-step
// snapshot rows into source block sums; moves prepared ahead of events.
struct DpGroup::Premap {
  PeerBuffers peers;
  void* old_buf = nullptr;
  void* replica = nullptr;
  const std::uint64_t* old_rows = nullptr;      // per-step snapshot rows (refreshed in place)
  const std::uint64_t* replica_rows = nullptr;
  std::vector<int> layout_members;  // the membership OLD and the replica are laid out over
  ew_shardmap* old_map = nullptr;
  ew_shardmap* rep_map = nullptr;
  std::set<int> covers;  // ranks whose entries are in the table
  std::int64_t n_words = 0;
  std::unique_ptr<DevArray<std::uint64_t>> landed, old_blocks, rep_blocks;
  std::unique_ptr<DevArray<std::uint32_t>> bad;
  std::map<std::pair<int, std::vector<int>>, std::unique_ptr<PreparedMove>> moves;

  explicit Premap(std::int64_t words) : n_words(words) {
    landed = std::make_unique<DevArray<std::uint64_t>>(words);
    old_blocks = std::make_unique<DevArray<std::uint64_t>>(words);
    rep_blocks = std::make_unique<DevArray<std::uint64_t>>(words);
    bad = std::make_unique<DevArray<std::uint32_t>>(4);
  }
  ~Premap() {
    moves.clear();
    peers.close();
    ew_shardmap_free(old_map);
    ew_shardmap_free(rep_map);
  }
  std::map<int, void*> mine() const {
    return {{static_cast<int>(BufRole::Old), old_buf},
            {static_cast<int>(BufRole::Replica), replica},
            {kLanded, landed->p},
            {kOldBlocks, old_blocks->p},
            {kReplicaBlocks, rep_blocks->p}};
  }
  bool covers_all(const std::vector<int>& ranks) const {
    for (int r : ranks)
      if (!covers.count(r)) return false;
    return true;
  }
  // this rank's source block sums of a move out of rp.src: from the
  // snapshot rows when they describe these buffers and this layout, else a
  // re-read of the buffers (stream-ordered either way)
  void source_sums(const ReshardPlan& rp, int me, const RankBuffers& bufs, int owner,
                   bool holder, std::int64_t block, ew_stream_t stream) const {
    const std::int64_t nb = n_words / 2;
    const bool same = layout_members == rp.old_members;
    if (same && old_rows && old_map && old_buf == bufs.old_buf)
      check(ew_rows_to_blocks(old_map, old_rows, old_blocks->p, nb, stream));
    else
      add_blocks(rp.src, me, bufs.old_buf, nullptr, old_blocks->p, nb, block, stream);
    if (!holder) return;
    if (same && replica_rows && rep_map && replica == bufs.replica)
      check(ew_rows_to_blocks(rep_map, replica_rows, rep_blocks->p, nb, stream));
    else
      add_blocks(rp.src, owner, bufs.replica, nullptr, rep_blocks->p, nb, block, stream);
  }
};

namespace {
std::int64_t group_words(const std::vector<std::int64_t>& layer_bytes, std::int64_t block) {
  std::int64_t total = 0;
  for (std::int64_t b : layer_bytes) total += b;
  return 2 * ((total + block - 1) / block);
}
}  // namespace

void DpGroup::premap(const RankBuffers& bufs, const std::uint64_t* old_rows,
                     const std::uint64_t* replica_rows) {
  if (ch_ == nullptr) throw std::invalid_argument("premap: a joiner is mapped by prepare_join");
  NvtxRange range("ew.premap");
  auto pm = std::make_unique<Premap>(group_words(layer_bytes_, opt_.block_bytes));
  pm->old_buf = bufs.old_buf;
  pm->replica = bufs.replica;
  pm->old_rows = old_rows;
  pm->replica_rows = replica_rows;
  pm->layout_members = members_;
  const ReshardPlan self = ReshardPlan::build(layer_bytes_, members_, members_);
  if (old_rows != nullptr) pm->old_map = make_map(shard_segments(self.src, me_), opt_.block_bytes);
  if (replica_rows != nullptr && bufs.replica != nullptr && members_.size() > 1)
    pm->rep_map = make_map(shard_segments(self.src, self.replica_of(me_)), opt_.block_bytes);
  pm->peers.exchange(*ch_, pm->mine());
  pm->covers.insert(members_.begin(), members_.end());
  pm_ = std::move(pm);
}

void DpGroup::prepare_move(EventKind kind, const std::vector<int>& targets, void* new_buf) {
  if (!pm_) throw std::logic_error("prepare_move: premap (members) / prepare_join (joiners) first");
  if (kind == EventKind::FailSlow) throw std::invalid_argument("prepare_move: no move for FailSlow");
  const bool join = kind == EventKind::ScaleOut;
  std::vector<int> t(targets.begin(), targets.end());
  std::sort(t.begin(), t.end());
  t.erase(std::unique(t.begin(), t.end()), t.end());
  std::vector<int> next;
  if (join) {
    next = members_;
    next.insert(next.end(), t.begin(), t.end());
    std::sort(next.begin(), next.end());
  } else {
    next = without(members_, std::set<int>(t.begin(), t.end()));
    if (std::binary_search(t.begin(), t.end(), me_)) return;  // a departing member has no part
  }
  if (!pm_->covers_all(next) || !pm_->covers_all(members_))
    throw std::invalid_argument("prepare_move: the participants are not mapped");
  if (new_buf == nullptr) throw std::invalid_argument("prepare_move: NEW buffer required");
  NvtxRange range("ew.prepare_move");
  auto mv = std::make_unique<PreparedMove>();
  mv->rp = std::make_unique<ReshardPlan>(ReshardPlan::build(layer_bytes_, members_, next));
  mv->new_buf = new_buf;
  pm_->peers.put(static_cast<int>(BufRole::New), me_, new_buf);
  mv->mv.exec = std::make_unique<ReshardExecutor>(*mv->rp, me_, false, opt_.block_bytes);
  mv->mv.exec->bind(pm_->peers, true);
  mv->mv.wire(pm_->peers, *mv->rp, me_, pm_->n_words);
  pm_->moves[{join ? 1 : 0, t}] = std::move(mv);
}

DpGroup::DpGroup(Channel& ch, const std::vector<std::int64_t>& layer_bytes, ew_comm* comm,
                 DpGroupOptions opt)
    : store_(ch.store()), name_(ch.name()), me_(ch.me()), ch_(&ch), layer_bytes_(layer_bytes),
      members_(ch.members()), comm_(comm), opt_(opt) {
  mb_sizes_.assign(members_.size(), opt_.per_slot_mbs);
  for (std::size_t i = 0; i < members_.size(); ++i)
    for (std::size_t j = i + 1; j < members_.size(); ++j)
      links_.insert(make_link(members_[i], members_[j]));
  if (opt_.prepare_comms && comm_ != nullptr) prepare();
}

DpGroup::DpGroup(Store& store, std::string group_name, const std::vector<std::int64_t>& layer_bytes,
                 std::vector<int> members, int me, DpGroupOptions opt)
    : store_(store), name_(std::move(group_name)), me_(me), ch_(nullptr),
      layer_bytes_(layer_bytes), members_(std::move(members)), opt_(opt) {
  std::sort(members_.begin(), members_.end());
  if (members_.empty()) throw std::invalid_argument("a joiner needs the group's members");
  if (index_of(members_, me_) >= 0)
    throw std::invalid_argument("rank " + std::to_string(me_) + " is already a member");
  // the members' link pool: the mesh over the current members (the DP mesh
  // after any departures, communicator.cpp:74-81)
  for (std::size_t i = 0; i < members_.size(); ++i)
    for (std::size_t j = i + 1; j < members_.size(); ++j)
      links_.insert(make_link(members_[i], members_[j]));
}

DpGroup::~DpGroup() {
  // ncclCommAbort throughout: a communicator that includes a departed member
  // cannot be destroyed collectively (its peer never arrives), and the group
  // may be torn down on any subset of its members
  for (auto& [d, c] : prepared_comms_) ew_comm_abort(c);
  prepared_comms_.clear();
  for (auto& [m, c] : standby_comms_) ew_comm_abort(c);
  standby_comms_.clear();
  ew_comm_abort(comm_);
  for (auto it = retired_.rbegin(); it != retired_.rend(); ++it) ew_comm_abort(*it);
}

void DpGroup::prepare() {
  std::vector<std::vector<int>> singles;
  for (int d : members_) singles.push_back({d});
  prepare(singles);
}

void DpGroup::prepare(const std::vector<std::vector<int>>& departures) {
  if (comm_ == nullptr || members_.size() < 2 || ch_ == nullptr) return;
  NvtxRange range("ew.prepare_comms");
  std::vector<std::vector<int>> sets;
  for (std::vector<int> d : departures) {
    std::sort(d.begin(), d.end());
    d.erase(std::unique(d.begin(), d.end()), d.end());
    if (d.empty() || d.size() >= members_.size())
      throw std::invalid_argument("prepare: a departure set must leave survivors");
    for (int x : d)
      if (index_of(members_, x) < 0)
        throw std::invalid_argument("prepare: member " + std::to_string(x) + " not in the group");
    if (std::find(sets.begin(), sets.end(), d) == sets.end()) sets.push_back(d);
  }
  for (auto& [d, c] : prepared_comms_) retired_.push_back(c);
  prepared_comms_.clear();
  for (auto it = retired_.rbegin(); it != retired_.rend(); ++it) ew_comm_abort(*it);
  retired_.clear();
  const int key = index_of(members_, me_);
  for (const std::vector<int>& d : sets) {
    const bool out = std::binary_search(d.begin(), d.end(), me_);
    ew_comm* c = nullptr;
    check(ew_comm_split(comm_, out ? -1 : 0, key, opt_.share_comm_resources ? 1 : 0, &c));
    if (c != nullptr) prepared_comms_[d] = c;
  }
  // one collective on each (NCCL connects lazily): the repair at failure
  // time is then a lookup of a live communicator.  One communicator at a
  // time across the group (host barrier between them): siblings that share
  // resources must never run concurrently, and the members of different
  // siblings would otherwise start them in different orders
  const DevArray<std::int64_t> one(1);
  for (const std::vector<int>& d : sets) {
    if (prepared_comms_.count(d)) check(ew_allreduce_i64(prepared_comms_.at(d), one.p, 1, nullptr));
    check(ew_device_sync());
    ch_->barrier();
  }
}

void DpGroup::prepare_join(const std::vector<int>& joiners) {
  std::set<int> add(joiners.begin(), joiners.end());
  if (add.empty()) throw std::invalid_argument("prepare_join: no joiners");
  for (int j : add)
    if (index_of(members_, j) >= 0)
      throw std::invalid_argument("joining member " + std::to_string(j) + " is already in the group");
  std::vector<int> next = members_;
  next.insert(next.end(), add.begin(), add.end());
  std::sort(next.begin(), next.end());
  NvtxRange range("ew.prepare_join");
  const int round = standby_rounds_[next]++;
  Channel all(store_, name_ + "/standby" + std::to_string(round) + ":" + csv(members_) + ">" +
                          csv(next), next, me_);
  // what the members run: a NCCL communicator (then the joiners need the
  // grown one) and a steady-state mapping (then the joiners join it)
  const bool joiner = add.count(me_) > 0;
  const std::vector<std::string> flags =
      all.allgather(joiner ? "j" : std::string(comm_ ? "n" : "-") + (pm_ ? "p" : "-"));
  bool nccl = true, members_mapped = true;
  for (const std::string& f : flags) {
    if (f == "j") continue;
    nccl = nccl && f[0] == 'n';
    members_mapped = members_mapped && f[1] == 'p';
  }
  ew_comm* c = nullptr;
  if (nccl) {
    c = init_comm(all);
    try {
      const DevArray<std::int64_t> one(1);
      check(ew_allreduce_i64(c, one.p, 1, nullptr));
      check(ew_device_sync());
    } catch (...) {
      ew_comm_abort(c);
      throw;
    }
  }
  if (members_mapped) {
    if (joiner) pm_ = std::make_unique<Premap>(group_words(layer_bytes_, opt_.block_bytes));
    pm_->peers.exchange(all, pm_->mine());
    pm_->covers.insert(next.begin(), next.end());
  }
  all.barrier();
  if (c != nullptr) {
    const auto it = standby_comms_.find(next);
    if (it != standby_comms_.end()) retired_.push_back(it->second);
    standby_comms_[next] = c;
  }
}

void DpGroup::commit_members(std::vector<int> next) {
  members_ = std::move(next);
  // later collectives of the group (prepare()) run over the new membership
  own_ch_ = std::make_unique<Channel>(store_, name_ + "/members" + std::to_string(events_) + ":" +
                                                  csv(members_), members_, me_);
  ch_ = own_ch_.get();
}

MttrEvent DpGroup::recover(const std::vector<int>& departed, EventKind kind,
                           const RankBuffers& bufs, ew_stream_t stream, int step) {
  if (kind == EventKind::ScaleOut) return admit(departed, bufs, stream, step);
  if (kind == EventKind::FailSlow)
    throw std::invalid_argument("DpGroup::recover handles FailStop / ScaleIn / ScaleOut");
  if (ch_ == nullptr) throw std::invalid_argument("a joiner takes part in its ScaleOut first");
  std::set<int> gone(departed.begin(), departed.end());
  for (int d : gone)
    if (index_of(members_, d) < 0)
      throw std::invalid_argument("departed member " + std::to_string(d) + " is not in the group");
  if (gone.count(me_)) throw std::invalid_argument("a departed member does not recover");
  const std::vector<int> survivors = without(members_, gone);
  MttrEvent ev;
  ev.step = step;
  ev.kind = to_string(kind);
  NvtxRange range("ew.recover");
  const auto t0 = Clock::now();
  nvtxRangePushA("ew.comm_repair");

  // comm repair: the edit plan (communicator.cpp:54-105), then the NCCL
  // communicator: a prepared split (lookup) or a shrink at failure time;
  // its first collective is part of the repair
  ElasticEvent e;
  e.kind = kind;
  e.targets = std::vector<DeviceId>(gone.begin(), gone.end());
  const EditPlan edit = plan_edit({CommGroup{"dp", members_, GroupTopology::Mesh}}, e, links_);
  for (const Link& l : edit.links_to_remove) links_.erase(l);
  links_.insert(edit.links_to_add.begin(), edit.links_to_add.end());
  const auto t_edit = Clock::now();
  ew_comm* new_comm = nullptr;
  if (comm_ != nullptr) {
    const std::vector<int> key(gone.begin(), gone.end());
    if (prepared_comms_.count(key)) {
      new_comm = prepared_comms_.at(key);
      prepared_comms_.erase(key);
      ev.phases["comm_prepared"] = 1.0;
    } else {
      std::vector<int> ranks;
      for (int d : gone) ranks.push_back(index_of(members_, d));  // ranks of the CURRENT comm
      check(ew_comm_shrink(comm_, ranks.data(), static_cast<int>(ranks.size()), 0, &new_comm));
      ev.phases["comm_prepared"] = 0.0;
    }
    const auto t_c = Clock::now();
    const DevArray<std::int64_t> one(1);
    check(ew_allreduce_i64(new_comm, one.p, 1, stream));
    check(ew_stream_sync(stream));
    ev.phases["comm_acquire_s"] = seconds(t_edit, t_c);
    ev.phases["first_collective_s"] = seconds(t_c, Clock::now());
  }
  ev.phases["plan_edit_s"] = seconds(t0, t_edit);
  const auto t1 = Clock::now();
  ev.comm_repair_s = seconds(t0, t1);
  nvtxRangePop();
  nvtxRangePushA("ew.reshape");

  // dataflow: the global batch over the survivors (dataflow.cpp:52-69)
  MicrobatchAssignment mb;
  for (std::size_t i = 0; i < members_.size(); ++i) mb.slots.push_back(static_cast<int>(i));
  mb.per_slot_mbs = mb_sizes_;
  mb.num_microbatches = opt_.num_microbatches;
  std::vector<int> idx;
  for (int s : survivors) idx.push_back(index_of(members_, s));
  const MicrobatchAssignment next = reshard_microbatches(mb, idx);
  const auto t2 = Clock::now();
  ev.other_s = seconds(t1, t2);
  nvtxRangePop();
  NvtxRange remap("ew.remap");

  // remap
  // SnapshotRing::step_tag (param_fabric.hpp:42): the state a survivor moves
  // must be the event's step; a mismatch fails the verdict
  const bool stale = snapshot_step_ >= 0 && snapshot_step_ != step;
  if (prepared_ != nullptr && gone.size() == 1 && prepared_->members() == members_) {
    ev.verified = prepared_->recover(*gone.begin(), stream, &ev, stale);
  } else {
    Channel sc(store_, name_ + "/event" + std::to_string(events_), survivors, me_);
    const ReshardPlan rp = ReshardPlan::build(layer_bytes_, members_, survivors);
    const std::int64_t n_words = 2 * rp.n_blocks(opt_.block_bytes);
    const int owner = rp.replica_of(me_);
    const bool holder = owner >= 0 && rp.failed.count(owner) > 0;
    if (holder && bufs.replica == nullptr)
      throw std::invalid_argument("this rank holds the departed member's replica: pass it");
    const auto tp = Clock::now();
    // the steady-state mapping serves when every survivor passes the buffers
    // it premapped (one store round)
    const bool mine_mapped = pm_ && pm_->covers_all(survivors) && pm_->n_words == n_words &&
                             pm_->old_buf == bufs.old_buf &&
                             (!holder || pm_->replica == bufs.replica);
    const bool mapped = sc.sum(mine_mapped ? 0 : 1) == 0;
    std::unique_ptr<Premap> fresh;
    if (!mapped) fresh = std::make_unique<Premap>(n_words);
    Premap& pm = mapped ? *pm_ : *fresh;
    check(ew_memset_async(pm.old_blocks->p, 0, n_words * 8, stream));
    check(ew_memset_async(pm.rep_blocks->p, 0, n_words * 8, stream));
    pm.source_sums(rp, me_, bufs, owner, holder, opt_.block_bytes, stream);
    const auto ts = Clock::now();
    ev.phases["sums_s"] = seconds(tp, ts);
    if (!mapped) {
      fresh->old_buf = bufs.old_buf;
      fresh->replica = holder ? bufs.replica : nullptr;
      fresh->peers.exchange(sc, fresh->mine());
    }
    // a move prepared for exactly this departure set and NEW buffer skips
    // the lowering and the program build
    PreparedMove* ready = nullptr;
    if (mapped) {
      const auto it = pm_->moves.find({0, std::vector<int>(gone.begin(), gone.end())});
      if (it != pm_->moves.end() && it->second->new_buf == bufs.new_buf) ready = it->second.get();
    }
    VerifiedMove local;
    VerifiedMove& mv = ready ? ready->mv : local;
    if (!ready) {
      pm.peers.put(static_cast<int>(BufRole::New), me_, bufs.new_buf);
      mv.exec = std::make_unique<ReshardExecutor>(rp, me_, false, opt_.block_bytes);
      mv.exec->bind(pm.peers, true);
      mv.wire(pm.peers, rp, me_, n_words);
    }
    ev.phases["plan_s"] = ready ? 0.0 : rp.plan_seconds;
    ev.phases["map_bind_s"] = seconds(tp, Clock::now());
    ev.phases["bind_s"] = seconds(ts, Clock::now());
    ev.phases["premapped"] = mapped ? 1.0 : 0.0;
    ev.phases["prepared"] = ready ? 1.0 : 0.0;
    sc.barrier();  // every survivor bound and its source sums ready
    ev.verified = run_move(*mv.exec, *mv.verifier, pm.landed->p, n_words, pm.bad->p, nullptr, 0.0,
                           sc, stream, &ev, stale);
  }
  ++events_;
  ev.remap_s = seconds(t2, Clock::now());

  // commit the new membership; the communicators of other departures were
  // built over the old membership
  mb_sizes_ = next.per_slot_mbs;
  commit_members(survivors);
  if (comm_ != nullptr) {
    // the parent and the other departures' communicators include the
    // departed member: retired (aborted later, never destroyed collectively)
    for (auto& [d, c] : prepared_comms_) retired_.push_back(c);
    prepared_comms_.clear();
    for (auto& [m, c] : standby_comms_) retired_.push_back(c);
    standby_comms_.clear();
    retired_.push_back(comm_);
    comm_ = new_comm;
  }
  return ev;
}

MttrEvent DpGroup::admit(const std::vector<int>& joined, const RankBuffers& bufs,
                         ew_stream_t stream, int step) {
  std::set<int> add(joined.begin(), joined.end());
  if (add.empty()) throw std::invalid_argument("ScaleOut without joiners");
  for (int j : add)
    if (index_of(members_, j) >= 0)
      throw std::invalid_argument("joining member " + std::to_string(j) + " is already in the group");
  const bool joiner = add.count(me_) > 0;
  if (!joiner && index_of(members_, me_) < 0)
    throw std::invalid_argument("rank " + std::to_string(me_) + " is neither a member nor a joiner");
  if (bufs.new_buf == nullptr) throw std::invalid_argument("ScaleOut: pass the NEW buffer");
  if (!joiner && bufs.old_buf == nullptr)
    throw std::invalid_argument("ScaleOut: a member passes its OLD shard");
  std::vector<int> next = members_;
  next.insert(next.end(), add.begin(), add.end());
  std::sort(next.begin(), next.end());
  MttrEvent ev;
  ev.step = step;
  ev.kind = to_string(EventKind::ScaleOut);
  NvtxRange range("ew.admit");
  const auto t0 = Clock::now();
  nvtxRangePushA("ew.comm_repair");

  // comm repair: the groups after the event hold the joiners
  // (comm_edit_time, sim.cpp:436-450); plan_edit adds the links incident to
  // them that the pool lacks (communicator.cpp:65-70)
  ElasticEvent e;
  e.kind = EventKind::ScaleOut;
  e.targets = std::vector<DeviceId>(add.begin(), add.end());
  const EditPlan edit = plan_edit({CommGroup{"dp", next, GroupTopology::Mesh}}, e, links_);
  for (const Link& l : edit.links_to_remove) links_.erase(l);
  links_.insert(edit.links_to_add.begin(), edit.links_to_add.end());
  const auto t_edit = Clock::now();
  // rendezvous of members and joiners; the members hand the joiners the
  // group's state: NCCL in use, event count, micro-batch sizes.  Everyone
  // says whether it holds the standby communicator of this membership.
  Channel all(store_, name_ + "/join" + std::to_string(step) + ":" + csv(members_) + ">" +
                          csv(next), next, me_);
  const bool has_standby = standby_comms_.count(next) > 0;
  const std::string mine = std::string(has_standby ? "s" : "-") + ";" +
                           (joiner ? std::string("j") : std::string(comm_ ? "1" : "0") + ";" +
                                                            std::to_string(events_) + ";" +
                                                            csv(mb_sizes_));
  const std::vector<std::string> blobs = all.allgather(mine);
  bool all_standby = true;
  for (const std::string& b : blobs) all_standby = all_standby && !b.empty() && b[0] == 's';
  const std::string& head = blobs[static_cast<std::size_t>(index_of(next, members_.front()))];
  // head = "<s|->;<nccl>;<events>;<mb sizes>"
  const std::size_t p1 = head.find(';', 2), p2 = head.find(';', p1 + 1);
  if (head.size() < 4 || p1 == std::string::npos || p2 == std::string::npos)
    throw std::runtime_error("ScaleOut: malformed group state from the members");
  const bool nccl = head[2] == '1';
  if (joiner) {
    events_ = std::stoi(head.substr(p1 + 1, p2 - p1 - 1));
    mb_sizes_ = parse_csv(head.substr(p2 + 1));
  }
  ew_comm* new_comm = nullptr;
  if (nccl) {
    if (all_standby) {
      new_comm = standby_comms_.at(next);
      standby_comms_.erase(next);
      ev.phases["comm_prepared"] = 1.0;
    } else {
      if (has_standby) {  // not every participant built it: unusable
        retired_.push_back(standby_comms_.at(next));
        standby_comms_.erase(next);
      }
      new_comm = init_comm(all);
      ev.phases["comm_prepared"] = 0.0;
    }
    const auto t_c = Clock::now();
    const DevArray<std::int64_t> one(1);
    check(ew_allreduce_i64(new_comm, one.p, 1, stream));
    check(ew_stream_sync(stream));
    ev.phases["comm_acquire_s"] = seconds(t_edit, t_c);  // rendezvous + communicator
    ev.phases["first_collective_s"] = seconds(t_c, Clock::now());
  }
  ev.phases["plan_edit_s"] = seconds(t0, t_edit);
  const auto t1 = Clock::now();
  ev.comm_repair_s = seconds(t0, t1);
  nvtxRangePop();
  nvtxRangePushA("ew.reshape");

  // dataflow: the global batch re-dealt over the grown group (dataflow.cpp:52-69)
  MicrobatchAssignment mb;
  for (std::size_t i = 0; i < members_.size(); ++i) mb.slots.push_back(static_cast<int>(i));
  mb.per_slot_mbs = mb_sizes_;
  mb.num_microbatches = opt_.num_microbatches;
  std::vector<int> idx(next.size());
  for (std::size_t i = 0; i < next.size(); ++i) idx[i] = static_cast<int>(i);
  const MicrobatchAssignment nmb = reshard_microbatches(mb, idx);
  const auto t2 = Clock::now();
  ev.other_s = seconds(t1, t2);
  nvtxRangePop();

  // remap: the members' shards re-cut over the grown group; joiners only
  // receive.  Conservation: the landed sums of every new member equal the
  // source sums of every old member.
  {
    NvtxRange remap("ew.remap");
    const auto tp = Clock::now();
    const ReshardPlan rp = ReshardPlan::build(layer_bytes_, members_, next);
    const std::int64_t n_words = 2 * rp.n_blocks(opt_.block_bytes);
    const bool mine_mapped = pm_ && pm_->covers_all(next) && pm_->n_words == n_words &&
                             (joiner || pm_->old_buf == bufs.old_buf);
    const bool mapped = all.sum(mine_mapped ? 0 : 1) == 0;
    std::unique_ptr<Premap> fresh;
    if (!mapped) fresh = std::make_unique<Premap>(n_words);
    Premap& pm = mapped ? *pm_ : *fresh;
    check(ew_memset_async(pm.old_blocks->p, 0, n_words * 8, stream));
    check(ew_memset_async(pm.rep_blocks->p, 0, n_words * 8, stream));
    if (!joiner) pm.source_sums(rp, me_, bufs, -1, false, opt_.block_bytes, stream);
    const auto ts = Clock::now();
    ev.phases["sums_s"] = seconds(tp, ts);
    if (!mapped) {
      fresh->old_buf = joiner ? nullptr : bufs.old_buf;
      fresh->peers.exchange(all, fresh->mine());
    }
    PreparedMove* ready = nullptr;
    if (mapped) {
      const auto it = pm_->moves.find({1, std::vector<int>(add.begin(), add.end())});
      if (it != pm_->moves.end() && it->second->new_buf == bufs.new_buf) ready = it->second.get();
    }
    VerifiedMove local;
    VerifiedMove& mv = ready ? ready->mv : local;
    if (!ready) {
      pm.peers.put(static_cast<int>(BufRole::New), me_, bufs.new_buf);
      mv.exec = std::make_unique<ReshardExecutor>(rp, me_, false, opt_.block_bytes);
      mv.exec->bind(pm.peers, true);
      mv.wire(pm.peers, rp, me_, n_words);
    }
    ev.phases["plan_s"] = ready ? 0.0 : rp.plan_seconds;
    ev.phases["map_bind_s"] = seconds(tp, Clock::now());
    ev.phases["bind_s"] = seconds(ts, Clock::now());
    ev.phases["premapped"] = mapped ? 1.0 : 0.0;
    ev.phases["prepared"] = ready ? 1.0 : 0.0;
    all.barrier();  // every participant bound and its source sums ready
    const bool stale = !joiner && snapshot_step_ >= 0 && snapshot_step_ != step;
    ev.verified = run_move(*mv.exec, *mv.verifier, pm.landed->p, n_words, pm.bad->p, nullptr, 0.0,
                           all, stream, &ev, stale);
  }
  ++events_;
  ev.remap_s = seconds(t2, Clock::now());

  mb_sizes_ = nmb.per_slot_mbs;
  commit_members(next);
  if (nccl) {
    // every communicator of the old membership is retired (the departure
    // splits were built over it); the grown one serves the (d) reduce
    for (auto& [d, c] : prepared_comms_) retired_.push_back(c);
    prepared_comms_.clear();
    if (comm_ != nullptr) retired_.push_back(comm_);
    comm_ = new_comm;
  }
  return ev;
}

// --------------------------------------------------------- InPlaceExecutor

struct InPlaceExecutor::Phase {
  ew_copy_program* direct = nullptr;
  ew_copy_program* staged = nullptr;
  ew_copy_program* flush = nullptr;
  ~Phase() {
    ew_copy_program_free(direct);
    ew_copy_program_free(staged);
    ew_copy_program_free(flush);
  }
};

namespace {

// NEW's segment map restricted to packed offsets [lo, hi), re-based at `pad`
// with a leading pad segment (nothing lands there) so the map stays packed.
std::vector<Segment> clip_segments(const std::vector<Segment>& segs, std::int64_t lo,
                                   std::int64_t hi, std::int64_t pad) {
  std::vector<Segment> out;
  for (const Segment& s : segs) {
    const std::int64_t x = std::max(s.local_off, lo), y = std::min(s.local_off + s.length, hi);
    if (y <= x) continue;
    if (out.empty() && pad > 0)
      out.push_back({s.global_lo + (x - s.local_off) - pad, pad, 0});
    out.push_back({s.global_lo + (x - s.local_off), y - x, x - lo + pad});
  }
  return out;
}

ew_copy_program* program(const std::vector<CopyDesc>& copies, const std::vector<void*>& table,
                         int tr, int me, ew_shardmap* verify_map) {
  std::vector<ew_copy_desc> d;
  for (const CopyDesc& c : copies)
    d.push_back({static_cast<std::int32_t>(c.src_role), c.src_rank,
                 static_cast<std::int32_t>(c.dst_role), c.dst_rank, c.src_off, c.dst_off,
                 c.bytes});
  ew_copy_program* p = nullptr;
  if (verify_map != nullptr)
    check(ew_copy_program_create_verified(d.data(), static_cast<std::int64_t>(d.size()),
                                          table.data(), tr, me, verify_map, &p));
  else
    check(ew_copy_program_create(d.data(), static_cast<std::int64_t>(d.size()), table.data(), tr,
                                 me, &p));
  return p;
}

}  // namespace

InPlaceExecutor::InPlaceExecutor(Channel& ch, const ReshardPlan& rp, void* buf, void* replica,
                                 InPlaceOptions opt)
    : rp_(rp), me_(ch.me()), opt_(opt), buf_(buf) {
  std::int64_t biggest = 0;
  for (int r : rp_.new_members) biggest = std::max(biggest, shard_bytes(rp_.dst, r));
  std::int64_t phase = opt_.phase_bytes;
  if (phase <= 0)  // ~28 phases: profiles/r01_config_d_inplace_sweep_70gb.log
    phase = std::min<std::int64_t>(std::int64_t{8} << 30,
                                   std::max<std::int64_t>(std::int64_t{256} << 20, biggest / 28));
  sched_ = inplace_schedule(rp_.layer_bytes, rp_.src, rp_.dst, rp_.failed, opt_.stage_bytes,
                            phase, opt_.slack);
  const bool in_new = std::find(rp_.new_members.begin(), rp_.new_members.end(), me_) !=
                      rp_.new_members.end();
  const bool in_old = std::find(rp_.old_members.begin(), rp_.old_members.end(), me_) !=
                      rp_.old_members.end();
  const int n_new = static_cast<int>(rp_.new_members.size());
  if (in_new) {
    flags_ = dalloc<unsigned long long>(std::max(2, n_new));
    check(ew_memset_async(flags_, 0, 8 * std::max(2, n_new), nullptr));
    check(ew_device_sync());
  }
  std::map<int, void*> mine = {{kFlags, flags_}};
  if (in_old && !rp_.failed.count(me_)) mine[static_cast<int>(BufRole::Old)] = buf_;
  if (replica != nullptr) mine[static_cast<int>(BufRole::Replica)] = replica;
  peers_.exchange(ch, mine);
  if (!in_new) {
    ch.barrier();
    return;
  }
  try {
    for (int k = 0; k < sched_.ring && sched_.stage_alloc > 0; ++k)
      staging_.push_back(dalloc<std::uint8_t>(std::max<std::int64_t>(16, sched_.stage_alloc)));
    int top = me_;
    for (int m : rp_.old_members) top = std::max(top, m);
    for (int m : rp_.new_members) top = std::max(top, m);
    const int tr = top + 1;
    std::vector<void*> table(3 * static_cast<std::size_t>(tr), nullptr);
    for (int role = 0; role < 2; ++role)
      for (int m = 0; m < tr; ++m) table[static_cast<std::size_t>(role) * tr + m] = peers_.get(role, m);
    table[2 * static_cast<std::size_t>(tr) + me_] = buf_;
    const std::vector<CopyDesc> copies =
        reshard_copies(rp_.plan, rp_.src, rp_.dst, rp_.failed, &rp_.ring, me_, false);
    const std::vector<Segment> new_segs = shard_segments(rp_.dst, me_);
    maps_.push_back(make_map(new_segs, opt_.block_bytes));
    const InPlaceRanges& rr = sched_.ranks.at(me_);
    for (std::size_t j = 0; j < sched_.phases.size(); ++j) {
      auto ph = std::make_unique<Phase>();
      const auto [dlo, dhi] = rr.direct[j];
      const std::vector<CopyDesc> d = clip_copies(copies, dlo, dhi, dlo);
      if (!d.empty()) ph->direct = program(d, table, tr, me_, maps_.front());
      const auto [slo, shi] = rr.staged[j];
      if (shi > slo) {
        void* st = staging_[j % static_cast<std::size_t>(sched_.ring)];
        const std::int64_t pad = slo % 16;  // staging keeps NEW's alignment mod 16
        std::vector<void*> t2 = table;
        t2[2 * static_cast<std::size_t>(tr) + me_] = st;
        maps_.push_back(make_map(clip_segments(new_segs, slo, shi, pad), opt_.block_bytes));
        ph->staged = program(clip_copies(copies, slo, shi, pad), t2, tr, me_, maps_.back());
        const void* src = static_cast<std::uint8_t*>(st) + pad;
        void* dst = static_cast<std::uint8_t*>(buf_) + slo;
        const std::int64_t bytes = shi - slo;
        const int remote = 0;
        check(ew_copy_program_create_raw(&src, &dst, &bytes, &remote, 1, &ph->flush));
      }
      phases_.push_back(std::move(ph));
    }
    barrier_ = make_barrier(peers_, rp_.new_members, me_, 0);
    const int n_streams = std::max(1, opt_.gather_streams) - 1 + 2;  // extra gathers + sync + flush
    for (int k = 0; k < n_streams; ++k) {
      cudaStream_t s = nullptr;
      cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
      streams_.push_back(s);
    }
  } catch (...) {
    release();
    throw;
  }
  ch.barrier();
}

InPlaceExecutor::~InPlaceExecutor() { release(); }

void InPlaceExecutor::release() {
  for (void* s : streams_) cudaStreamDestroy(static_cast<cudaStream_t>(s));
  streams_.clear();
  phases_.clear();
  for (ew_shardmap* m : maps_) ew_shardmap_free(m);
  maps_.clear();
  if (barrier_ != nullptr) ew_peer_barrier_free(barrier_);
  barrier_ = nullptr;
  peers_.close();
  for (void* p : staging_) dfree(p);
  staging_.clear();
  dfree(flags_);
  flags_ = nullptr;
}

void InPlaceExecutor::launch(ew_stream_t stream, std::uint64_t* block_sums) {
  if (barrier_ == nullptr) return;  // not a member of the target layout
  const int ng = std::max(1, opt_.gather_streams);
  cudaStream_t main = reinterpret_cast<cudaStream_t>(stream);
  std::vector<cudaStream_t> gs = {main};
  for (int k = 0; k < ng - 1; ++k) gs.push_back(static_cast<cudaStream_t>(streams_[k]));
  cudaStream_t ys = static_cast<cudaStream_t>(streams_[ng - 1]);
  cudaStream_t fs = static_cast<cudaStream_t>(streams_[ng]);
  std::vector<cudaEvent_t> events;
  auto event = [&](cudaStream_t s) {
    cudaEvent_t e = nullptr;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
    events.push_back(e);
    return e;
  };
  const cudaEvent_t start = event(main);
  for (std::size_t k = 1; k < gs.size(); ++k) cudaStreamWaitEvent(gs[k], start, 0);
  cudaStreamWaitEvent(ys, start, 0);
  cudaStreamWaitEvent(fs, start, 0);
  const int* veto = nullptr;
  check(ew_peer_barrier_error_flag(barrier_, &veto));
  std::vector<cudaEvent_t> bar;
  std::vector<cudaEvent_t> flushed;
  const int slack = sched_.slack, ring = sched_.ring;
  for (std::size_t j = 0; j < phases_.size(); ++j) {
    cudaStream_t g = gs[j % gs.size()];
    const long k = static_cast<long>(j) - slack - 1;
    if (k >= 0) cudaStreamWaitEvent(g, bar[static_cast<std::size_t>(k)], 0);  // all read R_k
    if (static_cast<long>(j) >= ring && flushed[j - ring] != nullptr)
      cudaStreamWaitEvent(g, flushed[j - ring], 0);  // staging buffer free again
    const Phase& ph = *phases_[j];
    if (ph.staged) check(ew_copy_program_launch_guarded(ph.staged, 0, 0, block_sums, veto, g));
    if (ph.direct) check(ew_copy_program_launch_guarded(ph.direct, 0, 0, block_sums, veto, g));
    cudaStreamWaitEvent(ys, event(g), 0);
    check(ew_peer_barrier_wait(barrier_, opt_.barrier_timeout_s, ys));  // all read R_j
    bar.push_back(event(ys));
    if (ph.flush) {
      cudaStreamWaitEvent(fs, bar.back(), 0);
      check(ew_copy_program_launch_guarded(ph.flush, opt_.flush_ctas, 0, nullptr, veto, fs));
      flushed.push_back(event(fs));
    } else {
      flushed.push_back(nullptr);
    }
  }
  for (std::size_t k = 1; k < gs.size(); ++k) cudaStreamWaitEvent(main, event(gs[k]), 0);
  cudaStreamWaitEvent(main, event(ys), 0);
  cudaStreamWaitEvent(main, event(fs), 0);
  for (cudaEvent_t e : events) cudaEventDestroy(e);  // released once their waits resolve
}

bool InPlaceExecutor::timed_out() const {
  if (barrier_ == nullptr) return false;
  int t = 0;
  check(ew_peer_barrier_timed_out(barrier_, &t));
  return t != 0;
}

}  // namespace elaskit::b200
