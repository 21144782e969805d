// Runtime services of libelaskit_b200: error state, device memory, CUDA IPC
// peer mappings (the B200 "links" of the dynamic communicator) and the NCCL
// communicator used by the weighted reduce (d).
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "kernels/ew_device.cuh"

namespace ew {

namespace {
thread_local std::string g_last_error;
}

int set_error(int status, const std::string& msg) {
  g_last_error = msg;
  return status;
}

int cuda_status(cudaError_t e, const char* what) {
  return set_error(EW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                                    cudaGetErrorString(e) + ")");
}

__global__ void write_u64_kernel(volatile unsigned long long* p, unsigned long long v) {
  __threadfence_system();  // the stream's earlier writes (a D2H image) come first
  *p = v;
  __threadfence_system();
}

int num_sms() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    n = 148;
  cache[dev] = n;
  return n;
}

}  // namespace ew

using namespace ew;

namespace {

int nccl_status(ncclResult_t r, const char* what) {
  return set_error(EW_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

#define EW_NCCL_TRY(expr)                                 \
  do {                                                    \
    ncclResult_t _r = (expr);                             \
    if (_r != ncclSuccess) return nccl_status(_r, #expr); \
  } while (0)

struct IpcMapping {
  void* base = nullptr;
  int refs = 0;
};
std::mutex g_ipc_mu;
std::map<std::string, IpcMapping> g_ipc_by_handle;  // handle bytes -> mapping
// returned ptr -> (handle bytes, opens of this ptr): one mapping can be
// opened several times (same or different offsets); every open is closed once
std::map<void*, std::pair<std::string, int>> g_ipc_by_ptr;

}  // namespace

struct ew_comm {
  ncclComm_t nccl = nullptr;
  int rank = -1;
  int nranks = 0;
};

extern "C" {

const char* ew_last_error(void) { return g_last_error.c_str(); }
const char* ew_version(void) { return "elaskit-b200 0.1 (sm_100a)"; }

int ew_device_count(int* n) {
  if (n == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  *n = 0;
  const cudaError_t e = cudaGetDeviceCount(n);
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver) {
    *n = 0;
    cudaGetLastError();
    return EW_OK;
  }
  EW_CUDA_TRY(e);
  return EW_OK;
}

int ew_set_device(int device) {
  EW_CUDA_TRY(cudaSetDevice(device));
  return EW_OK;
}

int ew_peer_access_enable(int peer_device) {
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free error state
    return EW_OK;
  }
  EW_CUDA_TRY(e);
  return EW_OK;
}

int ew_alloc(int64_t bytes, void** out) {
  if (out == nullptr || bytes < 0) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_alloc: bad arguments");
  *out = nullptr;
  if (bytes == 0) return EW_OK;
  EW_CUDA_TRY(cudaMalloc(out, static_cast<size_t>(bytes)));
  return EW_OK;
}

int ew_free(void* ptr) {
  if (ptr == nullptr) return EW_OK;
  EW_CUDA_TRY(cudaFree(ptr));
  return EW_OK;
}

int ew_memset_async(void* ptr, int value, int64_t bytes, ew_stream_t stream) {
  if (bytes == 0) return EW_OK;
  EW_CUDA_TRY(cudaMemsetAsync(ptr, value, static_cast<size_t>(bytes), (cudaStream_t)stream));
  return EW_OK;
}

int ew_memcpy_async(void* dst, const void* src, int64_t bytes, ew_stream_t stream) {
  if (bytes == 0) return EW_OK;
  EW_CUDA_TRY(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDefault,
                              (cudaStream_t)stream));
  return EW_OK;
}

int ew_stream_sync(ew_stream_t stream) {
  EW_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  return EW_OK;
}

int ew_device_sync(void) {
  EW_CUDA_TRY(cudaDeviceSynchronize());
  return EW_OK;
}

int ew_ipc_get_handle(const void* ptr, void* handle64, int64_t* offset) {
  if (ptr == nullptr || handle64 == nullptr || offset == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_ipc_get_handle: NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle is 64 bytes");
  cudaIpcMemHandle_t h;
  EW_CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(ptr)));
  // the handle names the whole allocation (e.g. a caching-allocator segment):
  // find its base through the driver's cuMemGetAddressRange
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = nullptr;
  if (get_range == nullptr) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    EW_CUDA_TRY(cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &fn, 12000,
                                                 cudaEnableDefault, &q));
    if (fn == nullptr || q != cudaDriverEntryPointSuccess)
      return set_error(EW_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    get_range = reinterpret_cast<GetRange>(fn);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, static_cast<unsigned long long>(reinterpret_cast<uintptr_t>(ptr))) != 0)
    return set_error(EW_ERR_CUDA, "cuMemGetAddressRange failed");
  std::memcpy(handle64, &h, 64);
  *offset = static_cast<int64_t>(reinterpret_cast<uintptr_t>(ptr) - base);
  return EW_OK;
}

int ew_ipc_open(const void* handle64, int64_t offset, void** out) {
  if (handle64 == nullptr || out == nullptr || offset < 0)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_ipc_open: bad arguments");
  const std::string key(static_cast<const char*>(handle64), 64);
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  IpcMapping& m = g_ipc_by_handle[key];
  if (m.refs == 0) {
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    const cudaError_t e = cudaIpcOpenMemHandle(&m.base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      g_ipc_by_handle.erase(key);
      return cuda_status(e, "cudaIpcOpenMemHandle");
    }
  }
  ++m.refs;
  void* p = static_cast<char*>(m.base) + offset;
  auto& slot = g_ipc_by_ptr[p];
  slot.first = key;
  ++slot.second;
  *out = p;
  return EW_OK;
}

int ew_ipc_close(void* ptr) {
  std::lock_guard<std::mutex> lock(g_ipc_mu);
  const auto it = g_ipc_by_ptr.find(ptr);
  if (it == g_ipc_by_ptr.end()) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_ipc_close: unknown pointer");
  const std::string key = it->second.first;
  if (--it->second.second == 0) g_ipc_by_ptr.erase(it);
  IpcMapping& m = g_ipc_by_handle[key];
  if (--m.refs == 0) {
    const cudaError_t e = cudaIpcCloseMemHandle(m.base);
    g_ipc_by_handle.erase(key);
    EW_CUDA_TRY(e);
  }
  return EW_OK;
}

int ew_host_register(void* host, int64_t bytes, void** dev_ptr) {
  if (host == nullptr || bytes <= 0 || dev_ptr == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_host_register: bad arguments");
  EW_CUDA_TRY(cudaHostRegister(host, static_cast<size_t>(bytes),
                               cudaHostRegisterPortable | cudaHostRegisterMapped));
  const cudaError_t e = cudaHostGetDevicePointer(dev_ptr, host, 0);
  if (e != cudaSuccess) {
    cudaHostUnregister(host);
    return cuda_status(e, "cudaHostGetDevicePointer");
  }
  return EW_OK;
}

int ew_write_u64_async(void* dev_ptr, uint64_t value, ew_stream_t stream) {
  if (dev_ptr == nullptr || (reinterpret_cast<uintptr_t>(dev_ptr) & 7))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_write_u64_async: NULL or unaligned");
  ew::write_u64_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(
      static_cast<volatile unsigned long long*>(dev_ptr), value);
  EW_CUDA_TRY(cudaGetLastError());
  return EW_OK;
}

int ew_host_unregister(void* host) {
  if (host == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "ew_host_unregister: NULL");
  EW_CUDA_TRY(cudaHostUnregister(host));
  return EW_OK;
}

// ---- NCCL communicator ----

int ew_comm_unique_id(void* id128) {
  if (id128 == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  EW_NCCL_TRY(ncclGetUniqueId(&id));
  std::memcpy(id128, &id, 128);
  return EW_OK;
}

int ew_comm_init(const void* id128, int nranks, int rank, ew_comm** out) {
  if (id128 == nullptr || out == nullptr || nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_comm_init: bad arguments");
  ncclUniqueId id;
  std::memcpy(&id, id128, 128);
  auto* c = new ew_comm();
  const ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_status(r, "ncclCommInitRank");
  }
  c->rank = rank;
  c->nranks = nranks;
  *out = c;
  return EW_OK;
}

int ew_comm_shrink(ew_comm* parent, const int* exclude_ranks, int n_exclude, int abort,
                   ew_comm** out) {
  if (parent == nullptr || out == nullptr || n_exclude < 0 || (n_exclude > 0 && !exclude_ranks))
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_comm_shrink: bad arguments");
  *out = nullptr;
  auto* c = new ew_comm();
  // A planned departure reuses the parent's buffers and connections
  // (shrinkShare), so only the membership edit is paid; after a crash
  // (abort) nothing of the parent can be trusted and it is rebuilt.
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.shrinkShare = abort ? 0 : 1;
  const ncclResult_t r =
      ncclCommShrink(parent->nccl, const_cast<int*>(exclude_ranks), n_exclude, &c->nccl, &cfg,
                     abort ? NCCL_SHRINK_ABORT : NCCL_SHRINK_DEFAULT);
  if (r != ncclSuccess) {
    delete c;
    return nccl_status(r, "ncclCommShrink");
  }
  if (c->nccl == nullptr) {  // this rank was excluded
    delete c;
    return EW_OK;
  }
  ncclCommUserRank(c->nccl, &c->rank);
  ncclCommCount(c->nccl, &c->nranks);
  *out = c;
  return EW_OK;
}

int ew_comm_split(ew_comm* parent, int color, int key, int share, ew_comm** out) {
  if (parent == nullptr || out == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_comm_split: bad arguments");
  *out = nullptr;
  auto* c = new ew_comm();
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.splitShare = share ? 1 : 0;
  const ncclResult_t r =
      ncclCommSplit(parent->nccl, color < 0 ? NCCL_SPLIT_NOCOLOR : color, key, &c->nccl, &cfg);
  if (r != ncclSuccess) {
    delete c;
    return nccl_status(r, "ncclCommSplit");
  }
  if (c->nccl == nullptr) {  // NCCL_SPLIT_NOCOLOR: not a member of any child
    delete c;
    return EW_OK;
  }
  ncclCommUserRank(c->nccl, &c->rank);
  ncclCommCount(c->nccl, &c->nranks);
  *out = c;
  return EW_OK;
}

int ew_comm_abort(ew_comm* comm) {
  if (comm == nullptr) return EW_OK;
  const ncclResult_t r = ncclCommAbort(comm->nccl);
  delete comm;
  if (r != ncclSuccess) return nccl_status(r, "ncclCommAbort");
  return EW_OK;
}

int ew_comm_rank(const ew_comm* comm, int* rank, int* nranks) {
  if (comm == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL comm");
  if (rank) *rank = comm->rank;
  if (nranks) *nranks = comm->nranks;
  return EW_OK;
}

int ew_comm_destroy(ew_comm* comm) {
  if (comm == nullptr) return EW_OK;
  const ncclResult_t r = ncclCommDestroy(comm->nccl);
  delete comm;
  EW_NCCL_TRY(r);
  return EW_OK;
}

int ew_allreduce_i64(ew_comm* comm, int64_t* buf, int64_t n, ew_stream_t stream) {
  if (comm == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL comm");
  EW_NCCL_TRY(ncclAllReduce(buf, buf, static_cast<size_t>(n), ncclInt64, ncclSum, comm->nccl,
                            (cudaStream_t)stream));
  return EW_OK;
}

int ew_allreduce_u64(ew_comm* comm, uint64_t* buf, int64_t n, ew_stream_t stream) {
  if (comm == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL comm");
  EW_NCCL_TRY(ncclAllReduce(buf, buf, static_cast<size_t>(n), ncclUint64, ncclSum, comm->nccl,
                            (cudaStream_t)stream));
  return EW_OK;
}

int ew_allreduce_max_f64(ew_comm* comm, double* buf, int64_t n, ew_stream_t stream) {
  if (comm == nullptr) return set_error(EW_ERR_INVALID_ARGUMENT, "NULL comm");
  EW_NCCL_TRY(ncclAllReduce(buf, buf, static_cast<size_t>(n), ncclFloat64, ncclMax, comm->nccl,
                            (cudaStream_t)stream));
  return EW_OK;
}

int ew_weighted_reduce(ew_comm* comm, const float* const* units, const double* weights,
                       int n_units, int64_t total_units, int64_t n_elems, int64_t* ws_acc,
                       double* ws_max, float* out, int* frac_bits_out, ew_stream_t stream) {
  if (comm == nullptr || ws_acc == nullptr || ws_max == nullptr || out == nullptr ||
      frac_bits_out == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_weighted_reduce: NULL argument");
  if (int st = ew_weighted_absmax(units, weights, n_units, n_elems, ws_max, stream)) return st;
  if (int st = ew_allreduce_max_f64(comm, ws_max, 1, stream)) return st;
  double gmax = 0.0;
  EW_CUDA_TRY(cudaMemcpyAsync(&gmax, ws_max, sizeof(double), cudaMemcpyDeviceToHost,
                              (cudaStream_t)stream));
  EW_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
  int f = 0;
  if (int st = ew_fixed_point_bits(gmax, total_units, &f)) return st;
  if (int st = ew_weighted_fold(units, weights, n_units, n_elems, f, ws_acc, 0, stream)) return st;
  if (int st = ew_allreduce_i64(comm, ws_acc, n_elems, stream)) return st;
  if (int st = ew_fixed_to_float(ws_acc, n_elems, f, out, stream)) return st;
  *frac_bits_out = f;
  return EW_OK;
}

int ew_weighted_reduce_async(ew_comm* comm, const float* const* units, const double* weights,
                             int n_units, int64_t total_units, int64_t n_elems, int64_t* ws_acc,
                             double* ws_max, int* ws_bits, float* out, ew_stream_t stream) {
  if (comm == nullptr || ws_acc == nullptr || ws_max == nullptr || ws_bits == nullptr ||
      out == nullptr)
    return set_error(EW_ERR_INVALID_ARGUMENT, "ew_weighted_reduce_async: NULL argument");
  // every step stream-ordered on the device: no host round trip, capturable
  // in a CUDA graph together with the collectives
  if (int st = ew_weighted_absmax(units, weights, n_units, n_elems, ws_max, stream)) return st;
  if (int st = ew_allreduce_max_f64(comm, ws_max, 1, stream)) return st;
  if (int st = ew_fixed_point_bits_async(ws_max, total_units, ws_bits, stream)) return st;
  if (int st = ew_weighted_fold_dev(units, weights, n_units, n_elems, ws_bits, ws_acc, 0, nullptr,
                                    stream))
    return st;
  if (int st = ew_allreduce_i64(comm, ws_acc, n_elems, stream)) return st;
  return ew_fixed_to_float_dev(ws_acc, n_elems, ws_bits, out, stream);
}

}  // extern "C"
