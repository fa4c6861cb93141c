// dist.cpp -- row-sharded multi-GPU sgemm (one process per GPU).
//
// The paper's distributed model: data distributed by rows,
// each rank runs its own block (distribute(i); rank conditional
// q = get_rank()), communication is explicit
// (send/receive) and C is never gathered.
// For gemm the only exchange is B: NCCL broadcast from the root over
// NVLink/NVSwitch, in K-chunks on a dedicated comm stream; the GEMM of chunk c
// (beta_c = beta for c = 0, else 1) runs on the caller's stream as soon as
// chunk c has arrived, so chunk c+1 streams while chunk c computes.
//
// NCCL is loaded with dlopen (the same libnccl.so.2 torch uses), so the
// single-GPU library has no link-time NCCL dependency.
//
// SM sharing: the GEMM is a persistent kernel that would occupy every SM (and
// all registers) for the whole chunk, so a concurrently enqueued NCCL kernel
// could not start until it finished -- no overlap.  The communicator is created
// with maxCTAs = kCommCtas and the chunk GEMMs leave kCommCtas SMs free.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <chrono>
#include <thread>
#include <vector>

#include "tm_internal.h"

namespace {

// Minimal NCCL ABI (stable since NCCL 2.x; matches nccl.h).
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclFloat32 = 7 } ncclDataType_t;
// ncclConfig_t as of NCCL 2.28 (nccl.h ncclConfig_v22800); the size/version
// fields let older/newer libraries interpret it.
struct NcclConfig {
  size_t size;
  unsigned int magic;
  unsigned int version;
  int blocking, cgaClusterSize, minCTAs, maxCTAs;
  const char* netName;
  int splitShare, trafficClass;
  const char* commName;
  int collnetEnable, CTAPolicy, shrinkShare, nvlsCTAs, nChannelsPerNetPeer, nvlinkCentricSched;
};
constexpr int kNcclUndefInt = static_cast<int>(0x80000000);
constexpr int kCommCtasDefault = 16;

int comm_ctas() {
  static const int v = [] {
    const char* e = std::getenv("TM_DIST_COMM_SMS");  // tuning knob (bench only)
    return e ? std::max(0, std::atoi(e)) : kCommCtasDefault;
  }();
  return v;
}

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, NcclConfig*) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  // point-to-point (the blur's border-row exchange)
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, NcclConfig*) = nullptr;
  bool ok = false;
};

Nccl g_nccl;
std::once_flag g_nccl_once;

void load_nccl() {
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    const char* p = std::getenv("TM_NCCL_PATH");
    if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) return;
  g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
  g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
  g_nccl.CommInitRankConfig =
      reinterpret_cast<decltype(g_nccl.CommInitRankConfig)>(dlsym(h, "ncclCommInitRankConfig"));
  g_nccl.GetVersion = reinterpret_cast<decltype(g_nccl.GetVersion)>(dlsym(h, "ncclGetVersion"));
  g_nccl.CommGetAsyncError =
      reinterpret_cast<decltype(g_nccl.CommGetAsyncError)>(dlsym(h, "ncclCommGetAsyncError"));
  g_nccl.CommAbort = reinterpret_cast<decltype(g_nccl.CommAbort)>(dlsym(h, "ncclCommAbort"));
  g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
  g_nccl.Broadcast = reinterpret_cast<decltype(g_nccl.Broadcast)>(dlsym(h, "ncclBroadcast"));
  g_nccl.AllGather = reinterpret_cast<decltype(g_nccl.AllGather)>(dlsym(h, "ncclAllGather"));
  g_nccl.Send = reinterpret_cast<decltype(g_nccl.Send)>(dlsym(h, "ncclSend"));
  g_nccl.Recv = reinterpret_cast<decltype(g_nccl.Recv)>(dlsym(h, "ncclRecv"));
  g_nccl.GroupStart = reinterpret_cast<decltype(g_nccl.GroupStart)>(dlsym(h, "ncclGroupStart"));
  g_nccl.GroupEnd = reinterpret_cast<decltype(g_nccl.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
  g_nccl.CommSplit = reinterpret_cast<decltype(g_nccl.CommSplit)>(dlsym(h, "ncclCommSplit"));
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.Broadcast && g_nccl.AllGather;
}

bool nccl() {
  std::call_once(g_nccl_once, load_nccl);
  return g_nccl.ok;
}

constexpr int kMaxChunks = 16;

tm_status set_flag(cudaStream_t s, unsigned* flag, unsigned value) { return tmk::stream_write_u32(s, flag, value); }

// Loopback link model (projections, TM_LOOPBACK_LINK_GBS = R GB/s): a
// rank's transfer stream starts a clock before its first chunk and, after
// chunk c (its device copy in modes 0-2), blocks until
//   t0 + (chain_pos * piece_bytes + bytes of chunks 0..c) / R,
// so chunk c arrives no earlier than a pipelined chain (or ring) of links of
// rate R delivers it to the rank at position chain_pos.  The clock and the
// waits are host functions on the transfer stream (cudaLaunchHostFunc): they
// hold the stream without occupying an SM, so the GEMMs keep theirs.
struct LinkClock {
  std::chrono::steady_clock::time_point t0;
};
struct LinkWait {
  LinkClock* clock;
  double ns;
};
void CUDART_CB link_start(void* p) { static_cast<LinkClock*>(p)->t0 = std::chrono::steady_clock::now(); }
void CUDART_CB link_until(void* p) {
  const LinkWait* w = static_cast<const LinkWait*>(p);
  std::this_thread::sleep_until(w->clock->t0 + std::chrono::nanoseconds(static_cast<long long>(w->ns)));
}
// SMs the loopback's GEMMs leave free.  NCCL model (modes 0-2): as many as
// the NCCL schedule leaves to NCCL's kernels -- the loopback's same-device
// copies are kernels too (scripts/r02/ce_probe.cu: a 256 MiB device-to-device
// copy waits 3 ms behind a kernel that holds every SM's thread slots).
// Copy-engine model (modes 3, 4): none; the chunks are not copied at all
// (peer-to-peer copies between devices run on the copy engines, which one
// device cannot emulate), only released on the link model's schedule.
int loopback_reserve(int mode) {
  if (mode >= 3) return 0;
  static const int v = [] {
    const char* e = std::getenv("TM_LOOPBACK_RESERVE");
    return e ? std::max(1, std::atoi(e)) : comm_ctas();
  }();
  return v;
}
double loopback_link_gbs(int mode) {
  const char* e = std::getenv("TM_LOOPBACK_LINK_GBS");
  const double v = e ? std::atof(e) : 0.0;
  return mode >= 3 && v <= 0.0 ? 700.0 : v;
}

}  // namespace

namespace tmk {

// Stream memory operations through the runtime's driver entry-point query (no
// link-time libcuda dependency): no kernel, no SM; ordered in the stream like
// any other operation (the write after all earlier work, with a memory barrier).
namespace {
template <class Fn>
Fn driver_fn(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
    return reinterpret_cast<Fn>(p);
  return nullptr;
}
using WriteValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WaitValue32Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using AddressRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
}  // namespace

tm_status stream_write_u32(cudaStream_t s, unsigned* flag, unsigned value) {
  static const WriteValue32Fn fn = driver_fn<WriteValue32Fn>("cuStreamWriteValue32");
  if (!fn) return TM_ERR_CUDA;
  return fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value, 0) == CUDA_SUCCESS
             ? TM_OK
             : TM_ERR_CUDA;
}

tm_status stream_wait_u32(cudaStream_t s, const unsigned* flag, unsigned value) {
  static const WaitValue32Fn fn = driver_fn<WaitValue32Fn>("cuStreamWaitValue32");
  if (!fn) return TM_ERR_CUDA;
  // CU_STREAM_WAIT_VALUE_GEQ (0): until (int32)(*flag - value) >= 0 -- epochs wrap safely
  return fn(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), value, 0) == CUDA_SUCCESS
             ? TM_OK
             : TM_ERR_CUDA;
}

tm_status device_allocation(const void* p, void** base, size_t* bytes) {
  static const AddressRangeFn fn = driver_fn<AddressRangeFn>("cuMemGetAddressRange");
  if (!fn) return TM_ERR_CUDA;
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS) return TM_ERR_INVALID_VALUE;
  *base = reinterpret_cast<void*>(b);
  if (bytes) *bytes = sz;
  return TM_OK;
}

int dist_comm_ctas() { return comm_ctas(); }

}  // namespace tmk

struct tm_comm_s {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_start = nullptr;
  cudaEvent_t ev_chunk[kMaxChunks] = {};
  uint64_t bytes_received = 0;
  unsigned* chunk_flags = nullptr;  // [kMaxChunks] device arrival flags (fused mode)
  unsigned epoch = 0;               // fused-mode call counter (the flag value of this call)
  // SUMMA (tm_sgemm_summa): row / column communicators of the last grid,
  // double-buffered panel buffers, their events
  int summa_pr = 0, summa_pc = 0;
  ncclComm_t row_comm = nullptr, col_comm = nullptr;
  float* panel_buf = nullptr;
  size_t panel_bytes = 0;
  cudaEvent_t ev_ready[2] = {}, ev_used[2] = {};
};

extern "C" {

tm_status tm_dist_rows(int64_t m, int nranks, int rank, int64_t* row0, int64_t* rows) {
  if (m < 0 || nranks < 1 || rank < 0 || rank >= nranks || !row0 || !rows) return TM_ERR_INVALID_VALUE;
  const int64_t q = m / nranks, r = m % nranks;
  *rows = q + (rank < r ? 1 : 0);
  *row0 = static_cast<int64_t>(rank) * q + (rank < r ? rank : r);
  return TM_OK;
}

tm_status tm_comm_get_unique_id(tm_unique_id* out) {
  if (!out) return TM_ERR_INVALID_VALUE;
  if (!nccl()) return TM_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == sizeof(tm_unique_id), "unique id size");
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return TM_ERR_NCCL;
  std::memcpy(out->bytes, id.internal, sizeof(id));
  return TM_OK;
}

tm_status tm_comm_init(tm_comm_t* out, int nranks, int rank, const tm_unique_id* id) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return TM_ERR_INVALID_VALUE;
  if (!nccl()) return TM_ERR_NCCL;
  tm_comm_s* c = new (std::nothrow) tm_comm_s;
  if (!c) return TM_ERR_OUT_OF_MEMORY;
  c->rank = rank;
  c->nranks = nranks;
  if (cudaGetDevice(&c->device) != cudaSuccess) { delete c; return TM_ERR_CUDA; }
  ncclUniqueId nid;
  std::memcpy(nid.internal, id->bytes, sizeof(nid));
  int ver = 0;
  if (g_nccl.GetVersion) g_nccl.GetVersion(&ver);
  ncclResult_t r;
  if (g_nccl.CommInitRankConfig && ver >= 22800 && comm_ctas() > 0) {
    NcclConfig cfg = {sizeof(NcclConfig), 0xcafebeef, static_cast<unsigned>(ver),
                      kNcclUndefInt, kNcclUndefInt, kNcclUndefInt, kNcclUndefInt, nullptr, kNcclUndefInt,
                      kNcclUndefInt, nullptr, kNcclUndefInt, kNcclUndefInt, kNcclUndefInt, kNcclUndefInt,
                      kNcclUndefInt, kNcclUndefInt};
    cfg.maxCTAs = comm_ctas();
    cfg.minCTAs = std::min(comm_ctas(), 4);
    r = g_nccl.CommInitRankConfig(&c->comm, nranks, nid, rank, &cfg);
  } else {
    r = g_nccl.CommInitRank(&c->comm, nranks, nid, rank);
  }
  if (r != ncclSuccess) { delete c; return TM_ERR_NCCL; }
  bool ok = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; ok && i < kMaxChunks; ++i)
    ok = cudaEventCreateWithFlags(&c->ev_chunk[i], cudaEventDisableTiming) == cudaSuccess;
  ok = ok && cudaMalloc(&c->chunk_flags, kMaxChunks * sizeof(unsigned)) == cudaSuccess &&
       cudaMemset(c->chunk_flags, 0, kMaxChunks * sizeof(unsigned)) == cudaSuccess;
  if (!ok) {
    tm_comm_destroy(c);
    return TM_ERR_CUDA;
  }
  *out = c;
  return TM_OK;
}

tm_status tm_comm_destroy(tm_comm_t c) {
  if (!c) return TM_ERR_INVALID_VALUE;
  tm_status st = TM_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm && g_nccl.CommDestroy(c->comm) != ncclSuccess) st = TM_ERR_NCCL;  // null after an abort
  for (int i = 0; i < kMaxChunks; ++i)
    if (c->ev_chunk[i]) cudaEventDestroy(c->ev_chunk[i]);
  if (c->ev_start) cudaEventDestroy(c->ev_start);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->chunk_flags) cudaFree(c->chunk_flags);
  if (c->row_comm) g_nccl.CommDestroy(c->row_comm);
  if (c->col_comm) g_nccl.CommDestroy(c->col_comm);
  if (c->panel_buf) cudaFree(c->panel_buf);
  for (int i = 0; i < 2; ++i) {
    if (c->ev_ready[i]) cudaEventDestroy(c->ev_ready[i]);
    if (c->ev_used[i]) cudaEventDestroy(c->ev_used[i]);
  }
  delete c;
  return st;
}

tm_status tm_comm_rank(tm_comm_t c, int* rank, int* nranks) {
  if (!c || !rank || !nranks) return TM_ERR_INVALID_VALUE;
  *rank = c->rank;
  *nranks = c->nranks;
  return TM_OK;
}

tm_status tm_comm_check(tm_comm_t c, int abort_on_error) {
  if (!c || !c->comm) return TM_ERR_INVALID_VALUE;
  if (!g_nccl.CommGetAsyncError) return TM_OK;
  ncclResult_t async = ncclSuccess;
  if (g_nccl.CommGetAsyncError(c->comm, &async) != ncclSuccess) return TM_ERR_NCCL;
  if (async == ncclSuccess || static_cast<int>(async) == 7 /* ncclInProgress */) return TM_OK;
  if (abort_on_error && g_nccl.CommAbort) {
    g_nccl.CommAbort(c->comm);
    c->comm = nullptr;
  }
  return TM_ERR_NCCL;
}

tm_status tm_comm_bytes_received(tm_comm_t c, uint64_t* bytes) {
  if (!c || !bytes) return TM_ERR_INVALID_VALUE;
  *bytes = c->bytes_received;
  return TM_OK;
}

static int choose_chunks(int64_t k, int nranks) {
  if (nranks <= 1) return 1;
  // Uniform chunks (the fused schedule's flag granularity): at least 512
  // K-rows; at most 8.
  int64_t c = k / 512;
  if (c > 8) c = 8;
  if (c < 1) c = 1;
  return static_cast<int>(c);
}

// Uniform plan: nch chunks of kc rows (multiple of 32), the last ragged.
static int uniform_plan(int64_t k, int nranks, int64_t* bounds) {
  const int nch = choose_chunks(k, nranks);
  const int64_t kc = ((k + nch - 1) / nch + 31) / 32 * 32;
  int n = 0;
  bounds[0] = 0;
  for (int64_t k0 = 0; k0 < k; k0 += kc) bounds[++n] = std::min(k, k0 + kc);
  return n;
}

// The chunked schedule's K-chunks: geometric, each twice the previous,
// starting at max(512, k/32) rows (multiples of 32); a remainder of at most
// half the last chunk is merged into it, a larger one becomes its own chunk.
// Rationale: chunk 0 is the exposed transfer, so it is
// small; chunk c+1 arrives while chunk c's GEMM runs as long as the link moves
// a K-row faster than the GEMM consumes it divided by the growth factor (at
// 16384^3 / P = 8: 0.26 us of GEMM vs 0.09 us of NVLink per K-row, margin
// 1.4x), and every chunk boundary costs a launch tail and a round trip of C,
// so few, growing chunks beat many uniform ones.  TM_DIST_CHUNKS=uniform
// selects the uniform plan (measurement knob).
static int chunk_plan(int64_t k, int nranks, int64_t* bounds) {
  bounds[0] = 0;
  if (k <= 0) return 0;
  if (nranks <= 1) {
    bounds[1] = k;
    return 1;
  }
  static const bool uniform = [] {
    const char* e = std::getenv("TM_DIST_CHUNKS");
    return e && std::strcmp(e, "uniform") == 0;
  }();
  if (uniform) return uniform_plan(k, nranks, bounds);
  int64_t s = std::max<int64_t>(512, (k / 32 + 31) / 32 * 32);
  int n = 0;
  int64_t sum = 0;
  while (n < kMaxChunks && sum + s <= k) {
    sum += s;
    bounds[++n] = sum;
    s *= 2;
  }
  const int64_t rest = k - sum;
  if (n == 0) {
    bounds[++n] = k;
  } else if (rest > 0) {
    const int64_t last = bounds[n] - bounds[n - 1];
    if (rest * 2 > last && n < kMaxChunks) bounds[++n] = k;
    else bounds[n] = k;
  }
  return n;
}

tm_status tm_dist_chunk(int64_t k, int nranks, int idx, int64_t* k0, int64_t* kr) {
  if (k < 0 || nranks < 1 || !k0 || !kr) return TM_ERR_INVALID_VALUE;
  int64_t bounds[kMaxChunks + 1];
  const int count = chunk_plan(k, nranks, bounds);
  if (idx < 0) {
    *k0 = count;
    *kr = count ? bounds[count] - bounds[count - 1] : 0;  // the largest (last) chunk
    return TM_OK;
  }
  if (idx >= count) return TM_ERR_INVALID_VALUE;
  *k0 = bounds[idx];
  *kr = bounds[idx + 1] - bounds[idx];
  return TM_OK;
}

}  // extern "C"

namespace {

// Whether the GEMM of chunk c is expected to run while later chunks are still
// being transferred, i.e. needs SMs left free for the broadcast kernels.  Model:
// chunk c's GEMM starts when chunk 0 has arrived plus c chunk-GEMM times;
// the broadcast ends after all chunks at the link rate.  Chunk GEMMs past that
// point get every SM (the 16 reserved SMs are ~11% of the machine).  If the
// estimate is optimistic the only cost is a broadcast kernel waiting for SMs
// (no GEMM ever waits inside a kernel on the broadcast).  Rates: NVLink ~700
// GB/s per rank, 3xTF32 GEMM ~240 TFLOP/s (measured C5; TM_DIST_LINK_GBS and
// TM_DIST_GEMM_TFLOPS override them).
bool chunk_overlaps_transfer(const int64_t* bounds, int c, int nchunks, int64_t rows, int64_t n, int64_t ldb) {
  static const double link = [] { const char* e = std::getenv("TM_DIST_LINK_GBS"); return e ? std::atof(e) : 700.0; }();
  static const double gemm = [] { const char* e = std::getenv("TM_DIST_GEMM_TFLOPS"); return e ? std::atof(e) : 240.0; }();
  if (link <= 0.0 || gemm <= 0.0) return true;
  const double per_row_xfer = 4.0 * static_cast<double>(ldb) / (link * 1e9);
  const double per_row_gemm = 2.0 * static_cast<double>(rows) * static_cast<double>(n) / (gemm * 1e12);
  // chunk c's GEMM starts after chunk 0 arrived and chunks 0..c-1 computed;
  // the broadcast ends after all of B crossed the link
  const double start = static_cast<double>(bounds[1]) * per_row_xfer + static_cast<double>(bounds[c]) * per_row_gemm;
  return start < static_cast<double>(bounds[nchunks]) * per_row_xfer;
}

// The per-rank schedule of the row-sharded GEMM, shared by the NCCL mode and
// the single-process loopback mode.  `xfer(p, count)` enqueues the transfer of
// `count` floats of B at `p` from the root on `comm_stream` (ncclBroadcast, or
// a device copy in loopback); the GEMM of chunk c waits only for chunk c.
template <class Xfer>
tm_status dist_schedule(int nranks, int rank, int root, int64_t m, int64_t n, int64_t k, float alpha,
                        const float* A_local, int64_t lda, float* B, int64_t ldb, float beta, float* C_local,
                        int64_t ldc, cudaStream_t stream, cudaStream_t comm_stream, cudaEvent_t ev_start,
                        cudaEvent_t* ev_chunk, uint64_t* bytes_received, Xfer&& xfer, int reserve_sms = -1) {
  int64_t row0 = 0, rows = 0;
  tm_dist_rows(m, nranks, rank, &row0, &rows);
  const bool reads_ab = alpha != 0.0f && k > 0 && n > 0;
  if (!reads_ab || nranks == 1) {
    // Nothing to exchange (P == 1, or B is not read): exactly tm_sgemm.
    return tm_sgemm(rows, n, k, alpha, A_local, lda, B, ldb, beta, C_local, ldc, stream);
  }
  if (!B || ldb < (n > 1 ? n : 1)) return TM_ERR_INVALID_VALUE;
  int64_t bounds[kMaxChunks + 1];
  const int nchunks = chunk_plan(k, nranks, bounds);
  if (cudaEventRecord(ev_start, stream) != cudaSuccess) return TM_ERR_CUDA;
  if (cudaStreamWaitEvent(comm_stream, ev_start, 0) != cudaSuccess) return TM_ERR_CUDA;
  nvtxRangePushA("tm_sgemm_dist schedule");
  struct Pop {
    ~Pop() { nvtxRangePop(); }
  } pop;
  for (int c = 0; c < nchunks; ++c) {
    const int64_t k0 = bounds[c], kr = bounds[c + 1] - bounds[c];
    // Root sends in place; the last row's padding beyond n is inside k*ldb.
    const size_t count = static_cast<size_t>(kr) * static_cast<size_t>(ldb);
    tm_status st = xfer(B + k0 * ldb, count);
    if (st != TM_OK) return st;
    if (rank != root && bytes_received) *bytes_received += count * 4;
    if (cudaEventRecord(ev_chunk[c], comm_stream) != cudaSuccess) return TM_ERR_CUDA;
  }
  for (int c = 0; c < nchunks; ++c) {
    const int64_t k0 = bounds[c], kr = bounds[c + 1] - bounds[c];
    if (cudaStreamWaitEvent(stream, ev_chunk[c], 0) != cudaSuccess) return TM_ERR_CUDA;
    if (rows > 0) {
      tmk::GemmArgs ga{rows, n, kr, alpha, c == 0 ? beta : 1.0f, A_local + k0, lda, B + k0 * ldb, ldb, C_local, ldc};
      const int reserve = reserve_sms >= 0 ? reserve_sms
                          : chunk_overlaps_transfer(bounds, c, nchunks, rows, n, ldb) ? comm_ctas() : 0;
      tm_status st = tmk::sgemm_reserve(ga, stream, reserve);
      if (st != TM_OK) return st;
    }
  }
  return TM_OK;
}

// Fused single-launch schedule (SURVEY.md 8(e) "Fused alternative"): ONE
// persistent GEMM over the full K on `stream`, while B's K-chunks arrive on
// `comm_stream`; after each chunk's transfer a stream memory operation sets
// flags[c] = epoch, and the GEMM's TMA producers wait for that flag before they
// load any stage of chunk c (tc_gemm.cuh wait_chunk_flag).  Unlike the chunked
// schedule there is one launch tail instead of nchunks and C is read and
// written once (no beta chain); the cost is that the first wave of tiles is
// paced by the transfer.  The root's GEMM is not gated (its B is complete).
// Falls back to the chunked schedule when the tensor-core path cannot take the
// operands (alignment).  reserve: SMs left to the transfer kernels (NCCL); the
// copy-engine loopback transport needs none.
template <class Xfer>
tm_status dist_fused_schedule(int nranks, int rank, int root, int64_t m, int64_t n, int64_t k, float alpha,
                              const float* A_local, int64_t lda, float* B, int64_t ldb, float beta, float* C_local,
                              int64_t ldc, cudaStream_t stream, cudaStream_t comm_stream, cudaEvent_t ev_start,
                              cudaEvent_t* ev_chunk, unsigned* flags, unsigned epoch, int reserve,
                              uint64_t* bytes_received, Xfer&& xfer) {
  int64_t row0 = 0, rows = 0;
  tm_dist_rows(m, nranks, rank, &row0, &rows);
  const bool reads_ab = alpha != 0.0f && k > 0 && n > 0;
  if (!reads_ab || nranks == 1)
    return tm_sgemm(rows, n, k, alpha, A_local, lda, B, ldb, beta, C_local, ldc, stream);
  if (!B || ldb < (n > 1 ? n : 1)) return TM_ERR_INVALID_VALUE;
  tmk::GemmArgs ga{rows, n, k, alpha, beta, A_local, lda, B, ldb, C_local, ldc};
  if (rows > 0 && !tmk::tc_plan_ok(ga))
    return dist_schedule(nranks, rank, root, m, n, k, alpha, A_local, lda, B, ldb, beta, C_local, ldc, stream,
                         comm_stream, ev_start, ev_chunk, bytes_received, xfer, reserve == comm_ctas() ? -1 : reserve);
  int64_t bounds[kMaxChunks + 1];
  const int nchunks = uniform_plan(k, nranks, bounds);  // flags cover equal chunks of kc rows
  const int64_t kc = bounds[1];
  (void)nchunks;
  if (cudaEventRecord(ev_start, stream) != cudaSuccess) return TM_ERR_CUDA;
  if (cudaStreamWaitEvent(comm_stream, ev_start, 0) != cudaSuccess) return TM_ERR_CUDA;
  nvtxRangePushA("tm_sgemm_dist fused schedule");
  struct Pop {
    ~Pop() { nvtxRangePop(); }
  } pop;
  int c = 0;
  for (int64_t k0 = 0; k0 < k; k0 += kc, ++c) {
    const int64_t kr = (k0 + kc <= k) ? kc : k - k0;
    const size_t count = static_cast<size_t>(kr) * static_cast<size_t>(ldb);
    tm_status st = xfer(B + k0 * ldb, count);
    if (st != TM_OK) return st;
    if (rank != root && bytes_received) *bytes_received += count * 4;
    if ((st = set_flag(comm_stream, flags + c, epoch)) != TM_OK) return st;
  }
  if (cudaEventRecord(ev_chunk[0], comm_stream) != cudaSuccess) return TM_ERR_CUDA;
  if (rows > 0) {
    if (rank != root) {
      ga.kflags = flags;
      ga.kepoch = epoch;
      ga.kchunk = kc;
    }
    tm_status st = tmk::sgemm_reserve(ga, stream, reserve);
    if (st != TM_OK) return st;
  }
  // the call completes (stream-ordered) only when B has fully arrived
  return cudaStreamWaitEvent(stream, ev_chunk[0], 0) == cudaSuccess ? TM_OK : TM_ERR_CUDA;
}

// All-gather variant: B arrives pre-sharded by k-rows (rank r owns rows
// [r*kr, (r+1)*kr), kr = k/P).  The GEMM on the own shard needs no
// communication and runs first, overlapping the gather (`gather()` enqueues it
// on comm_stream); the other K ranges follow once it lands.
template <class Gather>
tm_status allgather_schedule(int nranks, int rank, int64_t m, int64_t n, int64_t k, float alpha, const float* A_local,
                             int64_t lda, const float* B_shard, float* B_full, int64_t ldb, float beta,
                             float* C_local, int64_t ldc, cudaStream_t stream, cudaStream_t comm_stream,
                             cudaEvent_t ev_start, cudaEvent_t ev_done, uint64_t* bytes_received, Gather&& gather) {
  if (k % nranks != 0) return TM_ERR_INVALID_VALUE;
  int64_t row0 = 0, rows = 0;
  tm_dist_rows(m, nranks, rank, &row0, &rows);
  const bool reads_ab = alpha != 0.0f && k > 0 && n > 0;
  if (!reads_ab) return tm_sgemm(rows, n, k, alpha, A_local, lda, B_full, ldb, beta, C_local, ldc, stream);
  if (!B_shard || !B_full || ldb < (n > 1 ? n : 1)) return TM_ERR_INVALID_VALUE;
  const int64_t kr = k / nranks, k0 = rank * kr;
  const int reserve = nranks > 1 ? comm_ctas() : 0;
  if (cudaEventRecord(ev_start, stream) != cudaSuccess) return TM_ERR_CUDA;
  if (cudaStreamWaitEvent(comm_stream, ev_start, 0) != cudaSuccess) return TM_ERR_CUDA;
  const size_t count = static_cast<size_t>(kr) * static_cast<size_t>(ldb);
  tm_status st = gather(count);
  if (st != TM_OK) return st;
  if (bytes_received) *bytes_received += count * 4 * static_cast<uint64_t>(nranks - 1);
  if (cudaEventRecord(ev_done, comm_stream) != cudaSuccess) return TM_ERR_CUDA;
  if (rows == 0) return cudaStreamWaitEvent(stream, ev_done, 0) == cudaSuccess ? TM_OK : TM_ERR_CUDA;
  tmk::GemmArgs own{rows, n, kr, alpha, beta, A_local + k0, lda, B_shard, ldb, C_local, ldc};
  st = tmk::sgemm_reserve(own, stream, reserve);
  if (st != TM_OK) return st;
  if (cudaStreamWaitEvent(stream, ev_done, 0) != cudaSuccess) return TM_ERR_CUDA;
  if (k0 > 0) {
    tmk::GemmArgs lo{rows, n, k0, alpha, 1.0f, A_local, lda, B_full, ldb, C_local, ldc};
    st = tmk::sgemm_reserve(lo, stream, 0);  // the gather is complete: every SM
    if (st != TM_OK) return st;
  }
  if (k0 + kr < k) {
    tmk::GemmArgs hi{rows, n, k - k0 - kr, alpha, 1.0f, A_local + k0 + kr, lda, B_full + (k0 + kr) * ldb, ldb, C_local, ldc};
    st = tmk::sgemm_reserve(hi, stream, 0);
    if (st != TM_OK) return st;
  }
  return TM_OK;
}

// ---------------------------------------------------------------- SUMMA
// 2-D sharding ("2-D SUMMA-style sharding for larger
// P"): ranks form a pr x pc grid, rank r = (i, j) = (r / pc, r % pc) owns
//   C[rows_i, cols_j],  A[rows_i, ka_j],  B[kb_i, cols_j]
// with rows_i = tm_dist_rows(m, pr, i), cols_j = tm_dist_rows(n, pc, j),
// ka_j = tm_dist_rows(k, pc, j), kb_i = tm_dist_rows(k, pr, i).  K is cut into
// panels lying inside one A column block and one B row block; for panel p the
// owner (i, ja(p)) of A(i, p) broadcasts it along grid row i, the owner
// (ib(p), j) of B(p, j) along grid column j, and every rank accumulates
// C_ij = alpha * A(i,p) B(p,j) + beta_p C_ij (beta for the first panel, then
// 1).  Double-buffered: panel p+1 is packed and broadcast while panel p's GEMM
// runs.  Per rank the traffic is the A and B panels of its grid row / column
// (~ k (m/pr + n/pc) floats) instead of all of B (k n) for the 1-D schedule.

constexpr int64_t kSummaPanelMax = 2048;

// Panel boundaries: the union of the A (over pc) and B (over pr) K
// partitions, each interval split into pieces of at most kSummaPanelMax.
static int summa_panels(int64_t k, int pr, int pc, std::vector<int64_t>& b) {
  b.assign(1, 0);
  if (k <= 0) return 0;
  std::vector<int64_t> cuts;
  for (int j = 0; j < pc; ++j) {
    int64_t r0, rr;
    tm_dist_rows(k, pc, j, &r0, &rr);
    cuts.push_back(r0 + rr);
  }
  for (int i = 0; i < pr; ++i) {
    int64_t r0, rr;
    tm_dist_rows(k, pr, i, &r0, &rr);
    cuts.push_back(r0 + rr);
  }
  std::sort(cuts.begin(), cuts.end());
  int64_t prev = 0;
  for (int64_t c : cuts) {
    if (c <= prev) continue;
    const int64_t pieces = (c - prev + kSummaPanelMax - 1) / kSummaPanelMax;
    for (int64_t q = 1; q <= pieces; ++q) b.push_back(prev + (c - prev) * q / pieces);
    prev = c;
  }
  return static_cast<int>(b.size()) - 1;
}

// The grid block owning K index k0 under tm_dist_rows(k, parts, .).
static int owner_of(int64_t k, int parts, int64_t k0, int64_t* start) {
  for (int q = 0; q < parts; ++q) {
    int64_t r0, rr;
    tm_dist_rows(k, parts, q, &r0, &rr);
    if (k0 >= r0 && k0 < r0 + rr) {
      *start = r0;
      return q;
    }
  }
  *start = 0;
  return 0;
}

struct SummaBlocks {  // one rank's view: its blocks and those of the panel owners
  int64_t rows, cols;                 // of C_ij
  int64_t lda_panel, ldb_panel;       // packed panel pitches (multiples of 4)
};

// Per-rank SUMMA schedule.  `deliver(p, ja, ka0, ib, kb0, k0, kr, Apan, Bpan)`
// enqueues on comm_stream the arrival of A(i, [k0, k0+kr)) packed as rows x kr
// (pitch lda_panel) in Apan and B([k0, k0+kr), j) as kr x cols (pitch
// ldb_panel) in Bpan; ja / ib own them, ka0 / kb0 are the owners' first K
// indices.  panel_buf holds 2 x (A panel + B panel).
template <class Deliver>
tm_status summa_schedule(int pr, int pc, int rank, int64_t m, int64_t n, int64_t k, float alpha, float beta,
                         float* C_local, int64_t ldc, cudaStream_t stream, cudaStream_t comm_stream,
                         cudaEvent_t ev_start, cudaEvent_t* ev_ready, cudaEvent_t* ev_used, float* panel_buf,
                         Deliver&& deliver) {
  const int i = rank / pc, j = rank % pc;
  int64_t r0, rows, c0, cols;
  tm_dist_rows(m, pr, i, &r0, &rows);
  tm_dist_rows(n, pc, j, &c0, &cols);
  if (alpha == 0.0f || k == 0)  // every rank alike: nothing to exchange
    return tm_sgemm(rows, cols, 0, 0.0f, nullptr, 1, nullptr, std::max<int64_t>(1, cols), beta, C_local, ldc, stream);
  // A rank with an empty block still takes part in its row's and column's
  // broadcasts (ranks of a grid row share `rows`, of a column `cols`).
  std::vector<int64_t> b;
  const int np = summa_panels(k, pr, pc, b);
  int64_t maxkr = 0;
  for (int p = 0; p < np; ++p) maxkr = std::max(maxkr, b[p + 1] - b[p]);
  const int64_t lda_p = (maxkr + 3) / 4 * 4, ldb_p = (cols + 3) / 4 * 4;
  const size_t a_elems = static_cast<size_t>(rows) * lda_p, b_elems = static_cast<size_t>(maxkr) * ldb_p;
  if (cudaEventRecord(ev_start, stream) != cudaSuccess) return TM_ERR_CUDA;
  if (cudaStreamWaitEvent(comm_stream, ev_start, 0) != cudaSuccess) return TM_ERR_CUDA;
  nvtxRangePushA("tm_sgemm_summa schedule");
  struct Pop {
    ~Pop() { nvtxRangePop(); }
  } pop;
  for (int p = 0; p < np; ++p) {
    const int s = p & 1;
    float* Apan = panel_buf + s * (a_elems + b_elems);
    float* Bpan = Apan + a_elems;
    const int64_t k0 = b[p], kr = b[p + 1] - b[p];
    int64_t ka0 = 0, kb0 = 0;
    const int ja = owner_of(k, pc, k0, &ka0), ib = owner_of(k, pr, k0, &kb0);
    if (p >= 2 && cudaStreamWaitEvent(comm_stream, ev_used[s], 0) != cudaSuccess) return TM_ERR_CUDA;
    tm_status st = deliver(p, ja, ka0, ib, kb0, k0, kr, Apan, lda_p, Bpan, ldb_p);
    if (st != TM_OK) return st;
    if (cudaEventRecord(ev_ready[s], comm_stream) != cudaSuccess) return TM_ERR_CUDA;
    if (cudaStreamWaitEvent(stream, ev_ready[s], 0) != cudaSuccess) return TM_ERR_CUDA;
    if (rows > 0 && cols > 0) {
      tmk::GemmArgs ga{rows, cols, kr, alpha, p == 0 ? beta : 1.0f, Apan, lda_p, Bpan, ldb_p, C_local, ldc};
      if ((st = tmk::sgemm_reserve(ga, stream, 0)) != TM_OK) return st;
    }
    if (cudaEventRecord(ev_used[s], stream) != cudaSuccess) return TM_ERR_CUDA;
  }
  return TM_OK;
}

// Bytes of the two panel buffers (A and B, double-buffered) for rank `rank`.
static size_t summa_buffer_bytes(int pr, int pc, int rank, int64_t m, int64_t n, int64_t k) {
  int64_t r0, rows, c0, cols;
  tm_dist_rows(m, pr, rank / pc, &r0, &rows);
  tm_dist_rows(n, pc, rank % pc, &c0, &cols);
  std::vector<int64_t> b;
  const int np = summa_panels(k, pr, pc, b);
  int64_t maxkr = 0;
  for (int p = 0; p < np; ++p) maxkr = std::max(maxkr, b[p + 1] - b[p]);
  const size_t a = static_cast<size_t>(rows) * ((maxkr + 3) / 4 * 4), bb = static_cast<size_t>(maxkr) * ((cols + 3) / 4 * 4);
  return 2 * (a + bb) * 4;
}

// Row-distributed blur (Fig. 5 Code 3).  Rank r owns
// output rows [row0, row0 + rows) of the N-2 (tm_dist_rows(N-2, P, r)) and the
// matching input rows in lin[0, rows); the two border rows lin[rows, rows + 2)
// come from rank r+1 (its lin[0, 2)), the last rank's are the caller's.
// `exchange(send_buf, recv_buf, count)` enqueues on comm_stream the send of
// this rank's first two rows to r-1 (send_buf null on rank 0) and the receive
// of r+1's into the border region (recv_buf null on the last rank).  The
// interior rows [0, rows - 2) need no border and run while it is in flight.
template <class Exchange>
tm_status blur_dist_schedule(int nranks, int rank, int64_t N, int64_t M, float* lin, int64_t ldi, float* lout,
                             int64_t ldo, cudaStream_t stream, cudaStream_t comm_stream, cudaEvent_t ev_start,
                             cudaEvent_t ev_halo, uint64_t* bytes_received, Exchange&& exchange) {
  if (N < 3 || M < 3 || ldi < 3 * M || ldo < 3 * (M - 2) || !lin || !lout) return TM_ERR_INVALID_VALUE;
  if (nranks > 1 && (N - 2) / nranks < 2) return TM_ERR_INVALID_VALUE;
  int64_t row0 = 0, rows = 0;
  tm_dist_rows(N - 2, nranks, rank, &row0, &rows);
  {  // lout must not overlap lin (rows + 2 input rows)
    const uintptr_t i0 = reinterpret_cast<uintptr_t>(lin), o0 = reinterpret_cast<uintptr_t>(lout);
    const uintptr_t ib = static_cast<uintptr_t>(((rows + 1) * ldi + 3 * M) * 4);
    const uintptr_t ob = static_cast<uintptr_t>(((rows - 1) * ldo + 3 * (M - 2)) * 4);
    if (i0 < o0 + ob && o0 < i0 + ib) return TM_ERR_INVALID_VALUE;
  }
  int sms = 0;
  tm_status st = tmk::device_sms(&sms);
  if (st != TM_OK) return st;
  const bool last = rank == nranks - 1;
  if (nranks == 1 || (last && rank == 0))
    return tmk::launch_blur(0, rows, M, lin, ldi, lout, ldo, sms, stream);
  // two rows of the paper's M*2*3 contiguous elements, here row pitch ldi
  const size_t count = static_cast<size_t>(ldi + 3 * M);
  if (cudaEventRecord(ev_start, stream) != cudaSuccess) return TM_ERR_CUDA;
  if (cudaStreamWaitEvent(comm_stream, ev_start, 0) != cudaSuccess) return TM_ERR_CUDA;
  nvtxRangePushA("tm_blur_dist schedule");
  struct Pop {
    ~Pop() { nvtxRangePop(); }
  } pop;
  st = exchange(rank > 0 ? lin : nullptr, last ? nullptr : lin + rows * ldi, count);
  if (st != TM_OK) return st;
  if (!last && bytes_received) *bytes_received += count * 4;
  if (cudaEventRecord(ev_halo, comm_stream) != cudaSuccess) return TM_ERR_CUDA;
  if (last) {  // border rows are local: one launch, then join the send
    st = tmk::launch_blur(0, rows, M, lin, ldi, lout, ldo, sms, stream);
    if (st != TM_OK) return st;
    return cudaStreamWaitEvent(stream, ev_halo, 0) == cudaSuccess ? TM_OK : TM_ERR_CUDA;
  }
  st = tmk::launch_blur(0, rows - 2, M, lin, ldi, lout, ldo, sms, stream);  // interior, overlaps the exchange
  if (st != TM_OK) return st;
  if (cudaStreamWaitEvent(stream, ev_halo, 0) != cudaSuccess) return TM_ERR_CUDA;
  return tmk::launch_blur(rows - 2, rows, M, lin, ldi, lout, ldo, sms, stream);
}

}  // namespace

extern "C" {

tm_status tm_sgemm_dist(tm_comm_t comm, int64_t m, int64_t n, int64_t k, float alpha, const float* A_local,
                        int64_t lda, float* B, int64_t ldb, int root, float beta, float* C_local, int64_t ldc,
                        void* stream_) {
  if (!comm || root < 0 || root >= comm->nranks || m < 0 || n < 0 || k < 0) return TM_ERR_INVALID_VALUE;
  auto xfer = [&](float* p, size_t count) -> tm_status {
    return g_nccl.Broadcast(p, p, count, ncclFloat32, root, comm->comm, comm->stream) == ncclSuccess ? TM_OK
                                                                                                    : TM_ERR_NCCL;
  };
  return dist_schedule(comm->nranks, comm->rank, root, m, n, k, alpha, A_local, lda, B, ldb, beta, C_local, ldc,
                       static_cast<cudaStream_t>(stream_), comm->stream, comm->ev_start, comm->ev_chunk,
                       &comm->bytes_received, xfer);
}

tm_status tm_sgemm_dist_fused(tm_comm_t comm, int64_t m, int64_t n, int64_t k, float alpha, const float* A_local,
                              int64_t lda, float* B, int64_t ldb, int root, float beta, float* C_local, int64_t ldc,
                              void* stream_) {
  if (!comm || root < 0 || root >= comm->nranks || m < 0 || n < 0 || k < 0) return TM_ERR_INVALID_VALUE;
  auto xfer = [&](float* p, size_t count) -> tm_status {
    return g_nccl.Broadcast(p, p, count, ncclFloat32, root, comm->comm, comm->stream) == ncclSuccess ? TM_OK
                                                                                                    : TM_ERR_NCCL;
  };
  return dist_fused_schedule(comm->nranks, comm->rank, root, m, n, k, alpha, A_local, lda, B, ldb, beta, C_local,
                             ldc, static_cast<cudaStream_t>(stream_), comm->stream, comm->ev_start, comm->ev_chunk,
                             comm->chunk_flags, ++comm->epoch, comm_ctas(), &comm->bytes_received, xfer);
}

tm_status tm_sgemm_dist_loopback(int nranks, int root, int mode, int64_t m, int64_t n, int64_t k, float alpha,
                                 const float* const* A_locals, int64_t lda, float* const* Bs, int64_t ldb,
                                 float beta, float* const* C_locals, int64_t ldc, uint64_t* bytes_received,
                                 void* stream_) {
  if (nranks < 1 || root < 0 || root >= nranks || !A_locals || !Bs || !C_locals || m < 0 || n < 0 || k < 0 ||
      mode < 0 || mode > 4)
    return TM_ERR_INVALID_VALUE;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_start = nullptr, ev_chunk[kMaxChunks] = {};
  tm_status st = TM_OK;
  bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; ok && i < kMaxChunks; ++i)
    ok = cudaEventCreateWithFlags(&ev_chunk[i], cudaEventDisableTiming) == cudaSuccess;
  unsigned* flags = nullptr;  // fused mode: per-chunk arrival flags, zeroed once (rank r's epoch is r + 1)
  LinkClock clock;                 // link model (host functions on the transfer stream)
  std::vector<LinkWait> waits;
  waits.reserve(kMaxChunks);
  if (ok && (mode == 2 || mode == 4))
    ok = cudaMalloc(&flags, kMaxChunks * sizeof(unsigned)) == cudaSuccess &&
         cudaMemsetAsync(flags, 0, kMaxChunks * sizeof(unsigned), stream) == cudaSuccess;
  if (!ok) st = TM_ERR_CUDA;
  const double link_gbs = loopback_link_gbs(mode);
  if (bytes_received)
    for (int r = 0; r < nranks; ++r) bytes_received[r] = 0;
  // Ranks run one after another on this device; rank r's "broadcast" copies
  // the root's chunk into rank r's B (the root's own transfer is a no-op).
  if (mode == 1 && k % nranks != 0) st = TM_ERR_INVALID_VALUE;
  // All-gather emulation needs every rank's shard before any rank's gather
  // overwrites the rest of its buffer: keep a copy of all shards.
  float* shards = nullptr;
  const int64_t kr = (mode == 1 && nranks > 0) ? k / nranks : 0;
  if (st == TM_OK && mode == 1 && kr > 0) {
    if (cudaMalloc(&shards, static_cast<size_t>(k) * ldb * 4) != cudaSuccess) st = TM_ERR_OUT_OF_MEMORY;
    for (int q = 0; st == TM_OK && q < nranks; ++q)
      if (cudaMemcpyAsync(shards + q * kr * ldb, Bs[q] + q * kr * ldb, static_cast<size_t>(kr) * ldb * 4,
                          cudaMemcpyDeviceToDevice, stream) != cudaSuccess)
        st = TM_ERR_CUDA;
    if (st == TM_OK && cudaStreamSynchronize(stream) != cudaSuccess) st = TM_ERR_CUDA;
  }
  for (int r = 0; st == TM_OK && r < nranks; ++r) {
    if (mode != 1) {
      const float* root_B = Bs[root];
      const int pos = (r - root + nranks) % nranks;                       // chain position
      const double piece_bytes = 128.0 * static_cast<double>(ldb) * 4.0;  // the CE chain's piece
      double sent = 0.0;
      auto xfer = [&](float* p, size_t count) -> tm_status {
        if (r == root) return TM_OK;
        if (link_gbs > 0.0 && p == Bs[r]) {  // first chunk: start the link clock
          waits.clear();
          if (cudaLaunchHostFunc(cs, link_start, &clock) != cudaSuccess) return TM_ERR_CUDA;
        }
        const float* src = root_B + (p - Bs[r]);
        if (mode < 3 && cudaMemcpyAsync(p, src, count * 4, cudaMemcpyDeviceToDevice, cs) != cudaSuccess)
          return TM_ERR_CUDA;
        if (link_gbs > 0.0) {  // projection: the chunk arrives no earlier than the modelled link delivers it
          sent += count * 4.0;
          waits.push_back({&clock, (pos * piece_bytes + sent) / link_gbs});
          if (cudaLaunchHostFunc(cs, link_until, &waits.back()) != cudaSuccess) return TM_ERR_CUDA;
        }
        return TM_OK;
      };
      const int reserve = loopback_reserve(mode);
      if (mode == 0 || mode == 3)
        st = dist_schedule(nranks, r, root, m, n, k, alpha, A_locals[r], lda, Bs[r], ldb, beta, C_locals[r], ldc,
                           stream, cs, ev_start, ev_chunk, bytes_received ? &bytes_received[r] : nullptr, xfer,
                           mode == 3 ? reserve : -1);
      else  // flags of simulated rank r carry epoch r + 1 (flags are never reset within the call)
        st = dist_fused_schedule(nranks, r, root, m, n, k, alpha, A_locals[r], lda, Bs[r], ldb, beta, C_locals[r],
                                 ldc, stream, cs, ev_start, ev_chunk, flags, static_cast<unsigned>(r + 1),
                                 reserve, bytes_received ? &bytes_received[r] : nullptr, xfer);
    } else {
      auto gather = [&](size_t count) -> tm_status {
        for (int q = 0; q < nranks; ++q) {
          if (q == r) continue;
          if (cudaMemcpyAsync(Bs[r] + q * kr * ldb, shards + q * kr * ldb, count * 4, cudaMemcpyDeviceToDevice, cs) !=
              cudaSuccess)
            return TM_ERR_CUDA;
        }
        return TM_OK;
      };
      st = allgather_schedule(nranks, r, m, n, k, alpha, A_locals[r], lda, Bs[r] + r * kr * ldb, Bs[r], ldb, beta,
                              C_locals[r], ldc, stream, cs, ev_start, ev_chunk[0],
                              bytes_received ? &bytes_received[r] : nullptr, gather);
    }
    if (st == TM_OK && cudaStreamSynchronize(stream) != cudaSuccess) st = TM_ERR_CUDA;
  }
  if (shards) cudaFree(shards);
  if (cs) cudaStreamSynchronize(cs);
  if (flags) cudaFree(flags);
  for (int i = 0; i < kMaxChunks; ++i)
    if (ev_chunk[i]) cudaEventDestroy(ev_chunk[i]);
  if (ev_start) cudaEventDestroy(ev_start);
  if (cs) cudaStreamDestroy(cs);
  return st;
}

tm_status tm_sgemm_dist_allgather(tm_comm_t comm, int64_t m, int64_t n, int64_t k, float alpha,
                                  const float* A_local, int64_t lda, const float* B_shard, float* B_full,
                                  int64_t ldb, float beta, float* C_local, int64_t ldc, void* stream_) {
  if (!comm || m < 0 || n < 0 || k < 0) return TM_ERR_INVALID_VALUE;
  auto gather = [&](size_t count) -> tm_status {
    return g_nccl.AllGather(B_shard, B_full, count, ncclFloat32, comm->comm, comm->stream) == ncclSuccess
               ? TM_OK
               : TM_ERR_NCCL;
  };
  return allgather_schedule(comm->nranks, comm->rank, m, n, k, alpha, A_local, lda, B_shard, B_full, ldb, beta,
                            C_local, ldc, static_cast<cudaStream_t>(stream_), comm->stream, comm->ev_start,
                            comm->ev_chunk[0], &comm->bytes_received, gather);
}

tm_status tm_blur_dist(tm_comm_t comm, int64_t N, int64_t M, float* lin, int64_t ldi, float* lout, int64_t ldo,
                       void* stream_) {
  if (!comm) return TM_ERR_INVALID_VALUE;
  if (comm->nranks > 1 && !(g_nccl.Send && g_nccl.Recv && g_nccl.GroupStart && g_nccl.GroupEnd)) return TM_ERR_NCCL;
  const int r = comm->rank;
  auto exchange = [&](const float* send_buf, float* recv_buf, size_t count) -> tm_status {
    if (g_nccl.GroupStart() != ncclSuccess) return TM_ERR_NCCL;
    bool ok = true;
    if (send_buf) ok = g_nccl.Send(send_buf, count, ncclFloat32, r - 1, comm->comm, comm->stream) == ncclSuccess;
    if (ok && recv_buf) ok = g_nccl.Recv(recv_buf, count, ncclFloat32, r + 1, comm->comm, comm->stream) == ncclSuccess;
    const bool ended = g_nccl.GroupEnd() == ncclSuccess;
    return ok && ended ? TM_OK : TM_ERR_NCCL;
  };
  return blur_dist_schedule(comm->nranks, r, N, M, lin, ldi, lout, ldo, static_cast<cudaStream_t>(stream_),
                            comm->stream, comm->ev_start, comm->ev_chunk[0], &comm->bytes_received, exchange);
}

tm_status tm_blur_dist_loopback(int nranks, int64_t N, int64_t M, float* const* lins, int64_t ldi,
                                float* const* louts, int64_t ldo, uint64_t* bytes_received, void* stream_) {
  if (nranks < 1 || !lins || !louts) return TM_ERR_INVALID_VALUE;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_start = nullptr, ev_halo = nullptr;
  tm_status st = TM_OK;
  if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ev_halo, cudaEventDisableTiming) != cudaSuccess)
    st = TM_ERR_CUDA;
  if (bytes_received)
    for (int r = 0; r < nranks; ++r) bytes_received[r] = 0;
  // Ranks one after another; rank r's receive copies rank r+1's first two rows
  // (its send is the matching receive of rank r-1, so it moves nothing here).
  for (int r = 0; st == TM_OK && r < nranks; ++r) {
    auto exchange = [&](const float*, float* recv_buf, size_t count) -> tm_status {
      if (!recv_buf) return TM_OK;
      return cudaMemcpyAsync(recv_buf, lins[r + 1], count * 4, cudaMemcpyDeviceToDevice, cs) == cudaSuccess
                 ? TM_OK
                 : TM_ERR_CUDA;
    };
    st = blur_dist_schedule(nranks, r, N, M, lins[r], ldi, louts[r], ldo, stream, cs, ev_start, ev_halo,
                            bytes_received ? &bytes_received[r] : nullptr, exchange);
    if (st == TM_OK && cudaStreamSynchronize(stream) != cudaSuccess) st = TM_ERR_CUDA;
  }
  if (cs) cudaStreamSynchronize(cs);
  if (ev_halo) cudaEventDestroy(ev_halo);
  if (ev_start) cudaEventDestroy(ev_start);
  if (cs) cudaStreamDestroy(cs);
  return st;
}

tm_status tm_summa_panel(int64_t k, int pr, int pc, int idx, int64_t* k0, int64_t* kr) {
  if (k < 0 || pr < 1 || pc < 1 || !k0 || !kr) return TM_ERR_INVALID_VALUE;
  std::vector<int64_t> b;
  const int np = summa_panels(k, pr, pc, b);
  if (idx < 0) {
    *k0 = np;
    *kr = 0;
    return TM_OK;
  }
  if (idx >= np) return TM_ERR_INVALID_VALUE;
  *k0 = b[idx];
  *kr = b[idx + 1] - b[idx];
  return TM_OK;
}

tm_status tm_sgemm_summa(tm_comm_t comm, int pr, int pc, int64_t m, int64_t n, int64_t k, float alpha,
                         const float* A_local, int64_t lda, const float* B_local, int64_t ldb, float beta,
                         float* C_local, int64_t ldc, void* stream_) {
  if (!comm || pr < 1 || pc < 1 || pr * pc != comm->nranks || m < 0 || n < 0 || k < 0) return TM_ERR_INVALID_VALUE;
  const int r = comm->rank, i = r / pc, j = r % pc;
  int64_t r0, rows, c0, cols, a0, ka, b0, kb;
  tm_dist_rows(m, pr, i, &r0, &rows);
  tm_dist_rows(n, pc, j, &c0, &cols);
  tm_dist_rows(k, pc, j, &a0, &ka);
  tm_dist_rows(k, pr, i, &b0, &kb);
  if (rows > 0 && cols > 0 && (!C_local || ldc < std::max<int64_t>(1, cols))) return TM_ERR_INVALID_VALUE;
  const bool reads_ab = alpha != 0.0f && k > 0;
  if (reads_ab && ((ka > 0 && rows > 0 && (!A_local || lda < ka)) || (kb > 0 && cols > 0 && (!B_local || ldb < cols))))
    return TM_ERR_INVALID_VALUE;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  if (comm->nranks == 1)
    return tm_sgemm(m, n, k, alpha, A_local, lda, B_local, ldb, beta, C_local, ldc, stream);
  if (!g_nccl.CommSplit || !g_nccl.GroupStart || !g_nccl.GroupEnd) return TM_ERR_NCCL;
  if (comm->summa_pr != pr || comm->summa_pc != pc) {  // collective: every rank switches grid together
    if (comm->row_comm) g_nccl.CommDestroy(comm->row_comm);
    if (comm->col_comm) g_nccl.CommDestroy(comm->col_comm);
    comm->row_comm = comm->col_comm = nullptr;
    if (g_nccl.CommSplit(comm->comm, i, j, &comm->row_comm, nullptr) != ncclSuccess ||
        g_nccl.CommSplit(comm->comm, j, i, &comm->col_comm, nullptr) != ncclSuccess)
      return TM_ERR_NCCL;
    comm->summa_pr = pr;
    comm->summa_pc = pc;
    for (int q = 0; q < 2; ++q) {
      if (!comm->ev_ready[q] && cudaEventCreateWithFlags(&comm->ev_ready[q], cudaEventDisableTiming) != cudaSuccess)
        return TM_ERR_CUDA;
      if (!comm->ev_used[q] && cudaEventCreateWithFlags(&comm->ev_used[q], cudaEventDisableTiming) != cudaSuccess)
        return TM_ERR_CUDA;
    }
  }
  const size_t need = summa_buffer_bytes(pr, pc, r, m, n, k);
  if (need > comm->panel_bytes) {
    if (comm->panel_buf) {
      cudaStreamSynchronize(comm->stream);
      cudaStreamSynchronize(stream);
      cudaFree(comm->panel_buf);
      comm->panel_buf = nullptr;
      comm->panel_bytes = 0;
    }
    if (cudaMalloc(&comm->panel_buf, need) != cudaSuccess) return TM_ERR_OUT_OF_MEMORY;
    comm->panel_bytes = need;
  }
  auto deliver = [&](int, int ja, int64_t ka0, int ib, int64_t kb0, int64_t k0, int64_t kr, float* Apan,
                     int64_t lda_p, float* Bpan, int64_t ldb_p) -> tm_status {
    // owners pack their panel (a strided 2-D copy), then both broadcasts
    if (j == ja && rows > 0 &&
        cudaMemcpy2DAsync(Apan, lda_p * 4, A_local + (k0 - ka0), lda * 4, kr * 4, rows, cudaMemcpyDeviceToDevice,
                          comm->stream) != cudaSuccess)
      return TM_ERR_CUDA;
    if (i == ib && cols > 0 &&
        cudaMemcpy2DAsync(Bpan, ldb_p * 4, B_local + (k0 - kb0) * ldb, ldb * 4, cols * 4, kr,
                          cudaMemcpyDeviceToDevice, comm->stream) != cudaSuccess)
      return TM_ERR_CUDA;
    if (g_nccl.GroupStart() != ncclSuccess) return TM_ERR_NCCL;
    bool ok = true;
    if (pc > 1 && rows > 0)
      ok = g_nccl.Broadcast(Apan, Apan, static_cast<size_t>(rows) * lda_p, ncclFloat32, ja, comm->row_comm,
                            comm->stream) == ncclSuccess;
    if (ok && pr > 1 && cols > 0)
      ok = g_nccl.Broadcast(Bpan, Bpan, static_cast<size_t>(kr) * ldb_p, ncclFloat32, ib, comm->col_comm,
                            comm->stream) == ncclSuccess;
    const bool ended = g_nccl.GroupEnd() == ncclSuccess;
    if (!(ok && ended)) return TM_ERR_NCCL;
    if (j != ja) comm->bytes_received += static_cast<uint64_t>(rows) * lda_p * 4;
    if (i != ib) comm->bytes_received += static_cast<uint64_t>(kr) * ldb_p * 4;
    return TM_OK;
  };
  return summa_schedule(pr, pc, r, m, n, k, alpha, beta, C_local, ldc, stream, comm->stream, comm->ev_start,
                        comm->ev_ready, comm->ev_used, comm->panel_buf, deliver);
}

tm_status tm_sgemm_summa_loopback(int pr, int pc, int64_t m, int64_t n, int64_t k, float alpha,
                                  const float* const* A_locals, const int64_t* ldas, const float* const* B_locals,
                                  const int64_t* ldbs, float beta, float* const* C_locals, const int64_t* ldcs,
                                  uint64_t* bytes_received, void* stream_) {
  if (pr < 1 || pc < 1 || !A_locals || !ldas || !B_locals || !ldbs || !C_locals || !ldcs || m < 0 || n < 0 || k < 0)
    return TM_ERR_INVALID_VALUE;
  const int P = pr * pc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_start = nullptr, ev_ready[2] = {}, ev_used[2] = {};
  float* buf = nullptr;
  size_t need = 0;
  for (int r = 0; r < P; ++r) need = std::max(need, summa_buffer_bytes(pr, pc, r, m, n, k));
  tm_status st = TM_OK;
  bool ok = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) == cudaSuccess;
  for (int q = 0; ok && q < 2; ++q)
    ok = cudaEventCreateWithFlags(&ev_ready[q], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&ev_used[q], cudaEventDisableTiming) == cudaSuccess;
  if (ok && need) ok = cudaMalloc(&buf, need) == cudaSuccess;
  if (!ok) st = TM_ERR_CUDA;
  if (bytes_received)
    for (int r = 0; r < P; ++r) bytes_received[r] = 0;
  // Ranks one after another; every rank's panels are packed straight from the
  // owners' blocks (the broadcast of the NCCL entry point).
  for (int r = 0; st == TM_OK && r < P; ++r) {
    const int i = r / pc, j = r % pc;
    int64_t r0, rows, c0, cols;
    tm_dist_rows(m, pr, i, &r0, &rows);
    tm_dist_rows(n, pc, j, &c0, &cols);
    auto deliver = [&](int, int ja, int64_t ka0, int ib, int64_t kb0, int64_t k0, int64_t kr, float* Apan,
                       int64_t lda_p, float* Bpan, int64_t ldb_p) -> tm_status {
      const int oa = i * pc + ja, ob = ib * pc + j;  // owner ranks
      if (rows > 0 && cudaMemcpy2DAsync(Apan, lda_p * 4, A_locals[oa] + (k0 - ka0), ldas[oa] * 4, kr * 4, rows,
                                        cudaMemcpyDeviceToDevice, cs) != cudaSuccess)
        return TM_ERR_CUDA;
      if (cols > 0 && cudaMemcpy2DAsync(Bpan, ldb_p * 4, B_locals[ob] + (k0 - kb0) * ldbs[ob], ldbs[ob] * 4,
                                        cols * 4, kr, cudaMemcpyDeviceToDevice, cs) != cudaSuccess)
        return TM_ERR_CUDA;
      if (bytes_received) {
        if (oa != r) bytes_received[r] += static_cast<uint64_t>(rows) * lda_p * 4;
        if (ob != r) bytes_received[r] += static_cast<uint64_t>(kr) * ldb_p * 4;
      }
      return TM_OK;
    };
    st = summa_schedule(pr, pc, r, m, n, k, alpha, beta, C_locals[r], ldcs[r], stream, cs, ev_start, ev_ready,
                        ev_used, buf, deliver);
    if (st == TM_OK && cudaStreamSynchronize(stream) != cudaSuccess) st = TM_ERR_CUDA;
  }
  if (cs) cudaStreamSynchronize(cs);
  if (buf) cudaFree(buf);
  for (int q = 0; q < 2; ++q) {
    if (ev_ready[q]) cudaEventDestroy(ev_ready[q]);
    if (ev_used[q]) cudaEventDestroy(ev_used[q]);
  }
  if (ev_start) cudaEventDestroy(ev_start);
  if (cs) cudaStreamDestroy(cs);
  return st;
}

}  // extern "C"
