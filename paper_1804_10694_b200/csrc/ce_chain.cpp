// ce_chain.cpp -- copy-engine chain broadcast of B for the row-sharded sgemm
// ("a copy-engine chain broadcast (no SM contention)").
//
// The paper's distributed model moves data with explicit send/receive
// between ranks that each own a row block.
// Here the one exchange, B from the root to every rank, runs as a pipelined
// chain root -> r+1 -> r+2 ... over CUDA IPC mappings of the peers' buffers:
// each rank PUSHES every piece of B it holds into its successor's B with a
// cudaMemcpyAsync to the peer's mapping -- between devices a peer-to-peer copy
// over NVLink, executed by the copy engines -- then writes the successor's
// arrival flag for that piece with a stream memory operation
// (cuStreamWriteValue32, ordered after the copy, with a memory barrier).  No
// kernel moves data between GPUs, so the GEMM keeps all 148 SMs (the NCCL
// schedule leaves 16 to NCCL's kernels).  Within ONE device a device-to-device
// cudaMemcpyAsync is a kernel (scripts/r02/ce_probe.cu: a 256 MiB copy waits
// 3 ms behind a kernel holding every SM's thread slots), so the tests, whose
// processes share one GPU, check correctness only, not overlap.
//
// Flow control (credits): before the first piece of a call is pushed, the
// successor must have declared its B free for this call: every rank writes
// its predecessor's "ready" flag on its own compute stream at the start of the
// call, i.e. after its previous call's GEMMs stopped reading B.  All flags are
// epochs (one per call, identical on every rank since calls are collective),
// compared with wrap-safe int32 differences, so they are never reset.
//
// Flags live in one small device allocation per rank, exported by CUDA IPC:
//   flags[0]         = ready: my successor may receive epoch e (written by the successor)
//   flags[1 + p]     = piece p of B has arrived in my B    (written by the predecessor)
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "tm_internal.h"

namespace {

constexpr int kMaxPieces = 4096;
constexpr int kMaxChunksCe = 16;
constexpr int64_t kPieceRows = 128;  // K-rows per forwarded piece (8 MiB at n = 16384)

}  // namespace

struct tm_ce_s {
  int nranks = 1, rank = 0, device = 0;
  unsigned* flags = nullptr;          // local [1 + kMaxPieces]
  unsigned* succ_flags = nullptr;     // successor's flags (IPC-mapped)
  unsigned* pred_flags = nullptr;     // predecessor's flags (IPC-mapped)
  int succ = -1, pred = -1;           // chain neighbours of the last connect (root-relative below)
  std::vector<void*> peer_flags;      // every peer's flags, opened at connect (nullptr for self)
  std::map<std::string, void*> opened;  // IPC handle bytes -> mapped base
  cudaStream_t recv = nullptr, send = nullptr;
  cudaEvent_t ev_start = nullptr, ev_send_done = nullptr, ev_recv_done = nullptr;
  cudaEvent_t ev_chunk[kMaxChunksCe] = {};
  unsigned epoch = 0;
  uint64_t bytes_received = 0;
};

namespace {

tm_status open_handle(tm_ce_s* ce, const tm_ipc_buf& h, void** out) {
  const std::string key(reinterpret_cast<const char*>(h.bytes), sizeof(h.bytes));
  auto it = ce->opened.find(key);
  if (it == ce->opened.end()) {
    cudaIpcMemHandle_t mh;
    static_assert(sizeof(mh) <= sizeof(h.bytes), "IPC handle size");
    std::memcpy(&mh, h.bytes, sizeof(mh));
    void* base = nullptr;
    if (cudaIpcOpenMemHandle(&base, mh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return TM_ERR_CUDA;
    }
    it = ce->opened.emplace(key, base).first;
  }
  *out = static_cast<char*>(it->second) + h.offset;
  return TM_OK;
}

}  // namespace

extern "C" {

tm_status tm_ipc_export(const void* ptr, tm_ipc_buf* out) {
  if (!ptr || !out) return TM_ERR_INVALID_VALUE;
  void* base = nullptr;
  tm_status st = tmk::device_allocation(ptr, &base, nullptr);
  if (st != TM_OK) return st;
  cudaIpcMemHandle_t mh;
  if (cudaIpcGetMemHandle(&mh, base) != cudaSuccess) {
    cudaGetLastError();
    return TM_ERR_CUDA;
  }
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->bytes, &mh, sizeof(mh));
  out->offset = static_cast<const char*>(ptr) - static_cast<const char*>(base);
  return TM_OK;
}

tm_status tm_ce_create(tm_ce_t* out, int nranks, int rank, tm_ipc_buf* my_flags) {
  if (!out || !my_flags || nranks < 1 || rank < 0 || rank >= nranks) return TM_ERR_INVALID_VALUE;
  tm_ce_s* ce = new (std::nothrow) tm_ce_s;
  if (!ce) return TM_ERR_OUT_OF_MEMORY;
  ce->nranks = nranks;
  ce->rank = rank;
  bool ok = cudaGetDevice(&ce->device) == cudaSuccess &&
            cudaMalloc(&ce->flags, (1 + kMaxPieces) * sizeof(unsigned)) == cudaSuccess &&
            cudaMemset(ce->flags, 0, (1 + kMaxPieces) * sizeof(unsigned)) == cudaSuccess &&
            cudaDeviceSynchronize() == cudaSuccess &&
            cudaStreamCreateWithFlags(&ce->recv, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamCreateWithFlags(&ce->send, cudaStreamNonBlocking) == cudaSuccess &&
            cudaEventCreateWithFlags(&ce->ev_start, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ce->ev_send_done, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&ce->ev_recv_done, cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; ok && i < kMaxChunksCe; ++i)
    ok = cudaEventCreateWithFlags(&ce->ev_chunk[i], cudaEventDisableTiming) == cudaSuccess;
  if (!ok) {
    tm_ce_destroy(ce);
    return TM_ERR_CUDA;
  }
  tm_status st = tm_ipc_export(ce->flags, my_flags);
  if (st != TM_OK) {
    tm_ce_destroy(ce);
    return st;
  }
  *out = ce;
  return TM_OK;
}

tm_status tm_ce_connect(tm_ce_t ce, const tm_ipc_buf* all_flags) {
  if (!ce || !all_flags) return TM_ERR_INVALID_VALUE;
  ce->peer_flags.assign(ce->nranks, nullptr);
  for (int r = 0; r < ce->nranks; ++r) {
    if (r == ce->rank) continue;
    void* p = nullptr;
    tm_status st = open_handle(ce, all_flags[r], &p);
    if (st != TM_OK) return st;
    ce->peer_flags[r] = p;
  }
  return TM_OK;
}

tm_status tm_ce_destroy(tm_ce_t ce) {
  if (!ce) return TM_ERR_INVALID_VALUE;
  if (ce->send) cudaStreamSynchronize(ce->send);
  if (ce->recv) cudaStreamSynchronize(ce->recv);
  for (auto& kv : ce->opened) cudaIpcCloseMemHandle(kv.second);
  for (int i = 0; i < kMaxChunksCe; ++i)
    if (ce->ev_chunk[i]) cudaEventDestroy(ce->ev_chunk[i]);
  if (ce->ev_start) cudaEventDestroy(ce->ev_start);
  if (ce->ev_send_done) cudaEventDestroy(ce->ev_send_done);
  if (ce->ev_recv_done) cudaEventDestroy(ce->ev_recv_done);
  if (ce->send) cudaStreamDestroy(ce->send);
  if (ce->recv) cudaStreamDestroy(ce->recv);
  if (ce->flags) cudaFree(ce->flags);
  delete ce;
  return TM_OK;
}

tm_status tm_ce_bytes_received(tm_ce_t ce, uint64_t* bytes) {
  if (!ce || !bytes) return TM_ERR_INVALID_VALUE;
  *bytes = ce->bytes_received;
  return TM_OK;
}

tm_status tm_sgemm_dist_ce(tm_ce_t ce, int64_t m, int64_t n, int64_t k, float alpha, const float* A_local,
                           int64_t lda, float* B, int64_t ldb, const tm_ipc_buf* all_B, int root, float beta,
                           float* C_local, int64_t ldc, int fused, void* stream_) {
  if (!ce || root < 0 || root >= ce->nranks || m < 0 || n < 0 || k < 0) return TM_ERR_INVALID_VALUE;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int P = ce->nranks, r = ce->rank;
  int64_t row0 = 0, rows = 0;
  tm_dist_rows(m, P, r, &row0, &rows);
  const bool reads_ab = alpha != 0.0f && k > 0 && n > 0;
  if (!reads_ab || P == 1) return tm_sgemm(rows, n, k, alpha, A_local, lda, B, ldb, beta, C_local, ldc, stream);
  if (!B || !all_B || ldb < (n > 1 ? n : 1)) return TM_ERR_INVALID_VALUE;
  if (static_cast<int>(ce->peer_flags.size()) != P) return TM_ERR_INVALID_VALUE;  // not connected
  const int pos = (r - root + P) % P;
  const int pred = pos > 0 ? (r - 1 + P) % P : -1;
  const int succ = pos < P - 1 ? (r + 1) % P : -1;
  float* succ_B = nullptr;
  if (succ >= 0) {
    void* p = nullptr;
    tm_status st = open_handle(ce, all_B[succ], &p);
    if (st != TM_OK) return st;
    succ_B = static_cast<float*>(p);
  }
  // pieces: kPieceRows K-rows (doubling if k is huge), aligned with the chunk
  // plan's boundaries (multiples of 512 but the end)
  int64_t piece = kPieceRows;
  while ((k + piece - 1) / piece > kMaxPieces) piece *= 2;
  const int npieces = static_cast<int>((k + piece - 1) / piece);
  int64_t nch = 0, kr_last = 0;
  tm_dist_chunk(k, P, -1, &nch, &kr_last);
  if (nch > kMaxChunksCe) return TM_ERR_INTERNAL;
  const unsigned epoch = ++ce->epoch;
  unsigned* flags = ce->flags;
  unsigned* pieces_in = flags + 1;
  nvtxRangePushA("tm_sgemm_dist_ce schedule");
  struct Pop {
    ~Pop() { nvtxRangePop(); }
  } pop;
  tm_status st = TM_OK;
  // 1. credit to the predecessor: my B is free for this call (stream-ordered
  //    after my previous GEMMs stopped reading it)
  if (pred >= 0 && (st = tmk::stream_write_u32(stream, static_cast<unsigned*>(ce->peer_flags[pred]), epoch)) != TM_OK)
    return st;
  if (cudaEventRecord(ce->ev_start, stream) != cudaSuccess) return TM_ERR_CUDA;
  // 2. send stream: push every piece to the successor once it is here and the
  //    successor has given its credit
  if (succ >= 0) {
    if (cudaStreamWaitEvent(ce->send, ce->ev_start, 0) != cudaSuccess) return TM_ERR_CUDA;
    if ((st = tmk::stream_wait_u32(ce->send, flags, epoch)) != TM_OK) return st;
    unsigned* succ_in = static_cast<unsigned*>(ce->peer_flags[succ]) + 1;
    for (int p = 0; p < npieces; ++p) {
      const int64_t k0 = p * piece, kr = std::min(piece, k - k0);
      if (pred >= 0 && (st = tmk::stream_wait_u32(ce->send, pieces_in + p, epoch)) != TM_OK) return st;
      const size_t bytes = static_cast<size_t>(kr) * static_cast<size_t>(ldb) * 4;
      if (cudaMemcpyAsync(succ_B + k0 * ldb, B + k0 * ldb, bytes, cudaMemcpyDeviceToDevice, ce->send) != cudaSuccess)
        return TM_ERR_CUDA;
      if ((st = tmk::stream_write_u32(ce->send, succ_in + p, epoch)) != TM_OK) return st;
    }
    if (cudaEventRecord(ce->ev_send_done, ce->send) != cudaSuccess) return TM_ERR_CUDA;
  }
  // 3. receive stream: chunk c is here once its last piece's flag is set
  //    (the predecessor pushes pieces in order on one stream)
  if (pred >= 0) {
    if (cudaStreamWaitEvent(ce->recv, ce->ev_start, 0) != cudaSuccess) return TM_ERR_CUDA;
    ce->bytes_received += static_cast<uint64_t>(k) * static_cast<uint64_t>(ldb) * 4;
  }
  // 4. compute on the caller's stream, every SM
  if (rows > 0 && fused) {
    tmk::GemmArgs ga{rows, n, k, alpha, beta, A_local, lda, B, ldb, C_local, ldc};
    if (!tmk::tc_plan_ok(ga)) fused = 0;
    if (fused) {
      if (pred >= 0) {
        ga.kflags = pieces_in;
        ga.kepoch = epoch;
        ga.kchunk = piece;
      }
      if ((st = tmk::sgemm_reserve(ga, stream, 0)) != TM_OK) return st;
    }
  }
  if (!fused) {
    for (int c = 0; c < nch; ++c) {
      int64_t k0 = 0, kr = 0;
      tm_dist_chunk(k, P, c, &k0, &kr);
      if (pred >= 0) {
        const int last_piece = static_cast<int>((k0 + kr - 1) / piece);
        if ((st = tmk::stream_wait_u32(ce->recv, pieces_in + last_piece, epoch)) != TM_OK) return st;
        if (cudaEventRecord(ce->ev_chunk[c], ce->recv) != cudaSuccess) return TM_ERR_CUDA;
        if (cudaStreamWaitEvent(stream, ce->ev_chunk[c], 0) != cudaSuccess) return TM_ERR_CUDA;
      }
      if (rows > 0) {
        tmk::GemmArgs ga{rows, n, kr, alpha, c == 0 ? beta : 1.0f, A_local + k0, lda, B + k0 * ldb, ldb, C_local, ldc};
        if ((st = tmk::sgemm_reserve(ga, stream, 0)) != TM_OK) return st;
      }
    }
  } else if (pred >= 0) {
    // the call completes only when all of B has arrived
    if ((st = tmk::stream_wait_u32(ce->recv, pieces_in + npieces - 1, epoch)) != TM_OK) return st;
  }
  // 5. join: B must not be touched by the caller before the pushes out of it
  //    (and into it) are complete
  if (pred >= 0) {
    if (cudaEventRecord(ce->ev_recv_done, ce->recv) != cudaSuccess) return TM_ERR_CUDA;
    if (cudaStreamWaitEvent(stream, ce->ev_recv_done, 0) != cudaSuccess) return TM_ERR_CUDA;
  }
  if (succ >= 0 && cudaStreamWaitEvent(stream, ce->ev_send_done, 0) != cudaSuccess) return TM_ERR_CUDA;
  return TM_OK;
}

}  // extern "C"
