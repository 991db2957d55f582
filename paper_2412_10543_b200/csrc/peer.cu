// Peer-memory exchange of the corpus-sharded search.
//
// The sharded path scores every query against every rank's corpus shard, so
// query q's P sorted lists live on P GPUs; rank r merges the queries of its
// slice [r*nq/P, (r+1)*nq/P).  Instead of a NCCL all-to-all, each rank's
// scatter kernel stores its key rows directly into the owners' receive
// regions (CUDA IPC mappings: NVLink / NVSwitch stores for remote owners,
// local stores for itself) and the last block to finish raises this rank's
// epoch flag in every region; the owner's merge kernel (retrieval.cu,
// merge_topk64_kernel<true>) waits on the P flags in-kernel and reads the
// lists with ld.global.cv.  Keys are 8 bytes (distance bits << 32 | id), so
// a region's list for (parity, source) is [slice_cap][k] uint64.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>

#include "retrieval.cuh"

namespace rs {
namespace {

// One thread per key; consecutive threads walk a row, and rows of one owner
// are contiguous at the destination, so the remote stores coalesce.
__global__ void __launch_bounds__(256) peer_scatter_kernel(const uint64_t* __restrict__ keys, int64_t nq,
                                                           const __grid_constant__ rs_peer_exchange ex,
                                                           uint32_t epoch) {
  const int k = ex.k;
  const int64_t total = nq * k;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = t / k;
    peer_row(ex, nq, q, epoch)[t - q * k] = keys[t];
  }
  peer_signal(ex, epoch);
}


}  // namespace

int check_peer_exchange(const rs_peer_exchange* ex) {
  RS_REQUIRE(ex != nullptr, "exchange is NULL");
  RS_REQUIRE(ex->world >= 1 && ex->world <= RS_PEER_MAX, "world out of range (%d)", ex->world);
  RS_REQUIRE(ex->rank >= 0 && ex->rank < ex->world, "rank out of range (%d)", ex->rank);
  RS_REQUIRE(ex->k >= 1 && ex->k <= 255, "k out of range (%d)", ex->k);
  RS_REQUIRE(ex->slice_cap >= 1, "slice_cap must be positive");
  for (int r = 0; r < ex->world; ++r) RS_REQUIRE(ex->region[r] != nullptr, "region %d is NULL", r);
  return RS_OK;
}

int launch_peer_scatter(const rs_peer_exchange& ex, const uint64_t* keys, int64_t nq, uint32_t epoch,
                        cudaStream_t st) {
  // nq == 0 still launches one block: the flags must advance with the epoch
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(nq * ex.k, 256), 148 * 4));
  peer_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(keys, nq, ex, epoch);
  RS_CHECK_LAUNCH("peer_scatter_kernel");
  return RS_OK;
}

}  // namespace rs

extern "C" int rs_peer_region_bytes(int32_t world, int64_t slice_cap, int32_t k, uint64_t* bytes) {
  RS_REQUIRE(world >= 1 && world <= RS_PEER_MAX && slice_cap >= 1 && k >= 1 && bytes, "bad arguments");
  *bytes = rs::kPeerKeysOff + 2ull * uint64_t(world) * uint64_t(slice_cap) * uint64_t(k) * 8ull;
  return RS_OK;
}

extern "C" int rs_peer_alloc(uint64_t bytes, int32_t device, void** region, void* ipc_handle) {
  RS_REQUIRE(bytes >= rs::kPeerKeysOff && region && ipc_handle, "bad arguments");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  rs::DeviceGuard g(device);
  void* p = nullptr;
  RS_CHECK_CUDA(cudaMalloc(&p, bytes), "cudaMalloc(peer region)");
  cudaError_t e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();  // zeroed before any peer can map it
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    rs::set_error("peer region: %s", cudaGetErrorString(e));
    return RS_ERR_CUDA;
  }
  memcpy(ipc_handle, &h, sizeof(h));
  *region = p;
  return RS_OK;
}

extern "C" int rs_peer_open(const void* ipc_handle, int32_t device, void** region) {
  RS_REQUIRE(ipc_handle && region, "bad arguments");
  rs::DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  void* p = nullptr;
  RS_CHECK_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  *region = p;
  return RS_OK;
}

extern "C" int rs_peer_close(void* region) {
  RS_REQUIRE(region, "region is NULL");
  RS_CHECK_CUDA(cudaIpcCloseMemHandle(region), "cudaIpcCloseMemHandle");
  return RS_OK;
}

extern "C" int rs_peer_free(void* region) {
  RS_REQUIRE(region, "region is NULL");
  RS_CHECK_CUDA(cudaFree(region), "cudaFree(peer region)");
  return RS_OK;
}

extern "C" int rs_peer_scatter_keys(const rs_peer_exchange* ex, const uint64_t* keys, int64_t nq, uint32_t epoch,
                                    void* stream) {
  int rc = rs::check_peer_exchange(ex);
  if (rc) return rc;
  RS_REQUIRE(nq >= 0 && (nq == 0 || keys), "bad arguments");
  RS_REQUIRE(rs::ceil_div(nq, ex->world) <= ex->slice_cap, "nq %lld exceeds world x slice_cap", (long long)nq);
  return rs::launch_peer_scatter(*ex, keys, nq, epoch, rs::as_stream(stream));
}

extern "C" int rs_peer_merge_topk(const rs_peer_exchange* ex, int64_t nq, uint32_t epoch, int32_t k,
                                  const rs_config* cfg, float* D, int64_t* I, int32_t timeout_ms, void* stream) {
  int rc = rs::check_peer_exchange(ex);
  if (rc) return rc;
  RS_REQUIRE(nq >= 0 && k >= 1 && k <= 128 && timeout_ms >= 0, "bad arguments");
  RS_REQUIRE(rs::ceil_div(nq, ex->world) <= ex->slice_cap, "nq %lld exceeds world x slice_cap", (long long)nq);
  const int64_t q0 = (int64_t(ex->rank) * nq) / ex->world, q1 = (int64_t(ex->rank + 1) * nq) / ex->world;
  // an empty slice still waits: the next exchange may reuse a parity buffer
  // only after every rank's merge of this one has seen all sources arrive
  RS_REQUIRE(q1 == q0 || (D && I), "D/I are NULL");
  void* own = ex->region[ex->rank];
  rs::PeerWait pw;
  pw.flags = rs::peer_flags(own);
  pw.n = ex->world;
  pw.epoch = epoch;
  pw.error = rs::peer_error(own);
  pw.timeout_ns = uint64_t(timeout_ms ? timeout_ms : 60000) * 1000000ull;
  const uint64_t* lists = rs::peer_keys(own) + int64_t(epoch & 1u) * ex->world * ex->slice_cap * ex->k;
  return rs::launch_merge_wait(lists, q1 - q0, ex->world, ex->k, /*list_stride=*/ex->slice_cap * ex->k,
                               /*q_stride=*/ex->k, k, cfg, D, I, pw, rs::as_stream(stream));
}

extern "C" int rs_peer_error(const rs_peer_exchange* ex, int32_t clear, int32_t* error) {
  int rc = rs::check_peer_exchange(ex);
  if (rc) return rc;
  RS_REQUIRE(error, "error is NULL");
  int32_t* e = rs::peer_error(ex->region[ex->rank]);
  RS_CHECK_CUDA(cudaMemcpy(error, e, sizeof(int32_t), cudaMemcpyDeviceToHost), "read peer error");
  if (clear) RS_CHECK_CUDA(cudaMemset(e, 0, sizeof(int32_t)), "clear peer error");
  return RS_OK;
}
