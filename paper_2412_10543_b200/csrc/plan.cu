// §8(f2): per-call expansion of chosen configs — memory.plan_calls
// (memory.py:89-150) for a batch, as a CSR of rs_call records.
//   stuff       1 SINGLE call over the concatenated chunks
//   map_rerank  n RERANK calls, one per chunk
//   map_reduce  n MAPPER calls producing `interlen` tokens + 1 REDUCER that
//               depends on all mappers
// with the reference's checks in its order: InvalidChunkCount, positive
// interlen, then each call's context-window check (memory.py:81-86).
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rs_common.cuh"

namespace rs {
namespace {

struct PlanConst {
  int64_t pt, C, T, O, max_ctx;
  int32_t max_chunks;
};

enum : uint8_t { K_SINGLE = 0, K_MAPPER = 1, K_REDUCER = 2, K_RERANK = 3 };

__device__ __forceinline__ int64_t buffered(int64_t tokens, int64_t pt) { return (102 * tokens * pt + 99) / 100; }

// number of calls of query i's plan (0 when the reference raises / no config)
__device__ __forceinline__ int64_t plan_count(const rs_config& c, int64_t q, const PlanConst& P, uint8_t& st) {
  if (c.status != RS_SELECT_BEST_FIT && c.status != RS_SELECT_FALLBACK) {
    st = RS_PLAN_NONE;
    return 0;
  }
  const int64_t n = c.num_chunks;
  if (n < 1 || n > P.max_chunks) {
    st = RS_PLAN_INVALID_CHUNKS;
    return 0;
  }
  st = RS_PLAN_OK;
  if (c.method == RS_STUFF) {
    if (q + n * P.C + P.T + P.O > P.max_ctx) st = RS_PLAN_CONTEXT_OVERFLOW;
    return st == RS_PLAN_OK ? 1 : 0;
  }
  if (c.method == RS_MAP_RERANK) {
    if (q + P.C + P.T + P.O > P.max_ctx) st = RS_PLAN_CONTEXT_OVERFLOW;
    return st == RS_PLAN_OK ? n : 0;
  }
  const int64_t il = c.interlen;
  if (il <= 0) {
    st = RS_PLAN_BAD_INTERLEN;
    return 0;
  }
  if (q + P.C + P.T + il > P.max_ctx || q + n * il + P.T + P.O > P.max_ctx) st = RS_PLAN_CONTEXT_OVERFLOW;
  return st == RS_PLAN_OK ? n + 1 : 0;
}

__global__ void plan_count_kernel(const rs_config* __restrict__ cfg, const int32_t* __restrict__ qlen, int64_t n,
                                  PlanConst P, int64_t* __restrict__ counts, uint8_t* __restrict__ status) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n; i += int64_t(gridDim.x) * blockDim.x) {
    if (i == n) {
      counts[i] = 0;  // the scan's last output is the total
      continue;
    }
    uint8_t st;
    counts[i] = plan_count(cfg[i], qlen[i], P, st);
    if (status) status[i] = st;
  }
}

__global__ void plan_fill_kernel(const rs_config* __restrict__ cfg, const int32_t* __restrict__ qlen, int64_t n,
                                 PlanConst P, const int64_t* __restrict__ offsets, rs_call* __restrict__ calls,
                                 int64_t* __restrict__ total) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const rs_config c = cfg[i];
    const int64_t q = qlen[i];
    rs_call* out = calls + offsets[i];
    const int64_t cnt = offsets[i + 1] - offsets[i];
    int64_t sum = 0;
    if (cnt > 0) {
      const int64_t nc = c.num_chunks;
      rs_call x{};
      if (c.method == RS_STUFF) {
        x.prompt_tokens = int32_t(q + nc * P.C + P.T);
        x.max_output_tokens = int32_t(P.O);
        x.kv_bytes = buffered(x.prompt_tokens + P.O, P.pt);
        x.kind = K_SINGLE;
        out[0] = x;
        sum = x.kv_bytes;
      } else if (c.method == RS_MAP_RERANK) {
        x.prompt_tokens = int32_t(q + P.C + P.T);
        x.max_output_tokens = int32_t(P.O);
        x.kv_bytes = buffered(x.prompt_tokens + P.O, P.pt);
        x.kind = K_RERANK;
        for (int64_t j = 0; j < nc; ++j) {
          x.index = uint16_t(j);
          out[j] = x;
        }
        sum = nc * x.kv_bytes;
      } else {
        const int64_t il = c.interlen;
        x.prompt_tokens = int32_t(q + P.C + P.T);
        x.max_output_tokens = int32_t(il);
        x.kv_bytes = buffered(x.prompt_tokens + il, P.pt);
        x.kind = K_MAPPER;
        for (int64_t j = 0; j < nc; ++j) {
          x.index = uint16_t(j);
          out[j] = x;
        }
        rs_call r{};
        r.prompt_tokens = int32_t(q + nc * il + P.T);
        r.max_output_tokens = int32_t(P.O);
        r.kv_bytes = buffered(r.prompt_tokens + P.O, P.pt);
        r.kind = K_REDUCER;
        r.index = 0;  // LlmCall default index (memory.py:540-547)
        out[nc] = r;
        sum = nc * x.kv_bytes + r.kv_bytes;
      }
    }
    if (total) total[i] = sum;
  }
}

size_t cub_temp_bytes(int64_t n) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int64_t*)nullptr, (int64_t*)nullptr, int(n + 1));
  return t;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace
}  // namespace rs

extern "C" size_t rs_plan_calls_workspace_size(int64_t n) {
  if (n < 0) n = 0;
  return rs::align256(sizeof(int64_t) * (n + 1)) + rs::align256(rs::cub_temp_bytes(n));
}

extern "C" int rs_plan_calls(const rs_config* configs, const int32_t* qlen, int64_t n, const rs_select_params* p,
                             int64_t max_context_tokens, int64_t* offsets, rs_call* calls, int64_t* total_bytes,
                             uint8_t* status, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace rs;
  RS_REQUIRE(p != nullptr, "params is NULL");
  RS_REQUIRE(p->out_budget > 0, "out_budget must be positive");
  RS_REQUIRE(p->per_token_bytes > 0 && p->chunk_size > 0 && p->template_tokens >= 0 && p->max_chunks >= 1,
             "bad select params");
  RS_REQUIRE(max_context_tokens > 0, "max_context_tokens must be positive");
  RS_REQUIRE(n >= 0 && n < (int64_t(1) << 31), "n out of range");
  RS_REQUIRE(offsets != nullptr, "offsets is NULL");
  if (n == 0) {
    RS_CHECK_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t), as_stream(stream)), "cudaMemsetAsync");
    return RS_OK;
  }
  RS_REQUIRE(configs && qlen, "NULL device pointer");
  RS_REQUIRE(workspace && workspace_bytes >= rs_plan_calls_workspace_size(n), "workspace too small");
  PlanConst P{p->per_token_bytes, p->chunk_size, p->template_tokens, p->out_budget, max_context_tokens,
              p->max_chunks};
  cudaStream_t st = as_stream(stream);
  const unsigned blocks = unsigned(std::min<int64_t>(ceil_div(n + 1, 256), 4096));
  if (calls == nullptr) {
    int64_t* counts = reinterpret_cast<int64_t*>(workspace);
    void* temp = static_cast<char*>(workspace) + align256(sizeof(int64_t) * (n + 1));
    size_t temp_bytes = cub_temp_bytes(n);
    plan_count_kernel<<<blocks, 256, 0, st>>>(configs, qlen, n, P, counts, status);
    RS_CHECK_LAUNCH("plan_count_kernel");
    RS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offsets, int(n + 1), st),
                  "cub::DeviceScan::ExclusiveSum");
    count_launch();
    return RS_OK;
  }
  plan_fill_kernel<<<blocks, 256, 0, st>>>(configs, qlen, n, P, offsets, calls, total_bytes);
  RS_CHECK_LAUNCH("plan_fill_kernel");
  return RS_OK;
}
