// Cost table of every pruned candidate: for each query, every config of its
// pruned space in enumerate_candidates order (mapping.py:129-156) with its
// whole-plan KV bytes (plan_bytes, memory.py:164-195) and the critical-path
// delay of its plan under the prefill/decode cost model (call_latency,
// sim.py:84-92; independent calls dispatched with concurrency
// running_before + j as in sim.py:223-229, a map_reduce reducer after its
// mappers).  best_fit_select only needs the bytes (select.cu); this table is
// the north star's "evaluate every candidate" output for callers that weigh
// delay too.  Count pass (grid sizes) -> CUB exclusive scan -> fill pass with
// one warp per query, lanes strided over its grid.
#include <cub/device/device_scan.cuh>

#include "cost_model.cuh"

namespace rs {
namespace {

__global__ void cost_count_kernel(const rs_space* __restrict__ spaces, int64_t n, SelConst P,
                                  int64_t* __restrict__ counts) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= n; i += int64_t(gridDim.x) * blockDim.x)
    counts[i] = i < n ? Grid(spaces[i], P).G : 0;  // the scan's last output is the total
}

// Plan delay of one candidate.  With non-negative cost terms the latency is
// non-decreasing in the concurrency (each rounded step is monotone), so the
// max over the independent calls is the last call's latency — bit-identical
// to the sequential fmax; otherwise the calls are scanned.
__device__ __forceinline__ double plan_delay(int m, int64_t q, int64_t nc, int64_t il, int64_t c0, const SelConst& P) {
  if (m == RS_STUFF) return fmax(0.0, call_latency(q + nc * P.C + P.T, P.O, c0, P.a, P.b, P.s));
  const int64_t out = m == RS_MAP_RERANK ? P.O : il;
  double d = 0.0;
  if (P.a >= 0.0 && P.b >= 0.0 && P.s >= 0.0) {
    d = call_latency(q + P.C + P.T, out, c0 + nc - 1, P.a, P.b, P.s);
  } else {
    for (int64_t j = 0; j < nc; ++j) d = fmax(d, call_latency(q + P.C + P.T, out, c0 + j, P.a, P.b, P.s));
  }
  if (m == RS_MAP_REDUCE) d = __dadd_rn(d, call_latency(q + nc * il + P.T, P.O, c0, P.a, P.b, P.s));
  return d;
}

__global__ void __launch_bounds__(256) cost_fill_kernel(const rs_space* __restrict__ spaces,
                                                        const int32_t* __restrict__ qlen,
                                                        const int32_t* __restrict__ running, int64_t n, SelConst P,
                                                        const int64_t* __restrict__ offsets,
                                                        rs_candidate* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (qi >= n) return;
  const Grid gr(spaces[qi], P);
  const int64_t q = qlen[qi];
  const int64_t c0 = running ? running[qi] : 0;
  rs_candidate* dst = out + offsets[qi];
  const int64_t rr_call = buffered(q + P.C + P.T + P.O, P.pt);
  for (int64_t g = lane; g < gr.G; g += 32) {
    rs_config c{};
    gr.decode(g, P, c);
    const int64_t nc = c.num_chunks, il = c.interlen;
    rs_candidate x{};
    x.method = c.method;
    x.num_chunks = c.num_chunks;
    x.interlen = c.interlen;
    if (c.method == RS_MAP_RERANK)
      x.kv_bytes = nc * rr_call;
    else if (c.method == RS_STUFF)
      x.kv_bytes = buffered(q + nc * P.C + P.T + P.O, P.pt);
    else
      x.kv_bytes = nc * buffered(q + P.C + P.T + il, P.pt) + buffered(q + nc * il + P.T + P.O, P.pt);
    x.delay = P.has_cost ? plan_delay(c.method, q, nc, il, c0, P) : 0.0;
    dst[g] = x;
  }
}

size_t scan_temp_bytes(int64_t n) {
  size_t t = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, t, (const int64_t*)nullptr, (int64_t*)nullptr, int(n + 1));
  return t;
}
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// int64 range guard of the whole table (the per-query one of select.cu,
// evaluated on the host-visible bounds the kernel would hit)
__global__ void cost_guard_kernel(const rs_space* __restrict__ spaces, const int32_t* __restrict__ qlen, int64_t n,
                                  SelConst P, int32_t* __restrict__ bad) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const Grid gr(spaces[i], P);
    const int64_t nmax = gr.n_hi > P.max_chunks ? gr.n_hi : P.max_chunks;
    const int64_t per = P.C > gr.il_hi ? P.C : gr.il_hi;
    const int64_t tail = P.O > gr.il_hi ? P.O : gr.il_hi;
    const int64_t tmax = int64_t(qlen[i]) + nmax * per + P.T + tail;
    bool b = nmax > 65535 || per > (int64_t(1) << 30) || tmax > P.tok_limit;
    if (!b) b = buffered(tmax, P.pt) > (int64_t)(INT64_MAX / 2) / (nmax + 1);
    if (b) atomicExch(bad, 1);
  }
}

}  // namespace
}  // namespace rs

extern "C" size_t rs_candidate_costs_workspace_size(int64_t n) {
  if (n < 0) n = 0;
  return rs::align256(sizeof(int64_t) * (n + 1)) + rs::align256(rs::scan_temp_bytes(n));
}

extern "C" int rs_candidate_costs(const rs_space* spaces, const int32_t* qlen, const int32_t* running_before,
                                  int64_t n, const rs_select_params* params, const rs_cost_model* cost,
                                  int64_t* offsets, rs_candidate* out, void* workspace, size_t workspace_bytes,
                                  void* stream) {
  using namespace rs;
  RS_REQUIRE(n >= 0 && n < (int64_t(1) << 31), "n out of range");
  RS_REQUIRE(offsets != nullptr, "offsets is NULL");
  SelConst P;
  int rc = make_const(params, cost, &P);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    RS_CHECK_CUDA(cudaMemsetAsync(offsets, 0, sizeof(int64_t), st), "cudaMemsetAsync");
    return RS_OK;
  }
  RS_REQUIRE(spaces && qlen, "NULL device pointer");
  const unsigned blocks = unsigned(std::min<int64_t>(ceil_div(n + 1, 256), 4096));
  if (out == nullptr) {
    RS_REQUIRE(workspace && workspace_bytes >= rs_candidate_costs_workspace_size(n), "workspace too small");
    int64_t* counts = reinterpret_cast<int64_t*>(workspace);
    void* temp = static_cast<char*>(workspace) + align256(sizeof(int64_t) * (n + 1));
    size_t temp_bytes = scan_temp_bytes(n);
    cost_count_kernel<<<blocks, 256, 0, st>>>(spaces, n, P, counts);
    RS_CHECK_LAUNCH("cost_count_kernel");
    RS_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, counts, offsets, int(n + 1), st),
                  "cub::DeviceScan::ExclusiveSum");
    count_launch();
    return RS_OK;
  }
  int32_t* bad = reinterpret_cast<int32_t*>(workspace);
  RS_REQUIRE(workspace && workspace_bytes >= sizeof(int32_t), "workspace too small");
  RS_CHECK_CUDA(cudaMemsetAsync(bad, 0, sizeof(int32_t), st), "cudaMemsetAsync");
  cost_guard_kernel<<<blocks, 256, 0, st>>>(spaces, qlen, n, P, bad);
  RS_CHECK_LAUNCH("cost_guard_kernel");
  int32_t hbad = 0;
  RS_CHECK_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync");
  RS_CHECK_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  if (hbad) {
    set_error("KV byte arithmetic exceeds int64 for some query of the batch");
    return RS_ERR_OVERFLOW;
  }
  cost_fill_kernel<<<unsigned(ceil_div(n * 32, 256)), 256, 0, st>>>(spaces, qlen, running_before, n, P, offsets,
                                                                    out);
  RS_CHECK_LAUNCH("cost_fill_kernel");
  return RS_OK;
}
