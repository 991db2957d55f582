// K4 gate_prune: the confidence gate + Algorithm-1 pruning for a batch,
// bit-exact with applying the reference gate to the queries IN ORDER:
//   gate_profile      profiler.py:467-486   map_profile     mapping.py:106-126
//   RecentSpaceWindow profiler.py:138-153   hull_of_spaces  mapping.py:180-200
//
// The only serial coupling is the window: a rejected query sees the hull of
// the last <= 10 ACCEPTED spaces before it (plus the carried-in window).  The
// window contents are a pure function of the accepted-query ranks, so the
// batch is solved with a scan instead of a loop:
//   1. map + accept flags + per-block accept counts      (one thread / query)
//   2. exclusive scan of the block counts                (one block)
//   3. per-query accepted rank, compaction of accepted indices
//   4. hull over the <= 10 predecessors for rejected queries, new window.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rs_common.cuh"

namespace rs {
namespace {

constexpr int kBlock = 1024;

struct GateWs {  // carved out of the caller's workspace
  int32_t* flag;    // [n]   accepted?
  int32_t* rank;    // [n]   accepted queries strictly before i (within batch)
  int32_t* acc_idx; // [n]   index of the r-th accepted query
  int32_t* block;   // [nb+1] block counts -> exclusive offsets, [nb] = total
  rs_window* carry; // copy of the carried-in window
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

size_t ws_layout(int64_t n, char* base, GateWs* ws) {
  const int64_t nb = ceil_div(n > 0 ? n : 1, kBlock);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* p = base ? base + off : nullptr;
    off = align_up(off + bytes);
    return p;
  };
  GateWs w{};
  w.flag = (int32_t*)take(sizeof(int32_t) * n);
  w.rank = (int32_t*)take(sizeof(int32_t) * n);
  w.acc_idx = (int32_t*)take(sizeof(int32_t) * n);
  w.block = (int32_t*)take(sizeof(int32_t) * (nb + 1));
  w.carry = (rs_window*)take(sizeof(rs_window));
  if (ws) *ws = w;
  return off;
}

__device__ __forceinline__ rs_space map_profile(const rs_profile& p, int max_chunks) {
  // mapping.py:106-126: methods by (joint, complexity); chunks [p, 3p]
  // clamped to [1, max_chunks] (IntRange.clamp_to, types.py:53-54)
  rs_space s{};
  if (!p.needs_joint_reasoning)
    s.methods = RS_MAP_RERANK;
  else if (!p.complexity_high)
    s.methods = RS_STUFF;
  else
    s.methods = RS_STUFF | RS_MAP_REDUCE;
  const int lo = p.pieces_required, hi = 3 * int(p.pieces_required);
  s.num_chunks_lo = (uint16_t)min(max(lo, 1), max_chunks);
  s.num_chunks_hi = (uint16_t)min(max(hi, 1), max_chunks);
  if (s.methods & RS_MAP_REDUCE) {
    s.interlen_lo = p.summary_lo;
    s.interlen_hi = p.summary_hi;
  }
  return s;
}

__global__ void __launch_bounds__(kBlock) gate_map_kernel(const rs_profile* __restrict__ prof, int64_t n,
                                                          double thr, int max_chunks,
                                                          rs_space* __restrict__ out, GateWs ws) {
  const int64_t i = int64_t(blockIdx.x) * kBlock + threadIdx.x;
  int acc = 0;
  if (i < n) {
    const rs_profile p = prof[i];
    acc = p.confidence >= thr;  // profiler.py:481, IEEE double compare
    if (acc) out[i] = map_profile(p, max_chunks);
    ws.flag[i] = acc;
  }
  const int cnt = __syncthreads_count(acc);
  if (threadIdx.x == 0) ws.block[blockIdx.x] = cnt;
}

__global__ void __launch_bounds__(kBlock) gate_scan_kernel(GateWs ws, int64_t nb,
                                                           const rs_window* __restrict__ window_in) {
  __shared__ int32_t warp_sums[32];
  __shared__ int32_t carry;
  if (threadIdx.x == 0) carry = 0;
  if (threadIdx.x == 0) *ws.carry = *window_in;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < nb; base += kBlock) {
    const int64_t j = base + threadIdx.x;
    const int32_t v = j < nb ? ws.block[j] : 0;
    int32_t x = v;  // inclusive warp scan
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) warp_sums[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int32_t w = warp_sums[lane];
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, off);
        if (lane >= off) w += y;
      }
      warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int32_t excl = carry + (wid ? warp_sums[wid - 1] : 0) + x - v;
    if (j < nb) ws.block[j] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) ws.block[nb] = carry;
}

__global__ void __launch_bounds__(kBlock) gate_rank_kernel(int64_t n, GateWs ws) {
  __shared__ int32_t warp_cnt[32];
  const int64_t i = int64_t(blockIdx.x) * kBlock + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int acc = (i < n) ? ws.flag[i] : 0;
  const unsigned bal = __ballot_sync(0xffffffffu, acc);
  if (lane == 0) warp_cnt[wid] = __popc(bal);
  __syncthreads();
  if (wid == 0) {
    int32_t w = warp_cnt[lane];
    int32_t x = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    warp_cnt[lane] = x - w;  // exclusive over warps
  }
  __syncthreads();
  if (i < n) {
    const int32_t r = ws.block[blockIdx.x] + warp_cnt[wid] + __popc(bal & ((1u << lane) - 1u));
    ws.rank[i] = r;
    if (acc) ws.acc_idx[r] = (int32_t)i;
  }
}

__device__ __forceinline__ const rs_space& window_entry(int64_t t, int32_t w0, const rs_window& carry,
                                                        const int32_t* acc_idx, const rs_space* out) {
  // entry t of (carried window ++ batch accepted spaces)
  return t < w0 ? carry.spaces[t] : out[acc_idx[t - w0]];
}

__global__ void __launch_bounds__(kBlock) gate_hull_kernel(int64_t n, GateWs ws, rs_space dflt,
                                                           rs_space* __restrict__ out,
                                                           rs_window* __restrict__ window_out) {
  const int64_t i = int64_t(blockIdx.x) * kBlock + threadIdx.x;
  const rs_window& carry = *ws.carry;
  const int32_t w0 = carry.len;
  if (i < n && !ws.flag[i]) {
    const int64_t end = int64_t(w0) + ws.rank[i];
    const int64_t beg = end > RS_WINDOW_CAPACITY ? end - RS_WINDOW_CAPACITY : 0;
    rs_space s;
    if (end == 0) {
      s = dflt;  // `window.hull() or default_space` (profiler.py:485)
    } else {
      const rs_space& f = window_entry(beg, w0, carry, ws.acc_idx, out);
      int m = 0, lo = f.num_chunks_lo, hi = f.num_chunks_hi, a = -1, b = -1;
      for (int64_t t = beg; t < end; ++t) {
        const rs_space& e = window_entry(t, w0, carry, ws.acc_idx, out);
        m |= e.methods;
        lo = min(lo, (int)e.num_chunks_lo);
        hi = max(hi, (int)e.num_chunks_hi);
        if (e.methods & RS_MAP_REDUCE) {
          a = a < 0 ? e.interlen_lo : min(a, (int)e.interlen_lo);
          b = b < 0 ? e.interlen_hi : max(b, (int)e.interlen_hi);
        }
      }
      s = rs_space{};
      s.methods = (uint16_t)m;
      s.num_chunks_lo = (uint16_t)lo;
      s.num_chunks_hi = (uint16_t)hi;
      if (m & RS_MAP_REDUCE) {  // mapping.py:196-199
        s.interlen_lo = (uint16_t)(a < 0 ? 30 : a);
        s.interlen_hi = (uint16_t)(a < 0 ? 200 : b);
      }
    }
    s.gate_fallback = 1;
    s.reserved = 0;
    out[i] = s;
  }
  if (i == 0) {
    // window after the batch: last <= 10 of (carried ++ all accepted)
    const int64_t total = int64_t(w0) + ws.block[gridDim.x];
    const int64_t beg = total > RS_WINDOW_CAPACITY ? total - RS_WINDOW_CAPACITY : 0;
    rs_window w{};
    for (int64_t t = beg; t < total; ++t) {
      rs_space e = window_entry(t, w0, carry, ws.acc_idx, out);
      e.gate_fallback = 0;
      w.spaces[t - beg] = e;
    }
    w.len = (int32_t)(total - beg);
    *window_out = w;
  }
}

// Batches of <= kBlock queries (and the scalar drop-in, n = 1): the four
// steps above in ONE block and one launch — accept flags, the block-wide
// exclusive scan of the accepted ranks, the compaction and the hulls all in
// shared memory.
__global__ void __launch_bounds__(kBlock) gate_small_kernel(const rs_profile* __restrict__ prof, int n, double thr,
                                                            int max_chunks, rs_space dflt,
                                                            rs_space* __restrict__ out,
                                                            rs_window* __restrict__ window_io) {
  __shared__ rs_space s_sp[kBlock];   // accepted spaces by batch index
  __shared__ int32_t s_acc_idx[kBlock];
  __shared__ int32_t warp_cnt[32];
  __shared__ int32_t s_total;
  __shared__ rs_window carry;
  const int i = threadIdx.x;
  const int lane = i & 31, wid = i >> 5;
  if (i == 0) carry = *window_io;
  int acc = 0;
  if (i < n) {
    const rs_profile p = prof[i];
    acc = p.confidence >= thr;  // profiler.py:481, IEEE double compare
    if (acc) {
      const rs_space sp = map_profile(p, max_chunks);
      s_sp[i] = sp;
      out[i] = sp;
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, acc);
  if (lane == 0) warp_cnt[wid] = __popc(bal);
  __syncthreads();
  if (wid == 0) {
    const int32_t w = warp_cnt[lane];
    int32_t x = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    warp_cnt[lane] = x - w;  // exclusive over warps
    if (lane == 31) s_total = x;
  }
  __syncthreads();
  const int32_t rank = warp_cnt[wid] + __popc(bal & ((1u << lane) - 1u));
  if (acc) s_acc_idx[rank] = i;
  __syncthreads();
  const int32_t total_acc = s_total;
  const int32_t w0 = carry.len;
  auto entry = [&](int32_t t) -> const rs_space& { return t < w0 ? carry.spaces[t] : s_sp[s_acc_idx[t - w0]]; };
  if (i < n && !acc) {
    const int32_t end = w0 + rank;
    const int32_t beg = end > RS_WINDOW_CAPACITY ? end - RS_WINDOW_CAPACITY : 0;
    rs_space s;
    if (end == 0) {
      s = dflt;  // `window.hull() or default_space` (profiler.py:485)
    } else {
      const rs_space& f = entry(beg);
      int m = 0, lo = f.num_chunks_lo, hi = f.num_chunks_hi, a = -1, b = -1;
      for (int32_t t = beg; t < end; ++t) {
        const rs_space& e = entry(t);
        m |= e.methods;
        lo = min(lo, (int)e.num_chunks_lo);
        hi = max(hi, (int)e.num_chunks_hi);
        if (e.methods & RS_MAP_REDUCE) {
          a = a < 0 ? e.interlen_lo : min(a, (int)e.interlen_lo);
          b = b < 0 ? e.interlen_hi : max(b, (int)e.interlen_hi);
        }
      }
      s = rs_space{};
      s.methods = (uint16_t)m;
      s.num_chunks_lo = (uint16_t)lo;
      s.num_chunks_hi = (uint16_t)hi;
      if (m & RS_MAP_REDUCE) {  // mapping.py:196-199
        s.interlen_lo = (uint16_t)(a < 0 ? 30 : a);
        s.interlen_hi = (uint16_t)(a < 0 ? 200 : b);
      }
    }
    s.gate_fallback = 1;
    s.reserved = 0;
    out[i] = s;
  }
  if (i == 0) {
    const int32_t total = w0 + total_acc;
    const int32_t beg = total > RS_WINDOW_CAPACITY ? total - RS_WINDOW_CAPACITY : 0;
    rs_window w{};
    for (int32_t t = beg; t < total; ++t) {
      rs_space e = entry(t);
      e.gate_fallback = 0;
      w.spaces[t - beg] = e;
    }
    w.len = total - beg;
    *window_io = w;
  }
}

}  // namespace
}  // namespace rs

extern "C" size_t rs_prune_gate_workspace_size(int64_t n) {
  return rs::ws_layout(n < 0 ? 0 : n, nullptr, nullptr);
}

extern "C" int rs_prune_gate(const rs_profile* profiles, int64_t n, const rs_gate_params* params,
                             rs_window* window_io, rs_space* spaces_out, void* workspace,
                             size_t workspace_bytes, void* stream) {
  using namespace rs;
  RS_REQUIRE(params != nullptr, "params is NULL");
  RS_REQUIRE(params->threshold > 0.0 && params->threshold <= 1.0,
             "threshold must be in (0, 1], got %g", params->threshold);
  RS_REQUIRE(params->max_chunks >= 1, "max_chunks must be >= 1");
  RS_REQUIRE(n >= 0 && n < (int64_t(1) << 31), "n out of range");
  if (n == 0) return RS_OK;
  RS_REQUIRE(profiles && window_io && spaces_out && workspace, "NULL device pointer");
  GateWs ws;
  const size_t need = ws_layout(n, (char*)workspace, &ws);
  RS_REQUIRE(workspace_bytes >= need, "workspace too small (%zu < %zu)", workspace_bytes, need);
  cudaStream_t st = as_stream(stream);
  rs_space dflt = params->default_space;
  dflt.gate_fallback = 1;
  if (n <= kBlock) {  // one block, one launch
    gate_small_kernel<<<1, kBlock, 0, st>>>(profiles, int(n), params->threshold, params->max_chunks, dflt,
                                            spaces_out, window_io);
    RS_CHECK_LAUNCH("gate_small_kernel");
    return RS_OK;
  }
  const int64_t nb = ceil_div(n, kBlock);
  gate_map_kernel<<<(unsigned)nb, kBlock, 0, st>>>(profiles, n, params->threshold, params->max_chunks,
                                                  spaces_out, ws);
  RS_CHECK_LAUNCH("gate_map_kernel");
  gate_scan_kernel<<<1, kBlock, 0, st>>>(ws, nb, window_io);
  RS_CHECK_LAUNCH("gate_scan_kernel");
  gate_rank_kernel<<<(unsigned)nb, kBlock, 0, st>>>(n, ws);
  RS_CHECK_LAUNCH("gate_rank_kernel");
  gate_hull_kernel<<<(unsigned)nb, kBlock, 0, st>>>(n, ws, dflt, spaces_out, window_io);
  RS_CHECK_LAUNCH("gate_hull_kernel");
  return RS_OK;
}
