// Shared device pieces of the config path's cost model (select.cu,
// costs.cu): the selection scalars, the exact int64 KV-byte model
// (memory.py:70-78), the IEEE-exact call latency (sim.py:84-92) and the
// candidate grid of a pruned space (mapping.py:129-156).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ragsched_b200.h"
#include "rs_common.cuh"

namespace rs {

struct SelConst {
  int64_t pt;        // per-token bytes
  int64_t C, T, O;   // chunk size, template tokens, out budget
  int64_t tok_limit; // largest token count whose 102*tok*pt+99 fits int64
  int64_t pa;        // 102*pt = 100*pa + pb (the fast exact form of buffered())
  int32_t pb;
  int32_t max_chunks, cstep, istep, allow_fallback;
  int32_t has_cost;
  double a, b, s;    // CostModel
};

__device__ __forceinline__ int64_t buffered(int64_t tokens, int64_t pt) {
  return (102 * tokens * pt + 99) / 100;  // memory.py:76-78
}

// The same value without a 64-bit division: with 102*pt = 100*pa + pb,
// (102*pt*t + 99) / 100 = pa*t + (pb*t + 99) / 100 exactly (100*pa*t is a
// multiple of 100); pb*t + 99 fits uint32 for t < kFastTok.
constexpr int64_t kFastTok = 20000000;
__device__ __forceinline__ int64_t buffered_fast(int32_t t, int64_t pa, int32_t pb) {
  return pa * int64_t(t) + int64_t((uint32_t(pb) * uint32_t(t) + 99u) / 100u);
}

// sim.py:84-92 in the reference's IEEE-double evaluation order, no FMA.
__device__ __forceinline__ double call_latency(int64_t prompt, int64_t out, int64_t conc, double a,
                                               double b, double s) {
  const double prefill = __dmul_rn(a, __ll2double_rn(prompt));
  const double dil = __dadd_rn(1.0, __dmul_rn(s, __ll2double_rn(conc)));
  const double decode = __dmul_rn(__dmul_rn(__ll2double_rn(out), b), dil);
  return __dadd_rn(prefill, decode);
}

// Grid of one pruned space (enumerate_candidates, mapping.py:129-156, with
// IntRange.values(step), types.py:59-60): method-major RR, ST, MR; n
// ascending; il ascending inside MR.  Flat index g -> config without
// materialising the list.
struct Grid {
  int m;
  int64_t n_lo, n_hi, il_lo, il_hi, nn, ni, n_rr, n_st, G;
  __device__ __forceinline__ Grid(const rs_space& sp, const SelConst& P) {
    m = sp.methods;
    n_lo = sp.num_chunks_lo;
    n_hi = sp.num_chunks_hi;
    il_lo = sp.interlen_lo;
    il_hi = sp.interlen_hi;
    nn = (n_hi >= n_lo) ? (n_hi - n_lo) / P.cstep + 1 : 0;
    ni = ((m & RS_MAP_REDUCE) && il_hi >= il_lo) ? (il_hi - il_lo) / P.istep + 1 : 0;
    n_rr = (m & RS_MAP_RERANK) ? nn : 0;
    n_st = (m & RS_STUFF) ? nn : 0;
    G = n_rr + n_st + nn * ni;
  }
  __device__ __forceinline__ void decode(int64_t g, const SelConst& P, rs_config& c) const {
    if (g < n_rr) {
      c.method = RS_MAP_RERANK;
      c.num_chunks = (uint16_t)(n_lo + g * P.cstep);
    } else if (g < n_rr + n_st) {
      c.method = RS_STUFF;
      c.num_chunks = (uint16_t)(n_lo + (g - n_rr) * P.cstep);
    } else {
      const int64_t r = g - n_rr - n_st;
      const int64_t i_n = r / ni;
      c.method = RS_MAP_REDUCE;
      c.num_chunks = (uint16_t)(n_lo + i_n * P.cstep);
      c.interlen = (uint16_t)(il_lo + (r - i_n * ni) * P.istep);
    }
  }
};

inline int make_const(const rs_select_params* p, const rs_cost_model* cost, SelConst* out) {
  RS_REQUIRE(p != nullptr, "params is NULL");
  RS_REQUIRE(p->per_token_bytes > 0, "per_token_bytes must be positive");
  RS_REQUIRE(p->chunk_size > 0, "chunk_size must be positive");
  RS_REQUIRE(p->out_budget > 0, "out_budget must be positive");
  RS_REQUIRE(p->template_tokens >= 0, "template_tokens must be non-negative");
  RS_REQUIRE(p->max_chunks >= 1, "max_chunks must be >= 1");
  RS_REQUIRE(p->chunk_step >= 1 && p->interlen_step >= 1, "granularity steps must be at least 1");
  SelConst c{};
  c.pt = p->per_token_bytes;
  c.C = p->chunk_size;
  c.T = p->template_tokens;
  c.O = p->out_budget;
  c.tok_limit = (INT64_MAX - 99) / (102 * c.pt);
  c.pa = (102 * c.pt) / 100;
  c.pb = int32_t((102 * c.pt) % 100);
  c.max_chunks = p->max_chunks;
  c.cstep = p->chunk_step;
  c.istep = p->interlen_step;
  c.allow_fallback = p->allow_fallback;
  if (cost) {
    c.has_cost = 1;
    c.a = cost->prefill_secs_per_token;
    c.b = cost->decode_secs_per_token_base;
    c.s = cost->batch_slowdown_per_seq;
  }
  *out = c;
  return RS_OK;
}


}  // namespace rs
