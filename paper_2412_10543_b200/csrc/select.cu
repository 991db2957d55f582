// K3 config_select: batched best-fit + fallback selection with the KV-memory
// and prefill/decode delay cost models, bit-exact with the reference:
//   buffered_bytes   memory.py:76-78      plan_bytes        memory.py:164-195
//   best_fit_select  scheduler.py:127-156 fallback_config   scheduler.py:159-191
//   decision order   scheduler.py:335-378 call_latency      sim.py:84-92
//
// One warp per query.  The reference enumerates the grid, stable-sorts it by
// bytes and scans in reverse (O(C log C)); that is exactly the arg-max of the
// pair (bytes, grid index) over the fitting candidates, which a warp computes
// with a strided scan and a 5-step shuffle reduction — no sort, no
// materialised candidate list.  All byte arithmetic is int64 (intermediates
// reach 6.3e11 at the north-star shapes); an up-front per-query bound turns
// any int64 overflow into RS_SELECT_OVERFLOW instead of a wrong answer.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rs_common.cuh"

namespace rs {
namespace {

struct SelConst {
  int64_t pt;        // per-token bytes
  int64_t C, T, O;   // chunk size, template tokens, out budget
  int64_t tok_limit; // largest token count whose 102*tok*pt+99 fits int64
  int32_t max_chunks, cstep, istep, allow_fallback;
  int32_t has_cost;
  double a, b, s;    // CostModel
};

__device__ __forceinline__ int64_t buffered(int64_t tokens, int64_t pt) {
  return (102 * tokens * pt + 99) / 100;  // memory.py:76-78
}

// sim.py:84-92 in the reference's IEEE-double evaluation order, no FMA.
__device__ __forceinline__ double call_latency(int64_t prompt, int64_t out, int64_t conc, double a,
                                               double b, double s) {
  const double prefill = __dmul_rn(a, __ll2double_rn(prompt));
  const double dil = __dadd_rn(1.0, __dmul_rn(s, __ll2double_rn(conc)));
  const double decode = __dmul_rn(__dmul_rn(__ll2double_rn(out), b), dil);
  return __dadd_rn(prefill, decode);
}

__device__ __forceinline__ void warp_argmax(int64_t& b, int32_t& g) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const int64_t ob = __shfl_xor_sync(0xffffffffu, b, off);
    const int32_t og = __shfl_xor_sync(0xffffffffu, g, off);
    if (ob > b || (ob == b && og > g)) {
      b = ob;
      g = og;
    }
  }
}

__global__ void __launch_bounds__(256) select_kernel(const rs_space* __restrict__ spaces,
                                                     const rs_profile* __restrict__ profiles,
                                                     const int32_t* __restrict__ qlen,
                                                     const int64_t* __restrict__ free_bytes, int64_t n,
                                                     SelConst P, const int32_t* __restrict__ running,
                                                     double* __restrict__ delay,
                                                     rs_config* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t qi = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (qi >= n) return;

  const rs_space sp = spaces[qi];
  const int64_t q = qlen[qi];
  const int64_t fr = free_bytes[qi];
  const int m = sp.methods;
  const int64_t n_lo = sp.num_chunks_lo, n_hi = sp.num_chunks_hi;
  const int64_t il_lo = sp.interlen_lo, il_hi = sp.interlen_hi;

  // grid extents (IntRange.values(step), types.py:59-60)
  const int64_t nn = (n_hi >= n_lo) ? (n_hi - n_lo) / P.cstep + 1 : 0;
  const int64_t ni = ((m & RS_MAP_REDUCE) && il_hi >= il_lo) ? (il_hi - il_lo) / P.istep + 1 : 0;
  const int64_t n_rr = (m & RS_MAP_RERANK) ? nn : 0;
  const int64_t n_st = (m & RS_STUFF) ? nn : 0;
  const int64_t G = n_rr + n_st + nn * ni;

  // int64 range guard (conservative bound over every candidate + fallback)
  {
    const int64_t nmax = n_hi > P.max_chunks ? n_hi : P.max_chunks;
    const int64_t per = P.C > il_hi ? P.C : il_hi;
    const int64_t tail = P.O > il_hi ? P.O : il_hi;
    const int64_t tmax = q + nmax * per + P.T + tail;
    bool bad = nmax > 65535 || per > (int64_t(1) << 30) || q > (int64_t(1) << 40) ||
               tmax > P.tok_limit;
    if (!bad) bad = buffered(tmax, P.pt) > (int64_t)(INT64_MAX / 2) / (nmax + 1);
    if (bad) {
      if (lane == 0) {
        rs_config c{};
        c.status = RS_SELECT_OVERFLOW;
        out[qi] = c;
        if (delay) delay[qi] = 0.0;
      }
      return;
    }
  }

  const int64_t rr_call = buffered(q + P.C + P.T + P.O, P.pt);  // one rerank call
  int64_t best_b = -1;
  int32_t best_g = -1;
  for (int64_t g = lane; g < G; g += 32) {
    int64_t bytes;
    if (g < n_rr) {
      const int64_t nc = n_lo + g * P.cstep;
      bytes = nc * rr_call;
    } else if (g < n_rr + n_st) {
      const int64_t nc = n_lo + (g - n_rr) * P.cstep;
      bytes = buffered(q + nc * P.C + P.T + P.O, P.pt);
    } else {
      const int64_t r = g - n_rr - n_st;
      const int64_t i_n = r / ni;
      const int64_t nc = n_lo + i_n * P.cstep;
      const int64_t il = il_lo + (r - i_n * ni) * P.istep;
      bytes = nc * buffered(q + P.C + P.T + il, P.pt) + buffered(q + nc * il + P.T + P.O, P.pt);
    }
    if (bytes <= fr && bytes >= best_b) {  // g ascends per lane: ties -> later g
      best_b = bytes;
      best_g = (int32_t)g;
    }
  }
  warp_argmax(best_b, best_g);

  rs_config c{};
  if (best_g >= 0) {
    const int64_t g = best_g;
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
    c.kv_bytes = best_b;
    c.status = RS_SELECT_BEST_FIT;
  } else if (P.allow_fallback) {
    // fallback_config (scheduler.py:159-191): never map_reduce, ignores the space
    if (!profiles[qi].needs_joint_reasoning) {
      int64_t k = fr / rr_call;  // free >= 0 in the reference; negatives give k < 1 either way
      if (k > P.max_chunks) k = P.max_chunks;
      if (k >= 1) {
        c.method = RS_MAP_RERANK;
        c.num_chunks = (uint16_t)k;
        c.kv_bytes = k * rr_call;
        c.status = RS_SELECT_FALLBACK;
      } else {
        c.status = RS_SELECT_MUST_QUEUE;
      }
    } else {
      // largest k in [max_chunks .. 1] whose stuff plan fits
      int64_t kb = -1, kbytes = 0;
      for (int64_t k = P.max_chunks - lane; k >= 1; k -= 32) {
        const int64_t b = buffered(q + k * P.C + P.T + P.O, P.pt);
        if (b <= fr && k > kb) {
          kb = k;
          kbytes = b;
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const int64_t ok = __shfl_xor_sync(0xffffffffu, kb, off);
        const int64_t obytes = __shfl_xor_sync(0xffffffffu, kbytes, off);
        if (ok > kb) {
          kb = ok;
          kbytes = obytes;
        }
      }
      if (kb >= 1) {
        c.method = RS_STUFF;
        c.num_chunks = (uint16_t)kb;
        c.kv_bytes = kbytes;
        c.status = RS_SELECT_FALLBACK;
      } else {
        c.status = RS_SELECT_MUST_QUEUE;
      }
    }
  } else {
    c.status = RS_SELECT_MUST_QUEUE;
  }

  if (lane == 0) out[qi] = c;

  if (P.has_cost && lane == 0) {
    // Critical-path delay of the admitted plan (plan_calls memory.py:117-148,
    // sim.dispatch concurrency sim.py:226-228): j-th independent call runs
    // with running_before + j sequences; a reducer waits for its mappers and
    // then runs with running_before.
    double d = 0.0;
    if (c.status == RS_SELECT_BEST_FIT || c.status == RS_SELECT_FALLBACK) {
      const int64_t c0 = running ? running[qi] : 0;
      const int64_t nc = c.num_chunks;
      if (c.method == RS_STUFF) {
        d = fmax(d, call_latency(q + nc * P.C + P.T, P.O, c0, P.a, P.b, P.s));
      } else if (c.method == RS_MAP_RERANK) {
        for (int64_t j = 0; j < nc; ++j)
          d = fmax(d, call_latency(q + P.C + P.T, P.O, c0 + j, P.a, P.b, P.s));
      } else {
        const int64_t il = c.interlen;
        for (int64_t j = 0; j < nc; ++j)
          d = fmax(d, call_latency(q + P.C + P.T, il, c0 + j, P.a, P.b, P.s));
        d = __dadd_rn(d, call_latency(q + nc * il + P.T, P.O, c0, P.a, P.b, P.s));
      }
    }
    delay[qi] = d;
  }
}

__global__ void call_latency_kernel(const int64_t* __restrict__ prompt, const int64_t* __restrict__ outt,
                                    const int64_t* __restrict__ conc, int64_t n, double a, double b,
                                    double s, double* __restrict__ res) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    res[i] = call_latency(prompt[i], outt[i], conc[i], a, b, s);
}

__global__ void plan_bytes_kernel(const uint8_t* __restrict__ method, const int32_t* __restrict__ nch,
                                  const int32_t* __restrict__ il, const int32_t* __restrict__ qlen,
                                  int64_t n, SelConst P, int64_t* __restrict__ res) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = qlen[i], nc = nch[i];
    int64_t b;
    if (method[i] == RS_STUFF)
      b = buffered(q + nc * P.C + P.T + P.O, P.pt);
    else if (method[i] == RS_MAP_RERANK)
      b = nc * buffered(q + P.C + P.T + P.O, P.pt);
    else
      b = nc * buffered(q + P.C + P.T + il[i], P.pt) + buffered(q + nc * il[i] + P.T + P.O, P.pt);
    res[i] = b;
  }
}

int make_const(const rs_select_params* p, const rs_cost_model* cost, SelConst* out) {
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

}  // namespace
}  // namespace rs

extern "C" int rs_select(const rs_space* spaces, const rs_profile* profiles, const int32_t* qlen,
                         const int64_t* free_bytes, int64_t n, const rs_select_params* params,
                         const rs_cost_model* cost, const int32_t* running_before, double* delay_out,
                         rs_config* out, void* stream) {
  using namespace rs;
  RS_REQUIRE(n >= 0, "n must be non-negative");
  if (n == 0) return RS_OK;
  RS_REQUIRE(spaces && qlen && free_bytes && out, "NULL device pointer");
  RS_REQUIRE(profiles || (params && !params->allow_fallback), "profiles required by the fallback");
  RS_REQUIRE(!cost || delay_out, "delay_out required when cost is given");
  SelConst c;
  int rc = make_const(params, cost, &c);
  if (rc) return rc;
  const int64_t threads = n * 32;
  const int64_t blocks = ceil_div(threads, 256);
  RS_REQUIRE(blocks < (int64_t(1) << 31), "batch too large");
  select_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(spaces, profiles, qlen, free_bytes, n, c,
                                                                 running_before, delay_out, out);
  RS_CHECK_LAUNCH("select_kernel");
  return RS_OK;
}

extern "C" int rs_call_latency(const int64_t* prompt_tokens, const int64_t* max_output_tokens,
                               const int64_t* concurrent_seqs, int64_t n, const rs_cost_model* cost,
                               double* out, void* stream) {
  using namespace rs;
  RS_REQUIRE(n >= 0 && cost, "bad arguments");
  if (n == 0) return RS_OK;
  const int64_t blocks = std::min<int64_t>(ceil_div(n, 256), 4096);
  call_latency_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(
      prompt_tokens, max_output_tokens, concurrent_seqs, n, cost->prefill_secs_per_token,
      cost->decode_secs_per_token_base, cost->batch_slowdown_per_seq, out);
  RS_CHECK_LAUNCH("call_latency_kernel");
  return RS_OK;
}

extern "C" int rs_plan_bytes(const uint8_t* method, const int32_t* num_chunks, const int32_t* interlen,
                             const int32_t* qlen, int64_t n, const rs_select_params* params, int64_t* out,
                             void* stream) {
  using namespace rs;
  RS_REQUIRE(n >= 0, "n must be non-negative");
  if (n == 0) return RS_OK;
  SelConst c;
  int rc = make_const(params, nullptr, &c);
  if (rc) return rc;
  const int64_t blocks = std::min<int64_t>(ceil_div(n, 256), 4096);
  plan_bytes_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(method, num_chunks, interlen, qlen, n,
                                                                     c, out);
  RS_CHECK_LAUNCH("plan_bytes_kernel");
  return RS_OK;
}
