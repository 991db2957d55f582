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

#include "cost_model.cuh"
#include "rs_common.cuh"

namespace rs {
namespace {

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

// int64 range guard: a conservative bound over every candidate and the
// fallback; true = the query's byte arithmetic could overflow.
__device__ __forceinline__ int64_t query_tmax(const Grid& gr, int64_t q, const SelConst& P) {
  const int64_t nmax = gr.n_hi > P.max_chunks ? gr.n_hi : P.max_chunks;
  const int64_t per = P.C > gr.il_hi ? P.C : gr.il_hi;
  const int64_t tail = P.O > gr.il_hi ? P.O : gr.il_hi;
  return q + nmax * per + P.T + tail;  // bounds every token count of the query's candidates and fallback
}
__device__ __forceinline__ bool range_overflow(const Grid& gr, int64_t q, const SelConst& P) {
  const int64_t nmax = gr.n_hi > P.max_chunks ? gr.n_hi : P.max_chunks;
  const int64_t per = P.C > gr.il_hi ? P.C : gr.il_hi;
  const int64_t tmax = query_tmax(gr, q, P);
  bool bad = nmax > 65535 || per > (int64_t(1) << 30) || q > (int64_t(1) << 40) || tmax > P.tok_limit ||
             gr.G >= (int64_t(1) << 30);  // grid indices are int32 in the scan
  if (!bad) bad = buffered(tmax, P.pt) > (int64_t)(INT64_MAX / 2) / (nmax + 1);
  return bad;
}

// best_fit_select (scheduler.py:127-156), warp-collective: arg-max of
// (bytes, grid index) over the candidates with bytes <= fr.  On a fit sets
// c.{method,num_chunks,interlen,kv_bytes} and status BEST_FIT; returns false
// (c untouched) when nothing fits.
//
// Each lane walks its grid indices g = lane, lane + 32, ... in increasing
// order through the three method blocks (so ">=" keeps the later g on byte
// ties); the map_reduce block is walked as (i_n, i_il) with an incremental
// carry instead of a per-candidate division, and token counts below
// kFastTok use the division-free buffered_fast.
template <bool FAST>
__device__ __forceinline__ void best_fit_scan(const Grid& gr, int64_t q, int64_t fr, const SelConst& P, int lane,
                                              int64_t& best_b, int32_t& best_g) {
  auto buf = [&](int64_t t) -> int64_t {
    if constexpr (FAST) return buffered_fast(int32_t(t), P.pa, P.pb);
    else return buffered(t, P.pt);
  };
  const int64_t rr_call = buf(q + P.C + P.T + P.O);  // one rerank call
  const int32_t nn = int32_t(gr.nn);
  // map_rerank block: g = i
  for (int32_t i = lane; i < int32_t(gr.n_rr); i += 32) {
    const int64_t bytes = (gr.n_lo + int64_t(i) * P.cstep) * rr_call;
    if (bytes <= fr && bytes >= best_b) {
      best_b = bytes;
      best_g = i;
    }
  }
  // stuff block: g = n_rr + i
  for (int32_t i = lane; i < int32_t(gr.n_st); i += 32) {
    const int64_t nc = gr.n_lo + int64_t(i) * P.cstep;
    const int64_t bytes = buf(q + nc * P.C + P.T + P.O);
    if (bytes <= fr && bytes >= best_b) {
      best_b = bytes;
      best_g = int32_t(gr.n_rr) + i;
    }
  }
  // map_reduce block: g = n_rr + n_st + i_n * ni + i_il
  const int32_t ni = int32_t(gr.ni);
  const int32_t n_mr = nn * ni;
  if (n_mr > 0) {
    const int32_t off = int32_t(gr.n_rr + gr.n_st);
    const int32_t dn = 32 / ni, dil = 32 % ni;  // per-step carry of (i_n, i_il)
    int32_t i_n = lane / ni, i_il = lane % ni;
    for (int32_t r = lane; r < n_mr; r += 32) {
      const int64_t nc = gr.n_lo + int64_t(i_n) * P.cstep;
      const int64_t il = gr.il_lo + int64_t(i_il) * P.istep;
      const int64_t bytes = nc * buf(q + P.C + P.T + il) + buf(q + nc * il + P.T + P.O);
      if (bytes <= fr && bytes >= best_b) {
        best_b = bytes;
        best_g = off + r;
      }
      i_n += dn;
      i_il += dil;
      if (i_il >= ni) {
        i_il -= ni;
        ++i_n;
      }
    }
  }
}

__device__ __forceinline__ bool best_fit_warp(const Grid& gr, int64_t q, int64_t fr, const SelConst& P, int lane,
                                              rs_config& c) {
  int64_t best_b = -1;
  int32_t best_g = -1;
  if (query_tmax(gr, q, P) < kFastTok)  // warp-uniform
    best_fit_scan<true>(gr, q, fr, P, lane, best_b, best_g);
  else
    best_fit_scan<false>(gr, q, fr, P, lane, best_b, best_g);
  warp_argmax(best_b, best_g);
  if (best_g < 0) return false;
  gr.decode(best_g, P, c);
  c.kv_bytes = best_b;
  c.status = RS_SELECT_BEST_FIT;
  return true;
}

// fallback_config (scheduler.py:159-191), warp-collective: never map_reduce,
// ignores the space.  Sets status FALLBACK or MUST_QUEUE.
__device__ __forceinline__ void fallback_warp(bool joint, int64_t q, int64_t fr, const SelConst& P, int lane,
                                              rs_config& c) {
  const int64_t rr_call = buffered(q + P.C + P.T + P.O, P.pt);
  if (!joint) {
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
    return;
  }
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

#ifndef RS_SELECT_MIN_BLOCKS
#define RS_SELECT_MIN_BLOCKS 4  // <= 64 registers: 4 blocks of 256 per SM (issue-bound kernel)
#endif
__global__ void __launch_bounds__(256, RS_SELECT_MIN_BLOCKS) select_kernel(const rs_space* __restrict__ spaces,
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
  const Grid gr(sp, P);

  if (range_overflow(gr, q, P)) {
    if (lane == 0) {
      rs_config c{};
      c.status = RS_SELECT_OVERFLOW;
      out[qi] = c;
      if (delay) delay[qi] = 0.0;
    }
    return;
  }

  rs_config c{};
  if (!best_fit_warp(gr, q, fr, P, lane, c)) {
    if (P.allow_fallback)
      fallback_warp(profiles[qi].needs_joint_reasoning != 0, q, fr, P, lane, c);
    else
      c.status = RS_SELECT_MUST_QUEUE;
  }

  if (lane == 0) out[qi] = c;

  if (P.has_cost) {
    // Critical-path delay of the admitted plan (plan_calls memory.py:117-148,
    // sim.dispatch concurrency sim.py:226-228): j-th independent call runs
    // with running_before + j sequences; a reducer waits for its mappers and
    // then runs with running_before.  Lanes take calls j = lane, lane + 32..;
    // the max is exact in any order, so the warp reduction is bit-identical
    // to the sequential scan.
    double d = 0.0;
    if (c.status == RS_SELECT_BEST_FIT || c.status == RS_SELECT_FALLBACK) {
      const int64_t c0 = running ? running[qi] : 0;
      const int64_t nc = c.num_chunks;
      if (c.method == RS_STUFF) {
        d = call_latency(q + nc * P.C + P.T, P.O, c0, P.a, P.b, P.s);
      } else {
        const int64_t out = c.method == RS_MAP_RERANK ? P.O : int64_t(c.interlen);
        for (int64_t j = lane; j < nc; j += 32) d = fmax(d, call_latency(q + P.C + P.T, out, c0 + j, P.a, P.b, P.s));
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, off));
        if (c.method == RS_MAP_REDUCE)
          d = __dadd_rn(d, call_latency(q + nc * int64_t(c.interlen) + P.T, P.O, c0, P.a, P.b, P.s));
      }
    }
    if (lane == 0) delay[qi] = d;
  }
}

// plan_calls' raising checks for a chosen config (memory.py:106-145, in the
// reference's order): chunk count, then per call kind the context window
// (memory.py:81-86), map_reduce's intermediate length before its mappers.
// Also returns the independent calls (CallPlan.independent_calls, memory.py
// :66-67): every call but a map_reduce reducer, all of one size per plan.
__device__ __forceinline__ int plan_check(const rs_config& c, int64_t q, const SelConst& P, int64_t ctx,
                                          int64_t& n_indep, int64_t& indep_bytes) {
  const int64_t n = c.num_chunks;
  if (n < 1 || n > P.max_chunks) return RS_ADMIT_INVALID_CHUNKS;
  if (c.method == RS_STUFF) {
    if (q + n * P.C + P.T + P.O > ctx) return RS_ADMIT_CONTEXT_OVERFLOW;
    n_indep = 1;
    indep_bytes = buffered(q + n * P.C + P.T + P.O, P.pt);
  } else if (c.method == RS_MAP_RERANK) {
    if (q + P.C + P.T + P.O > ctx) return RS_ADMIT_CONTEXT_OVERFLOW;
    n_indep = n;
    indep_bytes = buffered(q + P.C + P.T + P.O, P.pt);
  } else {
    const int64_t il = c.interlen;
    if (il <= 0) return RS_ADMIT_BAD_INTERLEN;
    if (q + P.C + P.T + il > ctx) return RS_ADMIT_CONTEXT_OVERFLOW;
    if (q + n * il + P.T + P.O > ctx) return RS_ADMIT_CONTEXT_OVERFLOW;
    n_indep = n;
    indep_bytes = buffered(q + P.C + P.T + il, P.pt);
  }
  return RS_ADMIT_DRAINED;  // ok
}

// FIFO admission chain: the new-query loop of Scheduler.step
// (scheduler.py:397-410) over _try_admit_new (:335-395) and the memory
// accounting of _start_run (:281-333).  The chain is serial through the free
// bytes (each admission lowers them by its admitted independent calls; a
// map_reduce reducer is deferred), so one warp walks the queue in order and
// evaluates each query's candidates lane-parallel; queue records are
// prefetched 32 at a time (lane j loads entry base + j) and broadcast with
// shuffles, keeping global-load latency off the serial path.
__global__ void __launch_bounds__(32) admit_fifo_kernel(const rs_space* __restrict__ spaces,
                                                        const rs_profile* __restrict__ profiles,
                                                        const uint8_t* __restrict__ has_profile,
                                                        const int32_t* __restrict__ qlen, int64_t n, SelConst P,
                                                        int64_t capacity, int64_t used0, int64_t ctx,
                                                        rs_config* __restrict__ configs,
                                                        rs_admit_info* __restrict__ info,
                                                        rs_admit_result* __restrict__ result) {
  const int lane = threadIdx.x;
  int64_t used = used0;
  int64_t i = 0;
  int32_t stop = RS_ADMIT_DRAINED;
  for (int64_t base = 0; base < n && stop == RS_ADMIT_DRAINED; base += 32) {
    // prefetch 32 queue entries: lane j holds entry base + j
    uint2 sp_lo = make_uint2(0, 0), sp_hi = make_uint2(0, 0);
    int32_t ql = 0;
    uint32_t joint = 0, hasp = 1;
    if (base + lane < n) {
      const uint4 v = reinterpret_cast<const uint4*>(spaces)[base + lane];
      sp_lo = make_uint2(v.x, v.y);
      sp_hi = make_uint2(v.z, v.w);
      ql = qlen[base + lane];
      if (profiles) joint = profiles[base + lane].needs_joint_reasoning;
      if (has_profile) hasp = has_profile[base + lane];
    }
    const int cnt = int(n - base < 32 ? n - base : 32);
    for (int t = 0; t < cnt; ++t) {
      i = base + t;
      uint4 v;
      v.x = __shfl_sync(0xffffffffu, sp_lo.x, t);
      v.y = __shfl_sync(0xffffffffu, sp_lo.y, t);
      v.z = __shfl_sync(0xffffffffu, sp_hi.x, t);
      v.w = __shfl_sync(0xffffffffu, sp_hi.y, t);
      rs_space sp;
      memcpy(&sp, &v, sizeof(sp));
      const int64_t q = __shfl_sync(0xffffffffu, ql, t);
      const bool jt = __shfl_sync(0xffffffffu, joint, t) != 0;
      const bool hp = __shfl_sync(0xffffffffu, hasp, t) != 0;
      const int64_t fr = capacity - used;
      const Grid gr(sp, P);

      rs_config c{};
      int64_t n_adm = 0, adm_bytes = 0;
      bool fixed = false;
      if (range_overflow(gr, q, P)) {
        stop = RS_ADMIT_OVERFLOW;
      } else {
        // best fit first, whatever the mode (scheduler.py:339-351)
        bool ok = best_fit_warp(gr, q, fr, P, lane, c);
        if (!ok && P.allow_fallback) {
          if (!hp) {
            stop = RS_ADMIT_NO_PROFILE;  // scheduler.py:356-359
          } else {
            fallback_warp(jt, q, fr, P, lane, c);
            ok = c.status == RS_SELECT_FALLBACK;
            if (!ok) stop = used == 0 ? RS_ADMIT_IMPOSSIBLE : RS_ADMIT_BLOCKED;  // :374-378
          }
        } else if (!ok) {
          // fixed-config baseline (scheduler.py:380-395): exactly one
          // candidate, admitted call by call in index order while each fits
          fixed = true;
          if (gr.G != 1) {
            stop = RS_ADMIT_FIXED_SPACE;
          } else {
            gr.decode(0, P, c);
            int64_t n_ind = 0, per = 0;
            const int rc = plan_check(c, q, P, ctx, n_ind, per);
            if (rc != RS_ADMIT_DRAINED) {
              stop = rc;
            } else if (per > capacity) {
              stop = RS_ADMIT_IMPOSSIBLE;
            } else if (per > fr) {
              stop = RS_ADMIT_BLOCKED;
            } else {
              const int64_t nc = c.num_chunks;
              c.kv_bytes = c.method == RS_STUFF        ? per
                           : c.method == RS_MAP_RERANK ? nc * per
                                                       : nc * per + buffered(q + nc * c.interlen + P.T + P.O, P.pt);
              c.status = RS_SELECT_BEST_FIT;
              n_adm = fr / per < n_ind ? fr / per : n_ind;
              adm_bytes = n_adm * per;
            }
          }
        }
        if (ok && !fixed) {
          int64_t n_ind = 0, per = 0;
          const int rc = plan_check(c, q, P, ctx, n_ind, per);
          if (rc != RS_ADMIT_DRAINED) {
            stop = rc;
          } else {
            // admit_all_independent: every independent call fits by construction
            // (their sum is at most plan_bytes <= free); the host re-checks
            n_adm = n_ind;
            adm_bytes = n_ind * per;
          }
        }
      }
      if (stop != RS_ADMIT_DRAINED) {
        // the chosen (or fixed) config of the entry that raised, for the
        // caller's error message
        if (lane == 0) configs[i] = c;
        break;
      }
      used += adm_bytes;
      if (lane == 0) {
        configs[i] = c;
        rs_admit_info a{};
        a.admitted_bytes = adm_bytes;
        a.admitted_calls = int32_t(n_adm);
        a.fixed_path = fixed ? 1 : 0;
        info[i] = a;
      }
    }
  }
  if (lane == 0) {
    rs_admit_result r{};
    r.admitted = stop == RS_ADMIT_DRAINED ? n : i;
    r.used_bytes = used;
    r.stop = stop;
    *result = r;
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

extern "C" int rs_admit_fifo(const rs_space* spaces, const rs_profile* profiles, const uint8_t* has_profile,
                             const int32_t* qlen, int64_t n, const rs_select_params* params,
                             const rs_admit_params* admit, rs_config* configs, rs_admit_info* info,
                             rs_admit_result* result, void* stream) {
  using namespace rs;
  RS_REQUIRE(n >= 0, "n must be non-negative");
  RS_REQUIRE(admit != nullptr && result != nullptr, "NULL argument");
  RS_REQUIRE(n == 0 || (spaces && qlen && configs && info), "NULL device pointer");
  RS_REQUIRE(n == 0 || profiles || (params && !params->allow_fallback), "profiles required by the fallback");
  RS_REQUIRE(admit->capacity_bytes > 0, "capacity_bytes must be positive");
  RS_REQUIRE(admit->used_bytes >= 0 && admit->used_bytes <= admit->capacity_bytes, "used_bytes outside [0, capacity]");
  RS_REQUIRE(admit->max_context_tokens > 0, "max_context_tokens must be positive");
  SelConst c;
  int rc = make_const(params, nullptr, &c);
  if (rc) return rc;
  admit_fifo_kernel<<<1, 32, 0, as_stream(stream)>>>(spaces, profiles, has_profile, qlen, n, c,
                                                     admit->capacity_bytes, admit->used_bytes,
                                                     admit->max_context_tokens, configs, info, result);
  RS_CHECK_LAUNCH("admit_fifo_kernel");
  return RS_OK;
}
