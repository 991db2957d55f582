// Retrieval: the index handle (rs_index_*), row norms, the CUDA-core fused
// score+top-k kernel (fp32 corpora and a bf16 cross-check path), the k-way
// top-k merge (K2) and the search planner.  FAISS IndexFlatL2 semantics
// (PAPER.md:653): D = |q|^2 + |c|^2 - 2<q,c> clamped at 0, ascending, ties to
// the lower chunk id, missing results I = -1 / D = +inf.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "retrieval.cuh"
#include "topk_rows.cuh"

namespace rs {
namespace {

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) {
  return v;
}
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}

// ---- squared norms: one warp per row, fp32 accumulate ---------------------
// For an fp32 matrix headed for the 3xTF32 kernel the same pass also writes
// the tf32 residuals lo = x - trunc_tf32(x) (the tensor core reads an fp32
// operand as tf32 by dropping the low 13 mantissa bits; the residual is exact
// in fp32), so the split costs no extra read of x.
__device__ __forceinline__ float tf32_residual(float v) {
  return v - __uint_as_float(__float_as_uint(v) & 0xffffe000u);
}

template <typename T>
__global__ void __launch_bounds__(256) row_norms_kernel(const T* __restrict__ x, int64_t n, int dim,
                                                        float* __restrict__ out, unsigned int* __restrict__ max_bits,
                                                        float* __restrict__ lo) {
  const int lane = threadIdx.x & 31;
  float mx = 0.0f;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const T* row = x + r * dim;
    float s = 0.0f;
    for (int i = lane; i < dim; i += 32) {
      const float v = to_f(row[i]);
      s = fmaf(v, v, s);
      if constexpr (sizeof(T) == 4) {
        if (lo) lo[r * dim + i] = tf32_residual(v);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) out[r] = s;
    mx = fmaxf(mx, s);
  }
  // running max of the (non-negative) norms: unsigned order == float order
  if (max_bits && lane == 0 && mx > 0.0f) atomicMax(max_bits, __float_as_uint(mx));
}

// ---- CUDA-core fused score + top-k ------------------------------------------
// CTA = 64 queries x 64 corpus rows per tile, 256 threads each holding a 4x4
// micro-tile of dot products; distances go through a smem tile and one thread
// per query feeds its RowTopK.
constexpr int BQ = kSimtBQ, BC = kSimtBC, BKS = 32;

template <typename T, int KCAP, int BUF>
__global__ void __launch_bounds__(256) score_topk_simt_kernel(const T* __restrict__ Q, const float* __restrict__ qn,
                                                              int64_t nq, const T* __restrict__ C,
                                                              const float* __restrict__ cn, int64_t n, int dim, int k,
                                                              int64_t id_base, int qtiles, int segments,
                                                              int64_t seg_rows, uint64_t* __restrict__ part) {
  __shared__ float As[BKS][BQ + 4];
  __shared__ float Bs[BKS][BC + 4];
  __shared__ float Sd[BQ][BC + 1];
  extern __shared__ uint64_t simt_dyn[];  // heap [KCAP][BQ] then buffer [BUF][BQ]
  uint64_t* heap = simt_dyn;
  uint64_t* bufm = simt_dyn + KCAP * BQ;
  const int tid = threadIdx.x;
  const int tq = tid >> 4, tc = tid & 15;
  const int64_t units = int64_t(qtiles) * segments;
  RowTopK<BQ, BUF> rt{heap, bufm, tid & (BQ - 1), k, 0, 0, 0.0f};

  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int seg = int(u / qtiles);
    const int qt = int(u - int64_t(seg) * qtiles);
    const int64_t r0 = int64_t(seg) * seg_rows;
    const int64_t r1 = std::min<int64_t>(n, r0 + seg_rows);
    const int64_t q0 = int64_t(qt) * BQ;
    if (tid < BQ) rt.reset();
    for (int64_t c0 = r0; c0 < r1; c0 += BC) {
      float acc[4][4] = {};
      for (int k0 = 0; k0 < dim; k0 += BKS) {
#pragma unroll
        for (int i = 0; i < (BQ * BKS) / 256; ++i) {
          const int idx = tid + i * 256;
          const int rr = idx / BKS, kk = idx % BKS;
          const int64_t qrow = q0 + rr, crow = c0 + rr;
          const bool kin = k0 + kk < dim;
          As[kk][rr] = (qrow < nq && kin) ? to_f(Q[qrow * dim + k0 + kk]) : 0.0f;
          Bs[kk][rr] = (crow < r1 && kin) ? to_f(C[crow * dim + k0 + kk]) : 0.0f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < BKS; ++kk) {
          float a[4], b[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            a[i] = As[kk][tq + 16 * i];
            b[i] = Bs[kk][tc + 16 * i];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t qrow = q0 + tq + 16 * i;
        const float qv = qrow < nq ? qn[qrow] : 0.0f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int64_t crow = c0 + tc + 16 * j;
          const float cv = crow < r1 ? cn[crow] : 0.0f;
          Sd[tq + 16 * i][tc + 16 * j] = l2_from_dot(qv + cv, acc[i][j]);
        }
      }
      __syncthreads();
      if (tid < BQ) {
        const int valid = int(std::min<int64_t>(BC, r1 - c0));
        const uint32_t id0 = uint32_t(id_base + c0);
        for (int c = 0; c < BC; c += 16) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (c + j < valid) rt.offer(Sd[tid][c + j], id0 + c + j);
          if (__any_sync(0xffffffffu, rt.nb > BUF - 16)) rt.flush();
        }
      }
      __syncthreads();
    }
    if (tid < BQ && q0 + tid < nq) rt.finish(part + ((q0 + tid) * segments + seg) * k);
  }
}

// ---- K2: k-way merge of sorted key lists (one warp per query) -----------------
// List l of query q: keys[q * q_stride + l * list_stride + j], j < k_in, sorted
// ascending (kEmptyKey-padded).  Tournament: every lane tracks the head of
// lists lane, lane+32, ...; per output the warp arg-min picks the winner list
// and only the owning lane advances and rescans.
constexpr int kMergeWarps = 8;

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, uint32_t(v), src);
  const uint32_t hi = __shfl_sync(0xffffffffu, uint32_t(v >> 32), src);
  return (uint64_t(hi) << 32) | lo;
}

__global__ void __launch_bounds__(kMergeWarps * 32) merge_topk_kernel(
    const uint64_t* __restrict__ keys, int64_t nq, int nlists, int k_in, int64_t list_stride, int64_t q_stride,
    int k, const rs_config* __restrict__ keep, float* __restrict__ D, int64_t* __restrict__ I,
    uint64_t* __restrict__ keys_out) {
  extern __shared__ uint8_t heads_all[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint8_t* heads = heads_all + size_t(w) * nlists;
  for (int64_t q = int64_t(blockIdx.x) * kMergeWarps + w; q < nq; q += int64_t(gridDim.x) * kMergeWarps) {
    const uint64_t* base = keys + q * q_stride;
    for (int l = lane; l < nlists; l += 32) heads[l] = 0;
    __syncwarp();
    // lane-local minimum over its lists
    uint64_t best = kEmptyKey;
    int best_l = -1;
    for (int l = lane; l < nlists; l += 32) {
      const uint64_t v = base[int64_t(l) * list_stride];
      if (v < best || best_l < 0) {
        best = v;
        best_l = l;
      }
    }
    int limit = k;
    if (keep) {
      const rs_config c = keep[q];
      limit = (c.status == RS_SELECT_BEST_FIT || c.status == RS_SELECT_FALLBACK) ? c.num_chunks : 0;
      if (limit > k) limit = k;
    }
    for (int j = 0; j < k; ++j) {
      uint64_t v = best;
      int src = lane;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const uint64_t ov = shfl_u64(v, lane ^ off);
        const int os = __shfl_xor_sync(0xffffffffu, src, off);
        if (ov < v || (ov == v && os < src)) {
          v = ov;
          src = os;
        }
      }
      const bool real = v != kEmptyKey && j < limit;
      if (lane == 0) {
        if (keys_out) keys_out[q * k + j] = real ? v : kEmptyKey;
        if (D) D[q * k + j] = real ? key_dist(v) : __int_as_float(0x7f800000);
        if (I) I[q * k + j] = real ? int64_t(uint32_t(v)) : int64_t(-1);
      }
      if (v == kEmptyKey || j + 1 >= limit) {
        // remaining outputs are padding
        for (int jj = j + 1 + lane; jj < k; jj += 32) {
          if (keys_out) keys_out[q * k + jj] = kEmptyKey;
          if (D) D[q * k + jj] = __int_as_float(0x7f800000);
          if (I) I[q * k + jj] = -1;
        }
        break;
      }
      if (lane == src) {
        // advance the winning list, rescan this lane's heads
        const int h = heads[best_l] + 1;
        heads[best_l] = (uint8_t)h;
        best = kEmptyKey;
        int bl = -1;
        for (int l = lane; l < nlists; l += 32) {
          const int hh = heads[l];
          const uint64_t cand = hh < k_in ? base[int64_t(l) * list_stride + hh] : kEmptyKey;
          if (cand < best || bl < 0) {
            best = cand;
            bl = l;
          }
        }
        best_l = bl;
      }
      __syncwarp();
    }
    __syncwarp();
  }
}

// k-way merge for up to 64 lists per query, all state in registers: lane
// l owns lists l and l + 32, holding each list's current head and the key
// after it (prefetched, so the winner's global load leaves the critical
// path).  The warp's minimum key is found with two 32-bit REDUX reductions
// (distance bits, then the id among lanes tied on distance) and a ballot —
// ids are unique, so the (distance, id) minimum is unique too.
//
// Modes.  kMergeWait (the owner's merge of the peer exchange, peer.cu): the
// lists are written by other GPUs over NVLink while the kernel starts, so
// each block first waits on the sources' epoch flags and then reads the keys
// with ld.global.cv.  kMergeScatter (the last step of a sharded search): each
// output row is stored straight into its slice owner's region (peer_row, over
// NVLink for remote owners) and the grid signals the owners at the end — the
// merge and the exchange are one kernel.
constexpr int kMergePlain = 0, kMergeWait = 1, kMergeScatter = 2;

struct PeerArgs {
  PeerWait wait;
  rs_peer_exchange ex;
  uint32_t epoch;
};
template <bool WAIT>
__device__ __forceinline__ uint64_t merge_key(const uint64_t* p) {
  if constexpr (WAIT) return __ldcv(reinterpret_cast<const unsigned long long*>(p));
  return *p;
}

__device__ __forceinline__ void peer_wait(const PeerWait& pw) {
  if (threadIdx.x == 0) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int s = 0; s < pw.n; ++s) {
      for (;;) {
        uint32_t f;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(f) : "l"(pw.flags + s) : "memory");
        if (int32_t(f - pw.epoch) >= 0) break;
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > pw.timeout_ns) {  // a source never arrived: flag it, merge what is there
          atomicExch(pw.error, 1);
          s = pw.n;
          break;
        }
        __nanosleep(200);
      }
    }
  }
  __syncthreads();
}

// One query's 64-list tournament (the warp): emits the first `limit` keys of
// the merged order through emit(j, key) (lane 0) and returns how many it
// emitted (fewer when every list runs out).
template <bool WAIT, typename Emit>
__device__ __forceinline__ int warp_merge64(const uint64_t* base, int nlists, int k_in, int64_t list_stride,
                                            int limit, Emit emit) {
  // named registers, not arrays: a [tb]-indexed array would live in local memory
  const int lane = threadIdx.x & 31;
  const uint64_t* lp0 = base + int64_t(lane) * list_stride;
  const uint64_t* lp1 = base + int64_t(lane + 32) * list_stride;
  uint64_t cur0 = lane < nlists ? merge_key<WAIT>(lp0) : kEmptyKey;
  uint64_t nxt0 = (lane < nlists && k_in > 1) ? merge_key<WAIT>(lp0 + 1) : kEmptyKey;
  uint64_t cur1 = lane + 32 < nlists ? merge_key<WAIT>(lp1) : kEmptyKey;
  uint64_t nxt1 = (lane + 32 < nlists && k_in > 1) ? merge_key<WAIT>(lp1 + 1) : kEmptyKey;
  int head0 = 0, head1 = 0;
  int j = 0;
  for (; j < limit; ++j) {
    const bool tb = cur1 < cur0;
    const uint64_t mine = tb ? cur1 : cur0;
    const uint32_t hi = uint32_t(mine >> 32);
    const uint32_t dmin = __reduce_min_sync(0xffffffffu, hi);
    const uint32_t idmin = __reduce_min_sync(0xffffffffu, hi == dmin ? uint32_t(mine) : 0xffffffffu);
    const uint64_t v = (uint64_t(dmin) << 32) | idmin;
    if (v == kEmptyKey) break;  // every list is exhausted
    const unsigned win = __ballot_sync(0xffffffffu, mine == v);
    if (lane == 0) emit(j, v);
    if (lane == __ffs(win) - 1) {
      // advance the winning list: the prefetched key moves up, the next one is requested
      if (tb) {
        cur1 = nxt1;
        ++head1;
        nxt1 = head1 + 1 < k_in ? merge_key<WAIT>(lp1 + head1 + 1) : kEmptyKey;
      } else {
        cur0 = nxt0;
        ++head0;
        nxt0 = head0 + 1 < k_in ? merge_key<WAIT>(lp0 + head0 + 1) : kEmptyKey;
      }
    }
  }
  return j;
}

__device__ __forceinline__ int keep_limit(const rs_config* keep, int64_t q, int k) {
  if (!keep) return k;
  const rs_config c = keep[q];
  const int limit = (c.status == RS_SELECT_BEST_FIT || c.status == RS_SELECT_FALLBACK) ? c.num_chunks : 0;
  return limit > k ? k : limit;
}

template <int MODE>
__global__ void __launch_bounds__(kMergeWarps * 32) merge_topk64_kernel(
    const uint64_t* keys, int64_t nq, int nlists, int k_in, int64_t list_stride, int64_t q_stride,
    int k, const rs_config* __restrict__ keep, float* __restrict__ D, int64_t* __restrict__ I,
    uint64_t* __restrict__ keys_out, const __grid_constant__ PeerArgs pa) {
  constexpr bool WAIT = MODE == kMergeWait;
  if constexpr (WAIT) peer_wait(pa.wait);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t q = int64_t(blockIdx.x) * kMergeWarps + w; q < nq; q += int64_t(gridDim.x) * kMergeWarps) {
    uint64_t* orow = MODE == kMergeScatter ? peer_row(pa.ex, nq, q, pa.epoch) : keys_out ? keys_out + q * k : nullptr;
    const int j = warp_merge64<WAIT>(keys + q * q_stride, nlists, k_in, list_stride, keep_limit(keep, q, k),
                                     [&](int jj, uint64_t v) {
                                       if (orow) orow[jj] = v;
                                       if (D) D[q * k + jj] = key_dist(v);
                                       if (I) I[q * k + jj] = int64_t(uint32_t(v));
                                     });
    for (int jj = j + lane; jj < k; jj += 32) {  // padding past the limit / the lists
      if (orow) orow[jj] = kEmptyKey;
      if (D) D[q * k + jj] = __int_as_float(0x7f800000);
      if (I) I[q * k + jj] = -1;
    }
  }
  if constexpr (MODE == kMergeScatter) peer_signal(pa.ex, pa.epoch);
}

__global__ void fill_empty_kernel(int64_t n, float* D, int64_t* I, uint64_t* keys) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    if (D) D[i] = __int_as_float(0x7f800000);
    if (I) I[i] = -1;
    if (keys) keys[i] = kEmptyKey;
  }
}

// One sorted list per query (the join after a single-shard search): the
// merge is a prefix copy with the keep limit, one thread per output slot.
__global__ void copy_topk_kernel(const uint64_t* __restrict__ keys, int64_t nq, int k_in, int64_t q_stride, int k,
                                 const rs_config* __restrict__ keep, float* __restrict__ D, int64_t* __restrict__ I,
                                 uint64_t* __restrict__ keys_out) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nq * k; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t q = t / k;
    const int j = int(t - q * k);
    int limit = k;
    if (keep) {
      const rs_config c = keep[q];
      limit = (c.status == RS_SELECT_BEST_FIT || c.status == RS_SELECT_FALLBACK) ? c.num_chunks : 0;
      if (limit > k) limit = k;
    }
    const uint64_t v = j < k_in && j < limit ? keys[q * q_stride + j] : kEmptyKey;
    const bool real = v != kEmptyKey;
    if (keys_out) keys_out[t] = v;
    if (D) D[t] = real ? key_dist(v) : __int_as_float(0x7f800000);
    if (I) I[t] = real ? int64_t(uint32_t(v)) : int64_t(-1);
  }
}

int launch_merge(const uint64_t* keys, int64_t nq, int nlists, int k_in, int64_t list_stride, int64_t q_stride,
                 int k, const rs_config* keep, float* D, int64_t* I, uint64_t* keys_out, cudaStream_t st) {
  RS_REQUIRE(nlists >= 1 && nlists <= 4096, "nlists out of range (%d)", nlists);
  RS_REQUIRE(k_in >= 1 && k_in <= 255, "k_in out of range (%d)", k_in);
  if (nlists == 1) {
    const int64_t blocks = std::min<int64_t>(ceil_div(nq * k, 256), 148 * 16);
    copy_topk_kernel<<<(unsigned)blocks, 256, 0, st>>>(keys, nq, k_in, q_stride, k, keep, D, I, keys_out);
    RS_CHECK_LAUNCH("copy_topk_kernel");
    return RS_OK;
  }
  const size_t smem = size_t(kMergeWarps) * nlists;
  const int64_t blocks = std::min<int64_t>(ceil_div(nq, kMergeWarps), 65535);
  if (nlists <= 64) {
    merge_topk64_kernel<kMergePlain><<<(unsigned)blocks, kMergeWarps * 32, 0, st>>>(
        keys, nq, nlists, k_in, list_stride, q_stride, k, keep, D, I, keys_out, PeerArgs{});
    RS_CHECK_LAUNCH("merge_topk64_kernel");
    return RS_OK;
  }
  if (smem > 48 * 1024) {
    RS_CHECK_CUDA(cudaFuncSetAttribute(merge_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
                  "cudaFuncSetAttribute(merge_topk_kernel)");
  }
  merge_topk_kernel<<<(unsigned)blocks, kMergeWarps * 32, smem, st>>>(keys, nq, nlists, k_in, list_stride, q_stride,
                                                                       k, keep, D, I, keys_out);
  RS_CHECK_LAUNCH("merge_topk_kernel");
  return RS_OK;
}

// Exact fp32 re-rank of the 3xTF32 candidates.  The tensor core accumulates
// each MMA's products into the fp32 TMEM accumulator with truncation, so at
// d = 768 a near neighbour's dot (~0.9) drifts by ~1.4e-5 relative — above the
// north star's 1e-5 fp32 tolerance.  The fused kernel therefore keeps
// kc = k + kRefineExtra candidates per query, and the kernel below recomputes
// their distances with fp32 FMAs on CUDA cores (lanes over the dimension,
// float4 loads, in-group reduction; error ~1e-7), ranks them by (distance, id)
// and emits the top k — the FAISS semantics the oracle checks, at a cost of
// nq * kc * d FMAs (negligible next to the GEMM).
//
// One CTA per query, three phases, one launch (the merge of the per-segment
// lists, the scoring and the ranking were three kernels in round 1):
//  1. all threads copy the query's lists (nlists x k_in keys, contiguous) into
//     shared memory in one coalesced pass, then warp 0 merges them into the kc
//     smallest keys (warp_merge64 over shared memory: the round-2 version
//     walked the lists in global memory, one dependent L2 round trip per
//     merged key, and the other warps idled at the barrier);
//  2. all warps score them, one candidate row per warp at a time: every lane
//     issues its (up to 8) float4 loads of the row at once (the query row is
//     staged in shared memory in phase 1), so a row costs one DRAM round
//     trip, then a 5-step butterfly;
//  3. warps 0-1 rank the exact keys (thread t owns candidate t) and write the
//     top k with the keep limit.  Keys are unique except padding.
#ifndef RS_REFINE_WARPS
#define RS_REFINE_WARPS 4  // 8 / 4 / 2 measured at cfg1: 46.5 / 35.5 / 51 us (profiles/r2_refine.md)
#endif
constexpr int kRefineWarps = RS_REFINE_WARPS;
constexpr int kRefineVec = 8;  // float4 loads per lane per 1024-element slice of a row
__global__ void __launch_bounds__(kRefineWarps * 32, 32 / kRefineWarps) refine_fp32_kernel(
    const uint64_t* __restrict__ lists, int nlists, int k_in, int64_t list_stride, int64_t q_stride, int kc,
    const float* __restrict__ Q, const float* __restrict__ qn, const float* __restrict__ C,
    const float* __restrict__ cn, int64_t nq, int dim, int64_t id_base, int k, const rs_config* __restrict__ keep,
    float* __restrict__ D, int64_t* __restrict__ I, uint64_t* __restrict__ keys_out) {
  extern __shared__ uint64_t refine_smem[];
  uint64_t* cand = refine_smem;         // [64]
  uint64_t* exact = refine_smem + 64;   // [64]
  float4* qsm = reinterpret_cast<float4*>(refine_smem + 128);  // [dim / 4]: the query row
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int d4 = dim / 4;
  uint64_t* lsm = refine_smem + 128 + 2 * d4;  // [nlists][k_in] (a float4 is two 8-byte words)
  const int nkeys = nlists * k_in;
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    const uint64_t* lq = lists + q * q_stride;
    for (int t = threadIdx.x; t < nkeys; t += kRefineWarps * 32) {
      const int l = t / k_in;
      lsm[t] = lq[int64_t(l) * list_stride + (t - l * k_in)];
    }
    const float4* qv = reinterpret_cast<const float4*>(Q + q * dim);
    for (int t = threadIdx.x; t < d4; t += kRefineWarps * 32) qsm[t] = __ldg(qv + t);
    __syncthreads();
    if (w == 0) {  // 1. candidates
      const int got = warp_merge64<false>(lsm, nlists, k_in, k_in, kc, [&](int j, uint64_t v) { cand[j] = v; });
      for (int j = got + lane; j < 64; j += 32) cand[j] = kEmptyKey;
    } else if (w == 1) {
      for (int j = kc + lane; j < 64; j += 32) exact[j] = kEmptyKey;
    }
    __syncthreads();
    const float qq = qn[q];
    for (int j = w; j < kc; j += kRefineWarps) {  // 2. exact distances, one row per warp
      const uint64_t key = cand[j];
      if (key == kEmptyKey) {  // warp-uniform
        if (lane == 0) exact[j] = kEmptyKey;
        continue;
      }
      const int64_t row = int64_t(uint32_t(key)) - id_base;
      const float4* cv = reinterpret_cast<const float4*>(C + row * dim);
      float acc = 0.0f;
      for (int base = 0; base < d4; base += 32 * kRefineVec) {
        float4 b[kRefineVec];  // the row's loads all in flight; the query comes from shared memory
#pragma unroll
        for (int i = 0; i < kRefineVec; ++i) {
          const int x = base + lane + 32 * i;
          if (x < d4) b[i] = __ldg(cv + x);
        }
#pragma unroll
        for (int i = 0; i < kRefineVec; ++i) {
          if (base + lane + 32 * i < d4) {
            const float4 a = qsm[base + lane + 32 * i];
            acc = fmaf(a.x, b[i].x, acc);
            acc = fmaf(a.y, b[i].y, acc);
            acc = fmaf(a.z, b[i].z, acc);
            acc = fmaf(a.w, b[i].w, acc);
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) {
        float dist = fmaf(-2.0f, acc, qq + cn[row]);
        dist = dist > 0.0f ? dist : 0.0f;  // FAISS clamps round-off at 0 (and NaN -> 0)
        exact[j] = (uint64_t(__float_as_uint(dist)) << 32) | uint32_t(key);
      }
    }
    __syncthreads();
    if (threadIdx.x < 64) {  // 3. rank: thread t owns candidate t
      const int t = threadIdx.x;
      const uint64_t mine = exact[t];
      int r = 0;
#pragma unroll 8
      for (int j = 0; j < 64; ++j) {
        const uint64_t o = exact[j];
        r += (o < mine || (o == mine && j < t)) ? 1 : 0;
      }
      if (r < k) {
        const int limit = keep_limit(keep, q, k);
        const bool real = mine != kEmptyKey && r < limit;
        if (keys_out) keys_out[q * k + r] = real ? mine : kEmptyKey;
        if (D) D[q * k + r] = real ? key_dist(mine) : __int_as_float(0x7f800000);
        if (I) I[q * k + r] = real ? int64_t(uint32_t(mine)) : int64_t(-1);
      }
    }
    __syncthreads();
  }
}

// lists: the fused search's per-segment tf32 lists (nlists sorted lists of
// k_in keys per query); more than 64 lists are first merged to one list of kc
// (into `scratch`, nq * kc keys).
int launch_refine_fp32(const uint64_t* lists, int nlists, int k_in, int64_t list_stride, int64_t q_stride,
                       uint64_t* scratch, int kc, const float* Q, const float* qn, const float* C, const float* cn,
                       int64_t nq, int dim, int64_t id_base, int k, const rs_config* keep, float* D, int64_t* I,
                       uint64_t* keys_out, int sms, cudaStream_t st) {
  RS_REQUIRE(kc >= k && kc <= 64 && dim % 4 == 0, "refine: bad shape");
  if (nlists > 64) {
    int rc = launch_merge(lists, nq, nlists, k_in, list_stride, q_stride, kc, nullptr, nullptr, nullptr, scratch, st);
    if (rc) return rc;
    lists = scratch;
    nlists = 1;
    k_in = kc;
    list_stride = kc;
    q_stride = kc;
  }
  // cand + exact (1 KB), the query row, the lists (<= 64 x 255 keys)
  const size_t smem = size_t(128 + 2 * (dim / 4) + nlists * k_in) * sizeof(uint64_t);
  RS_REQUIRE(smem <= 160 * 1024, "refine: %d lists x %d keys at d = %d exceed shared memory", nlists, k_in, dim);
  if (smem > 48 * 1024) {
    static bool opted = false;
    if (!opted) {
      RS_CHECK_CUDA(cudaFuncSetAttribute(refine_fp32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024),
                    "cudaFuncSetAttribute(refine_fp32_kernel)");
      opted = true;
    }
  }
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(nq, int64_t(sms) * (64 / kRefineWarps)));
  refine_fp32_kernel<<<(unsigned)blocks, kRefineWarps * 32, smem, st>>>(lists, nlists, k_in, list_stride, q_stride,
                                                                         kc, Q, qn, C, cn, nq, dim, id_base, k, keep,
                                                                         D, I, keys_out);
  RS_CHECK_LAUNCH("refine_fp32_kernel");
  return RS_OK;
}

int launch_norms(const void* x, int64_t n, int dim, int dtype, float* out, cudaStream_t st,
                 float* max_out, float* lo) {
  if (n <= 0) return RS_OK;
  const int64_t blocks = std::min<int64_t>(ceil_div(n * 32, 256), 148 * 64);
  unsigned int* mb = reinterpret_cast<unsigned int*>(max_out);
  if (dtype == RS_BF16)
    row_norms_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, st>>>((const __nv_bfloat16*)x, n, dim, out, mb,
                                                                      nullptr);
  else
    row_norms_kernel<float><<<(unsigned)blocks, 256, 0, st>>>((const float*)x, n, dim, out, mb, lo);
  RS_CHECK_LAUNCH("row_norms_kernel");
  return RS_OK;
}

template <typename T, int KCAP, int BUF>
constexpr size_t simt_dyn_bytes() {
  return size_t(KCAP + BUF) * BQ * sizeof(uint64_t);
}

template <typename T, int KCAP, int BUF>
int simt_prepare() {
  static bool done = false;
  if (!done) {
    RS_CHECK_CUDA(cudaFuncSetAttribute(score_topk_simt_kernel<T, KCAP, BUF>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(simt_dyn_bytes<T, KCAP, BUF>())),
                  "cudaFuncSetAttribute(score_topk_simt_kernel)");
    done = true;
  }
  return RS_OK;
}

template <typename T, int KCAP, int BUF>
int launch_simt_t(const void* Q, const float* qn, int64_t nq, const void* C, const float* cn, int64_t n, int dim,
                  int k, int64_t id_base, const SearchPlan& plan, uint64_t* part, cudaStream_t st) {
  int rc = simt_prepare<T, KCAP, BUF>();
  if (rc) return rc;
  score_topk_simt_kernel<T, KCAP, BUF><<<plan.ctas, 256, simt_dyn_bytes<T, KCAP, BUF>(), st>>>(
      (const T*)Q, qn, nq, (const T*)C, cn, n, dim, k, id_base, plan.qtiles, plan.segments, plan.seg_rows, part);
  RS_CHECK_LAUNCH("score_topk_simt_kernel");
  return RS_OK;
}

template <typename T, int KCAP, int BUF>
int simt_occ() {
  int occ = 1;
  simt_prepare<T, KCAP, BUF>();
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, score_topk_simt_kernel<T, KCAP, BUF>, 256,
                                                simt_dyn_bytes<T, KCAP, BUF>());
  return occ > 0 ? occ : 1;
}

int simt_ctas_per_sm(int dtype, int k) {
  if (dtype == RS_BF16) return k <= 40 ? simt_occ<__nv_bfloat16, 40, 32>() : simt_occ<__nv_bfloat16, 128, 32>();
  return k <= 40 ? simt_occ<float, 40, 32>() : simt_occ<float, 128, 32>();
}

int launch_simt(int dtype, const void* Q, const float* qn, int64_t nq, const void* C, const float* cn, int64_t n,
                int dim, int k, int64_t id_base, const SearchPlan& plan, uint64_t* part, cudaStream_t st) {
  if (dtype == RS_BF16)
    return k <= 40 ? launch_simt_t<__nv_bfloat16, 40, 32>(Q, qn, nq, C, cn, n, dim, k, id_base, plan, part, st)
                   : launch_simt_t<__nv_bfloat16, 128, 32>(Q, qn, nq, C, cn, n, dim, k, id_base, plan, part, st);
  return k <= 40 ? launch_simt_t<float, 40, 32>(Q, qn, nq, C, cn, n, dim, k, id_base, plan, part, st)
                 : launch_simt_t<float, 128, 32>(Q, qn, nq, C, cn, n, dim, k, id_base, plan, part, st);
}

}  // namespace

int launch_merge_wait(const uint64_t* keys, int64_t nq, int nlists, int k_in, int64_t list_stride, int64_t q_stride,
                      int k, const rs_config* keep, float* D, int64_t* I, const PeerWait& pw, cudaStream_t st) {
  RS_REQUIRE(nlists >= 1 && nlists <= 64, "nlists out of range (%d)", nlists);
  RS_REQUIRE(k_in >= 1 && k_in <= 255, "k_in out of range (%d)", k_in);
  // nq == 0: one block that only waits (keeps the exchange's epoch chain)
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(nq, kMergeWarps), 65535));
  PeerArgs pa{};
  pa.wait = pw;
  merge_topk64_kernel<kMergeWait><<<(unsigned)blocks, kMergeWarps * 32, 0, st>>>(keys, nq, nlists, k_in, list_stride,
                                                                                q_stride, k, keep, D, I, nullptr, pa);
  RS_CHECK_LAUNCH("merge_topk64_kernel<wait>");
  return RS_OK;
}

int launch_merge_to_peers(const uint64_t* keys, int64_t nq, int nlists, int k_in, int64_t list_stride,
                          int64_t q_stride, const rs_peer_exchange& ex, uint32_t epoch, cudaStream_t st) {
  RS_REQUIRE(nlists >= 1 && nlists <= 64, "nlists out of range (%d)", nlists);
  RS_REQUIRE(k_in >= 1 && k_in <= 255 && nq >= 1, "bad arguments");
  const int64_t blocks = std::min<int64_t>(ceil_div(nq, kMergeWarps), 65535);
  PeerArgs pa{};
  pa.ex = ex;
  pa.epoch = epoch;
  merge_topk64_kernel<kMergeScatter><<<(unsigned)blocks, kMergeWarps * 32, 0, st>>>(
      keys, nq, nlists, k_in, list_stride, q_stride, ex.k, nullptr, nullptr, nullptr, nullptr, pa);
  RS_CHECK_LAUNCH("merge_topk64_kernel<scatter>");
  return RS_OK;
}

// ---- per-chunk norm minima (the pair kernel's dot bound) ------------------------
__global__ void chunk_min_kernel(const float* __restrict__ norms, int64_t c_lo, int64_t c_hi, int64_t r1,
                                 float* __restrict__ cmin) {
  const int lane = threadIdx.x & 31;
  for (int64_t c = c_lo + ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5); c < c_hi;
       c += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int64_t r = c * 32 + lane;
    float v = r < r1 ? norms[r] : __int_as_float(0x7f800000);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, off));
    if (lane == 0) cmin[c] = v;
  }
}

int launch_chunk_min(const float* norms, int64_t r0, int64_t r1, float* cmin, cudaStream_t st) {
  if (r1 <= r0) return RS_OK;
  const int64_t c_lo = r0 / 32, c_hi = ceil_div(r1, 32);
  const int64_t blocks = std::min<int64_t>(ceil_div((c_hi - c_lo) * 32, 256), 148 * 16);
  chunk_min_kernel<<<(unsigned)blocks, 256, 0, st>>>(norms, c_lo, c_hi, r1, cmin);
  RS_CHECK_LAUNCH("chunk_min_kernel");
  return RS_OK;
}

// ---- planner -----------------------------------------------------------------
SearchPlan plan_search(int64_t nq, int64_t n, int bq, int bn, int ctas_capacity, int64_t row_bytes, bool share_l2) {
  SearchPlan best;
  const int64_t qt = ceil_div(std::max<int64_t>(nq, 1), bq);
  const int64_t nt = ceil_div(std::max<int64_t>(n, 1), bn);
  // With several query tiles the CTAs of one round share a segment through L2:
  // about ceil(ctas/qtiles)+1 segments are streamed at once, and together they
  // must stay L2-resident (ncu at 10M x 1024: 48 MB segments re-read the
  // corpus 17x from DRAM).  Budget 64 MB of the 126 MB L2 for the corpus
  // window (the query tiles are pinned evict_last next to it).
  int64_t max_tps = nt;
  // (The CTA-pair kernel schedules units dynamically in segment-major order,
  // so its concurrent units stay in lockstep without a segment-size cap and
  // long segments keep the per-column top-k candidate rate low; it passes
  // share_l2 = false.)
  if (share_l2 && qt > 1) {
    const int64_t concurrent = ceil_div(ctas_capacity, qt) + 1;
    max_tps = std::max<int64_t>(1, (int64_t(64) << 20) / (concurrent * int64_t(bn) * row_bytes));
  }
  // partial lists (8-byte keys, written then merged) must stay a small
  // fraction of the work: <= 4 GB, costed against the GEMM time below
  const int64_t list_bytes_per_seg = qt * int64_t(bq) * 40 * 8 * 2;
  const double tile_secs = 2.0 * bq * bn * (row_bytes / 2) / (1.2e15 / std::max(ctas_capacity, 1));
  double best_cost = 1e300;
  for (int64_t tps = nt; tps >= 1;) {
    const int64_t segs = ceil_div(nt, tps);
    if (segs > kMaxSegments) break;
    if (tps <= max_tps && (segs * list_bytes_per_seg <= (int64_t(4) << 30) || best_cost == 1e300)) {
      const int64_t units = qt * segs;
      const int64_t rounds = ceil_div(units, ctas_capacity);
      // per-unit overhead ~1 tile (pipeline fill + list write) + the merge's HBM traffic
      const double list_cost = double(segs * list_bytes_per_seg) / 6.5e12 / tile_secs;
      const double cost = double(rounds) * double(tps + 1) + list_cost;
      if (cost < best_cost) {
        best_cost = cost;
        best.qtiles = int32_t(qt);
        best.segments = int32_t(segs);
        best.seg_rows = tps * bn;
        best.ctas = int32_t(std::min<int64_t>(units, ctas_capacity));
      }
    }
    // next distinct segment count
    const int64_t nxt = ceil_div(nt, segs + 1);
    tps = (nxt < tps) ? nxt : tps - 1;
  }
  return best;
}

}  // namespace rs

// ============================ rs_index =========================================
using rs::DeviceGuard;

struct rs_index {
  int32_t dim = 0, dtype = 0, device = 0, algo = RS_ALGO_AUTO;
  int32_t walk_bias = 0;  // test hook (rs_index_set_walk_bias)
  int32_t seg_rows_override = 0;  // tuning knob (rs_index_set_segment_rows): 0 = the planner's choice
  int32_t probe_mode = 0;         // rs_index_set_probe: 0 off (default), 1 on (when the shape allows one)
  int32_t last_probe_rows = 0;    // rows the last search's probe pass scanned (0 = none)
  int64_t capacity = 0, ntotal = 0;
  void* data = nullptr;
  float* norms = nullptr;
  float* norm_max = nullptr;  // device scalar: max squared norm over the shard
  int32_t* sched_counter = nullptr;  // pair kernel: [0] units, [1] bursts, [2] finished CTAs, [3 + s] frontier of
                                     // segment s, [3 + kMaxSegments + u] position of unit u (drift limiter)
  // burst merge (rs_index_set_burst_merge): mode, the automatic choice, and the
  // last pair launch's burst count, posted by its last CTA to pinned memory
  int32_t burst_mode = -1;
  bool coop_active = false;
  uint32_t* burst_host = nullptr;
  double burst_tiles = 0.0;  // (32-row, 256-row) tiles of the launch whose count was copied last
  float* cmin = nullptr;      // [ceil(capacity/256)*8 + 8]: min squared norm per 32-row chunk
  float* lo = nullptr;        // fp32 index: [capacity, dim] tf32 residuals x - trunc_tf32(x) (3xTF32 path)
  float* qlo = nullptr;       // per-search query residuals [qlo_cap, dim]
  int64_t qlo_cap = 0;
  uint64_t* cand = nullptr;   // fp32 path with > 64 lists: merged 3xTF32 candidates [nq, kc] before the re-rank
  size_t cand_cap = 0;        // bytes
  float* qnorm = nullptr;
  uint32_t* qtau = nullptr;   // pair kernel: per-query shared k-th distance (threshold sharing)
  int64_t qnorm_cap = 0;
  uint64_t* part = nullptr;
  size_t part_cap = 0;  // bytes
  uint64_t* skeys = nullptr;  // rs_index_search_scatter: local key rows when the merge cannot store to peers
  size_t skeys_cap = 0;       // bytes
  rs::SearchPlan last;
  int32_t last_algo = 0;
  // optional per-search timing of the fused score kernel (event ring)
  bool timing = false;
  static constexpr int kRing = 512;
  cudaEvent_t ev_start[kRing] = {}, ev_stop[kRing] = {};
  int ev_next = 0, ev_pending = 0;
};

namespace {
size_t esize(int dtype) { return dtype == RS_BF16 ? 2 : 4; }

int ensure_ws(rs_index* ix, int64_t nq, size_t part_bytes) {
  if (ix->dtype == RS_F32 && nq > ix->qlo_cap) {
    if (ix->qlo) cudaFree(ix->qlo);
    ix->qlo = nullptr;
    RS_CHECK_CUDA(cudaMalloc(&ix->qlo, sizeof(float) * size_t(nq) * ix->dim), "cudaMalloc(query tf32 residuals)");
    ix->qlo_cap = nq;
  }
  if (nq > ix->qnorm_cap) {
    if (ix->qnorm) cudaFree(ix->qnorm);
    ix->qnorm = nullptr;
    RS_CHECK_CUDA(cudaMalloc(&ix->qnorm, sizeof(float) * nq), "cudaMalloc(qnorm)");
    if (ix->qtau) cudaFree(ix->qtau);
    ix->qtau = nullptr;
    RS_CHECK_CUDA(cudaMalloc(&ix->qtau, sizeof(uint32_t) * nq * rs::kSharedBoundWords), "cudaMalloc(qtau)");
    ix->qnorm_cap = nq;
  }
  if (part_bytes > ix->part_cap) {
    if (ix->part) cudaFree(ix->part);
    ix->part = nullptr;
    RS_CHECK_CUDA(cudaMalloc(&ix->part, part_bytes), "cudaMalloc(partial top-k)");
    ix->part_cap = part_bytes;
  }
  return RS_OK;
}

// Concrete kernel for a search: the CTA-pair tcgen05 kernel (default; bf16,
// or 3xTF32 for an fp32 corpus), the single-CTA tcgen05 kernel on request
// (bf16), else the CUDA-core kernel (k > 40, odd dims, or on request).
int choose_algo(const rs_index* ix, int k) {
  const bool tc_ok = k <= rs::kTcMaxK && (ix->dtype == RS_BF16 ? ix->dim % 8 == 0 : ix->dim % 4 == 0);
  if (ix->algo == RS_ALGO_SIMT || !tc_ok) return RS_ALGO_SIMT;
  if (ix->algo == RS_ALGO_TCGEN05_1SM && ix->dtype == RS_BF16) return RS_ALGO_TCGEN05_1SM;
  return RS_ALGO_TCGEN05;
}

// small batches take the CTA pair's M = 128 tile: one tile, no padding rows
bool pair_small(int64_t nq) { return nq <= rs::kSmallBatchMax && rs::kPairGroup == 1 && rs::kPairEpiGroups == 1; }

rs::SearchPlan make_plan(const rs_index* ix, int algo, int64_t nq, int64_t n, int k) {
  using namespace rs;
  const int sms = sm_count(ix->device);
  if (algo == RS_ALGO_TCGEN05) {  // units of one cluster: kPairGroup pair tiles
    // tile cost in bf16-equivalent K: 3 tf32 passes at half the bf16 rate
    const int64_t eq_row_bytes = int64_t(ix->dim) * 2 * (ix->dtype == RS_BF16 ? 1 : 6);
    const bool small = pair_small(nq);
    SearchPlan p = plan_search(nq, n, pair_tile_rows(small) * kPairGroup, kTcBN, sms / (2 * kPairGroup),
                               eq_row_bytes, /*share_l2=*/false);
    if (ix->seg_rows_override > 0) {  // fixed segment length (rounded to whole tiles)
      const int64_t tps = std::max<int64_t>(1, ix->seg_rows_override / kTcBN);
      const int64_t nt = ceil_div(std::max<int64_t>(n, 1), kTcBN);
      p.segments = int32_t(std::min<int64_t>(ceil_div(nt, std::min(tps, nt)), kMaxSegments));
      p.seg_rows = ceil_div(nt, p.segments) * kTcBN;
      p.segments = int32_t(ceil_div(nt * kTcBN, p.seg_rows));
      p.ctas = int32_t(std::min<int64_t>(int64_t(p.qtiles) * p.segments, sms / (2 * kPairGroup)));
    }
    p.lists_per_seg = small ? 2 : kPairEpiGroups;
    const int pairs = sms / (2 * kPairGroup);
    const int64_t units = int64_t(p.qtiles) * p.segments;
#ifndef RS_PAIR_SYNC_PARTIAL_ROUND  // experiment: also a single round with up to qtiles - 1 idle pairs (measured: no gain, profiles/r2_drift_limiter.md)
#define RS_PAIR_SYNC_PARTIAL_ROUND 0
#endif
    const bool one_round = RS_PAIR_SYNC_PARTIAL_ROUND ? (units <= pairs && units > pairs - p.qtiles) : units == pairs;
    p.sync_tiles = (kPairGroup == 1 && !small && p.qtiles >= 2 && p.qtiles <= kSyncMaxQtiles && one_round)
                       ? RS_PAIR_SYNC_TILES : 0;
    return p;
  }
  if (algo == RS_ALGO_TCGEN05_1SM) return plan_search(nq, n, kTcBM, kTcBN, sms, int64_t(ix->dim) * 2, true);
  return plan_search(nq, n, kSimtBQ, kSimtBC, sms * simt_ctas_per_sm(ix->dtype, k),
                     int64_t(ix->dim) * esize(ix->dtype), true);
}

// Probe pass of the CTA-pair kernel (rs_index_set_probe; measured and off by
// default).  When every unit of a search runs in about one round (cfg1: 1,000
// queries x 100k rows, 72 units of 22 tiles), every per-segment list starts
// empty at the same time and a unit's first tiles admit nearly every column
// (45% of cfg1's epilogue busy cycles).  The probe runs the same kernel first
// over the corpus's first S rows, one tile per segment (one round of units),
// and folds the kCas-th smallest of those lists' rank-ceil(k/kCas) distances
// into qtau: a valid bound of every query's final k-th distance (>= k real
// rows at or below it, distances bit-identical to the main launch's), so the
// main launch's lists admit from their first tile.  Results are bit-identical
// with or without it.  Measured at cfg1 (ncu launch list): the main launch
// 641 -> 622 us, but the probe itself 105 us — its one-tile lists are all cold
// start, the cost it was meant to remove — so the default is off.  Returns
// the probe's plan (segments = 0: no probe).
constexpr int kProbeMinLists = 4 * rs::kPairEpiGroups;  // the cascade needs kCas disjoint lists
rs::SearchPlan probe_plan(const rs_index* ix, int algo, int64_t nq, const rs::SearchPlan& main) {
  using namespace rs;
  SearchPlan pp = main;
  pp.segments = 0;
  if (algo != RS_ALGO_TCGEN05 || ix->probe_mode != 1 || pair_small(nq) || kPairGroup != 1) return pp;
  const int pairs = sm_count(ix->device) / 2;
  const int64_t tiles = ix->ntotal / kTcBN;  // whole tiles only (no partial-tile rows)
  const int64_t segs = std::min<int64_t>({int64_t(pairs / std::max(main.qtiles, 1)), 16, tiles / 16});
  if (segs < kProbeMinLists) return pp;
  pp.segments = int32_t(segs);
  pp.seg_rows = kTcBN;
  pp.sync_tiles = 0;
  pp.ctas = int32_t(std::min<int64_t>(int64_t(main.qtiles) * segs, pairs));
  return pp;
}

// Lean or cooperative pair-kernel variant (rs_index_set_burst_merge).  In the
// automatic mode the previous launch's burst count (posted to pinned memory by
// its last CTA; read without a synchronisation, so possibly one search stale) is normalised by
// that launch's (32-row, 256-row) tile visits: isotropic data measures
// ~1e-4 bursty flushes per visit, a doc-contiguous corpus 0.03-0.2
// (profiles/r2_burst_merge.md).
constexpr double kBurstOn = 4e-3, kBurstOff = 1e-3;
bool burst_choice(rs_index* ix) {
  if (ix->burst_mode >= 0) return ix->burst_mode != 0;
  if (ix->burst_tiles > 0.0) {
    const double rate = double(*reinterpret_cast<volatile uint32_t*>(ix->burst_host)) / ix->burst_tiles;
    if (rate > kBurstOn) ix->coop_active = true;
    else if (rate < kBurstOff) ix->coop_active = false;
  }
  return ix->coop_active;
}

// partial lists for (queries x this shard) -> part; returns the plan
int run_partial(rs_index* ix, const void* queries, int64_t nq, int k, int64_t id_base, cudaStream_t st,
                rs::SearchPlan* plan_out, int algo_for_k = -1) {
  using namespace rs;
  // algo_for_k: the user's k when this pass keeps more candidates than k (the
  // fp32 re-rank pass), so the kernel choice follows the user's k
  const int algo = choose_algo(ix, algo_for_k >= 0 ? algo_for_k : k);
  RS_REQUIRE(!((ix->algo == RS_ALGO_TCGEN05 || ix->algo == RS_ALGO_TCGEN05_1SM) && algo == RS_ALGO_SIMT),
             "tcgen05 path needs 16-byte rows (bf16 dim %% 8, fp32 dim %% 4) and k <= %d", kTcMaxK);
  RS_REQUIRE(!(ix->algo == RS_ALGO_TCGEN05_1SM && ix->dtype != RS_BF16), "the single-CTA tcgen05 kernel is bf16-only");
  const SearchPlan plan = make_plan(ix, algo, nq, ix->ntotal, k);
  const SearchPlan pplan = probe_plan(ix, algo, nq, plan);
  // the probe's lists go to the same buffer, overwritten by the main launch
  const size_t part_bytes = size_t(nq) * std::max(plan.lists(), pplan.lists()) * k * sizeof(uint64_t);
  int rc = ensure_ws(ix, nq, part_bytes);
  if (rc) return rc;
  // 3xTF32 (fp32 corpus on the tensor cores): the same pass splits the queries
  const bool tf_split = ix->dtype == RS_F32 && algo == RS_ALGO_TCGEN05;
  rc = launch_norms(queries, nq, ix->dim, ix->dtype, ix->qnorm, st, nullptr, tf_split ? ix->qlo : nullptr);
  if (rc) return rc;
  const int slot = ix->ev_next;
  if (ix->timing) {
    if (!ix->ev_start[slot]) {
      RS_CHECK_CUDA(cudaEventCreate(&ix->ev_start[slot]), "cudaEventCreate");
      RS_CHECK_CUDA(cudaEventCreate(&ix->ev_stop[slot]), "cudaEventCreate");
    }
    RS_CHECK_CUDA(cudaEventRecord(ix->ev_start[slot], st), "cudaEventRecord");
  }
  if (algo != RS_ALGO_SIMT) {
    const bool pair = algo == RS_ALGO_TCGEN05;
    const bool tf = ix->dtype == RS_F32;
    CUtensorMap tmq, tmc, tmql, tmcl;
    const int crows = pair ? kTcBN / 2 / kPairGroup : kTcBN;
    const bool small = pair && pair_small(nq);
    const int qrows = pair ? pair_tile_rows(small) / 2 : kTcBM;  // query rows per CTA
    rc = encode_kmajor_map(&tmq, queries, nq, ix->dim, qrows, ix->dtype);
    if (rc) return rc;
    rc = encode_kmajor_map(&tmc, ix->data, ix->ntotal, ix->dim, crows, ix->dtype);
    if (rc) return rc;
    if (tf) {  // 3xTF32: the residuals (the queries' from launch_norms above, the corpus's from add)
      rc = encode_kmajor_map(&tmql, ix->qlo, nq, ix->dim, qrows, RS_F32);
      if (rc) return rc;
      if (RS_TF32_STORED_LO) {
        rc = encode_kmajor_map(&tmcl, ix->lo, ix->ntotal, ix->dim, crows, RS_F32);
        if (rc) return rc;
      }
    }
    if (pair) {
      const bool coop = burst_choice(ix);
      const bool count = ix->burst_mode < 0;  // automatic: this launch's count, for the next search's choice
      const bool probe = pplan.segments > 0;
      ix->last_probe_rows = probe ? int32_t(int64_t(pplan.segments) * pplan.seg_rows) : 0;
      if (probe) {  // the same kernel over the first rows (probe_plan), then fold the bound
        rc = launch_score_topk_pair(tmq, tf ? &tmql : nullptr, tmc, (tf && RS_TF32_STORED_LO) ? &tmcl : nullptr,
                                    ix->qnorm, ix->norms, ix->cmin, nq, ix->last_probe_rows, ix->dim, k, id_base,
                                    pplan, small, ix->part, ix->sched_counter, 0, ix->qtau, coop, nullptr, st);
        if (rc == RS_OK) rc = launch_fold_probe_bounds(ix->qtau, nq, st);
        if (rc) return rc;
      }
      rc = launch_score_topk_pair(tmq, tf ? &tmql : nullptr, tmc, (tf && RS_TF32_STORED_LO) ? &tmcl : nullptr,
                                  ix->qnorm, ix->norms, ix->cmin, nq, ix->ntotal, ix->dim, k, id_base, plan, small,
                                  ix->part, ix->sched_counter, ix->walk_bias, ix->qtau, coop,
                                  count ? ix->burst_host : nullptr, st, probe);
      if (rc == RS_OK && count)
        ix->burst_tiles = double(plan.qtiles) * pair_tile_rows(small) / 32.0 * double(ceil_div(ix->ntotal, kTcBN));
    } else {
      rc = launch_score_topk_tc(tmq, tmc, ix->qnorm, ix->norms, nq, ix->ntotal, ix->dim, k, id_base, plan, ix->part,
                                st);
    }
  } else {
    rc = launch_simt(ix->dtype, queries, ix->qnorm, nq, ix->data, ix->norms, ix->ntotal, ix->dim, k, id_base, plan,
                     ix->part, st);
  }
  if (rc) return rc;
  if (ix->timing) {
    RS_CHECK_CUDA(cudaEventRecord(ix->ev_stop[slot], st), "cudaEventRecord");
    ix->ev_next = (slot + 1) % rs_index::kRing;
    if (ix->ev_pending < rs_index::kRing) ++ix->ev_pending;
  }
  ix->last = plan;
  ix->last_algo = algo;
  *plan_out = plan;
  return RS_OK;
}

int check_search_args(const rs_index* ix, const void* q, int64_t nq, int32_t k, int64_t id_base) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  RS_REQUIRE(nq >= 0, "nq must be non-negative");
  RS_REQUIRE(k >= 1 && k <= 128, "k must be in [1, 128], got %d", k);
  RS_REQUIRE(nq == 0 || q != nullptr, "queries is NULL");
  RS_REQUIRE(id_base >= 0 && id_base + ix->ntotal < (int64_t(1) << 32) - 1,
             "global chunk ids must fit in uint32 (id_base %lld + ntotal %lld)", (long long)id_base,
             (long long)ix->ntotal);
  return RS_OK;
}
}  // namespace

extern "C" int rs_index_create(int32_t dim, int32_t dtype, int64_t capacity, int32_t device, rs_index** out) {
  RS_REQUIRE(out != nullptr, "out is NULL");
  RS_REQUIRE(dim >= 1 && dim <= 65536, "dim out of range");
  RS_REQUIRE(dtype == RS_F32 || dtype == RS_BF16, "dtype must be RS_F32 or RS_BF16");
  RS_REQUIRE(capacity >= 0, "capacity must be non-negative");
  if (!rs_device_supported(device)) {
    rs::set_error("device %d is not an sm_100 (B200) GPU", device);
    return RS_ERR_UNSUPPORTED;
  }
  DeviceGuard g(device);
  rs_index* ix = new rs_index();
  ix->dim = dim;
  ix->dtype = dtype;
  ix->device = device;
  ix->capacity = capacity;
  if (capacity > 0) {
    cudaError_t e = cudaMalloc(&ix->data, size_t(capacity) * dim * esize(dtype));
    // + one column tile of padding: the fused kernel bulk-copies whole 16-byte
    // granules of norms past the last row of a partial tile
    if (e == cudaSuccess) e = cudaMalloc(&ix->norms, sizeof(float) * (capacity + rs::kTcBN));
    if (e == cudaSuccess) e = cudaMalloc(&ix->norm_max, sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&ix->sched_counter,
                                             sizeof(int32_t) * (3 + rs::kMaxSegments * (1 + rs::kSyncMaxQtiles)));
    if (e == cudaSuccess) e = cudaHostAlloc(&ix->burst_host, sizeof(uint32_t), cudaHostAllocDefault);
    if (e == cudaSuccess) *ix->burst_host = 0;
    if (e == cudaSuccess && dtype == RS_F32 && RS_TF32_STORED_LO && dim % 4 == 0)
      e = cudaMalloc(&ix->lo, size_t(capacity) * dim * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&ix->cmin, sizeof(float) * (rs::ceil_div(capacity, 256) * 8 + 8));
    if (e == cudaSuccess) e = cudaMemset(ix->norm_max, 0, sizeof(float));
    if (e != cudaSuccess) {
      rs::set_error("cudaMalloc(corpus %lld x %d): %s", (long long)capacity, dim, cudaGetErrorString(e));
      if (ix->data) cudaFree(ix->data);
      delete ix;
      return RS_ERR_OOM;
    }
  }
  *out = ix;
  return RS_OK;
}

extern "C" int rs_index_enable_timing(rs_index* ix, int32_t enable) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  ix->timing = enable != 0;
  ix->ev_pending = 0;
  return RS_OK;
}

extern "C" int rs_index_kernel_times(rs_index* ix, float* ms_out, int32_t max, int32_t* count) {
  RS_REQUIRE(ix != nullptr && count != nullptr, "NULL argument");
  DeviceGuard g(ix->device);
  const int n = ix->ev_pending < max ? ix->ev_pending : max;
  for (int i = 0; i < n; ++i) {
    // oldest first
    const int slot = (ix->ev_next - ix->ev_pending + i + rs_index::kRing) % rs_index::kRing;
    float ms = 0.0f;
    RS_CHECK_CUDA(cudaEventElapsedTime(&ms, ix->ev_start[slot], ix->ev_stop[slot]), "cudaEventElapsedTime");
    if (ms_out) ms_out[i] = ms;
  }
  *count = n;
  ix->ev_pending = 0;
  return RS_OK;
}

extern "C" int rs_index_destroy(rs_index* ix) {
  if (!ix) return RS_OK;
  DeviceGuard g(ix->device);
  for (int i = 0; i < rs_index::kRing; ++i) {
    if (ix->ev_start[i]) cudaEventDestroy(ix->ev_start[i]);
    if (ix->ev_stop[i]) cudaEventDestroy(ix->ev_stop[i]);
  }
  cudaFree(ix->data);
  cudaFree(ix->norms);
  cudaFree(ix->norm_max);
  cudaFree(ix->sched_counter);
  if (ix->burst_host) cudaFreeHost(ix->burst_host);
  cudaFree(ix->lo);
  cudaFree(ix->cmin);
  cudaFree(ix->qlo);
  cudaFree(ix->cand);
  cudaFree(ix->qnorm);
  cudaFree(ix->qtau);
  cudaFree(ix->part);
  cudaFree(ix->skeys);
  delete ix;
  return RS_OK;
}

extern "C" int rs_index_add(rs_index* ix, const void* emb, int64_t n, void* stream) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  RS_REQUIRE(n >= 0, "n must be non-negative");
  if (n == 0) return RS_OK;
  RS_REQUIRE(emb != nullptr, "embeddings is NULL");
  RS_REQUIRE(ix->ntotal + n <= ix->capacity, "index capacity exceeded (%lld + %lld > %lld)",
             (long long)ix->ntotal, (long long)n, (long long)ix->capacity);
  DeviceGuard g(ix->device);
  cudaStream_t st = rs::as_stream(stream);
  const size_t row = size_t(ix->dim) * esize(ix->dtype);
  RS_CHECK_CUDA(cudaMemcpyAsync((char*)ix->data + size_t(ix->ntotal) * row, emb, size_t(n) * row,
                                cudaMemcpyDeviceToDevice, st),
                "cudaMemcpyAsync(add)");
  // + the 3xTF32 residuals of the new rows (fp32, dim % 4 == 0: the tcgen05 path exists)
  int rc = rs::launch_norms((char*)ix->data + size_t(ix->ntotal) * row, n, ix->dim, ix->dtype,
                            ix->norms + ix->ntotal, st, ix->norm_max,
                            ix->lo ? ix->lo + size_t(ix->ntotal) * ix->dim : nullptr);
  if (rc) return rc;
  rc = rs::launch_chunk_min(ix->norms, ix->ntotal, ix->ntotal + n, ix->cmin, st);
  if (rc) return rc;
  ix->ntotal += n;
  return RS_OK;
}

extern "C" int rs_index_reset(rs_index* ix) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  ix->ntotal = 0;
  if (ix->norm_max) {
    DeviceGuard g(ix->device);
    RS_CHECK_CUDA(cudaMemset(ix->norm_max, 0, sizeof(float)), "cudaMemset(norm_max)");
  }
  return RS_OK;
}

extern "C" int rs_index_ntotal(const rs_index* ix, int64_t* out) {
  RS_REQUIRE(ix && out, "NULL argument");
  *out = ix->ntotal;
  return RS_OK;
}

extern "C" int rs_index_data(const rs_index* ix, const void** emb, const float** norms) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  if (emb) *emb = ix->data;
  if (norms) *norms = ix->norms;
  return RS_OK;
}

extern "C" int rs_index_set_segment_rows(rs_index* ix, int32_t rows) {
  RS_REQUIRE(ix != nullptr && rows >= 0, "bad arguments");
  ix->seg_rows_override = rows;
  return RS_OK;
}

extern "C" int rs_index_set_probe(rs_index* ix, int32_t mode) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  RS_REQUIRE(mode == 0 || mode == 1, "probe mode must be 0 or 1, got %d", mode);
  ix->probe_mode = mode;
  return RS_OK;
}

extern "C" int rs_index_last_probe_rows(const rs_index* ix, int32_t* rows) {
  RS_REQUIRE(ix != nullptr && rows != nullptr, "NULL argument");
  *rows = ix->last_probe_rows;
  return RS_OK;
}

extern "C" int rs_index_set_burst_merge(rs_index* ix, int32_t mode) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  RS_REQUIRE(mode >= -1 && mode <= 1, "burst merge mode must be -1 (auto), 0 or 1, got %d", mode);
  ix->burst_mode = mode;
  ix->burst_tiles = 0.0;
  if (mode >= 0) ix->coop_active = mode != 0;
  return RS_OK;
}

extern "C" int rs_index_burst_merge_active(rs_index* ix, int32_t* active) {
  RS_REQUIRE(ix != nullptr && active != nullptr, "NULL argument");
  if (ix->burst_mode >= 0) {
    *active = ix->burst_mode;
    return RS_OK;
  }
  // the automatic choice the next search makes from the counts copied so far
  DeviceGuard g(ix->device);
  *active = burst_choice(ix) ? 1 : 0;
  return RS_OK;
}

extern "C" int rs_index_set_walk_bias(rs_index* ix, int32_t bias) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  RS_REQUIRE(bias >= 0 && bias < (1 << 16), "walk bias out of range (%d)", bias);
  ix->walk_bias = bias;
  return RS_OK;
}

extern "C" int rs_index_set_algo(rs_index* ix, int32_t algo) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  RS_REQUIRE(algo >= RS_ALGO_AUTO && algo <= RS_ALGO_TCGEN05_1SM, "unknown algo %d", algo);
  ix->algo = algo;
  return RS_OK;
}

extern "C" int rs_index_reserve(rs_index* ix, int64_t nq_max, int32_t k) {
  using namespace rs;
  RS_REQUIRE(ix != nullptr && nq_max >= 0 && k >= 1, "bad arguments");
  DeviceGuard g(ix->device);
  // worst case over the expected corpus size (capacity)
  const int algo = choose_algo(ix, k);
  // the fp32 tensor-core search keeps k + kRefineExtra candidates per list
  const int kk = (ix->dtype == RS_F32 && algo == RS_ALGO_TCGEN05) ? k + kRefineExtra : k;
  const SearchPlan plan = make_plan(ix, algo, nq_max, std::max<int64_t>(ix->capacity, 1), kk);
  return ensure_ws(ix, nq_max, size_t(nq_max) * plan.lists() * kk * sizeof(uint64_t));
}

extern "C" int rs_index_last_plan(const rs_index* ix, int32_t* segments, int32_t* qtiles, int32_t* ctas,
                                  int32_t* algo) {
  RS_REQUIRE(ix != nullptr, "index is NULL");
  if (segments) *segments = ix->last.segments;
  if (qtiles) *qtiles = ix->last.qtiles;
  if (ctas) *ctas = ix->last.ctas;
  if (algo) *algo = ix->last_algo;
  return RS_OK;
}

static int search_impl(rs_index* ix, const void* queries, int64_t nq, int32_t k, int64_t id_base,
                       const rs_config* keep, float* D, int64_t* I, uint64_t* keys, void* stream,
                       const rs_peer_exchange* px = nullptr, uint32_t epoch = 0) {
  using namespace rs;
  int rc = check_search_args(ix, queries, nq, k, id_base);
  if (rc) return rc;
  DeviceGuard g(ix->device);
  cudaStream_t st = as_stream(stream);
  if (px && nq > 0) {  // the key rows are built locally unless the final merge stores them to the peers
    const size_t kb = size_t(nq) * k * sizeof(uint64_t);
    if (kb > ix->skeys_cap) {
      if (ix->skeys) cudaFree(ix->skeys);
      ix->skeys = nullptr;
      RS_CHECK_CUDA(cudaMalloc(&ix->skeys, kb), "cudaMalloc(scatter keys)");
      ix->skeys_cap = kb;
    }
    keys = ix->skeys;
  }
  // after a local result: the peer scatter of its key rows (nq == 0 still signals)
  auto finish = [&](int r) { return (r || !px) ? r : launch_peer_scatter(*px, keys, nq, epoch, st); };
  if (nq == 0) return finish(RS_OK);
  if (ix->ntotal == 0) {
    fill_empty_kernel<<<(unsigned)std::min<int64_t>(ceil_div(nq * k, 256), 4096), 256, 0, st>>>(nq * k, D, I, keys);
    RS_CHECK_LAUNCH("fill_empty_kernel");
    return finish(RS_OK);
  }
  SearchPlan plan;
  if (ix->dtype == RS_F32 && choose_algo(ix, k) == RS_ALGO_TCGEN05) {
    // 3xTF32 candidates (kc per query) -> exact fp32 re-rank to k
    const int kc = k + kRefineExtra;  // <= kTcMaxK + kRefineExtra: the tf32 lists' capacity
    rc = run_partial(ix, queries, nq, kc, id_base, st, &plan, k);
    if (rc) return rc;
    if (plan.lists() > 64) {  // the candidate lists are merged to one list of kc first
      const size_t cb = size_t(nq) * kc * sizeof(uint64_t);
      if (cb > ix->cand_cap) {
        if (ix->cand) cudaFree(ix->cand);
        ix->cand = nullptr;
        RS_CHECK_CUDA(cudaMalloc(&ix->cand, cb), "cudaMalloc(refine candidates)");
        ix->cand_cap = cb;
      }
    }
    return finish(launch_refine_fp32(ix->part, plan.lists(), kc, kc, int64_t(plan.lists()) * kc, ix->cand, kc,
                                     static_cast<const float*>(queries), ix->qnorm,
                                     static_cast<const float*>(ix->data), ix->norms, nq, ix->dim, id_base, k, keep,
                                     D, I, keys, sm_count(ix->device), st));
  }
  rc = run_partial(ix, queries, nq, k, id_base, st, &plan);
  if (rc) return rc;
  if (px && plan.lists() <= 64)  // the merge and the exchange in one kernel
    return launch_merge_to_peers(ix->part, nq, plan.lists(), k, /*list_stride=*/k,
                                 /*q_stride=*/int64_t(plan.lists()) * k, *px, epoch, st);
  return finish(launch_merge(ix->part, nq, plan.lists(), k, /*list_stride=*/k, /*q_stride=*/int64_t(plan.lists()) * k,
                             k, keep, D, I, keys, st));
}

extern "C" int rs_index_search(rs_index* ix, const void* queries, int64_t nq, int32_t k, int64_t id_base,
                               const rs_config* keep, float* D, int64_t* I, void* stream) {
  RS_REQUIRE(nq == 0 || (D != nullptr && I != nullptr), "D/I are NULL");
  return search_impl(ix, queries, nq, k, id_base, keep, D, I, nullptr, stream);
}

extern "C" int rs_index_search_keys(rs_index* ix, const void* queries, int64_t nq, int32_t k, int64_t id_base,
                                    uint64_t* keys, void* stream) {
  RS_REQUIRE(nq == 0 || keys != nullptr, "keys is NULL");
  return search_impl(ix, queries, nq, k, id_base, nullptr, nullptr, nullptr, keys, stream);
}

extern "C" int rs_index_search_scatter(rs_index* ix, const void* queries, int64_t nq, int32_t k, int64_t id_base,
                                       const rs_peer_exchange* ex, uint32_t epoch, void* stream) {
  int rc = rs::check_peer_exchange(ex);
  if (rc) return rc;
  RS_REQUIRE(ex->k == k, "k (%d) must equal the exchange's k (%d)", k, ex->k);
  RS_REQUIRE(nq >= 0 && rs::ceil_div(nq, ex->world) <= ex->slice_cap, "nq %lld exceeds world x slice_cap",
             (long long)nq);
  return search_impl(ix, queries, nq, k, id_base, nullptr, nullptr, nullptr, nullptr, stream, ex, epoch);
}

extern "C" int rs_merge_topk(const uint64_t* keys, int64_t nq, int32_t nlists, int32_t k_in, int64_t list_stride,
                             int32_t k, const rs_config* cfg, float* D, int64_t* I, void* stream) {
  RS_REQUIRE(nq >= 0 && k >= 1 && k <= 128, "bad arguments");
  if (nq == 0) return RS_OK;
  RS_REQUIRE(D && I, "D/I are NULL");
  return rs::launch_merge(keys, nq, nlists, k_in, list_stride, /*q_stride=*/k_in, k, cfg, D, I, nullptr,
                          rs::as_stream(stream));
}

extern "C" int rs_row_norms(const void* x, int64_t n, int32_t dim, int32_t dtype, float* out, void* stream) {
  RS_REQUIRE(n >= 0 && dim >= 1 && (dtype == RS_F32 || dtype == RS_BF16), "bad arguments");
  if (n == 0) return RS_OK;
  return rs::launch_norms(x, n, dim, dtype, out, rs::as_stream(stream), nullptr, nullptr);
}
