// Streaming per-row top-k used by the fused score+select epilogues.
//
// One thread owns one query row.  Scores arrive in ascending chunk-id order.
// A candidate passes a register threshold test (d <= tau, tau = current k-th
// best distance) and is appended to a small per-row buffer in shared memory
// (a predicated store — no divergence on the common reject path).  When any
// lane of the warp nears a full buffer the whole warp flushes in lockstep:
// each lane pushes its buffered keys into its own bounded max-heap (root =
// current k-th best), then refreshes tau.  Keys are packed u64
// (fp32 distance bits << 32 | uint32 chunk id) so the heap order is exactly
// (distance asc, id asc) — the north star's lower-index tie rule.
//
// Shared-memory layout is slot-major ([slot][row]) so lanes touching the
// same slot hit consecutive 8-byte words.
#pragma once

#include <stdint.h>

namespace rs {

__device__ __forceinline__ uint64_t make_key(float d, uint32_t id) {
  return (uint64_t(__float_as_uint(d)) << 32) | id;
}
__device__ __forceinline__ float key_dist(uint64_t k) { return __uint_as_float(uint32_t(k >> 32)); }

template <int ROWS, int BUF>
struct RowTopK {
  uint64_t* heap;  // [k][ROWS]   (slot-major)
  uint64_t* buf;   // [BUF][ROWS]
  int row;
  int k;
  int nk;  // heap size
  int nb;  // buffered candidates
  float tau;

  __device__ __forceinline__ void reset() {
    nk = 0;
    nb = 0;
    tau = __int_as_float(0x7f800000);  // +inf
  }

  __device__ __forceinline__ uint64_t& H(int i) { return heap[i * ROWS + row]; }

  // Predicated append of one candidate.
  __device__ __forceinline__ void offer(float d, uint32_t id) {
    if (d <= tau) append(d, id);
  }
  __device__ __forceinline__ void append(float d, uint32_t id) {
    buf[nb * ROWS + row] = make_key(d, id);
    ++nb;
  }

  __device__ void push(uint64_t key) {
    if (nk < k) {  // sift up
      int i = nk++;
      while (i > 0) {
        const int p = (i - 1) >> 1;
        const uint64_t pk = H(p);
        if (pk >= key) break;
        H(i) = pk;
        i = p;
      }
      H(i) = key;
    } else if (key < H(0)) {  // replace root, sift down
      int i = 0;
      for (;;) {
        int c = 2 * i + 1;
        if (c >= nk) break;
        uint64_t ck = H(c);
        if (c + 1 < nk) {
          const uint64_t c2 = H(c + 1);
          if (c2 > ck) {
            ck = c2;
            ++c;
          }
        }
        if (ck <= key) break;
        H(i) = ck;
        i = c;
      }
      H(i) = key;
    }
  }

  __device__ void flush() {
    for (int j = 0; j < nb; ++j) push(buf[j * ROWS + row]);
    nb = 0;
    if (nk == k) tau = key_dist(H(0));
  }

  // Heap-sort in place (ascending) and write k keys (kEmpty-padded).
  __device__ void finish(uint64_t* __restrict__ out) {
    flush();
    for (int end = nk - 1; end > 0; --end) {
      const uint64_t top = H(0);
      const uint64_t key = H(end);
      H(end) = top;
      int i = 0;
      for (;;) {
        int c = 2 * i + 1;
        if (c >= end) break;
        uint64_t ck = H(c);
        if (c + 1 < end) {
          const uint64_t c2 = H(c + 1);
          if (c2 > ck) {
            ck = c2;
            ++c;
          }
        }
        if (ck <= key) break;
        H(i) = ck;
        i = c;
      }
      H(i) = key;
    }
    for (int j = 0; j < k; ++j) out[j] = j < nk ? H(j) : ~0ull;
  }
};

// Epilogue fast path for 8 columns of one query row (fp32 dots `r` from
// TMEM, corpus norms `cn` in smem): 3 instructions per score (FADD
// |q|^2+|c|^2, FFMA -2<q,c>, FSETP d <= tau, the compiler folds the 8 compares
// into FMNMX3 + one FSETP) plus one warp vote per group; candidate append and
// heap maintenance only run when some lane of the warp has a candidate (rare
// once the heaps are full).  Exact: the filter uses the same rounded distance
// that is stored.
template <int ROWS, int BUF, int CHECK, bool FULL>
__device__ __forceinline__ void epi_group8(RowTopK<ROWS, BUF>& rt, const uint32_t* r, const float* cn, float qnv,
                                           uint32_t id, int lim) {
  static_assert(BUF >= CHECK, "buffer must hold one group");
  const float4 a = *reinterpret_cast<const float4*>(cn);
  const float4 b = *reinterpret_cast<const float4*>(cn + 4);
  const float cv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  float e[8];
  bool hit = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    e[j] = fmaf(-2.0f, __uint_as_float(r[j]), qnv + cv[j]);
    hit |= (FULL || j < lim) && e[j] <= rt.tau;
  }
  if (__any_sync(0xffffffffu, hit)) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if ((FULL || j < lim) && e[j] <= rt.tau) rt.append(e[j] > 0.0f ? e[j] : 0.0f, id + j);
    if (__any_sync(0xffffffffu, rt.nb > BUF - CHECK)) rt.flush();
  }
}

// Distance from the fused epilogue: ||q||^2 + ||c||^2 - 2<q,c>, negative
// round-off clamped to 0 (FAISS exhaustive_L2sqr_blas); NaN maps to 0 too.
__device__ __forceinline__ float l2_from_dot(float qn_plus_cn, float dot) {
  const float d = fmaf(-2.0f, dot, qn_plus_cn);
  return d > 0.0f ? d : 0.0f;
}

}  // namespace rs
