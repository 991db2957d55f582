// Streaming per-row top-k used by the fused score+select epilogues.
//
// One thread owns one query row.  Scores arrive in ascending chunk-id order.
// A candidate passes a register threshold test (d <= tau, tau = current k-th
// best distance) and is appended to a small per-row buffer in shared memory
// (predicated stores through a running write pointer — no divergence on the
// reject path).  When any lane of the warp nears a full buffer the whole warp
// flushes in lockstep: each lane pushes its buffered keys into its own bounded
// max-heap (root = current k-th best), then refreshes tau.  Keys are packed
// u64 (fp32 distance bits << 32 | uint32 chunk id) so the heap order is
// exactly (distance asc, id asc) — the north star's lower-index tie rule.
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
  float qn = 0.0f;      // this row's |q|^2 (epilogues that compute distances here)
  uint32_t wp = 0;      // shared-window byte address of the next buffer slot (append_raw)

  __device__ __forceinline__ uint32_t buf_base() const {
    return static_cast<uint32_t>(__cvta_generic_to_shared(buf + row));
  }

  __device__ __forceinline__ void reset() {
    nk = 0;
    nb = 0;
    tau = __int_as_float(0x7f800000);  // +inf
    wp = buf_base();
  }

  __device__ __forceinline__ uint64_t& H(int i) { return heap[i * ROWS + row]; }

  // Predicated append of one clamped candidate.
  __device__ __forceinline__ void offer(float d, uint32_t id) {
    if (d <= tau) append(d, id);
  }
  __device__ __forceinline__ void append(float d, uint32_t id) {
    buf[nb * ROWS + row] = make_key(d, id);
    ++nb;
  }
  // Append an unclamped distance through the write pointer (2 instructions
  // when predicated); negative round-off is clamped to 0 at flush time.
  __device__ __forceinline__ void append_raw(float e, uint32_t id) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(wp), "r"(id), "r"(__float_as_uint(e)) : "memory");
    wp += ROWS * 8;
  }
  __device__ __forceinline__ int buffered() const { return nb + int((wp - buf_base()) / (ROWS * 8)); }

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

#ifdef RS_TOPK_PROFILE
  unsigned long long flush_cycles = 0, flushes = 0;
  __device__ void flush() {
    const long long t0 = clock64();
    flush_impl();
    flush_cycles += clock64() - t0;
    ++flushes;
  }
  __device__ void flush_impl() {
#else
  __device__ void flush() {
#endif
    const int n = buffered();
    for (int j = 0; j < n; ++j) {
      uint64_t key = buf[j * ROWS + row];
      if (!(key_dist(key) > 0.0f)) key &= 0xffffffffull;  // clamp negative / -0 distances to +0
      push(key);
    }
    nb = 0;
    wp = buf_base();
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
// heap maintenance only run when some lane of the warp has a candidate.
// Exact: the filter uses the same rounded distance that is stored.
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

// ---------------------------------------------------------------------------
// Register-resident streaming top-k (the CTA-pair kernel's epilogue state).
//
// Profiling the smem heap showed each epilogue warp spending ~30% of the
// kernel in flushes: a heap sift is a chain of dependent shared-memory loads
// (~500 cycles per push) and one warp per scheduler cannot hide it.  Here the
// current best KREG (distance, id) pairs live in registers as a sorted list;
// inserting a candidate is a fully unrolled, branch-free compare/select sweep
// (each slot depends only on the old values of itself and its predecessor, so
// all KREG updates issue back to back).  Candidates still go through the smem
// append buffer (cheap predicated stores) and are inserted in batches.
//
// Order: the list is sorted by a u32 key = (distance bits << 1) | phase
// (distances are non-negative floats, so their bit patterns are ordered and
// 31 bits wide), inserted with a strict "<".  Within one phase candidates
// arrive with increasing chunk ids, so a strict "<" puts a new element after
// equal distances of its own phase — the (distance asc, id asc) tie rule
// without comparing ids.  A caller that streams a row range out of id order
// (the pair kernel joins a corpus segment at its frontier tile and wraps
// around) switches to phase 0 at the wrap: every later id is lower than every
// id seen before it, and phase 0 sorts before phase 1 at equal distance, so
// the rule stays exact at the same cost.
#ifndef RS_TOPK_COUNTERS  // event counters in the profiling build (-DRS_PAIR_PROFILE=1)
#if defined(RS_PAIR_PROFILE)
#define RS_TOPK_COUNTERS RS_PAIR_PROFILE
#else
#define RS_TOPK_COUNTERS 0
#endif
#endif
#ifndef RS_TOPK_COOP
#define RS_TOPK_COOP 6  // buffered candidates from which a lane may be merged cooperatively (0 = never)
#endif
#ifndef RS_TOPK_COOP_RANK
#define RS_TOPK_COOP_RANK 1  // cooperative merge by slot ranks (1) or by a bitonic sort of all elements (0)
#endif
#ifndef RS_TOPK_CHECK_GROUPS
#define RS_TOPK_CHECK_GROUPS 2  // 8-column groups per buffer check in epi_chunk32b (1 or 2)
#endif
#ifndef RS_TOPK_COOP_GAIN
#define RS_TOPK_COOP_GAIN 5  // ...and that lane holds at least this many more than every other lane
#endif
// Warp-cooperative sort behind RegTopK::flush for a burst lane (a document
// of consecutive chunks puts up to 32 candidates of one query in one
// 32-column chunk, and the lockstep insert would cost the warp one KREG-wide
// sweep per candidate).  The scratch holds the lane's KREG sorted list
// entries (key, id); every lane takes two of 64 elements (four of 128 when
// KREG + BUF > 64) — list entries,
// then the lane's admitted buffer entries (sbuf: its slot 0), then kEmpty —
// packed u64 (key << 32 | id); a 21-stage (28) bitonic sort over the warp orders
// them and the first KREG go back to the scratch.  u64 order on (key, id) is
// exactly the sequential insert's order: within a phase equal keys arrive
// with ascending ids, and the phase bit in the key orders the two phases.
// Not inlined: ~1k instructions that only bursts execute stay out of the
// epilogue's ~10 inlined flush sites.  (A per-candidate cooperative variant
// — ballot rank + shuffle shift — was slower.)
template <int KREG, int ROWS, int BUF>
__device__ __noinline__ void coop_sort64(uint32_t scr, uint32_t sbuf, int ns, uint32_t kt, uint32_t ph) {
  constexpr int E = KREG + BUF <= 64 ? 2 : 4;  // elements per lane: 64 or 128 in all
  static_assert(KREG % 2 == 0 && KREG + BUF <= 32 * E, "cooperative merge capacity");
  constexpr uint32_t kEmptyKey = 0xff000001u;
  const int lane = int(threadIdx.x & 31);
  unsigned long long v[E];
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int e = E * lane + s;
    uint32_t a = kEmptyKey, b = 0xffffffffu;
    if (e < KREG) {
      asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(scr + e * 8));
    } else if (e - KREG < ns) {
      uint32_t cid, dbits;
      asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(cid), "=r"(dbits) : "r"(sbuf + (e - KREG) * ROWS * 8));
      // clamp negative round-off (and -0, NaN) to +0, as the lockstep flush
      const uint32_t xk = ((__uint_as_float(dbits) > 0.0f ? dbits : 0u) << 1) | ph;
      if (xk < kt) {
        a = xk;
        b = cid;
      }
    }
    v[s] = (static_cast<unsigned long long>(a) << 32) | b;
  }
  // bitonic sort of the 32*E elements (element e = E*lane + s), ascending
#pragma unroll
  for (int size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride < E) {  // partner in the same lane
#pragma unroll
        for (int s = 0; s < E; ++s) {
          if (s & stride) continue;
          const int e = E * lane + s;
          const bool asc = (e & size) == 0;
          const unsigned long long x = v[s], y = v[s + stride];
          const bool sw = asc ? y < x : x < y;
          v[s] = sw ? y : x;
          v[s + stride] = sw ? x : y;
        }
      } else {
#pragma unroll
        for (int s = 0; s < E; ++s) {
          const int e = E * lane + s;
          const unsigned long long o = __shfl_xor_sync(0xffffffffu, v[s], stride / E);
          const bool keep_min = ((e & stride) == 0) == ((e & size) == 0);
          v[s] = keep_min ? (o < v[s] ? o : v[s]) : (o < v[s] ? v[s] : o);
        }
      }
    }
  }
  __syncwarp();  // every lane read the scratch before it is rewritten
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int e = E * lane + s;
    if (e < KREG)
      asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(scr + e * 8), "r"(uint32_t(v[s] >> 32)),
                   "r"(uint32_t(v[s]))
                   : "memory");
  }
  __syncwarp();
}

// Rank merge (the default cooperative merge, RS_TOPK_COOP_RANK = 1): the
// list is already sorted, so instead of sorting all KREG + n elements each
// element's output slot is computed directly.  Lane t < n holds buffer entry
// t (admitted or kEmpty), lanes hold list entries t and t + 32; a list entry
// lands at its index plus the buffer keys below it, a buffer entry at the
// buffer keys below it (ties by index) plus the list keys at or below it.
// Two loops of shared-memory broadcasts (n + KREG compares per lane) instead
// of a 21-stage shuffle network.  Keys are unique except kEmpty padding, and
// the tie rules make the slots a permutation.
template <int KREG, int ROWS, int BUF>
__device__ __noinline__ void coop_rank_merge(uint32_t scr, uint32_t sbuf, int ns, uint32_t kt, uint32_t ph) {
  static_assert(KREG <= 64 && BUF <= 32, "rank merge: two list entries and one buffer entry per lane");
  constexpr unsigned long long kE = (static_cast<unsigned long long>(0xff000001u) << 32) | 0xffffffffu;
  const int lane = int(threadIdx.x & 31);
  const uint32_t bscr = scr + KREG * 8;  // BUF packed buffer keys after the list
  auto ld_entry = [](uint32_t addr) -> unsigned long long {
    uint32_t a, b;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(addr));
    return (static_cast<unsigned long long>(a) << 32) | b;
  };
  unsigned long long bv = kE;
  if (lane < ns) {
    uint32_t cid, dbits;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(cid), "=r"(dbits) : "r"(sbuf + lane * ROWS * 8));
    // clamp negative round-off (and -0, NaN) to +0, as the lockstep flush
    const uint32_t xk = ((__uint_as_float(dbits) > 0.0f ? dbits : 0u) << 1) | ph;
    if (xk < kt) bv = (static_cast<unsigned long long>(xk) << 32) | cid;
  }
  if (lane < ns)
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(bscr + lane * 8), "r"(uint32_t(bv >> 32)), "r"(uint32_t(bv))
                 : "memory");
  const unsigned long long l0 = lane < KREG ? ld_entry(scr + lane * 8) : kE;
  const unsigned long long l1 = lane + 32 < KREG ? ld_entry(scr + (lane + 32) * 8) : kE;
  __syncwarp();
  int pb = 0, p0 = lane, p1 = lane + 32;
#pragma unroll 4
  for (int i = 0; i < ns; ++i) {
    const unsigned long long b = ld_entry(bscr + i * 8);
    pb += (b < bv || (b == bv && i < lane)) ? 1 : 0;
    p0 += b < l0 ? 1 : 0;
    p1 += b < l1 ? 1 : 0;
  }
#pragma unroll 8
  for (int j = 0; j < KREG; ++j) pb += ld_entry(scr + j * 8) <= bv ? 1 : 0;
  __syncwarp();  // every lane read the list before it is rewritten
  auto st_entry = [](uint32_t addr, unsigned long long v) {
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(uint32_t(v >> 32)), "r"(uint32_t(v)) : "memory");
  };
  if (lane < ns && pb < KREG) st_entry(scr + pb * 8, bv);
  if (lane < KREG && p0 < KREG) st_entry(scr + p0 * 8, l0);
  if (lane + 32 < KREG && p1 < KREG) st_entry(scr + p1 * 8, l1);
  __syncwarp();
}

// COOP = false: the same list without the cooperative merge code (the lean
// kernel variant; its flushes still count bursts, see flush()).
template <int KREG, int ROWS, int BUF, bool COOP = true>
struct RegTopK {
  uint32_t key[KREG];  // (distance bits << 1) | phase
  uint32_t id[KREG];
  int k;          // <= KREG
  float tau;      // distance of the current k-th best, +inf until k candidates seen
  uint32_t ktau;  // admission key: min(key of the current k-th best, seedk)
  uint32_t seedk; // shared-threshold seed (see seed()), kEmpty when none
  uint32_t kthk;  // key of the current k-th best (kEmpty until k entries)
  uint32_t phase; // 1 until the walk wraps to lower ids, then 0
  uint32_t bursts = 0;  // flushes that found a burst lane (warp-uniform; the host's variant choice)
  float qn;       // this row's |q|^2
  uint32_t wbase; // shared-window byte address of this row's buffer slot 0
  uint32_t wp;    // next free buffer slot
#if RS_TOPK_COUNTERS
  // event counts (tuning builds): slow-path groups, appends, flushes, inserts
  uint32_t c_groups = 0, c_appends = 0, c_flushes = 0, c_inserts = 0, c_coop = 0;
#define RS_TOPK_COUNT(field, n) (field) += (n)
#else
#define RS_TOPK_COUNT(field, n) ((void)0)
#endif

  static constexpr uint32_t kEmpty = 0xff000001u;  // +inf, phase 1

  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int j = 0; j < KREG; ++j) {
      key[j] = kEmpty;
      id[j] = 0xffffffffu;
    }
    tau = __int_as_float(0x7f800000);
    ktau = kEmpty;
    seedk = kEmpty;
    kthk = kEmpty;
    phase = 1;
    wp = wbase;
  }

  __device__ __forceinline__ void append_raw(float e, uint32_t cid) {
    RS_TOPK_COUNT(c_appends, 1);
    asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(wp), "r"(cid), "r"(__float_as_uint(e)) : "memory");
    wp += ROWS * 8;
  }
  __device__ __forceinline__ int buffered() const { return int((wp - wbase) / (ROWS * 8)); }

  __device__ __forceinline__ void insert(uint32_t xk, uint32_t xid) {
#pragma unroll
    for (int j = KREG - 1; j >= 1; --j) {
      const bool lt_prev = xk < key[j - 1];
      const bool lt_cur = xk < key[j];
      id[j] = lt_prev ? id[j - 1] : (lt_cur ? xid : id[j]);
      key[j] = lt_prev ? key[j - 1] : (lt_cur ? xk : key[j]);
    }
    const bool lt0 = xk < key[0];
    id[0] = lt0 ? xid : id[0];
    key[0] = lt0 ? xk : key[0];
  }

  __device__ __forceinline__ void refresh_tau() {
    uint32_t t = key[0];
#pragma unroll
    for (int j = 1; j < KREG; ++j)
      if (j == k - 1) t = key[j];
    kthk = t;
    ktau = t < seedk ? t : seedk;
    tau = __uint_as_float(ktau >> 1);
  }

  // Shared threshold: dist_bits is the k-th best distance of SOME k real rows
  // of this query (another unit's list), hence >= the final k-th distance;
  // only candidates at or below it can reach the final top-k.  The seed key
  // (bits + 1) << 1 admits every candidate with distance <= that value, in
  // either phase (exact ties are kept; the merge orders them by id), so the
  // unit's list may end with fewer than k real entries — it never loses one
  // the global top-k needs.
  __device__ __forceinline__ void seed(uint32_t dist_bits) {
    if (dist_bits >= 0x7f800000u) return;  // +inf / no bound yet
    const uint32_t s = (dist_bits + 1u) << 1;
    if (s < seedk) {
      seedk = s;
      if (s < ktau) {
        ktau = s;
        tau = __uint_as_float(s >> 1);
      }
    }
  }
  // distance bits of the current k-th best (0x7f800000 = +inf until k entries)
  __device__ __forceinline__ uint32_t kth_bits() const { return kthk >> 1; }
  // distance bits of the r-th best (1-based, r <= k; +inf when fewer entries)
  __device__ __forceinline__ uint32_t rank_bits(int r) const {
    uint32_t t = key[0];
#pragma unroll
    for (int j = 1; j < KREG; ++j)
      if (j == r - 1) t = key[j];
    return t >> 1;
  }

  // Cooperative merge of ONE lane's list with its buffered candidates, by the
  // whole warp (coop_rank_merge above; coop_sort64 with RS_TOPK_COOP_RANK=0):
  // lane src publishes its KREG sorted entries to the warp's scratch, the
  // warp merges them with src's admitted buffer entries, src reloads the
  // first KREG.
  uint32_t sbase;  // shared-window byte address of this warp's (KREG + BUF) x 8-byte scratch
  __device__ __forceinline__ void coop_merge(int src, int ns, uint32_t kt) {
    const int lane = int(threadIdx.x & 31);
    if (lane == src) {
#pragma unroll
      for (int j = 0; j < KREG; j += 2)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sbase + j * 8), "r"(key[j]), "r"(id[j]),
                     "r"(key[j + 1]), "r"(id[j + 1])
                     : "memory");
    }
    __syncwarp();
#if RS_TOPK_COOP_RANK
    coop_rank_merge<KREG, ROWS, BUF>(sbase, wbase + uint32_t(src - lane) * 8u, ns, kt, phase);
#else
    coop_sort64<KREG, ROWS, BUF>(sbase, wbase + uint32_t(src - lane) * 8u, ns, kt, phase);
#endif
    if (lane == src) {
#pragma unroll
      for (int j = 0; j < KREG; j += 2)
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(key[j]), "=r"(id[j]), "=r"(key[j + 1]), "=r"(id[j + 1])
                     : "r"(sbase + j * 8));
    }
    __syncwarp();  // src read the scratch before the next merge rewrites it
  }

  // Warp-collective: every lane inserts its buffered candidates (lockstep over
  // the warp's largest buffer; lanes past their own count insert kEmpty = no-op).
  // Lockstep costs the warp one KREG-wide sweep per candidate of its FULLEST
  // lane, so a lane that holds RS_TOPK_COOP_GAIN or more candidates beyond
  // every other lane (a burst) is merged cooperatively first, fullest first.
  // SITE = false: a flush site that never merges cooperatively (nor counts).
  template <bool SITE = true>
  __device__ __forceinline__ void flush() {
    int n = buffered();
#if RS_TOPK_COOP
    if (SITE) {
      const int lane = int(threadIdx.x & 31);
      bool first = true;
#pragma unroll 1
      for (;;) {
        const int top = __reduce_max_sync(0xffffffffu, n);
        if (top < RS_TOPK_COOP) break;
        const int src = __ffs(__ballot_sync(0xffffffffu, n == top)) - 1;
        const int second = __reduce_max_sync(0xffffffffu, lane == src ? 0 : n);
        if (top - second < RS_TOPK_COOP_GAIN) break;
        if (first) ++bursts;
        first = false;
        if constexpr (!COOP) break;
        RS_TOPK_COUNT(c_coop, 1);
        coop_merge(src, top, __shfl_sync(0xffffffffu, ktau, src));
        if (lane == src) n = 0;
      }
    }
#endif
    const int nmax = __reduce_max_sync(0xffffffffu, n);
    RS_TOPK_COUNT(c_flushes, 1);
#ifdef RS_EXP_NO_INSERT  // timing experiment only (wrong results): candidates are dropped
    if (nmax < 0)
#endif
    for (int j = 0; j < nmax; ++j) {
      uint32_t lo = 0, hi = 0;
      if (j < n) asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(wbase + j * ROWS * 8));
      // clamp negative round-off (and -0, NaN) to +0: bit pattern 0
      const uint32_t xk = j < n ? ((__uint_as_float(hi) > 0.0f ? hi : 0u) << 1) | phase : kEmpty;
      if (__any_sync(0xffffffffu, xk < ktau)) {
        RS_TOPK_COUNT(c_inserts, 1);
        insert(xk < ktau ? xk : kEmpty, lo);
      }
    }
    wp = wbase;
    refresh_tau();
  }

  // Write the k best keys (call the warp-collective flush() first, with the
  // whole warp converged; this part is per lane).
  __device__ __forceinline__ void finish(uint64_t* __restrict__ out) const {
#pragma unroll
    for (int j = 0; j < KREG; ++j)
      if (j < k) out[j] = (key[j] >> 1) >= 0x7f800000u ? ~0ull : (uint64_t(key[j] >> 1) << 32) | id[j];
  }
};

// Exact distances and predicated appends of 8 columns for RegTopK (the slow
// path of epi_chunk32b).
template <int KREG, int ROWS, int BUF, int CHECK, bool FULL, bool CHK = true, bool COOP = true>
__device__ __forceinline__ void epi_group8r(RegTopK<KREG, ROWS, BUF, COOP>& rt, const uint32_t* r, const float* cn,
                                            uint32_t id, int lim) {
  static_assert(BUF >= CHECK, "buffer must hold the groups between two checks");
  RS_TOPK_COUNT(rt.c_groups, 1);
  const float4 a = *reinterpret_cast<const float4*>(cn);
  const float4 b = *reinterpret_cast<const float4*>(cn + 4);
  const float2 q2 = make_float2(rt.qn, rt.qn);
  const float2 m2 = make_float2(-2.0f, -2.0f);
  const float2 e0 = __ffma2_rn(make_float2(__uint_as_float(r[0]), __uint_as_float(r[1])), m2,
                               __fadd2_rn(q2, make_float2(a.x, a.y)));
  const float2 e1 = __ffma2_rn(make_float2(__uint_as_float(r[2]), __uint_as_float(r[3])), m2,
                               __fadd2_rn(q2, make_float2(a.z, a.w)));
  const float2 e2 = __ffma2_rn(make_float2(__uint_as_float(r[4]), __uint_as_float(r[5])), m2,
                               __fadd2_rn(q2, make_float2(b.x, b.y)));
  const float2 e3 = __ffma2_rn(make_float2(__uint_as_float(r[6]), __uint_as_float(r[7])), m2,
                               __fadd2_rn(q2, make_float2(b.z, b.w)));
  const float e[8] = {e0.x, e0.y, e1.x, e1.y, e2.x, e2.y, e3.x, e3.y};
#pragma unroll
  for (int j = 0; j < 8; ++j)
    if ((FULL || j < lim) && e[j] <= rt.tau) rt.append_raw(e[j], id + j);
  if (CHK && __any_sync(0xffffffffu, rt.buffered() > BUF - CHECK)) rt.flush();
}

// Bound-filtered epilogue (epi_chunk32b below).  For the columns of a 32-column chunk,
//   e_j = |q|^2 + |c_j|^2 - 2<q,c_j>  >=  |q|^2 + min_chunk|c|^2 - 2<q,c_j>,
// so e_j <= tau needs <q,c_j> >= thr = (|q|^2 + min|c|^2 - tau) / 2 (minus a
// rounding margin, chunk_threshold).  The fast path is therefore the raw TMEM
// dots alone — an 8-way max, one compare, one warp vote — and only groups
// where some lane of the warp passes compute the exact distances (the same
// FADD2/FFMA2 rounding as epi_group8r) and append.  With normalised corpora
// the bound is tight; otherwise it is looser but never drops a candidate.
// A whole 32-column TMEM chunk through the dot bound: four independent 8-way
// max trees, four votes, and a single branch in the common case that no lane
// of the warp has a candidate anywhere in the chunk (a one-warp-per-SMSP
// epilogue is latency-bound, so the short dependency chains and the single
// branch matter more than the instruction count).
template <int KREG, int ROWS, int BUF, int CHECK, bool FULL, bool COOP>
__device__ __forceinline__ void epi_chunk32b(RegTopK<KREG, ROWS, BUF, COOP>& rt, const uint32_t* r, const float* cn,
                                             uint32_t id, int lim, float thr) {
  float m[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      v[j] = (FULL || g * 8 + j < lim) ? __uint_as_float(r[g * 8 + j]) : -__int_as_float(0x7f800000);
    m[g] = fmaxf(fmaxf(fmaxf(v[0], v[1]), fmaxf(v[2], v[3])), fmaxf(fmaxf(v[4], v[5]), fmaxf(v[6], v[7])));
  }
  uint32_t hit = 0;
#pragma unroll
  for (int g = 0; g < 4; ++g) hit |= __any_sync(0xffffffffu, m[g] >= thr) ? (1u << g) : 0u;
  if (hit == 0) return;
#if RS_TOPK_CHECK_GROUPS == 1
#pragma unroll
  for (int g = 0; g < 4; ++g)
    if (hit & (1u << g)) {
      if (FULL)
        epi_group8r<KREG, ROWS, BUF, CHECK, true, true, COOP>(rt, r + g * 8, cn + g * 8, id + g * 8, 8);
      else
        epi_group8r<KREG, ROWS, BUF, CHECK, false, true, COOP>(rt, r + g * 8, cn + g * 8, id + g * 8, lim - g * 8);
    }
#else
  // one buffer check per two groups (half the inlined flush sites; CHECK
  // then covers 16 columns)
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (hit & (1u << g)) {
      if (FULL)
        epi_group8r<KREG, ROWS, BUF, CHECK, true, false, COOP>(rt, r + g * 8, cn + g * 8, id + g * 8, 8);
      else
        epi_group8r<KREG, ROWS, BUF, CHECK, false, false, COOP>(rt, r + g * 8, cn + g * 8, id + g * 8, lim - g * 8);
    }
    if ((g & 1) && (hit & (3u << (g - 1))) && __any_sync(0xffffffffu, rt.buffered() > BUF - CHECK)) rt.flush();
  }
#endif
}

// Dot threshold of a chunk whose smallest corpus norm is cmin (see
// epi_chunk32b); +inf tau (list not full) gives -inf: everything passes.  The
// margin covers the fp32 rounding of both this bound and the exact distance.
__device__ __forceinline__ float chunk_threshold(float qn, float cmin, float tau) {
  const float t = 0.5f * (qn + cmin - tau);
  return t - 1e-6f * (fabsf(qn) + fabsf(cmin) + fabsf(tau)) - 1e-30f;
}

// Distance from the fused epilogue: ||q||^2 + ||c||^2 - 2<q,c>, negative
// round-off clamped to 0 (FAISS exhaustive_L2sqr_blas); NaN maps to 0 too.
__device__ __forceinline__ float l2_from_dot(float qn_plus_cn, float dot) {
  const float d = fmaf(-2.0f, dot, qn_plus_cn);
  return d > 0.0f ? d : 0.0f;
}

}  // namespace rs
