// K1 score_topk, CTA-pair variant (sm_100a, cta_group::2) — the default bf16
// retrieval kernel.
//
// Same fused exact-L2 + streaming top-k as score_topk_sm100.cu, but two CTAs
// on the two SMs of a TPC cooperate on a 256-query x 256-chunk tile with one
// tcgen05.mma.cta_group::2 (M=256, N=256, K=16):
//   * CTA r stages query rows [256*qt + 128*r, +128) (A half) and corpus rows
//     [c0 + 128*r, +128) (B half) per k-block — each SM pulls 32 KB per
//     512-cycle k-block (64 B/clk) instead of the 48 KB (96 B/clk) of the
//     single-CTA tile, and the freed shared memory buys a deeper TMA ring;
//   * the leader CTA (rank 0) issues the MMAs; its TMEM receives query rows
//     0-127 of the tile and the peer's TMEM rows 128-255, all 256 chunk
//     columns each, so every CTA's epilogue owns 128 queries x 256 chunks;
//   * the epilogue keeps each query's running top-k in REGISTERS (RegTopK,
//     topk_rows.cuh): a branch-free 3-instruction-per-score filter appends
//     candidates to a small smem buffer, flushed in warp-wide batches into a
//     sorted register list (no shared-memory heap latency chains);
//   * units (query tile, corpus segment) are handed out DYNAMICALLY in
//     segment-major order (one atomic per unit, published to both CTAs of
//     the pair through a 4-deep smem ring): the units in flight are always
//     consecutive, so the CTAs streaming a segment for different query tiles
//     stay together and the segment is read from HBM about once (a static
//     round-robin let pairs drift apart: ncu showed the 20 GB corpus read
//     17x from DRAM).
//
// Synchronisation (all mbarriers):
//   full[s]   leader only; the leader's producer arms 2 x 32 KB, both CTAs'
//             TMA loads complete on it (.cta_group::2 TMA, mapa address)
//   empty[s]  both CTAs; leader MMA commit multicasts to both
//   tfull[a]  both CTAs; 2 arrivals: the local norm bulk-copy (expect_tx) and
//             the leader's MMA commit (multicast)
//   tempty[a] leader: 8 warp arrivals (4 local + 4 remote from the peer);
//             peer: its 4 local warps (gates its own norm copy)
//   ufull[i]  both CTAs: unit id published (leader producer; remote for peer)
//   uempty[i] leader: 11 consumers read the slot (5 local + 6 remote)
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "retrieval.cuh"
#include "sm100_ptx.cuh"
#include "topk_rows.cuh"

namespace rs {
namespace {

using namespace sm100;

#ifndef RS_PAIR_STAGES
#define RS_PAIR_STAGES 6
#endif
#ifndef RS_TOPK_COOP_ALL_SITES
#define RS_TOPK_COOP_ALL_SITES 1  // 0: the walk-wrap and unit-end flushes stay lockstep-only
#endif
#ifndef RS_PAIR_BUF
// candidate buffer slots per row: one check per RS_TOPK_CHECK_GROUPS 8-column
// groups flushes above 8 buffered, so a check interval of 16 columns needs 24
// (swept 8..48 with one check per group and 5/6 stages: 6 x 16 was best then)
#define RS_PAIR_BUF (8 + 8 * RS_TOPK_CHECK_GROUPS)
#endif

constexpr int BM = 128;         // query rows per CTA (TMEM lanes)
constexpr int BN = kTcBN;       // corpus columns per tile (both CTAs)
constexpr int HB = BN / 2;      // corpus rows staged per CTA
#ifndef RS_PAIR_STAGES_TF32
#define RS_PAIR_STAGES_TF32 3
#endif
// Drift limiter (RS_PAIR_SYNC_TILES, retrieval.cuh; the plan enables it):
// a unit's producer does not start a tile more than sync_tiles tiles past the
// slowest running unit of its segment (bounded wait), so the segment's rows
// are read from DRAM once instead of once per drifting pair.
constexpr int32_t kSyncIdle = 0x7f7f7f7f;  // prog[] of a unit not running (memset 0x7f)
constexpr uint64_t kSyncMaxWaitNs = 20000;  // per tile: a stalled partner never stalls a unit for long
// corpus tiles prefetched into L2 ahead of the TMA loads (0 = off)
#ifndef RS_PAIR_PREFETCH
#define RS_PAIR_PREFETCH 0
#endif
constexpr int KREG = kTcMaxK;   // register top-k capacity, bf16 (k <= 40)
// tf32 path: the candidate pass keeps k + kRefineExtra rows for the exact
// re-rank, so its lists hold up to kTcMaxK + kRefineExtra (every k <= 40 keeps
// its 8 spare candidates)
constexpr int KREG_TF32 = kTcMaxK + kRefineExtra;
// candidate buffer per row; a warp flushes when one of its lanes holds more
// than BUF - CHECK entries, so every flush batches many candidates per lane
constexpr int BUF = RS_PAIR_BUF;
constexpr int CHECK = 8 * RS_TOPK_CHECK_GROUPS;  // candidates one check interval can add per row
constexpr int EPI_COLS = 32;    // TMEM columns per tcgen05.ld
#ifndef RS_PAIR_EPI_PAIRED
#define RS_PAIR_EPI_PAIRED 0       // 1: two loads per tcgen05.wait::ld
#endif
constexpr int ROW_BYTES = 128;  // one SWIZZLE_128B row of a k-block (64 bf16 / 32 fp32)
constexpr int B_BYTES = HB * ROW_BYTES;
constexpr int TMEM_COLS = 2 * BN;
constexpr int EG = kPairEpiGroups;       // epilogue warp groups (column slices)
constexpr int CPG = BN / EG;             // tile columns per epilogue group
constexpr int EPI_THREADS = 128 * EG;
constexpr int NUM_THREADS = 128 + EPI_THREADS;
// Warp roles.  The SM's warp arbiter favours HIGHER warp ids, so the latency-
// critical single-thread roles (TMA producer, MMA issuer) take the top ids and
// the epilogue warps the bottom ones (epilogue warp w reads TMEM lane quadrant
// w % 4, so it must start at a multiple of 4).
#ifndef RS_PAIR_ROLES_HIGH
#define RS_PAIR_ROLES_HIGH 1
#endif
#if RS_PAIR_ROLES_HIGH
constexpr int EPI_WARP0 = 0;
constexpr int WARP_TMEM = 4 * EG + 1;
constexpr int WARP_PROD = 4 * EG + 2;
constexpr int WARP_MMA = 4 * EG + 3;
constexpr int WARP_CVT = 4 * EG;  // tf32 path: the corpus residual converter
#else
constexpr int WARP_CVT = 3;
constexpr int EPI_WARP0 = 4;
constexpr int WARP_PROD = 0;
constexpr int WARP_MMA = 1;
constexpr int WARP_TMEM = 2;
#endif
static_assert(CPG % 32 == 0, "column slice must be whole TMEM loads");
constexpr int G = kPairGroup;   // pairs per cluster sharing each corpus tile (TMA multicast)
constexpr int CL = 2 * G;       // cluster size (CTAs)
constexpr int BPIECE = HB / G;  // corpus rows each CTA loads and multicasts per k-block
constexpr int URING = 4;        // unit-id ring depth
// readers of a unit-ring slot: every CTA's norm/MMA thread + 4 epilogue warps,
// and every producer except the scheduling one (cluster rank 0)
constexpr uint32_t UCONSUMERS = (2 + 4 * EG) * CL - 1;
static_assert(HB % G == 0 && BPIECE % 8 == 0, "corpus piece must be whole swizzle atoms");

template <int S>
struct __align__(8) SmemTailT {
  uint64_t full[S];
  uint64_t braw[S];  // tf32 path: this CTA's raw corpus tile landed (local TMA)
  uint64_t empty[S];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint64_t ufull[URING];
  uint64_t uempty[URING];
  int32_t uid[URING];
  int32_t ustart[URING];  // absolute frontier tile the unit starts at
  uint32_t tmem_base;
  int32_t cvt_stop;  // tf32 path: stages the producer issued (set when it is done)
};

// Operand precision.  bf16: one kind::f16 MMA per 16-element k-step.  fp32
// (TF = true, "3xTF32"): each operand x is fed as hi = x (the tensor core
// reads the top 19 bits, i.e. tf32 truncation) and lo = x - trunc_tf32(x)
// (exact in fp32, precomputed: the corpus at add(), the queries per search),
// and every 8-element k-step issues lo*hi + hi*lo + hi*hi into the same fp32
// TMEM accumulator.  The accumulator's truncating adds leave ~1e-5 relative
// error on large dots at d = 768, so the fp32 search keeps k + 8 candidates
// and re-ranks them exactly (refine_score_kernel + refine_rank_kernel, retrieval.cu).
//
// Pair tile height.  SM = false: M = 256 (128 query rows per CTA), the
// accumulator of a tile fills 256 TMEM columns of all 128 lanes.  SM = true
// (small batches, nq <= 128): M = 128 (64 rows per CTA), so a lone query
// tile wastes no MMA work on padding rows; tcgen05's 2-CTA M = 128 data path
// puts rows 0-31 / 32-63 in lane quadrants 0 / 1 for tile columns 0-127 and
// again in quadrants 2 / 3 for columns 128-255, 128 TMEM columns per tile.
// Each epilogue warp then owns half the columns of 32 rows, so a row keeps
// two top-k lists per unit (merged downstream like the segments).
//
// With RS_TF32_STORED_LO = 0 (a measured-slower option; the default streams
// precomputed residuals) the corpus residual is formed in shared memory: each CTA's raw fp32 corpus tile arrives by a local TMA on
// braw[s]; the converter warp writes lo = x - trunc_tf32(x) next to it,
// issues fence.proxy.async (generic-proxy stores -> the tensor core's async
// proxy) and arrives on the leader's full[s], which therefore counts the
// producer's expect_tx arrival plus both CTAs' converter arrivals.  The
// corpus is then streamed at 4 bytes per element and stored once.
template <bool TF, bool SM = false>
struct Cfg {
  static constexpr int BK = TF ? 32 : 64;  // elements per k-block (one 128-byte row)
  static constexpr int NT = TF ? 2 : 1;    // tiles per operand per stage (hi, lo)
  static constexpr int BMv = SM ? 64 : BM;  // query rows per CTA
  static constexpr int PMv = 2 * BMv;      // query rows per pair tile (the MMA's M)
  static constexpr int A_BYTESv = BMv * ROW_BYTES;
  static constexpr int ACC_COLS = SM ? BN / 2 : BN;  // TMEM columns per accumulator buffer
  static constexpr int LPS = SM ? 2 : EG;            // top-k lists per (query, segment)
  static constexpr int STAGES = TF ? RS_PAIR_STAGES_TF32 : RS_PAIR_STAGES;
  static constexpr int STAGE_BYTES = NT * (A_BYTESv + B_BYTES);
  static constexpr int OFF_B = NT * A_BYTESv;  // stage layout: A hi | [A lo] | B hi | [B lo]
  static constexpr uint32_t IDESC = TF ? umma_idesc_tf32_f32(PMv, BN) : umma_idesc_bf16_f32(PMv, BN);
  using Tail = SmemTailT<STAGES>;
  static constexpr int KR = TF ? KREG_TF32 : KREG;  // register top-k capacity
  static constexpr size_t OFF_BUF = size_t(STAGES) * STAGE_BYTES;
  static constexpr size_t OFF_CN = OFF_BUF + size_t(BUF) * EPI_THREADS * 8;
  static constexpr size_t OFF_SCR = OFF_CN + 2 * BN * sizeof(float);  // per epilogue warp: (KR + BUF) x 8 B (coop_merge)
  static constexpr size_t OFF_TAIL = OFF_SCR + size_t(EPI_THREADS / 32) * (KR + BUF) * 8;
  static constexpr size_t SMEM_BYTES = OFF_TAIL + sizeof(Tail);
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
};

struct Params {
  const float* qn;
  const float* cn;
  const float* cmin;  // per 32-row chunk of the shard: min squared norm (the epilogue's dot bound)
  int64_t nq, n;
  int32_t kblocks;
  int32_t k;
  int64_t id_base;
  int32_t qtiles, segments;
  int64_t seg_rows;
  uint64_t* part;
  int32_t* counter;  // dynamic unit counter (zeroed before the launch)
  uint32_t* bursts;  // flushes that found a burst lane, summed over warps (zeroed)
  int32_t* done;     // CTAs finished (zeroed): the last one posts *bursts to bursts_host
  uint32_t* bursts_host;  // pinned host word (device-accessible under unified addressing) or null
  int32_t* seg_pos;  // per segment: absolute tile index the most advanced pair last started (zeroed)
  int32_t* prog;     // drift limiter: per unit, the absolute tile it is loading (kSyncIdle when not running)
  int32_t sync_tiles;  // drift limiter window (0 = off)
  int32_t walk_bias; // test hook: unit of query tile qt starts walk_bias*(qt+1) tiles past the frontier
  uint32_t* qtau;    // per query: best k-th distance bits published by any unit (memset 0xff per search)
  uint32_t* qcas;    // per query: the kCas smallest rank-r distances of finished lists (r = ceil(k/kCas))
  int32_t cas_rank;  // r
  int64_t cunits;    // cluster units = (qtiles / G) * segments
};

__device__ __forceinline__ void unit_coords(int64_t u, const Params& p, int& qt, int& seg, int64_t& r0,
                                            int64_t& r1) {
  seg = int(u / p.qtiles);
  qt = int(u - int64_t(seg) * p.qtiles);
  r0 = int64_t(seg) * p.seg_rows;
  r1 = r0 + p.seg_rows;
  if (r1 > p.n) r1 = p.n;
}

// Frontier join: a unit streams its segment's T tiles starting at the tile
// the most advanced pair on that segment is loading (absolute index `start`)
// and wraps around, so every pair on a segment reads the same corpus rows at
// about the same time whenever it joined — the segment's rows are fetched
// from HBM about once and served to the other query tiles from L2.  (In
// plain ascending order the dynamically scheduled pairs drift apart by
// fractions of a unit; ncu measured the 20 GB corpus read 8x from DRAM at
// 10M x 1024, and the DRAM power cost ~10% of the SM clock under the cap.)
struct TileWalk {
  int64_t r0, r1, ntiles, first;  // first = start mod ntiles
  __device__ __forceinline__ TileWalk(int64_t r0_, int64_t r1_, int32_t start) : r0(r0_), r1(r1_) {
    ntiles = (r1 - r0 + BN - 1) / BN;
    first = ntiles > 0 ? int64_t(start) % ntiles : 0;
  }
  __device__ __forceinline__ bool wrapped(int64_t j) const { return first + j >= ntiles; }
  __device__ __forceinline__ int64_t c0(int64_t j) const {
    int64_t t = first + j;
    if (t >= ntiles) t -= ntiles;
    return r0 + t * BN;
  }
};

// Shared admission bound of a query (threshold sharing across units).  Two
// valid upper bounds of the query's final k-th distance:
//  * qtau: the smallest k-th distance any list has reached (a list's k
//    entries are real rows), published every 4 tiles and at unit end;
//  * qcas[kCas-1]: each finished list inserts its rank-r distance (r =
//    ceil(k/kCas)) into a per-query cascade of kCas atomicMin slots, so
//    slot kCas-1 holds the kCas-th smallest of them — kCas disjoint lists
//    (distinct segments / column halves) with >= r rows each at or below
//    it, i.e. >= k rows.  Once a few segments of a query are done this is
//    far tighter than any single list's k-th distance, so later units admit
//    ~k/kCas candidates instead of ~k.  With RS_PAIR_CAS_MULTI a list
//    inserts its rank-r, 2r, ... distances: the value at rank j*r stands for
//    the list's rows of rank ((j-1)r, jr], disjoint from every other inserted
//    value's rows, so slot kCas-1 is still backed by kCas*r >= k rows — and
//    one list with many near rows (a document of consecutive chunks) now
//    tightens the bound by itself.
constexpr int kCas = RS_PAIR_CAS;
static_assert(1 + kCas == kSharedBoundWords, "qtau allocation (retrieval.cu)");
__device__ __forceinline__ uint32_t shared_bound(const Params& p, int64_t qrow) {
  const uint32_t a = ld_relaxed_gpu_u32(p.qtau + qrow);
  const uint32_t b = ld_relaxed_gpu_u32(p.qcas + qrow * kCas + (kCas - 1));
  return a < b ? a : b;
}
// Concurrent insertion into ascending slots by an atomicMin cascade: each
// level keeps min(v, old) and passes max(v, old) down, so (values being
// conserved per level) slot i ends as the (i+1)-th smallest inserted value,
// and at any moment slot i's value is backed by i+1 distinct inserts.
__device__ __forceinline__ void cascade_min_insert(uint32_t* slots, uint32_t v) {
#pragma unroll
  for (int i = 0; i < kCas; ++i) {
    const uint32_t old = atomicMin(slots + i, v);
    v = v > old ? v : old;
    if (v == 0xffffffffu) break;
  }
}

// Consumer side of the unit ring: wait for slot i, read the unit id, release
// the slot to the leader's producer.  Returns the unit (-1 = no more work).
template <class SmemTail>
__device__ __forceinline__ void release_unit(SmemTail* tail, uint32_t i, bool scheduler) {
  if (scheduler)
    mbar_arrive(&tail->uempty[i % URING]);
  else
    mbar_arrive_cluster(mapa_shared(smem_u32(&tail->uempty[i % URING]), 0));
}
template <class SmemTail>
__device__ __forceinline__ int next_unit(SmemTail* tail, uint32_t i, bool scheduler, bool arrive, int32_t& start) {
  const int slot = int(i % URING);
  mbar_wait_cluster(&tail->ufull[slot], (i / URING) & 1);
  const int u = *reinterpret_cast<volatile int32_t*>(&tail->uid[slot]);
  start = *reinterpret_cast<volatile int32_t*>(&tail->ustart[slot]);
  if (arrive) release_unit(tail, i, scheduler);
  return u;
}

// Optional per-role cycle accounting (tuning builds: -DRS_PAIR_PROFILE=1;
// read back with tools/pair_profile.py).
#ifndef RS_PAIR_PROFILE
#define RS_PAIR_PROFILE 0
#endif
#if RS_PAIR_PROFILE
// [cta][0..7]: role cycles (below); [cta][8..11]: epilogue event counts summed
// over the CTA's epilogue lanes (warp-collective events once per warp):
// slow-path 8-column groups, candidate appends, flushes, warp insert steps
__device__ unsigned long long g_pair_prof[1024][16];
#define PROF(slot, stmt)                       \
  do {                                         \
    const long long _t0 = clock64();           \
    stmt;                                      \
    prof[slot] += clock64() - _t0;             \
  } while (0)
#else
#define PROF(slot, stmt) stmt
#endif

template <bool TF, bool SM, bool COOP>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    score_topk_pair_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmql,
                           const __grid_constant__ CUtensorMap tmc, const __grid_constant__ CUtensorMap tmcl,
                           const Params p) {
  using C = Cfg<TF, SM>;
  using SmemTail = typename C::Tail;
  constexpr int STAGES = C::STAGES;
  // no static shared memory: the dynamic window starts at the CTA's shared
  // base, 1024-aligned as SWIZZLE_128B requires
  extern __shared__ __align__(1024) uint8_t smem[];
  SmemTail* tail = reinterpret_cast<SmemTail*>(smem + C::OFF_TAIL);
  float* cns = reinterpret_cast<float*>(smem + C::OFF_CN);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t half = rank & 1;           // CTA within its pair
  const int pp = int(rank >> 1);            // pair within the cluster
  const uint32_t pair_leader = rank & ~1u;  // issues the pair's MMAs
  const bool leader = half == 0;
  const bool scheduler = rank == 0;         // hands out cluster units
  const uint16_t mc_half = uint16_t(((1u << CL) - 1u) / 3u << half);  // CTAs {2p'+half}: 0b0101.. << half
  if ((smem_u32(smem) & 1023u) != 0) __trap();

  if (warp == WARP_PROD && lane == 0) {
    tma_prefetch_desc(&tmq);
    tma_prefetch_desc(&tmc);
    if (TF) {
      tma_prefetch_desc(&tmql);
      tma_prefetch_desc(&tmcl);
    }
  }
  if (warp == WARP_MMA && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&tail->full[s], (TF && !RS_TF32_STORED_LO) ? 3 : 1);
      mbar_init(&tail->braw[s], 1);
      mbar_init(&tail->empty[s], G);  // one MMA commit per pair of the cluster
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tail->tfull[a], 2);
      mbar_init(&tail->tempty[a], leader ? 8 * EG : 4 * EG);
    }
    for (int i = 0; i < URING; ++i) {
      mbar_init(&tail->ufull[i], 1);
      mbar_init(&tail->uempty[i], scheduler ? UCONSUMERS : 1);
    }
    tail->cvt_stop = 0x7fffffff;
    fence_barrier_init();
  }
  if (warp == WARP_TMEM) {
    tmem_alloc_pair(&tail->tmem_base, TMEM_COLS);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem_base = tail->tmem_base;
#if RS_PAIR_PROFILE
  unsigned long long prof[8] = {};
  const long long t_start = clock64();
#endif

  if (warp == WARP_PROD) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs): own A half + own B half per k-block;
      //       the leader's producer also schedules the units =====
      const uint64_t pol_q = policy_evict_last();
      const uint64_t pol_c = p.qtiles == 1 ? policy_evict_first() : policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      int32_t issued = 0;  // k-block stages issued (the tf32 converter's stop count)
      for (uint32_t i = 0;; ++i) {
        int u;
        int32_t start = 0;
        if (scheduler) {
          const int slot = int(i % URING);
          mbar_wait(&tail->uempty[slot], ((i / URING) & 1) ^ 1);
          u = atomicAdd(p.counter, 1);
          if (u >= p.cunits) u = -1;
          if (u >= 0) {
            const int64_t uu = int64_t(u) * G;
            start = ld_relaxed_gpu_s32(p.seg_pos + uu / p.qtiles) + p.walk_bias * int32_t(uu % p.qtiles + 1);
          }
          tail->uid[slot] = u;
          tail->ustart[slot] = start;
          for (uint32_t c = 1; c < CL; ++c) {
            st_shared_cluster_u32(mapa_shared(smem_u32(&tail->uid[slot]), c), uint32_t(u));
            st_shared_cluster_u32(mapa_shared(smem_u32(&tail->ustart[slot]), c), uint32_t(start));
          }
          mbar_arrive(&tail->ufull[slot]);
          for (uint32_t c = 1; c < CL; ++c)  // release: orders the remote stores above
            mbar_arrive_cluster(mapa_shared(smem_u32(&tail->ufull[slot]), c));
        } else {
          u = next_unit(tail, i, false, true, start);
        }
        if (u < 0) break;
        int qt, seg;
        int64_t r0, r1;
        unit_coords(int64_t(u) * G + pp, p, qt, seg, r0, r1);
        const TileWalk walk(r0, r1, start);
        for (int64_t j = 0; j < walk.ntiles; ++j) {
          const int64_t c0 = walk.c0(j);
          if (scheduler) red_max_relaxed_gpu_s32(p.seg_pos + seg, start + int32_t(j));
          if (RS_PAIR_SYNC_TILES > 0 && scheduler && p.sync_tiles > 0) {
            // publish this unit's position, then wait while it is more than
            // sync_tiles past the slowest running unit of the segment (the
            // slowest never waits, so every unit progresses)
            const int32_t pos = start + int32_t(j);
            st_relaxed_gpu_s32(p.prog + u, pos);
            uint64_t t0 = 0;
            for (;;) {
              int32_t m = kSyncIdle;
              for (int q2 = 0; q2 < p.qtiles; ++q2) {
                if (q2 == qt) continue;
                const int32_t v = ld_relaxed_gpu_s32(p.prog + int64_t(seg) * p.qtiles + q2);
                m = v < m ? v : m;
              }
              if (m == kSyncIdle || pos - m <= p.sync_tiles) break;
              uint64_t t;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
              if (t0 == 0) t0 = t;
              else if (t - t0 > kSyncMaxWaitNs) break;
              __nanosleep(128);
            }
            if (j + 1 == walk.ntiles) st_relaxed_gpu_s32(p.prog + u, kSyncIdle);
          }
          for (int kb = 0; kb < p.kblocks; ++kb) {
            PROF(0, mbar_wait(&tail->empty[stage], phase ^ 1));
            uint8_t* sa = smem + size_t(stage) * C::STAGE_BYTES;
            const uint32_t full_leader = mapa_shared(smem_u32(&tail->full[stage]), pair_leader);
            const int32_t kx = kb * C::BK;
            const int32_t qrow0 = qt * C::PMv + int(half) * C::BMv;
#ifdef RS_EXP_HALF_A  // timing experiment only (wrong results): the query tile is reloaded every other tile
            const bool load_a = (j & 1) == 0;
            if (leader) mbar_arrive_expect_tx(&tail->full[stage], 2 * (C::STAGE_BYTES - (load_a ? 0 : C::A_BYTESv)));
            if (load_a) tma_load_2d_pair(&tmq, full_leader, sa, kx, qrow0, pol_q);
#else
            if (leader) {
              // tf32 + in-kernel residual: only the query halves complete on full[s] by TMA
              const uint32_t tx = (TF && !RS_TF32_STORED_LO) ? 2 * C::NT * C::A_BYTESv : 2 * C::STAGE_BYTES;
              mbar_arrive_expect_tx(&tail->full[stage], tx);
            }
            tma_load_2d_pair(&tmq, full_leader, sa, kx, qrow0, pol_q);
#endif
            if (TF) tma_load_2d_pair(&tmql, full_leader, sa + C::A_BYTESv, kx, qrow0, pol_q);
            if (G == 1) {
#ifdef RS_EXP_L2_CORPUS_ROWS  // timing experiment only (wrong results): corpus reads wrap in an L2-sized window
              const int32_t crow0 = int32_t(c0 % RS_EXP_L2_CORPUS_ROWS) + int(half) * HB;
#else
              const int32_t crow0 = int32_t(c0) + int(half) * HB;
#endif
              if (TF && !RS_TF32_STORED_LO) {
                mbar_arrive_expect_tx(&tail->braw[stage], B_BYTES);
                tma_load_2d(&tmc, &tail->braw[stage], sa + C::OFF_B, kx, crow0, pol_c);
              } else {
                tma_load_2d_pair(&tmc, full_leader, sa + C::OFF_B, kx, crow0, pol_c);
                if (TF) tma_load_2d_pair(&tmcl, full_leader, sa + C::OFF_B + B_BYTES, kx, crow0, pol_c);
              }
              if (RS_PAIR_PREFETCH > 0 && j + RS_PAIR_PREFETCH < walk.ntiles) {
                // the same box RS_PAIR_PREFETCH tiles ahead: the DRAM miss of the
                // first unit to reach a tile no longer stalls the units in lockstep
                const int32_t prow = int32_t(walk.c0(j + RS_PAIR_PREFETCH)) + int(half) * HB;
                tma_prefetch_2d(&tmc, kx, prow);
                if (TF && RS_TF32_STORED_LO) tma_prefetch_2d(&tmcl, kx, prow);
              }
            } else {
              // piece pp of this half's corpus rows, written into the same smem
              // offset of every CTA holding this half in the cluster's G pairs
              tma_load_2d_pair_mc(&tmc, full_leader, sa + C::OFF_B + pp * BPIECE * ROW_BYTES, kx,
                                  int32_t(c0) + int(half) * HB + pp * BPIECE, mc_half, pol_c);
            }
            ++issued;
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      if (TF && !RS_TF32_STORED_LO) {
        // no more tiles: publish the stage count, then wake the converter on
        // the next stage's barrier once its previous use has drained (so the
        // arrival cannot complete a second phase the converter has not seen)
        mbar_wait(&tail->empty[stage], phase ^ 1);
        *reinterpret_cast<volatile int32_t*>(&tail->cvt_stop) = issued;
        mbar_arrive(&tail->braw[stage]);
      }
    }
  } else if (TF && !RS_TF32_STORED_LO && warp == WARP_CVT) {
    // ===== tf32 residual converter (both CTAs): lo = x - trunc_tf32(x) of
    //       this CTA's corpus half, written beside the raw tile =====
    int stage = 0, done = 0;
    uint32_t phase = 0;
    const uint32_t full_leader0 = mapa_shared(smem_u32(&tail->full[0]), pair_leader);
    for (;;) {
      mbar_wait(&tail->braw[stage], phase);
      // the barrier completed either by a corpus tile or by the producer's
      // final arrival, which follows its store of the issued-stage count
      if (done == *reinterpret_cast<volatile int32_t*>(&tail->cvt_stop)) break;
      ++done;
      const float4* src = reinterpret_cast<const float4*>(smem + size_t(stage) * C::STAGE_BYTES + C::OFF_B);
      float4* dst = reinterpret_cast<float4*>(smem + size_t(stage) * C::STAGE_BYTES + C::OFF_B + B_BYTES);
#pragma unroll 4
      for (int i = lane; i < B_BYTES / 16; i += 32) {
        float4 v = src[i];
        v.x -= __uint_as_float(__float_as_uint(v.x) & 0xffffe000u);
        v.y -= __uint_as_float(__float_as_uint(v.y) & 0xffffe000u);
        v.z -= __uint_as_float(__float_as_uint(v.z) & 0xffffe000u);
        v.w -= __uint_as_float(__float_as_uint(v.w) & 0xffffe000u);
        dst[i] = v;
      }
      fence_proxy_async_shared();  // the tensor core reads these stores through the async proxy
      __syncwarp();
      if (lane == 0) {
        if (leader)
          mbar_arrive(&tail->full[stage]);
        else
          mbar_arrive_cluster(full_leader0 + uint32_t(stage) * 8u);
      }
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == WARP_MMA) {
    if (lane == 0) {
      // ===== leader: MMA issuer; both: corpus-norm staging per tile =====
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tile_iter = 0;
      for (uint32_t i = 0;; ++i) {
        int32_t start;
        const int u = next_unit(tail, i, scheduler, true, start);
        if (u < 0) break;
        int qt, seg;
        int64_t r0, r1;
        unit_coords(int64_t(u) * G + pp, p, qt, seg, r0, r1);
        const TileWalk walk(r0, r1, start);
        for (int64_t j = 0; j < walk.ntiles; ++j, ++tile_iter) {
          const int64_t c0 = walk.c0(j);
          const uint32_t acc = tile_iter & 1;
          // leader: both epilogues released TMEM buffer acc; peer: own epilogue released cns[acc]
          PROF(1, mbar_wait(&tail->tempty[acc], ((tile_iter >> 1) & 1) ^ 1));
          tc_fence_after();
          {
            // this tile's corpus norms for the epilogue (the index pads the
            // norms array, so rounding the copy up to 16 B stays in bounds)
            const int valid = int(r1 - c0 < BN ? r1 - c0 : BN);
            const uint32_t bytes = uint32_t((valid + 3) & ~3) * 4u;
            mbar_arrive_expect_tx(&tail->tfull[acc], bytes);
            bulk_copy_g2s(cns + acc * BN, p.cn + c0, bytes, &tail->tfull[acc]);
          }
          if (!leader) continue;
          const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
          for (int kb = 0; kb < p.kblocks; ++kb) {
            if (TF && !RS_TF32_STORED_LO)  // the peer's converter stores are released at cluster scope
              PROF(2, mbar_wait_cluster(&tail->full[stage], phase));
            else
              PROF(2, mbar_wait(&tail->full[stage], phase));
            tc_fence_after();
            const uint32_t a_addr = smem_u32(smem + size_t(stage) * C::STAGE_BYTES);
            const uint32_t b_addr = a_addr + C::OFF_B;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // 4 MMA k-steps of 32 bytes per 128-byte k-block
              if constexpr (!TF) {
                umma_bf16_ss_pair(d_tmem, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                                  C::IDESC, (kb | kk) != 0);
              } else {
                const uint64_t ahi = umma_desc_sw128(a_addr + kk * 32);
                const uint64_t alo = umma_desc_sw128(a_addr + C::A_BYTESv + kk * 32);
                const uint64_t bhi = umma_desc_sw128(b_addr + kk * 32), blo = umma_desc_sw128(b_addr + B_BYTES + kk * 32);
                umma_tf32_ss_pair(d_tmem, alo, bhi, C::IDESC, (kb | kk) != 0);  // small terms first
                umma_tf32_ss_pair(d_tmem, ahi, blo, C::IDESC, 1);
                umma_tf32_ss_pair(d_tmem, ahi, bhi, C::IDESC, 1);
              }
            }
            umma_commit_pair_mc(&tail->empty[stage], uint16_t((1u << CL) - 1u));  // every CTA of the cluster
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit_pair_mc(&tail->tfull[acc], uint16_t(0x3u << (2 * pp)));
        }
      }
    }
  } else if (warp >= EPI_WARP0 && warp < EPI_WARP0 + 4 * EG) {
    // ===== epilogue (both CTAs): 128 queries x 256 chunks per tile =====
    const int ew = (warp - EPI_WARP0) & 3;  // == warp % 4: the TMEM lane quadrant this warp may read
    // column slice of every tile this warp filters, and the list it feeds:
    // M = 256: warp group eg owns [eg*CPG, (eg+1)*CPG) of its quadrant's rows;
    // M = 128: quadrant ew holds rows (ew&1)*32.. for tile columns (ew>>1)*128..
    const int eg = SM ? (ew >> 1) : ((warp - EPI_WARP0) >> 2);
    constexpr int SLICE = SM ? BN / 2 : CPG;
    const int row = SM ? (ew & 1) * 32 + lane : ew * 32 + lane;
    const int tcol0 = SM ? eg * SLICE : 0;  // tile column held at this accumulator's TMEM column 0
    const int et = (warp - EPI_WARP0) * 32 + lane;
    RegTopK<C::KR, EPI_THREADS, BUF, COOP> rt;
    rt.k = p.k;
    rt.wbase = smem_u32(smem + C::OFF_BUF) + uint32_t(et) * 8u;
    rt.sbase = smem_u32(smem + C::OFF_SCR) + uint32_t(warp - EPI_WARP0) * uint32_t(C::KR + BUF) * 8u;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tail->tempty[0]), pair_leader);
    const uint32_t tempty_leader1 = mapa_shared(smem_u32(&tail->tempty[1]), pair_leader);
    uint32_t tile_iter = 0;
#if RS_PAIR_PROFILE
    unsigned long long busy_all = 0, busy_early = 0, n_early = 0;
#endif
    for (uint32_t i = 0;; ++i) {
      int32_t start;
      const int u = next_unit(tail, i, scheduler, false, start);
      __syncwarp();
      if (lane == 0) release_unit(tail, i, scheduler);  // one release per warp, after every lane read the slot
      if (u < 0) break;
      int qt, seg;
      int64_t r0, r1;
      unit_coords(int64_t(u) * G + pp, p, qt, seg, r0, r1);
      const int64_t qrow = int64_t(qt) * C::PMv + int64_t(half) * C::BMv + row;
      const bool real_row = qrow < p.nq;
      rt.qn = real_row ? p.qn[qrow] : 0.0f;
      rt.reset();
#ifndef RS_PAIR_NO_SHARED_TAU
      // threshold sharing: start from the best k-th distance any unit of this
      // query has published (units of other segments, finished or running)
      if (real_row) rt.seed(shared_bound(p, qrow));
      uint32_t tau_pending = 0xffffffffu;
#endif
      const TileWalk walk(r0, r1, start);
      for (int64_t j = 0; j < walk.ntiles; ++j, ++tile_iter) {
        const int64_t c0 = walk.c0(j);
        // ids below every one seen so far from here on: flush the earlier
        // phase's candidates, then tag the rest phase 0 (RegTopK ordering)
        if (rt.phase && walk.wrapped(j)) {
          rt.template flush<RS_TOPK_COOP_ALL_SITES>();
          rt.phase = 0;
        }
        const uint32_t acc = tile_iter & 1;
        const int valid = int(r1 - c0 < BN ? r1 - c0 : BN);
        const float* cn_t = cns + acc * BN;
#ifndef RS_PAIR_NO_SHARED_TAU
        // every 4th tile: fetch the shared threshold (consumed after the tile)
        if ((j & 3) == 0 && real_row) tau_pending = shared_bound(p, qrow);
#endif
        // the tile's eight 32-column norm minima, loaded before the wait
        const float4 cm0 = __ldg(reinterpret_cast<const float4*>(p.cmin + (c0 >> 5)));
        const float4 cm1 = __ldg(reinterpret_cast<const float4*>(p.cmin + (c0 >> 5)) + 1);
        PROF(3, mbar_wait(&tail->tfull[acc], (tile_iter >> 1) & 1));
        tc_fence_after();
#if RS_PAIR_PROFILE
        const long long t_tile0 = clock64();
#endif
        const uint32_t t_row = tmem_base + (uint32_t(ew * 32) << 16) + acc * C::ACC_COLS - tcol0;
        const uint32_t id0 = uint32_t(p.id_base + c0);
        // this chunk's dot bound (epi_chunk32b)
        auto chunk_thr = [&](int base) -> float {
          const int ci = base >> 5;
          const float4 ch = ci < 4 ? cm0 : cm1;
          const int cj = ci & 3;
          const float cmin = cj < 2 ? (cj == 0 ? ch.x : ch.y) : (cj == 2 ? ch.z : ch.w);
#ifdef RS_EXP_NO_SLOW  // timing experiment only (wrong results): no candidate ever passes the bound
          (void)cmin;
          return __int_as_float(0x7f800000);
#else
          return chunk_threshold(rt.qn, cmin, rt.tau);
#endif
        };
        auto filter = [&](const uint32_t(&r)[EPI_COLS], int base, float thr) {
#ifdef RS_PAIR_EPI_NOP  // timing experiment only: the MMA pipeline without the top-k work
          if (__uint_as_float(r[0]) == 12345.0f) rt.append_raw(0.0f, id0);
          return;
#endif
          if (base + EPI_COLS <= valid)
            epi_chunk32b<C::KR, EPI_THREADS, BUF, CHECK, true, COOP>(rt, r, cn_t + base, id0 + base, EPI_COLS, thr);
          else
            epi_chunk32b<C::KR, EPI_THREADS, BUF, CHECK, false, COOP>(rt, r, cn_t + base, id0 + base, valid - base, thr);
        };
#if RS_PAIR_EPI_PAIRED
        // two 32-column loads in flight per wait (4 waits per 256-column tile)
#pragma unroll 1
        for (int base = eg * SLICE; base < (eg + 1) * SLICE; base += 2 * EPI_COLS) {
          if (base >= valid) break;  // warp-uniform
          const bool two = base + EPI_COLS < valid;
          uint32_t r0[EPI_COLS], r1[EPI_COLS];
          __syncwarp();
          tmem_ld_32x32b_x32(t_row + base, r0);
          if (two) tmem_ld_32x32b_x32(t_row + base + EPI_COLS, r1);
          const float thr0 = chunk_thr(base);
          tmem_wait_ld();
          filter(r0, base, thr0);
          if (two) filter(r1, base + EPI_COLS, chunk_thr(base + EPI_COLS));
        }
#else
#pragma unroll 1
        for (int base = eg * SLICE; base < (eg + 1) * SLICE; base += EPI_COLS) {
          if (base >= valid) break;  // warp-uniform
          uint32_t r[EPI_COLS];
          __syncwarp();
          tmem_ld_32x32b_x32(t_row + base, r);
          const float thr = chunk_thr(base);  // computed while the load is in flight
          PROF(6, tmem_wait_ld());
          PROF(4, filter(r, base, thr));
        }
#endif
#ifndef RS_PAIR_NO_SHARED_TAU
        if ((j & 3) == 0 && real_row) {
          // publish this list's k-th best (a bound for every other unit of
          // the query), then adopt the fetched one
          const uint32_t kb = rt.kth_bits();
          if (kb < 0x7f800000u && kb < tau_pending) red_min_relaxed_gpu_u32(p.qtau + qrow, kb);
          rt.seed(tau_pending);
        }
#endif
#if RS_PAIR_PROFILE
        {  // busy epilogue cycles of this tile: the first 4 tiles of a unit vs all
          const long long dt = clock64() - t_tile0;
          busy_all += dt;
          if (j < 4) {
            busy_early += dt;
            ++n_early;
          }
        }
#endif
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          // the TMEM reads completed (tcgen05.wait::ld), so a relaxed remote
          // arrive suffices (a release at cluster scope costs a MEMBAR.GPU)
          mbar_arrive(&tail->tempty[acc]);
          if (!leader) mbar_arrive_cluster_relaxed(acc ? tempty_leader1 : tempty_leader0);
        }
      }
      // every lane flushes (warp-collective), then writes its row if it is a real query
      PROF(5, rt.template flush<RS_TOPK_COOP_ALL_SITES>());
#ifndef RS_PAIR_NO_SHARED_TAU
      if (real_row) {
        if (rt.kth_bits() < 0x7f800000u) red_min_relaxed_gpu_u32(p.qtau + qrow, rt.kth_bits());
        // this finished list holds >= j*r rows at or below its rank-j*r
        // distance: insert it into the query's kCas-smallest cascade (ranks
        // r, 2r, ... with RS_PAIR_CAS_MULTI; see shared_bound)
        uint32_t* cas = p.qcas + qrow * kCas;
        const uint32_t cut = RS_PAIR_CAS_MULTI ? ld_relaxed_gpu_u32(cas + (kCas - 1)) : 0xffffffffu;
#pragma unroll 1
        for (int j = 1; j <= (RS_PAIR_CAS_MULTI ? kCas : 1); ++j) {
          const uint32_t rb = rt.rank_bits(j * p.cas_rank);
          if (rb >= 0x7f800000u || rb >= cut) break;  // ranks ascend: so do the rest
          cascade_min_insert(cas, rb);
        }
      }
#endif
      if (qrow < p.nq) rt.finish(p.part + ((qrow * p.segments + seg) * C::LPS + eg) * p.k);
    }
    if (lane == 0 && rt.bursts) atomicAdd(p.bursts, rt.bursts);  // the host's lean / cooperative choice
#if RS_PAIR_PROFILE && RS_TOPK_COUNTERS
    if (blockIdx.x < 1024) {
      const uint32_t cnt[5] = {rt.c_groups, rt.c_appends, rt.c_flushes, rt.c_inserts, rt.c_coop};
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        // groups / flushes / inserts are warp-uniform events: count them once per warp
        const uint32_t v = i == 1 ? __reduce_add_sync(0xffffffffu, cnt[i]) : cnt[i];
        if (lane == 0) atomicAdd(&g_pair_prof[blockIdx.x][8 + i], (unsigned long long)v);
      }
    }
#endif
#if RS_PAIR_PROFILE
    if (lane == 0 && blockIdx.x < 1024) {  // [13] busy cycles in a unit's first 4 tiles, [14] in all, [15] first-4 tiles
      atomicAdd(&g_pair_prof[blockIdx.x][13], busy_early);
      atomicAdd(&g_pair_prof[blockIdx.x][14], busy_all);
      atomicAdd(&g_pair_prof[blockIdx.x][15], n_early);
    }
#endif
  }
#if RS_PAIR_PROFILE
  prof[7] = clock64() - t_start;
  if (lane == 0 && warp < 8 && blockIdx.x < 1024) {
    for (int i = 0; i < 8; ++i)
      if (prof[i]) atomicAdd(&g_pair_prof[blockIdx.x][i], prof[i] / ((warp >= EPI_WARP0 && i == 7) ? 4 : 1));
  }
#endif

  __syncwarp();
  tc_fence_before();
  cluster_sync();  // the peer's smem / TMEM stay alive until the leader's MMAs are done
  if (warp == WARP_TMEM) {
    tc_fence_after();
    tmem_dealloc_pair(tmem_base, TMEM_COLS);
  }
  // the last CTA to finish posts the launch's burst count straight to pinned
  // host memory (the host's lean / cooperative choice for the next search):
  // no copy in the stream, no synchronisation
  if (p.bursts_host && threadIdx.x == 0) {  // every warp of this CTA added its count before cluster_sync
    __threadfence();
    if (atomicAdd(p.done, 1) == int(gridDim.x) - 1) {
      __threadfence();
      *reinterpret_cast<volatile uint32_t*>(p.bursts_host) = atomicAdd(p.bursts, 0u);
    }
  }
}

}  // namespace

#if RS_PAIR_PROFILE
extern "C" int rs_debug_pair_profile(unsigned long long* host_out, int nblocks) {
  cudaDeviceSynchronize();
  return int(cudaMemcpyFromSymbol(host_out, g_pair_prof, sizeof(unsigned long long) * 16 * nblocks));
}
extern "C" int rs_debug_pair_profile_reset() {
  static unsigned long long zeros[1024][16];
  return int(cudaMemcpyToSymbol(g_pair_prof, zeros, sizeof(zeros)));
}
#endif

namespace {

template <bool TF, bool SM, bool COOP>
int set_smem_attr() {
  static bool done = false;
  if (!done) {
    RS_CHECK_CUDA(cudaFuncSetAttribute(score_topk_pair_kernel<TF, SM, COOP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(Cfg<TF, SM>::SMEM_BYTES)),
                  "cudaFuncSetAttribute(score_topk_pair_kernel)");
    done = true;
  }
  return RS_OK;
}

template <bool TF, bool SM, bool COOP>
int launch_t(const CUtensorMap& tmq, const CUtensorMap& tmql, const CUtensorMap& tmc, const CUtensorMap& tmcl,
             const Params& p, int ctas, cudaStream_t st) {
  int rc = set_smem_attr<TF, SM, COOP>();
  if (rc) return rc;
  score_topk_pair_kernel<TF, SM, COOP>
      <<<CL * ctas, NUM_THREADS, Cfg<TF, SM>::SMEM_BYTES, st>>>(tmq, tmql, tmc, tmcl, p);
  RS_CHECK_LAUNCH("score_topk_pair_kernel");
  return RS_OK;
}

}  // namespace

// After the probe pass (the same kernel over the first rows of the corpus,
// one tile per segment): fold each query's cascade bound into qtau.  Slot
// kCas-1 is backed by kCas disjoint probe lists with >= cas_rank rows each at
// or below it (>= k real rows), so it is a valid bound of the query's final
// k-th distance by itself; the cascade is then restarted by the main launch,
// whose lists overlap the probe's rows and must not combine with its entries.
__global__ void fold_probe_bounds_kernel(uint32_t* __restrict__ qtau, int64_t nq) {
  const int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const uint32_t b = qtau[nq + q * kCas + (kCas - 1)];
  if (b < qtau[q]) qtau[q] = b;
}

int launch_fold_probe_bounds(uint32_t* qtau, int64_t nq, cudaStream_t st) {
  if (nq <= 0) return RS_OK;
  fold_probe_bounds_kernel<<<unsigned((nq + 255) / 256), 256, 0, st>>>(qtau, nq);
  RS_CHECK_LAUNCH("fold_probe_bounds_kernel");
  return RS_OK;
}

int pair_tile_rows(bool small) { return small ? Cfg<false, true>::PMv : Cfg<false, false>::PMv; }

int launch_score_topk_pair(const CUtensorMap& tmq, const CUtensorMap* tmql, const CUtensorMap& tmc,
                           const CUtensorMap* tmcl, const float* qn, const float* cn, const float* cmin, int64_t nq,
                           int64_t n, int dim, int k, int64_t id_base, const SearchPlan& plan, bool small,
                           uint64_t* part, int32_t* counter, int32_t walk_bias, uint32_t* qtau, bool coop,
                           uint32_t* bursts_host, cudaStream_t st, bool keep_tau) {
  const bool tf = tmql != nullptr;
  RS_REQUIRE(!tf || !RS_TF32_STORED_LO || tmcl != nullptr, "tf32 path with stored residuals needs the corpus lo map");
  RS_REQUIRE(!tf || G == 1, "the tf32 path has no multicast (RS_PAIR_GROUP) variant");
  RS_REQUIRE(k >= 1 && k <= (tf ? KREG_TF32 : KREG), "k (%d) exceeds the register top-k capacity (%d)", k,
             tf ? KREG_TF32 : KREG);
  RS_REQUIRE(!small || G == 1, "the M = 128 variant has no multicast (RS_PAIR_GROUP) variant");
  // (its epilogue splits columns by lane quadrant, not by warp group)
  RS_REQUIRE(!small || EG == 1, "the M = 128 variant has one epilogue warp group");
  RS_REQUIRE(plan.lists_per_seg == (small ? 2 : kPairEpiGroups), "plan lists per segment do not match the kernel");
  RS_REQUIRE(plan.segments >= 1 && plan.segments <= kMaxSegments, "segments out of range (%d)", plan.segments);
  RS_CHECK_CUDA(cudaMemsetAsync(counter, 0, sizeof(int32_t) * (3 + plan.segments), st),
                "cudaMemsetAsync(unit counter, burst count, finished CTAs, segment frontiers)");
  // keep_tau: qtau already holds a bound of this search's queries (the probe
  // pass, fold_probe_bounds); only the cascade of finished lists restarts
  RS_CHECK_CUDA(cudaMemsetAsync(keep_tau ? qtau + nq : qtau, 0xff,
                                sizeof(uint32_t) * size_t(nq) * (keep_tau ? kCas : 1 + kCas), st),
                "cudaMemsetAsync(shared bounds)");
  Params p{};
  p.qn = qn;
  p.cn = cn;
  p.cmin = cmin;
  p.nq = nq;
  p.n = n;
  const int bk = tf ? Cfg<true>::BK : Cfg<false>::BK;
  p.kblocks = (dim + bk - 1) / bk;
  p.k = k;
  p.id_base = id_base;
  // the plan counts cluster units (G pair tiles); the kernel works in pair
  // tiles, padded to a multiple of G (pad rows are >= nq)
  p.qtiles = plan.qtiles * G;
  p.segments = plan.segments;
  p.seg_rows = plan.seg_rows;
  p.part = part;
  p.counter = counter;
  p.bursts = reinterpret_cast<uint32_t*>(counter + 1);
  p.done = counter + 2;
  p.bursts_host = bursts_host;
  p.seg_pos = counter + 3;
  // drift limiter: the plan's choice (make_plan), G == 1 only
  RS_REQUIRE(plan.sync_tiles == 0 || (G == 1 && p.qtiles <= kSyncMaxQtiles), "drift limiter plan out of range");
  p.sync_tiles = RS_PAIR_SYNC_TILES > 0 ? plan.sync_tiles : 0;
  p.prog = counter + 3 + kMaxSegments;
  if (p.sync_tiles > 0)
    RS_CHECK_CUDA(cudaMemsetAsync(p.prog, 0x7f, sizeof(int32_t) * size_t(p.qtiles) * plan.segments, st),
                  "cudaMemsetAsync(unit positions)");
  p.walk_bias = walk_bias;
  p.qtau = qtau;
  p.qcas = qtau + nq;  // the caller allocates nq * (1 + kCas) words
  p.cas_rank = (k + kCas - 1) / kCas;
  p.cunits = int64_t(plan.qtiles) * plan.segments;
  const CUtensorMap& ql = tf ? *tmql : tmq;
  const CUtensorMap& cl = (tf && tmcl) ? *tmcl : tmc;
  if (coop) {
    if (tf) return small ? launch_t<true, true, true>(tmq, ql, tmc, cl, p, plan.ctas, st)
                         : launch_t<true, false, true>(tmq, ql, tmc, cl, p, plan.ctas, st);
    return small ? launch_t<false, true, true>(tmq, ql, tmc, cl, p, plan.ctas, st)
                 : launch_t<false, false, true>(tmq, ql, tmc, cl, p, plan.ctas, st);
  }
  if (tf) return small ? launch_t<true, true, false>(tmq, ql, tmc, cl, p, plan.ctas, st)
                       : launch_t<true, false, false>(tmq, ql, tmc, cl, p, plan.ctas, st);
  return small ? launch_t<false, true, false>(tmq, ql, tmc, cl, p, plan.ctas, st)
               : launch_t<false, false, false>(tmq, ql, tmc, cl, p, plan.ctas, st);
}

}  // namespace rs
