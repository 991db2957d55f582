// Internal interfaces between the retrieval translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "rs_common.cuh"

namespace rs {

// Work split of one search over a corpus shard: the corpus is cut into
// `segments` contiguous row ranges of `seg_rows` rows (a multiple of the
// kernel's column tile) and the queries into `qtiles` row tiles; a unit is
// (query tile, segment) and writes one sorted top-k list per query row to
// part[(row * segments + segment) * k].  Units are ordered segment-major so the
// CTAs that run concurrently stream the same corpus segment (L2 reuse).
struct SearchPlan {
  int32_t qtiles = 0;
  int32_t segments = 0;
  int64_t seg_rows = 0;
  int32_t ctas = 0;
  int32_t lists_per_seg = 1;  // sorted lists a unit writes per query (epilogue groups)
  int32_t sync_tiles = 0;     // pair kernel drift limiter window (0 = off)
  int32_t lists() const { return segments * lists_per_seg; }
};

// In-kernel wait of the peer-exchange merge (peer.cu): every flag of
// flags[0..n) must reach `epoch` (wrapping compare) before the lists are read;
// after timeout_ns the kernel sets *error = 1 and merges what is there.
struct PeerWait {
  const uint32_t* flags = nullptr;
  int32_t n = 0;
  uint32_t epoch = 0;
  int32_t* error = nullptr;
  uint64_t timeout_ns = 0;
};

// K2 merge (nlists <= 64) that first waits on `pw` (lists written by peers)
int launch_merge_wait(const uint64_t* keys, int64_t nq, int nlists, int k_in, int64_t list_stride, int64_t q_stride,
                      int k, const rs_config* keep, float* D, int64_t* I, const PeerWait& pw, cudaStream_t st);

// ---- peer-exchange regions (peer.cu; layout documented in ragsched_b200.h) ----
constexpr size_t kPeerCounterOff = 256;  // uint32, after flags[RS_PEER_MAX]
constexpr size_t kPeerErrorOff = 260;    // int32
constexpr size_t kPeerKeysOff = 512;
__host__ __device__ inline uint32_t* peer_flags(void* r) { return static_cast<uint32_t*>(r); }
__host__ __device__ inline uint32_t* peer_counter(void* r) {
  return reinterpret_cast<uint32_t*>(static_cast<char*>(r) + kPeerCounterOff);
}
__host__ __device__ inline int32_t* peer_error(void* r) {
  return reinterpret_cast<int32_t*>(static_cast<char*>(r) + kPeerErrorOff);
}
__host__ __device__ inline uint64_t* peer_keys(void* r) {
  return reinterpret_cast<uint64_t*>(static_cast<char*>(r) + kPeerKeysOff);
}

// first query row of rank o's slice of an nq batch (dist.shard_range)
__host__ __device__ inline int64_t peer_slice_lo(int64_t nq, int o, int world) { return (int64_t(o) * nq) / world; }

// Where query q's key row (this rank's shard list) goes: the owner's region,
// list (epoch parity, source ex.rank), row q - slice_lo(owner).
__device__ __forceinline__ uint64_t* peer_row(const rs_peer_exchange& ex, int64_t nq, int64_t q, uint32_t epoch) {
  const int W = ex.world;
  int o = int((q * W) / nq);
  while (o + 1 < W && q >= peer_slice_lo(nq, o + 1, W)) ++o;
  while (q < peer_slice_lo(nq, o, W)) --o;
  const int64_t par = epoch & 1u;
  return peer_keys(ex.region[o]) + ((par * W + ex.rank) * ex.slice_cap + (q - peer_slice_lo(nq, o, W))) * ex.k;
}

// Block epilogue of a kernel that stored key rows with peer_row: every
// thread's stores are ordered before its block's arrival; the last block of
// the grid raises flags[rank] = epoch in every region (release, system
// scope) and resets the arrival counter.  All threads of every block call it.
__device__ __forceinline__ void peer_signal(const rs_peer_exchange& ex, uint32_t epoch) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t* counter = peer_counter(ex.region[ex.rank]);
    const uint32_t prev = atomicAdd(counter, 1u);
    if (prev == gridDim.x - 1) {
      *counter = 0;  // every block has arrived; the next exchange is stream-ordered after this one
      __threadfence_system();
      for (int s = 0; s < ex.world; ++s) {
        uint32_t* f = peer_flags(ex.region[s]) + ex.rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
      }
    }
  }
}

int check_peer_exchange(const rs_peer_exchange* ex);
// the scatter kernel: key rows [nq, ex.k] -> owners' regions, then the signal
int launch_peer_scatter(const rs_peer_exchange& ex, const uint64_t* keys, int64_t nq, uint32_t epoch, cudaStream_t st);
// the K2 merge of a search whose output rows go straight to the owners'
// regions (nlists <= 64, k == ex.k), then the signal
int launch_merge_to_peers(const uint64_t* keys, int64_t nq, int nlists, int k_in, int64_t list_stride,
                          int64_t q_stride, const rs_peer_exchange& ex, uint32_t epoch, cudaStream_t st);

// upper bound of SearchPlan::segments (plan_search never exceeds it)
constexpr int kMaxSegments = 4096;
// Pair kernel drift limiter.  With few query tiles every unit of a segment
// streams the same corpus rows at once, but the dynamically scheduled pairs
// drift apart by more than the segment's share of L2 and the laggard re-reads
// the rows from DRAM (cfg4 corpus, nq 512: 1.39x the corpus).  A unit's
// producer then waits (bounded, per tile) while it is more than
// RS_PAIR_SYNC_TILES tiles past the slowest running unit of its segment.
// Enabled by make_plan when 2 <= query tiles <= kSyncMaxQtiles and the units
// are exactly one round of pairs (on B200: 2 query tiles x 37 segments).
// Measured (cfg4 corpus, tools/r2d_gpu5-7.sh, profiles/r2_drift_limiter.md):
// nq 512 DRAM 28.4 -> 20.7 GB per launch (1.01x the corpus), +3-11% q/s;
// nq 384 +5-7%; with more rounds of units the waits cost about what the
// re-reads do (nq 1024, 2 rounds: +0.5-4%) or more (nq 768, 3 rounds: -4 to
// -6.5%; nq 2048: -6%), and cfg1 (72 units) gains nothing, so it stays off
// there.  Unit positions live after the segment frontiers in the schedule
// counters.
#ifndef RS_PAIR_SYNC_TILES
#define RS_PAIR_SYNC_TILES 2
#endif
constexpr int kSyncMaxQtiles = 4;

SearchPlan plan_search(int64_t nq, int64_t n, int bq, int bn, int ctas_capacity, int64_t row_bytes,
                       bool share_l2);

// tcgen05/TMA/TMEM bf16 kernel (score_topk_sm100.cu).
constexpr int kTcMaxK = 40;
// fp32 (3xTF32) path: 1 (default) = residuals precomputed at add() and
// streamed as a second tensor; 0 = the corpus tf32 residual is formed in shared
// memory by the pair kernel's converter warp (corpus stored and streamed once;
// measured slower: cfg1 0.99M vs 1.45M q/s, the one converter warp limits)
#ifndef RS_TF32_STORED_LO
#define RS_TF32_STORED_LO 1
#endif
// fp32 (3xTF32) path: extra candidates kept for the exact fp32 re-rank
constexpr int kRefineExtra = 8;
constexpr int kTcBM = 128;
constexpr int kTcBN = 256;
size_t tc_smem_bytes();
int launch_score_topk_tc(const CUtensorMap& tmq, const CUtensorMap& tmc, const float* qn, const float* cn,
                         int64_t nq, int64_t n, int dim, int k, int64_t id_base, const SearchPlan& plan,
                         uint64_t* part, cudaStream_t st);
// CTA-pair (cta_group::2) variant, 256 queries per pair tile (score_topk_sm100_pair.cu).
// kPairGroup pairs form one cluster and share each corpus tile through TMA
// multicast (they work on consecutive query tiles of the same segment).
// (Measured: multicast does not pay on B200 — per-SM smem ingress, not L2
// output, bounds the operand feed — so the default is 1, no multicast.)
#ifndef RS_PAIR_GROUP
#define RS_PAIR_GROUP 1
#endif
constexpr int kPairGroup = RS_PAIR_GROUP;
// Epilogue warp groups per CTA: each owns a column slice of every tile and
// keeps its own top-k per query, so a (query, segment) unit emits this many
// sorted lists.
#ifndef RS_PAIR_EPI_GROUPS
#define RS_PAIR_EPI_GROUPS 1  // 2 measured no faster on B200 (and doubles the partial lists)
#endif
constexpr int kPairEpiGroups = RS_PAIR_EPI_GROUPS;
// tmql / tmcl: the fp32 path's lo maps (3xTF32), NULL for bf16.
int launch_score_topk_pair(const CUtensorMap& tmq, const CUtensorMap* tmql, const CUtensorMap& tmc,
                           const CUtensorMap* tmcl, const float* qn, const float* cn, const float* cmin, int64_t nq,
                           int64_t n, int dim, int k, int64_t id_base, const SearchPlan& plan, bool small,
                           uint64_t* part, int32_t* counter, int32_t walk_bias, uint32_t* qtau, bool coop,
                           uint32_t* bursts_host, cudaStream_t st, bool keep_tau = false);
// qtau[q] = min(qtau[q], cascade slot kCas-1) after a probe launch
int launch_fold_probe_bounds(uint32_t* qtau, int64_t nq, cudaStream_t st);
// query rows per pair tile: 256, or 128 for the small-batch (M = 128) variant
int pair_tile_rows(bool small);
// 32-bit words of shared-bound state per query the pair kernel needs (qtau + cascade)
#ifndef RS_PAIR_CAS
#define RS_PAIR_CAS 4  // cascade slots per query (score_topk_sm100_pair.cu)
#endif
#ifndef RS_PAIR_CAS_MULTI
#define RS_PAIR_CAS_MULTI 0  // 1: every finished list inserts ranks r, 2r, ... (not only r)
#endif
constexpr int64_t kSharedBoundWords = 1 + RS_PAIR_CAS;
// queries up to which a search uses the M = 128 pair tile (one tile, no padding rows)
constexpr int64_t kSmallBatchMax = 128;
// per 32-row chunk minimum of the squared norms over rows [r0, r1) of a shard
// (recomputes every chunk the range touches)
int launch_chunk_min(const float* norms, int64_t r0, int64_t r1, float* cmin, cudaStream_t st);
int encode_kmajor_bf16_map(CUtensorMap* map, const void* base, int64_t rows, int dim, int box_rows);
// dtype RS_BF16 or RS_F32: 128-byte boxes (64 bf16 / 32 fp32) x box_rows, SWIZZLE_128B.
int encode_kmajor_map(CUtensorMap* map, const void* base, int64_t rows, int dim, int box_rows, int dtype);

// CUDA-core kernel for fp32 (and bf16 cross-checks), retrieval.cu.
constexpr int kSimtBQ = 64;
constexpr int kSimtBC = 64;

}  // namespace rs
