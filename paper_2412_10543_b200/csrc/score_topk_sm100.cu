// K1 score_topk (sm_100a): fused exact-L2 scoring GEMM + streaming top-k.
//
// Replaces FAISS IndexFlatL2.search for a bf16 corpus shard.
// The score matrix never reaches HBM: each CTA keeps the fp32 dot products of
// a 128-query x 256-chunk tile in TMEM, and its epilogue warps turn them into
// distances and filter them into per-query top-k heaps in shared memory.
//
//   warp 0      TMA producer: query tile A [128 x 64] + corpus tile B [256 x 64]
//               per k-block into a STAGES-deep smem ring (128 B swizzle)
//   warp 1      MMA issuer (one thread): tcgen05.mma.kind::f16, M=128 N=256
//               K=16, fp32 accumulators in TMEM, double-buffered (2 x 256 cols)
//   warp 2      TMEM allocator
//   warps 4-7   epilogue: tcgen05.ld 32 columns at a time, d = |q|^2+|c|^2-2qc,
//               threshold filter -> RowTopK (topk_rows.cuh); one thread per query
//
// Work = units (query tile, corpus segment), persistent CTAs, segment-major
// order (see SearchPlan).  Each unit writes one sorted top-k list per query;
// merge_topk (retrieval.cu) combines the segment lists.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "retrieval.cuh"
#include "sm100_ptx.cuh"
#include "topk_rows.cuh"

namespace rs {
namespace {

using namespace sm100;

constexpr int BM = kTcBM;
constexpr int BN = kTcBN;
constexpr int BK = 64;  // bf16 elements per k-block = 128-byte rows
constexpr int STAGES = 3;
constexpr int KCAP = kTcMaxK;
constexpr int BUF = 24;
constexpr int CHECK = 8;  // flush check granularity (BUF - CHECK = flush trigger)
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 2 * BN;
constexpr int NUM_THREADS = 256;
constexpr int EPI_WARP0 = 4;
constexpr uint32_t IDESC = umma_idesc_bf16_f32(BM, BN);

struct __align__(8) SmemTail {
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tfull[2];
  uint64_t tempty[2];
  uint32_t tmem_base;
};

constexpr size_t OFF_HEAP = size_t(STAGES) * STAGE_BYTES;
constexpr size_t OFF_BUF = OFF_HEAP + size_t(KCAP) * BM * 8;
constexpr size_t OFF_CN = OFF_BUF + size_t(BUF) * BM * 8;
constexpr size_t OFF_TAIL = OFF_CN + 2 * BN * sizeof(float);
constexpr size_t SMEM_BYTES = OFF_TAIL + sizeof(SmemTail) + 1024;  // + alignment slack

struct Params {
  const float* qn;
  const float* cn;
  int64_t nq, n;
  int32_t kblocks;
  int32_t k;
  int64_t id_base;
  int32_t qtiles, segments;
  int64_t seg_rows;
  uint64_t* part;
};

__device__ __forceinline__ void unit_coords(int64_t u, const Params& p, int& qt, int& seg, int64_t& r0,
                                            int64_t& r1) {
  seg = int(u / p.qtiles);
  qt = int(u - int64_t(seg) * p.qtiles);
  r0 = int64_t(seg) * p.seg_rows;
  r1 = r0 + p.seg_rows;
  if (r1 > p.n) r1 = p.n;
}

template <bool FULL>
__device__ __forceinline__ void epi_group(RowTopK<BM, BUF>& rt, const uint32_t* r, const float* cn, float qnv,
                                          uint32_t id, int lim) {
  epi_group8<BM, BUF, CHECK, FULL>(rt, r, cn, qnv, id, lim);
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    score_topk_tc_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmc,
                         const Params p) {
  // The kernel has no static shared memory, so the dynamic window starts at
  // the CTA's shared-memory base (1024-aligned, as SWIZZLE_128B requires);
  // indexing the array directly keeps every access in the shared window
  // (LDS/STS rather than generic loads).
  extern __shared__ __align__(1024) uint8_t smem[];
  if ((smem_u32(smem) & 1023u) != 0) __trap();
  SmemTail* tail = reinterpret_cast<SmemTail*>(smem + OFF_TAIL);
  uint64_t* heap = reinterpret_cast<uint64_t*>(smem + OFF_HEAP);
  uint64_t* buf = reinterpret_cast<uint64_t*>(smem + OFF_BUF);
  float* cns = reinterpret_cast<float*>(smem + OFF_CN);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t units = int64_t(p.qtiles) * p.segments;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmq);
    tma_prefetch_desc(&tmc);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&tail->full[s], 1);
      mbar_init(&tail->empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tail->tfull[a], 2);  // cnorm bulk copy (expect_tx) + MMA commit
      mbar_init(&tail->tempty[a], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc(&tail->tmem_base, TMEM_COLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = tail->tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_q = policy_evict_last();   // query tiles are re-read per corpus tile
      // corpus: streamed exactly once when a single query tile exists; otherwise
      // the qtiles CTAs of a round share each segment through L2
      const uint64_t pol_c = p.qtiles == 1 ? policy_evict_first() : policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int qt, seg;
        int64_t r0, r1;
        unit_coords(u, p, qt, seg, r0, r1);
        for (int64_t c0 = r0; c0 < r1; c0 += BN) {
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&tail->empty[stage], phase ^ 1);
            uint8_t* sa = smem + size_t(stage) * STAGE_BYTES;
            mbar_arrive_expect_tx(&tail->full[stage], STAGE_BYTES);
            tma_load_2d(&tmq, &tail->full[stage], sa, kb * BK, qt * BM, pol_q);
            tma_load_2d(&tmc, &tail->full[stage], sa + A_BYTES, kb * BK, int32_t(c0), pol_c);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      int stage = 0;
      uint32_t phase = 0;
      uint32_t tile_iter = 0;
      for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int qt, seg;
        int64_t r0, r1;
        unit_coords(u, p, qt, seg, r0, r1);
        for (int64_t c0 = r0; c0 < r1; c0 += BN, ++tile_iter) {
          const uint32_t acc = tile_iter & 1;
          mbar_wait(&tail->tempty[acc], ((tile_iter >> 1) & 1) ^ 1);
          tc_fence_after();
          {
            // stage this tile's corpus norms for the epilogue (the index pads
            // the norms array, so rounding the copy up to 16 B stays in bounds)
            const int valid = int(r1 - c0 < BN ? r1 - c0 : BN);
            const uint32_t bytes = uint32_t((valid + 3) & ~3) * 4u;
            mbar_arrive_expect_tx(&tail->tfull[acc], bytes);
            bulk_copy_g2s(cns + acc * BN, p.cn + c0, bytes, &tail->tfull[acc]);
          }
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < p.kblocks; ++kb) {
            mbar_wait(&tail->full[stage], phase);
            tc_fence_after();
            const uint32_t a_addr = smem_u32(smem + size_t(stage) * STAGE_BYTES);
            const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              umma_bf16_ss(d_tmem, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32), IDESC,
                           (kb | kk) != 0);
            }
            umma_commit(&tail->empty[stage]);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          umma_commit(&tail->tfull[acc]);
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ===== epilogue: TMEM -> distances -> per-query top-k =====
    const int ew = warp - EPI_WARP0;  // == warp % 4: the TMEM lane quadrant this warp may read
    const int row = ew * 32 + lane;
    RowTopK<BM, BUF> rt{heap, buf, row, p.k, 0, 0, 0.0f};
    uint32_t tile_iter = 0;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
      int qt, seg;
      int64_t r0, r1;
      unit_coords(u, p, qt, seg, r0, r1);
      const int64_t qrow = int64_t(qt) * BM + row;
      const float qnv = qrow < p.nq ? p.qn[qrow] : 0.0f;
      rt.reset();
      for (int64_t c0 = r0; c0 < r1; c0 += BN, ++tile_iter) {
        const uint32_t acc = tile_iter & 1;
        const int valid = int(r1 - c0 < BN ? r1 - c0 : BN);
        const float* cn_t = cns + acc * BN;
        mbar_wait(&tail->tfull[acc], (tile_iter >> 1) & 1);
        tc_fence_after();
        const uint32_t t_row = tmem_base + (uint32_t(ew * 32) << 16) + acc * BN;
        const uint32_t id0 = uint32_t(p.id_base + c0);
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          if (ch * 32 >= valid) break;  // warp-uniform
          uint32_t r[32];
          __syncwarp();
          tmem_ld_32x32b_x32(t_row + ch * 32, r);
          tmem_wait_ld();
          if (ch * 32 + 32 <= valid) {
#pragma unroll
            for (int g = 0; g < 32; g += CHECK)
              epi_group<true>(rt, r + g, cn_t + ch * 32 + g, qnv, id0 + ch * 32 + g, CHECK);
          } else {
#pragma unroll
            for (int g = 0; g < 32; g += CHECK)
              epi_group<false>(rt, r + g, cn_t + ch * 32 + g, qnv, id0 + ch * 32 + g, valid - ch * 32 - g);
          }
        }
        tc_fence_before();
        mbar_arrive(&tail->tempty[acc]);
      }
      if (qrow < p.nq) rt.finish(p.part + (qrow * p.segments + seg) * p.k);
    }
  }

  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, TMEM_COLS);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  }
  return fn;
}

}  // namespace

size_t tc_smem_bytes() { return SMEM_BYTES; }

int encode_kmajor_map(CUtensorMap* map, const void* base, int64_t rows, int dim, int box_rows, int dtype) {
  EncodeTiledFn fn = get_encode_fn();
  if (!fn) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return RS_ERR_UNSUPPORTED;
  }
  const int es = dtype == RS_BF16 ? 2 : 4;
  RS_REQUIRE((int64_t(dim) * es) % 16 == 0, "TMA path needs 16-byte rows (dim %d)", dim);
  RS_REQUIRE((reinterpret_cast<uintptr_t>(base) & 15) == 0, "embedding base must be 16-byte aligned");
  const cuuint64_t dims[2] = {cuuint64_t(dim), cuuint64_t(rows > 0 ? rows : 1)};
  const cuuint64_t strides[1] = {cuuint64_t(dim) * es};
  // one 128-byte (SWIZZLE_128B) row per k-block: 64 bf16 or 32 fp32 elements
  const cuuint32_t box[2] = {cuuint32_t(128 / es), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, dtype == RS_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", int(r));
    return RS_ERR_CUDA;
  }
  return RS_OK;
}

int encode_kmajor_bf16_map(CUtensorMap* map, const void* base, int64_t rows, int dim, int box_rows) {
  return encode_kmajor_map(map, base, rows, dim, box_rows, RS_BF16);
}

int launch_score_topk_tc(const CUtensorMap& tmq, const CUtensorMap& tmc, const float* qn, const float* cn,
                         int64_t nq, int64_t n, int dim, int k, int64_t id_base, const SearchPlan& plan,
                         uint64_t* part, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    RS_CHECK_CUDA(cudaFuncSetAttribute(score_topk_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(SMEM_BYTES)),
                  "cudaFuncSetAttribute(score_topk_tc_kernel)");
    attr_set = true;
  }
  Params p{};
  p.qn = qn;
  p.cn = cn;
  p.nq = nq;
  p.n = n;
  p.kblocks = (dim + BK - 1) / BK;
  p.k = k;
  p.id_base = id_base;
  p.qtiles = plan.qtiles;
  p.segments = plan.segments;
  p.seg_rows = plan.seg_rows;
  p.part = part;
  score_topk_tc_kernel<<<plan.ctas, NUM_THREADS, SMEM_BYTES, st>>>(tmq, tmc, p);
  RS_CHECK_LAUNCH("score_topk_tc_kernel");
  return RS_OK;
}

}  // namespace rs
