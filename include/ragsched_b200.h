/*
 * ragsched_b200 — C ABI of the B200-native METIS per-query hot path.
 *
 * Drop-in boundary for the data-parallel path of the reference package
 * `ragsched` (/root/reference/pkg/src/ragsched/):
 *
 *   confidence gate + Algorithm-1 pruning  profiler.py:467-486, mapping.py:106-126,
 *                                          mapping.py:180-200 (window hull)
 *   KV-memory + best-fit + fallback        memory.py:70-78, memory.py:164-195,
 *                                          scheduler.py:127-191, order of
 *                                          Scheduler._try_admit_new scheduler.py:335-378
 *   prefill/decode delay model             sim.py:42-57, sim.py:84-92 (call_latency),
 *                                          dispatch order sim.py:223-229
 *   dense chunk retrieval                  absent from the reference; the
 *                                          paper's FAISS IndexFlatL2 `index.search(q, k)`
 *
 *
 * The reference has no FFI of its own (it is pure Python; its callers resolve
 * these functions by module attribute, scheduler.py:340/:360,
 * profiler.py:534-541).  The Python package paper_2412_10543_b200 binds this
 * header with ctypes (see INTEGRATION.md for the binding a ragsched
 * maintainer would add).
 *
 * Conventions
 *  - every pointer argument documented "device" is a device pointer (cudaMalloc /
 *    torch CUDA tensor data); "host" pointers are plain host memory;
 *  - every launch takes a cudaStream_t passed as `void*` and is stream-ordered;
 *    no entry point synchronises the device except rs_index_add/… where noted;
 *  - return value 0 = RS_OK, otherwise an RS_ERR_* code; rs_last_error()
 *    returns a thread-local message for the last failure.  Nothing throws.
 *  - the library never falls back to the CPU.
 */
#ifndef RAGSCHED_B200_H
#define RAGSCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 1

enum rs_status {
  RS_OK = 0,
  RS_ERR_INVALID_ARG = 1, /* reference: ValueError                              */
  RS_ERR_CUDA = 2,
  RS_ERR_UNSUPPORTED = 3, /* e.g. no sm_100 device                              */
  RS_ERR_OOM = 4,
  RS_ERR_OVERFLOW = 5     /* int64 byte arithmetic would overflow               */
};

/* Synthesis-method bits in the reference grid order METHOD_ORDER (mapping.py:24). */
enum rs_method { RS_MAP_RERANK = 1, RS_STUFF = 2, RS_MAP_REDUCE = 4 };

/* Per-query decision (Scheduler._try_admit_new, scheduler.py:335-378). */
enum rs_select_status {
  RS_SELECT_BEST_FIT = 0,   /* best_fit_select returned a config                 */
  RS_SELECT_FALLBACK = 1,   /* best_fit_select -> None, fallback_config -> config */
  RS_SELECT_MUST_QUEUE = 2, /* both None: the query stays queued                 */
  RS_SELECT_OVERFLOW = 3    /* inputs exceed the int64 byte range (error)        */
};

/* QueryProfile (mapping.py:31-48), 16 bytes. */
typedef struct rs_profile {
  uint8_t complexity_high;
  uint8_t needs_joint_reasoning;
  uint16_t pieces_required;
  uint16_t summary_lo, summary_hi; /* summary_len_range                         */
  double confidence;
} rs_profile;

/* PrunedConfigSpace (mapping.py:51-83), 16 bytes.  interlen_lo/hi are 0 when
 * RS_MAP_REDUCE is not in `methods` (the reference's None range). */
typedef struct rs_space {
  uint16_t methods;
  uint16_t num_chunks_lo, num_chunks_hi;
  uint16_t interlen_lo, interlen_hi;
  uint16_t gate_fallback; /* GateDecision.used_fallback (profiler.py:157-163)   */
  uint32_t reserved;
} rs_space;

/* Chosen RagConfig (types.py:66-81) plus its whole-plan bytes, 16 bytes. */
typedef struct rs_config {
  int64_t kv_bytes;    /* plan_bytes(...) of the chosen config (memory.py:164)  */
  uint8_t method;      /* rs_method bit; 0 when status != BEST_FIT/FALLBACK     */
  uint8_t status;      /* rs_select_status                                      */
  uint16_t num_chunks;
  uint16_t interlen;   /* 0 == None                                             */
  uint16_t reserved;
} rs_config;

/* Scalars of best_fit_select / fallback_config (scheduler.py:127-191). */
typedef struct rs_select_params {
  int64_t per_token_bytes; /* bytes_per_kv_token(model), memory.py:70-73          */
  int32_t chunk_size;      /* DatasetMeta.chunk_size                              */
  int32_t out_budget;
  int32_t template_tokens; /* DEFAULT_TEMPLATE_TOKENS = 64 (types.py:13)          */
  int32_t max_chunks;      /* DEFAULT_MAX_CHUNKS = 35 (types.py:12)               */
  int32_t chunk_step;      /* EnumGranularity (mapping.py:86-95)                  */
  int32_t interlen_step;
  int32_t allow_fallback;  /* SchedulerParams.allow_fallback (scheduler.py:55)    */
  int32_t reserved;
} rs_select_params;

/* CostModel latency terms (sim.py:42-57). */
typedef struct rs_cost_model {
  double prefill_secs_per_token;
  double decode_secs_per_token_base;
  double batch_slowdown_per_seq;
} rs_cost_model;

/* gate_profile parameters (profiler.py:467-477). */
typedef struct rs_gate_params {
  double threshold;       /* GATE_THRESHOLD = 0.90; must be in (0, 1]          */
  rs_space default_space; /* DEFAULT_FALLBACK_SPACE = stuff [1,5]               */
  int32_t max_chunks;
  int32_t reserved;
} rs_gate_params;

/* Gate window carried across batches: RecentSpaceWindow (profiler.py:138-153). */
#define RS_WINDOW_CAPACITY 10
typedef struct rs_window {
  rs_space spaces[RS_WINDOW_CAPACITY]; /* oldest first                           */
  int32_t len;
  int32_t reserved[3];
} rs_window;

/* ---- library ------------------------------------------------------------ */
int rs_abi_version(void);
const char* rs_last_error(void);
/* 1 when `device` is an sm_100 part this library was compiled for. */
int rs_device_supported(int device);

/* ---- config path ---------------------------------------------------------
 * rs_prune_gate: gate_profile applied to a batch IN ORDER (the window couples
 * each query to the last <=10 accepted before it).  profiles/spaces_out are
 * device arrays of n; window_io is a device rs_window read as the carry-in
 * state and overwritten with the state after the batch; workspace is a device
 * buffer of rs_prune_gate_workspace_size(n) bytes.  Replaces, per query,
 * QueryProfiler.gate -> gate_profile -> map_profile | window.hull()
 * (profiler.py:534-541, :467-486). */
size_t rs_prune_gate_workspace_size(int64_t n);
int rs_prune_gate(const rs_profile* profiles, int64_t n, const rs_gate_params* params /* host */,
                  rs_window* window_io, rs_space* spaces_out, void* workspace, size_t workspace_bytes,
                  void* stream);

/* rs_select: best_fit_select then fallback_config for every query
 * independently (scheduler.py:127-191 in the order of :335-378).  spaces,
 * profiles (only .needs_joint_reasoning is read, by the fallback — the
 * reference passes `pending.profile`, scheduler.py:360-369; may be NULL when
 * allow_fallback == 0), qlen (query_token_len) and free_bytes are device
 * arrays of n.  If `cost` is non-NULL, delay_out (device, n doubles) receives
 * the chosen plan's critical-path delay under call_latency (sim.py:84-92)
 * with the sim's dispatch concurrency (sim.py:223-229) starting from
 * running_before[i] (device, may be NULL = 0). */
int rs_select(const rs_space* spaces, const rs_profile* profiles, const int32_t* qlen,
              const int64_t* free_bytes, int64_t n, const rs_select_params* params /* host */,
              const rs_cost_model* cost /* host, nullable */, const int32_t* running_before,
              double* delay_out, rs_config* out, void* stream);

/* rs_call_latency: sim.call_latency (sim.py:84-92) element-wise, bit-exact
 * IEEE double in the reference's evaluation order. */
int rs_call_latency(const int64_t* prompt_tokens, const int64_t* max_output_tokens,
                    const int64_t* concurrent_seqs, int64_t n, const rs_cost_model* cost /* host */,
                    double* out, void* stream);

/* rs_plan_bytes: memory.plan_bytes (memory.py:164-195) element-wise over
 * configs (method bit, num_chunks, interlen) and query lengths. */
int rs_plan_bytes(const uint8_t* method, const int32_t* num_chunks, const int32_t* interlen,
                  const int32_t* qlen, int64_t n, const rs_select_params* params /* host */,
                  int64_t* out, void* stream);

/* ---- per-call expansion (memory.plan_calls, memory.py:89-150) --------------
 * One LlmCall (memory.py:43-56), 24 bytes.  kind: 0 SINGLE (stuff),
 * 1 MAPPER, 2 REDUCER, 3 RERANK (CallKind order of memory.py:29-33).  A
 * map_reduce reducer depends on all mappers of its plan (the preceding
 * num_chunks calls); no other call has dependencies. */
typedef struct rs_call {
  int64_t kv_bytes;           /* buffered_bytes(prompt + max_output, per_token) */
  int32_t prompt_tokens;
  int32_t max_output_tokens;
  uint16_t index;             /* LlmCall.index */
  uint8_t kind;
  uint8_t reserved0;
  uint32_t reserved1;
} rs_call;

enum rs_plan_status {
  RS_PLAN_OK = 0,
  RS_PLAN_NONE = 1,            /* config is MustQueue / overflow: no calls      */
  RS_PLAN_INVALID_CHUNKS = 2,  /* InvalidChunkCount (memory.py:108-109)          */
  RS_PLAN_CONTEXT_OVERFLOW = 3,/* ContextOverflow (memory.py:81-86)              */
  RS_PLAN_BAD_INTERLEN = 4     /* map_reduce without positive intermediate_length */
};

/* rs_plan_calls: expand n chosen configs (rs_config from rs_select) into
 * their calls.  Pass 1 (calls == NULL): writes offsets[0..n] (exclusive scan
 * of the per-query call counts; offsets[n] = total calls) — size the calls
 * buffer from it.  Pass 2: fills calls[offsets[i] .. offsets[i+1]) and, if
 * non-NULL, total_bytes[i] (CallPlan.total_bytes) and status[i].  Queries
 * whose plan raises in the reference get 0 calls and their RS_PLAN_* status.
 * max_context_tokens is ModelSpec.max_context_tokens.  Workspace: device
 * buffer of rs_plan_calls_workspace_size(n) bytes. */
size_t rs_plan_calls_workspace_size(int64_t n);
int rs_plan_calls(const rs_config* configs, const int32_t* qlen, int64_t n,
                  const rs_select_params* params /* host */, int64_t max_context_tokens, int64_t* offsets,
                  rs_call* calls, int64_t* total_bytes, uint8_t* status, void* workspace,
                  size_t workspace_bytes, void* stream);

/* ---- cost table of every pruned candidate ---------------------------------
 * For each query i, every config of its space in enumerate_candidates order
 * (mapping.py:129-156): method, num_chunks, interlen, plan_bytes
 * (memory.py:164-195) and — if `cost` is non-NULL — the plan's critical-path
 * delay: the max of the independent calls' call_latency (sim.py:84-92) with
 * concurrency running_before[i] + j (sim.py:223-229; NULL = 0), plus the
 * reducer's latency for map_reduce.  Two passes like rs_plan_calls: out ==
 * NULL writes offsets[0..n] (exclusive scan of the grid sizes; offsets[n] =
 * total); then out[offsets[i] .. offsets[i+1]) are filled.  Returns
 * RS_ERR_OVERFLOW if some query's byte arithmetic would exceed int64. */
typedef struct rs_candidate {
  int64_t kv_bytes;
  double delay;
  uint8_t method;      /* rs_method bit */
  uint8_t reserved0;
  uint16_t num_chunks;
  uint16_t interlen;   /* 0 == None */
  uint16_t reserved1;
} rs_candidate;
size_t rs_candidate_costs_workspace_size(int64_t n);
int rs_candidate_costs(const rs_space* spaces, const int32_t* qlen, const int32_t* running_before, int64_t n,
                       const rs_select_params* params /* host */, const rs_cost_model* cost /* host, nullable */,
                       int64_t* offsets, rs_candidate* out, void* workspace, size_t workspace_bytes,
                       void* stream);

/* ---- profile ingestion (parse_profile_text, profiler.py:203-254) -----------
 * Host routine (the answers are strings on the host): parse n estimator
 * answers — UTF-8, answer i = text[offsets[i] .. offsets[i+1]) — into
 * rs_profile records with confidence[i] (NULL = 1.0), the clamped-field bits
 * and, if line_numbers is non-NULL, the line of each field (n x 4: complexity,
 * joint_reasoning, pieces, summary_range; -1 = absent).  status[i] is
 * RS_PARSE_UNPARSEABLE where the reference raises UnparseableAnswer.
 * nthreads <= 0 uses every hardware thread.  All pointers are host memory. */
enum rs_parse_status { RS_PARSE_OK = 0, RS_PARSE_UNPARSEABLE = 1 };
enum rs_clamped_bits { RS_CLAMPED_PIECES = 1, RS_CLAMPED_SUMMARY = 2 };
int rs_parse_profiles(const char* text, const int64_t* offsets, int64_t n, const double* confidence,
                      rs_profile* out, uint8_t* clamped, int32_t* line_numbers, uint8_t* status, int32_t nthreads);
/* Per-field answer confidences (_per_field_confidences, profiler.py:427-464;
 * the remote estimator's gate confidence is their minimum, :417-418): answer
 * i (text[offsets[i] .. offsets[i+1]), UTF-8) came with the tokens
 * [tok_offsets[i], tok_offsets[i+1]); token t's text is
 * tok_text[tok_text_offsets[t] .. tok_text_offsets[t+1]) (UTF-8, its length
 * counts code points) and its log-prob tok_lp[t] (tok_has_lp[t] = 0: None).
 * Each token falls on the answer line (str.splitlines(keepends=True)) its
 * starting character offset lies in; a field's confidence is exp(mean of its
 * line's log-probs) — the mean as CPython 3.12's sum() computes it
 * (Neumaier-compensated), then math.exp — or 1.0 without log-probs.  Answers
 * with no tokens or that do not parse give 1.0 for every field.  out: n x 4
 * doubles (complexity, joint_reasoning, pieces, summary_range).  Host memory;
 * nthreads <= 0 uses every hardware thread. */
int rs_field_confidences(const char* text, const int64_t* offsets, int64_t n, const int64_t* tok_offsets,
                         const char* tok_text, const int64_t* tok_text_offsets, const double* tok_lp,
                         const uint8_t* tok_has_lp, double* out, int32_t nthreads);

/* ---- FIFO admission chain (Scheduler.step, scheduler.py:397-410) ----------
 * The new-query loop of Scheduler.step: for the waiting queue in FIFO order,
 * _try_admit_new (scheduler.py:335-395) — best_fit_select against the free
 * bytes left by the admissions before it, else fallback_config (if
 * allow_fallback), else stop — and the accounting of _start_run (:281-333):
 * every independent call of the chosen plan is admitted, a map_reduce
 * reducer is deferred.  With allow_fallback == 0 the fixed-config baseline
 * path (:380-395) runs instead: the space must hold exactly one candidate,
 * whose independent calls are admitted in index order while each fits.
 * The backlog pass that precedes the loop (_admit_backlog, :257-270) stays
 * with the caller, which owns the per-call state. */
typedef struct rs_admit_params {
  int64_t capacity_bytes;     /* Scheduler.capacity_bytes                         */
  int64_t used_bytes;         /* Scheduler.used_bytes when the loop starts         */
  int64_t max_context_tokens; /* ModelSpec.max_context_tokens (plan_calls checks)  */
} rs_admit_params;

typedef struct rs_admit_info { /* per admitted queue entry, 16 bytes */
  int64_t admitted_bytes;      /* KV bytes of the calls admitted now              */
  int32_t admitted_calls;      /* independent calls admitted now (index prefix)   */
  int32_t fixed_path;          /* 1: the baseline path admitted it call by call
                                  (_start_run admit_all_independent = False)     */
} rs_admit_info;

enum rs_admit_stop {
  RS_ADMIT_DRAINED = 0,          /* every entry admitted                               */
  RS_ADMIT_BLOCKED = 1,          /* _try_admit_new -> None: the head waits              */
  RS_ADMIT_NO_PROFILE = 2,       /* SchedulingImpossible: fallback needs a profile (:356-359) */
  RS_ADMIT_IMPOSSIBLE = 3,       /* SchedulingImpossible: cannot fit an empty scheduler (:374-377, :388-391) */
  RS_ADMIT_FIXED_SPACE = 4,      /* SchedulingImpossible: baseline space not one config (:383-386) */
  RS_ADMIT_INVALID_CHUNKS = 5,   /* InvalidChunkCount from plan_calls (memory.py:108-109) */
  RS_ADMIT_CONTEXT_OVERFLOW = 6, /* ContextOverflow from plan_calls (memory.py:81-86)   */
  RS_ADMIT_BAD_INTERLEN = 7,     /* ValueError: map_reduce without intermediate_length  */
  RS_ADMIT_OVERFLOW = 8          /* inputs exceed the int64 byte range (error)          */
};

typedef struct rs_admit_result { /* device, written once per call */
  int64_t admitted;   /* entries admitted: configs/info[0 .. admitted) are valid       */
  int64_t used_bytes; /* Scheduler.used_bytes after them                               */
  int32_t stop;       /* rs_admit_stop; for != DRAINED it concerns entry `admitted`     */
  int32_t reserved;
} rs_admit_result;

/* spaces/profiles/has_profile/qlen: device arrays of the n waiting entries in
 * queue order (has_profile may be NULL = all present; profiles may be NULL
 * when allow_fallback == 0).  configs/info: device, n entries.  result:
 * device.  One launch, stream-ordered. */
int rs_admit_fifo(const rs_space* spaces, const rs_profile* profiles, const uint8_t* has_profile,
                  const int32_t* qlen, int64_t n, const rs_select_params* params /* host */,
                  const rs_admit_params* admit /* host */, rs_config* configs, rs_admit_info* info,
                  rs_admit_result* result, void* stream);

/* ---- retrieval (FAISS IndexFlatL2 semantics) ----------------
 * An index owns one corpus shard in HBM: row-major [ntotal, dim] embeddings of
 * `dtype` plus fp32 squared norms.  Search returns, per query, the k smallest
 * D = ||q||^2 + ||c||^2 - 2<q,c> (fp32 accumulate, clamped at 0), ascending,
 * ties to the lower chunk id; missing entries are I = -1, D = +inf.
 * Chunk ids are id_base + row (id_base = the shard's first global id).
 * An index handle owns its search workspace (partial lists, query norms, the
 * kernel's unit counter and shared thresholds): searches on ONE handle must be
 * ordered on one stream (or synchronised); use one handle per concurrent
 * stream.  Distinct handles are independent. */
enum rs_dtype { RS_F32 = 0, RS_BF16 = 1 };
/* RS_ALGO_TCGEN05: CTA-pair tcgen05 kernel (default: bf16, or 3xTF32 + an
 * exact fp32 re-rank for an fp32 corpus; an M = 128 pair tile for nq <= 128);
 * RS_ALGO_TCGEN05_1SM: single-CTA tcgen05 kernel (bf16); RS_ALGO_SIMT: CUDA
 * cores (also k > 40). */
enum rs_algo { RS_ALGO_AUTO = 0, RS_ALGO_SIMT = 1, RS_ALGO_TCGEN05 = 2, RS_ALGO_TCGEN05_1SM = 3 };

typedef struct rs_index rs_index;

int rs_index_create(int32_t dim, int32_t dtype, int64_t capacity, int32_t device, rs_index** out);
int rs_index_destroy(rs_index* index);
/* Append n device rows (copied; norms computed on device). */
int rs_index_add(rs_index* index, const void* embeddings, int64_t n, void* stream);
int rs_index_reset(rs_index* index);
int rs_index_ntotal(const rs_index* index, int64_t* out);
/* Device pointers of the stored corpus / norms (read-only views). */
int rs_index_data(const rs_index* index, const void** embeddings, const float** norms);
int rs_index_set_algo(rs_index* index, int32_t algo);
/* Test hook (0 in production): every CTA-pair kernel unit of query tile qt
 * starts its corpus-segment walk bias*(qt+1) tiles past the segment frontier,
 * so the out-of-id-order (wrap-around) top-k path runs deterministically. */
int rs_index_set_walk_bias(rs_index* index, int32_t bias);
/* Tuning knob of the CTA-pair kernel's schedule: corpus rows per segment
 * (rounded down to whole 256-row tiles; 0 = the planner's choice).  Shorter
 * segments keep a segment L2-resident for units that join it late, at the cost
 * of more partial lists to merge. */
int rs_index_set_segment_rows(rs_index* index, int32_t rows);
/* The CTA-pair kernel's burst merge (a query's candidates arriving as a burst
 * in one epilogue lane, e.g. a document's consecutive chunks, merged by the
 * whole warp).  mode -1 (default): automatic — the lean kernel variant runs
 * until a search reports more than RS_BURST_ON bursty flushes per
 * (32 query rows x 256-row tile), then the cooperative variant until the rate
 * falls below RS_BURST_OFF; 0: always lean; 1: always cooperative.  Both
 * variants return bit-identical results; only the timing differs.
 * rs_index_burst_merge_active reports the variant the next search will use. */
int rs_index_set_burst_merge(rs_index* index, int32_t mode);
/* Probe pass of the CTA-pair kernel (an experiment, off by default): before
 * the main launch, the same kernel scans the corpus's first rows (one 256-row
 * tile per segment, one round of units) and seeds every query's shared
 * admission bound with a valid upper bound of its final k-th distance, so the
 * main launch's per-segment lists do not start cold.  mode 0 (default): off;
 * 1: on whenever the shape allows (>= 4 probe lists per query).  Results are
 * bit-identical either way; measured slower at cfg1.
 * rs_index_last_probe_rows reports the rows the last search's probe scanned
 * (0 = no probe). */
int rs_index_set_probe(rs_index* index, int32_t mode);
int rs_index_last_probe_rows(const rs_index* index, int32_t* rows);
int rs_index_burst_merge_active(rs_index* index, int32_t* active);
/* Preallocate the search workspace for up to nq_max queries of k results. */
int rs_index_reserve(rs_index* index, int64_t nq_max, int32_t k);
/* Search: queries device [nq, dim] of the index dtype; D device [nq,k] fp32,
 * I device [nq,k] int64.  If `keep` (device, nq rs_config) is non-NULL only
 * the first keep[q].num_chunks results of a selected query are returned
 * (the join of PAPER.md:377); MustQueue queries get none. */
int rs_index_search(rs_index* index, const void* queries, int64_t nq, int32_t k, int64_t id_base,
                    const rs_config* keep, float* D, int64_t* I, void* stream);
/* Same search, but emits the per-query sorted top-k as packed keys
 * (fp32 distance bits << 32 | uint32 global id; UINT64_MAX = missing) for a
 * later cross-shard rs_merge_topk. */
int rs_index_search_keys(rs_index* index, const void* queries, int64_t nq, int32_t k,
                         int64_t id_base, uint64_t* keys, void* stream);
/* Last search's work split (segments of the corpus, query tiles, grid). */
int rs_index_last_plan(const rs_index* index, int32_t* segments, int32_t* qtiles, int32_t* ctas,
                       int32_t* algo);

/* k-way merge of sorted key lists: list l of query q starts at
 * keys[l*list_stride + q*k_in]; produces the k smallest by (distance, id).
 * If `cfg` is non-NULL only the first cfg[q].num_chunks results are kept
 * (the join "retrieve the selected number of chunks") and the
 * rest are I = -1 / D = +inf. */
int rs_merge_topk(const uint64_t* keys, int64_t nq, int32_t nlists, int32_t k_in, int64_t list_stride,
                  int32_t k, const rs_config* cfg, float* D, int64_t* I, void* stream);

/* ---- peer-memory key exchange (multi-GPU, one process per GPU) -----------
 * The exchange step of the corpus-sharded search (the
 * reference has none — it replaces the NCCL all-to-all of dist.py): every
 * rank stores the key rows of query slice r (r*nq/world .. (r+1)*nq/world)
 * straight into rank r's receive region over NVLink / NVSwitch, and rank r's
 * merge waits in-kernel on the sources' epoch flags, then merges its slice.
 * Regions are plain cudaMalloc allocations shared by CUDA IPC; the caller
 * moves the 64-byte handles between processes (e.g. torch.distributed).
 * Region layout: uint32 flags[RS_PEER_MAX] (flags[s] = last epoch source s
 * delivered) | uint32 counter | int32 error | pad to 512 B | uint64
 * keys[2 (epoch parity)][world (source)][slice_cap][k].  Epochs start at 1
 * and increase by one per exchange; a rank may run at most one exchange
 * ahead of the slowest peer's merge (guaranteed by stream order, since each
 * rank's next scatter follows its own merge, which waits for every peer). */
#define RS_PEER_MAX 64
typedef struct rs_peer_exchange {
  int32_t rank, world; /* world <= RS_PEER_MAX                                  */
  int32_t k;           /* keys per query row                                    */
  int32_t reserved;
  int64_t slice_cap;   /* >= ceil(nq / world) for every nq exchanged            */
  void* region[RS_PEER_MAX]; /* every rank's region as mapped in THIS process   */
} rs_peer_exchange;

int rs_peer_region_bytes(int32_t world, int64_t slice_cap, int32_t k, uint64_t* bytes);
/* cudaMalloc + zero-fill on `device`; ipc_handle receives 64 bytes. */
int rs_peer_alloc(uint64_t bytes, int32_t device, void** region, void* ipc_handle);
int rs_peer_open(const void* ipc_handle, int32_t device, void** region);
int rs_peer_close(void* region);
int rs_peer_free(void* region);
/* keys: device [nq, k] packed keys of this rank's shard (rs_index_search_keys);
 * stores them into the owners' regions (parity epoch & 1); the last block to
 * finish raises flags[rank] = epoch in every region (release, system scope). */
int rs_peer_scatter_keys(const rs_peer_exchange* ex, const uint64_t* keys, int64_t nq, uint32_t epoch,
                         void* stream);
/* This rank's slice of the batch of nq queries: waits until every source's
 * flag reaches `epoch` (at most timeout_ms; 0 = 60000), then the k-way merge
 * of the world lists with rs_merge_topk's contract (D/I [slice, k]).  A
 * timeout sets the region's error word (rs_peer_error) instead of hanging. */
int rs_peer_merge_topk(const rs_peer_exchange* ex, int64_t nq, uint32_t epoch, int32_t k, const rs_config* cfg,
                       float* D, int64_t* I, int32_t timeout_ms, void* stream);
/* Reads (and optionally clears) this rank's error word; synchronous. */
int rs_peer_error(const rs_peer_exchange* ex, int32_t clear, int32_t* error);
/* rs_index_search_keys fused with rs_peer_scatter_keys: the search's final
 * k-way merge stores each query's key row straight into its slice owner's
 * region and the same kernel raises the epoch flags (k must equal ex->k;
 * searches whose final step is not that merge build the rows locally and
 * scatter them).  Follow with rs_peer_merge_topk on every rank. */
int rs_index_search_scatter(rs_index* index, const void* queries, int64_t nq, int32_t k, int64_t id_base,
                            const rs_peer_exchange* ex, uint32_t epoch, void* stream);

/* Squared L2 norms of n rows of `dtype` (fp32 accumulate). */
int rs_row_norms(const void* x, int64_t n, int32_t dim, int32_t dtype, float* out, void* stream);

/* ---- measurement hooks (bench / profiling) --------------------------------
 * Kernels launched by this library since load (all entry points). */
uint64_t rs_launch_count(void);
/* When enabled, every search brackets its fused score kernel with CUDA events
 * on the launching stream; rs_index_kernel_times returns the durations (ms)
 * recorded since the previous call (the streams must be synchronised). */
int rs_index_enable_timing(rs_index* index, int32_t enable);
int rs_index_kernel_times(rs_index* index, float* ms_out, int32_t max, int32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* RAGSCHED_B200_H */
