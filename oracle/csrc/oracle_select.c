/* C restatement of the reference config path — TEST INFRASTRUCTURE / CPU
 * BASELINE ONLY (see oracle/__init__.py).
 *
 * Follows the reference algorithm step by step so it can be timed as "the
 * reference's CPU path" at C speed:
 *   enumerate_candidates   mapping.py:129-156   (grid order, method-major)
 *   plan_bytes             memory.py:164-195    (closed form, 2% buffer)
 *   best_fit_select        scheduler.py:127-156 (stable sort by bytes, reverse scan)
 *   fallback_config        scheduler.py:159-191
 *   gate_profile           profiler.py:467-486  (+ RecentSpaceWindow :138-153,
 *                                                hull_of_spaces mapping.py:180-200)
 * Queries are independent in select, so the batch is split over OpenMP
 * threads; the gate is order-dependent and runs serially.
 * Encodings match oracle/config_oracle.py.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { RERANK = 1, STUFF = 2, REDUCE = 4 };

typedef struct {
    int64_t per_token_bytes;
    int32_t chunk_size, out_budget, template_tokens, max_chunks, chunk_step, interlen_step;
} oracle_params;

static inline int64_t buffered(int64_t tokens, int64_t per_tok) {
    return (102 * tokens * per_tok + 99) / 100;
}

static inline int64_t plan_bytes(int64_t q, int m, int64_t n, int64_t il, const oracle_params* p) {
    const int64_t c = p->chunk_size, t = p->template_tokens, o = p->out_budget, pt = p->per_token_bytes;
    if (m == STUFF) return buffered(q + n * c + t + o, pt);
    if (m == RERANK) return n * buffered(q + c + t + o, pt);
    return n * buffered(q + c + t + il, pt) + buffered(q + n * il + t + o, pt);
}

typedef struct { int64_t bytes; int32_t idx; int16_t m; int16_t pad; int32_t n, il; } cand_t;

/* (bytes, grid index) ascending == Python's stable sort by bytes */
static int cmp_cand(const void* a, const void* b) {
    const cand_t* x = (const cand_t*)a;
    const cand_t* y = (const cand_t*)b;
    if (x->bytes != y->bytes) return x->bytes < y->bytes ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

static int64_t grid_size(const int32_t* s, const oracle_params* p) {
    const int64_t nn = s[2] >= s[1] ? (s[2] - s[1]) / p->chunk_step + 1 : 0;
    const int64_t ni = (s[0] & REDUCE) && s[4] >= s[3] ? (s[4] - s[3]) / p->interlen_step + 1 : 0;
    return ((s[0] & RERANK) ? nn : 0) + ((s[0] & STUFF) ? nn : 0) + nn * ni;
}

/* returns status 0 best-fit, 1 fallback, 2 must-queue */
static int select_one(const int32_t* s, int joint, int64_t q, int64_t free_b, const oracle_params* p,
                      int allow_fallback, cand_t* scratch, int32_t* cfg, int64_t* bytes) {
    int64_t g = 0;
    static const int order[3] = {RERANK, STUFF, REDUCE};
    for (int mi = 0; mi < 3; ++mi) {
        const int m = order[mi];
        if (!(s[0] & m)) continue;
        for (int64_t n = s[1]; n <= s[2]; n += p->chunk_step) {
            if (m == REDUCE) {
                for (int64_t il = s[3]; il <= s[4]; il += p->interlen_step) {
                    cand_t* c = &scratch[g];
                    c->bytes = plan_bytes(q, m, n, il, p); c->idx = (int32_t)g; c->m = (int16_t)m;
                    c->n = (int32_t)n; c->il = (int32_t)il; ++g;
                }
            } else {
                cand_t* c = &scratch[g];
                c->bytes = plan_bytes(q, m, n, 0, p); c->idx = (int32_t)g; c->m = (int16_t)m;
                c->n = (int32_t)n; c->il = 0; ++g;
            }
        }
    }
    qsort(scratch, (size_t)g, sizeof(cand_t), cmp_cand);
    for (int64_t i = g - 1; i >= 0; --i) {
        if (scratch[i].bytes <= free_b) {
            cfg[0] = scratch[i].m; cfg[1] = scratch[i].n; cfg[2] = scratch[i].il;
            *bytes = scratch[i].bytes;
            return 0;
        }
    }
    if (allow_fallback) {
        if (!joint) {
            const int64_t call = buffered(q + p->chunk_size + p->template_tokens + p->out_budget,
                                          p->per_token_bytes);
            int64_t k = free_b / call;
            if (k > p->max_chunks) k = p->max_chunks;
            if (k >= 1) {
                cfg[0] = RERANK; cfg[1] = (int32_t)k; cfg[2] = 0; *bytes = k * call;
                return 1;
            }
        } else {
            for (int64_t k = p->max_chunks; k >= 1; --k) {
                const int64_t b = plan_bytes(q, STUFF, k, 0, p);
                if (b <= free_b) {
                    cfg[0] = STUFF; cfg[1] = (int32_t)k; cfg[2] = 0; *bytes = b;
                    return 1;
                }
            }
        }
    }
    cfg[0] = cfg[1] = cfg[2] = 0; *bytes = 0;
    return 2;
}

int oracle_select_batch(int64_t n, const int32_t* spaces, const uint8_t* joint, const int32_t* qlen,
                        const int64_t* free_b, const oracle_params* p, int allow_fallback,
                        int32_t* out_cfg, int64_t* out_bytes, uint8_t* out_status, int nthreads) {
    int64_t gmax = 1;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t g = grid_size(spaces + 5 * i, p);
        if (g > gmax) gmax = g;
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int err = 0;
#pragma omp parallel
    {
        cand_t* scratch = (cand_t*)malloc((size_t)gmax * sizeof(cand_t));
        if (!scratch) {
#pragma omp atomic write
            err = 1;
        } else {
#pragma omp for schedule(static)
            for (int64_t i = 0; i < n; ++i) {
                out_status[i] = (uint8_t)select_one(spaces + 5 * i, joint[i], qlen[i], free_b[i], p,
                                                    allow_fallback, scratch, out_cfg + 3 * i,
                                                    out_bytes + i);
            }
            free(scratch);
        }
    }
    return err;
}

/* ---- gate: map_profile + window hull, strictly in order ---------------- */

static void map_profile(const int32_t* pr, int max_chunks, int32_t* s) {
    /* pr = cx, joint, pieces, s_lo, s_hi */
    const int m = !pr[1] ? RERANK : (!pr[0] ? STUFF : (STUFF | REDUCE));
    int lo = pr[2], hi = 3 * pr[2];
    lo = lo < 1 ? 1 : (lo > max_chunks ? max_chunks : lo);
    hi = hi < 1 ? 1 : (hi > max_chunks ? max_chunks : hi);
    s[0] = m; s[1] = lo; s[2] = hi;
    s[3] = (m & REDUCE) ? pr[3] : 0;
    s[4] = (m & REDUCE) ? pr[4] : 0;
}

int oracle_gate_batch(int64_t n, const int32_t* profiles, const double* conf, double threshold,
                      const int32_t* default_space, int max_chunks, int32_t* window, int32_t* win_len,
                      int32_t* out_spaces, uint8_t* out_fallback) {
    /* window: ring of 10 spaces (oldest first), *win_len entries valid on entry/exit */
    int len = *win_len;
    for (int64_t i = 0; i < n; ++i) {
        int32_t* o = out_spaces + 5 * i;
        if (conf[i] >= threshold) {
            map_profile(profiles + 5 * i, max_chunks, o);
            if (len == 10) {
                memmove(window, window + 5, 9 * 5 * sizeof(int32_t));
                len = 9;
            }
            memcpy(window + 5 * len, o, 5 * sizeof(int32_t));
            ++len;
            out_fallback[i] = 0;
        } else if (len == 0) {
            memcpy(o, default_space, 5 * sizeof(int32_t));
            out_fallback[i] = 1;
        } else {
            int m = 0, lo = window[1], hi = window[2], a = -1, b = -1;
            for (int w = 0; w < len; ++w) {
                const int32_t* s = window + 5 * w;
                m |= s[0];
                if (s[1] < lo) lo = s[1];
                if (s[2] > hi) hi = s[2];
                if (s[0] & REDUCE) {
                    if (a < 0) { a = s[3]; b = s[4]; }
                    else { if (s[3] < a) a = s[3]; if (s[4] > b) b = s[4]; }
                }
            }
            if (m & REDUCE) { if (a < 0) { a = 30; b = 200; } } else { a = 0; b = 0; }
            o[0] = m; o[1] = lo; o[2] = hi; o[3] = a; o[4] = b;
            out_fallback[i] = 1;
        }
    }
    *win_len = len;
    return 0;
}
