/*
 * TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  See wf_oracle.h.
 *
 * Plain-C restatement of the reference's sequential engine.  Each function
 * cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  Pinned against tests/golden/ (vectors produced by the
 * unmodified reference via oracle/_ref); see tests/test_oracle.py.
 */
#include "wf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

/* ---- RNG: include/walkforge/rng.hpp ---------------------------------------- */

#define WFO_GAMMA 0x9E3779B97F4A7C15ULL /* rng.hpp:62 */
#define WFO_SALT 0xA3EC647659359ACDULL  /* rng.hpp:63 */
#define WFO_TRIAL_CAP (1u << 20)        /* sampler.hpp:27 */
#define WFO_NO_ALIAS 0xFFFFFFFFu        /* sampler.hpp:26 */
#define WFO_NO_EDGE UINT64_MAX          /* engine.hpp:337 */

static inline uint64_t wfo_mix(uint64_t z) { /* rng.hpp:55-59 */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t state;
} wfo_rng;

static inline wfo_rng wfo_rng_make(uint64_t seed, uint64_t stream) { /* rng.hpp:23-24 */
    wfo_rng r;
    r.state = wfo_mix(wfo_mix(seed + WFO_GAMMA) ^ wfo_mix(stream ^ WFO_SALT));
    return r;
}

static inline uint64_t wfo_next(wfo_rng* r) { /* rng.hpp:26-30 */
    r->state += WFO_GAMMA;
    return wfo_mix(r->state);
}

static inline uint32_t wfo_index(wfo_rng* r, uint32_t n) { /* rng.hpp:34-38 */
    return (uint32_t)(((unsigned __int128)wfo_next(r) * n) >> 64);
}

static inline double wfo_real(wfo_rng* r, double bound) { /* rng.hpp:42-47 */
    double u = (double)(wfo_next(r) >> 11) * 0x1.0p-53;
    double x = u * bound;
    return x < bound ? x : nextafter(bound, 0.0);
}

void wfo_rng_probe(uint64_t seed, uint64_t stream, uint32_t draws, uint64_t* out) {
    wfo_rng r = wfo_rng_make(seed, stream);
    for (uint32_t i = 0; i < draws; ++i) out[i] = wfo_next(&r);
}

void wfo_rng_index_real(uint64_t seed, uint64_t stream, uint32_t n, double bound, uint32_t* idx,
                        double* real) {
    wfo_rng r = wfo_rng_make(seed, stream);
    *idx = wfo_index(&r, n);
    *real = wfo_real(&r, bound);
}

/* ---- errors ------------------------------------------------------------------ */

typedef struct {
    int code;
    char msg[256];
} wfo_err;

static void wfo_set(wfo_err* e, int code, const char* fmt, ...) {
    if (e->code != WF_OK) return;
    e->code = code;
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(e->msg, sizeof(e->msg), fmt, ap);
    va_end(ap);
}

/* ---- graph helpers: include/walkforge/graph.hpp, src/graph.cpp -------------- */

typedef struct {
    const wfo_graph* g;
    double max_weight;   /* graph.cpp:175-178 */
    int sorted;          /* graph.cpp:164-174 */
} wfo_gview;

static inline uint32_t wfo_degree(const wfo_graph* g, uint32_t v) {
    return (uint32_t)(g->offsets[v + 1] - g->offsets[v]);
}

static int wfo_has_edge(const wfo_gview* gv, uint32_t src, uint32_t dst) { /* graph.cpp:182-188 */
    const uint32_t* ns = gv->g->neighbors + gv->g->offsets[src];
    uint64_t n = gv->g->offsets[src + 1] - gv->g->offsets[src];
    if (gv->sorted) { /* std::binary_search: lower_bound then equality */
        uint64_t lo = 0, hi = n;
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (ns[mid] < dst) lo = mid + 1; else hi = mid;
        }
        return lo < n && ns[lo] == dst;
    }
    for (uint64_t i = 0; i < n; ++i)
        if (ns[i] == dst) return 1;
    return 0;
}

/* ---- programs: include/walkforge/algorithms.hpp, program.hpp -------------- */

enum { WT_UNBIASED = 0, WT_STATIC = 1, WT_DYNAMIC = 2 }; /* program.hpp:17 */

typedef struct {
    int kind;
    int walker_type;
    int has_max_weight;   /* BoundedWeightProgram, program.hpp:55-58 */
    int prechecked;       /* PreCheckedProgram, program.hpp:81-84 */
    int preferred;        /* SamplerPreferringProgram, -1 none */
    double stop;          /* PPR */
    uint32_t length;
    int weighted;
    double inv_a, inv_b, first, bound;
    const uint32_t* schema;
    uint32_t schema_len;
} wfo_prog;

typedef struct {
    uint64_t id;
    uint32_t* path;
    uint64_t len, cap;
    wfo_rng rng;
} wfo_walker;

static int wfo_prog_init(wfo_prog* p, const wfo_gview* gv, const wf_program_desc* d, wfo_err* e) {
    memset(p, 0, sizeof(*p));
    p->kind = d->kind;
    p->preferred = -1;
    switch (d->kind) {
        case WF_PROGRAM_PPR: /* algorithms.hpp:20-37 */
            if (!(d->termination > 0.0 && d->termination <= 1.0)) {
                wfo_set(e, WF_ERR_CONFIG, "termination probability must be in (0, 1], got %f",
                        d->termination);
                return 0;
            }
            p->walker_type = WT_UNBIASED;
            p->stop = d->termination;
            p->has_max_weight = 1;
            p->bound = 1.0;
            return 1;
        case WF_PROGRAM_DEEPWALK: /* algorithms.hpp:41-67 */
            if (d->target_length < 1) {
                wfo_set(e, WF_ERR_CONFIG, "target length must be >= 1");
                return 0;
            }
            if (d->weighted && gv->g->weights == NULL) {
                wfo_set(e, WF_ERR_CONFIG, "weighted walks need a graph with edge weights");
                return 0;
            }
            p->walker_type = WT_STATIC;
            p->length = d->target_length;
            p->weighted = d->weighted != 0;
            p->bound = p->weighted ? gv->max_weight : 1.0;
            p->has_max_weight = 1;
            p->prechecked = 1;
            return 1;
        case WF_PROGRAM_NODE2VEC: /* algorithms.hpp:79-133 */
            if (!(isfinite(d->a) && d->a > 0.0)) {
                wfo_set(e, WF_ERR_CONFIG, "return parameter a must be positive and finite");
                return 0;
            }
            if (!(isfinite(d->b) && d->b > 0.0)) {
                wfo_set(e, WF_ERR_CONFIG, "in-out parameter b must be positive and finite");
                return 0;
            }
            if (d->target_length < 1) {
                wfo_set(e, WF_ERR_CONFIG, "target length must be >= 1");
                return 0;
            }
            if (d->weighted && gv->g->weights == NULL) {
                wfo_set(e, WF_ERR_CONFIG, "weighted walks need a graph with edge weights");
                return 0;
            }
            p->walker_type = WT_DYNAMIC;
            p->preferred = WF_SAMPLER_OREJ;
            p->length = d->target_length;
            p->weighted = d->weighted != 0;
            p->inv_a = 1.0 / d->a;
            p->inv_b = 1.0 / d->b;
            p->first = p->inv_a;
            if (1.0 > p->first) p->first = 1.0;
            if (p->inv_b > p->first) p->first = p->inv_b;
            p->bound = p->weighted ? p->first * gv->max_weight : p->first;
            p->has_max_weight = 1;
            p->prechecked = 1;
            return 1;
        case WF_PROGRAM_METAPATH: { /* algorithms.hpp:141-173 */
            if (gv->g->labels == NULL) {
                wfo_set(e, WF_ERR_CONFIG, "meta-path walks need a graph with edge labels");
                return 0;
            }
            if (d->schema_len == 0) {
                wfo_set(e, WF_ERR_CONFIG, "meta-path schema must be non-empty");
                return 0;
            }
            int present[256] = {0};
            for (uint64_t i = 0; i < gv->g->edge_count; ++i) present[gv->g->labels[i]] = 1;
            for (uint32_t i = 0; i < d->schema_len; ++i) {
                if (d->schema[i] > 255 || !present[d->schema[i]]) {
                    wfo_set(e, WF_ERR_CONFIG, "schema label %u does not occur in the graph",
                            d->schema[i]);
                    return 0;
                }
            }
            p->walker_type = WT_DYNAMIC;
            p->schema = d->schema;
            p->schema_len = d->schema_len;
            p->prechecked = 1;
            return 1;
        }
        case WF_PROGRAM_UNIFORM: /* algorithms.hpp:177-193 */
            if (d->target_length < 1) {
                wfo_set(e, WF_ERR_CONFIG, "target length must be >= 1");
                return 0;
            }
            p->walker_type = WT_UNBIASED;
            p->length = d->target_length;
            p->has_max_weight = 1;
            p->bound = 1.0;
            p->prechecked = 1;
            return 1;
        default:
            wfo_set(e, WF_ERR_CONFIG, "unknown program kind %d", d->kind);
            return 0;
    }
}

/* weight(Q, e); q == NULL in static contexts (program.hpp:39-42). */
static double wfo_weight(const wfo_prog* p, const wfo_gview* gv, const wfo_walker* q,
                         uint64_t edge) {
    const wfo_graph* g = gv->g;
    switch (p->kind) {
        case WF_PROGRAM_DEEPWALK: /* algorithms.hpp:49-51 */
            return p->weighted ? (double)g->weights[edge] : 1.0;
        case WF_PROGRAM_NODE2VEC: { /* algorithms.hpp:103-119 */
            double w;
            if (q->len - 1 == 0) {
                w = p->first;
            } else {
                uint32_t dst = g->neighbors[edge];
                uint32_t prev = q->path[q->len - 2];
                if (dst == prev) w = p->inv_a;
                else if (wfo_has_edge(gv, prev, dst)) w = 1.0;
                else w = p->inv_b;
            }
            return p->weighted ? w * (double)g->weights[edge] : w;
        }
        case WF_PROGRAM_METAPATH: /* algorithms.hpp:164-166 */
            return (uint32_t)g->labels[edge] == p->schema[q->len - 1] ? 1.0 : 0.0;
        default: /* PPR, Uniform: algorithms.hpp:30, 186 */
            return 1.0;
    }
}

/* update(Q, e): the only place a program draws (program.hpp:43-45). */
static int wfo_update(const wfo_prog* p, wfo_walker* q) {
    switch (p->kind) {
        case WF_PROGRAM_PPR: return wfo_real(&q->rng, 1.0) < p->stop; /* algorithms.hpp:31 */
        case WF_PROGRAM_METAPATH: return q->len - 1 >= p->schema_len; /* algorithms.hpp:167 */
        default: return q->len >= p->length;                          /* algorithms.hpp:58,120,187 */
    }
}

static int wfo_finished(const wfo_prog* p, const wfo_walker* q) { /* program.hpp:86-93 */
    if (!p->prechecked) return 0;
    if (p->kind == WF_PROGRAM_METAPATH) return q->len - 1 >= p->schema_len;
    return q->len >= p->length;
}

/* ---- samplers: include/walkforge/sampler.hpp ------------------------------ */

/* cumulative_upper_index, sampler.hpp:48-60 */
static uint32_t wfo_upper_index(const double* cum, uint32_t n, double x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = lo + (hi - lo) / 2;
        if (x < cum[mid]) hi = mid; else lo = mid + 1;
    }
    return lo;
}

typedef struct {
    double split;
    uint32_t first, second, first_dst, second_dst;
} wfo_slot; /* EngineAliasSlot, engine.hpp:22-28 */

typedef struct {
    double* scaled;
    uint32_t* small;
    uint32_t* large;
    uint64_t cap;
} wfo_vose_scratch;

static void wfo_scratch_reserve(wfo_vose_scratch* s, uint64_t n) {
    if (n <= s->cap) return;
    s->scaled = realloc(s->scaled, n * sizeof(double));
    s->small = realloc(s->small, 2 * n * sizeof(uint32_t)); /* smalls + demoted larges */
    s->large = realloc(s->large, n * sizeof(uint32_t));
    s->cap = n;
}

/* vose_build with FIFO worklists (sampler.hpp:89-120) writing decorated slots
 * (build_alias_slots, engine.hpp:118-127).  dst == NULL writes undecorated
 * slots with second = WFO_NO_ALIAS for leftovers (alias_init). */
static void wfo_vose(const double* w, uint32_t n, double sum, const uint32_t* dst,
                     wfo_slot* out, wfo_vose_scratch* s) {
    wfo_scratch_reserve(s, n);
    uint64_t ns = 0, nl = 0;
    for (uint32_t i = 0; i < n; ++i) {
        s->scaled[i] = w[i] * n / sum;
        if (s->scaled[i] < 1.0) s->small[ns++] = i; else s->large[nl++] = i;
    }
    uint64_t sh = 0, lh = 0;
    while (sh < ns && lh < nl) {
        uint32_t sm = s->small[sh++];
        uint32_t lg = s->large[lh];
        out[sm].split = s->scaled[sm];
        out[sm].first = sm;
        out[sm].second = lg;
        s->scaled[lg] -= 1.0 - s->scaled[sm];
        if (s->scaled[lg] < 1.0) {
            lh++;
            s->small[ns++] = lg;
        }
    }
    for (uint64_t i = sh; i < ns; ++i) {
        uint32_t k = s->small[i];
        out[k].split = 1.0; out[k].first = k; out[k].second = WFO_NO_ALIAS;
    }
    for (uint64_t i = lh; i < nl; ++i) {
        uint32_t k = s->large[i];
        out[k].split = 1.0; out[k].first = k; out[k].second = WFO_NO_ALIAS;
    }
    if (dst) {
        for (uint32_t i = 0; i < n; ++i) {
            if (out[i].second == WFO_NO_ALIAS) out[i].second = out[i].first;
            out[i].first_dst = dst[out[i].first];
            out[i].second_dst = dst[out[i].second];
        }
    }
}

/* checked_weight_sum, sampler.cpp:28-43 */
static int wfo_checked_sum(const double* w, uint32_t n, double* sum, wfo_err* e) {
    if (n == 0) { wfo_set(e, WF_ERR_DISTRIBUTION, "empty weight sequence"); return 0; }
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) {
        if (!isfinite(w[i]) || w[i] < 0.0) {
            wfo_set(e, WF_ERR_DISTRIBUTION, "weights must be finite and non-negative");
            return 0;
        }
        s += w[i];
    }
    if (!(s > 0.0)) { wfo_set(e, WF_ERR_DISTRIBUTION, "weights sum to zero"); return 0; }
    *sum = s;
    return 1;
}

int wfo_alias_init(const double* weights, uint32_t n, double* split, uint32_t* first,
                   uint32_t* second, char* err, int errlen) { /* sampler.cpp:57-69 */
    wfo_err e = {WF_OK, {0}};
    double sum;
    if (!wfo_checked_sum(weights, n, &sum, &e)) {
        if (err) snprintf(err, errlen, "%s", e.msg);
        return e.code;
    }
    wfo_slot* slots = malloc((size_t)n * sizeof(wfo_slot));
    wfo_vose_scratch s = {0};
    wfo_vose(weights, n, sum, NULL, slots, &s);
    for (uint32_t i = 0; i < n; ++i) {
        split[i] = slots[i].split; first[i] = slots[i].first; second[i] = slots[i].second;
    }
    free(slots); free(s.scaled); free(s.small); free(s.large);
    return WF_OK;
}

/* ---- static tables: preprocess_static, engine.hpp:190-251 ------------------- */

typedef struct {
    int kind;
    wfo_slot* alias;     /* E */
    double* its;         /* E */
    double* rej_p_star;  /* V */
    uint8_t* exhausted;  /* V */
} wfo_tables;

static int wfo_check_weight(double w, wfo_err* e) { /* engine.hpp:97-101 */
    if (!isfinite(w) || w < 0.0) {
        wfo_set(e, WF_ERR_CONTRACT, "program emitted a weight that is negative or not finite");
        return 0;
    }
    return 1;
}

static int wfo_preprocess(const wfo_prog* p, const wfo_gview* gv, int kind, wfo_tables* t,
                          wfo_err* e) {
    const wfo_graph* g = gv->g;
    memset(t, 0, sizeof(*t));
    t->kind = kind;
    if (p->walker_type == WT_DYNAMIC) {
        wfo_set(e, WF_ERR_CONFIG,
                "cannot preprocess a dynamic program; its weights depend on the walker");
        return 0;
    }
    if (kind != WF_SAMPLER_ITS && kind != WF_SAMPLER_ALIAS && kind != WF_SAMPLER_REJ) {
        wfo_set(e, WF_ERR_CONFIG, "static tables exist for ITS, ALIAS, and REJ only");
        return 0;
    }
    t->exhausted = calloc(g->vertex_count, 1);
    if (kind == WF_SAMPLER_ITS) t->its = calloc(g->edge_count ? g->edge_count : 1, sizeof(double));
    else if (kind == WF_SAMPLER_ALIAS) t->alias = calloc(g->edge_count ? g->edge_count : 1, sizeof(wfo_slot));
    else t->rej_p_star = calloc(g->vertex_count, sizeof(double));
    double* w = NULL;
    uint64_t wcap = 0;
    wfo_vose_scratch s = {0};
    for (uint32_t v = 0; v < g->vertex_count; ++v) {
        uint64_t base = g->offsets[v];
        uint32_t d = wfo_degree(g, v);
        if (d == 0) continue;
        if (d > wcap) { wcap = d; w = realloc(w, wcap * sizeof(double)); }
        double sum = 0.0, mx = 0.0;
        for (uint32_t i = 0; i < d; ++i) {
            double x = wfo_weight(p, gv, NULL, base + i);
            if (!wfo_check_weight(x, e)) { free(w); return 0; }
            w[i] = x;
            sum += x;
            if (x > mx) mx = x;
        }
        if (!(sum > 0.0)) { t->exhausted[v] = 1; continue; }
        if (kind == WF_SAMPLER_ITS) {
            double run = 0.0;
            for (uint32_t i = 0; i < d; ++i) { run += w[i]; t->its[base + i] = run; }
        } else if (kind == WF_SAMPLER_ALIAS) {
            wfo_vose(w, d, sum, g->neighbors + base, t->alias + base, &s);
        } else {
            t->rej_p_star[v] = mx;
        }
    }
    free(w); free(s.scaled); free(s.small); free(s.large);
    return 1;
}

static void wfo_tables_free(wfo_tables* t) {
    free(t->alias); free(t->its); free(t->rej_p_star); free(t->exhausted);
}

/* ---- run resolution: resolve_flow / ResolvedRun, engine.hpp:255-294 -------- */

enum { FLOW_DIRECT = 0, FLOW_TABLES = 1, FLOW_GATHERED = 2 };

typedef struct {
    wfo_prog prog;
    wfo_gview gv;
    int kind, flow;
    double orej_bound;
    uint32_t trial_cap;
    wfo_tables tables;
} wfo_run_ctx;

static const char* wfo_type_name(int t) {
    return t == WT_UNBIASED ? "unbiased" : (t == WT_STATIC ? "static" : "dynamic");
}

static int wfo_resolve(wfo_run_ctx* r, const wf_exec_options* o, wfo_err* e) {
    int kind = (o && o->sampler >= 0) ? o->sampler
               : (r->prog.preferred >= 0 ? r->prog.preferred
                  : (r->prog.walker_type == WT_UNBIASED ? WF_SAMPLER_NAIVE
                     : r->prog.walker_type == WT_STATIC ? WF_SAMPLER_ALIAS : WF_SAMPLER_ITS));
    int use_tables = o ? o->use_static_tables != 0 : 1;
    r->kind = kind;
    if (kind == WF_SAMPLER_NAIVE) {
        if (r->prog.walker_type != WT_UNBIASED) {
            wfo_set(e, WF_ERR_CONFIG, "NAIVE assumes a uniform distribution; the program is %s",
                    wfo_type_name(r->prog.walker_type));
            return 0;
        }
        r->flow = FLOW_DIRECT;
    } else if (kind == WF_SAMPLER_OREJ) {
        r->flow = FLOW_DIRECT;
    } else if (r->prog.walker_type == WT_DYNAMIC) {
        r->flow = FLOW_GATHERED;
    } else {
        r->flow = use_tables ? FLOW_TABLES : FLOW_GATHERED;
    }
    r->trial_cap = (o && o->rej_trial_cap) ? o->rej_trial_cap : WFO_TRIAL_CAP;
    if (kind == WF_SAMPLER_OREJ) { /* resolve_orej_bound, engine.hpp:103-114 */
        if (!r->prog.has_max_weight) {
            wfo_set(e, WF_ERR_CONFIG, "O-REJ needs a program with max_weight()");
            return 0;
        }
        double b = r->prog.bound;
        if (!isfinite(b) || b <= 0.0) {
            wfo_set(e, WF_ERR_CONTRACT, "max_weight() must be positive and finite");
            return 0;
        }
        r->orej_bound = b;
    }
    if (r->flow == FLOW_TABLES) {
        if (!wfo_preprocess(&r->prog, &r->gv, kind, &r->tables, e)) return 0;
    }
    return 1;
}

/* ---- the step: StepDriver::step, engine.hpp:342-426 ----------------------- */

typedef struct {
    double* reals;      /* ITS cumulative / REJ raw weights */
    double* weights;    /* ALIAS gather temp */
    wfo_slot* alias;
    uint64_t cap;
    wfo_vose_scratch vs;
} wfo_tctx; /* TransitionContext, engine.hpp:46-55 */

static void wfo_tctx_reserve(wfo_tctx* c, uint64_t n) {
    if (n <= c->cap) return;
    c->reals = realloc(c->reals, n * sizeof(double));
    c->weights = realloc(c->weights, n * sizeof(double));
    c->alias = realloc(c->alias, n * sizeof(wfo_slot));
    c->cap = n;
}

static void wfo_tctx_free(wfo_tctx* c) {
    free(c->reals); free(c->weights); free(c->alias);
    free(c->vs.scaled); free(c->vs.small); free(c->vs.large);
}

/* rej_generate, sampler.hpp:152-164; mode 0: O-REJ lazy program weight
 * (checked), 1: tables REJ weight(null, e), 2: gathered weights array. */
static uint32_t wfo_rej(const wfo_run_ctx* r, wfo_walker* q, uint64_t base, uint32_t d,
                        double p_star, int mode, const double* gathered, wfo_err* e) {
    for (uint32_t trial = 1; trial <= r->trial_cap; ++trial) {
        uint32_t x = wfo_index(&q->rng, d);
        double y = wfo_real(&q->rng, p_star);
        double w;
        if (mode == 0) {
            w = wfo_weight(&r->prog, &r->gv, q, base + x);
            if (!wfo_check_weight(w, e)) return 0;
        } else if (mode == 1) {
            w = wfo_weight(&r->prog, &r->gv, NULL, base + x);
        } else {
            w = gathered[x];
        }
        if (y < w) return x;
    }
    wfo_set(e, WF_ERR_REJECTION_CAP,
            "rejection sampling exceeded %u trials; asserted bound does not match the weights",
            r->trial_cap);
    return 0;
}

/* gather, engine.hpp:134-184 */
static int wfo_gather(const wfo_run_ctx* r, const wfo_walker* q, wfo_tctx* c, double* p_star,
                      wfo_err* e) {
    const wfo_graph* g = r->gv.g;
    uint32_t v = q->path[q->len - 1];
    uint64_t base = g->offsets[v];
    uint32_t d = wfo_degree(g, v);
    if (d == 0) return 0;
    wfo_tctx_reserve(c, d);
    double* w = r->kind == WF_SAMPLER_ALIAS ? c->weights : c->reals;
    double sum = 0.0, mx = 0.0;
    for (uint32_t i = 0; i < d; ++i) {
        double x = wfo_weight(&r->prog, &r->gv, q, base + i);
        if (!wfo_check_weight(x, e)) return 0;
        w[i] = x;
        sum += x;
        if (x > mx) mx = x;
    }
    if (!(sum > 0.0)) return 0;
    if (r->kind == WF_SAMPLER_ITS) {
        double run = 0.0;
        for (uint32_t i = 0; i < d; ++i) { run += w[i]; c->reals[i] = run; }
    } else if (r->kind == WF_SAMPLER_ALIAS) {
        wfo_vose(w, d, sum, g->neighbors + base, c->alias, &c->vs);
    } else if (r->kind == WF_SAMPLER_REJ) {
        *p_star = mx;
    } else {
        wfo_set(e, WF_ERR_CONFIG, "gather feeds ITS, ALIAS, or REJ");
        return 0;
    }
    return 1;
}

static uint64_t wfo_step(const wfo_run_ctx* r, wfo_walker* q, wfo_tctx* c, wfo_err* e) {
    const wfo_graph* g = r->gv.g;
    uint32_t v = q->path[q->len - 1];
    uint64_t base = g->offsets[v];
    uint32_t d = wfo_degree(g, v);
    uint32_t pick = 0;
    if (r->flow == FLOW_DIRECT) {
        if (d == 0) return WFO_NO_EDGE;
        if (r->kind == WF_SAMPLER_NAIVE) pick = wfo_index(&q->rng, d);
        else pick = wfo_rej(r, q, base, d, r->orej_bound, 0, NULL, e);
    } else if (r->flow == FLOW_TABLES) {
        if (d == 0 || r->tables.exhausted[v]) return WFO_NO_EDGE;
        if (r->kind == WF_SAMPLER_ITS) {
            const double* cum = r->tables.its + base;
            double x = wfo_real(&q->rng, cum[d - 1]);
            pick = wfo_upper_index(cum, d, x);
        } else if (r->kind == WF_SAMPLER_ALIAS) {
            const wfo_slot* s = &r->tables.alias[base + wfo_index(&q->rng, d)];
            pick = wfo_real(&q->rng, 1.0) < s->split ? s->first : s->second;
        } else {
            pick = wfo_rej(r, q, base, d, r->tables.rej_p_star[v], 1, NULL, e);
        }
    } else {
        double p_star = 0.0;
        if (!wfo_gather(r, q, c, &p_star, e)) return WFO_NO_EDGE;
        if (r->kind == WF_SAMPLER_ITS) {
            double x = wfo_real(&q->rng, c->reals[d - 1]);
            pick = wfo_upper_index(c->reals, d, x);
        } else if (r->kind == WF_SAMPLER_ALIAS) {
            const wfo_slot* s = &c->alias[wfo_index(&q->rng, d)];
            pick = wfo_real(&q->rng, 1.0) < s->split ? s->first : s->second;
        } else {
            pick = wfo_rej(r, q, base, d, p_star, 2, c->reals, e);
        }
    }
    if (e->code != WF_OK) return WFO_NO_EDGE;
    uint64_t edge = base + pick;
    if (q->len == q->cap) {
        q->cap = q->cap ? 2 * q->cap : 16;
        q->path = realloc(q->path, q->cap * sizeof(uint32_t));
    }
    q->path[q->len++] = g->neighbors[edge];
    return edge;
}

/* ---- the run: run_sequential, engine.hpp:440-504 ----------------------------- */

typedef struct {
    const wfo_run_ctx* r;
    const wf_query_spec* spec;
    const uint64_t* qids;
    uint64_t lo, hi;
    uint64_t seed;
    int discard;
    /* outputs */
    uint64_t* lens;
    uint8_t* status;
    uint32_t* verts;
    uint64_t nverts, capverts;
    uint64_t steps;
    wfo_err err;
} wfo_worker;

static uint32_t wfo_source_at(const wf_query_spec* s, uint64_t qid) { /* walker.hpp:70-77 */
    switch (s->mode) {
        case WF_QUERY_ONE_PER_VERTEX: return (uint32_t)qid;
        case WF_QUERY_FROM_SOURCE: return s->source;
        default: return s->sources[qid];
    }
}

static void* wfo_worker_main(void* arg) {
    wfo_worker* w = arg;
    wfo_tctx c = {0};
    wfo_walker q = {0};
    for (uint64_t i = w->lo; i < w->hi; ++i) {
        uint64_t qid = w->qids ? w->qids[i] : i;
        q.id = qid;
        q.rng = wfo_rng_make(w->seed, qid);
        q.len = 0;
        if (q.cap == 0) { q.cap = 16; q.path = malloc(q.cap * sizeof(uint32_t)); }
        q.path[q.len++] = wfo_source_at(w->spec, qid);
        int st = WF_WALK_DEAD_END;
        if (wfo_finished(&w->r->prog, &q)) {
            st = WF_WALK_COMPLETE;
        } else {
            for (;;) {
                uint64_t edge = wfo_step(w->r, &q, &c, &w->err);
                if (w->err.code != WF_OK) goto done;
                if (edge == WFO_NO_EDGE) break;
                w->steps += 1;
                if (wfo_update(&w->r->prog, &q)) { st = WF_WALK_COMPLETE; break; }
            }
        }
        if (!w->discard) {
            w->lens[i - w->lo] = q.len;
            w->status[i - w->lo] = (uint8_t)st;
            if (w->nverts + q.len > w->capverts) {
                w->capverts = 2 * (w->nverts + q.len) + 1024;
                w->verts = realloc(w->verts, w->capverts * sizeof(uint32_t));
            }
            memcpy(w->verts + w->nverts, q.path, q.len * sizeof(uint32_t));
            w->nverts += q.len;
        }
    }
done:
    free(q.path);
    wfo_tctx_free(&c);
    return NULL;
}

static double wfo_now(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + ts.tv_nsec * 1e-9;
}

static void wfo_gview_init(wfo_gview* gv, const wfo_graph* g) { /* finalize_stats, graph.cpp:161-180 */
    gv->g = g;
    gv->sorted = 1;
    for (uint32_t v = 0; v < g->vertex_count && gv->sorted; ++v)
        for (uint64_t e = g->offsets[v] + 1; e < g->offsets[v + 1]; ++e)
            if (g->neighbors[e - 1] > g->neighbors[e]) { gv->sorted = 0; break; }
    gv->max_weight = 0.0;
    if (g->weights)
        for (uint64_t e = 0; e < g->edge_count; ++e)
            if ((double)g->weights[e] > gv->max_weight) gv->max_weight = g->weights[e];
}

static int wfo_finish_err(const wfo_err* e, char* err, int errlen) {
    if (err && errlen > 0) snprintf(err, errlen, "%s", e->msg);
    return e->code;
}

int wfo_run(const wfo_graph* g, const wf_program_desc* prog, const wf_query_spec* spec,
            const wf_exec_options* opts, const uint64_t* qids, uint64_t n_qids, int threads,
            int discard, wfo_result* out, char* err, int errlen) {
    wfo_err e = {WF_OK, {0}};
    memset(out, 0, sizeof(*out));
    /* QuerySpec::validate, walker.cpp:89-109 */
    uint64_t total = spec->mode == WF_QUERY_ONE_PER_VERTEX ? g->vertex_count : spec->count;
    if (spec->mode == WF_QUERY_FROM_SOURCE && spec->source >= g->vertex_count) {
        wfo_set(&e, WF_ERR_CONFIG, "query source %u is not a vertex (V=%u)", spec->source,
                g->vertex_count);
        return wfo_finish_err(&e, err, errlen);
    }
    if (spec->mode == WF_QUERY_FROM_LIST) {
        for (uint64_t i = 0; i < spec->count; ++i) {
            if (spec->sources[i] >= g->vertex_count) {
                wfo_set(&e, WF_ERR_CONFIG, "query source %u is not a vertex (V=%u)",
                        spec->sources[i], g->vertex_count);
                return wfo_finish_err(&e, err, errlen);
            }
        }
    }
    wfo_run_ctx r;
    memset(&r, 0, sizeof(r));
    wfo_gview_init(&r.gv, g);
    if (!wfo_prog_init(&r.prog, &r.gv, prog, &e)) return wfo_finish_err(&e, err, errlen);
    double t0 = wfo_now();
    if (!wfo_resolve(&r, opts, &e)) {
        wfo_tables_free(&r.tables);
        return wfo_finish_err(&e, err, errlen);
    }
    out->preprocess_seconds = wfo_now() - t0;
    uint64_t n = qids ? n_qids : total;
    if (threads < 1) threads = 1;
    wfo_worker* ws = calloc(threads, sizeof(wfo_worker));
    pthread_t* th = calloc(threads, sizeof(pthread_t));
    uint64_t* lens = discard ? NULL : malloc((n ? n : 1) * sizeof(uint64_t));
    uint8_t* status = discard ? NULL : malloc(n ? n : 1);
    double t1 = wfo_now();
    for (int w = 0; w < threads; ++w) { /* worker_range, engine.hpp:296-298 */
        ws[w].r = &r;
        ws[w].spec = spec;
        ws[w].qids = qids;
        ws[w].lo = n * (uint64_t)w / threads;
        ws[w].hi = n * (uint64_t)(w + 1) / threads;
        ws[w].seed = opts ? opts->seed : 0;
        ws[w].discard = discard;
        ws[w].lens = lens ? lens + ws[w].lo : NULL;
        ws[w].status = status ? status + ws[w].lo : NULL;
        if (threads > 1) pthread_create(&th[w], NULL, wfo_worker_main, &ws[w]);
        else wfo_worker_main(&ws[w]);
    }
    if (threads > 1)
        for (int w = 0; w < threads; ++w) pthread_join(th[w], NULL);
    out->exec_seconds = wfo_now() - t1;
    for (int w = 0; w < threads && e.code == WF_OK; ++w)
        if (ws[w].err.code != WF_OK) e = ws[w].err;
    if (e.code == WF_OK) {
        out->n = n;
        for (int w = 0; w < threads; ++w) out->total_steps += ws[w].steps;
        if (!discard) {
            out->offsets = malloc((n + 1) * sizeof(uint64_t));
            uint64_t pos = 0;
            for (uint64_t i = 0; i < n; ++i) { out->offsets[i] = pos; pos += lens[i]; }
            out->offsets[n] = pos;
            out->vertices = malloc((pos ? pos : 1) * sizeof(uint32_t));
            for (int w = 0; w < threads; ++w)
                memcpy(out->vertices + out->offsets[ws[w].lo], ws[w].verts,
                       ws[w].nverts * sizeof(uint32_t));
            out->status = status;
            status = NULL;
        }
    }
    for (int w = 0; w < threads; ++w) free(ws[w].verts);
    free(ws); free(th); free(lens); free(status);
    wfo_tables_free(&r.tables);
    return wfo_finish_err(&e, err, errlen);
}

void wfo_result_free(wfo_result* r) {
    free(r->offsets); free(r->vertices); free(r->status);
    memset(r, 0, sizeof(*r));
}

int wfo_static_tables(const wfo_graph* g, const wf_program_desc* prog, int sampler,
                      double* alias_split, uint32_t* alias_first_dst, uint32_t* alias_second_dst,
                      double* its_cumulative, double* rej_p_star, uint8_t* exhausted, char* err,
                      int errlen) {
    wfo_err e = {WF_OK, {0}};
    wfo_gview gv;
    wfo_gview_init(&gv, g);
    wfo_prog p;
    if (!wfo_prog_init(&p, &gv, prog, &e)) return wfo_finish_err(&e, err, errlen);
    wfo_tables t;
    if (!wfo_preprocess(&p, &gv, sampler, &t, &e)) {
        wfo_tables_free(&t);
        return wfo_finish_err(&e, err, errlen);
    }
    if (exhausted) memcpy(exhausted, t.exhausted, g->vertex_count);
    for (uint64_t i = 0; t.alias && i < g->edge_count; ++i) {
        if (alias_split) alias_split[i] = t.alias[i].split;
        if (alias_first_dst) alias_first_dst[i] = t.alias[i].first_dst;
        if (alias_second_dst) alias_second_dst[i] = t.alias[i].second_dst;
    }
    if (its_cumulative && t.its) memcpy(its_cumulative, t.its, g->edge_count * sizeof(double));
    if (rej_p_star && t.rej_p_star) memcpy(rej_p_star, t.rej_p_star, g->vertex_count * sizeof(double));
    wfo_tables_free(&t);
    return WF_OK;
}

/* ---- synthetic R-MAT CSR, multithreaded --------------------- */

#define WFO_RMAT_SALT 0x524D4154454447ULL
#define WFO_WEIGHT_SALT 0x57464757454947ULL /* graph.cpp:26 */
#define WFO_LABEL_SALT 0x5746474C41424CULL  /* graph.cpp:27 */

typedef struct {
    uint64_t premix;
    uint32_t scale, t1, t2, t3;
} wfo_rmat_gen;

static inline void wfo_rmat_edge(const wfo_rmat_gen* g, uint64_t i, uint32_t* s, uint32_t* d) {
    wfo_rng r;
    r.state = wfo_mix(g->premix ^ wfo_mix(i ^ WFO_SALT));
    uint32_t ss = 0, dd = 0;
    for (uint32_t lvl = 0; lvl < g->scale; lvl += 2) {
        uint64_t x = wfo_next(&r);
        for (int h = 0; h < 2; ++h) {
            uint32_t l = lvl + h;
            if (l >= g->scale) break;
            uint32_t u = h == 0 ? (uint32_t)(x >> 32) : (uint32_t)x;
            uint32_t bit = 1u << (g->scale - 1 - l);
            if (u >= g->t1) {
                if (u < g->t2) dd |= bit;
                else if (u < g->t3) ss |= bit;
                else { ss |= bit; dd |= bit; }
            }
        }
    }
    *s = ss;
    *d = dd;
}

typedef struct {
    const wfo_rmat_gen* gen;
    uint64_t lo, hi;
    uint32_t* deg;           /* pass 0 */
    uint64_t* cursor;        /* pass 1 */
    /* R-MAT hubs are the low ids: their counts and cursors are per thread
     * (no shared cache lines), the rest use atomics */
    uint32_t hot;            /* vertices [0, hot) */
    uint32_t* hot_deg;       /* pass 0: this thread's counts */
    uint64_t* hot_cur;       /* pass 1: this thread's cursors */
    uint32_t* raw;           /* pass 1 */
    /* pass 2/3: vertex range */
    uint32_t vlo, vhi;
    const uint64_t* off0;
    uint32_t* ndeg;
    const uint64_t* off1;
    uint32_t* out;
    int pass;
    /* attributes */
    uint64_t elo, ehi, wmix, lmix;
    float* w;
    uint8_t* lab;
    uint32_t label_count;
} wfo_rmat_job;

/* Sorts a neighbour segment: insertion sort when short, else an LSD radix
 * sort with 11-bit digits through `tmp` (same result as any sort; the order of
 * equal ids does not matter because duplicates are merged right after). */
static void wfo_sort_u32(uint32_t* x, uint64_t n, uint32_t** tmp, uint64_t* tmp_n) {
    if (n <= 32) {
        for (uint64_t i = 1; i < n; ++i) {
            uint32_t v = x[i];
            uint64_t k = i;
            while (k > 0 && x[k - 1] > v) { x[k] = x[k - 1]; --k; }
            x[k] = v;
        }
        return;
    }
    if (*tmp_n < n) {
        free(*tmp);
        *tmp = malloc(n * sizeof(uint32_t));
        *tmp_n = n;
    }
    uint32_t* a = x;
    uint32_t* b = *tmp;
    for (int shift = 0; shift < 32; shift += 11) {
        uint64_t cnt[2049] = {0};
        for (uint64_t i = 0; i < n; ++i) ++cnt[((a[i] >> shift) & 2047) + 1];
        if (cnt[((a[0] >> shift) & 2047) + 1] == n) continue; /* one digit value: already ordered */
        for (int d = 0; d < 2048; ++d) cnt[d + 1] += cnt[d];
        for (uint64_t i = 0; i < n; ++i) b[cnt[(a[i] >> shift) & 2047]++] = a[i];
        uint32_t* t = a;
        a = b;
        b = t;
    }
    if (a != x) memcpy(x, a, n * sizeof(uint32_t));
}

static void* wfo_rmat_worker(void* arg) {
    wfo_rmat_job* j = arg;
    if (j->pass == 0 || j->pass == 1) {
        for (uint64_t i = j->lo; i < j->hi; ++i) {
            uint32_t s, d;
            wfo_rmat_edge(j->gen, i, &s, &d);
            if (s == d) continue;
            if (j->pass == 0) {
                if (s < j->hot) ++j->hot_deg[s];
                else __atomic_fetch_add(&j->deg[s], 1u, __ATOMIC_RELAXED);
                if (d < j->hot) ++j->hot_deg[d];
                else __atomic_fetch_add(&j->deg[d], 1u, __ATOMIC_RELAXED);
            } else {
                j->raw[s < j->hot ? j->hot_cur[s]++ : __atomic_fetch_add(&j->cursor[s], 1ull, __ATOMIC_RELAXED)] = d;
                j->raw[d < j->hot ? j->hot_cur[d]++ : __atomic_fetch_add(&j->cursor[d], 1ull, __ATOMIC_RELAXED)] = s;
            }
        }
    } else if (j->pass == 2) { /* sort + count distinct */
        uint32_t* tmp = NULL;
        uint64_t tmp_n = 0;
        for (uint32_t v = j->vlo; v < j->vhi; ++v) {
            uint64_t a = j->off0[v], n = j->off0[v + 1] - a;
            if (n > 1) wfo_sort_u32(j->raw + a, n, &tmp, &tmp_n);
            uint32_t c = 0;
            for (uint64_t e = 0; e < n; ++e) c += (e == 0 || j->raw[a + e] != j->raw[a + e - 1]);
            j->ndeg[v] = c;
        }
        free(tmp);
    } else if (j->pass == 3) { /* compact */
        for (uint32_t v = j->vlo; v < j->vhi; ++v) {
            uint64_t a = j->off0[v], n = j->off0[v + 1] - a, w = j->off1[v];
            for (uint64_t e = 0; e < n; ++e)
                if (e == 0 || j->raw[a + e] != j->raw[a + e - 1]) j->out[w++] = j->raw[a + e];
        }
    } else { /* attributes: synthetic_weight / synthetic_label, graph.cpp:279-287 */
        for (uint64_t e = j->elo; e < j->ehi; ++e) {
            if (j->w) {
                wfo_rng r;
                r.state = wfo_mix(j->wmix ^ wfo_mix(e ^ WFO_SALT));
                j->w[e] = (float)(1.0 + wfo_real(&r, 4.0));
            }
            if (j->lab) {
                wfo_rng r;
                r.state = wfo_mix(j->lmix ^ wfo_mix(e ^ WFO_SALT));
                j->lab[e] = (uint8_t)wfo_index(&r, j->label_count);
            }
        }
    }
    return NULL;
}

static void wfo_run_jobs(wfo_rmat_job* jobs, int n) {
    pthread_t* th = calloc(n, sizeof(pthread_t));
    for (int i = 0; i < n; ++i) pthread_create(&th[i], NULL, wfo_rmat_worker, &jobs[i]);
    for (int i = 0; i < n; ++i) pthread_join(th[i], NULL);
    free(th);
}

static uint32_t wfo_thr32(double x) {
    double t = floor(x * 4294967296.0);
    return t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t;
}

int wfo_rmat_csr(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                 int weighted, uint32_t label_count, int threads, wfo_csr* out) {
    memset(out, 0, sizeof(*out));
    if (scale < 1 || scale > 31 || edge_factor < 1) return WF_ERR_CONFIG;
    if (threads <= 0) threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    wfo_rmat_gen gen = {wfo_mix((seed ^ WFO_RMAT_SALT) + WFO_GAMMA), scale, wfo_thr32(a),
                        wfo_thr32(a + b), wfo_thr32(a + b + c)};
    const uint32_t V = 1u << scale;
    const uint64_t n = (uint64_t)edge_factor << scale;
    uint32_t* deg = calloc(V, sizeof(uint32_t));
    wfo_rmat_job* jobs = calloc(threads, sizeof(wfo_rmat_job));
    const uint32_t hot = V < (1u << 18) ? V : (1u << 18);
    for (int t = 0; t < threads; ++t) {
        jobs[t].gen = &gen;
        jobs[t].lo = n * t / threads;
        jobs[t].hi = n * (t + 1) / threads;
        jobs[t].deg = deg;
        jobs[t].hot = hot;
        jobs[t].hot_deg = calloc(hot, sizeof(uint32_t));
        jobs[t].hot_cur = malloc(hot * sizeof(uint64_t));
        jobs[t].pass = 0;
    }
    wfo_run_jobs(jobs, threads);
    for (int t = 0; t < threads; ++t)
        for (uint32_t v = 0; v < hot; ++v) deg[v] += jobs[t].hot_deg[v];
    uint64_t* off0 = malloc((V + 1ull) * sizeof(uint64_t));
    off0[0] = 0;
    for (uint32_t v = 0; v < V; ++v) off0[v + 1] = off0[v] + deg[v];
    free(deg);
    uint64_t E0 = off0[V];
    uint32_t* raw = malloc((E0 ? E0 : 1) * sizeof(uint32_t));
    uint64_t* cursor = malloc(V * sizeof(uint64_t));
    memcpy(cursor, off0, V * sizeof(uint64_t));
    /* each thread's hot cursors start at its own slice of the segment */
    for (uint32_t v = 0; v < hot; ++v) {
        uint64_t at = off0[v];
        for (int t = 0; t < threads; ++t) {
            jobs[t].hot_cur[v] = at;
            at += jobs[t].hot_deg[v];
        }
    }
    for (int t = 0; t < threads; ++t) {
        jobs[t].cursor = cursor;
        jobs[t].raw = raw;
        jobs[t].pass = 1;
    }
    wfo_run_jobs(jobs, threads);
    free(cursor);
    for (int t = 0; t < threads; ++t) {
        free(jobs[t].hot_deg);
        free(jobs[t].hot_cur);
        jobs[t].hot_deg = NULL;
        jobs[t].hot_cur = NULL;
    }
    uint32_t* ndeg = malloc(V * sizeof(uint32_t));
    /* vertex ranges balanced by edges: R-MAT hubs sit at low ids */
    uint32_t* cut = malloc((threads + 1) * sizeof(uint32_t));
    cut[0] = 0;
    for (int t = 1, v = 0; t <= threads; ++t) {
        uint64_t target = E0 * (uint64_t)t / threads;
        while ((uint32_t)v < V && off0[v] < target) ++v;
        cut[t] = t == threads ? V : (uint32_t)v;
    }
    for (int t = 0; t < threads; ++t) {
        jobs[t].vlo = cut[t];
        jobs[t].vhi = cut[t + 1];
        jobs[t].off0 = off0;
        jobs[t].ndeg = ndeg;
        jobs[t].pass = 2;
    }
    wfo_run_jobs(jobs, threads);
    uint64_t* off1 = malloc((V + 1ull) * sizeof(uint64_t));
    off1[0] = 0;
    for (uint32_t v = 0; v < V; ++v) off1[v + 1] = off1[v] + ndeg[v];
    free(ndeg);
    uint64_t E = off1[V];
    uint32_t* nbr = malloc((E + 8) * sizeof(uint32_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t].off1 = off1;
        jobs[t].out = nbr;
        jobs[t].pass = 3;
    }
    wfo_run_jobs(jobs, threads);
    free(raw);
    free(off0);
    free(cut);
    float* w = weighted ? malloc((E ? E : 1) * sizeof(float)) : NULL;
    uint8_t* lab = label_count ? malloc(E ? E : 1) : NULL;
    if (w || lab) {
        for (int t = 0; t < threads; ++t) {
            jobs[t].elo = E * t / threads;
            jobs[t].ehi = E * (t + 1) / threads;
            jobs[t].wmix = wfo_mix((seed ^ WFO_WEIGHT_SALT) + WFO_GAMMA);
            jobs[t].lmix = wfo_mix((seed ^ WFO_LABEL_SALT) + WFO_GAMMA);
            jobs[t].w = w;
            jobs[t].lab = lab;
            jobs[t].label_count = label_count;
            jobs[t].pass = 4;
        }
        wfo_run_jobs(jobs, threads);
    }
    free(jobs);
    out->vertex_count = V;
    out->edge_count = E;
    out->offsets = off1;
    out->neighbors = nbr;
    out->weights = w;
    out->labels = lab;
    return WF_OK;
}

void wfo_rmat_free(wfo_csr* g) {
    free(g->offsets); free(g->neighbors); free(g->weights); free(g->labels);
    memset(g, 0, sizeof(*g));
}
