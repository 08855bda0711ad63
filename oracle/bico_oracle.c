/*
 * bico_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference's BICO clustering-feature engine
 * (`/root/reference/pkg/src/piecy/coreset.py`, class BicoEngine).  Only the
 * test-suite, `__graft_entry__.smoke()` and the `cpu_baseline` / `--impl
 * reference` legs of bench.py may load this library.  The product path in
 * `paper_1502_04265_b200/` never links or calls it.
 *
 * Semantics followed (file:line in coreset.py):
 *   insert / validation / total weight ........... :264-281
 *   bootstrap buffering, exact-bytes distinctness . :283-295
 *   build: T0 = min positive pairwise sq * m / 16 . :297-305, :479-489
 *   live insert loop ............................. :307-310
 *   one descent (_absorb) with inlined capacity ... :312-372
 *   open ......................................... :374-377, _Node :191-201
 *   group add / nearest (first index wins ties) .. :146-180
 *   rebuild: T*=2, sort (-weight, index), reattach  :381-421, :454-463
 *   features (DFS pre-order) / extract ........... :425-451
 *   bootstrap-time features (aggregated pending) . :429-432, :466-476
 *
 * All scalar decision arithmetic keeps the reference's operation order
 * (no FMA contraction: build with -ffp-contract=off).  Dot products are plain
 * left-to-right fp64 sums; the reference uses OpenBLAS ddot/dgemv whose
 * summation order is CPU-kernel dependent, so those values agree to ~1e-16
 * relative, not bit-for-bit (SURVEY.md §8a parity contract).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t *members;  /* node ids in position order */
    int64_t size, cap;
} group_t;

typedef struct {
    int dim;
    int64_t budget, sample_cap;
    int64_t total_weight;
    double threshold;
    int built;
    int64_t num_features, next_index;
    /* node storage (slots are never reused; rebuild merges leave holes) */
    int64_t ncap, nnodes;
    int64_t *w, *index, *children;
    double *q, *sn, *rn, *s, *ref;
    /* groups; group 0 is the root */
    group_t *groups;
    int64_t ngroups, gcap;
    /* bootstrap state */
    double *pend_x; int64_t *pend_w; int64_t npend, pcap;
    double *dist_x; int64_t ndist, dcap;       /* distinct keys, first-seen order */
    int64_t *htab; int64_t hcap;              /* open addressing over dist_x rows */
} bico_t;

static double dot(const double *a, const double *b, int d) {
    double acc = 0.0;
    for (int i = 0; i < d; ++i) acc += a[i] * b[i];
    return acc;
}

static uint64_t hash_bytes(const double *x, int d) {
    const unsigned char *p = (const unsigned char *)x;
    uint64_t h = 1469598103934665603ULL;
    for (size_t i = 0; i < (size_t)d * 8; ++i) { h ^= p[i]; h *= 1099511628211ULL; }
    return h;
}

static void *xrealloc(void *p, size_t n) { void *q = realloc(p, n ? n : 1); if (!q) abort(); return q; }

bico_t *bico_create(int dim, int64_t budget, int64_t bootstrap_cap) {
    bico_t *e = (bico_t *)calloc(1, sizeof(bico_t));
    e->dim = dim; e->budget = budget;
    e->sample_cap = budget + 1 < bootstrap_cap ? budget + 1 : bootstrap_cap;
    e->hcap = 64;
    e->htab = (int64_t *)malloc(sizeof(int64_t) * e->hcap);
    for (int64_t i = 0; i < e->hcap; ++i) e->htab[i] = -1;
    return e;
}

void bico_destroy(bico_t *e) {
    if (!e) return;
    free(e->w); free(e->index); free(e->children); free(e->q); free(e->sn); free(e->rn);
    free(e->s); free(e->ref);
    for (int64_t g = 0; g < e->ngroups; ++g) free(e->groups[g].members);
    free(e->groups);
    free(e->pend_x); free(e->pend_w); free(e->dist_x); free(e->htab);
    free(e);
}

/* ---------------------------------------------------------------- groups */
static int64_t new_group(bico_t *e) {
    if (e->ngroups == e->gcap) {
        e->gcap = e->gcap ? 2 * e->gcap : 64;
        e->groups = (group_t *)xrealloc(e->groups, sizeof(group_t) * e->gcap);
    }
    group_t *g = &e->groups[e->ngroups];
    g->members = NULL; g->size = 0; g->cap = 0;
    return e->ngroups++;
}

static void group_add(bico_t *e, int64_t gid, int64_t node) {   /* coreset.py:146-156 */
    group_t *g = &e->groups[gid];
    if (g->size == g->cap) {
        g->cap = g->cap ? 2 * g->cap : 8;
        g->members = (int64_t *)xrealloc(g->members, sizeof(int64_t) * g->cap);
    }
    g->members[g->size++] = node;
    e->rn[node] = dot(e->ref + node * e->dim, e->ref + node * e->dim, e->dim);
}

/* nearest reference of a group: position + part (|r|^2 - 2 r.x); -1 if empty.
 * coreset.py:158-180 -- strict '<' keeps the lowest position on ties. */
static int64_t group_nearest(const bico_t *e, int64_t gid, const double *x, double *part) {
    const group_t *g = &e->groups[gid];
    int64_t best = -1; double bp = INFINITY;
    for (int64_t p = 0; p < g->size; ++p) {
        int64_t j = g->members[p];
        double v = e->rn[j] + (-2.0 * dot(e->ref + j * e->dim, x, e->dim));
        if (best < 0 || v < bp) { best = p; bp = v; }
    }
    *part = bp;
    return best;
}

/* ----------------------------------------------------------------- nodes */
static int64_t new_node(bico_t *e) {
    if (e->nnodes == e->ncap) {
        int64_t c = e->ncap ? 2 * e->ncap : 256;
        size_t d = (size_t)e->dim;
        e->w = (int64_t *)xrealloc(e->w, sizeof(int64_t) * c);
        e->index = (int64_t *)xrealloc(e->index, sizeof(int64_t) * c);
        e->children = (int64_t *)xrealloc(e->children, sizeof(int64_t) * c);
        e->q = (double *)xrealloc(e->q, sizeof(double) * c);
        e->sn = (double *)xrealloc(e->sn, sizeof(double) * c);
        e->rn = (double *)xrealloc(e->rn, sizeof(double) * c);
        e->s = (double *)xrealloc(e->s, sizeof(double) * c * d);
        e->ref = (double *)xrealloc(e->ref, sizeof(double) * c * d);
        e->ncap = c;
    }
    return e->nnodes++;
}

/* _open: coreset.py:374-377 with _Node.__init__ :191-198 */
static void open_node(bico_t *e, int64_t gid, const double *x, double x_sq, int64_t w) {
    int64_t j = new_node(e);
    int d = e->dim;
    double fw = (double)w;
    e->w[j] = w;
    for (int i = 0; i < d; ++i) e->s[j * d + i] = fw * x[i];
    e->q[j] = fw * x_sq;
    e->sn[j] = (double)(w * w) * x_sq;
    memcpy(e->ref + j * d, x, sizeof(double) * d);
    e->children[j] = -1;
    e->index[j] = e->next_index++;
    group_add(e, gid, j);
    e->num_features++;
}

static void rebuild(bico_t *e);

/* _absorb: coreset.py:312-372.  Returns copies placed. */
static int64_t absorb(bico_t *e, const double *x, double x_sq, int64_t remaining) {
    const double T = e->threshold;
    int64_t gid = 0;
    double radius_sq = T;
    int64_t placed = 0;
    int d = e->dim;
    for (;;) {
        double part;
        int64_t pos = group_nearest(e, gid, x, &part);
        if (pos < 0 || part + x_sq > radius_sq) {
            if (e->num_features < e->budget) {
                open_node(e, gid, x, x_sq, remaining);
                return placed + remaining;
            }
            open_node(e, gid, x, x_sq, 1);
            rebuild(e);
            return placed + 1;
        }
        int64_t j = e->groups[gid].members[pos];
        int64_t n = e->w[j];
        double fn = (double)n;
        double norm_over_n = e->sn[j] / fn;
        double err = e->q[j] - norm_over_n;
        if (err < 0.0) err = 0.0;
        double dt = dot(e->s + j * d, x, d);
        double dist_sq = x_sq - (2.0 * dt - norm_over_n) / fn;
        if (dist_sq < 0.0) dist_sq = 0.0;
        double slack = fn * dist_sq - T + err;
        int64_t take;
        if (slack <= 0.0) {
            take = remaining;
        } else {
            double limit = (fn * T - fn * err) / slack;
            if (limit >= (double)remaining) take = remaining;
            else if (limit > 0.0) take = (int64_t)limit;
            else take = 0;
        }
        if (take > 0) {
            e->w[j] = n + take;
            double *s = e->s + j * d;
            if (take == 1) { for (int i = 0; i < d; ++i) s[i] += x[i]; }
            else { double ft = (double)take; for (int i = 0; i < d; ++i) s[i] += ft * x[i]; }
            e->q[j] += (double)take * x_sq;
            e->sn[j] += 2.0 * (double)take * dt + (double)(take * take) * x_sq;
            placed += take;
            remaining -= take;
            if (remaining == 0) return placed;
        }
        if (e->children[j] < 0) e->children[j] = new_group(e);
        gid = e->children[j];
        radius_sq *= 0.25;
    }
}

static void insert_live(bico_t *e, const double *x, double x_sq, int64_t w) {
    int64_t remaining = w;
    while (remaining > 0) remaining -= absorb(e, x, x_sq, remaining);
}

/* ---------------------------------------------------------------- rebuild */
static const bico_t *g_sort_engine;
static int rebuild_cmp(const void *pa, const void *pb) {   /* coreset.py:454-455 */
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    const bico_t *e = g_sort_engine;
    if (e->w[a] != e->w[b]) return e->w[a] > e->w[b] ? -1 : 1;
    return e->index[a] < e->index[b] ? -1 : (e->index[a] > e->index[b]);
}

static void collect(bico_t *e, int64_t gid, int64_t *out, int64_t *cnt) {  /* :458-463 */
    group_t *g = &e->groups[gid];
    for (int64_t p = 0; p < g->size; ++p) {
        int64_t j = g->members[p];
        out[(*cnt)++] = j;
        if (e->children[j] >= 0) { collect(e, e->children[j], out, cnt); e->children[j] = -1; }
    }
}

static void reattach(bico_t *e, int64_t node) {   /* coreset.py:395-421 */
    int d = e->dim;
    double T = e->threshold;
    int64_t gid = 0;
    double radius_sq = T;
    const double *ref = e->ref + node * d;
    double ref_sq = dot(ref, ref, d);
    double *msum = (double *)malloc(sizeof(double) * d);
    for (;;) {
        double part;
        int64_t pos = group_nearest(e, gid, ref, &part);
        if (pos < 0 || part + ref_sq > radius_sq) {
            group_add(e, gid, node);
            e->num_features++;
            break;
        }
        int64_t h = e->groups[gid].members[pos];
        int64_t mw = e->w[h] + e->w[node];
        for (int i = 0; i < d; ++i) msum[i] = e->s[h * d + i] + e->s[node * d + i];
        double mq = e->q[h] + e->q[node];
        double mn = dot(msum, msum, d);
        if (mq - mn / (double)mw <= T) {
            e->w[h] = mw;
            memcpy(e->s + h * d, msum, sizeof(double) * d);
            e->q[h] = mq;
            e->sn[h] = mn;
            e->w[node] = 0;   /* merged away */
            break;
        }
        if (e->children[h] < 0) e->children[h] = new_group(e);
        gid = e->children[h];
        radius_sq *= 0.25;
    }
    free(msum);
}

static void rebuild(bico_t *e) {   /* coreset.py:381-393 */
    while (e->num_features > e->budget) {
        e->threshold *= 2.0;
        int64_t *nodes = (int64_t *)malloc(sizeof(int64_t) * (e->num_features + 1));
        int64_t cnt = 0;
        collect(e, 0, nodes, &cnt);
        g_sort_engine = e;
        qsort(nodes, cnt, sizeof(int64_t), rebuild_cmp);
        for (int64_t g = 0; g < e->ngroups; ++g) free(e->groups[g].members);
        e->ngroups = 0;
        new_group(e);   /* fresh roots */
        e->num_features = 0;
        for (int64_t i = 0; i < cnt; ++i) reattach(e, nodes[i]);
        free(nodes);
    }
}

/* ------------------------------------------------------------- bootstrap */
static int64_t dist_lookup(bico_t *e, const double *x, uint64_t h, int insert) {
    int d = e->dim;
    uint64_t mask = (uint64_t)e->hcap - 1;
    for (uint64_t i = h & mask;; i = (i + 1) & mask) {
        int64_t k = e->htab[i];
        if (k < 0) {
            if (!insert) return -1;
            e->htab[i] = e->ndist;  /* caller appends the key */
            return -2;
        }
        if (memcmp(e->dist_x + k * d, x, sizeof(double) * d) == 0) return k;
    }
}

static void dist_grow(bico_t *e) {
    int64_t nc = e->hcap * 2;
    int64_t *t = (int64_t *)malloc(sizeof(int64_t) * nc);
    for (int64_t i = 0; i < nc; ++i) t[i] = -1;
    for (int64_t k = 0; k < e->ndist; ++k) {
        uint64_t h = hash_bytes(e->dist_x + k * e->dim, e->dim);
        for (uint64_t i = h & (nc - 1);; i = (i + 1) & (nc - 1))
            if (t[i] < 0) { t[i] = k; break; }
    }
    free(e->htab); e->htab = t; e->hcap = nc;
}

static void min_pairwise_build(bico_t *e);

static void bootstrap(bico_t *e, const double *x, int64_t w) {   /* coreset.py:283-295 */
    int d = e->dim;
    if (e->npend > 0 && memcmp(e->pend_x + (e->npend - 1) * d, x, sizeof(double) * d) == 0) {
        e->pend_w[e->npend - 1] += w;
    } else {
        if (e->npend == e->pcap) {
            e->pcap = e->pcap ? 2 * e->pcap : 64;
            e->pend_x = (double *)xrealloc(e->pend_x, sizeof(double) * e->pcap * d);
            e->pend_w = (int64_t *)xrealloc(e->pend_w, sizeof(int64_t) * e->pcap);
        }
        memcpy(e->pend_x + e->npend * d, x, sizeof(double) * d);
        e->pend_w[e->npend++] = w;
    }
    uint64_t h = hash_bytes(x, d);
    if (dist_lookup(e, x, h, 1) == -2) {
        if (e->ndist == e->dcap) {
            e->dcap = e->dcap ? 2 * e->dcap : 64;
            e->dist_x = (double *)xrealloc(e->dist_x, sizeof(double) * e->dcap * d);
        }
        memcpy(e->dist_x + e->ndist * d, x, sizeof(double) * d);
        e->ndist++;
        if (e->ndist * 2 > e->hcap) dist_grow(e);
        if (e->ndist > e->budget) min_pairwise_build(e);
    }
}

/* _min_pairwise_sq (coreset.py:479-489) on the first sample_cap distinct keys,
 * then _build (:297-305). */
static void min_pairwise_build(bico_t *e) {
    int d = e->dim;
    int64_t ns = e->ndist < e->sample_cap ? e->ndist : e->sample_cap;
    const double *S = e->dist_x;
    double mn;
    if (ns < 2) {
        mn = 1.0;
    } else {
        double *nrm = (double *)malloc(sizeof(double) * ns);
        double nmax = -INFINITY;
        for (int64_t i = 0; i < ns; ++i) { nrm[i] = dot(S + i * d, S + i * d, d); if (nrm[i] > nmax) nmax = nrm[i]; }
        mn = INFINITY; int any = 0;
        for (int64_t i = 0; i < ns; ++i)
            for (int64_t j = 0; j < ns; ++j) {
                if (i == j) continue;
                double v = (nrm[i] + nrm[j]) - 2.0 * dot(S + i * d, S + j * d, d);
                if (v > 0.0) { any = 1; if (v < mn) mn = v; }
            }
        if (!any) mn = 1e-12 * (nmax > 1.0 ? nmax : 1.0);
        free(nrm);
    }
    e->threshold = mn * (double)e->budget / 16.0;
    e->built = 1;
    new_group(e);   /* roots */
    /* replay pending in order */
    int64_t np = e->npend;
    double *px = e->pend_x; int64_t *pw = e->pend_w;
    e->pend_x = NULL; e->pend_w = NULL; e->npend = 0; e->pcap = 0;
    free(e->dist_x); e->dist_x = NULL; e->ndist = 0; e->dcap = 0;
    for (int64_t i = 0; i < e->hcap; ++i) e->htab[i] = -1;
    for (int64_t i = 0; i < np; ++i) {
        const double *x = px + i * d;
        insert_live(e, x, dot(x, x, d), pw[i]);
    }
    free(px); free(pw);
}

/* ------------------------------------------------------------ public API */
/* Returns 0 ok, -1 non-finite coordinates, -2 overflow, -3 bad weight. */
int bico_insert(bico_t *e, const double *x, int64_t w) {   /* coreset.py:264-281 */
    if (w < 1) return -3;
    double x_sq = dot(x, x, e->dim);
    if (!isfinite(x_sq)) {
        for (int i = 0; i < e->dim; ++i) if (!isfinite(x[i])) return -1;
        return -2;
    }
    e->total_weight += w;
    if (!e->built) bootstrap(e, x, w);
    else insert_live(e, x, x_sq, w);
    return 0;
}

/* Inserts rows in order; stops at the first invalid row.  Returns the number
 * of rows consumed; *status receives the error of the failing row (or 0). */
int64_t bico_insert_block(bico_t *e, const double *X, const int64_t *W, int64_t n, int *status) {
    *status = 0;
    for (int64_t i = 0; i < n; ++i) {
        int rc = bico_insert(e, X + i * e->dim, W ? W[i] : 1);
        if (rc) { *status = rc; return i; }
    }
    return n;
}

int64_t bico_num_features(const bico_t *e) { return e->built ? e->num_features : e->ndist; }
double bico_threshold(const bico_t *e) { return e->threshold; }
int64_t bico_total_weight(const bico_t *e) { return e->total_weight; }
int bico_built(const bico_t *e) { return e->built; }

/* features(): coreset.py:425-441 (DFS pre-order), bootstrap form :429-432.
 * Writes up to cap rows; returns the feature count. */
static void dfs(const bico_t *e, int64_t gid, int level, int64_t *cnt, int64_t cap,
                int32_t *lv, int64_t *w, double *s, double *q, double *ref) {
    const group_t *g = &e->groups[gid];
    int d = e->dim;
    for (int64_t p = 0; p < g->size; ++p) {
        int64_t j = g->members[p];
        int64_t k = (*cnt)++;
        if (k < cap) {
            if (lv) lv[k] = level;
            if (w) w[k] = e->w[j];
            if (s) memcpy(s + k * d, e->s + j * d, sizeof(double) * d);
            if (q) q[k] = e->q[j];
            if (ref) memcpy(ref + k * d, e->ref + j * d, sizeof(double) * d);
        }
        if (e->children[j] >= 0) dfs(e, e->children[j], level + 1, cnt, cap, lv, w, s, q, ref);
    }
}

int64_t bico_features(const bico_t *e, int64_t cap, int32_t *lv, int64_t *w, double *s,
                      double *q, double *ref) {
    int d = e->dim;
    if (!e->built) {
        /* _aggregate_pending: per exact location, first-occurrence order.  The
         * distinct-key table is kept in first-seen order, which is exactly the
         * first-occurrence order of the pending list. */
        int64_t nd = e->ndist;
        if (cap == 0) return nd;
        int64_t *tw = (int64_t *)calloc(nd ? nd : 1, sizeof(int64_t));
        for (int64_t i = 0; i < e->npend; ++i) {
            const double *x = e->pend_x + i * d;
            int64_t k = dist_lookup((bico_t *)e, x, hash_bytes(x, d), 0);
            tw[k] += e->pend_w[i];
        }
        for (int64_t k = 0; k < nd && k < cap; ++k) {
            const double *x = e->dist_x + k * d;
            double fw = (double)tw[k];
            if (lv) lv[k] = 1;
            if (w) w[k] = tw[k];
            if (s) for (int i = 0; i < d; ++i) s[k * d + i] = fw * x[i];
            if (q) q[k] = fw * dot(x, x, d);
            if (ref) memcpy(ref + k * d, x, sizeof(double) * d);
        }
        free(tw);
        return nd;
    }
    int64_t cnt = 0;
    dfs(e, 0, 1, &cnt, cap, lv, w, s, q, ref);
    return cnt;
}

/* extract_coreset: coreset.py:443-451 -- row = s / n, weight n. */
int64_t bico_extract(const bico_t *e, int64_t cap, double *pts, int64_t *wts) {
    int d = e->dim;
    int64_t nf = bico_features(e, 0, NULL, NULL, NULL, NULL, NULL);
    if (nf == 0) return 0;
    int64_t *w = (int64_t *)malloc(sizeof(int64_t) * nf);
    double *s = (double *)malloc(sizeof(double) * nf * d);
    bico_features(e, nf, NULL, w, s, NULL, NULL);
    for (int64_t k = 0; k < nf && k < cap; ++k) {
        double fw = (double)w[k];
        for (int i = 0; i < d; ++i) pts[k * d + i] = s[k * d + i] / fw;
        wts[k] = w[k];
    }
    free(w); free(s);
    return nf;
}
