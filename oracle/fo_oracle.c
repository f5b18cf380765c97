/*
 * fo_oracle.c -- CPU restatement of the reference `fuseopt` candidate-scoring
 * path (contraction -> durations -> discrete-event simulation), its
 * batch-expand step (CPython MT19937 + random_apply) and Alg. 1.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline; it is never linked into, called by, or shipped with the product
 * (paper_2209_12769_b200/).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.
 *
 * Pinned against golden vectors produced by the unmodified reference
 * (tests/golden/make_golden.py); see tests/test_oracle_golden.py.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to the reference's pkg/src/fuseopt/).
 *
 * Compiled with -ffp-contract=off: the reference's fp64 arithmetic is plain
 * IEEE add/mul (CPython floats), so no fused multiply-adds may appear.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_CYCLE 1
#define ORC_MISSING_COST 2
#define ORC_NEGATIVE_DURATION 3
#define ORC_DIM_MISMATCH 4
#define ORC_INVALID_ARG 5

/* op kinds (graph.py:29-32) */
#define KIND_COMPUTE 0
#define KIND_PARAMETER 1
#define KIND_CONTROL 2

/* cost provider kinds */
#define PROV_PROFILE 0 /* make_cost_providers (estimator.py:801-824) */
#define PROV_HW_ORACLE 1 /* oracle_providers, noise == 0 (workloads.py:294-304) */

/* estimator variants (estimator.py:254-257) */
#define VAR_NONE -1 /* model=None: fused groups -> MissingCost (estimator.py:815) */
#define VAR_ANALYTIC 0
#define VAR_LINEAR 1
#define VAR_MP 2

/* ------------------------------------------------------------------------ */
/* graph + model descriptions (caller-owned arrays, copied by orc_prepare)   */

typedef struct {
    int32_t V, E, A;
    const int32_t *op_kind;      /* [V] */
    const int64_t *op_out_bytes; /* [V] */
    const double *op_prof;       /* [V] lookup(profile, op); NaN = missing */
    const double *op_compute;    /* [V] OpNode.compute_us; NaN = None */
    const int32_t *op_slot;      /* [V] vocab slot for the one-hot */
    const int32_t *e_src, *e_dst; /* [E] op indices; sorted by (src, dst) */
    const int64_t *e_bytes;       /* [E] */
    const int32_t *ar_prod;       /* [A] producer op index; ARs in id order */
    const int64_t *ar_bytes;      /* [A] */
} orc_graph_desc;

typedef struct {
    int32_t provider;  /* PROV_* */
    int32_t variant;   /* VAR_* */
    double comm_C, comm_D;
    double launch, mem; /* analytic model params or hw oracle params */
    int32_t layers, hidden, feat_dim;
    const double *W_emb;   /* [hidden x feat_dim] */
    const double *W_layer; /* [layers x hidden x hidden] */
    const double *W_r, *A1, *c1, *A2, *c2, *a3;
    double c3;
    const double *node_mean, *node_std; /* [feat_dim] or NULL */
    const double *lin_w;                /* [12] */
    double lin_b;
    const double *agg_mean, *agg_std; /* [12] or NULL */
    double out_scale;
} orc_model;

typedef struct {
    int32_t V, E, A;
    int32_t *op_kind;
    int64_t *op_out_bytes;
    double *op_prof, *op_compute;
    int32_t *op_slot;
    int32_t *e_src, *e_dst;
    int64_t *e_bytes;
    int32_t *ar_prod;
    int64_t *ar_bytes;
    /* derived (graph.py:122-154) */
    int32_t *out_ptr, *out_e; /* out edges per op */
    int32_t *in_ptr, *in_e;   /* in edges per op */
    int32_t *arp_ptr, *arp;   /* ARs per producer op */
    uint8_t *agg;             /* per edge: _consumes_aggregate (graph.py:225-235) */
    int64_t *in_bytes;        /* per op: sum of all in-edge bytes (estimator.py:171) */
} orc_static;

static void *xmalloc(size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p) abort();
    return p;
}
static void *xcalloc(size_t n, size_t s) {
    void *p = calloc(n ? n : 1, s ? s : 1);
    if (!p) abort();
    return p;
}
#define DUP_ARR(dst, src, n, T)                       \
    do {                                              \
        (dst) = (T *)xmalloc(sizeof(T) * (size_t)(n)); \
        if (n) memcpy((dst), (src), sizeof(T) * (size_t)(n)); \
    } while (0)

static void csr_build(int n, int m, const int32_t *key, int32_t **ptr_out, int32_t **idx_out) {
    int32_t *ptr = (int32_t *)xcalloc((size_t)n + 1, sizeof(int32_t));
    int32_t *idx = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)m);
    for (int i = 0; i < m; i++) ptr[key[i] + 1]++;
    for (int i = 0; i < n; i++) ptr[i + 1] += ptr[i];
    int32_t *fill = (int32_t *)xmalloc(sizeof(int32_t) * ((size_t)n + 1));
    memcpy(fill, ptr, sizeof(int32_t) * ((size_t)n + 1));
    for (int i = 0; i < m; i++) idx[fill[key[i]]++] = i; /* stable: keeps input order */
    free(fill);
    *ptr_out = ptr;
    *idx_out = idx;
}

orc_static *orc_prepare(const orc_graph_desc *d) {
    orc_static *s = (orc_static *)xcalloc(1, sizeof(orc_static));
    s->V = d->V; s->E = d->E; s->A = d->A;
    DUP_ARR(s->op_kind, d->op_kind, d->V, int32_t);
    DUP_ARR(s->op_out_bytes, d->op_out_bytes, d->V, int64_t);
    DUP_ARR(s->op_prof, d->op_prof, d->V, double);
    DUP_ARR(s->op_compute, d->op_compute, d->V, double);
    DUP_ARR(s->op_slot, d->op_slot, d->V, int32_t);
    DUP_ARR(s->e_src, d->e_src, d->E, int32_t);
    DUP_ARR(s->e_dst, d->e_dst, d->E, int32_t);
    DUP_ARR(s->e_bytes, d->e_bytes, d->E, int64_t);
    DUP_ARR(s->ar_prod, d->ar_prod, d->A, int32_t);
    DUP_ARR(s->ar_bytes, d->ar_bytes, d->A, int64_t);
    csr_build(s->V, s->E, s->e_src, &s->out_ptr, &s->out_e);
    csr_build(s->V, s->E, s->e_dst, &s->in_ptr, &s->in_e);
    csr_build(s->V, s->A, s->ar_prod, &s->arp_ptr, &s->arp);
    s->agg = (uint8_t *)xcalloc((size_t)s->E, 1);
    for (int e = 0; e < s->E; e++) {
        int src = s->e_src[e], dst = s->e_dst[e];
        /* graph.py:231-235: src produces an AR, dst has no out-edges, dst produces no AR */
        s->agg[e] = (s->arp_ptr[src + 1] > s->arp_ptr[src]) && (s->out_ptr[dst + 1] == s->out_ptr[dst]) &&
                    (s->arp_ptr[dst + 1] == s->arp_ptr[dst]);
    }
    s->in_bytes = (int64_t *)xcalloc((size_t)s->V, sizeof(int64_t));
    for (int e = 0; e < s->E; e++) s->in_bytes[s->e_dst[e]] += s->e_bytes[e];
    return s;
}

void orc_free(orc_static *s) {
    if (!s) return;
    free(s->op_kind); free(s->op_out_bytes); free(s->op_prof); free(s->op_compute); free(s->op_slot);
    free(s->e_src); free(s->e_dst); free(s->e_bytes); free(s->ar_prod); free(s->ar_bytes);
    free(s->out_ptr); free(s->out_e); free(s->in_ptr); free(s->in_e); free(s->arp_ptr); free(s->arp);
    free(s->agg); free(s->in_bytes);
    free(s);
}

/* ------------------------------------------------------------------------ */
/* fusion-state index (graph.py:117-159)                                     */

typedef struct {
    int32_t G, B;
    int32_t *gid;              /* [G] sorted group ids */
    int32_t *mptr, *mem;       /* members per group (op index asc), all memberships */
    uint8_t *mdup;             /* membership is a duplicated (replica) one */
    int32_t *ngi, *rgi;        /* [V] group index of normal / replica membership */
    int32_t *bid;              /* [B] sorted bucket ids */
    int32_t *bptr, *bmem;      /* ARs per bucket (AR index asc) */
    int32_t *bki;              /* [A] bucket index per AR */
} orc_index;

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

static int uniq_sorted(int32_t *v, int n) {
    int k = 0;
    for (int i = 0; i < n; i++)
        if (k == 0 || v[k - 1] != v[i]) v[k++] = v[i];
    return k;
}

static int find_i32(const int32_t *v, int n, int32_t x) {
    int lo = 0, hi = n - 1;
    while (lo <= hi) {
        int mid = (lo + hi) >> 1;
        if (v[mid] == x) return mid;
        if (v[mid] < x) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

static void index_free(orc_index *ix) {
    free(ix->gid); free(ix->mptr); free(ix->mem); free(ix->mdup); free(ix->ngi); free(ix->rgi);
    free(ix->bid); free(ix->bptr); free(ix->bmem); free(ix->bki);
    memset(ix, 0, sizeof(*ix));
}

static void index_build(const orc_static *s, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt,
                        orc_index *ix) {
    int V = s->V, A = s->A;
    int32_t *ids = (int32_t *)xmalloc(sizeof(int32_t) * (2 * (size_t)V + 1));
    int n = 0;
    for (int v = 0; v < V; v++) {
        ids[n++] = ngid[v];
        if (rgid[v] >= 0) ids[n++] = rgid[v];
    }
    qsort(ids, (size_t)n, sizeof(int32_t), cmp_i32);
    ix->G = uniq_sorted(ids, n);
    ix->gid = ids;
    ix->ngi = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(V ? V : 1));
    ix->rgi = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(V ? V : 1));
    ix->mptr = (int32_t *)xcalloc((size_t)ix->G + 1, sizeof(int32_t));
    for (int v = 0; v < V; v++) {
        ix->ngi[v] = find_i32(ix->gid, ix->G, ngid[v]);
        ix->rgi[v] = rgid[v] >= 0 ? find_i32(ix->gid, ix->G, rgid[v]) : -1;
        ix->mptr[ix->ngi[v] + 1]++;
        if (ix->rgi[v] >= 0) ix->mptr[ix->rgi[v] + 1]++;
    }
    for (int g = 0; g < ix->G; g++) ix->mptr[g + 1] += ix->mptr[g];
    int M = ix->mptr[ix->G];
    ix->mem = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(M ? M : 1));
    ix->mdup = (uint8_t *)xmalloc((size_t)(M ? M : 1));
    int32_t *fill = (int32_t *)xmalloc(sizeof(int32_t) * ((size_t)ix->G + 1));
    memcpy(fill, ix->mptr, sizeof(int32_t) * ((size_t)ix->G + 1));
    for (int v = 0; v < V; v++) { /* ascending op index -> members sorted */
        int g = ix->ngi[v];
        ix->mdup[fill[g]] = 0;
        ix->mem[fill[g]++] = v;
        if (ix->rgi[v] >= 0) {
            g = ix->rgi[v];
            ix->mdup[fill[g]] = 1;
            ix->mem[fill[g]++] = v;
        }
    }
    free(fill);
    int32_t *bids = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(A ? A : 1));
    memcpy(bids, bkt, sizeof(int32_t) * (size_t)A);
    qsort(bids, (size_t)A, sizeof(int32_t), cmp_i32);
    ix->B = uniq_sorted(bids, A);
    ix->bid = bids;
    ix->bki = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(A ? A : 1));
    for (int a = 0; a < A; a++) ix->bki[a] = find_i32(ix->bid, ix->B, bkt[a]);
    csr_build(ix->B, A, ix->bki, &ix->bptr, &ix->bmem);
}

static inline int export_gi(const orc_index *ix, int op) { /* graph.py:158-159 */
    return ix->rgi[op] >= 0 ? ix->rgi[op] : ix->ngi[op];
}
static inline int in_group(const orc_index *ix, int op, int g) {
    return ix->ngi[op] == g || ix->rgi[op] == g;
}

/* sorted-unique pair lists -> CSR */
typedef struct { int32_t a, b; } pair_t;
static int cmp_pair(const void *x, const void *y) {
    const pair_t *p = (const pair_t *)x, *q = (const pair_t *)y;
    if (p->a != q->a) return (p->a > q->a) - (p->a < q->a);
    return (p->b > q->b) - (p->b < q->b);
}
static void pairs_to_csr(pair_t *p, int n, int nodes, int32_t **ptr, int32_t **idx, int *m_out) {
    qsort(p, (size_t)n, sizeof(pair_t), cmp_pair);
    int m = 0;
    for (int i = 0; i < n; i++)
        if (m == 0 || p[m - 1].a != p[i].a || p[m - 1].b != p[i].b) p[m++] = p[i];
    *ptr = (int32_t *)xcalloc((size_t)nodes + 1, sizeof(int32_t));
    *idx = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    for (int i = 0; i < m; i++) { (*ptr)[p[i].a + 1]++; (*idx)[i] = p[i].b; }
    for (int i = 0; i < nodes; i++) (*ptr)[i + 1] += (*ptr)[i];
    if (m_out) *m_out = m;
}

/* Joint schedule deps over nodes [groups (id order) | buckets (id order)]
 * (graph.py:215-274).  dptr/dep: deps of each node (sorted unique). */
static void schedule_deps(const orc_static *s, const orc_index *ix, int32_t **dptr, int32_t **dep) {
    int G = ix->G;
    size_t cap = 2 * (size_t)s->E * 2 + (size_t)s->A * 4 + 16;
    pair_t *p = (pair_t *)xmalloc(sizeof(pair_t) * cap);
    int n = 0;
    for (int e = 0; e < s->E; e++) {
        int src = s->e_src[e], dst = s->e_dst[e];
        int copies[2] = {ix->ngi[dst], ix->rgi[dst]};
        if (!s->agg[e]) { /* group_group_deps (graph.py:249-261) */
            int sg = export_gi(ix, src);
            for (int c = 0; c < 2; c++) {
                int g = copies[c];
                if (g < 0 || in_group(ix, src, g)) continue;
                if ((size_t)n + 1 >= cap) { cap *= 2; p = (pair_t *)realloc(p, sizeof(pair_t) * cap); }
                p[n].a = g; p[n].b = sg; n++;
            }
        } else { /* group_bucket_deps (graph.py:237-247) */
            for (int k = s->arp_ptr[src]; k < s->arp_ptr[src + 1]; k++) {
                int a = s->arp[k];
                for (int c = 0; c < 2; c++) {
                    int g = copies[c];
                    if (g < 0) continue;
                    if ((size_t)n + 1 >= cap) { cap *= 2; p = (pair_t *)realloc(p, sizeof(pair_t) * cap); }
                    p[n].a = g; p[n].b = G + ix->bki[a]; n++;
                }
            }
        }
    }
    for (int a = 0; a < s->A; a++) { /* bucket_ready_deps (graph.py:215-223) */
        if ((size_t)n + 1 >= cap) { cap *= 2; p = (pair_t *)realloc(p, sizeof(pair_t) * cap); }
        p[n].a = G + ix->bki[a]; p[n].b = export_gi(ix, s->ar_prod[a]); n++;
    }
    pairs_to_csr(p, n, G + ix->B, dptr, dep, NULL);
    free(p);
}

/* Kahn over deps (graph.py:487-502) */
static int deps_acyclic(int nodes, const int32_t *dptr, const int32_t *dep) {
    int32_t *indeg = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(nodes ? nodes : 1));
    pair_t *rp = (pair_t *)xmalloc(sizeof(pair_t) * (size_t)(dptr[nodes] ? dptr[nodes] : 1));
    for (int v = 0; v < nodes; v++) {
        indeg[v] = dptr[v + 1] - dptr[v];
        for (int k = dptr[v]; k < dptr[v + 1]; k++) { rp[k].a = dep[k]; rp[k].b = v; }
    }
    int32_t *sptr, *succ;
    pairs_to_csr(rp, dptr[nodes], nodes, &sptr, &succ, NULL);
    int32_t *stack = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(nodes ? nodes : 1));
    int top = 0, seen = 0;
    for (int v = 0; v < nodes; v++) if (indeg[v] == 0) stack[top++] = v;
    while (top) {
        int u = stack[--top];
        seen++;
        for (int k = sptr[u]; k < sptr[u + 1]; k++)
            if (--indeg[succ[k]] == 0) stack[top++] = succ[k];
    }
    free(indeg); free(rp); free(sptr); free(succ); free(stack);
    return seen == nodes;
}

/* ------------------------------------------------------------------------ */
/* group_io (graph.py:181-213)                                                */

static void group_io(const orc_static *s, const orc_index *ix, int64_t *internal, int64_t *ext_in, int64_t *ext_out) {
    int G = ix->G;
    memset(internal, 0, sizeof(int64_t) * (size_t)G);
    memset(ext_in, 0, sizeof(int64_t) * (size_t)G);
    memset(ext_out, 0, sizeof(int64_t) * (size_t)G);
    uint8_t *visible = (uint8_t *)xcalloc((size_t)s->V, 1);
    for (int e = 0; e < s->E; e++) {
        int src = s->e_src[e], dst = s->e_dst[e];
        int copies[2] = {ix->ngi[dst], ix->rgi[dst]};
        for (int c = 0; c < 2; c++) {
            int g = copies[c];
            if (g < 0) continue;
            if (in_group(ix, src, g)) internal[g] += s->e_bytes[e];
            else { ext_in[g] += s->e_bytes[e]; visible[src] = 1; }
        }
    }
    for (int v = 0; v < s->V; v++) {
        if (visible[v] || s->out_ptr[v + 1] == s->out_ptr[v] || s->arp_ptr[v + 1] > s->arp_ptr[v])
            ext_out[export_gi(ix, v)] += s->op_out_bytes[v];
    }
    free(visible);
}

/* ------------------------------------------------------------------------ */
/* CPython 3.12 built-in sum() over floats: Neumaier-compensated
 * (Objects/bltinmodule.c builtin_sum_impl).  The reference sums member
 * times with sum() (estimator.py:186, :442; workloads.py:284).              */

typedef struct { double f, c; int n; } pysum_t;
static void pysum_add(pysum_t *s, double x) {
    if (s->n++ == 0) { s->f = 0.0 + x; s->c = 0.0; return; }
    double t = s->f + x;
    if (fabs(s->f) >= fabs(x)) s->c += (s->f - t) + x;
    else s->c += (x - t) + s->f;
    s->f = t;
}
static double pysum_get(const pysum_t *s) {
    double f = s->f;
    if (s->c != 0.0 && isfinite(s->c)) f += s->c;
    return s->n ? f : 0.0;
}

/* ------------------------------------------------------------------------ */
/* estimator (estimator.py:131-470)                                          */

static double softplus(double z) { /* np.logaddexp(0, z) */
    if (z == 0.0) return 0.6931471805599453; /* ln 2 */
    if (z > 0) return z + log1p(exp(-z));
    return log1p(exp(z));
}

/* _longest_path_nodes (estimator.py:131-154) over member-local edges */
static int longest_path(int n, int ne, const int32_t *ls, const int32_t *ld) {
    if (n == 0) return 0;
    int32_t *indeg = (int32_t *)xcalloc((size_t)n, sizeof(int32_t));
    int32_t *depth = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
    int32_t *order = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)n);
    for (int i = 0; i < ne; i++) indeg[ld[i]]++;
    int head = 0, tail = 0;
    for (int i = 0; i < n; i++) { depth[i] = 1; if (indeg[i] == 0) order[tail++] = i; }
    while (head < tail) {
        int u = order[head++];
        for (int i = 0; i < ne; i++)
            if (ls[i] == u && --indeg[ld[i]] == 0) order[tail++] = ld[i];
    }
    /* depth relaxation in topological order (the reference's BFS-by-levels
     * order is also topological; the max is order-independent) */
    for (int k = 0; k < tail; k++) {
        int u = order[k];
        for (int i = 0; i < ne; i++)
            if (ls[i] == u && depth[ld[i]] < depth[u] + 1) depth[ld[i]] = depth[u] + 1;
    }
    int best = 0;
    for (int i = 0; i < n; i++) if (depth[i] > best) best = depth[i];
    free(indeg); free(depth); free(order);
    return best;
}

/* predict_fused for one multi-member group (estimator.py:462-470, via
 * featurize estimator.py:157-191).  Returns status. */
static int predict_group(const orc_static *s, const orc_model *m, const orc_index *ix, int g,
                         const int64_t *io_int, const int64_t *io_in, const int64_t *io_out, double *out) {
    int n = ix->mptr[g + 1] - ix->mptr[g];
    const int32_t *mem = ix->mem + ix->mptr[g];
    for (int i = 0; i < n; i++)
        if (isnan(s->op_prof[mem[i]])) return ORC_MISSING_COST; /* lookup -> UnknownOp */
    if (m->variant == VAR_ANALYTIC) { /* estimator.py:434-446 */
        pysum_t acc = {0.0, 0.0, 0};
        for (int i = 0; i < n; i++) {
            int v = mem[i];
            double raw = (s->op_prof[v] - m->launch) - m->mem * (double)(s->in_bytes[v] + s->op_out_bytes[v]);
            pysum_add(&acc, raw);
        }
        double pred = (pysum_get(&acc) + m->launch) + m->mem * (double)(io_in[g] + io_out[g]);
        *out = pred > 1e-9 ? pred : 1e-9;
        return ORC_OK;
    }
    /* internal edges, member-local indices, in graph edge order (estimator.py:173-177) */
    int cap = 0;
    for (int i = 0; i < n; i++) cap += s->out_ptr[mem[i] + 1] - s->out_ptr[mem[i]];
    int32_t *ls = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(cap + 1));
    int32_t *ld = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(cap + 1));
    int ne = 0;
    for (int e = 0; e < s->E; e++) {
        int a = -1, b = -1;
        for (int i = 0; i < n; i++) { if (mem[i] == s->e_src[e]) a = i; if (mem[i] == s->e_dst[e]) b = i; }
        if (a >= 0 && b >= 0) { ls[ne] = a; ld[ne] = b; ne++; }
    }
    int st = ORC_OK;
    if (m->variant == VAR_LINEAR) { /* estimator.py:117-128, 341-345, 421-426 */
        pysum_t acc = {0.0, 0.0, 0};
        for (int i = 0; i < n; i++) pysum_add(&acc, s->op_prof[mem[i]]);
        double total = pysum_get(&acc);
        double agg[6] = {(double)n, total, (double)io_int[g], (double)io_in[g], (double)io_out[g],
                         (double)longest_path(n, ne, ls, ld)};
        double fs[12];
        for (int k = 0; k < 6; k++) { fs[k] = log1p(agg[k]); fs[6 + k] = agg[k]; }
        if (m->agg_mean) for (int k = 0; k < 12; k++) fs[k] = (fs[k] - m->agg_mean[k]) / m->agg_std[k];
        double z = 0.0;
        for (int k = 0; k < 12; k++) z = z + m->lin_w[k] * fs[k];
        z = z + m->lin_b;
        double pred = softplus(z) * m->out_scale;
        *out = pred > 1e-9 ? pred : 1e-9;
    } else if (m->variant == VAR_MP) { /* estimator.py:321-389 */
        int h = m->hidden, F = m->feat_dim;
        double *x = (double *)xcalloc((size_t)n * F, sizeof(double));
        for (int i = 0; i < n; i++) {
            int v = mem[i];
            double c = s->op_prof[v], in = (double)s->in_bytes[v], o = (double)s->op_out_bytes[v];
            x[i * F + 0] = log1p(c); x[i * F + 1] = c;
            x[i * F + 2] = log1p(in); x[i * F + 3] = in;
            x[i * F + 4] = log1p(o); x[i * F + 5] = o;
            int slot = s->op_slot[v];
            if (6 + slot < F) x[i * F + 6 + slot] = 1.0;
            if (m->node_mean)
                for (int k = 0; k < F; k++) x[i * F + k] = (x[i * F + k] - m->node_mean[k]) / m->node_std[k];
        }
        /* mean aggregation matrix (estimator.py:348-355) */
        double *M = (double *)xcalloc((size_t)n * n, sizeof(double));
        for (int i = 0; i < n; i++) M[i * n + i] = 1.0;
        for (int k = 0; k < ne; k++) { M[ls[k] * n + ld[k]] = 1.0; M[ld[k] * n + ls[k]] = 1.0; }
        for (int i = 0; i < n; i++) {
            double rs = 0.0;
            for (int j = 0; j < n; j++) rs += M[i * n + j];
            for (int j = 0; j < n; j++) M[i * n + j] /= rs;
        }
        double *H = (double *)xmalloc(sizeof(double) * (size_t)n * h);
        double *P = (double *)xmalloc(sizeof(double) * (size_t)n * h);
        for (int i = 0; i < n; i++)
            for (int c = 0; c < h; c++) {
                double acc = 0.0;
                for (int k = 0; k < F; k++) acc += x[i * F + k] * m->W_emb[c * F + k];
                H[i * h + c] = acc;
            }
        for (int l = 0; l < m->layers; l++) {
            const double *W = m->W_layer + (size_t)l * h * h;
            for (int i = 0; i < n; i++)
                for (int c = 0; c < h; c++) {
                    double acc = 0.0;
                    for (int j = 0; j < n; j++) acc += M[i * n + j] * H[j * h + c];
                    P[i * h + c] = acc;
                }
            for (int i = 0; i < n; i++)
                for (int c = 0; c < h; c++) {
                    double acc = 0.0;
                    for (int k = 0; k < h; k++) acc += P[i * h + k] * W[c * h + k];
                    H[i * h + c] = acc > 0.0 ? acc : 0.0;
                }
        }
        double *sv = (double *)xcalloc((size_t)h, sizeof(double));
        double *r = (double *)xmalloc(sizeof(double) * (size_t)h);
        double *d1 = (double *)xmalloc(sizeof(double) * (size_t)h);
        double *d2 = (double *)xmalloc(sizeof(double) * (size_t)h);
        for (int i = 0; i < n; i++) for (int c = 0; c < h; c++) sv[c] += H[i * h + c];
        for (int c = 0; c < h; c++) {
            double acc = 0.0;
            for (int k = 0; k < h; k++) acc += m->W_r[c * h + k] * sv[k];
            r[c] = acc > 0.0 ? acc : 0.0;
        }
        for (int c = 0; c < h; c++) {
            double acc = 0.0;
            for (int k = 0; k < h; k++) acc += m->A1[c * h + k] * r[k];
            acc += m->c1[c];
            d1[c] = acc > 0.0 ? acc : 0.0;
        }
        for (int c = 0; c < h; c++) {
            double acc = 0.0;
            for (int k = 0; k < h; k++) acc += m->A2[c * h + k] * d1[k];
            acc += m->c2[c];
            d2[c] = acc > 0.0 ? acc : 0.0;
        }
        double z = 0.0;
        for (int k = 0; k < h; k++) z += m->a3[k] * d2[k];
        z += m->c3;
        double pred = softplus(z) * m->out_scale;
        *out = pred > 1e-9 ? pred : 1e-9;
        free(x); free(M); free(H); free(P); free(sv); free(r); free(d1); free(d2);
    } else {
        st = ORC_MISSING_COST;
    }
    free(ls); free(ld);
    return st;
}

/* durations of every schedule node, in node order; the first failing node
 * decides the status (simulator.py:38-50, :62).  Returns status; *bad = node. */
static int node_durations(const orc_static *s, const orc_model *m, const orc_index *ix, double *dur, int *bad) {
    int G = ix->G;
    int64_t *io_int = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(G + 1));
    int64_t *io_in = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(G + 1));
    int64_t *io_out = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(G + 1));
    group_io(s, ix, io_int, io_in, io_out);
    int st = ORC_OK;
    *bad = -1;
    for (int g = 0; g < G && st == ORC_OK; g++) {
        int n = ix->mptr[g + 1] - ix->mptr[g];
        const int32_t *mem = ix->mem + ix->mptr[g];
        double d = 0.0;
        if (m->provider == PROV_HW_ORACLE) { /* oracle_time, noise 0 (workloads.py:276-291) */
            int all_param = 1;
            pysum_t acc = {0.0, 0.0, 0};
            for (int i = 0; i < n; i++) {
                if (s->op_kind[mem[i]] != KIND_PARAMETER) all_param = 0;
                double c = s->op_compute[mem[i]];
                pysum_add(&acc, isnan(c) ? 0.0 : c);
            }
            d = all_param ? 0.0 : (pysum_get(&acc) + m->launch) + m->mem * (double)(io_in[g] + io_out[g]);
        } else if (n == 1) { /* estimator.py:810-814 */
            int v = mem[0];
            if (s->op_kind[v] == KIND_PARAMETER) d = 0.0;
            else if (isnan(s->op_prof[v])) st = ORC_MISSING_COST;
            else d = s->op_prof[v];
        } else {
            if (m->variant == VAR_NONE) st = ORC_MISSING_COST; /* estimator.py:815-818 */
            else st = predict_group(s, m, ix, g, io_int, io_in, io_out, &d);
        }
        if (st == ORC_OK && d < 0) st = ORC_NEGATIVE_DURATION;
        if (st != ORC_OK) *bad = g;
        dur[g] = d;
    }
    for (int b = 0; b < ix->B && st == ORC_OK; b++) { /* estimator.py:821-822 -> comm.py:45-49 */
        int64_t tot = 0;
        for (int k = ix->bptr[b]; k < ix->bptr[b + 1]; k++) tot += s->ar_bytes[ix->bmem[k]];
        double d = m->comm_C * (double)tot + m->comm_D;
        if (d < 0) { st = ORC_NEGATIVE_DURATION; *bad = G + b; }
        dur[G + b] = d;
    }
    free(io_int); free(io_in); free(io_out);
    return st;
}

/* ------------------------------------------------------------------------ */
/* simulator (simulator.py:53-140)                                           */

typedef struct { double k0; int64_t k1; int32_t k2; } hent_t; /* (rt|end, tiebreak|seq, node) */

static int hless(const hent_t *a, const hent_t *b) {
    if (a->k0 != b->k0) return a->k0 < b->k0;
    if (a->k1 != b->k1) return a->k1 < b->k1;
    return a->k2 < b->k2;
}
typedef struct { hent_t *v; int n; } heap_t;
static void hpush(heap_t *h, hent_t e) {
    int i = h->n++;
    h->v[i] = e;
    while (i > 0) {
        int p = (i - 1) >> 1;
        if (!hless(&h->v[i], &h->v[p])) break;
        hent_t t = h->v[i]; h->v[i] = h->v[p]; h->v[p] = t; i = p;
    }
}
static hent_t hpop(heap_t *h) {
    hent_t top = h->v[0];
    h->v[0] = h->v[--h->n];
    int i = 0;
    for (;;) {
        int l = 2 * i + 1, r = l + 1, m = i;
        if (l < h->n && hless(&h->v[l], &h->v[m])) m = l;
        if (r < h->n && hless(&h->v[r], &h->v[m])) m = r;
        if (m == i) break;
        hent_t t = h->v[i]; h->v[i] = h->v[m]; h->v[m] = t; i = m;
    }
    return top;
}

typedef struct {
    int32_t *c_id; double *c_start, *c_end; int32_t n_c; /* compute events */
    int32_t *b_id; double *b_start, *b_end; int32_t n_b; /* comm events */
} orc_timeline;

static int simulate_nodes(const orc_index *ix, const int32_t *dptr, const int32_t *dep, const double *dur,
                          const int64_t *tb, double *makespan, orc_timeline *tl) {
    int G = ix->G, N = ix->G + ix->B;
    int st = ORC_OK;
    int32_t *indeg = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(N + 1));
    pair_t *rp = (pair_t *)xmalloc(sizeof(pair_t) * (size_t)(dptr[N] + 1));
    for (int v = 0; v < N; v++) {
        indeg[v] = dptr[v + 1] - dptr[v];
        for (int k = dptr[v]; k < dptr[v + 1]; k++) { rp[k].a = dep[k]; rp[k].b = v; }
    }
    int32_t *sptr, *succ;
    pairs_to_csr(rp, dptr[N], N, &sptr, &succ, NULL);
    free(rp);
    double *finish = (double *)xmalloc(sizeof(double) * (size_t)(N + 1));
    heap_t ready[2], comp;
    ready[0].v = (hent_t *)xmalloc(sizeof(hent_t) * (size_t)(N + 1)); ready[0].n = 0;
    ready[1].v = (hent_t *)xmalloc(sizeof(hent_t) * (size_t)(N + 1)); ready[1].n = 0;
    comp.v = (hent_t *)xmalloc(sizeof(hent_t) * 4); comp.n = 0;
    for (int v = 0; v < N; v++)
        if (indeg[v] == 0) {
            hent_t e = {0.0, tb[v], v};
            hpush(&ready[v >= G], e);
        }
    int running[2] = {-1, -1};
    int64_t seq = 0;
    int done = 0;
    double now = 0.0, mk = 0.0;
    if (tl) { tl->n_c = 0; tl->n_b = 0; }
    while (done < N) {
        while (comp.n && comp.v[0].k0 <= now) { /* simulator.py:122-125 */
            hent_t c = hpop(&comp);
            int node = c.k2;
            running[node >= G] = -1;
            finish[node] = c.k0;
            done++;
            for (int k = sptr[node]; k < sptr[node + 1]; k++) { /* finish_node, simulator.py:88-96 */
                int sc = succ[k];
                if (--indeg[sc] == 0) {
                    double rt = 0.0;
                    for (int q = dptr[sc]; q < dptr[sc + 1]; q++) if (finish[dep[q]] > rt) rt = finish[dep[q]];
                    hent_t e = {rt, tb[sc], sc};
                    hpush(&ready[sc >= G], e);
                }
            }
        }
        if (done >= N) break;
        int started = 0;
        for (int lane = 0; lane < 2; lane++) { /* start_available, simulator.py:98-115 */
            if (running[lane] < 0 && ready[lane].n) {
                hent_t r = hpop(&ready[lane]);
                int node = r.k2;
                double start = now > r.k0 ? now : r.k0;
                double end = start + dur[node];
                running[lane] = node;
                if (end > mk) mk = end;
                if (tl) {
                    if (lane == 0) { tl->c_id[tl->n_c] = ix->gid[node]; tl->c_start[tl->n_c] = start; tl->c_end[tl->n_c++] = end; }
                    else { tl->b_id[tl->n_b] = ix->bid[node - G]; tl->b_start[tl->n_b] = start; tl->b_end[tl->n_b++] = end; }
                }
                hent_t c = {end, seq++, node};
                hpush(&comp, c);
                started = 1;
            }
        }
        if (started) continue;
        if (comp.n) { now = comp.v[0].k0; continue; }
        st = ORC_CYCLE; /* simulator.py:133 */
        break;
    }
    *makespan = st == ORC_OK ? mk : 0.0;
    free(indeg); free(sptr); free(succ); free(finish); free(ready[0].v); free(ready[1].v); free(comp.v);
    return st;
}

/* cost() of one candidate (simulator.py:143-145).  tl may be NULL; if set its
 * arrays must hold >= V+V / A entries.  Returns status. */
int orc_cost(const orc_static *s, const orc_model *m, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt,
             double *cost_out, orc_timeline *tl, int32_t *bad_node_id) {
    orc_index ix;
    index_build(s, ngid, rgid, bkt, &ix);
    int N = ix.G + ix.B;
    int32_t *dptr, *dep;
    schedule_deps(s, &ix, &dptr, &dep);
    double *dur = (double *)xmalloc(sizeof(double) * (size_t)(N + 1));
    int bad;
    int st = node_durations(s, m, &ix, dur, &bad);
    if (bad_node_id) *bad_node_id = bad < 0 ? -1 : (bad < ix.G ? ix.gid[bad] : ix.bid[bad - ix.G]);
    double mk = 0.0;
    if (st == ORC_OK) {
        int64_t *tb = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(N + 1));
        for (int g = 0; g < ix.G; g++) tb[g] = ix.mem[ix.mptr[g]]; /* min member (simulator.py:63) */
        for (int b = 0; b < ix.B; b++) tb[ix.G + b] = ix.bmem[ix.bptr[b]]; /* min AR (simulator.py:64) */
        st = simulate_nodes(&ix, dptr, dep, dur, tb, &mk, tl);
        free(tb);
    }
    *cost_out = mk;
    free(dptr); free(dep); free(dur);
    index_free(&ix);
    return st;
}

/* Batch scoring: K candidates laid out [K x V], [K x V], [K x A]. */
void orc_cost_batch(const orc_static *s, const orc_model *m, const int32_t *ngid, const int32_t *rgid,
                    const int32_t *bkt, int32_t K, double *cost_out, int32_t *status_out) {
    for (int i = 0; i < K; i++)
        status_out[i] = orc_cost(s, m, ngid + (size_t)i * s->V, rgid + (size_t)i * s->V, bkt + (size_t)i * s->A,
                                 &cost_out[i], NULL, NULL);
}

/* Per-group durations (node order: groups by id, then buckets by id) for the
 * estimator parity tests.  gid_out/bid_out receive the ids; returns G + B or
 * -status. */
int orc_node_durations(const orc_static *s, const orc_model *m, const int32_t *ngid, const int32_t *rgid,
                       const int32_t *bkt, int32_t *gid_out, int32_t *bid_out, double *dur_out, int32_t *G_out,
                       int64_t *io_out3) {
    orc_index ix;
    index_build(s, ngid, rgid, bkt, &ix);
    int bad;
    int st = node_durations(s, m, &ix, dur_out, &bad);
    for (int g = 0; g < ix.G; g++) gid_out[g] = ix.gid[g];
    for (int b = 0; b < ix.B; b++) bid_out[b] = ix.bid[b];
    *G_out = ix.G;
    if (io_out3) {
        int64_t *a = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(ix.G + 1));
        int64_t *b = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(ix.G + 1));
        int64_t *c = (int64_t *)xmalloc(sizeof(int64_t) * (size_t)(ix.G + 1));
        group_io(s, &ix, a, b, c);
        for (int g = 0; g < ix.G; g++) { io_out3[3 * g] = a[g]; io_out3[3 * g + 1] = b[g]; io_out3[3 * g + 2] = c[g]; }
        free(a); free(b); free(c);
    }
    int n = ix.G + ix.B;
    index_free(&ix);
    return st == ORC_OK ? n : -st;
}

/* ------------------------------------------------------------------------ */
/* CPython random.Random: MT19937 + init_by_array + _randbelow
 * (search.py:88, :119; rewrite.py:250)                                     */

typedef struct { uint32_t mt[624]; int mti; } orc_rng;

static void mt_init_genrand(orc_rng *r, uint32_t s) {
    r->mt[0] = s;
    for (int i = 1; i < 624; i++) r->mt[i] = 1812433253U * (r->mt[i - 1] ^ (r->mt[i - 1] >> 30)) + (uint32_t)i;
    r->mti = 624;
}
static void mt_init_by_array(orc_rng *r, const uint32_t *key, int len) {
    mt_init_genrand(r, 19650218U);
    int i = 1, j = 0;
    int k = 624 > len ? 624 : len;
    for (; k; k--) {
        r->mt[i] = (r->mt[i] ^ ((r->mt[i - 1] ^ (r->mt[i - 1] >> 30)) * 1664525U)) + key[j] + (uint32_t)j;
        i++; j++;
        if (i >= 624) { r->mt[0] = r->mt[623]; i = 1; }
        if (j >= len) j = 0;
    }
    for (k = 623; k; k--) {
        r->mt[i] = (r->mt[i] ^ ((r->mt[i - 1] ^ (r->mt[i - 1] >> 30)) * 1566083941U)) - (uint32_t)i;
        i++;
        if (i >= 624) { r->mt[0] = r->mt[623]; i = 1; }
    }
    r->mt[0] = 0x80000000U;
}
static uint32_t mt_next(orc_rng *r) {
    static const uint32_t mag01[2] = {0x0U, 0x9908b0dfU};
    uint32_t y;
    if (r->mti >= 624) {
        int kk;
        for (kk = 0; kk < 624 - 397; kk++) {
            y = (r->mt[kk] & 0x80000000U) | (r->mt[kk + 1] & 0x7fffffffU);
            r->mt[kk] = r->mt[kk + 397] ^ (y >> 1) ^ mag01[y & 1U];
        }
        for (; kk < 623; kk++) {
            y = (r->mt[kk] & 0x80000000U) | (r->mt[kk + 1] & 0x7fffffffU);
            r->mt[kk] = r->mt[kk + (397 - 624)] ^ (y >> 1) ^ mag01[y & 1U];
        }
        y = (r->mt[623] & 0x80000000U) | (r->mt[0] & 0x7fffffffU);
        r->mt[623] = r->mt[396] ^ (y >> 1) ^ mag01[y & 1U];
        r->mti = 0;
    }
    y = r->mt[r->mti++];
    y ^= (y >> 11);
    y ^= (y << 7) & 0x9d2c5680U;
    y ^= (y << 15) & 0xefc60000U;
    y ^= (y >> 18);
    return y;
}
void orc_rng_seed(orc_rng *r, uint64_t seed) { /* random_seed() for a non-negative int */
    uint32_t key[2];
    int len = 0;
    key[len++] = (uint32_t)(seed & 0xffffffffU);
    if (seed >> 32) key[len++] = (uint32_t)(seed >> 32);
    mt_init_by_array(r, key, len);
}
uint32_t orc_rng_getrandbits(orc_rng *r, int k) { return mt_next(r) >> (32 - k); } /* 1 <= k <= 32 */
uint32_t orc_rng_randbelow(orc_rng *r, uint32_t n) {
    int k = 0;
    for (uint32_t t = n; t; t >>= 1) k++;
    uint32_t v = orc_rng_getrandbits(r, k);
    while (v >= n) v = orc_rng_getrandbits(r, k);
    return v;
}
int32_t orc_rng_size(void) { return (int32_t)sizeof(orc_rng); }

/* ------------------------------------------------------------------------ */
/* rewrites (rewrite.py:45-263)                                              */

typedef struct {
    orc_index ix;
    int32_t *sptr, *succ; /* contracted succs per group (graph.py:161-171), group index order */
    int32_t *pptr, *pred; /* contracted preds (graph.py:173-179) */
    uint8_t *compute_ok;  /* rewrite.py:45-46 */
    uint8_t *has_dup;
} orc_adj;

static void adj_build(const orc_static *s, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, orc_adj *a) {
    index_build(s, ngid, rgid, bkt, &a->ix);
    orc_index *ix = &a->ix;
    pair_t *p = (pair_t *)xmalloc(sizeof(pair_t) * (2 * (size_t)s->E + 1));
    int n = 0;
    for (int e = 0; e < s->E; e++) {
        int src = s->e_src[e], dst = s->e_dst[e];
        int sg = export_gi(ix, src);
        int copies[2] = {ix->ngi[dst], ix->rgi[dst]};
        for (int c = 0; c < 2; c++) {
            int g = copies[c];
            if (g < 0 || in_group(ix, src, g)) continue;
            p[n].a = sg; p[n].b = g; n++;
        }
    }
    pairs_to_csr(p, n, ix->G, &a->sptr, &a->succ, NULL);
    for (int i = 0; i < n; i++) { int t = p[i].a; p[i].a = p[i].b; p[i].b = t; }
    pairs_to_csr(p, n, ix->G, &a->pptr, &a->pred, NULL);
    free(p);
    a->compute_ok = (uint8_t *)xmalloc((size_t)ix->G + 1);
    a->has_dup = (uint8_t *)xmalloc((size_t)ix->G + 1);
    for (int g = 0; g < ix->G; g++) {
        a->compute_ok[g] = 1;
        a->has_dup[g] = 0;
        for (int k = ix->mptr[g]; k < ix->mptr[g + 1]; k++) {
            if (s->op_kind[ix->mem[k]] != KIND_COMPUTE) a->compute_ok[g] = 0;
            if (ix->mdup[k]) a->has_dup[g] = 1;
        }
    }
}
static void adj_free(orc_adj *a) {
    index_free(&a->ix);
    free(a->sptr); free(a->succ); free(a->pptr); free(a->pred); free(a->compute_ok); free(a->has_dup);
}

static int state_valid(const orc_static *s, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt) {
    /* rewrite_candidate_ok (graph.py:505-512) */
    orc_index ix;
    index_build(s, ngid, rgid, bkt, &ix);
    int32_t *dptr, *dep;
    schedule_deps(s, &ix, &dptr, &dep);
    int ok = deps_acyclic(ix.G + ix.B, dptr, dep);
    free(dptr); free(dep);
    index_free(&ix);
    return ok;
}

/* fusible_pairs (rewrite.py:49-61) with the DUP filter (rewrite.py:242-247).
 * Returns the count; if want >= 0 stores that pair. */
static int fusible_pairs(const orc_adj *a, int dup_filter, int want, int *og, int *pg) {
    int cnt = 0;
    for (int g = 0; g < a->ix.G; g++) {
        if (!a->compute_ok[g]) continue;
        for (int k = a->pptr[g]; k < a->pptr[g + 1]; k++) {
            int p = a->pred[k];
            if (!a->compute_ok[p]) continue;
            if (dup_filter && a->has_dup[p]) continue;
            if (cnt == want) { *og = g; *pg = p; }
            cnt++;
        }
    }
    return cnt;
}

/* neighbors_allreduce (rewrite.py:156-178): marks[] over bucket indices */
static void neighbors(const orc_static *s, const orc_adj *a, int b, uint8_t *gmark, uint8_t *bmark) {
    const orc_index *ix = &a->ix;
    memset(gmark, 0, (size_t)ix->G + 1);
    memset(bmark, 0, (size_t)ix->B + 1);
    for (int k = ix->bptr[b]; k < ix->bptr[b + 1]; k++) {
        int g = export_gi(ix, s->ar_prod[ix->bmem[k]]);
        gmark[g] = 1;
    }
    /* nearby = own | succs(own) | preds(own) */
    uint8_t *own = (uint8_t *)xmalloc((size_t)ix->G + 1);
    memcpy(own, gmark, (size_t)ix->G + 1);
    for (int g = 0; g < ix->G; g++) {
        if (!own[g]) continue;
        for (int k = a->sptr[g]; k < a->sptr[g + 1]; k++) gmark[a->succ[k]] = 1;
        for (int k = a->pptr[g]; k < a->pptr[g + 1]; k++) gmark[a->pred[k]] = 1;
    }
    free(own);
    for (int o = 0; o < ix->B; o++) {
        if (o == b) continue;
        for (int k = ix->bptr[o]; k < ix->bptr[o + 1]; k++)
            if (gmark[export_gi(ix, s->ar_prod[ix->bmem[k]])]) { bmark[o] = 1; break; }
    }
}

/* bucket_pairs (rewrite.py:212-219) */
static int bucket_pairs(const orc_static *s, const orc_adj *a, int want, int *bo, int *bn) {
    int cnt = 0;
    uint8_t *gm = (uint8_t *)xmalloc((size_t)a->ix.G + 1);
    uint8_t *bm = (uint8_t *)xmalloc((size_t)a->ix.B + 1);
    for (int b = 0; b < a->ix.B; b++) {
        neighbors(s, a, b, gm, bm);
        for (int o = 0; o < a->ix.B; o++) {
            if (!bm[o]) continue;
            if (cnt == want) { *bo = b; *bn = o; }
            cnt++;
        }
    }
    free(gm); free(bm);
    return cnt;
}

#define M_NONDUP 0
#define M_DUP 1
#define M_AR 2

/* fuse_nondup (rewrite.py:64-96); writes the candidate into (n2, r2).  */
static int fuse_nondup(const orc_static *s, const orc_adj *a, int og, int pg, const int32_t *ng, const int32_t *rg,
                       const int32_t *bk, int32_t *n2, int32_t *r2) {
    const orc_index *ix = &a->ix;
    if (og == pg) return 0;
    for (int v = 0; v < s->V; v++) /* groups share a member (rewrite.py:76-79) */
        if (in_group(ix, v, og) && in_group(ix, v, pg)) return 0;
    if (!a->compute_ok[og] || !a->compute_ok[pg]) return 0;
    int32_t merged = ix->gid[og] < ix->gid[pg] ? ix->gid[og] : ix->gid[pg];
    for (int v = 0; v < s->V; v++) {
        n2[v] = (ix->ngi[v] == og || ix->ngi[v] == pg) ? merged : ng[v];
        r2[v] = (ix->rgi[v] >= 0 && (ix->rgi[v] == og || ix->rgi[v] == pg)) ? merged : rg[v];
    }
    return state_valid(s, n2, r2, bk);
}

/* fuse_dup (rewrite.py:99-153) */
static int fuse_dup(const orc_static *s, const orc_adj *a, int og, int pg, const int32_t *ng, const int32_t *rg,
                    const int32_t *bk, int32_t *n2, int32_t *r2) {
    const orc_index *ix = &a->ix;
    if (og == pg) return 0;
    for (int v = 0; v < s->V; v++)
        if (in_group(ix, v, og) && in_group(ix, v, pg)) return 0;
    if (!a->compute_ok[og] || !a->compute_ok[pg]) return 0;
    int feeds_ar = 0;
    for (int k = ix->mptr[pg]; k < ix->mptr[pg + 1]; k++) {
        int v = ix->mem[k];
        if (ix->rgi[v] >= 0) return 0; /* rewrite.py:116-118 */
        if (s->arp_ptr[v + 1] > s->arp_ptr[v]) feeds_ar = 1;
    }
    int other = 0;
    for (int k = a->sptr[pg]; k < a->sptr[pg + 1]; k++)
        if (a->succ[k] != og) other = 1;
    if (!other && !feeds_ar) return fuse_nondup(s, a, og, pg, ng, rg, bk, n2, r2); /* rewrite.py:124-130 */
    int32_t merged = ix->gid[og] < ix->gid[pg] ? ix->gid[og] : ix->gid[pg];
    int32_t replica = ix->gid[ix->G - 1] + 1; /* rewrite.py:138 */
    for (int v = 0; v < s->V; v++) {
        n2[v] = ng[v];
        r2[v] = rg[v];
        if (ix->ngi[v] == og) n2[v] = merged;
        if (ix->rgi[v] >= 0 && ix->rgi[v] == og) r2[v] = merged;
        if (ix->ngi[v] == pg) { n2[v] = merged; r2[v] = replica; }
    }
    return state_valid(s, n2, r2, bk);
}

/* fuse_allreduce (rewrite.py:181-209) */
static int fuse_ar(const orc_static *s, const orc_adj *a, int bo, int bn, const int32_t *ng, const int32_t *rg,
                   const int32_t *bk, int32_t *b2) {
    const orc_index *ix = &a->ix;
    int32_t merged = ix->bid[bo] < ix->bid[bn] ? ix->bid[bo] : ix->bid[bn];
    for (int k = 0; k < s->A; k++) b2[k] = (ix->bki[k] == bo || ix->bki[k] == bn) ? merged : bk[k];
    return state_valid(s, ng, rg, b2);
}

/* random_apply (rewrite.py:222-263): state updated in place; returns applied_any */
int orc_random_apply(const orc_static *s, int32_t *ng, int32_t *rg, int32_t *bk, int method, int n, orc_rng *r) {
    int V = s->V, A = s->A;
    int32_t *n2 = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(V + 1));
    int32_t *r2 = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(V + 1));
    int32_t *b2 = (int32_t *)xmalloc(sizeof(int32_t) * (size_t)(A + 1));
    int applied = 0;
    for (int it = 0; it < n; it++) {
        orc_adj a;
        adj_build(s, ng, rg, bk, &a);
        int x = -1, y = -1, cnt;
        if (method == M_AR) cnt = bucket_pairs(s, &a, -1, &x, &y);
        else cnt = fusible_pairs(&a, method == M_DUP, -1, &x, &y);
        if (cnt == 0) { adj_free(&a); break; }
        int idx = (int)orc_rng_randbelow(r, (uint32_t)cnt);
        if (method == M_AR) bucket_pairs(s, &a, idx, &x, &y);
        else fusible_pairs(&a, method == M_DUP, idx, &x, &y);
        int ok;
        if (method == M_NONDUP) ok = fuse_nondup(s, &a, x, y, ng, rg, bk, n2, r2);
        else if (method == M_DUP) ok = fuse_dup(s, &a, x, y, ng, rg, bk, n2, r2);
        else ok = fuse_ar(s, &a, x, y, ng, rg, bk, b2);
        if (ok) {
            if (method == M_AR) memcpy(bk, b2, sizeof(int32_t) * (size_t)A);
            else { memcpy(ng, n2, sizeof(int32_t) * (size_t)V); memcpy(rg, r2, sizeof(int32_t) * (size_t)V); }
            applied = 1;
        }
        adj_free(&a);
    }
    free(n2); free(r2); free(b2);
    return applied;
}

/* candidate i of the random batch: Random(seed), then nondup, dup, ar with
 * n = randint(0, beta) each, accumulating. */
void orc_make_candidate(const orc_static *s, uint64_t seed, int beta, int32_t *ng, int32_t *rg, int32_t *bk) {
    orc_rng r;
    orc_rng_seed(&r, seed);
    for (int m = 0; m < 3; m++) {
        int n = (int)orc_rng_randbelow(&r, (uint32_t)beta + 1);
        orc_random_apply(s, ng, rg, bk, m, n, &r);
    }
}

/* ------------------------------------------------------------------------ */
/* canonical state hash: equality semantics of canonical_hash (graph.py:559-580)
 * for a fixed graph -- the state is the set of (members, duplicated) group
 * tuples plus the set of bucket member tuples; ids are canonicalised away.   */

static uint64_t mix64(uint64_t x) {
    x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27; x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}
uint64_t orc_state_hash(const orc_static *s, const int32_t *ng, const int32_t *rg, const int32_t *bk) {
    orc_index ix;
    index_build(s, ng, rg, bk, &ix);
    uint64_t h = 0x9e3779b97f4a7c15ULL;
    for (int g = 0; g < ix.G; g++) {
        uint64_t gh = 0x1234567ULL;
        for (int k = ix.mptr[g]; k < ix.mptr[g + 1]; k++)
            gh = mix64(gh ^ ((uint64_t)(ix.mem[k] + 1) * 2 + ix.mdup[k]));
        h += mix64(gh + 0x51ULL);
    }
    for (int b = 0; b < ix.B; b++) {
        uint64_t bh = 0x7654321ULL;
        for (int k = ix.bptr[b]; k < ix.bptr[b + 1]; k++) bh = mix64(bh ^ (uint64_t)(ix.bmem[k] + 1));
        h += mix64(bh + 0xb7ULL);
    }
    index_free(&ix);
    return h;
}

/* ------------------------------------------------------------------------ */
/* backtracking search, Alg. 1 (search.py:84-155)                           */

typedef struct {
    double alpha;
    int32_t beta, max_unchanged, methods_mask; /* bit m = method m enabled */
    uint64_t seed;
    int64_t max_steps; /* 0 = unlimited (stands in for time_budget_s) */
} orc_search_cfg;

typedef struct {
    int32_t step; int8_t method; double cost, best; int32_t queue_len; int8_t enqueued;
} orc_trace_rec;

typedef struct { uint64_t key; double val; uint8_t used; } hs_ent;
typedef struct { hs_ent *t; size_t cap, n; } hset;
static void hs_init(hset *h) { h->cap = 1024; h->n = 0; h->t = (hs_ent *)xcalloc(h->cap, sizeof(hs_ent)); }
static hs_ent *hs_find(hset *h, uint64_t k, int insert) {
    if (insert && (h->n + 1) * 2 > h->cap) {
        hset nh; nh.cap = h->cap * 2; nh.n = 0; nh.t = (hs_ent *)xcalloc(nh.cap, sizeof(hs_ent));
        for (size_t i = 0; i < h->cap; i++)
            if (h->t[i].used) { hs_ent *e = hs_find(&nh, h->t[i].key, 1); e->val = h->t[i].val; }
        free(h->t); *h = nh;
    }
    size_t i = (size_t)mix64(k) & (h->cap - 1);
    while (h->t[i].used) {
        if (h->t[i].key == k) return &h->t[i];
        i = (i + 1) & (h->cap - 1);
    }
    if (!insert) return NULL;
    h->t[i].used = 1; h->t[i].key = k; h->n++;
    return &h->t[i];
}

typedef struct { double c; int64_t seq; uint64_t h; int32_t slot; } qent_t;
static int qless(const qent_t *a, const qent_t *b) {
    if (a->c != b->c) return a->c < b->c;
    return a->seq < b->seq; /* seq unique -> never compares h / graph */
}

/* Returns status; writes best state, counters and up to trace_cap records. */
int orc_search(const orc_static *s, const orc_model *m, const orc_search_cfg *cfg, int32_t *best_ng, int32_t *best_rg,
               int32_t *best_bk, double *best_cost_out, int64_t *counters /* steps, evaluated, enqueued, n_trace */,
               orc_trace_rec *trace, int64_t trace_cap) {
    int V = s->V, A = s->A;
    size_t W = (size_t)(2 * V + A);
    size_t pool_cap = 256, pool_n = 0;
    int32_t *pool = (int32_t *)xmalloc(sizeof(int32_t) * W * pool_cap);
    orc_rng rng;
    orc_rng_seed(&rng, cfg->seed);
    hset cache, seen;
    hs_init(&cache); hs_init(&seen);
    int64_t evaluated = 0, enq = 0, steps = 0, ntr = 0;
    int st = ORC_OK;
    /* g0 = default state passed in best_* */
    memcpy(pool, best_ng, sizeof(int32_t) * V);
    memcpy(pool + V, best_rg, sizeof(int32_t) * V);
    memcpy(pool + 2 * V, best_bk, sizeof(int32_t) * A);
    pool_n = 1;
    uint64_t h0 = orc_state_hash(s, pool, pool + V, pool + 2 * V);
    double c0;
    st = orc_cost(s, m, pool, pool + V, pool + 2 * V, &c0, NULL, NULL);
    if (st) goto done;
    evaluated = 1;
    hs_find(&cache, h0, 1)->val = c0;
    hs_find(&seen, h0, 1);
    double best = c0;
    int32_t best_slot = 0;
    size_t qcap = 1024;
    qent_t *q = (qent_t *)xmalloc(sizeof(qent_t) * qcap);
    int qn = 0;
    int64_t qseq = 1;
    q[qn++] = (qent_t){c0, 0, h0, 0};
    int unchanged = 0;
    int32_t *cand = (int32_t *)xmalloc(sizeof(int32_t) * W);
    while (qn && unchanged < cfg->max_unchanged) {
        if (cfg->max_steps && steps >= cfg->max_steps) break;
        /* heappop */
        qent_t cur = q[0];
        q[0] = q[--qn];
        for (int i = 0;;) {
            int l = 2 * i + 1, r = l + 1, mm = i;
            if (l < qn && qless(&q[l], &q[mm])) mm = l;
            if (r < qn && qless(&q[r], &q[mm])) mm = r;
            if (mm == i) break;
            qent_t t = q[i]; q[i] = q[mm]; q[mm] = t; i = mm;
        }
        steps++;
        int requeued = 0;
        for (int meth = 0; meth < 3; meth++) {
            if (!(cfg->methods_mask & (1 << meth))) continue;
            int n = (int)orc_rng_randbelow(&rng, (uint32_t)cfg->beta + 1);
            memcpy(cand, pool + W * (size_t)cur.slot, sizeof(int32_t) * W);
            int applied = orc_random_apply(s, cand, cand + V, cand + 2 * V, meth, n, &rng);
            uint64_t h = applied ? orc_state_hash(s, cand, cand + V, cand + 2 * V) : cur.h;
            hs_ent *ce = hs_find(&cache, h, 0);
            double c;
            if (ce) c = ce->val;
            else {
                st = orc_cost(s, m, cand, cand + V, cand + 2 * V, &c, NULL, NULL);
                if (st) { free(q); free(cand); goto done; }
                hs_find(&cache, h, 1)->val = c;
                evaluated++;
            }
            int slot = -1;
            if (c < best) {
                best = c;
                if (pool_n == pool_cap) { pool_cap *= 2; pool = (int32_t *)realloc(pool, sizeof(int32_t) * W * pool_cap); }
                memcpy(pool + W * pool_n, cand, sizeof(int32_t) * W);
                slot = (int)pool_n++;
                best_slot = slot;
                unchanged = 0;
            } else unchanged++;
            int entered = 0;
            if (c <= cfg->alpha * best) {
                int push = 0;
                if (!hs_find(&seen, h, 0)) { hs_find(&seen, h, 1); push = 1; enq++; }
                else if (h == cur.h && !requeued) { push = 1; requeued = 1; }
                if (push) {
                    if (slot < 0) {
                        if (pool_n == pool_cap) { pool_cap *= 2; pool = (int32_t *)realloc(pool, sizeof(int32_t) * W * pool_cap); }
                        memcpy(pool + W * pool_n, cand, sizeof(int32_t) * W);
                        slot = (int)pool_n++;
                    }
                    if (qn == (int)qcap) { qcap *= 2; q = (qent_t *)realloc(q, sizeof(qent_t) * qcap); }
                    q[qn] = (qent_t){c, qseq++, h, slot};
                    for (int i = qn++; i > 0;) {
                        int p = (i - 1) >> 1;
                        if (!qless(&q[i], &q[p])) break;
                        qent_t t = q[i]; q[i] = q[p]; q[p] = t; i = p;
                    }
                    entered = 1;
                }
            }
            if (trace && ntr < trace_cap)
                trace[ntr] = (orc_trace_rec){(int32_t)steps, (int8_t)meth, c, best, qn, (int8_t)entered};
            ntr++;
        }
    }
    free(q); free(cand);
    memcpy(best_ng, pool + W * (size_t)best_slot, sizeof(int32_t) * V);
    memcpy(best_rg, pool + W * (size_t)best_slot + V, sizeof(int32_t) * V);
    memcpy(best_bk, pool + W * (size_t)best_slot + 2 * V, sizeof(int32_t) * A);
    *best_cost_out = best;
done:
    counters[0] = steps; counters[1] = evaluated; counters[2] = enq; counters[3] = ntr;
    free(pool); free(cache.t); free(seen.t);
    return st;
}
