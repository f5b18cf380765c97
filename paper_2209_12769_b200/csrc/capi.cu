// capi.cu -- C-ABI entry points (include/disco_b200.h): graph handle, cost
// model upload, batched scoring, single-candidate simulate/timeline.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "fo_internal.h"

namespace fo {

static thread_local std::string g_last_error;
std::atomic<int64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int status, const std::string &msg) {
    g_last_error = msg;
    return status;
}

#define CUDA_TRY(expr)                                                                     \
    do {                                                                                   \
        cudaError_t _e = (expr);                                                           \
        if (_e != cudaSuccess)                                                             \
            return fail(FO_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

int ensure_workspace(fo_graph *g, int VB, int slots, WsLayout *L, bool big, int nws, int alt) {
    *L = ws_layout(g->V, g->E, g->A, VB, g->pairs_max, big ? g->V : kMpCapDefault, nws);
    size_t need = (size_t)L->total * (size_t)slots;
    // alt 0: the handle's workspace, 1: the search's second lane, 2..: submission slots 1..
    char *&buf = big ? g->d_ws_big : (alt >= 2 ? g->sub[alt - 1].ws : alt ? g->d_ws_alt : g->d_ws);
    size_t &have = big ? g->ws_big_bytes : (alt >= 2 ? g->sub[alt - 1].ws_bytes : alt ? g->ws_alt_bytes : g->ws_bytes);
    if (need > have) {
        if (buf) cudaFree(buf);
        buf = nullptr;
        have = 0;
        CUDA_TRY(cudaMalloc(&buf, need));
        have = need;
    }
    return FO_OK;
}

static int launch(fo_graph *g, const void *ngid, const void *rgid, const void *bkt, int idx16, int K, int VB,
                  int precision, double *cost, int32_t *status, const double *ext_dur, TimelineOut tl,
                  double *dur_out, int32_t *bad_out, int32_t *ngroups_out, cudaStream_t stream,
                  const DeltaIn *delta = nullptr, int alt_ws = 0, int first_retry = 0) {
    ScoreGeo geo = score_geometry(g->dg, K, g->num_sms, precision);
    const int nws = score_team_warps(geo);
    WsLayout L = ws_layout(g->V, g->E, g->A, VB, g->pairs_max, kMpCapDefault, nws);
    // bound the per-slot workspace to an HBM budget: 45 % of the device's
    // memory (80 GB on a B200), which keeps one full wave of candidates
    // resident even at 50k ops (~17 MB of scratch each; measured 20.9k ->
    // 67.9k cand/s on configs[4] against the former 16 GB).  FO_WS_BUDGET_GB
    // overrides.
    static const char *wsb = getenv("FO_WS_BUDGET_GB");
    size_t budget = (size_t)16 << 30;
    if (wsb && atoi(wsb) > 0) budget = (size_t)atoi(wsb) << 30;
    else {
        if (!g->mem_total) {  // queried once per handle: it sits on the launch path
            size_t fr = 0;
            if (cudaMemGetInfo(&fr, &g->mem_total) != cudaSuccess) g->mem_total = budget;
        }
        budget = std::max(budget, g->mem_total / 100 * 45);
    }
    const int per_block = score_slots(geo) / geo.grid;
    int max_blocks = (int)std::max<size_t>(1, budget / ((size_t)L.total * per_block));
    geo.grid = std::min(geo.grid, max_blocks);
    int slots = score_slots(geo);
    int st = ensure_workspace(g, VB, slots, &L, false, nws, alt_ws);
    if (st) return st;
    char *wsp = alt_ws >= 2 ? g->sub[alt_ws - 1].ws : alt_ws ? g->d_ws_alt : g->d_ws;
    cudaError_t e = launch_score(g->dg, ngid, rgid, bkt, idx16, K, VB, precision, wsp, L, geo,
                                 cost, status, ext_dur, tl,
                                 dur_out, bad_out, ngroups_out, stream, first_retry, delta);
    g_launches++;
    if (e != cudaSuccess) return fail(FO_CUDA_ERROR, std::string("score kernel launch: ") + cudaGetErrorString(e));
    if (g->V > kMpCapDefault) {
        // second pass, same stream: only candidates whose fused groups exceeded
        // the first pass's estimator scratch, with scratch for whole-graph groups
        WsLayout Lb;
        ScoreGeo gb = geo;
        gb.sm_bytes = 0;
        // latency geometry: a block per candidate, so the very large MP groups
        // (the reason for this pass) run on the whole team (FO_RETRY_TEAM=0: a warp each)
        const char *rt = getenv("FO_RETRY_TEAM");
        gb.team = rt ? rt[0] == '1' : 1;
        const int per_block = gb.team ? 1 : score_warps_per_block();
        gb.grid = gb.team ? std::min(K, 4 * g->num_sms)
                          : std::min(std::max(1, (K + per_block - 1) / per_block), g->num_sms);
        Lb = ws_layout(g->V, g->E, g->A, VB, g->pairs_max, g->V);
        gb.grid = std::min<int>(gb.grid, (int)std::max<size_t>(1, budget / ((size_t)Lb.total * per_block)));
        st = ensure_workspace(g, VB, gb.grid * per_block, &Lb, true, 1);
        if (st) return st;
        e = launch_score(g->dg, ngid, rgid, bkt, idx16, K, VB, precision, g->d_ws_big, Lb, gb, cost, status, ext_dur, tl,
                         dur_out, bad_out, ngroups_out, stream, 1, delta);
        g_launches++;
        if (e != cudaSuccess) return fail(FO_CUDA_ERROR, std::string("score retry launch: ") + cudaGetErrorString(e));
    }
    return FO_OK;
}

int score_device(fo_graph *g, const void *ngid, const void *rgid, const void *bkt, int idx16, int K, int VB,
                 int precision, double *cost, int32_t *status, cudaStream_t stream, int alt_ws) {
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    if (!g->model_set) return fail(FO_INVALID_ARG, "no cost model set (fo_graph_set_cost_model)");
    if (K <= 0) return FO_OK;
    if (VB <= 0) return fail(FO_INVALID_ARG, "gid_bound must be > 0");
    if (idx16 && (VB > 32767 || g->A > 32767)) return fail(FO_INVALID_ARG, "int16 encoding needs gid_bound and A <= 32767");
    CUDA_TRY(cudaSetDevice(g->device));
    TimelineOut tl{};
    return launch(g, ngid, rgid, bkt, idx16, K, VB, precision, cost, status, nullptr, tl, nullptr, nullptr, nullptr,
                  stream, nullptr, alt_ws);
}

// sparse candidates against the resident parent (fo_set_parent).  slot k > 0:
// submission slot k's own scratch (incremental workspace, estimator queue,
// memo tables, general-kernel workspace), so batches can run on several
// streams at once (fo_score_delta_submit).
int score_delta_device(fo_graph *g, const int32_t *off, const int32_t *chg, int K, int precision, double *cost,
                       int32_t *status, cudaStream_t stream, int slot) {
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    if (!g->model_set) return fail(FO_INVALID_ARG, "no cost model set (fo_graph_set_cost_model)");
    if (!g->d_parent) return fail(FO_INVALID_ARG, "no parent state set (fo_set_parent)");
    if (K <= 0) return FO_OK;
    CUDA_TRY(cudaSetDevice(g->device));
    // the slot's memo tables stand in for the handle's while this batch is
    // launched (kernel arguments are copied at launch)
    MemoEnt *memo_save[2] = {g->dg.memo[0], g->dg.memo[1]};
    struct Restore {
        fo_graph *g;
        MemoEnt *m[2];
        ~Restore() { g->dg.memo[0] = m[0]; g->dg.memo[1] = m[1]; }
    } restore{g, {memo_save[0], memo_save[1]}};
    if (slot && g->dg.memo[0]) {
        const size_t slots = (size_t)g->dg.memo_mask + 1;
        void *&m = g->sub[slot].memo;
        if (!m) {
            CUDA_TRY(cudaMalloc(&m, 2 * slots * sizeof(MemoEnt)));
            CUDA_TRY(cudaMemset(m, 0, 2 * slots * sizeof(MemoEnt)));
        }
        g->dg.memo[0] = (MemoEnt *)m;
        g->dg.memo[1] = (MemoEnt *)m + slots;
    }
    TimelineOut tl{};
    DeltaIn d;
    d.base = g->d_parent;
    d.off = off;
    d.chg = chg;
    const int pi = precision == FO_PREC_FP64 ? 1 : 0;
    const bool inc = g->delta_mode && g->plan_ok[pi] && g->plan_pv[pi] == g->parent_ver && g->plan_mv[pi] == g->model_ver;
    if (inc) {
        // incremental kernel; candidates it hands back (kRetryGeneral) take the general kernel
        const IncPlan &p = g->plan[pi];
        IncLayout L = inc_layout(g->V, g->E, g->A, p.VB, p.P, 2 * (p.NN + 2) <= 3600);  // indegrees in smem: 7 blocks of 4 warps still fit
        int bps = score_inc_blocks_per_sm(L, precision);
        if (bps <= 0) {
            L = inc_layout(g->V, g->E, g->A, p.VB, p.P, false);
            bps = score_inc_blocks_per_sm(L, precision);
        }
        const int warps = score_warps_per_block();
        const int grid = std::max(1, std::min(g->num_sms * std::max(bps, 1), (K + warps - 1) / warps));
        char *&ws = slot ? g->sub[slot].ws_inc : g->d_ws_inc;
        size_t &ws_bytes = slot ? g->sub[slot].ws_inc_bytes : g->ws_inc_bytes;
        void *&q = slot ? g->sub[slot].inc_q : g->d_inc_q;
        size_t &q_bytes = slot ? g->sub[slot].inc_q_bytes : g->inc_q_bytes;
        const size_t need = (size_t)L.total * grid * warps;
        if (need > ws_bytes) {
            if (ws) CUDA_TRY(cudaFree(ws));
            ws = nullptr;
            ws_bytes = 0;
            CUDA_TRY(cudaMalloc(&ws, need));
            // member marks of the estimator kernel start at -1 (every byte 0xff)
            CUDA_TRY(cudaMemset(ws, 0xff, need));
            ws_bytes = need;
        }
        const int qcap = kIncQueuePerCand * std::min(K, grid * warps);
        const size_t qneed = 64 + (size_t)qcap * 48;
        if (qneed > q_bytes) {
            if (q) CUDA_TRY(cudaFree(q));
            q = nullptr;
            q_bytes = 0;
            CUDA_TRY(cudaMalloc(&q, qneed));
            CUDA_TRY(cudaMemset(q, 0, 64));  // queue count, fast-forward counters (fo_inc_stats)
            q_bytes = qneed;
        }
        cudaError_t e = launch_score_inc(g->dg, p, L, off, chg, K, precision, ws, grid, (IncQ *)((char *)q + 64),
                                         (int *)q, qcap, cost, status, stream, g->delta_mode == 2);
        // kernels launched: setup, estimator and event loop per chunk of one candidate per warp
        g_launches += (int64_t)((K + grid * warps - 1) / (grid * warps)) * (g->dg.phase_stop == 1 ? 1 : 3);
        if (e != cudaSuccess) return fail(FO_CUDA_ERROR, std::string("incremental score launch: ") + cudaGetErrorString(e));
        if (g->delta_mode == 2) return FO_OK;  // diagnostic: hand-backs stay visible as status 101
        return launch(g, nullptr, nullptr, nullptr, 0, K, 2 * g->V + 2, precision, cost, status, nullptr, tl, nullptr,
                      nullptr, nullptr, stream, &d, slot ? slot + 1 : 0, 2);
    }
    return launch(g, nullptr, nullptr, nullptr, 0, K, 2 * g->V + 2, precision, cost, status, nullptr, tl, nullptr,
                  nullptr, nullptr, stream, &d, slot ? slot + 1 : 0);
}

}  // namespace fo

using namespace fo;

static int ensure_plan(fo_graph *g, int precision);  // incremental delta scoring (below)

extern "C" {

const char *fo_last_error(void) { return fo::g_last_error.c_str(); }
int64_t fo_kernel_launches(void) { return fo::g_launches.load(); }

int fo_score_geometry(fo_graph *g, int32_t K, int32_t precision, int32_t *out4) {
    if (!g || !out4 || K <= 0) return fail(FO_INVALID_ARG, "bad arguments");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    CUDA_TRY(cudaSetDevice(g->device));
    const ScoreGeo geo = score_geometry(g->dg, K, g->num_sms, precision);
    out4[0] = geo.team ? 1 : 0;
    out4[1] = geo.grid;
    out4[2] = geo.blocks_per_sm;
    out4[3] = geo.sm_bytes;
    return FO_OK;
}

int fo_set_estimator_arith(fo_graph *g, int32_t mode) {
    if (!g || mode < 0 || mode > 2) return fail(FO_INVALID_ARG, "mode must be 0 (FFMA), 1 (TF32) or 2 (3xTF32)");
    g->dg.mp_arith = mode;
    return FO_OK;
}

int fo_inc_stats(fo_graph *g, int32_t precision, int64_t *out6) {
    if (!g || !out6) return fail(FO_INVALID_ARG, "bad arguments");
    const int pi = precision == FO_PREC_FP64 ? 1 : 0;
    unsigned long long c[3] = {0, 0, 0};
    if (g->d_inc_q) {
        CUDA_TRY(cudaSetDevice(g->device));
        CUDA_TRY(cudaDeviceSynchronize());
        CUDA_TRY(cudaMemcpy(c, (char *)g->d_inc_q + 16, sizeof(c), cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemset((char *)g->d_inc_q + 16, 0, sizeof(c)));
    }
    const bool ok = g->plan_ok[pi] != 0;
    out6[0] = (int64_t)c[0];
    out6[1] = (int64_t)c[1];
    out6[2] = (int64_t)c[2];
    out6[3] = ok ? g->plan_iters[pi] : 0;
    out6[4] = ok ? g->plan[pi].nsnap : 0;
    out6[5] = ok ? g->plan[pi].snap_S : 0;
    return FO_OK;
}

int fo_set_delta_mode(fo_graph *g, int32_t mode) {
    if (!g || mode < 0 || mode > 2) return fail(FO_INVALID_ARG, "mode must be 0, 1 or 2");
    g->delta_mode = mode;
    return FO_OK;
}

int fo_set_phase_stop(fo_graph *g, int32_t phase) {
    if (!g || phase < 0 || phase > 2) return fail(FO_INVALID_ARG, "phase must be 0, 1 or 2");
    g->dg.phase_stop = phase;
    return FO_OK;
}

int fo_graph_create(const fo_graph_desc *d, int32_t device, fo_graph **out) {
    if (!d || !out) return fail(FO_INVALID_ARG, "null argument");
    const int V = d->n_ops, E = d->n_edges, A = d->n_allreduces;
    if (V < 0 || E < 0 || A < 0) return fail(FO_INVALID_ARG, "negative sizes");
    for (int e = 0; e < E; e++)
        if (d->edge_src[e] < 0 || d->edge_src[e] >= V || d->edge_dst[e] < 0 || d->edge_dst[e] >= V)
            return fail(FO_INVALID_ARG, "edge endpoint out of range");
    for (int a = 0; a < A; a++)
        if (d->ar_producer[a] < 0 || d->ar_producer[a] >= V) return fail(FO_INVALID_ARG, "AllReduce producer out of range");
    fo_graph *g = new fo_graph();
    g->device = device;
    g->V = V; g->E = E; g->A = A;
    g->op_kind.assign(d->op_kind, d->op_kind + V);
    g->op_out.assign(d->op_out_bytes, d->op_out_bytes + V);
    g->op_prof.assign(d->op_profile_us, d->op_profile_us + V);
    g->op_compute.assign(d->op_compute_us, d->op_compute_us + V);
    g->e_src.assign(d->edge_src, d->edge_src + E);
    g->e_dst.assign(d->edge_dst, d->edge_dst + E);
    g->e_bytes.assign(d->edge_bytes, d->edge_bytes + E);
    g->ar_prod.assign(d->ar_producer, d->ar_producer + A);
    g->ar_bytes.assign(d->ar_bytes, d->ar_bytes + A);
    // CSRs (graph.py:128-154): stable, so per-op edge lists keep (src, dst) order
    auto csr = [](int n, const std::vector<int32_t> &key, std::vector<int32_t> &ptr, std::vector<int32_t> &idx) {
        ptr.assign(n + 1, 0);
        idx.assign(key.size(), 0);
        for (int32_t k : key) ptr[k + 1]++;
        for (int i = 0; i < n; i++) ptr[i + 1] += ptr[i];
        std::vector<int32_t> cur(ptr.begin(), ptr.end() - 1);
        for (size_t i = 0; i < key.size(); i++) idx[cur[key[i]]++] = (int32_t)i;
    };
    csr(V, g->e_dst, g->in_ptr, g->in_e);
    csr(V, g->e_src, g->out_ptr, g->out_e);
    csr(V, g->ar_prod, g->arp_ptr, g->arp);
    g->agg.assign(E, 0);
    g->op_in.assign(V, 0);
    int64_t pairs = A;
    for (int e = 0; e < E; e++) {
        int s = g->e_src[e], t = g->e_dst[e];
        int nar = g->arp_ptr[s + 1] - g->arp_ptr[s];
        // _consumes_aggregate (graph.py:231-235)
        g->agg[e] = nar > 0 && g->out_ptr[t + 1] == g->out_ptr[t] && g->arp_ptr[t + 1] == g->arp_ptr[t];
        g->op_in[t] += g->e_bytes[e];
        pairs += g->agg[e] ? 2 * nar : 2;
    }
    if (pairs > INT32_MAX / 2) { delete g; return fail(FO_INVALID_ARG, "graph too large"); }
    g->pairs_max = (int32_t)pairs;

    if (device < 0) {  // host-only handle: the native batch-expand engine without a device
        *out = g;
        return FO_OK;
    }
    cudaError_t ce = cudaSetDevice(device);
    if (ce == cudaSuccess) ce = cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
    // one allocation for the static arrays
    struct Seg { const void *src; size_t bytes; size_t off; };
    std::vector<uint8_t> kind8(V);
    for (int v = 0; v < V; v++) kind8[v] = (uint8_t)g->op_kind[v];
    Seg segs[] = {
        {g->e_src.data(), 4u * E, 0}, {g->e_dst.data(), 4u * E, 0}, {g->e_bytes.data(), 8u * E, 0},
        {g->agg.data(), (size_t)E, 0}, {g->in_ptr.data(), 4u * (V + 1), 0}, {g->in_e.data(), 4u * E, 0},
        {g->out_ptr.data(), 4u * (V + 1), 0}, {g->out_e.data(), 4u * E, 0}, {g->arp_ptr.data(), 4u * (V + 1), 0},
        {g->arp.data(), 4u * A, 0}, {g->ar_prod.data(), 4u * A, 0}, {g->ar_bytes.data(), 8u * A, 0},
        {kind8.data(), (size_t)V, 0}, {g->op_prof.data(), 8u * V, 0}, {g->op_compute.data(), 8u * V, 0},
        {g->op_out.data(), 8u * V, 0}, {g->op_in.data(), 8u * V, 0},
    };
    size_t total = 0;
    for (auto &s : segs) { s.off = total; total += al256(s.bytes + 1); }
    if (ce == cudaSuccess) ce = cudaMalloc(&g->d_static, total);
    for (auto &s : segs)
        if (ce == cudaSuccess && s.bytes) ce = cudaMemcpy((char *)g->d_static + s.off, s.src, s.bytes, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
        std::string m = std::string("fo_graph_create: ") + cudaGetErrorString(ce);
        fo_graph_destroy(g);
        return fail(FO_CUDA_ERROR, m);
    }
    char *b = (char *)g->d_static;
    DGraph &dg = g->dg;
    dg.V = V; dg.E = E; dg.A = A;
    dg.e_src = (const int32_t *)(b + segs[0].off);
    dg.e_dst = (const int32_t *)(b + segs[1].off);
    dg.e_bytes = (const int64_t *)(b + segs[2].off);
    dg.e_agg = (const uint8_t *)(b + segs[3].off);
    dg.in_ptr = (const int32_t *)(b + segs[4].off);
    dg.in_e = (const int32_t *)(b + segs[5].off);
    dg.out_ptr = (const int32_t *)(b + segs[6].off);
    dg.out_e = (const int32_t *)(b + segs[7].off);
    dg.arp_ptr = (const int32_t *)(b + segs[8].off);
    dg.arp = (const int32_t *)(b + segs[9].off);
    dg.ar_prod = (const int32_t *)(b + segs[10].off);
    dg.ar_bytes = (const int64_t *)(b + segs[11].off);
    dg.op_kind = (const uint8_t *)(b + segs[12].off);
    dg.op_prof = (const double *)(b + segs[13].off);
    dg.op_compute = (const double *)(b + segs[14].off);
    dg.op_out = (const int64_t *)(b + segs[15].off);
    dg.op_in = (const int64_t *)(b + segs[16].off);
    dg.pairs_max = g->pairs_max;
    *out = g;
    return FO_OK;
}

int fo_graph_destroy(fo_graph *g) {
    if (!g) return FO_OK;
    if (g->device < 0) { delete g; return FO_OK; }
    cudaSetDevice(g->device);
    if (g->stream) cudaStreamSynchronize(g->stream);
    if (g->d_static) cudaFree(g->d_static);
    if (g->d_model) cudaFree(g->d_model);
    if (g->d_ws) cudaFree(g->d_ws);
    if (g->d_ws_big) cudaFree(g->d_ws_big);
    if (g->d_ws_alt) cudaFree(g->d_ws_alt);
    if (g->d_memo) cudaFree(g->d_memo);
    if (g->d_keys) cudaFree(g->d_keys);
    if (g->d_io) cudaFree(g->d_io);
    if (g->d_parent) cudaFree(g->d_parent);
    for (void *pl : g->d_plan)
        if (pl) cudaFree(pl);
    for (void *pl : g->d_snap)
        if (pl) cudaFree(pl);
    if (g->d_ws_inc) cudaFree(g->d_ws_inc);
    if (g->d_inc_q) cudaFree(g->d_inc_q);
    for (auto &u : g->sub) {
        if (u.ws_inc) cudaFree(u.ws_inc);
        if (u.inc_q) cudaFree(u.inc_q);
        if (u.memo) cudaFree(u.memo);
        if (u.ws) cudaFree(u.ws);
        if (u.stream) cudaStreamDestroy(u.stream);
    }
    if (g->h_pinned) cudaFreeHost(g->h_pinned);
    for (auto &sl : g->aslot) {
        if (sl.done) cudaEventSynchronize(sl.done);
        if (sl.d) cudaFree(sl.d);
        if (sl.h2d) cudaEventDestroy(sl.h2d);
        if (sl.kdone) cudaEventDestroy(sl.kdone);
        if (sl.done) cudaEventDestroy(sl.done);
    }
    if (g->hstream) cudaStreamDestroy(g->hstream);
    if (g->dstream) cudaStreamDestroy(g->dstream);
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
    return FO_OK;
}

int fo_graph_set_cost_model(fo_graph *g, const fo_cost_model *m) {
    if (!g || !m) return fail(FO_INVALID_ARG, "null argument");
    std::lock_guard<std::mutex> lk(g->mu);
    g->model_ver++;  // invalidates the incremental plans
    DGraph &dg = g->dg;
    dg.provider = m->provider;
    dg.variant = m->variant;
    dg.C = m->comm_C;
    dg.D = m->comm_D;
    dg.launch = m->launch_us;
    dg.mem = m->mem_us_per_byte;
    dg.out_scale = m->out_scale;
    dg.layers = 0;
    dg.lin_norm = 0;
    dg.emb = dg.emb_mean = dg.emb_std = nullptr;
    if (m->provider != FO_PROVIDER_PROFILE && m->provider != FO_PROVIDER_HW_ORACLE)
        return fail(FO_INVALID_ARG, "unknown provider");
    if (!(m->comm_C >= 0) || !(m->comm_D >= 0)) return fail(FO_INVALID_ARG, "C and D must be non-negative");
    const int V = g->V;
    dg.noise = 0.0;
    dg.kpre = dg.okb = nullptr;
    dg.oko = nullptr;
    dg.kpre_len = 0;
    if (m->provider == FO_PROVIDER_HW_ORACLE && m->hw_noise != 0.0) {
        // jitter keys (workloads.py:254-273): prefix | per-op fragments | offsets
        if (!(m->hw_noise >= 0.0 && m->hw_noise <= 0.5)) return fail(FO_INVALID_ARG, "noise fraction must lie in [0, 0.5]");
        if (!m->hw_key_prefix || m->hw_key_prefix_len < 0 || !m->op_key_bytes || !m->op_key_off)
            return fail(FO_INVALID_ARG, "jitter needs the key prefix and per-op key fragments");
        const int64_t nb = m->op_key_off[V];
        size_t o_off = al256((size_t)m->hw_key_prefix_len + 8), o_b = o_off + al256(8 * ((size_t)V + 1));
        size_t tot = o_b + al256((size_t)nb + 8);
        dg.noise = m->hw_noise;
        dg.kpre_len = m->hw_key_prefix_len;
        if (g->device >= 0) {
            CUDA_TRY(cudaSetDevice(g->device));
            if (g->d_keys) { cudaFree(g->d_keys); g->d_keys = nullptr; }
            CUDA_TRY(cudaMalloc(&g->d_keys, tot));
            char *b = (char *)g->d_keys;
            CUDA_TRY(cudaMemcpy(b, m->hw_key_prefix, m->hw_key_prefix_len, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(b + o_off, m->op_key_off, 8 * ((size_t)V + 1), cudaMemcpyHostToDevice));
            if (nb) CUDA_TRY(cudaMemcpy(b + o_b, m->op_key_bytes, nb, cudaMemcpyHostToDevice));
            dg.kpre = (const uint8_t *)b;
            dg.oko = (const int64_t *)(b + o_off);
            dg.okb = (const uint8_t *)(b + o_b);
        }
    }
    if (m->provider == FO_PROVIDER_PROFILE && m->variant == FO_EST_LINEAR) {
        if (!m->params || m->n_params != 13) return fail(FO_DIM_MISMATCH, "linear model needs w[12] and b");
        for (int i = 0; i < 12; i++) dg.lin_w[i] = m->params[i];
        dg.lin_b = m->params[12];
        if (m->norm_mean && m->norm_std) {
            dg.lin_norm = 1;
            for (int i = 0; i < 12; i++) { dg.agg_mean[i] = m->norm_mean[i]; dg.agg_std[i] = m->norm_std[i]; }
        }
    }
    if (m->provider == FO_PROVIDER_PROFILE && m->variant == FO_EST_MESSAGE_PASSING) {
        const int h = m->hidden, F = m->feat_dim, L = m->layers;
        if (h < 1 || h > kHidden) return fail(FO_UNSUPPORTED, "hidden size must be in [1, 32] on the device");
        if (F < 6 || L < 0) return fail(FO_DIM_MISMATCH, "bad feature dimension / layers");
        int64_t need = (int64_t)h * F + (int64_t)(L + 3) * h * h + 3 * h + 1;
        if (!m->params || m->n_params != need) return fail(FO_DIM_MISMATCH, "message-passing parameter count mismatch");
        if (!m->op_vocab_slot) return fail(FO_INVALID_ARG, "op_vocab_slot required");
        for (int v = 0; v < V; v++)
            if (m->op_vocab_slot[v] < 0 || 6 + m->op_vocab_slot[v] >= F)
                return fail(FO_DIM_MISMATCH, "vocab slot outside W_emb");
        const double *p = m->params;
        const double *Wemb = p;
        const double *Wl = Wemb + (int64_t)h * F;
        const double *Wr = Wl + (int64_t)L * h * h;
        const double *A1 = Wr + h * h;
        const double *c1 = A1 + h * h;
        const double *A2 = c1 + h;
        const double *c2 = A2 + h * h;
        const double *a3 = c2 + h;
        const double c3 = a3[h];
        // per-op embedded features H0 = standardize(X) @ W_emb^T (estimator.py:321-338, :369)
        std::vector<double> H0((size_t)V * kHidden, 0.0), x(F);
        for (int v = 0; v < V; v++) {
            double c = g->op_prof[v], in = (double)g->op_in[v], o = (double)g->op_out[v];
            std::fill(x.begin(), x.end(), 0.0);
            x[0] = std::log1p(c); x[1] = c; x[2] = std::log1p(in); x[3] = in; x[4] = std::log1p(o); x[5] = o;
            x[6 + m->op_vocab_slot[v]] = 1.0;
            if (m->norm_mean && m->norm_std)
                for (int k = 0; k < F; k++) x[k] = (x[k] - m->norm_mean[k]) / m->norm_std[k];
            for (int ch = 0; ch < h; ch++) {
                double acc = 0.0;
                for (int k = 0; k < F; k++) acc += x[k] * Wemb[ch * F + k];
                H0[(size_t)v * kHidden + ch] = acc;
            }
        }
        MpLayout ml = mp_layout(L);
        std::vector<double> W(ml.total, 0.0);
        auto put_t = [&](int64_t off, const double *M) {  // W^T, zero padded to 32x32
            for (int r = 0; r < h; r++)
                for (int k = 0; k < h; k++) W[off + k * 32 + r] = M[r * h + k];
        };
        for (int l = 0; l < L; l++) put_t(ml.wl + (int64_t)l * 1024, Wl + (int64_t)l * h * h);
        put_t(ml.wr, Wr);
        put_t(ml.a1, A1);
        put_t(ml.a2, A2);
        for (int r = 0; r < h; r++) { W[ml.c1 + r] = c1[r]; W[ml.c2 + r] = c2[r]; W[ml.a3 + r] = a3[r]; }
        W[ml.c3] = c3;
        std::vector<float> H0f(H0.begin(), H0.end()), Wf(W.begin(), W.end());
        size_t oH0d = 0, oH0f = al256(H0.size() * 8), oWd = oH0f + al256(H0f.size() * 4 + 4),
               oWf = oWd + al256(W.size() * 8), oE = oWf + al256(Wf.size() * 4),
               oNm = oE + al256((size_t)h * F * 8), tot = oNm + al256((size_t)2 * F * 8);
        const bool has_norm = m->norm_mean && m->norm_std;
        if (g->device < 0) { g->model_set = true; return FO_OK; }
        CUDA_TRY(cudaSetDevice(g->device));
        if (g->d_model) { cudaFree(g->d_model); g->d_model = nullptr; }
        CUDA_TRY(cudaMalloc(&g->d_model, tot));
        char *b = (char *)g->d_model;
        if (!H0.empty()) {
            CUDA_TRY(cudaMemcpy(b + oH0d, H0.data(), H0.size() * 8, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(b + oH0f, H0f.data(), H0f.size() * 4, cudaMemcpyHostToDevice));
        }
        CUDA_TRY(cudaMemcpy(b + oWd, W.data(), W.size() * 8, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(b + oWf, Wf.data(), Wf.size() * 4, cudaMemcpyHostToDevice));
        // W_emb and node_norm for feature-level prediction (fo_predict_features)
        CUDA_TRY(cudaMemcpy(b + oE, Wemb, (size_t)h * F * 8, cudaMemcpyHostToDevice));
        if (has_norm) {
            CUDA_TRY(cudaMemcpy(b + oNm, m->norm_mean, (size_t)F * 8, cudaMemcpyHostToDevice));
            CUDA_TRY(cudaMemcpy(b + oNm + (size_t)F * 8, m->norm_std, (size_t)F * 8, cudaMemcpyHostToDevice));
        }
        dg.emb = (const double *)(b + oE);
        dg.emb_mean = has_norm ? (const double *)(b + oNm) : nullptr;
        dg.emb_std = has_norm ? (const double *)(b + oNm + (size_t)F * 8) : nullptr;
        dg.emb_h = h;
        dg.emb_F = F;
        // estimator memo: 2 x 2^20 slots, cleared whenever the model changes
        const char *mlog = getenv("FO_MEMO_LOG2");  // tuning override: slots per precision
        const size_t slots = (size_t)1 << (mlog ? std::max(10, std::min(24, atoi(mlog))) : 20);
        if (g->d_memo && g->memo_slots != slots) { cudaFree(g->d_memo); g->d_memo = nullptr; }
        g->memo_slots = slots;
        if (!g->d_memo) CUDA_TRY(cudaMalloc(&g->d_memo, 2 * slots * sizeof(MemoEnt)));
        CUDA_TRY(cudaMemset(g->d_memo, 0, 2 * slots * sizeof(MemoEnt)));
        for (auto &u : g->sub)  // re-made empty on demand
            if (u.memo) { cudaFree(u.memo); u.memo = nullptr; }
        dg.memo[0] = (MemoEnt *)g->d_memo;
        dg.memo[1] = (MemoEnt *)g->d_memo + slots;
        dg.memo_mask = (uint32_t)(slots - 1);
        dg.H0d = (const double *)(b + oH0d);
        dg.H0f = (const float *)(b + oH0f);
        dg.Wd = (const double *)(b + oWd);
        dg.Wf = (const float *)(b + oWf);
        dg.layers = L;
    }
    g->model_set = true;
    return FO_OK;
}

int fo_batch_best(const double *cost, const int32_t *status, int32_t K, int64_t id_offset, double *out_pair,
                  void *stream) {
    if (!cost || !out_pair || K < 0) return fail(FO_INVALID_ARG, "bad arguments");
    cudaError_t e = launch_batch_best(cost, status, K, id_offset, out_pair, (cudaStream_t)stream);
    g_launches++;
    if (e != cudaSuccess) return fail(FO_CUDA_ERROR, std::string("batch_best launch: ") + cudaGetErrorString(e));
    return FO_OK;
}

int fo_pairs_best(const double *pairs, int32_t n, double *out_pair, void *stream) {
    if (!pairs || !out_pair || n < 0) return fail(FO_INVALID_ARG, "bad arguments");
    cudaError_t e = launch_batch_best(pairs, nullptr, n, 0, out_pair, (cudaStream_t)stream, 1);
    g_launches++;
    if (e != cudaSuccess) return fail(FO_CUDA_ERROR, std::string("pairs_best launch: ") + cudaGetErrorString(e));
    return FO_OK;
}

int fo_memo_clear(fo_graph *g, void *stream) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    if (!g->d_memo) return FO_OK;
    cudaStream_t s = stream ? (cudaStream_t)stream : g->stream;  // NULL: the handle's own stream
    CUDA_TRY(cudaMemsetAsync(g->d_memo, 0, 2 * ((size_t)g->dg.memo_mask + 1) * sizeof(MemoEnt), s));
    for (auto &u : g->sub)  // the submission streams' tables
        if (u.memo) CUDA_TRY(cudaMemsetAsync(u.memo, 0, 2 * ((size_t)g->dg.memo_mask + 1) * sizeof(MemoEnt), s));
    return FO_OK;
}

int fo_memo_enable(fo_graph *g, int32_t enable) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    std::lock_guard<std::mutex> lk(g->mu);
    const size_t slots = (size_t)g->dg.memo_mask + 1;
    if (enable && g->d_memo) {
        g->dg.memo[0] = (MemoEnt *)g->d_memo;
        g->dg.memo[1] = (MemoEnt *)g->d_memo + slots;
    } else {
        g->dg.memo[0] = g->dg.memo[1] = nullptr;
    }
    return FO_OK;
}

int fo_score(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t K, int32_t gid_bound,
             int32_t precision, double *cost_out, int32_t *status_out, void *stream) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    std::lock_guard<std::mutex> lk(g->mu);
    return score_device(g, ngid, rgid, bkt, 0, K, gid_bound, precision, cost_out, status_out, (cudaStream_t)stream);
}

int fo_score_i16(fo_graph *g, const int16_t *ngid, const int16_t *rgid, const int16_t *bkt, int32_t K,
                 int32_t gid_bound, int32_t precision, double *cost_out, int32_t *status_out, void *stream) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    std::lock_guard<std::mutex> lk(g->mu);
    return score_device(g, ngid, rgid, bkt, 1, K, gid_bound, precision, cost_out, status_out, (cudaStream_t)stream);
}

static int ensure_io(fo_graph *g, size_t bytes) {
    if (bytes > g->io_bytes) {
        if (g->d_io) cudaFree(g->d_io);
        g->d_io = nullptr;
        g->io_bytes = 0;
        CUDA_TRY(cudaMalloc(&g->d_io, bytes));
        g->io_bytes = bytes;
    }
    return FO_OK;
}

int fo_predict_features(fo_graph *g, int32_t n, const int32_t *op_slot, const double *compute_us,
                        const int64_t *in_bytes, const int64_t *out_bytes, int32_t m, const int32_t *edges,
                        const double *aggregates, int32_t precision, double *pred_out) {
    if (!g || !pred_out || n < 0 || m < 0 || (n && (!compute_us || !in_bytes || !out_bytes || !op_slot)) ||
        (m && !edges) || !aggregates)
        return fail(FO_INVALID_ARG, "bad arguments");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    if (!g->model_set) return fail(FO_INVALID_ARG, "no cost model set");
    if (g->dg.provider != FO_PROVIDER_PROFILE)
        return fail(FO_UNSUPPORTED, "feature-level prediction needs a profile-provider estimator");
    if (precision != FO_PREC_FP64 && precision != FO_PREC_FP32) return fail(FO_INVALID_ARG, "bad precision");
    if (g->dg.variant != FO_EST_ANALYTIC && g->dg.variant != FO_EST_LINEAR &&
        (g->dg.variant != FO_EST_MESSAGE_PASSING || !g->dg.emb))
        return fail(FO_DIM_MISMATCH, "no usable fused-op estimator loaded (parameter shapes do not match)");
    if (n > 8192) return fail(FO_UNSUPPORTED, "group too large for feature-level prediction (> 8192 ops)");
    const DGraph &dg = g->dg;
    if (dg.variant == FO_EST_MESSAGE_PASSING)
        for (int i = 0; i < n; i++)
            if (op_slot[i] < 0 || 6 + op_slot[i] >= dg.emb_F) return fail(FO_DIM_MISMATCH, "vocab slot outside W_emb");
    for (int q = 0; q < m; q++)
        if (edges[2 * q] < 0 || edges[2 * q] >= n || edges[2 * q + 1] < 0 || edges[2 * q + 1] >= n)
            return fail(FO_INVALID_ARG, "edge endpoint outside the group");
    std::lock_guard<std::mutex> lk(g->mu);
    CUDA_TRY(cudaSetDevice(g->device));
    const size_t o_slot = 0, o_c = al256((size_t)n * 4 + 4), o_in = o_c + al256((size_t)n * 8 + 8),
                 o_out = o_in + al256((size_t)n * 8 + 8), o_e = o_out + al256((size_t)n * 8 + 8),
                 o_ptr = o_e + al256((size_t)m * 8 + 8), o_nb = o_ptr + al256((size_t)n * 4 + 8),
                 o_H0 = o_nb + al256(((size_t)2 * m + 1 + n) * 4), o_H = o_H0 + al256((size_t)n * 32 * 8 + 8),
                 o_P = o_H + al256((size_t)n * 32 * 8 + 8), o_pred = o_P + al256((size_t)n * 32 * 8 + 8),
                 tot = o_pred + 256;
    int st = ensure_io(g, tot);
    if (st) return st;
    char *b = (char *)g->d_io;
    cudaStream_t s = g->stream;
    if (n) {
        CUDA_TRY(cudaMemcpyAsync(b + o_slot, op_slot, (size_t)n * 4, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(b + o_c, compute_us, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(b + o_in, in_bytes, (size_t)n * 8, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(b + o_out, out_bytes, (size_t)n * 8, cudaMemcpyHostToDevice, s));
    }
    if (m) CUDA_TRY(cudaMemcpyAsync(b + o_e, edges, (size_t)m * 8, cudaMemcpyHostToDevice, s));
    FeatIn fi;
    fi.n = n; fi.m = m;
    for (int q = 0; q < 6; q++) fi.agg[q] = aggregates[q];
    fi.slot = (const int32_t *)(b + o_slot);
    fi.edges = (const int32_t *)(b + o_e);
    fi.c = (const double *)(b + o_c);
    fi.in = (const long long *)(b + o_in);
    fi.out = (const long long *)(b + o_out);
    fi.nbptr = (int32_t *)(b + o_ptr);
    fi.nb = (int32_t *)(b + o_nb);
    fi.H0 = b + o_H0; fi.H = b + o_H; fi.P = b + o_P;
    cudaError_t e = launch_predict_features(dg, fi, precision, (double *)(b + o_pred), s);
    g_launches++;
    if (e != cudaSuccess) return fail(FO_CUDA_ERROR, std::string("predict_features launch: ") + cudaGetErrorString(e));
    CUDA_TRY(cudaMemcpyAsync(pred_out, b + o_pred, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FO_OK;
}

static int score_host_impl(fo_graph *g, const void *ngid, const void *rgid, const void *bkt, int es, int32_t K,
                           int32_t gid_bound, int32_t precision, double *cost_out, int32_t *status_out) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    std::lock_guard<std::mutex> lk(g->mu);
    if (K <= 0) return FO_OK;
    CUDA_TRY(cudaSetDevice(g->device));
    size_t nv = (size_t)K * g->V * es, na = (size_t)K * g->A * es;
    size_t o_r = al256(nv), o_b = o_r + al256(nv), o_c = o_b + al256(na + 4), o_s = o_c + al256((size_t)K * 8);
    int st = ensure_io(g, o_s + al256((size_t)K * 4));
    if (st) return st;
    char *b = (char *)g->d_io;
    cudaStream_t s = g->stream;
    if (nv) {
        CUDA_TRY(cudaMemcpyAsync(b, ngid, nv, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(b + o_r, rgid, nv, cudaMemcpyHostToDevice, s));
    }
    if (na) CUDA_TRY(cudaMemcpyAsync(b + o_b, bkt, na, cudaMemcpyHostToDevice, s));
    st = score_device(g, b, b + o_r, b + o_b, es == 2, K, gid_bound, precision, (double *)(b + o_c),
                      (int32_t *)(b + o_s), s);
    if (st) return st;
    CUDA_TRY(cudaMemcpyAsync(cost_out, b + o_c, (size_t)K * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status_out, b + o_s, (size_t)K * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FO_OK;
}

int fo_score_host(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t K,
                  int32_t gid_bound, int32_t precision, double *cost_out, int32_t *status_out) {
    return score_host_impl(g, ngid, rgid, bkt, 4, K, gid_bound, precision, cost_out, status_out);
}

int fo_score_host_i16(fo_graph *g, const int16_t *ngid, const int16_t *rgid, const int16_t *bkt, int32_t K,
                      int32_t gid_bound, int32_t precision, double *cost_out, int32_t *status_out) {
    return score_host_impl(g, ngid, rgid, bkt, 2, K, gid_bound, precision, cost_out, status_out);
}

int fo_score_delta(fo_graph *g, const int32_t *offsets, const int32_t *changes, int32_t K, int32_t precision,
                   double *cost_out, int32_t *status_out, void *stream) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    std::lock_guard<std::mutex> lk(g->mu);
    CUDA_TRY(cudaSetDevice(g->device));
    int st = ensure_plan(g, precision);
    if (st) return st;
    return score_delta_device(g, offsets, changes, K, precision, cost_out, status_out, (cudaStream_t)stream);
}

int fo_score_delta_slot(fo_graph *g, int32_t slot, const int32_t *offsets, const int32_t *changes, int32_t K,
                        int32_t precision, int32_t clear_memo, double *cost_out, int32_t *status_out, void *stream) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    if (slot < 0 || slot >= fo_graph::kSubmitSlots) return fail(FO_INVALID_ARG, "slot out of range");
    if (slot > 0 && g->V > kMpCapDefault)
        return fail(FO_INVALID_ARG, "graphs whose groups outgrow the estimator scratch have one scratch slot");
    std::lock_guard<std::mutex> lk(g->mu);
    CUDA_TRY(cudaSetDevice(g->device));
    int st = ensure_plan(g, precision);
    if (st) return st;
    cudaStream_t s = (cudaStream_t)stream;
    if (clear_memo && g->d_memo && (slot == 0 || g->sub[slot].memo)) {  // this slot's table of this precision
        const size_t slots = (size_t)g->dg.memo_mask + 1;
        MemoEnt *tab = (MemoEnt *)(slot ? g->sub[slot].memo : g->d_memo) + (precision == FO_PREC_FP64 ? slots : 0);
        CUDA_TRY(cudaMemsetAsync(tab, 0, slots * sizeof(MemoEnt), s));
    }
    return score_delta_device(g, offsets, changes, K, precision, cost_out, status_out, s, slot);
}

// sparse-candidate offsets: offsets[0] == 0 and non-decreasing, so every
// candidate's change range lies inside the staged changes buffer.  (Indices
// inside one candidate must be distinct: duplicates race in K1.)
static bool offsets_ok(const int32_t *offsets, int32_t K) {
    if (!offsets || offsets[0] != 0) return false;
    for (int32_t k = 0; k < K; k++)
        if (offsets[k + 1] < offsets[k]) return false;
    return true;
}

int fo_score_delta_host(fo_graph *g, const int32_t *offsets, const int32_t *changes, int32_t K, int32_t precision,
                        double *cost_out, int32_t *status_out) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    std::lock_guard<std::mutex> lk(g->mu);
    if (K <= 0) return FO_OK;
    if (!offsets_ok(offsets, K)) return fail(FO_INVALID_ARG, "bad offsets (offsets[0] != 0 or decreasing)");
    CUDA_TRY(cudaSetDevice(g->device));
    int st = ensure_plan(g, precision);  // before staging: building it uses the same staging buffer
    if (st) return st;
    const size_t nc = (size_t)offsets[K];
    size_t o_c = al256(4 * ((size_t)K + 1)), o_cost = o_c + al256(8 * nc + 8), o_s = o_cost + al256((size_t)K * 8);
    st = ensure_io(g, o_s + al256((size_t)K * 4));
    if (st) return st;
    char *b = (char *)g->d_io;
    cudaStream_t s = g->stream;
    CUDA_TRY(cudaMemcpyAsync(b, offsets, 4 * ((size_t)K + 1), cudaMemcpyHostToDevice, s));
    if (nc) CUDA_TRY(cudaMemcpyAsync(b + o_c, changes, 8 * nc, cudaMemcpyHostToDevice, s));
    st = score_delta_device(g, (const int32_t *)b, (const int32_t *)(b + o_c), K, precision, (double *)(b + o_cost),
                            (int32_t *)(b + o_s), s);
    if (st) return st;
    CUDA_TRY(cudaMemcpyAsync(cost_out, b + o_cost, (size_t)K * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(status_out, b + o_s, (size_t)K * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return FO_OK;
}

// Pipelined form of fo_score_delta_host.  Slot t % 2 owns its device
// staging; H2D runs on one copy stream (then signals the compute stream) and
// D2H on another (after the kernel), so consecutive submissions overlap
// transfers with the other batch's kernel.  A slot is reused only after its previous
// submission's D2H completed.
int fo_score_delta_submit(fo_graph *g, const int32_t *offsets, const int32_t *changes, int32_t K, int32_t precision,
                          int32_t clear_memo, double *cost_out, int32_t *status_out, int64_t *ticket_out) {
    if (!g || !ticket_out) return fail(FO_INVALID_ARG, "null argument");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    std::lock_guard<std::mutex> lk(g->mu);
    if (K < 0 || !offsets_ok(offsets, K)) return fail(FO_INVALID_ARG, "bad offsets (offsets[0] != 0 or decreasing)");
    CUDA_TRY(cudaSetDevice(g->device));
    {
        const int pst = ensure_plan(g, precision);
        if (pst) return pst;
    }
    if (!g->hstream) CUDA_TRY(cudaStreamCreateWithFlags(&g->hstream, cudaStreamNonBlocking));
    if (!g->dstream) CUDA_TRY(cudaStreamCreateWithFlags(&g->dstream, cudaStreamNonBlocking));
    const int64_t t = g->next_ticket;
    fo_graph::AsyncSlot &sl = g->aslot[t % fo_graph::kSubmitSlots];
    if (!sl.h2d) {
        CUDA_TRY(cudaEventCreateWithFlags(&sl.h2d, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&sl.kdone, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    }
    if (sl.ticket >= 0) CUDA_TRY(cudaEventSynchronize(sl.done));  // slot free: its last D2H landed
    const size_t nc = (size_t)offsets[K];
    const size_t o_c = al256(4 * ((size_t)K + 1)), o_cost = o_c + al256(8 * nc + 8),
                 o_s = o_cost + al256((size_t)K * 8 + 8), need = o_s + al256((size_t)K * 4 + 4);
    if (sl.bytes < need) {
        if (sl.d) CUDA_TRY(cudaFree(sl.d));
        sl.d = nullptr;
        sl.bytes = 0;
        CUDA_TRY(cudaMalloc(&sl.d, need));
        sl.bytes = need;
    }
    char *b = sl.d;
    // consecutive submissions alternate between two compute streams with
    // their own scratch, so a batch's setup runs in the previous batch's
    // event-loop tail (graphs whose fused groups outgrow the estimator scratch
    // share one second-pass workspace: one stream)
    static const int nstreams = getenv("FO_SUBMIT_STREAMS") ? std::max(1, std::min(fo_graph::kSubmitSlots, atoi(getenv("FO_SUBMIT_STREAMS"))))
                                                           : fo_graph::kSubmitSlots;
    const int ks = g->V <= kMpCapDefault ? (int)(t % nstreams) : 0;
    if (ks && !g->sub[ks].stream) CUDA_TRY(cudaStreamCreateWithFlags(&g->sub[ks].stream, cudaStreamNonBlocking));
    cudaStream_t hs = g->hstream, ds = g->dstream, s = ks ? g->sub[ks].stream : g->stream;
    CUDA_TRY(cudaMemcpyAsync(b, offsets, 4 * ((size_t)K + 1), cudaMemcpyHostToDevice, hs));
    if (nc) CUDA_TRY(cudaMemcpyAsync(b + o_c, changes, 8 * nc, cudaMemcpyHostToDevice, hs));
    CUDA_TRY(cudaEventRecord(sl.h2d, hs));
    CUDA_TRY(cudaStreamWaitEvent(s, sl.h2d, 0));
    if (clear_memo && g->d_memo && (!ks || g->sub[ks].memo)) {  // only the table this precision's estimator reads
        const size_t slots = (size_t)g->dg.memo_mask + 1;
        MemoEnt *tab = (MemoEnt *)(ks ? g->sub[ks].memo : g->d_memo) + (precision == FO_PREC_FP64 ? slots : 0);
        CUDA_TRY(cudaMemsetAsync(tab, 0, slots * sizeof(MemoEnt), s));
    }
    int st = score_delta_device(g, (const int32_t *)b, (const int32_t *)(b + o_c), K, precision,
                                (double *)(b + o_cost), (int32_t *)(b + o_s), s, ks);
    if (st) return st;
    CUDA_TRY(cudaEventRecord(sl.kdone, s));
    CUDA_TRY(cudaStreamWaitEvent(ds, sl.kdone, 0));
    if (K) {
        CUDA_TRY(cudaMemcpyAsync(cost_out, b + o_cost, (size_t)K * 8, cudaMemcpyDeviceToHost, ds));
        CUDA_TRY(cudaMemcpyAsync(status_out, b + o_s, (size_t)K * 4, cudaMemcpyDeviceToHost, ds));
    }
    CUDA_TRY(cudaEventRecord(sl.done, ds));
    sl.ticket = t;
    g->next_ticket = t + 1;
    *ticket_out = t;
    return FO_OK;
}

int fo_score_wait(fo_graph *g, int64_t ticket) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    std::lock_guard<std::mutex> lk(g->mu);
    if (ticket < 0 || ticket >= g->next_ticket) return fail(FO_INVALID_ARG, "unknown ticket");
    const fo_graph::AsyncSlot &sl = g->aslot[ticket % fo_graph::kSubmitSlots];
    // a slot that moved on to a later ticket already waited for this one
    if (sl.ticket == ticket) CUDA_TRY(cudaEventSynchronize(sl.done));
    return FO_OK;
}

// single candidate through device temporaries (simulate / timeline / durations)
static int single(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int VB, int precision,
                  const double *durations, bool want_tl, bool want_dur, std::vector<char> &hout, size_t *offs) {
    const int V = g->V, A = g->A;
    size_t GMx = 2 * (size_t)V + 1, NMx = GMx + A + 1;
    size_t o[16];
    size_t t = 0;
    auto take = [&](int i, size_t bytes) { o[i] = t; t += al256(bytes + 8); };
    take(0, 4u * V); take(1, 4u * V); take(2, 4u * A);      // state
    take(3, 8); take(4, 4);                                  // cost, status
    take(5, 8 * NMx);                                        // ext durations
    take(6, 4 * GMx); take(7, 8 * GMx); take(8, 8 * GMx);    // compute events
    take(9, 4u * (A + 1)); take(10, 8u * (A + 1)); take(11, 8u * (A + 1));  // comm events
    take(12, 4); take(13, 4);                                // counts
    take(14, 8 * NMx);                                       // dur out
    take(15, 16);                                            // bad, ngroups
    int st = ensure_io(g, t);
    if (st) return st;
    char *b = (char *)g->d_io;
    cudaStream_t s = g->stream;
    CUDA_TRY(cudaMemsetAsync(b, 0, t, s));
    if (V) {
        CUDA_TRY(cudaMemcpyAsync(b + o[0], ngid, 4u * V, cudaMemcpyHostToDevice, s));
        CUDA_TRY(cudaMemcpyAsync(b + o[1], rgid, 4u * V, cudaMemcpyHostToDevice, s));
    }
    if (A) CUDA_TRY(cudaMemcpyAsync(b + o[2], bkt, 4u * A, cudaMemcpyHostToDevice, s));
    const double *ext = nullptr;
    if (durations) {
        // caller passes G + B entries; the count is only known on the device, so
        // copy the maximum the caller may have supplied (sized by the shim)
        CUDA_TRY(cudaMemcpyAsync(b + o[5], durations, 8 * NMx, cudaMemcpyHostToDevice, s));
        ext = (const double *)(b + o[5]);
    }
    TimelineOut tl{};
    if (want_tl) {
        tl.c_id = (int32_t *)(b + o[6]); tl.c_start = (double *)(b + o[7]); tl.c_end = (double *)(b + o[8]);
        tl.b_id = (int32_t *)(b + o[9]); tl.b_start = (double *)(b + o[10]); tl.b_end = (double *)(b + o[11]);
        tl.n_c = (int32_t *)(b + o[12]); tl.n_b = (int32_t *)(b + o[13]);
    }
    int32_t *bad = (int32_t *)(b + o[15]);
    st = launch(g, b + o[0], b + o[1], b + o[2], 0, 1, VB, precision,
                (double *)(b + o[3]), (int32_t *)(b + o[4]), ext, tl, want_dur ? (double *)(b + o[14]) : nullptr, bad,
                bad + 1, s);
    if (st) return st;
    hout.resize(t);
    CUDA_TRY(cudaMemcpyAsync(hout.data(), b, t, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    for (int i = 0; i < 16; i++) offs[i] = o[i];
    return FO_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Parent plan of the incremental delta path (score_inc.cuh), per precision:
// the parent's contracted schedule DAG in gid space -- the dependency slots
// of graph.py:215-261 as a successor CSR with each slot's position, node
// records (duration, tie-break rank, existence), group / bucket members and
// the level-0 ready runs.  Durations come from the general kernel on the
// parent itself, so the plan carries exactly the general path's values.
// Only the MP estimator with profile lookups takes this path (the analytic /
// linear / hardware-oracle providers depend on group_io of neighbours).
// Run the parent's event loop once on the device (inc_record_kernel) and keep
// every node's push iteration plus a loop snapshot every S iterations in the
// plan, so candidates start at the last iteration they share with the parent.
// The recorded makespan must equal the general kernel's parent cost bit for
// bit; otherwise (or with FO_INC_NO_SNAP set) candidates start at level 0.
static int record_parent_loop(fo_graph *g, int pi, const char *parent_cost) {
    IncPlan &p = g->plan[pi];
    if (g->d_snap[pi]) { CUDA_TRY(cudaFree(g->d_snap[pi])); g->d_snap[pi] = nullptr; }
    g->plan_iters[pi] = 0;
    if (getenv("FO_INC_NO_SNAP") || p.n_exist < 16) return FO_OK;
    const int S = std::max(4, (p.n_exist + 63) / 64), maxsnap = p.n_exist / S;
    const int64_t stride = inc_snap_stride(p.NN);
    const size_t o_push = 0, o_fin = al256(2 * (size_t)(p.NN + 2)), o_out = 2 * o_fin, o_snap = o_out + 256;
    const size_t total = o_snap + (size_t)maxsnap * stride;
    CUDA_TRY(cudaMalloc(&g->d_snap[pi], total));
    char *b = (char *)g->d_snap[pi];
    CUDA_TRY(cudaMemsetAsync(b + o_out, 0, 16, g->stream));
    CUDA_TRY(launch_inc_record(p, (uint16_t *)(b + o_push), (uint16_t *)(b + o_fin), b + o_snap, S, maxsnap, b + o_out,
                               g->stream));
    int32_t out[5];
    CUDA_TRY(cudaMemcpyAsync(out, b + o_out, 20, cudaMemcpyDeviceToHost, g->stream));
    CUDA_TRY(cudaStreamSynchronize(g->stream));
    double mk;
    memcpy(&mk, out + 2, 8);
    if (out[1] != FO_OK || memcmp(&mk, parent_cost, 8) != 0 || out[0] <= 0) return FO_OK;  // level 0 only
    p.push = (const uint16_t *)(b + o_push);
    p.fin = (const uint16_t *)(b + o_fin);
    p.snap = b + o_snap;
    p.snap_S = S;
    p.nsnap = out[0];
    p.snap_stride = (int32_t)stride;
    g->plan_iters[pi] = out[4];
    return FO_OK;
}

static int build_plan(fo_graph *g, int precision) {
    const int pi = precision == FO_PREC_FP64 ? 1 : 0;
    g->plan_ok[pi] = 0;
    g->plan_pv[pi] = g->parent_ver;
    g->plan_mv[pi] = g->model_ver;
    const DGraph &dg = g->dg;
    if (!g->model_set || dg.provider != FO_PROVIDER_PROFILE || dg.variant != FO_EST_MESSAGE_PASSING) return FO_OK;
    const int V = g->V, E = g->E, A = g->A, VB = 2 * V + 2, NN = VB + A;
    if (NN >= 65535 || (int)g->h_parent.size() != 2 * V + A) return FO_OK;
    const int32_t *pn = g->h_parent.data(), *pr = pn + V, *pb = pn + 2 * V;
    std::vector<char> h;
    size_t o[16];
    const int stop = g->dg.phase_stop;  // the parent's full durations, whatever the measurement hook says
    g->dg.phase_stop = 0;
    int st = single(g, pn, pr, pb, VB, precision, nullptr, false, true, h, o);
    g->dg.phase_stop = stop;
    if (st) return st;
    if (*(const int32_t *)(h.data() + o[4]) != FO_OK) return FO_OK;  // the parent itself fails: general path
    const double *dur_c = (const double *)(h.data() + o[14]);
    std::vector<int> gcnt(VB, 0), gmin(VB, INT_MAX), bcnt(A, 0), bmin(A, INT_MAX);
    std::vector<int64_t> bbytes(A, 0);
    for (int v = 0; v < V; v++) {
        gcnt[pn[v]]++;
        gmin[pn[v]] = std::min(gmin[pn[v]], v);
        if (pr[v] >= 0) { gcnt[pr[v]]++; gmin[pr[v]] = std::min(gmin[pr[v]], v); }
    }
    for (int a = 0; a < A; a++) {
        bcnt[pb[a]]++;
        bmin[pb[a]] = std::min(bmin[pb[a]], a);
        bbytes[pb[a]] += g->ar_bytes[a];
    }
    std::vector<int32_t> mptr(VB + 1, 0), bptr(A + 1, 0);
    for (int x = 0; x < VB; x++) mptr[x + 1] = mptr[x] + gcnt[x];
    for (int b = 0; b < A; b++) bptr[b + 1] = bptr[b] + bcnt[b];
    std::vector<uint16_t> mem(std::max(mptr[VB], 1)), bmem(std::max(A, 1));
    {
        std::vector<int32_t> cur(mptr.begin(), mptr.end() - 1);
        for (int v = 0; v < V; v++) {  // ascending: member lists come out sorted
            mem[cur[pn[v]]++] = (uint16_t)v;
            if (pr[v] >= 0) mem[cur[pr[v]]++] = (uint16_t)v;
        }
        std::vector<int32_t> cb(bptr.begin(), bptr.end() - 1);
        for (int a = 0; a < A; a++) bmem[cb[pb[a]]++] = (uint16_t)a;
    }
    std::vector<double> dur(NN, 0.0);
    std::vector<uint16_t> prank(NN, 0);
    std::vector<uint8_t> exists(NN, 0);
    int r = 0;
    for (int x = 0; x < VB; x++)
        if (gcnt[x]) { dur[x] = dur_c[r++]; exists[x] = 1; }
    const int G = r;
    for (int b = 0; b < A; b++)
        if (bcnt[b]) { dur[VB + b] = dur_c[r++]; exists[VB + b] = 1; }
    (void)G;
    for (int x = 0; x < VB; x++) {
        if (!gcnt[x]) continue;
        const int t = gmin[x], other = pn[t] == x ? pr[t] : pn[t];
        prank[x] = (uint16_t)(2 * t + ((other >= 0 && gmin[other] == t && other < x) ? 1 : 0));  // simulator.py:63
    }
    for (int b = 0; b < A; b++)
        if (bcnt[b]) prank[VB + b] = (uint16_t)bmin[b];
    // dependency slots (graph.py:215-261), each recording its CSR position
    auto exp_of = [&](int v) { return pr[v] >= 0 ? pr[v] : pn[v]; };
    std::vector<int32_t> pos_e(2 * (size_t)E + 1, -1), agg_off(E + 1, 0), pos_ar(A + 1, -1);
    for (int e = 0; e < E; e++) {
        const int s = g->e_src[e];
        agg_off[e + 1] = agg_off[e] + (g->agg[e] ? 2 * (g->arp_ptr[s + 1] - g->arp_ptr[s]) : 0);
    }
    std::vector<int32_t> pos_agg(agg_off[E] + 1, -1);
    std::vector<int32_t> ssrc, stgt;
    std::vector<int32_t *> spos;
    auto slot = [&](int src, int tgt, int32_t *pos) { ssrc.push_back(src); stgt.push_back(tgt); spos.push_back(pos); };
    for (int e = 0; e < E; e++) {
        const int s = g->e_src[e], d = g->e_dst[e];
        for (int k = 0; k < 2; k++) {
            const int gid = k ? pr[d] : pn[d];
            if (gid < 0) continue;
            if (!g->agg[e]) {
                if (pn[s] != gid && pr[s] != gid) slot(exp_of(s), gid, &pos_e[2 * e + k]);
            } else {
                for (int q = g->arp_ptr[s], j = 0; q < g->arp_ptr[s + 1]; q++, j++)
                    slot(VB + pb[g->arp[q]], gid, &pos_agg[agg_off[e] + 2 * j + k]);
            }
        }
    }
    for (int a = 0; a < A; a++) slot(exp_of(g->ar_prod[a]), VB + pb[a], &pos_ar[a]);
    const int P = (int)ssrc.size();
    if (P > 32767) return FO_OK;  // successor positions are 15-bit in the ready entries
    std::vector<int32_t> sptr(NN + 1, 0);
    for (int i = 0; i < P; i++) sptr[ssrc[i] + 1]++;
    for (int n = 0; n < NN; n++) sptr[n + 1] += sptr[n];
    std::vector<uint32_t> succ(std::max(P, 1));
    std::vector<int32_t> indeg(NN, 0);
    {
        std::vector<int32_t> cur(sptr.begin(), sptr.end() - 1);
        for (int i = 0; i < P; i++) {
            const int q = cur[ssrc[i]]++;
            *spos[i] = q;
            succ[q] = ((uint32_t)prank[stgt[i]] << 16) | (uint32_t)stgt[i];
            indeg[stgt[i]]++;
        }
    }
    std::vector<IncNode> rec(NN);
    std::vector<uint16_t> indeg16(NN + 2, 0);
    int n_exist = 0;
    std::vector<std::pair<int, int>> rdy_g, rdy_b;
    for (int n = 0; n < NN; n++) {
        if (indeg[n] > 16383) return FO_OK;  // bit 15 of a candidate's indegree marks patched nodes
        rec[n] = IncNode{dur[n], (uint16_t)sptr[n], (uint16_t)sptr[n + 1], prank[n], exists[n], 0};
        indeg16[n] = (uint16_t)indeg[n];
        n_exist += exists[n];
        if (exists[n] && indeg[n] == 0) (n < VB ? rdy_g : rdy_b).push_back({prank[n], n});
    }
    std::sort(rdy_g.begin(), rdy_g.end());
    std::sort(rdy_b.begin(), rdy_b.end());
    std::vector<uint16_t> ready;
    for (auto &x : rdy_g) ready.push_back((uint16_t)x.second);
    for (auto &x : rdy_b) ready.push_back((uint16_t)x.second);
    if (ready.empty()) ready.push_back(0);
    std::vector<uint16_t> gcnt16(VB), gmin16(VB), bcnt16(std::max(A, 1)), bmin16(std::max(A, 1));
    for (int x = 0; x < VB; x++) { gcnt16[x] = (uint16_t)gcnt[x]; gmin16[x] = gcnt[x] ? (uint16_t)gmin[x] : 0; }
    for (int b = 0; b < A; b++) { bcnt16[b] = (uint16_t)bcnt[b]; bmin16[b] = bcnt[b] ? (uint16_t)bmin[b] : 0; }
    if (getenv("FO_PLAN_DUMP")) {  // debugging aid: checksums of the plan's arrays
        auto h64 = [](const void *p, size_t n) {
            uint64_t h = 1469598103934665603ull;
            for (size_t i = 0; i < n; i++) h = (h ^ ((const uint8_t *)p)[i]) * 1099511628211ull;
            return (unsigned long long)h;
        };
        fprintf(stderr, "plan pv=%d prec=%d NN=%d P=%d n_exist=%d ready=%d/%d rec=%llx indeg=%llx succ=%llx dur=%llx pos_e=%llx pos_agg=%llx pos_ar=%llx mem=%llx parent=%llx\n",
                g->parent_ver, precision, NN, P, n_exist, (int)rdy_g.size(), (int)rdy_b.size(),
                h64(rec.data(), sizeof(IncNode) * NN), h64(indeg16.data(), 2 * indeg16.size()), h64(succ.data(), 4 * succ.size()),
                h64(dur.data(), 8 * dur.size()), h64(pos_e.data(), 4 * pos_e.size()), h64(pos_agg.data(), 4 * pos_agg.size()),
                h64(pos_ar.data(), 4 * pos_ar.size()), h64(mem.data(), 2 * mem.size()), h64(pn, 4 * (2 * (size_t)V + A)));
    }
    // one device allocation
    struct Seg { const void *src; size_t bytes; size_t off; };
    Seg segs[] = {
        {rec.data(), sizeof(IncNode) * NN, 0}, {indeg16.data(), 2 * indeg16.size(), 0},
        {succ.data(), 4 * succ.size(), 0}, {gcnt16.data(), 2 * gcnt16.size(), 0}, {gmin16.data(), 2 * gmin16.size(), 0},
        {mptr.data(), 4 * mptr.size(), 0}, {mem.data(), 2 * mem.size(), 0}, {bcnt16.data(), 2 * bcnt16.size(), 0},
        {bmin16.data(), 2 * bmin16.size(), 0}, {bbytes.data(), 8 * bbytes.size(), 0}, {bptr.data(), 4 * bptr.size(), 0},
        {bmem.data(), 2 * bmem.size(), 0}, {pos_e.data(), 4 * pos_e.size(), 0}, {agg_off.data(), 4 * agg_off.size(), 0},
        {pos_agg.data(), 4 * pos_agg.size(), 0}, {pos_ar.data(), 4 * pos_ar.size(), 0}, {ready.data(), 2 * ready.size(), 0},
    };
    size_t total = 0;
    for (auto &sg : segs) { sg.off = total; total += al256(sg.bytes + 8); }
    if (g->d_plan[pi]) { CUDA_TRY(cudaFree(g->d_plan[pi])); g->d_plan[pi] = nullptr; }
    CUDA_TRY(cudaMalloc(&g->d_plan[pi], total));
    char *b = (char *)g->d_plan[pi];
    for (auto &sg : segs)
        if (sg.bytes) CUDA_TRY(cudaMemcpy(b + sg.off, sg.src, sg.bytes, cudaMemcpyHostToDevice));
    IncPlan &p = g->plan[pi];
    p.V = V; p.E = E; p.A = A; p.VB = VB; p.NN = NN; p.P = P; p.n_exist = n_exist;
    p.n_ready_g = (int)rdy_g.size();
    p.n_ready_b = (int)rdy_b.size();
    p.rec = (const IncNode *)(b + segs[0].off);
    p.indeg = (const uint16_t *)(b + segs[1].off);
    p.succ = (const uint32_t *)(b + segs[2].off);
    p.gcnt = (const uint16_t *)(b + segs[3].off);
    p.gmin = (const uint16_t *)(b + segs[4].off);
    p.mptr = (const int32_t *)(b + segs[5].off);
    p.mem = (const uint16_t *)(b + segs[6].off);
    p.bcnt = (const uint16_t *)(b + segs[7].off);
    p.bmin = (const uint16_t *)(b + segs[8].off);
    p.bbytes = (const int64_t *)(b + segs[9].off);
    p.bptr = (const int32_t *)(b + segs[10].off);
    p.bmem = (const uint16_t *)(b + segs[11].off);
    p.pos_e = (const int32_t *)(b + segs[12].off);
    p.agg_off = (const int32_t *)(b + segs[13].off);
    p.pos_agg = (const int32_t *)(b + segs[14].off);
    p.pos_ar = (const int32_t *)(b + segs[15].off);
    p.pnn = g->d_parent;
    p.prr = g->d_parent + V;
    p.pbk = g->d_parent + 2 * V;
    p.ready = (const uint16_t *)(b + segs[16].off);
    p.push = nullptr;
    p.fin = nullptr;
    p.snap = nullptr;
    p.snap_S = 1;
    p.nsnap = 0;
    p.snap_stride = 0;
    st = record_parent_loop(g, pi, h.data() + o[3]);
    if (st) return st;
    g->plan_ok[pi] = 1;
    return FO_OK;
}

// (re)build the plan of this precision when the parent or the cost model changed
static int ensure_plan(fo_graph *g, int precision) {
    const int pi = precision == FO_PREC_FP64 ? 1 : 0;
    if (!g->delta_mode || !g->d_parent) return FO_OK;
    if (g->plan_pv[pi] == g->parent_ver && g->plan_mv[pi] == g->model_ver) return FO_OK;
    return build_plan(g, precision);
}

extern "C" {

int fo_simulate(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t gid_bound,
                int32_t precision, const double *durations, int32_t *c_id, double *c_start, double *c_end,
                int32_t *n_compute, int32_t *b_id, double *b_start, double *b_end, int32_t *n_comm, double *makespan,
                int32_t *bad_node_out) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    std::lock_guard<std::mutex> lk(g->mu);
    if (!g->model_set && !durations) return fail(FO_INVALID_ARG, "no cost model set");
    CUDA_TRY(cudaSetDevice(g->device));
    std::vector<char> h;
    size_t o[16];
    int st = single(g, ngid, rgid, bkt, gid_bound, precision, durations, true, false, h, o);
    if (st) return st;
    int status = *(int32_t *)(h.data() + o[4]);
    *makespan = *(double *)(h.data() + o[3]);
    int nc = *(int32_t *)(h.data() + o[12]), nb = *(int32_t *)(h.data() + o[13]);
    if (n_compute) *n_compute = nc;
    if (n_comm) *n_comm = nb;
    if (c_id) {
        memcpy(c_id, h.data() + o[6], 4u * nc);
        memcpy(c_start, h.data() + o[7], 8u * nc);
        memcpy(c_end, h.data() + o[8], 8u * nc);
    }
    if (b_id) {
        memcpy(b_id, h.data() + o[9], 4u * nb);
        memcpy(b_start, h.data() + o[10], 8u * nb);
        memcpy(b_end, h.data() + o[11], 8u * nb);
    }
    if (bad_node_out) *bad_node_out = *(int32_t *)(h.data() + o[15]);
    if (status == 100) return fail(FO_UNSUPPORTED, "fused group larger than the device estimator scratch");
    return status;
}

int fo_node_durations(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t gid_bound,
                      int32_t precision, double *dur_out, int32_t *n_groups_out, int32_t *bad_node_out) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    if (g->device < 0) return fail(FO_CUDA_ERROR, "graph handle was created without a device");
    std::lock_guard<std::mutex> lk(g->mu);
    if (!g->model_set) return fail(FO_INVALID_ARG, "no cost model set");
    CUDA_TRY(cudaSetDevice(g->device));
    std::vector<char> h;
    size_t o[16];
    int st = single(g, ngid, rgid, bkt, gid_bound, precision, nullptr, false, true, h, o);
    if (st) return st;
    int G = *(int32_t *)(h.data() + o[15] + 4);
    *n_groups_out = G;
    // the number of buckets is the number of distinct bucket ids
    std::vector<char> seen(g->A + 1, 0);
    int B = 0;
    for (int a = 0; a < g->A; a++)
        if (bkt[a] >= 0 && bkt[a] < g->A && !seen[bkt[a]]) { seen[bkt[a]] = 1; B++; }
    memcpy(dur_out, h.data() + o[14], 8u * (G + B));
    if (bad_node_out) *bad_node_out = *(int32_t *)(h.data() + o[15]);
    int status = *(int32_t *)(h.data() + o[4]);
    if (status == 100) return fail(FO_UNSUPPORTED, "fused group larger than the device estimator scratch");
    return status;
}

}  // extern "C"
