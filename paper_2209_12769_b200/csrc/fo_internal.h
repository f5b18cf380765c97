// Internal declarations shared by the CUDA scoring kernels (score.cu), the
// C-ABI layer (capi.cu) and the native batch-expand / search engine
// (engine.cpp).  Not part of the public ABI (include/disco_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/disco_b200.h"

namespace fo {

constexpr int kHidden = 32;  // lane = hidden channel in the message-passing kernel

struct MemoEnt {  // estimator memo slot (score.cu)
    unsigned long long k1, k2;
    double v;
    unsigned long long pad;
};

// Device-side view of one graph + cost model, passed by value to kernels.
struct DGraph {
    int32_t V, E, A;
    // static graph (SoA, build_graph order)
    const int32_t *e_src, *e_dst;
    const int64_t *e_bytes;
    const uint8_t *e_agg;       // _consumes_aggregate (graph.py:225-235)
    const int32_t *in_ptr, *in_e;   // edge indices by destination op
    const int32_t *out_ptr, *out_e; // edge indices by source op
    const int32_t *arp_ptr, *arp;   // AllReduces by producer op
    const int32_t *ar_prod;
    const int64_t *ar_bytes;
    const uint8_t *op_kind;
    const double *op_prof;      // lookup(profile, op) or NaN
    const double *op_compute;   // OpNode.compute_us or NaN
    const int64_t *op_out, *op_in;
    // message passing (lane = channel; hidden padded to 32 with zeros)
    const float *H0f;           // [V][32]  X_std @ W_emb^T per op (estimator.py:369)
    const double *H0d;
    const float *Wf;            // packed transposed weights, see mp_layout()
    const double *Wd;
    int32_t layers;
    // cost model
    int32_t provider, variant;
    double C, D, launch, mem, out_scale;
    double lin_w[12], lin_b, agg_mean[12], agg_std[12];
    int32_t lin_norm;
    int32_t pairs_max;          // bound on contracted dependency pairs per candidate
    MemoEnt *memo[2];           // MP predictions by member set: [fp32, fp64]
    uint32_t memo_mask;
    int32_t phase_stop;         // measurement hook: launches stop after K1 (1) or K2 (2); 0 = full
    int32_t mp_arith;           // FP32 MP transforms: 0 FFMA, 1 TF32 tensor cores, 2 3xTF32 tensor cores
    // MP embedding for feature-level prediction (fo_predict_features): W_emb
    // [h][F] row-major and the node_norm mean / std [F] (nullptr: none)
    const double *emb, *emb_mean, *emb_std;
    int32_t emb_h, emb_F;
    // hardware-oracle jitter (workloads.py:254-291): noise, "{seed}|" prefix,
    // per-op content-key fragments (CSR over ops)
    double noise;
    const uint8_t *kpre;
    int32_t kpre_len;
    const uint8_t *okb;
    const int64_t *oko;
};

// Packed message-passing weights (float or double), all transposed so lane c
// reads element [k][c]:  W_l^T (L x 32 x 32) | W_r^T | A1^T | A2^T | c1 | c2 | a3 | c3
struct MpLayout {
    int64_t wl, wr, a1, a2, c1, c2, a3, c3, total;
};
__host__ __device__ inline MpLayout mp_layout(int layers) {
    MpLayout m;
    m.wl = 0;
    m.wr = (int64_t)layers * 1024;
    m.a1 = m.wr + 1024;
    m.a2 = m.a1 + 1024;
    m.c1 = m.a2 + 1024;
    m.c2 = m.c1 + 32;
    m.a3 = m.c2 + 32;
    m.c3 = m.a3 + 32;
    m.total = m.c3 + 32;
    return m;
}

// Per-warp workspace (one candidate at a time), byte offsets.
struct WsLayout {
    int64_t gmap, bmap, g2id, b2id, nn, rr, bki, gmin, gcnt, bmin, btot, indeg, scnt, sptr, succ, prank, dur, fused,
        gptr, gmem, gint, gin, gout, vis, zl, csim, rank, tlid;
    // per-warp fused-group scratch: copy w at gs0 + w * gs_stride, fields relative to the copy
    int64_t gs0, gs_stride, g_msort, g_lidx, g_zl, g_nbptr, g_nb, g_mark, g_H, g_P;
    int64_t total;
    int32_t mpcap;
};
WsLayout ws_layout(int V, int E, int A, int VB, int pairs_max, int mpcap, int nws = 1);
constexpr int kMpCapDefault = 2048;  // fused-group size the per-warp MP scratch holds

struct TimelineOut {
    int32_t *c_id;
    double *c_start, *c_end;
    int32_t *n_c;
    int32_t *b_id;
    double *b_start, *b_end;
    int32_t *n_b;
};

// Launch geometry: persistent grid and the per-warp shared-memory arena.
struct ScoreGeo {
    int grid, blocks_per_sm, sm_nodes, sm_pairs, sm_bytes;
    int team;  // 1: one 128-thread block per candidate (latency mode)
};
ScoreGeo score_geometry(const DGraph &g, int K, int num_sms, int precision);
// Sparse candidates: a resident parent state (ngid[V] | rgid[V] | bkt[A],
// int32) and, per candidate k, changes [off[k], off[k+1]) of (index, value)
// pairs over that concatenated index space.
struct DeltaIn {
    const int32_t *base = nullptr, *off = nullptr, *chg = nullptr;
};
// Kernel launch (score.cu).  ext_dur / tl / dur_out / bad_out are optional and
// only used with K == 1.
cudaError_t launch_score(const DGraph &g, const void *ngid, const void *rgid, const void *bkt, int idx16, int K,
                         int VB, int precision, char *ws, const WsLayout &L, const ScoreGeo &geo,
                         double *cost_out, int32_t *status_out, const double *ext_dur, TimelineOut tl,
                         double *dur_out, int32_t *bad_out, int32_t *ngroups_out, cudaStream_t stream,
                         int retry_only = 0, const DeltaIn *delta = nullptr);
int score_warps_per_block();
int score_slots(const ScoreGeo &geo);       // workspace slots a launch uses
int score_team_warps(const ScoreGeo &geo);  // warps per candidate
// predict_fused (estimator.py:462-470) from one group's features, one warp
struct FeatIn {
    int32_t n, m;
    const int32_t *slot, *edges;  // vocab slot per node; (src, dst) local pairs
    const double *c;
    const long long *in, *out;
    double agg[6];                // SubgraphFeatures.aggregate_vector()
    int32_t *nbptr, *nb;          // scratch: n + 1, 2m
    char *H0, *H, *P;             // scratch: n x 32 T each
};
cudaError_t launch_predict_features(const DGraph &g, const FeatIn &in, int precision, double *pred_out,
                                    cudaStream_t stream);
// ---------------------------------------------------------------------------
// Incremental scoring of sparse candidates (score_inc.cuh).  A sparse
// candidate is a handful of (index, value) changes against the resident
// parent, so its contracted schedule DAG is the parent's with a handful of
// nodes patched.  The parent's DAG is contracted ONCE per parent ("plan",
// built on the host by fo_set_parent's first scoring call) in gid space:
// group node = engine group id [0, VB), bucket node = VB + bucket id.  Per
// candidate the kernel derives only the changed dependency slots and the
// nodes they touch; the event loop walks the parent's successor lists (read
// only, shared by every warp of an SM, so L1-resident) plus a few rebuilt
// lists, with the candidate's indegrees in shared memory.
struct __align__(16) IncNode {  // parent node record, 16 B: one 128-bit load per released node
    double dur;
    uint16_t sb, se;  // successor range in IncPlan::succ (bit 15 of sb: rebuilt list, candidates only)
    uint16_t prank;   // tie-break rank (simulator.py:63-64): 2 * min member + replica bit, or min AR
    uint8_t exists, pad;
};
struct IncPlan {
    int32_t V, E, A, VB, NN, P, n_exist, n_ready_g, n_ready_b;
    const IncNode *rec;        // [NN]
    const uint16_t *indeg;     // [NN + pad]
    const uint32_t *succ;      // [P] (prank << 16) | target
    const uint16_t *gcnt, *gmin;                 // [VB]
    const int32_t *mptr; const uint16_t *mem;    // group members, ascending: [VB + 1], [mptr[VB]]
    const uint16_t *bcnt, *bmin; const int64_t *bbytes;  // [A]
    const int32_t *bptr; const uint16_t *bmem;   // bucket members (AR indices): [A + 1], [A]
    const int32_t *pos_e;      // [2E] parent succ position of non-aggregate slot (e, copy), -1 inactive
    const int32_t *agg_off;    // [E + 1] first aggregate slot of edge e (2 per AllReduce of its source)
    const int32_t *pos_agg;    // [agg_off[E]]
    const int32_t *pos_ar;     // [A] bucket <- export(producer) slot
    const int32_t *pnn, *prr, *pbk;  // the parent state (engine ids)
    const uint16_t *ready;     // level-0 ready nodes: lane g [0, n_ready_g), lane b after, each by prank
    // the parent's own event loop, recorded once per plan (inc_record_kernel):
    const uint16_t *push;      // [NN] loop iteration + 1 in which the node became ready (0: level 0, 0xffff: never)
    const uint16_t *fin;       // [NN] loop iteration + 1 in which it finished
    const char *snap;          // loop state at the top of iteration j * snap_S, j = 1 .. nsnap (IncSnap layout)
    int32_t snap_S, nsnap, snap_stride;
};
struct IncLayout {  // per-warp global scratch (byte offsets) and shared-memory arena
    int64_t hdr, chg, rem, add, dn, work, dirty, mem, pcsr, ring, indeg, gs0, total;
    int64_t g_msort, g_lidx, g_zl, g_nbptr, g_nb, g_mark, g_H, g_P;
    int32_t mem_cap, pcsr_cap, mpcap;
    int32_t ring_g, ring_b;  // ready-run ring sizes (powers of two >= the nodes of each lane: no overflow)
    int32_t s_indeg, s_pbm, s_abm, s_lbm, s_tbm, s_ppre, s_cbm, s_cnt, s_bytes;  // setup kernel smem (per warp)
    int32_t k_indeg, k_pbm, k_ppre, k_tbm, k_ring, k_state, k_bytes;  // event-loop kernel smem (k_indeg < 0: global)
    int32_t NW, CW, RW, s_rbm, s_chg, s_cpre, s_acnt;
};
constexpr int kIncMaxChg = 64, kIncMaxOps = 256, kIncMaxDirty = 192;
constexpr int kRetryGeneral = 101;  // internal status: the incremental kernel hands the candidate to score_kernel
constexpr int kIncPending = 102;    // internal status: set up, waiting for the event-loop kernel
IncLayout inc_layout(int V, int E, int A, int VB, int P, bool smem_indeg);
struct IncQ;
cudaError_t launch_score_inc(const DGraph &g, const IncPlan &p, const IncLayout &L, const int32_t *off,
                             const int32_t *chg, int K, int precision, char *ws, int grid, IncQ *queue, int *qcount,
                             int qcap, double *cost_out, int32_t *status_out, cudaStream_t stream, int diag = 0);
constexpr int kIncQueuePerCand = kIncMaxDirty;  // estimator queue entries per candidate: never full (a claimed memo slot always gets its value)
int score_inc_blocks_per_sm(const IncLayout &L, int precision);
// record the parent's event loop into the plan's push / snapshot arrays;
// out: {nsnap, status} as int32 then the makespan as a double (16 bytes)
int64_t inc_snap_stride(int NN);
cudaError_t launch_inc_record(const IncPlan &p, uint16_t *push, uint16_t *fin, char *snap, int S, int maxsnap,
                              void *out, cudaStream_t stream);

cudaError_t launch_batch_best(const double *cost, const int32_t *status, int K, int64_t id_offset, double *out,
                              cudaStream_t stream, int pairs = 0);

}  // namespace fo

// Host-side handle behind the opaque fo_graph.
struct fo_graph {
    int device = 0;
    int V = 0, E = 0, A = 0;
    // host copies
    std::vector<int32_t> op_kind, e_src, e_dst, ar_prod;
    std::vector<int64_t> op_out, op_in, e_bytes, ar_bytes;
    std::vector<double> op_prof, op_compute;
    std::vector<int32_t> in_ptr, in_e, out_ptr, out_e, arp_ptr, arp;
    std::vector<uint8_t> agg;
    int32_t pairs_max = 0;
    // device buffers
    void *d_static = nullptr;  // one allocation for the static graph
    void *d_model = nullptr;   // H0 + weights
    void *d_memo = nullptr;    // estimator memo tables
    size_t memo_slots = 0;     // slots per precision
    void *d_keys = nullptr;    // hardware-oracle jitter key bytes
    fo::DGraph dg{};
    bool model_set = false;
    // scoring workspace
    char *d_ws = nullptr;
    size_t ws_bytes = 0;
    char *d_ws_big = nullptr;  // second-pass workspace for fused groups beyond kMpCapDefault
    size_t ws_big_bytes = 0;
    char *d_ws_alt = nullptr;  // a second first-pass workspace: concurrent batches on another stream
    size_t ws_alt_bytes = 0;
    // host API staging
    void *d_io = nullptr;
    // resident parent of sparse (delta) candidates, engine ids
    int32_t *d_parent = nullptr;
    std::vector<int32_t> h_parent;
    size_t io_bytes = 0;
    void *h_pinned = nullptr;
    size_t pinned_bytes = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 0;
    size_t mem_total = 0;  // device memory (workspace budget)
    // fo_score_delta_submit / fo_score_wait: kSubmitSlots in-flight submissions;
    // H2D and D2H on their own streams so one batch's transfers overlap another's
    // kernels, and the kernels of consecutive submissions on their own compute
    // streams (slot 0: the handle's stream) with their own scratch (Sub)
    static constexpr int kSubmitSlots = 4;
    struct AsyncSlot {
        char *d = nullptr;
        size_t bytes = 0;
        cudaEvent_t h2d = nullptr, kdone = nullptr, done = nullptr;
        int64_t ticket = -1;
    } aslot[kSubmitSlots];
    struct Sub {  // slots 1.. (slot 0 uses the handle's own scratch)
        char *ws_inc = nullptr;
        size_t ws_inc_bytes = 0;
        void *inc_q = nullptr;
        size_t inc_q_bytes = 0;
        void *memo = nullptr;
        char *ws = nullptr;  // general-kernel first-pass workspace
        size_t ws_bytes = 0;
        cudaStream_t stream = nullptr;
    } sub[kSubmitSlots];
    cudaStream_t hstream = nullptr, dstream = nullptr;
    int64_t next_ticket = 0;
    // incremental delta scoring (score_inc.cuh): the parent's plan per
    // precision, rebuilt when the parent or the cost model changes
    int parent_ver = 0, model_ver = 0;
    void *d_plan[2] = {nullptr, nullptr};
    void *d_snap[2] = {nullptr, nullptr};  // the parent loop record of each plan
    int plan_iters[2] = {0, 0};             // the parent loop's iterations
    fo::IncPlan plan[2]{};
    int plan_pv[2] = {-1, -1}, plan_mv[2] = {-1, -1};
    int plan_ok[2] = {0, 0};
    char *d_ws_inc = nullptr;
    size_t ws_inc_bytes = 0;
    void *d_inc_q = nullptr;  // estimator queue (IncQ entries) + its counter
    size_t inc_q_bytes = 0;
    int delta_mode = 1;  // 1: incremental kernel when the plan allows it; 0: general kernel only
    std::mutex mu;
};

namespace fo {
void set_error(const std::string &msg);
int fail(int status, const std::string &msg);
int xchg_round(fo_xchg *x, int64_t round, const double *best, int R, int active);  // xchg.cpp
void xchg_final(fo_xchg *x, const double *best, int R);
void xchg_attach_cfg(fo_xchg *x, int64_t seed_offset, int every);
// Ensure the handle's workspace can hold `slots` warps for gid bound VB.
int ensure_workspace(fo_graph *g, int VB, int slots, WsLayout *L, bool big = false, int nws = 1, int alt = 0);
// Score K device-resident candidates (used by fo_score and the search engine).
int score_device(fo_graph *g, const void *ngid, const void *rgid, const void *bkt, int idx16, int K, int VB,
                 int precision, double *cost, int32_t *status, cudaStream_t stream, int alt_ws = 0);
int score_delta_device(fo_graph *g, const int32_t *off, const int32_t *chg, int K, int precision, double *cost,
                       int32_t *status, cudaStream_t stream, int slot = 0);
}  // namespace fo
