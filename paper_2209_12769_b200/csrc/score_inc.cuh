// score_inc.cuh -- incremental scoring of sparse candidates (included by
// score.cu inside namespace fo; it reuses that file's warp helpers, the MP
// forward, the estimator memo and the ring-buffer ready runs).
//
// A sparse candidate is (index, value) changes over ngid | rgid | bkt against
// the resident parent.  The reference rebuilds the whole contraction for
// every candidate (_Index, graph.py:117-274; simulate, simulator.py:61-62);
// here the parent's contraction exists once (IncPlan, host-built) and a
// candidate only re-derives what its changes touch:
//
//   setup  the dependency SLOTS whose endpoints changed (one slot per
//          (edge, copy of the consumer) -- graph.py:237-261 -- per
//          (aggregate edge, AllReduce, copy), and per AllReduce -- :215-223):
//          each is removed from / added to the parent's DAG; the nodes they
//          leave or enter and the groups / buckets whose membership changed
//          become PATCHED nodes (new duration, tie-break rank, existence,
//          successor list)
//   K2     durations of the patched groups: profile lookup for singletons,
//          the MP forward (estimator.py:363-389, memoised) for fused groups,
//          C * bytes + D for buckets (comm.py:45-49)
//   K3     the event loop of simulator.py:117-140 over the parent's successor
//          lists (read only and shared by every warp of the SM, so they stay
//          in L1), the rebuilt lists of patched nodes, and the candidate's
//          indegrees in shared memory
//
// Anything outside the fast path's bounds (more changes than kIncMaxChg, a
// ring or scratch overflow, a missing profile entry, an invalid id) ends the
// candidate with kRetryGeneral and the general kernel scores it instead, so
// results and error statuses are the general path's by construction.

struct IncDirty {  // a patched node of one candidate (sorted by node id)
    double dur;
    uint16_t prank, sb, se;
    uint8_t exists, fused;
};
struct IncWork {  // setup record of a patched node, in discovery order
    int32_t node, cnt, mn, mb, me, pad;
    int64_t bytes;
    unsigned long long h1, h2;  // member-set hash of a fused group (the memo key)
};

constexpr int kIncRingG = 128, kIncRingB = 64;  // shared-memory ready-run capacities per lane
// estimator kernel: member sets up to this size keep H / P in shared memory
// (16 KB per block either way: more would cost the fp64 kernel a resident block)
template <typename T>
constexpr int kIncMpSmem = sizeof(T) == 8 ? 8 : 16;

IncLayout inc_layout(int V, int E, int A, int VB, int P, bool smem_indeg) {
    IncLayout L{};
    const int NN = VB + A;
    int64_t o = 0;
    auto take = [&](int64_t bytes) { int64_t r = o; o = (o + bytes + 15) & ~int64_t(15); return r; };  // int4 / Ent16 entries
    L.mem_cap = 2 * V + A + 64;
    L.pcsr_cap = std::min<int64_t>(P + kIncMaxOps + 64, 32767);
    L.hdr = take(16);
    L.chg = take(8 * kIncMaxChg);
    L.rem = take(16 * kIncMaxOps);
    L.add = take(16 * kIncMaxOps);
    L.dn = take(4 * kIncMaxDirty);
    L.work = take(sizeof(IncWork) * kIncMaxDirty);
    L.dirty = take(sizeof(IncDirty) * (kIncMaxDirty + 1) + 2 * kIncMaxDirty);  // + rank -> slot map
    L.mem = take(4 * (int64_t)L.mem_cap);
    L.pcsr = take(4 * (int64_t)L.pcsr_cap);
    L.ring_g = kIncRingG;
    L.ring_b = kIncRingB;
    L.ring = 0;
    L.indeg = smem_indeg ? -1 : take(2 * (int64_t)(NN + 2));
    const int64_t cap = std::min(V, kMpCapDefault);
    L.mpcap = (int)cap;
    L.gs0 = o;
    int64_t q = 0;
    auto sub = [&](int64_t bytes) { int64_t r = q; q = align8(q + bytes); return r; };
    L.g_msort = sub(4 * (cap + 1));
    L.g_lidx = sub(4 * (int64_t)V);
    L.g_zl = sub(4 * (cap + 1));
    L.g_nbptr = sub(4 * (cap + 1));
    L.g_nb = sub(4 * (2 * (int64_t)E + 1));
    L.g_mark = sub(4 * (int64_t)V);
    L.g_H = sub(8 * cap * kHidden);
    L.g_P = sub(8 * cap * kHidden);
    o += q;
    L.total = ((o + 255) & ~int64_t(255)) + 256;  // per-warp slots stay 256-byte aligned
    // per-warp shared-memory arena
    L.NW = (NN + 31) / 32;
    L.CW = (2 * V + A + 31) / 32;
    int32_t s = 0;
    auto stake = [&](int32_t bytes) { int32_t r = s; s = (s + bytes + 15) & ~15; return r; };
    L.s_indeg = -1;  // the setup kernel keeps no indegrees
    L.s_pbm = stake(4 * L.NW);
    L.s_abm = stake(4 * L.NW);
    L.s_lbm = stake(4 * L.NW);
    L.s_tbm = -1;
    L.s_ppre = stake(2 * L.NW + 2);
    L.s_cbm = stake(4 * L.CW);
    L.s_cnt = stake(4 * 8);
    L.RW = (P + 31) / 32;
    L.s_rbm = stake(4 * L.RW);         // removed parent successor positions
    L.s_chg = stake(8 * kIncMaxChg);   // the sorted changes
    L.s_cpre = stake(L.CW + 4);        // their bitmap word prefix
    L.s_acnt = stake(4 * kIncMaxDirty); // added slots per patched node
    L.s_bytes = s;
    s = 0;
    L.k_indeg = smem_indeg ? stake(2 * (NN + 2)) : -1;
    L.k_pbm = stake(4 * L.NW);
    L.k_ppre = stake(2 * L.NW + 2);
    L.k_tbm = stake(4 * L.NW);
    L.k_ring = stake(8 * (kIncRingG + kIncRingB));
    L.k_state = stake(128);  // IncK3State: prep -> run hand-off
    L.k_bytes = s;
    return L;
}

struct IncQ {  // a member set queued for the estimator kernel
    const int *mem;  // ascending op indices, in the queuing warp's scratch
    int32_t slot;    // memo slot that also receives the prediction, or -1
    int32_t n;
    double v;        // the prediction (read by the queuing candidate)
    unsigned long long h1, h2;  // the set's memo key
    int64_t pad;
};

struct IncArgs {
    DGraph g;
    IncPlan p;
    IncLayout L;
    const int32_t *doff, *dchg;
    IncQ *queue;
    int *qcount;
    int qcap;
    MemoEnt *memo;  // this precision's memo table, or nullptr (memo off)
    int K;
    char *ws;
    double *cost_out;
    int32_t *status_out;
    int stop_after;
    int diag;  // fo_set_delta_mode 2: hand-backs keep a status that says why
    unsigned long long *stats;  // diag: event-loop fast-forward counters (fo_inc_stats), or nullptr
};

// counters in the per-warp shared arena
enum { kCRem = 0, kCAdd = 1, kCDirty = 2, kCMem = 3, kCPcsr = 4, kCFail = 5, kCExist = 6 };

struct IncCtx {
    const IncArgs *a;
    int2 *chg;
    int4 *rem;
    int4 *add;  // (source, target, the target's parent rank, 0)
    int *dn;
    IncWork *work;
    IncDirty *dirty;
    uint16_t *r2s;
    int *mem;
    uint32_t *pcsr;
    Ent16 *ring;
    uint16_t *indeg;
    uint32_t *pbm, *abm, *lbm, *tbm, *cbm, *rbm;
    uint8_t *cpre;  // changed-index bitmap word prefix (<= 64 changes)
    uint32_t *acnt; // per patched rank: added slots, then their fill cursor
    uint16_t *ppre;
    int *cnt;
    int *hdr;  // hand-off from the setup kernel to the event-loop kernel: nd, nrem, nadd, N
    int nchg;
};

__device__ __forceinline__ bool ibit(const uint32_t *bm, int i) { return (bm[i >> 5] >> (i & 31)) & 1u; }

// candidate value at index i of ngid | rgid | bkt: the parent's unless changed
// (the sorted change list is in index order, so a changed index's position
// is its rank in the changed-index bitmap: a word prefix plus a popcount)
__device__ __forceinline__ int icval(const IncCtx &c, int i, int pv) {
    const uint32_t w = c.cbm[i >> 5];
    if (!((w >> (i & 31)) & 1u)) return pv;
    return c.chg[(int)c.cpre[i >> 5] + __popc(w & ((1u << (i & 31)) - 1u))].y;
}
__device__ __forceinline__ int inn(const IncCtx &c, int v) { return icval(c, v, c.a->p.pnn[v]); }
__device__ __forceinline__ int irr(const IncCtx &c, int v) { return icval(c, c.a->p.V + v, c.a->p.prr[v]); }
__device__ __forceinline__ int ibk(const IncCtx &c, int a) { return icval(c, 2 * c.a->p.V + a, c.a->p.pbk[a]); }
__device__ __forceinline__ bool iop_changed(const IncCtx &c, int v) {
    return ibit(c.cbm, v) || ibit(c.cbm, c.a->p.V + v);
}
// a setup failure hands the candidate to the general kernel; the code says why
// (visible as status 110 + code in the diagnostic mode, fo_set_delta_mode 2)
__device__ __forceinline__ void ifail(const IncCtx &c, int code = 1) { c.cnt[kCFail] = code; }

__device__ void imark(const IncCtx &c, int n, int flags) {
    const uint32_t b = 1u << (n & 31);
    if (flags & 1) atomicOr(&c.abm[n >> 5], b);
    if (flags & 2) atomicOr(&c.lbm[n >> 5], b);
    if (atomicOr(&c.pbm[n >> 5], b) & b) return;
    const int s = atomicAdd(&c.cnt[kCDirty], 1);
    if (s >= kIncMaxDirty) { ifail(c, 2); return; }
    c.dn[s] = n;
}

// one dependency slot before (parent) and after (candidate) the changes
__device__ void islot(const IncCtx &c, int pos, bool oact, int osrc, int otgt, bool nact, int nsrc, int ntgt) {
    if (oact && nact && osrc == nsrc && otgt == ntgt) return;
    if (oact) {
        const int s = atomicAdd(&c.cnt[kCRem], 1);
        if (s >= kIncMaxOps || pos < 0) ifail(c, 3);
        else c.rem[s] = make_int4(pos, osrc, otgt, 0);
    }
    if (nact) {
        const int s = atomicAdd(&c.cnt[kCAdd], 1);
        if (s >= kIncMaxOps) ifail(c, 4);
        else c.add[s] = make_int4(nsrc, ntgt, c.a->p.rec[ntgt].prank, 0);  // rank loaded here, lanes in parallel
    }
}

// aggregate edge e, j-th AllReduce a of its source: bucket(a) -> every copy of
// the consumer (graph.py:237-247)
__device__ void iagg_slots(const IncCtx &c, int e, int j, int a, int pnd, int prd, int cnd, int crd) {
    const IncPlan &p = c.a->p;
    const int osrc = p.VB + p.pbk[a], nsrc = p.VB + ibk(c, a);
    const int base = p.agg_off[e] + 2 * j;
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const int ot = k ? prd : pnd, nt = k ? crd : cnd;
        islot(c, ot >= 0 ? p.pos_agg[base + k] : -1, ot >= 0, osrc, ot, nt >= 0, nsrc, nt);
    }
}

// every slot of edge e (graph.py:249-261 non-aggregate, :237-247 aggregate)
__device__ void iedge_slots(const IncCtx &c, int e) {
    const DGraph &g = c.a->g;
    const IncPlan &p = c.a->p;
    const int s = g.e_src[e], d = g.e_dst[e];
    const int pnd = p.pnn[d], prd = p.prr[d], cnd = inn(c, d), crd = irr(c, d);
    if (!g.e_agg[e]) {
        const int pns = p.pnn[s], prs = p.prr[s], cns = inn(c, s), crs = irr(c, s);
        const int osrc = prs >= 0 ? prs : pns, nsrc = crs >= 0 ? crs : cns;  // export group (graph.py:158-159)
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int ot = k ? prd : pnd, nt = k ? crd : cnd;
            const bool oact = ot >= 0 && pns != ot && prs != ot, nact = nt >= 0 && cns != nt && crs != nt;
            islot(c, oact ? p.pos_e[2 * e + k] : -1, oact, osrc, ot, nact, nsrc, nt);
        }
    } else {
        for (int q = g.arp_ptr[s], j = 0; q < g.arp_ptr[s + 1]; q++, j++) iagg_slots(c, e, j, g.arp[q], pnd, prd, cnd, crd);
    }
}

// bucket(a) <- export(producer(a)) (graph.py:215-223)
__device__ void iar_slot(const IncCtx &c, int a) {
    const IncPlan &p = c.a->p;
    const int pr = c.a->g.ar_prod[a];
    const int po = p.prr[pr] >= 0 ? p.prr[pr] : p.pnn[pr];
    const int cr = irr(c, pr), co = cr >= 0 ? cr : inn(c, pr);
    islot(c, p.pos_ar[a], true, po, p.VB + p.pbk[a], true, co, p.VB + ibk(c, a));
}

__device__ __forceinline__ int irank(const IncCtx &c, int n) {
    const uint32_t w = c.pbm[n >> 5];
    return (int)c.ppre[n >> 5] + __popc(w & ((1u << (n & 31)) - 1u));
}

extern __shared__ __align__(16) char fo_inc_smem[];  // the dynamic arena, addressed by 32-bit offsets

// A ready entry is one u64 in a shared-memory ring: (level << 16 | prank) in
// the high word -- the reference's (rt, tiebreak, id) order -- and the node
// (bit 16: patched) in the low word.  The node's record (duration, successor
// range) is read when it starts: the parent's from the L1-resident plan, a
// patched node's from the candidate's table.
__device__ __forceinline__ unsigned long long inc_ent(uint32_t key, unsigned t, unsigned patched) {
    return ((unsigned long long)key << 32) | (patched << 16) | t;
}

// the record of a patched node (rare): the candidate's table at its rank
__device__ __noinline__ IncDirty inc_patched_rec(const IncDirty *__restrict__ dirty, uint32_t s_pbm, uint32_t s_ppre,
                                                 unsigned t) {
    const uint32_t w = ((const uint32_t *)(fo_inc_smem + s_pbm))[t >> 5];
    const uint16_t *ppre = (const uint16_t *)(fo_inc_smem + s_ppre);
    return dirty[(int)ppre[t >> 5] + __popc(w & ((1u << (t & 31)) - 1u))];
}

// push into a ready run (sorted ring); keys only grow, so an append is the
// common case.  false when the ring is full.
__device__ __forceinline__ bool inc_push(unsigned long long *buf, unsigned m, int head, int &tail, uint32_t &last,
                                         unsigned long long x) {
    const uint32_t key = (uint32_t)(x >> 32);  // keys are unique: the high word orders the entries
    if (tail - head > (int)m) return false;
    // last bounds the run's keys from above (an emptied run keeps the bound,
    // and a smaller key then takes the insertion path, which is correct too)
    if (key >= last) {
        buf[(tail++) & m] = x;
        last = key;
        return true;
    }
    int i = tail++;
    while (i > head) {
        const unsigned long long q = buf[(i - 1) & m];
        if ((uint32_t)(q >> 32) <= key) break;
        buf[i & m] = q;
        i--;
    }
    buf[i & m] = x;
    return true;
}

// Loop state at the top of one iteration of inc_ring_loop: the state a
// candidate starts from -- level 0 (all zero, idle lanes) or a snapshot of the
// parent's own loop (IncSnap).  head / tail are absolute run positions (head =
// nodes started on the lane so far).
struct IncLoopState {
    int32_t headg, tailg, headb, tailb;
    uint32_t sb0, se0, sb1, se1;  // successor ranges of the running nodes
    unsigned long long end0, end1, nowb;
    uint32_t level, iter;
    uint32_t run0, run1;  // the running nodes (snapshots only)
};
// A snapshot: the state, then the ready runs' entries (head first), then the
// parent's indegrees (NN + 2 u16).
constexpr int kIncSnapRuns = 128, kIncSnapDeg = kIncSnapRuns + 8 * (kIncRingG + kIncRingB);
int64_t inc_snap_stride(int NN) { return kIncSnapDeg + ((2 * (int64_t)(NN + 2) + 127) & ~int64_t(127)); }

// Recording hooks of the parent's loop (inc_record_kernel only).
struct IncRecOut {
    uint16_t *push, *fin;  // iteration + 1 in which a node became ready / finished
    char *snap;
    int S, maxsnap;
    int64_t stride;
    int *nsnap, *iters;
};

// The event loop (simulator.py:117-140) of ring_loop over the parent's
// successor lists and the candidate's rebuilt ones.  Indegrees (SI), the
// patched bitmap and the ready rings in shared memory, 32-bit addressed.
// Starts from the state st (level 0, or a parent snapshot whose iterations
// the candidate shares).  false on ring overflow.  REC: the parent's own run,
// recording every node's push iteration and a snapshot every S iterations.
template <bool SI, bool REC = false>
__device__ __forceinline__ bool inc_ring_loop(const IncPlan &p, const uint32_t *__restrict__ csucc,
                                              const IncDirty *__restrict__ dirty, uint16_t *__restrict__ gindeg,
                                              uint32_t s_indeg, uint32_t s_pbm, uint32_t s_ppre, uint32_t s_ring,
                                              const IncLoopState &st, int N, double *cost_out, int32_t *status_out,
                                              const IncRecOut *ro = nullptr) {
    const uint32_t *__restrict__ psucc = p.succ;
    const IncNode *__restrict__ rec = p.rec;
    uint16_t *__restrict__ indeg = SI ? (uint16_t *)(fo_inc_smem + s_indeg) : gindeg;
    unsigned long long *rg = (unsigned long long *)(fo_inc_smem + s_ring);
    unsigned long long *rb = rg + kIncRingG;
    constexpr unsigned mg = kIncRingG - 1, mb = kIncRingB - 1;
    const unsigned VB = (unsigned)p.VB;
    int headg = st.headg, tailg = st.tailg, headb = st.headb, tailb = st.tailb;
    unsigned sb0 = st.sb0, se0 = st.se0, sb1 = st.sb1, se1 = st.se1;
    // End times are kept as the bit patterns of non-negative doubles, which
    // order like the values: integer compares and min.  An idle lane holds +inf.
    constexpr unsigned long long kIdle = 0x7ff0000000000000ull;
    unsigned long long end0 = st.end0, end1 = st.end1;
    double now = __longlong_as_double((long long)st.nowb);  // its bit pattern orders like an end time
    uint32_t level = st.level;
    uint32_t lastg = tailg > headg ? (uint32_t)(rg[(tailg - 1) & mg] >> 32) : 0u;
    uint32_t lastb = tailb > headb ? (uint32_t)(rb[(tailb - 1) & mb] >> 32) : 0u;
    uint32_t it = st.iter;  // REC: the iteration being run, + 1
    uint32_t run0 = 0xffffu, run1 = 0xffffu;  // REC: the running nodes
    auto release = [&](unsigned qb, unsigned qe) -> bool {
        // walk the list by pointer and count: nothing to re-select per entry
        const uint32_t *__restrict__ q = ((qb & 0x8000u) ? csucc : psucc) + (qb & 0x7fffu);
        for (int n = (int)qe - (int)(qb & 0x7fffu); n > 0; n--, q++) {
            const uint32_t e = *q;
            const unsigned t = e & 0xffffu;
            const unsigned d = (unsigned)indeg[t] - 1u;  // bit 15: the node is patched
            indeg[t] = (uint16_t)d;
            if ((d & 0x7fffu) == 0) {
                const unsigned pt = d >> 15;
                // the parent's rank travels in the successor entry; a patched node's is its own
                const uint32_t pr = pt ? inc_patched_rec(dirty, s_pbm, s_ppre, t).prank : (e >> 16);
                const unsigned long long x = inc_ent(level | pr, t, pt);
                if (!(t < VB ? inc_push(rg, mg, headg, tailg, lastg, x) : inc_push(rb, mb, headb, tailb, lastb, x)))
                    return false;
                if constexpr (REC) ro->push[t] = (uint16_t)it;
            }
        }
        return true;
    };
    auto node_rec = [&](unsigned long long x, double &dur, unsigned &sb, unsigned &se) {
        const unsigned t = (unsigned)x & 0xffffu;
        if (x & 0x10000ull) {
            const IncDirty r = inc_patched_rec(dirty, s_pbm, s_ppre, t);
            dur = r.dur;
            sb = r.sb;
            se = r.se;
        } else {  // one 128-bit load: duration, then the successor range (sb | se << 16)
            const uint4 r = __ldg((const uint4 *)(rec + t));
            dur = __hiloint2double((int)r.y, (int)r.x);
            sb = r.z & 0xffffu;
            se = r.z >> 16;
        }
    };
    // start_available (simulator.py:98-115): compute lane, then comm lane;
    // start = max(now, rt) = now because rt is a drained completion time
    auto start = [&]() {
        if ((uint32_t)(end0 >> 32) == (uint32_t)(kIdle >> 32) && headg < tailg) {  // idle: +inf's high word
            double d;
            const unsigned long long x = rg[(headg++) & mg];
            node_rec(x, d, sb0, se0);
            end0 = (unsigned long long)__double_as_longlong(__dadd_rn(now, d));
            if constexpr (REC) run0 = (unsigned)x & 0xffffu;
        }
        if ((uint32_t)(end1 >> 32) == (uint32_t)(kIdle >> 32) && headb < tailb) {
            double d;
            const unsigned long long x = rb[(headb++) & mb];
            node_rec(x, d, sb1, se1);
            end1 = (unsigned long long)__double_as_longlong(__dadd_rn(now, d));
            if constexpr (REC) run1 = (unsigned)x & 0xffffu;
        }
    };
    start();  // from a snapshot: a no-op (the state is taken right after a start)
    for (;;) {
        if constexpr (REC) {
            if (it > 0 && it % ro->S == 0 && (int)(it / ro->S) <= ro->maxsnap) {
                const int j = it / ro->S;
                char *sp = ro->snap + (int64_t)(j - 1) * ro->stride;
                IncLoopState *h = (IncLoopState *)sp;
                *h = IncLoopState{headg, tailg, headb, tailb, sb0,  se0,   sb1, se1,
                                  end0,  end1,  (unsigned long long)__double_as_longlong(now), level, it, run0, run1};
                unsigned long long *eg = (unsigned long long *)(sp + kIncSnapRuns), *eb = eg + kIncRingG;
                for (int i = headg; i < tailg; i++) eg[i - headg] = rg[i & mg];
                for (int i = headb; i < tailb; i++) eb[i - headb] = rb[i & mb];
                const uint32_t *src = (const uint32_t *)indeg;
                uint32_t *dst = (uint32_t *)(sp + kIncSnapDeg);
                for (int i = 0; i < (p.NN + 2) / 2; i++) dst[i] = src[i];
                *ro->nsnap = j;
            }
            it++;
        }
        // drain every lane ending at the next completion time (simulator.py:122-132):
        // c0 / c1 say which lanes end then; an idle lane's +inf never does
        // unless both are idle (+inf's high word: the loop ends)
        const bool c0 = end0 <= end1, c1 = end1 <= end0;
        const unsigned long long t = c0 ? end0 : end1;
        if ((uint32_t)(t >> 32) == (uint32_t)(kIdle >> 32)) break;
        if (t > (unsigned long long)__double_as_longlong(now)) {
            now = __longlong_as_double((long long)t);
            level += 0x10000u;
        }
        if (c0) {
            end0 = kIdle;
            if constexpr (REC) ro->fin[run0] = (uint16_t)it;
            if (!release(sb0, se0)) return false;
        }
        if (c1) {
            end1 = kIdle;
            if constexpr (REC) ro->fin[run1] = (uint16_t)it;
            if (!release(sb1, se1)) return false;
        }
        start();
    }
    if constexpr (REC) *ro->iters = (int)it;
    const int done = headg + headb;
    *cost_out = done == N ? now : 0.0;  // makespan = last completion time (simulator.py:135-139)
    *status_out = done == N ? FO_OK : FO_CYCLE;  // simulator.py:133
    return true;
}

// insert one ready entry into a level-0 run (kept sorted by key)
__device__ __forceinline__ bool inc_ring_insert(unsigned long long *buf, unsigned m, int &tail, unsigned long long x) {
    uint32_t last = tail > 0 ? (uint32_t)(buf[(tail - 1) & m] >> 32) : 0u;
    return inc_push(buf, m, 0, tail, last, x);
}

// Look member sets up in the memo and claim a slot for every new one (its
// prediction is filled in by the estimator kernel), all lanes of the warp at
// once.  A slot another thread is still writing (k1 == 2) is re-read on the
// next round -- lanes never spin on each other.  slot -1: no slot along the
// probe sequence (the set is queued privately).
__device__ __forceinline__ void memo_claim_warp(MemoEnt *t, unsigned mask, bool active, unsigned long long h1,
                                                unsigned long long h2, int &slot, bool &fresh) {
    int probe = 0;
    bool done = !active;
    slot = -1;
    fresh = true;
    while (__any_sync(FULL, !done)) {
        if (!done) {
            const unsigned i = (unsigned)(h1 + probe) & mask;
            MemoEnt *e = &t[i];
            const unsigned long long k = atomicCAS(&e->k1, 0ull, 2ull);
            if (k == 0) {
                e->k2 = h2;
                e->v = __longlong_as_double(0x7ff8000000000000ll);
                __threadfence();
                atomicExch(&e->k1, h1);
                slot = (int)i;
                done = true;
            } else if (k == h1) {
                __threadfence();
                if (*(volatile unsigned long long *)&e->k2 == h2) {
                    slot = (int)i;
                    fresh = false;
                    done = true;
                } else if (++probe >= kMemoProbe) done = true;
            } else if (k != 2 && ++probe >= kMemoProbe) {
                done = true;
            }
        }
        __syncwarp();
    }
}

template <typename T>
__device__ void score_one_inc(const IncArgs &a, int k, const IncCtx &c0, const GroupScratch &gs, int lane) {
    IncCtx c = c0;
    const DGraph &g = a.g;
    const IncPlan &p = a.p;
    const IncLayout &L = a.L;
    const int V = p.V, A = p.A, VB = p.VB;
    auto retry = [&]() {
        if (lane == 0) { a.cost_out[k] = 0.0; a.status_out[k] = a.diag ? 110 + c.cnt[kCFail] : kRetryGeneral; }
    };
    // ---- changes: load, validate, sort by index, changed-index bitmap
    const int cb = a.doff[k], ce = a.doff[k + 1];
    const int nchg = ce - cb;
    if (cb < 0 || nchg < 0 || ce > a.doff[a.K] || nchg > kIncMaxChg) { retry(); return; }
    for (int i = lane; i < L.CW; i += 32) c.cbm[i] = 0;
    for (int i = lane; i < L.NW; i += 32) { c.pbm[i] = 0; c.abm[i] = 0; c.lbm[i] = 0; }
    for (int i = lane; i < L.RW; i += 32) c.rbm[i] = 0;
    if (lane < 8) c.cnt[lane] = 0;
    unsigned long long key0 = ~0ull, key1 = ~0ull;  // (index << 32) | value, two per lane
    bool bad = false;
    auto load = [&](int i) -> unsigned long long {
        if (i >= nchg) return ~0ull;
        const int idx = a.dchg[2 * (cb + i)], val = a.dchg[2 * (cb + i) + 1];
        if (idx < 0 || idx >= 2 * V + A) { bad = true; return ~0ull; }
        if (idx < V ? (val < 0 || val >= VB) : idx < 2 * V ? (val < -1 || val >= VB) : (val < 0 || val >= A)) bad = true;
        return ((unsigned long long)(unsigned)idx << 32) | (unsigned)val;
    };
    key0 = load(lane);
    key1 = load(lane + 32);
    if (__any_sync(FULL, bad)) { retry(); return; }
    // bitonic sort of 64 keys held as (key0 of lanes 0..31, key1 of lanes 0..31)
    for (int kk = 2; kk <= 64; kk <<= 1)
        for (int j = kk >> 1; j > 0; j >>= 1) {
            if (j == 32) {  // partner is the same lane's other key
                const bool up = ((lane & kk) == 0);
                const unsigned long long lo = min(key0, key1), hi = max(key0, key1);
                key0 = up ? lo : hi;
                key1 = up ? hi : lo;
            } else {
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    unsigned long long &x = h ? key1 : key0;
                    const int i = lane + 32 * h;
                    const unsigned long long y = __shfl_xor_sync(FULL, x, j);
                    const bool up = ((i & kk) == 0), lower = (i & j) == 0;
                    const unsigned long long lo = min(x, y), hi = max(x, y);
                    x = (lower == up) ? lo : hi;
                }
            }
        }
    __syncwarp();
    c.nchg = nchg;
    if (lane < nchg) c.chg[lane] = make_int2((int)(key0 >> 32), (int)(unsigned)key0);
    if (lane + 32 < nchg) c.chg[lane + 32] = make_int2((int)(key1 >> 32), (int)(unsigned)key1);
    __syncwarp();
    for (int i = lane; i < nchg; i += 32) {
        const int idx = c.chg[i].x;
        atomicOr(&c.cbm[idx >> 5], 1u << (idx & 31));
        if (i > 0 && c.chg[i - 1].x == idx) bad = true;  // one change per index
    }
    __syncwarp();
    {  // word prefix of the changed-index bitmap (icval's rank)
        int carry = 0;
        for (int base = 0; base < L.CW; base += 32) {
            const int i = base + lane;
            const int x = i < L.CW ? __popc(c.cbm[i]) : 0;
            int v = x;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(FULL, v, d);
                if (lane >= d) v += y;
            }
            if (i < L.CW) c.cpre[i] = (uint8_t)(carry + v - x);
            carry += __shfl_sync(FULL, v, 31);
        }
    }
    __syncwarp();
    // every changed op keeps a normal group distinct from its replica group
    for (int i = lane; i < nchg; i += 32) {
        const int idx = c.chg[i].x;
        if (idx < 2 * V) {
            const int v = idx < V ? idx : idx - V;
            if (inn(c, v) == irr(c, v)) bad = true;
        }
    }
    if (__any_sync(FULL, bad)) { retry(); return; }

    // ---- changed dependency slots (removed from / added to the parent DAG)
    for (int i = lane; i < nchg; i += 32) {
        const int idx = c.chg[i].x;
        if (idx < 2 * V) {
            const int v = idx < V ? idx : idx - V;
            if (idx >= V && ibit(c.cbm, v)) continue;  // the op's ngid change covers it
            for (int q = g.in_ptr[v]; q < g.in_ptr[v + 1]; q++) iedge_slots(c, g.in_e[q]);
            for (int q = g.out_ptr[v]; q < g.out_ptr[v + 1]; q++) {
                const int e = g.out_e[q];
                if (!iop_changed(c, g.e_dst[e])) iedge_slots(c, e);  // else the consumer's in-edges cover it
            }
            for (int q = g.arp_ptr[v]; q < g.arp_ptr[v + 1]; q++) iar_slot(c, g.arp[q]);
        } else {
            const int aa = idx - 2 * V, s = g.ar_prod[aa];
            if (iop_changed(c, s)) continue;  // the producer's slots cover it
            iar_slot(c, aa);
            int j = 0;
            for (int q = g.arp_ptr[s]; q < g.arp_ptr[s + 1]; q++, j++)
                if (g.arp[q] == aa) break;
            for (int q = g.out_ptr[s]; q < g.out_ptr[s + 1]; q++) {
                const int e = g.out_e[q], d = g.e_dst[e];
                if (g.e_agg[e] && !iop_changed(c, d)) {
                    const int pnd = p.pnn[d], prd = p.prr[d];
                    iagg_slots(c, e, j, aa, pnd, prd, pnd, prd);
                }
            }
        }
    }
    // ---- patched nodes: groups / buckets whose membership changed (attribute)
    for (int i = lane; i < nchg; i += 32) {
        const int idx = c.chg[i].x, val = c.chg[i].y;
        if (idx < V) { imark(c, p.pnn[idx], 1); imark(c, val, 1); }
        else if (idx < 2 * V) {
            if (p.prr[idx - V] >= 0) imark(c, p.prr[idx - V], 1);
            if (val >= 0) imark(c, val, 1);
        } else { imark(c, VB + p.pbk[idx - 2 * V], 1); imark(c, VB + val, 1); }
    }
    __syncwarp();
    if (c.cnt[kCFail]) { retry(); return; }
    // members of attribute-patched groups / buckets
    const int n_attr = c.cnt[kCDirty];
    for (int s = lane; s < n_attr; s += 32) {
        const int n = c.dn[s];
        IncWork wk{n, -1, -1, 0, 0, 0, 0};
        if (n < VB) {
            int cnt = 0;
            for (int q = p.mptr[n]; q < p.mptr[n + 1]; q++) {
                const int u = p.mem[q];
                cnt += (inn(c, u) == n || irr(c, u) == n);
            }
            for (int i = 0; i < nchg; i++) {
                const int idx = c.chg[i].x;
                if (idx >= 2 * V) break;
                const int v = idx < V ? idx : idx - V;
                if (idx >= V && ibit(c.cbm, v)) continue;
                if ((inn(c, v) == n || irr(c, v) == n) && p.pnn[v] != n && p.prr[v] != n) cnt++;
            }
            const int mb = atomicAdd(&c.cnt[kCMem], cnt);
            if (mb + cnt > L.mem_cap) { ifail(c, 5); c.work[s] = wk; continue; }
            int o = mb;
            for (int q = p.mptr[n]; q < p.mptr[n + 1]; q++) {
                const int u = p.mem[q];
                if (inn(c, u) == n || irr(c, u) == n) c.mem[o++] = u;
            }
            for (int i = 0; i < nchg; i++) {
                const int idx = c.chg[i].x;
                if (idx >= 2 * V) break;
                const int v = idx < V ? idx : idx - V;
                if (idx >= V && ibit(c.cbm, v)) continue;
                if ((inn(c, v) == n || irr(c, v) == n) && p.pnn[v] != n && p.prr[v] != n) {
                    int j = o++;  // insertion into the ascending run
                    while (j > mb && c.mem[j - 1] > v) { c.mem[j] = c.mem[j - 1]; j--; }
                    c.mem[j] = v;
                }
            }
            wk.cnt = cnt;
            wk.mn = cnt ? c.mem[mb] : -1;
            wk.mb = mb;
            wk.me = mb + cnt;
        } else {
            const int b = n - VB;
            int cnt = 0, mn = INT_MAX;
            long long bytes = 0;
            for (int q = p.bptr[b]; q < p.bptr[b + 1]; q++) {
                const int ar = p.bmem[q];
                if (ibk(c, ar) == b) { cnt++; mn = min(mn, ar); bytes += g.ar_bytes[ar]; }
            }
            for (int i = 0; i < nchg; i++) {
                const int idx = c.chg[i].x;
                if (idx < 2 * V) continue;
                const int ar = idx - 2 * V;
                if (c.chg[i].y == b && p.pbk[ar] != b) { cnt++; mn = min(mn, ar); bytes += g.ar_bytes[ar]; }
            }
            wk.cnt = cnt;
            wk.mn = cnt ? mn : -1;
            wk.bytes = bytes;
        }
        c.work[s] = wk;
    }
    __syncwarp();
    // groups whose tie-break rank depends on a patched group's min member
    // (simulator.py:63: the replica bit of 2 * min + bit), and the sources of
    // every removed / added slot (their successor lists are rebuilt)
    for (int s = lane; s < n_attr; s += 32) {
        const int n = c.dn[s];
        if (n >= VB) continue;
        const int ts[2] = {p.gcnt[n] > 0 ? (int)p.gmin[n] : -1, c.work[s].mn};
        for (int h = 0; h < 2; h++) {
            if (ts[h] < 0) continue;
            const int y0 = inn(c, ts[h]), y1 = irr(c, ts[h]);
            if (y0 >= 0 && y0 != n) imark(c, y0, 0);
            if (y1 >= 0 && y1 != n) imark(c, y1, 0);
        }
    }
    const int nrem = min(c.cnt[kCRem], kIncMaxOps), nadd = min(c.cnt[kCAdd], kIncMaxOps);
    for (int i = lane; i < nrem; i += 32) {
        imark(c, c.rem[i].y, 2);
        atomicOr(&c.rbm[c.rem[i].x >> 5], 1u << (c.rem[i].x & 31));
    }
    for (int i = lane; i < nadd; i += 32) imark(c, c.add[i].x, 2);
    __syncwarp();
    if (c.cnt[kCFail]) { retry(); return; }
    const int nd = c.cnt[kCDirty];
    // rank of a patched node = its position among patched nodes by id
    {
        int carry = 0;
        for (int base = 0; base < L.NW; base += 32) {
            const int i = base + lane;
            const int x = i < L.NW ? __popc(c.pbm[i]) : 0;
            int v = x;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(FULL, v, d);
                if (lane >= d) v += y;
            }
            if (i < L.NW) c.ppre[i] = (uint16_t)(carry + v - x);
            carry += __shfl_sync(FULL, v, 31);
        }
    }
    __syncwarp();
    for (int s = lane; s < nd; s += 32) c.r2s[irank(c, c.dn[s])] = (uint16_t)s;
    __syncwarp();
    // patched records: existence, rank, duration (singletons, buckets), list range
    int exist_delta = 0;
    for (int s = lane; s < nd; s += 32) {
        const int n = c.dn[s];
        const bool attr = s < n_attr;
        const IncNode pr = p.rec[n];
        IncDirty dd{pr.dur, pr.prank, pr.sb, pr.se, pr.exists, 0};
        if (n < VB) {
            const int cnt = attr ? c.work[s].cnt : p.gcnt[n];
            const int mn = attr ? c.work[s].mn : (p.gcnt[n] ? (int)p.gmin[n] : -1);
            dd.exists = cnt > 0;
            if (cnt > 0) {
                const int cn = inn(c, mn), cr = irr(c, mn);
                const int other = cn == n ? cr : cn;
                int gmo = -1;
                if (other >= 0) {
                    const bool oattr = ibit(c.abm, other);
                    gmo = oattr ? c.work[c.r2s[irank(c, other)]].mn : (p.gcnt[other] ? (int)p.gmin[other] : -1);
                }
                dd.prank = (uint16_t)(2 * mn + ((other >= 0 && gmo == mn && other < n) ? 1 : 0));
                if (attr) {
                    if (cnt == 1) {  // estimator.py:810-814
                        if (g.op_kind[mn] == 1) dd.dur = 0.0;
                        else {
                            dd.dur = g.op_prof[mn];
                            if (isnan(dd.dur)) ifail(c, 6);  // MissingCost: the general path reports it
                        }
                    } else {
                        dd.fused = 1;
                        if (cnt > L.mpcap) ifail(c, 7);
                    }
                }
            }
        } else if (attr) {
            const IncWork wk = c.work[s];
            dd.exists = wk.cnt > 0;
            if (wk.cnt > 0) {
                dd.prank = (uint16_t)wk.mn;
                dd.dur = __dadd_rn(__dmul_rn(g.C, (double)wk.bytes), g.D);  // comm.py:45-49
            }
        }
        if (attr) exist_delta += (int)dd.exists - (int)pr.exists;
        c.dirty[irank(c, n)] = dd;
    }
    exist_delta = __reduce_add_sync(FULL, exist_delta);
    __syncwarp();
    if (c.cnt[kCFail]) { retry(); return; }
    // ---- K2 registration.  The MP prediction is a function of the member set
    // alone (estimator.py:167-177: per-op features, member-internal edges), so
    // each patched fused group's set is looked up in the memo; new sets are
    // queued and the estimator kernel runs one warp per queued set.  The
    // record holds the memo slot (>= 0) or -(queue index) - 1 until K3.
    // One lane per fused group: every lookup of the candidate is in flight at once.
    for (int r0 = 0; r0 < nd; r0 += 32) {
        const int r = r0 + lane;
        bool mine = r < nd && c.dirty[r].fused;
        int slot = -1;
        bool fresh = true;
        if (mine) {
            const int ws = c.r2s[r];
            const IncWork wk = c.work[ws];
            const int *mem = c.mem + wk.mb;
            unsigned long long s1 = 0, s2 = 0;
            bool miss = false;
            for (int i = 0; i < wk.cnt; i++) {  // set_hash's two commutative sums, one lane
                const int m = mem[i];
                miss |= isnan(g.op_prof[m]);  // MissingCost (estimator.py:170): the general path reports it
                s1 += smix((unsigned long long)m * 2 + 1);
                s2 += smix(((unsigned long long)m << 32) ^ 0x5bd1e995ull);
            }
            if (miss) ifail(c, 8);
            const unsigned long long h1 = smix(s1 + (unsigned long long)wk.cnt) | 1ull;
            const unsigned long long h2 = smix(s2 ^ ((unsigned long long)wk.cnt * 0xff51afd7ed558ccdull));
            c.work[ws].h1 = h1;
            c.work[ws].h2 = h2;
        }
        if (a.memo) {
            const IncWork &wk = c.work[c.r2s[min(r, nd - 1)]];
            memo_claim_warp(a.memo, g.memo_mask, mine, mine ? wk.h1 : 0ull, mine ? wk.h2 : 0ull, slot, fresh);
        }
        // new sets are queued (one atomic per warp); a memo hit keeps its slot
        const bool q = mine && (fresh || slot < 0);
        const unsigned qm = __ballot_sync(FULL, q);
        const int leader = qm ? __ffs(qm) - 1 : 0;
        int qbase = 0;
        if (qm && lane == leader) qbase = atomicAdd(a.qcount, __popc(qm));
        qbase = __shfl_sync(FULL, qbase, leader);
        if (q) {
            const int qi = qbase + __popc(qm & lanemask_lt());
            if (qi >= a.qcap) ifail(c, 9);
            else {
                const IncWork wk = c.work[c.r2s[r]];
                IncQ e;
                e.mem = c.mem + wk.mb;
                e.slot = slot;
                e.n = wk.cnt;
                e.v = 0.0;
                e.h1 = wk.h1;
                e.h2 = wk.h2;
                e.pad = 0;
                a.queue[qi] = e;
                c.dirty[r].dur = __longlong_as_double(-(long long)qi - 1);
            }
        } else if (mine) {
            c.dirty[r].dur = __longlong_as_double((long long)slot);
        }
    }
    __syncwarp();
    if (c.cnt[kCFail]) { retry(); return; }
    if (a.stop_after == 1) {
        if (lane == 0) { a.cost_out[k] = 0.0; a.status_out[k] = FO_OK; }
        return;
    }
    // ---- rebuilt successor lists of list-patched nodes: the parent's entries
    // that stay, then the node's added slots (in any order: the event loop
    // orders ready entries by key).  Added slots are counted and placed per
    // source rank, one lane per slot.
    uint32_t *acnt = c.acnt;
    for (int r = lane; r < nd; r += 32) acnt[r] = 0;
    __syncwarp();
    for (int i = lane; i < nadd; i += 32) atomicAdd(&acnt[irank(c, c.add[i].x)], 1u);
    __syncwarp();
    for (int s = lane; s < nd; s += 32) {
        const int n = c.dn[s];
        if (!ibit(c.lbm, n)) continue;
        const int r = irank(c, n);
        const IncNode pr = p.rec[n];
        int keep = 0;
        for (int q = pr.sb; q < pr.se; q++) keep += !ibit(c.rbm, q);
        const int cnt = keep + (int)acnt[r];
        const int o0 = atomicAdd(&c.cnt[kCPcsr], cnt);
        if (o0 + cnt > L.pcsr_cap) { ifail(c, 10); continue; }
        int o = o0;
        for (int q = pr.sb; q < pr.se; q++)
            if (!ibit(c.rbm, q)) c.pcsr[o++] = p.succ[q];
        acnt[r] = (uint32_t)o;  // where the added slots go
        IncDirty &dd = c.dirty[r];
        dd.sb = (uint16_t)(0x8000 | o0);
        dd.se = (uint16_t)(o0 + cnt);
    }
    __syncwarp();
    if (c.cnt[kCFail]) { retry(); return; }
    for (int i = lane; i < nadd; i += 32) {
        const int4 ad = c.add[i];
        if (!ibit(c.lbm, ad.x)) { ifail(c, 10); continue; }
        // the parent's rank (patched targets are re-ranked at release)
        c.pcsr[atomicAdd(&acnt[irank(c, ad.x)], 1u)] = ((uint32_t)ad.z << 16) | (uint32_t)ad.y;
    }
    __syncwarp();
    if (c.cnt[kCFail]) { retry(); return; }
    // hand-off to the event-loop kernel: counts in the header, lists in the scratch
    if (lane == 0) {
        c.hdr[0] = nd;
        c.hdr[1] = nrem;
        c.hdr[2] = nadd;
        c.hdr[3] = p.n_exist + exist_delta;
        a.status_out[k] = kIncPending;
    }
}

__device__ __forceinline__ IncCtx inc_ctx(const IncArgs &a, int wid, char *sm) {
    const IncLayout &L = a.L;
    char *wsb = a.ws + (int64_t)wid * L.total;
    IncCtx c;
    c.a = &a;
    c.hdr = (int *)(wsb + L.hdr);
    c.chg = (int2 *)(sm + L.s_chg);
    c.rem = (int4 *)(wsb + L.rem);
    c.add = (int4 *)(wsb + L.add);
    c.dn = (int *)(wsb + L.dn);
    c.work = (IncWork *)(wsb + L.work);
    c.dirty = (IncDirty *)(wsb + L.dirty);
    c.r2s = (uint16_t *)(c.dirty + kIncMaxDirty + 1);
    c.mem = (int *)(wsb + L.mem);
    c.pcsr = (uint32_t *)(wsb + L.pcsr);
    c.ring = (Ent16 *)(wsb + L.ring);
    c.indeg = L.s_indeg >= 0 ? (uint16_t *)(sm + L.s_indeg) : (uint16_t *)(wsb + L.indeg);
    c.pbm = (uint32_t *)(sm + L.s_pbm);
    c.abm = (uint32_t *)(sm + L.s_abm);
    c.lbm = (uint32_t *)(sm + L.s_lbm);
    c.tbm = nullptr;
    c.rbm = (uint32_t *)(sm + L.s_rbm);
    c.cpre = (uint8_t *)(sm + L.s_cpre);
    c.ppre = (uint16_t *)(sm + L.s_ppre);
    c.cbm = (uint32_t *)(sm + L.s_cbm);
    c.acnt = (uint32_t *)(sm + L.s_acnt);
    c.cnt = (int *)(sm + L.s_cnt);
    c.nchg = 0;
    return c;
}

// Setup + K2 of candidates [k0, k0 + warps): one warp each.
template <typename T>
__global__ void __launch_bounds__(kWarps * 32, 9) score_kernel_inc(const __grid_constant__ IncArgs a, int k0) {
    const int lane = threadIdx.x & 31;
    const int wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int k = k0 + wid;
    if (k >= a.K) return;
    const IncLayout &L = a.L;
    const IncCtx c = inc_ctx(a, wid, fo_inc_smem + (threadIdx.x >> 5) * L.s_bytes);
    char *gb = a.ws + (int64_t)wid * L.total + L.gs0;
    const GroupScratch gs{(int *)(gb + L.g_msort), (int *)(gb + L.g_lidx), (int *)(gb + L.g_zl),
                          (int *)(gb + L.g_nbptr), (int *)(gb + L.g_nb), (int *)(gb + L.g_mark),
                          gb + L.g_H, gb + L.g_P};
    score_one_inc<T>(a, k, c, gs, lane);
}

// K2: the estimator over the queued member sets, one warp per set.  The
// member-local undirected neighbour lists (in-edges, then out-edges, the
// general kernel's order; estimator.py:173-177, :348-355) come from a binary
// search in the ascending member list, then mp_forward (estimator.py:363-389).
template <typename T>
__global__ void __launch_bounds__(kWarps * 32, 7) score_kernel_inc_mp(const __grid_constant__ IncArgs a) {
    const int lane = threadIdx.x & 31;
    const int wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int nw = gridDim.x * kWarps;
    const DGraph &g = a.g;
    const IncLayout &L = a.L;
    char *gb = a.ws + (int64_t)wid * L.total + L.gs0;
    const GroupScratch gs{(int *)(gb + L.g_msort), (int *)(gb + L.g_lidx), (int *)(gb + L.g_zl),
                          (int *)(gb + L.g_nbptr), (int *)(gb + L.g_nb), (int *)(gb + L.g_mark),
                          gb + L.g_H, gb + L.g_P};
    const int nq = min(*a.qcount, a.qcap);
    for (int qi = wid; qi < nq; qi += nw) {
        const IncQ q = a.queue[qi];
        const int *mem = q.mem;
        const int n = q.n;
        if (n < 2 || n > L.mpcap || (const char *)mem < a.ws || (const char *)mem >= a.ws + (int64_t)nw * L.total) {
            if (lane == 0) a.queue[qi].v = __longlong_as_double(0x7ff8000000000000ll);  // K3 hands it back
            continue;
        }
        for (int i = lane; i < n; i += 32) {
            const int v = mem[i];
            gs.zl[i] = (g.in_ptr[v + 1] - g.in_ptr[v]) + (g.out_ptr[v + 1] - g.out_ptr[v]);
        }
        __syncwarp();
        warp_exscan(gs.zl, gs.nbptr, n, lane);
        // local index of an op among the (ascending) members, -1 outside the set
        auto local = [&](int op) {
            int lo = 0, hi = n - 1;
            while (lo < hi) {
                const int m = (lo + hi) >> 1;
                if (mem[m] < op) lo = m + 1;
                else hi = m;
            }
            return mem[lo] == op ? lo : -1;
        };
        for (int i = lane; i < n; i += 32) {
            const int v = mem[i];
            const int o = gs.nbptr[i];
            int cc = 0;
            for (int e = g.in_ptr[v]; e < g.in_ptr[v + 1]; e++) {
                const int j = local(g.e_src[g.in_e[e]]);
                if (j < 0) continue;
                bool dup = false;
                for (int t = 0; t < cc; t++) dup |= (gs.nb[o + t] == j);
                if (!dup) gs.nb[o + cc++] = j;
            }
            for (int e = g.out_ptr[v]; e < g.out_ptr[v + 1]; e++) {
                const int j = local(g.e_dst[g.out_e[e]]);
                if (j < 0) continue;
                bool dup = false;
                for (int t = 0; t < cc; t++) dup |= (gs.nb[o + t] == j);
                if (!dup) gs.nb[o + cc++] = j;
            }
            gs.msort[i] = cc;
        }
        __syncwarp();
        if (lane == 0) {  // compact rows into a dense CSR
            int o = 0;
            for (int i = 0; i < n; i++) {
                const int s0 = gs.nbptr[i], cc = gs.msort[i];
                for (int t = 0; t < cc; t++) gs.nb[o + t] = gs.nb[s0 + t];
                gs.nbptr[i] = o;
                o += cc;
            }
            gs.nbptr[n] = o;
        }
        __syncwarp();
        // node states H and aggregates P of sets up to kIncMpSmem members in the
        // warp's shared memory, larger sets in its global scratch
        T *sh = (T *)(fo_inc_smem + (threadIdx.x >> 5) * (2 * kIncMpSmem<T> * 32 * sizeof(T)));
        const bool in_smem = n <= kIncMpSmem<T>;
        const double pred = mp_forward<T>(g, mem, n, gs.nbptr, gs.nb, in_smem ? sh : (T *)gs.H,
                                          in_smem ? sh + kIncMpSmem<T> * 32 : (T *)gs.P, lane);
        if (lane == 0) {
            a.queue[qi].v = pred;  // the queuing candidate reads this
            if (q.slot >= 0 && a.memo[q.slot].k1 == q.h1 && a.memo[q.slot].k2 == q.h2)
                a.memo[q.slot].v = pred;  // later hits read the memo
        }
        __syncwarp();
    }
}

// K3 of the same candidates, in two phases.  Prep (the whole warp, one
// candidate after the other): the candidate's indegrees (the parent's, minus
// removed, plus added slots), the patched-node ranks and the ready runs in
// the candidate's shared-memory region, from level 0 or a parent snapshot.
// Run (one lane per candidate, all of the warp's candidates at once): the
// event loop.  The loops of different candidates of one parent take the same
// branches most of the time, so a warp instruction advances many of them.
struct IncK3State {
    IncLoopState st;
    int32_t k, wid, N, mode;  // mode 0: nothing to run, 1: from level 0, 2: from a snapshot
};

template <bool SI>
__device__ __forceinline__ void inc_k3_prep(const IncArgs &a, int k0, int wid, int n, int lane, uint32_t wsm) {
    const IncLayout &L = a.L;
    IncK3State *ks = (IncK3State *)(fo_inc_smem + wsm + L.k_state);
    if (lane == 0) ks->mode = 0;
    const int k = k0 + wid;
    if (wid >= n || k >= a.K || a.status_out[k] != kIncPending) return;
    const IncPlan &p = a.p;
    char *wsb = a.ws + (int64_t)wid * L.total;
    const int *hdr = (const int *)(wsb + L.hdr);
    const int nd = hdr[0], nrem = hdr[1], nadd = hdr[2], N = hdr[3];
    const int *dn = (const int *)(wsb + L.dn);
    const int4 *rem = (const int4 *)(wsb + L.rem);
    const int4 *add = (const int4 *)(wsb + L.add);
    const IncDirty *dirty = (const IncDirty *)(wsb + L.dirty);
    uint16_t *indeg = SI ? (uint16_t *)(fo_inc_smem + wsm + L.k_indeg) : (uint16_t *)(wsb + L.indeg);
    uint32_t *pbm = (uint32_t *)(fo_inc_smem + wsm + L.k_pbm);
    uint16_t *ppre = (uint16_t *)(fo_inc_smem + wsm + L.k_ppre);
    uint32_t *tbm = (uint32_t *)(fo_inc_smem + wsm + L.k_tbm);
    unsigned long long *rg = (unsigned long long *)(fo_inc_smem + wsm + L.k_ring), *rb = rg + kIncRingG;
    const int NN = p.NN;
    if (a.stop_after == 2) {  // phase timing only (fo_set_phase_stop)
        if (lane == 0) { a.cost_out[k] = 0.0; a.status_out[k] = FO_OK; }
        return;
    }
    // durations of patched fused groups, computed by the estimator kernel: a
    // queued set reads its queue entry, a memo hit its slot -- checked against
    // the set's key (a memo clear racing on another stream hands the
    // candidate to the general kernel instead of reading a foreign value)
    bool stale = false;
    const IncWork *work = (const IncWork *)(wsb + L.work);
    const uint16_t *r2s = (const uint16_t *)(dirty + kIncMaxDirty + 1);
    for (int r = lane; r < nd; r += 32) {
        IncDirty &dd = ((IncDirty *)dirty)[r];
        if (!dd.fused) continue;
        const long long ref = __double_as_longlong(dd.dur);
        if (ref < 0) {
            dd.dur = a.queue[-ref - 1].v;
            stale |= isnan(dd.dur);
        } else {
            const MemoEnt *e = &a.memo[ref];
            const IncWork &wk = work[r2s[r]];
            const double v = e->v;
            stale |= e->k1 != wk.h1 || e->k2 != wk.h2 || isnan(v);
            dd.dur = v;
        }
    }
    if (__any_sync(FULL, stale)) {
        if (lane == 0) { a.cost_out[k] = 0.0; a.status_out[k] = a.diag ? 103 : kRetryGeneral; }
        return;
    }
    for (int i = lane; i < L.NW; i += 32) { pbm[i] = 0; tbm[i] = 0; }
    __syncwarp();
    for (int s = lane; s < nd; s += 32) {
        const int n = dn[s];
        atomicOr(&pbm[n >> 5], 1u << (n & 31));
    }
    __syncwarp();
    {
        int carry = 0;
        for (int base = 0; base < L.NW; base += 32) {
            const int i = base + lane;
            const int x = i < L.NW ? __popc(pbm[i]) : 0;
            int v = x;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(FULL, v, d);
                if (lane >= d) v += y;
            }
            if (i < L.NW) ppre[i] = (uint16_t)(carry + v - x);
            carry += __shfl_sync(FULL, v, 31);
        }
    }
    // Fast-forward: the candidate's loop equals the parent's up to the first
    // iteration in which the parent makes a touched node ready (a patched node
    // with a new record, or the target of a removed / added slot) -- before
    // it, every started node and every indegree decrement is the parent's.
    // Start from the parent's latest snapshot at or before that iteration,
    // unless the candidate would have made a touched node ready earlier (a
    // target that lost its remaining predecessors: indegree 0 at the
    // snapshot), checked below.
    int j = 0;
    if (p.nsnap > 0) {
        unsigned c = 0xffffu;
        for (int s = lane; s < nd; s += 32) {
            // A patched node whose record (existence, rank, duration) is the
            // parent's differs only in its successor list, i.e. in the slots
            // removed / added at its finish: their targets bound the cut, and
            // a slot whose source finished before the snapshot is left out of
            // the indegrees.  Any other patched node: when it becomes ready.
            const int n = dn[s];
            const IncDirty dd = dirty[(int)ppre[n >> 5] + __popc(pbm[n >> 5] & ((1u << (n & 31)) - 1u))];
            const IncNode pr = p.rec[n];
            const bool same = dd.exists == pr.exists &&
                              (!dd.exists || (dd.prank == pr.prank && __double_as_longlong(dd.dur) ==
                                                                          __double_as_longlong(pr.dur)));
            if (!same) c = min(c, (unsigned)__ldg(&p.push[n]));
        }
        for (int i = lane; i < nrem; i += 32) c = min(c, (unsigned)__ldg(&p.push[rem[i].z]));
        for (int i = lane; i < nadd; i += 32) c = min(c, (unsigned)__ldg(&p.push[add[i].y]));
        c = __reduce_min_sync(FULL, c);
        j = c == 0 ? 0 : min((int)(c - 1) / p.snap_S, p.nsnap);
    }
    const char *sp = j ? p.snap + (int64_t)(j - 1) * p.snap_stride : nullptr;
    // the candidate's indegrees: the parent's (at level 0 or at the snapshot),
    // minus removed, plus added slots; bit 15 marks patched nodes
    // (a slot counts while its source has not finished: at level 0 every
    // slot; at the snapshot of iteration si, those whose source finishes in
    // the parent at iteration si or later -- sources of changed slots start
    // and end as in the parent up to the cut)
    auto build_indeg = [&](const uint16_t *base, int si) {
        {
            const uint32_t *src = (const uint32_t *)base;
            uint32_t *dst = (uint32_t *)indeg;
            for (int i = lane; i < (NN + 1) / 2; i += 32) dst[i] = __ldg(&src[i]);
        }
        __syncwarp();
        for (int i = lane; i < nrem; i += 32) {
            const int4 r = rem[i];
            if (si && (int)__ldg(&p.fin[r.y]) <= si) continue;
            atomicAdd((unsigned *)indeg + (r.z >> 1), (r.z & 1) ? 0xffff0000u : 0xffffffffu);
        }
        for (int i = lane; i < nadd; i += 32) {
            const int4 r = add[i];
            if (si && (int)__ldg(&p.fin[r.x]) <= si) continue;
            atomicAdd((unsigned *)indeg + (r.y >> 1), (r.y & 1) ? 0x10000u : 1u);
        }
        __syncwarp();
        for (int s = lane; s < nd; s += 32) {  // bit 15 of a patched node's indegree (read by the event loop)
            const int n = dn[s];
            atomicOr((unsigned *)indeg + (n >> 1), (n & 1) ? 0x80000000u : 0x8000u);
        }
        __syncwarp();
    };
    for (int i = lane; i < nrem; i += 32) atomicOr(&tbm[rem[i].z >> 5], 1u << (rem[i].z & 31));
    for (int i = lane; i < nadd; i += 32) atomicOr(&tbm[add[i].y >> 5], 1u << (add[i].y & 31));
    __syncwarp();
    for (int i = lane; i < L.NW; i += 32) tbm[i] |= pbm[i];
    __syncwarp();
    auto exists_c = [&](int n) -> bool {  // the node exists in the candidate
        if ((pbm[n >> 5] >> (n & 31)) & 1u)
            return dirty[(int)ppre[n >> 5] + __popc(pbm[n >> 5] & ((1u << (n & 31)) - 1u))].exists;
        return p.rec[n].exists;
    };
    build_indeg(j ? (const uint16_t *)(sp + kIncSnapDeg) : p.indeg, j * p.snap_S);
    if (j) {
        bool early = false;
        for (int wi = lane; wi < L.NW; wi += 32) {
            uint32_t m = tbm[wi];
            while (m) {
                const int n = wi * 32 + __ffs(m) - 1;
                m &= m - 1;
                // ready in the candidate but not yet in the parent at the snapshot
                early |= n < NN && (indeg[n] & 0x7fff) == 0 && exists_c(n) && (int)__ldg(&p.push[n]) > j * p.snap_S;
            }
        }
        if (__any_sync(FULL, early)) {  // the candidate diverges before the snapshot
            j = 0;
            build_indeg(p.indeg, 0);
        }
    }
    if (a.stats && lane == 0) {
        atomicAdd(&a.stats[0], 1ull);
        atomicAdd(&a.stats[1], j ? 1ull : 0ull);
        atomicAdd(&a.stats[2], j ? (unsigned long long)((const IncLoopState *)sp)->iter : 0ull);
    }
    IncLoopState st{};
    constexpr unsigned long long kIdle = 0x7ff0000000000000ull;
    st.end0 = kIdle;
    st.end1 = kIdle;
    bool over = false;
    if (j) {
        st = *(const IncLoopState *)sp;
        // ready nodes the snapshot holds may have rebuilt successor lists
        // (patched, same record): their entries read the candidate's
        const unsigned long long *eg = (const unsigned long long *)(sp + kIncSnapRuns), *eb = eg + kIncRingG;
        auto fix = [&](unsigned long long x) {
            const unsigned n = (unsigned)x & 0xffffu;
            return ((pbm[n >> 5] >> (n & 31)) & 1u) ? x | 0x10000ull : x;
        };
        for (int i = lane; i < st.tailg - st.headg; i += 32) rg[(st.headg + i) & (kIncRingG - 1)] = fix(eg[i]);
        for (int i = lane; i < st.tailb - st.headb; i += 32) rb[(st.headb + i) & (kIncRingB - 1)] = fix(eb[i]);
    } else {
        // level-0 ready runs: the parent's (sorted by rank) without touched
        // nodes; the touched nodes that are ready are inserted by the run phase
        int hgb[2] = {0, 0};
        for (int lanei = 0; lanei < 2; lanei++) {
            const uint16_t *src = p.ready + (lanei ? p.n_ready_g : 0);
            const int n0 = lanei ? p.n_ready_b : p.n_ready_g;
            unsigned long long *buf = lanei ? rb : rg;
            const int cap = lanei ? kIncRingB : kIncRingG;
            int h = 0;
            for (int base = 0; base < n0; base += 32) {
                const int i = base + lane;
                const int n = i < n0 ? src[i] : 0;
                const bool keep = i < n0 && !((tbm[n >> 5] >> (n & 31)) & 1u);
                const unsigned m = __ballot_sync(FULL, keep);
                const int pos = h + __popc(m & lanemask_lt());
                if (keep && pos < cap) buf[pos] = inc_ent(p.rec[n].prank, n, 0);
                h += __popc(m);
            }
            hgb[lanei] = h;
            over |= h > cap;
        }
        st.tailg = hgb[0];
        st.tailb = hgb[1];
    }
    __syncwarp();
    if (lane != 0) return;
    if (over) {
        a.cost_out[k] = 0.0;
        a.status_out[k] = a.diag ? 104 : kRetryGeneral;  // a ready run outgrew its ring: the general kernel scores it
        return;
    }
    ks->st = st;
    ks->k = k;
    ks->wid = wid;
    ks->N = N;
    ks->mode = j ? 2 : 1;
}

// the run phase of one candidate (one lane)
template <bool SI>
__device__ __forceinline__ void inc_k3_run(const IncArgs &a, uint32_t wsm) {
    const IncLayout &L = a.L;
    const IncK3State *ks = (const IncK3State *)(fo_inc_smem + wsm + L.k_state);
    const int mode = ks->mode;
    if (mode == 0) return;
    const IncPlan &p = a.p;
    const int k = ks->k, N = ks->N, NN = p.NN, VB = p.VB;
    IncLoopState st = ks->st;
    char *wsb = a.ws + (int64_t)ks->wid * L.total;
    const IncDirty *dirty = (const IncDirty *)(wsb + L.dirty);
    const uint32_t *pcsr = (const uint32_t *)(wsb + L.pcsr);
    uint16_t *indeg = SI ? (uint16_t *)(fo_inc_smem + wsm + L.k_indeg) : (uint16_t *)(wsb + L.indeg);
    const uint32_t *pbm = (const uint32_t *)(fo_inc_smem + wsm + L.k_pbm);
    const uint16_t *ppre = (const uint16_t *)(fo_inc_smem + wsm + L.k_ppre);
    const uint32_t *tbm = (const uint32_t *)(fo_inc_smem + wsm + L.k_tbm);
    unsigned long long *rg = (unsigned long long *)(fo_inc_smem + wsm + L.k_ring), *rb = rg + kIncRingG;
    constexpr unsigned long long kIdle = 0x7ff0000000000000ull;
    bool over = false;
    if (mode == 2) {
        // the running nodes of the snapshot may have rebuilt successor lists
        auto fix_run = [&](uint32_t n, uint32_t &sb, uint32_t &se) {
            if (n < (uint32_t)NN && ((pbm[n >> 5] >> (n & 31)) & 1u)) {
                const IncDirty dd = dirty[(int)ppre[n >> 5] + __popc(pbm[n >> 5] & ((1u << (n & 31)) - 1u))];
                sb = dd.sb;
                se = dd.se;
            }
        };
        if (st.end0 != kIdle) fix_run(st.run0, st.sb0, st.se0);
        if (st.end1 != kIdle) fix_run(st.run1, st.sb1, st.se1);
    } else {
        // the touched nodes that are ready at level 0, inserted in rank order
        for (int wi = 0; wi < L.NW && !over; wi++) {
            uint32_t m = tbm[wi];
            while (m && !over) {
                const int n = wi * 32 + __ffs(m) - 1;
                m &= m - 1;
                if (n >= NN || (indeg[n] & 0x7fff) != 0) continue;
                unsigned long long x;
                if ((pbm[n >> 5] >> (n & 31)) & 1u) {
                    const IncDirty dd = dirty[(int)ppre[n >> 5] + __popc(pbm[n >> 5] & ((1u << (n & 31)) - 1u))];
                    if (!dd.exists) continue;
                    x = inc_ent(dd.prank, n, 1);
                } else {
                    const IncNode r = p.rec[n];
                    if (!r.exists) continue;
                    x = inc_ent(r.prank, n, 0);
                }
                over = !(n < VB ? inc_ring_insert(rg, kIncRingG - 1, st.tailg, x)
                                : inc_ring_insert(rb, kIncRingB - 1, st.tailb, x));
            }
        }
    }
    if (over || !inc_ring_loop<SI>(p, pcsr, dirty, SI ? nullptr : indeg, wsm + L.k_indeg, wsm + L.k_pbm,
                                   wsm + L.k_ppre, wsm + L.k_ring, st, N, a.cost_out + k, a.status_out + k)) {
        a.cost_out[k] = 0.0;
        a.status_out[k] = a.diag ? 104 : kRetryGeneral;  // a ready run outgrew its ring: the general kernel scores it
    }
}

// K3 over the candidates [k0, k0 + n): one warp each (prep), then its lane 0
// (run).  One lane per candidate with several candidates per warp, so that
// their loops share instructions, measured 2.5x slower at 16 per warp: the
// loops diverge within a few events and the warp serialises them.
template <bool SI>
__global__ void __launch_bounds__(kWarps * 32, 10) score_kernel_inc_k3(const __grid_constant__ IncArgs a, int k0, int n) {
    const int lane = threadIdx.x & 31;
    const int wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const uint32_t wsm = (uint32_t)((threadIdx.x >> 5) * a.L.k_bytes);
    inc_k3_prep<SI>(a, k0, wid, n, lane, wsm);
    __syncwarp();
    if (lane == 0) inc_k3_run<SI>(a, wsm);
}

// The parent's own event loop, once per plan (one warp; lane 0 runs it):
// every node's push iteration and a snapshot of the loop state every S
// iterations, which candidates fast-forward to (score_kernel_inc_k3).
__global__ void inc_record_kernel(const __grid_constant__ IncPlan p, IncRecOut ro, int32_t *out) {
    const int lane = threadIdx.x;
    const int NN = p.NN, NW = (NN + 31) / 32;
    const uint32_t s_indeg = 0, s_pbm = (uint32_t)((2 * (NN + 2) + 15) & ~15), s_ppre = s_pbm + 4 * NW,
                   s_ring = (s_ppre + 2 * NW + 2 + 15) & ~15u;
    uint16_t *indeg = (uint16_t *)fo_inc_smem;
    uint32_t *pbm = (uint32_t *)(fo_inc_smem + s_pbm);
    for (int i = lane; i < (NN + 2) / 2; i += 32) ((uint32_t *)indeg)[i] = ((const uint32_t *)p.indeg)[i];
    for (int i = lane; i < NW; i += 32) pbm[i] = 0;
    for (int i = lane; i < NN; i += 32) ro.push[i] = ro.fin[i] = 0xffffu;
    __syncwarp();
    if (lane != 0) return;
    unsigned long long *rg = (unsigned long long *)(fo_inc_smem + s_ring), *rb = rg + kIncRingG;
    if (p.n_ready_g > kIncRingG || p.n_ready_b > kIncRingB || p.n_exist >= 65000) { out[1] = 1; return; }
    for (int i = 0; i < p.n_ready_g; i++) {
        const int n = p.ready[i];
        rg[i] = inc_ent(p.rec[n].prank, n, 0);
        ro.push[n] = 0;
    }
    for (int i = 0; i < p.n_ready_b; i++) {
        const int n = p.ready[p.n_ready_g + i];
        rb[i] = inc_ent(p.rec[n].prank, n, 0);
        ro.push[n] = 0;
    }
    IncLoopState st{};
    st.tailg = p.n_ready_g;
    st.tailb = p.n_ready_b;
    st.end0 = st.end1 = 0x7ff0000000000000ull;
    ro.nsnap = out;
    *out = 0;
    double *mk = (double *)(out + 2);
    const bool ok = inc_ring_loop<true, true>(p, nullptr, nullptr, nullptr, s_indeg, s_pbm, s_ppre, s_ring, st,
                                               p.n_exist, mk, out + 1, &ro);
    if (!ok) out[1] = 2;
}

cudaError_t launch_inc_record(const IncPlan &p, uint16_t *push, uint16_t *fin, char *snap, int S, int maxsnap,
                              void *out, cudaStream_t stream) {
    const int NN = p.NN, NW = (NN + 31) / 32;
    const size_t s_pbm = (2 * (NN + 2) + 15) & ~15, s_ring = (s_pbm + 6 * NW + 2 + 15) & ~(size_t)15;
    const size_t smem = s_ring + 8 * (kIncRingG + kIncRingB);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(inc_record_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    IncRecOut ro{push, fin, snap, S, maxsnap, inc_snap_stride(NN), nullptr, (int32_t *)out + 4};
    inc_record_kernel<<<1, 32, smem, stream>>>(p, ro, (int32_t *)out);
    return cudaGetLastError();
}

template <typename KF>
static int inc_occ(KF kf, int smem_per_block) {
    int n = 0;
    if (smem_per_block > 48 * 1024) cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_per_block);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kf, kWarps * 32, smem_per_block);
    return n;
}
template <typename T>
static int inc_blocks_per_sm_q(int setup_smem, int k3_smem) {
    return std::min({inc_occ(score_kernel_inc<T>, setup_smem), inc_occ(score_kernel_inc_k3<true>, k3_smem),
                     inc_occ(score_kernel_inc_k3<false>, k3_smem)});
}

int score_inc_blocks_per_sm(const IncLayout &L, int precision) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    const std::pair<int, int> key(L.s_bytes * 65536 + L.k_bytes, precision);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    const int n = precision == FO_PREC_FP64 ? inc_blocks_per_sm_q<double>(L.s_bytes * kWarps, L.k_bytes * kWarps)
                                            : inc_blocks_per_sm_q<float>(L.s_bytes * kWarps, L.k_bytes * kWarps);
    cache[key] = n;
    return n;
}

cudaError_t launch_score_inc(const DGraph &g, const IncPlan &p, const IncLayout &L, const int32_t *off,
                             const int32_t *chg, int K, int precision, char *ws, int grid, IncQ *queue, int *qcount,
                             int qcap, double *cost_out, int32_t *status_out, cudaStream_t stream, int diag) {
    IncArgs a;
    a.diag = diag;
    a.stats = diag ? (unsigned long long *)((char *)qcount + 16) : nullptr;
    a.g = g;
    a.p = p;
    a.L = L;
    a.doff = off;
    a.dchg = chg;
    a.queue = queue;
    a.qcount = qcount;
    a.qcap = qcap;
    a.memo = g.memo[precision == FO_PREC_FP64 ? 1 : 0];
    a.K = K;
    a.ws = ws;
    a.cost_out = cost_out;
    a.status_out = status_out;
    a.stop_after = g.phase_stop;
    const size_t smem = (size_t)L.s_bytes * kWarps;
    const int per_launch = grid * kWarps;  // one candidate per warp per launch
    const bool fp64 = precision == FO_PREC_FP64;
    const size_t ksmem = (size_t)L.k_bytes * kWarps;
    for (int k0 = 0; k0 < K; k0 += per_launch) {
        cudaError_t e = cudaMemsetAsync(qcount, 0, sizeof(int), stream);
        if (e != cudaSuccess) return e;
        const int n = std::min(per_launch, K - k0);
        if (fp64) score_kernel_inc<double><<<grid, kWarps * 32, smem, stream>>>(a, k0);
        else score_kernel_inc<float><<<grid, kWarps * 32, smem, stream>>>(a, k0);
        if (a.stop_after == 1) continue;
        if (fp64) score_kernel_inc_mp<double><<<grid, kWarps * 32, kWarps * 2 * kIncMpSmem<double> * 32 * 8, stream>>>(a);
        else score_kernel_inc_mp<float><<<grid, kWarps * 32, kWarps * 2 * kIncMpSmem<float> * 32 * 4, stream>>>(a);
        if (L.k_indeg >= 0) score_kernel_inc_k3<true><<<grid, kWarps * 32, ksmem, stream>>>(a, k0, n);
        else score_kernel_inc_k3<false><<<grid, kWarps * 32, ksmem, stream>>>(a, k0, n);
    }
    return cudaGetLastError();
}
