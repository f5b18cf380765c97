// engine.cpp -- native batch-expand and the lock-stepped backtracking search.
//
// * CPython random.Random restated (MT19937 + init_by_array + _randbelow),
//   because every draw of the reference's search and rewrites goes through it
//   (search.py:88, :119; rewrite.py:250).
// * The three rewrites with the reference's choice enumeration order, id
//   assignment and validity rule (rewrite.py:49-263, graph.py:505-512).
// * Alg. 1 (search.py:84-155) for R independent seeds advanced in lock step:
//   each round expands every active seed on host threads and scores all of
//   their candidates in ONE device batch (score.cu), then replays the
//   reference's accept/prune bookkeeping in method order.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "fo_internal.h"

namespace fo {

// ---------------------------------------------------------------------------
// CPython random.Random

struct PyRng {
    uint32_t mt[624];
    int mti = 625;

    void init_genrand(uint32_t s) {
        mt[0] = s;
        for (int i = 1; i < 624; i++) mt[i] = 1812433253u * (mt[i - 1] ^ (mt[i - 1] >> 30)) + (uint32_t)i;
        mti = 624;
    }
    // random_seed(int) -> init_by_array over the 32-bit words of |seed|
    explicit PyRng(uint64_t seed) {
        uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
        int klen = (seed >> 32) ? 2 : 1;
        init_genrand(19650218u);
        int i = 1, j = 0;
        for (int k = std::max(624, klen); k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
            if (++i >= 624) { mt[0] = mt[623]; i = 1; }
            if (++j >= klen) j = 0;
        }
        for (int k = 623; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
            if (++i >= 624) { mt[0] = mt[623]; i = 1; }
        }
        mt[0] = 0x80000000u;
    }
    uint32_t next() {
        if (mti >= 624) {
            static const uint32_t mag[2] = {0u, 0x9908b0dfu};
            int k = 0;
            uint32_t y;
            for (; k < 624 - 397; k++) {
                y = (mt[k] & 0x80000000u) | (mt[k + 1] & 0x7fffffffu);
                mt[k] = mt[k + 397] ^ (y >> 1) ^ mag[y & 1u];
            }
            for (; k < 623; k++) {
                y = (mt[k] & 0x80000000u) | (mt[k + 1] & 0x7fffffffu);
                mt[k] = mt[k - 227] ^ (y >> 1) ^ mag[y & 1u];
            }
            y = (mt[623] & 0x80000000u) | (mt[0] & 0x7fffffffu);
            mt[623] = mt[396] ^ (y >> 1) ^ mag[y & 1u];
            mti = 0;
        }
        uint32_t y = mt[mti++];
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        return y;
    }
    // _randbelow_with_getrandbits(n), n >= 1
    uint32_t below(uint32_t n) {
        int k = 32 - __builtin_clz(n);
        uint32_t r = next() >> (32 - k);
        while (r >= n) r = next() >> (32 - k);
        return r;
    }
};

// ---------------------------------------------------------------------------
// fusion state + derived index (graph.py:117-274)

struct State {
    std::vector<int32_t> ng, rg, bk;
};

enum { M_NONDUP = 0, M_DUP = 1, M_AR = 2 };

struct Engine;

struct Index {
    int G = 0, B = 0;
    std::vector<int32_t> gid, bid;      // sorted ids of groups / buckets
    std::vector<int32_t> nn, rr, bki;   // per op / per AR: node index
    std::vector<int32_t> mptr, mem;     // members per group (ascending op), all memberships
    std::vector<uint8_t> mdup, compute_ok, has_dup, feeds_ar, has_rep;
    std::vector<int32_t> sptr, succ, pptr, pred;  // contracted adjacency, sorted unique
    std::vector<int32_t> bptr, bex;               // per bucket: export groups of members (sorted unique)
    std::vector<int32_t> xbptr, xb;               // per group: buckets listing it in bex (inverse)
};

// Per-thread scratch: every buffer the rewrite loop needs, reused across
// iterations (no allocation, no thread-local lookups in the hot loop).
struct Scratch {
    std::vector<int32_t> gnode, bnode, cur, from, to, ptr, adj, indeg, stack, stamp, bstamp, near, nbrs;
    std::vector<int32_t> ps, pt;
    std::vector<std::pair<int32_t, int32_t>> pairs;
    Index ix;
    State cand;
};

// sorted-unique CSR from (src, dst) pairs via counting sort + per-row insertion sort
static void csr_unique(int n, const std::vector<int32_t> &src, const std::vector<int32_t> &dst,
                       std::vector<int32_t> &ptr, std::vector<int32_t> &out, std::vector<int32_t> &cur) {
    ptr.assign(n + 1, 0);
    for (int32_t x : src) ptr[x + 1]++;
    for (int i = 0; i < n; i++) ptr[i + 1] += ptr[i];
    out.resize(src.size());
    cur.assign(ptr.begin(), ptr.end() - 1);
    for (size_t i = 0; i < src.size(); i++) out[cur[src[i]]++] = dst[i];
    int w = 0;
    int32_t *o = out.data();
    for (int i = 0; i < n; i++) {
        int b = ptr[i], e = ptr[i + 1];
        ptr[i] = w;
        if (e - b > 32) std::sort(o + b, o + e);
        else
            for (int k = b + 1; k < e; k++) {
                int32_t x = o[k];
                int j = k - 1;
                while (j >= b && o[j] > x) { o[j + 1] = o[j]; j--; }
                o[j + 1] = x;
            }
        for (int k = b; k < e; k++)
            if (k == b || o[k] != o[w - 1]) o[w++] = o[k];
    }
    ptr[n] = w;
    out.resize(w);
}

struct Engine {
    const fo_graph *g;
    int V, E, A, VB;  // VB: gid bound used for every state this engine emits
    explicit Engine(const fo_graph *gr) : g(gr), V(gr->V), E(gr->E), A(gr->A), VB(2 * gr->V + 2) {}

    State default_state() const {
        State s;
        s.ng.resize(V);
        s.rg.assign(V, -1);
        s.bk.resize(A);
        for (int v = 0; v < V; v++) s.ng[v] = v;
        for (int a = 0; a < A; a++) s.bk[a] = a;
        return s;
    }

    // group ids -> dense node order; returns G.  gnode sized VB.
    int number_groups(const State &s, std::vector<int32_t> &gnode, std::vector<int32_t> *gid) const {
        gnode.assign(VB, -1);
        int32_t *gn = gnode.data();
        for (int v = 0; v < V; v++) {
            gn[s.ng[v]] = 0;
            if (s.rg[v] >= 0) gn[s.rg[v]] = 0;
        }
        int G = 0;
        if (gid) gid->clear();
        for (int i = 0; i < VB; i++)
            if (gn[i] == 0) {
                if (gid) gid->push_back(i);
                gn[i] = G++;
            }
        return G;
    }

    int number_buckets(const State &s, std::vector<int32_t> &bnode, std::vector<int32_t> *bid) const {
        bnode.assign(A, -1);
        for (int a = 0; a < A; a++) bnode[s.bk[a]] = 0;
        int B = 0;
        if (bid) bid->clear();
        for (int i = 0; i < A; i++)
            if (bnode[i] == 0) {
                if (bid) bid->push_back(i);
                bnode[i] = B++;
            }
        return B;
    }

    void build(const State &s, Index &ix, Scratch &sc, bool buckets = true) const {
        ix.G = number_groups(s, sc.gnode, &ix.gid);
        const int G = ix.G;
        const int32_t *gn = sc.gnode.data();
        ix.nn.resize(V);
        ix.rr.resize(V);
        for (int v = 0; v < V; v++) {
            ix.nn[v] = gn[s.ng[v]];
            ix.rr[v] = s.rg[v] >= 0 ? gn[s.rg[v]] : -1;
        }
        // members, ascending op index
        ix.mptr.assign(G + 1, 0);
        for (int v = 0; v < V; v++) {
            ix.mptr[ix.nn[v] + 1]++;
            if (ix.rr[v] >= 0) ix.mptr[ix.rr[v] + 1]++;
        }
        for (int i = 0; i < G; i++) ix.mptr[i + 1] += ix.mptr[i];
        ix.mem.resize(ix.mptr[G]);
        ix.mdup.resize(ix.mptr[G]);
        sc.cur.assign(ix.mptr.begin(), ix.mptr.end() - 1);
        ix.compute_ok.assign(G, 1);
        ix.has_dup.assign(G, 0);
        ix.feeds_ar.assign(G, 0);
        ix.has_rep.assign(G, 0);
        for (int v = 0; v < V; v++) {
            const bool notc = g->op_kind[v] != 0, far = g->arp_ptr[v + 1] > g->arp_ptr[v], rep = ix.rr[v] >= 0;
            int x = ix.nn[v];
            ix.mdup[sc.cur[x]] = 0;
            ix.mem[sc.cur[x]++] = v;
            if (notc) ix.compute_ok[x] = 0;
            if (far) ix.feeds_ar[x] = 1;
            if (rep) ix.has_rep[x] = 1;  // some member has a replica (rewrite.py:116)
            if (rep) {
                x = ix.rr[v];
                ix.mdup[sc.cur[x]] = 1;
                ix.mem[sc.cur[x]++] = v;
                if (notc) ix.compute_ok[x] = 0;
                if (far) ix.feeds_ar[x] = 1;
                ix.has_dup[x] = 1;
                ix.has_rep[x] = 1;
            }
        }
        // contracted succs/preds over ALL edges (graph.py:161-179)
        sc.ps.clear();
        sc.pt.clear();
        for (int e = 0; e < E; e++) {
            int sv = g->e_src[e], dv = g->e_dst[e];
            int ns = ix.nn[sv], rs = ix.rr[sv], ex = rs >= 0 ? rs : ns;
            int c0 = ix.nn[dv], c1 = ix.rr[dv];
            if (c0 != ns && c0 != rs) { sc.ps.push_back(ex); sc.pt.push_back(c0); }
            if (c1 >= 0 && c1 != ns && c1 != rs) { sc.ps.push_back(ex); sc.pt.push_back(c1); }
        }
        csr_unique(G, sc.ps, sc.pt, ix.sptr, ix.succ, sc.cur);
        csr_unique(G, sc.pt, sc.ps, ix.pptr, ix.pred, sc.cur);
        if (!buckets) return;  // op-fusion moves never read the bucket structures
        // buckets: export groups of their members, and the inverse
        ix.B = number_buckets(s, sc.bnode, &ix.bid);
        ix.bki.resize(A);
        sc.ps.clear();
        sc.pt.clear();
        for (int a = 0; a < A; a++) {
            ix.bki[a] = sc.bnode[s.bk[a]];
            int pv = g->ar_prod[a];
            sc.ps.push_back(ix.bki[a]);
            sc.pt.push_back(ix.rr[pv] >= 0 ? ix.rr[pv] : ix.nn[pv]);
        }
        csr_unique(ix.B, sc.ps, sc.pt, ix.bptr, ix.bex, sc.cur);
        csr_unique(G, sc.pt, sc.ps, ix.xbptr, ix.xb, sc.cur);
    }

    // rewrite_candidate_ok (graph.py:505-512): Kahn over the joint schedule
    // dependency multigraph (multiplicity does not change acyclicity).
    bool valid(const State &s, Scratch &sc) const {
        const int G = number_groups(s, sc.gnode, nullptr);
        const int B = number_buckets(s, sc.bnode, nullptr);
        const int N = G + B;
        const int32_t *gn = sc.gnode.data(), *bn = sc.bnode.data();
        auto &from = sc.from, &to = sc.to;
        from.clear();
        to.clear();
        for (int e = 0; e < E; e++) {
            int sv = g->e_src[e], dv = g->e_dst[e];
            int c0 = gn[s.ng[dv]], c1 = s.rg[dv] >= 0 ? gn[s.rg[dv]] : -1;
            if (!g->agg[e]) {
                int ns = gn[s.ng[sv]], rs = s.rg[sv] >= 0 ? gn[s.rg[sv]] : -1, ex = rs >= 0 ? rs : ns;
                if (c0 != ns && c0 != rs) { from.push_back(ex); to.push_back(c0); }
                if (c1 >= 0 && c1 != ns && c1 != rs) { from.push_back(ex); to.push_back(c1); }
            } else {
                for (int q = g->arp_ptr[sv]; q < g->arp_ptr[sv + 1]; q++) {
                    int b = G + bn[s.bk[g->arp[q]]];
                    from.push_back(b); to.push_back(c0);
                    if (c1 >= 0) { from.push_back(b); to.push_back(c1); }
                }
            }
        }
        for (int a = 0; a < A; a++) {
            int pv = g->ar_prod[a];
            from.push_back(s.rg[pv] >= 0 ? gn[s.rg[pv]] : gn[s.ng[pv]]);
            to.push_back(G + bn[s.bk[a]]);
        }
        auto &ptr = sc.ptr, &adj = sc.adj, &indeg = sc.indeg, &stack = sc.stack;
        ptr.assign(N + 1, 0);
        indeg.assign(N, 0);
        adj.resize(from.size());
        for (size_t i = 0; i < from.size(); i++) { ptr[from[i] + 1]++; indeg[to[i]]++; }
        for (int i = 0; i < N; i++) ptr[i + 1] += ptr[i];
        sc.cur.assign(ptr.begin(), ptr.end() - 1);
        for (size_t i = 0; i < from.size(); i++) adj[sc.cur[from[i]]++] = to[i];
        stack.clear();
        for (int i = 0; i < N; i++)
            if (!indeg[i]) stack.push_back(i);
        int seen = 0;
        while (!stack.empty()) {
            int u = stack.back();
            stack.pop_back();
            seen++;
            for (int k = ptr[u]; k < ptr[u + 1]; k++)
                if (--indeg[adj[k]] == 0) stack.push_back(adj[k]);
        }
        return seen == N;
    }

    // fusible_pairs (rewrite.py:49-61) + DUP filter (rewrite.py:242-247), in order
    void fusible_pairs(const Index &ix, bool dup, std::vector<std::pair<int32_t, int32_t>> &out) const {
        out.clear();
        for (int x = 0; x < ix.G; x++) {
            if (!ix.compute_ok[x]) continue;
            for (int k = ix.pptr[x]; k < ix.pptr[x + 1]; k++) {
                int p = ix.pred[k];
                if (!ix.compute_ok[p] || (dup && ix.has_dup[p])) continue;
                out.emplace_back(x, p);
            }
        }
    }

    // bucket_pairs (rewrite.py:212-219) via neighbors_allreduce (rewrite.py:156-178):
    // nearby = own | succs(own) | preds(own); neighbours = buckets exporting from nearby
    void bucket_pairs(const Index &ix, Scratch &sc, std::vector<std::pair<int32_t, int32_t>> &out) const {
        out.clear();
        sc.stamp.assign(ix.G, -1);
        sc.bstamp.assign(ix.B, -1);
        for (int b = 0; b < ix.B; b++) {
            sc.near.clear();
            auto mark = [&](int x) {
                if (sc.stamp[x] != b) { sc.stamp[x] = b; sc.near.push_back(x); }
            };
            for (int k = ix.bptr[b]; k < ix.bptr[b + 1]; k++) {
                int x = ix.bex[k];
                mark(x);
                for (int q = ix.sptr[x]; q < ix.sptr[x + 1]; q++) mark(ix.succ[q]);
                for (int q = ix.pptr[x]; q < ix.pptr[x + 1]; q++) mark(ix.pred[q]);
            }
            sc.nbrs.clear();
            for (int x : sc.near)
                for (int q = ix.xbptr[x]; q < ix.xbptr[x + 1]; q++) {
                    int o = ix.xb[q];
                    if (o != b && sc.bstamp[o] != b) { sc.bstamp[o] = b; sc.nbrs.push_back(o); }
                }
            std::sort(sc.nbrs.begin(), sc.nbrs.end());
            for (int o : sc.nbrs) out.emplace_back(b, o);
        }
    }

    // topo_order (graph.py:536-556): Kahn over the contracted group graph,
    // ties to the smallest (min member op, group id).  False on a cycle.
    bool topo_groups(const Index &ix, std::vector<int32_t> &order) const {
        const int G = ix.G;
        std::vector<int32_t> indeg(G);
        for (int x = 0; x < G; x++) indeg[x] = ix.pptr[x + 1] - ix.pptr[x];
        using Key = std::pair<int32_t, int32_t>;  // (min member, dense id == id order)
        std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
        for (int x = 0; x < G; x++)
            if (!indeg[x]) heap.emplace(ix.mem[ix.mptr[x]], x);
        order.clear();
        while (!heap.empty()) {
            int x = heap.top().second;
            heap.pop();
            order.push_back(x);
            for (int k = ix.sptr[x]; k < ix.sptr[x + 1]; k++) {
                int h = ix.succ[k];
                if (--indeg[h] == 0) heap.emplace(ix.mem[ix.mptr[h]], h);
            }
        }
        return (int)order.size() == G;
    }

    // o in neighbors_allreduce(b) (rewrite.py:156-178), dense bucket indices
    bool bucket_neighbor(const Index &ix, Scratch &sc, int b, int o) const {
        if (o == b) return false;
        sc.stamp.assign(ix.G, 0);
        for (int k = ix.bptr[b]; k < ix.bptr[b + 1]; k++) {
            int x = ix.bex[k];
            sc.stamp[x] = 1;
            for (int q = ix.sptr[x]; q < ix.sptr[x + 1]; q++) sc.stamp[ix.succ[q]] = 1;
            for (int q = ix.pptr[x]; q < ix.pptr[x + 1]; q++) sc.stamp[ix.pred[q]] = 1;
        }
        for (int k = ix.bptr[o]; k < ix.bptr[o + 1]; k++)
            if (sc.stamp[ix.bex[k]]) return true;
        return false;
    }

    void compact(State &s, Scratch &sc) const {  // monotone relabel of group ids to 0..G-1
        number_groups(s, sc.gnode, nullptr);
        for (int v = 0; v < V; v++) {
            s.ng[v] = sc.gnode[s.ng[v]];
            if (s.rg[v] >= 0) s.rg[v] = sc.gnode[s.rg[v]];
        }
    }

    // fuse_nondup (rewrite.py:64-96) / fuse_dup (rewrite.py:99-153)
    bool fuse_ops(const State &s, const Index &ix, int og, int pg, bool dup, State &out, Scratch &sc) const {
        if (og == pg) return false;
        for (int k = ix.mptr[pg]; k < ix.mptr[pg + 1]; k++) {  // groups share a member (rewrite.py:76-79)
            int v = ix.mem[k];
            if (ix.nn[v] == og || ix.rr[v] == og) return false;
        }
        if (!ix.compute_ok[og] || !ix.compute_ok[pg]) return false;
        int32_t gidx = ix.gid[og], gidp = ix.gid[pg];
        int32_t merged = std::min(gidx, gidp);
        out = s;
        if (dup) {
            if (ix.has_rep[pg]) return false;  // rewrite.py:116-118
            bool other = false;
            for (int k = ix.sptr[pg]; k < ix.sptr[pg + 1]; k++) other |= ix.succ[k] != og;
            if (other || ix.feeds_ar[pg]) {
                int32_t replica = ix.gid[ix.G - 1] + 1;  // rewrite.py:138
                if (replica >= VB) {  // ids only matter by order: compact, then recompute
                    compact(out, sc);
                    merged = std::min(og, pg);
                    replica = ix.G;
                }
                for (int k = ix.mptr[og]; k < ix.mptr[og + 1]; k++) {
                    int v = ix.mem[k];
                    if (ix.mdup[k]) out.rg[v] = merged; else out.ng[v] = merged;
                }
                for (int k = ix.mptr[pg]; k < ix.mptr[pg + 1]; k++) {
                    int v = ix.mem[k];
                    out.ng[v] = merged;
                    out.rg[v] = replica;
                }
                return valid(out, sc);
            }
        }
        for (int x : {og, pg})
            for (int k = ix.mptr[x]; k < ix.mptr[x + 1]; k++) {
                int v = ix.mem[k];
                if (ix.mdup[k]) out.rg[v] = merged; else out.ng[v] = merged;
            }
        return valid(out, sc);
    }

    // fuse_allreduce (rewrite.py:181-209)
    bool fuse_ar(const State &s, const Index &ix, int bo, int bn, State &out, Scratch &sc) const {
        int32_t merged = std::min(ix.bid[bo], ix.bid[bn]);
        out = s;
        for (int a = 0; a < A; a++)
            if (ix.bki[a] == bo || ix.bki[a] == bn) out.bk[a] = merged;
        return valid(out, sc);
    }

    // random_apply (rewrite.py:222-263); state updated in place
    bool random_apply(State &s, int method, int n, PyRng &rng, Scratch &sc) const {
        bool applied = false, stale = true;
        for (int it = 0; it < n; it++) {
            if (stale) {  // a rejected draw leaves the state, its index and its choice list unchanged
                build(s, sc.ix, sc, method == M_AR);
                if (method == M_AR) bucket_pairs(sc.ix, sc, sc.pairs);
                else fusible_pairs(sc.ix, method == M_DUP, sc.pairs);
                stale = false;
            }
            if (sc.pairs.empty()) break;
            auto pr = sc.pairs[rng.below((uint32_t)sc.pairs.size())];
            bool ok = method == M_AR ? fuse_ar(s, sc.ix, pr.first, pr.second, sc.cand, sc)
                                     : fuse_ops(s, sc.ix, pr.first, pr.second, method == M_DUP, sc.cand, sc);
            if (ok) {
                std::swap(s, sc.cand);
                applied = true;
                stale = true;
            }
        }
        return applied;
    }

    // canonical state hash: the state is a set of (members, duplicated) group
    // tuples plus a set of bucket member tuples (graph.py:559-580)
    static uint64_t mix(uint64_t x) {
        x += 0x9e3779b97f4a7c15ull;
        x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
        x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
        return x ^ (x >> 31);
    }
    uint64_t hash(const State &s) const {
        // group content hashes accumulated per group id (ops visited ascending)
        thread_local std::vector<uint64_t> acc, bacc;
        thread_local std::vector<uint8_t> used, bused;
        acc.assign(VB, 0);
        used.assign(VB, 0);
        for (int v = 0; v < V; v++) {
            int x = s.ng[v];
            acc[x] = mix(acc[x] ^ (uint64_t)(2 * v + 2));
            used[x] = 1;
            if (s.rg[v] >= 0) {
                x = s.rg[v];
                acc[x] = mix(acc[x] ^ (uint64_t)(2 * v + 3));
                used[x] = 1;
            }
        }
        uint64_t h = 0x6a09e667f3bcc909ull;
        for (int i = 0; i < VB; i++)
            if (used[i]) h += mix(acc[i] + 0x3c6ef372fe94f82bull);
        bacc.assign(A, 0);
        bused.assign(A, 0);
        for (int a = 0; a < A; a++) {
            int b = s.bk[a];
            bacc[b] = mix(bacc[b] ^ (uint64_t)(a + 1));
            bused[b] = 1;
        }
        for (int b = 0; b < A; b++)
            if (bused[b]) h += mix(bacc[b] + 0xa54ff53a5f1d36f1ull);
        return h;
    }

    bool load_state(const int32_t *ng, const int32_t *rg, const int32_t *bk, State &s) const {
        s = default_state();
        if (!ng) return true;
        std::vector<int32_t> ids;
        for (int v = 0; v < V; v++) {
            if (ng[v] < 0 || rg[v] < -1) return false;
            ids.push_back(ng[v]);
            if (rg[v] >= 0) ids.push_back(rg[v]);
        }
        std::sort(ids.begin(), ids.end());
        ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
        auto rank = [&](int32_t x) { return (int32_t)(std::lower_bound(ids.begin(), ids.end(), x) - ids.begin()); };
        for (int v = 0; v < V; v++) {
            s.ng[v] = rank(ng[v]);
            s.rg[v] = rg[v] >= 0 ? rank(rg[v]) : -1;
        }
        for (int a = 0; a < A; a++) {
            if (bk[a] < 0 || bk[a] >= A) return false;
            s.bk[a] = bk[a];
        }
        return true;
    }
};

// ---------------------------------------------------------------------------
// Incremental rewrite engine.  Engine::random_apply
// rebuilds the whole index after every accepted rewrite and runs a full Kahn
// pass per draw: O(V + E) per draw, ~50 ms per candidate at 50k ops.  Inc
// keeps the index live instead:
//   * per group id: members, flags, and four sorted-unique rows -- contracted
//     preds / succs over all edges (graph.py:161-179) and joint schedule
//     preds / succs with the bucket nodes (graph.py:215-274); bucket nodes
//     carry their joint rows too.  A merge recomputes only the rows of the
//     merged node and of its neighbours, from their member ops' edges.
//   * the fusible-pair list (rewrite.py:49-61) as per-group counts in a
//     Fenwick tree over group ids, so the k-th pair in the reference's order
//     is found without materialising the list.
//   * a topological order of the joint graph.  A merge of u and v is cyclic
//     iff a node reachable from the merged node's successors can reach it,
//     and every such node lies strictly between pos(u) and pos(v): the
//     validity test is a DFS bounded to that window (rewrite_candidate_ok,
//     graph.py:505-512), and an accepted merge reorders only that window
//     (Pearce-Kelly: the window's ancestors of the merged node, then the
//     merged node, then its descendants).
//   * a duplicate fusion that leaves a replica never needs the test: the
//     merged group takes the consumer's position and the replica the
//     producer's, and every new dependency runs forward in the old order.
// Draw sequence, accept/reject decisions and ids equal Engine::random_apply
// (cross-checked by tests/test_native_cpu.py with FO_ENGINE=full).

struct Inc {
    const fo_graph *g = nullptr;
    int V = 0, E = 0, A = 0, VB = 0, NJ = 0;
    std::vector<int32_t> ng, rg, bk;  // fusion state (engine ids)
    int maxid = -1;                   // largest live group id
    // groups by id
    std::vector<uint8_t> alive, cok, hdup, far, hrep;
    std::vector<int32_t> moff, mlen, mpool;  // members (op << 1 | dup), ascending op
    // rows: kind 0 contracted preds, 1 contracted succs (groups only),
    // 2 joint preds, 3 joint succs (groups [0, VB), bucket b at VB + b)
    std::vector<int32_t> roff[4], rlen[4], rpool;
    std::vector<int32_t> pos;  // topological position in the joint graph
    // buckets by id: member ARs ascending, total bytes
    std::vector<int32_t> boff, blen, bpool;
    std::vector<int64_t> btot;
    // fusible-pair counts per group id for the nondup (0) and dup (1) rules,
    // Fenwick trees over ids, kept current across every rewrite
    int method = -1;
    std::vector<int32_t> cnt[2], fen[2];
    int64_t tot[2] = {0, 0};
    int64_t total = 0;
    // AR method: materialised bucket pairs
    std::vector<std::pair<int32_t, int32_t>> arpairs;
    // scratch
    std::vector<int32_t> t0, t1, t2, t3, mark, stk, F, Bk, nb, gen, ihead;
    std::vector<std::pair<int32_t, int32_t>> iv;
    int32_t gen_no = 0;
    // undo journal: a candidate is applied to a shared index and rolled back
    // (checkpoint / undo), so per-candidate cost is the rewrites' footprint,
    // not a copy of the index
    bool jon = false, rebuilt = false;
    std::vector<std::pair<int32_t *, int32_t>> j32;
    std::vector<std::pair<uint8_t *, uint8_t>> j8;
    std::vector<std::pair<int64_t *, int64_t>> j64;
    size_t cp_m = 0, cp_r = 0, cp_b = 0;
    int cp_maxid = -1;
    int64_t cp_tot[2] = {0, 0};
    void S(int32_t &r, int32_t v) {
        if (jon) j32.emplace_back(&r, r);
        r = v;
    }
    void S(uint8_t &r, uint8_t v) {
        if (jon) j8.emplace_back(&r, r);
        r = v;
    }
    void S(int64_t &r, int64_t v) {
        if (jon) j64.emplace_back(&r, r);
        r = v;
    }
    void checkpoint() {
        jon = true;
        rebuilt = false;
        j32.clear();
        j8.clear();
        j64.clear();
        cp_m = mpool.size();
        cp_r = rpool.size();
        cp_b = bpool.size();
        cp_maxid = maxid;
        cp_tot[0] = tot[0];
        cp_tot[1] = tot[1];
    }
    // false when a rebuild (id compaction) happened: the caller recopies the base
    bool undo() {
        jon = false;
        if (rebuilt) return false;
        for (size_t i = j32.size(); i-- > 0;) *j32[i].first = j32[i].second;
        for (size_t i = j8.size(); i-- > 0;) *j8[i].first = j8[i].second;
        for (size_t i = j64.size(); i-- > 0;) *j64[i].first = j64[i].second;
        mpool.resize(cp_m);
        rpool.resize(cp_r);
        bpool.resize(cp_b);
        maxid = cp_maxid;
        tot[0] = cp_tot[0];
        tot[1] = cp_tot[1];
        return true;
    }

    const int32_t *row(int k, int n) const { return rpool.data() + roff[k][n]; }
    int rowlen(int k, int n) const { return rlen[k][n]; }
    bool member(int s, int c) const { return ng[s] == c || rg[s] == c; }
    int exportg(int s) const { return rg[s] >= 0 ? rg[s] : ng[s]; }

    void store(int k, int n, std::vector<int32_t> &t) {
        std::sort(t.begin(), t.end());
        t.erase(std::unique(t.begin(), t.end()), t.end());
        if (!jon && (int)t.size() <= rlen[k][n]) {  // shrinking rows rewrite in place
            std::copy(t.begin(), t.end(), rpool.begin() + roff[k][n]);
        } else {
            S(roff[k][n], (int32_t)rpool.size());
            rpool.insert(rpool.end(), t.begin(), t.end());
        }
        S(rlen[k][n], (int32_t)t.size());
    }

    // the four rows of group x from its member ops' edges
    void rows_group(int x) {
        t0.clear();
        t1.clear();
        const int32_t *m = mpool.data() + moff[x];
        for (int i = 0; i < mlen[x]; i++) {
            const int d = m[i] >> 1;
            for (int q = g->in_ptr[d]; q < g->in_ptr[d + 1]; q++) {
                const int e = g->in_e[q], s = g->e_src[e];
                const bool inside = member(s, x);
                if (!inside) t0.push_back(exportg(s));
                if (!g->agg[e]) {
                    if (!inside) t1.push_back(exportg(s));
                } else {
                    for (int r = g->arp_ptr[s]; r < g->arp_ptr[s + 1]; r++) t1.push_back(VB + bk[g->arp[r]]);
                }
            }
        }
        store(0, x, t0);
        store(2, x, t1);
        t0.clear();
        t1.clear();
        for (int i = 0; i < mlen[x]; i++) {
            const int s = m[i] >> 1;
            if (exportg(s) != x) continue;
            const int ns = ng[s], rs = rg[s];
            for (int q = g->out_ptr[s]; q < g->out_ptr[s + 1]; q++) {
                const int e = g->out_e[q], d = g->e_dst[e];
                const int c0 = ng[d], c1 = rg[d];
                if (c0 != ns && c0 != rs) {
                    t0.push_back(c0);
                    if (!g->agg[e]) t1.push_back(c0);
                }
                if (c1 >= 0 && c1 != ns && c1 != rs) {
                    t0.push_back(c1);
                    if (!g->agg[e]) t1.push_back(c1);
                }
            }
            for (int r = g->arp_ptr[s]; r < g->arp_ptr[s + 1]; r++) t1.push_back(VB + bk[g->arp[r]]);
        }
        store(1, x, t0);
        store(3, x, t1);
    }

    // joint rows of bucket b: producers' export groups in, aggregate consumers out
    void rows_bucket(int b) {
        t0.clear();
        t1.clear();
        const int32_t *m = bpool.data() + boff[b];
        for (int i = 0; i < blen[b]; i++) {
            const int s = g->ar_prod[m[i]];
            t0.push_back(exportg(s));
            for (int q = g->out_ptr[s]; q < g->out_ptr[s + 1]; q++) {
                const int e = g->out_e[q];
                if (!g->agg[e]) continue;
                const int d = g->e_dst[e];
                t1.push_back(ng[d]);
                if (rg[d] >= 0) t1.push_back(rg[d]);
            }
        }
        store(2, VB + b, t0);
        store(3, VB + b, t1);
    }

    void group_flags(int x) {
        cok[x] = 1;
        hdup[x] = far[x] = hrep[x] = 0;
        const int32_t *m = mpool.data() + moff[x];
        for (int i = 0; i < mlen[x]; i++) {
            const int v = m[i] >> 1;
            if (g->op_kind[v] != 0) cok[x] = 0;
            if (g->arp_ptr[v + 1] > g->arp_ptr[v]) far[x] = 1;
            if (m[i] & 1) hdup[x] = 1;
            if (rg[v] >= 0) hrep[x] = 1;
        }
    }

    // full build from a state (ids < VB); false when the joint graph is cyclic
    bool build(const fo_graph *gr, const State &s, int vb) {
        g = gr;
        V = gr->V;
        E = gr->E;
        A = gr->A;
        VB = vb;
        NJ = VB + A;
        ng = s.ng;
        rg = s.rg;
        bk = s.bk;
        alive.assign(VB, 0);
        cok.assign(VB, 0);
        hdup.assign(VB, 0);
        far.assign(VB, 0);
        hrep.assign(VB, 0);
        moff.assign(VB, 0);
        mlen.assign(VB, 0);
        for (int v = 0; v < V; v++) {
            mlen[ng[v]]++;
            if (rg[v] >= 0) mlen[rg[v]]++;
        }
        int o = 0;
        maxid = -1;
        for (int x = 0; x < VB; x++) {
            moff[x] = o;
            o += mlen[x];
            if (mlen[x]) {
                alive[x] = 1;
                maxid = x;
            }
            mlen[x] = 0;
        }
        mpool.assign(o, 0);
        for (int v = 0; v < V; v++) {  // ascending op: member lists come out sorted
            mpool[moff[ng[v]] + mlen[ng[v]]++] = v << 1;
            if (rg[v] >= 0) mpool[moff[rg[v]] + mlen[rg[v]]++] = (v << 1) | 1;
        }
        for (int x = 0; x < VB; x++)
            if (alive[x]) group_flags(x);
        boff.assign(A, 0);
        blen.assign(A, 0);
        btot.assign(A, 0);
        for (int a = 0; a < A; a++) {
            blen[bk[a]]++;
            btot[bk[a]] += g->ar_bytes[a];
        }
        o = 0;
        for (int b = 0; b < A; b++) {
            boff[b] = o;
            o += blen[b];
            blen[b] = 0;
        }
        bpool.assign(o, 0);
        for (int a = 0; a < A; a++) bpool[boff[bk[a]] + blen[bk[a]]++] = a;
        for (int k = 0; k < 4; k++) {
            roff[k].assign(NJ, 0);
            rlen[k].assign(NJ, 0);
        }
        rpool.clear();
        rpool.reserve(4 * (size_t)E + 4 * (size_t)A + 1024);
        for (int x = 0; x < VB; x++)
            if (alive[x]) rows_group(x);
        for (int b = 0; b < A; b++)
            if (blen[b]) rows_bucket(b);
        // topological positions of the joint graph (Kahn, LIFO: chains stay contiguous)
        pos.assign(NJ, 0);
        std::vector<int32_t> indeg(NJ, 0);
        stk.clear();
        int nodes = 0;
        for (int n = 0; n < NJ; n++) {
            const bool live = n < VB ? alive[n] : blen[n - VB] > 0;
            if (!live) continue;
            nodes++;
            indeg[n] = rlen[2][n];
            if (!indeg[n]) stk.push_back(n);
        }
        int p = 0;
        while (!stk.empty()) {
            const int u = stk.back();
            stk.pop_back();
            pos[u] = p++;
            const int32_t *r = row(3, u);
            for (int i = 0; i < rlen[3][u]; i++)
                if (--indeg[r[i]] == 0) stk.push_back(r[i]);
        }
        mark.assign(NJ, 0);
        gen.assign(NJ, 0);
        gen_no = 0;
        method = -1;
        init_counts();
        return p == nodes;
    }

    // ---- fusible pairs in the reference's order (rewrite.py:49-61, :242-247)
    bool qual(int p, int r) const { return cok[p] && !(r == 1 && hdup[p]); }
    void count_of(int x, int c[2]) const {
        c[0] = c[1] = 0;
        if (!alive[x] || !cok[x]) return;
        const int32_t *r = row(0, x);
        for (int i = 0; i < rlen[0][x]; i++) {
            const int p = r[i];
            if (cok[p]) {
                c[0]++;
                c[1] += !hdup[p];
            }
        }
    }
    void fen_add(int r, int x, int d) {
        for (int i = x + 1; i <= VB; i += i & -i) S(fen[r][i], fen[r][i] + d);
        tot[r] += d;
    }
    void recount(int x) {
        int c[2];
        count_of(x, c);
        for (int r = 0; r < 2; r++)
            if (c[r] != cnt[r][x]) {
                fen_add(r, x, c[r] - cnt[r][x]);
                S(cnt[r][x], c[r]);
            }
        if (method == M_NONDUP || method == M_DUP) total = tot[method == M_DUP];
    }
    void init_counts() {
        for (int r = 0; r < 2; r++) {
            cnt[r].assign(VB, 0);
            fen[r].assign(VB + 1, 0);
            tot[r] = 0;
        }
        for (int x = 0; x < VB; x++) {
            int c[2];
            count_of(x, c);
            for (int r = 0; r < 2; r++) {
                cnt[r][x] = c[r];
                tot[r] += c[r];
                fen[r][x + 1] += c[r];
            }
        }
        for (int r = 0; r < 2; r++)
            for (int i = 1; i <= VB; i++) {
                const int j = i + (i & -i);
                if (j <= VB) fen[r][j] += fen[r][i];
            }
    }
    void prepare_op_pairs(int m) {
        method = m;
        total = tot[m == M_DUP];
    }
    std::pair<int, int> select(int64_t k) const {  // k-th pair, 0-based
        const int rr = method == M_DUP;
        const std::vector<int32_t> &f = fen[rr];
        int x = 0;
        int step = 1;
        while (step * 2 <= VB) step *= 2;
        for (; step; step >>= 1)
            if (x + step <= VB && f[x + step] <= k) {
                x += step;
                k -= f[x];
            }
        // group x (0-based) holds the pair; k-th qualifying pred
        const int32_t *r = row(0, x);
        for (int i = 0; i < rlen[0][x]; i++)
            if (qual(r[i], rr) && k-- == 0) return {x, r[i]};
        return {-1, -1};
    }

    // ---- bucket pairs (rewrite.py:156-178, :212-219)
    void prepare_ar_pairs() {
        method = M_AR;
        arpairs.clear();
        // inverse: group -> buckets exporting from it (bex = joint preds of a
        // bucket), as (group, bucket) pairs sorted by group; ihead[x] (stamped
        // by gen == gi) is the first pair of group x
        iv.clear();
        for (int b = 0; b < A; b++)
            if (blen[b]) {
                const int32_t *r = row(2, VB + b);
                for (int i = 0; i < rlen[2][VB + b]; i++) iv.emplace_back(r[i], b);
            }
        std::sort(iv.begin(), iv.end());
        if ((int)ihead.size() < VB) ihead.assign(VB, 0);
        const int32_t gi = ++gen_no;
        for (int i = (int)iv.size() - 1; i >= 0; i--) {
            ihead[iv[i].first] = i;
            gen[iv[i].first] = gi;
        }
        for (int b = 0; b < A; b++) {
            if (!blen[b]) continue;
            t0.clear();
            const int32_t *r = row(2, VB + b);
            // nearby groups
            for (int i = 0; i < rlen[2][VB + b]; i++) {
                const int x = r[i];
                t0.push_back(x);
                const int32_t *s1 = row(1, x);
                t0.insert(t0.end(), s1, s1 + rlen[1][x]);
                const int32_t *p1 = row(0, x);
                t0.insert(t0.end(), p1, p1 + rlen[0][x]);
            }
            t1.clear();
            for (int x : t0) {
                if (gen[x] != gi) continue;  // no bucket exports from x
                for (int q = ihead[x]; q < (int)iv.size() && iv[q].first == x; q++)
                    if (iv[q].second != b) t1.push_back(iv[q].second);
            }
            std::sort(t1.begin(), t1.end());
            t1.erase(std::unique(t1.begin(), t1.end()), t1.end());
            for (int o : t1) arpairs.emplace_back(b, o);
        }
        total = (int64_t)arpairs.size();
    }

    // ---- validity of merging joint nodes u, v (rewrite_candidate_ok)
    // IN marks (gen == gin) the merged node's in-neighbours; the DFS from its
    // successors, bounded to positions < max(pos u, pos v), fails on reaching
    // one.  F collects the visited window.
    bool acyclic_merge(int u, int v, int32_t gin) {
        const int P = std::max(pos[u], pos[v]);
        const int32_t gv = ++gen_no;
        F.clear();
        stk.clear();
        for (int w : {u, v}) {
            const int32_t *r = row(3, w);
            for (int i = 0; i < rlen[3][w]; i++) {
                const int y = r[i];
                if (y == u || y == v || pos[y] >= P || gen[y] == gv) continue;
                gen[y] = gv;
                stk.push_back(y);
            }
        }
        while (!stk.empty()) {
            const int y = stk.back();
            stk.pop_back();
            if (mark[y] == gin) return false;
            F.push_back(y);
            const int32_t *r = row(3, y);
            for (int i = 0; i < rlen[3][y]; i++) {
                const int z = r[i];
                if (z == u || z == v || pos[z] >= P || gen[z] == gv) continue;
                gen[z] = gv;
                stk.push_back(z);
            }
        }
        return true;
    }
    // reorder the window after merging u, v into keep (Pearce-Kelly): the
    // merged node's ancestors inside the window (Bk), then it, then F
    void reorder(int u, int v, int keep, int32_t gin) {
        const int L = std::min(pos[u], pos[v]);
        const int32_t gb = ++gen_no;
        Bk.clear();
        stk.clear();
        for (int n : t2)  // in-neighbours of the merged node
            if (pos[n] > L && gen[n] != gb) {
                gen[n] = gb;
                stk.push_back(n);
            }
        while (!stk.empty()) {
            const int y = stk.back();
            stk.pop_back();
            Bk.push_back(y);
            const int32_t *r = row(2, y);
            for (int i = 0; i < rlen[2][y]; i++) {
                const int z = r[i];
                if (z == u || z == v || pos[z] <= L || gen[z] == gb) continue;
                gen[z] = gb;
                stk.push_back(z);
            }
        }
        (void)gin;
        auto by_pos = [&](int a, int b) { return pos[a] < pos[b]; };
        std::sort(Bk.begin(), Bk.end(), by_pos);
        std::sort(F.begin(), F.end(), by_pos);
        t3.clear();
        for (int n : Bk) t3.push_back(pos[n]);
        for (int n : F) t3.push_back(pos[n]);
        t3.push_back(pos[u]);
        t3.push_back(pos[v]);
        std::sort(t3.begin(), t3.end());
        int i = 0;
        for (int n : Bk) S(pos[n], t3[i++]);
        S(pos[keep], t3[i++]);
        for (int n : F) S(pos[n], t3[i++]);
    }

    // in-neighbours of the group merging og and pg (exclusion relative to the
    // merged member set, graph.py:245-262), marked with a fresh generation; the
    // list lands in t2
    int32_t mark_in_groups(int og, int pg) {
        const int32_t gi = ++gen_no;
        t2.clear();
        auto add = [&](int n) {
            if (mark[n] != gi) {
                mark[n] = gi;
                t2.push_back(n);
            }
        };
        for (int x : {og, pg}) {
            const int32_t *m = mpool.data() + moff[x];
            for (int i = 0; i < mlen[x]; i++) {
                const int d = m[i] >> 1;
                for (int q = g->in_ptr[d]; q < g->in_ptr[d + 1]; q++) {
                    const int e = g->in_e[q], s = g->e_src[e];
                    if (g->agg[e]) {
                        for (int r = g->arp_ptr[s]; r < g->arp_ptr[s + 1]; r++) add(VB + bk[g->arp[r]]);
                    } else if (!member(s, og) && !member(s, pg)) {
                        add(exportg(s));
                    }
                }
            }
        }
        return gi;
    }

    // neighbours of nodes (all row kinds), excluding the nodes themselves -> nb
    void collect_neighbours(std::initializer_list<int> nodes) {
        const int32_t gg = ++gen_no;
        nb.clear();
        for (int n : nodes) gen[n] = gg;
        for (int n : nodes)
            for (int k = 0; k < 4; k++) {
                if (k < 2 && n >= VB) continue;
                const int32_t *r = row(k, n);
                for (int i = 0; i < rlen[k][n]; i++)
                    if (gen[r[i]] != gg) {
                        gen[r[i]] = gg;
                        nb.push_back(r[i]);
                    }
            }
    }
    void refresh(int n) {
        if (n < VB) {
            if (alive[n]) rows_group(n);
        } else if (blen[n - VB]) {
            rows_bucket(n - VB);
        }
    }
    void kill_group(int x) {
        S(alive[x], 0);
        S(mlen[x], 0);
        for (int k = 0; k < 4; k++) S(rlen[k][x], 0);
        while (maxid >= 0 && !alive[maxid]) maxid--;
    }
    // merge member lists of x and y into a fresh slot for id keep
    void merge_members(int x, int y, int keep, bool y_normal_only) {
        t0.clear();
        const int32_t *a = mpool.data() + moff[x], *b = mpool.data() + moff[y];
        int i = 0, j = 0;
        while (i < mlen[x] || j < mlen[y]) {
            if (j >= mlen[y] || (i < mlen[x] && (a[i] >> 1) < (b[j] >> 1))) t0.push_back(a[i++]);
            else t0.push_back(y_normal_only ? (b[j++] & ~1) : b[j++]);
        }
        S(moff[keep], (int32_t)mpool.size());
        S(mlen[keep], (int32_t)t0.size());
        mpool.insert(mpool.end(), t0.begin(), t0.end());
    }

    // non-duplicate fusion of pg into og (rewrite.py:64-96); false if rejected
    bool try_nondup(int og, int pg) {
        if (og == pg) return false;
        {
            const int32_t *m = mpool.data() + moff[pg];
            for (int i = 0; i < mlen[pg]; i++)
                if (member(m[i] >> 1, og)) return false;  // groups share a member
        }
        if (!cok[og] || !cok[pg]) return false;
        const int32_t gin = mark_in_groups(og, pg);
        if (!acyclic_merge(og, pg, gin)) return false;
        const int keep = std::min(og, pg), dead = std::max(og, pg);
        reorder(og, pg, keep, gin);
        collect_neighbours({og, pg});
        // state: every membership of og / pg moves to keep (duplicated stays duplicated)
        for (int x : {og, pg}) {
            const int32_t *m = mpool.data() + moff[x];
            for (int i = 0; i < mlen[x]; i++) {
                const int v = m[i] >> 1;
                if (m[i] & 1) S(rg[v], keep); else S(ng[v], keep);
            }
        }
        merge_members(og, pg, keep, false);
        const uint8_t fd = hdup[og] | hdup[pg], ff = far[og] | far[pg], fr = hrep[og] | hrep[pg];
        kill_group(dead);
        S(alive[keep], 1);
        S(cok[keep], 1);
        S(hdup[keep], fd);
        S(far[keep], ff);
        S(hrep[keep], fr);
        if (keep > maxid) maxid = keep;
        rows_group(keep);
        for (int n : nb) refresh(n);
        recount(keep);
        recount(dead);
        for (int n : nb)
            if (n < VB) recount(n);
        return true;
    }
    // relabel group ids to 0..G-1 in id order (Engine::compact) and rebuild;
    // og / pg follow their groups
    void compact_rebuild(int &og, int &pg) {
        std::vector<int32_t> rank(VB, -1);
        int G = 0;
        for (int x = 0; x < VB; x++)
            if (alive[x]) rank[x] = G++;
        State s;
        s.ng.resize(V);
        s.rg.resize(V);
        for (int v = 0; v < V; v++) {
            s.ng[v] = rank[ng[v]];
            s.rg[v] = rg[v] >= 0 ? rank[rg[v]] : -1;
        }
        s.bk = bk;
        og = rank[og];
        pg = rank[pg];
        const int m = method;
        const bool j = jon;
        build(g, s, VB);
        jon = j;
        rebuilt = true;
        if (m >= 0 && m != M_AR) prepare_op_pairs(m);
        else method = m;
    }

    // duplicate fusion (rewrite.py:99-153); degrades to nondup without other
    // consumers.  The replica path needs no acyclicity test (see above).
    bool try_dup(int og, int pg) {
        if (og == pg) return false;
        {
            const int32_t *m = mpool.data() + moff[pg];
            for (int i = 0; i < mlen[pg]; i++)
                if (member(m[i] >> 1, og)) return false;
        }
        if (!cok[og] || !cok[pg]) return false;
        if (hrep[pg]) return false;  // rewrite.py:116-118
        bool other = far[pg] != 0;
        {
            const int32_t *r = row(1, pg);
            for (int i = 0; i < rlen[1][pg]; i++) other |= r[i] != og;
        }
        if (!other) return try_nondup(og, pg);
        if (maxid + 1 >= VB) compact_rebuild(og, pg);
        const int R = maxid + 1;  // rewrite.py:138
        const int keep = std::min(og, pg), dead = std::max(og, pg);
        const int po = pos[og], pp = pos[pg];
        collect_neighbours({og, pg});
        // replica member list first (pg's slot may be reused by keep)
        {
            const int32_t *m = mpool.data() + moff[pg];
            t1.clear();
            for (int i = 0; i < mlen[pg]; i++) t1.push_back(m[i] | 1);
            S(moff[R], (int32_t)mpool.size());
            S(mlen[R], (int32_t)t1.size());
            mpool.insert(mpool.end(), t1.begin(), t1.end());
        }
        {
            const int32_t *m = mpool.data() + moff[og];
            for (int i = 0; i < mlen[og]; i++) {
                const int v = m[i] >> 1;
                if (m[i] & 1) S(rg[v], keep); else S(ng[v], keep);
            }
            m = mpool.data() + moff[pg];
            for (int i = 0; i < mlen[pg]; i++) {
                const int v = m[i] >> 1;
                S(ng[v], keep);
                S(rg[v], R);
            }
        }
        merge_members(og, pg, keep, true);
        const uint8_t fd = hdup[og], ff = far[og] | far[pg], fr_p = far[pg];
        kill_group(dead);
        S(alive[keep], 1);
        S(cok[keep], 1);
        S(hdup[keep], fd);
        S(far[keep], ff);
        S(hrep[keep], 1);
        S(alive[R], 1);
        S(cok[R], 1);
        S(hdup[R], 1);
        S(far[R], fr_p);
        S(hrep[R], 1);
        maxid = std::max(maxid, R);
        S(pos[keep], po);
        S(pos[R], pp);
        rows_group(keep);
        rows_group(R);
        for (int n : nb) refresh(n);
        recount(keep);
        recount(dead);
        recount(R);
        for (int n : nb)
            if (n < VB) recount(n);
        return true;
    }

    // AllReduce fusion of buckets bo, bn (rewrite.py:181-209)
    bool try_ar(int bo, int bn) {
        const int u = VB + bo, v = VB + bn;
        const int32_t gi = ++gen_no;
        t2.clear();
        for (int w : {u, v}) {
            const int32_t *r = row(2, w);
            for (int i = 0; i < rlen[2][w]; i++)
                if (mark[r[i]] != gi) {
                    mark[r[i]] = gi;
                    t2.push_back(r[i]);
                }
        }
        if (!acyclic_merge(u, v, gi)) return false;
        const int keep = std::min(bo, bn), dead = std::max(bo, bn);
        reorder(u, v, VB + keep, gi);
        collect_neighbours({u, v});
        t0.clear();
        const int32_t *a = bpool.data() + boff[bo], *b = bpool.data() + boff[bn];
        int i = 0, j = 0;
        while (i < blen[bo] || j < blen[bn]) {
            if (j >= blen[bn] || (i < blen[bo] && a[i] < b[j])) t0.push_back(a[i++]);
            else t0.push_back(b[j++]);
        }
        for (int x : t0) S(bk[x], keep);
        const int64_t bt = btot[bo] + btot[bn];
        S(btot[dead], 0);
        S(btot[keep], bt);
        S(blen[dead], 0);
        S(rlen[2][VB + dead], 0);
        S(rlen[3][VB + dead], 0);
        S(boff[keep], (int32_t)bpool.size());
        S(blen[keep], (int32_t)t0.size());
        bpool.insert(bpool.end(), t0.begin(), t0.end());
        rows_bucket(keep);
        for (int n : nb) refresh(n);
        return true;
    }

    // random_apply (rewrite.py:222-263) on the live state
    bool random_apply(int m, int n, PyRng &rng) {
        if (n <= 0) return false;
        if (m == M_AR) prepare_ar_pairs();
        else prepare_op_pairs(m);
        bool applied = false;
        for (int it = 0; it < n; it++) {
            if (total == 0) break;
            const uint32_t k = rng.below((uint32_t)total);
            bool ok;
            if (m == M_AR) {
                const auto pr = arpairs[k];
                ok = try_ar(pr.first, pr.second);
                if (ok) prepare_ar_pairs();
            } else {
                const auto pr = select(k);
                ok = m == M_DUP ? try_dup(pr.first, pr.second) : try_nondup(pr.first, pr.second);
            }
            applied |= ok;
        }
        return applied;
    }

    void to_state(State &s) const {
        s.ng = ng;
        s.rg = rg;
        s.bk = bk;
    }
};

// FO_ENGINE=full selects the full-rebuild Engine path (cross-checking only)
static bool use_full_engine() {
    const char *e = getenv("FO_ENGINE");
    return e && std::strcmp(e, "full") == 0;
}

}  // namespace fo

using namespace fo;

extern "C" {

extern "C++" {
// Candidate k: random.Random(seeds[k]) then, per enabled method, n =
// randint(0, beta) accumulating random_apply steps from the base state;
// emit(k, state) runs on the generating thread.
template <typename Emit>
static int generate(fo_graph *g, const State &base, const Engine &eng, const uint64_t *seeds, int32_t K, int32_t beta,
                    int32_t methods_mask, int32_t n_threads, Emit emit) {
    if (n_threads <= 0) n_threads = omp_get_max_threads();
    Inc inc0;
    const bool full = use_full_engine() || !inc0.build(g, base, eng.VB);
    static std::atomic<uint64_t> calls{0};
    const uint64_t epoch = ++calls;
#pragma omp parallel for num_threads(n_threads) schedule(dynamic, 1)
    for (int k = 0; k < K; k++) {
        PyRng rng(seeds[k]);
        if (full) {
            thread_local Scratch sc;
            State s = base;
            for (int m = 0; m < 3; m++) {
                if (!(methods_mask & (1 << m))) continue;
                int n = (int)rng.below((uint32_t)beta + 1);
                eng.random_apply(s, m, n, rng, sc);
            }
            emit(k, s.ng.data(), s.rg.data(), s.bk.data());
            continue;
        }
        // one copy of the base index per thread and call; candidates roll back
        thread_local Inc w;
        thread_local uint64_t w_epoch = 0;
        if (w_epoch != epoch) {
            w = inc0;
            w_epoch = epoch;
        }
        w.checkpoint();
        for (int m = 0; m < 3; m++) {
            if (!(methods_mask & (1 << m))) continue;
            int n = (int)rng.below((uint32_t)beta + 1);
            w.random_apply(m, n, rng);
        }
        emit(k, w.ng.data(), w.rg.data(), w.bk.data());
        if (!w.undo()) w = inc0;
    }
    return FO_OK;
}
}  // extern "C++"

int fo_make_candidates(fo_graph *g, const int32_t *base_ngid, const int32_t *base_rgid, const int32_t *base_bkt,
                       const uint64_t *seeds, int32_t K, int32_t beta, int32_t methods_mask, int32_t n_threads,
                       int32_t *ngid_out, int32_t *rgid_out, int32_t *bkt_out, int32_t *gid_bound_out) {
    if (!g || !seeds || K < 0 || beta < 0) return fail(FO_INVALID_ARG, "bad arguments");
    Engine eng(g);
    State base;
    if (!eng.load_state(base_ngid, base_rgid, base_bkt, base)) return fail(FO_INVALID_ARG, "bad base state");
    const int V = g->V, A = g->A;
    generate(g, base, eng, seeds, K, beta, methods_mask, n_threads,
             [&](int k, const int32_t *ng, const int32_t *rg, const int32_t *bk) {
                 std::copy(ng, ng + V, ngid_out + (int64_t)k * V);
                 std::copy(rg, rg + V, rgid_out + (int64_t)k * V);
                 std::copy(bk, bk + A, bkt_out + (int64_t)k * A);
             });
    if (gid_bound_out) *gid_bound_out = eng.VB;
    return FO_OK;
}

// Sparse form: changes of each candidate against the (id-ranked) base state as
// (index, value) pairs over ngid | rgid | bkt -- the fo_score_delta input.
int fo_make_candidates_delta(fo_graph *g, const int32_t *base_ngid, const int32_t *base_rgid, const int32_t *base_bkt,
                             const uint64_t *seeds, int32_t K, int32_t beta, int32_t methods_mask, int32_t n_threads,
                             int32_t *offsets_out, int32_t *changes_out, int64_t cap_pairs) {
    if (!g || !seeds || K < 0 || beta < 0 || !offsets_out) return fail(FO_INVALID_ARG, "bad arguments");
    Engine eng(g);
    State base;
    if (!eng.load_state(base_ngid, base_rgid, base_bkt, base)) return fail(FO_INVALID_ARG, "bad base state");
    const int V = g->V, A = g->A;
    std::vector<std::vector<int32_t>> per(K);
    generate(g, base, eng, seeds, K, beta, methods_mask, n_threads,
             [&](int k, const int32_t *ng, const int32_t *rg, const int32_t *bk) {
                 auto &d = per[k];
                 d.clear();
                 for (int v = 0; v < V; v++)
                     if (ng[v] != base.ng[v]) { d.push_back(v); d.push_back(ng[v]); }
                 for (int v = 0; v < V; v++)
                     if (rg[v] != base.rg[v]) { d.push_back(V + v); d.push_back(rg[v]); }
                 for (int a = 0; a < A; a++)
                     if (bk[a] != base.bk[a]) { d.push_back(2 * V + a); d.push_back(bk[a]); }
             });
    int64_t n = 0;
    offsets_out[0] = 0;
    for (int k = 0; k < K; k++) {
        n += (int64_t)per[k].size() / 2;
        if (n > INT32_MAX) return fail(FO_INVALID_ARG, "too many changes");
        offsets_out[k + 1] = (int32_t)n;
    }
    if (n > cap_pairs || (n > 0 && !changes_out)) return fail(FO_INVALID_ARG, "changes capacity too small");
    for (int k = 0; k < K; k++) std::copy(per[k].begin(), per[k].end(), changes_out + 2 * (int64_t)offsets_out[k]);
    return FO_OK;
}

// Resident parent of sparse candidates: ids ranked like the engine's base state.
int fo_set_parent(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    Engine eng(g);
    State s;
    if (!eng.load_state(ngid, rgid, bkt, s)) return fail(FO_INVALID_ARG, "bad parent state");
    const int V = g->V, A = g->A;
    g->h_parent.resize(2 * (size_t)V + A);
    std::copy(s.ng.begin(), s.ng.end(), g->h_parent.begin());
    std::copy(s.rg.begin(), s.rg.end(), g->h_parent.begin() + V);
    std::copy(s.bk.begin(), s.bk.end(), g->h_parent.begin() + 2 * V);
    g->parent_ver++;  // invalidates the incremental plans (capi.cu ensure_plan)
    if (g->device < 0) return FO_OK;
    if (cudaSetDevice(g->device) != cudaSuccess) return fail(FO_CUDA_ERROR, "cudaSetDevice");
    if (!g->d_parent && cudaMalloc(&g->d_parent, 4 * g->h_parent.size() + 4) != cudaSuccess)
        return fail(FO_CUDA_ERROR, "parent alloc");
    if (cudaMemcpyAsync(g->d_parent, g->h_parent.data(), 4 * g->h_parent.size(), cudaMemcpyHostToDevice, g->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(g->stream) != cudaSuccess)
        return fail(FO_CUDA_ERROR, "parent upload");
    return FO_OK;
}

int fo_random_apply(fo_graph *g, int32_t *ngid, int32_t *rgid, int32_t *bkt, int32_t method, int32_t n,
                    uint32_t *mt_state, int32_t *applied_out) {
    if (!g || !ngid || !rgid || !bkt || !mt_state || method < 0 || method > 2 || n < 0)
        return fail(FO_INVALID_ARG, "bad arguments");
    Engine eng(g);
    State s;
    if (!eng.load_state(ngid, rgid, bkt, s)) return fail(FO_INVALID_ARG, "bad state");
    PyRng rng(0);
    std::copy(mt_state, mt_state + 624, rng.mt);
    rng.mti = (int)mt_state[624];
    bool applied;
    Inc w;
    if (use_full_engine() || !w.build(g, s, eng.VB)) {
        Scratch sc;
        applied = eng.random_apply(s, method, n, rng, sc);
    } else {
        applied = w.random_apply(method, n, rng);
        w.to_state(s);
    }
    std::copy(rng.mt, rng.mt + 624, mt_state);
    mt_state[624] = (uint32_t)rng.mti;
    std::copy(s.ng.begin(), s.ng.end(), ngid);
    std::copy(s.rg.begin(), s.rg.end(), rgid);
    std::copy(s.bk.begin(), s.bk.end(), bkt);
    if (applied_out) *applied_out = applied ? 1 : 0;
    return FO_OK;
}

int fo_expand_all(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t cap,
                  int32_t *ngid_out, int32_t *rgid_out, int32_t *bkt_out, int32_t *n_out) {
    if (!g || !n_out) return fail(FO_INVALID_ARG, "bad arguments");
    Engine eng(g);
    State s;
    if (!eng.load_state(ngid, rgid, bkt, s)) return fail(FO_INVALID_ARG, "bad state");
    Scratch sc;
    Index ix;
    eng.build(s, ix, sc);
    std::vector<State> out;
    State cand;
    // exhaustive_search's per-graph enumeration (search.py:185-206)
    std::vector<std::pair<int32_t, int32_t>> fp, bp;
    eng.fusible_pairs(ix, false, fp);
    for (auto pr : fp) {
        int x = pr.first, y = pr.second;
        if (eng.fuse_ops(s, ix, x, y, false, cand, sc)) out.push_back(cand);
        bool other = ix.feeds_ar[y];
        for (int k = ix.sptr[y]; k < ix.sptr[y + 1]; k++) other |= ix.succ[k] != x;
        if (other && !ix.has_rep[y] && eng.fuse_ops(s, ix, x, y, true, cand, sc)) out.push_back(cand);
    }
    eng.bucket_pairs(ix, sc, bp);
    for (auto pr : bp)
        if (eng.fuse_ar(s, ix, pr.first, pr.second, cand, sc)) out.push_back(cand);
    *n_out = (int32_t)out.size();
    if ((int)out.size() > cap) return fail(FO_INVALID_ARG, "output capacity too small");
    const int V = g->V, A = g->A;
    for (size_t k = 0; k < out.size(); k++) {
        std::copy(out[k].ng.begin(), out[k].ng.end(), ngid_out + k * V);
        std::copy(out[k].rg.begin(), out[k].rg.end(), rgid_out + k * V);
        std::copy(out[k].bk.begin(), out[k].bk.end(), bkt_out + k * A);
    }
    return FO_OK;
}

// Rewrite primitives on one state (rewrite.py:49-219), ids as ranks of the
// state's group / bucket ids.  kind 0: fusible_pairs, 1: the same with the
// duplicate-fusion filter (rewrite.py:242-247), 2: bucket_pairs, 3: every
// contracted (group, predecessor) pair.
int fo_rewrite_pairs(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t kind,
                     int32_t *pairs_out, int32_t cap, int32_t *n_out) {
    if (!g || !n_out || kind < 0 || kind > 3) return fail(FO_INVALID_ARG, "bad arguments");
    Engine eng(g);
    State s;
    if (!eng.load_state(ngid, rgid, bkt, s)) return fail(FO_INVALID_ARG, "bad state");
    Scratch sc;
    Index ix;
    eng.build(s, ix, sc, kind == 2);
    std::vector<std::pair<int32_t, int32_t>> v;
    if (kind == 2) eng.bucket_pairs(ix, sc, v);
    else if (kind == 3)  // every (group, contracted predecessor) pair (graph.py:161-179)
        for (int x = 0; x < ix.G; x++)
            for (int k = ix.pptr[x]; k < ix.pptr[x + 1]; k++) v.emplace_back(x, ix.pred[k]);
    else eng.fusible_pairs(ix, kind == 1, v);
    *n_out = (int32_t)v.size();
    if ((int64_t)v.size() > cap) return fail(FO_INVALID_ARG, "pair capacity too small");
    for (size_t i = 0; i < v.size(); i++) {
        pairs_out[2 * i] = v[i].first;
        pairs_out[2 * i + 1] = v[i].second;
    }
    return FO_OK;
}

// fuse_nondup / fuse_dup (a = consumer group, b = predecessor group) or
// fuse_allreduce (a = bucket, b = neighbour; the caller checks adjacency,
// rewrite.py:185-186); the state is rewritten in place when applied.
int fo_rewrite_apply(fo_graph *g, int32_t *ngid, int32_t *rgid, int32_t *bkt, int32_t method, int32_t a, int32_t b,
                     int32_t *applied_out) {
    if (!g || !ngid || !rgid || !bkt || !applied_out || method < 0 || method > 2)
        return fail(FO_INVALID_ARG, "bad arguments");
    Engine eng(g);
    State s, out;
    if (!eng.load_state(ngid, rgid, bkt, s)) return fail(FO_INVALID_ARG, "bad state");
    Scratch sc;
    Index ix;
    eng.build(s, ix, sc, method == M_AR);
    const int n = method == M_AR ? ix.B : ix.G;
    if (a < 0 || a >= n || b < 0 || b >= n) return fail(FO_INVALID_ARG, "unknown group or bucket");
    bool ok = false;
    if (method == M_AR) {
        ok = a != b && eng.fuse_ar(s, ix, a, b, out, sc);
    } else {
        bool adjacent = false;  // pred_gid in contracted_preds[op_gid] (rewrite.py:72-73)
        for (int k = ix.pptr[a]; k < ix.pptr[a + 1]; k++) adjacent |= ix.pred[k] == b;
        ok = adjacent && eng.fuse_ops(s, ix, a, b, method == M_DUP, out, sc);
    }
    *applied_out = ok ? 1 : 0;
    if (ok) {
        std::copy(out.ng.begin(), out.ng.end(), ngid);
        std::copy(out.rg.begin(), out.rg.end(), rgid);
        std::copy(out.bk.begin(), out.bk.end(), bkt);
    }
    return FO_OK;
}

// greedy_postorder_fusion (search.py:228-244): ops in reverse topological
// order; each op's current normal group is non-duplicate-fused with its first
// predecessor group (ascending id) for which the rewrite is valid.
int fo_greedy_postorder(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt,
                        int32_t *ngid_out, int32_t *rgid_out, int32_t *bkt_out) {
    if (!g || !ngid_out || !rgid_out || !bkt_out) return fail(FO_INVALID_ARG, "bad arguments");
    Engine eng(g);
    State s, cand;
    if (!eng.load_state(ngid, rgid, bkt, s)) return fail(FO_INVALID_ARG, "bad state");
    Scratch sc;
    Index ix;
    eng.build(s, ix, sc, false);
    std::vector<int32_t> topo, ops;
    if (!eng.topo_groups(ix, topo)) return fail(FO_CYCLE, "contracted group graph is cyclic");
    for (int x : topo)
        for (int k = ix.mptr[x]; k < ix.mptr[x + 1]; k++) ops.push_back(ix.mem[k]);
    for (size_t i = ops.size(); i-- > 0;) {
        const int x = ix.nn[ops[i]];
        for (int k = ix.pptr[x]; k < ix.pptr[x + 1]; k++) {
            if (eng.fuse_ops(s, ix, x, ix.pred[k], false, cand, sc)) {
                std::swap(s, cand);
                eng.build(s, ix, sc, false);
                break;
            }
        }
    }
    std::copy(s.ng.begin(), s.ng.end(), ngid_out);
    std::copy(s.rg.begin(), s.rg.end(), rgid_out);
    std::copy(s.bk.begin(), s.bk.end(), bkt_out);
    return FO_OK;
}

// topo_order (graph.py:536-556): group ids in the deterministic topological
// order of the contracted group graph
int fo_topo_order(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t *gid_out,
                  int32_t *n_out) {
    if (!g || !gid_out || !n_out) return fail(FO_INVALID_ARG, "bad arguments");
    Engine eng(g);
    State s;
    if (!eng.load_state(ngid, rgid, bkt, s)) return fail(FO_INVALID_ARG, "bad state");
    Scratch sc;
    Index ix;
    eng.build(s, ix, sc, false);
    std::vector<int32_t> topo;
    if (!eng.topo_groups(ix, topo)) return fail(FO_CYCLE, "contracted group graph is cyclic");
    for (size_t i = 0; i < topo.size(); i++) gid_out[i] = ix.gid[topo[i]];
    *n_out = (int32_t)topo.size();
    return FO_OK;
}

// threshold_allreduce_fusion (search.py:247-302): buckets in production order
// (order[] = bucket ids by simulated start; NULL: contracted topological
// production order), consecutive neighbours merged while the merged size stays
// within threshold_bytes.
int fo_threshold_ar(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int64_t threshold_bytes,
                    const int32_t *order, int32_t n_order, int32_t *ngid_out, int32_t *rgid_out, int32_t *bkt_out) {
    if (!g || !ngid_out || !rgid_out || !bkt_out) return fail(FO_INVALID_ARG, "bad arguments");
    if (threshold_bytes <= 0) return fail(FO_INVALID_ARG, "threshold must be > 0");
    Engine eng(g);
    State s, cand;
    if (!eng.load_state(ngid, rgid, bkt, s)) return fail(FO_INVALID_ARG, "bad state");
    Scratch sc;
    Index ix;
    eng.build(s, ix, sc, true);
    const int A = g->A;
    std::vector<int32_t> ord;
    if (order) {
        if (n_order != ix.B) return fail(FO_INVALID_ARG, "order must list every bucket once");
        std::vector<uint8_t> seen(A, 0);
        for (int i = 0; i < n_order; i++) {
            int b = order[i];
            if (b < 0 || b >= A || seen[b] || !std::binary_search(ix.bid.begin(), ix.bid.end(), b))
                return fail(FO_INVALID_ARG, "order must list every bucket once");
            seen[b] = 1;
            ord.push_back(b);
        }
    } else {  // production key (max topo position of member producers' export groups, min member)
        std::vector<int32_t> topo, pos(ix.G);
        if (!eng.topo_groups(ix, topo)) return fail(FO_CYCLE, "contracted group graph is cyclic");
        for (int i = 0; i < ix.G; i++) pos[topo[i]] = i;
        std::vector<std::pair<std::pair<int32_t, int32_t>, int32_t>> key(ix.B, {{-1, INT32_MAX}, 0});
        for (int a = 0; a < A; a++) {
            const int b = ix.bki[a], pv = g->ar_prod[a];
            const int ex = ix.rr[pv] >= 0 ? ix.rr[pv] : ix.nn[pv];
            key[b].first.first = std::max(key[b].first.first, pos[ex]);
            key[b].first.second = std::min(key[b].first.second, a);
            key[b].second = ix.bid[b];
        }
        std::sort(key.begin(), key.end());
        for (auto &k : key) ord.push_back(k.second);
    }
    std::vector<int64_t> tot(A, 0);
    for (int a = 0; a < A; a++) tot[s.bk[a]] += g->ar_bytes[a];
    std::vector<int32_t> alias(A);
    for (int b : ord) alias[b] = b;
    auto dense = [&](int b) { return (int)(std::lower_bound(ix.bid.begin(), ix.bid.end(), b) - ix.bid.begin()); };
    int acc = -1;
    for (int b : ord) {
        const int live = alias[b];
        if (acc < 0) {
            acc = live;
            continue;
        }
        if (tot[acc] + tot[live] <= threshold_bytes && eng.bucket_neighbor(ix, sc, dense(acc), dense(live)) &&
            eng.fuse_ar(s, ix, dense(acc), dense(live), cand, sc)) {
            std::swap(s, cand);
            eng.build(s, ix, sc, true);
            const int merged = std::min(acc, live);
            const int64_t t = tot[acc] + tot[live];
            for (int k : ord)
                if (alias[k] == acc || alias[k] == live) alias[k] = merged;
            tot[merged] = t;
            acc = merged;
            continue;
        }
        acc = live;
    }
    std::copy(s.ng.begin(), s.ng.end(), ngid_out);
    std::copy(s.rg.begin(), s.rg.end(), rgid_out);
    std::copy(s.bk.begin(), s.bk.end(), bkt_out);
    return FO_OK;
}

int fo_state_hash(fo_graph *g, const int32_t *ngid, const int32_t *rgid, const int32_t *bkt, int32_t K,
                  uint64_t *hash_out) {
    if (!g) return fail(FO_INVALID_ARG, "null graph");
    Engine eng(g);
    for (int k = 0; k < K; k++) {
        State s;
        if (!eng.load_state(ngid + (int64_t)k * g->V, rgid + (int64_t)k * g->V, bkt + (int64_t)k * g->A, s))
            return fail(FO_INVALID_ARG, "bad state");
        hash_out[k] = eng.hash(s);
    }
    return FO_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// lock-stepped backtracking search (search.py:84-155)

struct fo_search {
    fo_graph *g = nullptr;
    fo_search_cfg cfg{};
    Engine *eng = nullptr;
    struct QE {
        double c;
        int64_t seq;
        uint64_t h;
        int32_t slot;
        bool operator>(const QE &o) const { return c != o.c ? c > o.c : seq > o.seq; }
    };
    struct Seed {
        PyRng rng{0};
        std::vector<State> pool;
        std::priority_queue<QE, std::vector<QE>, std::greater<QE>> queue;
        std::unordered_set<uint64_t> seen;
        std::unordered_map<uint64_t, double> cache;
        int64_t seq = 1, steps = 0, evaluated = 0, enqueued = 0;
        int unchanged = 0;
        double best = 0.0;
        int32_t best_slot = 0;
        bool active = true;
        int status = FO_OK;
        std::vector<fo_trace_rec> trace;
        // per-step scratch
        QE cur{};
        int ncand = 0;
        State cand[3];
        int meth[3];
        uint64_t h[3];
        int64_t batch_pos[3];
        Scratch sc;
        Inc inc0;  // incremental index of the popped state (methods roll back)
        // speculation (one step ahead): costs of the candidates of every state
        // the next step may pop, scored in the same device batch.  They enter
        // the reference-visible cache only when that step really evaluates them.
        std::unordered_map<uint64_t, std::pair<double, int32_t>> spec;
        int nbr = 0;
        State br_cand[4][3];
        uint64_t br_h[4][3];
        int br_n[4];
        int64_t br_pos[4][3];
        const State *br_state[4];
        uint64_t br_hs[4];
        // the branch expansions stay valid for the next pop: the seed's rng
        // does not move between them, so a pop of branch q's exact state
        // reuses its candidates and post-expansion rng instead of expanding again
        int br_avail = 0;
        State br_src[4];
        PyRng br_rng[4]{PyRng(0), PyRng(0), PyRng(0), PyRng(0)};
        int br_meth[4][3];
    };
    // one in-flight device batch: pinned staging, device buffers, results
    struct Lane {
        int32_t *h_buf = nullptr;
        size_t h_cap = 0;
        char *d_buf = nullptr;
        size_t d_cap = 0;
        double *h_cost = nullptr;
        int32_t *h_status = nullptr;
        size_t hc_cap = 0;
        int n = 0;
        cudaEvent_t done = nullptr, e0 = nullptr, e1 = nullptr;
        cudaStream_t stream = nullptr;  // lane 1: its own stream and workspace (concurrent halves)
        int alt = 0;
    };
    std::vector<Seed> seeds;
    Lane lanes[2];
    double device_ms = 0, expand_ms = 0;
    double launch_ms = 0, wait_ms = 0, replay_ms = 0;  // host-side split (FO_SEARCH_PROFILE)
    double put_ms = 0, issue_ms = 0;
    int64_t scored = 0, host_steps = 0;
    int64_t rounds = 0;  // device rounds run (fo_search_rounds)
    bool started = false;
    fo_xchg *x = nullptr;      // the multi-GPU exchange (fo_xchg_attach)
    int64_t x_round = 0;
    fo_round_fn cb = nullptr;  // per-round hook of fo_search_run_cb
    void *cb_ctx = nullptr;
    int64_t cb_round = 0;
    bool cb_stop = false;
    std::vector<double> cb_best;
    bool spec = false;  // one-step speculation (latency-bound rounds: few seeds)
    int spec_at = -1;   // switch speculation on once this few seeds are active (-1: never)
};

static int lane_reserve(fo_search *S, fo_search::Lane &L, int n) {
    const size_t W = 2 * (size_t)S->g->V + S->g->A;
    if ((size_t)n * W > L.h_cap) {
        if (L.h_buf) cudaFreeHost(L.h_buf);
        L.h_buf = nullptr;
        size_t cap = std::max((size_t)n * W, L.h_cap * 2);
        if (cudaMallocHost(&L.h_buf, cap * 4) != cudaSuccess) return fail(FO_CUDA_ERROR, "pinned alloc");
        L.h_cap = cap;
    }
    if ((size_t)n > L.hc_cap) {
        if (L.h_cost) cudaFreeHost(L.h_cost);
        if (L.h_status) cudaFreeHost(L.h_status);
        size_t cap = std::max((size_t)n, L.hc_cap * 2);
        if (cudaMallocHost(&L.h_cost, cap * 8) != cudaSuccess || cudaMallocHost(&L.h_status, cap * 4) != cudaSuccess)
            return fail(FO_CUDA_ERROR, "pinned alloc");
        L.hc_cap = cap;
    }
    size_t need = ((W * n * 4 + 255) & ~size_t(255)) + 16 * (size_t)n + 256;
    if (need > L.d_cap) {  // geometric: cudaFree synchronises the device
        if (L.d_buf) cudaFree(L.d_buf);
        L.d_buf = nullptr;
        need = std::max(need, 2 * L.d_cap);
        if (cudaMalloc(&L.d_buf, need) != cudaSuccess) return fail(FO_CUDA_ERROR, "search batch alloc");
        L.d_cap = need;
    }
    if (!L.done) {
        cudaEventCreateWithFlags(&L.done, cudaEventDisableTiming);
        cudaEventCreate(&L.e0);
        cudaEventCreate(&L.e1);
    }
    return FO_OK;
}

// bytes per id in the staged batch: int16 whenever the ids fit (half the H2D)
static size_t id_bytes(const fo_search *S) { return (S->eng->VB <= 32767 && S->g->A <= 32767) ? 2 : 4; }

// write candidate j of an n-candidate batch (SoA [ng * n | rg * n | bk * n])
static void lane_put(fo_search *S, fo_search::Lane &L, int n, int j, const State &s) {
    const int V = S->g->V, A = S->g->A;
    if (id_bytes(S) == 2) {
        int16_t *b = (int16_t *)L.h_buf;
        std::copy(s.ng.begin(), s.ng.end(), b + (size_t)j * V);
        std::copy(s.rg.begin(), s.rg.end(), b + (size_t)V * n + (size_t)j * V);
        std::copy(s.bk.begin(), s.bk.end(), b + (size_t)2 * V * n + (size_t)j * A);
        return;
    }
    std::copy(s.ng.begin(), s.ng.end(), L.h_buf + (size_t)j * V);
    std::copy(s.rg.begin(), s.rg.end(), L.h_buf + (size_t)V * n + (size_t)j * V);
    std::copy(s.bk.begin(), s.bk.end(), L.h_buf + (size_t)2 * V * n + (size_t)j * A);
}

// H2D, score, D2H on the handle's stream; asynchronous until lane_wait
static int lane_launch(fo_search *S, fo_search::Lane &L, int n) {
    fo_graph *g = S->g;
    const int V = g->V, A = g->A;
    const size_t W = 2 * (size_t)V + A;
    L.n = n;
    if (n == 0) return FO_OK;
    char *db = L.d_buf;
    const size_t eb = id_bytes(S);
    size_t cost_off = (W * n * eb + 255) & ~size_t(255);
    const char *dn = db, *dr = dn + (size_t)V * n * eb, *dk = dr + (size_t)V * n * eb;
    double *dc = (double *)(db + cost_off);
    int32_t *ds = (int32_t *)(dc + n);
    cudaStream_t st = L.stream ? L.stream : g->stream;
    if (cudaMemcpyAsync(db, L.h_buf, W * n * eb, cudaMemcpyHostToDevice, st) != cudaSuccess)
        return fail(FO_CUDA_ERROR, "search batch H2D");
    cudaEventRecord(L.e0, st);
    int rc = score_device(g, dn, dr, dk, eb == 2, n, S->eng->VB, S->cfg.precision, dc, ds, st, L.alt);
    if (rc) return rc;
    cudaEventRecord(L.e1, st);
    cudaMemcpyAsync(L.h_cost, dc, 8 * (size_t)n, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(L.h_status, ds, 4 * (size_t)n, cudaMemcpyDeviceToHost, st);
    cudaEventRecord(L.done, st);
    return FO_OK;
}

static int lane_wait(fo_search *S, fo_search::Lane &L) {
    if (L.n == 0) return FO_OK;
    if (cudaEventSynchronize(L.done) != cudaSuccess) return fail(FO_CUDA_ERROR, "search batch sync");
    float ms = 0;
    cudaEventElapsedTime(&ms, L.e0, L.e1);
    S->device_ms += ms;
    S->scored += L.n;
    return FO_OK;
}

// eval_cost(g0) once per seed (search.py:101-102); the same state -> one score
static int search_start(fo_search *S) {
    if (S->started) return FO_OK;
    auto &L = S->lanes[0];
    int rc = lane_reserve(S, L, 1);
    if (rc) return rc;
    lane_put(S, L, 1, 0, S->seeds[0].pool[0]);
    if ((rc = lane_launch(S, L, 1)) || (rc = lane_wait(S, L))) return rc;
    for (auto &sd : S->seeds) {
        sd.status = L.h_status[0];
        if (L.h_status[0]) { sd.active = false; continue; }
        sd.best = L.h_cost[0];
        sd.evaluated = 1;
        sd.cache[sd.cur.h] = L.h_cost[0];
        sd.queue.push({L.h_cost[0], 0, sd.cur.h, 0});
    }
    S->started = true;
    return FO_OK;
}

// one Alg. 1 step's batch-expand from state H (search.py:112-119): for each
// enabled method, n = randint(0, beta) rewrites from H (rewrite.py:222-263)
static void expand_step(const fo_search *S, const State &H, uint64_t hH, PyRng &rng, Inc &inc, Scratch &sc,
                        State *cand, int *meth, uint64_t *h, int &ncand) {
    const Engine &eng = *S->eng;
    bool built = false, inc_ok = !use_full_engine();
    ncand = 0;
    for (int m = 0; m < 3; m++) {
        if (!(S->cfg.methods_mask & (1 << m))) continue;
        int n = (int)rng.below((uint32_t)S->cfg.beta + 1);
        int j = ncand++;
        bool applied = false;
        if (inc_ok && n > 0 && !built) {  // one index of the popped state serves all methods
            inc_ok = inc.build(S->g, H, eng.VB);
            built = true;
        }
        if (inc_ok && n > 0) {
            inc.checkpoint();
            applied = inc.random_apply(m, n, rng);
            if (applied) inc.to_state(cand[j]);
            else cand[j] = H;
            if (!inc.undo()) inc.build(S->g, H, eng.VB);
        } else {
            cand[j] = H;
            applied = eng.random_apply(cand[j], m, n, rng, sc);
        }
        if (meth) meth[j] = m;
        h[j] = applied ? eng.hash(cand[j]) : hH;
    }
}

static bool step_known(const fo_search::Seed &sd) {
    for (int j = 0; j < sd.ncand; j++)
        if (!sd.cache.count(sd.h[j]) && !sd.spec.count(sd.h[j])) return false;
    return true;
}

static void replay_seed(fo_search *S, fo_search::Seed &sd, const fo_search::Lane *L);

// every active seed in [lo, hi) pops and generates its step's candidates.
// With speculation, steps whose candidates were all scored speculatively are
// replayed on the host at once, and the pending step's successors are expanded
// for every state the next pop can return.
static void search_expand(fo_search *S, int lo, int hi) {
    auto t0 = std::chrono::steady_clock::now();
    int nthreads = S->cfg.n_threads > 0 ? S->cfg.n_threads : omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
    for (int r = lo; r < hi; r++) {
        auto &sd = S->seeds[r];
        sd.ncand = 0;
        sd.nbr = 0;
        for (;;) {
            if (!sd.active) break;
            if (sd.queue.empty() || sd.unchanged >= S->cfg.max_unchanged) { sd.active = false; break; }
            sd.cur = sd.queue.top();
            sd.queue.pop();
            sd.steps++;
            int hit = -1;
            for (int q = 0; q < sd.br_avail && hit < 0; q++)
                if (sd.br_hs[q] == sd.cur.h && sd.br_src[q].ng == sd.pool[sd.cur.slot].ng &&
                    sd.br_src[q].rg == sd.pool[sd.cur.slot].rg && sd.br_src[q].bk == sd.pool[sd.cur.slot].bk)
                    hit = q;
            sd.br_avail = 0;
            if (hit >= 0) {
                sd.ncand = sd.br_n[hit];
                for (int j = 0; j < sd.ncand; j++) {
                    sd.cand[j] = sd.br_cand[hit][j];
                    sd.h[j] = sd.br_h[hit][j];
                    sd.meth[j] = sd.br_meth[hit][j];
                }
                sd.rng = sd.br_rng[hit];
            } else {
                expand_step(S, sd.pool[sd.cur.slot], sd.cur.h, sd.rng, sd.inc0, sd.sc, sd.cand, sd.meth, sd.h,
                            sd.ncand);
            }
            if (S->spec && step_known(sd)) {
                replay_seed(S, sd, nullptr);
#pragma omp atomic
                S->host_steps++;
                continue;
            }
            break;
        }
        if (!S->spec || sd.ncand == 0) continue;
        // the next pop is the queue's current top or one of this step's candidates
        int nb = 0;
        auto add = [&](const State *st, uint64_t hs) {
            for (int q = 0; q < nb; q++)
                if (sd.br_hs[q] == hs) return;
            sd.br_state[nb] = st;
            sd.br_hs[nb++] = hs;
        };
        for (int j = 0; j < sd.ncand; j++) add(&sd.cand[j], sd.h[j]);
        if (!sd.queue.empty()) add(&sd.pool[sd.queue.top().slot], sd.queue.top().h);
        sd.nbr = nb;
    }
    if (S->spec) {  // branch expansions, flattened over (seed, branch)
        std::vector<std::pair<int, int>> work;
        for (int r = lo; r < hi; r++)
            for (int q = 0; q < S->seeds[r].nbr; q++) work.emplace_back(r, q);
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
        for (int w = 0; w < (int)work.size(); w++) {
            auto &sd = S->seeds[work[w].first];
            const int q = work[w].second;
            thread_local Inc inc;
            thread_local Scratch sc;
            PyRng rng = sd.rng;  // the next step continues this seed's draws
            expand_step(S, *sd.br_state[q], sd.br_hs[q], rng, inc, sc, sd.br_cand[q], sd.br_meth[q], sd.br_h[q],
                        sd.br_n[q]);
            sd.br_src[q] = *sd.br_state[q];
            sd.br_rng[q] = rng;
        }
        for (int r = lo; r < hi; r++) S->seeds[r].br_avail = S->seeds[r].nbr;
    }
    S->expand_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// batch every uncached candidate of seeds [lo, hi) (dedupe within a step) and launch
static int search_launch(fo_search *S, fo_search::Lane &L, int lo, int hi) {
    int n = 0;
    for (int r = lo; r < hi; r++) {
        auto &sd = S->seeds[r];
        std::unordered_map<uint64_t, int64_t> inb;  // hash -> batch position (this seed)
        for (int j = 0; j < sd.ncand; j++) {
            sd.batch_pos[j] = -1;
            if (sd.cache.count(sd.h[j]) || sd.spec.count(sd.h[j])) continue;
            auto it = inb.find(sd.h[j]);
            if (it != inb.end()) sd.batch_pos[j] = it->second;
            else inb[sd.h[j]] = sd.batch_pos[j] = n++;
        }
        for (int q = 0; q < sd.nbr; q++)
            for (int j = 0; j < sd.br_n[q]; j++) {
                const uint64_t hh = sd.br_h[q][j];
                sd.br_pos[q][j] = -1;
                if (sd.cache.count(hh) || sd.spec.count(hh) || inb.count(hh)) continue;
                inb[hh] = sd.br_pos[q][j] = n++;
            }
    }
    auto t0 = std::chrono::steady_clock::now();
    if (n > 0) {
        int rc = lane_reserve(S, L, n);
        if (rc) return rc;
        const int nthreads = S->cfg.n_threads > 0 ? S->cfg.n_threads : omp_get_max_threads();
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 4) if (hi - lo > 8)
        for (int r = lo; r < hi; r++) {
            auto &sd = S->seeds[r];
            for (int j = 0; j < sd.ncand; j++)  // duplicates write the same state twice
                if (sd.batch_pos[j] >= 0) lane_put(S, L, n, (int)sd.batch_pos[j], sd.cand[j]);
            for (int q = 0; q < sd.nbr; q++)
                for (int j = 0; j < sd.br_n[q]; j++)
                    if (sd.br_pos[q][j] >= 0) lane_put(S, L, n, (int)sd.br_pos[q][j], sd.br_cand[q][j]);
        }
    }
    auto t1 = std::chrono::steady_clock::now();
    int rc = lane_launch(S, L, n);
    auto t2 = std::chrono::steady_clock::now();
    S->put_ms += std::chrono::duration<double, std::milli>(t1 - t0).count();
    S->issue_ms += std::chrono::duration<double, std::milli>(t2 - t1).count();
    return rc;
}

// replay the accept / prune bookkeeping of a seed's pending step in method
// order (search.py:120-146).  Costs come from the cache, the batch, or the
// speculation table -- the last two count as this step's evaluations.
static void replay_seed(fo_search *S, fo_search::Seed &sd, const fo_search::Lane *L) {
    bool requeued = false;
    for (int j = 0; j < sd.ncand; j++) {
        double c;
        auto it = sd.cache.find(sd.h[j]);
        if (it != sd.cache.end()) c = it->second;
        else {
            int32_t st;
            if (L && sd.batch_pos[j] >= 0) {
                const int p = (int)sd.batch_pos[j];
                st = L->h_status[p];
                c = L->h_cost[p];
            } else {
                const auto &e = sd.spec.at(sd.h[j]);
                c = e.first;
                st = e.second;
            }
            if (st) { sd.status = st; sd.active = false; break; }
            sd.cache[sd.h[j]] = c;
            sd.evaluated++;
        }
        int slot = -1;
        if (c < sd.best) {
            sd.best = c;
            sd.pool.push_back(sd.cand[j]);
            slot = (int)sd.pool.size() - 1;
            sd.best_slot = slot;
            sd.unchanged = 0;
        } else sd.unchanged++;
        int entered = 0;
        if (c <= S->cfg.alpha * sd.best) {
            bool push = false;
            if (!sd.seen.count(sd.h[j])) { sd.seen.insert(sd.h[j]); push = true; sd.enqueued++; }
            else if (sd.h[j] == sd.cur.h && !requeued) { push = true; requeued = true; }
            if (push) {
                if (slot < 0) {
                    if (sd.h[j] == sd.cur.h) slot = sd.cur.slot;
                    else { sd.pool.push_back(sd.cand[j]); slot = (int)sd.pool.size() - 1; }
                }
                sd.queue.push({c, sd.seq++, sd.h[j], slot});
                entered = 1;
            }
        }
        sd.trace.push_back({(int32_t)sd.steps, sd.meth[j], c, sd.best, (int32_t)sd.queue.size(), entered});
    }
    sd.ncand = 0;
}

static void search_replay(fo_search *S, fo_search::Lane &L, int lo, int hi) {
    const int nthreads = S->cfg.n_threads > 0 ? S->cfg.n_threads : omp_get_max_threads();
    // seeds are independent: their bookkeeping replays in parallel
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 4) if (hi - lo > 8)
    for (int r = lo; r < hi; r++) {
        auto &sd = S->seeds[r];
        for (int q = 0; q < sd.nbr; q++)  // speculative results first (not yet evaluations)
            for (int j = 0; j < sd.br_n[q]; j++)
                if (sd.br_pos[q][j] >= 0) {
                    const int p = (int)sd.br_pos[q][j];
                    sd.spec.emplace(sd.br_h[q][j], std::make_pair(L.h_cost[p], L.h_status[p]));
                }
        sd.nbr = 0;
        if (sd.ncand) replay_seed(S, sd, &L);
    }
}

static int count_active(fo_search *S, double *best_cost_out) {
    int active = 0;
    for (size_t r = 0; r < S->seeds.size(); r++) {
        if (S->seeds[r].active) active++;
        if (best_cost_out) best_cost_out[r] = S->seeds[r].best;
    }
    return active;
}

// the per-round hook (fo_search_run_cb); false once it asked to stop
static bool round_hook(fo_search *S) {
    if (!S->cb && !S->x) return true;
    const int R = (int)S->seeds.size();
    S->cb_best.resize(R);
    int active = 0;
    for (int r = 0; r < R; r++) {
        S->cb_best[r] = S->seeds[r].best;
        active += S->seeds[r].active;
    }
    if (S->x && xchg_round(S->x, S->x_round++, S->cb_best.data(), R, active) != FO_OK) S->cb_stop = true;
    if (S->cb && S->cb(S->cb_ctx, S->cb_round++, active, S->cb_best.data(), R) != 0) S->cb_stop = true;
    return !S->cb_stop;
}

extern "C" {

int fo_search_create(fo_graph *g, const fo_search_cfg *cfg, const uint64_t *seeds, int32_t R, const int32_t *ngid0,
                     const int32_t *rgid0, const int32_t *bkt0, fo_search **out) {
    if (!g || !cfg || !seeds || R <= 0 || !out) return fail(FO_INVALID_ARG, "bad arguments");
    if (cfg->alpha < 1 || cfg->beta < 1 || cfg->max_unchanged < 1 || !(cfg->methods_mask & 7))
        return fail(FO_INVALID_ARG, "invalid search config (search.py:53-61)");
    if (!g->model_set) return fail(FO_INVALID_ARG, "no cost model set");
    fo_search *S = new fo_search();
    S->g = g;
    S->cfg = *cfg;
    S->eng = new Engine(g);
    State s0;
    if (!S->eng->load_state(ngid0, rgid0, bkt0, s0)) { delete S->eng; delete S; return fail(FO_INVALID_ARG, "bad start state"); }
    S->seeds.resize(R);
    uint64_t h0 = S->eng->hash(s0);
    for (int r = 0; r < R; r++) {
        auto &sd = S->seeds[r];
        sd.rng = PyRng(seeds[r]);
        sd.pool.push_back(s0);
        sd.seen.insert(h0);
        sd.cur.h = h0;
    }
    // speculation pays while a round is latency-bound (few seeds): each round
    // then advances a seed by two steps.  FO_SEARCH_SPEC=0/1 overrides.
    // Long searches end with a tail of few active seeds, so speculation also
    // switches on when the active count falls to FO_SEARCH_SPEC_AT (default 32).
    const char *sp = getenv("FO_SEARCH_SPEC");
    S->spec = sp ? sp[0] == '1' : R <= 32;
    const char *sa = getenv("FO_SEARCH_SPEC_AT");
    S->spec_at = sp ? -1 : (sa ? atoi(sa) : 32);
    cudaSetDevice(g->device);
    *out = S;
    return FO_OK;
}

// One round: every active search does one step of Alg. 1; all of their
// candidates are scored in ONE device batch.
// eval_cost(g0) for every seed (search.py:101-102) without a step: what a
// search whose time budget is already spent reports
int fo_search_start(fo_search *S, double *best_cost_out) {
    if (!S) return fail(FO_INVALID_ARG, "null search");
    std::lock_guard<std::mutex> lk(S->g->mu);
    cudaSetDevice(S->g->device);
    int rc = search_start(S);
    if (rc) return rc;
    count_active(S, best_cost_out);
    return FO_OK;
}

int fo_search_round(fo_search *S, int32_t *active_out, double *best_cost_out) {
    if (!S) return fail(FO_INVALID_ARG, "null search");
    fo_graph *g = S->g;
    std::lock_guard<std::mutex> lk(g->mu);
    cudaSetDevice(g->device);
    int rc = search_start(S);
    if (rc) return rc;
    const int R = (int)S->seeds.size();
    if (!S->spec && S->spec_at >= 0 && count_active(S, nullptr) <= S->spec_at) S->spec = true;
    search_expand(S, 0, R);
    if ((rc = search_launch(S, S->lanes[0], 0, R)) || (rc = lane_wait(S, S->lanes[0]))) return rc;
    search_replay(S, S->lanes[0], 0, R);
    S->rounds++;
    *active_out = count_active(S, best_cost_out);
    return FO_OK;
}

// Run every search to completion (or max_rounds steps per seed) in native
// code.  With R >= 2 the seeds are split in two halves whose device batches
// alternate with the other half's host-side expand, so host and device
// overlap; each seed's own step sequence is unchanged.
static bool any_active(const fo_search *S, int lo, int hi) {
    for (int r = lo; r < hi; r++)
        if (S->seeds[r].active) return true;
    return false;
}

// up to `limit` rounds (< 0: no limit), one batch in flight; returns rounds run
static int run_single(fo_search *S, int64_t limit, int &rc) {
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const int R = (int)S->seeds.size();
    int64_t it = 0;
    rc = FO_OK;
    for (; (limit < 0 || it < limit) && any_active(S, 0, R); it++) {
        search_expand(S, 0, R);
        const auto t0 = clk::now();
        if ((rc = search_launch(S, S->lanes[0], 0, R))) return (int)it;
        const auto t1 = clk::now();
        if ((rc = lane_wait(S, S->lanes[0]))) return (int)it;
        const auto t2 = clk::now();
        search_replay(S, S->lanes[0], 0, R);
        S->launch_ms += ms(t0, t1);
        S->wait_ms += ms(t1, t2);
        S->replay_ms += ms(t2, clk::now());
        if (!round_hook(S)) return (int)it + 1;
    }
    return (int)it;
}

// seeds split in two halves whose host expand overlaps the other half's device
// batch; up to `limit` rounds, both lanes drained on return
static int run_pipelined(fo_search *S, int64_t limit, int &rc) {
    const int R = (int)S->seeds.size(), mid = R / 2;
    auto &LA = S->lanes[0], &LB = S->lanes[1];
    // the halves' batches are latency-bound: on two streams with two workspaces
    // they run concurrently (not when a second pass would share its scratch)
    if (!LB.stream && S->g->V <= kMpCapDefault) {
        if (cudaStreamCreateWithFlags(&LB.stream, cudaStreamNonBlocking) == cudaSuccess) LB.alt = 1;
        else LB.stream = nullptr;
    }
    bool b_inflight = false;
    int64_t it = 0;
    rc = FO_OK;
    if (!any_active(S, 0, R)) return 0;
    search_expand(S, 0, mid);
    if ((rc = search_launch(S, LA, 0, mid))) return 0;
    using clk = std::chrono::steady_clock;
    auto ms = [](clk::time_point x, clk::time_point y) { return std::chrono::duration<double, std::milli>(y - x).count(); };
    for (; limit < 0 || it < limit; it++) {
        auto t0 = clk::now();
        if (b_inflight) {
            if ((rc = lane_wait(S, LB))) return (int)it;
            search_replay(S, LB, mid, R);
        }
        auto t1 = clk::now();
        S->wait_ms += ms(t0, t1);
        bool b_live = any_active(S, mid, R) && !S->cb_stop;
        if (b_live) {
            search_expand(S, mid, R);  // overlaps A's device batch
            auto t2 = clk::now();
            if ((rc = search_launch(S, LB, mid, R))) return (int)it;
            S->launch_ms += ms(t2, clk::now());
        }
        b_inflight = b_live;
        auto t3 = clk::now();
        if ((rc = lane_wait(S, LA))) return (int)it;
        search_replay(S, LA, 0, mid);
        S->wait_ms += ms(t3, clk::now());
        round_hook(S);  // a round: half A done, half B's in flight
        bool a_live = any_active(S, 0, mid) && !S->cb_stop;
        if (!a_live && !b_inflight) { it++; break; }
        if (a_live && (limit < 0 || it + 1 < limit)) {
            search_expand(S, 0, mid);  // overlaps B's device batch
            auto t4 = clk::now();
            if ((rc = search_launch(S, LA, 0, mid))) return (int)it;
            S->launch_ms += ms(t4, clk::now());
        } else {
            LA.n = 0;
            if (!b_inflight) { it++; break; }
        }
    }
    if (b_inflight) {
        if ((rc = lane_wait(S, LB))) return (int)it;
        search_replay(S, LB, mid, R);
    }
    if ((rc = lane_wait(S, LA))) return (int)it;
    if (LA.n) search_replay(S, LA, 0, mid);
    LA.n = LB.n = 0;
    return (int)it;
}

static int search_run(fo_search *S, int64_t max_rounds, int32_t *active_out);

int fo_search_run(fo_search *S, int64_t max_rounds, int32_t *active_out) {
    if (!S) return fail(FO_INVALID_ARG, "null search");
    S->cb_stop = false;
    const int rc = search_run(S, max_rounds, active_out);
    if (rc) return rc;
    if (S->cb_stop) return FO_CUDA_ERROR;  // the exchange failed (fo_last_error says why)
    return FO_OK;
}

int fo_xchg_attach(fo_search *S, fo_xchg *x, int64_t seed_offset, int32_t every) {
    if (!S || every < 1) return fail(FO_INVALID_ARG, "bad attach arguments");
    S->x = x;
    S->x_round = 0;
    if (x) xchg_attach_cfg(x, seed_offset, every);
    return FO_OK;
}

int fo_search_run_cb(fo_search *S, int64_t max_rounds, fo_round_fn fn, void *ctx, int32_t *active_out) {
    if (!S) return fail(FO_INVALID_ARG, "null search");
    S->cb = fn;
    S->cb_ctx = ctx;
    S->cb_round = 0;
    S->cb_stop = false;
    const int rc = search_run(S, max_rounds, active_out);
    const bool stopped = S->cb_stop;
    S->cb = nullptr;
    S->cb_ctx = nullptr;
    if (rc) return rc;
    return stopped ? fail(FO_INVALID_ARG, "the round callback stopped the search") : FO_OK;
}

static int search_run(fo_search *S, int64_t max_rounds, int32_t *active_out) {
    fo_graph *g = S->g;
    std::lock_guard<std::mutex> lk(g->mu);
    cudaSetDevice(g->device);
    int rc = search_start(S);
    if (rc) return rc;
    const int R = (int)S->seeds.size();
    using clk = std::chrono::steady_clock;
    auto left = [&](int64_t it) { return max_rounds <= 0 ? (int64_t)-1 : std::max<int64_t>(0, max_rounds - it); };
    auto cap = [](int64_t l, int64_t n) { return l < 0 ? n : std::min(l, n); };
    // Probe rounds pick the schedule by measured wall time per round: one batch
    // of all seeds, or two halves whose host expand overlaps the other half's
    // device batch (a half batch is not half the time: search batches are
    // latency-bound).  Speculating drivers (few seeds) keep one batch.
    int64_t it = 0;
    bool pipeline = false;
    if (R > 1 && !S->spec) {
        const int probe = 8;
        auto t0 = clk::now();
        int n1 = run_single(S, cap(left(it), probe), rc);
        if (rc) return rc;
        it += n1;
        const double w1 = std::chrono::duration<double>(clk::now() - t0).count() / std::max(n1, 1);
        t0 = clk::now();
        int n2 = S->cb_stop ? 0 : run_pipelined(S, cap(left(it), probe), rc);
        if (rc) return rc;
        it += n2;
        const double w2 = std::chrono::duration<double>(clk::now() - t0).count() / std::max(n2, 1);
        pipeline = n1 > 0 && n2 > 0 && w2 < w1;
    }
    // the rest in chunks, so speculation can switch on for the tail
    for (;;) {
        const int64_t rest = left(it);
        if (rest == 0 || !any_active(S, 0, R) || S->cb_stop) break;
        if (!S->spec && S->spec_at >= 0 && count_active(S, nullptr) <= S->spec_at) S->spec = true;
        const int64_t chunk = S->spec || S->spec_at < 0 ? rest : cap(rest, 32);
        const int n = pipeline && !S->spec ? run_pipelined(S, chunk, rc) : run_single(S, chunk, rc);
        if (rc) return rc;
        it += n;
        if (n == 0 || S->cb_stop) break;
    }
    S->rounds += it;
    if (active_out) *active_out = count_active(S, nullptr);
    if (S->x) {  // the closing exchanges carry the run's final bests
        std::vector<double> b(S->seeds.size());
        for (size_t r = 0; r < b.size(); r++) b[r] = S->seeds[r].best;
        xchg_final(S->x, b.data(), (int)b.size());
    }
    if (getenv("FO_SEARCH_PROFILE"))
        fprintf(stderr, "fo_search_run: rounds %lld pipeline %d spec %d (host-only steps %lld) device %.1f ms expand %.1f ms launch %.1f ms (put %.1f, issue %.1f) wait %.1f ms replay %.1f ms\n",
                (long long)it, (int)pipeline, (int)S->spec, (long long)S->host_steps, S->device_ms, S->expand_ms,
                S->launch_ms, S->put_ms, S->issue_ms, S->wait_ms, S->replay_ms);
    return FO_OK;
}

int fo_search_result(fo_search *S, int32_t r, double *best_cost, int64_t *counters4, int32_t *best_ngid,
                     int32_t *best_rgid, int32_t *best_bkt, fo_trace_rec *trace, int64_t trace_cap) {
    if (!S || r < 0 || r >= (int)S->seeds.size()) return fail(FO_INVALID_ARG, "bad search index");
    auto &sd = S->seeds[r];
    if (best_cost) *best_cost = sd.best;
    if (counters4) {
        counters4[0] = sd.steps;
        counters4[1] = sd.evaluated;
        counters4[2] = sd.enqueued;
        counters4[3] = (int64_t)sd.trace.size();
    }
    const State &b = sd.pool[sd.best_slot];
    if (best_ngid) std::copy(b.ng.begin(), b.ng.end(), best_ngid);
    if (best_rgid) std::copy(b.rg.begin(), b.rg.end(), best_rgid);
    if (best_bkt) std::copy(b.bk.begin(), b.bk.end(), best_bkt);
    if (trace)
        for (int64_t i = 0; i < (int64_t)sd.trace.size() && i < trace_cap; i++) trace[i] = sd.trace[i];
    return sd.status;
}

int fo_search_timing(fo_search *S, double *device_ms, double *expand_ms, int64_t *scored) {
    if (!S) return fail(FO_INVALID_ARG, "null search");
    if (device_ms) *device_ms = S->device_ms;
    if (expand_ms) *expand_ms = S->expand_ms;
    if (scored) *scored = S->scored;
    return FO_OK;
}

int fo_search_rounds(fo_search *S, int64_t *rounds_out) {
    if (!S || !rounds_out) return fail(FO_INVALID_ARG, "null argument");
    *rounds_out = S->rounds;
    return FO_OK;
}

int fo_search_destroy(fo_search *S) {
    if (!S) return FO_OK;
    for (auto &L : S->lanes) {
        if (L.d_buf) cudaFree(L.d_buf);
        if (L.stream) cudaStreamDestroy(L.stream);
        if (L.h_buf) cudaFreeHost(L.h_buf);
        if (L.h_cost) cudaFreeHost(L.h_cost);
        if (L.h_status) cudaFreeHost(L.h_status);
        if (L.done) cudaEventDestroy(L.done);
        if (L.e0) cudaEventDestroy(L.e0);
        if (L.e1) cudaEventDestroy(L.e1);
    }
    delete S->eng;
    delete S;
    return FO_OK;
}

}  // extern "C"
