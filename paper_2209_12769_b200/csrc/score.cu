// score.cu -- the fused candidate-scoring kernel for sm_100a.
//
// One warp scores one candidate fusion state end to end, persistently looping
// over candidates (candidate k -> warp k mod nwarps):
//
//   K1 pack/contract   group numbering, per-group tie-break keys, bucket sizes
//                      and the contracted schedule DAG as a successor CSR with
//                      multiplicities (graph.py:117-274)                   [warp-parallel]
//   K2 estimate        per fused group: message passing with lane = hidden
//                      channel (estimator.py:321-389), or the analytic /
//                      linear / hardware-oracle closed forms          [warp-parallel]
//   K3 simulate        the two-lane discrete-event loop of simulator.py:53-140
//                      with (rt, tiebreak, id) ready keys            [lane 0, fp64]
//
// fp64 schedule arithmetic (max and +) is bit-exact against the reference;
// the file is compiled with -fmad=false so no multiply-add is contracted
// except the explicit fma() in the message-passing transforms.
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "fo_internal.h"

#include <map>
#include <mutex>

namespace fo {

#define FULL 0xffffffffu
constexpr int kWarps = 4;          // warps per block
constexpr int kRetryLarge = 100;   // internal status: fused group larger than the MP scratch (L.mpcap)

static inline int64_t align8(int64_t x) { return (x + 7) & ~int64_t(7); }

WsLayout ws_layout(int V, int E, int A, int VB, int pairs_max, int mpcap, int nws) {
    WsLayout L{};
    L.mpcap = mpcap;
    int64_t GM = (int64_t)(VB < 2 * V ? VB : 2 * V) + 1;
    int64_t NM = GM + A + 1;
    int64_t cap = V < mpcap ? V : mpcap;
    int64_t o = 0;
    auto take = [&](int64_t bytes) { int64_t r = o; o = align8(o + bytes); return r; };
    L.gmap = take(4 * (int64_t)VB);
    L.bmap = take(4 * (int64_t)A);
    L.g2id = take(4 * GM);
    L.b2id = take(4 * (int64_t)A);
    L.nn = take(4 * (int64_t)V);
    L.rr = take(4 * (int64_t)V);
    L.bki = take(4 * (int64_t)A);
    L.gmin = take(4 * GM);
    L.gcnt = take(4 * GM);
    L.bmin = take(4 * (int64_t)A);
    L.btot = take(8 * (int64_t)A);
    L.indeg = take(4 * NM);
    L.scnt = take(4 * (NM + 1));
    L.sptr = take(4 * (NM + 1));
    L.succ = take(4 * (int64_t)(pairs_max + 1));
    L.prank = take(4 * NM);
    L.dur = take(8 * NM);
    L.fused = take(4 * GM);
    L.gptr = take(4 * (GM + 1));
    L.gmem = take(4 * (2 * (int64_t)V + 1));
    L.gint = take(8 * GM);
    L.gin = take(8 * GM);
    L.gout = take(8 * GM);
    L.vis = take(4 * (int64_t)V);
    L.zl = take(4 * 2 * NM);
    L.rank = take(4 * (2 * (int64_t)V + A + 64));
    L.tlid = take(4 * NM);
    L.csim = take(4 * (NM + 2) * 2 + 8 * (int64_t)(pairs_max + 2) + std::max<int64_t>(24 * (GM + A + 4), 16 * 2 * 256) + 64);
    // per-warp fused-group scratch, one copy per warp of the team
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
    L.gs_stride = align8(q) + 128;
    L.gs0 = take(L.gs_stride * (nws > 0 ? nws : 1));
    L.total = align8(o) + 128;
    return L;
}

// ---------------------------------------------------------------------------
// warp helpers

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Flags (0/1) in arr[0..n) -> ranks; inv[rank] = i.  Returns the count.
__device__ int warp_rank_flags(int *arr, int *inv, int n, int lane) {
    int carry = 0;
    for (int base = 0; base < n; base += 32) {
        int i = base + lane;
        int f = (i < n) ? arr[i] : 0;
        unsigned m = __ballot_sync(FULL, f != 0);
        int r = carry + __popc(m & lanemask_lt());
        if (f) { arr[i] = r; inv[r] = i; }
        carry += __popc(m);
    }
    __syncwarp();
    return carry;
}

// Exclusive scan of in[0..n) into out[0..n]; returns the total.
__device__ int warp_exscan(const int *in, int *out, int n, int lane) {
    int carry = 0;
    for (int base = 0; base < n; base += 32) {
        int i = base + lane;
        int x = (i < n) ? in[i] : 0;
        int v = x;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int y = __shfl_up_sync(FULL, v, d);
            if (lane >= d) v += y;
        }
        if (i < n) out[i] = carry + v - x;
        carry += __shfl_sync(FULL, v, 31);
    }
    if (lane == 0) out[n] = carry;
    __syncwarp();
    return carry;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    return v;
}

// ---------------------------------------------------------------------------
// team primitives: a candidate is scored by a team of TEAM threads -- one warp
// (throughput mode: thousands of candidates in flight) or one 128-thread block
// (latency mode: search-round batches).  TEAM == 32 compiles to warp intrinsics.

struct TeamShm {
    int wsum[32];
    long long wll[32];
    double part[4][32];  // per-warp partial readouts (team MP forward)
    double bcast;
    int flag;
};

template <int TEAM>
__device__ __forceinline__ void tsync() {
    if constexpr (TEAM == 32) __syncwarp();
    else __syncthreads();
}
template <int TEAM>
__device__ __forceinline__ bool tany(bool p) {
    if constexpr (TEAM == 32) return __any_sync(FULL, p);
    else return __syncthreads_or(p) != 0;
}
// exclusive prefix count of a flag over one chunk of TEAM items; total out
template <int TEAM>
__device__ __forceinline__ int tprefix(bool f, int &total, TeamShm *ts, int tid) {
    unsigned m = __ballot_sync(FULL, f);
    int pre = __popc(m & lanemask_lt());
    if constexpr (TEAM == 32) {
        total = __popc(m);
        return pre;
    } else {
        const int wid = tid >> 5;
        if ((tid & 31) == 0) ts->wsum[wid] = __popc(m);
        __syncthreads();
        int off = 0, tot = 0;
#pragma unroll
        for (int i = 0; i < TEAM / 32; i++) {
            int c = ts->wsum[i];
            off += i < wid ? c : 0;
            tot += c;
        }
        __syncthreads();
        total = tot;
        return off + pre;
    }
}
// exclusive prefix sum of x over one chunk of TEAM items; total out
template <int TEAM>
__device__ __forceinline__ int tscan(int x, int &total, TeamShm *ts, int tid) {
    const int lane = tid & 31;
    int v = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int y = __shfl_up_sync(FULL, v, d);
        if (lane >= d) v += y;
    }
    int wtot = __shfl_sync(FULL, v, 31);
    if constexpr (TEAM == 32) {
        total = wtot;
        return v - x;
    } else {
        const int wid = tid >> 5;
        if (lane == 0) ts->wsum[wid] = wtot;
        __syncthreads();
        int off = 0, tot = 0;
#pragma unroll
        for (int i = 0; i < TEAM / 32; i++) {
            int c = ts->wsum[i];
            off += i < wid ? c : 0;
            tot += c;
        }
        __syncthreads();
        total = tot;
        return off + v - x;
    }
}
template <int TEAM>
__device__ __forceinline__ long long tmin(long long v, TeamShm *ts, int tid) {
#pragma unroll
    for (int d = 16; d; d >>= 1) v = min(v, __shfl_xor_sync(FULL, v, d));
    if constexpr (TEAM == 32) {
        return v;
    } else {
        if ((tid & 31) == 0) ts->wll[tid >> 5] = v;
        __syncthreads();
        long long r = ts->wll[0];
#pragma unroll
        for (int i = 1; i < TEAM / 32; i++) r = min(r, ts->wll[i]);
        __syncthreads();
        return r;
    }
}
// flags (0/1) in arr[0..n) -> ranks; inv[rank] = i when inv != nullptr
template <int TEAM>
__device__ int team_rank_flags(int *arr, int *inv, int n, TeamShm *ts, int tid) {
    int carry = 0;
    for (int base = 0; base < n; base += TEAM) {
        int i = base + tid;
        int f = (i < n) ? arr[i] : 0;
        int tot;
        int r = carry + tprefix<TEAM>(f != 0, tot, ts, tid);
        if (f) {
            arr[i] = r;
            if (inv) inv[r] = i;
        }
        carry += tot;
    }
    tsync<TEAM>();
    return carry;
}
// exclusive scan of in[0..n) into out[0..n] (out[n] = total)
template <int TEAM, typename O>
__device__ int team_exscan(const int *in, O *out, int n, TeamShm *ts, int tid) {
    int carry = 0;
    for (int base = 0; base < n; base += TEAM) {
        int i = base + tid;
        int x = (i < n) ? in[i] : 0, tot;
        int e = tscan<TEAM>(x, tot, ts, tid);
        if (i < n) out[i] = (O)(carry + e);
        carry += tot;
    }
    if (tid == 0) out[n] = (O)carry;
    tsync<TEAM>();
    return carry;
}

// CPython 3.12 sum() over floats is Neumaier-compensated (bltinmodule.c
// builtin_sum_impl); the reference sums member times with it
// (estimator.py:186, :442; workloads.py:284).
struct PySum {
    double f = 0.0, c = 0.0;
    int n = 0;
    __device__ __forceinline__ void add(double x) {
        if (n++ == 0) { f = x; return; }
        double t = __dadd_rn(f, x);
        if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
        else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
        f = t;
    }
    __device__ __forceinline__ double get() const { return (c != 0.0 && isfinite(c)) ? __dadd_rn(f, c) : f; }
};

// Group-level estimator memo: the message-passing prediction is
// a pure function of the member set (per-op features, member-internal edges),
// so predictions are cached per graph handle in an open-addressing table keyed
// by two independent 64-bit set hashes.  k1 == 0 empty, 2 pending, odd ready.
__device__ __forceinline__ unsigned long long smix(unsigned long long x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
// commutative hashes of the member set, warp-wide (order independent)
__device__ __forceinline__ void set_hash(const int *mem, int n, int lane, unsigned long long &h1,
                                         unsigned long long &h2) {
    unsigned long long a = 0, b = 0;
    #pragma unroll 4
    for (int i = lane; i < n; i += 32) {
        a += smix((unsigned long long)mem[i] * 2 + 1);
        b += smix(((unsigned long long)mem[i] << 32) ^ 0x5bd1e995ull);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        a += __shfl_xor_sync(FULL, a, d);
        b += __shfl_xor_sync(FULL, b, d);
    }
    h1 = smix(a + (unsigned long long)n) | 1ull;
    h2 = smix(b ^ ((unsigned long long)n * 0xff51afd7ed558ccdull));
}
constexpr int kMemoProbe = 16;
__device__ __forceinline__ bool memo_get(const MemoEnt *t, unsigned mask, unsigned long long h1, unsigned long long h2,
                                         double *v) {
    for (int p = 0; p < kMemoProbe; p++) {
        const MemoEnt *e = &t[(unsigned)(h1 + p) & mask];
        unsigned long long k = *(volatile const unsigned long long *)&e->k1;
        if (k == 0) return false;
        if (k == h1) {
            __threadfence();
            if (*(volatile const unsigned long long *)&e->k2 == h2) {
                *v = *(volatile const double *)&e->v;
                return true;
            }
        }
    }
    return false;
}
__device__ __forceinline__ void memo_put(MemoEnt *t, unsigned mask, unsigned long long h1, unsigned long long h2,
                                         double v) {
    for (int p = 0; p < kMemoProbe; p++) {
        MemoEnt *e = &t[(unsigned)(h1 + p) & mask];
        unsigned long long k = atomicCAS(&e->k1, 0ull, 2ull);
        if (k == 0) {
            e->k2 = h2;
            e->v = v;
            __threadfence();
            atomicExch(&e->k1, h1);
            return;
        }
        if (k == h1) return;  // already present
    }
}

// ---------------------------------------------------------------------------
// Hardware-oracle jitter (workloads.py:254-273): blake2b with an 8-byte
// digest over "{seed}|{content key}", where the key is the members' fragments
// "{op_code}:{input_shape_key}:{compute_us}" in ascending op order joined by
// ';', then "|{internal},{external_in},{external_out}".  One thread streams the
// message through a 128-byte block buffer (RFC 7693).
__device__ __constant__ uint64_t kB2bIv[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                                              0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                                              0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
__device__ __constant__ uint8_t kB2bSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

struct Blake2b64 {
    uint64_t h[8];
    uint64_t m[16];  // current block as little-endian words
    uint64_t t;      // bytes compressed so far
    int n;           // bytes in the current block

    __device__ __forceinline__ static uint64_t rotr(uint64_t x, int r) { return (x >> r) | (x << (64 - r)); }
    __device__ void init() {
        for (int i = 0; i < 8; i++) h[i] = kB2bIv[i];
        h[0] ^= 0x01010000ull ^ 8ull;  // digest_size 8, no key
        for (int i = 0; i < 16; i++) m[i] = 0;
        t = 0;
        n = 0;
    }
    __device__ void compress(bool last) {
        uint64_t v[16];
        for (int i = 0; i < 8; i++) { v[i] = h[i]; v[i + 8] = kB2bIv[i]; }
        v[12] ^= t;
        if (last) v[14] = ~v[14];
        for (int r = 0; r < 12; r++) {
            const uint8_t *sg = kB2bSigma[r];
#define FO_B2B_G(a, b, c, d, x, y)               \
    a = a + b + x; d = rotr(d ^ a, 32);          \
    c = c + d; b = rotr(b ^ c, 24);              \
    a = a + b + y; d = rotr(d ^ a, 16);          \
    c = c + d; b = rotr(b ^ c, 63);
            FO_B2B_G(v[0], v[4], v[8], v[12], m[sg[0]], m[sg[1]]);
            FO_B2B_G(v[1], v[5], v[9], v[13], m[sg[2]], m[sg[3]]);
            FO_B2B_G(v[2], v[6], v[10], v[14], m[sg[4]], m[sg[5]]);
            FO_B2B_G(v[3], v[7], v[11], v[15], m[sg[6]], m[sg[7]]);
            FO_B2B_G(v[0], v[5], v[10], v[15], m[sg[8]], m[sg[9]]);
            FO_B2B_G(v[1], v[6], v[11], v[12], m[sg[10]], m[sg[11]]);
            FO_B2B_G(v[2], v[7], v[8], v[13], m[sg[12]], m[sg[13]]);
            FO_B2B_G(v[3], v[4], v[9], v[14], m[sg[14]], m[sg[15]]);
#undef FO_B2B_G
        }
        for (int i = 0; i < 8; i++) h[i] ^= v[i] ^ v[i + 8];
    }
    __device__ void put(uint8_t c) {
        if (n == 128) {  // a full block is compressed only once more data follows
            t += 128;
            compress(false);
            for (int i = 0; i < 16; i++) m[i] = 0;
            n = 0;
        }
        m[n >> 3] |= (uint64_t)c << (8 * (n & 7));
        n++;
    }
    __device__ void put(const uint8_t *p, int64_t len) {
        for (int64_t i = 0; i < len; i++) put(p[i]);
    }
    __device__ void put_uint(unsigned long long x) {  // decimal, like str(int)
        char d[20];
        int k = 0;
        do { d[k++] = (char)('0' + x % 10); x /= 10; } while (x);
        while (k) put((uint8_t)d[--k]);
    }
    __device__ uint64_t digest() {
        t += n;
        compress(true);
        return h[0];  // the 8-byte digest, read little-endian
    }
};

// 1 + noise * (2u - 1), u = digest / 2^64 (workloads.py:256-264); ops[] ascending
__device__ __noinline__ double hw_jitter(const DGraph &g, const int *ops, int n, long long internal, long long ext_in,
                            long long ext_out) {
    Blake2b64 b;
    b.init();
    b.put(g.kpre, g.kpre_len);
    for (int i = 0; i < n; i++) {
        if (i) b.put((uint8_t)';');
        const int v = ops[i];
        b.put(g.okb + g.oko[v], g.oko[v + 1] - g.oko[v]);
    }
    b.put((uint8_t)'|');
    b.put_uint((unsigned long long)internal);
    b.put((uint8_t)',');
    b.put_uint((unsigned long long)ext_in);
    b.put((uint8_t)',');
    b.put_uint((unsigned long long)ext_out);
    const double u = __dmul_rn(__ull2double_rn(b.digest()), 0x1p-64);
    return __dadd_rn(1.0, __dmul_rn(g.noise, __dsub_rn(__dmul_rn(2.0, u), 1.0)));
}

// Drop dead workspace lines from L2 without writing them back
// (discard.global.L2): the per-warp scratch of ~4,000 resident candidates
// exceeds the 126 MB L2, and write-backs of dead setup arrays were most of
// the kernel's DRAM traffic.  Only whole 128-byte lines inside the range.
__device__ __forceinline__ void l2_discard(const void *p, int64_t bytes, int tid, int nthreads) {
    uintptr_t lo = ((uintptr_t)p + 127) & ~uintptr_t(127);
    uintptr_t hi = ((uintptr_t)p + (uintptr_t)bytes) & ~uintptr_t(127);
    for (uintptr_t a = lo + (uintptr_t)tid * 128; a < hi; a += (uintptr_t)nthreads * 128) {
        size_t ga = __cvta_generic_to_global((const void *)a);
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(ga) : "memory");
    }
}

// numpy logaddexp(0, z) (estimator.py:297-298)
__device__ __forceinline__ double softplus_d(double z) {
    if (z == 0.0) return 0.6931471805599453;
    if (z > 0.0) return __dadd_rn(z, log1p(exp(-z)));
    return log1p(exp(z));
}

// ---------------------------------------------------------------------------
// message-passing forward for one fused group (estimator.py:363-389),
// lane = hidden channel.  mem[0..n) sorted op indices of the members.

template <typename T>
struct MpW;
template <>
struct MpW<float> {
    static __device__ __forceinline__ const float *W(const DGraph &g) { return g.Wf; }
    static __device__ __forceinline__ const float *H0(const DGraph &g) { return g.H0f; }
};
template <>
struct MpW<double> {
    static __device__ __forceinline__ const double *W(const DGraph &g) { return g.Wd; }
    static __device__ __forceinline__ const double *H0(const DGraph &g) { return g.H0d; }
};

template <typename T>
__device__ __forceinline__ T fmaT(T a, T b, T c);
template <>
__device__ __forceinline__ float fmaT<float>(float a, float b, float c) { return __fmaf_rn(a, b, c); }
template <>
__device__ __forceinline__ double fmaT<double>(double a, double b, double c) { return __fma_rn(a, b, c); }

// dense 32x32 transform: out[c] = sum_k x[k] * Wt[k][c]  (x distributed over lanes)
template <typename T>
__device__ __forceinline__ T mat32(const T *__restrict__ Wt, T x, int lane) {
    T acc = T(0);
#pragma unroll 8
    for (int k = 0; k < 32; k++) acc = fmaT<T>(__shfl_sync(FULL, x, k), __ldg(&Wt[k * 32 + lane]), acc);
    return acc;
}

// ---- tensor-core option for the FP32 layer transforms (north star: tensor
// cores only if the result stays within tolerance).  H = relu(P @ W_l^T) as
// m16n8k8 TF32 MMAs: rows = member nodes (16 per tile), 4 n8 tiles of output
// channels, 4 k8 steps.  SPLIT adds the 3xTF32 correction terms (x = hi + lo,
// hi * hi + hi * lo + lo * hi), recovering ~FP32 accuracy.
__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                 "{%0,%1,%2,%3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <bool SPLIT>
__device__ void mma_transform(const float *__restrict__ Wt, const float *P, float *H, int n, int lane) {
    const int gq = lane >> 2, tq = lane & 3;
    for (int m0 = 0; m0 < n; m0 += 16) {
        float acc[4][4] = {};
        const int r0 = m0 + gq, r1 = m0 + gq + 8;
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 8) {
            const float af[4] = {r0 < n ? P[r0 * 32 + k0 + tq] : 0.f, r1 < n ? P[r1 * 32 + k0 + tq] : 0.f,
                                 r0 < n ? P[r0 * 32 + k0 + tq + 4] : 0.f, r1 < n ? P[r1 * 32 + k0 + tq + 4] : 0.f};
            uint32_t ah[4], al[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                ah[i] = to_tf32(af[i]);
                al[i] = to_tf32(af[i] - __uint_as_float(ah[i]));
            }
#pragma unroll
            for (int nt = 0; nt < 4; nt++) {
                const float w0 = __ldg(&Wt[(k0 + tq) * 32 + nt * 8 + gq]), w1 = __ldg(&Wt[(k0 + tq + 4) * 32 + nt * 8 + gq]);
                const uint32_t bh0 = to_tf32(w0), bh1 = to_tf32(w1);
                if (SPLIT) {
                    const uint32_t bl0 = to_tf32(w0 - __uint_as_float(bh0)), bl1 = to_tf32(w1 - __uint_as_float(bh1));
                    mma_tf32(acc[nt], al, bh0, bh1);  // small terms first
                    mma_tf32(acc[nt], ah, bl0, bl1);
                }
                mma_tf32(acc[nt], ah, bh0, bh1);
            }
        }
        __syncwarp();  // every lane has read its P rows before H (which may alias nothing) is written
#pragma unroll
        for (int nt = 0; nt < 4; nt++) {
            const int c = nt * 8 + 2 * tq;
            if (r0 < n) { H[r0 * 32 + c] = fmaxf(acc[nt][0], 0.f); H[r0 * 32 + c + 1] = fmaxf(acc[nt][1], 0.f); }
            if (r1 < n) { H[r1 * 32 + c] = fmaxf(acc[nt][2], 0.f); H[r1 * 32 + c + 1] = fmaxf(acc[nt][3], 0.f); }
        }
    }
}

template <typename T>
__device__ double mp_forward(const DGraph &g, const int *mem, int n, const int *nbptr, const int *nb, T *H, T *P,
                             int lane) {
    const MpLayout ml = mp_layout(g.layers);
    const T *W = MpW<T>::W(g);
    const T *H0 = MpW<T>::H0(g);
    for (int i = 0; i < n; i++) H[i * 32 + lane] = __ldg(&H0[(int64_t)mem[i] * 32 + lane]);
    __syncwarp();
    for (int l = 0; l < g.layers; l++) {
        const T *Wt = W + ml.wl + (int64_t)l * 1024;
        // mean aggregation over {i} U undirected internal neighbours (estimator.py:348-355, :374)
        for (int i = 0; i < n; i++) {
            int b = nbptr[i], e = nbptr[i + 1];
            T acc = H[i * 32 + lane];
            for (int q = b; q < e; q++) acc += H[nb[q] * 32 + lane];
            P[i * 32 + lane] = acc / T(1 + e - b);
        }
        __syncwarp();
        if constexpr (sizeof(T) == 4) {
            if (g.mp_arith) {  // tensor-core option (measured)
                if (g.mp_arith == 2) mma_transform<true>((const float *)Wt, (const float *)P, (float *)H, n, lane);
                else mma_transform<false>((const float *)Wt, (const float *)P, (float *)H, n, lane);
                __syncwarp();
                continue;
            }
        }
        // H = relu(P @ W_l^T) (estimator.py:375-376); two nodes share each weight load
        for (int i = 0; i < n; i += 2) {
            const bool two = i + 1 < n;
            T p0 = P[i * 32 + lane], p1 = two ? P[(i + 1) * 32 + lane] : T(0);
            T a0 = T(0), a1 = T(0);
#pragma unroll 8
            for (int k = 0; k < 32; k++) {
                T wk = __ldg(&Wt[k * 32 + lane]);
                a0 = fmaT<T>(__shfl_sync(FULL, p0, k), wk, a0);
                a1 = fmaT<T>(__shfl_sync(FULL, p1, k), wk, a1);
            }
            H[i * 32 + lane] = a0 > T(0) ? a0 : T(0);
            if (two) H[(i + 1) * 32 + lane] = a1 > T(0) ? a1 : T(0);
        }
        __syncwarp();
    }
    // sum readout + dense head (estimator.py:380-389)
    T s = T(0);
    for (int i = 0; i < n; i++) s += H[i * 32 + lane];
    T r = mat32<T>(W + ml.wr, s, lane);
    r = r > T(0) ? r : T(0);
    T d1 = mat32<T>(W + ml.a1, r, lane) + __ldg(&W[ml.c1 + lane]);
    d1 = d1 > T(0) ? d1 : T(0);
    T d2 = mat32<T>(W + ml.a2, d1, lane) + __ldg(&W[ml.c2 + lane]);
    d2 = d2 > T(0) ? d2 : T(0);
    T z = warp_sum<T>(__ldg(&W[ml.a3 + lane]) * d2) + __ldg(&W[ml.c3]);
    double pred = __dmul_rn(softplus_d((double)z), g.out_scale);
    return pred > 1e-9 ? pred : 1e-9;
}

// ---------------------------------------------------------------------------

// Workspace arrays are base + offset, the offsets read from the __grid_constant__
// launch parameters, so no pointer table occupies registers.
struct Ws {
    char *b;
    const WsLayout *L;
    __device__ __forceinline__ int *gmap() const { return (int *)(b + L->gmap); }
    __device__ __forceinline__ int *bmap() const { return (int *)(b + L->bmap); }
    __device__ __forceinline__ int *g2id() const { return (int *)(b + L->g2id); }
    __device__ __forceinline__ int *b2id() const { return (int *)(b + L->b2id); }
    __device__ __forceinline__ int *nn() const { return (int *)(b + L->nn); }
    __device__ __forceinline__ int *rr() const { return (int *)(b + L->rr); }
    __device__ __forceinline__ int *bki() const { return (int *)(b + L->bki); }
    __device__ __forceinline__ int *gmin() const { return (int *)(b + L->gmin); }
    __device__ __forceinline__ int *gcnt() const { return (int *)(b + L->gcnt); }
    __device__ __forceinline__ int *bmin() const { return (int *)(b + L->bmin); }
    __device__ __forceinline__ long long *btot() const { return (long long *)(b + L->btot); }
    __device__ __forceinline__ int *indeg() const { return (int *)(b + L->indeg); }
    __device__ __forceinline__ int *scnt() const { return (int *)(b + L->scnt); }
    __device__ __forceinline__ int *sptr() const { return (int *)(b + L->sptr); }
    __device__ __forceinline__ int *succ() const { return (int *)(b + L->succ); }
    __device__ __forceinline__ int *prank() const { return (int *)(b + L->prank); }
    __device__ __forceinline__ double *dur() const { return (double *)(b + L->dur); }
    __device__ __forceinline__ int *fused() const { return (int *)(b + L->fused); }
    __device__ __forceinline__ int *gptr() const { return (int *)(b + L->gptr); }
    __device__ __forceinline__ int *gmem() const { return (int *)(b + L->gmem); }
    __device__ __forceinline__ long long *gint() const { return (long long *)(b + L->gint); }
    __device__ __forceinline__ long long *gin() const { return (long long *)(b + L->gin); }
    __device__ __forceinline__ long long *gout() const { return (long long *)(b + L->gout); }
    __device__ __forceinline__ int *vis() const { return (int *)(b + L->vis); }
    __device__ __forceinline__ int *zl() const { return (int *)(b + L->zl); }
    __device__ __forceinline__ int *rank() const { return (int *)(b + L->rank); }
    __device__ __forceinline__ int *tlid() const { return (int *)(b + L->tlid); }
    __device__ __forceinline__ char *csim() const { return (char *)(b + L->csim); }
};

__device__ __forceinline__ Ws ws_at(char *base, const WsLayout &L) { return Ws{base, &L}; }

// one warp's fused-group scratch (team mode keeps one copy per warp)
struct GroupScratch {
    int *msort, *lidx, *zl, *nbptr, *nb, *mark;
    char *H, *P;
};
__device__ __forceinline__ GroupScratch group_scratch(const Ws &w, int wid) {
    const WsLayout &L = *w.L;
    char *b = w.b + L.gs0 + (int64_t)wid * L.gs_stride;
    return GroupScratch{(int *)(b + L.g_msort), (int *)(b + L.g_lidx), (int *)(b + L.g_zl), (int *)(b + L.g_nbptr),
                        (int *)(b + L.g_nb), (int *)(b + L.g_mark), b + L.g_H, b + L.g_P};
}

struct ScoreArgs {
    DGraph g;
    const void *ngid, *rgid, *bkt;  // int32, or int16 when idx16
    const int32_t *dbase, *doff, *dchg;  // sparse candidates (DeltaIn) when dbase != nullptr
    int idx16;
    int retry_only;  // 1: second pass over candidates flagged kRetryLarge; 2: first pass over kRetryGeneral ones
    int stop_after;  // measurement hook (fo_set_phase_stop): 1 = after K1, 2 = after K2, 0 = full
    int K, VB;
    int sm_nodes, sm_pairs, sm_bytes;  // per-warp shared-memory simulation arena
    char *ws;
    WsLayout L;
    double *cost_out;
    int32_t *status_out;
    const double *ext_dur;
    TimelineOut tl;
    double *dur_out;
    int32_t *bad_out;
    int32_t *ngroups_out;
};

__device__ __forceinline__ bool in_grp(const Ws &w, int op, int gn) { return w.nn()[op] == gn || w.rr()[op] == gn; }
__device__ __forceinline__ int export_of(const Ws &w, int op) { return w.rr()[op] >= 0 ? w.rr()[op] : w.nn()[op]; }

// status packed with the failing node so a warp min picks the first node in
// schedule order (simulator.py:62 evaluates durations in node order)
__device__ __forceinline__ long long pack_bad(int node, int code) { return ((long long)node << 8) | code; }

// Ready-set keys: (level, prank, node) packed in a u64 -- level counts the
// distinct completion times so far, so (level, prank) orders exactly like the
// reference's (rt, tiebreak, id) heap entries (simulator.py:63-77, :95-96).
// Keys are pushed in non-decreasing level order, so each lane's ready set is
// an insertion-sorted run [head, tail) of one array: O(1) pops, and a push
// only moves past same-level entries.
constexpr int kKeyNodeBits = 20;
__device__ __forceinline__ unsigned long long make_key(unsigned long long level, unsigned prank, unsigned node) {
    return (level << 40) | ((unsigned long long)prank << kKeyNodeBits) | node;
}
// A ready entry carries everything the loop needs when the node starts and
// completes, loaded when the node is released (off the pop critical path).
struct ReadyEnt {
    unsigned long long key;
    double dur;
    unsigned sb, se;  // successor range
};
__device__ __forceinline__ void ready_push(ReadyEnt *buf, int head, int &tail, const ReadyEnt &x) {
    int i = tail++;
    while (i > head) {
        ReadyEnt p = buf[i - 1];
        if (p.key <= x.key) break;
        buf[i] = p;
        i--;
    }
    buf[i] = x;
}

// successor entry -> (prank, node)
template <typename SE>
__device__ __forceinline__ unsigned se_node(SE e);
template <>
__device__ __forceinline__ unsigned se_node<uint32_t>(uint32_t e) { return e & 0xffffu; }
template <>
__device__ __forceinline__ unsigned se_node<unsigned long long>(unsigned long long e) { return (unsigned)(e & 0xfffffu); }
template <typename SE>
__device__ __forceinline__ unsigned se_prank(SE e);
template <>
__device__ __forceinline__ unsigned se_prank<uint32_t>(uint32_t e) { return e >> 16; }
template <>
__device__ __forceinline__ unsigned se_prank<unsigned long long>(unsigned long long e) { return (unsigned)(e >> 20); }
template <typename SE>
__device__ __forceinline__ SE se_make(unsigned prank, unsigned node);
template <>
__device__ __forceinline__ uint32_t se_make<uint32_t>(unsigned prank, unsigned node) { return (prank << 16) | node; }
template <>
__device__ __forceinline__ unsigned long long se_make<unsigned long long>(unsigned prank, unsigned node) {
    return ((unsigned long long)prank << 20) | node;
}

// hide a pointer's derivation from the compiler, so it stays one register
// pair instead of a base plus a spilled offset re-read at every use
template <typename T>
__device__ __forceinline__ T *opaque_ptr(T *p) {
    asm("mov.b64 %0, %0;" : "+l"(p));
    return p;
}

template <bool TL, typename IT, typename SE>
__device__ __forceinline__ void event_loop(const ScoreArgs &a, int k, const double *__restrict__ dur,
                                           const IT *__restrict__ sptr, IT *__restrict__ indeg_,
                                           const SE *__restrict__ succ_, ReadyEnt *__restrict__ bufg,
                                           ReadyEnt *__restrict__ bufb, const Ws &w, int G, int N, int hg, int hb) {
    IT *__restrict__ indeg = opaque_ptr(indeg_);
    const SE *__restrict__ succ = opaque_ptr(succ_);
    int headg = 0, tailg = hg, headb = 0, tailb = hb;
    int run0 = -1, run1 = -1, done = 0, nc = 0, nb = 0, st = FO_OK;
    unsigned sb0 = 0, se0 = 0, sb1 = 0, se1 = 0;
    double end0 = 0.0, end1 = 0.0, now = 0.0, last = 0.0;
    unsigned long long level = 0;
    for (;;) {
        // start_available (simulator.py:98-115): compute lane, then comm lane;
        // start = max(now, rt) = now because rt is a drained completion time
        if (run0 < 0 && headg < tailg) {
            ReadyEnt x = bufg[headg++];
            run0 = (int)(x.key & ((1u << kKeyNodeBits) - 1));
            end0 = __dadd_rn(now, x.dur);
            sb0 = x.sb;
            se0 = x.se;
            if (TL) { a.tl.c_id[nc] = w.g2id()[run0]; a.tl.c_start[nc] = now; a.tl.c_end[nc] = end0; nc++; }
        }
        if (run1 < 0 && headb < tailb) {
            ReadyEnt x = bufb[headb++];
            run1 = (int)(x.key & ((1u << kKeyNodeBits) - 1));
            end1 = __dadd_rn(now, x.dur);
            sb1 = x.sb;
            se1 = x.se;
            if (TL) { a.tl.b_id[nb] = w.b2id()[run1 - G]; a.tl.b_start[nb] = now; a.tl.b_end[nb] = end1; nb++; }
        }
        if (run0 < 0 && run1 < 0) {
            if (done != N) st = FO_CYCLE;  // simulator.py:133
            break;
        }
        // advance to the next completion and drain every lane ending there
        // (simulator.py:122-132); equal ends share one level
        now = run0 < 0 ? end1 : (run1 < 0 ? end0 : (end0 < end1 ? end0 : end1));
        if (now > last) { last = now; level++; }
#pragma unroll
        for (int t = 0; t < 2; t++) {
            if ((t == 0 ? run0 : run1) < 0 || (t == 0 ? end0 : end1) != now) continue;
            const unsigned qb = t == 0 ? sb0 : sb1, qe = t == 0 ? se0 : se1;
            if (t == 0) run0 = -1; else run1 = -1;
            done++;
            for (unsigned q = qb; q < qe; q++) {  // finish_node (simulator.py:88-96)
                SE e = succ[q];
                unsigned s = se_node<SE>(e);
                // issue the release-time loads together with the indegree load
                IT d = indeg[s] - 1;
                ReadyEnt x;
                x.dur = dur[s];
                x.sb = sptr[s];
                x.se = sptr[s + 1];
                indeg[s] = d;
                if (d == 0) {
                    x.key = make_key(level, se_prank<SE>(e), s);
                    if ((int)s < G) ready_push(bufg, headg, tailg, x);
                    else ready_push(bufb, headb, tailb, x);
                }
            }
        }
    }
    a.cost_out[k] = st == FO_OK ? now : 0.0;  // makespan = last completion time
    a.status_out[k] = st;
    if (TL) { *a.tl.n_c = nc; *a.tl.n_b = nb; }
    if (a.bad_out) *a.bad_out = -1;
}

// Small-graph loop with 16-byte ready entries in two ring buffers of
// kRing slots: keys are (level << 16 | prank), so a ring only holds the
// currently ready nodes and its working set stays in L1.  Returns false on
// ring overflow (the caller reruns the linear-buffer loop).
constexpr int kRing = 256;
struct __align__(16) Ent16 {  // one 128-bit load / store per ready entry
    uint32_t key;
    uint16_t sb, se;
    double dur;
};
__device__ __forceinline__ bool ring_push(Ent16 *buf, int head, int &tail, const Ent16 &x) {
    if (tail - head >= kRing) return false;
    int i = tail++;
    while (i > head) {
        Ent16 p = buf[(i - 1) & (kRing - 1)];
        if (p.key <= x.key) break;
        buf[i & (kRing - 1)] = p;
        i--;
    }
    buf[i & (kRing - 1)] = x;
    return true;
}

// append without reading the ring when the key is not below the last one
// pushed (the common case: levels only grow); lastkey is the ring's max key
__device__ __forceinline__ bool ring_push_t(Ent16 *buf, int head, int &tail, uint32_t &lastkey, const Ent16 &x) {
    if (tail - head >= kRing) return false;
    if (tail == head || x.key >= lastkey) {
        buf[(tail++) & (kRing - 1)] = x;
        lastkey = x.key;
        return true;
    }
    return ring_push(buf, head, tail, x);
}

__device__ __forceinline__ bool ring_loop(const ScoreArgs &a, int k, const double *__restrict__ dur,
                                          const uint16_t *__restrict__ sptr, uint16_t *__restrict__ indeg_,
                                          const uint32_t *__restrict__ succ, Ent16 *__restrict__ rg,
                                          Ent16 *__restrict__ rb, int G, int N, int hg, int hb) {
    uint16_t *__restrict__ indeg = opaque_ptr(indeg_);  // measured: a spilled offset otherwise
    int headg = 0, tailg = hg, headb = 0, tailb = hb;
    int run0 = 0, run1 = 0;  // lane busy flags as full registers (bools get byte-packed)
    unsigned sb0 = 0, se0 = 0, sb1 = 0, se1 = 0;
    double end0 = 0.0, end1 = 0.0, now = 0.0;
    uint32_t level = 0;
    uint32_t lastg = hg > 0 ? rg[(hg - 1) & (kRing - 1)].key : 0u;
    uint32_t lastb = hb > 0 ? rb[(hb - 1) & (kRing - 1)].key : 0u;
    // finish_node (simulator.py:88-96); false on ring overflow
    auto release = [&](unsigned qb, unsigned qe) -> bool {
        for (unsigned q = qb; q < qe; q++) {
            const uint32_t e = succ[q];
            const unsigned s = e & 0xffffu;
            const int d = indeg[s] - 1;
            Ent16 x;  // release-time loads issued with the indegree load
            x.dur = dur[s];
            x.sb = sptr[s];
            x.se = sptr[s + 1];
            indeg[s] = (uint16_t)d;
            if (d == 0) {
                x.key = level | (e >> 16);
                if (!((int)s < G ? ring_push_t(rg, headg, tailg, lastg, x) : ring_push_t(rb, headb, tailb, lastb, x)))
                    return false;
            }
        }
        return true;
    };
    // start_available (simulator.py:98-115): compute lane, then comm lane
    auto start = [&]() {
        if (!run0 && headg < tailg) {
            const Ent16 x = rg[(headg++) & (kRing - 1)];
            run0 = 1;
            end0 = __dadd_rn(now, x.dur);
            sb0 = x.sb;
            se0 = x.se;
        }
        if (!run1 && headb < tailb) {
            const Ent16 x = rb[(headb++) & (kRing - 1)];
            run1 = 1;
            end1 = __dadd_rn(now, x.dur);
            sb1 = x.sb;
            se1 = x.se;
        }
    };
    start();
    while (run0 || run1) {
        // next completion; every lane ending then drains before any start
        const bool c0 = run0 && (!run1 || end0 <= end1);
        const bool c1 = run1 && (!run0 || end1 <= end0);
        const double t = c0 ? end0 : end1;
        if (t > now) { now = t; level += 0x10000u; }
        if (c0) {
            run0 = 0;
            if (!release(sb0, se0)) return false;
        }
        if (c1) {
            run1 = 0;
            if (!release(sb1, se1)) return false;
        }
        start();
    }
    const int done = headg + headb;  // every started node has completed once both lanes are idle
    a.cost_out[k] = done == N ? now : 0.0;  // makespan = last completion time (simulator.py:135-139)
    a.status_out[k] = done == N ? FO_OK : FO_CYCLE;  // simulator.py:133
    if (a.bad_out) *a.bad_out = -1;
    return true;
}

template <typename IT, typename SE, int TEAM>
__device__ void simulate_compact(const ScoreArgs &a, int k, const Ws &w, int tid, int G, int N, TeamShm *ts) {
    // compact copies of the contracted DAG for the serial loop: narrow indices,
    // successor entries carrying the successor's tie-break rank
    IT *sptr = (IT *)w.csim();
    IT *indeg = sptr + (N + 2);
    SE *succ = (SE *)(((uintptr_t)(indeg + N + 2) + 15) & ~uintptr_t(15));
    const int P = w.sptr()[N];
    ReadyEnt *bufg = (ReadyEnt *)(((uintptr_t)(succ + P + 1) + 15) & ~uintptr_t(15));
    ReadyEnt *bufb = bufg + G + 1;
    #pragma unroll 4
    for (int i = tid; i <= N; i += TEAM) sptr[i] = (IT)w.sptr()[i];
    #pragma unroll 4
    for (int i = tid; i < N; i += TEAM) indeg[i] = (IT)w.indeg()[i];
    #pragma unroll 4
    for (int q = tid; q < P; q += TEAM) {
        int s = w.succ()[q];
        succ[q] = se_make<SE>((unsigned)w.prank()[s], (unsigned)s);
    }
    // setup-only arrays are dead from here on: drop them from L2
    {
        const int V = a.g.V, A = a.g.A;
        tsync<TEAM>();
        l2_discard(w.gmap(), 4ll * a.VB, tid, TEAM);
        l2_discard(w.nn(), 4ll * V, tid, TEAM);
        l2_discard(w.rr(), 4ll * V, tid, TEAM);
        l2_discard(w.gmin(), 4ll * G, tid, TEAM);
        l2_discard(w.gcnt(), 4ll * G, tid, TEAM);
        l2_discard(w.scnt(), 4ll * (N + 1), tid, TEAM);
        l2_discard(w.succ(), 4ll * P, tid, TEAM);
        l2_discard(w.bki(), 4ll * A, tid, TEAM);
    }
    // initial ready set: nodes with no deps at rt = 0.0 (level 0), keys sorted
    int hg = 0, hb = 0;
    for (int base = 0; base < N; base += TEAM) {
        int i = base + tid;
        bool z = i < N && w.indeg()[i] == 0;
        bool zg = z && i < G, zb = z && !zg;
        int tg, tb;
        int pg = tprefix<TEAM>(zg, tg, ts, tid), pb = tprefix<TEAM>(zb, tb, ts, tid);
        if (zg) w.zl()[hg + pg] = i;
        if (zb) w.zl()[N + hb + pb] = i;
        hg += tg;
        hb += tb;
    }
    tsync<TEAM>();
    if (tid == 0) {
        bool done = false;
        if (sizeof(IT) == 2 && !a.tl.c_id && hg <= kRing && hb <= kRing) {
            Ent16 *rg = (Ent16 *)bufg, *rb = rg + kRing;
            for (int q = 0; q < hg + hb; q++) {  // level-0 runs: node order == prank order per lane
                int i = q < hg ? w.zl()[q] : w.zl()[N + q - hg];
                Ent16 x;
                x.key = (uint32_t)w.prank()[i];
                x.dur = w.dur()[i];
                x.sb = (uint16_t)w.sptr()[i];
                x.se = (uint16_t)w.sptr()[i + 1];
                int t = q < hg ? q : q - hg;
                int dummy = t;
                ring_push(q < hg ? rg : rb, 0, dummy, x);
            }
            done = ring_loop(a, k, w.dur(), (const uint16_t *)sptr, (uint16_t *)indeg, (const uint32_t *)succ, rg, rb,
                             G, N, hg, hb);
            if (!done)  // ring overflow: restore the indegrees and rerun with linear buffers
                for (int i = 0; i < N; i++) indeg[i] = (IT)w.indeg()[i];
        }
        if (!done) {
            int t = 0;
            for (int q = 0; q < hg + hb; q++) {
                int i = q < hg ? w.zl()[q] : w.zl()[N + q - hg];
                ReadyEnt x;
                x.key = make_key(0, (unsigned)w.prank()[i], (unsigned)i);
                x.dur = w.dur()[i];
                x.sb = (unsigned)w.sptr()[i];
                x.se = (unsigned)w.sptr()[i + 1];
                if (q == hg) t = 0;
                ready_push(q < hg ? bufg : bufb, 0, t, x);
            }
            if (a.tl.c_id) event_loop<true, IT, SE>(a, k, w.dur(), sptr, indeg, succ, bufg, bufb, w, G, N, hg, hb);
            else event_loop<false, IT, SE>(a, k, w.dur(), sptr, indeg, succ, bufg, bufb, w, G, N, hg, hb);
        }
    }
    tsync<TEAM>();
}

// Shared-memory simulation.  Nodes are renumbered into tie-break order --
// groups by (min member, id), buckets by min AllReduce -- so a ready key is
// just (level << 16 | lane-local node): level counts distinct completion
// times, and (level, node) orders exactly like the reference's
// (rt, tiebreak, id) heap entries (simulator.py:63-77, :95-96).  All hot
// state (durations, successor CSR, indegrees, ready runs) sits in the warp's
// shared-memory arena.  Returns false when the candidate does not fit.
// Per-node record of the shared-memory loop: everything a node needs when it
// starts (duration) and completes (successor range) in one 16-byte load.
struct __align__(16) NodeRec {
    double dur;
    uint16_t sb, se;
    uint32_t pad;
};

template <bool TL>
__device__ __forceinline__ void smem_loop(const ScoreArgs &a, int k, const NodeRec *rec, uint16_t *indeg,
                                          const uint16_t *succ, uint32_t *rg, uint32_t *rb, const int *tlid, int G,
                                          int N, int hg, int hb) {
    int headg = 0, tailg = hg, headb = 0, tailb = hb;
    int run0 = -1, run1 = -1, done = 0, nc = 0, nb = 0;
    unsigned sb0 = 0, se0 = 0, sb1 = 0, se1 = 0;
    double end0 = 0.0, end1 = 0.0, now = 0.0;
    uint32_t level = 0;
    uint32_t lastg = hg > 0 ? rg[hg - 1] : 0u, lastb = hb > 0 ? rb[hb - 1] : 0u;  // max key in each run
    // release the successors of a completed node (finish_node, simulator.py:88-96)
    auto release = [&](unsigned qb, unsigned qe) {
        for (unsigned q = qb; q < qe; q++) {
            const int s = succ[q];
            const int d = indeg[s] - 1;
            indeg[s] = (uint16_t)d;
            if (d == 0) {
                const bool isg = s < G;
                uint32_t *r = isg ? rg : rb;
                const int h = isg ? headg : headb;
                int i = isg ? tailg++ : tailb++;
                const uint32_t key = level | (uint32_t)(isg ? s : s - G);
                uint32_t &last = isg ? lastg : lastb;
                if (i == h || key >= last) {
                    last = key;
                } else {
                    while (i > h && r[i - 1] > key) { r[i] = r[i - 1]; i--; }
                }
                r[i] = key;
            }
        }
    };
    // start_available (simulator.py:98-115): compute lane then comm lane;
    // start = max(now, rt) = now because rt is a drained completion time
    auto start = [&]() {
        if (run0 < 0 && headg < tailg) {
            run0 = (int)(rg[headg++] & 0xffffu);
            const NodeRec r = rec[run0];
            end0 = __dadd_rn(now, r.dur);
            sb0 = r.sb;
            se0 = r.se;
            if (TL) { a.tl.c_id[nc] = tlid[run0]; a.tl.c_start[nc] = now; a.tl.c_end[nc] = end0; nc++; }
        }
        if (run1 < 0 && headb < tailb) {
            run1 = G + (int)(rb[headb++] & 0xffffu);
            const NodeRec r = rec[run1];
            end1 = __dadd_rn(now, r.dur);
            sb1 = r.sb;
            se1 = r.se;
            if (TL) { a.tl.b_id[nb] = tlid[run1]; a.tl.b_start[nb] = now; a.tl.b_end[nb] = end1; nb++; }
        }
    };
    start();
    while (run0 >= 0 || run1 >= 0) {
        // next completion; every lane ending then is drained before any start
        // (simulator.py:122-132).  Equal completion times share one level.
        const bool c0 = run0 >= 0 && (run1 < 0 || end0 <= end1);
        const bool c1 = run1 >= 0 && (run0 < 0 || end1 <= end0);
        const double t = c0 ? end0 : end1;
        if (t > now) { now = t; level += 0x10000u; }
        if (c0) { run0 = -1; done++; release(sb0, se0); }
        if (c1) { run1 = -1; done++; release(sb1, se1); }
        start();
    }
    const int st = done == N ? FO_OK : FO_CYCLE;  // simulator.py:133
    a.cost_out[k] = st == FO_OK ? now : 0.0;
    a.status_out[k] = st;
    if (TL) { *a.tl.n_c = nc; *a.tl.n_b = nb; }
    if (a.bad_out) *a.bad_out = -1;
}

template <int TEAM>
__device__ bool simulate_smem(const ScoreArgs &a, int k, const Ws &w, int tid, int G, int N, char *sm, TeamShm *ts) {
    const int V = a.g.V, A = a.g.A, B = N - G;
    const int P = w.sptr()[N];
    const int cn = a.sm_nodes, cp = a.sm_pairs;
    if (sm == nullptr || N > cn || P > cp || N >= 65536 || 2 * V + A >= 65536) return false;
    NodeRec *rec = (NodeRec *)sm;
    uint16_t *sptr = (uint16_t *)(rec + cn);  // exclusive scan scratch (cn + 2)
    uint16_t *indeg = sptr + cn + 2;
    uint16_t *succ = indeg + cn;
    uint32_t *ready = (uint32_t *)(succ + cp);  // cp is even: 4-byte aligned, stays a shared-space pointer
    // sim order: rank of prank among groups / of min AR among buckets
    int *rk = w.rank();  // [0, 2V) group pranks, [2V, 2V + A) bucket pranks
    #pragma unroll 4
    for (int i = tid; i < 2 * V + A; i += TEAM) rk[i] = 0;
    tsync<TEAM>();
    #pragma unroll 4
    for (int i = tid; i < N; i += TEAM) rk[i < G ? w.prank()[i] : 2 * V + w.prank()[i]] = 1;
    tsync<TEAM>();
    team_rank_flags<TEAM>(rk, nullptr, 2 * V, ts, tid);
    team_rank_flags<TEAM>(rk + 2 * V, nullptr, A, ts, tid);
    int *sim = w.zl();       // [0, N): setup node -> sim node
    int *cnt = w.zl() + N;   // [N, 2N): successor counts in sim order
    #pragma unroll 4
    for (int i = tid; i < N; i += TEAM) {
        int j = i < G ? rk[w.prank()[i]] : G + rk[2 * V + w.prank()[i]];
        sim[i] = j;
        cnt[j] = w.sptr()[i + 1] - w.sptr()[i];
        rec[j].dur = w.dur()[i];
        indeg[j] = (uint16_t)w.indeg()[i];
        if (a.tl.c_id) w.tlid()[j] = i < G ? w.g2id()[i] : w.b2id()[i - G];
    }
    tsync<TEAM>();
    team_exscan<TEAM>(cnt, sptr, N, ts, tid);  // successor counts -> sptr (u16)
#pragma unroll 4
    for (int j = tid; j < N; j += TEAM) { rec[j].sb = sptr[j]; rec[j].se = sptr[j + 1]; }
    #pragma unroll 4
    for (int i = tid; i < N; i += TEAM) {
        int o = sptr[sim[i]];
        for (int q = w.sptr()[i]; q < w.sptr()[i + 1]; q++) succ[o++] = (uint16_t)sim[w.succ()[q]];
    }
    // initial ready runs: indegree-0 nodes at level 0, already in key order
    uint32_t *rg = ready, *rb = ready + G;
    int hg = 0, hb = 0;
    tsync<TEAM>();
    for (int base = 0; base < N; base += TEAM) {
        int j = base + tid;
        bool z = j < N && indeg[j] == 0;
        bool zg = z && j < G, zb = z && j >= G;
        int tg, tb;
        int pg = tprefix<TEAM>(zg, tg, ts, tid), pb = tprefix<TEAM>(zb, tb, ts, tid);
        if (zg) rg[hg + pg] = (uint32_t)j;
        if (zb) rb[hb + pb] = (uint32_t)(j - G);
        hg += tg;
        hb += tb;
    }
    tsync<TEAM>();
    if (tid == 0) {
        if (a.tl.c_id) smem_loop<true>(a, k, rec, indeg, succ, rg, rb, w.tlid(), G, N, hg, hb);
        else smem_loop<false>(a, k, rec, indeg, succ, rg, rb, w.tlid(), G, N, hg, hb);
    }
    tsync<TEAM>();
    (void)B;
    return true;
}

// Team-level MP forward for very large fused groups (second pass, latency
// geometry): lane = hidden channel within a warp, nodes split across the
// team's warps, a team barrier between the aggregation and transform halves of
// each layer.  The readout sums each warp's nodes, then the warps in order.
template <typename T, int TEAM>
__device__ double mp_forward_team(const DGraph &g, const int *mem, int n, const int *nbptr, const int *nb, T *H, T *P,
                                  int tid, TeamShm *ts) {
    constexpr int NW = TEAM / 32;
    const int lane = tid & 31, wid = tid >> 5;
    const MpLayout ml = mp_layout(g.layers);
    const T *W = MpW<T>::W(g);
    const T *H0 = MpW<T>::H0(g);
    for (int i = wid; i < n; i += NW) H[i * 32 + lane] = __ldg(&H0[(int64_t)mem[i] * 32 + lane]);
    tsync<TEAM>();
    for (int l = 0; l < g.layers; l++) {
        const T *Wt = W + ml.wl + (int64_t)l * 1024;
        for (int i = wid; i < n; i += NW) {  // mean aggregation (estimator.py:348-355, :374)
            int b = nbptr[i], e = nbptr[i + 1];
            T acc = H[i * 32 + lane];
            for (int q = b; q < e; q++) acc += H[nb[q] * 32 + lane];
            P[i * 32 + lane] = acc / T(1 + e - b);
        }
        tsync<TEAM>();
        for (int i = wid; i < n; i += 2 * NW) {  // relu(P @ W_l^T), two nodes per weight load
            const int i1 = i + NW;
            const bool two = i1 < n;
            T p0 = P[i * 32 + lane], p1 = two ? P[i1 * 32 + lane] : T(0);
            T a0 = T(0), a1 = T(0);
#pragma unroll 8
            for (int k = 0; k < 32; k++) {
                T wk = __ldg(&Wt[k * 32 + lane]);
                a0 = fmaT<T>(__shfl_sync(FULL, p0, k), wk, a0);
                a1 = fmaT<T>(__shfl_sync(FULL, p1, k), wk, a1);
            }
            H[i * 32 + lane] = a0 > T(0) ? a0 : T(0);
            if (two) H[i1 * 32 + lane] = a1 > T(0) ? a1 : T(0);
        }
        tsync<TEAM>();
    }
    T part = T(0);
    for (int i = wid; i < n; i += NW) part += H[i * 32 + lane];
    ts->part[wid][lane] = (double)part;
    tsync<TEAM>();
    double pred = 0.0;
    if (wid == 0) {
        T s = T(0);
        for (int q = 0; q < NW; q++) s += (T)ts->part[q][lane];
        T r = mat32<T>(W + ml.wr, s, lane);
        r = r > T(0) ? r : T(0);
        T d1 = mat32<T>(W + ml.a1, r, lane) + __ldg(&W[ml.c1 + lane]);
        d1 = d1 > T(0) ? d1 : T(0);
        T d2 = mat32<T>(W + ml.a2, d1, lane) + __ldg(&W[ml.c2 + lane]);
        d2 = d2 > T(0) ? d2 : T(0);
        T z = warp_sum<T>(__ldg(&W[ml.a3 + lane]) * d2) + __ldg(&W[ml.c3]);
        pred = __dmul_rn(softplus_d((double)z), g.out_scale);
        pred = pred > 1e-9 ? pred : 1e-9;
        if (tid == 0) ts->bcast = pred;
    }
    tsync<TEAM>();
    return ts->bcast;
}

// One very large MP fused group (n > the per-warp scratch), the whole team:
// canonical member order, member-local undirected neighbour lists, memo,
// team MP forward (estimator.py:157-191, :363-389).  Scratch: copy 0.
template <typename T, int TEAM>
__device__ void process_group_team(const ScoreArgs &a, const Ws &w, const GroupScratch &gs, int f, int tid,
                                   long long &badk, TeamShm *ts) {
    const DGraph &g = a.g;
    const int V = g.V, lane = tid & 31, wid = tid >> 5;
    const int gi = w.fused()[f];
    const int b0 = w.gptr()[f], n = w.gptr()[f + 1] - b0;
    int *mem = w.gmem() + b0;
    // members ascending: mark, then a team prefix scan over ops
    for (int v = tid; v < V; v += TEAM) gs.mark[v] = 0;
    tsync<TEAM>();
    for (int i = tid; i < n; i += TEAM) gs.mark[mem[i]] = 1;
    tsync<TEAM>();
    int o = 0;
    for (int base = 0; base < V; base += TEAM) {
        const int v = base + tid;
        const bool m = v < V && gs.mark[v];
        int tot;
        const int pos = tprefix<TEAM>(m, tot, ts, tid);
        if (m) mem[o + pos] = v;
        o += tot;
    }
    tsync<TEAM>();
    // memo (member-set hash, as the warp path)
    MemoEnt *memo = g.memo[sizeof(T) == 8];
    unsigned long long mh1 = 0, mh2 = 0;
    if (wid == 0) {
        set_hash(mem, n, lane, mh1, mh2);
        double mv = 0.0;
        bool hit = false;
        if (lane == 0 && memo) hit = memo_get(memo, g.memo_mask, mh1, mh2, &mv);
        if (lane == 0) { ts->flag = hit; ts->bcast = mv; }
    }
    tsync<TEAM>();
    if (ts->flag) {
        if (tid == 0) w.dur()[gi] = ts->bcast;
        tsync<TEAM>();
        return;
    }
    bool miss = false;
    for (int i = tid; i < n; i += TEAM) miss |= isnan(g.op_prof[mem[i]]);
    if (tany<TEAM>(miss)) { badk = min(badk, pack_bad(gi, FO_MISSING_COST)); return; }
    for (int i = tid; i < n; i += TEAM) gs.lidx[mem[i]] = i;
    tsync<TEAM>();
    for (int i = tid; i < n; i += TEAM) {
        const int v = mem[i];
        gs.zl[i] = (g.in_ptr[v + 1] - g.in_ptr[v]) + (g.out_ptr[v + 1] - g.out_ptr[v]);
    }
    tsync<TEAM>();
    team_exscan<TEAM>(gs.zl, gs.nbptr, n, ts, tid);
    for (int i = tid; i < n; i += TEAM) {  // unique neighbours inside the group
        const int v = mem[i];
        const int o2 = gs.nbptr[i];
        int c = 0;
        for (int q = g.in_ptr[v]; q < g.in_ptr[v + 1]; q++) {
            const int s2 = g.e_src[g.in_e[q]];
            if (!in_grp(w, s2, gi)) continue;
            const int j = gs.lidx[s2];
            bool dup = false;
            for (int t = 0; t < c; t++) dup |= (gs.nb[o2 + t] == j);
            if (!dup) gs.nb[o2 + c++] = j;
        }
        for (int q = g.out_ptr[v]; q < g.out_ptr[v + 1]; q++) {
            const int d2 = g.e_dst[g.out_e[q]];
            if (!in_grp(w, d2, gi)) continue;
            const int j = gs.lidx[d2];
            bool dup = false;
            for (int t = 0; t < c; t++) dup |= (gs.nb[o2 + t] == j);
            if (!dup) gs.nb[o2 + c++] = j;
        }
        gs.msort[i] = c;
    }
    tsync<TEAM>();
    if (tid == 0) {  // compact rows into a dense CSR
        int oo = 0;
        for (int i = 0; i < n; i++) {
            const int s0 = gs.nbptr[i], c = gs.msort[i];
            for (int t = 0; t < c; t++) gs.nb[oo + t] = gs.nb[s0 + t];
            gs.nbptr[i] = oo;
            oo += c;
        }
        gs.nbptr[n] = oo;
    }
    tsync<TEAM>();
    const double pred = mp_forward_team<T, TEAM>(g, mem, n, gs.nbptr, gs.nb, (T *)gs.H, (T *)gs.P, tid, ts);
    if (tid == 0) {
        w.dur()[gi] = pred;
        if (memo) memo_put(memo, g.memo_mask, mh1, mh2, pred);
    }
    tsync<TEAM>();
}

// One fused group (K2), warp-level: lane = hidden channel for message passing.
template <typename T>
__device__ void process_group(const ScoreArgs &a, const Ws &w, const GroupScratch &gs, int f, int lane, bool hw,
                              long long &badk) {
    const DGraph &g = a.g;
    const int V = g.V;
    const int gi = w.fused()[f];
    const int b0 = w.gptr()[f], n = w.gptr()[f + 1] - b0;
    int *mem = w.gmem() + b0;
    unsigned long long mh1 = 0, mh2 = 0;
    MemoEnt *memo = (!hw && g.variant == FO_EST_MESSAGE_PASSING) ? g.memo[sizeof(T) == 8] : nullptr;
    if (memo) {
        set_hash(mem, n, lane, mh1, mh2);
        double mv = 0.0;
        bool hit = false;
        if (lane == 0) hit = memo_get(memo, g.memo_mask, mh1, mh2, &mv);
        hit = __shfl_sync(FULL, hit, 0);
        if (hit) {
            if (lane == 0) w.dur()[gi] = mv;
            return;
        }
    }
    if (n > a.L.mpcap && !hw && (g.variant == FO_EST_MESSAGE_PASSING || g.variant == FO_EST_LINEAR)) {
        badk = min(badk, pack_bad(gi, kRetryLarge));
        return;
    }
    // sort members ascending (estimator.py:160, node order = ascending op id)
    if (n <= 32) {
        int x = lane < n ? mem[lane] : INT_MAX;
        for (int kk = 2; kk <= 32; kk <<= 1)
            for (int j = kk >> 1; j > 0; j >>= 1) {
                int y = __shfl_xor_sync(FULL, x, j);
                bool up = ((lane & kk) == 0);
                bool lower = (lane & j) == 0;
                int lo = min(x, y), hi = max(x, y);
                x = (lower == up) ? lo : hi;
            }
        if (lane < n) mem[lane] = x;
    } else {  // large groups: mark members, then a ballot scan over ops yields them in order
        int *mark = gs.mark;
        #pragma unroll 4
        for (int v = lane; v < V; v += 32) mark[v] = 0;
        __syncwarp();
        #pragma unroll 4
        for (int i = lane; i < n; i += 32) mark[mem[i]] = 1;
        __syncwarp();
        int o = 0;
        for (int base = 0; base < V; base += 32) {
            int v = base + lane;
            bool m = v < V && mark[v];
            unsigned bm = __ballot_sync(FULL, m);
            if (m) mem[o + __popc(bm & lanemask_lt())] = v;
            o += __popc(bm);
        }
    }
    __syncwarp();
    double d = 0.0;
    if (hw) {  // oracle_time (workloads.py:281-291): sum in ascending member order
        if (lane == 0) {
            bool all_param = true;
            PySum comp;
            for (int i = 0; i < n; i++) {
                int v = mem[i];
                if (g.op_kind[v] != 1) all_param = false;
                double c = g.op_compute[v];
                comp.add(isnan(c) ? 0.0 : c);
            }
            d = all_param ? 0.0
                          : __dadd_rn(__dadd_rn(comp.get(), g.launch),
                                      __dmul_rn(g.mem, (double)(w.gin()[gi] + w.gout()[gi])));
        }
        d = __shfl_sync(FULL, d, 0);
        if (lane == 0) w.dur()[gi] = d;
        return;
    }
    // featurize -> lookup for every member (estimator.py:170)
    bool miss = false;
    #pragma unroll 4
    for (int i = lane; i < n; i += 32) miss |= isnan(g.op_prof[mem[i]]);
    if (__any_sync(FULL, miss)) { badk = min(badk, pack_bad(gi, FO_MISSING_COST)); return; }
    if (g.variant == FO_EST_ANALYTIC) {  // estimator.py:434-446
        if (lane == 0) {
            PySum sum;
            for (int i = 0; i < n; i++) {
                int v = mem[i];
                double raw = __dsub_rn(__dsub_rn(g.op_prof[v], g.launch),
                                       __dmul_rn(g.mem, (double)(g.op_in[v] + g.op_out[v])));
                sum.add(raw);
            }
            double pred = __dadd_rn(__dadd_rn(sum.get(), g.launch), __dmul_rn(g.mem, (double)(w.gin()[gi] + w.gout()[gi])));
            w.dur()[gi] = pred > 1e-9 ? pred : 1e-9;
        }
        return;
    }
    // member-local undirected neighbour lists (estimator.py:173-177, :348-355)
    #pragma unroll 4
    for (int i = lane; i < n; i += 32) gs.lidx[mem[i]] = i;
    __syncwarp();
    #pragma unroll 4
    for (int i = lane; i < n; i += 32) {
        int v = mem[i];
        gs.zl[i] = (g.in_ptr[v + 1] - g.in_ptr[v]) + (g.out_ptr[v + 1] - g.out_ptr[v]);
    }
    __syncwarp();
    warp_exscan(gs.zl, gs.nbptr, n, lane);
    int dirE = 0;  // directed internal edges (linear variant's longest path)
    #pragma unroll 4
    for (int i = lane; i < n; i += 32) {
        int v = mem[i];
        int o = gs.nbptr[i], c = 0;
        for (int q = g.in_ptr[v]; q < g.in_ptr[v + 1]; q++) {
            int s = g.e_src[g.in_e[q]];
            if (!in_grp(w, s, gi)) continue;
            dirE++;
            int j = gs.lidx[s];
            bool dup = false;
            for (int t = 0; t < c; t++) dup |= (gs.nb[o + t] == j);
            if (!dup) gs.nb[o + c++] = j;
        }
        for (int q = g.out_ptr[v]; q < g.out_ptr[v + 1]; q++) {
            int d2 = g.e_dst[g.out_e[q]];
            if (!in_grp(w, d2, gi)) continue;
            int j = gs.lidx[d2];
            bool dup = false;
            for (int t = 0; t < c; t++) dup |= (gs.nb[o + t] == j);
            if (!dup) gs.nb[o + c++] = j;
        }
        gs.zl[i] = c;
    }
    __syncwarp();
    // compact rows in place: nbptr -> [start, start + count)
    // (store counts as end pointers in msort to keep nbptr monotone)
    #pragma unroll 4
    for (int i = lane; i < n; i += 32) gs.msort[i] = gs.zl[i];
    __syncwarp();
    if (g.variant == FO_EST_MESSAGE_PASSING) {
        // compact neighbour rows into a dense CSR (msort holds the counts)
        if (lane == 0) {
            int o = 0;
            for (int i = 0; i < n; i++) {
                int s0 = gs.nbptr[i], c = gs.msort[i];
                for (int t = 0; t < c; t++) gs.nb[o + t] = gs.nb[s0 + t];
                gs.nbptr[i] = o;
                o += c;
            }
            gs.nbptr[n] = o;
        }
        __syncwarp();
        double pred = mp_forward<T>(g, mem, n, gs.nbptr, gs.nb, (T *)gs.H, (T *)gs.P, lane);
        if (lane == 0) {
            w.dur()[gi] = pred;
            if (memo) memo_put(memo, g.memo_mask, mh1, mh2, pred);
        }
    } else {  // LINEAR (estimator.py:117-128, 341-345, 421-426)
        dirE = __reduce_add_sync(FULL, dirE);
        if (lane == 0) {
            // longest path in nodes over the directed internal edges (estimator.py:131-154)
            int *depth = gs.msort;  // reuse: counts no longer needed
            for (int i = 0; i < n; i++) depth[i] = 1;
            for (int it = 0; it < n; it++) {
                bool ch = false;
                for (int i = 0; i < n; i++) {
                    int v = mem[i];
                    for (int q = g.in_ptr[v]; q < g.in_ptr[v + 1]; q++) {
                        int s = g.e_src[g.in_e[q]];
                        if (!in_grp(w, s, gi)) continue;
                        int j = gs.lidx[s];
                        if (depth[j] + 1 > depth[i]) { depth[i] = depth[j] + 1; ch = true; }
                    }
                }
                if (!ch) break;
            }
            int lp = 0;
            for (int i = 0; i < n; i++) lp = max(lp, depth[i]);
            PySum tot;
            for (int i = 0; i < n; i++) tot.add(g.op_prof[mem[i]]);
            const double total = tot.get();
            double agg[6] = {(double)n, total, (double)w.gint()[gi], (double)w.gin()[gi], (double)w.gout()[gi],
                             (double)lp};
            double fs[12];
            for (int q = 0; q < 6; q++) { fs[q] = log1p(agg[q]); fs[6 + q] = agg[q]; }
            if (g.lin_norm)
                for (int q = 0; q < 12; q++) fs[q] = __ddiv_rn(__dsub_rn(fs[q], g.agg_mean[q]), g.agg_std[q]);
            double z = 0.0;
            for (int q = 0; q < 12; q++) z = __dadd_rn(z, __dmul_rn(g.lin_w[q], fs[q]));
            z = __dadd_rn(z, g.lin_b);
            double pred = __dmul_rn(softplus_d(z), g.out_scale);
            w.dur()[gi] = pred > 1e-9 ? pred : 1e-9;
        }
    }
    __syncwarp();
}

template <typename T, int TEAM>
__device__ void score_one(const ScoreArgs &a, int k, const Ws &w, int tid, char *sm, TeamShm *ts) {
    constexpr int NW = TEAM / 32;
    const int lane = tid & 31, wid = tid >> 5;
    const DGraph &g = a.g;
    const int V = g.V, E = g.E, A = g.A, VB = a.VB;
    // candidate encoding: int32 or int16 ids (the int16 form halves the bytes moved)
    auto ldid = [&](const void *p, int64_t i) -> int {
        return a.idx16 ? (int)((const int16_t *)p)[i] : ((const int32_t *)p)[i];
    };
    const int64_t ob = (int64_t)k * V, oa = (int64_t)k * A;

    // ---- K1: group / bucket numbering (ids -> node order, graph.py:269-273)
    #pragma unroll 4
    for (int i = tid; i < VB; i += TEAM) w.gmap()[i] = 0;
    #pragma unroll 4
    for (int i = tid; i < A; i += TEAM) w.bmap()[i] = 0;
    tsync<TEAM>();
    bool bad = false;
    if (a.dbase) {
        // sparse candidate: the resident parent (read by every candidate of the
        // batch, so it is served from L2) with this candidate's changes applied
        const int32_t *pb = a.dbase;
        #pragma unroll 4
        for (int v = tid; v < V; v += TEAM) {
            w.nn()[v] = pb[v];
            w.rr()[v] = pb[V + v];
        }
        #pragma unroll 4
        for (int i = tid; i < A; i += TEAM) w.bki()[i] = pb[2 * V + i];
        tsync<TEAM>();
        const int c0 = a.doff[k], c1 = a.doff[k + 1];
        if (c0 < 0 || c1 < c0 || c1 > a.doff[a.K]) bad = true;  // offsets must be non-decreasing
        else for (int c = c0 + tid; c < c1; c += TEAM) {
            const int idx = a.dchg[2 * c], val = a.dchg[2 * c + 1];
            if (idx < 0 || idx >= 2 * V + A) { bad = true; continue; }
            if (idx < V) w.nn()[idx] = val;
            else if (idx < 2 * V) w.rr()[idx - V] = val;
            else w.bki()[idx - 2 * V] = val;
        }
        tsync<TEAM>();
        #pragma unroll 4
        for (int v = tid; v < V; v += TEAM) {
            const int x = w.nn()[v], y = w.rr()[v];
            if (x < 0 || x >= VB || y < -1 || y >= VB || x == y) { bad = true; continue; }
            w.gmap()[x] = 1;
            if (y >= 0) w.gmap()[y] = 1;
        }
        #pragma unroll 4
        for (int i = tid; i < A; i += TEAM) {
            const int x = w.bki()[i];
            if (x < 0 || x >= A) { bad = true; continue; }
            w.bmap()[x] = 1;
        }
    } else {
        #pragma unroll 4
        for (int v = tid; v < V; v += TEAM) {
            int x = ldid(a.ngid, ob + v), y = ldid(a.rgid, ob + v);
            if (x < 0 || x >= VB || y < -1 || y >= VB || x == y) { bad = true; continue; }
            w.gmap()[x] = 1;
            if (y >= 0) w.gmap()[y] = 1;
            w.nn()[v] = x;
            w.rr()[v] = y;
        }
        #pragma unroll 4
        for (int i = tid; i < A; i += TEAM) {
            int x = ldid(a.bkt, oa + i);
            if (x < 0 || x >= A) { bad = true; continue; }
            w.bmap()[x] = 1;
            w.bki()[i] = x;
        }
    }
    if (tany<TEAM>(bad)) {
        if (tid == 0) { a.cost_out[k] = 0.0; a.status_out[k] = FO_INVALID_ARG; }
        return;
    }
    tsync<TEAM>();
    const int G = team_rank_flags<TEAM>(w.gmap(), a.tl.c_id ? w.g2id() : nullptr, VB, ts, tid);
    const int B = team_rank_flags<TEAM>(w.bmap(), a.tl.c_id ? w.b2id() : nullptr, A, ts, tid);
    const int N = G + B;
    #pragma unroll 4
    for (int v = tid; v < V; v += TEAM) {
        w.nn()[v] = w.gmap()[w.nn()[v]];
        int y = w.rr()[v];
        w.rr()[v] = y >= 0 ? w.gmap()[y] : -1;
    }
    #pragma unroll 4
    for (int i = tid; i < A; i += TEAM) w.bki()[i] = w.bmap()[w.bki()[i]];
    #pragma unroll 4
    for (int i = tid; i < G; i += TEAM) { w.gmin()[i] = INT_MAX; w.gcnt()[i] = 0; }
    #pragma unroll 4
    for (int i = tid; i < B; i += TEAM) { w.bmin()[i] = INT_MAX; w.btot()[i] = 0; }
    #pragma unroll 4
    for (int i = tid; i < N; i += TEAM) { w.indeg()[i] = 0; w.scnt()[i] = 0; }
    tsync<TEAM>();

    // per-group min member / size, per-bucket min AR / total bytes
    #pragma unroll 4
    for (int v = tid; v < V; v += TEAM) {
        int x = w.nn()[v], y = w.rr()[v];
        atomicMin(&w.gmin()[x], v);
        atomicAdd(&w.gcnt()[x], 1);
        if (y >= 0) { atomicMin(&w.gmin()[y], v); atomicAdd(&w.gcnt()[y], 1); }
    }
    #pragma unroll 4
    for (int i = tid; i < A; i += TEAM) {
        int b = w.bki()[i];
        atomicMin(&w.bmin()[b], i);
        atomicAdd((unsigned long long *)&w.btot()[b], (unsigned long long)g.ar_bytes[i]);
    }
    tsync<TEAM>();

    // contracted schedule DAG with multiplicities (graph.py:237-274):
    //   non-aggregate edge s->d: every copy C of d not holding s waits for export(s)
    //   aggregate edge s->d:     every copy C of d waits for bucket(a), a in ARs(s)
    //   bucket b:                waits for export(producer(a)), a in b
    for (int pass = 0; pass < 2; pass++) {
        #pragma unroll 4
        for (int e = tid; e < E; e += TEAM) {
            int s = g.e_src[e], d = g.e_dst[e];
            int c0 = w.nn()[d], c1 = w.rr()[d];
            if (!g.e_agg[e]) {
                int ex = export_of(w, s);
                int ns = w.nn()[s], rs = w.rr()[s];
                if (c0 != ns && c0 != rs) {
                    if (pass == 0) { atomicAdd(&w.scnt()[ex], 1); atomicAdd(&w.indeg()[c0], 1); }
                    else w.succ()[atomicAdd(&w.scnt()[ex], 1)] = c0;
                }
                if (c1 >= 0 && c1 != ns && c1 != rs) {
                    if (pass == 0) { atomicAdd(&w.scnt()[ex], 1); atomicAdd(&w.indeg()[c1], 1); }
                    else w.succ()[atomicAdd(&w.scnt()[ex], 1)] = c1;
                }
            } else {
                for (int q = g.arp_ptr[s]; q < g.arp_ptr[s + 1]; q++) {
                    int bn = G + w.bki()[g.arp[q]];
                    if (pass == 0) {
                        atomicAdd(&w.scnt()[bn], c1 >= 0 ? 2 : 1);
                        atomicAdd(&w.indeg()[c0], 1);
                        if (c1 >= 0) atomicAdd(&w.indeg()[c1], 1);
                    } else {
                        w.succ()[atomicAdd(&w.scnt()[bn], 1)] = c0;
                        if (c1 >= 0) w.succ()[atomicAdd(&w.scnt()[bn], 1)] = c1;
                    }
                }
            }
        }
        #pragma unroll 4
        for (int i = tid; i < A; i += TEAM) {
            int bn = G + w.bki()[i];
            int ex = export_of(w, g.ar_prod[i]);
            if (pass == 0) { atomicAdd(&w.scnt()[ex], 1); atomicAdd(&w.indeg()[bn], 1); }
            else w.succ()[atomicAdd(&w.scnt()[ex], 1)] = bn;
        }
        tsync<TEAM>();
        if (pass == 0) {
            team_exscan<TEAM>(w.scnt(), w.sptr(), N, ts, tid);
            #pragma unroll 4
            for (int i = tid; i < N; i += TEAM) w.scnt()[i] = w.sptr()[i];  // fill cursors
            tsync<TEAM>();
        }
    }

    // tie-break ranks (simulator.py:63-64): group key (min member, id), bucket key min AR.
    // prank = 2*min_member + (1 if the other group sharing that min member has a smaller id)
    #pragma unroll 4
    for (int gi = tid; gi < G; gi += TEAM) {
        int t = w.gmin()[gi];
        int other = (w.nn()[t] == gi) ? w.rr()[t] : w.nn()[t];
        int sub = (other >= 0 && w.gmin()[other] == t && other < gi) ? 1 : 0;
        int pr = 2 * t + sub;
        w.prank()[gi] = pr;
    }
    #pragma unroll 4
    for (int b = tid; b < B; b += TEAM) {
        int pr = w.bmin()[b];
        w.prank()[G + b] = pr;
    }

    if (a.stop_after == 1) {  // phase timing only (fo_set_phase_stop)
        if (tid == 0) { a.cost_out[k] = 0.0; a.status_out[k] = FO_OK; }
        return;
    }
    // ---- K2: durations of every node (simulator.py:62)
    long long badk = LLONG_MAX;
    if (!a.ext_dur) {  // (external durations replace these; the two must not race)
        #pragma unroll 4
        for (int b = tid; b < B; b += TEAM) {  // comm.py:45-49
            double d = __dadd_rn(__dmul_rn(g.C, (double)w.btot()[b]), g.D);
            w.dur()[G + b] = d;
            if (d < 0.0) badk = min(badk, pack_bad(G + b, FO_NEGATIVE_DURATION));
        }
    }
    if (a.ext_dur) {
        #pragma unroll 4
        for (int i = tid; i < N; i += TEAM) {
            double d = a.ext_dur[i];
            w.dur()[i] = d;
            if (!(d >= 0.0)) badk = min(badk, pack_bad(i, FO_NEGATIVE_DURATION));
        }
    } else {
        const bool hw = g.provider == FO_PROVIDER_HW_ORACLE;
        const bool need_io = hw || g.variant == FO_EST_ANALYTIC || g.variant == FO_EST_LINEAR;
        if (need_io) {  // group_io (graph.py:181-213)
            #pragma unroll 4
            for (int i = tid; i < G; i += TEAM) { w.gint()[i] = 0; w.gin()[i] = 0; w.gout()[i] = 0; }
            #pragma unroll 4
            for (int v = tid; v < V; v += TEAM) w.vis()[v] = 0;
            tsync<TEAM>();
            #pragma unroll 4
            for (int e = tid; e < E; e += TEAM) {
                int s = g.e_src[e], d = g.e_dst[e];
                unsigned long long by = (unsigned long long)g.e_bytes[e];
                int cs[2] = {w.nn()[d], w.rr()[d]};
                for (int c = 0; c < 2; c++) {
                    int C = cs[c];
                    if (C < 0) continue;
                    if (in_grp(w, s, C)) atomicAdd((unsigned long long *)&w.gint()[C], by);
                    else { atomicAdd((unsigned long long *)&w.gin()[C], by); w.vis()[s] = 1; }
                }
            }
            tsync<TEAM>();
            #pragma unroll 4
            for (int v = tid; v < V; v += TEAM) {
                if (w.vis()[v] || g.out_ptr[v + 1] == g.out_ptr[v] || g.arp_ptr[v + 1] > g.arp_ptr[v])
                    atomicAdd((unsigned long long *)&w.gout()[export_of(w, v)], (unsigned long long)g.op_out[v]);
            }
            tsync<TEAM>();
        }
        // singletons (estimator.py:810-814 / workloads.py:276-291) and the fused-group list
        int nf = 0;
        for (int base = 0; base < G; base += TEAM) {
            int gi = base + tid;
            bool fused = false;
            if (gi < G) {
                int n = w.gcnt()[gi];
                if (n == 1) {
                    int v = w.gmin()[gi];
                    double d;
                    if (hw) {
                        double c = g.op_compute[v];
                        d = g.op_kind[v] == 1 ? 0.0
                                              : __dadd_rn(__dadd_rn(isnan(c) ? 0.0 : c, g.launch),
                                                          __dmul_rn(g.mem, (double)(w.gin()[gi] + w.gout()[gi])));
                    } else if (g.op_kind[v] == 1) {
                        d = 0.0;
                    } else {
                        d = g.op_prof[v];
                        if (isnan(d)) { badk = min(badk, pack_bad(gi, FO_MISSING_COST)); d = 0.0; }
                    }
                    w.dur()[gi] = d;
                } else {
                    w.dur()[gi] = 0.0;
                    if (!hw && g.variant == FO_EST_NONE) badk = min(badk, pack_bad(gi, FO_MISSING_COST));
                    else if (!hw && g.variant == FO_EST_INVALID) badk = min(badk, pack_bad(gi, FO_DIM_MISMATCH));
                    else fused = true;
                }
            }
            int tot;
            int pos = tprefix<TEAM>(fused, tot, ts, tid);
            if (fused) w.fused()[nf + pos] = gi;
            nf += tot;
        }
        tsync<TEAM>();
        if (nf > 0) {
            // member lists of fused groups (order fixed below by sorting)
            #pragma unroll 4
            for (int f = tid; f < nf; f += TEAM) w.zl()[f] = w.gcnt()[w.fused()[f]];
            tsync<TEAM>();
            team_exscan<TEAM>(w.zl(), w.gptr(), nf, ts, tid);
            // group -> fused position via prank scratch-free map: reuse gcnt as position+1 marker
            #pragma unroll 4
            for (int f = tid; f < nf; f += TEAM) w.gcnt()[w.fused()[f]] = -(f + 1);
            tsync<TEAM>();
            #pragma unroll 4
            for (int f = tid; f < nf; f += TEAM) w.zl()[f] = w.gptr()[f];
            tsync<TEAM>();
            #pragma unroll 4
            for (int v = tid; v < V; v += TEAM) {
                int x = w.nn()[v], y = w.rr()[v];
                int fx = w.gcnt()[x];
                if (fx < 0) w.gmem()[atomicAdd(&w.zl()[-fx - 1], 1)] = v;
                if (y >= 0) {
                    int fy = w.gcnt()[y];
                    if (fy < 0) w.gmem()[atomicAdd(&w.zl()[-fy - 1], 1)] = v;
                }
            }
            tsync<TEAM>();
            if (TEAM > 32 && a.retry_only == 1) {
                // second pass (whole-graph scratch, one copy): groups one at a
                // time; the very large MP groups use the whole team
                const GroupScratch gs = group_scratch(w, 0);
                for (int f = 0; f < nf; f++) {
                    const int nn_f = w.gptr()[f + 1] - w.gptr()[f];
                    if (!hw && g.variant == FO_EST_MESSAGE_PASSING && nn_f > kMpCapDefault) {
                        process_group_team<T, TEAM>(a, w, gs, f, tid, badk, ts);
                    } else {
                        if (wid == 0) process_group<T>(a, w, gs, f, lane, hw, badk);
                        tsync<TEAM>();
                    }
                }
            } else {
                const GroupScratch gs = group_scratch(w, wid);
                for (int f = wid; f < nf; f += NW) process_group<T>(a, w, gs, f, lane, hw, badk);
            }
            tsync<TEAM>();
        }
    }
    // hardware-oracle jitter (noise > 0): one cold pass over the groups once
    // their base times exist; members ascending (fused lists are sorted)
    if (g.provider == FO_PROVIDER_HW_ORACLE && g.noise != 0.0 && !a.ext_dur) {
        tsync<TEAM>();
        for (int gi = tid; gi < G; gi += TEAM) {
            const double d = w.dur()[gi];
            if (d == 0.0) continue;  // all-parameter group (workloads.py:282-283)
            const int c = w.gcnt()[gi];
            const int *ops = c < 0 ? w.gmem() + w.gptr()[-c - 1] : w.gmin() + gi;
            const int n = c < 0 ? w.gptr()[-c] - w.gptr()[-c - 1] : 1;
            w.dur()[gi] = __dmul_rn(d, hw_jitter(g, ops, n, w.gint()[gi], w.gin()[gi], w.gout()[gi]));
        }
        tsync<TEAM>();
    }
    // first failing node in node order decides the error (simulator.py:62)
    badk = tmin<TEAM>(badk, ts, tid);
    tsync<TEAM>();
    if (a.dur_out) {
        #pragma unroll 4
        for (int i = tid; i < N; i += TEAM) a.dur_out[i] = w.dur()[i];
        if (tid == 0) *a.ngroups_out = G;
    }
    if (badk != LLONG_MAX) {
        if (tid == 0) {
            a.cost_out[k] = 0.0;
            a.status_out[k] = (int)(badk & 0xff);
            if (a.bad_out) *a.bad_out = (int)(badk >> 8);
        }
        return;
    }

    if (a.stop_after == 2) {  // phase timing only (fo_set_phase_stop)
        if (tid == 0) { a.cost_out[k] = 0.0; a.status_out[k] = FO_OK; }
        return;
    }
    // ---- K3: two-lane discrete-event simulation (simulator.py:66-140)
    const bool small = N < 65536 && w.sptr()[N] < 65536 && 2 * V < 65536;
    if (!small && (N >= (1 << kKeyNodeBits) || 2 * V >= (1 << kKeyNodeBits))) {
        if (tid == 0) { a.cost_out[k] = 0.0; a.status_out[k] = FO_UNSUPPORTED; }
        return;
    }
    if (simulate_smem<TEAM>(a, k, w, tid, G, N, sm, ts)) return;
    if (small) simulate_compact<uint16_t, uint32_t, TEAM>(a, k, w, tid, G, N, ts);
    else simulate_compact<uint32_t, unsigned long long, TEAM>(a, k, w, tid, G, N, ts);
}

template <typename T>
__global__ void __launch_bounds__(kWarps * 32, 7) score_kernel(const __grid_constant__ ScoreArgs a) {
    const int lane = threadIdx.x & 31;
    const int wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
    const int nw = gridDim.x * kWarps;
    extern __shared__ __align__(16) char smem_arena[];
    Ws w = ws_at(a.ws + (int64_t)wid * a.L.total, a.L);
    char *sm = a.sm_bytes > 0 ? smem_arena + (threadIdx.x >> 5) * a.sm_bytes : nullptr;
    for (int k = wid; k < a.K; k += nw) {
        if (a.retry_only && a.status_out[k] != (a.retry_only == 1 ? kRetryLarge : kRetryGeneral)) continue;
        score_one<T, 32>(a, k, w, lane, sm, nullptr);
    }
}

// Latency mode: one 128-thread block scores one candidate (setup loops over
// 128 threads, fused groups spread over the 4 warps, event loop on thread 0).
constexpr int kTeam = 128;
template <typename T>
__global__ void __launch_bounds__(kTeam, 4) score_kernel_team(const __grid_constant__ ScoreArgs a) {
    extern __shared__ __align__(16) char smem_arena[];
    __shared__ TeamShm ts;
    Ws w = ws_at(a.ws + (int64_t)blockIdx.x * a.L.total, a.L);
    char *sm = a.sm_bytes > 0 ? smem_arena : nullptr;
    for (int k = blockIdx.x; k < a.K; k += gridDim.x) {
        if (a.retry_only && a.status_out[k] != (a.retry_only == 1 ? kRetryLarge : kRetryGeneral)) continue;
        score_one<T, kTeam>(a, k, w, threadIdx.x, sm, &ts);
        __syncthreads();
    }
}

// predict_fused from features (estimator.py:462-470) on one warp: the
// closed forms as in K2, or the MP forward over embedded node features
// (estimator.py:321-389) -- the embedding in the host's operation order, the
// neighbour lists in edge order, like the graph path.
template <typename T>
__global__ void predict_features_kernel(DGraph g, FeatIn in, double *pred_out) {
    const int lane = threadIdx.x;
    const int n = in.n;
    if (g.variant == FO_EST_ANALYTIC) {  // estimator.py:434-446
        if (lane == 0) {
            PySum sum;
            for (int i = 0; i < n; i++)
                sum.add(__dsub_rn(__dsub_rn(in.c[i], g.launch), __dmul_rn(g.mem, (double)(in.in[i] + in.out[i]))));
            const double pred =
                __dadd_rn(__dadd_rn(sum.get(), g.launch), __dmul_rn(g.mem, __dadd_rn(in.agg[3], in.agg[4])));
            *pred_out = pred > 1e-9 ? pred : 1e-9;
        }
        return;
    }
    if (g.variant == FO_EST_LINEAR) {  // estimator.py:117-128, :341-345, :421-426
        if (lane == 0) {
            double fs[12];
            for (int q = 0; q < 6; q++) { fs[q] = log1p(in.agg[q]); fs[6 + q] = in.agg[q]; }
            if (g.lin_norm)
                for (int q = 0; q < 12; q++) fs[q] = __ddiv_rn(__dsub_rn(fs[q], g.agg_mean[q]), g.agg_std[q]);
            double z = 0.0;
            for (int q = 0; q < 12; q++) z = __dadd_rn(z, __dmul_rn(g.lin_w[q], fs[q]));
            z = __dadd_rn(z, g.lin_b);
            const double pred = __dmul_rn(softplus_d(z), g.out_scale);
            *pred_out = pred > 1e-9 ? pred : 1e-9;
        }
        return;
    }
    // message passing: H0 = std(X) @ W_emb^T per node, in double, like the host
    T *H0 = (T *)in.H0;
    const int F = g.emb_F, h = g.emb_h;
    for (int i = 0; i < n; i++) {
        double acc = 0.0;
        if (lane < h) {
            const double c = in.c[i], ib = (double)in.in[i], ob = (double)in.out[i];
            for (int k = 0; k < F; k++) {
                double x = k == 0 ? log1p(c) : k == 1 ? c : k == 2 ? log1p(ib) : k == 3 ? ib : k == 4 ? log1p(ob)
                         : k == 5 ? ob : (k == 6 + in.slot[i] ? 1.0 : 0.0);
                if (g.emb_mean) x = __ddiv_rn(__dsub_rn(x, g.emb_mean[k]), g.emb_std[k]);
                acc = __dadd_rn(acc, __dmul_rn(x, g.emb[(int64_t)lane * F + k]));
            }
        }
        H0[i * 32 + lane] = (T)acc;
    }
    // unique undirected neighbours: in-edges, then out-edges, in edge order
    // (warp scan over the edge list per node, ballot-ordered appends)
    int o = 0;
    for (int i = 0; i < n; i++) {
        const int start = o;
        if (lane == 0) in.nbptr[i] = start;
        for (int pass = 0; pass < 2; pass++)
            for (int q0 = 0; q0 < in.m; q0 += 32) {
                const int q = q0 + lane;
                int j = -1;
                if (q < in.m) {
                    const int s2 = in.edges[2 * q], d2 = in.edges[2 * q + 1];
                    j = pass == 0 ? (d2 == i ? s2 : -1) : (s2 == i ? d2 : -1);
                }
                unsigned hit = __ballot_sync(FULL, j >= 0);
                while (hit) {
                    const int src = __ffs(hit) - 1;
                    hit &= hit - 1;
                    const int jj = __shfl_sync(FULL, j, src);
                    bool dup = false;
                    for (int t = start + lane; t < o; t += 32) dup |= in.nb[t] == jj;
                    if (!__any_sync(FULL, dup)) {
                        if (lane == 0) in.nb[o] = jj;
                        o++;
                    }
                    __syncwarp();
                }
            }
    }
    if (lane == 0) in.nbptr[n] = o;
    DGraph g2 = g;  // the per-call embeddings stand in for the per-op table
    if (sizeof(T) == 8) g2.H0d = (const double *)H0;
    else g2.H0f = (const float *)H0;
    // mem = identity: node i reads H0[i]
    int *mem = in.nb + 2 * in.m + 1;
    for (int i = lane; i < n; i += 32) mem[i] = i;
    __syncwarp();
    const double pred = mp_forward<T>(g2, mem, n, in.nbptr, in.nb, (T *)in.H, (T *)in.P, lane);
    if (lane == 0) *pred_out = pred;
}

cudaError_t launch_predict_features(const DGraph &g, const FeatIn &in, int precision, double *pred_out,
                                    cudaStream_t stream) {
    if (precision == FO_PREC_FP64) predict_features_kernel<double><<<1, 32, 0, stream>>>(g, in, pred_out);
    else predict_features_kernel<float><<<1, 32, 0, stream>>>(g, in, pred_out);
    return cudaGetLastError();
}

// Per-round best (cost, candidate id) of a scored batch: one block, strict-<
// order (the lowest id wins among equal costs, search.py:124, :214).  Non-OK
// candidates are skipped.  out = {cost, id}; (inf, -1) for an empty batch.
// pairs != 0: cost holds (cost, id) pairs (an all-gathered exchange buffer)
__global__ void batch_best_kernel(const double *__restrict__ cost, const int32_t *__restrict__ status, int K,
                                  int64_t id_offset, double *out, int pairs) {
    __shared__ double sc[32];
    __shared__ long long si[32];
    double bc = __longlong_as_double(0x7ff0000000000000ll);
    long long bi = LLONG_MAX;
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        if (status && status[k] != 0) continue;
        double c = pairs ? cost[2 * k] : cost[k];
        long long id = pairs ? (long long)cost[2 * k + 1] : k;
        if (pairs && id < 0) continue;
        if (c < bc || (c == bc && id < bi)) { bc = c; bi = id; }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        double oc = __shfl_xor_sync(FULL, bc, d);
        long long oi = __shfl_xor_sync(FULL, bi, d);
        if (oc < bc || (oc == bc && oi < bi)) { bc = oc; bi = oi; }
    }
    if ((threadIdx.x & 31) == 0) { sc[threadIdx.x >> 5] = bc; si[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x < 32) {
        int nw = blockDim.x >> 5;
        bc = threadIdx.x < nw ? sc[threadIdx.x] : __longlong_as_double(0x7ff0000000000000ll);
        bi = threadIdx.x < nw ? si[threadIdx.x] : LLONG_MAX;
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            double oc = __shfl_xor_sync(FULL, bc, d);
            long long oi = __shfl_xor_sync(FULL, bi, d);
            if (oc < bc || (oc == bc && oi < bi)) { bc = oc; bi = oi; }
        }
        if (threadIdx.x == 0) {
            out[0] = bc;
            out[1] = bi == LLONG_MAX ? -1.0 : (double)(bi + (pairs ? 0 : id_offset));
        }
    }
}

cudaError_t launch_batch_best(const double *cost, const int32_t *status, int K, int64_t id_offset, double *out,
                              cudaStream_t stream, int pairs) {
    batch_best_kernel<<<1, 512, 0, stream>>>(cost, status, K, id_offset, out, pairs);
    return cudaGetLastError();
}

int score_warps_per_block() { return kWarps; }

template <typename T>
static int blocks_per_sm_query(int smem_per_block, bool team) {
    int n = 0;
    if (team) {
        if (smem_per_block > 48 * 1024)
            cudaFuncSetAttribute(score_kernel_team<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_per_block);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, score_kernel_team<T>, kTeam, smem_per_block);
    } else {
        if (smem_per_block > 48 * 1024)
            cudaFuncSetAttribute(score_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_per_block);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, score_kernel<T>, kWarps * 32, smem_per_block);
    }
    return n;
}

// occupancy queries are cached: they sit on the per-launch host path
template <typename T>
static int blocks_per_sm(int smem_per_block, bool team) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, int> cache;
    const std::pair<int, int> key(smem_per_block, team ? 1 : 0);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    int n = blocks_per_sm_query<T>(smem_per_block, team);
    std::lock_guard<std::mutex> lk(mu);
    cache[key] = n;
    return n;
}

ScoreGeo score_geometry(const DGraph &g, int K, int num_sms, int precision) {
    ScoreGeo geo{};
    const int V = g.V, E = g.E, A = g.A;
    // arena sized for typical candidates (groups ~ ops); larger ones use the global path
    int64_t n = std::min<int64_t>(2 * (int64_t)V + A + 1, (int64_t)V + V / 8 + A + 32);
    int64_t p = (std::min<int64_t>(g.pairs_max, (int64_t)E + E / 4 + A + 32) + 1) & ~int64_t(1);
    int64_t bytes = (16 * n + 2 * (n + 2) + 2 * n + 2 * p + 4 + 4 * n + 15) & ~int64_t(15);
    const bool fp64 = precision == FO_PREC_FP64;
    const bool arena_fits = bytes <= 200 * 1024 && n < 65536;
    // Batches that fit in one wave of 128-thread blocks (search rounds) take
    // one block per candidate: the setup phases then run 4x wider, halving
    // the per-candidate latency; larger batches take one warp per candidate.
    const char *tenv = getenv("FO_TEAM");  // tuning override, read per launch
    if (tenv) {
        geo.team = tenv[0] == '1';
    } else {
        int sm_t = arena_fits ? (int)bytes : 0;
        int per_sm_t = fp64 ? blocks_per_sm<double>(sm_t, true) : blocks_per_sm<float>(sm_t, true);
        if (per_sm_t <= 0) per_sm_t = fp64 ? blocks_per_sm<double>(0, true) : blocks_per_sm<float>(0, true);
        geo.team = K <= num_sms * std::max(per_sm_t, 1);
    }
    const int per_block = geo.team ? 1 : kWarps;  // arenas per block
    geo.sm_nodes = (int)n;
    geo.sm_pairs = (int)p;
    // The shared-memory arena takes the L1 capacity the global-workspace setup
    // phase lives on (measured slower for full batches), so only small batches
    // (latency-bound, one block per SM at most) take it.
    const char *env = getenv("FO_SIM_SMEM");  // tuning override, read per launch
    const bool arena_on = env ? env[0] == '1' : K <= num_sms * kWarps;
    geo.sm_bytes = (arena_on && arena_fits && bytes * per_block <= 200 * 1024) ? (int)bytes : 0;
    int per_sm = fp64 ? blocks_per_sm<double>(geo.sm_bytes * per_block, geo.team)
                      : blocks_per_sm<float>(geo.sm_bytes * per_block, geo.team);
    if (per_sm <= 0) {  // arena does not fit: global-memory simulation only
        geo.sm_bytes = 0;
        per_sm = fp64 ? blocks_per_sm<double>(0, geo.team) : blocks_per_sm<float>(0, geo.team);
    }
    static const char *bps = getenv("FO_BLOCKS_PER_SM");  // tuning override
    if (bps && atoi(bps) > 0) per_sm = std::min(per_sm, atoi(bps));
    int want = geo.team ? K : (K + kWarps - 1) / kWarps;
    int maxb = num_sms * std::max(per_sm, 1);
    geo.grid = std::max(1, std::min(want, maxb));
    geo.blocks_per_sm = per_sm;
    return geo;
}

cudaError_t launch_score(const DGraph &g, const void *ngid, const void *rgid, const void *bkt, int idx16, int K,
                         int VB, int precision, char *ws, const WsLayout &L, const ScoreGeo &geo,
                         double *cost_out, int32_t *status_out, const double *ext_dur, TimelineOut tl,
                         double *dur_out, int32_t *bad_out, int32_t *ngroups_out, cudaStream_t stream, int retry_only,
                         const DeltaIn *delta) {
    ScoreArgs a;
    a.retry_only = retry_only;
    a.stop_after = g.phase_stop;
    a.dbase = delta ? delta->base : nullptr;
    a.doff = delta ? delta->off : nullptr;
    a.dchg = delta ? delta->chg : nullptr;
    a.g = g;
    a.ngid = ngid;
    a.rgid = rgid;
    a.bkt = bkt;
    a.idx16 = idx16;
    a.K = K;
    a.VB = VB;
    a.sm_nodes = geo.sm_nodes;
    a.sm_pairs = geo.sm_pairs;
    a.sm_bytes = geo.sm_bytes;
    a.ws = ws;
    a.L = L;
    a.cost_out = cost_out;
    a.status_out = status_out;
    a.ext_dur = ext_dur;
    a.tl = tl;
    a.dur_out = dur_out;
    a.bad_out = bad_out;
    a.ngroups_out = ngroups_out;
    const bool fp64 = precision == FO_PREC_FP64;
    if (geo.team) {
        size_t smem = (size_t)geo.sm_bytes;
        if (fp64) score_kernel_team<double><<<geo.grid, kTeam, smem, stream>>>(a);
        else score_kernel_team<float><<<geo.grid, kTeam, smem, stream>>>(a);
    } else {
        size_t smem = (size_t)geo.sm_bytes * kWarps;
        if (fp64) score_kernel<double><<<geo.grid, kWarps * 32, smem, stream>>>(a);
        else score_kernel<float><<<geo.grid, kWarps * 32, smem, stream>>>(a);
    }
    return cudaGetLastError();
}

int score_slots(const ScoreGeo &geo) { return geo.team ? geo.grid : geo.grid * kWarps; }
int score_team_warps(const ScoreGeo &geo) { return geo.team ? kTeam / 32 : 1; }

#include "score_inc.cuh"

}  // namespace fo
