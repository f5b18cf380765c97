// xchg.cpp -- the multi-GPU search's per-round exchange, natively over NCCL.
//
// Each rank of a sharded lock-stepped search (parallel.py ShardedSearch)
// posts, after every round, its best (cost, global seed id) and its count of
// live seeds; one ncclAllGather of 3 doubles per rank combines them and every
// rank keeps the global best of each exchange -- the strict-< tie-break of
// search.py:124 (lowest id among equal costs).  The exchange is posted from
// the search's native round hook on a stream of its own and waited `lag`
// exchanges late (an event per slot), so a round costs a few CUDA API calls
// and never waits for another rank's same round.
//
// Stop protocol: a rank whose run is over (seeds done, or max_rounds) keeps
// posting exchanges with 0 live seeds, one per exchange it waits, until it
// waits one whose global live count is 0; every rank then holds `lag`
// exchanges in flight, so all ranks post the same number and leave together.
//
// NCCL is bound at run time (dlopen): the library torch already loaded when
// there is one, so one NCCL serves the process.

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <array>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <limits>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fo_internal.h"

namespace {

struct NcclApi {
    void *lib = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_init_rank_config)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *) = nullptr;
    ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
};

const NcclApi *nccl_api(std::string &err) {
    static NcclApi api;
    static bool tried = false;
    if (tried) {
        if (!api.lib) err = "NCCL (libnccl.so.2) could not be loaded";
        return api.lib ? &api : nullptr;
    }
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // torch's, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        err = "NCCL (libnccl.so.2) could not be loaded";
        return nullptr;
    }
    api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
    api.comm_init_rank_config = (decltype(api.comm_init_rank_config))dlsym(h, "ncclCommInitRankConfig");
    api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
    api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
    api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.comm_destroy || !api.error_string) {
        err = "NCCL symbols missing";
        return nullptr;
    }
    api.lib = h;
    return &api;
}

}  // namespace

struct fo_xchg {
    const NcclApi *api = nullptr;
    ncclComm_t comm = nullptr;
    cudaStream_t st = nullptr;
    int rank = 0, world = 1, lag = 1, device = 0;
    double *d_send = nullptr, *d_recv = nullptr;  // [(lag + 1) * 3], [(lag + 1) * 3 * world]
    double *h_send = nullptr, *h_recv = nullptr;  // pinned mirrors
    std::vector<cudaEvent_t> ev;
    std::deque<int> pending;
    int64_t posted = 0;
    std::vector<double> hist;  // (cost, seed id) of every exchange waited
    double last_cost = std::numeric_limits<double>::infinity(), last_id = std::numeric_limits<double>::infinity();
    double final_cost = 0, final_id = 0;  // the run's final best (xchg_final), posted by the closing exchanges
    bool has_final = false;
    int64_t seed_offset = 0;
    int every = 1;
    std::string err;
    // the posts run on a thread of their own: the search's round hook only
    // queues (cost, id, active) -- a post's CUDA / NCCL calls can block on a
    // deep stream, and the search's next round must not wait for them
    std::thread worker;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<std::array<double, 3>> queue;
    bool closing = false;
    std::atomic<bool> failed{false};
};

namespace fo {

// wait for the oldest exchange in flight; returns the global live-seed count (< 0: error)
static int64_t xchg_wait(fo_xchg *x) {
    const int k = x->pending.front();
    x->pending.pop_front();
    if (cudaEventSynchronize(x->ev[k]) != cudaSuccess) {
        x->err = "exchange sync failed";
        return -1;
    }
    const double *a = x->h_recv + (size_t)k * 3 * x->world;
    int best = 0;
    double total = 0;
    for (int r = 0; r < x->world; r++) {
        total += a[3 * r + 2];
        const double c = a[3 * r], i = a[3 * r + 1];
        if (c < a[3 * best] || (c == a[3 * best] && i < a[3 * best + 1])) best = r;  // strict <, lowest id
    }
    x->hist.push_back(a[3 * best]);
    x->hist.push_back(a[3 * best + 1]);
    return (int64_t)std::llround(total);
}

// post one exchange of (cost, id, active); waits the oldest once more than lag are in flight
static int xchg_post(fo_xchg *x, double cost, double id, int active) {
    const int k = (int)(x->posted % (x->lag + 1));  // its previous exchange was waited
    double *hs = x->h_send + 3 * k;
    hs[0] = cost;
    hs[1] = id;
    hs[2] = (double)active;
    x->last_cost = cost;
    x->last_id = id;
    if (cudaMemcpyAsync(x->d_send + 3 * k, hs, 3 * sizeof(double), cudaMemcpyHostToDevice, x->st) != cudaSuccess) {
        x->err = "exchange H2D";
        return FO_CUDA_ERROR;
    }
    const ncclResult_t r = x->api->all_gather(x->d_send + 3 * k, x->d_recv + (size_t)3 * k * x->world, 3, ncclFloat64,
                                              x->comm, x->st);
    if (r != ncclSuccess) {
        x->err = std::string("ncclAllGather: ") + x->api->error_string(r);
        return FO_CUDA_ERROR;
    }
    if (cudaMemcpyAsync(x->h_recv + (size_t)3 * k * x->world, x->d_recv + (size_t)3 * k * x->world,
                        3 * sizeof(double) * x->world, cudaMemcpyDeviceToHost, x->st) != cudaSuccess ||
        cudaEventRecord(x->ev[k], x->st) != cudaSuccess) {
        x->err = "exchange D2H";
        return FO_CUDA_ERROR;
    }
    x->pending.push_back(k);
    x->posted++;
    while ((int)x->pending.size() > x->lag)
        if (xchg_wait(x) < 0) return FO_CUDA_ERROR;
    return FO_OK;
}

static void xchg_stop_worker(fo_xchg *x) {
    if (!x->worker.joinable()) return;
    {
        std::lock_guard<std::mutex> lk(x->mu);
        x->closing = true;
    }
    x->cv.notify_one();
    x->worker.join();
}

static void xchg_worker(fo_xchg *x) {
    cudaSetDevice(x->device);
    for (;;) {
        std::array<double, 3> it;
        {
            std::unique_lock<std::mutex> lk(x->mu);
            x->cv.wait(lk, [&] { return x->closing || !x->queue.empty(); });
            if (x->queue.empty()) return;  // closing and drained
            it = x->queue.front();
            x->queue.pop_front();
        }
        if (!x->failed && xchg_post(x, it[0], it[1], (int)it[2]) != FO_OK) x->failed = true;
    }
}

// the search's round hook: this rank's best (first minimum: lowest seed id) and live seeds
int xchg_round(fo_xchg *x, int64_t round, const double *best, int R, int active) {
    if (x->failed) return fail(FO_CUDA_ERROR, "the search exchange failed: " + x->err);
    if ((round + 1) % x->every != 0) return FO_OK;
    int j = -1;
    for (int r = 0; r < R; r++)
        if (j < 0 || best[r] < best[j]) j = r;
    const double inf = std::numeric_limits<double>::infinity();
    const double c = j < 0 ? inf : best[j], id = j < 0 ? inf : (double)(x->seed_offset + j);
    {
        std::lock_guard<std::mutex> lk(x->mu);
        x->queue.push_back({c, id, (double)active});
    }
    x->cv.notify_one();
    return FO_OK;
}

void xchg_attach_cfg(fo_xchg *x, int64_t seed_offset, int every) {
    x->seed_offset = seed_offset;
    x->every = every;
}

// the run is over on this rank: record its final best for the closing exchanges
void xchg_final(fo_xchg *x, const double *best, int R) {
    int j = -1;
    for (int r = 0; r < R; r++)
        if (j < 0 || best[r] < best[j]) j = r;
    if (j >= 0) {
        x->final_cost = best[j];
        x->final_id = (double)(x->seed_offset + j);
        x->has_final = true;
    }
}

}  // namespace fo

using namespace fo;

extern "C" {

int fo_xchg_unique_id(uint8_t *out128) {
    if (!out128) return fail(FO_INVALID_ARG, "null id");
    std::string err;
    const NcclApi *api = nccl_api(err);
    if (!api) return fail(FO_CUDA_ERROR, err);
    ncclUniqueId id;
    const ncclResult_t r = api->get_unique_id(&id);
    if (r != ncclSuccess) return fail(FO_CUDA_ERROR, std::string("ncclGetUniqueId: ") + api->error_string(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    memcpy(out128, &id, 128);
    return FO_OK;
}

int fo_xchg_create(const uint8_t *id128, int32_t rank, int32_t world, int32_t device, int32_t lag, fo_xchg **out) {
    if (!id128 || !out || world < 1 || rank < 0 || rank >= world || lag < 1 || lag > 4096)
        return fail(FO_INVALID_ARG, "bad exchange arguments");
    std::string err;
    const NcclApi *api = nccl_api(err);
    if (!api) return fail(FO_CUDA_ERROR, err);
    if (cudaSetDevice(device) != cudaSuccess) return fail(FO_CUDA_ERROR, "cudaSetDevice");
    auto *x = new fo_xchg;
    x->api = api;
    x->rank = rank;
    x->world = world;
    x->device = device;
    x->lag = lag;
    ncclUniqueId id;
    memcpy(&id, id128, 128);
    // one CTA: an exchange kernel waits on the GPU for the slowest rank's post,
    // and every CTA it holds is an SM the search's own kernels lose meanwhile
    // (measured: 4 GPUs, BERT 256 seeds 11.6 s at NCCL's default, 7.1 s at one CTA)
    ncclResult_t r;
    if (api->comm_init_rank_config) {
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.minCTAs = 1;
        cfg.maxCTAs = 1;
        r = api->comm_init_rank_config(&x->comm, world, id, rank, &cfg);  // collective: every rank joins
    } else {
        r = api->comm_init_rank(&x->comm, world, id, rank);
    }
    if (r != ncclSuccess) {
        delete x;
        return fail(FO_CUDA_ERROR, std::string("ncclCommInitRank: ") + api->error_string(r));
    }
    const int n = lag + 1;
    bool ok = cudaStreamCreateWithFlags(&x->st, cudaStreamNonBlocking) == cudaSuccess &&
              cudaMalloc(&x->d_send, sizeof(double) * 3 * n) == cudaSuccess &&
              cudaMalloc(&x->d_recv, sizeof(double) * 3 * n * world) == cudaSuccess &&
              cudaMallocHost(&x->h_send, sizeof(double) * 3 * n) == cudaSuccess &&
              cudaMallocHost(&x->h_recv, sizeof(double) * 3 * n * world) == cudaSuccess;
    x->ev.assign(n, nullptr);
    for (int k = 0; k < n && ok; k++) ok = cudaEventCreateWithFlags(&x->ev[k], cudaEventDisableTiming | cudaEventBlockingSync) == cudaSuccess;  // the worker sleeps, no core spins
    if (!ok) {
        fo_xchg_destroy(x);
        return fail(FO_CUDA_ERROR, "exchange buffers");
    }
    x->worker = std::thread(xchg_worker, x);
    *out = x;
    return FO_OK;
}

int fo_xchg_finish(fo_xchg *x) {
    if (!x) return fail(FO_INVALID_ARG, "null exchange");
    if (cudaSetDevice(x->device) != cudaSuccess) return fail(FO_CUDA_ERROR, "cudaSetDevice");
    xchg_stop_worker(x);  // every queued post is out
    if (x->failed) return fail(FO_CUDA_ERROR, "the search exchange failed: " + x->err);
    if (x->has_final) {
        x->last_cost = x->final_cost;
        x->last_id = x->final_id;
    }
    while ((int)x->pending.size() < x->lag)
        if (xchg_post(x, x->last_cost, x->last_id, 0) != FO_OK) return fail(FO_CUDA_ERROR, x->err);
    for (;;) {
        const int64_t total = xchg_wait(x);
        if (total < 0) return fail(FO_CUDA_ERROR, x->err);
        if (total == 0) break;
        if (xchg_post(x, x->last_cost, x->last_id, 0) != FO_OK) return fail(FO_CUDA_ERROR, x->err);
    }
    while (!x->pending.empty())
        if (xchg_wait(x) < 0) return fail(FO_CUDA_ERROR, x->err);
    return FO_OK;
}

int fo_xchg_history(fo_xchg *x, double *out2, int64_t cap, int64_t *n_out) {
    if (!x) return fail(FO_INVALID_ARG, "null exchange");
    const int64_t n = (int64_t)x->hist.size() / 2;
    if (n_out) *n_out = n;
    if (out2)
        for (int64_t i = 0; i < n && i < cap; i++) {
            out2[2 * i] = x->hist[2 * i];
            out2[2 * i + 1] = x->hist[2 * i + 1];
        }
    return FO_OK;
}

int fo_xchg_destroy(fo_xchg *x) {
    if (!x) return FO_OK;
    xchg_stop_worker(x);
    cudaSetDevice(x->device);
    if (x->st) cudaStreamSynchronize(x->st);
    for (auto e : x->ev)
        if (e) cudaEventDestroy(e);
    if (x->comm) x->api->comm_destroy(x->comm);
    if (x->st) cudaStreamDestroy(x->st);
    if (x->d_send) cudaFree(x->d_send);
    if (x->d_recv) cudaFree(x->d_recv);
    if (x->h_send) cudaFreeHost(x->h_send);
    if (x->h_recv) cudaFreeHost(x->h_recv);
    delete x;
    return FO_OK;
}

}  // extern "C"
