// partition.cu — the single-design multi-GPU mode: nets (hence WA entries and the
// net-arc pin pairs fused into WA) are split into contiguous ranges of the WA block list balanced by
// net-pin entries; every rank folds only its entries into a partial cell gradient, and one NCCL
// all-reduce (sum) over [partial d_cell | WA / HPWL / PP block partials] completes the gradient and the
// objective terms on every rank.  Density, the Adam step and the timing refresh are replicated, so the
// positions stay identical across ranks without further traffic.  NCCL is loaded at run time
// (dlopen), only when a communicator is requested.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "gp_kernels.cuh"

namespace tdpg {

int api_fail(int kind, const std::string& msg);

// Entry weight of every WA block, in the session's block order (session.cu: classes N = 2..8 of 256
// nets each in size-stable order, then the other nets 16 per block).
std::vector<long long> wa_block_weights(int N, const int* net_start)
{
    constexpr int kMaxN = 8, kB = 256, kGen = 16;
    auto size = [&](int n) { return net_start[n + 1] - net_start[n]; };
    auto cls = [&](int k) { return (k >= 2 && k <= kMaxN) ? k : 0; };
    std::vector<int> cnt(kMaxN + 1, 0);
    std::vector<long long> gen_sizes;
    for (int n = 0; n < N; ++n) {
        const int k = cls(size(n));
        ++cnt[k];
        if (k == 0) gen_sizes.push_back(size(n));
    }
    std::vector<long long> w;
    for (int k = 2; k <= kMaxN; ++k)
        for (int i = 0; i < cnt[k]; i += kB) w.push_back(static_cast<long long>(k) * std::min(kB, cnt[k] - i));
    for (size_t i = 0; i < gen_sizes.size(); i += kGen) {
        long long e = 0;
        for (size_t j = i; j < std::min(gen_sizes.size(), i + kGen); ++j) e += gen_sizes[j];
        w.push_back(e);
    }
    return w;
}

// Contiguous block ranges, rank r owning [b[r], b[r+1]), cut where the entry prefix crosses r/world.
std::vector<int> partition_bounds(const std::vector<long long>& w, int world)
{
    long long total = 0;
    for (long long x : w) total += x;
    std::vector<int> b(world + 1, static_cast<int>(w.size()));
    b[0] = 0;
    long long pre = 0;
    int r = 1;
    for (size_t i = 0; i < w.size() && r < world; ++i) {
        pre += w[i];
        while (r < world && pre * world >= total * r) b[r++] = static_cast<int>(i + 1);
    }
    return b;
}

namespace {

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

Nccl& nccl()
{
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.h) break;
        }
        if (!n.h) return;
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(n.h, "ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(n.h, "ncclCommInitRank"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(n.h, "ncclAllReduce"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(n.h, "ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(n.h, "ncclGetErrorString"));
    });
    if (!n.h || !n.get_unique_id || !n.comm_init_rank || !n.all_reduce)
        throw Error(TDPG_ERR_CUDA, "nccl error: libnccl.so.2 could not be loaded");
    return n;
}

void nccl_check(ncclResult_t r, const char* what)
{
    if (r != ncclSuccess)
        throw Error(TDPG_ERR_CUDA, std::string("nccl error: ") + (nccl().error_string ? nccl().error_string(r) : "?") +
                                       " (" + what + ")");
}

} // namespace

// Sum-all-reduce of `n` doubles in place on the session stream (capturable into a CUDA graph).
void comm_allreduce(tdpg_session* s, double* buf, size_t n)
{
    nccl_check(nccl().all_reduce(buf, buf, n, ncclFloat64, ncclSum, static_cast<ncclComm_t>(s->comm), s->st),
               "ncclAllReduce");
}

// Sum-all-reduce of the fixed-point density grid (int64: exact and order independent, so every rank holds
// bitwise the single-GPU grid) on stream `st` (capturable).
void comm_allreduce_i64(tdpg_session* s, long long* buf, size_t n, cudaStream_t st)
{
    nccl_check(nccl().all_reduce(buf, buf, n, ncclInt64, ncclSum, static_cast<ncclComm_t>(s->comm), st),
               "ncclAllReduce (density grid)");
}

void comm_destroy(tdpg_session* s)
{
    if (s->comm && nccl().comm_destroy) nccl().comm_destroy(static_cast<ncclComm_t>(s->comm));
    s->comm = nullptr;
}

void set_partition(tdpg_session* s, int rank, int world)
{
    if (world < 1 || rank < 0 || rank >= world)
        throw Error(TDPG_ERR_VALIDATION, "validation error: partition rank must be in [0, world)");
    const auto b = partition_bounds(wa_block_weights(s->N, s->h_net_start.data()), world);
    if (b.back() != s->n_wa_blocks && !(s->n_wa_blocks == 1 && b.back() == 0))
        throw Error(TDPG_ERR_INTERNAL, "partition plan does not match the WA block layout");
    s->part_rank = rank, s->part_world = world, s->part_comm1 = false;
    s->part_b0 = b[rank], s->part_b1 = world == 1 ? s->n_wa_blocks : b[rank + 1];
    engine_release(s); // the iteration graph depends on the partition: tdpg_engine_init again
}

} // namespace tdpg

using namespace tdpg;

#define API_BEGIN try {
#define API_END                                                                   \
    return TDPG_OK;                                                               \
    }                                                                             \
    catch (const ::tdpg::Error& e) { return ::tdpg::api_fail(e.kind, e.what()); } \
    catch (const std::exception& e) { return ::tdpg::api_fail(TDPG_ERR_INTERNAL, e.what()); }

extern "C" {

int tdpg_partition_plan(int32_t n_nets, const int32_t* net_start, int32_t world, int32_t* bounds,
                        int64_t* rank_entries)
{
    API_BEGIN
    if (world < 1) throw Error(TDPG_ERR_VALIDATION, "validation error: world must be >= 1");
    const auto w = wa_block_weights(n_nets, net_start);
    const auto b = partition_bounds(w, world);
    for (int r = 0; r <= world; ++r) bounds[r] = b[r];
    if (rank_entries)
        for (int r = 0; r < world; ++r) {
            long long e = 0;
            for (int i = b[r]; i < b[r + 1]; ++i) e += w[i];
            rank_entries[r] = e;
        }
    API_END
}

int tdpg_set_partition(tdpg_session* s, int32_t rank, int32_t world)
{
    API_BEGIN
    set_partition(s, rank, world);
    API_END
}

int tdpg_comm_unique_id(uint8_t id[128])
{
    API_BEGIN
    ncclUniqueId u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    static_assert(sizeof u == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, sizeof u);
    API_END
}

int tdpg_comm_init(tdpg_session* s, int32_t rank, int32_t world, const uint8_t id[128])
{
    API_BEGIN
    set_partition(s, rank, world);
    comm_destroy(s);
    // TDPG_COMM_WORLD1=1: a one-rank communicator still drives the partitioned engine (its graph with the
    // NCCL all-reduces captured in it), so that path runs on a single GPU (tests/test_partition_gpu.py)
    const char* w1 = std::getenv("TDPG_COMM_WORLD1");
    s->part_comm1 = world == 1 && w1 && std::atoi(w1) != 0;
    if (world > 1 || s->part_comm1) {
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof u);
        CK(cudaSetDevice(s->device));
        ncclComm_t c = nullptr;
        nccl_check(nccl().comm_init_rank(&c, world, u, rank), "ncclCommInitRank");
        s->comm = c;
    }
    API_END
}

// Device time of the partitioned iteration's two collectives alone (the int64 density grid, then the
// gradient buffer of n_red doubles), averaged over `iters` back-to-back pairs on the session stream; every
// rank must call it (collective).  The engine's buffers are reused: the grid is zero between iterations
// and the gradient buffer is rebuilt by the next iteration.
int tdpg_comm_bench(tdpg_session* s, int32_t iters, int64_t n_red, double ms[2])
{
    API_BEGIN
    if (!s->comm) throw Error(TDPG_ERR_VALIDATION, "validation error: tdpg_comm_bench needs a communicator");
    if (!s->grid.valid()) throw Error(TDPG_ERR_VALIDATION, "validation error: no density grid (engine_init first)");
    DBuf<double> buf;
    buf.alloc(static_cast<size_t>(std::max<int64_t>(n_red, 1)));
    buf.zero(s->st);
    cudaEvent_t e[3];
    for (auto& x : e) CK(cudaEventCreate(&x));
    float t0 = 0, t1 = 0;
    const size_t B = static_cast<size_t>(s->grid.bins());
    CK(cudaEventRecord(e[0], s->st));
    for (int i = 0; i < iters; ++i) comm_allreduce_i64(s, s->grid.acc.p, B, s->st);
    CK(cudaEventRecord(e[1], s->st));
    for (int i = 0; i < iters; ++i) comm_allreduce(s, buf.p, static_cast<size_t>(n_red));
    CK(cudaEventRecord(e[2], s->st));
    CK(cudaEventSynchronize(e[2]));
    CK(cudaEventElapsedTime(&t0, e[0], e[1]));
    CK(cudaEventElapsedTime(&t1, e[1], e[2]));
    for (auto& x : e) cudaEventDestroy(x);
    ms[0] = t0 / std::max(iters, 1), ms[1] = t1 / std::max(iters, 1);
    API_END
}

} // extern "C"
