// common.cuh — shared device/host plumbing for the tdpg engine (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tdpg.h"

namespace tdpg {

// Programmatic dependent launch (sm_90+): a kernel launched with programmatic stream serialization may
// start once every block of the kernel before it has called pdl_trigger(); pdl_wait() then blocks until
// that kernel has completed and its writes are visible.  Code before pdl_wait() may only read data that
// no kernel still in flight writes.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... P, typename... A>
inline cudaError_t launch_pdl(void (*k)(P...), unsigned grid, unsigned block, cudaStream_t st, bool pdl, A&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid), cfg.blockDim = dim3(block), cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at, cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
}

// Bumped by every device (re)allocation: captured CUDA graphs hold raw pointers, so an engine re-captures
// its graphs when this moved since the capture (a grow-only scratch that another API call enlarged).
inline std::atomic<unsigned long long>& dbuf_epoch()
{
    static std::atomic<unsigned long long> e{0};
    return e;
}

// Exception carrying a C-ABI status; converted at the extern "C" boundary.
struct Error : std::runtime_error {
    int kind;
    Error(int k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

[[noreturn]] inline void cuda_fail(cudaError_t e, const char* what, const char* file, int line)
{
    throw Error(TDPG_ERR_CUDA, std::string("cuda error: ") + cudaGetErrorString(e) + " (" + what + " at " + file +
                                   ":" + std::to_string(line) + ")");
}

#define CK(x)                                                              \
    do {                                                                   \
        cudaError_t e_ = (x);                                              \
        if (e_ != cudaSuccess) ::tdpg::cuda_fail(e_, #x, __FILE__, __LINE__); \
    } while (0)

#define CK_LAUNCH() CK(cudaGetLastError())

// Owning device buffer.
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept
    {
        if (this != &o) {
            release();
            p = o.p, n = o.n;
            o.p = nullptr, o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void release()
    {
        if (p) {
            cudaFree(p);
            ++dbuf_epoch();
        }
        p = nullptr, n = 0;
    }
    void alloc(size_t count)
    {
        release();
        n = count;
        if (count) {
            CK(cudaMalloc(&p, count * sizeof(T)));
            ++dbuf_epoch();
            static const bool trace = [] { const char* e = std::getenv("TDPG_TRACE_ALLOC"); return e && *e == '1'; }();
            if (trace) std::fprintf(stderr, "dbuf alloc %zu x %zu B (epoch %llu)\n", count, sizeof(T), dbuf_epoch().load());
        }
    }
    // grow-only
    void reserve(size_t count)
    {
        if (count > n) alloc(count + count / 4 + 16);
    }
    void upload(const T* h, size_t count, cudaStream_t s)
    {
        if (count > n) alloc(count);
        if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
    void download(T* h, size_t count, cudaStream_t s) const
    {
        if (count) CK(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    void zero(cudaStream_t s, size_t count = SIZE_MAX)
    {
        if (count == SIZE_MAX) count = n;
        if (count) CK(cudaMemsetAsync(p, 0, count * sizeof(T), s));
    }
    T* get() const { return p; }
    operator T*() const { return p; }
};

// The device's default memory pool keeps freed memory cached (no release back to the driver at sync
// points), so the stream-ordered scratch below is recycled across session creations.
inline void pool_keep()
{
    static const bool once = [] {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        cudaGetLastError();
        return true;
    }();
    (void)once;
}

// Stream-ordered scratch buffer (session creation): cudaMallocAsync / cudaFreeAsync on one stream, so
// temporaries cost neither a device-wide synchronisation on free nor a driver allocation on reuse.
template <typename T>
struct TBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t st = nullptr;
    explicit TBuf(cudaStream_t s) : st(s) {}
    TBuf(size_t count, cudaStream_t s) : st(s) { alloc(count); }
    TBuf(const TBuf&) = delete;
    TBuf& operator=(const TBuf&) = delete;
    ~TBuf() { release(); }
    void release()
    {
        if (p) cudaFreeAsync(p, st);
        p = nullptr, n = 0;
    }
    void alloc(size_t count)
    {
        release();
        n = count;
        if (count) {
            pool_keep();
            CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), st));
        }
    }
    void reserve(size_t count)
    {
        if (count > n) alloc(count + count / 4 + 16);
    }
    void upload(const T* h, size_t count, cudaStream_t s)
    {
        if (count > n) alloc(count);
        if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void upload(const std::vector<T>& v, cudaStream_t s) { upload(v.data(), v.size(), s); }
    void download(T* h, size_t count, cudaStream_t s) const
    {
        if (count) CK(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    void zero(cudaStream_t s, size_t count = SIZE_MAX)
    {
        if (count == SIZE_MAX) count = n;
        if (count) CK(cudaMemsetAsync(p, 0, count * sizeof(T), s));
    }
    operator T*() const { return p; }
};

// Pinned host buffer.
template <typename T>
struct HBuf {
    T* p = nullptr;
    size_t n = 0;
    HBuf() = default;
    HBuf(const HBuf&) = delete;
    HBuf& operator=(const HBuf&) = delete;
    ~HBuf()
    {
        if (p) cudaFreeHost(p);
    }
    void reserve(size_t count)
    {
        if (count <= n) return;
        if (p) cudaFreeHost(p);
        n = count + count / 4 + 16;
        CK(cudaMallocHost(&p, n * sizeof(T)));
    }
    T& operator[](size_t i) { return p[i]; }
};

inline unsigned blocks_for(long long n, int threads) { return static_cast<unsigned>((n + threads - 1) / threads); }

// ---- device helpers --------------------------------------------------------
// std::min / std::max semantics (first argument kept unless strictly beaten).
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum (fixed tree order) — result valid in thread 0.
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double* sh)
{
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (w == 0) {
        r = lane < BLOCK / 32 ? sh[lane] : 0.0;
        r = warp_sum(r);
    }
    __syncthreads();
    return r;
}

// Three deterministic block sums in one shared round (results valid in thread 0); sh >= 3 * BLOCK / 32.
template <int BLOCK>
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* sh)
{
    a = warp_sum(a), b = warp_sum(b), c = warp_sum(c);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    constexpr int NW = BLOCK / 32;
    if (lane == 0) sh[w] = a, sh[NW + w] = b, sh[2 * NW + w] = c;
    __syncthreads();
    if (w == 0) {
        a = warp_sum(lane < NW ? sh[lane] : 0.0);
        b = warp_sum(lane < NW ? sh[NW + lane] : 0.0);
        c = warp_sum(lane < NW ? sh[2 * NW + lane] : 0.0);
    }
}

// Orderable 64-bit key of a double (ascending key == ascending value, -0 < +0).
__device__ __forceinline__ uint64_t double_key(double d)
{
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

} // namespace tdpg
