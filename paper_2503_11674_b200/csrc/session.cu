// session.cu — session lifetime, netlist upload, timing-graph build, C-ABI plumbing.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <memory>
#include <mutex>
#include <thread>

#include "engine.cuh"

using namespace tdpg;

namespace {
thread_local std::string g_err;
thread_local int g_kind = 0;
} // namespace

namespace tdpg {

int api_fail(int kind, const std::string& msg)
{
    g_err = msg;
    g_kind = kind;
    return kind;
}

} // namespace tdpg

#define API_BEGIN try {
#define API_END                                                     \
    return TDPG_OK;                                                 \
    }                                                               \
    catch (const ::tdpg::Error& e) { return ::tdpg::api_fail(e.kind, e.what()); } \
    catch (const std::bad_alloc&) { return ::tdpg::api_fail(TDPG_ERR_INTERNAL, "out of host memory"); } \
    catch (const std::exception& e) { return ::tdpg::api_fail(TDPG_ERR_INTERNAL, e.what()); }


namespace tdpg {

void* cub_scratch(tdpg_session* s, size_t bytes)
{
    s->cub_tmp.reserve(bytes);
    return s->cub_tmp.p;
}

__global__ void k_gather_anchor(int P, const int* __restrict__ L_pin, const double2* __restrict__ anchor,
                                double2* __restrict__ L_anchor)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P) L_anchor[i] = anchor[L_pin[i]];
}

// Kernel: pin positions (netlist.cpp:23-32): anchor + offset, two IEEE adds.
// Fixed-cell baseline (density.cpp:75-93): exact overlap areas, accumulated in the grid's fixed point
// (integer atomics commute, so the baseline is the same bits whatever the order), then converted.
__global__ void k_fixed_baseline(int C, const double2* xy, const double2* wh, const uint8_t* fixed, double x0,
                                 double y0, double bw, double bh, int nx, int ny, double scale,
                                 unsigned long long* base_q)
{
    // Fixed cells are few; one thread per fixed cell.
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C || !fixed[c]) return;
    const double xl = xy[c].x, xh = xl + wh[c].x, yl = xy[c].y, yh = yl + wh[c].y;
    const int bx0 = max(0, static_cast<int>(floor((xl - x0) / bw)));
    const int bx1 = min(nx - 1, static_cast<int>(floor((xh - x0) / bw)));
    const int by0 = max(0, static_cast<int>(floor((yl - y0) / bh)));
    const int by1 = min(ny - 1, static_cast<int>(floor((yh - y0) / bh)));
    for (int bx = bx0; bx <= bx1; ++bx)
        for (int by = by0; by <= by1; ++by) {
            const double ox = smin(xh, x0 + (bx + 1) * bw) - smax(xl, x0 + bx * bw);
            const double oy = smin(yh, y0 + (by + 1) * bh) - smax(yl, y0 + by * bh);
            if (ox > 0.0 && oy > 0.0)
                atomicAdd(&base_q[static_cast<long long>(bx) * ny + by],
                          static_cast<unsigned long long>(__double2ll_rn(ox * oy * scale)));
        }
}

__global__ void k_fixed_to_double(long long B, double* base, double inv_scale)
{
    const long long i = blockIdx.x * 256LL + threadIdx.x;
    if (i < B) base[i] = static_cast<double>(reinterpret_cast<const long long*>(base)[i]) * inv_scale;
}

void refresh_fixed_baseline(tdpg_session* s)
{
    Grid& g = s->grid;
    if (!g.valid() || !g.has_fixed) return;
    g.base.zero(s->st); // (as int64 zeros)
    k_fixed_baseline<<<blocks_for(s->C, 256), 256, 0, s->st>>>(s->C, s->cell_xy, s->cell_wh, s->cell_fixed, g.x0,
                                                                g.y0, g.bw, g.bh, g.nx, g.ny, g.scale,
                                                                reinterpret_cast<unsigned long long*>(g.base.p));
    k_fixed_to_double<<<blocks_for(g.bins(), 256), 256, 0, s->st>>>(g.bins(), g.base, g.inv_scale);
    CK_LAUNCH();
}

// Entry layout on the device (session creation): net `order[i]`'s pins go to their WA slots — for a class
// net of k pins at pos0[k] + block * 256 k + t + j * 256 (slot-major blocks), for a generic net contiguous
// from gen_start[i] — with the owner cell (or -1 - pin for terminals) and the pin offset.
struct EntryLayout {
    int net0[9], pos0[9];
    int gen0, gen1;
};

__global__ void k_entry_layout(int N, EntryLayout L, const int* __restrict__ order, const int* __restrict__ gen_start,
                               const int* __restrict__ net_start, const int* __restrict__ net_pins,
                               const int* __restrict__ pin_cell, const double2* __restrict__ pin_off,
                               int* __restrict__ e_cell, double2* __restrict__ e_off, int* __restrict__ pin_entry,
                               int* __restrict__ pin_net)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int n = order[i], b0 = net_start[n], k = net_start[n + 1] - b0;
    int base, stride;
    if (i >= L.gen0 && i < L.gen1) {
        base = gen_start[i], stride = 1;
    } else {
        const int q = i - L.net0[k];
        base = L.pos0[k] + (q / 256) * 256 * k + q % 256, stride = 256;
    }
    for (int j = 0; j < k; ++j) {
        const int p = net_pins[b0 + j], id = base + j * stride;
        const int c = pin_cell[p];
        e_cell[id] = c >= 0 ? c : -1 - p;
        e_off[id] = pin_off[p];
        pin_entry[p] = id;
        pin_net[p] = n;
    }
}

// Sink order of each net (pin_pairs.cpp:22-34 accumulates a driver's pair terms in ascending sink pin id):
// rank of every sink by pin id (O(k^2) per net, for nets of up to kRankOnDevice pins; the host sorts the
// few larger ones), the class nets' 3-bit slot words, the generic nets' slot lists, and per sink its
// (net index, slot) and driver.
constexpr int kRankOnDevice = 256;
__global__ void k_pair_tables(int N, int gen0, int gen1, const int* __restrict__ order,
                              const int* __restrict__ gen_start, const int* __restrict__ net_start,
                              const int* __restrict__ net_pins, uint32_t* __restrict__ ord, int* __restrict__ gen_ord,
                              int* __restrict__ pin_loc, int* __restrict__ pin_driver)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int n = order[i], b0 = net_start[n], k = net_start[n + 1] - b0;
    const int drv = net_pins[b0];
    const bool generic = i >= gen0 && i < gen1;
    uint32_t w = 0;
    for (int j = 1; j < k; ++j) {
        const int pj = net_pins[b0 + j];
        pin_driver[pj] = drv;
        if (k > kRankOnDevice) continue; // (a generic net: gen_ord from the host)
        int r = 0;
        for (int q = 1; q < k; ++q) r += net_pins[b0 + q] < pj ? 1 : 0; // (pins on a net are distinct)
        if (generic) {
            gen_ord[gen_start[i] + r] = j;
        } else {
            w |= static_cast<uint32_t>(j) << (3 * r);
            pin_loc[pj] = (i << 3) | j;
        }
    }
    if (!generic) ord[i] = w;
}

__global__ void k_offnet_flags(int P, const int* __restrict__ pin_cell, const int* __restrict__ pin_entry,
                               int* __restrict__ flag)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p <= P) flag[p] = (p < P && pin_entry[p] < 0 && pin_cell[p] >= 0) ? 1 : 0;
}

// off-net cell pins take slot pos + rank; every cell pin is keyed by its cell for the fold CSR (terminals
// sort last) and counted into its cell's start (exclusive-scanned after)
__global__ void k_offnet_slots(int P, int pos, int C, const int* __restrict__ pin_cell, const int* __restrict__ flag,
                               const int* __restrict__ rank, int* __restrict__ pin_entry, int* __restrict__ key,
                               int* __restrict__ val, int* __restrict__ ces)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    if (flag[p]) pin_entry[p] = pos + rank[p];
    const int c = pin_cell[p];
    key[p] = c >= 0 ? c : C;
    val[p] = p;
    if (c >= 0) atomicAdd(&ces[c], 1);
}

__global__ void k_fold_entries(int n, const int* __restrict__ pin_sorted, const int* __restrict__ pin_entry,
                               int* __restrict__ ce)
{
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) ce[j] = pin_entry[pin_sorted[j]];
}

// Host copies of the pin -> entry and pin -> net maps (built on the device at creation), for the one-off
// API calls that map entry gradients back to pins on the host.
void host_pin_maps(tdpg_session* s)
{
    if (s->h_pin_maps_valid) return;
    s->h_pin_entry.resize(s->P), s->h_pin_net.resize(s->P);
    s->pin_entry.download(s->h_pin_entry.data(), s->P, s->st);
    s->pin_net.download(s->h_pin_net.data(), s->P, s->st);
    CK(cudaStreamSynchronize(s->st));
    s->h_pin_maps_valid = true;
}

__global__ void k_set_terminals(int P, const int* __restrict__ pin_cell, const double2* __restrict__ xy,
                                double2* __restrict__ anchor)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < P && pin_cell[p] < 0) anchor[p] = xy[p];
}

void upload_positions(tdpg_session* s, const double* xy)
{
    s->cell_xy.reserve(static_cast<size_t>(s->C));
    upload_bytes_staged(s->cell_xy.p, xy, sizeof(double2) * static_cast<size_t>(s->C), s->st);
    s->sta_valid = false;
    s->pin_xy_external = false;
    refresh_fixed_baseline(s);
}

// DensityGrid ctor (density.cpp:53-64).
void ensure_grid(tdpg_session* s, int nx, int ny, double td)
{
    if (nx < 1 || ny < 1) throw Error(TDPG_ERR_VALIDATION, "validation error: density grid must be at least 1x1");
    Grid& g = s->grid;
    if (g.nx == nx && g.ny == ny && g.td == td) return;
    g.nx = nx, g.ny = ny, g.td = td;
    g.x0 = s->core[0], g.y0 = s->core[1];
    g.bw = (s->core[2] - s->core[0]) / nx;
    g.bh = (s->core[3] - s->core[1]) / ny;
    g.cap = td * g.bw * g.bh;
    double mov = 0.0, all = 0.0, amax = 0.0;
    bool fixed = false;
    for (int c = 0; c < s->C; ++c) {
        const double a = s->h_cell_w[c] * s->h_cell_h[c];
        all += a;
        if (!s->h_cell_fixed[c]) mov += a, amax = std::max(amax, a);
        else fixed = true;
    }
    g.total_movable = mov;
    g.has_fixed = fixed;
    g.n_movable = 0;
    for (int c = 0; c < s->C; ++c) g.n_movable += s->h_cell_fixed[c] ? 0 : 1;
    g.wide_w = 1.99 * g.bw, g.wide_h = 1.99 * g.bh;
    {
        std::vector<int> wide;
        for (int c = 0; c < s->C; ++c)
            if (!s->h_cell_fixed[c] && (s->h_cell_w[c] > g.wide_w || s->h_cell_h[c] > g.wide_h)) wide.push_back(c);
        g.n_wide = static_cast<int>(wide.size());
        g.wide.upload(wide, s->st);
    }
    // Fixed point: every bin's movable occupancy is <= total area, keep 2 bits of headroom.
    int ex = 0;
    std::frexp(std::max(all, 1e-300), &ex);
    const int k = std::min(60 - ex, 1000);
    g.scale = std::ldexp(1.0, k);
    g.inv_scale = std::ldexp(1.0, -k);
    // an entry is area * wx * wy * scale with weights <= 0.75 (x2 margin): below 2^45 -> two limbs (a 23-bit low
    // part and a signed high part below 2^22, 256 of them per bin and block within int32), else three
    g.limbs = (2.0 * amax * g.scale < std::ldexp(1.0, 45)) ? 2 : 3;
    const long long B = g.bins();
    g.acc.alloc(B);
    g.acc.zero(s->st);
    g.excess.alloc(B);
    if (fixed) {
        g.base.alloc(B);
        refresh_fixed_baseline(s);
    } else {
        g.base.release();
    }
    if (g.model == 1) g.electro.ensure(nx, ny);
}

// Density model of the session's grid (0 = bin overflow, 1 = electrostatic); plans are made here, never
// inside a graph capture.
void set_density_model(tdpg_session* s, int model)
{
    if (model != 0 && model != 1)
        throw Error(TDPG_ERR_VALIDATION, "validation error: density_model must be \"overflow\" or \"electrostatic\"");
    s->grid.model = model;
    if (model == 1 && s->grid.valid()) s->grid.electro.ensure(s->grid.nx, s->grid.ny);
}

} // namespace tdpg

namespace {

// TDPG_TRACE_CREATE=1: wall time of each session-creation phase on stderr
struct PhaseTimer {
    bool on = std::getenv("TDPG_TRACE_CREATE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what)
    {
        if (!on) return;
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[tdpg create] %-28s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

// Host loop over [0, n) split into contiguous chunks on up to 16 threads (session creation at 1M+ cells).
template <typename F>
void par_for(long long n, F&& f, long long min_chunk = 1 << 15)
{
    const long long hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const int nt = static_cast<int>(std::max(1LL, std::min(hw, (n + min_chunk - 1) / min_chunk)));
    if (nt <= 1) {
        if (n > 0) f(0LL, n);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(nt - 1);
    for (int t = 1; t < nt; ++t) th.emplace_back([&f, n, nt, t] { f(n * t / nt, n * (t + 1) / nt); });
    f(0LL, n / nt);
    for (auto& x : th) x.join();
}

// Host -> device copies of the netlist-sized arrays through a process-wide pinned staging pair: each
// 32 MB chunk is copied in by several threads while the previous chunk's DMA runs (pageable copies run
// at ~5 GB/s, single threaded).  Small copies take the plain path.
struct Stager {
    static constexpr size_t kChunk = size_t(32) << 20;
    char* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    std::mutex mu;
    double ms_wait = 0, ms_copy = 0, ms_issue = 0; // (TDPG_TRACE_CREATE)
    size_t bytes = 0;
};

Stager& stager()
{
    static Stager* s = new Stager; // (never freed: lives for the process, like the CUDA context)
    return *s;
}

// Page-locked (cudaHostAlloc'd or cudaHostRegister'ed) host memory: the DMA engines read / write it directly,
// so the staging copy would only add a host memcpy.
bool host_pinned(const void* p)
{
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError(); // (clear the sticky-free query error)
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

void upload_bytes(void* dst, const void* src, size_t bytes, cudaStream_t st)
{
    if (bytes == 0) return;
    if (bytes < (size_t(4) << 20)) { // (pageable: the driver stages it before returning)
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    if (host_pinned(src)) { // DMA straight from the caller's buffer, which it may reuse once we return
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        CK(cudaStreamSynchronize(st));
        return;
    }
    Stager& S = stager();
    std::lock_guard<std::mutex> lock(S.mu);
    if (!S.buf[0]) {
        for (int k = 0; k < 2; ++k) {
            CK(cudaHostAlloc(reinterpret_cast<void**>(&S.buf[k]), Stager::kChunk, cudaHostAllocPortable));
            CK(cudaEventCreateWithFlags(&S.ev[k], cudaEventDisableTiming));
        }
    }
    int k = 0;
    for (size_t off = 0; off < bytes; off += Stager::kChunk, k ^= 1) {
        const size_t n = std::min(Stager::kChunk, bytes - off);
        const auto t0 = std::chrono::steady_clock::now();
        CK(cudaEventSynchronize(S.ev[k])); // the DMA that last read this half is done
        const auto t1 = std::chrono::steady_clock::now();
        const char* from = static_cast<const char*>(src) + off;
        char* to = S.buf[k];
        par_for(static_cast<long long>(n), [&](long long lo, long long hi) { std::memcpy(to + lo, from + lo, hi - lo); },
                size_t(4) << 20);
        const auto t2 = std::chrono::steady_clock::now();
        CK(cudaMemcpyAsync(static_cast<char*>(dst) + off, to, n, cudaMemcpyHostToDevice, st));
        CK(cudaEventRecord(S.ev[k], st));
        const auto t3 = std::chrono::steady_clock::now();
        S.ms_wait += std::chrono::duration<double, std::milli>(t1 - t0).count();
        S.ms_copy += std::chrono::duration<double, std::milli>(t2 - t1).count();
        S.ms_issue += std::chrono::duration<double, std::milli>(t3 - t2).count();
        S.bytes += n;
    }
}

} // namespace

namespace tdpg {

// Device -> host counterpart of upload_bytes (stream-ordered on `st`, synchronous for the caller): each
// 32 MB chunk lands in a pinned half by DMA and is copied out by several host threads while the next
// chunk's DMA runs.  Small copies take the plain path (the caller synchronises).
void download_bytes(void* dst, const void* src, size_t bytes, cudaStream_t st)
{
    if (bytes == 0) return;
    if (bytes < (size_t(4) << 20) || host_pinned(dst)) {
        CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return;
    }
    Stager& S = stager();
    std::lock_guard<std::mutex> lock(S.mu);
    if (!S.buf[0]) {
        for (int k = 0; k < 2; ++k) {
            CK(cudaHostAlloc(reinterpret_cast<void**>(&S.buf[k]), Stager::kChunk, cudaHostAllocPortable));
            CK(cudaEventCreateWithFlags(&S.ev[k], cudaEventDisableTiming));
        }
    }
    const size_t nch = (bytes + Stager::kChunk - 1) / Stager::kChunk;
    auto issue = [&](size_t c) {
        const size_t off = c * Stager::kChunk, n = std::min(Stager::kChunk, bytes - off);
        CK(cudaEventSynchronize(S.ev[c & 1])); // (the half's previous user is done)
        CK(cudaMemcpyAsync(S.buf[c & 1], static_cast<const char*>(src) + off, n, cudaMemcpyDeviceToHost, st));
        CK(cudaEventRecord(S.ev[c & 1], st));
    };
    issue(0);
    for (size_t c = 0; c < nch; ++c) {
        if (c + 1 < nch) issue(c + 1);
        CK(cudaEventSynchronize(S.ev[c & 1]));
        const size_t off = c * Stager::kChunk, n = std::min(Stager::kChunk, bytes - off);
        char* to = static_cast<char*>(dst) + off;
        const char* from = S.buf[c & 1];
        par_for(static_cast<long long>(n), [&](long long lo, long long hi) { std::memcpy(to + lo, from + lo, hi - lo); },
                size_t(4) << 20);
    }
}

void upload_bytes_staged(void* dst, const void* src, size_t bytes, cudaStream_t st) { upload_bytes(dst, src, bytes, st); }

} // namespace tdpg

namespace {

template <typename T>
void upload_fast(DBuf<T>& b, const T* h, size_t count, cudaStream_t st)
{
    if (count > b.n) b.alloc(count);
    upload_bytes(b.p, h, count * sizeof(T), st);
}
template <typename T>
void upload_fast(DBuf<T>& b, const std::vector<T>& v, cudaStream_t st)
{
    upload_fast(b, v.data(), v.size(), st);
}

void check_netlist(const tdpg_netlist* d)
{
    auto bad = [](const std::string& m) { throw Error(TDPG_ERR_VALIDATION, "validation error: " + m); };
    if (d->n_cells < 0 || d->n_pins < 0 || d->n_nets < 0) bad("negative sizes");
    std::atomic<int> err{0}; // first failure kind of the parallel checks (1 pin cell, 2 sinks, 3 pin id, 4 reuse)
    auto fail = [&](int k) {
        int z = 0;
        err.compare_exchange_strong(z, k);
    };
    par_for(d->n_pins, [&](long long lo, long long hi) {
        for (long long p = lo; p < hi; ++p)
            if (d->pin_cell[p] < -1 || d->pin_cell[p] >= d->n_cells) return fail(1);
    });
    if (err.load() == 1) bad("pin cell id out of range");
    if (d->net_start[0] != 0) bad("net_start[0] must be 0");
    std::unique_ptr<std::atomic<int>[]> owner(new std::atomic<int>[std::max(d->n_pins, 1)]);
    par_for(d->n_pins, [&](long long lo, long long hi) {
        for (long long p = lo; p < hi; ++p) owner[p].store(-1, std::memory_order_relaxed);
    });
    // (nets in ascending order per thread: the reported failure is one the sequential scan could report
    // first only up to the order of independent errors)
    par_for(d->n_nets, [&](long long lo, long long hi) {
        for (long long n = lo; n < hi; ++n) {
            if (d->net_start[n + 1] - d->net_start[n] < 2) return fail(2);
            for (int e = d->net_start[n]; e < d->net_start[n + 1]; ++e) {
                const int p = d->net_pins[e];
                if (p < 0 || p >= d->n_pins) return fail(3);
                int none = -1;
                if (!owner[p].compare_exchange_strong(none, static_cast<int>(n), std::memory_order_relaxed)) return fail(4);
            }
        }
    });
    switch (err.load()) {
    case 2: bad("net needs at least one sink");
    case 3: bad("net pin id out of range");
    case 4: bad("pin used by two nets");
    default: break;
    }
    for (int i = 0; i < d->n_sources; ++i)
        if (d->sources[i] < 0 || d->sources[i] >= d->n_pins) bad("source pin id out of range");
    for (int i = 0; i < d->n_endpoints; ++i)
        if (d->endpoints[i] < 0 || d->endpoints[i] >= d->n_pins) bad("endpoint pin id out of range");
}

} // namespace

extern "C" {

const char* tdpg_last_error(void) { return g_err.c_str(); }
int tdpg_last_error_kind(void) { return g_kind; }
const char* tdpg_version(void) { return "tdpg 0.1 (sm_100a, fp64)"; }

int tdpg_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

void tdpg_config_default(tdpg_config* c)
{
    std::memset(c, 0, sizeof *c); // placer.hpp:22-57
    c->gamma_frac = 0.01, c->grid_nx = 16, c->grid_ny = 16, c->target_density = 0.6, c->beta = 2.5e-5;
    c->m = 15, c->w0 = 10.0, c->w1 = 0.2, c->timing_start_iter = 500, c->k = 1, c->max_iters = 1500;
    c->mu = 1.05, c->lambda_max = 1e8, c->step0_frac = 0.01, c->step_decay = 0.999, c->adam_beta1 = 0.9;
    c->adam_beta2 = 0.999, c->adam_eps = 1e-8, c->seed = 1, c->init_jitter_frac = 0.02, c->threads = 1;
}

int tdpg_session_create(const tdpg_netlist* d, tdpg_session** out)
{
    API_BEGIN
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        throw Error(TDPG_ERR_CUDA, "cuda error: no CUDA device available (the tdpg engine has no CPU fallback)");
    }
    PhaseTimer pt;
    check_netlist(d);
    pt.mark("check_netlist");
    auto s = std::make_unique<tdpg_session>();
    CK(cudaGetDevice(&s->device));
    CK(cudaStreamCreateWithFlags(&s->st, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s->st_req, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s->st_cond, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&s->ev_sta_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_sta_join, cudaEventDisableTiming));
    s->C = d->n_cells, s->P = d->n_pins, s->N = d->n_nets, s->S = d->n_sources, s->EP = d->n_endpoints;
    s->E = d->net_start[d->n_nets];
    s->clock = d->clock_period, s->r_unit = d->r_unit, s->c_unit = d->c_unit;
    std::memcpy(s->core, d->core, sizeof s->core);
    const int C = s->C, P = s->P, N = s->N, E = s->E;
    // host copies kept for later host-side work (grid setup, jitter flags, partition bounds, endpoint
    // checks, one-off gradient mapping); arrays used only here are read from the caller's buffers
    s->h_cell_w.assign(d->cell_w, d->cell_w + C);
    s->h_cell_h.assign(d->cell_h, d->cell_h + C);
    s->h_cell_fixed.assign(d->cell_fixed, d->cell_fixed + C);
    s->h_pin_cell.assign(d->pin_cell, d->pin_cell + P);
    s->h_net_start.assign(d->net_start, d->net_start + N + 1);
    s->h_sources.assign(d->sources, d->sources + s->S);
    s->h_endpoints.assign(d->endpoints, d->endpoints + s->EP);
    if (d->pin_names) { // (all blank: nothing stored, messages print the blank names)
        bool any = false;
        for (int p = 0; p < P && !any; ++p) any = d->pin_names[p] && d->pin_names[p][0];
        if (any) {
            s->pin_names.resize(P);
            for (int p = 0; p < P; ++p) s->pin_names[p] = d->pin_names[p] ? d->pin_names[p] : "";
        } else {
            s->pin_names_blank = true;
        }
    }
    const int* net_pins = d->net_pins;
    const double* pin_off = d->pin_off;
    pt.mark("streams + host copies");
    s->h_is_source.assign(P, 0);
    s->h_is_endpoint.assign(P, 0);
    for (int v : s->h_sources) s->h_is_source[v] = 1;
    for (int v : s->h_endpoints) s->h_is_endpoint[v] = 1;
    // device netlist
    {
        std::vector<double2> wh(C);
        par_for(C, [&](long long lo, long long hi) {
            for (long long c = lo; c < hi; ++c) wh[c] = make_double2(d->cell_w[c], d->cell_h[c]);
        });
        upload_fast(s->cell_wh, wh, s->st); // (returns once the source is staged: temporaries may go)
    }
    upload_fast(s->cell_delay, d->cell_delay, C, s->st);
    upload_fast(s->cell_fixed, d->cell_fixed, C, s->st);
    upload_fast(s->pin_cell, d->pin_cell, P, s->st);
    upload_fast(s->pin_off, reinterpret_cast<const double2*>(d->pin_off), P, s->st);
    upload_fast(s->anchor, reinterpret_cast<const double2*>(d->pin_term), P, s->st);
    upload_fast(s->pin_dir, d->pin_dir, P, s->st);
    upload_fast(s->pin_cap, d->pin_cap, P, s->st);
    upload_fast(s->is_source, s->h_is_source, s->st);
    upload_fast(s->is_endpoint, s->h_is_endpoint, s->st);
    upload_fast(s->net_start, s->h_net_start, s->st);
    upload_fast(s->net_pins, net_pins, E, s->st);
    if (pt.on) {
        Stager& S = stager();
        std::fprintf(stderr, "[tdpg create]   staged %.1f MB: wait %.2f ms, copy %.2f ms, issue %.2f ms\n", S.bytes / 1e6,
                     S.ms_wait, S.ms_copy, S.ms_issue);
        S.ms_wait = S.ms_copy = S.ms_issue = 0, S.bytes = 0;
    }
    pt.mark("netlist upload");
    build_graph_device(s.get()); // build_timing_graph (timing_graph.cpp:49-138) on the device (graph.cu)
    sta_setup(s.get());
    pt.mark("timing graph (device)");
    // Net-pin entries in the WA layout: nets sorted (stably) by pin count; nets of N = 2..8 pins in
    // blocks of 256, slot-major inside a block (pin j of the block's t-th net at base + j*256 + t, so a
    // warp's loads and stores of one pin slot are contiguous); other nets (class 0) contiguous after.
    constexpr int kMaxN = 8, kB = 256;
    auto cls = [&](int n) { return (n >= 2 && n <= kMaxN) ? n : 0; };
    const int* ns = d->net_start;
    std::vector<int> cnt(kMaxN + 2, 0);
    for (int n = 0; n < N; ++n) cnt[cls(ns[n + 1] - ns[n]) + 1]++;
    for (int k = 0; k <= kMaxN; ++k) cnt[k + 1] += cnt[k];
    std::vector<int> order(std::max(N, 1)), fill(cnt.begin(), cnt.end() - 1);
    for (int n = 0; n < N; ++n) order[fill[cls(ns[n + 1] - ns[n])]++] = n;
    std::vector<int> gen_start(std::max(N, 1) + 1, 0);
    std::vector<int4> blk;
    int pos = 0;
    for (int k = 2; k <= kMaxN; ++k) {
        s->wa_cls_blk0[k] = static_cast<int>(blk.size());
        s->wa_cls_net0[k] = cnt[k], s->wa_cls_net1[k] = cnt[k + 1], s->wa_cls_pos0[k] = pos;
        // (the t-th net of a block at base + t, its pin j at + j * 256: k_entry_layout)
        for (int i = cnt[k]; i < cnt[k + 1]; i += kB) blk.push_back(make_int4(k, i, std::min(kB, cnt[k + 1] - i), pos + (i - cnt[k]) * k));
        pos += ((cnt[k + 1] - cnt[k] + kB - 1) / kB) * kB * k;
        s->wa_cls_nblk[k] = static_cast<int>(blk.size()) - s->wa_cls_blk0[k];
    }
    s->wa_cls_blk0[0] = static_cast<int>(blk.size());
    constexpr int kGenNets = 16; // generic nets per block: two per warp (half-warps for nets <= 16 pins)
    for (int i = cnt[0]; i < cnt[1]; i += kGenNets) blk.push_back(make_int4(0, i, std::min(kGenNets, cnt[1] - i), 0));
    s->wa_cls_nblk[0] = static_cast<int>(blk.size()) - s->wa_cls_blk0[0];
    for (int i = cnt[0]; i < cnt[1]; ++i) {
        const int n = order[i];
        gen_start[i] = pos;
        pos += ns[n + 1] - ns[n];
    }
    gen_start[cnt[1]] = pos; // sentinel: generic net i has gen_start[i + 1] - gen_start[i] pins
    s->wa_gen_nets = cnt[1];
    s->n_wa_blocks = static_cast<int>(blk.size());
    s->part_b0 = 0, s->part_b1 = s->n_wa_blocks; // whole design until tdpg_set_partition / tdpg_comm_init
    s->E_lay = pos;
    pt.mark("  WA layout: order + slots");
    if (blk.empty()) blk.push_back(make_int4(0, 0, 0, 0));
    upload_fast(s->net_by_size, order, s->st);
    upload_fast(s->wa_blk, blk, s->st);
    upload_fast(s->wa_gen_start, gen_start, s->st);
    {   // fused pin-pair tables (engine mode, k_pair_tables): per class-ordered net the sink slots in
        // ascending pin id (3 bits each), per generic net the same as a list; per sink pin its (net index,
        // slot) and its driver
        s->pp_ord.alloc(std::max(N, 1)), s->wa_gen_ord.alloc(std::max(pos, 1));
        s->pin_loc.alloc(std::max(P, 1)), s->pin_driver.alloc(std::max(P, 1));
        s->wa_gen_ord.zero(s->st), s->pp_ord.zero(s->st);
        CK(cudaMemsetAsync(s->pin_loc.p, 0xff, sizeof(int) * std::max(P, 1), s->st));
        CK(cudaMemsetAsync(s->pin_driver.p, 0xff, sizeof(int) * std::max(P, 1), s->st));
        if (N > 0)
            k_pair_tables<<<blocks_for(N, 256), 256, 0, s->st>>>(N, cnt[0], cnt[1], s->net_by_size, s->wa_gen_start,
                                                                s->net_start, s->net_pins, s->pp_ord, s->wa_gen_ord,
                                                                s->pin_loc, s->pin_driver);
        CK_LAUNCH();
        for (int i = cnt[0]; i < cnt[1]; ++i) { // generic nets too large for the device rank loop
            const int n = order[i], b0 = ns[n], k = ns[n + 1] - b0;
            if (k <= kRankOnDevice) continue;
            std::vector<std::pair<int, int>> sk;
            sk.reserve(k - 1);
            for (int j = 1; j < k; ++j) sk.emplace_back(net_pins[b0 + j], j);
            std::sort(sk.begin(), sk.end());
            std::vector<int> go(k - 1);
            for (int q = 0; q + 1 < k; ++q) go[q] = sk[q].second;
            CK(cudaMemcpyAsync(s->wa_gen_ord.p + gen_start[i], go.data(), sizeof(int) * (k - 1), cudaMemcpyHostToDevice,
                               s->st));
            CK(cudaStreamSynchronize(s->st)); // (go is a temporary)
        }
        s->pp_mask.alloc(std::max(N, 1));
        s->pp_mask.zero(s->st);
        s->ppw_e.alloc(std::max(pos, 1));
        s->ppw_e.zero(s->st);
        s->dl_w.alloc(std::max(P, 1));
        s->dl_w.zero(s->st);
    }
    pt.mark("  WA layout: pair tables");
    // entries, pin -> entry / net maps, off-net pin slots and the fold CSR, built on the device from the
    // uploaded netlist and the class order (host copies of the pin maps are made only if an API asks)
    {
        s->e_cell.alloc(std::max(pos, 1)), s->e_off.alloc(std::max(pos, 1));
        s->e_cell.zero(s->st), s->e_off.zero(s->st); // (padding slots of partial blocks read as cell 0 / 0)
        s->pin_entry.alloc(std::max(P, 1)), s->pin_net.alloc(std::max(P, 1));
        CK(cudaMemsetAsync(s->pin_entry.p, 0xff, sizeof(int) * std::max(P, 1), s->st)); // -1: no entry
        CK(cudaMemsetAsync(s->pin_net.p, 0xff, sizeof(int) * std::max(P, 1), s->st));
        EntryLayout L{};
        for (int k = 0; k <= kMaxN; ++k) L.net0[k] = s->wa_cls_net0[k], L.pos0[k] = s->wa_cls_pos0[k];
        L.gen0 = cnt[0], L.gen1 = cnt[1];
        if (N > 0)
            k_entry_layout<<<blocks_for(N, 256), 256, 0, s->st>>>(N, L, s->net_by_size, s->wa_gen_start, s->net_start,
                                                                 s->net_pins, s->pin_cell, s->pin_off, s->e_cell,
                                                                 s->e_off, s->pin_entry, s->pin_net);
        CK_LAUNCH();
        // cell pins on no net still take pin-pair gradient (pin_pairs.cpp:31-34 writes any pin): extra
        // slots after the laid-out entries, in ascending pin id
        cudaStream_t st = s->st;
        TBuf<int> flag(P + 1, st), rank(P + 1, st), key(std::max(P, 1), st), key_s(std::max(P, 1), st),
            val(std::max(P, 1), st), val_s(std::max(P, 1), st);
        if (P > 0) {
            k_offnet_flags<<<blocks_for(P + 1, 256), 256, 0, s->st>>>(P, s->pin_cell, s->pin_entry, flag);
            CK_LAUNCH();
            size_t b = 0;
            CK(cub::DeviceScan::ExclusiveSum(nullptr, b, flag.p, rank.p, P + 1, s->st));
            CK(cub::DeviceScan::ExclusiveSum(cub_scratch(s.get(), b), b, flag.p, rank.p, P + 1, s->st));
            int extra = 0;
            CK(cudaMemcpyAsync(&extra, rank.p + P, sizeof(int), cudaMemcpyDeviceToHost, s->st));
            // fold CSR: per cell, the entries of its pins in ascending pin id (stable sort of pins by cell)
            s->cell_ent_start.alloc(C + 1);
            TBuf<int> ccnt(C + 1, st);
            ccnt.zero(s->st);
            k_offnet_slots<<<blocks_for(P, 256), 256, 0, s->st>>>(P, pos, C, s->pin_cell, flag, rank, s->pin_entry, key,
                                                                  val, ccnt);
            CK_LAUNCH();
            int bits = 1;
            while ((1LL << bits) < static_cast<long long>(C) + 1) ++bits;
            CK(cub::DeviceRadixSort::SortPairs(nullptr, b, key.p, key_s.p, val.p, val_s.p, P, 0, bits, s->st));
            CK(cub::DeviceRadixSort::SortPairs(cub_scratch(s.get(), b), b, key.p, key_s.p, val.p, val_s.p, P, 0, bits, s->st));
            CK(cub::DeviceScan::ExclusiveSum(nullptr, b, ccnt.p, s->cell_ent_start.p, C + 1, s->st));
            CK(cub::DeviceScan::ExclusiveSum(cub_scratch(s.get(), b), b, ccnt.p, s->cell_ent_start.p, C + 1, s->st));
            CK(cudaStreamSynchronize(s->st));
            s->E_tot = pos + extra;
            int n_ce = 0;
            CK(cudaMemcpy(&n_ce, s->cell_ent_start.p + C, sizeof(int), cudaMemcpyDeviceToHost));
            s->cell_ent.alloc(std::max(n_ce, 1));
            if (n_ce > 0) {
                k_fold_entries<<<blocks_for(n_ce, 256), 256, 0, s->st>>>(n_ce, val_s, s->pin_entry, s->cell_ent);
                CK_LAUNCH();
            }
        } else {
            s->E_tot = pos;
            s->cell_ent_start.alloc(C + 1);
            CK(cudaMemsetAsync(s->cell_ent_start.p, 0, sizeof(int) * (C + 1), s->st));
            s->cell_ent.alloc(1);
        }
        CK(cudaStreamSynchronize(s->st)); // (the scratch buffers are freed on scope exit)
        s->h_pin_maps_valid = false;
    }
    pt.mark("  entries + fold CSR (device)");

    pt.mark("entries + fold CSR");
    // state buffers
    s->cell_xy.alloc(C);
    {   // Opt-in (TDPG_L2_PERSIST=1): an L2 persisting window over the cell positions.  Measured on B200
        // it gains nothing at 1M cells and costs 50% at 4M (the carve-out evicts the density grid), so
        // the default leaves L2 to the hardware policy.
        int max_persist = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, s->device);
        const size_t bytes = sizeof(double2) * static_cast<size_t>(std::max(C, 1));
        const char* pe = std::getenv("TDPG_L2_PERSIST");
        if (!(pe && std::atoi(pe) != 0)) max_persist = 0;
        if (max_persist > 0) {
            const size_t limit = std::min<size_t>(static_cast<size_t>(max_persist), 2 * bytes);
            if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, limit) == cudaSuccess) {
                cudaStreamAttrValue attr{};
                attr.accessPolicyWindow.base_ptr = s->cell_xy.p;
                attr.accessPolicyWindow.num_bytes = bytes;
                attr.accessPolicyWindow.hitRatio = std::min(1.0f, static_cast<float>(limit) / static_cast<float>(bytes));
                attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
                attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
                cudaStreamSetAttribute(s->st, cudaStreamAttributeAccessPolicyWindow, &attr);
            }
            cudaGetLastError();
        }
    }
    s->d_cell.alloc(C);
    s->dgrad.alloc(std::max(C, 1));
    s->dgrad.zero(s->st);
    s->grad_e.alloc(std::max(s->E_tot, 1));
    s->grad_e.zero(s->st);
    s->pin_xy.alloc(P);
    s->arr.alloc(P), s->req.alloc(P), s->slack.alloc(P);
    s->ak.alloc(P), s->rk.alloc(P), s->tie.alloc(P);
    s->pred.alloc(P), s->tie_list.alloc(std::max(P, 1));
    s->counters.alloc(16);
    s->h_small.reserve(64);
    CK(cudaStreamSynchronize(s->st));
    pt.mark("state buffers + sync");
    *out = s.release();
    API_END
}

int tdpg_session_destroy(tdpg_session* s)
{
    API_BEGIN
    delete s;
    API_END
}

int tdpg_graph_info(tdpg_session* s, int32_t counts[4], int32_t* level)
{
    API_BEGIN
    counts[0] = s->A_net, counts[1] = s->A_cell, counts[2] = s->L, counts[3] = s->L - 1;
    if (level) graph_host_level(s);
    if (level) std::memcpy(level, s->h_level.data(), s->h_level.size() * sizeof(int32_t));
    API_END
}

int tdpg_graph_arcs(tdpg_session* s, int32_t* from, int32_t* to, int32_t* kind, int32_t* owner)
{
    API_BEGIN
    const size_t A = static_cast<size_t>(s->A);
    graph_host_arcs(s);
    if (from) std::memcpy(from, s->h_arc_from.data(), A * sizeof(int32_t));
    if (to) std::memcpy(to, s->h_arc_to.data(), A * sizeof(int32_t));
    if (kind) std::memcpy(kind, s->h_arc_kind.data(), A * sizeof(int32_t));
    if (owner) std::memcpy(owner, s->h_arc_owner.data(), A * sizeof(int32_t));
    API_END
}

int tdpg_set_positions(tdpg_session* s, const double* xy)
{
    API_BEGIN
    upload_positions(s, xy);
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_set_terminal_positions(tdpg_session* s, const double* xy)
{
    API_BEGIN
    if (s->P == 0) return TDPG_OK;
    {   // terminal pins take the new positions (the other pins' anchors are unused)
        DBuf<double2> xy_d;
        xy_d.upload(reinterpret_cast<const double2*>(xy), s->P, s->st);
        k_set_terminals<<<blocks_for(s->P, 256), 256, 0, s->st>>>(s->P, s->pin_cell, xy_d, s->anchor);
        CK_LAUNCH();
        CK(cudaStreamSynchronize(s->st)); // (xy_d is freed on return)
    }
    if (s->L_anchor.p && s->L_pin.p) { // the level-major copy the STA sweeps read
        k_gather_anchor<<<blocks_for(s->P, 256), 256, 0, s->st>>>(s->P, s->L_pin, s->anchor, s->L_anchor);
        CK_LAUNCH();
    }
    s->sta_valid = false;
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_get_positions(tdpg_session* s, double* xy)
{
    API_BEGIN
    download_bytes(xy, s->cell_xy.p, sizeof(double2) * static_cast<size_t>(s->C), s->st);
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_set_density_model(tdpg_session* s, int32_t model)
{
    API_BEGIN
    set_density_model(s, model);
    API_END
}

int tdpg_density_fields(tdpg_session* s, double* rho, double* psi)
{
    API_BEGIN
    if (s->grid.model != 1 || s->grid.electro.nx == 0)
        throw Error(TDPG_ERR_VALIDATION, "validation error: no electrostatic density evaluated");
    const size_t B = static_cast<size_t>(s->grid.bins());
    if (rho) s->grid.electro.rho.download(rho, B, s->st);
    if (psi) s->grid.electro.psi.download(psi, B, s->st);
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_set_grid(tdpg_session* s, int32_t nx, int32_t ny, double td)
{
    API_BEGIN
    ensure_grid(s, nx, ny, td);
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_pp_set(tdpg_session* s, int64_t q, const int32_t* a, const int32_t* b, const double* w)
{
    API_BEGIN
    std::vector<std::pair<unsigned long long, double>> v(static_cast<size_t>(q));
    for (int64_t i = 0; i < q; ++i) {
        if (a[i] < 0 || b[i] < 0 || a[i] >= s->P || b[i] >= s->P)
            throw Error(TDPG_ERR_VALIDATION, "validation error: pin pair id out of range");
        v[static_cast<size_t>(i)] = {(static_cast<unsigned long long>(static_cast<uint32_t>(a[i])) << 32) |
                                         static_cast<uint32_t>(b[i]),
                                     w[i]};
    }
    std::sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    std::vector<unsigned long long> k(v.size());
    std::vector<double> ww(v.size());
    for (size_t i = 0; i < v.size(); ++i) k[i] = v[i].first, ww[i] = v[i].second;
    s->led_key.upload(k, s->st);
    s->led_w.upload(ww, s->st);
    s->Q = q;
    s->pp_dirty = true;
    if (s->E_tot > s->E_lay)
        CK(cudaMemsetAsync(s->grad_e.p + s->E_lay, 0, sizeof(double2) * (s->E_tot - s->E_lay), s->st));
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_pp_size(tdpg_session* s, int64_t* q)
{
    API_BEGIN
    *q = s->Q;
    API_END
}

int tdpg_pp_get(tdpg_session* s, int32_t* a, int32_t* b, double* w)
{
    API_BEGIN
    std::vector<unsigned long long> k(static_cast<size_t>(s->Q));
    s->led_key.download(k.data(), k.size(), s->st);
    if (w) s->led_w.download(w, static_cast<size_t>(s->Q), s->st);
    CK(cudaStreamSynchronize(s->st));
    for (size_t i = 0; i < k.size(); ++i) {
        if (a) a[i] = static_cast<int32_t>(k[i] >> 32);
        if (b) b[i] = static_cast<int32_t>(k[i] & 0xFFFFFFFFull);
    }
    API_END
}

} // extern "C"
