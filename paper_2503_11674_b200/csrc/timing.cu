// timing.cu — levelized STA (sta.cpp:33-143), rank-0 critical-path extraction with the
// enumerator's lexicographic tie rule (paths.cpp:12-189), collect_pin_pairs
// (paths.cpp:191-203) and the pin-pair weight ledger (pin_pairs.cpp:7-15), on the device.
#include <cub/cub.cuh>

#include <algorithm>
#include <functional>
#include <array>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "gp_kernels.cuh"

namespace tdpg {

int api_fail(int kind, const std::string& msg);

constexpr unsigned long long kNoKey = ~0ull;

// net_delay (sta.cpp:10-14): (r * L) * (c * L + cap), L = Manhattan(driver, sink).
__device__ __forceinline__ double net_delay(double2 a, double2 b, double cap, double r, double c)
{
    const double len = fabs(a.x - b.x) + fabs(a.y - b.y);
    return (r * len) * (c * len + cap);
}

__global__ void k_pin_xy(int P, const int* __restrict__ pin_cell, const double2* __restrict__ off,
                         const double2* __restrict__ cell_xy, const double2* __restrict__ anchor,
                         double2* __restrict__ pin_xy)
{
    pdl_trigger();
    pdl_wait();
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p < P) pin_xy[p] = pin_pos(p, pin_cell, off, cell_xy, anchor);
}

struct StaArgs {
    const int *lvl_pins, *in_start, *in_from, *out_start, *out_to, *pin_cell;
    const uint8_t *is_source, *is_endpoint, *pin_dir;
    const double *cell_delay, *pin_cap;
    const double2* pin_xy;
    double r, c, clock;
    double *arr, *req;
    uint8_t *ak, *rk, *tie;
    int *pred, *tie_list, *counters;
};

// propagate_arrival for one level (sta.cpp:41-62): max over known fan-in, strict '>' in
// ascending arc id; records the winning fan-in pin and whether another arc tied it exactly.
__device__ __forceinline__ void arrival_pin(int v, const StaArgs& a)
{
    if (a.is_source[v]) {
        a.arr[v] = 0.0, a.ak[v] = 1, a.pred[v] = -1, a.tie[v] = 0;
        return;
    }
    const bool sink = a.pin_dir[v] == 0;
    const int j0 = a.in_start[v], j1 = a.in_start[v + 1];
    double best = -INFINITY;
    bool found = false;
    int bu = -1, ntie = 0;
    if (j1 > j0) {
        const double2 pv = a.pin_xy[v];
        const double cap = a.pin_cap[v];
        const double dcell = sink ? 0.0 : a.cell_delay[a.pin_cell[v]];
        for (int j = j0; j < j1; ++j) {
            const int u = a.in_from[j];
            if (!a.ak[u]) continue;
            const double d = sink ? net_delay(a.pin_xy[u], pv, cap, a.r, a.c) : dcell;
            const double cand = a.arr[u] + d;
            if (!found || cand > best) {
                best = cand, found = true, bu = u, ntie = 1;
            } else if (cand == best) {
                ++ntie;
            }
        }
    }
    a.arr[v] = found ? best : 0.0;
    a.ak[v] = found ? 1 : 0;
    a.pred[v] = found ? bu : -1;
    a.tie[v] = ntie > 1;
    if (ntie > 1) a.tie_list[atomicAdd(&a.counters[0], 1)] = v;
}

__global__ void __launch_bounds__(kBlock) k_arrival(int lo, int hi, StaArgs a)
{
    const int i = lo + blockIdx.x * kBlock + threadIdx.x;
    if (i < hi) arrival_pin(a.lvl_pins[i], a);
}

// propagate_required for one level (sta.cpp:77-97): min over known fan-out, strict '<'.
__device__ __forceinline__ void required_pin(int u, const StaArgs& a)
{
    double best = INFINITY;
    bool found = false;
    if (a.is_endpoint[u]) best = a.clock, found = true;
    const int j0 = a.out_start[u], j1 = a.out_start[u + 1];
    if (j1 > j0) {
        const bool driver = a.pin_dir[u] == 1;
        const double2 pu = a.pin_xy[u];
        const double dcell = driver ? 0.0 : a.cell_delay[a.pin_cell[u]];
        for (int j = j0; j < j1; ++j) {
            const int t = a.out_to[j];
            if (!a.rk[t]) continue;
            const double d = driver ? net_delay(pu, a.pin_xy[t], a.pin_cap[t], a.r, a.c) : dcell;
            const double cand = a.req[t] - d;
            if (!found || cand < best) best = cand, found = true;
        }
    }
    a.req[u] = found ? best : a.clock;
    a.rk[u] = found ? 1 : 0;
}

__global__ void __launch_bounds__(kBlock) k_required(int lo, int hi, StaArgs a)
{
    const int i = lo + blockIdx.x * kBlock + threadIdx.x;
    if (i < hi) required_pin(a.lvl_pins[i], a);
}

// Push sweep over sink levels.  Every arc into an Input pin is a net arc from an Output pin and every arc
// into an Output pin is a cell arc from an Input pin (sta.cpp:16-21).  So only levels holding Input pins
// need a dependent launch: an Input pin reads its driver's arrival and pushes arr + cell delay into its
// cell's outputs with a 64-bit atomicMax on the order-preserving key of the double (exact: max/min need
// no rounding); backwards, it takes its outputs' required times and pushes req - net delay into its
// driver with atomicMin.  Each thread's work is one pin and its (small) cell fan-out, instead of an
// Output pin looping over a whole net.  A final pass per direction decodes the Output pins' keys; the
// arrival decode re-evaluates the fan-in to recover the first maximising arc (pred) and exact ties,
// exactly like propagate_arrival's strict '>' in ascending arc id (sta.cpp:51-58).
__device__ __forceinline__ double key_double(unsigned long long k)
{ // inverse of double_key
    const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}
constexpr unsigned long long kNoArr = 0ull, kNoReq = ~0ull;

__global__ void __launch_bounds__(kBlock) k_sta_init(int P, StaArgs a, bool pin_xy_from_cells,
                                                     const double2* __restrict__ off,
                                                     const double2* __restrict__ cell_xy,
                                                     const double2* __restrict__ anchor,
                                                     unsigned long long* __restrict__ akey,
                                                     unsigned long long* __restrict__ rkey)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p >= P) return;
    if (pin_xy_from_cells) const_cast<double2*>(a.pin_xy)[p] = pin_pos(p, a.pin_cell, off, cell_xy, anchor);
    akey[p] = a.is_source[p] ? double_key(0.0) : kNoArr;
    rkey[p] = a.is_endpoint[p] ? double_key(a.clock) : kNoReq;
}

__global__ void __launch_bounds__(kBlock) k_arr_push(int lo, int hi, const int* __restrict__ pins, StaArgs a,
                                                     unsigned long long* __restrict__ akey)
{
    const int i = lo + blockIdx.x * kBlock + threadIdx.x;
    if (i >= hi) return;
    const int t = pins[i];
    double best = 0.0;
    bool found = false;
    int bu = -1, ntie = 0;
    if (a.is_source[t]) {
        found = true;
    } else {
        const int j0 = a.in_start[t], j1 = a.in_start[t + 1];
        if (j1 > j0) {
            const double2 pt = a.pin_xy[t];
            const double cap = a.pin_cap[t];
            for (int j = j0; j < j1; ++j) { // net arcs from drivers (final: lower levels)
                const int u = a.in_from[j];
                const unsigned long long k = akey[u];
                if (k == kNoArr) continue;
                const double cand = key_double(k) + net_delay(a.pin_xy[u], pt, cap, a.r, a.c);
                if (!found || cand > best) {
                    best = cand, found = true, bu = u, ntie = 1;
                } else if (cand == best) {
                    ++ntie;
                }
            }
        }
    }
    a.arr[t] = found ? best : 0.0;
    a.ak[t] = found ? 1 : 0;
    a.pred[t] = found ? bu : -1;
    a.tie[t] = ntie > 1;
    if (ntie > 1) a.tie_list[atomicAdd(&a.counters[0], 1)] = t;
    if (!found) return;
    const int o0 = a.out_start[t], o1 = a.out_start[t + 1];
    if (o1 > o0) {
        const double cand = best + a.cell_delay[a.pin_cell[t]];
        const unsigned long long k = double_key(cand);
        for (int j = o0; j < o1; ++j) atomicMax(&akey[a.out_to[j]], k);
    }
}

__global__ void __launch_bounds__(kBlock) k_arr_decode(int n, const int* __restrict__ pins, StaArgs a,
                                                       const unsigned long long* __restrict__ akey)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const int v = pins[i];
    if (a.is_source[v]) {
        a.arr[v] = 0.0, a.ak[v] = 1, a.pred[v] = -1, a.tie[v] = 0;
        return;
    }
    const unsigned long long k = akey[v];
    if (k == kNoArr) {
        a.arr[v] = 0.0, a.ak[v] = 0, a.pred[v] = -1, a.tie[v] = 0;
        return;
    }
    const double best = key_double(k), dcell = a.cell_delay[a.pin_cell[v]];
    int bu = -1, ntie = 0;
    for (int j = a.in_start[v]; j < a.in_start[v + 1]; ++j) {
        const int u = a.in_from[j];
        if (!a.ak[u]) continue;
        if (a.arr[u] + dcell == best) {
            if (bu < 0) bu = u;
            ++ntie;
        }
    }
    a.arr[v] = best, a.ak[v] = 1, a.pred[v] = bu, a.tie[v] = ntie > 1;
    if (ntie > 1) a.tie_list[atomicAdd(&a.counters[0], 1)] = v;
}

__global__ void __launch_bounds__(kBlock) k_req_push(int lo, int hi, const int* __restrict__ pins, StaArgs a,
                                                     unsigned long long* __restrict__ rkey)
{
    const int i = lo + blockIdx.x * kBlock + threadIdx.x;
    if (i >= hi) return;
    const int t = pins[i];
    double best = INFINITY;
    bool found = false;
    if (a.is_endpoint[t]) best = a.clock, found = true;
    const int o0 = a.out_start[t], o1 = a.out_start[t + 1];
    if (o1 > o0) {
        const double dcell = a.cell_delay[a.pin_cell[t]];
        for (int j = o0; j < o1; ++j) { // cell arcs to outputs (final: higher levels)
            const unsigned long long k = rkey[a.out_to[j]];
            if (k == kNoReq) continue;
            const double cand = key_double(k) - dcell;
            if (!found || cand < best) best = cand, found = true;
        }
    }
    a.req[t] = found ? best : a.clock;
    a.rk[t] = found ? 1 : 0;
    if (!found) return;
    const int j0 = a.in_start[t], j1 = a.in_start[t + 1];
    if (j1 > j0) {
        const double2 pt = a.pin_xy[t];
        const double cap = a.pin_cap[t];
        for (int j = j0; j < j1; ++j) {
            const int u = a.in_from[j];
            atomicMin(&rkey[u], double_key(best - net_delay(a.pin_xy[u], pt, cap, a.r, a.c)));
        }
    }
}

__global__ void __launch_bounds__(kBlock) k_req_decode(int n, const int* __restrict__ pins, StaArgs a,
                                                       const unsigned long long* __restrict__ rkey)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const int u = pins[i];
    const unsigned long long k = rkey[u];
    a.req[u] = k == kNoReq ? a.clock : key_double(k);
    a.rk[u] = k == kNoReq ? 0 : 1;
}

// ---- the push sweep in level-major L-space (default) --------------------------------------------
// Same arithmetic as k_arr_push / k_req_push / decodes above, on the level-major copy of the graph
// (session.cu): a level's Input pins are one contiguous L range, so every per-pin load and store of a
// launch is coalesced and only the driver / fan-out accesses remain gathers.  A final pass writes the
// results back to pin order (and maps pred / tie-list entries back to pin ids).
struct LArgs {
    const int *in_start, *in_from, *out_start, *out_to, *cell, *pin;
    const uint8_t* flags;
    const double *cap, *cell_delay;
    const double2 *off, *anchor;
    double2* xy;
    double r, c, clock;
    double *arr, *req;
    uint8_t *ak, *rk, *tie;
    int* pred;
    unsigned long long *akey, *rkey;
    int *tie_list, *counters;
};

__global__ void __launch_bounds__(kBlock) k_L_init(int P, LArgs a, bool from_cells, const double2* __restrict__ cell_xy,
                                                   const double2* __restrict__ pin_xy)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= P) return;
    if (from_cells) { // pin_positions (netlist.cpp:23-32)
        const int c = a.cell[i];
        const double2 o = a.off[i], b = c >= 0 ? cell_xy[c] : a.anchor[i];
        a.xy[i] = make_double2(b.x + o.x, b.y + o.y);
    } else {
        a.xy[i] = pin_xy[a.pin[i]];
    }
    const uint8_t f = a.flags[i];
    if (!(f & 4)) return; // keys are read and pushed for Output pins only (Input pins store arr / req)
    a.akey[i] = (f & 1) ? double_key(0.0) : kNoArr;
    a.rkey[i] = (f & 2) ? double_key(a.clock) : kNoReq;
}

// Levels after the first are launched as programmatic dependents of the previous level: only the
// session-constant graph tables (written at session setup, never by a kernel of the refresh) are loaded
// before pdl_wait(); this refresh's pin positions and keys after it.
__global__ void __launch_bounds__(kBlock) k_L_arr_push(int lo, int hi, LArgs a)
{
    pdl_trigger();
    const int t = lo + blockIdx.x * kBlock + threadIdx.x;
    if (t >= hi) return;
    const uint8_t fl = a.flags[t];
    const int j0 = a.in_start[t], j1 = a.in_start[t + 1], o0 = a.out_start[t], o1 = a.out_start[t + 1];
    const double cap = a.cap[t], dcell = o1 > o0 ? a.cell_delay[a.cell[t]] : 0.0;
    const int u0 = j1 > j0 ? a.in_from[j0] : 0;
    pdl_wait();
    const double2 pt = a.xy[t], xu0 = a.xy[u0];
    double best = 0.0;
    bool found = false;
    int bu = -1, ntie = 0;
    if (fl & 1) {
        found = true;
    } else {
        if (j1 > j0) {
            for (int j = j0; j < j1; ++j) {
                const int u = j == j0 ? u0 : a.in_from[j];
                const unsigned long long k = a.akey[u];
                if (k == kNoArr) continue;
                const double cand = key_double(k) + net_delay(j == j0 ? xu0 : a.xy[u], pt, cap, a.r, a.c);
                if (!found || cand > best) {
                    best = cand, found = true, bu = u, ntie = 1;
                } else if (cand == best) {
                    ++ntie;
                }
            }
        }
    }
    a.arr[t] = found ? best : 0.0;
    a.ak[t] = found ? 1 : 0;
    a.pred[t] = found ? bu : -1;
    if (ntie > 1) a.tie_list[atomicAdd(&a.counters[0], 1)] = t;
    if (!found) return;
    if (o1 > o0) {
        const unsigned long long k = double_key(best + dcell);
        for (int j = o0; j < o1; ++j) atomicMax(&a.akey[a.out_to[j]], k);
    }
}

__global__ void __launch_bounds__(kBlock) k_L_arr_decode(int P, LArgs a)
{
    pdl_trigger();
    pdl_wait();
    const int v = blockIdx.x * kBlock + threadIdx.x;
    if (v >= P) return;
    const uint8_t f = a.flags[v];
    if (!(f & 4)) return; // Input pins were stored by the push
    if (f & 1) {
        a.arr[v] = 0.0, a.ak[v] = 1, a.pred[v] = -1;
        return;
    }
    const unsigned long long k = a.akey[v];
    if (k == kNoArr) {
        a.arr[v] = 0.0, a.ak[v] = 0, a.pred[v] = -1;
        return;
    }
    const double best = key_double(k), dcell = a.cell_delay[a.cell[v]];
    int bu = -1, ntie = 0;
    for (int j = a.in_start[v]; j < a.in_start[v + 1]; ++j) {
        const int u = a.in_from[j];
        if (!a.ak[u]) continue;
        if (a.arr[u] + dcell == best) {
            if (bu < 0) bu = u;
            ++ntie;
        }
    }
    a.arr[v] = best, a.ak[v] = 1, a.pred[v] = bu;
    if (ntie > 1) a.tie_list[atomicAdd(&a.counters[0], 1)] = v;
}

__global__ void __launch_bounds__(kBlock) k_L_req_push(int lo, int hi, LArgs a)
{
    pdl_trigger();
    const int t = lo + blockIdx.x * kBlock + threadIdx.x;
    if (t >= hi) return;
    const uint8_t fl = a.flags[t];
    const int o0 = a.out_start[t], o1 = a.out_start[t + 1], j0 = a.in_start[t], j1 = a.in_start[t + 1];
    const double dcell = o1 > o0 ? a.cell_delay[a.cell[t]] : 0.0;
    const double cap = a.cap[t];
    const int v0 = o1 > o0 ? a.out_to[o0] : 0;
    pdl_wait();
    const double2 pt = a.xy[t];
    double best = INFINITY;
    bool found = false;
    if (fl & 2) best = a.clock, found = true;
    if (o1 > o0) {
        for (int j = o0; j < o1; ++j) {
            const unsigned long long k = a.rkey[j == o0 ? v0 : a.out_to[j]];
            if (k == kNoReq) continue;
            const double cand = key_double(k) - dcell;
            if (!found || cand < best) best = cand, found = true;
        }
    }
    a.req[t] = found ? best : a.clock;
    a.rk[t] = found ? 1 : 0;
    if (!found) return;
    if (j1 > j0) {
        for (int j = j0; j < j1; ++j) {
            const int u = a.in_from[j];
            atomicMin(&a.rkey[u], double_key(best - net_delay(a.xy[u], pt, cap, a.r, a.c)));
        }
    }
}

__global__ void __launch_bounds__(kBlock) k_L_req_decode(int P, LArgs a)
{
    pdl_trigger();
    pdl_wait();
    const int u = blockIdx.x * kBlock + threadIdx.x;
    if (u >= P || !(a.flags[u] & 4)) return;
    const unsigned long long k = a.rkey[u];
    a.req[u] = k == kNoReq ? a.clock : key_double(k);
    a.rk[u] = k == kNoReq ? 0 : 1;
}

// L-space results back to pin order; pred and tie-list entries become pin ids.
// (pin positions are rebuilt in pin order by the coalesced k_pin_xy instead of scattered from L_xy, and the
// per-pin tie flags are never read back: ties travel in tie_list)
__global__ void __launch_bounds__(kBlock) k_L_to_pins(int P, LArgs a, double* __restrict__ arr,
                                                      double* __restrict__ req, uint8_t* __restrict__ ak,
                                                      uint8_t* __restrict__ rk, int* __restrict__ pred)
{
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i < a.counters[0]) a.tie_list[i] = a.pin[a.tie_list[i]];
    if (i >= P) return;
    const int p = a.pin[i], q = a.pred[i];
    arr[p] = a.arr[i], req[p] = a.req[i], ak[p] = a.ak[i], rk[p] = a.rk[i];
    pred[p] = q >= 0 ? a.pin[q] : -1;
}

// Grid-wide barrier for the persistent STA (all blocks co-resident: cooperative launch).  Arrival
// counter + generation word; the last block to arrive resets the counter and bumps the generation.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == nblocks - 1) {
            bar[0] = 0;
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// The whole level sweep in one launch: pin positions, arrival levels ascending, required levels
// descending (sta.cpp:33-102), a grid barrier between dependent levels instead of a kernel boundary.
__global__ void __launch_bounds__(kBlock) k_sta_persist(StaArgs a, const int* __restrict__ lvl_start, int L, int P,
                                                        bool pin_xy_from_cells, const double2* __restrict__ off,
                                                        const double2* __restrict__ cell_xy,
                                                        const double2* __restrict__ anchor, unsigned* bar)
{
    const unsigned nb = gridDim.x;
    const int tid = blockIdx.x * kBlock + threadIdx.x, nt = gridDim.x * kBlock;
    if (pin_xy_from_cells) {
        for (int p = tid; p < P; p += nt)
            const_cast<double2*>(a.pin_xy)[p] = pin_pos(p, a.pin_cell, off, cell_xy, anchor);
        grid_barrier(bar, nb);
    }
    for (int l = 0; l < L; ++l) {
        const int lo = lvl_start[l], hi = lvl_start[l + 1];
        for (int i = lo + tid; i < hi; i += nt) arrival_pin(a.lvl_pins[i], a);
        grid_barrier(bar, nb);
    }
    for (int l = L - 1; l >= 0; --l) {
        const int lo = lvl_start[l], hi = lvl_start[l + 1];
        for (int i = lo + tid; i < hi; i += nt) required_pin(a.lvl_pins[i], a);
        if (l > 0) grid_barrier(bar, nb);
    }
}

// compute_slacks + endpoint keys (sta.cpp:104-133, paths.cpp:77-87): orderable slack keys
// over the pin-sorted endpoint list so a stable radix sort yields (slack, pin) order.
__global__ void __launch_bounds__(kBlock) k_slack_keys(int P, int EP, const double* __restrict__ arr,
                                                       const double* __restrict__ req, double* __restrict__ slack,
                                                       const int* __restrict__ ep_sorted,
                                                       unsigned long long* __restrict__ keys, int* __restrict__ vals,
                                                       double* __restrict__ part)
{
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[kBlock / 32];
    __shared__ double shm[kBlock / 32];
    __shared__ int shc[kBlock / 32];
    const int n = max(P, EP);
    double tns = 0.0, wns = 0.0;
    int nv = 0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) {
        if (i < P) slack[i] = req[i] - arr[i];
        if (i < EP) {
            const int e = ep_sorted[i];
            const double s = req[e] - arr[e];
            const bool viol = s < 0.0;
            keys[i] = viol ? double_key(s) : kNoKey;
            vals[i] = e;
            if (viol) tns += s, wns = fmin(wns, s), ++nv;
        }
    }
    const double bt = block_sum<kBlock>(tns, sh);
    // block min / count
    double m = wns;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    int c = nv;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) shm[w] = m, shc[w] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = 0.0;
        int cc = 0;
        for (int k = 0; k < kBlock / 32; ++k) mm = fmin(mm, shm[k]), cc += shc[k];
        part[3 * blockIdx.x] = bt, part[3 * blockIdx.x + 1] = mm, part[3 * blockIdx.x + 2] = cc;
    }
}

// k_slack_keys on the L-space results (engine refresh): endpoint keys only, the per-pin slack array is
// not written (sta_materialize_pins does it when a caller needs it).
__global__ void __launch_bounds__(kBlock) k_slack_keys_L(int EP, const int* __restrict__ ep_sorted,
                                                         const int* __restrict__ L_of,
                                                         const double* __restrict__ L_arr,
                                                         const double* __restrict__ L_req,
                                                         unsigned long long* __restrict__ keys, int* __restrict__ vals,
                                                         double* __restrict__ part)
{
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[kBlock / 32];
    __shared__ double shm[kBlock / 32];
    __shared__ int shc[kBlock / 32];
    double tns = 0.0, wns = 0.0;
    int nv = 0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < EP; i += gridDim.x * kBlock) {
        const int e = ep_sorted[i], u = L_of[e];
        const double s = L_req[u] - L_arr[u];
        const bool viol = s < 0.0;
        keys[i] = viol ? double_key(s) : kNoKey;
        vals[i] = e;
        if (viol) tns += s, wns = fmin(wns, s), ++nv;
    }
    const double bt = block_sum<kBlock>(tns, sh);
    double m = wns;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    int c = nv;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) shm[w] = m, shc[w] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = 0.0;
        int cc = 0;
        for (int k = 0; k < kBlock / 32; ++k) mm = fmin(mm, shm[k]), cc += shc[k];
        part[3 * blockIdx.x] = bt, part[3 * blockIdx.x + 1] = mm, part[3 * blockIdx.x + 2] = cc;
    }
}

__global__ void k_slack_all(int P, const double* __restrict__ arr, const double* __restrict__ req,
                            double* __restrict__ slack)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p < P) slack[p] = req[p] - arr[p];
}

__global__ void k_sta_final(int nb, const double* part, double* out3)
{
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[kBlock / 32];
    double t = 0.0, m = 0.0, c = 0.0;
    for (int i = threadIdx.x; i < nb; i += kBlock) t += part[3 * i], m = fmin(m, part[3 * i + 1]), c += part[3 * i + 2];
    t = block_sum<kBlock>(t, sh);
    c = block_sum<kBlock>(c, sh);
    __shared__ double mins[kBlock];
    mins[threadIdx.x] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        double mm = 0.0;
        for (int k = 0; k < kBlock; ++k) mm = fmin(mm, mins[k]);
        out3[0] = t, out3[1] = mm, out3[2] = c;
    }
}

// Exact delay ties: the enumerator prefers the lexicographically smallest full pin
// sequence (paths.hpp:63-69).  Tie pins are resolved in level order so every
// predecessor path is final when compared.  One block; tie pins are rare.
__device__ int materialize(const int* pred, int v, int* buf)
{
    int n = 0;
    for (int u = v; u >= 0; u = pred[u]) ++n;
    int k = n;
    for (int u = v; u >= 0; u = pred[u]) buf[--k] = u;
    return n;
}

__global__ void k_resolve_ties(StaArgs a, const int* __restrict__ level, int L, int* scratch, int stride)
{
    const int ntie = a.counters[0];
    if (ntie == 0) return;
    int* b1 = scratch + static_cast<long long>(threadIdx.x) * 2 * stride;
    int* b2 = b1 + stride;
    for (int l = 1; l < L; ++l) {
        for (int t = threadIdx.x; t < ntie; t += blockDim.x) {
            const int v = a.tie_list[t];
            if (level[v] != l) continue;
            const bool sink = a.pin_dir[v] == 0;
            const double2 pv = a.pin_xy[v];
            int bu = -1, nb = 0;
            for (int j = a.in_start[v]; j < a.in_start[v + 1]; ++j) {
                const int u = a.in_from[j];
                if (!a.ak[u]) continue;
                const double d = sink ? net_delay(a.pin_xy[u], pv, a.pin_cap[v], a.r, a.c)
                                      : a.cell_delay[a.pin_cell[v]];
                if (a.arr[u] + d != a.arr[v]) continue;
                const int n1 = materialize(a.pred, u, b1);
                b1[n1] = v;
                if (bu < 0) {
                    for (int k = 0; k <= n1; ++k) b2[k] = b1[k];
                    nb = n1 + 1, bu = u;
                    continue;
                }
                // lexicographic compare of b1[0..n1] vs b2[0..nb)
                const int m = min(n1 + 1, nb);
                int k = 0;
                while (k < m && b1[k] == b2[k]) ++k;
                const bool less = (k < m) ? (b1[k] < b2[k]) : (n1 + 1 < nb);
                if (less) {
                    for (int q = 0; q <= n1; ++q) b2[q] = b1[q];
                    nb = n1 + 1, bu = u;
                }
            }
            if (bu >= 0) a.pred[v] = bu;
        }
        __syncthreads();
    }
}

// k_resolve_ties on the L-space results: tie_list holds L indices, paths are compared by pin id.
__device__ int materialize_L(const int* L_pred, const int* L_pin, int v, int* buf)
{
    int n = 0;
    for (int u = v; u >= 0; u = L_pred[u]) ++n;
    int k = n;
    for (int u = v; u >= 0; u = L_pred[u]) buf[--k] = L_pin[u];
    return n;
}

__global__ void k_resolve_ties_L(LArgs a, const int* __restrict__ level, int L, int* scratch, int stride)
{
    const int ntie = a.counters[0];
    if (ntie == 0) return;
    int* b1 = scratch + static_cast<long long>(threadIdx.x) * 2 * stride;
    int* b2 = b1 + stride;
    for (int l = 1; l < L; ++l) {
        for (int t = threadIdx.x; t < ntie; t += blockDim.x) {
            const int v = a.tie_list[t];
            const int pv_id = a.pin[v];
            if (level[pv_id] != l) continue;
            const bool sink = !(a.flags[v] & 4);
            const double2 pv = a.xy[v];
            int bu = -1, nb = 0;
            for (int j = a.in_start[v]; j < a.in_start[v + 1]; ++j) {
                const int u = a.in_from[j];
                if (!a.ak[u]) continue;
                const double d = sink ? net_delay(a.xy[u], pv, a.cap[v], a.r, a.c) : a.cell_delay[a.cell[v]];
                if (a.arr[u] + d != a.arr[v]) continue;
                const int n1 = materialize_L(a.pred, a.pin, u, b1);
                b1[n1] = pv_id;
                if (bu < 0) {
                    for (int k = 0; k <= n1; ++k) b2[k] = b1[k];
                    nb = n1 + 1, bu = u;
                    continue;
                }
                const int m = min(n1 + 1, nb);
                int k = 0;
                while (k < m && b1[k] == b2[k]) ++k;
                const bool less = (k < m) ? (b1[k] < b2[k]) : (n1 + 1 < nb);
                if (less) {
                    for (int q = 0; q <= n1; ++q) b2[q] = b1[q];
                    nb = n1 + 1, bu = u;
                }
            }
            if (bu >= 0) a.pred[v] = bu;
        }
        __syncthreads();
    }
}

// Backtrace of the rank-0 path of each selected endpoint: pass 1 counts pins and
// net hops (hops leaving an Output pin, paths.cpp:195-200), pass 2 writes them.
// selected(): with nvp (the STA's [tns, wns, violated] on the device) only the first
// min(n_req or all, violated) of the n slots are paths; the rest get length 0.
__device__ __forceinline__ int selected(int n, const double* nvp, int n_req)
{
    if (!nvp) return n;
    const int nv = static_cast<int>(nvp[2]);
    return min(n, n_req <= 0 ? nv : min(n_req, nv));
}

__global__ void k_bt_count(int n, const int* __restrict__ ep, const int* __restrict__ pred,
                           const uint8_t* __restrict__ pin_dir, int* __restrict__ len, int* __restrict__ hops,
                           const double* __restrict__ nvp = nullptr, int n_req = 0)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    if (i >= selected(n, nvp, n_req)) {
        len[i] = 0, hops[i] = 0;
        return;
    }
    int v = ep[i], l = 1, h = 0;
    for (int u = pred[v]; u >= 0; v = u, u = pred[v]) {
        ++l;
        h += pin_dir[u] == 1;
    }
    len[i] = l, hops[i] = h;
}

// mark_pair(): the pair of a hop is its net arc, identified by the sink pin; the first hit of a pair
// sets its bit and counts it (collect_pin_pairs' unique set, paths.cpp:89-102)
__device__ __forceinline__ void mark_pair(unsigned* bits, int* uniq, int sink)
{
    if (!bits) return;
    const unsigned m = 1u << (sink & 31);
    if (!(atomicOr(&bits[sink >> 5], m) & m)) atomicAdd(uniq, 1);
}

__global__ void k_bt_write(int n, const int* __restrict__ ep, const int* __restrict__ pred,
                           const uint8_t* __restrict__ pin_dir, const int* __restrict__ len,
                           const int* __restrict__ off, const int* __restrict__ hops, const int* __restrict__ hoff,
                           const double* __restrict__ arr, double clock, int* __restrict__ pins,
                           double* __restrict__ pslack, unsigned long long* __restrict__ hkey,
                           double* __restrict__ hslack, int* __restrict__ hidx, unsigned* __restrict__ bits = nullptr,
                           int* __restrict__ uniq = nullptr)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n || len[i] == 0) return;
    int v = ep[i];
    const double sl = clock - arr[v]; // path slack = clock - rank-0 delay (paths.cpp:123)
    pslack[i] = sl;
    int k = off[i] + len[i] - 1;
    int h = hoff[i] + hops[i] - 1;
    pins[k] = v;
    for (int u = pred[v]; u >= 0; v = u, u = pred[v]) {
        pins[--k] = u;
        if (pin_dir[u] == 1) {
            const unsigned lo = static_cast<unsigned>(min(u, v)), hi = static_cast<unsigned>(max(u, v));
            hkey[h] = (static_cast<unsigned long long>(lo) << 32) | hi;
            hslack[h] = sl;
            hidx[h] = h;
            --h;
            mark_pair(bits, uniq, v);
        }
    }
}

// One-pass backtrace of the selected endpoints into fixed-stride slots (path i's pins end at
// pins[i S + S - 1], its hits at keys[i SH + SH - 1], both written from the endpoint backwards), with the
// path slack, lengths and unique-pair bits; k_bt_compact then packs the slots by the scanned lengths.
// Level-major predecessors when L_of is given (an L-space-only STA), per-pin ones otherwise.
__device__ __forceinline__ bool refresh_active(const double* sta_out, const Ctrl* ctrl)
{
    return !(ctrl && ctrl->stopped) && sta_out[1] < 0.0;
}

// With ctrl (the engine's refresh: every violated endpoint while the refresh is active) the hit key is
// the sink pin of a violated path (the dense ledger's key, pin_pairs.cpp:11), else the pair key.
__global__ void k_bt_walk(int ub, const int* __restrict__ ep, const double* __restrict__ nvp, int n_req,
                          const int* __restrict__ L_of, const int* __restrict__ L_pin, const int* __restrict__ pred,
                          const uint8_t* __restrict__ L_flags, const uint8_t* __restrict__ pin_dir,
                          const double* __restrict__ arr, double clock, int S, int SH, int* __restrict__ pins,
                          unsigned long long* __restrict__ keys, int* __restrict__ len, int* __restrict__ hops,
                          double* __restrict__ pslack, unsigned* __restrict__ bits, int* __restrict__ uniq,
                          const Ctrl* __restrict__ ctrl = nullptr)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= ub) return;
    if (i >= (ctrl ? (refresh_active(nvp, ctrl) ? static_cast<int>(nvp[2]) : 0) : selected(ub, nvp, n_req))) {
        len[i] = 0, hops[i] = 0;
        return;
    }
    const int e = ep[i];
    int v = L_of ? L_of[e] : e, vp = e;
    const double sl = clock - arr[v]; // paths.cpp:123
    pslack[i] = sl;
    int* pp = pins + static_cast<long long>(i) * S;
    unsigned long long* kk = keys + static_cast<long long>(i) * SH;
    int k = S - 1, kh = SH - 1;
    pp[k] = e;
    for (int u = pred[v]; u >= 0; v = u, u = pred[v]) {
        const int up = L_of ? L_pin[u] : u;
        pp[--k] = up;
        if (L_of ? (L_flags[u] & 4) != 0 : pin_dir[u] == 1) { // a hop leaving an Output pin (paths.cpp:195-200)
            const unsigned lo = static_cast<unsigned>(min(up, vp)), hi = static_cast<unsigned>(max(up, vp));
            kk[kh--] = ctrl ? (sl < 0.0 ? static_cast<unsigned>(vp) : 0xFFFFFFFFu)
                            : (static_cast<unsigned long long>(lo) << 32) | hi;
            mark_pair(bits, uniq, vp);
        }
        vp = up;
    }
    len[i] = S - k, hops[i] = SH - 1 - kh;
}

__global__ void k_bt_compact(int ub, int S, int SH, const int* __restrict__ pins,
                             const unsigned long long* __restrict__ keys, const int* __restrict__ len,
                             const int* __restrict__ off, const int* __restrict__ hops, const int* __restrict__ hoff,
                             const double* __restrict__ pslack, int* __restrict__ out_pins,
                             unsigned long long* __restrict__ hkey, double* __restrict__ hslack,
                             int* __restrict__ hidx, unsigned* __restrict__ hkey32 = nullptr,
                             const long long* __restrict__ n_dev = nullptr)
{
    // n_dev (the refresh): the selected paths are the first *n_dev sorted endpoints; a fixed grid
    // strides over their slots only
    const long long n = n_dev ? min(static_cast<long long>(ub), *n_dev) : ub;
    const long long end = n * S;
    for (long long t = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; t < end;
         t += static_cast<long long>(gridDim.x) * kBlock) {
        const int i = static_cast<int>(t / S), j = static_cast<int>(t - static_cast<long long>(i) * S);
        const int l = len[i];
        if (j < l) out_pins[off[i] + j] = pins[static_cast<long long>(i) * S + S - l + j];
        const int nh = hops[i];
        if (j < nh) {
            const int h = hoff[i] + j;
            const unsigned long long key = keys[static_cast<long long>(i) * SH + SH - nh + j];
            if (hkey32) hkey32[h] = static_cast<unsigned>(key);
            else hkey[h] = key;
            hslack[h] = pslack[i];
            hidx[h] = h;
        }
    }
}


// update_pair_weights (pin_pairs.cpp:7-15) over hits sorted stably by pair: one thread per
// group of equal pairs applies the group's additions in hit order; new pairs enter at w0.
__global__ void k_ledger_groups(long long H, const unsigned long long* __restrict__ hk, const int* __restrict__ hidx,
                                const double* __restrict__ hslack, const unsigned long long* __restrict__ led_key,
                                double* __restrict__ led_w, long long Q, double wns, double w0, double w1,
                                uint8_t* __restrict__ new_flag, double* __restrict__ new_w)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= H) return;
    const unsigned long long key = hk[i];
    new_flag[i] = 0;
    if (key == kNoKey || (i > 0 && hk[i - 1] == key)) return;
    long long lo = 0, hi = Q;
    while (lo < hi) {
        const long long mid = (lo + hi) >> 1;
        if (led_key[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    const bool found = lo < Q && led_key[lo] == key;
    double w = found ? led_w[lo] : w0;
    long long j = found ? i : i + 1;
    for (; j < H && hk[j] == key; ++j) w += w1 * (hslack[hidx[j]] / wns);
    if (found) led_w[lo] = w;
    else new_flag[i] = 1, new_w[i] = w;
}

__global__ void k_iota(long long n, int* out)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i < n) out[i] = static_cast<int>(i);
}

__global__ void k_host_hit_keys(long long n, const int* a, const int* b, const double* s, unsigned long long* key,
                                int* idx)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= n) return;
    key[i] = s[i] < 0.0 ? (static_cast<unsigned long long>(static_cast<unsigned>(a[i])) << 32) | static_cast<unsigned>(b[i])
                        : kNoKey;
    idx[i] = static_cast<int>(i);
}

// apply_net_weights (placer.cpp:262-273)
__global__ void k_net_weights(int N, const int* __restrict__ net_start, const int* __restrict__ net_pins,
                              const double* __restrict__ slack, double wns, double* __restrict__ w)
{
    const int e = blockIdx.x * kBlock + threadIdx.x;
    if (e >= N) return;
    double r = 1.0;
    if (wns < 0.0) {
        double worst = slack[net_pins[net_start[e]]];
        for (int j = net_start[e] + 1; j < net_start[e + 1]; ++j) worst = smin(worst, slack[net_pins[j]]);
        if (worst < 0.0) r = 1.0 + (-worst) / (-wns);
    }
    w[e] = r;
}

// ---------------------------------------------------------------------------------------
StaArgs sta_args(tdpg_session* s)
{
    StaArgs a;
    a.lvl_pins = s->lvl_pins, a.in_start = s->in_start, a.in_from = s->in_from, a.out_start = s->out_start;
    a.out_to = s->out_to, a.pin_cell = s->pin_cell, a.is_source = s->is_source, a.is_endpoint = s->is_endpoint;
    a.pin_dir = s->pin_dir, a.cell_delay = s->cell_delay, a.pin_cap = s->pin_cap, a.pin_xy = s->pin_xy;
    a.r = s->r_unit, a.c = s->c_unit, a.clock = s->clock, a.arr = s->arr, a.req = s->req, a.ak = s->ak, a.rk = s->rk;
    a.tie = s->tie, a.pred = s->pred, a.tie_list = s->tie_list, a.counters = s->counters;
    return a;
}

// TDPG_STA_PIN_ORDER=1: the push sweep on pin-indexed arrays (A/B switch for the L-space copy).
static bool pin_order_push()
{
    static const bool on = [] {
        const char* e = std::getenv("TDPG_STA_PIN_ORDER");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

// TDPG_STA_ALL_LEVELS=1: the plain pull sweep, one launch per level over every pin (A/B switch).
static bool all_levels_sweep()
{
    static const bool on = [] {
        const char* e = std::getenv("TDPG_STA_ALL_LEVELS");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

// Full STA at the current positions; leaves endpoint keys in sort_k0/sort_v0 and
// [tns, wns, n_violated] in out3. Stream-ordered, no host sync.  The 2L per-level launches are
// captured once into a CUDA graph (re-captured only if a buffer it uses moved).
// TDPG_STA_PDL=0: launch the level sweep without programmatic dependent launch
static bool sta_pdl()
{
    static const bool on = [] {
        const char* e = std::getenv("TDPG_STA_PDL");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

static LArgs make_largs(tdpg_session* s)
{
    LArgs la;
    la.in_start = s->L_in_start, la.in_from = s->L_in_from, la.out_start = s->L_out_start;
    la.out_to = s->L_out_to, la.cell = s->L_cell, la.pin = s->L_pin, la.flags = s->L_flags;
    la.cap = s->L_cap, la.cell_delay = s->cell_delay, la.off = s->L_off, la.anchor = s->L_anchor;
    la.xy = s->L_xy, la.r = s->r_unit, la.c = s->c_unit, la.clock = s->clock;
    la.arr = s->L_arr, la.req = s->L_req, la.ak = s->L_ak, la.rk = s->L_rk, la.tie = s->L_tie;
    la.pred = s->L_pred, la.akey = s->sta_akey, la.rkey = s->sta_rkey;
    la.tie_list = s->tie_list, la.counters = s->counters;
    return la;
}

// The L-space sweep is the default; pin_space = false (the engine's k = 1 refresh) leaves the results
// there: endpoint keys and TNS / WNS straight from L-space, no per-pin arrays (s->pins_stale).
static bool l_space_sweep() { return !all_levels_sweep() && !pin_order_push(); }

// Per-pin arrays of an L-space-only sweep (arr, req, known flags, pred, tie list as pins, pin
// positions, slack), for callers that read them.
void sta_materialize_pins(tdpg_session* s)
{
    if (!s->pins_stale) return;
    const int P = s->P;
    const unsigned nbP = blocks_for(std::max(P, 1), kBlock);
    k_L_to_pins<<<nbP, kBlock, 0, s->st>>>(P, make_largs(s), s->arr, s->req, s->ak, s->rk, s->pred);
    if (!s->pin_xy_external)
        k_pin_xy<<<nbP, kBlock, 0, s->st>>>(P, s->pin_cell, s->pin_off, s->cell_xy, s->anchor, s->pin_xy);
    k_slack_all<<<nbP, kBlock, 0, s->st>>>(P, s->arr, s->req, s->slack);
    CK_LAUNCH();
    s->pins_stale = false;
}

void sta_record(tdpg_session* s, double* out3, bool pin_space)
{
    const bool lonly = !pin_space && l_space_sweep() && s->sta_grid <= 0;
    s->pins_stale = lonly;
    const int P = s->P;
    const bool persist = s->sta_grid > 0;
    if (!s->pin_xy_external && !persist && all_levels_sweep()) { // pin positions from the cells (netlist.cpp:23-32) unless given
        k_pin_xy<<<blocks_for(P, kBlock), kBlock, 0, s->st>>>(P, s->pin_cell, s->pin_off, s->cell_xy, s->anchor,
                                                              s->pin_xy);
        CK_LAUNCH();
    }
    CK(cudaMemsetAsync(s->counters.p, 0, sizeof(int) * 4, s->st));
    const StaArgs a = sta_args(s);
    if (persist) { // one cooperative launch for the whole sweep, pin positions included
        CK(cudaMemsetAsync(s->grid_bar.p, 0, 2 * sizeof(unsigned), s->st));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(s->sta_grid), cfg.blockDim = dim3(kBlock), cfg.stream = s->st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative, attr[0].val.cooperative = 1;
        cfg.attrs = attr, cfg.numAttrs = 1;
        CK(cudaLaunchKernelEx(&cfg, k_sta_persist, a, static_cast<const int*>(s->lvl_start.p), s->L, P,
                              !s->pin_xy_external,
                              static_cast<const double2*>(s->pin_off.p), static_cast<const double2*>(s->cell_xy.p),
                              static_cast<const double2*>(s->anchor.p), s->grid_bar.p));
    } else if (!all_levels_sweep() && !pin_order_push()) { // L-space push sweep (default)
        const LArgs la = make_largs(s);
        const unsigned nbP = blocks_for(P, kBlock);
        k_L_init<<<nbP, kBlock, 0, s->st>>>(P, la, !s->pin_xy_external, s->cell_xy, s->pin_xy);
        const bool pdl = sta_pdl();
        // required times do not depend on arrival times (sta.cpp:69-102): the backward sweep runs on a
        // second stream beside the forward one (both are latency-bound level chains)
        CK(cudaEventRecord(s->ev_sta_fork, s->st));
        CK(cudaStreamWaitEvent(s->st_req, s->ev_sta_fork, 0));
        bool first = true;
        for (int l = 0; l < s->L; ++l) {
            const int lo = s->h_L_in_lo[l], hi = s->h_L_in_hi[l];
            if (hi > lo) CK(launch_pdl(k_L_arr_push, blocks_for(hi - lo, kBlock), kBlock, s->st, pdl && !first, lo, hi, la));
            first = first && !(hi > lo);
        }
        CK(launch_pdl(k_L_arr_decode, nbP, kBlock, s->st, pdl, P, la));
        first = true;
        for (int l = s->L - 1; l >= 0; --l) {
            const int lo = s->h_L_in_lo[l], hi = s->h_L_in_hi[l];
            if (hi > lo)
                CK(launch_pdl(k_L_req_push, blocks_for(hi - lo, kBlock), kBlock, s->st_req, pdl && !first, lo, hi, la));
            first = first && !(hi > lo);
        }
        CK(launch_pdl(k_L_req_decode, nbP, kBlock, s->st_req, pdl && !first, P, la));
        CK(cudaEventRecord(s->ev_sta_join, s->st_req));
        CK(cudaStreamWaitEvent(s->st, s->ev_sta_join, 0));
        if (!lonly) {
            CK(launch_pdl(k_L_to_pins, nbP, kBlock, s->st, pdl, P, la, s->arr.p, s->req.p, s->ak.p, s->rk.p,
                          s->pred.p));
            if (!s->pin_xy_external)
                CK(launch_pdl(k_pin_xy, nbP, kBlock, s->st, pdl, P, s->pin_cell.p, s->pin_off.p, s->cell_xy.p,
                              s->anchor.p, s->pin_xy.p));
        }
    } else if (!all_levels_sweep()) { // push sweep over sink levels in pin order (see k_arr_push)
        k_sta_init<<<blocks_for(P, kBlock), kBlock, 0, s->st>>>(P, a, !s->pin_xy_external, s->pin_off, s->cell_xy,
                                                                 s->anchor, s->sta_akey, s->sta_rkey);
        for (int l = 0; l < s->L; ++l) {
            const int lo = s->h_sta_in_start[l], hi = s->h_sta_in_start[l + 1];
            if (hi > lo) k_arr_push<<<blocks_for(hi - lo, kBlock), kBlock, 0, s->st>>>(lo, hi, s->sta_in_pins, a,
                                                                                        s->sta_akey);
        }
        const int n_out = s->h_sta_out_start[s->L];
        if (n_out) k_arr_decode<<<blocks_for(n_out, kBlock), kBlock, 0, s->st>>>(n_out, s->sta_out_pins, a, s->sta_akey);
        CK_LAUNCH();
        for (int l = s->L - 1; l >= 0; --l) {
            const int lo = s->h_sta_in_start[l], hi = s->h_sta_in_start[l + 1];
            if (hi > lo) k_req_push<<<blocks_for(hi - lo, kBlock), kBlock, 0, s->st>>>(lo, hi, s->sta_in_pins, a,
                                                                                        s->sta_rkey);
        }
        if (n_out) k_req_decode<<<blocks_for(n_out, kBlock), kBlock, 0, s->st>>>(n_out, s->sta_out_pins, a, s->sta_rkey);
        CK_LAUNCH();
    } else {
    for (int l = 0; l < s->L; ++l) {
        const int lo = s->h_lvl_start[l], hi = s->h_lvl_start[l + 1];
        if (hi > lo) k_arrival<<<blocks_for(hi - lo, kBlock), kBlock, 0, s->st>>>(lo, hi, a);
    }
    CK_LAUNCH();
    for (int l = s->L - 1; l >= 0; --l) {
        const int lo = s->h_lvl_start[l], hi = s->h_lvl_start[l + 1];
        if (hi > lo) k_required<<<blocks_for(hi - lo, kBlock), kBlock, 0, s->st>>>(lo, hi, a);
    }
    CK_LAUNCH();
    }
    const int nb = std::max(1, std::min(148 * 4, static_cast<int>(blocks_for(std::max(P, s->EP), kBlock))));
    const bool pdl = sta_pdl();
    if (lonly)
        CK(launch_pdl(k_slack_keys_L, nb, kBlock, s->st, pdl, s->EP, s->ep_sorted.p, s->L_of.p, s->L_arr.p,
                      s->L_req.p, s->sort_k0.p, s->sort_v0.p, s->sta_part.p));
    else
        CK(launch_pdl(k_slack_keys, nb, kBlock, s->st, pdl, P, s->EP, s->arr.p, s->req.p, s->slack.p,
                      s->ep_sorted.p, s->sort_k0.p, s->sort_v0.p, s->sta_part.p));
    CK(launch_pdl(k_sta_final, 1, kBlock, s->st, pdl, nb, s->sta_part.p, out3));
}

// Size the persistent STA for co-residency (every block resident at once, cooperative launch).
// Opt-in (TDPG_STA_PERSIST=1): measured on B200 at 1M cells it is slower than one launch per level
// (1.32-1.68 ms vs 1.12 ms: the level sweep is bound by dependent gathers, not by launch gaps, and
// the co-resident grid holds fewer loads in flight than a full grid per level).
void sta_setup(tdpg_session* s)
{
    s->sta_grid = 0;
    const char* e = std::getenv("TDPG_STA_PERSIST");
    if (!(e && std::atoi(e) != 0)) return;
    int coop = 0, sms = 0, per_sm = 0;
    CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, s->device));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sta_persist, kBlock, 0));
    if (!coop || per_sm < 1) return;
    s->grid_bar.alloc(2);
    const char* b = std::getenv("TDPG_STA_BLOCKS_PER_SM");
    s->sta_grid = sms * std::max(1, std::min(per_sm, b ? std::atoi(b) : 2));
}

void run_sta_async(tdpg_session* s, double* out3, bool pin_space)
{
    const size_t ep = static_cast<size_t>(std::max(s->EP, 1));
    s->sort_k0.reserve(ep), s->sort_k1.reserve(ep), s->sort_v0.reserve(ep), s->sort_v1.reserve(ep);
    const int nb = std::max(1, std::min(148 * 4, static_cast<int>(blocks_for(std::max(s->P, s->EP), kBlock))));
    s->sta_part.reserve(3 * nb + 8);
    // the graph bakes buffer pointers and the constraints (kernel arguments) in: re-capture on any change
    auto bits = [](double x) { uint64_t u; std::memcpy(&u, &x, sizeof u); return u; };
    auto ptr = [](const void* p) { return static_cast<uint64_t>(reinterpret_cast<uintptr_t>(p)); };
    const std::array<uint64_t, 9> key = {ptr(s->pin_xy_external ? s->pin_xy.p : nullptr), ptr(s->cell_xy.p),
                                         ptr(s->sort_k0.p), ptr(s->sort_v0.p), ptr(s->sta_part.p), ptr(out3),
                                         bits(s->clock), bits(s->r_unit), bits(s->c_unit)};
    const bool lonly = !pin_space && l_space_sweep() && s->sta_grid <= 0;
    cudaGraphExec_t& gx = lonly ? s->sta_gexec_L : s->sta_gexec;
    std::array<uint64_t, 9>& gk = lonly ? s->sta_graph_key_L : s->sta_graph_key;
    if (!gx || key != gk) {
        if (gx) cudaGraphExecDestroy(gx), gx = nullptr;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(s->st, cudaStreamCaptureModeThreadLocal));
        sta_record(s, out3, !lonly);
        CK(cudaStreamEndCapture(s->st, &g));
        CK(cudaGraphInstantiate(&gx, g, 0));
        cudaGraphDestroy(g);
        gk = key;
    }
    CK(cudaGraphLaunch(gx, s->st));
    s->pins_stale = lonly;
}

void run_sta_dev(tdpg_session* s, bool pin_space)
{
    s->sta_out.reserve(4);
    run_sta_async(s, s->sta_out, pin_space);
    double h[3];
    s->sta_out.download(h, 3, s->st);
    CK(cudaStreamSynchronize(s->st));
    s->tns = h[0], s->wns = h[1];
    s->sta_valid = true;
    s->ties_resolved = false;
}

// Exact-delay ties of the last STA resolved to the lexicographically smallest path (idempotent).
void resolve_ties_dev(tdpg_session* s)
{
    sta_materialize_pins(s);
    if (s->ties_resolved) return;
    const int stride = s->L + 2;
    s->tie_scratch.reserve(static_cast<size_t>(kBlock) * 2 * stride);
    k_resolve_ties<<<1, kBlock, 0, s->st>>>(sta_args(s), s->d_level, s->L, s->tie_scratch, stride);
    CK_LAUNCH();
    s->ties_resolved = true;
}

// After a stable radix sort on the upper 32 bits of the endpoint keys: each run of equal upper halves among
// the first nv entries (the violated endpoints) is re-sorted by the full key with a stable insertion sort by
// the thread at its start, so the order is exactly the 64-bit stable sort's (slack, then pin).  Runs are a few
// entries (the upper half keeps ~6 significant digits of the slack).
__global__ void k_ep_fixup(const long long* __restrict__ nv_ptr, const double* __restrict__ nv_d,
                           unsigned long long* __restrict__ keys, int* __restrict__ vals)
{
    const long long nv = nv_ptr ? *nv_ptr : static_cast<long long>(nv_d[2]); // (sta_out[2]: violated count)
    for (long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; i + 1 < nv;
         i += static_cast<long long>(gridDim.x) * kBlock) {
        const unsigned hi = static_cast<unsigned>(keys[i] >> 32);
        if ((i > 0 && static_cast<unsigned>(keys[i - 1] >> 32) == hi) || static_cast<unsigned>(keys[i + 1] >> 32) != hi)
            continue; // not the start of a run of two or more
        long long e = i + 2;
        while (e < nv && static_cast<unsigned>(keys[e] >> 32) == hi) ++e;
        for (long long j = i + 1; j < e; ++j) { // stable: only strictly greater keys move
            const unsigned long long k = keys[j];
            const int v = vals[j];
            long long q = j - 1;
            while (q >= i && keys[q] > k) keys[q + 1] = keys[q], vals[q + 1] = vals[q], --q;
            keys[q + 1] = k, vals[q + 1] = v;
        }
    }
}

// TDPG_EP_SORT64=1: the endpoint sort over all 64 key bits (8 radix passes) instead of the upper 32 bits and
// the run fix-up (4 passes + one kernel); A/B switch.
bool ep_sort64()
{
    static const bool on = [] {
        const char* e = std::getenv("TDPG_EP_SORT64");
        return e && std::atoi(e) != 0;
    }();
    return on;
}

// violated_endpoints (paths.cpp:77-87) of the current STA: (slack, pin) order in sort_v1; returns
// how many endpoints violate.
int sorted_violated(tdpg_session* s)
{
    sta_materialize_pins(s);
    s->sta_out.reserve(4);
    double* out3 = s->sta_out.p;
    const int P = s->P;
    const int nb = std::max(1, std::min(148 * 4, static_cast<int>(blocks_for(std::max(P, s->EP), kBlock))));
    s->part.reserve(3 * nb + 8);
    const size_t ep = static_cast<size_t>(std::max(s->EP, 1));
    s->sort_k0.reserve(ep), s->sort_k1.reserve(ep), s->sort_v0.reserve(ep), s->sort_v1.reserve(ep);
    k_slack_keys<<<nb, kBlock, 0, s->st>>>(P, s->EP, s->arr, s->req, s->slack, s->ep_sorted, s->sort_k0, s->sort_v0,
                                           s->part);
    CK_LAUNCH();
    k_sta_final<<<1, kBlock, 0, s->st>>>(nb, s->part, out3);
    CK_LAUNCH();
    if (s->EP > 0) {
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, s->sort_k0.p, s->sort_k1.p, s->sort_v0.p, s->sort_v1.p, s->EP,
                                        0, 64, s->st);
        void* tmp = cub_scratch(s, bytes);
        const int lo_bit = ep_sort64() ? 0 : 32; // (upper halves, then the exact run fix-up)
        CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, s->sort_k0.p, s->sort_k1.p, s->sort_v0.p, s->sort_v1.p, s->EP,
                                           lo_bit, 64, s->st));
        if (lo_bit) {
            k_ep_fixup<<<std::max<unsigned>(1, std::min<unsigned>(blocks_for(s->EP, kBlock), 148 * 4)), kBlock, 0,
                         s->st>>>(nullptr, out3, s->sort_k1.p, s->sort_v1.p);
            CK_LAUNCH();
        }
    }
    double h[3];
    CK(cudaMemcpyAsync(h, out3, sizeof h, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    return static_cast<int>(h[2]);
}

static int bits_for(long long n);

// report_timing_endpoint(n, k = 1) on the current STA (paths.cpp:167-189).
void extract_endpoint_dev(tdpg_session* s, int n)
{
    if (!s->sta_valid) run_sta_dev(s, false);
    const bool Lsp = s->pins_stale; // the sweep's results are in L-space (no per-pin arrays)
    // exact ties first (the backtrace reads the resolved predecessors; host-side state, outside the graph)
    if (!Lsp) {
        resolve_ties_dev(s);
    } else if (!s->ties_resolved) {
        const int stride = s->L + 2;
        s->tie_scratch.reserve(static_cast<size_t>(kBlock) * 2 * stride);
        k_resolve_ties_L<<<1, kBlock, 0, s->st>>>(make_largs(s), s->d_level, s->L, s->tie_scratch, stride);
        CK_LAUNCH();
        s->ties_resolved = true;
    }
    const int EP = s->EP, P = s->P;
    // the selection size min(n, violated) stays on the device: the backtrace runs over an upper bound of
    // slots (zero-length past the selection), one host read brings back every count
    const int ub = (n <= 0) ? EP : std::min(n, EP);
    s->n_paths = 0, s->n_path_pins = 0, s->n_hits = 0, s->uniq_pairs = 0, s->uniq_endpoints = 0, s->candidates = 0;
    if (ub <= 0) return;
    // endpoint keys, the (slack, pin) sort, the backtrace lengths and their scans: a fixed-size sequence
    // of ~17 launches, replayed as one graph (re-captured when n, the STA form or any buffer changes)
    s->sta_out.reserve(4);
    double* out3 = s->sta_out.p;
    const int nb = std::max(1, std::min(148 * 4, static_cast<int>(blocks_for(std::max(P, EP), kBlock))));
    s->part.reserve(3 * nb + 8);
    const size_t ep = static_cast<size_t>(std::max(EP, 1));
    s->sort_k0.reserve(ep), s->sort_k1.reserve(ep), s->sort_v0.reserve(ep), s->sort_v1.reserve(ep);
    s->ex_len.reserve(ub), s->ex_hops.reserve(ub), s->ex_off.reserve(ub), s->ex_hoff.reserve(ub);
    s->ex_slack.reserve(ub);
    const int S = s->L + 1, SH = s->L / 2 + 2; // pins per path <= levels, hits <= Output pins on it
    s->ex_tmp_pins.reserve(static_cast<size_t>(ub) * S), s->ex_tmp_keys.reserve(static_cast<size_t>(ub) * SH);
    const size_t nbits = static_cast<size_t>(P) / 32 + 1;
    s->pair_bits.reserve(nbits);
    size_t b_sort = 0, b_scan = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b_sort, s->sort_k0.p, s->sort_k1.p, s->sort_v0.p, s->sort_v1.p, EP, 0,
                                    64, s->st);
    cub::DeviceScan::ExclusiveSum(nullptr, b_scan, s->ex_len.p, s->ex_off.p, ub, s->st);
    cub_scratch(s, std::max(b_sort, b_scan));
    const std::array<long long, 4> key = {n, ub, Lsp ? 1 : 0, static_cast<long long>(dbuf_epoch())};
    auto record = [&] {
        if (Lsp)
            k_slack_keys_L<<<nb, kBlock, 0, s->st>>>(EP, s->ep_sorted, s->L_of, s->L_arr, s->L_req, s->sort_k0,
                                                     s->sort_v0, s->part);
        else
            k_slack_keys<<<nb, kBlock, 0, s->st>>>(P, EP, s->arr, s->req, s->slack, s->ep_sorted, s->sort_k0,
                                                   s->sort_v0, s->part);
        k_sta_final<<<1, kBlock, 0, s->st>>>(nb, s->part, out3);
        size_t bytes = s->cub_tmp.n;
        const int lo_bit = ep_sort64() ? 0 : 32; // (upper halves, then the exact run fix-up)
        CK(cub::DeviceRadixSort::SortPairs(s->cub_tmp.p, bytes, s->sort_k0.p, s->sort_k1.p, s->sort_v0.p,
                                           s->sort_v1.p, EP, lo_bit, 64, s->st));
        if (lo_bit) {
            k_ep_fixup<<<std::max<unsigned>(1, std::min<unsigned>(blocks_for(EP, kBlock), 148 * 4)), kBlock, 0,
                         s->st>>>(nullptr, out3, s->sort_k1.p, s->sort_v1.p);
            CK_LAUNCH();
        }
        CK(cudaMemsetAsync(s->pair_bits.p, 0, nbits * sizeof(unsigned), s->st));
        CK(cudaMemsetAsync(s->counters.p + 1, 0, sizeof(int), s->st));
        k_bt_walk<<<blocks_for(ub, kBlock), kBlock, 0, s->st>>>(
            ub, s->sort_v1, out3, n, Lsp ? s->L_of.p : nullptr, s->L_pin, Lsp ? s->L_pred.p : s->pred.p, s->L_flags,
            s->pin_dir, Lsp ? s->L_arr.p : s->arr.p, s->clock, S, SH, s->ex_tmp_pins, s->ex_tmp_keys, s->ex_len,
            s->ex_hops, s->ex_slack, s->pair_bits, s->counters.p + 1);
        bytes = s->cub_tmp.n;
        CK(cub::DeviceScan::ExclusiveSum(s->cub_tmp.p, bytes, s->ex_len.p, s->ex_off.p, ub, s->st));
        bytes = s->cub_tmp.n;
        CK(cub::DeviceScan::ExclusiveSum(s->cub_tmp.p, bytes, s->ex_hops.p, s->ex_hoff.p, ub, s->st));
    };
    if (!s->ex_gexec || key != s->ex_key) {
        if (s->ex_gexec) cudaGraphExecDestroy(s->ex_gexec), s->ex_gexec = nullptr;
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(s->st, cudaStreamCaptureModeThreadLocal));
        record();
        CK(cudaStreamEndCapture(s->st, &g));
        CK(cudaGraphInstantiate(&s->ex_gexec, g, 0));
        cudaGraphDestroy(g);
        s->ex_key = key;
    }
    CK(cudaGraphLaunch(s->ex_gexec, s->st));
    int tail[5];
    double h3[3];
    CK(cudaMemcpyAsync(h3, out3, sizeof h3, cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(&tail[4], s->counters.p + 1, sizeof(int), cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(&tail[0], s->ex_off.p + ub - 1, sizeof(int), cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(&tail[1], s->ex_len.p + ub - 1, sizeof(int), cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(&tail[2], s->ex_hoff.p + ub - 1, sizeof(int), cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(&tail[3], s->ex_hops.p + ub - 1, sizeof(int), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    const int nv = static_cast<int>(h3[2]);
    const int np = (n <= 0) ? nv : std::min(n, nv);
    s->n_paths = np;
    s->uniq_endpoints = np, s->candidates = np; // k = 1: one path per selected endpoint
    if (np == 0) return;
    s->n_path_pins = static_cast<long long>(tail[0]) + tail[1];
    s->n_hits = static_cast<long long>(tail[2]) + tail[3];
    const long long H = s->n_hits;
    s->ex_pins.reserve(s->n_path_pins + 1);
    s->hit_key.reserve(H + 1), s->hit_slack.reserve(H + 1), s->hit_idx.reserve(H + 1);
    s->hit_key_s.reserve(H + 1), s->hit_idx_s.reserve(H + 1);
    // pack the fixed-stride slots (coalesced; the unique pairs were counted by the walk)
    k_bt_compact<<<blocks_for(static_cast<long long>(np) * S, kBlock), kBlock, 0, s->st>>>(
        np, S, SH, s->ex_tmp_pins, s->ex_tmp_keys, s->ex_len, s->ex_off, s->ex_hops, s->ex_hoff, s->ex_slack,
        s->ex_pins, s->hit_key, s->hit_slack, s->hit_idx);
    CK_LAUNCH();
    s->uniq_pairs = H > 0 ? tail[4] : 0;
    s->hits_sorted = false; // (sorted by ledger_update_dev when the ledger takes them)
}

// Apply the last sorted hits (hit_key_s / hit_idx_s / hit_slack) to the ledger.
void ledger_apply_sorted(tdpg_session* s, long long H, double wns, double w0, double w1)
{
    if (!(wns < 0.0) || H == 0) return;
    s->lg_flag.reserve(H), s->lg_w.reserve(H), s->lg_new_k.reserve(H), s->lg_new_w.reserve(H), s->lg_nsel.reserve(2);
    DBuf<uint8_t>& flag = s->lg_flag;
    DBuf<double>& nw = s->lg_w;
    const long long Q = s->Q;
    k_ledger_groups<<<blocks_for(H, kBlock), kBlock, 0, s->st>>>(H, s->hit_key_s, s->hit_idx_s, s->hit_slack,
                                                                 s->led_key, s->led_w, Q, wns, w0, w1, flag, nw);
    CK_LAUNCH();
    DBuf<unsigned long long>& new_k = s->lg_new_k;
    DBuf<double>& new_w = s->lg_new_w;
    DBuf<int>& n_sel = s->lg_nsel;
    size_t bytes = 0;
    cub::DeviceSelect::Flagged(nullptr, bytes, s->hit_key_s.p, flag.p, new_k.p, n_sel.p, static_cast<int>(H), s->st);
    void* tmp = cub_scratch(s, bytes);
    CK(cub::DeviceSelect::Flagged(tmp, bytes, s->hit_key_s.p, flag.p, new_k.p, n_sel.p, static_cast<int>(H), s->st));
    CK(cub::DeviceSelect::Flagged(tmp, bytes, nw.p, flag.p, new_w.p, n_sel.p, static_cast<int>(H), s->st));
    int M = 0;
    CK(cudaMemcpyAsync(&M, n_sel.p, sizeof(int), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    if (M == 0) return;
    const long long nq = Q + M;
    s->led_key2.reserve(nq), s->led_w2.reserve(nq);
    if (Q == 0) {
        CK(cudaMemcpyAsync(s->led_key2.p, new_k.p, M * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s->st));
        CK(cudaMemcpyAsync(s->led_w2.p, new_w.p, M * sizeof(double), cudaMemcpyDeviceToDevice, s->st));
    } else {
        bytes = 0;
        cub::DeviceMerge::MergePairs(nullptr, bytes, s->led_key.p, s->led_w.p, static_cast<int>(Q), new_k.p, new_w.p,
                                     M, s->led_key2.p, s->led_w2.p, ::cuda::std::less<>{}, s->st);
        tmp = cub_scratch(s, bytes);
        CK(cub::DeviceMerge::MergePairs(tmp, bytes, s->led_key.p, s->led_w.p, static_cast<int>(Q), new_k.p, new_w.p, M,
                                        s->led_key2.p, s->led_w2.p, ::cuda::std::less<>{}, s->st));
    }
    // copy back (not swap): the iteration graph holds the ledger pointers
    s->led_key.reserve(nq), s->led_w.reserve(nq);
    CK(cudaMemcpyAsync(s->led_key.p, s->led_key2.p, nq * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s->st));
    CK(cudaMemcpyAsync(s->led_w.p, s->led_w2.p, nq * sizeof(double), cudaMemcpyDeviceToDevice, s->st));
    s->Q = nq;
    s->pp_dirty = true;
}

void ledger_update_dev(tdpg_session* s, double wns, double w0, double w1, bool)
{
    const long long H = s->n_hits;
    if (!s->hits_sorted && H > 0) { // stable sort of the hits by pair (update_pair_weights order per pair)
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, s->hit_key.p, s->hit_key_s.p, s->hit_idx.p, s->hit_idx_s.p,
                                        static_cast<int>(H), 0, 64, s->st);
        void* tmp = cub_scratch(s, bytes);
        CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, s->hit_key.p, s->hit_key_s.p, s->hit_idx.p, s->hit_idx_s.p,
                                           static_cast<int>(H), 0, 64, s->st));
        s->hits_sorted = true;
    }
    ledger_apply_sorted(s, H, wns, w0, w1);
}

void net_weights_dev(tdpg_session* s)
{
    s->net_w.reserve(std::max(s->N, 1));
    k_net_weights<<<blocks_for(s->N, kBlock), kBlock, 0, s->st>>>(s->N, s->net_start, s->net_pins.p,
                                                                  s->slack, s->wns, s->net_w);
    CK_LAUNCH();
}

// =====================================================================================
// Engine-mode timing refresh (placer.cpp:415-435) with no host round trip: every size comes from
// device memory, every launch is sized for its capacity (endpoints, endpoints x levels), so the
// whole refresh is captured once as a CUDA graph.  The reference skips extraction and the ledger
// when wns >= 0; here the kernels read wns (sta_out[1]) and exit.
// =====================================================================================

__global__ void k_refresh_begin(const double* sta_out, Ctrl* ctrl, double* timing_row)
{
    if (ctrl->stopped) return;
    timing_row[0] = 1.0, timing_row[1] = sta_out[0], timing_row[2] = sta_out[1];
    ctrl->engaged = 1;
}

__global__ void k_bt_count_dev(int EP, const double* __restrict__ sta_out, const Ctrl* __restrict__ ctrl,
                               const int* __restrict__ ep, const int* __restrict__ pred,
                               const uint8_t* __restrict__ pin_dir, int* __restrict__ len, int* __restrict__ hops)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= EP) return;
    const int n_paths = refresh_active(sta_out, ctrl) ? static_cast<int>(sta_out[2]) : 0;
    if (i >= n_paths) {
        len[i] = 0, hops[i] = 0;
        return;
    }
    int v = ep[i], l = 1, h = 0;
    for (int u = pred[v]; u >= 0; v = u, u = pred[v]) ++l, h += pin_dir[u] == 1;
    len[i] = l, hops[i] = h;
}

// Paths into the capacity buffers; one hit per hop leaving an Output pin keyed by the hop's sink
// pin (each pair is a net arc: the sink identifies it), tagged with the path slack.
__global__ void k_bt_write_dev(int EP, const double* __restrict__ sta_out, const Ctrl* __restrict__ ctrl,
                               const int* __restrict__ ep, const int* __restrict__ pred,
                               const uint8_t* __restrict__ pin_dir, const int* __restrict__ len,
                               const int* __restrict__ off, const int* __restrict__ hops, const int* __restrict__ hoff,
                               const double* __restrict__ arr, double clock, int* __restrict__ pins,
                               double* __restrict__ pslack, unsigned* __restrict__ hkey,
                               double* __restrict__ hslack, int* __restrict__ hidx)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= EP || len[i] == 0) return;
    int v = ep[i];
    const double sl = clock - arr[v]; // paths.cpp:123
    pslack[i] = sl;
    int k = off[i] + len[i] - 1, h = hoff[i] + hops[i] - 1;
    pins[k] = v;
    for (int u = pred[v]; u >= 0; v = u, u = pred[v]) {
        pins[--k] = u;
        if (pin_dir[u] == 1) {
            hkey[h] = sl < 0.0 ? static_cast<unsigned>(v) : 0xFFFFFFFFu; // pin_pairs.cpp:11
            hslack[h] = sl;
            hidx[h] = h;
            --h;
        }
    }
}

__global__ void k_fill_u32(long long n, unsigned* p, unsigned v)
{
    for (long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * kBlock)
        p[i] = v;
}

// The pad past the packed hits up to the largest size class switch_by_count can pick for them:
// the smallest class >= nh is at most max(cap/64, 4 nh).
__global__ void k_fill_hit_pad(long long cap, const long long* __restrict__ n_hits, unsigned* p)
{
    const long long nh = min(cap, *n_hits), end = min(cap, max(cap >> 6, 4 * nh));
    for (long long i = nh + blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; i < end;
         i += static_cast<long long>(gridDim.x) * kBlock)
        p[i] = 0xFFFFFFFFu;
}

// update_pair_weights (pin_pairs.cpp:7-15) on the dense ledger: hits sorted stably by sink pin, so a
// pair's hits are one contiguous run in hit order and its weight is the serial sum over that run (kept
// serial: bitwise the reference's left-to-right additions).  Two kernels on two graph branches:
//  * k_ledger_dense: a run of at most kLedRun hits is summed by the thread at its start — run length
//    first (keys of one L1 line), then every term's gathers issued together, then the adds;
//  * k_ledger_long: longer runs (a pin shared by thousands of critical paths; one thread walking one
//    took 1.7 ms of a 1M refresh).  Each block scans a slice of the hits for long-run starts and sums
//    each such run cooperatively: 256 terms gathered and scaled in parallel (double-buffered), one
//    thread adding them in order.  Its critical path is the longest run's add chain, overlapped with
//    the short runs on the other branch.
constexpr int kLedRun = 32;
constexpr int kLedBlock = 256;
constexpr int kLedLongBlocks = 148 * 2;

__device__ __forceinline__ void ledger_store(const LedgerArgs& a, int v, double w, bool fresh)
{
    a.dl_w[v] = w;
    a.ppw_e[a.pin_entry[v]] = w;
    // new pairs counted with one atomic per warp (every thread of a first refresh adds one)
    const unsigned act = __activemask(), fm = __ballot_sync(act, fresh);
    if (fresh) {
        const int loc = a.pin_loc[v];
        if (loc >= 0) atomicOr(&a.pp_mask[loc >> 3], 1u << (loc & 7));
        if ((threadIdx.x & 31) == __ffs(fm) - 1) atomicAdd(a.q_count, static_cast<unsigned long long>(__popc(fm)));
    }
}

__device__ __forceinline__ long long ledger_hits(const LedgerArgs& a)
{
    return a.n_hits ? *a.n_hits : a.H;
}

__device__ __forceinline__ bool ledger_active(const LedgerArgs& a)
{
    return a.gen ? !(a.ctrl->stopped) && a.sta_out[1] < 0.0 : refresh_active(a.sta_out, a.ctrl);
}

__device__ __forceinline__ bool ledger_long_start(const unsigned* hk, long long i, long long H, unsigned& key)
{
    key = hk[i];
    return key != 0xFFFFFFFFu && (i == 0 || hk[i - 1] != key) && i + kLedRun < H && hk[i + kLedRun] == key;
}

__global__ void k_ledger_dense(long long cap, LedgerArgs a)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= cap || !ledger_active(a)) return;
    const long long H = ledger_hits(a); // (only the hits are sorted; the tail past them is stale)
    if (i >= H) return;
    const unsigned key = a.hk[i];
    if (key == 0xFFFFFFFFu || (i > 0 && a.hk[i - 1] == key)) return;
    int n = 1; // run length, at most kLedRun here (longer runs: k_ledger_long)
    while (n <= kLedRun && i + n < H && a.hk[i + n] == key) ++n;
    if (n > kLedRun) return;
    const double wns = a.sta_out[1];
    const int v = static_cast<int>(key);
    double w = a.dl_w[v];
    const bool fresh = !(w > 0.0); // weights start at w0 > 0 and never decrease
    int k = 0;
    if (fresh) w = a.w0, k = 1;
    for (; k < n; k += 8) { // eight terms' gathers in flight, then their adds in hit order
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = k + u < n ? a.hslack[a.hidx[i + k + u]] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (k + u < n) w += a.w1 * (t[u] / wns);
    }
    ledger_store(a, v, w, fresh);
}

__global__ void __launch_bounds__(kLedBlock) k_ledger_long(LedgerArgs a)
{
    __shared__ double term[2][kLedBlock];
    __shared__ long long found[kLedBlock];
    __shared__ int n_found;
    if (!ledger_active(a)) return;
    const long long H = ledger_hits(a);
    const double wns = a.sta_out[1];
    const int t = threadIdx.x;
    const long long slice = (H + gridDim.x - 1) / gridDim.x;
    const long long lo = blockIdx.x * slice, hi = H < lo + slice ? H : lo + slice;
    for (long long b0 = lo; b0 < hi; b0 += kLedBlock) {
        if (t == 0) n_found = 0;
        __syncthreads();
        unsigned key;
        if (b0 + t < hi && ledger_long_start(a.hk, b0 + t, H, key)) found[atomicAdd(&n_found, 1)] = b0 + t;
        __syncthreads();
        const int nf = n_found;
        for (int f = 0; f < nf; ++f) { // (the order among runs does not matter: disjoint keys)
            const long long i = found[f];
            key = a.hk[i];
            const int v = static_cast<int>(key);
            double w = a.dl_w[v]; // (read by every thread; only thread 0 uses it)
            const bool fresh = !(w > 0.0);
            if (fresh) w = a.w0;
            long long base = fresh ? i + 1 : i;
            auto gather = [&](long long bb, bool& in) {
                const long long j = bb + t;
                in = j < H && a.hk[j] == key; // (the run is contiguous: the lanes in it are a prefix)
                return in ? a.w1 * (a.hslack[a.hidx[j]] / wns) : 0.0;
            };
            bool in;
            term[0][t] = gather(base, in);
            int n = __syncthreads_count(in), cur = 0;
            for (;;) {
                const bool more = n == kLedBlock;
                double nxt = 0.0;
                bool in2 = false;
                if (more) nxt = gather(base + kLedBlock, in2); // next chunk in flight while thread 0 adds
                if (t == 0) {
                    int k = 0;
                    for (; k + 8 <= n; k += 8) {
                        double r[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) r[u] = term[cur][k + u];
#pragma unroll
                        for (int u = 0; u < 8; ++u) w += r[u];
                    }
                    for (; k < n; ++k) w += term[cur][k];
                }
                if (!more) break; // (block-uniform)
                term[cur ^ 1][t] = nxt;
                n = __syncthreads_count(in2);
                base += kLedBlock, cur ^= 1;
            }
            if (t == 0) ledger_store(a, v, w, fresh);
            __syncthreads();
        }
    }
}

// The two ledger kernels as two branches (s->st_req carries the long runs), joined on s->st; capturable.
void launch_ledger_update(tdpg_session* s, long long cap, const LedgerArgs& a)
{
    CK(cudaEventRecord(s->ev_sta_fork, s->st));
    CK(cudaStreamWaitEvent(s->st_req, s->ev_sta_fork, 0));
    k_ledger_long<<<kLedLongBlocks, kLedBlock, 0, s->st_req>>>(a);
    CK_LAUNCH();
    k_ledger_dense<<<blocks_for(cap, kBlock), kBlock, 0, s->st>>>(cap, a);
    CK_LAUNCH();
    CK(cudaEventRecord(s->ev_sta_join, s->st_req));
    CK(cudaStreamWaitEvent(s->st, s->ev_sta_join, 0));
}

__global__ void k_extract_counts(int EP, const double* __restrict__ sta_out, const Ctrl* __restrict__ ctrl,
                                 const int* __restrict__ len, const int* __restrict__ off,
                                 const int* __restrict__ hops, const int* __restrict__ hoff,
                                 long long* __restrict__ counts)
{
    const bool on = refresh_active(sta_out, ctrl) && EP > 0;
    counts[0] = on ? static_cast<long long>(sta_out[2]) : 0;
    counts[1] = on ? static_cast<long long>(off[EP - 1]) + len[EP - 1] : 0;
    counts[2] = on ? static_cast<long long>(hoff[EP - 1]) + hops[EP - 1] : 0;
    counts[3] += counts[0]; // engine totals over every refresh since engine_init (tdpg_engine_paths)
    counts[4] += counts[1];
}

__global__ void k_net_weights_dev(int N, const int* __restrict__ net_start, const int* __restrict__ net_pins,
                                  const double* __restrict__ slack, const double* __restrict__ sta_out,
                                  const Ctrl* __restrict__ ctrl, double* __restrict__ w)
{
    const int e = blockIdx.x * kBlock + threadIdx.x;
    if (e >= N || (ctrl && ctrl->stopped)) return;
    const double wns = sta_out[1];
    double r = 1.0;
    if (wns < 0.0) { // apply_net_weights (placer.cpp:262-273)
        double worst = slack[net_pins[net_start[e]]];
        for (int j = net_start[e] + 1; j < net_start[e + 1]; ++j) worst = smin(worst, slack[net_pins[j]]);
        if (worst < 0.0) r = 1.0 + (-worst) / (-wns);
    }
    w[e] = r;
}

void net_weights_engine(tdpg_session* s, const Ctrl* ctrl)
{
    if (!s->N) return;
    sta_materialize_pins(s);
    k_net_weights_dev<<<blocks_for(s->N, kBlock), kBlock, 0, s->st>>>(s->N, s->net_start, s->net_pins, s->slack,
                                                                      s->sta_out, ctrl, s->net_w);
    CK_LAUNCH();
}

static int bits_for(long long n)
{
    int b = 1;
    while ((1ll << b) <= n) ++b;
    return b;
}

// Reserve every buffer the engine refresh touches (before capture; pointers never move after).
void refresh_reserve(tdpg_session* s)
{
    const size_t EP = static_cast<size_t>(std::max(s->EP, 1));
    const size_t L = static_cast<size_t>(std::max(s->L, 1));
    // the refresh's path slots, hits and scans are int-indexed (cub counts, slot offsets): refuse designs
    // whose worst case would overflow them instead of corrupting memory
    if (EP * (L + 1) > static_cast<size_t>(INT_MAX) || EP * ((L + 1) / 2 + 1) > static_cast<size_t>(INT_MAX))
        throw Error(TDPG_ERR_VALIDATION, "validation error: design too large for the timing refresh: " +
                                             std::to_string(EP) + " endpoints x " + std::to_string(L + 1) +
                                             " levels exceed 2^31 path-pin slots");
    s->hcap = static_cast<long long>(EP) * static_cast<long long>((L + 1) / 2 + 1);
    const size_t H = static_cast<size_t>(s->hcap);
    s->sort_k0.reserve(EP), s->sort_k1.reserve(EP), s->sort_v0.reserve(EP), s->sort_v1.reserve(EP);
    s->ex_len.reserve(EP), s->ex_hops.reserve(EP), s->ex_off.reserve(EP), s->ex_hoff.reserve(EP);
    s->ex_slack.reserve(EP), s->ex_pins.reserve(EP * L + 1);
    s->ex_tmp_pins.reserve(EP * (L + 1)), s->ex_tmp_keys.reserve(EP * (L / 2 + 2)); // (k_bt_walk slots)
    s->eh_key.reserve(H), s->eh_key_s.reserve(H), s->eh_idx.reserve(H), s->eh_idx_s.reserve(H);
    s->eh_slack.reserve(H);
    s->ex_counts.reserve(8), s->q_count.reserve(2), s->sta_out.reserve(4);
    const int nb = std::max(1, std::min(148 * 4, static_cast<int>(blocks_for(std::max(s->P, s->EP), kBlock))));
    s->sta_part.reserve(3 * nb + 8);
    size_t b1 = 0, b2 = 0, b3 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b1, s->sort_k0.p, s->sort_k1.p, s->sort_v0.p, s->sort_v1.p,
                                    static_cast<int>(EP), 0, 64, s->st);
    cub::DeviceScan::ExclusiveSum(nullptr, b2, s->ex_len.p, s->ex_off.p, static_cast<int>(EP), s->st);
    cub::DeviceRadixSort::SortPairs(nullptr, b3, s->eh_key.p, s->eh_key_s.p, s->eh_idx.p, s->eh_idx_s.p,
                                    static_cast<int>(H), 0, 32, s->st);
    s->ep_kc.reserve(EP), s->ep_vc.reserve(EP), s->ep_flag.reserve(EP), s->ep_nv.reserve(4);
    size_t b4 = 0, b5 = 0;
    cub::DeviceSelect::Flagged(nullptr, b4, s->sort_k0.p, s->ep_flag.p, s->ep_kc.p, s->ep_nv.p + 1,
                               static_cast<int>(EP), s->st);
    cub::DeviceSelect::Flagged(nullptr, b5, s->sort_v0.p, s->ep_flag.p, s->ep_vc.p, s->ep_nv.p + 2,
                               static_cast<int>(EP), s->st);
    cub_scratch(s, std::max({b1, b2, b3, b4, b5}));
    s->tie_scratch.reserve(static_cast<size_t>(kBlock) * 2 * (s->L + 2));
    if (s->N) s->net_w.reserve(s->N);
}

__global__ void k_ep_violated(const double* __restrict__ sta_out, const Ctrl* __restrict__ ctrl,
                              long long* __restrict__ nv)
{
    nv[0] = refresh_active(sta_out, ctrl) ? static_cast<long long>(sta_out[2]) : 0;
}

__global__ void k_flag_keys(int n, const unsigned long long* __restrict__ keys, uint8_t* __restrict__ flag)
{
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n; i += gridDim.x * kBlock) flag[i] = keys[i] != kNoKey;
}

// kNoKey past the compacted violated keys, up to the size class being sorted
__global__ void k_pad_keys(long long n, const long long* __restrict__ nv, unsigned long long* __restrict__ keys)
{
    for (long long i = nv[1] + blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * kBlock)
        keys[i] = kNoKey;
}

// Size classes for a stream-ordered count known only on the device (cap/64, cap/16, cap/4, cap).
struct SizeClasses {
    long long c[4];
    int k;
};

__global__ void k_pick_class(const long long* __restrict__ n, SizeClasses sc, cudaGraphConditionalHandle h)
{
    const long long v = *n;
    unsigned k = static_cast<unsigned>(sc.k); // (no body when there is nothing to process)
    if (v > 0)
        for (k = 0; k + 1 < static_cast<unsigned>(sc.k) && v > sc.c[k]; ++k) {}
    cudaGraphSetConditional(h, k);
}

// Record body(stream, n) for the smallest size class n >= *d_n: under stream capture one SWITCH
// conditional node whose bodies are the size classes, selected on the device by k_pick_class (the
// graph stays host-sync-free); eagerly, body runs over the full capacity.
static bool size_classes_apply(tdpg_session* s, long long cap)
{
    static const bool off = [] { // TDPG_NO_COND=1: full-capacity bodies (profilers that skip conditional graphs)
        const char* e = std::getenv("TDPG_NO_COND");
        return e && std::atoi(e) != 0;
    }();
    if (off) return false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s->st, &cs));
    return cs == cudaStreamCaptureStatusActive && cap >= 64;
}

template <typename F>
void switch_by_count(tdpg_session* s, const long long* d_n, long long cap, F&& body)
{
    if (!size_classes_apply(s, cap)) {
        body(s->st, cap);
        return;
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    SizeClasses sc{};
    for (const long long c : {cap >> 6, cap >> 4, cap >> 2, cap})
        if (c > 0 && (sc.k == 0 || c > sc.c[sc.k - 1])) sc.c[sc.k++] = c;
    cudaGraph_t g = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t nd = 0;
    CK(cudaStreamGetCaptureInfo(s->st, &cs, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle h{};
    CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
    k_pick_class<<<1, 1, 0, s->st>>>(d_n, sc, h);
    CK_LAUNCH();
    CK(cudaStreamGetCaptureInfo(s->st, &cs, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams p{};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeSwitch;
    p.conditional.size = static_cast<unsigned>(sc.k);
    cudaGraphNode_t node = nullptr;
    CK(cudaGraphAddNode(&node, g, deps, nd, &p));
    for (int k = 0; k < sc.k; ++k) {
        CK(cudaStreamBeginCaptureToGraph(s->st_cond, p.conditional.phGraph_out[k], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
        body(s->st_cond, sc.c[k]);
        cudaGraph_t out = nullptr;
        CK(cudaStreamEndCapture(s->st_cond, &out));
    }
    CK(cudaStreamUpdateCaptureDependencies(s->st, &node, 1, cudaStreamSetCaptureDependencies));
}

// The whole refresh, stream-ordered and host-sync-free (captured by the engine).
// 0xFFFFFFFF keys past the device hit count, up to the size class the following sort may pick (or the
// whole capacity when size classes are off), so the sorted prefix holds exactly the hits.
void pad_hit_keys(tdpg_session* s, long long cap, const long long* n_dev, unsigned* keys)
{
    if (!size_classes_apply(s, cap))
        k_fill_u32<<<std::min<unsigned>(blocks_for(cap, kBlock), 148 * 8), kBlock, 0, s->st>>>(cap, keys, 0xFFFFFFFFu);
    else
        k_fill_hit_pad<<<std::min<unsigned>(blocks_for(cap, kBlock), 148 * 8), kBlock, 0, s->st>>>(cap, n_dev, keys);
    CK_LAUNCH();
}

bool capturing(tdpg_session* s)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s->st, &cs));
    return cs == cudaStreamCaptureStatusActive;
}

int bits_for_pins(int P) { return bits_for(P); }

void switch_hits_by_count(tdpg_session* s, const long long* d_n, long long cap,
                          const std::function<void(cudaStream_t, long long)>& body)
{
    switch_by_count(s, d_n, cap, body);
}

void refresh_begin(tdpg_session* s, Ctrl* ctrl, double* timing_row)
{
    k_refresh_begin<<<1, 1, 0, s->st>>>(s->sta_out, ctrl, timing_row);
    CK_LAUNCH();
}

void net_weights_record(tdpg_session* s, const Ctrl* ctrl)
{
    k_net_weights_dev<<<blocks_for(s->N, kBlock), kBlock, 0, s->st>>>(s->N, s->net_start, s->net_pins, s->slack,
                                                                      s->sta_out, ctrl, s->net_w);
    CK_LAUNCH();
}

// The endpoints in (slack, pin) order into sort_v1 (paths.cpp:77-87), from the keys sta_record left in
// sort_k0 / sort_v0.  Readers take only the first (violated-count) entries: when few fail, compact them
// stably and sort the smallest size class holding them; else sort every endpoint.  Capturable.
void sort_violated_endpoints(tdpg_session* s, const Ctrl* ctrl)
{
    const int EP = s->EP;
    k_ep_violated<<<1, 1, 0, s->st>>>(s->sta_out, ctrl, s->ep_nv);
    CK_LAUNCH();
    switch_by_count(s, s->ep_nv.p, EP, [&](cudaStream_t st, long long n) {
        size_t b = s->cub_tmp.n;
        const int lo_bit = ep_sort64() ? 0 : 32;
        auto fixup = [&] {
            if (lo_bit == 0) return;
            k_ep_fixup<<<std::max<unsigned>(1, std::min<unsigned>(blocks_for(n, kBlock), 148 * 4)), kBlock, 0, st>>>(
                s->ep_nv.p, nullptr, s->sort_k1.p, s->sort_v1.p);
            CK_LAUNCH();
        };
        if (n >= EP) {
            CK(cub::DeviceRadixSort::SortPairs(s->cub_tmp.p, b, s->sort_k0.p, s->sort_k1.p, s->sort_v0.p,
                                               s->sort_v1.p, EP, lo_bit, 64, st));
            fixup();
            return;
        }
        k_flag_keys<<<std::min<unsigned>(blocks_for(EP, kBlock), 148 * 4), kBlock, 0, st>>>(EP, s->sort_k0, s->ep_flag);
        CK_LAUNCH();
        CK(cub::DeviceSelect::Flagged(s->cub_tmp.p, b, s->sort_k0.p, s->ep_flag.p, s->ep_kc.p, s->ep_nv.p + 1, EP, st));
        b = s->cub_tmp.n;
        CK(cub::DeviceSelect::Flagged(s->cub_tmp.p, b, s->sort_v0.p, s->ep_flag.p, s->ep_vc.p, s->ep_nv.p + 2, EP, st));
        k_pad_keys<<<std::max<unsigned>(1, std::min<unsigned>(blocks_for(n, kBlock), 148 * 4)), kBlock, 0, st>>>(
            n, s->ep_nv, s->ep_kc);
        CK_LAUNCH();
        b = s->cub_tmp.n;
        CK(cub::DeviceRadixSort::SortPairs(s->cub_tmp.p, b, s->ep_kc.p, s->sort_k1.p, s->ep_vc.p, s->sort_v1.p,
                                           static_cast<int>(n), lo_bit, 64, st));
        fixup();
    });
}

void refresh_record(tdpg_session* s, Ctrl* ctrl, double* timing_row, double w0, double w1, bool net_weighting)
{
    // net weighting reads every pin's slack: keep the per-pin arrays then
    sta_record(s, s->sta_out, net_weighting);
    const bool lonly = s->pins_stale;
    k_refresh_begin<<<1, 1, 0, s->st>>>(s->sta_out, ctrl, timing_row);
    CK_LAUNCH();
    const int EP = s->EP;
    if (EP == 0) return;
    sort_violated_endpoints(s, ctrl);
    size_t bytes = 0;
    const int S = s->L + 1, SH = s->L / 2 + 2; // (k_bt_walk's slot strides)
    if (lonly) { // one backtrace pass into fixed-stride slots, packed after the scans (k_bt_compact)
        k_resolve_ties_L<<<1, kBlock, 0, s->st>>>(make_largs(s), s->d_level, s->L, s->tie_scratch, s->L + 2);
        k_bt_walk<<<blocks_for(EP, kBlock), kBlock, 0, s->st>>>(
            EP, s->sort_v1, s->sta_out, 0, s->L_of, s->L_pin, s->L_pred, s->L_flags, s->pin_dir, s->L_arr, s->clock,
            S, SH, s->ex_tmp_pins, s->ex_tmp_keys, s->ex_len, s->ex_hops, s->ex_slack, nullptr, nullptr, ctrl);
    } else {
        k_resolve_ties<<<1, kBlock, 0, s->st>>>(sta_args(s), s->d_level, s->L, s->tie_scratch, s->L + 2);
        k_bt_count_dev<<<blocks_for(EP, kBlock), kBlock, 0, s->st>>>(EP, s->sta_out, ctrl, s->sort_v1, s->pred,
                                                                     s->pin_dir, s->ex_len, s->ex_hops);
    }
    CK_LAUNCH();
    bytes = s->cub_tmp.n;
    CK(cub::DeviceScan::ExclusiveSum(s->cub_tmp.p, bytes, s->ex_len.p, s->ex_off.p, EP, s->st));
    bytes = s->cub_tmp.n;
    CK(cub::DeviceScan::ExclusiveSum(s->cub_tmp.p, bytes, s->ex_hops.p, s->ex_hoff.p, EP, s->st));
    k_extract_counts<<<1, 1, 0, s->st>>>(EP, s->sta_out, ctrl, s->ex_len, s->ex_off, s->ex_hops, s->ex_hoff,
                                         s->ex_counts);
    CK_LAUNCH();
    const long long H = s->hcap;
    if (!size_classes_apply(s, H)) // (switch_by_count sorts the full capacity then)
        k_fill_u32<<<std::min<unsigned>(blocks_for(H, kBlock), 148 * 8), kBlock, 0, s->st>>>(H, s->eh_key,
                                                                                             0xFFFFFFFFu);
    else
        k_fill_hit_pad<<<std::min<unsigned>(blocks_for(H, kBlock), 148 * 8), kBlock, 0, s->st>>>(
            H, s->ex_counts.p + 2, s->eh_key);
    CK_LAUNCH();
    if (lonly)
        k_bt_compact<<<std::min<unsigned>(blocks_for(static_cast<long long>(EP) * S, kBlock), 148 * 8), kBlock, 0,
                       s->st>>>(EP, S, SH, s->ex_tmp_pins, s->ex_tmp_keys, s->ex_len, s->ex_off, s->ex_hops,
                                s->ex_hoff, s->ex_slack, s->ex_pins, nullptr, s->eh_slack, s->eh_idx, s->eh_key,
                                s->ex_counts.p);
    else
        k_bt_write_dev<<<blocks_for(EP, kBlock), kBlock, 0, s->st>>>(EP, s->sta_out, ctrl, s->sort_v1, s->pred,
                                                                     s->pin_dir, s->ex_len, s->ex_off, s->ex_hops,
                                                                     s->ex_hoff, s->arr, s->clock, s->ex_pins,
                                                                     s->ex_slack, s->eh_key, s->eh_slack, s->eh_idx);
    CK_LAUNCH();
    // the hits are packed at the front (k_extract_counts' total); sort the smallest size class that holds them
    const int kbits = bits_for(s->P);
    switch_by_count(s, s->ex_counts.p + 2, H, [&](cudaStream_t st, long long n) {
        size_t b = s->cub_tmp.n;
        CK(cub::DeviceRadixSort::SortPairs(s->cub_tmp.p, b, s->eh_key.p, s->eh_key_s.p, s->eh_idx.p, s->eh_idx_s.p,
                                           static_cast<int>(n), 0, kbits, st));
    });
    {
        LedgerArgs la{};
        la.n_hits = s->ex_counts.p + 2, la.H = H, la.sta_out = s->sta_out, la.ctrl = ctrl, la.gen = false;
        la.hk = s->eh_key_s, la.hidx = s->eh_idx_s, la.hslack = s->eh_slack, la.w0 = w0, la.w1 = w1;
        la.dl_w = s->dl_w, la.ppw_e = s->ppw_e, la.pin_entry = s->pin_entry, la.pin_loc = s->pin_loc;
        la.pp_mask = s->pp_mask, la.q_count = s->q_count;
        launch_ledger_update(s, H, la);
    }
    if (net_weighting && s->N) {
        k_net_weights_dev<<<blocks_for(s->N, kBlock), kBlock, 0, s->st>>>(s->N, s->net_start, s->net_pins, s->slack,
                                                                          s->sta_out, ctrl, s->net_w);
        CK_LAUNCH();
    }
}

// Buffers tdpg_place touches after its loop (the sorted ledger, the final HPWL partials), reserved
// with the engine's own so that allocation-free runs can reuse the previous run's graphs.
void place_tail_reserve(tdpg_session* s)
{
    const int P = std::max(s->P, 1);
    s->dl_k0.reserve(P), s->dl_k1.reserve(P), s->dl_w0.reserve(P), s->dl_w1.reserve(P);
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, s->dl_k0.p, s->dl_k1.p, s->dl_w0.p, s->dl_w1.p, P, 0, 64, s->st);
    cub_scratch(s, bytes);
    s->part.reserve(2 * static_cast<size_t>(wa_blocks(s)) + 8);
    s->sta_out.reserve(4);
    s->led_key.reserve(static_cast<size_t>(P) + 1), s->led_w.reserve(static_cast<size_t>(P) + 1); // (Q <= P)
}

// The dense ledger's pairs (weight > 0), compacted in any order (the sort below fixes it).
__global__ void k_dense_compact(int P, const double* __restrict__ dl_w, const int* __restrict__ pin_driver,
                                unsigned long long* __restrict__ key, double* __restrict__ w, int* __restrict__ n)
{
    const int v = blockIdx.x * kBlock + threadIdx.x;
    if (v >= P) return;
    const double x = dl_w[v];
    const int d = pin_driver[v];
    if (!(x > 0.0 && d >= 0)) return;
    const unsigned lo = static_cast<unsigned>(min(v, d)), hi = static_cast<unsigned>(max(v, d));
    const int k = atomicAdd(n, 1);
    key[k] = (static_cast<unsigned long long>(lo) << 32) | hi;
    w[k] = x;
}

// Dense ledger -> the sorted (a, b, w) ledger of the session (tdpg_pp_get), after a run.
void dense_ledger_to_sorted(tdpg_session* s)
{
    const int P = s->P;
    if (P == 0) return;
    // persistent scratch: a per-call cudaMalloc / cudaFree of these (4 x 8P bytes) cost up to ~0.8 s when the
    // device heap is busy
    s->dl_k0.reserve(P), s->dl_k1.reserve(P), s->dl_w0.reserve(P), s->dl_w1.reserve(P);
    DBuf<unsigned long long>& k0 = s->dl_k0;
    DBuf<unsigned long long>& k1 = s->dl_k1;
    DBuf<double>& w0 = s->dl_w0;
    DBuf<double>& w1 = s->dl_w1;
    // only the Q pairs are sorted (by their key bits), not the P-slot dense array
    unsigned long long q = 0;
    CK(cudaMemcpyAsync(&q, s->q_count.p, sizeof q, cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemsetAsync(s->counters.p + 4, 0, sizeof(int), s->st));
    k_dense_compact<<<blocks_for(P, kBlock), kBlock, 0, s->st>>>(P, s->dl_w, s->pin_driver, k0, w0,
                                                                 s->counters.p + 4);
    CK_LAUNCH();
    CK(cudaStreamSynchronize(s->st));
    if (q) {
        size_t bytes = 0;
        const int kb = std::min(64, 32 + bits_for(P));
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0.p, k1.p, w0.p, w1.p, static_cast<int>(q), 0, kb, s->st);
        void* tmp = cub_scratch(s, bytes);
        CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, k0.p, k1.p, w0.p, w1.p, static_cast<int>(q), 0, kb, s->st));
    }
    s->led_key.reserve(q + 1), s->led_w.reserve(q + 1);
    if (q) {
        CK(cudaMemcpyAsync(s->led_key.p, k1.p, q * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s->st));
        CK(cudaMemcpyAsync(s->led_w.p, w1.p, q * sizeof(double), cudaMemcpyDeviceToDevice, s->st));
    }
    s->Q = static_cast<long long>(q);
    s->pp_dirty = true;
    CK(cudaStreamSynchronize(s->st));
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

int tdpg_pin_positions(tdpg_session* s, double* pin_xy)
{
    API_BEGIN
    k_pin_xy<<<blocks_for(s->P, kBlock), kBlock, 0, s->st>>>(s->P, s->pin_cell, s->pin_off, s->cell_xy, s->anchor,
                                                             s->pin_xy);
    CK_LAUNCH();
    s->pin_xy.download(reinterpret_cast<double2*>(pin_xy), s->P, s->st);
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_sta(tdpg_session* s, double* arr, double* req, double* slack, uint8_t* ak, uint8_t* rk, double* tns,
             double* wns)
{
    API_BEGIN
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s->st));
    run_sta_dev(s, arr || req || slack || ak || rk); // no per-pin outputs asked for: leave them in L-space
    CK(cudaEventRecord(e1, s->st));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    s->last_sta_ms = ms;
    cudaEventDestroy(e0), cudaEventDestroy(e1);
    const size_t P = static_cast<size_t>(s->P);
    if (arr) s->arr.download(arr, P, s->st);
    if (req) s->req.download(req, P, s->st);
    if (slack) s->slack.download(slack, P, s->st);
    if (ak) s->ak.download(ak, P, s->st);
    if (rk) s->rk.download(rk, P, s->st);
    CK(cudaStreamSynchronize(s->st));
    if (tns) *tns = s->tns;
    if (wns) *wns = s->wns;
    API_END
}

static void extract_timed(tdpg_session* s, int policy, int n, int k)
{
    if (k < 1) throw Error(TDPG_ERR_VALIDATION, "validation error: k must be >= 1");
    if (policy != 0 && policy != 1) throw Error(TDPG_ERR_VALIDATION, "validation error: policy must be \"endpoint\" or \"topn\"");
    // report_timing_endpoint(n, 1) reads the sweep in L-space; the other policies need the per-pin arrays
    if (!s->sta_valid) run_sta_dev(s, !(policy == 0 && k == 1));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s->st));
    if (policy == 0 && k == 1) extract_endpoint_dev(s, n);
    else extract_policy_dev(s, policy, n, k, false);
    CK(cudaEventRecord(e1, s->st));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    s->last_extract_ms = ms;
    cudaEventDestroy(e0), cudaEventDestroy(e1);
}

int tdpg_extract_endpoint(tdpg_session* s, int32_t n, int32_t k, int64_t counts[4])
{
    API_BEGIN
    extract_timed(s, 0, n, k);
    counts[0] = s->n_paths, counts[1] = s->n_path_pins, counts[2] = s->uniq_endpoints, counts[3] = s->uniq_pairs;
    API_END
}

int tdpg_extract(tdpg_session* s, int32_t policy, int32_t n, int32_t k, int64_t counts[5])
{
    API_BEGIN
    extract_timed(s, policy, n, k);
    counts[0] = s->n_paths, counts[1] = s->n_path_pins, counts[2] = s->uniq_endpoints, counts[3] = s->uniq_pairs;
    counts[4] = s->candidates;
    API_END
}

int tdpg_paths_counts(tdpg_session* s, int64_t counts[4])
{
    API_BEGIN
    counts[0] = s->n_paths, counts[1] = s->n_path_pins, counts[2] = s->uniq_endpoints, counts[3] = s->uniq_pairs;
    API_END
}

int tdpg_paths_candidates(tdpg_session* s, int64_t* candidates)
{
    API_BEGIN
    *candidates = s->candidates;
    API_END
}

int tdpg_paths_get(tdpg_session* s, int32_t* start, int32_t* pins, double* slack)
{
    API_BEGIN
    const int np = s->n_paths;
    if (np > 0) {
        if (start) {
            s->ex_off.download(start, np, s->st);
            CK(cudaStreamSynchronize(s->st));
            start[np] = static_cast<int32_t>(s->n_path_pins);
        }
        if (pins) s->ex_pins.download(pins, s->n_path_pins, s->st);
        if (slack) s->ex_slack.download(slack, np, s->st);
    } else if (start) {
        start[0] = 0;
    }
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_paths_hits(tdpg_session* s, int64_t* n_hits, int32_t* a, int32_t* b, double* slack)
{
    API_BEGIN
    *n_hits = s->n_hits;
    if (s->n_hits > 0 && (a || b || slack)) {
        std::vector<unsigned long long> k(s->n_hits);
        s->hit_key.download(k.data(), k.size(), s->st);
        if (slack) s->hit_slack.download(slack, s->n_hits, s->st);
        CK(cudaStreamSynchronize(s->st));
        for (size_t i = 0; i < k.size(); ++i) {
            if (a) a[i] = static_cast<int32_t>(k[i] >> 32);
            if (b) b[i] = static_cast<int32_t>(k[i] & 0xFFFFFFFFull);
        }
    }
    API_END
}

int tdpg_pp_update(tdpg_session* s, int64_t n, const int32_t* a, const int32_t* b, const double* sl, double wns,
                   double w0, double w1)
{
    API_BEGIN
    if (!(wns < 0.0) || n == 0) return TDPG_OK; // pin_pairs.cpp:9
    DBuf<int> da(n), db(n);
    DBuf<double> ds(n);
    da.upload(a, n, s->st), db.upload(b, n, s->st), ds.upload(sl, n, s->st);
    s->hit_key.reserve(n + 1), s->hit_idx.reserve(n + 1), s->hit_key_s.reserve(n + 1), s->hit_idx_s.reserve(n + 1);
    s->hit_slack.reserve(n + 1);
    k_host_hit_keys<<<blocks_for(n, kBlock), kBlock, 0, s->st>>>(n, da, db, ds, s->hit_key, s->hit_idx);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(s->hit_slack.p, ds.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s->st));
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, s->hit_key.p, s->hit_key_s.p, s->hit_idx.p, s->hit_idx_s.p,
                                    static_cast<int>(n), 0, 64, s->st);
    void* tmp = cub_scratch(s, bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, s->hit_key.p, s->hit_key_s.p, s->hit_idx.p, s->hit_idx_s.p,
                                       static_cast<int>(n), 0, 64, s->st));
    ledger_apply_sorted(s, n, wns, w0, w1);
    s->n_hits = 0; // host-provided hits are not an extraction result
    s->n_paths = 0;
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_set_pin_positions(tdpg_session* s, const double* pin_xy)
{
    API_BEGIN
    s->pin_xy.upload(reinterpret_cast<const double2*>(pin_xy), s->P, s->st);
    s->pin_xy_external = true;
    s->sta_valid = false;
    CK(cudaStreamSynchronize(s->st));
    API_END
}

int tdpg_sta_fetch(tdpg_session* s, double* arr, double* req, double* slack, uint8_t* ak, uint8_t* rk, double* tns,
                   double* wns)
{
    API_BEGIN
    if (!s->sta_valid) throw Error(TDPG_ERR_GRAPH, "graph error: no timing annotation (run tdpg_sta first)");
    sta_materialize_pins(s);
    const size_t P = static_cast<size_t>(s->P);
    if (arr) s->arr.download(arr, P, s->st);
    if (req) s->req.download(req, P, s->st);
    if (slack) s->slack.download(slack, P, s->st);
    if (ak) s->ak.download(ak, P, s->st);
    if (rk) s->rk.download(rk, P, s->st);
    CK(cudaStreamSynchronize(s->st));
    if (tns) *tns = s->tns;
    if (wns) *wns = s->wns;
    API_END
}

// PathEnumerator::path_to(pin, rank) for rank 0 (paths.cpp:44-55): the worst source->pin path.
int tdpg_path_to(tdpg_session* s, int32_t pin, int32_t rank, int32_t* pins, int32_t cap, int32_t* n_pins,
                 double* delay)
{
    API_BEGIN
    if (pin < 0 || pin >= s->P) throw Error(TDPG_ERR_VALIDATION, "validation error: pin id out of range");
    if (rank < 0) throw Error(TDPG_ERR_VALIDATION, "validation error: rank must be >= 0");
    if (rank > 0) { // rank-th record of the pin's k-best list (K = rank + 1)
        std::vector<std::vector<int>> paths;
        std::vector<double> d;
        kbest_paths_of(s, pin, rank + 1, paths, d);
        *n_pins = 0;
        if (static_cast<int>(paths.size()) <= rank) return TDPG_OK; // exhausted: nullptr in the reference
        const auto& p = paths[rank];
        if (static_cast<int>(p.size()) > cap)
            throw Error(TDPG_ERR_VALIDATION, "validation error: path longer than the output buffer");
        std::copy(p.begin(), p.end(), pins);
        *n_pins = static_cast<int32_t>(p.size());
        if (delay) *delay = d[rank];
        return TDPG_OK;
    }
    if (!s->sta_valid) run_sta_dev(s);
    resolve_ties_dev(s); // (materialises the per-pin arrays of an L-space-only STA)
    uint8_t known = 0;
    CK(cudaMemcpyAsync(&known, s->ak.p + pin, 1, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    *n_pins = 0;
    if (!known) return TDPG_OK; // no source reaches the pin: nullptr in the reference
    DBuf<int> ep(1), len(1), hops(1), off(1), hoff(1), out(std::max(cap, 1));
    DBuf<double> sl(1);
    ep.upload(&pin, 1, s->st);
    const int z = 0;
    off.upload(&z, 1, s->st), hoff.upload(&z, 1, s->st);
    k_bt_count<<<1, kBlock, 0, s->st>>>(1, ep, s->pred, s->pin_dir, len, hops);
    CK_LAUNCH();
    int L = 0;
    len.download(&L, 1, s->st);
    CK(cudaStreamSynchronize(s->st));
    if (L > cap) throw Error(TDPG_ERR_VALIDATION, "validation error: path longer than the output buffer");
    s->hit_key.reserve(L + 1), s->hit_slack.reserve(L + 1), s->hit_idx.reserve(L + 1);
    k_bt_write<<<1, kBlock, 0, s->st>>>(1, ep, s->pred, s->pin_dir, len, off, hops, hoff, s->arr, s->clock, out, sl,
                                        s->hit_key, s->hit_slack, s->hit_idx);
    CK_LAUNCH();
    out.download(pins, L, s->st);
    double a = 0.0;
    CK(cudaMemcpyAsync(&a, s->arr.p + pin, sizeof a, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    *n_pins = L;
    if (delay) *delay = a;
    s->n_hits = 0, s->n_paths = 0; // scratch hit buffers were reused
    API_END
}

// k_worst_paths_to (paths.cpp:57-72): EndpointError unless `endpoint` is a graph endpoint.
int tdpg_k_worst(tdpg_session* s, int32_t endpoint, int32_t k, int32_t* n_paths, int32_t* start, int32_t* pins,
                 int32_t cap, double* slack)
{
    API_BEGIN
    if (endpoint < 0 || endpoint >= s->P || !s->h_is_endpoint[endpoint])
        throw Error(TDPG_ERR_ENDPOINT, "validation error: pin " + std::to_string(endpoint) + " is not an endpoint");
    *n_paths = 0;
    if (start) start[0] = 0;
    if (k <= 0) return TDPG_OK;
    std::vector<std::vector<int>> paths;
    std::vector<double> d;
    kbest_paths_of(s, endpoint, k, paths, d);
    int off = 0;
    for (size_t i = 0; i < paths.size(); ++i) {
        if (off + static_cast<int>(paths[i].size()) > cap)
            throw Error(TDPG_ERR_VALIDATION, "validation error: paths exceed the output buffer");
        if (start) start[i] = off;
        std::copy(paths[i].begin(), paths[i].end(), pins + off);
        off += static_cast<int>(paths[i].size());
        if (slack) slack[i] = s->clock - d[i]; // paths.cpp:69
    }
    if (start) start[paths.size()] = off;
    *n_paths = static_cast<int32_t>(paths.size());
    API_END
}

int tdpg_last_timing_ms(tdpg_session* s, double* sta_ms, double* extract_ms)
{
    API_BEGIN
    if (sta_ms) *sta_ms = s->last_sta_ms;
    if (extract_ms) *extract_ms = s->last_extract_ms;
    API_END
}

} // extern "C"
