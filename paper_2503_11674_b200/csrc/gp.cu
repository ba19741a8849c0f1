// gp.cu — objective_and_gradient on the device (placer.cpp:275-343) and its kernels.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <cstdlib>

#include "gp_kernels.cuh"

namespace tdpg {

int api_fail(int kind, const std::string& msg);

// =====================================================================================
// WA wirelength, size-classed (the fast path).  Nets are sorted once by pin count; every
// block holds nets of one pin count N (2..kWaMaxN), so one thread per net runs a fully
// unrolled body with N known at compile time: pins in registers, no divergence, the
// max/min and the four exponential sums accumulated in the reference's pin order
// (wirelength.cpp:15-34), the 4 exps per pin computed once and reused for the gradient.
// Divisions by gamma and by the per-net sums become multiplications by reciprocals.
// Entries are laid out slot-major per block so each pin slot is one coalesced access;
// nets outside the classes (more pins) take k_wa_generic, one warp per net.
// =====================================================================================
template <int N>
__device__ __forceinline__ void wa_axis(const double (&x)[N], double inv_gamma, double (&g)[N], double& value,
                                        double& extent)
{
    double hi = x[0], lo = x[0];
#pragma unroll
    for (int i = 0; i < N; ++i) hi = smax(hi, x[i]), lo = smin(lo, x[i]);
    double eu[N], el[N];
    double s_max = 0.0, t_max = 0.0, s_min = 0.0, t_min = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        eu[i] = exp((x[i] - hi) * inv_gamma);
        el[i] = exp(-(x[i] - lo) * inv_gamma);
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
        s_max += eu[i];
        t_max += (x[i] - hi) * eu[i];
        s_min += el[i];
        t_min += (x[i] - lo) * el[i];
    }
    const double is_max = 1.0 / s_max, is_min = 1.0 / s_min;
    const double max_term = t_max * is_max, min_term = t_min * is_min;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double d_max = (eu[i] * is_max) * (1.0 + ((x[i] - hi) - max_term) * inv_gamma);
        const double d_min = (el[i] * is_min) * (1.0 - ((x[i] - lo) - min_term) * inv_gamma);
        g[i] = d_max - d_min;
    }
    value = (hi - lo) + (max_term - min_term);
    extent = hi - lo;
}

// Pin-pair attraction fused into WA (engine mode).  Every pair the engine's extraction creates is
// a net arc (driver, sink) (paths.cpp:195-200), so a net's pairs are exactly its sinks with a ledger
// weight, and both pins' positions are already in this thread's registers.  Per pin the reference
// accumulates pp.d_pin in map-key order (pin_pairs.cpp:22-34): a sink has one term, the driver one
// term per pair in ascending sink pin id (the per-net order word).  Sink term = (2w)(p_s - p_d)
// (quadratic) or w(p_s - p_d)/dist (linear) whichever pin is `first`; the driver subtracts them.
struct PPArgs {
    const uint32_t* mask;  // per class-ordered net: bit j = sink slot j has a pair
    const uint32_t* ord;   // per class-ordered net: sink slots in ascending pin id, 3 bits each
    const double* w_e;     // pair weight per WA entry slot (0 = no pair)
    double beta;
    int kind;              // 0 quadratic, 1 linear
};

template <int N>
__device__ __forceinline__ void pp_net(const PPArgs& pp, uint32_t mask, uint32_t ord, int base, const double (&x)[N],
                                       const double (&y)[N], double (&px)[N], double (&py)[N], double& val)
{
#pragma unroll
    for (int j = 0; j < N; ++j) px[j] = 0.0, py[j] = 0.0;
#pragma unroll
    for (int j = 1; j < N; ++j) {
        if (!(mask >> j & 1u)) continue;
        const double w = pp.w_e[base + j * kBlock];
        const double dx = x[j] - x[0], dy = y[j] - y[0];
        if (pp.kind == 0) {
            val += w * (dx * dx + dy * dy);
            px[j] = 2.0 * w * dx, py[j] = 2.0 * w * dy;
        } else {
            const double dist = sqrt(dx * dx + dy * dy);
            val += w * dist;
            if (dist > 0.0) px[j] = w * dx / dist, py[j] = w * dy / dist;
        }
    }
    double sx = 0.0, sy = 0.0; // driver: terms in ascending sink pin id
#pragma unroll
    for (int k = 0; k < N - 1; ++k) {
        const int j = (ord >> (3 * k)) & 7;
#pragma unroll
        for (int q = 1; q < N; ++q)
            if (q == j && (mask >> q & 1u)) sx -= px[q], sy -= py[q];
    }
    px[0] = sx, py[0] = sy;
}

template <int N>
__device__ __forceinline__ void wa_net_slots(int base, double w, const int* __restrict__ e_cell,
                                             const double2* __restrict__ e_off, const double2* __restrict__ cell_xy,
                                             const double2* __restrict__ anchor, double inv_gamma,
                                             double2* __restrict__ grad_e, double& wl, double& hp,
                                             const PPArgs* pp, uint32_t mask, uint32_t ord, double& ppv)
{
    double x[N], y[N], gx[N], gy[N];
#pragma unroll
    for (int i = 0; i < N; ++i) { // pin i of this net at base + i * 256 (slot-major block layout)
        const double2 p = entry_pos(__ldcs(e_cell + base + i * kBlock), __ldcs(e_off + base + i * kBlock), cell_xy,
                                    anchor);
        x[i] = p.x, y[i] = p.y;
    }
    double vx, vy, hx, hy;
    wa_axis<N>(x, inv_gamma, gx, vx, hx);
    wa_axis<N>(y, inv_gamma, gy, vy, hy);
    if (pp && mask) {
        double px[N], py[N];
        pp_net<N>(*pp, mask, ord, base, x, y, px, py, ppv);
        // fold term pin_grad + beta * pp.d_pin (placer.cpp:323)
#pragma unroll
        for (int i = 0; i < N; ++i)
            grad_e[base + i * kBlock] = make_double2(w * gx[i] + pp->beta * px[i], w * gy[i] + pp->beta * py[i]);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) grad_e[base + i * kBlock] = make_double2(w * gx[i], w * gy[i]);
    }
    wl = w * (vx + vy);
    hp = hx + hy;
}

constexpr int kWaMaxN = 8;
#ifndef WA_MINB
#define WA_MINB 1
#endif

// One launch per pin count N: thread t of block b owns the t-th net of the block.
template <int N>
__global__ void __launch_bounds__(kBlock, WA_MINB) k_wa_class(int blk0, const int4* __restrict__ blk,
                                                     const int* __restrict__ net_by_size,
                                                     const int* __restrict__ e_cell, const double2* __restrict__ e_off,
                                                     const double2* __restrict__ cell_xy,
                                                     const double2* __restrict__ anchor,
                                                     const double* __restrict__ net_w, double inv_gamma,
                                                     double2* __restrict__ grad_e, double* __restrict__ part_wl,
                                                     double* __restrict__ part_hp, PPArgs pp, double* __restrict__ part_pp,
                                                     const Ctrl* __restrict__ ctrl)
{
    __shared__ double sh[kBlock / 32];
    if (ctrl && ctrl->stopped) return;
    const int4 b = blk[blk0 + blockIdx.x]; // (N, first in net_by_size, count, entry base)
    double wl = 0.0, hp = 0.0, ppv = 0.0;
    if (static_cast<int>(threadIdx.x) < b.z) {
        const int i = b.y + threadIdx.x;
        const double w = net_w ? net_w[net_by_size[i]] : 1.0;
        const uint32_t mask = pp.mask ? pp.mask[i] : 0u;
        const uint32_t ord = mask ? pp.ord[i] : 0u;
        wa_net_slots<N>(b.w + threadIdx.x, w, e_cell, e_off, cell_xy, anchor, inv_gamma, grad_e, wl, hp,
                        pp.mask ? &pp : nullptr, mask, ord, ppv);
    }
    const double bw = block_sum<kBlock>(wl, sh);
    const double bh = block_sum<kBlock>(hp, sh);
    const double bp = part_pp ? block_sum<kBlock>(ppv, sh) : 0.0;
    if (threadIdx.x == 0) {
        part_wl[blk0 + blockIdx.x] = bw, part_hp[blk0 + blockIdx.x] = bh;
        if (part_pp) part_pp[blk0 + blockIdx.x] = bp;
    }
}

// Axis-split variant: two threads per net (lane pairs), one per axis, so a thread keeps only its axis's
// N coordinates and exponentials in registers (half the register footprint of wa_net_slots, twice the
// resident warps for latency hiding).  Each thread loads only its coordinate component (the pair's
// two 8-byte loads share a sector).  Everything that couples the axes — the net value w·(vx + vy), the
// HPWL, the pin-pair value w·(dx² + dy²) and the linear-loss distance — is formed after exchanging the
// partner's term with one shuffle, in the reference's operand order, so results are bitwise those of the
// one-thread form.
struct WaAxisArgs {
    // size-class layout (session.cu): blocks of class k are [cls_blk0[k], cls_blk0[k+1]), their nets
    // [cls_net0[k], cls_net1[k]) of net_by_size, their entries from cls_pos0[k] (k * 256 per block)
    int cls_blk0[10], cls_net0[9], cls_net1[9], cls_pos0[9];
    const int4* blk;
    const int* net_by_size;
    const int* e_cell;
    const double *e_off, *cell_xy, *anchor, *net_w;
    double inv_gamma;
    double *grad_e, *part_wl, *part_hp;
    PPArgs pp;
    double* part_pp;
};

// Block descriptor (N, first net, nets, entry base) of size-class block g from the kernel parameters:
// no table load ahead of the entry loads.
__device__ __forceinline__ int4 wa_blk_of(int g, const WaAxisArgs& A)
{
    int k = 2;
#pragma unroll
    for (int c = 3; c <= 8; ++c)
        if (g >= A.cls_blk0[c]) k = c;
    const int j = g - A.cls_blk0[k];
    const int net0 = A.cls_net0[k] + j * kBlock;
    return make_int4(k, net0, min(kBlock, A.cls_net1[k] - net0), A.cls_pos0[k] + j * kBlock * k);
}

template <int N>
__device__ __forceinline__ void wa_axis_block(const int4 b, int gblk, const WaAxisArgs& A, double* sh,
                                              const Ctrl* __restrict__ ctrl)
{
    const bool stop = ctrl && ctrl->stopped; // (checked after the entry loads are issued)
    const int* __restrict__ net_by_size = A.net_by_size;
    const int* __restrict__ e_cell = A.e_cell;
    const double* __restrict__ e_off = A.e_off;
    const double* __restrict__ cell_xy = A.cell_xy;
    const double* __restrict__ anchor = A.anchor;
    const double* __restrict__ net_w = A.net_w;
    const double inv_gamma = A.inv_gamma;
    double* __restrict__ grad_e = A.grad_e;
    const PPArgs& pp = A.pp;
    const int t = threadIdx.x >> 1, axis = threadIdx.x & 1;
    const bool on = t < b.z;
    const int base = b.w + (on ? t : 0);
    double x[N], g[N];
#pragma unroll
    for (int i = 0; i < N; ++i) { // entry_pos (netlist.cpp:28-29), this axis only
        const int e = base + i * kBlock;
        const int ec = __ldcs(e_cell + e);
        const double a = ec >= 0 ? cell_xy[2 * ec + axis] : anchor[2 * (-1 - ec) + axis];
        x[i] = a + __ldcs(e_off + 2 * e + axis);
    }
    if (stop) return; // (uniform over the block)
    // pin-pair operands: for the larger nets issued ahead of the WA math so their latency overlaps it
    // (measured: 6-8 pins 35 -> 28 us once the ledger is populated; the 2-5 group, at its 64-register
    // budget, only spills more)
    constexpr bool kEarlyPP = N >= 6;
    uint32_t mask = 0u, ord = 0u;
    double wts[N];
    if constexpr (kEarlyPP) {
        const int i_net0 = b.y + (on ? t : 0);
        mask = (on && pp.mask) ? pp.mask[i_net0] : 0u;
        ord = mask ? pp.ord[i_net0] : 0u;
#pragma unroll
        for (int j = 0; j < N; ++j) wts[j] = (j > 0 && (mask >> j & 1u)) ? pp.w_e[base + j * kBlock] : 0.0;
    }
    double v, ext;
    wa_axis<N>(x, inv_gamma, g, v, ext);
    const double v_other = __shfl_xor_sync(0xffffffffu, v, 1), e_other = __shfl_xor_sync(0xffffffffu, ext, 1);
    const int i_net = b.y + (on ? t : 0);
    const double w = net_w ? net_w[net_by_size[i_net]] : 1.0;
    double wl = 0.0, hp = 0.0, ppv = 0.0;
    if (on && axis == 0) wl = w * (v + v_other);   // w (vx + vy), on the x thread
    if (on && axis == 1) hp = e_other + ext;        // hx + hy, on the y thread (see the reduction below)
    if constexpr (!kEarlyPP) {
        mask = (on && pp.mask) ? pp.mask[i_net] : 0u;
        ord = mask ? pp.ord[i_net] : 0u;
    }
    double p[N];
#pragma unroll
    for (int i = 0; i < N; ++i) p[i] = 0.0;
    if (pp.mask) { // pin pairs of this net (pin_pairs.cpp:17-49), see pp_net
#pragma unroll
        for (int j = 1; j < N; ++j) {
            const double d = x[j] - x[0];
            const double d_other = __shfl_xor_sync(0xffffffffu, d, 1);
            if (!(mask >> j & 1u)) continue;
            const double wt = kEarlyPP ? wts[j] : pp.w_e[base + j * kBlock];
            const double dx = axis ? d_other : d, dy = axis ? d : d_other;
            if (pp.kind == 0) {
                if (axis == 0) ppv += wt * (dx * dx + dy * dy);
                p[j] = 2.0 * wt * d;
            } else {
                const double dist = sqrt(dx * dx + dy * dy);
                if (axis == 0) ppv += wt * dist;
                if (dist > 0.0) p[j] = wt * d / dist;
            }
        }
        double sd = 0.0; // driver: terms in ascending sink pin id
#pragma unroll
        for (int k = 0; k < N - 1; ++k) {
            const int j = (ord >> (3 * k)) & 7;
#pragma unroll
            for (int q = 1; q < N; ++q)
                if (q == j && (mask >> q & 1u)) sd -= p[q];
        }
        p[0] = sd;
    }
    if (on) {
#pragma unroll
        for (int i = 0; i < N; ++i) // fold term pin_grad + beta * pp.d_pin (placer.cpp:323)
            grad_e[2 * (base + i * kBlock) + axis] = mask ? w * g[i] + pp.beta * p[i] : w * g[i];
    }
    // block partials of (WA, HPWL, pair value) in one fixed-order tree: the net terms live on the
    // axis-0 (even) lanes, so even lanes carry WA and the pair value and odd lanes the HPWL through a
    // parity-preserving butterfly (offsets 16..2), then 16 warps x 3 values in one shared round
    double r1 = axis == 0 ? wl : hp, r2 = ppv;
#pragma unroll
    for (int o = 16; o > 1; o >>= 1) {
        r1 += __shfl_xor_sync(0xffffffffu, r1, o);
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    }
    double* s3 = sh; // [3][16]
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) s3[wid] = r1, s3[32 + wid] = r2;
    if (lane == 1) s3[16 + wid] = r1;
    __syncthreads();
    if (wid == 0) {
        double a = lane < 16 ? s3[lane] : s3[lane]; // lanes 0..15: WA, 16..31: HPWL
        double c = lane < 16 ? s3[32 + lane] : 0.0;
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (lane == 0) {
            A.part_wl[gblk] = a;
            if (A.part_pp) A.part_pp[gblk] = c;
        }
        if (lane == 16) A.part_hp[gblk] = a;
    }
}

template <int N>
__global__ void __launch_bounds__(2 * kBlock, (N <= 5 ? 2 : 1)) k_wa_axis(int blk0, WaAxisArgs A,
                                                                          const Ctrl* __restrict__ ctrl)
{
    __shared__ double sh[48];
    wa_axis_block<N>(wa_blk_of(blk0 + blockIdx.x, A), blk0 + blockIdx.x, A, sh, ctrl);
}

// Several size classes in one launch (their blocks are contiguous in the table): each block dispatches
// on its pin count; the register budget is the group's largest class.
// L2 prefetch of a byte range (TMA engine; 16-byte aligned, size a multiple of 16).
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes)
{
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <int LO, int HI, int MINB>
__global__ void __launch_bounds__(2 * kBlock, MINB) k_wa_axis_group(int blk0, WaAxisArgs A,
                                                                    const Ctrl* __restrict__ ctrl, int ahead)
{
    __shared__ double sh[48];
    const int g = blk0 + blockIdx.x;
    const int4 b = wa_blk_of(g, A);
    const int gridw = gridDim.x;
    switch (b.x) {
    case 2: if (LO <= 2 && 2 <= HI) wa_axis_block<(LO <= 2 && 2 <= HI) ? 2 : LO>(b, g, A, sh, ctrl); break;
    case 3: if (LO <= 3 && 3 <= HI) wa_axis_block<(LO <= 3 && 3 <= HI) ? 3 : LO>(b, g, A, sh, ctrl); break;
    case 4: if (LO <= 4 && 4 <= HI) wa_axis_block<(LO <= 4 && 4 <= HI) ? 4 : LO>(b, g, A, sh, ctrl); break;
    case 5: if (LO <= 5 && 5 <= HI) wa_axis_block<(LO <= 5 && 5 <= HI) ? 5 : LO>(b, g, A, sh, ctrl); break;
    case 6: if (LO <= 6 && 6 <= HI) wa_axis_block<(LO <= 6 && 6 <= HI) ? 6 : LO>(b, g, A, sh, ctrl); break;
    case 7: if (LO <= 7 && 7 <= HI) wa_axis_block<(LO <= 7 && 7 <= HI) ? 7 : LO>(b, g, A, sh, ctrl); break;
    case 8: if (LO <= 8 && 8 <= HI) wa_axis_block<(LO <= 8 && 8 <= HI) ? 8 : LO>(b, g, A, sh, ctrl); break;
    default: break;
    }
    // a block about one resident wave ahead (blocks are dispatched in order): its entry records into L2
    // now, so its first loads wait for L2 instead of DRAM
    if (ahead > 0 && threadIdx.x == 0 && blockIdx.x + ahead < gridw) {
        const int4 f = wa_blk_of(g + ahead, A);
        const unsigned n = static_cast<unsigned>(f.x) * kBlock;
        prefetch_l2(A.e_cell + f.w, n * 4u);
        prefetch_l2(A.e_off + 2 * static_cast<long long>(f.w), n * 16u);
        if (A.pp.w_e) prefetch_l2(A.pp.w_e + f.w, n * 8u);
    }
}

// Nets outside the classes (more than kWaMaxN pins): one warp per net, lanes stride over the
// pins (contiguous in the layout); max/min and the exponential sums reduced with shuffles.
__device__ __forceinline__ double wsum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void wa_axis_warp(int s0, int n, int axis, const int* __restrict__ e_cell,
                                             const double2* __restrict__ e_off, const double2* __restrict__ cell_xy,
                                             const double2* __restrict__ anchor, double inv_gamma, double w,
                                             double2* __restrict__ grad_e, double& value, double& extent)
{
    const int lane = threadIdx.x & 31;
    auto X = [&](int i) {
        const double2 p = entry_pos(e_cell[s0 + i], e_off[s0 + i], cell_xy, anchor);
        return axis ? p.y : p.x;
    };
    double hi = X(0), lo = hi;
    for (int i = lane; i < n; i += 32) {
        const double x = X(i);
        hi = smax(hi, x), lo = smin(lo, x);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        hi = smax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        lo = smin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    }
    double s_max = 0.0, t_max = 0.0, s_min = 0.0, t_min = 0.0;
    for (int i = lane; i < n; i += 32) {
        const double x = X(i);
        const double eu = exp((x - hi) * inv_gamma), el = exp(-(x - lo) * inv_gamma);
        s_max += eu, t_max += (x - hi) * eu, s_min += el, t_min += (x - lo) * el;
    }
    s_max = wsum(s_max), t_max = wsum(t_max), s_min = wsum(s_min), t_min = wsum(t_min);
    const double is_max = 1.0 / s_max, is_min = 1.0 / s_min;
    const double max_term = t_max * is_max, min_term = t_min * is_min;
    for (int i = lane; i < n; i += 32) {
        const double x = X(i);
        const double eu = exp((x - hi) * inv_gamma), el = exp(-(x - lo) * inv_gamma);
        const double d = (eu * is_max) * (1.0 + ((x - hi) - max_term) * inv_gamma) -
                         (el * is_min) * (1.0 - ((x - lo) - min_term) * inv_gamma);
        if (axis) grad_e[s0 + i].y = w * d;
        else grad_e[s0 + i].x = w * d;
    }
    value = (hi - lo) + (max_term - min_term);
    extent = hi - lo;
}

// One axis of a net of <= 32 pins, lane i holding pin i (lanes past the net hold the driver and
// contribute nothing): max/min and the four exponential sums by warp shuffles; returns the pin's
// unweighted gradient (wirelength.cpp:15-43).
__device__ __forceinline__ double wa_lane(double x, bool on, double inv_gamma, double& value, double& extent)
{
    double hi = x, lo = x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        hi = smax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        lo = smin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    }
    const double eu = on ? exp((x - hi) * inv_gamma) : 0.0;
    const double el = on ? exp(-(x - lo) * inv_gamma) : 0.0;
    const double s_max = wsum(eu), t_max = wsum((x - hi) * eu);
    const double s_min = wsum(el), t_min = wsum((x - lo) * el);
    const double is_max = 1.0 / s_max, is_min = 1.0 / s_min;
    const double max_term = t_max * is_max, min_term = t_min * is_min;
    value = (hi - lo) + (max_term - min_term);
    extent = hi - lo;
    return (eu * is_max) * (1.0 + ((x - hi) - max_term) * inv_gamma) -
           (el * is_min) * (1.0 - ((x - lo) - min_term) * inv_gamma);
}

// wa_lane over a W-lane segment of the warp (W = 16: two nets per warp).
template <int W>
__device__ __forceinline__ double wa_lane_w(double x, bool on, double inv_gamma, double& value, double& extent)
{
    double hi = x, lo = x;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
        hi = smax(hi, __shfl_xor_sync(0xffffffffu, hi, o, W));
        lo = smin(lo, __shfl_xor_sync(0xffffffffu, lo, o, W));
    }
    const double eu = on ? exp((x - hi) * inv_gamma) : 0.0;
    const double el = on ? exp(-(x - lo) * inv_gamma) : 0.0;
    double s_max = eu, t_max = (x - hi) * eu, s_min = el, t_min = (x - lo) * el;
#pragma unroll
    for (int o = W / 2; o > 0; o >>= 1) {
        s_max += __shfl_xor_sync(0xffffffffu, s_max, o, W), t_max += __shfl_xor_sync(0xffffffffu, t_max, o, W);
        s_min += __shfl_xor_sync(0xffffffffu, s_min, o, W), t_min += __shfl_xor_sync(0xffffffffu, t_min, o, W);
    }
    const double is_max = 1.0 / s_max, is_min = 1.0 / s_min;
    const double max_term = t_max * is_max, min_term = t_min * is_min;
    value = (hi - lo) + (max_term - min_term);
    extent = hi - lo;
    return (eu * is_max) * (1.0 + ((x - hi) - max_term) * inv_gamma) -
           (el * is_min) * (1.0 - ((x - lo) - min_term) * inv_gamma);
}

// One net of <= 16 pins per half-warp (lane `sub` of the segment holds pin `sub`): WA both axes and the
// net's pin pairs, the driver's pair terms summed in ascending sink pin id (kmax: the longer net of the
// two segments, so every lane runs the same shuffles).
__device__ __forceinline__ void wa_half_net(int sub, int s0, int n, int kmax, double w, const int* __restrict__ e_cell,
                                            const double2* __restrict__ e_off, const double2* __restrict__ cell_xy,
                                            const double2* __restrict__ anchor, double inv_gamma,
                                            double2* __restrict__ grad_e, const PPArgs& pp,
                                            const int* __restrict__ gen_ord, double& wl, double& hp, double& ppv)
{
    const bool live = n >= 2; // single-pin nets: zero gradient, no terms (wirelength.cpp:53)
    const bool on = live ? sub < n : sub == 0;
    // lanes past the net hold its first pin, so they leave the max / min butterflies unchanged
    const int q = sub < n ? sub : 0;
    const double2 p = n > 0 ? entry_pos(e_cell[s0 + q], e_off[s0 + q], cell_xy, anchor) : make_double2(0.0, 0.0);
    double vx, vy, hx, hy;
    const double gx = wa_lane_w<16>(p.x, on, inv_gamma, vx, hx);
    const double gy = wa_lane_w<16>(p.y, on, inv_gamma, vy, hy);
    double ex = w * gx, ey = w * gy;
    if (pp.w_e) {
        const double wt = (live && on && sub > 0) ? pp.w_e[s0 + sub] : 0.0;
        const double pdx = __shfl_sync(0xffffffffu, p.x, 0, 16), pdy = __shfl_sync(0xffffffffu, p.y, 0, 16);
        const double dx = p.x - pdx, dy = p.y - pdy;
        double px = 0.0, py = 0.0, pv = 0.0;
        if (wt != 0.0) {
            if (pp.kind == 0) {
                pv = wt * (dx * dx + dy * dy);
                px = 2.0 * wt * dx, py = 2.0 * wt * dy;
            } else {
                const double dist = sqrt(dx * dx + dy * dy);
                pv = wt * dist;
                if (dist > 0.0) px = wt * dx / dist, py = wt * dy / dist;
            }
            ex = ex + pp.beta * px, ey = ey + pp.beta * py;
        }
        const int o = (live && sub + 1 < n) ? gen_ord[s0 + sub] : 0;
        double sx = 0.0, sy = 0.0;
        for (int k = 0; k < kmax; ++k) {
            const int j = __shfl_sync(0xffffffffu, o, k, 16);
            const double gxj = __shfl_sync(0xffffffffu, px, j, 16), gyj = __shfl_sync(0xffffffffu, py, j, 16);
            const double vj = __shfl_sync(0xffffffffu, pv, j, 16), wj = __shfl_sync(0xffffffffu, wt, j, 16);
            if (sub == 0 && k + 1 < n && wj != 0.0) ppv += vj, sx -= gxj, sy -= gyj;
        }
        if (sub == 0) ex = ex + pp.beta * sx, ey = ey + pp.beta * sy;
    }
    if (sub < n) grad_e[s0 + sub] = live ? make_double2(ex, ey) : make_double2(0.0, 0.0);
    if (sub == 0 && live) wl += w * (vx + vy), hp += hx + hy;
}

// Block g holds generic nets [16 (g - gen_blk0), +16) of the order; a net's pin count is the difference of
// consecutive layout starts (gen_start has a sentinel), so no net table is read ahead of the entries.
__global__ void __launch_bounds__(kBlock) k_wa_generic(int blk0, int gen_blk0, int gen_nets,
                                                       const int* __restrict__ net_by_size,
                                                       const int* __restrict__ gen_start,
                                                       const int* __restrict__ e_cell,
                                                       const double2* __restrict__ e_off,
                                                       const double2* __restrict__ cell_xy,
                                                       const double2* __restrict__ anchor,
                                                       const double* __restrict__ net_w, double inv_gamma,
                                                       double2* __restrict__ grad_e, double* __restrict__ part_wl,
                                                       double* __restrict__ part_hp, PPArgs pp,
                                                       const int* __restrict__ gen_ord, double* __restrict__ part_pp,
                                                       const Ctrl* __restrict__ ctrl)
{
    __shared__ double sh[3 * kBlock / 32];
    const bool stop = ctrl && ctrl->stopped; // (checked once the net sizes are loaded)
    const int first = (blk0 + blockIdx.x - gen_blk0) * 16;
    const int4 b = make_int4(0, first, min(16, gen_nets - first), 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double wl = 0.0, hp = 0.0, ppv = 0.0;
    // nets in pairs per warp: two nets of <= 16 pins share the warp (a half each); otherwise the warp
    // takes them one after the other
    const int t0 = 2 * warp, t1 = t0 + 1;
    auto size_of = [&](int t) { return t < b.z ? gen_start[b.y + t + 1] - gen_start[b.y + t] : 0; };
    const int n0 = size_of(t0), n1 = size_of(t1);
    if (stop) return; // (uniform over the block)
    const bool halves = t0 < b.z && n0 <= 16 && n1 <= 16;
    if (halves) {
        const int seg = lane >> 4, t = seg ? t1 : t0, n = seg ? n1 : n0;
        const bool have = t < b.z;
        const int i = b.y + (have ? t : t0);
        const int s0 = gen_start[i];
        const double w = net_w ? net_w[net_by_size[i]] : 1.0;
        const int kmax = max(n0, n1) - 1;
        double wl_l = 0.0, hp_l = 0.0, pp_l = 0.0;
        wa_half_net(lane & 15, s0, have ? n : 0, kmax, w, e_cell, e_off, cell_xy, anchor, inv_gamma, grad_e, pp,
                    gen_ord, wl_l, hp_l, pp_l);
        wl += wl_l, hp += hp_l, ppv += pp_l;
    }
    for (int t = halves ? b.z : t0; t < b.z && t <= t1; ++t) { // one warp per net
        const int i = b.y + t;
        const int s0 = gen_start[i], n = gen_start[i + 1] - s0;
        const double w = net_w ? net_w[net_by_size[i]] : 1.0;
        if (n < 2) {
            for (int k = lane; k < n; k += 32) grad_e[s0 + k] = make_double2(0.0, 0.0);
            continue;
        }
        double vx, vy, hx, hy;
        if (n <= 32) { // one pin per lane, held in registers: one gather, exps computed once
            const bool on = lane < n;
            const double2 p = on ? entry_pos(e_cell[s0 + lane], e_off[s0 + lane], cell_xy, anchor)
                                 : entry_pos(e_cell[s0], e_off[s0], cell_xy, anchor);
            const double gx = wa_lane(p.x, on, inv_gamma, vx, hx);
            const double gy = wa_lane(p.y, on, inv_gamma, vy, hy);
            double ex = w * gx, ey = w * gy;
            if (pp.w_e) { // pin pairs of the net (pin_pairs.cpp:17-49), one sink per lane
                const double wt = (on && lane > 0) ? pp.w_e[s0 + lane] : 0.0;
                const double pdx = __shfl_sync(0xffffffffu, p.x, 0), pdy = __shfl_sync(0xffffffffu, p.y, 0);
                const double dx = p.x - pdx, dy = p.y - pdy;
                double px = 0.0, py = 0.0, pv = 0.0;
                if (wt != 0.0) {
                    if (pp.kind == 0) {
                        pv = wt * (dx * dx + dy * dy);
                        px = 2.0 * wt * dx, py = 2.0 * wt * dy;
                    } else {
                        const double dist = sqrt(dx * dx + dy * dy);
                        pv = wt * dist;
                        if (dist > 0.0) px = wt * dx / dist, py = wt * dy / dist;
                    }
                    ex = ex + pp.beta * px, ey = ey + pp.beta * py;
                }
                // the driver's terms and the net's value in ascending sink pin id (gen_ord), as the
                // reference accumulates them in map-key order
                const int o = lane + 1 < n ? gen_ord[s0 + lane] : 0;
                double sx = 0.0, sy = 0.0;
                for (int k = 0; k + 1 < n; ++k) {
                    const int j = __shfl_sync(0xffffffffu, o, k);
                    const double gxj = __shfl_sync(0xffffffffu, px, j), gyj = __shfl_sync(0xffffffffu, py, j);
                    const double vj = __shfl_sync(0xffffffffu, pv, j), wj = __shfl_sync(0xffffffffu, wt, j);
                    if (lane == 0 && wj != 0.0) ppv += vj, sx -= gxj, sy -= gyj; // counted once, by the driver
                }
                if (lane == 0) ex = ex + pp.beta * sx, ey = ey + pp.beta * sy;
            }
            if (on) grad_e[s0 + lane] = make_double2(ex, ey);
        } else {
            wa_axis_warp(s0, n, 0, e_cell, e_off, cell_xy, anchor, inv_gamma, w, grad_e, vx, hx);
            wa_axis_warp(s0, n, 1, e_cell, e_off, cell_xy, anchor, inv_gamma, w, grad_e, vy, hy);
        }
        if (lane == 0) wl += w * (vx + vy), hp += hx + hy;
        if (pp.w_e && n > 32) { // nets beyond a warp: lane 0 walks the sinks in ascending pin id
            __syncwarp();
            if (lane == 0) {
                const double2 pd = entry_pos(e_cell[s0], e_off[s0], cell_xy, anchor);
                double sx = 0.0, sy = 0.0;
                for (int k = 0; k + 1 < n; ++k) {
                    const int j = gen_ord[s0 + k];
                    const double wt = pp.w_e[s0 + j];
                    if (wt == 0.0) continue;
                    const double2 ps = entry_pos(e_cell[s0 + j], e_off[s0 + j], cell_xy, anchor);
                    const double dx = ps.x - pd.x, dy = ps.y - pd.y;
                    double gx = 0.0, gy = 0.0;
                    if (pp.kind == 0) {
                        ppv += wt * (dx * dx + dy * dy);
                        gx = 2.0 * wt * dx, gy = 2.0 * wt * dy;
                    } else {
                        const double dist = sqrt(dx * dx + dy * dy);
                        ppv += wt * dist;
                        if (dist > 0.0) gx = wt * dx / dist, gy = wt * dy / dist;
                    }
                    double2 ge = grad_e[s0 + j];
                    ge.x = ge.x + pp.beta * gx, ge.y = ge.y + pp.beta * gy;
                    grad_e[s0 + j] = ge;
                    sx -= gx, sy -= gy;
                }
                double2 gd = grad_e[s0];
                gd.x = gd.x + pp.beta * sx, gd.y = gd.y + pp.beta * sy;
                grad_e[s0] = gd;
            }
            __syncwarp();
        }
    }
    block_sum3<kBlock>(wl, hp, ppv, sh);
    if (threadIdx.x == 0) {
        part_wl[blk0 + blockIdx.x] = wl, part_hp[blk0 + blockIdx.x] = hp;
        if (part_pp) part_pp[blk0 + blockIdx.x] = ppv;
    }
}

// =====================================================================================
// Pin-pair attraction (pin_pairs.cpp:17-49).  One thread per pin that appears in the
// ledger; its incidences are in ledger (map-key) order, so the per-pin sum has the
// reference's accumulation order.  beta * sum is added onto the pin's WA entry gradient,
// which is exactly the reference fold term pin_grad + beta * pp.d_pin (placer.cpp:323).
// Pair values are summed once per pair (on the lower pin's side).
// =====================================================================================
__global__ void __launch_bounds__(kBlock) k_pin_pairs(const int* __restrict__ n_pins_dev, const int* __restrict__ pp_start,
                                                      const int* __restrict__ pp_entry, const int* __restrict__ pp_inc,
                                                      const unsigned long long* __restrict__ led_key,
                                                      const double* __restrict__ led_w,
                                                      const int* __restrict__ pin_cell,
                                                      const double2* __restrict__ pin_off,
                                                      const double2* __restrict__ cell_xy,
                                                      const double2* __restrict__ anchor, int kind, double beta,
                                                      int n_net_entries, double2* __restrict__ grad_e,
                                                      double* __restrict__ part_pp,
                                                      const Ctrl* __restrict__ ctrl)
{
    __shared__ double sh[kBlock / 32];
    if (ctrl && ctrl->stopped) return;
    const int n_pins = *n_pins_dev;
    double val = 0.0;
    for (int i = blockIdx.x * kBlock + threadIdx.x; i < n_pins; i += gridDim.x * kBlock) {
        double sx = 0.0, sy = 0.0;
        for (int j = pp_start[i]; j < pp_start[i + 1]; ++j) {
            const int inc = pp_inc[j];
            const int q = inc >> 1;
            const bool second = inc & 1;
            const unsigned long long key = led_key[q];
            const int a = static_cast<int>(key >> 32), b = static_cast<int>(key & 0xFFFFFFFFull);
            const double w = led_w[q];
            const double2 pa = pin_pos(a, pin_cell, pin_off, cell_xy, anchor);
            const double2 pb = pin_pos(b, pin_cell, pin_off, cell_xy, anchor);
            const double dx = pa.x - pb.x;
            const double dy = pa.y - pb.y;
            double gx, gy;
            if (kind == 0) {
                if (!second) val += w * (dx * dx + dy * dy);
                gx = 2.0 * w * dx;
                gy = 2.0 * w * dy;
            } else {
                const double dist = sqrt(dx * dx + dy * dy);
                if (!second) val += w * dist;
                if (!(dist > 0.0)) continue;
                gx = w * dx / dist;
                gy = w * dy / dist;
            }
            if (second) sx -= gx, sy -= gy;
            else sx += gx, sy += gy;
        }
        const int e = pp_entry[i];
        if (e >= n_net_entries) { // off-net pin: pin_grad is 0, slot holds 0 + beta * pp
            grad_e[e] = make_double2(0.0 + beta * sx, 0.0 + beta * sy);
        } else if (e >= 0) {
            double2 g = grad_e[e];
            g.x = g.x + beta * sx;
            g.y = g.y + beta * sy;
            grad_e[e] = g;
        }
    }
    const double bv = block_sum<kBlock>(val, sh);
    if (threadIdx.x == 0) part_pp[blockIdx.x] = bv;
}

// =====================================================================================
// Density (density.cpp:66-158).  Scatter: one thread per movable cell rasterises its
// quadratic B-spline footprint into int64 fixed-point accumulators (order-independent,
// hence run-to-run deterministic).  Bins: excess = max(0, occ - cap), value / overflow
// partial sums, accumulators reset for the next evaluation.
// =====================================================================================

// Scatter over cells in spatial order (perm, refreshed by sort_cells_spatial): the block's
// footprints usually cover a small window of bins, which is accumulated in shared memory
// with shared int64 atomics and flushed once per bin; blocks whose window does not fit
// fall back to global atomics.  Integer adds commute, so the result is bitwise the same
// whatever the order or the path.
constexpr int kWinBins = 4096; // 32 KB of int64 accumulators

// Fixed-point entries into shared 32-bit limbs with no-return adds (RED; a 64-bit shared atomicAdd compiles
// to a CAS spin loop on sm_100a): a block adds at most 256 entries per bin, so each limb is sized to hold
// 256 of its parts.  LIMBS = 2 (|q| < 2^45, Grid::limbs): an unsigned 23-bit low part and a signed high
// part; LIMBS = 3: 21-bit low and middle parts and a signed top.  The flush recombines the exact int64 sum.
template <int LIMBS>
struct SmemLimbs {
    unsigned* w;    // LIMBS arrays of `stride` limbs
    int stride;
    __device__ __forceinline__ void add(long long k, unsigned long long u) const
    {
        const long long q = static_cast<long long>(u);
        if constexpr (LIMBS == 2) {
            atomicAdd(w + k, static_cast<unsigned>(q & 0x7FFFFF));
            atomicAdd(reinterpret_cast<int*>(w + stride) + k, static_cast<int>(q >> 23));
        } else {
            atomicAdd(w + k, static_cast<unsigned>(q & 0x1FFFFF));
            atomicAdd(w + stride + k, static_cast<unsigned>((q >> 21) & 0x1FFFFF));
            atomicAdd(reinterpret_cast<int*>(w + 2 * stride) + k, static_cast<int>(q >> 42));
        }
    }
    __device__ __forceinline__ long long sum(int k) const
    {
        if constexpr (LIMBS == 2)
            return static_cast<long long>(w[k]) + static_cast<long long>(static_cast<int>(w[stride + k])) * (1LL << 23);
        else
            return static_cast<long long>(w[k]) + static_cast<long long>(w[stride + k]) * (1LL << 21) +
                   static_cast<long long>(static_cast<int>(w[2 * stride + k])) * (1LL << 42);
    }
};

// 64-bit fixed-point add into shared memory as two native 32-bit atomics with an explicit carry
// (a 64-bit shared atomicAdd compiles to a CAS spin loop, ATOMS.CAST.SPIN.64, on sm_100a).
struct SmemAcc {
    unsigned* lo;
    unsigned* hi;
    __device__ __forceinline__ void add(long long k, unsigned long long v) const
    {
        const unsigned vl = static_cast<unsigned>(v), vh = static_cast<unsigned>(v >> 32);
        const unsigned old = atomicAdd(lo + k, vl);
        const unsigned carry = (old + vl < old) ? 1u : 0u;
        if (vh + carry) atomicAdd(hi + k, vh + carry);
    }
};

struct GlobalAcc {
    unsigned long long* p;
    __device__ __forceinline__ void add(long long k, unsigned long long v) const { atomicAdd(p + k, v); }
};

template <typename Acc>
__device__ __noinline__ void scatter_cell_wide(const double2 p, const double2 s, const GridDev& g, const Acc& acc,
                                               long long row_stride, int col0, int row0)
{   // general footprint (cells wider than ~2 bins): any number of bins per axis
    const Axis ax = make_axis(p.x, p.x + s.x, g.x0, g.bw, g.inv_bw, g.nx);
    const Axis ay = make_axis(p.y, p.y + s.y, g.y0, g.bh, g.inv_bh, g.ny);
    const double area = s.x * s.y;
    for (int bx = ax.b0; bx <= ax.b1; ++bx) {
        const double wx = axis_w(ax, bx);
        if (wx == 0.0) continue;
        const double aw = area * wx;
        const long long row = static_cast<long long>(bx - row0) * row_stride - col0;
        for (int by = ay.b0; by <= ay.b1; ++by) {
            const long long q = __double2ll_rn(aw * axis_w(ay, by) * g.scale);
            if (q) acc.add(row + by, static_cast<unsigned long long>(q));
        }
    }
}

// Five-bin footprint (axis5) scatter: entry (i, j) = area * wx_i * wy_j (density.cpp:127), in fixed point.
template <typename Acc>
__device__ __forceinline__ void scatter_cell5(double area, int bx, int by, const double (&wx)[kF5],
                                              const double (&wy)[kF5], const GridDev& g, const Acc& acc,
                                              long long row_stride, int col0, int row0)
{
#pragma unroll
    for (int i = 0; i < kF5; ++i) {
        if (wx[i] == 0.0) continue;
        // (area * wx) * scale * wy == (area * wx) * wy * scale bitwise: scale is a power of two
        const double aws = (area * wx[i]) * g.scale;
        const long long row = static_cast<long long>(bx + i - row0) * row_stride + (by - col0);
#pragma unroll
        for (int j = 0; j < kF5; ++j) {
            const long long q = __double2ll_rn(aws * wy[j]);
            if (q) acc.add(row + j, static_cast<unsigned long long>(q));
        }
    }
}

__global__ void __launch_bounds__(kBlock) k_density_scatter_win(int n_mov, const int* __restrict__ perm,
                                                                const double2* __restrict__ cell_xy,
                                                                const double2* __restrict__ cell_wh, GridDev g,
                                                                unsigned long long* __restrict__ acc,
                                                                const Ctrl* __restrict__ ctrl,
                                                                double2* __restrict__ xy_sp, double2* __restrict__ wh_sp)
{
    __shared__ unsigned win_lo[kWinBins], win_hi[kWinBins];
    __shared__ int bb[4];
    const bool stop = ctrl && ctrl->stopped; // (checked once the cell loads are in flight)
    const int i = blockIdx.x * kBlock + threadIdx.x;
    const bool valid = i < n_mov;
    double2 p = make_double2(0, 0), s = make_double2(1, 1);
    int bx0 = INT_MAX, bx1 = INT_MIN, by0 = INT_MAX, by1 = INT_MIN;
    double wx[kF5], wy[kF5], dw[kF5];
    int bx = 0, by = 0;
    bool fast = false;
    if (valid) {
        const int c = perm[i];
        p = cell_xy[c], s = cell_wh[c];
        xy_sp[i] = p, wh_sp[i] = s; // (for k_dens_grad)
        // cells of Grid::wide are scattered by k_density_scatter_wide; every other cell spans at most
        // 1.99 pitches, so its footprint has at most five bins per axis (axis5 succeeds)
        fast = !(s.x > g.wide_w || s.y > g.wide_h) &&
               axis5(p.x, p.x + s.x, g.x0, g.bw, g.inv_bw, g.nx, bx, wx, dw) &&
               axis5(p.y, p.y + s.y, g.y0, g.bh, g.inv_bh, g.ny, by, wy, dw);
        if (fast)
            bx0 = max(bx, 0), bx1 = min(bx + kF5 - 1, g.nx - 1), by0 = max(by, 0), by1 = min(by + kF5 - 1, g.ny - 1);
    }
    if (stop) return; // (uniform over the block)
    if (threadIdx.x == 0) bb[0] = INT_MAX, bb[1] = INT_MIN, bb[2] = INT_MAX, bb[3] = INT_MIN;
    int a0 = bx0, a1 = bx1, c0 = by0, c1 = by1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 = min(a0, __shfl_xor_sync(0xffffffffu, a0, o)), a1 = max(a1, __shfl_xor_sync(0xffffffffu, a1, o));
        c0 = min(c0, __shfl_xor_sync(0xffffffffu, c0, o)), c1 = max(c1, __shfl_xor_sync(0xffffffffu, c1, o));
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && a0 <= a1) {
        atomicMin(&bb[0], a0), atomicMax(&bb[1], a1), atomicMin(&bb[2], c0), atomicMax(&bb[3], c1);
    }
    __syncthreads();
    const int X0 = bb[0], Y0 = bb[2];
    const long long W = static_cast<long long>(bb[1]) - X0 + 1, H = static_cast<long long>(bb[3]) - Y0 + 1;
    if (X0 > bb[1]) return; // no movable cell in this block
    const double area = s.x * s.y;
    if (W * H <= kWinBins) {
        for (int k = threadIdx.x; k < static_cast<int>(W * H); k += kBlock) win_lo[k] = 0u, win_hi[k] = 0u;
        __syncthreads();
        if (fast) scatter_cell5(area, bx, by, wx, wy, g, SmemAcc{win_lo, win_hi}, H, Y0, X0);
        __syncthreads();
        const int h = static_cast<int>(H), n = static_cast<int>(W * H);
        for (int k = threadIdx.x; k < n; k += kBlock) {
            const unsigned long long v = (static_cast<unsigned long long>(win_hi[k]) << 32) | win_lo[k];
            const int col = k / h;
            if (v) atomicAdd(&acc[static_cast<long long>(X0 + col) * g.ny + (Y0 + k - col * h)], v);
        }
    } else if (fast) {
        scatter_cell5(area, bx, by, wx, wy, g, GlobalAcc{acc}, g.ny, 0, 0);
    }
}

template <int LIMBS>
__global__ void __launch_bounds__(kBlock) k_density_scatter_limbs(int n_mov, const int* __restrict__ perm,
                                                                const double2* __restrict__ cell_xy,
                                                                const double2* __restrict__ cell_wh, GridDev g,
                                                                unsigned long long* __restrict__ acc,
                                                                const Ctrl* __restrict__ ctrl,
                                                                double2* __restrict__ xy_sp, double2* __restrict__ wh_sp)
{
    constexpr int kW = LIMBS == 2 ? kWinBins : 4000; // (3 limbs: 48 KB of static shared memory)
    __shared__ unsigned win[LIMBS * kW];
    const SmemLimbs<LIMBS> SA{win, kW};
    __shared__ int bb[4];
    const bool stop = ctrl && ctrl->stopped; // (checked once the cell loads are in flight)
    const int i = blockIdx.x * kBlock + threadIdx.x;
    const bool valid = i < n_mov;
    double2 p = make_double2(0, 0), s = make_double2(1, 1);
    int bx0 = INT_MAX, bx1 = INT_MIN, by0 = INT_MAX, by1 = INT_MIN;
    double wx[kF5], wy[kF5], dw[kF5];
    int bx = 0, by = 0;
    bool fast = false;
    if (valid) {
        const int c = perm[i];
        p = cell_xy[c], s = cell_wh[c];
        xy_sp[i] = p, wh_sp[i] = s; // (for k_dens_grad)
        // cells of Grid::wide are scattered by k_density_scatter_wide; every other cell spans at most
        // 1.99 pitches, so its footprint has at most five bins per axis (axis5 succeeds)
        fast = !(s.x > g.wide_w || s.y > g.wide_h) &&
               axis5(p.x, p.x + s.x, g.x0, g.bw, g.inv_bw, g.nx, bx, wx, dw) &&
               axis5(p.y, p.y + s.y, g.y0, g.bh, g.inv_bh, g.ny, by, wy, dw);
        if (fast)
            bx0 = max(bx, 0), bx1 = min(bx + kF5 - 1, g.nx - 1), by0 = max(by, 0), by1 = min(by + kF5 - 1, g.ny - 1);
    }
    if (stop) return; // (uniform over the block)
    if (threadIdx.x == 0) bb[0] = INT_MAX, bb[1] = INT_MIN, bb[2] = INT_MAX, bb[3] = INT_MIN;
    int a0 = bx0, a1 = bx1, c0 = by0, c1 = by1;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a0 = min(a0, __shfl_xor_sync(0xffffffffu, a0, o)), a1 = max(a1, __shfl_xor_sync(0xffffffffu, a1, o));
        c0 = min(c0, __shfl_xor_sync(0xffffffffu, c0, o)), c1 = max(c1, __shfl_xor_sync(0xffffffffu, c1, o));
    }
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && a0 <= a1) {
        atomicMin(&bb[0], a0), atomicMax(&bb[1], a1), atomicMin(&bb[2], c0), atomicMax(&bb[3], c1);
    }
    __syncthreads();
    const int X0 = bb[0], Y0 = bb[2];
    const long long W = static_cast<long long>(bb[1]) - X0 + 1, H = static_cast<long long>(bb[3]) - Y0 + 1;
    if (X0 > bb[1]) return; // no movable cell in this block
    const double area = s.x * s.y;
    if (W * H <= kW) {
        for (int k = threadIdx.x; k < static_cast<int>(W * H); k += kBlock)
#pragma unroll
            for (int l = 0; l < LIMBS; ++l) win[l * kW + k] = 0u;
        __syncthreads();
        if (fast) scatter_cell5(area, bx, by, wx, wy, g, SA, H, Y0, X0);
        __syncthreads();
        const int h = static_cast<int>(H), n = static_cast<int>(W * H);
        for (int k = threadIdx.x; k < n; k += kBlock) {
            const long long v = SA.sum(k);
            const int col = k / h;
            if (v) atomicAdd(&acc[static_cast<long long>(X0 + col) * g.ny + (Y0 + k - col * h)],
                             static_cast<unsigned long long>(v));
        }
    } else if (fast) {
        scatter_cell5(area, bx, by, wx, wy, g, GlobalAcc{acc}, g.ny, 0, 0);
    }
}

// Cells of Grid::wide: global int64 atomics (they are few), five-bin form when it applies.
__global__ void __launch_bounds__(kBlock) k_density_scatter_wide(int n, const int* __restrict__ wide,
                                                                 const double2* __restrict__ cell_xy,
                                                                 const double2* __restrict__ cell_wh, GridDev g,
                                                                 unsigned long long* __restrict__ acc,
                                                                 const Ctrl* __restrict__ ctrl)
{
    if (ctrl && ctrl->stopped) return;
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const int c = wide[i];
    const double2 p = cell_xy[c], s = cell_wh[c];
    double wx[kF5], wy[kF5], dw[kF5];
    int bx, by;
    if (axis5(p.x, p.x + s.x, g.x0, g.bw, g.inv_bw, g.nx, bx, wx, dw) &&
        axis5(p.y, p.y + s.y, g.y0, g.bh, g.inv_bh, g.ny, by, wy, dw))
        scatter_cell5(s.x * s.y, bx, by, wx, wy, g, GlobalAcc{acc}, g.ny, 0, 0);
    else
        scatter_cell_wide(p, s, g, GlobalAcc{acc}, g.ny, 0, 0);
}

// Spatial order of the movable cells: key = 8x8-bin tile of the cell's lower-left corner.
__global__ void k_spatial_keys(int C, const double2* __restrict__ cell_xy, const uint8_t* __restrict__ fixed,
                               GridDev g, int tiles_y, unsigned fixed_key, unsigned* __restrict__ keys,
                               int* __restrict__ vals)
{
    const int c = blockIdx.x * kBlock + threadIdx.x;
    if (c >= C) return;
    const double2 p = cell_xy[c];
    const int bx = min(g.nx - 1, max(0, static_cast<int>((p.x - g.x0) * g.inv_bw)));
    const int by = min(g.ny - 1, max(0, static_cast<int>((p.y - g.y0) * g.inv_bh)));
    keys[c] = fixed[c] ? fixed_key : static_cast<unsigned>((bx >> 3) * tiles_y + (by >> 3)); // fixed: last
    vals[c] = c;
}

// Grid-stride over bin pairs (16-byte loads/stores), four pairs per thread per step with every load issued
// before use; one pass: read the accumulator, reset it, write excess.  Per block one (value, overflow)
// partial in fixed order.
constexpr int kBinsBlocks = 148 * 4;

__global__ void __launch_bounds__(kBlock) k_density_bins(long long B, GridDev g, long long* __restrict__ acc,
                                                         const double* __restrict__ base,
                                                         double* __restrict__ excess, double* __restrict__ part_d,
                                                         const Ctrl* __restrict__ ctrl, double* __restrict__ rho)
{
    pdl_trigger();
    pdl_wait();
    __shared__ double sh[2][kBlock / 32];
    if (ctrl && ctrl->stopped) return;
    double v2 = 0.0, v1 = 0.0;
    auto one = [&](long long q, long long k) {
        const double mov = static_cast<double>(q) * g.inv_scale;
        const double occ = base ? base[k] + mov : mov;
        if (rho) rho[k] = occ; // electrostatic model: the charge map
        const double ex = smax(0.0, occ - g.cap);
        v2 += ex * ex;
        v1 += ex;
        return ex;
    };
    const long long pairs = B / 2, stride = static_cast<long long>(gridDim.x) * kBlock;
    constexpr int U = 4;
    for (long long p0 = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; p0 < pairs; p0 += U * stride) {
        longlong2 q[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = p0 + u * stride;
            q[u] = p < pairs ? reinterpret_cast<const longlong2*>(acc)[p] : make_longlong2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long p = p0 + u * stride;
            if (p >= pairs) break;
            reinterpret_cast<longlong2*>(acc)[p] = make_longlong2(0, 0);
            double2 ex;
            ex.x = one(q[u].x, 2 * p);
            ex.y = one(q[u].y, 2 * p + 1);
            reinterpret_cast<double2*>(excess)[p] = ex;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (B & 1)) { // odd bin count: the last bin
        const long long q = acc[B - 1];
        acc[B - 1] = 0;
        excess[B - 1] = one(q, B - 1);
    }
    v2 = warp_sum(v2), v1 = warp_sum(v1);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[0][w] = v2, sh[1][w] = v1;
    __syncthreads();
    if (w == 0) {
        double a = lane < kBlock / 32 ? sh[0][lane] : 0.0, b = lane < kBlock / 32 ? sh[1][lane] : 0.0;
        a = warp_sum(a), b = warp_sum(b);
        if (lane == 0) part_d[2 * blockIdx.x] = a, part_d[2 * blockIdx.x + 1] = b;
    }
}

// =====================================================================================
// Finalize: deterministic fixed-order sums of all partials -> objective terms, trace
// row, stop / non-finite flags, and the schedule values of this iteration.
// =====================================================================================


constexpr int kFinBlock = 1024;

__global__ void __launch_bounds__(kFinBlock) k_finalize(FinArgs a, Ctrl* ctrl, IterCur* cur)
{
    pdl_trigger(); // (k_cells may start its fold now; it waits for this kernel before reading cur)
    __shared__ double sh[kFinBlock / 32];
    __shared__ int skip;
    if (threadIdx.x == 0) skip = ctrl ? ctrl->stopped : 0;
    __syncthreads();
    if (skip) {
        if (threadIdx.x == 0) cur->do_adam = 0;
        return;
    }
    double r[5] = {0, 0, 0, 0, 0}; // wl, hpwl, pp, density value, overflow numerator
    // loads batched 8 deep (all issued before the adds) so the single block is not latency-serialised
    auto acc = [&](const double* p, int n, int stride, int off, double& out) {
        for (int i0 = threadIdx.x; i0 < n; i0 += 8 * kFinBlock) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * kFinBlock;
                v[u] = i < n ? p[static_cast<long long>(i) * stride + off] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) out += v[u];
        }
    };
    acc(a.part_wl, a.nb_wa, 1, 0, r[0]);
    acc(a.part_hp, a.nb_wa, 1, 0, r[1]);
    acc(a.part_pp, a.nb_pp, 1, 0, r[2]);
    acc(a.part_d, a.nb_d, 2, 0, r[3]);
    acc(a.part_d, a.nb_d, 2, 1, r[4]);
    {   // one fixed-order tree for all five sums
        __shared__ double sh5[5][kFinBlock / 32];
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
        for (int k = 0; k < 5; ++k) r[k] = warp_sum(r[k]);
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 5; ++k) sh5[k][w] = r[k];
        __syncthreads();
        if (w != 0) return;
#pragma unroll
        for (int k = 0; k < 5; ++k) r[k] = warp_sum(lane < kFinBlock / 32 ? sh5[k][lane] : 0.0);
    }
    (void)sh;
    double wl = r[0], hp = r[1], pp = r[2], d2 = r[3], d1 = r[4];
    if (threadIdx.x != 0) return;
    const int it = ctrl ? ctrl->iter : 0;
    const double lambda = a.sched ? a.sched[it].lambda : a.lambda_single;
    Terms t;
    t.wl = wl, t.hpwl = hp, t.pp = a.nb_pp ? pp : 0.0, t.density = d2;
    t.overflow = a.total_movable > 0.0 ? d1 / a.total_movable : 0.0;
    t.value = t.wl + lambda * t.density + a.beta * t.pp;
    *a.terms = t;
    const bool finite = isfinite(t.value) && isfinite(t.wl) && isfinite(t.density) && isfinite(t.pp);
    cur->lambda = lambda;
    cur->iter = it;
    cur->do_adam = 0;
    if (!ctrl) return;
    if (!finite) atomicMin(&ctrl->nonfinite_at, it);
    if (a.trace) {
        TraceRowDev r;
        r.iter = it;
        r.has_timing = a.timing_row && a.timing_row[0] != 0.0;
        r.tns = r.has_timing ? a.timing_row[1] : 0.0;
        r.wns = r.has_timing ? a.timing_row[2] : 0.0;
        r.hpwl = t.hpwl, r.overflow = t.overflow, r.wl_term = t.wl, r.density_term = t.density;
        r.pp_term = t.pp, r.lambda = lambda, r.beta_pp = a.beta * t.pp;
        a.trace[it] = r;
    }
    if (a.timing_row_clear) a.timing_row_clear[0] = 0.0;
    ctrl->rows = it + 1;
    if (ctrl->engaged && t.overflow <= a.stop_overflow) { // placer.cpp:459-462
        ctrl->stopped = 1;
        return;
    }
    if (a.sched) {
        cur->lr = a.sched[it].lr, cur->c1 = a.sched[it].c1, cur->c2 = a.sched[it].c2;
        cur->do_adam = 1;
    }
    ctrl->iter = it + 1;
}

// The two halves of k_finalize (engine iteration graph).  Each series is reduced with exactly
// k_finalize's thread layout and tree, so the terms are bitwise the single kernel's.
template <int K>
__device__ __forceinline__ bool fin_reduce(const double* const (&p)[K], const int (&n)[K], const int (&stride)[K],
                                           const int (&off)[K], double (&r)[K])
{
    for (int k = 0; k < K; ++k) r[k] = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k)
        for (int i0 = threadIdx.x; i0 < n[k]; i0 += 8 * kFinBlock) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * kFinBlock;
                v[u] = i < n[k] ? p[k][static_cast<long long>(i) * stride[k] + off[k]] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) r[k] += v[u];
        }
    __shared__ double sh[K][kFinBlock / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) r[k] = warp_sum(r[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) sh[k][w] = r[k];
    __syncthreads();
    if (w != 0) return false;
#pragma unroll
    for (int k = 0; k < K; ++k) r[k] = warp_sum(lane < kFinBlock / 32 ? sh[k][lane] : 0.0);
    return threadIdx.x == 0;
}

__global__ void __launch_bounds__(kFinBlock) k_fin_density(FinArgs a, Ctrl* ctrl, IterCur* cur)
{
    __shared__ int skip;
    if (threadIdx.x == 0) skip = ctrl->stopped;
    __syncthreads();
    if (skip) {
        if (threadIdx.x == 0) cur->do_adam = 0, cur->live = 0;
        return;
    }
    double r[2];
    if (!fin_reduce<2>({a.part_d, a.part_d}, {a.nb_d, a.nb_d}, {2, 2}, {0, 1}, r)) return;
    const int it = ctrl->iter;
    const double lambda = a.sched ? a.sched[it].lambda : a.lambda_single;
    const double overflow = a.total_movable > 0.0 ? r[1] / a.total_movable : 0.0;
    cur->lambda = lambda, cur->iter = it, cur->do_adam = 0, cur->live = 1, cur->stop = 0;
    cur->density = r[0], cur->overflow = overflow;
    // placer.cpp:459-462.  The flag the other kernels read is raised by k_fin_terms, after this iteration's
    // WA kernels: they run beside this kernel and must not see the stop before they have run.
    if (ctrl->engaged && overflow <= a.stop_overflow) {
        cur->stop = 1;
        return;
    }
    if (a.sched) {
        cur->lr = a.sched[it].lr, cur->c1 = a.sched[it].c1, cur->c2 = a.sched[it].c2;
        cur->do_adam = 1;
    }
    // (ctrl->iter advances in k_fin_terms: kernels beside this one — the partitioned engine's λ · density
    // gradient fold — still read this iteration's index)
}

__global__ void __launch_bounds__(kFinBlock) k_fin_terms(FinArgs a, Ctrl* ctrl, const IterCur* cur)
{
    if (!cur->live) return; // (uniform)
    double r[3];
    if (!fin_reduce<3>({a.part_wl, a.part_hp, a.part_pp}, {a.nb_wa, a.nb_wa, a.nb_pp}, {1, 1, 1}, {0, 0, 0}, r))
        return;
    const int it = cur->iter;
    const double lambda = cur->lambda;
    Terms t;
    t.wl = r[0], t.hpwl = r[1], t.pp = a.nb_pp ? r[2] : 0.0, t.density = cur->density;
    t.overflow = cur->overflow;
    t.value = t.wl + lambda * t.density + a.beta * t.pp;
    *a.terms = t;
    const bool finite = isfinite(t.value) && isfinite(t.wl) && isfinite(t.density) && isfinite(t.pp);
    if (!finite) atomicMin(&ctrl->nonfinite_at, it);
    if (a.trace) {
        TraceRowDev row;
        row.iter = it;
        row.has_timing = a.timing_row && a.timing_row[0] != 0.0;
        row.tns = row.has_timing ? a.timing_row[1] : 0.0;
        row.wns = row.has_timing ? a.timing_row[2] : 0.0;
        row.hpwl = t.hpwl, row.overflow = t.overflow, row.wl_term = t.wl, row.density_term = t.density;
        row.pp_term = t.pp, row.lambda = lambda, row.beta_pp = a.beta * t.pp;
        a.trace[it] = row;
    }
    if (a.timing_row_clear) a.timing_row_clear[0] = 0.0;
    ctrl->rows = it + 1;
    if (cur->stop) ctrl->stopped = 1;
    else ctrl->iter = it + 1;
}

// =====================================================================================
// Density gradient (density.cpp:148-156), one thread per movable cell in the scatter's spatial
// order, so neighbouring threads read neighbouring excess bins (L1 hits).  Regrouped per bin
// column: dgx = sum_bx area*dwx(bx) * 2*sum_by f(bx,by)*wy(by), dgy = sum_bx area*wx(bx) * 2*sum_by f*dwy.
// =====================================================================================
__device__ __noinline__ double2 dens_grad_wide(const double2 p, const double2 s, const GridDev& g,
                                               const double* __restrict__ excess, double fscale)
{   // general footprint (cells wider than ~2 bins)
    const Axis ax = make_axis(p.x, p.x + s.x, g.x0, g.bw, g.inv_bw, g.nx);
    const Axis ay = make_axis(p.y, p.y + s.y, g.y0, g.bh, g.inv_bh, g.ny);
    const double area = s.x * s.y;
    double dgx = 0.0, dgy = 0.0;
    for (int bx = ax.b0; bx <= ax.b1; ++bx) {
        double wx, dwx;
        axis_at(ax, bx, wx, dwx);
        if (wx == 0.0 && dwx == 0.0) continue;
        double sx = 0.0, sy = 0.0;
        for (int by = ay.b0; by <= ay.b1; ++by) {
            double wy, dwy;
            axis_at(ay, by, wy, dwy);
            if (wy == 0.0 && dwy == 0.0) continue;
            const double f = excess[static_cast<long long>(bx) * g.ny + by];
            sx += f * wy, sy += f * dwy;
        }
        dgx += (area * dwx) * (fscale * sx);
        dgy += (area * wx) * (fscale * sy);
    }
    return make_double2(dgx, dgy);
}

// Five-bin footprint gradient (axis5 on both axes): per bin column, dgx += area*dwx * fscale*sum f*wy,
// dgy += area*wx * fscale*sum f*dwy.  Only the in-grid bins of the footprint (span = D + 3 per axis) are
// read; the column sums are fused multiply-adds (within the 1e-9 density tolerance).
__device__ __forceinline__ double2 dens_grad5(int bx, int by, int sx_n, int sy_n, const double (&wx)[kF5],
                                              const double (&dwx)[kF5], const double (&wy)[kF5],
                                              const double (&dwy)[kF5], double area, const GridDev& g,
                                              const double* __restrict__ excess, double fscale)
{
    double dgx = 0.0, dgy = 0.0;
    // footprint bins inside the grid: a in [a0, a1), j in [j0, j1)
    const int a0 = max(0, -bx), a1 = min(sx_n, g.nx - bx), j0 = max(0, -by), j1 = min(sy_n, g.ny - by);
#pragma unroll
    for (int a = 0; a < kF5; ++a) {
        if (a < a0 || a >= a1) continue; // (outside the grid, or no support)
        const double* ex = excess + static_cast<long long>(bx + a) * g.ny + by;
        double f[kF5];
#pragma unroll
        for (int j = 0; j < kF5; ++j) f[j] = (j >= j0 && j < j1) ? ex[j] : 0.0;
        double sx = 0.0, sy = 0.0;
#pragma unroll
        for (int j = 0; j < kF5; ++j) sx = __fma_rn(f[j], wy[j], sx), sy = __fma_rn(f[j], dwy[j], sy);
        dgx += (area * dwx[a]) * (fscale * sx);
        dgy += (area * wx[a]) * (fscale * sy);
    }
    return make_double2(dgx, dgy);
}

// field = excess with fscale 2 (d sum excess^2, density.cpp:148-156) or the potential with fscale 1.
// Cells of Grid::wide are skipped here (k_dens_grad_wide).
__global__ void __launch_bounds__(kBlock, 4) k_dens_grad(int n_mov, const int* __restrict__ perm,
                                                      const double2* __restrict__ xy_sp,
                                                      const double2* __restrict__ wh_sp, GridDev g,
                                                      const double* __restrict__ excess, double2* __restrict__ dgrad,
                                                      const Ctrl* __restrict__ ctrl, double fscale)
{   // A programmatic dependent of the bins kernel: everything an earlier kernel of the iteration wrote (the
    // scatter's spatial-order copies, the excess field, the stop flag) is read after pdl_wait() — a kernel
    // may start once its primary's CTAs have exited, before their writes are guaranteed visible (loading
    // the scatter's copies before the wait was measured to read stale data under compute-sanitizer).
    pdl_trigger();
    pdl_wait();
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n_mov) return;
    const double2 p = xy_sp[i], s = wh_sp[i];
    const bool stop = ctrl && ctrl->stopped;
    if (stop || s.x > g.wide_w || s.y > g.wide_h) return;
    double wx[kF5], dwx[kF5], wy[kF5], dwy[kF5];
    int bx, by, nx5, ny5;
    axis5(p.x, p.x + s.x, g.x0, g.bw, g.inv_bw, g.nx, bx, wx, dwx, &nx5);
    axis5(p.y, p.y + s.y, g.y0, g.bh, g.inv_bh, g.ny, by, wy, dwy, &ny5);
    dgrad[perm[i]] = dens_grad5(bx, by, nx5, ny5, wx, dwx, wy, dwy, s.x * s.y, g, excess, fscale);
}

__global__ void __launch_bounds__(kBlock) k_dens_grad_wide(int n, const int* __restrict__ wide,
                                                           const double2* __restrict__ cell_xy,
                                                           const double2* __restrict__ cell_wh, GridDev g,
                                                           const double* __restrict__ excess,
                                                           double2* __restrict__ dgrad, const Ctrl* __restrict__ ctrl,
                                                           double fscale)
{
    if (ctrl && ctrl->stopped) return;
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    const int c = wide[i];
    const double2 p = cell_xy[c], s = cell_wh[c];
    double wx[kF5], dwx[kF5], wy[kF5], dwy[kF5];
    int bx, by, nx5, ny5;
    if (axis5(p.x, p.x + s.x, g.x0, g.bw, g.inv_bw, g.nx, bx, wx, dwx, &nx5) &&
        axis5(p.y, p.y + s.y, g.y0, g.bh, g.inv_bh, g.ny, by, wy, dwy, &ny5))
        dgrad[c] = dens_grad5(bx, by, nx5, ny5, wx, dwx, wy, dwy, s.x * s.y, g, excess, fscale);
    else
        dgrad[c] = dens_grad_wide(p, s, g, excess, fscale);
}

// =====================================================================================
// Cell kernel: gradient fold (placer.cpp:318-333) + lambda * density gradient + Adam
// (placer.cpp:345-356) + write-back / clamp (placer.cpp:472-476), one thread per cell.
// =====================================================================================
struct CellArgs {
    int C;
    const int* ent_start;
    const int* ent;
    const double2* grad_e;
    const uint8_t* fixed;
    double2* xy;
    const double2* wh;
    const double2* dgrad;
    double2* d_cell;    // optional gradient output
    const double2* folded; // partitioned mode: the all-reduced fold (skips the fold)
    bool dgrad_folded;     // ... which already holds lambda * density gradient (sharded density)
    double2* m;         // Adam state (iteration mode)
    double2* v;
    double b1, b2, eps;
    double core_x0, core_y0, core_x1, core_y1;
};

// In the iteration graph this is a programmatic dependent of k_finalize: its CTAs are resident when
// finalize ends, but everything is read after pdl_wait() — reading the WA kernels' entry gradients
// before it (they completed before finalize started) was measured to see stale data.
__global__ void __launch_bounds__(kBlock, 5) k_cells(CellArgs a, const IterCur* __restrict__ cur, Ctrl* ctrl)
{
    pdl_trigger();
    pdl_wait();
    const int c = blockIdx.x * kBlock + threadIdx.x;
    if (c >= a.C) return;
    double gx = 0.0, gy = 0.0;
    if (!a.folded) { // fold in ascending pin order (placer.cpp:318-325); loads batched 4 at a time
        const int j0 = a.ent_start[c], j1 = a.ent_start[c + 1];
        for (int j = j0; j < j1; j += 4) {
            double2 ge[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) ge[k] = (j + k < j1) ? a.grad_e[a.ent[j + k]] : make_double2(0.0, 0.0);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (j + k < j1) gx += ge[k].x, gy += ge[k].y;
        }
    }
    const bool fixed = a.fixed[c];
    const double2 dg = fixed ? make_double2(0.0, 0.0) : a.dgrad[c];
    if (a.folded) gx = a.folded[c].x, gy = a.folded[c].y;
    const bool adam = cur->do_adam;
    if (ctrl && !adam && !a.d_cell) return; // stopped: nothing to do
    if (fixed) {
        if (a.d_cell) a.d_cell[c] = make_double2(0.0, 0.0);
        return;
    }
    const double lambda = cur->lambda;
    if (!a.dgrad_folded) {
        gx += lambda * dg.x;
        gy += lambda * dg.y;
    }
    if (ctrl && !(isfinite(gx) && isfinite(gy))) atomicMin(&ctrl->nonfinite_at, cur->iter);
    if (a.d_cell) a.d_cell[c] = make_double2(gx, gy);
    if (!adam) return;
    const double2 p = a.xy[c], s = a.wh[c];
    double2 m = a.m[c], v = a.v[c];
    const double lr = cur->lr, c1 = cur->c1, c2 = cur->c2;
    m.x = a.b1 * m.x + (1.0 - a.b1) * gx;
    m.y = a.b1 * m.y + (1.0 - a.b1) * gy;
    v.x = a.b2 * v.x + (1.0 - a.b2) * gx * gx;
    v.y = a.b2 * v.y + (1.0 - a.b2) * gy * gy;
    double x = p.x - lr * (m.x / c1) / (sqrt(v.x / c2) + a.eps);
    double y = p.y - lr * (m.y / c1) / (sqrt(v.y / c2) + a.eps);
    const double xhi = a.core_x1 - s.x, yhi = a.core_y1 - s.y; // clamp_to_core, placer.cpp:99-103
    x = x < a.core_x0 ? a.core_x0 : (xhi < x ? xhi : x);
    y = y < a.core_y0 ? a.core_y0 : (yhi < y ? yhi : y);
    a.m[c] = m, a.v[c] = v;
    a.xy[c] = make_double2(x, y);
}

// Partitioned mode: this rank's share of the fold (placer.cpp:318-325) — entries of other ranks' nets
// hold 0 — into the all-reduce buffer.
__global__ void __launch_bounds__(kBlock) k_fold(int C, const int* __restrict__ ent_start, const int* __restrict__ ent,
                                                 const double2* __restrict__ grad_e, double2* __restrict__ out,
                                                 const Ctrl* __restrict__ ctrl)
{
    const int c = blockIdx.x * kBlock + threadIdx.x;
    if (c >= C || (ctrl && ctrl->stopped)) return;
    double gx = 0.0, gy = 0.0;
    for (int j = ent_start[c]; j < ent_start[c + 1]; ++j) {
        const double2 g = grad_e[ent[j]];
        gx += g.x, gy += g.y;
    }
    out[c] = make_double2(gx, gy);
}

// hpwl_total on caller-provided pin positions (wirelength.cpp:74-85), one thread per net.
__global__ void __launch_bounds__(kBlock) k_hpwl_pins(int N, const int* __restrict__ net_start,
                                                      const int* __restrict__ net_pins,
                                                      const double2* __restrict__ pin_xy, double* __restrict__ part)
{
    __shared__ double sh[kBlock / 32];
    const int e = blockIdx.x * kBlock + threadIdx.x;
    double h = 0.0;
    if (e < N) {
        const int s0 = net_start[e], s1 = net_start[e + 1];
        if (s1 - s0 >= 2) {
            const double2 p0 = pin_xy[net_pins[s0]];
            double xl = p0.x, xh = p0.x, yl = p0.y, yh = p0.y;
            for (int j = s0 + 1; j < s1; ++j) {
                const double2 p = pin_xy[net_pins[j]];
                xl = smin(xl, p.x), xh = smax(xh, p.x), yl = smin(yl, p.y), yh = smax(yh, p.y);
            }
            h = (xh - xl) + (yh - yl);
        }
    }
    h = block_sum<kBlock>(h, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = h;
}

// Adam on a flat device vector (AdamState::step for the reference-shaped host API).
__global__ void k_adam_flat(long long n, double* x, const double* g, double* m, double* v, double lr, double b1,
                            double b2, double eps, double c1, double c2)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= n) return;
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    x[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
}

// =====================================================================================
// host side
// =====================================================================================
GridDev grid_dev(const tdpg_session* s)
{
    const Grid& g = s->grid;
    return GridDev{g.nx, g.ny, g.x0, g.y0, g.bw, g.bh, g.cap, g.scale, g.inv_scale, g.total_movable, 1.0 / g.bw,
                   1.0 / g.bh, g.wide_w, g.wide_h};
}

int wa_blocks(const tdpg_session* s) { return std::max(1, s->n_wa_blocks); }
int pp_blocks(const tdpg_session*) { return 148 * 4; }
int bins_blocks(const tdpg_session* s)
{
    return std::max(1, std::min(kBinsBlocks, static_cast<int>(blocks_for((s->grid.bins() + 1) / 2, kBlock))));
}

// Per-pin incidence CSR of the ledger (rebuilt when the ledger changes).
__global__ void k_pp_inc_keys(long long Q, const unsigned long long* key, unsigned long long* out)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= Q) return;
    const unsigned long long k = key[i];
    out[2 * i] = (k >> 32 << 32) | static_cast<unsigned long long>(2 * i);
    out[2 * i + 1] = (k << 32) | static_cast<unsigned long long>(2 * i + 1);
}

__global__ void k_pp_csr(long long n, const unsigned long long* sorted, int* pp_inc, int* pin_of, int* head)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= n) return;
    const unsigned long long k = sorted[i];
    pp_inc[i] = static_cast<int>(k & 0xFFFFFFFFull);
    pin_of[i] = static_cast<int>(k >> 32);
    head[i] = (i == 0 || (sorted[i - 1] >> 32) != (k >> 32)) ? 1 : 0;
}

__global__ void k_pp_heads(long long n, const int* head, const int* head_pos, const int* pin_of, const int* pin_entry,
                           int* pp_start, int* pp_entry, int* n_pins_out)
{
    const long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x;
    if (i >= n) return;
    if (head[i]) {
        const int h = head_pos[i];
        pp_start[h] = static_cast<int>(i);
        pp_entry[h] = pin_entry[pin_of[i]];
    }
    if (i == n - 1) {
        const int total = head_pos[i] + head[i];
        pp_start[total] = static_cast<int>(n);
        *n_pins_out = total;
    }
}

void rebuild_pp_incidence(tdpg_session* s)
{
    if (!s->pp_dirty) return;
    s->pp_dirty = false;
    const long long Q = s->Q, n = 2 * Q;
    // capacity: every pair is a net arc, so Q <= A_net
    const size_t cap = static_cast<size_t>(std::max<long long>(n, 2LL * s->A_net)) + 2;
    s->pp_inc.reserve(cap);
    s->pp_start.reserve(cap + 1);
    s->pp_entry.reserve(cap);
    s->pp_pins.reserve(4); // pp_pins[0] = number of distinct pins (device)
    if (Q == 0) {
        s->pp_pins.zero(s->st, 1);
        s->n_pp_pins = 0;
        return;
    }
    s->sort_k0.reserve(cap), s->sort_k1.reserve(cap), s->sort_v0.reserve(cap), s->sort_v1.reserve(cap);
    k_pp_inc_keys<<<blocks_for(Q, kBlock), kBlock, 0, s->st>>>(Q, s->led_key, s->sort_k0);
    CK_LAUNCH();
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, s->sort_k0.p, s->sort_k1.p, static_cast<int>(n), 0, 64, s->st);
    void* tmp = cub_scratch(s, bytes);
    CK(cub::DeviceRadixSort::SortKeys(tmp, bytes, s->sort_k0.p, s->sort_k1.p, static_cast<int>(n), 0, 64, s->st));
    int* pin_of = s->sort_v0.p;
    int* head = s->sort_v1.p;
    int* head_pos = reinterpret_cast<int*>(s->sort_k0.p); // k0 free now (cap >= n ints)
    k_pp_csr<<<blocks_for(n, kBlock), kBlock, 0, s->st>>>(n, s->sort_k1, s->pp_inc, pin_of, head);
    CK_LAUNCH();
    bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, head, head_pos, static_cast<int>(n), s->st);
    tmp = cub_scratch(s, bytes);
    CK(cub::DeviceScan::ExclusiveSum(tmp, bytes, head, head_pos, static_cast<int>(n), s->st));
    k_pp_heads<<<blocks_for(n, kBlock), kBlock, 0, s->st>>>(n, head, head_pos, pin_of, s->pin_entry, s->pp_start,
                                                            s->pp_entry, s->pp_pins);
    CK_LAUNCH();
}

// TDPG_WA_GROUPS: 0 one launch per size class, 1 (default) classes 2-5 and 6-8 in two launches, 2 all
// in one (measured at 1M: 0.301 / 0.296 / 0.334 ms per iteration).
inline int wa_groups()
{
    static const int g = [] {
        const char* e = std::getenv("TDPG_WA_GROUPS");
        return e ? std::atoi(e) : 1;
    }();
    return g;
}

// TDPG_WA_AHEAD: prefetch distance unit of the WA kernels' L2 prefetch (the 2-5 group prefetches 4x, the
// 6-8 group 2x this many blocks ahead; 0 disables it).  Measured at 1M (WA serialised, bench): 0: 111-113 us,
// 37: 112, 74 (default): 107, 148: 110.
inline int wa_ahead()
{
    static const int a = [] {
        const char* e = std::getenv("TDPG_WA_AHEAD");
        return e ? std::atoi(e) : 74;
    }();
    return a;
}

// TDPG_WA_AXIS=0 selects the one-thread-per-net class kernels (A/B switch).
inline bool wa_axis_split()
{
    static const bool on = [] {
        const char* e = std::getenv("TDPG_WA_AXIS");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

WaAxisArgs wa_axis_args(tdpg_session* s, const double* nw, double inv_gamma, double* pw, double* ph, const PPArgs& pp,
                        double* ppart)
{
    WaAxisArgs A;
    A.blk = s->wa_blk, A.net_by_size = s->net_by_size, A.e_cell = s->e_cell;
    A.e_off = reinterpret_cast<const double*>(s->e_off.p), A.cell_xy = reinterpret_cast<const double*>(s->cell_xy.p);
    A.anchor = reinterpret_cast<const double*>(s->anchor.p), A.net_w = nw, A.inv_gamma = inv_gamma;
    A.grad_e = reinterpret_cast<double*>(s->grad_e.p), A.part_wl = pw, A.part_hp = ph, A.pp = pp, A.part_pp = ppart;
    for (int k = 0; k <= 8; ++k) {
        A.cls_blk0[k] = s->wa_cls_blk0[k], A.cls_net0[k] = s->wa_cls_net0[k], A.cls_net1[k] = s->wa_cls_net1[k];
        A.cls_pos0[k] = s->wa_cls_pos0[k];
    }
    A.cls_blk0[9] = s->wa_cls_blk0[0]; // (the generic blocks follow class 8; an empty class starts where
                                       // the next one does, so in wa_blk_of the last match wins)
    return A;
}

// The class's block range clipped to this rank's partition [part_b0, part_b1) (whole design at world 1).
inline bool wa_range(const tdpg_session* s, int cls, int& b0, int& nb)
{
    const int lo = s->part_active ? s->part_b0 : 0, hi = s->part_active ? s->part_b1 : s->n_wa_blocks;
    b0 = std::max(s->wa_cls_blk0[cls], lo);
    nb = std::min(s->wa_cls_blk0[cls] + s->wa_cls_nblk[cls], hi) - b0;
    return nb > 0;
}

template <int N>
void launch_wa_class(tdpg_session* s, const double* nw, double inv_gamma, double* pw, double* ph, const PPArgs& pp,
                     double* ppart, const Ctrl* ctrl, cudaStream_t st)
{
    int b0, nb;
    if (!wa_range(s, N, b0, nb)) return;
    if (wa_axis_split()) {
        k_wa_axis<N><<<nb, 2 * kBlock, 0, st>>>(b0, wa_axis_args(s, nw, inv_gamma, pw, ph, pp, ppart), ctrl);
        CK_LAUNCH();
        return;
    }
    k_wa_class<N><<<nb, kBlock, 0, st>>>(b0, s->wa_blk, s->net_by_size, s->e_cell,
                                                           s->e_off, s->cell_xy, s->anchor, nw, inv_gamma, s->grad_e,
                                                           pw, ph, pp, ppart, ctrl);
    CK_LAUNCH();
}

// WA (+ fused pin pairs when pp_fused: the engine's dense ledger) over all size classes.  The class
// kernels touch disjoint nets; with branch streams (graph capture) each class runs on its own branch
// so the small per-class grids overlap instead of draining the GPU one after another.
void launch_wirelength_pp(tdpg_session* s, double gamma, bool use_net_w, double* part_wl, double* part_hp,
                          bool pp_fused, int kind, double beta, double* part_pp, const Ctrl* ctrl,
                          const cudaStream_t* branch, int n_branch)
{
    const double* nw = use_net_w ? s->net_w.p : nullptr;
    const double ig = 1.0 / gamma;
    PPArgs pp{nullptr, nullptr, nullptr, beta, kind};
    if (pp_fused) pp = PPArgs{s->pp_mask.p, s->pp_ord.p, s->ppw_e.p, beta, kind};
    double* ppart = pp_fused ? part_pp : nullptr;
    auto st = [&](int k) { return n_branch > 0 ? branch[k % n_branch] : s->st; };
    const int groups = wa_groups();
    if (groups > 0 && wa_axis_split()) { // size classes merged into one or two launches
        const WaAxisArgs A = wa_axis_args(s, nw, ig, part_wl, part_hp, pp, ppart);
        auto range = [&](int lo, int hi, int& b0, int& nb) {
            const int plo = s->part_active ? s->part_b0 : 0, phi = s->part_active ? s->part_b1 : s->n_wa_blocks;
            b0 = std::max(s->wa_cls_blk0[lo], plo);
            nb = std::min(s->wa_cls_blk0[hi] + s->wa_cls_nblk[hi], phi) - b0;
            return nb > 0;
        };
        int b0, nb;
        if (groups == 1) {
            if (range(2, 5, b0, nb)) k_wa_axis_group<2, 5, 2><<<nb, 2 * kBlock, 0, st(1)>>>(b0, A, ctrl, 4 * wa_ahead());
            if (range(6, 8, b0, nb)) k_wa_axis_group<6, 8, 1><<<nb, 2 * kBlock, 0, st(2)>>>(b0, A, ctrl, 2 * wa_ahead());
        } else {
            if (range(2, 8, b0, nb)) k_wa_axis_group<2, 8, 1><<<nb, 2 * kBlock, 0, st(1)>>>(b0, A, ctrl, 2 * wa_ahead());
        }
        CK_LAUNCH();
    } else {
    launch_wa_class<2>(s, nw, ig, part_wl, part_hp, pp, ppart, ctrl, st(1));
    launch_wa_class<3>(s, nw, ig, part_wl, part_hp, pp, ppart, ctrl, st(2));
    launch_wa_class<4>(s, nw, ig, part_wl, part_hp, pp, ppart, ctrl, st(3));
    launch_wa_class<5>(s, nw, ig, part_wl, part_hp, pp, ppart, ctrl, st(4));
    launch_wa_class<6>(s, nw, ig, part_wl, part_hp, pp, ppart, ctrl, st(5));
    launch_wa_class<7>(s, nw, ig, part_wl, part_hp, pp, ppart, ctrl, st(6));
    launch_wa_class<8>(s, nw, ig, part_wl, part_hp, pp, ppart, ctrl, st(7));
    }
    int g0, gn;
    if (wa_range(s, 0, g0, gn)) {
        k_wa_generic<<<gn, kBlock, 0, st(0)>>>(g0, s->wa_cls_blk0[0], s->wa_gen_nets, s->net_by_size,
                                                              s->wa_gen_start, s->e_cell, s->e_off,
                                                              s->cell_xy, s->anchor, nw, ig, s->grad_e, part_wl,
                                                              part_hp, pp, s->wa_gen_ord, ppart, ctrl);
        CK_LAUNCH();
    }
}

void launch_wirelength(tdpg_session* s, double gamma, bool use_net_w, double* part_wl, double* part_hp, int nblk,
                       const Ctrl* ctrl)
{
    (void)nblk;
    launch_wirelength_pp(s, gamma, use_net_w, part_wl, part_hp, false, 0, 0.0, nullptr, ctrl, nullptr, 0);
}

void launch_wirelength(tdpg_session* s, double gamma, bool use_net_w, double* part_wl, double* part_hp, int nblk)
{
    launch_wirelength(s, gamma, use_net_w, part_wl, part_hp, nblk, nullptr);
}

void launch_pp(tdpg_session* s, int kind, double beta, double* part_pp, int nblk, const Ctrl* ctrl)
{
    k_pin_pairs<<<nblk, kBlock, 0, s->st>>>(s->pp_pins, s->pp_start, s->pp_entry, s->pp_inc, s->led_key, s->led_w,
                                            s->pin_cell, s->pin_off, s->cell_xy, s->anchor, kind, beta, s->E_lay,
                                            s->grad_e, part_pp, ctrl);
    CK_LAUNCH();
}

void launch_pp(tdpg_session* s, int kind, double beta, double* part_pp, int nblk)
{
    launch_pp(s, kind, beta, part_pp, nblk, nullptr);
}

// Refresh the spatial permutation of the movable cells (radix sort by 8x8-bin tile).
void sort_cells_spatial(tdpg_session* s)
{
    Grid& gr = s->grid;
    const int C = s->C;
    if (C == 0) return;
    gr.perm.reserve(C), gr.perm_keys.reserve(2 * static_cast<size_t>(C)), gr.perm_tmp.reserve(C);
    gr.xy_sp.reserve(C), gr.wh_sp.reserve(C);
    const GridDev g = grid_dev(s);
    const int tiles_y = (g.ny + 7) / 8, tiles_x = (g.nx + 7) / 8;
    unsigned* k0 = gr.perm_keys.p;
    unsigned* k1 = gr.perm_keys.p + C;
    const long long ntiles = static_cast<long long>(tiles_x) * tiles_y;
    k_spatial_keys<<<blocks_for(C, kBlock), kBlock, 0, s->st>>>(C, s->cell_xy, s->cell_fixed, g, tiles_y,
                                                                static_cast<unsigned>(ntiles), k0, gr.perm_tmp);
    CK_LAUNCH();
    int bits = 1; // keys 0..ntiles (fixed cells sort last)
    while ((1ll << bits) < ntiles + 1) ++bits;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0, k1, gr.perm_tmp.p, gr.perm.p, C, 0, 32, s->st);
    void* tmp = cub_scratch(s, bytes);
    CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, k1, gr.perm_tmp.p, gr.perm.p, C, 0, bits, s->st));
}

void launch_density_scatter_ctrl(tdpg_session* s, const Ctrl* ctrl);

void launch_density(tdpg_session* s, double* part_d, int nblk, const Ctrl* ctrl)
{
    const GridDev g = grid_dev(s);
    if (!ctrl) sort_cells_spatial(s); // one-off evaluations sort first; the loop sorts on its own schedule
    launch_density_scatter_ctrl(s, ctrl);
    launch_density_bins_ctrl(s, part_d, nblk, ctrl);
}

void launch_density(tdpg_session* s, double* part_d, int nblk) { launch_density(s, part_d, nblk, nullptr); }

// The windowed scatter kernel for this grid: no-return limb adds (2 or 3 limbs, Grid::limbs), or with
// TDPG_SCATTER_LIMBS=0 the carry-propagating two-word form (A/B switch; the grids are bitwise equal).
using ScatterKernel = void (*)(int, const int*, const double2*, const double2*, GridDev, unsigned long long*,
                               const Ctrl*, double2*, double2*);
ScatterKernel scatter_kernel(const tdpg_session* s)
{
    static const bool limbs = [] {
        const char* e = std::getenv("TDPG_SCATTER_LIMBS");
        return !(e && std::atoi(e) == 0);
    }();
    if (!limbs) return k_density_scatter_win;
    return s->grid.limbs == 2 ? k_density_scatter_limbs<2> : k_density_scatter_limbs<3>;
}

void launch_density_scatter_ctrl(tdpg_session* s, const Ctrl* ctrl)
{
    const GridDev g = grid_dev(s);
    const int n_mov = s->grid.n_movable;
    if (n_mov == 0) return;
    scatter_kernel(s)<<<blocks_for(n_mov, kBlock), kBlock, 0, s->st>>>(
        n_mov, s->grid.perm, s->cell_xy, s->cell_wh, g, reinterpret_cast<unsigned long long*>(s->grid.acc.p), ctrl,
        s->grid.xy_sp, s->grid.wh_sp);
    CK_LAUNCH();
    if (s->grid.n_wide > 0) {
        k_density_scatter_wide<<<blocks_for(s->grid.n_wide, kBlock), kBlock, 0, s->st>>>(
            s->grid.n_wide, s->grid.wide, s->cell_xy, s->cell_wh, g,
            reinterpret_cast<unsigned long long*>(s->grid.acc.p), ctrl);
        CK_LAUNCH();
    }
}

void launch_density_bins_ctrl(tdpg_session* s, double* part_d, int nblk, const Ctrl* ctrl)
{
    const GridDev g = grid_dev(s);
    const bool el = s->grid.model == 1;
    CK(launch_pdl(k_density_bins, nblk, kBlock, s->st, s->pdl_graph && s->grid.n_movable > 0, s->grid.bins(), g,
                  s->grid.acc.p, static_cast<const double*>(s->grid.has_fixed ? s->grid.base.p : nullptr),
                  s->grid.excess.p, part_d, ctrl, el ? s->grid.electro.rho.p : nullptr));
    if (el) { // potential, then the energy partials replace the overflow-penalty value partials
        electro_solve(s, s->st);
        electro_energy(s, part_d, nblk, ctrl, s->st);
    }
}

CellArgs cell_args(tdpg_session* s, double2* d_cell, double2* m, double2* v, double b1, double b2, double eps)
{
    CellArgs a;
    a.C = s->C;
    a.ent_start = s->cell_ent_start;
    a.ent = s->cell_ent;
    a.grad_e = s->grad_e;
    a.fixed = s->cell_fixed;
    a.xy = s->cell_xy;
    a.wh = s->cell_wh;
    a.dgrad = s->dgrad;
    a.d_cell = d_cell;
    a.folded = nullptr;
    a.dgrad_folded = false;
    a.m = m, a.v = v;
    a.b1 = b1, a.b2 = b2, a.eps = eps;
    a.core_x0 = s->core[0], a.core_y0 = s->core[1], a.core_x1 = s->core[2], a.core_y1 = s->core[3];
    return a;
}

void launch_dens_grad(tdpg_session* s, const Ctrl* ctrl, cudaStream_t st)
{
    const int n_mov = s->grid.n_movable;
    if (n_mov > 0) {
        const bool el = s->grid.model == 1;
        CK(launch_pdl(k_dens_grad, blocks_for(n_mov, kBlock), kBlock, st, s->pdl_graph,
                      n_mov, static_cast<const int*>(s->grid.perm.p), static_cast<const double2*>(s->grid.xy_sp.p),
                      static_cast<const double2*>(s->grid.wh_sp.p), grid_dev(s),
                      static_cast<const double*>(el ? s->grid.electro.psi.p : s->grid.excess.p), s->dgrad.p, ctrl,
                      el ? 1.0 : 2.0));
        if (s->grid.n_wide > 0) {
            k_dens_grad_wide<<<blocks_for(s->grid.n_wide, kBlock), kBlock, 0, st>>>(
                s->grid.n_wide, s->grid.wide, s->cell_xy, s->cell_wh, grid_dev(s),
                el ? s->grid.electro.psi.p : s->grid.excess.p, s->dgrad, ctrl, el ? 1.0 : 2.0);
            CK_LAUNCH();
        }
    }
}

// density gradient (unless the caller already enqueued it) then the cell kernel
void launch_cell_pass(tdpg_session* s, const CellArgs& ca, const IterCur* cur, Ctrl* ctrl, bool dens_grad = true)
{
    if (dens_grad) launch_dens_grad(s, ctrl, s->st);
    CK(launch_pdl(k_cells, blocks_for(s->C, kBlock), kBlock, s->st, s->pdl_graph, ca, cur, ctrl));
}

// One full objective_and_gradient evaluation at the session's positions.
Terms evaluate_objective(tdpg_session* s, double gamma, double lambda, double beta, int kind, bool use_net_w,
                         double* d_cell_host)
{
    if (!s->grid.valid()) throw Error(TDPG_ERR_VALIDATION, "validation error: density grid not set");
    const int nb_wa = wa_blocks(s), nb_pp = pp_blocks(s), nb_d = bins_blocks(s);
    s->part.reserve(2 * nb_wa + nb_pp + 2 * nb_d + 64);
    double* part_wl = s->part.p;
    double* part_hp = part_wl + nb_wa;
    double* part_pp = part_hp + nb_wa;
    double* part_d = part_pp + nb_pp;
    Terms* terms = reinterpret_cast<Terms*>(part_d + 2 * nb_d);
    IterCur* cur = reinterpret_cast<IterCur*>(terms + 1);
    launch_wirelength(s, gamma, use_net_w, part_wl, part_hp, nb_wa);
    const bool pp = s->Q > 0;
    if (pp) {
        rebuild_pp_incidence(s);
        launch_pp(s, kind, beta, part_pp, nb_pp);
    }
    launch_density(s, part_d, nb_d);
    FinArgs fa{};
    fa.part_wl = part_wl, fa.part_hp = part_hp, fa.part_pp = part_pp, fa.part_d = part_d;
    fa.nb_wa = nb_wa, fa.nb_pp = pp ? nb_pp : 0, fa.nb_d = nb_d;
    fa.total_movable = s->grid.total_movable, fa.beta = beta, fa.sched = nullptr, fa.lambda_single = lambda;
    fa.terms = terms;
    k_finalize<<<1, kFinBlock, 0, s->st>>>(fa, nullptr, cur);
    CK_LAUNCH();
    const CellArgs ca = cell_args(s, s->d_cell, nullptr, nullptr, 0, 0, 0);
    launch_cell_pass(s, ca, cur, nullptr);
    Terms t;
    CK(cudaMemcpyAsync(&t, terms, sizeof(Terms), cudaMemcpyDeviceToHost, s->st));
    if (d_cell_host) download_bytes(d_cell_host, s->d_cell.p, sizeof(double2) * static_cast<size_t>(s->C), s->st);
    CK(cudaStreamSynchronize(s->st));
    return t;
}

} // namespace tdpg

using namespace tdpg;

#define API_BEGIN try {
#define API_END                                                                   \
    return TDPG_OK;                                                               \
    }                                                                             \
    catch (const ::tdpg::Error& e) { return ::tdpg::api_fail(e.kind, e.what()); } \
    catch (const std::exception& e) { return ::tdpg::api_fail(TDPG_ERR_INTERNAL, e.what()); }

namespace {

void check_finite_terms(const Terms& t, const double* d_cell, int C)
{
    bool ok = std::isfinite(t.value) && std::isfinite(t.wl) && std::isfinite(t.density) && std::isfinite(t.pp);
    for (int i = 0; ok && d_cell && i < 2 * C; ++i) ok = std::isfinite(d_cell[i]);
    if (!ok) throw Error(TDPG_ERR_NONFINITE, "non-finite value: non-finite objective or gradient");
}

void set_net_w(tdpg_session* s, const double* net_w)
{
    if (!net_w) return;
    s->net_w.upload(net_w, static_cast<size_t>(s->N), s->st);
}

} // namespace

extern "C" {

int tdpg_wirelength(tdpg_session* s, double gamma, const double* net_w, double* wl, double* hpwl, double* pin_grad)
{
    API_BEGIN
    set_net_w(s, net_w);
    const int nb = wa_blocks(s);
    s->part.reserve(2 * nb + 8);
    launch_wirelength(s, gamma, net_w != nullptr, s->part.p, s->part.p + nb, nb);
    std::vector<double> part(2 * nb);
    s->part.download(part.data(), part.size(), s->st);
    std::vector<double2> ge;
    if (pin_grad) {
        ge.resize(s->E_tot);
        s->grad_e.download(ge.data(), ge.size(), s->st);
    }
    CK(cudaStreamSynchronize(s->st));
    double a = 0, b = 0;
    for (int i = 0; i < nb; ++i) a += part[i], b += part[nb + i];
    if (wl) *wl = a;
    if (hpwl) *hpwl = b;
    if (pin_grad) {
        host_pin_maps(s);
        std::fill(pin_grad, pin_grad + 2 * static_cast<size_t>(s->P), 0.0);
        for (int p = 0; p < s->P; ++p) {
            const int e = s->h_pin_entry[p];
            if (e >= 0 && s->h_pin_net[p] >= 0) pin_grad[2 * p] = ge[e].x, pin_grad[2 * p + 1] = ge[e].y;
        }
    }
    API_END
}

// Shared-memory atomics the windowed scatter issues at the session's positions (measurement aid for the
// roofline limiter): per non-zero footprint entry of a five-bin cell one low-limb atomic ([0]) and
// Grid::limbs - 1 upper-limb atomics ([1]), as k_density_scatter_limbs issues them.
__global__ void k_count_scatter_atomics(int n_mov, const int* __restrict__ perm, const double2* __restrict__ cell_xy,
                                        const double2* __restrict__ cell_wh, GridDev g, int limbs,
                                        unsigned long long* __restrict__ out)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    unsigned long long lo = 0, hi = 0;
    if (i < n_mov) {
        const int c = perm[i];
        const double2 p = cell_xy[c], s = cell_wh[c];
        double wx[kF5], wy[kF5], dw[kF5];
        int bx, by;
        if (!(s.x > g.wide_w || s.y > g.wide_h) && axis5(p.x, p.x + s.x, g.x0, g.bw, g.inv_bw, g.nx, bx, wx, dw) &&
            axis5(p.y, p.y + s.y, g.y0, g.bh, g.inv_bh, g.ny, by, wy, dw)) {
            const double area = s.x * s.y;
            for (int a = 0; a < kF5; ++a) {
                if (wx[a] == 0.0) continue;
                const double aw = area * wx[a];
                for (int j = 0; j < kF5; ++j) {
                    const long long q = __double2ll_rn(aw * wy[j] * g.scale);
                    lo += q != 0, hi += q != 0 ? limbs - 1 : 0;
                }
            }
        }
    }
    lo = warp_sum(lo), hi = warp_sum(hi);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, lo), atomicAdd(out + 1, hi);
}

int tdpg_density_atomics(tdpg_session* s, int64_t* lo_hi)
{
    API_BEGIN
    if (!s->grid.valid()) throw Error(TDPG_ERR_VALIDATION, "validation error: density grid not set");
    sort_cells_spatial(s);
    DBuf<unsigned long long> out(2);
    out.zero(s->st);
    const int n_mov = s->grid.n_movable;
    if (n_mov > 0)
        k_count_scatter_atomics<<<blocks_for(n_mov, kBlock), kBlock, 0, s->st>>>(n_mov, s->grid.perm, s->cell_xy,
                                                                                s->cell_wh, grid_dev(s), s->grid.limbs, out);
    CK_LAUNCH();
    unsigned long long h[2];
    out.download(h, 2, s->st);
    CK(cudaStreamSynchronize(s->st));
    lo_hi[0] = static_cast<int64_t>(h[0]), lo_hi[1] = static_cast<int64_t>(h[1]);
    API_END
}

int tdpg_density(tdpg_session* s, double* value, double* overflow, double* d_cell)
{
    API_BEGIN
    if (!s->grid.valid()) throw Error(TDPG_ERR_VALIDATION, "validation error: density grid not set");
    // Density alone = objective with the WA/PP contributions removed: run the density
    // kernels and the cell kernel with zero entry gradients and lambda = 1.
    const int nb_d = bins_blocks(s);
    s->part.reserve(2 * nb_d + 64);
    double* part_d = s->part.p;
    Terms* terms = reinterpret_cast<Terms*>(part_d + 2 * nb_d);
    IterCur* cur = reinterpret_cast<IterCur*>(terms + 1);
    launch_density(s, part_d, nb_d);
    FinArgs fa{};
    fa.part_d = part_d, fa.nb_d = nb_d, fa.total_movable = s->grid.total_movable, fa.lambda_single = 1.0;
    fa.terms = terms;
    k_finalize<<<1, kFinBlock, 0, s->st>>>(fa, nullptr, cur);
    CK_LAUNCH();
    if (d_cell) {
        s->grad_e.zero(s->st, s->E_tot);
        const CellArgs ca = cell_args(s, s->d_cell, nullptr, nullptr, 0, 0, 0);
        launch_cell_pass(s, ca, cur, nullptr);
        s->d_cell.download(reinterpret_cast<double2*>(d_cell), s->C, s->st);
    }
    Terms t;
    CK(cudaMemcpyAsync(&t, terms, sizeof(Terms), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    *value = t.density;
    *overflow = t.overflow;
    API_END
}

int tdpg_pp_loss(tdpg_session* s, int32_t kind, double* value, double* d_pin)
{
    API_BEGIN
    const int nb = pp_blocks(s);
    s->part.reserve(nb + 8);
    double v = 0.0;
    if (d_pin) std::fill(d_pin, d_pin + 2 * static_cast<size_t>(s->P), 0.0);
    if (s->Q > 0) {
        rebuild_pp_incidence(s);
        s->grad_e.zero(s->st, s->E_tot);
        launch_pp(s, kind, 1.0, s->part.p, nb);
        std::vector<double> part(nb);
        s->part.download(part.data(), nb, s->st);
        std::vector<double2> ge;
        if (d_pin) {
            ge.resize(s->E_tot);
            s->grad_e.download(ge.data(), ge.size(), s->st);
        }
        CK(cudaStreamSynchronize(s->st));
        for (double x : part) v += x;
        if (d_pin) host_pin_maps(s);
        if (d_pin)
            for (int p = 0; p < s->P; ++p) {
                const int e = s->h_pin_entry[p];
                if (e >= 0) d_pin[2 * p] = ge[e].x, d_pin[2 * p + 1] = ge[e].y;
            }
    }
    *value = v;
    API_END
}

int tdpg_objective(tdpg_session* s, double gamma, double lambda, double beta, int32_t pp_kind, const double* net_w,
                   double terms[6], double* d_cell)
{
    API_BEGIN
    if (net_w) set_net_w(s, net_w);
    std::vector<double> tmp;
    double* g = d_cell;
    if (!g) {
        tmp.resize(2 * static_cast<size_t>(s->C));
        g = tmp.data();
    }
    const Terms t = evaluate_objective(s, gamma, lambda, beta, pp_kind, net_w != nullptr, g);
    terms[0] = t.value, terms[1] = t.wl, terms[2] = t.density, terms[3] = t.pp, terms[4] = t.hpwl,
    terms[5] = t.overflow;
    check_finite_terms(t, g, s->C);
    API_END
}

int tdpg_hpwl_pins(tdpg_session* s, const double* pin_xy, double* hpwl)
{
    API_BEGIN
    DBuf<double2> pxy(std::max(s->P, 1));
    pxy.upload(reinterpret_cast<const double2*>(pin_xy), s->P, s->st);
    const int nb = std::max(1, static_cast<int>(blocks_for(s->N, kBlock)));
    DBuf<double> part(nb);
    k_hpwl_pins<<<nb, kBlock, 0, s->st>>>(s->N, s->net_start, s->net_pins, pxy, part);
    CK_LAUNCH();
    std::vector<double> h(nb);
    part.download(h.data(), nb, s->st);
    CK(cudaStreamSynchronize(s->st));
    double t = 0.0;
    for (double x : h) t += x;
    *hpwl = t;
    API_END
}

int tdpg_set_core(tdpg_session* s, const double core[4])
{
    API_BEGIN
    if (std::memcmp(s->core, core, sizeof s->core) != 0) {
        std::memcpy(s->core, core, sizeof s->core);
        s->grid.nx = 0; // the grid geometry follows the core; rebuilt by the next tdpg_set_grid
    }
    API_END
}

int tdpg_set_constraints(tdpg_session* s, double clock_period, double r_unit, double c_unit)
{
    API_BEGIN
    if (s->clock != clock_period || s->r_unit != r_unit || s->c_unit != c_unit) s->sta_valid = false;
    s->clock = clock_period, s->r_unit = r_unit, s->c_unit = c_unit;
    API_END
}

int tdpg_adam_step(int64_t n, double* x, const double* g, double* m, double* v, int32_t* t, double lr, double b1,
                   double b2, double eps)
{
    API_BEGIN
    if (tdpg_device_count() == 0) throw Error(TDPG_ERR_CUDA, "cuda error: no CUDA device available");
    ++*t;
    const double c1 = 1.0 - std::pow(b1, *t); // host-side scalars, bitwise std::pow like the reference
    const double c2 = 1.0 - std::pow(b2, *t);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    DBuf<double> dx(n), dg(n), dm(n), dv(n);
    dx.upload(x, n, st), dg.upload(g, n, st), dm.upload(m, n, st), dv.upload(v, n, st);
    k_adam_flat<<<blocks_for(n, kBlock), kBlock, 0, st>>>(n, dx, dg, dm, dv, lr, b1, b2, eps, c1, c2);
    CK_LAUNCH();
    dx.download(x, n, st), dm.download(m, n, st), dv.download(v, n, st);
    CK(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    API_END
}

} // extern "C"

// Placement-loop internals used by place.cu
namespace tdpg {
void launch_wirelength_ctrl(tdpg_session* s, double gamma, bool use_net_w, double* pw, double* ph, int nb,
                            const Ctrl* ctrl)
{
    launch_wirelength(s, gamma, use_net_w, pw, ph, nb, ctrl);
}
void launch_pp_ctrl(tdpg_session* s, int kind, double beta, double* pp, int nb, const Ctrl* ctrl)
{
    launch_pp(s, kind, beta, pp, nb, ctrl);
}
void launch_density_ctrl(tdpg_session* s, double* pd, int nb, const Ctrl* ctrl) { launch_density(s, pd, nb, ctrl); }
void launch_finalize(tdpg_session* s, const FinArgs& fa, Ctrl* ctrl, IterCur* cur)
{
    k_finalize<<<1, kFinBlock, 0, s->st>>>(fa, ctrl, cur);
    CK_LAUNCH();
}
void launch_fin_density(tdpg_session* s, const FinArgs& fa, Ctrl* ctrl, IterCur* cur, cudaStream_t st)
{
    (void)s;
    k_fin_density<<<1, kFinBlock, 0, st>>>(fa, ctrl, cur);
    CK_LAUNCH();
}
void launch_fin_terms(tdpg_session* s, const FinArgs& fa, Ctrl* ctrl, const IterCur* cur, cudaStream_t st)
{
    (void)s;
    k_fin_terms<<<1, kFinBlock, 0, st>>>(fa, ctrl, cur);
    CK_LAUNCH();
}
void launch_cells(tdpg_session* s, double2* d_cell, double2* m, double2* v, double b1, double b2, double eps,
                  const IterCur* cur, Ctrl* ctrl, bool dens_grad, const double2* folded, bool dgrad_folded)
{
    CellArgs ca = cell_args(s, d_cell, m, v, b1, b2, eps);
    ca.folded = folded;
    ca.dgrad_folded = dgrad_folded;
    launch_cell_pass(s, ca, cur, ctrl, dens_grad);
}

// Partitioned engine with the density sharded: this rank scatters the movable cells of its
// slice [lo, hi) of the spatial order (rank 0 also the wide cells); the int64 grid is summed across ranks
// (exact, order independent); bins are replicated; the density gradient is computed for the slice (the
// few wide cells on every rank) and lambda * gradient goes into this rank's share of the all-reduced fold.
void launch_density_scatter_part(tdpg_session* s, const Ctrl* ctrl, int lo, int hi, bool wide)
{
    const GridDev g = grid_dev(s);
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(s->grid.acc.p);
    if (hi > lo) {
        scatter_kernel(s)<<<blocks_for(hi - lo, kBlock), kBlock, 0, s->st>>>(
            hi - lo, s->grid.perm.p + lo, s->cell_xy, s->cell_wh, g, acc, ctrl, s->grid.xy_sp.p + lo,
            s->grid.wh_sp.p + lo);
        CK_LAUNCH();
    }
    if (wide && s->grid.n_wide > 0) {
        k_density_scatter_wide<<<blocks_for(s->grid.n_wide, kBlock), kBlock, 0, s->st>>>(
            s->grid.n_wide, s->grid.wide, s->cell_xy, s->cell_wh, g, acc, ctrl);
        CK_LAUNCH();
    }
}

void launch_dens_grad_part(tdpg_session* s, const Ctrl* ctrl, cudaStream_t st, int lo, int hi)
{
    const bool el = s->grid.model == 1;
    const double* field = el ? s->grid.electro.psi.p : s->grid.excess.p;
    if (hi > lo) {
        k_dens_grad<<<blocks_for(hi - lo, kBlock), kBlock, 0, st>>>(hi - lo, s->grid.perm.p + lo,
                                                                    s->grid.xy_sp.p + lo, s->grid.wh_sp.p + lo,
                                                                    grid_dev(s), field, s->dgrad, ctrl, el ? 1.0 : 2.0);
        CK_LAUNCH();
    }
    if (s->grid.n_wide > 0) {
        k_dens_grad_wide<<<blocks_for(s->grid.n_wide, kBlock), kBlock, 0, st>>>(
            s->grid.n_wide, s->grid.wide, s->cell_xy, s->cell_wh, grid_dev(s), field, s->dgrad, ctrl, el ? 1.0 : 2.0);
        CK_LAUNCH();
    }
}

__global__ void k_add_dgrad(int n, const int* __restrict__ perm, const uint8_t* __restrict__ fixed,
                            const double2* __restrict__ dgrad, const Sched* __restrict__ sched,
                            const Ctrl* __restrict__ ctrl, double2* __restrict__ fold)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n || ctrl->stopped) return;
    const int c = perm[i];
    if (fixed[c]) return;
    const double lambda = sched[ctrl->iter].lambda; // (what k_finalize publishes for this iteration)
    const double2 g = dgrad[c], f = fold[c];
    fold[c] = make_double2(f.x + lambda * g.x, f.y + lambda * g.y);
}

void launch_add_dgrad(tdpg_session* s, const Sched* sched, const Ctrl* ctrl, double2* fold, int lo, int hi)
{
    if (hi <= lo) return;
    k_add_dgrad<<<blocks_for(hi - lo, kBlock), kBlock, 0, s->st>>>(hi - lo, s->grid.perm.p + lo, s->cell_fixed,
                                                                   s->dgrad, sched, ctrl, fold);
    CK_LAUNCH();
}

void launch_fold(tdpg_session* s, double2* out, const Ctrl* ctrl)
{
    k_fold<<<blocks_for(s->C, kBlock), kBlock, 0, s->st>>>(s->C, s->cell_ent_start, s->cell_ent, s->grad_e, out, ctrl);
    CK_LAUNCH();
}
} // namespace tdpg
