// graph.cu — build_timing_graph (timing_graph.cpp:49-138) on the device, at session creation.
//
// Every step is integer work with a stable order, so the result is bitwise the reference's graph:
//  * arcs: net arcs in (net, sink) order (arc id e - n - 1 for entry e of net n), then cell arcs per cell
//    in (cell, input pin, output pin) order, both pin lists ascending (timing_graph.cpp:60-77) — counts
//    per cell, an exclusive scan, one thread per cell writing its block;
//  * in / out CSR: arc ids stably radix-sorted by to / from pin (ascending arc id within a pin);
//  * levels (Kahn, level = longest path from an in-degree-0 pin, :87-104): synchronous frontier rounds —
//    a pin leaves the graph in round r exactly when its longest incoming path has r arcs — with an
//    atomic in-degree countdown; a short round count means a cycle (:12-45, message built from the
//    remaining pins);
//  * reachability from the sources (:112-135): pulled level by level (every predecessor has a lower
//    level), then the first unreachable endpoint in the netlist's endpoint order is reported;
//  * the level-major copies the STA runs on (L-space, sta_in / sta_out pins): one stable sort by
//    (level, is-output) — per level its Input pins then its Output pins, ascending id.
// Host copies (level of every pin, the arc lists) are downloaded only when the API asks for them.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>
#include <vector>

#include "gp_kernels.cuh"

namespace tdpg {

namespace {

constexpr int kGB = 256;

int bits_for_n(long long n)
{
    int b = 1;
    while ((1ll << b) <= n) ++b;
    return b;
}

struct Tmp { // scratch for one CUB call at a time
    explicit Tmp(cudaStream_t st) : buf(st) {}
    TBuf<unsigned char> buf;
    void* get(size_t bytes)
    {
        buf.reserve(std::max<size_t>(bytes, 1));
        return buf.p;
    }
};

void sort_pairs(Tmp& t, const int* kin, int* kout, const int* vin, int* vout, int n, int bits, cudaStream_t st)
{
    if (n <= 0) return;
    size_t b = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, b, kin, kout, vin, vout, n, 0, bits, st));
    CK(cub::DeviceRadixSort::SortPairs(t.get(b), b, kin, kout, vin, vout, n, 0, bits, st));
}

void excl_sum(Tmp& t, const int* in, int* out, int n, cudaStream_t st)
{
    if (n <= 0) return;
    size_t b = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, n, st));
    CK(cub::DeviceScan::ExclusiveSum(t.get(b), b, in, out, n, st));
}

__global__ void k_iota(int n, int* __restrict__ v)
{
    for (int i = blockIdx.x * kGB + threadIdx.x; i < n; i += gridDim.x * kGB) v[i] = i;
}

// cell of every pin as a sort key (terminals last), and per cell the counts of its arc-eligible pins
__global__ void k_cell_keys(int P, int C, const int* __restrict__ pin_cell, int* __restrict__ key,
                            const uint8_t* __restrict__ dir, const uint8_t* __restrict__ is_src,
                            const uint8_t* __restrict__ is_ep, int* __restrict__ n_in, int* __restrict__ n_out,
                            int* __restrict__ cp_cnt)
{
    for (int p = blockIdx.x * kGB + threadIdx.x; p < P; p += gridDim.x * kGB) {
        const int c = pin_cell[p];
        key[p] = c >= 0 ? c : C;
        if (c < 0) continue;
        atomicAdd(&cp_cnt[c], 1);
        if (dir[p] == 0 && !is_ep[p]) atomicAdd(&n_in[c], 1);
        if (dir[p] == 1 && !is_src[p]) atomicAdd(&n_out[c], 1);
    }
}

__global__ void k_cell_arc_count(int C, const int* __restrict__ n_in, const int* __restrict__ n_out,
                                 int* __restrict__ cnt)
{
    for (int c = blockIdx.x * kGB + threadIdx.x; c < C; c += gridDim.x * kGB) cnt[c] = n_in[c] * n_out[c];
}

// net arcs: entry e of net n (not its driver) is arc e - n - 1
__global__ void k_net_arcs(int N, const int* __restrict__ net_start, const int* __restrict__ net_pins,
                           int* __restrict__ af, int* __restrict__ at, int* __restrict__ ak, int* __restrict__ ao)
{
    for (int n = blockIdx.x * kGB + threadIdx.x; n < N; n += gridDim.x * kGB) {
        const int b = net_start[n], e1 = net_start[n + 1];
        const int drv = net_pins[b];
        for (int e = b + 1; e < e1; ++e) {
            const int a = e - n - 1;
            af[a] = drv, at[a] = net_pins[e], ak[a] = 0, ao[a] = n;
        }
    }
}

// cell arcs: per cell, eligible inputs x eligible outputs in ascending pin order (timing_graph.cpp:67-77)
__global__ void k_cell_arcs(int C, int A_net, const int* __restrict__ cp_start, const int* __restrict__ cp,
                            const int* __restrict__ off, const uint8_t* __restrict__ dir,
                            const uint8_t* __restrict__ is_src, const uint8_t* __restrict__ is_ep,
                            int* __restrict__ af, int* __restrict__ at, int* __restrict__ ak, int* __restrict__ ao)
{
    for (int c = blockIdx.x * kGB + threadIdx.x; c < C; c += gridDim.x * kGB) {
        int a = A_net + off[c];
        const int lo = cp_start[c], hi = cp_start[c + 1];
        for (int i = lo; i < hi; ++i) {
            const int in = cp[i];
            if (dir[in] != 0 || is_ep[in]) continue;
            for (int j = lo; j < hi; ++j) {
                const int out = cp[j];
                if (dir[out] != 1 || is_src[out]) continue;
                af[a] = in, at[a] = out, ak[a] = 1, ao[a] = c;
                ++a;
            }
        }
    }
}

// histogram of a key array into counts[0..nbins)
__global__ void k_hist(int n, const int* __restrict__ key, int* __restrict__ cnt)
{
    for (int i = blockIdx.x * kGB + threadIdx.x; i < n; i += gridDim.x * kGB) atomicAdd(&cnt[key[i]], 1);
}

__global__ void k_gather_i(int n, const int* __restrict__ idx, const int* __restrict__ src, int* __restrict__ dst)
{
    for (int i = blockIdx.x * kGB + threadIdx.x; i < n; i += gridDim.x * kGB) dst[i] = src[idx[i]];
}

__global__ void k_indeg(int P, const int* __restrict__ in_start, int* __restrict__ indeg, int* __restrict__ level,
                        int* __restrict__ front, int* __restrict__ n_front)
{
    for (int p = blockIdx.x * kGB + threadIdx.x; p < P; p += gridDim.x * kGB) {
        indeg[p] = in_start[p + 1] - in_start[p];
        level[p] = 0;
        if (indeg[p] == 0) front[atomicAdd(n_front, 1)] = p;
    }
}

__global__ void k_kahn_round(int n, int r, const int* __restrict__ front, const int* __restrict__ out_start,
                             const int* __restrict__ out_to, int* __restrict__ indeg, int* __restrict__ level,
                             int* __restrict__ next, int* __restrict__ n_next)
{
    for (int i = blockIdx.x * kGB + threadIdx.x; i < n; i += gridDim.x * kGB) {
        const int u = front[i];
        for (int k = out_start[u]; k < out_start[u + 1]; ++k) {
            const int v = out_to[k];
            if (atomicSub(&indeg[v], 1) == 1) {
                level[v] = r + 1;
                next[atomicAdd(n_next, 1)] = v;
            }
        }
    }
}

__global__ void k_reach_level(int lo, int hi, const int* __restrict__ lvl_pins, const int* __restrict__ in_start,
                              const int* __restrict__ in_from, const uint8_t* __restrict__ is_src,
                              uint8_t* __restrict__ reach)
{
    for (int i = lo + blockIdx.x * kGB + threadIdx.x; i < hi; i += gridDim.x * kGB) {
        const int v = lvl_pins[i];
        uint8_t r = is_src[v];
        for (int k = in_start[v]; k < in_start[v + 1] && !r; ++k) r = reach[in_from[k]];
        reach[v] = r;
    }
}

__global__ void k_first_unreached(int n, const int* __restrict__ eps, const uint8_t* __restrict__ reach,
                                  int* __restrict__ first)
{
    for (int i = blockIdx.x * kGB + threadIdx.x; i < n; i += gridDim.x * kGB)
        if (!reach[eps[i]]) atomicMin(first, i);
}

// L-space key: 2 * level + (pin is an Output)
__global__ void k_lkeys(int P, const int* __restrict__ level, const uint8_t* __restrict__ dir, int* __restrict__ key)
{
    for (int p = blockIdx.x * kGB + threadIdx.x; p < P; p += gridDim.x * kGB) key[p] = 2 * level[p] + (dir[p] == 1);
}

__global__ void k_lspace_nodes(int P, const int* __restrict__ Lpin, int* __restrict__ Lidx,
                               const int* __restrict__ in_start, const int* __restrict__ out_start,
                               int* __restrict__ in_cnt, int* __restrict__ out_cnt, const uint8_t* __restrict__ is_src,
                               const uint8_t* __restrict__ is_ep, const uint8_t* __restrict__ dir,
                               const double* __restrict__ cap, const int* __restrict__ pin_cell,
                               const double2* __restrict__ off, const double2* __restrict__ term,
                               uint8_t* __restrict__ Lfl, double* __restrict__ Lcap, int* __restrict__ Lcell,
                               double2* __restrict__ Loff, double2* __restrict__ Lanc)
{
    for (int i = blockIdx.x * kGB + threadIdx.x; i < P; i += gridDim.x * kGB) {
        const int p = Lpin[i];
        Lidx[p] = i;
        in_cnt[i] = in_start[p + 1] - in_start[p];
        out_cnt[i] = out_start[p + 1] - out_start[p];
        Lfl[i] = static_cast<uint8_t>((is_src[p] ? 1 : 0) | (is_ep[p] ? 2 : 0) | (dir[p] == 1 ? 4 : 0));
        Lcap[i] = cap[p], Lcell[i] = pin_cell[p], Loff[i] = off[p], Lanc[i] = term[p];
    }
}

__global__ void k_lspace_edges(int P, const int* __restrict__ Lpin, const int* __restrict__ Lidx,
                               const int* __restrict__ in_start, const int* __restrict__ in_from,
                               const int* __restrict__ out_start, const int* __restrict__ out_to,
                               const int* __restrict__ Lis, const int* __restrict__ Los, int* __restrict__ Lif,
                               int* __restrict__ Lot)
{
    for (int i = blockIdx.x * kGB + threadIdx.x; i < P; i += gridDim.x * kGB) {
        const int p = Lpin[i];
        int d = Lis[i];
        for (int k = in_start[p]; k < in_start[p + 1]; ++k) Lif[d++] = Lidx[in_from[k]];
        d = Los[i];
        for (int k = out_start[p]; k < out_start[p + 1]; ++k) Lot[d++] = Lidx[out_to[k]];
    }
}

// the Input / Output pins of Lpin, each in level order
__global__ void k_split_io(int P, const int* __restrict__ Lpin, const int* __restrict__ lkey_sorted,
                           const int* __restrict__ seg_start, const int* __restrict__ in_base,
                           const int* __restrict__ out_base, int* __restrict__ ins, int* __restrict__ outs)
{
    for (int i = blockIdx.x * kGB + threadIdx.x; i < P; i += gridDim.x * kGB) {
        const int k = lkey_sorted[i], l = k >> 1;
        const int r = i - seg_start[k];
        if (k & 1) outs[out_base[l] + r] = Lpin[i];
        else ins[in_base[l] + r] = Lpin[i];
    }
}

unsigned grid_for(long long n) { return static_cast<unsigned>(std::min<long long>(std::max<long long>((n + kGB - 1) / kGB, 1), 148 * 16)); }

} // namespace

void build_graph_device(tdpg_session* s)
{
    cudaStream_t st = s->st;
    const int P = s->P, C = s->C, N = s->N;
    Tmp tmp(st);
    // ---- cell pins, ascending pin id per cell (netlist.cpp:12-14)
    TBuf<int> key(st), key_s(st), iota(st), cp(st), cp_cnt(st), cp_start(st), n_in(st), n_out(st);
    key.alloc(std::max(P, 1)), key_s.alloc(std::max(P, 1)), iota.alloc(std::max(P, 1)), cp.alloc(std::max(P, 1));
    cp_cnt.alloc(C + 1), cp_start.alloc(C + 1), n_in.alloc(std::max(C, 1)), n_out.alloc(std::max(C, 1));
    cp_cnt.zero(st), n_in.zero(st), n_out.zero(st);
    if (P) {
        k_iota<<<grid_for(P), kGB, 0, st>>>(P, iota);
        k_cell_keys<<<grid_for(P), kGB, 0, st>>>(P, C, s->pin_cell, key, s->pin_dir, s->is_source, s->is_endpoint,
                                                  n_in, n_out, cp_cnt);
        CK_LAUNCH();
        sort_pairs(tmp, key, key_s, iota, cp, P, bits_for_n(C + 1), st);
    }
    excl_sum(tmp, cp_cnt, cp_start, C + 1, st);
    // ---- arcs
    const int A_net = s->E - N;
    TBuf<int> ccnt(st), coff(st);
    ccnt.alloc(C + 1), coff.alloc(C + 1);
    ccnt.zero(st);
    if (C) k_cell_arc_count<<<grid_for(C), kGB, 0, st>>>(C, n_in, n_out, ccnt);
    excl_sum(tmp, ccnt, coff, C + 1, st);
    int A_cell = 0;
    CK(cudaMemcpyAsync(&A_cell, coff.p + C, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int A = A_net + A_cell;
    s->A_net = A_net, s->A_cell = A_cell, s->A = A;
    s->arc_from.alloc(std::max(A, 1)), s->arc_to.alloc(std::max(A, 1)), s->arc_kind.alloc(std::max(A, 1));
    s->arc_owner.alloc(std::max(A, 1));
    if (N) k_net_arcs<<<grid_for(N), kGB, 0, st>>>(N, s->net_start, s->net_pins, s->arc_from, s->arc_to,
                                                    s->arc_kind, s->arc_owner);
    if (C) k_cell_arcs<<<grid_for(C), kGB, 0, st>>>(C, A_net, cp_start, cp, coff, s->pin_dir, s->is_source,
                                                     s->is_endpoint, s->arc_from, s->arc_to, s->arc_kind,
                                                     s->arc_owner);
    CK_LAUNCH();
    // ---- in / out CSR: arc ids stably sorted by to / from
    TBuf<int> aiota(st), akey_s(st), in_a(st), out_a(st), cnt(st);
    aiota.alloc(std::max(A, 1)), akey_s.alloc(std::max(A, 1)), in_a.alloc(std::max(A, 1)), out_a.alloc(std::max(A, 1));
    cnt.alloc(2 * static_cast<size_t>(P) + 4); // (histograms over pins, levels and 2 * levels + 1)
    s->in_start.alloc(P + 1), s->out_start.alloc(P + 1), s->in_from.alloc(std::max(A, 1)), s->out_to.alloc(std::max(A, 1));
    const int pbits = bits_for_n(P);
    if (A) {
        k_iota<<<grid_for(A), kGB, 0, st>>>(A, aiota);
        sort_pairs(tmp, s->arc_to, akey_s, aiota, in_a, A, pbits, st);
        sort_pairs(tmp, s->arc_from, akey_s, aiota, out_a, A, pbits, st);
    }
    cnt.zero(st);
    if (A) k_hist<<<grid_for(A), kGB, 0, st>>>(A, s->arc_to, cnt);
    excl_sum(tmp, cnt, s->in_start, P + 1, st);
    cnt.zero(st);
    if (A) k_hist<<<grid_for(A), kGB, 0, st>>>(A, s->arc_from, cnt);
    excl_sum(tmp, cnt, s->out_start, P + 1, st);
    if (A) {
        k_gather_i<<<grid_for(A), kGB, 0, st>>>(A, in_a, s->arc_from, s->in_from);
        k_gather_i<<<grid_for(A), kGB, 0, st>>>(A, out_a, s->arc_to, s->out_to);
    }
    CK_LAUNCH();
    // ---- Kahn levels by synchronous frontier rounds
    TBuf<int> indeg(st), fa(st), fb(st), nf(st);
    indeg.alloc(std::max(P, 1)), fa.alloc(std::max(P, 1)), fb.alloc(std::max(P, 1)), nf.alloc(2);
    s->d_level.alloc(std::max(P, 1));
    HBuf<int>& hn = s->h_graph_small;
    hn.reserve(8);
    nf.zero(st);
    int done = 0, n_cur = 0, rounds = 0;
    if (P) {
        k_indeg<<<grid_for(P), kGB, 0, st>>>(P, s->in_start, indeg, s->d_level, fa, nf);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(hn.p, nf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        n_cur = hn[0];
    }
    int* cur = fa.p;
    int* nxt = fb.p;
    while (n_cur > 0) {
        done += n_cur;
        CK(cudaMemsetAsync(nf.p, 0, sizeof(int), st));
        k_kahn_round<<<grid_for(n_cur), kGB, 0, st>>>(n_cur, rounds, cur, s->out_start, s->out_to, indeg,
                                                       s->d_level, nxt, nf);
        CK_LAUNCH();
        CK(cudaMemcpyAsync(hn.p, nf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        n_cur = hn[0];
        std::swap(cur, nxt);
        ++rounds;
    }
    if (done != P) { // report_cycle (timing_graph.cpp:12-45): walk back through remaining pins
        std::vector<int> h_indeg(P), h_in_start(P + 1), h_in_from(std::max(A, 1));
        CK(cudaMemcpyAsync(h_indeg.data(), indeg.p, sizeof(int) * P, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(h_in_start.data(), s->in_start.p, sizeof(int) * (P + 1), cudaMemcpyDeviceToHost, st));
        if (A) CK(cudaMemcpyAsync(h_in_from.data(), s->in_from.p, sizeof(int) * A, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        auto name = [&](int p) {
            return s->pin_names.empty() ? (s->pin_names_blank ? std::string() : "p" + std::to_string(p)) : s->pin_names[p];
        };
        int start = -1;
        for (int p = 0; p < P; ++p)
            if (h_indeg[p] > 0) start = p;
        std::vector<int> seen(P, -1), walk;
        int c = start;
        while (seen[c] < 0) {
            seen[c] = static_cast<int>(walk.size());
            walk.push_back(c);
            for (int i = h_in_start[c]; i < h_in_start[c + 1]; ++i) {
                const int u = h_in_from[i];
                if (h_indeg[u] > 0) {
                    c = u;
                    break;
                }
            }
        }
        std::string msg;
        for (size_t i = static_cast<size_t>(seen[c]); i < walk.size(); ++i) {
            if (!msg.empty()) msg += " <- ";
            msg += name(walk[i]);
        }
        throw Error(TDPG_ERR_CYCLE, "validation error: combinational cycle: " + msg);
    }
    const int L = std::max(rounds, 1);
    s->L = L;
    // ---- pins by level (ascending id inside a level)
    s->lvl_pins.alloc(std::max(P, 1)), s->lvl_start.alloc(L + 1);
    if (P) sort_pairs(tmp, s->d_level, key_s, iota, s->lvl_pins, P, bits_for_n(L), st);
    cnt.zero(st);
    if (P) k_hist<<<grid_for(P), kGB, 0, st>>>(P, s->d_level, cnt);
    excl_sum(tmp, cnt, s->lvl_start, L + 1, st);
    s->h_lvl_start.resize(L + 1);
    CK(cudaMemcpyAsync(s->h_lvl_start.data(), s->lvl_start.p, sizeof(int) * (L + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!P) s->h_lvl_start.assign(L + 1, 0);
    // ---- endpoint reachability (timing_graph.cpp:112-135)
    {
        TBuf<uint8_t> reach(st);
        reach.alloc(std::max(P, 1));
        reach.zero(st);
        for (int l = 0; l < L; ++l) {
            const int lo = s->h_lvl_start[l], hi = s->h_lvl_start[l + 1];
            if (hi > lo)
                k_reach_level<<<grid_for(hi - lo), kGB, 0, st>>>(lo, hi, s->lvl_pins, s->in_start, s->in_from,
                                                                  s->is_source, reach);
        }
        CK_LAUNCH();
        TBuf<int> eps(st), first(st);
        eps.upload(s->h_endpoints, st);
        first.alloc(1);
        const int big = INT_MAX;
        CK(cudaMemcpyAsync(first.p, &big, sizeof(int), cudaMemcpyHostToDevice, st));
        if (s->EP) k_first_unreached<<<grid_for(s->EP), kGB, 0, st>>>(s->EP, eps, reach, first);
        CK_LAUNCH();
        int f = INT_MAX;
        CK(cudaMemcpyAsync(&f, first.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (f != INT_MAX) {
            const int e = s->h_endpoints[f];
            const std::string nm =
                s->pin_names.empty() ? (s->pin_names_blank ? std::string() : "p" + std::to_string(e)) : s->pin_names[e];
            throw Error(TDPG_ERR_VALIDATION, "validation error: endpoint \"" + nm + "\" unreachable from every source");
        }
    }
    // ---- level-major L-space: per level its Input pins then its Output pins, ascending id
    TBuf<int> Lpin(st), lkey_s(st), seg(st);
    Lpin.alloc(std::max(P, 1)), lkey_s.alloc(std::max(P, 1)), seg.alloc(2 * L + 1);
    if (P) {
        k_lkeys<<<grid_for(P), kGB, 0, st>>>(P, s->d_level, s->pin_dir, key);
        sort_pairs(tmp, key, lkey_s, iota, Lpin, P, bits_for_n(2 * L), st);
    }
    cnt.zero(st);
    if (P) k_hist<<<grid_for(P), kGB, 0, st>>>(P, key, cnt);
    excl_sum(tmp, cnt, seg, 2 * L + 1, st);
    std::vector<int> hseg(2 * L + 1);
    CK(cudaMemcpyAsync(hseg.data(), seg.p, sizeof(int) * (2 * L + 1), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!P) std::fill(hseg.begin(), hseg.end(), 0);
    s->h_L_in_lo.assign(L, 0), s->h_L_in_hi.assign(L, 0);
    s->h_sta_out_start.assign(L + 1, 0), s->h_sta_in_start.assign(L + 1, 0);
    for (int l = 0; l < L; ++l) {
        s->h_L_in_lo[l] = hseg[2 * l], s->h_L_in_hi[l] = hseg[2 * l + 1];
        s->h_sta_in_start[l + 1] = s->h_sta_in_start[l] + (hseg[2 * l + 1] - hseg[2 * l]);
        s->h_sta_out_start[l + 1] = s->h_sta_out_start[l] + (hseg[2 * l + 2] - hseg[2 * l + 1]);
    }
    {   // push-sweep tables: Input pins / Output pins, each grouped by level
        const int n_in = s->h_sta_in_start[L], n_out = s->h_sta_out_start[L];
        s->sta_in_pins.alloc(std::max(n_in, 1)), s->sta_out_pins.alloc(std::max(n_out, 1));
        s->sta_in_pins.zero(st), s->sta_out_pins.zero(st);
        TBuf<int> ib(st), ob(st);
        ib.upload(s->h_sta_in_start, st), ob.upload(s->h_sta_out_start, st);
        if (P) k_split_io<<<grid_for(P), kGB, 0, st>>>(P, Lpin, lkey_s, seg, ib, ob, s->sta_in_pins, s->sta_out_pins);
        CK_LAUNCH();
        s->sta_akey.alloc(std::max(P, 1)), s->sta_rkey.alloc(std::max(P, 1));
        CK(cudaStreamSynchronize(st)); // (ib / ob are freed on return)
    }
    {
        const size_t n = static_cast<size_t>(std::max(P, 1));
        s->L_of.alloc(n), s->L_pin.alloc(n), s->L_cell.alloc(n), s->L_flags.alloc(n), s->L_cap.alloc(n);
        s->L_off.alloc(n), s->L_anchor.alloc(n);
        s->L_in_start.alloc(P + 1), s->L_out_start.alloc(P + 1);
        s->L_in_from.alloc(std::max(A, 1)), s->L_out_to.alloc(std::max(A, 1));
        TBuf<int> icnt(st), ocnt(st);
        icnt.alloc(P + 1), ocnt.alloc(P + 1);
        icnt.zero(st), ocnt.zero(st);
        if (P) {
            CK(cudaMemcpyAsync(s->L_pin.p, Lpin.p, sizeof(int) * P, cudaMemcpyDeviceToDevice, st));
            k_lspace_nodes<<<grid_for(P), kGB, 0, st>>>(P, Lpin, s->L_of, s->in_start, s->out_start, icnt, ocnt,
                                                         s->is_source, s->is_endpoint, s->pin_dir, s->pin_cap,
                                                         s->pin_cell, s->pin_off, s->anchor, s->L_flags, s->L_cap,
                                                         s->L_cell, s->L_off, s->L_anchor);
            CK_LAUNCH();
        } else {
            s->L_of.zero(st), s->L_pin.zero(st), s->L_cell.zero(st), s->L_flags.zero(st), s->L_cap.zero(st);
            s->L_off.zero(st), s->L_anchor.zero(st);
        }
        excl_sum(tmp, icnt, s->L_in_start, P + 1, st);
        excl_sum(tmp, ocnt, s->L_out_start, P + 1, st);
        if (P) k_lspace_edges<<<grid_for(P), kGB, 0, st>>>(P, Lpin, s->L_of, s->in_start, s->in_from, s->out_start,
                                                            s->out_to, s->L_in_start, s->L_out_start, s->L_in_from,
                                                            s->L_out_to);
        CK_LAUNCH();
        s->L_pred.alloc(n), s->L_ak.alloc(n), s->L_rk.alloc(n), s->L_tie.alloc(n);
        s->L_arr.alloc(n), s->L_req.alloc(n), s->L_xy.alloc(n);
    }
    {   // endpoints ascending
        TBuf<int> e(st);
        e.upload(s->h_endpoints, st);
        s->ep_sorted.alloc(std::max(s->EP, 1));
        if (s->EP) {
            size_t b = 0;
            CK(cub::DeviceRadixSort::SortKeys(nullptr, b, e.p, s->ep_sorted.p, s->EP, 0, pbits, st));
            CK(cub::DeviceRadixSort::SortKeys(tmp.get(b), b, e.p, s->ep_sorted.p, s->EP, 0, pbits, st));
        }
        CK(cudaStreamSynchronize(st)); // (every temporary above is freed on return)
    }
    s->h_level_valid = false, s->h_arcs_valid = false;
}

// Host copies of the level array / the arc lists, downloaded on first use (tdpg_graph_info / _arcs).
void graph_host_level(tdpg_session* s)
{
    if (s->h_level_valid) return;
    s->h_level.resize(s->P);
    if (s->P) CK(cudaMemcpyAsync(s->h_level.data(), s->d_level.p, sizeof(int) * s->P, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    s->h_level_valid = true;
}

void graph_host_arcs(tdpg_session* s)
{
    if (s->h_arcs_valid) return;
    const size_t A = static_cast<size_t>(s->A);
    s->h_arc_from.resize(A), s->h_arc_to.resize(A), s->h_arc_kind.resize(A), s->h_arc_owner.resize(A);
    if (A) {
        CK(cudaMemcpyAsync(s->h_arc_from.data(), s->arc_from.p, 4 * A, cudaMemcpyDeviceToHost, s->st));
        CK(cudaMemcpyAsync(s->h_arc_to.data(), s->arc_to.p, 4 * A, cudaMemcpyDeviceToHost, s->st));
        CK(cudaMemcpyAsync(s->h_arc_kind.data(), s->arc_kind.p, 4 * A, cudaMemcpyDeviceToHost, s->st));
        CK(cudaMemcpyAsync(s->h_arc_owner.data(), s->arc_owner.p, 4 * A, cudaMemcpyDeviceToHost, s->st));
    }
    CK(cudaStreamSynchronize(s->st));
    s->h_arcs_valid = true;
}

} // namespace tdpg
