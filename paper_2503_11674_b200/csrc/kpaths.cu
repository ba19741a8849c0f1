// kpaths.cu — k worst paths per endpoint (report_timing_endpoint(n, k), paths.cpp:167-189), the topn
// policy (report_timing(n), paths.cpp:136-165), k_worst_paths_to (paths.cpp:57-72) and
// PathEnumerator::path_to(pin, rank) (paths.cpp:44-55) on the device.
//
// The reference enumerates lazily: per pin a list of found records and a heap holding one candidate
// per in-arc, the next unconsumed predecessor rank (paths.cpp:19-55).  Its output is therefore a
// deterministic function of the graph: the found list of pin v is the greedy merge of the in-arc
// streams found[u] + d(u, v), popping the largest delay first and breaking exact ties by the
// lexicographically smaller full pin sequence (CandidateOrder, paths.hpp:63-69).  Here that merge
// runs for every pin, level by level (all predecessors are final when a level starts), keeping the
// first K records of each list — exact, because a pin pops at most K times and never looks past rank
// K - 1 of a predecessor.  Records are (delay, predecessor pin, predecessor rank): a path is a chain,
// materialised only for output and for exact-delay ties.
//
// HBM layout: kb_delay double[P * K], kb_pred int2[P * K] (pred pin, pred rank; -1 for a source),
// kb_cnt int[P] (records found, <= K).
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <vector>

#include "gp_kernels.cuh"

namespace tdpg {

int api_fail(int kind, const std::string& msg);
void* cub_scratch(tdpg_session* s, size_t bytes);

namespace {

constexpr int kMaxFan = 32;   // in-arcs per pin handled by the merge (error beyond)
constexpr int kLocalPath = 64; // tie comparisons materialise paths up to this length in local memory

struct KbArgs {
    const int *lvl_pins, *in_start, *in_from, *pin_cell;
    const uint8_t *is_source, *pin_dir;
    const double *cell_delay, *pin_cap;
    const double2* pin_xy;
    double r, c;
    int K;
    double* kd;
    int2* kp;
    int* kc;
    int* err;
};

__device__ __forceinline__ double kb_net_delay(double2 a, double2 b, double cap, double r, double c)
{ // net_delay (sta.cpp:10-14)
    const double len = fabs(a.x - b.x) + fabs(a.y - b.y);
    return (r * len) * (c * len + cap);
}

__device__ int kb_len(const int2* kp, int K, int v, int r)
{
    int n = 1;
    for (int2 p = kp[static_cast<size_t>(v) * K + r]; p.x >= 0; p = kp[static_cast<size_t>(p.x) * K + p.y]) ++n;
    return n;
}

// pin at position i (0 = source) of the path (v, r) of length n
__device__ int kb_pin_at(const int2* kp, int K, int v, int r, int n, int i)
{
    for (int s = n - 1; s > i; --s) {
        const int2 p = kp[static_cast<size_t>(v) * K + r];
        v = p.x, r = p.y;
    }
    return v;
}

// Is path(u1, r1) ++ [v] lexicographically smaller than path(u2, r2) ++ [v]?  (std::vector operator<)
__device__ __noinline__ bool kb_lex_less(const int2* kp, int K, int u1, int r1, int u2, int r2, int v)
{
    const int n1 = kb_len(kp, K, u1, r1), n2 = kb_len(kp, K, u2, r2);
    if (n1 < kLocalPath && n2 < kLocalPath) {
        int b1[kLocalPath], b2[kLocalPath];
        int x = u1, y = r1;
        for (int i = n1 - 1; i >= 0; --i) {
            b1[i] = x;
            const int2 p = kp[static_cast<size_t>(x) * K + y];
            x = p.x, y = p.y;
        }
        x = u2, y = r2;
        for (int i = n2 - 1; i >= 0; --i) {
            b2[i] = x;
            const int2 p = kp[static_cast<size_t>(x) * K + y];
            x = p.x, y = p.y;
        }
        b1[n1] = v, b2[n2] = v;
        const int m = min(n1, n2) + 1;
        for (int i = 0; i < m; ++i)
            if (b1[i] != b2[i]) return b1[i] < b2[i];
        return n1 < n2;
    }
    const int m = min(n1, n2) + 1; // long paths: walk from the ends (quadratic, tie-only)
    for (int i = 0; i < m; ++i) {
        const int a = i < n1 ? kb_pin_at(kp, K, u1, r1, n1, i) : v;
        const int b = i < n2 ? kb_pin_at(kp, K, u2, r2, n2, i) : v;
        if (a != b) return a < b;
    }
    return n1 < n2;
}

// One level of the merge: thread per pin.
__global__ void __launch_bounds__(kBlock) k_kbest_level(int lo, int hi, KbArgs a)
{
    const int i = lo + blockIdx.x * kBlock + threadIdx.x;
    if (i >= hi) return;
    const int v = a.lvl_pins[i];
    const size_t base = static_cast<size_t>(v) * a.K;
    if (a.is_source[v]) { // initialize (paths.cpp:36-39)
        a.kd[base] = 0.0;
        a.kp[base] = make_int2(-1, -1);
        a.kc[v] = 1;
        return;
    }
    const int j0 = a.in_start[v], nf = a.in_start[v + 1] - j0;
    if (nf > kMaxFan) {
        atomicExch(a.err, 1);
        a.kc[v] = 0;
        return;
    }
    int ptr[kMaxFan];
    double dl[kMaxFan];
    const bool sink = a.pin_dir[v] == 0; // in-arcs of a sink are net arcs, of an output cell arcs
    const double2 pv = sink ? a.pin_xy[v] : make_double2(0.0, 0.0);
    const double cap = sink ? a.pin_cap[v] : 0.0;
    const double dcell = sink ? 0.0 : a.cell_delay[a.pin_cell[v]];
    for (int f = 0; f < nf; ++f) {
        const int u = a.in_from[j0 + f];
        ptr[f] = 0;
        dl[f] = sink ? kb_net_delay(a.pin_xy[u], pv, cap, a.r, a.c) : dcell;
    }
    int m = 0;
    for (; m < a.K; ++m) { // path_to's pop loop (paths.cpp:48-53)
        int bf = -1, bu = -1;
        double bd = 0.0;
        for (int f = 0; f < nf; ++f) {
            const int u = a.in_from[j0 + f];
            if (ptr[f] >= a.kc[u]) continue; // stream exhausted (no candidate pushed, paths.cpp:23)
            const double cd = a.kd[static_cast<size_t>(u) * a.K + ptr[f]] + dl[f]; // paths.cpp:25
            if (bf < 0 || cd > bd || (cd == bd && kb_lex_less(a.kp, a.K, u, ptr[f], bu, ptr[bf], v)))
                bf = f, bu = u, bd = cd;
        }
        if (bf < 0) break;
        a.kd[base + m] = bd;
        a.kp[base + m] = make_int2(bu, ptr[bf]);
        ++ptr[bf];
    }
    a.kc[v] = m;
}

// Per selected endpoint: paths kept (min(per, found)), their total pins.
__global__ void k_kb_count(int nsel, const int* __restrict__ ep, int per, const int2* __restrict__ kp,
                           const int* __restrict__ kc, int K, int* __restrict__ npath, int* __restrict__ npins)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= nsel) return;
    const int e = ep[i], c = min(per, kc[e]);
    int pins = 0;
    for (int r = 0; r < c; ++r) pins += kb_len(kp, K, e, r);
    npath[i] = c, npins[i] = pins;
}

// Candidate paths in (endpoint rank, path rank) order: pins source-first, slack = clock - delay
// (paths.cpp:69, :123).
__global__ void k_kb_write(int nsel, const int* __restrict__ ep, const int* __restrict__ npath,
                           const int* __restrict__ poff, const int* __restrict__ pinoff, const int2* __restrict__ kp,
                           const double* __restrict__ kd, int K, double clock, int* __restrict__ start,
                           int* __restrict__ len, int* __restrict__ pins, double* __restrict__ slack)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= nsel) return;
    const int e = ep[i];
    int o = pinoff[i];
    for (int r = 0; r < npath[i]; ++r) {
        const int p = poff[i] + r, n = kb_len(kp, K, e, r);
        start[p] = o, len[p] = n;
        slack[p] = clock - kd[static_cast<size_t>(e) * K + r];
        int v = e, rr = r;
        for (int k = o + n - 1; k >= o; --k) {
            pins[k] = v;
            const int2 q = kp[static_cast<size_t>(v) * K + rr];
            v = q.x, rr = q.y;
        }
        o += n;
    }
}

__global__ void k_kb_slack_keys(int np, const double* __restrict__ slack, unsigned long long* __restrict__ key,
                                int* __restrict__ idx)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p >= np) return;
    key[p] = double_key(slack[p]);
    idx[p] = p;
}

__device__ bool pins_less(const int* pins, int sa, int na, int sb, int nb)
{
    const int m = min(na, nb);
    for (int i = 0; i < m; ++i)
        if (pins[sa + i] != pins[sb + i]) return pins[sa + i] < pins[sb + i];
    return na < nb;
}

// report_timing's sort (paths.cpp:155-158): after a stable radix sort by slack, every group of equal
// slack is ordered by pin sequence (insertion sort by its head thread; equal slacks are rare).
__global__ void k_kb_fix_ties(int np, const unsigned long long* __restrict__ key, int* __restrict__ idx,
                              const int* __restrict__ start, const int* __restrict__ len, const int* __restrict__ pins)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= np || (i > 0 && key[i - 1] == key[i])) return;
    int j = i + 1;
    while (j < np && key[j] == key[i]) ++j;
    for (int a = i + 1; a < j; ++a) {
        const int x = idx[a];
        int b = a - 1;
        while (b >= i && pins_less(pins, start[x], len[x], start[idx[b]], len[idx[b]])) idx[b + 1] = idx[b], --b;
        idx[b + 1] = x;
    }
}

// topn completeness: an endpoint whose list was cut at K (< its per-endpoint budget) may hide paths
// that tie or beat the current n-th; flag it so the host retries with a larger K.
__global__ void k_kb_complete(int nsel, const int* __restrict__ ep, const int* __restrict__ kc, int K, int per,
                              const double* __restrict__ kd, double clock, const unsigned long long* __restrict__ skey,
                              long long np, int n, int* __restrict__ incomplete)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= nsel) return;
    const int e = ep[i];
    if (kc[e] < K || K >= per) return; // exhausted, or every budgeted path is present
    if (np < n) {
        atomicExch(incomplete, 1);
        return;
    }
    const unsigned long long last = double_key(clock - kd[static_cast<size_t>(e) * K + K - 1]);
    if (last <= skey[n - 1]) atomicExch(incomplete, 1);
}

// final paths: gather the first np candidates in `order` (topn) or take them as they are
__global__ void k_kb_gather_len(int np, const int* __restrict__ order, const int* __restrict__ len, int* __restrict__ out)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p < np) out[p] = len[order[p]];
}

__global__ void k_kb_gather(int np, const int* __restrict__ order, const int* __restrict__ cstart,
                            const int* __restrict__ clen, const int* __restrict__ cpins,
                            const double* __restrict__ cslack, const int* __restrict__ off, int* __restrict__ pins,
                            double* __restrict__ slack)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p >= np) return;
    const int q = order[p];
    for (int k = 0; k < clen[q]; ++k) pins[off[p] + k] = cpins[cstart[q] + k];
    slack[p] = cslack[q];
}

// collect_pin_pairs (paths.cpp:191-203): hops leaving an Output pin, per path.
__global__ void k_path_hops(int np, const int* __restrict__ start, const int* __restrict__ len,
                            const int* __restrict__ pins, const uint8_t* __restrict__ pin_dir, int* __restrict__ hops)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p >= np) return;
    int h = 0;
    for (int k = start[p]; k + 1 < start[p] + len[p]; ++k) h += pin_dir[pins[k]] == 1;
    hops[p] = h;
}

__global__ void k_path_hits(int np, const int* __restrict__ start, const int* __restrict__ len,
                            const int* __restrict__ pins, const double* __restrict__ slack,
                            const uint8_t* __restrict__ pin_dir, const int* __restrict__ hoff,
                            unsigned long long* __restrict__ hkey, double* __restrict__ hslack, int* __restrict__ hidx,
                            unsigned* __restrict__ sink_key)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p >= np) return;
    int h = hoff[p];
    const double sl = slack[p];
    for (int k = start[p]; k + 1 < start[p] + len[p]; ++k) {
        const int u = pins[k], v = pins[k + 1];
        if (pin_dir[u] != 1) continue;
        const unsigned lo = static_cast<unsigned>(min(u, v)), hi = static_cast<unsigned>(max(u, v));
        hkey[h] = (static_cast<unsigned long long>(lo) << 32) | hi;
        hslack[h] = sl;
        hidx[h] = h;
        if (sink_key) sink_key[h] = sl < 0.0 ? static_cast<unsigned>(v) : 0xFFFFFFFFu; // pin_pairs.cpp:11
        ++h;
    }
}

__global__ void k_unique_last(int np, const int* __restrict__ start, const int* __restrict__ len,
                              const int* __restrict__ pins, int* __restrict__ flag, int* __restrict__ count)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p >= np) return;
    if (atomicExch(&flag[pins[start[p] + len[p] - 1]], 1) == 0) atomicAdd(count, 1);
}

__global__ void k_count_heads64(long long n, const unsigned long long* __restrict__ k, int* __restrict__ out)
{
    int c = 0;
    for (long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * kBlock)
        c += (i == 0 || k[i - 1] != k[i]);
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

template <typename T>
T read1(tdpg_session* s, const T* p)
{
    T v{};
    CK(cudaMemcpyAsync(&v, p, sizeof(T), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    return v;
}

void exclusive_scan(tdpg_session* s, const int* in, int* out, int n)
{
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s->st);
    void* tmp = cub_scratch(s, bytes);
    CK(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n, s->st));
}

} // namespace

// ---- the engine's timing refresh with k > 1 paths per endpoint (report_timing_endpoint(n, k),
// placer.cpp:424-429) as one captured graph: every count lives on the device, buffers are sized for the
// worst case (every endpoint violated, k paths each, L + 1 pins per path), sorts run over the smallest
// size class holding the data (conditional graph node) — no host synchronisation inside the loop.
__device__ __forceinline__ int active_nv(const double* __restrict__ sta_out, const Ctrl* __restrict__ ctrl)
{
    return (!ctrl->stopped && sta_out[1] < 0.0) ? static_cast<int>(sta_out[2]) : 0;
}

__global__ void k_kb_count_dev(int cap, const double* __restrict__ sta_out, const Ctrl* __restrict__ ctrl,
                               const int* __restrict__ ep, int per, const int2* __restrict__ kp,
                               const int* __restrict__ kc, int K, int* __restrict__ npath, int* __restrict__ npins)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= cap) return;
    if (i >= active_nv(sta_out, ctrl)) {
        npath[i] = 0, npins[i] = 0;
        return;
    }
    const int e = ep[i], c = min(per, kc[e]);
    int pins = 0;
    for (int r = 0; r < c; ++r) pins += kb_len(kp, K, e, r);
    npath[i] = c, npins[i] = pins;
}

__global__ void k_kb_write_dev(int cap, const double* __restrict__ sta_out, const Ctrl* __restrict__ ctrl,
                               const int* __restrict__ ep, const int* __restrict__ npath, const int* __restrict__ poff,
                               const int* __restrict__ pinoff, const int2* __restrict__ kp,
                               const double* __restrict__ kd, int K, double clock, int* __restrict__ start,
                               int* __restrict__ len, int* __restrict__ pins, double* __restrict__ slack)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= cap || i >= active_nv(sta_out, ctrl)) return;
    const int e = ep[i];
    int o = pinoff[i];
    for (int r = 0; r < npath[i]; ++r) {
        const int p = poff[i] + r, n = kb_len(kp, K, e, r);
        start[p] = o, len[p] = n;
        slack[p] = clock - kd[static_cast<size_t>(e) * K + r];
        int v = e, rr = r;
        for (int k = o + n - 1; k >= o; --k) {
            pins[k] = v;
            const int2 q = kp[static_cast<size_t>(v) * K + rr];
            v = q.x, rr = q.y;
        }
        o += n;
    }
}

// totals of a capacity-sized count / exclusive-offset pair: out = off[n-1] + cnt[n-1]
__global__ void k_kb_totals(int n, const int* __restrict__ poff, const int* __restrict__ npath,
                            const int* __restrict__ pinoff, const int* __restrict__ npins, int* __restrict__ dn,
                            long long* __restrict__ ex_counts)
{
    const int np = poff[n - 1] + npath[n - 1], pins = pinoff[n - 1] + npins[n - 1];
    dn[0] = np, dn[1] = pins;
    ex_counts[0] = np, ex_counts[1] = pins;
    ex_counts[3] += np, ex_counts[4] += pins; // (engine totals, tdpg_engine_paths)
}

__global__ void k_path_hops_dev(int cap, const int* __restrict__ dn, const int* __restrict__ start,
                                const int* __restrict__ len, const int* __restrict__ pins,
                                const uint8_t* __restrict__ pin_dir, int* __restrict__ hops)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p >= cap) return;
    int h = 0;
    if (p < dn[0])
        for (int k = start[p]; k + 1 < start[p] + len[p]; ++k) h += pin_dir[pins[k]] == 1;
    hops[p] = h;
}

__global__ void k_hits_total(int n, const int* __restrict__ hoff, const int* __restrict__ hops,
                             long long* __restrict__ H, long long* __restrict__ ex_counts)
{
    H[0] = static_cast<long long>(hoff[n - 1]) + hops[n - 1];
    ex_counts[2] = H[0];
}

// collect_pin_pairs (paths.cpp:191-203) keyed by sink pin for the dense ledger (pin_pairs.cpp:11)
__global__ void k_path_hits_dev(int cap, const int* __restrict__ dn, const int* __restrict__ start,
                                const int* __restrict__ len, const int* __restrict__ pins,
                                const double* __restrict__ slack, const uint8_t* __restrict__ pin_dir,
                                const int* __restrict__ hoff, double* __restrict__ hslack, int* __restrict__ hidx,
                                unsigned* __restrict__ sink_key)
{
    const int p = blockIdx.x * kBlock + threadIdx.x;
    if (p >= cap || p >= dn[0]) return;
    int h = hoff[p];
    const double sl = slack[p];
    for (int k = start[p]; k + 1 < start[p] + len[p]; ++k) {
        const int u = pins[k], v = pins[k + 1];
        if (pin_dir[u] != 1) continue;
        hslack[h] = sl;
        hidx[h] = h;
        sink_key[h] = sl < 0.0 ? static_cast<unsigned>(v) : 0xFFFFFFFFu;
        ++h;
    }
}

// The K-best lists of every pin at the current STA's pin positions.
void kbest_build(tdpg_session* s, int K)
{
    sta_materialize_pins(s);
    const size_t P = static_cast<size_t>(std::max(s->P, 1));
    const double bytes = static_cast<double>(P) * K * (sizeof(double) + sizeof(int2));
    if (K < 1 || bytes > 48e9)
        throw Error(TDPG_ERR_VALIDATION, "validation error: k = " + std::to_string(K) +
                                             " paths per pin exceed the device memory budget for this design");
    if (s->kb_K != K) {
        s->kb_delay.alloc(P * K), s->kb_pred.alloc(P * K);
        s->kb_K = K;
    }
    s->kb_cnt.reserve(P);
    s->counters.reserve(8);
    CK(cudaMemsetAsync(s->counters.p + 2, 0, sizeof(int), s->st));
    KbArgs a;
    a.lvl_pins = s->lvl_pins, a.in_start = s->in_start, a.in_from = s->in_from, a.pin_cell = s->pin_cell;
    a.is_source = s->is_source, a.pin_dir = s->pin_dir, a.cell_delay = s->cell_delay, a.pin_cap = s->pin_cap;
    a.pin_xy = s->pin_xy, a.r = s->r_unit, a.c = s->c_unit, a.K = K;
    a.kd = s->kb_delay, a.kp = s->kb_pred, a.kc = s->kb_cnt, a.err = s->counters.p + 2;
    for (int l = 0; l < s->L; ++l) {
        const int lo = s->h_lvl_start[l], hi = s->h_lvl_start[l + 1];
        if (hi > lo) k_kbest_level<<<blocks_for(hi - lo, kBlock), kBlock, 0, s->st>>>(lo, hi, a);
    }
    CK_LAUNCH();
    if (capturing(s)) return; // (the engine checks the flag after its run: kbest_check)
    if (read1(s, s->counters.p + 2))
        throw Error(TDPG_ERR_INTERNAL, "path enumeration: a pin has more than 32 in-arcs");
}

void kbest_check(tdpg_session* s)
{
    if (s->kb_K > 0 && read1(s, s->counters.p + 2))
        throw Error(TDPG_ERR_INTERNAL, "path enumeration: a pin has more than 32 in-arcs");
}

// Worst-case capacities of the k-best engine refresh (every endpoint violated, K paths of <= L + 1 pins
// and <= (L + 1) / 2 + 1 hops each); every buffer sized before capture.
void kbest_refresh_reserve(tdpg_session* s, int K)
{
    const size_t P = static_cast<size_t>(std::max(s->P, 1));
    if (s->kb_K != K) {
        s->kb_delay.alloc(P * K), s->kb_pred.alloc(P * K);
        s->kb_K = K;
    }
    s->kb_cnt.reserve(P);
    s->counters.reserve(8);
    const long long EP = std::max(s->EP, 1), L = std::max(s->L, 1);
    const long long npc = EP * K, pinc = npc * (L + 1), hc = npc * ((L + 1) / 2 + 1);
    if (pinc > INT_MAX || hc > INT_MAX)
        throw Error(TDPG_ERR_VALIDATION, "validation error: k = " + std::to_string(K) +
                                             " paths per endpoint exceed the 2^31 path-pin capacity for this design");
    KbScratch& X = s->kbx;
    X.npath.reserve(EP), X.npins.reserve(EP), X.poff.reserve(EP), X.pinoff.reserve(EP);
    X.cstart.reserve(npc + 1), X.clen.reserve(npc + 1), X.cslack.reserve(npc + 1), X.cpins.reserve(pinc + 1);
    X.flag.reserve(npc + 1), X.order.reserve(npc + 1); // (hops / hop offsets)
    s->kh_key.reserve(hc + 1), s->kh_key_s.reserve(hc + 1), s->kh_idx_s.reserve(hc + 1);
    s->hit_slack.reserve(hc + 1), s->hit_idx.reserve(hc + 1);
    s->kb_dn.reserve(4), s->kb_H.reserve(2);
    s->kb_hcap = hc;
    size_t b1 = 0, b2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, b1, X.npath.p, X.poff.p, static_cast<int>(npc), s->st);
    cub::DeviceRadixSort::SortPairs(nullptr, b2, s->kh_key.p, s->kh_key_s.p, s->hit_idx.p, s->kh_idx_s.p,
                                    static_cast<int>(hc), 0, 32, s->st);
    cub_scratch(s, std::max(b1, b2));
}

void launch_ledger_update(tdpg_session* s, long long cap, const LedgerArgs& a);

// The k > 1 endpoint-policy refresh (placer.cpp:415-435): STA with per-pin results, violated endpoints
// in (slack, pin) order, the k-best lists, the first k paths of every violated endpoint, their hits keyed
// by sink pin, the dense-ledger update, net weights.  Recorded into the engine's refresh graph.
void refresh_record_kbest(tdpg_session* s, Ctrl* ctrl, double* timing_row, double w0, double w1,
                          bool net_weighting, int K)
{
    sta_record(s, s->sta_out, true); // (the k-best merge reads per-pin arrival and positions)
    refresh_begin(s, ctrl, timing_row);
    const int EP = s->EP;
    if (EP == 0) return;
    sort_violated_endpoints(s, ctrl);
    kbest_build(s, K);
    KbScratch& X = s->kbx;
    const int npc = EP * K;
    k_kb_count_dev<<<blocks_for(EP, kBlock), kBlock, 0, s->st>>>(EP, s->sta_out, ctrl, s->sort_v1, K, s->kb_pred,
                                                                 s->kb_cnt, K, X.npath, X.npins);
    CK_LAUNCH();
    size_t b = s->cub_tmp.n;
    CK(cub::DeviceScan::ExclusiveSum(s->cub_tmp.p, b, X.npath.p, X.poff.p, EP, s->st));
    b = s->cub_tmp.n;
    CK(cub::DeviceScan::ExclusiveSum(s->cub_tmp.p, b, X.npins.p, X.pinoff.p, EP, s->st));
    k_kb_write_dev<<<blocks_for(EP, kBlock), kBlock, 0, s->st>>>(EP, s->sta_out, ctrl, s->sort_v1, X.npath, X.poff,
                                                                 X.pinoff, s->kb_pred, s->kb_delay, K, s->clock,
                                                                 X.cstart, X.clen, X.cpins, X.cslack);
    CK_LAUNCH();
    k_kb_totals<<<1, 1, 0, s->st>>>(EP, X.poff, X.npath, X.pinoff, X.npins, s->kb_dn, s->ex_counts);
    CK_LAUNCH();
    int* hops = X.flag.p;
    int* hoff = X.order.p;
    k_path_hops_dev<<<blocks_for(npc, kBlock), kBlock, 0, s->st>>>(npc, s->kb_dn, X.cstart, X.clen, X.cpins,
                                                                   s->pin_dir, hops);
    CK_LAUNCH();
    b = s->cub_tmp.n;
    CK(cub::DeviceScan::ExclusiveSum(s->cub_tmp.p, b, hops, hoff, npc, s->st));
    k_hits_total<<<1, 1, 0, s->st>>>(npc, hoff, hops, s->kb_H, s->ex_counts);
    CK_LAUNCH();
    k_path_hits_dev<<<blocks_for(npc, kBlock), kBlock, 0, s->st>>>(npc, s->kb_dn, X.cstart, X.clen, X.cpins,
                                                                   X.cslack, s->pin_dir, hoff, s->hit_slack,
                                                                   s->hit_idx, s->kh_key);
    CK_LAUNCH();
    pad_hit_keys(s, s->kb_hcap, s->kb_H.p, s->kh_key.p);
    const int kbits = bits_for_pins(s->P);
    switch_hits_by_count(s, s->kb_H.p, s->kb_hcap, [&](cudaStream_t st, long long n) {
        size_t bb = s->cub_tmp.n;
        CK(cub::DeviceRadixSort::SortPairs(s->cub_tmp.p, bb, s->kh_key.p, s->kh_key_s.p, s->hit_idx.p, s->kh_idx_s.p,
                                           static_cast<int>(n), 0, kbits, st));
    });
    LedgerArgs la{};
    la.n_hits = s->kb_H.p, la.H = s->kb_hcap, la.sta_out = s->sta_out, la.ctrl = ctrl, la.gen = true;
    la.hk = s->kh_key_s, la.hidx = s->kh_idx_s, la.hslack = s->hit_slack, la.w0 = w0, la.w1 = w1;
    la.dl_w = s->dl_w, la.ppw_e = s->ppw_e, la.pin_entry = s->pin_entry, la.pin_loc = s->pin_loc;
    la.pp_mask = s->pp_mask, la.q_count = s->q_count;
    launch_ledger_update(s, s->kb_hcap, la);
    if (net_weighting && s->N) net_weights_record(s, ctrl);
}

// Observer rounds of the k-best refresh: this round's paths into the session's report buffers.
void kbest_refresh_publish(tdpg_session* s)
{
    int dn[2];
    CK(cudaMemcpyAsync(dn, s->kb_dn.p, sizeof dn, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    const int np = dn[0];
    const long long pins = dn[1];
    KbScratch& X = s->kbx;
    s->ex_off.reserve(np + 1), s->ex_len.reserve(np + 1), s->ex_slack.reserve(np + 1), s->ex_pins.reserve(pins + 1);
    if (np > 0) {
        CK(cudaMemcpyAsync(s->ex_off.p, X.cstart.p, sizeof(int) * np, cudaMemcpyDeviceToDevice, s->st));
        CK(cudaMemcpyAsync(s->ex_len.p, X.clen.p, sizeof(int) * np, cudaMemcpyDeviceToDevice, s->st));
        CK(cudaMemcpyAsync(s->ex_slack.p, X.cslack.p, sizeof(double) * np, cudaMemcpyDeviceToDevice, s->st));
        CK(cudaMemcpyAsync(s->ex_pins.p, X.cpins.p, sizeof(int) * pins, cudaMemcpyDeviceToDevice, s->st));
    }
    s->n_paths = np, s->n_path_pins = pins, s->n_hits = 0, s->candidates = np;
}

// Endpoint-sorted violated endpoints of the current STA (paths.cpp:77-87) into sort_v1; returns their count.
int sorted_violated(tdpg_session* s);

// report_timing_endpoint(n, k) (policy 0) / report_timing(n) (policy 1) on the current STA.  n <= 0
// selects every violated endpoint (placer.cpp:424-429).  Results land in the session's extraction
// buffers (ex_off / ex_pins / ex_slack, hits); with sink_keys the engine's dense-ledger hit keys too.
void extract_policy_dev(tdpg_session* s, int policy, int n, int k, bool sink_keys)
{
    if (!s->sta_valid) run_sta_dev(s);
    const int nv = sorted_violated(s);
    if (n <= 0) n = nv;
    const int nsel = std::min(n, nv);
    const int per = policy == 1 ? n : k;
    s->n_paths = 0, s->n_path_pins = 0, s->n_hits = 0, s->uniq_pairs = 0, s->uniq_endpoints = 0;
    s->candidates = policy == 1 ? static_cast<long long>(nsel) * n : 0;
    s->hits_sorted = false;
    if (nsel <= 0 || per <= 0) return;
    const int* ep = s->sort_v1.p;
    // session-owned grow-only scratch: no cudaMalloc / cudaFree (device-synchronising) per extraction
    KbScratch& X = s->kbx;
    DBuf<int>&npath = X.npath, &npins = X.npins, &poff = X.poff, &pinoff = X.pinoff;
    npath.reserve(nsel), npins.reserve(nsel), poff.reserve(nsel), pinoff.reserve(nsel);
    int K = policy == 1 ? std::min(per, 16) : per;
    long long np = 0, npins_tot = 0;
    DBuf<int>&cstart = X.cstart, &clen = X.clen, &cpins = X.cpins, &order = X.order;
    DBuf<double>& cslack = X.cslack;
    DBuf<unsigned long long>&key0 = X.key0, &key1 = X.key1;
    DBuf<int>& idx0 = X.idx0;
    for (;;) {
        kbest_build(s, K);
        k_kb_count<<<blocks_for(nsel, kBlock), kBlock, 0, s->st>>>(nsel, ep, per, s->kb_pred, s->kb_cnt, K, npath,
                                                                   npins);
        CK_LAUNCH();
        exclusive_scan(s, npath, poff, nsel);
        exclusive_scan(s, npins, pinoff, nsel);
        np = static_cast<long long>(read1(s, poff.p + nsel - 1)) + read1(s, npath.p + nsel - 1);
        npins_tot = static_cast<long long>(read1(s, pinoff.p + nsel - 1)) + read1(s, npins.p + nsel - 1);
        if (np > INT_MAX || npins_tot > INT_MAX)
            throw Error(TDPG_ERR_VALIDATION, "validation error: path report exceeds 2^31 entries");
        cstart.reserve(np + 1), clen.reserve(np + 1), cslack.reserve(np + 1), cpins.reserve(npins_tot + 1);
        k_kb_write<<<blocks_for(nsel, kBlock), kBlock, 0, s->st>>>(nsel, ep, npath, poff, pinoff, s->kb_pred,
                                                                   s->kb_delay, K, s->clock, cstart, clen, cpins,
                                                                   cslack);
        CK_LAUNCH();
        if (policy == 0) break;
        // topn: order all candidates by (slack, pins), then check that no cut list could still compete
        key0.reserve(np + 1), key1.reserve(np + 1), idx0.reserve(np + 1), order.reserve(np + 1);
        if (np > 0) {
            k_kb_slack_keys<<<blocks_for(np, kBlock), kBlock, 0, s->st>>>(static_cast<int>(np), cslack, key0, idx0);
            CK_LAUNCH();
            size_t bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, bytes, key0.p, key1.p, idx0.p, order.p, static_cast<int>(np), 0,
                                            64, s->st);
            void* tmp = cub_scratch(s, bytes);
            CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, key0.p, key1.p, idx0.p, order.p, static_cast<int>(np), 0,
                                               64, s->st));
            k_kb_fix_ties<<<blocks_for(np, kBlock), kBlock, 0, s->st>>>(static_cast<int>(np), key1, order, cstart,
                                                                        clen, cpins);
            CK_LAUNCH();
        }
        if (K >= per) break;
        CK(cudaMemsetAsync(s->counters.p + 3, 0, sizeof(int), s->st));
        k_kb_complete<<<blocks_for(nsel, kBlock), kBlock, 0, s->st>>>(nsel, ep, s->kb_cnt, K, per, s->kb_delay,
                                                                      s->clock, key1, np, n, s->counters.p + 3);
        CK_LAUNCH();
        if (!read1(s, s->counters.p + 3)) break;
        K = static_cast<int>(std::min<long long>(per, 4LL * K));
    }
    // final paths
    const int nfin = policy == 1 ? static_cast<int>(std::min<long long>(np, n)) : static_cast<int>(np);
    s->ex_off.reserve(nfin + 1), s->ex_len.reserve(nfin + 1), s->ex_slack.reserve(nfin + 1);
    if (policy == 0) {
        CK(cudaMemcpyAsync(s->ex_off.p, cstart.p, sizeof(int) * nfin, cudaMemcpyDeviceToDevice, s->st));
        CK(cudaMemcpyAsync(s->ex_len.p, clen.p, sizeof(int) * nfin, cudaMemcpyDeviceToDevice, s->st));
        CK(cudaMemcpyAsync(s->ex_slack.p, cslack.p, sizeof(double) * nfin, cudaMemcpyDeviceToDevice, s->st));
        s->ex_pins.reserve(npins_tot + 1);
        CK(cudaMemcpyAsync(s->ex_pins.p, cpins.p, sizeof(int) * npins_tot, cudaMemcpyDeviceToDevice, s->st));
        s->n_path_pins = npins_tot;
        s->candidates = np; // paths.cpp:181-184
    } else if (nfin > 0) {
        k_kb_gather_len<<<blocks_for(nfin, kBlock), kBlock, 0, s->st>>>(nfin, order, clen, s->ex_len);
        CK_LAUNCH();
        exclusive_scan(s, s->ex_len, s->ex_off, nfin);
        s->n_path_pins = static_cast<long long>(read1(s, s->ex_off.p + nfin - 1)) + read1(s, s->ex_len.p + nfin - 1);
        s->ex_pins.reserve(s->n_path_pins + 1);
        k_kb_gather<<<blocks_for(nfin, kBlock), kBlock, 0, s->st>>>(nfin, order, cstart, clen, cpins, cslack, s->ex_off,
                                                                    s->ex_pins, s->ex_slack);
        CK_LAUNCH();
    }
    s->n_paths = nfin;
    if (nfin == 0) return;
    // hits (collect_pin_pairs) and finish_report counters (paths.cpp:89-102)
    s->ex_hops.reserve(nfin + 1), s->ex_hoff.reserve(nfin + 1);
    k_path_hops<<<blocks_for(nfin, kBlock), kBlock, 0, s->st>>>(nfin, s->ex_off, s->ex_len, s->ex_pins, s->pin_dir,
                                                                s->ex_hops);
    CK_LAUNCH();
    exclusive_scan(s, s->ex_hops, s->ex_hoff, nfin);
    const long long H = static_cast<long long>(read1(s, s->ex_hoff.p + nfin - 1)) + read1(s, s->ex_hops.p + nfin - 1);
    s->n_hits = H;
    s->hit_key.reserve(H + 1), s->hit_slack.reserve(H + 1), s->hit_idx.reserve(H + 1);
    s->hit_key_s.reserve(H + 1), s->hit_idx_s.reserve(H + 1);
    if (sink_keys) s->kh_key.reserve(H + 1), s->kh_key_s.reserve(H + 1), s->kh_idx_s.reserve(H + 1);
    k_path_hits<<<blocks_for(nfin, kBlock), kBlock, 0, s->st>>>(nfin, s->ex_off, s->ex_len, s->ex_pins, s->ex_slack,
                                                                s->pin_dir, s->ex_hoff, s->hit_key, s->hit_slack,
                                                                s->hit_idx, sink_keys ? s->kh_key.p : nullptr);
    CK_LAUNCH();
    DBuf<int>& flag = X.flag;
    flag.reserve(std::max(s->P, 1));
    flag.zero(s->st, std::max(s->P, 1));
    CK(cudaMemsetAsync(s->counters.p + 4, 0, 2 * sizeof(int), s->st));
    k_unique_last<<<blocks_for(nfin, kBlock), kBlock, 0, s->st>>>(nfin, s->ex_off, s->ex_len, s->ex_pins, flag,
                                                                  s->counters.p + 4);
    CK_LAUNCH();
    if (H > 0) {
        size_t bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, bytes, s->hit_key.p, s->hit_key_s.p, s->hit_idx.p, s->hit_idx_s.p,
                                        static_cast<int>(H), 0, 64, s->st);
        void* tmp = cub_scratch(s, bytes);
        CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, s->hit_key.p, s->hit_key_s.p, s->hit_idx.p, s->hit_idx_s.p,
                                           static_cast<int>(H), 0, 64, s->st));
        k_count_heads64<<<std::min<unsigned>(blocks_for(H, kBlock), 148 * 4), kBlock, 0, s->st>>>(H, s->hit_key_s,
                                                                                                   s->counters.p + 5);
        CK_LAUNCH();
        if (sink_keys) {
            bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, bytes, s->kh_key.p, s->kh_key_s.p, s->hit_idx.p, s->kh_idx_s.p,
                                            static_cast<int>(H), 0, 32, s->st);
            tmp = cub_scratch(s, bytes);
            CK(cub::DeviceRadixSort::SortPairs(tmp, bytes, s->kh_key.p, s->kh_key_s.p, s->hit_idx.p, s->kh_idx_s.p,
                                               static_cast<int>(H), 0, 32, s->st));
        }
    }
    int cnt[2];
    CK(cudaMemcpyAsync(cnt, s->counters.p + 4, sizeof cnt, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    s->uniq_endpoints = cnt[0];
    s->uniq_pairs = H > 0 ? cnt[1] : 0;
    s->hits_sorted = true;
}

// PathEnumerator::path_to(pin, rank) / k_worst_paths_to(endpoint, k) on the current STA: K-best lists
// with K = rank + 1 (resp. k), the requested pin's records materialised on the host side.
void kbest_paths_of(tdpg_session* s, int pin, int K, std::vector<std::vector<int>>& paths, std::vector<double>& delay)
{
    if (!s->sta_valid) run_sta_dev(s);
    kbest_build(s, K);
    const int c = read1(s, s->kb_cnt.p + pin);
    std::vector<int2> kp;
    paths.clear(), delay.clear();
    if (c == 0) return;
    // the chains of the pin's records stay inside its fan-in cone: pull the whole table once (small
    // designs) or walk record by record (large ones)
    auto rec = [&](int v, int r) {
        int2 q;
        CK(cudaMemcpyAsync(&q, s->kb_pred.p + static_cast<size_t>(v) * K + r, sizeof q, cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
        return q;
    };
    std::vector<double> d(c);
    CK(cudaMemcpyAsync(d.data(), s->kb_delay.p + static_cast<size_t>(pin) * K, sizeof(double) * c,
                       cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    for (int r = 0; r < c; ++r) {
        std::vector<int> p;
        int v = pin, rr = r;
        while (v >= 0) {
            p.push_back(v);
            const int2 q = rec(v, rr);
            v = q.x, rr = q.y;
        }
        std::reverse(p.begin(), p.end());
        paths.push_back(std::move(p));
        delay.push_back(d[r]);
    }
}

} // namespace tdpg
