// tdp_api.cpp — the reference's tdp:: operator API implemented over the sm_100a engine (include/tdpg.h).
//
// A device session is created once per netlist and cached (keyed on the Netlist's address, sizes, storage
// addresses and a fixed-size content sample: O(1) per call), so per-iteration calls such as
// objective_and_gradient only upload positions.  Per-net calls on bare points (wa_wirelength, hpwl_net,
// pin_pair_loss, update_pair_weights) reuse one scratch session per point count.  Exceptions
// from the C-ABI are re-thrown as the reference's exception classes with the reference's messages.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <memory>
#include <sstream>
#include <mutex>
#include <thread>
#include <set>

#include <json.hpp> // nlohmann json (header-only, the reference's own JSON dependency)

#include "tdp/tdp_api.hpp"
#include "tdpg.h"

namespace tdp {

namespace {

std::string strip(const std::string& m, const char* prefix)
{
    const std::string p(prefix);
    return m.compare(0, p.size(), p) == 0 ? m.substr(p.size()) : m;
}

[[noreturn]] void rethrow(int kind)
{
    const std::string m = tdpg_last_error();
    switch (kind) {
    case TDPG_ERR_PARSE: throw ParseError(strip(m, "parse error: "));
    case TDPG_ERR_CYCLE: throw CycleError(strip(m, "validation error: combinational cycle: "));
    case TDPG_ERR_ENDPOINT: throw EndpointError(strip(m, "validation error: "));
    case TDPG_ERR_VALIDATION: throw ValidationError(strip(m, "validation error: "));
    case TDPG_ERR_GRAPH: throw GraphError(strip(m, "graph error: "));
    case TDPG_ERR_NONFINITE: throw NonFiniteError(strip(m, "non-finite value: "));
    case TDPG_ERR_INTERNAL: throw std::logic_error(m);
    default: throw std::runtime_error(m);
    }
}

void ck(int rc)
{
    if (rc != TDPG_OK) rethrow(rc);
}

// Flat SoA copy of a Netlist + constraints, owned alongside the session it created.
struct FlatNetlist {
    std::vector<double> cw, ch, cd, pt, po, pc;
    std::vector<uint8_t> cf, pd;
    std::vector<int32_t> pcell, ns, np, src, ep;
    std::vector<std::string> names;
    std::vector<const char*> name_ptrs;
    tdpg_netlist view{};

    FlatNetlist(const Netlist& nl, const DesignConstraints& c)
    {
        const size_t C = nl.cells.size(), P = nl.pins.size();
        cw.resize(C), ch.resize(C), cd.resize(C), cf.resize(C);
        for (size_t i = 0; i < C; ++i) {
            const Cell& cell = nl.cells[i];
            cw[i] = cell.width, ch[i] = cell.height, cd[i] = cell.delay, cf[i] = cell.is_fixed;
        }
        pcell.resize(P), pt.resize(2 * P), po.resize(2 * P), pd.resize(P), pc.resize(P);
        bool named = false;
        for (size_t i = 0; i < P; ++i) {
            const Pin& p = nl.pins[i];
            pcell[i] = p.cell;
            pt[2 * i] = p.terminal_pos.x, pt[2 * i + 1] = p.terminal_pos.y;
            po[2 * i] = p.offset.x, po[2 * i + 1] = p.offset.y;
            pd[i] = p.dir == PinDir::Output ? 1 : 0;
            pc[i] = p.load_cap;
            named = named || !p.name.empty();
        }
        if (named) { // (names only feed error messages: skipped when the netlist has none)
            names.reserve(P);
            for (const Pin& p : nl.pins) names.push_back(p.name);
        }
        size_t E = 0;
        for (const Net& n : nl.nets) E += 1 + n.sinks.size();
        ns.reserve(nl.nets.size() + 1), np.reserve(E);
        ns.push_back(0);
        for (const Net& n : nl.nets) {
            np.push_back(n.driver);
            for (int s : n.sinks) np.push_back(s);
            ns.push_back(static_cast<int32_t>(np.size()));
        }
        src.assign(nl.sources.begin(), nl.sources.end());
        ep.assign(nl.endpoints.begin(), nl.endpoints.end());
        for (const auto& s : names) name_ptrs.push_back(s.c_str());
        view.n_cells = static_cast<int32_t>(C), view.n_pins = static_cast<int32_t>(P);
        view.n_nets = static_cast<int32_t>(nl.nets.size());
        view.n_sources = static_cast<int32_t>(src.size()), view.n_endpoints = static_cast<int32_t>(ep.size());
        view.cell_w = cw.data(), view.cell_h = ch.data(), view.cell_delay = cd.data(), view.cell_fixed = cf.data();
        view.pin_cell = pcell.data(), view.pin_term = pt.data(), view.pin_off = po.data(), view.pin_dir = pd.data();
        view.pin_cap = pc.data(), view.net_start = ns.data(), view.net_pins = np.data(), view.sources = src.data();
        view.endpoints = ep.data(), view.clock_period = c.clock_period > 0 ? c.clock_period : 1.0;
        view.r_unit = c.r_unit, view.c_unit = c.c_unit;
        view.core[0] = c.core.x_lo, view.core[1] = c.core.y_lo, view.core[2] = c.core.x_hi, view.core[3] = c.core.y_hi;
        if (names.empty()) name_ptrs.assign(P, ""); // (all blank: the engine stores none)
        view.pin_names = name_ptrs.data();
    }
};

struct Sess {
    std::unique_ptr<FlatNetlist> flat;
    tdpg_session* s = nullptr;
    std::vector<std::size_t> fp;
    ~Sess()
    {
        if (s) tdpg_session_destroy(s);
    }
};

// Identity of a Netlist for the session cache, O(1) in the netlist size: the reference's Netlist is
// immutable after construction, so its address, its sizes and the addresses of its
// storage identify it; a fixed sample of 64 evenly spaced cells, pins and nets guards against a
// different netlist later built at a reused address.  (Round 1 hashed every byte: 0.3 s per call at 1M.)
std::vector<std::size_t> netlist_key(const Netlist& nl)
{
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* p, std::size_t n) {
        const auto* b = static_cast<const unsigned char*>(p);
        for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    };
    auto d = [&](double x) { mix(&x, sizeof x); };
    auto i32 = [&](int x) { mix(&x, sizeof x); };
    constexpr std::size_t kSample = 64;
    auto each = [&](std::size_t n, auto&& f) {
        const std::size_t step = std::max<std::size_t>(1, n / kSample);
        for (std::size_t i = 0; i < n; i += step) f(i);
        if (n) f(n - 1);
    };
    each(nl.cells.size(), [&](std::size_t i) {
        const Cell& c = nl.cells[i];
        d(c.width), d(c.height), d(c.delay), i32(c.is_fixed);
    });
    each(nl.pins.size(), [&](std::size_t i) {
        const Pin& p = nl.pins[i];
        i32(p.cell), d(p.terminal_pos.x), d(p.terminal_pos.y), d(p.offset.x), d(p.offset.y);
        i32(p.dir == PinDir::Output), d(p.load_cap);
    });
    each(nl.nets.size(), [&](std::size_t i) {
        const Net& n = nl.nets[i];
        i32(n.driver), i32(static_cast<int>(n.sinks.size()));
        if (!n.sinks.empty()) i32(n.sinks.front()), i32(n.sinks.back());
    });
    auto addr = [](const void* p) { return reinterpret_cast<std::size_t>(p); };
    return {nl.cells.size(), nl.pins.size(), nl.nets.size(), nl.sources.size(), nl.endpoints.size(),
            addr(nl.cells.data()), addr(nl.pins.data()), addr(nl.nets.data()), addr(nl.sources.data()),
            addr(nl.endpoints.data()), static_cast<std::size_t>(h)};
}

std::mutex g_mu;
std::map<const Netlist*, std::shared_ptr<Sess>> g_cache;

// A private device session (not cached): concurrent callers (run_compare's parallel rows) each own one.
std::shared_ptr<Sess> fresh_session(const Netlist& nl, const DesignConstraints& c)
{
    auto S = std::make_shared<Sess>();
    S->flat = std::make_unique<FlatNetlist>(nl, c);
    S->fp = netlist_key(nl);
    ck(tdpg_session_create(&S->flat->view, &S->s));
    ck(tdpg_set_constraints(S->s, c.clock_period > 0 ? c.clock_period : 1.0, c.r_unit, c.c_unit));
    return S;
}

// Device session for this netlist (rebuilt when the netlist or the core changed).
std::shared_ptr<Sess> session(const Netlist& nl, const DesignConstraints& c)
{
    std::lock_guard<std::mutex> lock(g_mu);
    auto fp = netlist_key(nl);
    auto it = g_cache.find(&nl);
    if (it != g_cache.end() && it->second->fp == fp) {
        ck(tdpg_set_constraints(it->second->s, c.clock_period > 0 ? c.clock_period : 1.0, c.r_unit, c.c_unit));
        return it->second;
    }
    auto S = std::make_shared<Sess>();
    S->flat = std::make_unique<FlatNetlist>(nl, c);
    S->fp = std::move(fp);
    ck(tdpg_session_create(&S->flat->view, &S->s));
    if (g_cache.size() > 64) g_cache.clear();
    g_cache[&nl] = S;
    return S;
}

// A design core for netlist-only calls: any nondegenerate rect works for STA/WA/PP.
DesignConstraints core_only(const Rect& core)
{
    DesignConstraints c;
    c.core = core.nondegenerate() ? core : Rect{0.0, 0.0, 1.0, 1.0};
    c.r_unit = c.c_unit = 1.0;
    c.clock_period = 1.0;
    return c;
}

// Point is two packed doubles, so a std::vector<Point> is already the C-ABI's flat (x, y) array: the
// engine reads the caller's positions in place and writes results straight into Point vectors.
static_assert(sizeof(Point) == 2 * sizeof(double), "Point must be two packed doubles");
struct FlatRef {
    const double* p;
    const double* data() const { return p; }
};
FlatRef flat_points(const std::vector<Point>& p) { return {reinterpret_cast<const double*>(p.data())}; }
double* flat_out(std::vector<Point>& p) { return reinterpret_cast<double*>(p.data()); }


// One-net scratch netlist of terminal pins at the given positions (pin 0 drives the rest).
struct PointNet {
    Netlist nl;
    explicit PointNet(std::span<const Point> pts)
    {
        for (std::size_t i = 0; i < pts.size(); ++i) {
            Pin p;
            p.name = "t" + std::to_string(i);
            p.terminal_pos = pts[i];
            p.dir = i == 0 ? PinDir::Output : PinDir::Input;
            nl.pins.push_back(p);
        }
        if (pts.size() >= 2) {
            Net n;
            n.name = "n";
            n.driver = 0;
            for (std::size_t i = 1; i < pts.size(); ++i) n.sinks.push_back(static_cast<int>(i));
            nl.nets.push_back(n);
        }
        nl.finalize();
    }
};

// Scratch session for calls on bare points: the one-net netlist of n terminal pins above, one per
// point count and thread, kept across calls and re-pointed with tdpg_set_terminal_positions.
tdpg_session* scratch_session(std::span<const Point> pts)
{
    struct Entry {
        std::unique_ptr<PointNet> net;
        std::shared_ptr<Sess> S;
    };
    thread_local std::map<std::size_t, Entry> cache;
    auto it = cache.find(pts.size());
    if (it == cache.end()) {
        if (cache.size() >= 16) cache.clear();
        Entry e{std::make_unique<PointNet>(pts), nullptr};
        e.S = fresh_session(e.net->nl, core_only({}));
        return cache.emplace(pts.size(), std::move(e)).first->second.S->s;
    }
    std::vector<double> xy(2 * pts.size());
    for (std::size_t i = 0; i < pts.size(); ++i) xy[2 * i] = pts[i].x, xy[2 * i + 1] = pts[i].y;
    ck(tdpg_set_terminal_positions(it->second.S->s, xy.data()));
    return it->second.S->s;
}

void set_core(tdpg_session* s, const Rect& r)
{
    const double core[4] = {r.x_lo, r.y_lo, r.x_hi, r.y_hi};
    ck(tdpg_set_core(s, core));
}

void ledger_upload(tdpg_session* s, const PinPairWeights& w)
{
    std::vector<int32_t> a, b;
    std::vector<double> ww;
    a.reserve(w.size()), b.reserve(w.size()), ww.reserve(w.size());
    for (const auto& [pr, x] : w) a.push_back(pr.first), b.push_back(pr.second), ww.push_back(x);
    ck(tdpg_pp_set(s, static_cast<int64_t>(a.size()), a.data(), b.data(), ww.data()));
}

PinPairWeights ledger_download(tdpg_session* s)
{
    int64_t q = 0;
    ck(tdpg_pp_size(s, &q));
    std::vector<int32_t> a(q), b(q);
    std::vector<double> w(q);
    if (q) ck(tdpg_pp_get(s, a.data(), b.data(), w.data()));
    PinPairWeights out;
    for (int64_t i = 0; i < q; ++i) out.emplace(std::make_pair(a[i], b[i]), w[i]);
    return out;
}

TimingAnnotation fetch_annotation(tdpg_session* s, const Netlist& nl)
{
    const std::size_t P = nl.pins.size();
    TimingAnnotation ann;
    ann.arr.resize(P), ann.req.resize(P), ann.slack.resize(P);
    std::vector<uint8_t> ak(P), rk(P);
    ck(tdpg_sta_fetch(s, ann.arr.data(), ann.req.data(), ann.slack.data(), ak.data(), rk.data(), &ann.tns, &ann.wns));
    ann.arr_known.assign(ak.begin(), ak.end());
    ann.req_known.assign(rk.begin(), rk.end());
    for (int e : nl.endpoints) ann.endpoint_slacks.emplace_back(e, ann.slack[static_cast<std::size_t>(e)]);
    return ann;
}

ExtractionReport fetch_report(tdpg_session* s, const Netlist& nl, int n, int k, const int64_t counts[5], double ms,
                              const char* policy = "endpoint")
{
    ExtractionReport r;
    r.policy = policy, r.n = n, r.k = k;
    const int np = static_cast<int>(counts[0]);
    std::vector<int32_t> start(np + 1), pins(std::max<int64_t>(counts[1], 1));
    std::vector<double> slack(std::max(np, 1));
    ck(tdpg_paths_get(s, start.data(), pins.data(), slack.data()));
    for (int i = 0; i < np; ++i)
        r.paths.push_back(CriticalPath{std::vector<int>(pins.begin() + start[i], pins.begin() + start[i + 1]), slack[i]});
    r.unique_endpoints = static_cast<int>(counts[2]);
    r.unique_pin_pairs = static_cast<int>(counts[3]);
    r.candidates_generated = counts[4];
    r.elapsed_ms = ms;
    (void)nl;
    return r;
}

// STA on the device at the given pin positions.
std::shared_ptr<Sess> sta_at(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                             const DesignConstraints& c)
{
    if (!graph.levelized || graph.level.size() != static_cast<std::size_t>(graph.num_pins))
        throw GraphError("timing graph is not levelized");
    auto S = session(nl, c);
    const auto xy = flat_points(pos);
    ck(tdpg_set_pin_positions(S->s, xy.data()));
    ck(tdpg_sta(S->s, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
    return S;
}

} // namespace

// ---- netlist -----------------------------------------------------------------------------------
void Netlist::finalize()
{ // netlist.cpp:5-21 semantics: per-cell ascending pin lists, owning net per pin, role flags
    cell_pins.assign(cells.size(), {});
    pin_net.assign(pins.size(), -1);
    pin_is_source.assign(pins.size(), false);
    pin_is_endpoint.assign(pins.size(), false);
    for (std::size_t p = 0; p < pins.size(); ++p)
        if (pins[p].cell >= 0) cell_pins[static_cast<std::size_t>(pins[p].cell)].push_back(static_cast<int>(p));
    for (std::size_t n = 0; n < nets.size(); ++n) {
        pin_net[static_cast<std::size_t>(nets[n].driver)] = static_cast<int>(n);
        for (int s : nets[n].sinks) pin_net[static_cast<std::size_t>(s)] = static_cast<int>(n);
    }
    for (int s : sources) pin_is_source[static_cast<std::size_t>(s)] = true;
    for (int e : endpoints) pin_is_endpoint[static_cast<std::size_t>(e)] = true;
}

PinPositions pin_positions(const Netlist& nl, const std::vector<Point>& cell_pos)
{
    auto S = session(nl, core_only({}));
    const auto xy = flat_points(cell_pos);
    ck(tdpg_set_positions(S->s, xy.data()));
    PinPositions out(nl.pins.size());
    ck(tdpg_pin_positions(S->s, flat_out(out)));
    return out;
}

// ---- timing graph ----------------------------------------------------------------------------------
TimingGraph build_timing_graph(const Netlist& nl)
{
    auto S = session(nl, core_only({}));
    TimingGraph g;
    g.num_pins = static_cast<int>(nl.pins.size());
    int32_t cnt[4];
    g.level.resize(nl.pins.size());
    ck(tdpg_graph_info(S->s, cnt, g.level.data()));
    g.num_net_arcs = cnt[0], g.num_cell_arcs = cnt[1];
    const std::size_t A = static_cast<std::size_t>(cnt[0]) + cnt[1];
    std::vector<int32_t> from(A), to(A), kind(A), owner(A);
    ck(tdpg_graph_arcs(S->s, from.data(), to.data(), kind.data(), owner.data()));
    g.arcs.resize(A);
    g.in_arcs.assign(nl.pins.size(), {});
    g.out_arcs.assign(nl.pins.size(), {});
    for (std::size_t a = 0; a < A; ++a) {
        g.arcs[a] = Arc{from[a], to[a], kind[a] ? ArcKind::CellArc : ArcKind::NetArc, owner[a]};
        g.out_arcs[static_cast<std::size_t>(from[a])].push_back(static_cast<int>(a));
        g.in_arcs[static_cast<std::size_t>(to[a])].push_back(static_cast<int>(a));
    }
    g.levels.assign(static_cast<std::size_t>(cnt[2]), {});
    for (std::size_t p = 0; p < nl.pins.size(); ++p) g.levels[static_cast<std::size_t>(g.level[p])].push_back(static_cast<int>(p));
    g.sources = nl.sources, g.endpoints = nl.endpoints;
    g.is_source.assign(nl.pins.size(), false);
    g.is_endpoint.assign(nl.pins.size(), false);
    for (int s : nl.sources) g.is_source[static_cast<std::size_t>(s)] = true;
    for (int e : nl.endpoints) g.is_endpoint[static_cast<std::size_t>(e)] = true;
    g.levelized = true;
    return g;
}

// ---- STA -------------------------------------------------------------------------------------------
double net_delay(const Point& a, const Point& b, double cap, const DesignConstraints& c)
{ // scalar convenience form of the device's net_delay (sta.cpp:10-14), same expression
    const double len = manhattan(a, b);
    return (c.r_unit * len) * (c.c_unit * len + cap);
}

double arc_delay(const Arc& arc, const Netlist& nl, const PinPositions& pos, const DesignConstraints& c)
{
    if (arc.kind == ArcKind::CellArc) return nl.cells[static_cast<std::size_t>(arc.owner)].delay;
    return net_delay(pos[static_cast<std::size_t>(arc.from)], pos[static_cast<std::size_t>(arc.to)],
                     nl.pins[static_cast<std::size_t>(arc.to)].load_cap, c);
}

std::vector<double> propagate_arrival(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                                      const DesignConstraints& c, std::vector<bool>* arr_known, int)
{
    auto S = sta_at(graph, nl, pos, c);
    TimingAnnotation a = fetch_annotation(S->s, nl);
    if (arr_known) *arr_known = a.arr_known;
    return a.arr;
}

std::vector<double> propagate_required(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                                       const DesignConstraints& c, std::vector<bool>* req_known, int)
{
    auto S = sta_at(graph, nl, pos, c);
    TimingAnnotation a = fetch_annotation(S->s, nl);
    if (req_known) *req_known = a.req_known;
    return a.req;
}

TimingAnnotation compute_slacks(const TimingGraph& graph, std::vector<double> arrivals, std::vector<double> required,
                                std::vector<bool> arr_known, std::vector<bool> req_known)
{ // glue over caller-supplied vectors (sta.cpp:104-120); the engine computes slacks on the device
    TimingAnnotation ann;
    ann.arr = std::move(arrivals), ann.req = std::move(required);
    ann.arr_known = std::move(arr_known), ann.req_known = std::move(req_known);
    ann.slack.resize(ann.arr.size());
    for (std::size_t p = 0; p < ann.arr.size(); ++p) ann.slack[p] = ann.req[p] - ann.arr[p];
    for (int e : graph.endpoints) ann.endpoint_slacks.emplace_back(e, ann.slack[static_cast<std::size_t>(e)]);
    std::tie(ann.tns, ann.wns) = tns_wns(ann.endpoint_slacks);
    return ann;
}

std::pair<double, double> tns_wns(const std::vector<std::pair<int, double>>& endpoint_slacks)
{
    double tns = 0.0, wns = 0.0;
    for (const auto& [pin, s] : endpoint_slacks)
        if (s < 0.0) {
            tns += s;
            if (s < wns) wns = s;
        }
    return {tns, wns};
}

TimingAnnotation run_sta(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                         const DesignConstraints& c, int)
{
    auto S = sta_at(graph, nl, pos, c);
    return fetch_annotation(S->s, nl);
}

// ---- paths -----------------------------------------------------------------------------------------
PathEnumerator::PathEnumerator(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                               const DesignConstraints& c)
    : graph_(graph), netlist_(nl), pos_(pos), constraints_(c)
{
}

const PathEnumerator::Record* PathEnumerator::path_to(int pin, std::size_t rank)
{
    const auto key = std::make_pair(pin, rank);
    if (auto it = found_.find(key); it != found_.end()) return &it->second;
    if (none_.count(key)) return nullptr;
    auto S = sta_at(graph_, netlist_, pos_, constraints_);
    std::vector<int32_t> buf(static_cast<std::size_t>(graph_.levels.size()) + 2);
    int32_t n = 0;
    double delay = 0.0;
    ck(tdpg_path_to(S->s, pin, static_cast<int32_t>(rank), buf.data(), static_cast<int32_t>(buf.size()), &n, &delay));
    if (n == 0) {
        none_[key] = true;
        return nullptr;
    }
    Record r;
    r.delay = delay;
    r.pins.assign(buf.begin(), buf.begin() + n);
    return &found_.emplace(key, std::move(r)).first->second;
}

std::vector<CriticalPath> k_worst_paths_to(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                                           const DesignConstraints& c, const TimingAnnotation&, int endpoint, int k)
{
    if (endpoint < 0 || endpoint >= graph.num_pins || !graph.is_endpoint[static_cast<std::size_t>(endpoint)])
        throw EndpointError("pin " + std::to_string(endpoint) + " is not an endpoint");
    std::vector<CriticalPath> out;
    if (k <= 0) return out;
    auto S = sta_at(graph, nl, pos, c);
    const std::size_t cap = static_cast<std::size_t>(k) * (graph.levels.size() + 2);
    std::vector<int32_t> start(static_cast<std::size_t>(k) + 1), pins(cap);
    std::vector<double> slack(static_cast<std::size_t>(k));
    int32_t np = 0;
    ck(tdpg_k_worst(S->s, endpoint, k, &np, start.data(), pins.data(), static_cast<int32_t>(cap), slack.data()));
    for (int i = 0; i < np; ++i)
        out.push_back(CriticalPath{std::vector<int>(pins.begin() + start[i], pins.begin() + start[i + 1]), slack[i]});
    return out;
}

namespace {
// report_timing (policy 1) / report_timing_endpoint (policy 0) through tdpg_extract.  The C-ABI's
// n <= 0 means "every violated endpoint"; the reference's own n <= 0 clips the selection to nothing
// (paths.cpp:147, :178), so that case never reaches the device.
ExtractionReport extract_report(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                                const DesignConstraints& c, const TimingAnnotation& ann, int n, int k, int policy)
{
    const auto t0 = std::chrono::steady_clock::now();
    ExtractionReport r;
    r.policy = policy ? "topn" : "endpoint", r.n = n, r.k = policy ? n : k;
    if (n <= 0) {
        if (policy) { // candidates_generated = violated.size() * n (paths.cpp:149)
            long long nv = 0;
            for (const auto& [pin, slack] : ann.endpoint_slacks) nv += slack < 0.0;
            r.candidates_generated = n < 0 ? nv * n : 0;
        }
        return r;
    }
    auto S = sta_at(graph, nl, pos, c);
    int64_t counts[5];
    ck(tdpg_extract(S->s, policy, n, k, counts));
    r = fetch_report(S->s, nl, n, policy ? n : k, counts, 0.0, policy ? "topn" : "endpoint");
    r.elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return r;
}
} // namespace

ExtractionReport report_timing(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                               const DesignConstraints& c, const TimingAnnotation& ann, int n, int)
{
    return extract_report(graph, nl, pos, c, ann, n, 1, 1);
}

ExtractionReport report_timing_endpoint(const TimingGraph& graph, const Netlist& nl, const PinPositions& pos,
                                        const DesignConstraints& c, const TimingAnnotation& ann, int n, int k, int)
{
    return extract_report(graph, nl, pos, c, ann, n, k, 0);
}

std::vector<PairHit> collect_pin_pairs(const Netlist& nl, const std::vector<CriticalPath>& paths)
{ // glue over caller-supplied paths (paths.cpp:191-203); the engine produces hits on the device
    std::vector<PairHit> hits;
    for (const auto& path : paths)
        for (std::size_t i = 0; i + 1 < path.pins.size(); ++i) {
            if (nl.pins[static_cast<std::size_t>(path.pins[i])].dir != PinDir::Output) continue;
            hits.push_back(PairHit{std::minmax(path.pins[i], path.pins[i + 1]), path.slack});
        }
    return hits;
}

// ---- pin pairs -------------------------------------------------------------------------------------
void update_pair_weights(PinPairWeights& weights, const std::vector<PairHit>& hits, double wns, double w0, double w1)
{
    if (!(wns < 0.0) || hits.empty()) return;
    int max_pin = 0;
    for (const auto& [pr, w] : weights) max_pin = std::max({max_pin, pr.first, pr.second});
    for (const auto& h : hits) max_pin = std::max({max_pin, h.pair.first, h.pair.second});
    std::size_t cap = 2; // (pin ids index the ledger only: a power-of-two capacity keeps one scratch session)
    while (cap < static_cast<std::size_t>(max_pin) + 1) cap *= 2;
    std::vector<Point> pts(cap);
    tdpg_session* S = scratch_session(std::span<const Point>(pts));
    ledger_upload(S, weights);
    std::vector<int32_t> a, b;
    std::vector<double> sl;
    for (const auto& h : hits) a.push_back(h.pair.first), b.push_back(h.pair.second), sl.push_back(h.path_slack);
    ck(tdpg_pp_update(S, static_cast<int64_t>(a.size()), a.data(), b.data(), sl.data(), wns, w0, w1));
    weights = ledger_download(S);
}

PinPairLossResult pin_pair_loss(const PinPairWeights& weights, const PinPositions& pins, std::size_t num_pins,
                                PairLossKind kind)
{
    PinPairLossResult out;
    out.d_pin.assign(num_pins, Point{});
    if (weights.empty() || pins.empty()) return out;
    tdpg_session* S = scratch_session(std::span<const Point>(pins.data(), pins.size()));
    ledger_upload(S, weights);
    std::vector<double> d(2 * pins.size());
    ck(tdpg_pp_loss(S, kind == PairLossKind::Linear ? 1 : 0, &out.value, d.data()));
    for (std::size_t p = 0; p < std::min(num_pins, pins.size()); ++p) out.d_pin[p] = Point{d[2 * p], d[2 * p + 1]};
    return out;
}

// ---- wirelength ------------------------------------------------------------------------------------
NetTermGrad wa_wirelength(std::span<const Point> pin_pos, double gamma)
{
    NetTermGrad out;
    out.d_pin.assign(pin_pos.size(), Point{});
    if (pin_pos.size() < 2) return out;
    tdpg_session* S = scratch_session(pin_pos);
    double wl = 0.0, hp = 0.0;
    std::vector<double> g(2 * pin_pos.size());
    ck(tdpg_wirelength(S, gamma, nullptr, &wl, &hp, g.data()));
    out.value = wl;
    for (std::size_t i = 0; i < pin_pos.size(); ++i) out.d_pin[i] = Point{g[2 * i], g[2 * i + 1]};
    return out;
}

double hpwl_net(std::span<const Point> pin_pos)
{
    if (pin_pos.size() < 2) return 0.0;
    tdpg_session* S = scratch_session(pin_pos);
    double h = 0.0;
    std::vector<double> xy(2 * pin_pos.size());
    for (std::size_t i = 0; i < pin_pos.size(); ++i) xy[2 * i] = pin_pos[i].x, xy[2 * i + 1] = pin_pos[i].y;
    ck(tdpg_hpwl_pins(S, xy.data(), &h));
    return h;
}

double hpwl_total(const Netlist& nl, const PinPositions& pos)
{
    auto S = session(nl, core_only({}));
    const auto xy = flat_points(pos);
    double h = 0.0;
    ck(tdpg_hpwl_pins(S->s, xy.data(), &h));
    return h;
}

// ---- density ----------------------------------------------------------------------------------------
DensityGrid::DensityGrid(const Netlist&, const Rect& core, int nx, int ny, double target_density)
    : core_(core), nx_(nx), ny_(ny), target_density_(target_density)
{
    if (nx < 1 || ny < 1) throw ValidationError("density grid must be at least 1x1");
}

DensityResult DensityGrid::evaluate(const Netlist& nl, const std::vector<Point>& cell_pos, int) const
{
    auto S = session(nl, core_only(core_));
    set_core(S->s, core_);
    const auto xy = flat_points(cell_pos);
    ck(tdpg_set_positions(S->s, xy.data()));
    ck(tdpg_set_grid(S->s, nx_, ny_, target_density_));
    DensityResult r;
    r.d_cell.resize(nl.cells.size());
    ck(tdpg_density(S->s, &r.value, &r.overflow, flat_out(r.d_cell)));
    return r;
}

// ---- placer -------------------------------------------------------------------------------------------
namespace {
std::string fmt17(double v)
{
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

tdpg_config to_c(const OptimizerConfig& c)
{
    tdpg_config k;
    tdpg_config_default(&k);
    k.gamma_frac = c.gamma_frac, k.grid_nx = c.grid_nx, k.grid_ny = c.grid_ny, k.target_density = c.target_density;
    k.beta = c.beta, k.pp_loss = c.pp_loss == PairLossKind::Linear, k.net_weighting = c.net_weighting, k.m = c.m;
    k.w0 = c.w0, k.w1 = c.w1, k.timing_start_iter = c.timing_start_iter;
    k.extraction = c.extraction == ExtractionPolicy::TopN, k.k = c.k, k.max_iters = c.max_iters;
    k.stop_overflow = c.stop_overflow, k.mu = c.mu, k.lambda0 = c.lambda0, k.lambda_max = c.lambda_max;
    k.step0_frac = c.step0_frac, k.step_decay = c.step_decay, k.adam_beta1 = c.adam_beta1;
    k.adam_beta2 = c.adam_beta2, k.adam_eps = c.adam_eps, k.seed = c.seed, k.init_jitter_frac = c.init_jitter_frac;
    k.threads = c.threads;
    return k;
}
} // namespace

std::string metrics_to_csv(const MetricTrace& trace)
{ // placer.cpp:234-260 format
    std::string out = "iter,hpwl,overflow,tns,wns,wl_term,density_term,pp_term,lambda,beta_pp\n";
    for (const TraceRow& r : trace) {
        out += std::to_string(r.iter) + ',' + fmt17(r.hpwl) + ',' + fmt17(r.overflow) + ',';
        if (r.has_timing) out += fmt17(r.tns);
        out += ',';
        if (r.has_timing) out += fmt17(r.wns);
        out += ',' + fmt17(r.wl_term) + ',' + fmt17(r.density_term) + ',' + fmt17(r.pp_term) + ',' + fmt17(r.lambda) +
               ',' + fmt17(r.beta_pp) + '\n';
    }
    return out;
}

std::string weights_to_json(const PinPairWeights& weights, const Netlist& nl)
{ // placer.cpp:486-499: {pairs:[{a,b,weight}]} with pin names, in pin-id order
    nlohmann::json arr = nlohmann::json::array();
    for (const auto& [pr, w] : weights) {
        nlohmann::json item;
        item["a"] = nl.pins[static_cast<std::size_t>(pr.first)].name;
        item["b"] = nl.pins[static_cast<std::size_t>(pr.second)].name;
        item["weight"] = w;
        arr.push_back(item);
    }
    nlohmann::json j;
    j["pairs"] = arr;
    return j.dump(2) + "\n";
}

// ---- configuration I/O (placer.cpp:22-232, the reference's rules and messages) -------------------------
namespace {
using nlohmann::json;

void reject_unknown_keys(const json& obj, std::initializer_list<const char*> allowed)
{
    for (auto it = obj.begin(); it != obj.end(); ++it)
        if (std::none_of(allowed.begin(), allowed.end(), [&](const char* k) { return it.key() == k; }))
            throw ParseError("config: unknown key \"" + it.key() + "\"");
}

template <typename T, typename Pred>
void get_field(const json& j, const char* key, T& out, Pred ok, const char* what)
{
    if (!j.contains(key)) return;
    if (!ok(j[key])) throw ParseError(std::string("config: \"") + key + "\" must be " + what);
    out = j[key].get<T>();
}

void require_positive(double v, const char* what)
{
    if (!(v > 0.0)) throw ValidationError(std::string("config: ") + what + " must be > 0");
}

void validate_config(const OptimizerConfig& c)
{ // placer.cpp:68-90
    if (c.grid_nx < 1 || c.grid_ny < 1) throw ValidationError("config: density grid must be at least 1x1");
    require_positive(c.target_density, "target_density");
    require_positive(c.gamma_frac, "gamma_frac");
    if (c.beta < 0.0) throw ValidationError("config: beta must be >= 0");
    if (c.m < 1) throw ValidationError("config: m must be >= 1");
    require_positive(c.w0, "w0");
    if (c.w1 < 0.0) throw ValidationError("config: w1 must be >= 0");
    if (c.timing_start_iter < 0) throw ValidationError("config: timing_start_iter must be >= 0");
    if (c.k < 1) throw ValidationError("config: k must be >= 1");
    if (c.max_iters < 0) throw ValidationError("config: max_iters must be >= 0");
    if (c.stop_overflow < 0.0) throw ValidationError("config: stop_overflow must be >= 0");
    require_positive(c.mu, "mu");
    require_positive(c.lambda_max, "lambda_max");
    require_positive(c.step0_frac, "step0_frac");
    if (!(c.step_decay > 0.0 && c.step_decay <= 1.0)) throw ValidationError("config: step_decay must be in (0, 1]");
    if (!(c.adam_beta1 >= 0.0 && c.adam_beta1 < 1.0) || !(c.adam_beta2 >= 0.0 && c.adam_beta2 < 1.0))
        throw ValidationError("config: adam betas must be in [0, 1)");
    require_positive(c.adam_eps, "adam_eps");
    if (c.init_jitter_frac < 0.0) throw ValidationError("config: init_jitter_frac must be >= 0");
    if (c.threads < 1) throw ValidationError("config: threads must be >= 1");
}
} // namespace

OptimizerConfig config_from_json(const std::string& text)
{
    json j;
    try {
        j = json::parse(text);
    } catch (const json::parse_error& e) {
        throw ParseError(std::string("config: ") + e.what());
    }
    if (!j.is_object()) throw ParseError("config: expected a JSON object");
    reject_unknown_keys(j, {"name", "gamma_frac", "grid_nx", "grid_ny", "target_density", "beta", "pp_loss",
                            "net_weighting", "m", "w0", "w1", "timing_start_iter", "extraction", "k", "max_iters",
                            "stop_overflow", "mu", "lambda0", "lambda_max", "step0_frac", "step_decay", "adam_beta1",
                            "adam_beta2", "adam_eps", "seed", "init_jitter_frac", "threads"});
    const auto num = [](const json& v) { return v.is_number(); };
    const auto integer = [](const json& v) { return v.is_number_integer(); };
    const auto boolean = [](const json& v) { return v.is_boolean(); };
    const auto str = [](const json& v) { return v.is_string(); };
    OptimizerConfig c;
    get_field(j, "name", c.name, str, "a string"); // (the reference's order: the first bad key is reported)
    get_field(j, "gamma_frac", c.gamma_frac, num, "a number");
    get_field(j, "grid_nx", c.grid_nx, integer, "an integer");
    get_field(j, "grid_ny", c.grid_ny, integer, "an integer");
    get_field(j, "target_density", c.target_density, num, "a number");
    get_field(j, "beta", c.beta, num, "a number");
    get_field(j, "mu", c.mu, num, "a number");
    get_field(j, "m", c.m, integer, "an integer");
    get_field(j, "w0", c.w0, num, "a number");
    get_field(j, "w1", c.w1, num, "a number");
    get_field(j, "timing_start_iter", c.timing_start_iter, integer, "an integer");
    get_field(j, "k", c.k, integer, "an integer");
    get_field(j, "max_iters", c.max_iters, integer, "an integer");
    get_field(j, "stop_overflow", c.stop_overflow, num, "a number");
    get_field(j, "lambda_max", c.lambda_max, num, "a number");
    get_field(j, "step0_frac", c.step0_frac, num, "a number");
    get_field(j, "step_decay", c.step_decay, num, "a number");
    get_field(j, "adam_beta1", c.adam_beta1, num, "a number");
    get_field(j, "adam_beta2", c.adam_beta2, num, "a number");
    get_field(j, "adam_eps", c.adam_eps, num, "a number");
    get_field(j, "init_jitter_frac", c.init_jitter_frac, num, "a number");
    get_field(j, "threads", c.threads, integer, "an integer");
    get_field(j, "net_weighting", c.net_weighting, boolean, "a boolean");
    if (j.contains("seed")) {
        if (!j["seed"].is_number_unsigned() && !j["seed"].is_number_integer())
            throw ParseError("config: \"seed\" must be an integer");
        c.seed = j["seed"].get<std::uint64_t>();
    }
    if (j.contains("pp_loss")) {
        std::string s;
        get_field(j, "pp_loss", s, str, "a string");
        if (s == "quadratic") c.pp_loss = PairLossKind::Quadratic;
        else if (s == "linear") c.pp_loss = PairLossKind::Linear;
        else throw ParseError("config: pp_loss must be \"quadratic\" or \"linear\"");
    }
    if (j.contains("extraction")) {
        std::string s;
        get_field(j, "extraction", s, str, "a string");
        if (s == "endpoint") c.extraction = ExtractionPolicy::Endpoint;
        else if (s == "topn") c.extraction = ExtractionPolicy::TopN;
        else throw ParseError("config: extraction must be \"endpoint\" or \"topn\"");
    }
    if (j.contains("lambda0")) {
        const char* msg = "config: lambda0 must be \"auto\" or a positive number";
        if (j["lambda0"].is_string()) {
            if (j["lambda0"].get<std::string>() != "auto") throw ParseError(msg);
            c.lambda0 = 0.0;
        } else if (j["lambda0"].is_number()) {
            c.lambda0 = j["lambda0"].get<double>();
            if (!(c.lambda0 > 0.0)) throw ParseError(msg);
        } else {
            throw ParseError(msg);
        }
    }
    validate_config(c);
    return c;
}

std::string config_to_json(const OptimizerConfig& c)
{
    json j;
    j["name"] = c.name;
    j["gamma_frac"] = c.gamma_frac;
    j["grid_nx"] = c.grid_nx;
    j["grid_ny"] = c.grid_ny;
    j["target_density"] = c.target_density;
    j["beta"] = c.beta;
    j["pp_loss"] = c.pp_loss == PairLossKind::Quadratic ? "quadratic" : "linear";
    j["net_weighting"] = c.net_weighting;
    j["m"] = c.m;
    j["w0"] = c.w0;
    j["w1"] = c.w1;
    j["timing_start_iter"] = c.timing_start_iter;
    j["extraction"] = c.extraction == ExtractionPolicy::Endpoint ? "endpoint" : "topn";
    j["k"] = c.k;
    j["max_iters"] = c.max_iters;
    j["stop_overflow"] = c.stop_overflow;
    j["mu"] = c.mu;
    if (c.lambda0 > 0.0) j["lambda0"] = c.lambda0;
    else j["lambda0"] = "auto";
    j["lambda_max"] = c.lambda_max;
    j["step0_frac"] = c.step0_frac;
    j["step_decay"] = c.step_decay;
    j["adam_beta1"] = c.adam_beta1;
    j["adam_beta2"] = c.adam_beta2;
    j["adam_eps"] = c.adam_eps;
    j["seed"] = c.seed;
    j["init_jitter_frac"] = c.init_jitter_frac;
    j["threads"] = c.threads;
    return j.dump(2) + "\n";
}

OptimizerConfig load_config(const std::string& path)
{
    std::ifstream in(path);
    if (!in) throw ParseError("cannot open config file: " + path);
    std::stringstream ss;
    ss << in.rdbuf();
    return config_from_json(ss.str());
}

void save_config(const OptimizerConfig& config, const std::string& path)
{
    std::ofstream out(path);
    if (!out) throw ParseError("cannot write config file: " + path);
    out << config_to_json(config);
}

ObjectiveResult objective_and_gradient(const Netlist& nl, const std::vector<Point>& cell_pos, const DensityGrid& grid,
                                       const PinPairWeights& weights, const std::vector<double>& net_weights,
                                       double gamma, double lambda, double beta, PairLossKind kind, int)
{
    if (!net_weights.empty() && net_weights.size() != nl.nets.size())
        throw ValidationError("net weight count does not match net count");
    auto S = session(nl, core_only(grid.core()));
    set_core(S->s, grid.core());
    if (cell_pos.size() != nl.cells.size()) throw ValidationError("cell position count does not match cell count");
    // Point is two packed doubles: the positions go to the device and the gradient comes back in place,
    // with no intermediate copies (the per-iteration host cost of a reference-style loop)
    static_assert(sizeof(Point) == 2 * sizeof(double), "Point must be two packed doubles");
    ck(tdpg_set_positions(S->s, reinterpret_cast<const double*>(cell_pos.data())));
    ck(tdpg_set_grid(S->s, grid.nx(), grid.ny(), grid.target_density()));
    ledger_upload(S->s, weights);
    double terms[6];
    ObjectiveResult r;
    r.d_cell.resize(nl.cells.size());
    ck(tdpg_objective(S->s, gamma, lambda, beta, kind == PairLossKind::Linear ? 1 : 0,
                      net_weights.empty() ? nullptr : net_weights.data(), terms,
                      reinterpret_cast<double*>(r.d_cell.data())));
    r.value = terms[0], r.wl_term = terms[1], r.density_term = terms[2], r.pp_term = terms[3], r.hpwl = terms[4];
    r.overflow = terms[5];
    return r;
}

std::vector<double> apply_net_weights(const TimingAnnotation& ann, const Netlist& nl)
{ // glue over a caller-supplied annotation (placer.cpp:262-273); the engine applies it on the device
    std::vector<double> w(nl.nets.size(), 1.0);
    if (ann.wns >= 0.0) return w;
    for (std::size_t e = 0; e < nl.nets.size(); ++e) {
        double worst = ann.slack[static_cast<std::size_t>(nl.nets[e].driver)];
        for (int s : nl.nets[e].sinks) worst = std::min(worst, ann.slack[static_cast<std::size_t>(s)]);
        if (worst < 0.0) w[e] = 1.0 + (-worst) / (-ann.wns);
    }
    return w;
}

void AdamState::step(std::vector<double>& x, const std::vector<double>& grad, double lr, double beta1, double beta2,
                     double eps)
{
    int32_t tt = t;
    ck(tdpg_adam_step(static_cast<int64_t>(x.size()), x.data(), grad.data(), m.data(), v.data(), &tt, lr, beta1, beta2,
                      eps));
    t = tt;
}

namespace {
struct ObserverCtx {
    tdpg_session* s;
    const Netlist* nl;
    const TimingRoundObserver* obs;
    int policy, k;
};

void observer_trampoline(void* user, int32_t iter)
{
    auto* c = static_cast<ObserverCtx*>(user);
    const TimingAnnotation ann = fetch_annotation(c->s, *c->nl);
    int64_t counts[5];
    ck(tdpg_paths_counts(c->s, counts));
    ck(tdpg_paths_candidates(c->s, &counts[4]));
    long long n_fail = 0; // the round extracts for n = n_fail (placer.cpp:424-429)
    for (const auto& [pin, slack] : ann.endpoint_slacks) n_fail += slack < 0.0;
    const int n = static_cast<int>(n_fail);
    ExtractionReport r = fetch_report(c->s, *c->nl, n, c->policy ? n : c->k, counts, 0.0,
                                      c->policy ? "topn" : "endpoint");
    if (ann.wns >= 0.0) r = ExtractionReport{}; // the round was skipped (placer.cpp:422-432)
    (*c->obs)(iter, ann, r);
}
} // namespace

namespace {
PlacementOutcome place_on(const std::shared_ptr<Sess>& S, const Design& design, const OptimizerConfig& config,
                          const TimingRoundObserver& observer, double* final_hpwl);
} // namespace

PlacementOutcome run_placement(const Design& design, const OptimizerConfig& config, const TimingRoundObserver& observer)
{
    return place_on(session(design.netlist, design.constraints), design, config, observer, nullptr);
}

namespace {
PlacementOutcome place_on(const std::shared_ptr<Sess>& S, const Design& design, const OptimizerConfig& config,
                          const TimingRoundObserver& observer, double* final_hpwl)
{
    const Netlist& nl = design.netlist;
    set_core(S->s, design.constraints.core);
    const auto xy = flat_points(design.positions);
    ck(tdpg_set_positions(S->s, xy.data()));
    std::vector<uint8_t> expl(design.pos_explicit.begin(), design.pos_explicit.end());
    expl.resize(nl.cells.size(), 0);
    const tdpg_config cfg = to_c(config);
    std::vector<tdpg_trace_row> rows(static_cast<std::size_t>(std::max(config.max_iters, 1)));
    int32_t n_rows = 0, stop = 0;
    double fin[3];
    ObserverCtx ctx{S->s, &nl, &observer, cfg.extraction, cfg.k};
    ck(tdpg_set_round_callback(S->s, observer ? observer_trampoline : nullptr, &ctx));
    const int rc = tdpg_place(S->s, &cfg, expl.data(), rows.data(), &n_rows, &stop, fin);
    tdpg_set_round_callback(S->s, nullptr, nullptr);
    ck(rc);
    PlacementOutcome out;
    out.positions.resize(nl.cells.size());
    ck(tdpg_get_positions(S->s, flat_out(out.positions)));
    for (int i = 0; i < n_rows; ++i) {
        const tdpg_trace_row& r = rows[static_cast<std::size_t>(i)];
        TraceRow t;
        t.iter = r.iter, t.hpwl = r.hpwl, t.overflow = r.overflow, t.has_timing = r.has_timing != 0, t.tns = r.tns;
        t.wns = r.wns, t.wl_term = r.wl_term, t.density_term = r.density_term, t.pp_term = r.pp_term;
        t.lambda = r.lambda, t.beta_pp = r.beta_pp;
        out.trace.push_back(t);
    }
    out.pair_weights = ledger_download(S->s);
    out.final_timing = fetch_annotation(S->s, nl); // tdpg_place ran STA at the returned positions
    out.iterations = n_rows;
    out.stop_reason = stop ? "overflow" : "max_iters";
    if (final_hpwl) *final_hpwl = fin[2];
    return out;
}

std::string fmt_g(double v, const char* spec)
{
    char buf[64];
    std::snprintf(buf, sizeof buf, spec, v);
    return buf;
}

std::string csv_escape(const std::string& s)
{
    if (s.find_first_of(",\"\n") == std::string::npos) return s;
    std::string out = "\"";
    for (char c : s) {
        if (c == '"') out += "\"\"";
        else out += c;
    }
    return out + "\"";
}
} // namespace

// run_compare (compare.cpp:37-95): coverage columns on one frozen snapshot, then every configuration in
// full; with `parallel` the full runs execute concurrently on private device sessions (own streams).
CompareReport run_compare(const Design& design, const std::vector<OptimizerConfig>& configs, bool parallel)
{
    if (configs.size() < 2) throw ValidationError("compare: need >= 2 configurations");
    for (const OptimizerConfig& c : configs)
        if (c.seed != configs.front().seed)
            throw ValidationError("compare: all configurations must share one seed (config \"" + c.name +
                                  "\" differs)");
    CompareReport report;
    report.rows.resize(configs.size());
    OptimizerConfig snap_cfg = configs.front();
    snap_cfg.beta = 0.0;
    snap_cfg.net_weighting = false;
    snap_cfg.max_iters = std::min(snap_cfg.max_iters, snap_cfg.timing_start_iter);
    snap_cfg.timing_start_iter = snap_cfg.max_iters + 1;
    snap_cfg.stop_overflow = 0.0;
    const PlacementOutcome snapshot = run_placement(design, snap_cfg);
    const TimingGraph graph = build_timing_graph(design.netlist);
    const PinPositions snap_pins = pin_positions(design.netlist, snapshot.positions);
    const TimingAnnotation snap_ann = run_sta(graph, design.netlist, snap_pins, design.constraints);
    int n_fail = 0;
    for (const auto& [pin, slack] : snap_ann.endpoint_slacks) n_fail += slack < 0.0;
    for (std::size_t i = 0; i < configs.size(); ++i) { // coverage (serial: the cached session)
        CompareRow& row = report.rows[i];
        row.config_name = configs[i].name;
        if (n_fail <= 0) continue;
        try {
            const ExtractionReport ext =
                configs[i].extraction == ExtractionPolicy::Endpoint
                    ? report_timing_endpoint(graph, design.netlist, snap_pins, design.constraints, snap_ann, n_fail,
                                             configs[i].k)
                    : report_timing(graph, design.netlist, snap_pins, design.constraints, snap_ann, n_fail);
            row.unique_endpoints = ext.unique_endpoints;
            row.unique_pin_pairs = ext.unique_pin_pairs;
            row.candidates_generated = ext.candidates_generated;
        } catch (const std::exception& e) {
            row.error = e.what();
        }
    }
    auto run = [&](std::size_t i, bool priv) {
        CompareRow& row = report.rows[i];
        if (!row.error.empty()) return;
        try {
            const auto t0 = std::chrono::steady_clock::now();
            double h = 0.0;
            const auto S = priv ? fresh_session(design.netlist, design.constraints)
                                : session(design.netlist, design.constraints);
            const PlacementOutcome outcome = place_on(S, design, configs[i], {}, &h);
            row.runtime_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            row.tns = outcome.final_timing.tns;
            row.wns = outcome.final_timing.wns;
            row.hpwl = h; // hpwl_total at the final positions (tdpg_place)
            row.ok = true;
        } catch (const std::exception& e) {
            row.ok = false;
            row.error = e.what();
        }
    };
    if (parallel) {
        std::vector<std::thread> ts;
        for (std::size_t i = 0; i < configs.size(); ++i) ts.emplace_back(run, i, true);
        for (auto& t : ts) t.join();
    } else {
        for (std::size_t i = 0; i < configs.size(); ++i) run(i, false);
    }
    return report;
}

std::string compare_to_csv(const CompareReport& report)
{ // compare.cpp:97-122
    std::string out = "config,status,tns,wns,hpwl,runtime_s,unique_endpoints,unique_pin_pairs,candidates_generated\n";
    for (const CompareRow& r : report.rows) {
        out += csv_escape(r.config_name) + ',' + (r.ok ? std::string("ok") : csv_escape(r.error)) + ',';
        out += fmt_g(r.tns, "%.17g") + ',' + fmt_g(r.wns, "%.17g") + ',' + fmt_g(r.hpwl, "%.17g") + ',';
        out += fmt_g(r.runtime_s, "%.3f") + ',' + std::to_string(r.unique_endpoints) + ',';
        out += std::to_string(r.unique_pin_pairs) + ',' + std::to_string(r.candidates_generated) + '\n';
    }
    return out;
}

std::string compare_to_table(const CompareReport& report)
{ // compare.cpp:124-150
    std::string out;
    char line[256];
    std::snprintf(line, sizeof line, "%-24s %-6s %14s %12s %14s %10s %8s %8s %12s\n", "config", "status", "tns",
                  "wns", "hpwl", "runtime_s", "uniq_ep", "uniq_pp", "candidates");
    out += line;
    out += std::string(24 + 1 + 6 + 1 + 14 + 1 + 12 + 1 + 14 + 1 + 10 + 1 + 8 + 1 + 8 + 1 + 12, '-') + '\n';
    for (const CompareRow& r : report.rows) {
        if (r.ok)
            std::snprintf(line, sizeof line, "%-24s %-6s %14.4f %12.4f %14.2f %10.2f %8d %8d %12lld\n",
                          r.config_name.c_str(), "ok", r.tns, r.wns, r.hpwl, r.runtime_s, r.unique_endpoints,
                          r.unique_pin_pairs, r.candidates_generated);
        else
            std::snprintf(line, sizeof line, "%-24s %-6s %s\n", r.config_name.c_str(), "error", r.error.c_str());
        out += line;
    }
    return out;
}

} // namespace tdp
