// ref_harness.cpp — TEST INFRASTRUCTURE ONLY (checker + CPU baseline).
//
// A thin extern "C" shim over the reference's own, unmodified sources
// (/root/reference/proj/src/*.cpp, compiled from where they lie by
// oracle/Makefile into oracle/_ref/libtdpref.so).  It converts the flat
// tdpg_netlist view (include/tdpg.h) into a tdp::Design and calls the
// reference functions directly, so the tests and bench.py's CPU baseline
// can run the reference itself on exactly the inputs the GPU engine sees.
// Nothing in the product links or loads this file.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <random>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "tdp/compare.hpp"
#include "tdp/density.hpp"
#include "tdp/design_io.hpp"
#include "tdp/errors.hpp"
#include "tdp/generator.hpp"
#include "tdp/netlist.hpp"
#include "tdp/paths.hpp"
#include "tdp/pin_pairs.hpp"
#include "tdp/placer.hpp"
#include "tdp/rng.hpp"
#include "tdp/sta.hpp"
#include "tdp/timing_graph.hpp"
#include "tdp/wirelength.hpp"
#include "tdpg.h"
#include "fixtures.hpp" // the reference's own test fixtures (proj/tests/fixtures.hpp)

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

template <typename F>
int guard(F&& f)
{
    try {
        f();
        return 0;
    } catch (const tdp::CycleError& e) {
        g_err = e.what(), g_kind = TDPG_ERR_CYCLE;
    } catch (const tdp::EndpointError& e) {
        g_err = e.what(), g_kind = TDPG_ERR_ENDPOINT;
    } catch (const tdp::ValidationError& e) {
        g_err = e.what(), g_kind = TDPG_ERR_VALIDATION;
    } catch (const tdp::ParseError& e) {
        g_err = e.what(), g_kind = TDPG_ERR_PARSE;
    } catch (const tdp::GraphError& e) {
        g_err = e.what(), g_kind = TDPG_ERR_GRAPH;
    } catch (const tdp::NonFiniteError& e) {
        g_err = e.what(), g_kind = TDPG_ERR_NONFINITE;
    } catch (const std::exception& e) {
        g_err = e.what(), g_kind = TDPG_ERR_INTERNAL;
    }
    return g_kind;
}

struct RefSession {
    tdp::Design design;
    std::unique_ptr<tdp::TimingGraph> graph;
    tdp::ExtractionReport report;
    std::vector<tdp::PairHit> hits;
    tdp::PinPairWeights ledger;
    tdp::PlacementOutcome outcome;
    std::string csv;
    std::string json;

    const tdp::TimingGraph& g()
    {
        if (!graph) graph = std::make_unique<tdp::TimingGraph>(tdp::build_timing_graph(design.netlist));
        return *graph;
    }
};

std::vector<tdp::Point> to_points(const double* xy, std::size_t n)
{
    std::vector<tdp::Point> p(n);
    for (std::size_t i = 0; i < n; ++i) p[i] = tdp::Point{xy[2 * i], xy[2 * i + 1]};
    return p;
}

void from_points(const std::vector<tdp::Point>& p, double* xy)
{
    for (std::size_t i = 0; i < p.size(); ++i) xy[2 * i] = p[i].x, xy[2 * i + 1] = p[i].y;
}

tdp::Design to_design(const tdpg_netlist* d, const double* xy, const uint8_t* pos_explicit)
{
    tdp::Design out;
    tdp::Netlist& nl = out.netlist;
    nl.cells.resize(static_cast<std::size_t>(d->n_cells));
    for (int c = 0; c < d->n_cells; ++c) {
        tdp::Cell& cell = nl.cells[static_cast<std::size_t>(c)];
        cell.name = "c" + std::to_string(c);
        cell.width = d->cell_w[c];
        cell.height = d->cell_h[c];
        cell.delay = d->cell_delay[c];
        cell.is_fixed = d->cell_fixed[c] != 0;
    }
    nl.pins.resize(static_cast<std::size_t>(d->n_pins));
    for (int p = 0; p < d->n_pins; ++p) {
        tdp::Pin& pin = nl.pins[static_cast<std::size_t>(p)];
        pin.name = "p" + std::to_string(p);
        pin.cell = d->pin_cell[p];
        pin.terminal_pos = tdp::Point{d->pin_term[2 * p], d->pin_term[2 * p + 1]};
        pin.offset = tdp::Point{d->pin_off[2 * p], d->pin_off[2 * p + 1]};
        pin.dir = d->pin_dir[p] ? tdp::PinDir::Output : tdp::PinDir::Input;
        pin.load_cap = d->pin_cap[p];
    }
    nl.nets.resize(static_cast<std::size_t>(d->n_nets));
    for (int n = 0; n < d->n_nets; ++n) {
        tdp::Net& net = nl.nets[static_cast<std::size_t>(n)];
        net.name = "n" + std::to_string(n);
        net.driver = d->net_pins[d->net_start[n]];
        for (int e = d->net_start[n] + 1; e < d->net_start[n + 1]; ++e) net.sinks.push_back(d->net_pins[e]);
    }
    nl.sources.assign(d->sources, d->sources + d->n_sources);
    nl.endpoints.assign(d->endpoints, d->endpoints + d->n_endpoints);
    out.constraints.clock_period = d->clock_period;
    out.constraints.r_unit = d->r_unit;
    out.constraints.c_unit = d->c_unit;
    out.constraints.core = tdp::Rect{d->core[0], d->core[1], d->core[2], d->core[3]};
    out.positions = to_points(xy, static_cast<std::size_t>(d->n_cells));
    out.pos_explicit.resize(static_cast<std::size_t>(d->n_cells));
    for (int c = 0; c < d->n_cells; ++c) out.pos_explicit[static_cast<std::size_t>(c)] = pos_explicit ? pos_explicit[c] != 0 : true;
    nl.finalize();
    return out;
}

tdp::PinPairWeights to_ledger(int64_t q, const int32_t* a, const int32_t* b, const double* w)
{
    tdp::PinPairWeights out;
    for (int64_t i = 0; i < q; ++i) out[{a[i], b[i]}] = w[i];
    return out;
}

double ms_since(std::chrono::steady_clock::time_point t0)
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_last_error_kind(void) { return g_kind; }

int ref_create(const tdpg_netlist* d, const double* xy, const uint8_t* pos_explicit, void** out)
{
    return guard([&] {
        auto s = std::make_unique<RefSession>();
        s->design = to_design(d, xy, pos_explicit);
        *out = s.release();
    });
}

int ref_validate(void* h) { return guard([&] { tdp::validate_design(static_cast<RefSession*>(h)->design); }); }

void ref_destroy(void* h) { delete static_cast<RefSession*>(h); }

int ref_set_positions(void* h, const double* xy)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        s->design.positions = to_points(xy, s->design.netlist.cells.size());
    });
}

int ref_graph(void* h, int32_t counts[4], int32_t* level, int32_t* arc_from, int32_t* arc_to, int32_t* arc_kind,
              int32_t* arc_owner)
{
    return guard([&] {
        const tdp::TimingGraph& g = static_cast<RefSession*>(h)->g();
        counts[0] = g.num_net_arcs;
        counts[1] = g.num_cell_arcs;
        counts[2] = static_cast<int32_t>(g.levels.size());
        counts[3] = static_cast<int32_t>(g.levels.size()) - 1;
        if (level)
            for (std::size_t p = 0; p < g.level.size(); ++p) level[p] = g.level[p];
        for (std::size_t a = 0; a < g.arcs.size(); ++a) {
            if (arc_from) arc_from[a] = g.arcs[a].from;
            if (arc_to) arc_to[a] = g.arcs[a].to;
            if (arc_kind) arc_kind[a] = g.arcs[a].kind == tdp::ArcKind::CellArc ? 1 : 0;
            if (arc_owner) arc_owner[a] = g.arcs[a].owner;
        }
    });
}

int ref_pin_positions(void* h, double* pin_xy)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        from_points(tdp::pin_positions(s->design.netlist, s->design.positions), pin_xy);
    });
}

int ref_sta(void* h, int threads, double* arr, double* req, double* slack, uint8_t* ak, uint8_t* rk, double* tns,
            double* wns, double* elapsed_ms)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        const tdp::TimingGraph& g = s->g();
        const auto pos = tdp::pin_positions(s->design.netlist, s->design.positions);
        const auto t0 = std::chrono::steady_clock::now();
        const tdp::TimingAnnotation ann = tdp::run_sta(g, s->design.netlist, pos, s->design.constraints, threads);
        if (elapsed_ms) *elapsed_ms = ms_since(t0);
        const std::size_t n = ann.arr.size();
        for (std::size_t p = 0; p < n; ++p) {
            if (arr) arr[p] = ann.arr[p];
            if (req) req[p] = ann.req[p];
            if (slack) slack[p] = ann.slack[p];
            if (ak) ak[p] = ann.arr_known[p] ? 1 : 0;
            if (rk) rk[p] = ann.req_known[p] ? 1 : 0;
        }
        if (tns) *tns = ann.tns;
        if (wns) *wns = ann.wns;
    });
}

// policy 0 = endpoint(n, k), 1 = topn(n).  n <= 0 selects every violated endpoint.
// counts = n_paths, total_pins, unique_endpoints, unique_pin_pairs, candidates_generated.
int ref_extract(void* h, int policy, int n, int k, int threads, int64_t counts[5], double* sta_ms,
                double* extract_ms)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        const tdp::TimingGraph& g = s->g();
        const auto pos = tdp::pin_positions(s->design.netlist, s->design.positions);
        auto t0 = std::chrono::steady_clock::now();
        const tdp::TimingAnnotation ann = tdp::run_sta(g, s->design.netlist, pos, s->design.constraints, threads);
        if (sta_ms) *sta_ms = ms_since(t0);
        if (n <= 0) {
            n = 0;
            for (const auto& [pin, slack] : ann.endpoint_slacks)
                if (slack < 0.0) ++n;
        }
        t0 = std::chrono::steady_clock::now();
        if (policy == 0)
            s->report = tdp::report_timing_endpoint(g, s->design.netlist, pos, s->design.constraints, ann, n, k, threads);
        else
            s->report = tdp::report_timing(g, s->design.netlist, pos, s->design.constraints, ann, n, threads);
        if (extract_ms) *extract_ms = ms_since(t0);
        s->hits = tdp::collect_pin_pairs(s->design.netlist, s->report.paths);
        int64_t total = 0;
        for (const auto& p : s->report.paths) total += static_cast<int64_t>(p.pins.size());
        counts[0] = static_cast<int64_t>(s->report.paths.size());
        counts[1] = total;
        counts[2] = s->report.unique_endpoints;
        counts[3] = s->report.unique_pin_pairs;
        counts[4] = s->report.candidates_generated;
    });
}

int ref_paths_get(void* h, int32_t* start, int32_t* pins, double* slack, int64_t* n_hits)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        int32_t off = 0;
        for (std::size_t i = 0; i < s->report.paths.size(); ++i) {
            const auto& p = s->report.paths[i];
            if (start) start[i] = off;
            if (pins) std::memcpy(pins + off, p.pins.data(), p.pins.size() * sizeof(int32_t));
            if (slack) slack[i] = p.slack;
            off += static_cast<int32_t>(p.pins.size());
        }
        if (start) start[s->report.paths.size()] = off;
        if (n_hits) *n_hits = static_cast<int64_t>(s->hits.size());
    });
}

int ref_hits_get(void* h, int32_t* a, int32_t* b, double* slack)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        for (std::size_t i = 0; i < s->hits.size(); ++i) {
            a[i] = s->hits[i].pair.first;
            b[i] = s->hits[i].pair.second;
            slack[i] = s->hits[i].path_slack;
        }
    });
}

int ref_k_worst(void* h, int endpoint, int k, int32_t* n_paths, int32_t* start, int32_t* pins, double* slack,
                int32_t cap_pins)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        const tdp::TimingGraph& g = s->g();
        const auto pos = tdp::pin_positions(s->design.netlist, s->design.positions);
        const tdp::TimingAnnotation ann = tdp::run_sta(g, s->design.netlist, pos, s->design.constraints);
        const auto paths = tdp::k_worst_paths_to(g, s->design.netlist, pos, s->design.constraints, ann, endpoint, k);
        *n_paths = static_cast<int32_t>(paths.size());
        int32_t off = 0;
        for (std::size_t i = 0; i < paths.size(); ++i) {
            start[i] = off;
            for (int p : paths[i].pins)
                if (off < cap_pins) pins[off++] = p;
            slack[i] = paths[i].slack;
        }
        start[paths.size()] = off;
    });
}

int ref_wa(int n, const double* xy, double gamma, double* value, double* grad)
{
    return guard([&] {
        const auto pts = to_points(xy, static_cast<std::size_t>(n));
        const tdp::NetTermGrad r = tdp::wa_wirelength(pts, gamma);
        *value = r.value;
        from_points(r.d_pin, grad);
    });
}

int ref_hpwl(void* h, double* out)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        *out = tdp::hpwl_total(s->design.netlist, tdp::pin_positions(s->design.netlist, s->design.positions));
    });
}

int ref_density(void* h, int nx, int ny, double td, int threads, double* value, double* overflow, double* d_cell,
                double* elapsed_ms)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        const tdp::DensityGrid grid(s->design.netlist, s->design.constraints.core, nx, ny, td);
        const auto t0 = std::chrono::steady_clock::now();
        const tdp::DensityResult r = grid.evaluate(s->design.netlist, s->design.positions, threads);
        if (elapsed_ms) *elapsed_ms = ms_since(t0);
        *value = r.value;
        *overflow = r.overflow;
        if (d_cell) from_points(r.d_cell, d_cell);
    });
}

int ref_pp_loss(int64_t q, const int32_t* a, const int32_t* b, const double* w, int64_t n_pins, const double* pin_xy,
                int kind, double* value, double* d_pin)
{
    return guard([&] {
        const auto ledger = to_ledger(q, a, b, w);
        const auto pos = to_points(pin_xy, static_cast<std::size_t>(n_pins));
        const tdp::PinPairLossResult r = tdp::pin_pair_loss(
            ledger, pos, static_cast<std::size_t>(n_pins), kind ? tdp::PairLossKind::Linear : tdp::PairLossKind::Quadratic);
        *value = r.value;
        from_points(r.d_pin, d_pin);
    });
}

// Ledger update held in the session: set, update, then fetch size + arrays.
int ref_pp_update(void* h, int64_t q, const int32_t* a, const int32_t* b, const double* w, int64_t n_hits,
                  const int32_t* ha, const int32_t* hb, const double* hs, double wns, double w0, double w1, int64_t* q_out)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        s->ledger = to_ledger(q, a, b, w);
        std::vector<tdp::PairHit> hits(static_cast<std::size_t>(n_hits));
        for (int64_t i = 0; i < n_hits; ++i) hits[static_cast<std::size_t>(i)] = tdp::PairHit{{ha[i], hb[i]}, hs[i]};
        tdp::update_pair_weights(s->ledger, hits, wns, w0, w1);
        *q_out = static_cast<int64_t>(s->ledger.size());
    });
}

int ref_pp_ledger_get(void* h, int32_t* a, int32_t* b, double* w)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        std::size_t i = 0;
        for (const auto& [pair, weight] : s->ledger) {
            a[i] = pair.first;
            b[i] = pair.second;
            w[i] = weight;
            ++i;
        }
    });
}

// terms = value, wl, density, pp, hpwl, overflow
int ref_objective(void* h, int nx, int ny, double td, double gamma, double lambda, double beta, int kind,
                  const double* net_w, int64_t q, const int32_t* a, const int32_t* b, const double* w, int threads,
                  double terms[6], double* d_cell, double* elapsed_ms)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        const tdp::DensityGrid grid(s->design.netlist, s->design.constraints.core, nx, ny, td);
        const auto ledger = to_ledger(q, a, b, w);
        std::vector<double> nw;
        if (net_w) nw.assign(net_w, net_w + s->design.netlist.nets.size());
        const auto t0 = std::chrono::steady_clock::now();
        const tdp::ObjectiveResult r = tdp::objective_and_gradient(
            s->design.netlist, s->design.positions, grid, ledger, nw, gamma, lambda, beta,
            kind ? tdp::PairLossKind::Linear : tdp::PairLossKind::Quadratic, threads);
        if (elapsed_ms) *elapsed_ms = ms_since(t0);
        terms[0] = r.value;
        terms[1] = r.wl_term;
        terms[2] = r.density_term;
        terms[3] = r.pp_term;
        terms[4] = r.hpwl;
        terms[5] = r.overflow;
        if (d_cell) from_points(r.d_cell, d_cell);
    });
}

int ref_adam_step(int64_t n, double* x, const double* g, double* m, double* v, int32_t* t, double lr, double b1,
                  double b2, double eps)
{
    return guard([&] {
        tdp::AdamState st(static_cast<std::size_t>(n));
        st.m.assign(m, m + n);
        st.v.assign(v, v + n);
        st.t = *t;
        std::vector<double> xv(x, x + n), gv(g, g + n);
        st.step(xv, gv, lr, b1, b2, eps);
        std::memcpy(x, xv.data(), static_cast<std::size_t>(n) * sizeof(double));
        std::memcpy(m, st.m.data(), static_cast<std::size_t>(n) * sizeof(double));
        std::memcpy(v, st.v.data(), static_cast<std::size_t>(n) * sizeof(double));
        *t = st.t;
    });
}

// run_placement with a JSON config (config_from_json semantics).  Results are held
// in the session: final positions via ref_get_positions, metrics CSV via ref_text.
int ref_place(void* h, const char* config_json, double final_[3], int32_t* iterations, int32_t* stop_overflow,
              int64_t* n_pairs, double* elapsed_ms)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        const tdp::OptimizerConfig cfg =
            (config_json && *config_json) ? tdp::config_from_json(config_json) : tdp::OptimizerConfig{};
        const auto t0 = std::chrono::steady_clock::now();
        s->outcome = tdp::run_placement(s->design, cfg);
        if (elapsed_ms) *elapsed_ms = ms_since(t0);
        final_[0] = s->outcome.final_timing.tns;
        final_[1] = s->outcome.final_timing.wns;
        final_[2] = tdp::hpwl_total(s->design.netlist, tdp::pin_positions(s->design.netlist, s->outcome.positions));
        *iterations = s->outcome.iterations;
        *stop_overflow = s->outcome.stop_reason == "overflow" ? 1 : 0;
        s->ledger = s->outcome.pair_weights;
        *n_pairs = static_cast<int64_t>(s->ledger.size());
        s->csv = tdp::metrics_to_csv(s->outcome.trace);
    });
}

// bench.py's reference arm: run_placement's loop (placer.cpp:358-484) driven through the reference's
// own public functions — objective_and_gradient, AdamState::step, run_sta, report_timing_endpoint /
// report_timing, collect_pin_pairs, update_pair_weights, apply_net_weights — with a thread count per
// phase (the reference's STA / objective are fastest at nproc threads, its extraction at one
// thread, where the enumerator memoises prefixes).  Every loop step is the reference's, in its order;
// only the per-phase `threads` argument differs from run_placement(cfg.threads).  Per iteration: wall ms
// (refresh included), refresh ms and extracted paths (0 on non-timing iterations).
int ref_place_bench(void* h, const char* config_json, int threads_obj, int threads_sta, int threads_ex,
                    double* iter_ms, double* refresh_ms, int64_t* paths, int64_t* pairs_end, double final_[3],
                    int32_t* n_rows, tdpg_trace_row* trace)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        const tdp::OptimizerConfig config =
            (config_json && *config_json) ? tdp::config_from_json(config_json) : tdp::OptimizerConfig{};
        const tdp::Design& design = s->design;
        const tdp::Netlist& nl = design.netlist;
        const tdp::DesignConstraints& dc = design.constraints;
        const tdp::TimingGraph& graph = s->g();
        std::vector<tdp::Point> pos = design.positions;
        auto clamp = [&](tdp::Point& p, const tdp::Cell& cell) { // clamp_to_core (placer.cpp:99-103)
            p.x = std::clamp(p.x, dc.core.x_lo, dc.core.x_hi - cell.width);
            p.y = std::clamp(p.y, dc.core.y_lo, dc.core.y_hi - cell.height);
        };
        const double span = dc.core.span();
        const double gamma = config.gamma_frac * span;
        std::mt19937_64 rng(config.seed); // placer.cpp:375-382
        for (std::size_t c = 0; c < nl.cells.size(); ++c) {
            const tdp::Cell& cell = nl.cells[c];
            if (cell.is_fixed || design.pos_explicit[c]) continue;
            pos[c].x += tdp::rng_uniform(rng, -1.0, 1.0) * config.init_jitter_frac * dc.core.width();
            pos[c].y += tdp::rng_uniform(rng, -1.0, 1.0) * config.init_jitter_frac * dc.core.height();
            clamp(pos[c], cell);
        }
        const tdp::DensityGrid grid(nl, dc.core, config.grid_nx, config.grid_ny, config.target_density);
        tdp::PinPairWeights pairs;
        std::vector<double> net_weights;
        double lambda = config.lambda0;
        if (lambda <= 0.0) { // placer.cpp:388-402
            const tdp::ObjectiveResult wl_only = tdp::objective_and_gradient(nl, pos, grid, {}, {}, gamma, 0.0, 0.0,
                                                                             config.pp_loss, threads_obj);
            const tdp::DensityResult d0 = grid.evaluate(nl, pos, threads_obj);
            double wl_l1 = 0.0, d_l1 = 0.0;
            for (std::size_t c = 0; c < nl.cells.size(); ++c) {
                if (nl.cells[c].is_fixed) continue;
                wl_l1 += std::abs(wl_only.d_cell[c].x) + std::abs(wl_only.d_cell[c].y);
                d_l1 += std::abs(d0.d_cell[c].x) + std::abs(d0.d_cell[c].y);
            }
            lambda = (wl_l1 > 0.0 && d_l1 > 0.0) ? wl_l1 / d_l1 : 1.0;
        }
        const double lambda_cap = lambda * config.lambda_max;
        tdp::AdamState adam(2 * nl.cells.size());
        std::vector<double> flat(2 * nl.cells.size()), grad_flat(2 * nl.cells.size());
        bool timing_engaged = false;
        int rows = 0;
        for (int iter = 0; iter < config.max_iters; ++iter) {
            const auto t0 = std::chrono::steady_clock::now();
            refresh_ms[iter] = 0.0, paths[iter] = 0;
            bool sta_row = false;
            double row_tns = 0.0, row_wns = 0.0;
            if (iter >= config.timing_start_iter && (iter - config.timing_start_iter) % config.m == 0) {
                timing_engaged = true;
                const tdp::PinPositions ppos = tdp::pin_positions(nl, pos);
                const tdp::TimingAnnotation ann = tdp::run_sta(graph, nl, ppos, dc, threads_sta);
                sta_row = true, row_tns = ann.tns, row_wns = ann.wns;
                tdp::ExtractionReport report;
                if (ann.wns < 0.0) {
                    int n_fail = 0;
                    for (const auto& [pin, slack] : ann.endpoint_slacks)
                        if (slack < 0.0) ++n_fail;
                    report = config.extraction == tdp::ExtractionPolicy::Endpoint
                                 ? tdp::report_timing_endpoint(graph, nl, ppos, dc, ann, n_fail, config.k, threads_ex)
                                 : tdp::report_timing(graph, nl, ppos, dc, ann, n_fail, threads_ex);
                    const std::vector<tdp::PairHit> hits = tdp::collect_pin_pairs(nl, report.paths);
                    tdp::update_pair_weights(pairs, hits, ann.wns, config.w0, config.w1);
                }
                if (config.net_weighting) net_weights = tdp::apply_net_weights(ann, nl);
                refresh_ms[iter] = ms_since(t0);
                paths[iter] = static_cast<int64_t>(report.paths.size());
            }
            const tdp::ObjectiveResult obj = tdp::objective_and_gradient(nl, pos, grid, pairs, net_weights, gamma, lambda,
                                                                         config.beta, config.pp_loss, threads_obj);
            if (trace) { // TraceRow (placer.cpp:445-457)
                tdpg_trace_row& r = trace[iter];
                r.iter = iter, r.has_timing = sta_row ? 1 : 0, r.hpwl = obj.hpwl, r.overflow = obj.overflow;
                r.tns = row_tns, r.wns = row_wns, r.wl_term = obj.wl_term, r.density_term = obj.density_term;
                r.pp_term = obj.pp_term, r.lambda = lambda, r.beta_pp = config.beta * obj.pp_term;
            }
            ++rows;
            if (timing_engaged && obj.overflow <= config.stop_overflow) {
                iter_ms[iter] = ms_since(t0);
                break;
            }
            for (std::size_t c = 0; c < nl.cells.size(); ++c) {
                flat[2 * c] = pos[c].x, flat[2 * c + 1] = pos[c].y;
                grad_flat[2 * c] = obj.d_cell[c].x, grad_flat[2 * c + 1] = obj.d_cell[c].y;
            }
            const double lr = config.step0_frac * span * std::pow(config.step_decay, iter);
            adam.step(flat, grad_flat, lr, config.adam_beta1, config.adam_beta2, config.adam_eps);
            for (std::size_t c = 0; c < nl.cells.size(); ++c) {
                if (nl.cells[c].is_fixed) continue;
                pos[c] = tdp::Point{flat[2 * c], flat[2 * c + 1]};
                clamp(pos[c], nl.cells[c]);
            }
            lambda = std::min(lambda * config.mu, lambda_cap);
            iter_ms[iter] = ms_since(t0);
        }
        *n_rows = rows;
        *pairs_end = static_cast<int64_t>(pairs.size());
        const tdp::TimingAnnotation fin = tdp::run_sta(graph, nl, tdp::pin_positions(nl, pos), dc, threads_sta);
        final_[0] = fin.tns, final_[1] = fin.wns;
        final_[2] = tdp::hpwl_total(nl, tdp::pin_positions(nl, pos));
        s->outcome.positions = std::move(pos);
        s->ledger = std::move(pairs);
    });
}

int ref_place_positions(void* h, double* xy)
{
    return guard([&] { from_points(static_cast<RefSession*>(h)->outcome.positions, xy); });
}

const char* ref_place_csv(void* h) { return static_cast<RefSession*>(h)->csv.c_str(); }

// run_compare + compare_to_csv (compare.cpp:37-122) with JSON configs; the CSV via ref_place_csv.
int ref_compare(void* h, const char* const* config_jsons, int32_t n, int32_t parallel)
{
    return guard([&] {
        auto* s = static_cast<RefSession*>(h);
        std::vector<tdp::OptimizerConfig> cfgs;
        for (int32_t i = 0; i < n; ++i) cfgs.push_back(tdp::config_from_json(config_jsons[i]));
        s->csv = tdp::compare_to_csv(tdp::run_compare(s->design, cfgs, parallel != 0));
    });
}

// generate_synthetic: the design is held in a fresh session; fetch with ref_design_*.
int ref_generate(uint64_t seed, int cells, int registers, double fanout, double fail_frac, double r_unit,
                 double c_unit, void** out, double* elapsed_ms)
{
    return guard([&] {
        tdp::GeneratorSpec spec;
        spec.seed = seed;
        spec.n_cells = cells;
        spec.n_registers = registers;
        spec.avg_fanout = fanout;
        spec.target_fail_fraction = fail_frac;
        spec.r_unit = r_unit;
        spec.c_unit = c_unit;
        auto s = std::make_unique<RefSession>();
        const auto t0 = std::chrono::steady_clock::now();
        s->design = tdp::generate_synthetic(spec);
        if (elapsed_ms) *elapsed_ms = ms_since(t0);
        *out = s.release();
    });
}

// counts = n_cells, n_pins, n_nets, n_net_pins, n_sources, n_endpoints
int ref_design_counts(void* h, int64_t counts[6])
{
    return guard([&] {
        const auto& nl = static_cast<RefSession*>(h)->design.netlist;
        int64_t e = 0;
        for (const auto& n : nl.nets) e += 1 + static_cast<int64_t>(n.sinks.size());
        counts[0] = static_cast<int64_t>(nl.cells.size());
        counts[1] = static_cast<int64_t>(nl.pins.size());
        counts[2] = static_cast<int64_t>(nl.nets.size());
        counts[3] = e;
        counts[4] = static_cast<int64_t>(nl.sources.size());
        counts[5] = static_cast<int64_t>(nl.endpoints.size());
    });
}

// Fills caller-allocated arrays shaped like tdpg_netlist (const cast: the caller owns them).
int ref_design_fetch(void* h, tdpg_netlist* out, double* positions, uint8_t* pos_explicit)
{
    return guard([&] {
        const auto& d = static_cast<RefSession*>(h)->design;
        const auto& nl = d.netlist;
        auto* cw = const_cast<double*>(out->cell_w);
        auto* ch = const_cast<double*>(out->cell_h);
        auto* cd = const_cast<double*>(out->cell_delay);
        auto* cf = const_cast<uint8_t*>(out->cell_fixed);
        for (std::size_t c = 0; c < nl.cells.size(); ++c) {
            cw[c] = nl.cells[c].width;
            ch[c] = nl.cells[c].height;
            cd[c] = nl.cells[c].delay;
            cf[c] = nl.cells[c].is_fixed ? 1 : 0;
            positions[2 * c] = d.positions[c].x;
            positions[2 * c + 1] = d.positions[c].y;
            pos_explicit[c] = d.pos_explicit[c] ? 1 : 0;
        }
        auto* pc = const_cast<int32_t*>(out->pin_cell);
        auto* pt = const_cast<double*>(out->pin_term);
        auto* po = const_cast<double*>(out->pin_off);
        auto* pd = const_cast<uint8_t*>(out->pin_dir);
        auto* pcap = const_cast<double*>(out->pin_cap);
        for (std::size_t p = 0; p < nl.pins.size(); ++p) {
            pc[p] = nl.pins[p].cell;
            pt[2 * p] = nl.pins[p].terminal_pos.x;
            pt[2 * p + 1] = nl.pins[p].terminal_pos.y;
            po[2 * p] = nl.pins[p].offset.x;
            po[2 * p + 1] = nl.pins[p].offset.y;
            pd[p] = nl.pins[p].dir == tdp::PinDir::Output ? 1 : 0;
            pcap[p] = nl.pins[p].load_cap;
        }
        auto* ns = const_cast<int32_t*>(out->net_start);
        auto* np = const_cast<int32_t*>(out->net_pins);
        int32_t e = 0;
        for (std::size_t n = 0; n < nl.nets.size(); ++n) {
            ns[n] = e;
            np[e++] = nl.nets[n].driver;
            for (int s : nl.nets[n].sinks) np[e++] = s;
        }
        ns[nl.nets.size()] = e;
        std::memcpy(const_cast<int32_t*>(out->sources), nl.sources.data(), nl.sources.size() * sizeof(int32_t));
        std::memcpy(const_cast<int32_t*>(out->endpoints), nl.endpoints.data(), nl.endpoints.size() * sizeof(int32_t));
        out->clock_period = d.constraints.clock_period;
        out->r_unit = d.constraints.r_unit;
        out->c_unit = d.constraints.c_unit;
        out->core[0] = d.constraints.core.x_lo;
        out->core[1] = d.constraints.core.y_lo;
        out->core[2] = d.constraints.core.x_hi;
        out->core[3] = d.constraints.core.y_hi;
    });
}

// Design JSON round trip through the reference's own I/O (for the JSON fixtures).
int ref_design_from_json(const char* text, void** out)
{
    return guard([&] {
        auto s = std::make_unique<RefSession>();
        s->design = tdp::design_from_json(text);
        *out = s.release();
    });
}

const char* ref_design_to_json(void* h)
{
    auto* s = static_cast<RefSession*>(h);
    s->json = tdp::design_to_json(s->design);
    return s->json.c_str();
}

// The reference's fixture designs: 0 T1, 1 T2, 2 diamond(a, b), 3 trunk16, 4 random_design(seed, max_cells).
int ref_fixture(int which, uint64_t seed, double a, double b, int max_cells, void** out)
{
    return guard([&] {
        auto s = std::make_unique<RefSession>();
        switch (which) {
        case 0: s->design = tdptest::make_t1(); break;
        case 1: s->design = tdptest::make_t2(); break;
        case 2: s->design = tdptest::make_diamond(a, b); break;
        case 3: s->design = tdptest::make_trunk16(); break;
        default: s->design = tdptest::random_design(seed, max_cells); break;
        }
        *out = s.release();
    });
}

const char* ref_default_config(void)
{
    static std::string text = tdp::config_to_json(tdp::OptimizerConfig{});
    return text.c_str();
}

} // extern "C"
