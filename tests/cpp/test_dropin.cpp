// test_dropin.cpp — the reference's C++ operator API (tdp::, libtdp_b200.so over the sm_100a engine),
// exercised the way the reference's own unit tests use it; known answers from
// /root/reference/proj/tests/{test_sta,test_paths,test_placer,test_netlist}.cpp.
// Prints one line per check; exit code = number of failures.  Needs a CUDA device.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "tdp/compare.hpp"
#include "tdp/density.hpp"
#include "tdp/errors.hpp"
#include "tdp/netlist.hpp"
#include "tdp/paths.hpp"
#include "tdp/pin_pairs.hpp"
#include "tdp/placer.hpp"
#include "tdp/sta.hpp"
#include "tdp/timing_graph.hpp"
#include "tdp/wirelength.hpp"

using namespace tdp;

static int g_fail = 0;
#define CHECK(cond)                                                              \
    do {                                                                         \
        if (!(cond)) {                                                           \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);        \
            ++g_fail;                                                            \
        }                                                                        \
    } while (0)

static bool near(double a, double b, double tol = 1e-12) { return std::abs(a - b) <= tol * std::max(1.0, std::abs(b)); }

// Small in-memory designs (same geometry as the reference fixtures).
struct Build {
    Design d;
    Build(double clock, double r, double c)
    {
        d.constraints.core = Rect{0, 0, 10, 10};
        d.constraints.clock_period = clock, d.constraints.r_unit = r, d.constraints.c_unit = c;
    }
    int cell(const char* n, double delay, Point at)
    {
        d.netlist.cells.push_back(Cell{n, 1, 1, false, delay});
        d.positions.push_back(at);
        d.pos_explicit.push_back(true);
        return static_cast<int>(d.netlist.cells.size()) - 1;
    }
    int pin(const std::string& n, int cell, bool out)
    {
        Pin p;
        p.name = n, p.cell = cell, p.dir = out ? PinDir::Output : PinDir::Input;
        d.netlist.pins.push_back(p);
        return static_cast<int>(d.netlist.pins.size()) - 1;
    }
    int term(const std::string& n, Point at, bool out)
    {
        Pin p;
        p.name = n, p.terminal_pos = at, p.dir = out ? PinDir::Output : PinDir::Input;
        d.netlist.pins.push_back(p);
        return static_cast<int>(d.netlist.pins.size()) - 1;
    }
    void net(const std::string& n, int drv, std::vector<int> sinks) { d.netlist.nets.push_back(Net{n, drv, sinks}); }
    Design done()
    {
        d.netlist.finalize();
        return d;
    }
};

static Design t1(double clock = 10.0)
{ // PI -> A -> B -> C -> PO, r = c = 1, cells at (0,0), (3,0), (3,4)
    Build b(clock, 1, 1);
    const int A = b.cell("A", 1, {0, 0}), B = b.cell("B", 1, {3, 0}), C = b.cell("C", 1, {3, 4});
    const int pi = b.term("PI", {0, 0}, true);
    const int ai = b.pin("A.in", A, false), ao = b.pin("A.out", A, true);
    const int bi = b.pin("B.in", B, false), bo = b.pin("B.out", B, true);
    const int ci = b.pin("C.in", C, false), co = b.pin("C.out", C, true);
    const int po = b.term("PO", {3, 4}, false);
    b.net("n0", pi, {ai}), b.net("n1", ao, {bi}), b.net("n2", bo, {ci}), b.net("n3", co, {po});
    b.d.netlist.sources = {pi}, b.d.netlist.endpoints = {po};
    return b.done();
}

static Design diamond(double da, double db)
{
    Build b(10, 1, 1);
    const int A = b.cell("A", da, {0, 0}), B = b.cell("B", db, {0, 0}), M = b.cell("M", 1, {0, 0});
    const int s = b.term("S", {0, 0}, true);
    const int ai = b.pin("A.in", A, false), ao = b.pin("A.out", A, true);
    const int bi = b.pin("B.in", B, false), bo = b.pin("B.out", B, true);
    const int ma = b.pin("M.a", M, false), mb = b.pin("M.b", M, false), mo = b.pin("M.out", M, true);
    const int ep = b.term("EP", {0, 0}, false);
    b.net("nS", s, {ai, bi}), b.net("nA", ao, {ma}), b.net("nB", bo, {mb}), b.net("nM", mo, {ep});
    b.d.netlist.sources = {s}, b.d.netlist.endpoints = {ep};
    return b.done();
}

static Design t2()
{
    Build b(10, 1, 1);
    const int X = b.cell("X", 7, {0, 0}), Y = b.cell("Y", 6, {0, 0}), Z = b.cell("Z", 13, {0, 0}), M = b.cell("M", 8, {0, 0});
    const int s = b.term("S", {0, 0}, true);
    const int xi = b.pin("X.in", X, false), xo = b.pin("X.out", X, true);
    const int yi = b.pin("Y.in", Y, false), yo = b.pin("Y.out", Y, true);
    const int zi = b.pin("Z.in", Z, false), zo = b.pin("Z.out", Z, true);
    const int ma = b.pin("M.a", M, false), mb = b.pin("M.b", M, false), mo = b.pin("M.out", M, true);
    const int e1 = b.term("EP1", {0, 0}, false), e2 = b.term("EP2", {0, 0}, false);
    b.net("nS", s, {xi, yi, zi}), b.net("nX", xo, {ma}), b.net("nY", yo, {mb}), b.net("nM", mo, {e1}),
        b.net("nZ", zo, {e2});
    b.d.netlist.sources = {s}, b.d.netlist.endpoints = {e1, e2};
    return b.done();
}

int main()
{
    { // test_sta.cpp:55-77 + test_netlist.cpp:252-269
        const Design d = t1();
        const TimingGraph g = build_timing_graph(d.netlist);
        CHECK(g.num_net_arcs == 4 && g.num_cell_arcs == 3 && g.levelized);
        CHECK(g.level[0] == 0 && g.level[7] == 7);
        const TimingAnnotation t = run_sta(g, d.netlist, pin_positions(d.netlist, d.positions), d.constraints);
        const double arr[8] = {0, 0, 1, 10, 11, 27, 28, 28}, req[8] = {-18, -18, -17, -8, -7, 9, 10, 10};
        for (int p = 0; p < 8; ++p) CHECK(t.arr[p] == arr[p] && t.req[p] == req[p] && t.slack[p] == -18.0);
        CHECK(t.tns == -18.0 && t.wns == -18.0 && t.endpoint_slacks.size() == 1);
        CHECK(hpwl_total(d.netlist, pin_positions(d.netlist, d.positions)) == 7.0);
        const auto rep = report_timing_endpoint(g, d.netlist, pin_positions(d.netlist, d.positions), d.constraints, t, 1, 1);
        const auto hits = collect_pin_pairs(d.netlist, rep.paths);
        CHECK(hits.size() == 4 && hits[0].pair == std::make_pair(0, 1) && hits[3].pair == std::make_pair(6, 7));
        std::printf("ok   t1 sta / graph / hpwl / pairs\n");
    }
    { // test_paths.cpp:42-82: diamond k = 1, the equal-delay tie, EndpointError
        for (double db : {5.0, 7.0}) {
            const Design d = diamond(7, db);
            const TimingGraph g = build_timing_graph(d.netlist);
            const auto pos = pin_positions(d.netlist, d.positions);
            const auto t = run_sta(g, d.netlist, pos, d.constraints);
            const auto k1 = k_worst_paths_to(g, d.netlist, pos, d.constraints, t, 8, 1);
            CHECK(k1.size() == 1 && k1[0].pins == (std::vector<int>{0, 1, 2, 5, 7, 8}) && k1[0].slack == 2.0);
            bool threw = false;
            try {
                k_worst_paths_to(g, d.netlist, pos, d.constraints, t, 7, 1);
            } catch (const EndpointError& e) {
                threw = std::string(e.what()).find("is not an endpoint") != std::string::npos;
            }
            CHECK(threw);
            PathEnumerator en(g, d.netlist, pos, d.constraints);
            const auto* r0 = en.path_to(7, 0);
            CHECK(r0 && r0->delay == 8.0 && r0->pins == (std::vector<int>{0, 1, 2, 5, 7}));
        }
        std::printf("ok   diamond paths / tie / EndpointError / PathEnumerator rank 0\n");
    }
    { // test_paths.cpp:42-103: k worst paths, the tie order for k = 2, path_to ranks and exhaustion
        const Design d = diamond(7, 5);
        const TimingGraph g = build_timing_graph(d.netlist);
        const auto pos = pin_positions(d.netlist, d.positions);
        const auto t = run_sta(g, d.netlist, pos, d.constraints);
        const auto k2 = k_worst_paths_to(g, d.netlist, pos, d.constraints, t, 8, 2);
        CHECK(k2.size() == 2 && k2[1].pins == (std::vector<int>{0, 3, 4, 6, 7, 8}) && k2[1].slack == 4.0);
        CHECK(k_worst_paths_to(g, d.netlist, pos, d.constraints, t, 8, 3).size() == 2);
        PathEnumerator en(g, d.netlist, pos, d.constraints);
        const auto* r1 = en.path_to(7, 1);
        CHECK(r1 && r1->delay == 6.0 && en.path_to(7, 2) == nullptr);
        const Design e = diamond(7, 7);
        const TimingGraph ge = build_timing_graph(e.netlist);
        const auto pe = pin_positions(e.netlist, e.positions);
        const auto te = run_sta(ge, e.netlist, pe, e.constraints);
        const auto tie = k_worst_paths_to(ge, e.netlist, pe, e.constraints, te, 8, 2);
        CHECK(tie.size() == 2 && tie[0].slack == tie[1].slack && tie[0].pins < tie[1].pins);
        std::printf("ok   k worst paths / path_to ranks / tie order\n");
    }
    { // test_paths.cpp:105-139: topn piles onto the worst endpoint; n beyond the violated set
        const Design d = t2();
        const TimingGraph g = build_timing_graph(d.netlist);
        const auto pos = pin_positions(d.netlist, d.positions);
        const auto t = run_sta(g, d.netlist, pos, d.constraints);
        const auto r = report_timing(g, d.netlist, pos, d.constraints, t, 2);
        CHECK(r.policy == "topn" && r.paths.size() == 2 && r.paths[0].slack == -5.0 && r.paths[1].slack == -4.0);
        CHECK(r.unique_endpoints == 1 && r.candidates_generated == 4 && r.unique_pin_pairs == 5);
        const auto r10 = report_timing(g, d.netlist, pos, d.constraints, t, 10);
        CHECK(r10.paths.size() == 3 && r10.candidates_generated == 20 && r10.unique_endpoints == 2);
        std::printf("ok   topn policy\n");
    }
    { // compare.cpp:37-95: two configs on a tight T2, serial and parallel give the same rows
        Design d = t2();
        d.constraints.clock_period = 2.0;
        OptimizerConfig a, b;
        a.name = "endpoint", a.max_iters = 30, a.timing_start_iter = 10, a.m = 5, a.grid_nx = a.grid_ny = 8;
        b = a, b.name = "topn", b.extraction = ExtractionPolicy::TopN;
        const CompareReport s = run_compare(d, {a, b}, false), p = run_compare(d, {a, b}, true);
        CHECK(s.rows.size() == 2 && s.rows[0].ok && s.rows[1].ok);
        for (int i = 0; i < 2; ++i)
            CHECK(s.rows[i].tns == p.rows[i].tns && s.rows[i].hpwl == p.rows[i].hpwl &&
                  s.rows[i].candidates_generated == p.rows[i].candidates_generated);
        CHECK(compare_to_csv(s).rfind("config,status,tns,wns,hpwl,runtime_s,", 0) == 0);
        b.seed = 2;
        bool threw = false;
        try {
            run_compare(d, {a, b});
        } catch (const ValidationError& e) {
            threw = std::string(e.what()).find("share one seed") != std::string::npos;
        }
        CHECK(threw);
        std::printf("ok   run_compare / compare_to_csv\n");
    }
    { // test_paths.cpp:105-139 endpoint policy counters
        const Design d = t2();
        const TimingGraph g = build_timing_graph(d.netlist);
        const auto pos = pin_positions(d.netlist, d.positions);
        const auto t = run_sta(g, d.netlist, pos, d.constraints);
        CHECK(t.tns == -8.0 && t.wns == -5.0);
        if (t.tns != -8.0 || t.wns != -5.0) std::printf("     t2 tns %.17g wns %.17g\n", t.tns, t.wns);
        const auto r = report_timing_endpoint(g, d.netlist, pos, d.constraints, t, 2, 1);
        CHECK(r.policy == "endpoint" && r.paths.size() == 2 && r.paths[0].slack == -5.0 && r.paths[1].slack == -3.0);
        CHECK(r.unique_endpoints == 2 && r.candidates_generated == 2 && r.unique_pin_pairs == 5);
        std::printf("ok   t2 endpoint report\n");
    }
    { // test_placer.cpp:56-65, 283-299, 346-362, 509-520
        const std::vector<Point> two = {{0, 0}, {10, 0}};
        const NetTermGrad w = wa_wirelength(two, 1.0);
        CHECK(std::abs(w.value - 10.0 * std::tanh(5.0)) <= 1e-13 && w.d_pin[0].x < 0 && w.d_pin[0].y == 0.0);
        PinPairWeights pw;
        pw[{0, 1}] = 10.0;
        const auto q = pin_pair_loss(pw, {{0, 0}, {3, 4}}, 2, PairLossKind::Quadratic);
        CHECK(q.value == 250.0 && q.d_pin[0].x == -60.0 && q.d_pin[0].y == -80.0 && q.d_pin[1].x == 60.0);
        const auto l = pin_pair_loss(pw, {{0, 0}, {3, 4}}, 2, PairLossKind::Linear);
        CHECK(l.value == 50.0 && l.d_pin[0].x == -6.0 && l.d_pin[0].y == -8.0);
        PinPairWeights led;
        update_pair_weights(led, {{{1, 2}, -400.0}}, -500.0, 10.0, 0.2);
        CHECK((led.size() == 1 && led[std::make_pair(1, 2)] == 10.0));
        update_pair_weights(led, {{{1, 2}, -400.0}}, -500.0, 10.0, 0.2);
        CHECK(near(led[std::make_pair(1, 2)], 10.16));
        AdamState adam(1);
        std::vector<double> x = {5.0};
        adam.step(x, {3.0}, 0.1, 0.9, 0.999, 1e-8);
        CHECK(std::abs(x[0] - 4.9) <= 4.9e-8);
        adam.step(x, {3.0}, 0.1, 0.9, 0.999, 1e-8);
        CHECK(std::abs(x[0] - 4.8) <= 4.8e-7 && adam.t == 2);
        std::printf("ok   wa / pin pairs / ledger / adam\n");
    }
    { // objective_and_gradient: finite terms; NonFiniteError on an infinite coordinate (test_placer.cpp:498-505)
        const Design d = t1();
        const DensityGrid grid(d.netlist, d.constraints.core, 4, 4, 0.9);
        const ObjectiveResult r = objective_and_gradient(d.netlist, d.positions, grid, {}, {}, 0.1, 0.5, 0.1);
        CHECK(std::isfinite(r.value) && r.hpwl == 7.0 && r.d_cell.size() == 3);
        std::vector<Point> bad = d.positions;
        bad[1].x = INFINITY;
        bool threw = false;
        try {
            objective_and_gradient(d.netlist, bad, grid, {}, {}, 0.1, 0.5, 0.1);
        } catch (const NonFiniteError&) {
            threw = true;
        }
        CHECK(threw);
        std::printf("ok   objective / NonFiniteError\n");
    }
    { // run_placement schedule + observer (test_placer.cpp:709-804)
        const Design d = t1(2.0);
        OptimizerConfig c;
        c.max_iters = 40, c.timing_start_iter = 10, c.m = 5, c.grid_nx = 8, c.grid_ny = 8, c.target_density = 1e-6;
        std::vector<int> rounds;
        const PlacementOutcome out =
            run_placement(d, c, [&](int iter, const TimingAnnotation& a, const ExtractionReport& r) {
                rounds.push_back(iter);
                CHECK(a.wns < 0.0 && !r.paths.empty());
            });
        CHECK(out.stop_reason == "max_iters" && out.iterations == 40 && out.trace.size() == 40);
        CHECK(rounds == (std::vector<int>{10, 15, 20, 25, 30, 35}));
        for (const TraceRow& row : out.trace) CHECK(row.has_timing == (row.iter >= 10 && (row.iter - 10) % 5 == 0));
        CHECK(out.trace.back().pp_term > 0.0 && !out.pair_weights.empty());
        CHECK(metrics_to_csv(out.trace).rfind("iter,hpwl,overflow,tns,wns", 0) == 0);
        std::printf("ok   run_placement schedule / observer\n");
    }
    { // combinational cycle (test_netlist.cpp:295-317)
        Build b(10, 1, 1);
        const int U = b.cell("u0", 1, {0, 0}), V = b.cell("u1", 1, {0, 0});
        const int ui = b.pin("u0.i", U, false), uo = b.pin("u0.o", U, true);
        const int vi = b.pin("u1.i", V, false), vo = b.pin("u1.o", V, true);
        b.net("a", uo, {vi}), b.net("b", vo, {ui});
        const Design d = b.done();
        bool threw = false;
        try {
            build_timing_graph(d.netlist);
        } catch (const CycleError& e) {
            threw = std::string(e.what()).find("combinational cycle") != std::string::npos &&
                    std::string(e.what()).find("u0.o") != std::string::npos;
        }
        CHECK(threw);
        std::printf("ok   CycleError\n");
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "PASSED", g_fail);
    return g_fail;
}
