// Host overhead of the C++ drop-in's per-iteration call: tdp::objective_and_gradient (placer.cpp:275-343)
// on the bench's 1M design read from its binary design file, the way a reference-style loop calls it
// (std::vector<Point> in, ObjectiveResult with the cell gradient out).  Prints the wall time of the first
// call (device session creation) and of repeated calls against the device time of one objective
// evaluation.  Usage: dropin_overhead DESIGN.tdpb [reps]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "tdp/tdp_api.hpp"
#include "tdpg.h"

int main(int argc, char** argv)
{
    if (argc < 2) return std::fprintf(stderr, "usage: %s DESIGN.tdpb [reps]\n", argv[0]), 2;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
    int64_t cnt[6];
    if (tdpg_design_bin_info(argv[1], cnt, nullptr) != TDPG_OK) return std::fprintf(stderr, "%s\n", tdpg_last_error()), 1;
    const int C = static_cast<int>(cnt[0]), P = static_cast<int>(cnt[1]), N = static_cast<int>(cnt[2]);
    std::vector<double> cw(C), ch(C), cd(C), pt(2 * P), po(2 * P), pc(P), pos(2 * C);
    std::vector<uint8_t> cf(C), pd(P), pe(C);
    std::vector<int32_t> pcell(P), ns(N + 1), np(cnt[3]), src(cnt[4]), ep(cnt[5]);
    tdpg_netlist d{};
    d.n_cells = C, d.n_pins = P, d.n_nets = N, d.n_sources = static_cast<int>(cnt[4]), d.n_endpoints = static_cast<int>(cnt[5]);
    d.cell_w = cw.data(), d.cell_h = ch.data(), d.cell_delay = cd.data(), d.cell_fixed = cf.data();
    d.pin_cell = pcell.data(), d.pin_term = pt.data(), d.pin_off = po.data(), d.pin_dir = pd.data();
    d.pin_cap = pc.data(), d.net_start = ns.data(), d.net_pins = np.data(), d.sources = src.data();
    d.endpoints = ep.data();
    if (tdpg_design_bin_read(argv[1], &d, pos.data(), pe.data(), nullptr, 0) != TDPG_OK)
        return std::fprintf(stderr, "%s\n", tdpg_last_error()), 1;
    // the reference's Netlist (netlist.hpp) built from the arrays
    tdp::Netlist nl;
    nl.cells.resize(C), nl.pins.resize(P), nl.nets.resize(N);
    for (int c = 0; c < C; ++c) nl.cells[c].width = cw[c], nl.cells[c].height = ch[c], nl.cells[c].delay = cd[c],
                                nl.cells[c].is_fixed = cf[c] != 0;
    for (int p = 0; p < P; ++p) {
        tdp::Pin& q = nl.pins[p];
        q.cell = pcell[p], q.terminal_pos = {pt[2 * p], pt[2 * p + 1]}, q.offset = {po[2 * p], po[2 * p + 1]};
        q.dir = pd[p] ? tdp::PinDir::Output : tdp::PinDir::Input, q.load_cap = pc[p];
    }
    for (int n = 0; n < N; ++n) {
        nl.nets[n].driver = np[ns[n]];
        nl.nets[n].sinks.assign(np.begin() + ns[n] + 1, np.begin() + ns[n + 1]);
    }
    nl.sources.assign(src.begin(), src.end()), nl.endpoints.assign(ep.begin(), ep.end());
    nl.finalize();
    std::vector<tdp::Point> xy(C);
    for (int c = 0; c < C; ++c) xy[c] = {pos[2 * c], pos[2 * c + 1]};
    const tdp::Rect core{d.core[0], d.core[1], d.core[2], d.core[3]};
    const tdp::DensityGrid grid(nl, core, 1024, 1024, 0.6);
    const tdp::PinPairWeights w;
    const std::vector<double> nw;
    const double gamma = 0.01 * core.span();
    using clk = std::chrono::steady_clock;
    { // CUDA context + module load on a one-net design first, so call 0 below is the 1M session creation
        tdp::Netlist tiny;
        tiny.cells.resize(2);
        for (auto& c : tiny.cells) c.width = c.height = 1.0;
        tiny.pins.resize(2);
        tiny.pins[0].cell = 0, tiny.pins[0].dir = tdp::PinDir::Output, tiny.pins[1].cell = 1;
        tiny.nets.resize(1);
        tiny.nets[0].driver = 0, tiny.nets[0].sinks = {1};
        tiny.finalize();
        const tdp::Rect tc{0, 0, 10, 10};
        const auto t0 = clk::now();
        tdp::objective_and_gradient(tiny, {{1, 1}, {5, 5}}, tdp::DensityGrid(tiny, tc, 4, 4, 0.6), w, nw, 1.0, 1e-3, 0.0);
        std::printf("warm-up (CUDA context, module load): %.1f ms\n",
                    std::chrono::duration<double, std::milli>(clk::now() - t0).count());
    }
    for (int r = 0; r <= reps; ++r) {
        if (r > 0) xy[r % C].x += 1e-9; // (positions change between calls, as in a loop)
        const auto t0 = clk::now();
        const tdp::ObjectiveResult res = tdp::objective_and_gradient(nl, xy, grid, w, nw, gamma, 1e-3, 0.0);
        const double ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        std::printf("call %d: %.2f ms (value %.6e, |d_cell| = %zu)%s\n", r, ms, res.value, res.d_cell.size(),
                    r == 0 ? "  <- includes the device session creation" : "");
    }
    return 0;
}
