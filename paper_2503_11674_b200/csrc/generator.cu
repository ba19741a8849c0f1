// generator.cu — generate_synthetic (generator.cpp:60-263) with the same mt19937_64
// stream and the same draws, but without the reference's quadratic scans:
//   * shallow-driver fallback (generator.cpp:39-42): the list of drivers below the depth
//     bound only grows and keeps driver order, so it is maintained incrementally;
//   * idle-driver pick for primary outputs (generator.cpp:198-204): a Fenwick tree over
//     "idle, non-terminal" drivers gives the k-th idle driver in O(log N);
//   * net assembly (generator.cpp:209-217): connections are bucketed per driver in
//     creation order (stable counting sort) instead of rescanned per driver.
// Register slots use 64-bit arithmetic; the reference's int expression
// (r + 1) * total_slots overflows above ~1.4e5 cells (generator.cpp:90).
// The clock calibration runs the coarse placement (coarse_config, generator.cpp:47-58)
// on the GPU engine.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <random>
#include <vector>

#include "engine.cuh"

struct tdpg_design {
    std::vector<double> cell_w, cell_h, cell_delay, pin_term, pin_off, pin_cap, positions;
    std::vector<uint8_t> cell_fixed, pin_dir;
    std::vector<int> pin_cell, net_start, net_pins, sources, endpoints;
    double clock = 1.0, r_unit = 1e-4, c_unit = 1e-4, core[4] = {0, 0, 0, 0};
    tdpg_netlist view() const
    {
        tdpg_netlist v{};
        v.n_cells = static_cast<int32_t>(cell_w.size());
        v.n_pins = static_cast<int32_t>(pin_cell.size());
        v.n_nets = static_cast<int32_t>(net_start.size()) - 1;
        v.n_sources = static_cast<int32_t>(sources.size());
        v.n_endpoints = static_cast<int32_t>(endpoints.size());
        v.cell_w = cell_w.data(), v.cell_h = cell_h.data(), v.cell_delay = cell_delay.data();
        v.cell_fixed = cell_fixed.data(), v.pin_cell = pin_cell.data(), v.pin_term = pin_term.data();
        v.pin_off = pin_off.data(), v.pin_dir = pin_dir.data(), v.pin_cap = pin_cap.data();
        v.net_start = net_start.data(), v.net_pins = net_pins.data(), v.sources = sources.data();
        v.endpoints = endpoints.data(), v.clock_period = clock, v.r_unit = r_unit, v.c_unit = c_unit;
        std::memcpy(v.core, core, sizeof core);
        v.pin_names = nullptr;
        return v;
    }
};

namespace tdpg {
int api_fail(int kind, const std::string& msg);
}

namespace {

using tdpg::Error;

constexpr int kLocalityWindow = 30;
constexpr double kLocalityProb = 0.7;
constexpr int kMaxDepth = 20;

struct Rng { // include/tdp/rng.hpp:13-28
    std::mt19937_64 g;
    explicit Rng(uint64_t s) : g(s) {}
    double unit() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }
    int64_t integer(int64_t lo, int64_t hi)
    {
        const auto range = static_cast<uint64_t>(hi - lo) + 1;
        return lo + static_cast<int64_t>(g() % range);
    }
};

int pick_driver_index(Rng& rng, int n) // generator.cpp:22-27
{
    if (n > kLocalityWindow && rng.unit() < kLocalityProb)
        return static_cast<int>(rng.integer(n - kLocalityWindow, n - 1));
    return static_cast<int>(rng.integer(0, n - 1));
}

struct Fenwick {
    std::vector<int> t;
    int n = 0, top = 1;
    void init(int cap)
    {
        n = cap;
        t.assign(cap + 1, 0);
        top = 1;
        while (top * 2 <= n) top *= 2;
    }
    void add(int i, int d)
    {
        for (++i; i <= n; i += i & -i) t[i] += d;
    }
    int kth(int k) const // 0-based k-th set position
    {
        int pos = 0;
        for (int step = top; step; step >>= 1)
            if (pos + step <= n && t[pos + step] <= k) pos += step, k -= t[pos];
        return pos;
    }
};

void generate(uint64_t seed, int n_cells, int n_registers, double avg_fanout, double fail_frac, double r_unit,
              double c_unit, tdpg_design& D)
{
    auto gen_err = [](const char* m) { throw Error(TDPG_ERR_VALIDATION, std::string("validation error: generator: ") + m); };
    if (n_cells < 1) gen_err("n_cells must be >= 1");
    if (!(avg_fanout > 0.0)) gen_err("avg_fanout must be > 0");
    if (avg_fanout > n_cells) gen_err("avg_fanout exceeds cell count");
    if (!(fail_frac >= 0.0 && fail_frac <= 1.0)) gen_err("target_fail_fraction must be in [0, 1]");
    if (!(r_unit > 0.0 && c_unit > 0.0)) gen_err("r_unit and c_unit must be > 0");

    const int n_regs = n_registers >= 0 ? n_registers : n_cells / 10;
    const int n_pi = std::max(2, n_cells / 20);
    const int n_po = std::max(2, n_cells / 20);
    const int n_drivers_total = n_pi + n_cells + n_regs;
    const double mean_in = std::clamp((avg_fanout * n_drivers_total - n_regs - n_po) / n_cells, 1.0, 8.0);

    Rng rng(seed);
    const int total_slots = n_cells + n_regs;
    std::vector<uint8_t> slot_is_reg(total_slots, 0);
    for (int r = 0; r < n_regs; ++r)
        slot_is_reg[static_cast<size_t>((static_cast<int64_t>(r) + 1) * total_slots / (n_regs + 1))] = 1;

    const size_t est_pins = static_cast<size_t>(n_pi + n_po) + static_cast<size_t>(total_slots) * 5;
    D.pin_cell.reserve(est_pins), D.pin_term.reserve(2 * est_pins), D.pin_off.reserve(2 * est_pins);
    D.pin_dir.reserve(est_pins), D.pin_cap.reserve(est_pins);
    auto add_pin = [&](int cell, double tx, double ty, double ox, double oy, uint8_t dir, double cap) {
        D.pin_cell.push_back(cell);
        D.pin_term.push_back(tx), D.pin_term.push_back(ty);
        D.pin_off.push_back(ox), D.pin_off.push_back(oy);
        D.pin_dir.push_back(dir);
        D.pin_cap.push_back(cap);
        return static_cast<int>(D.pin_cell.size()) - 1;
    };

    std::vector<int> drivers, sink_count, depth, shallow;
    std::vector<std::pair<int, int>> conns; // (sink pin, driver index), creation order
    drivers.reserve(n_drivers_total), sink_count.reserve(n_drivers_total), depth.reserve(n_drivers_total);
    auto new_driver = [&](int pin, int d) {
        if (d < kMaxDepth) shallow.push_back(static_cast<int>(drivers.size()));
        drivers.push_back(pin), sink_count.push_back(0), depth.push_back(d);
    };
    auto add_conn = [&](int sink, int idx) {
        conns.emplace_back(sink, idx);
        ++sink_count[idx];
    };
    auto pick_shallow = [&]() { // generator.cpp:32-43
        const int n = static_cast<int>(depth.size());
        for (int a = 0; a < 16; ++a) {
            const int idx = pick_driver_index(rng, n);
            if (depth[idx] < kMaxDepth) return idx;
        }
        return shallow[static_cast<size_t>(rng.integer(0, static_cast<int64_t>(shallow.size()) - 1))];
    };

    std::vector<int> unit_scaled;
    for (int i = 0; i < n_pi; ++i) {
        const int p = add_pin(-1, 0.0, (i + 0.5) / n_pi, 0.0, 0.0, 1, 0.0);
        unit_scaled.push_back(p);
        D.sources.push_back(p);
        new_driver(p, 0);
    }
    D.cell_w.reserve(total_slots), D.cell_h.reserve(total_slots), D.cell_delay.reserve(total_slots);
    for (int slot = 0; slot < total_slots; ++slot) {
        const double w = rng.uniform(400.0, 800.0);
        const double h = rng.uniform(400.0, 800.0);
        const double delay = rng.uniform(0.5, 1.5);
        const int cell = static_cast<int>(D.cell_w.size());
        if (slot_is_reg[slot]) {
            const double dx = rng.uniform(0.0, w), dy = rng.uniform(0.0, h);
            const double cap = rng.uniform(0.5, 2.0);
            const int d_pin = add_pin(cell, 0.0, 0.0, dx, dy, 0, cap);
            D.endpoints.push_back(d_pin);
            add_conn(d_pin, pick_driver_index(rng, static_cast<int>(drivers.size())));
            const double qx = rng.uniform(0.0, w), qy = rng.uniform(0.0, h);
            const int q_pin = add_pin(cell, 0.0, 0.0, qx, qy, 1, 0.0);
            D.sources.push_back(q_pin);
            new_driver(q_pin, 0);
        } else {
            const int n_in = static_cast<int>(mean_in) + (rng.unit() < mean_in - std::floor(mean_in) ? 1 : 0);
            int depth_in = 0;
            for (int i = 0; i < std::max(1, n_in); ++i) {
                const double dx = rng.uniform(0.0, w), dy = rng.uniform(0.0, h);
                const double cap = rng.uniform(0.5, 2.0);
                const int pin = add_pin(cell, 0.0, 0.0, dx, dy, 0, cap);
                const int idx = pick_shallow();
                depth_in = std::max(depth_in, depth[idx]);
                add_conn(pin, idx);
            }
            const double ox = rng.uniform(0.0, w), oy = rng.uniform(0.0, h);
            const int o = add_pin(cell, 0.0, 0.0, ox, oy, 1, 0.0);
            new_driver(o, depth_in + 1);
        }
        D.cell_w.push_back(w), D.cell_h.push_back(h), D.cell_delay.push_back(delay);
    }
    // primary outputs prefer idle, non-terminal drivers (generator.cpp:187-206)
    const int nd = static_cast<int>(drivers.size());
    Fenwick idle;
    idle.init(nd);
    int n_idle = 0;
    for (int d = 0; d < nd; ++d)
        if (sink_count[d] == 0 && D.pin_cell[drivers[d]] >= 0) idle.add(d, 1), ++n_idle;
    for (int i = 0; i < n_po; ++i) {
        const double cap = rng.uniform(0.5, 2.0);
        const int p = add_pin(-1, 1.0, (i + 0.5) / n_po, 0.0, 0.0, 0, cap);
        unit_scaled.push_back(p);
        D.endpoints.push_back(p);
        int idx;
        if (n_idle > 0) idx = idle.kth(static_cast<int>(rng.integer(0, n_idle - 1)));
        else idx = static_cast<int>(rng.integer(0, nd - 1));
        if (sink_count[idx] == 0 && D.pin_cell[drivers[idx]] >= 0) idle.add(idx, -1), --n_idle;
        add_conn(p, idx);
    }
    // one net per driver with sinks, in driver order; sinks in connection order
    std::vector<int> start(nd + 1, 0);
    for (const auto& c : conns) start[c.second + 1]++;
    for (int d = 0; d < nd; ++d) start[d + 1] += start[d];
    std::vector<int> bucket(conns.size());
    {
        std::vector<int> f(start.begin(), start.end() - 1);
        for (const auto& c : conns) bucket[f[c.second]++] = c.first;
    }
    D.net_start.reserve(nd + 1);
    D.net_pins.reserve(conns.size() + nd);
    D.net_start.push_back(0);
    for (int d = 0; d < nd; ++d) {
        if (sink_count[d] == 0) continue;
        D.net_pins.push_back(drivers[d]);
        for (int j = start[d]; j < start[d + 1]; ++j) D.net_pins.push_back(bucket[j]);
        D.net_start.push_back(static_cast<int>(D.net_pins.size()));
    }
    // core at 75% utilisation (generator.cpp:219-231)
    double area = 0.0;
    for (size_t c = 0; c < D.cell_w.size(); ++c) area += D.cell_w[c] * D.cell_h[c];
    const double side = std::ceil(std::sqrt(area / 0.75));
    D.core[0] = 0.0, D.core[1] = 0.0, D.core[2] = side, D.core[3] = side;
    for (int p : unit_scaled) {
        D.pin_term[2 * p] = D.core[0] + D.pin_term[2 * p] * (D.core[2] - D.core[0]);
        D.pin_term[2 * p + 1] = D.core[1] + D.pin_term[2 * p + 1] * (D.core[3] - D.core[1]);
    }
    D.clock = 1.0, D.r_unit = r_unit, D.c_unit = c_unit;
    D.cell_fixed.assign(D.cell_w.size(), 0);
    D.positions.resize(2 * D.cell_w.size());
    for (size_t c = 0; c < D.cell_w.size(); ++c) {
        D.positions[2 * c] = D.core[0] + (D.core[2] - D.core[0] - D.cell_w[c]) / 2.0;
        D.positions[2 * c + 1] = D.core[1] + (D.core[3] - D.core[1] - D.cell_h[c]) / 2.0;
    }
}

// Clock at the (1 - fail_frac) quantile of endpoint arrivals after the coarse
// placement (generator.cpp:246-260).
void calibrate(tdpg_design& D, uint64_t seed, double fail_frac)
{
    tdpg_session* s = nullptr;
    const tdpg_netlist v = D.view();
    if (tdpg_session_create(&v, &s) != TDPG_OK) throw Error(tdpg_last_error_kind(), tdpg_last_error());
    std::unique_ptr<tdpg_session, int (*)(tdpg_session*)> guard(s, tdpg_session_destroy);
    if (tdpg_set_positions(s, D.positions.data()) != TDPG_OK) throw Error(tdpg_last_error_kind(), tdpg_last_error());
    tdpg_config c;
    tdpg_config_default(&c); // coarse_config (generator.cpp:47-58)
    c.beta = 0.0, c.max_iters = 300, c.timing_start_iter = 300, c.stop_overflow = 0.0, c.seed = seed, c.threads = 1;
    std::vector<uint8_t> expl(D.cell_w.size(), 0);
    double fin[3];
    int32_t rows = 0, stop = 0;
    if (tdpg_place(s, &c, expl.data(), nullptr, &rows, &stop, fin) != TDPG_OK)
        throw Error(tdpg_last_error_kind(), tdpg_last_error());
    std::vector<double> arr(v.n_pins);
    if (tdpg_sta(s, arr.data(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr) != TDPG_OK)
        throw Error(tdpg_last_error_kind(), tdpg_last_error());
    std::vector<double> a;
    a.reserve(D.endpoints.size());
    for (int e : D.endpoints) a.push_back(arr[e]);
    std::sort(a.begin(), a.end());
    const int n_ep = static_cast<int>(a.size());
    const int n_pass = std::clamp(static_cast<int>(std::lround((1.0 - fail_frac) * n_ep)), 0, n_ep);
    double clock;
    if (n_pass == 0) clock = std::max(a.front() * 0.95, 1e-9);
    else if (n_pass == n_ep) clock = a.back() * 1.05;
    else clock = 0.5 * (a[n_pass - 1] + a[n_pass]);
    D.clock = clock;
}

} // namespace

#define API_BEGIN try {
#define API_END                                                                   \
    return TDPG_OK;                                                               \
    }                                                                             \
    catch (const ::tdpg::Error& e) { return ::tdpg::api_fail(e.kind, e.what()); } \
    catch (const std::exception& e) { return ::tdpg::api_fail(TDPG_ERR_INTERNAL, e.what()); }

extern "C" {

int tdpg_generate(uint64_t seed, int32_t n_cells, int32_t n_registers, double avg_fanout, double fail_frac,
                  double r_unit, double c_unit, int32_t do_calibrate, tdpg_design** out)
{
    API_BEGIN
    *out = nullptr;
    auto d = std::make_unique<tdpg_design>();
    generate(seed, n_cells, n_registers, avg_fanout, fail_frac, r_unit, c_unit, *d);
    if (do_calibrate) calibrate(*d, seed, fail_frac);
    *out = d.release();
    API_END
}

int tdpg_design_view(tdpg_design* d, tdpg_netlist* view, const double** positions)
{
    API_BEGIN
    *view = d->view();
    if (positions) *positions = d->positions.data();
    API_END
}

int tdpg_design_set_clock(tdpg_design* d, double clock)
{
    API_BEGIN
    d->clock = clock;
    API_END
}

int tdpg_design_destroy(tdpg_design* d)
{
    API_BEGIN
    delete d;
    API_END
}

} // extern "C"
