// tdp_api.hpp — the reference's C++ operator API (namespace tdp, /root/reference/proj/include/tdp/*.hpp)
// re-declared over the B200 engine.  Callers of the reference keep compiling unchanged: every
// reference header name (tdp/sta.hpp, tdp/paths.hpp, ...) includes this file.  Types are plain data
// with the reference's field names; the functions run on the GPU through the C-ABI (include/tdpg.h).
// Every hot-path function runs on the device (k > 1 paths and the topn policy included); the host keeps
// only input/output glue (config JSON, CSV/JSON serialisation, type conversion).
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <functional>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace tdp {

// ---- geometry (geometry.hpp:8-40) ----------------------------------------------------------
struct Point {
    double x = 0.0, y = 0.0;
    bool operator==(const Point&) const = default;
    Point operator+(const Point& o) const { return {x + o.x, y + o.y}; }
    Point operator-(const Point& o) const { return {x - o.x, y - o.y}; }
};

inline double manhattan(const Point& a, const Point& b) { return std::abs(a.x - b.x) + std::abs(a.y - b.y); }

struct Rect {
    double x_lo = 0.0, y_lo = 0.0, x_hi = 0.0, y_hi = 0.0;
    bool operator==(const Rect&) const = default;
    double width() const { return x_hi - x_lo; }
    double height() const { return y_hi - y_lo; }
    double span() const { return width() > height() ? width() : height(); }
    bool contains(const Rect& r) const { return r.x_lo >= x_lo && r.y_lo >= y_lo && r.x_hi <= x_hi && r.y_hi <= y_hi; }
    bool nondegenerate() const { return x_hi > x_lo && y_hi > y_lo; }
};

// ---- errors (errors.hpp:9-42): same classes, same what() prefixes ---------------------------
struct ParseError : std::runtime_error {
    explicit ParseError(const std::string& m) : std::runtime_error("parse error: " + m) {}
};
struct ValidationError : std::runtime_error {
    explicit ValidationError(const std::string& m) : std::runtime_error("validation error: " + m) {}
};
struct CycleError : ValidationError {
    explicit CycleError(const std::string& m) : ValidationError("combinational cycle: " + m) {}
};
struct EndpointError : ValidationError {
    explicit EndpointError(const std::string& m) : ValidationError(m) {}
};
struct GenerationError : ValidationError {
    explicit GenerationError(const std::string& m) : ValidationError(m) {}
};
struct MismatchError : ValidationError {
    explicit MismatchError(const std::string& m) : ValidationError(m) {}
};
struct GraphError : std::runtime_error {
    explicit GraphError(const std::string& m) : std::runtime_error("graph error: " + m) {}
};
struct NonFiniteError : std::runtime_error {
    explicit NonFiniteError(const std::string& m) : std::runtime_error("non-finite value: " + m) {}
};

// ---- netlist (netlist.hpp:11-93) ---------------------------------------------------------------
enum class PinDir { Input, Output };
constexpr int kTerminal = -1;

struct Cell {
    std::string name;
    double width = 0.0, height = 0.0;
    bool is_fixed = false;
    double delay = 1.0;
    bool operator==(const Cell&) const = default;
};

struct Pin {
    std::string name;
    int cell = kTerminal;
    Point terminal_pos, offset;
    PinDir dir = PinDir::Input;
    double load_cap = 0.0;
    bool is_terminal() const { return cell == kTerminal; }
    bool operator==(const Pin&) const = default;
};

struct Net {
    std::string name;
    int driver = -1;
    std::vector<int> sinks;
    bool operator==(const Net&) const = default;
};

struct DesignConstraints {
    double clock_period = 0.0, r_unit = 0.0, c_unit = 0.0, default_cell_delay = 1.0;
    Rect core;
    bool operator==(const DesignConstraints&) const = default;
};

struct Netlist {
    std::vector<Cell> cells;
    std::vector<Pin> pins;
    std::vector<Net> nets;
    std::vector<int> sources, endpoints;
    std::vector<std::vector<int>> cell_pins;
    std::vector<int> pin_net;
    std::vector<bool> pin_is_source, pin_is_endpoint;
    void finalize();
    bool operator==(const Netlist& o) const
    {
        return cells == o.cells && pins == o.pins && nets == o.nets && sources == o.sources && endpoints == o.endpoints;
    }
};

struct Design {
    Netlist netlist;
    DesignConstraints constraints;
    std::vector<Point> positions;
    std::vector<bool> pos_explicit;
    bool operator==(const Design&) const = default;
};

using PinPositions = std::vector<Point>;
PinPositions pin_positions(const Netlist& netlist, const std::vector<Point>& cell_pos);

// ---- timing graph (timing_graph.hpp:10-43) -----------------------------------------------------
enum class ArcKind { NetArc, CellArc };
struct Arc {
    int from = -1, to = -1;
    ArcKind kind = ArcKind::NetArc;
    int owner = -1;
};
struct TimingGraph {
    int num_pins = 0;
    std::vector<Arc> arcs;
    std::vector<std::vector<int>> in_arcs, out_arcs;
    std::vector<int> sources, endpoints;
    std::vector<bool> is_source, is_endpoint;
    std::vector<int> level;
    std::vector<std::vector<int>> levels;
    bool levelized = false;
    int num_net_arcs = 0, num_cell_arcs = 0;
};
TimingGraph build_timing_graph(const Netlist& netlist);

// ---- STA (sta.hpp:12-51) -------------------------------------------------------------------
struct TimingAnnotation {
    std::vector<double> arr, req, slack;
    std::vector<bool> arr_known, req_known;
    std::vector<std::pair<int, double>> endpoint_slacks;
    double tns = 0.0, wns = 0.0;
};
double net_delay(const Point& source_pos, const Point& sink_pos, double sink_cap, const DesignConstraints& constraints);
double arc_delay(const Arc& arc, const Netlist& netlist, const PinPositions& pos, const DesignConstraints& constraints);
std::vector<double> propagate_arrival(const TimingGraph& graph, const Netlist& netlist, const PinPositions& pos,
                                      const DesignConstraints& constraints, std::vector<bool>* arr_known = nullptr,
                                      int threads = 1);
std::vector<double> propagate_required(const TimingGraph& graph, const Netlist& netlist, const PinPositions& pos,
                                       const DesignConstraints& constraints, std::vector<bool>* req_known = nullptr,
                                       int threads = 1);
TimingAnnotation compute_slacks(const TimingGraph& graph, std::vector<double> arrivals, std::vector<double> required,
                                std::vector<bool> arr_known, std::vector<bool> req_known);
std::pair<double, double> tns_wns(const std::vector<std::pair<int, double>>& endpoint_slacks);
TimingAnnotation run_sta(const TimingGraph& graph, const Netlist& netlist, const PinPositions& pos,
                         const DesignConstraints& constraints, int threads = 1);

// ---- paths (paths.hpp:15-110) ------------------------------------------------------------------
struct CriticalPath {
    std::vector<int> pins;
    double slack = 0.0;
    bool operator==(const CriticalPath&) const = default;
};
struct ExtractionReport {
    std::string policy;
    int n = 0, k = 0;
    std::vector<CriticalPath> paths;
    int unique_endpoints = 0, unique_pin_pairs = 0;
    long long candidates_generated = 0;
    double elapsed_ms = 0.0;
};
struct PairHit {
    std::pair<int, int> pair;
    double path_slack = 0.0;
};

class PathEnumerator {
  public:
    PathEnumerator(const TimingGraph& graph, const Netlist& netlist, const PinPositions& pos,
                   const DesignConstraints& constraints);
    struct Record {
        double delay = 0.0;
        std::vector<int> pins;
    };
    // any rank: rank 0 from the k = 1 backtrace, rank > 0 from the device k-best lists (csrc/kpaths.cu)
    const Record* path_to(int pin, std::size_t rank);

  private:
    const TimingGraph& graph_;
    const Netlist& netlist_;
    const PinPositions& pos_;
    const DesignConstraints& constraints_;
    std::map<std::pair<int, std::size_t>, Record> found_;
    std::map<std::pair<int, std::size_t>, bool> none_;
};

std::vector<CriticalPath> k_worst_paths_to(const TimingGraph& graph, const Netlist& netlist, const PinPositions& pos,
                                           const DesignConstraints& constraints, const TimingAnnotation& annotation,
                                           int endpoint, int k);
ExtractionReport report_timing(const TimingGraph& graph, const Netlist& netlist, const PinPositions& pos,
                               const DesignConstraints& constraints, const TimingAnnotation& annotation, int n,
                               int threads = 1);
ExtractionReport report_timing_endpoint(const TimingGraph& graph, const Netlist& netlist, const PinPositions& pos,
                                        const DesignConstraints& constraints, const TimingAnnotation& annotation,
                                        int n, int k, int threads = 1);
std::vector<PairHit> collect_pin_pairs(const Netlist& netlist, const std::vector<CriticalPath>& paths);

// ---- pin pairs (pin_pairs.hpp:16-40) -------------------------------------------------------------
using PinPairWeights = std::map<std::pair<int, int>, double>;
void update_pair_weights(PinPairWeights& weights, const std::vector<PairHit>& hits, double wns, double w0, double w1);
enum class PairLossKind { Quadratic, Linear };
struct PinPairLossResult {
    double value = 0.0;
    std::vector<Point> d_pin;
};
PinPairLossResult pin_pair_loss(const PinPairWeights& weights, const PinPositions& pins, std::size_t num_pins,
                                PairLossKind kind = PairLossKind::Quadratic);

// ---- wirelength (wirelength.hpp:11-26) -------------------------------------------------------------
struct NetTermGrad {
    double value = 0.0;
    std::vector<Point> d_pin;
};
NetTermGrad wa_wirelength(std::span<const Point> pin_pos, double gamma);
double hpwl_net(std::span<const Point> pin_pos);
double hpwl_total(const Netlist& netlist, const PinPositions& pos);

// ---- density (density.hpp:10-37) -----------------------------------------------------------------
struct DensityResult {
    double value = 0.0, overflow = 0.0;
    std::vector<Point> d_cell;
};
class DensityGrid {
  public:
    DensityGrid(const Netlist& netlist, const Rect& core, int nx, int ny, double target_density);
    DensityResult evaluate(const Netlist& netlist, const std::vector<Point>& cell_pos, int threads = 1) const;
    int nx() const { return nx_; }
    int ny() const { return ny_; }
    const Rect& core() const { return core_; }
    double target_density() const { return target_density_; }

  private:
    Rect core_;
    int nx_, ny_;
    double target_density_;
};

// ---- placer (placer.hpp:17-143) --------------------------------------------------------------------
enum class ExtractionPolicy { Endpoint, TopN };
struct OptimizerConfig {
    std::string name = "default";
    double gamma_frac = 0.01;
    int grid_nx = 16, grid_ny = 16;
    double target_density = 0.6, beta = 2.5e-5;
    PairLossKind pp_loss = PairLossKind::Quadratic;
    bool net_weighting = false;
    int m = 15;
    double w0 = 10.0, w1 = 0.2;
    int timing_start_iter = 500;
    ExtractionPolicy extraction = ExtractionPolicy::Endpoint;
    int k = 1, max_iters = 1500;
    double stop_overflow = 0.0, mu = 1.05, lambda0 = 0.0, lambda_max = 1e8, step0_frac = 0.01, step_decay = 0.999;
    double adam_beta1 = 0.9, adam_beta2 = 0.999, adam_eps = 1e-8;
    std::uint64_t seed = 1;
    double init_jitter_frac = 0.02;
    int threads = 1;
};
struct TraceRow {
    int iter = 0;
    double hpwl = 0.0, overflow = 0.0;
    bool has_timing = false;
    double tns = 0.0, wns = 0.0, wl_term = 0.0, density_term = 0.0, pp_term = 0.0, lambda = 0.0, beta_pp = 0.0;
};
/// JSON round-trip with unknown-key rejection (placer.hpp:58-65, placer.cpp:107-232): host-side
/// configuration I/O, same keys, messages and formatting as the reference.
OptimizerConfig config_from_json(const std::string& text);
std::string config_to_json(const OptimizerConfig& config);
OptimizerConfig load_config(const std::string& path);
void save_config(const OptimizerConfig& config, const std::string& path);
using MetricTrace = std::vector<TraceRow>;
std::string metrics_to_csv(const MetricTrace& trace);
struct ObjectiveResult {
    double value = 0.0, wl_term = 0.0, density_term = 0.0, pp_term = 0.0, hpwl = 0.0, overflow = 0.0;
    std::vector<Point> d_cell;
};
ObjectiveResult objective_and_gradient(const Netlist& netlist, const std::vector<Point>& cell_pos,
                                       const DensityGrid& grid, const PinPairWeights& weights,
                                       const std::vector<double>& net_weights, double gamma, double lambda,
                                       double beta, PairLossKind pp_loss = PairLossKind::Quadratic, int threads = 1);
std::vector<double> apply_net_weights(const TimingAnnotation& annotation, const Netlist& netlist);
struct AdamState {
    explicit AdamState(std::size_t n) : m(n, 0.0), v(n, 0.0) {}
    void step(std::vector<double>& x, const std::vector<double>& grad, double lr, double beta1, double beta2,
              double eps);
    std::vector<double> m, v;
    int t = 0;
};
struct PlacementOutcome {
    std::vector<Point> positions;
    MetricTrace trace;
    PinPairWeights pair_weights;
    TimingAnnotation final_timing;
    int iterations = 0;
    std::string stop_reason;
};
using TimingRoundObserver =
    std::function<void(int iter, const TimingAnnotation& annotation, const ExtractionReport& report)>;
PlacementOutcome run_placement(const Design& design, const OptimizerConfig& config,
                               const TimingRoundObserver& observer = {});
std::string weights_to_json(const PinPairWeights& weights, const Netlist& netlist);

// ---- ablation harness (include/tdp/compare.hpp) ------------------------------------------------------
struct CompareRow {
    std::string config_name;
    bool ok = false;
    std::string error;
    double tns = 0.0, wns = 0.0, hpwl = 0.0, runtime_s = 0.0;
    int unique_endpoints = 0, unique_pin_pairs = 0;
    long long candidates_generated = 0;
};
struct CompareReport {
    std::vector<CompareRow> rows;
};
CompareReport run_compare(const Design& design, const std::vector<OptimizerConfig>& configs, bool parallel = false);
std::string compare_to_csv(const CompareReport& report);
std::string compare_to_table(const CompareReport& report);

} // namespace tdp
