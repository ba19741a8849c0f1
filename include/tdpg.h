/*
 * tdpg.h — C-ABI of the B200-native timing-driven global placement engine.
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes, returns
 * an int status (TDPG_OK == 0) and never lets a C++ exception cross the ABI.
 * On failure the thread-local message from tdpg_last_error() carries the
 * reference's exception text (proj/include/tdp/errors.hpp:9-42, e.g.
 * "non-finite value: ... at iteration N", "combinational cycle: ...") and
 * tdpg_last_error_kind() the exception class.
 *
 * One session = one design resident in HBM (structure-of-arrays netlist,
 * levelized timing-graph CSR, density grid, pin-pair ledger, optimizer
 * state).  Host pointers are read/written synchronously; functions named
 * *_dev operate on device-resident state only and are stream-ordered.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   tdpg_session_create      Netlist::finalize + build_timing_graph   src/netlist.cpp:5-21, src/timing_graph.cpp:49-138
 *   tdpg_pin_positions       pin_positions                            src/netlist.cpp:23-32
 *   tdpg_wirelength          wa_wirelength per net + hpwl_total       src/wirelength.cpp:49-58, :74-85
 *   tdpg_density             DensityGrid::evaluate                    src/density.cpp:66-158
 *   tdpg_pp_loss             pin_pair_loss                            src/pin_pairs.cpp:17-49
 *   tdpg_pp_set/get/update   PinPairWeights + update_pair_weights     include/tdp/pin_pairs.hpp:16, src/pin_pairs.cpp:7-15
 *   tdpg_objective           objective_and_gradient                   src/placer.cpp:275-343
 *   tdpg_adam_step           AdamState::step                          src/placer.cpp:345-356
 *   tdpg_sta                 run_sta (arrival/required/slack/tns/wns) src/sta.cpp:33-143
 *   tdpg_extract_endpoint    report_timing_endpoint (n, k)            src/paths.cpp:167-189
 *   tdpg_extract             report_timing_endpoint / report_timing   src/paths.cpp:136-189
 *   tdpg_k_worst             k_worst_paths_to                         src/paths.cpp:57-72
 *   tdpg_paths_hits          collect_pin_pairs                        src/paths.cpp:191-203
 *   tdpg_place               run_placement                            src/placer.cpp:358-484
 *   tdpg_generate            generate_synthetic                       src/generator.cpp:60-263
 */
#ifndef TDPG_H
#define TDPG_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TDPG_OK = 0,
    TDPG_ERR_PARSE = 1,       /* tdp::ParseError                       */
    TDPG_ERR_VALIDATION = 2,  /* tdp::ValidationError                  */
    TDPG_ERR_CYCLE = 3,       /* tdp::CycleError (a ValidationError)   */
    TDPG_ERR_ENDPOINT = 4,    /* tdp::EndpointError (a ValidationError) */
    TDPG_ERR_GRAPH = 5,       /* tdp::GraphError                       */
    TDPG_ERR_NONFINITE = 6,   /* tdp::NonFiniteError                   */
    TDPG_ERR_CUDA = 7,        /* CUDA runtime failure / no device      */
    TDPG_ERR_INTERNAL = 9
};

/* Flat structure-of-arrays view of tdp::Design (include/tdp/netlist.hpp:11-93).
 * Pin ids, cell ids and net ids are array indices, as in the reference.  */
typedef struct tdpg_netlist {
    int32_t n_cells;
    int32_t n_pins;
    int32_t n_nets;
    int32_t n_sources;
    int32_t n_endpoints;
    const double* cell_w;      /* [n_cells]   Cell::width                     */
    const double* cell_h;      /* [n_cells]   Cell::height                    */
    const double* cell_delay;  /* [n_cells]   Cell::delay                     */
    const uint8_t* cell_fixed; /* [n_cells]   Cell::is_fixed                  */
    const int32_t* pin_cell;   /* [n_pins]    owner cell id or -1 (terminal)  */
    const double* pin_term;    /* [2*n_pins]  terminal_pos (x, y)             */
    const double* pin_off;     /* [2*n_pins]  offset (x, y)                   */
    const uint8_t* pin_dir;    /* [n_pins]    0 = Input, 1 = Output           */
    const double* pin_cap;     /* [n_pins]    load_cap                        */
    const int32_t* net_start;  /* [n_nets+1]  CSR into net_pins               */
    const int32_t* net_pins;   /* [net_start[n_nets]] driver, then sinks      */
    const int32_t* sources;    /* [n_sources]                                 */
    const int32_t* endpoints;  /* [n_endpoints]                               */
    double clock_period;
    double r_unit;
    double c_unit;
    double core[4];            /* x_lo, y_lo, x_hi, y_hi                      */
    const char* const* pin_names; /* optional [n_pins], only for error text  */
} tdpg_netlist;

/* OptimizerConfig (include/tdp/placer.hpp:22-57), same field meaning. */
typedef struct tdpg_config {
    double gamma_frac;
    int32_t grid_nx, grid_ny;
    double target_density;
    double beta;
    int32_t pp_loss;           /* 0 quadratic, 1 linear                       */
    int32_t net_weighting;     /* bool                                        */
    int32_t m;
    double w0, w1;
    int32_t timing_start_iter;
    int32_t extraction;        /* 0 endpoint, 1 topn (both on the device)     */
    int32_t k;
    int32_t max_iters;
    double stop_overflow;
    double mu;
    double lambda0;            /* <= 0 selects gradient-norm balancing        */
    double lambda_max;
    double step0_frac;
    double step_decay;
    double adam_beta1, adam_beta2, adam_eps;
    uint64_t seed;
    double init_jitter_frac;
    int32_t threads;           /* accepted for drop-in parity; ignored        */
    int32_t density_model;     /* extension: 0 bin overflow (the reference), 1 electrostatic (DCT Poisson) */
} tdpg_config;

void tdpg_config_default(tdpg_config* cfg);

/* One TraceRow (include/tdp/placer.hpp:67-79). */
typedef struct tdpg_trace_row {
    int32_t iter;
    int32_t has_timing;
    double hpwl, overflow, tns, wns, wl_term, density_term, pp_term, lambda, beta_pp;
} tdpg_trace_row;

typedef struct tdpg_session tdpg_session;

const char* tdpg_last_error(void);
int tdpg_last_error_kind(void);
const char* tdpg_version(void);
int tdpg_device_count(void);

/* ---- session -------------------------------------------------------- */
int tdpg_session_create(const tdpg_netlist* nl, tdpg_session** out);
int tdpg_session_destroy(tdpg_session* s);
/* Timing graph facts: counts[0..3] = n_net_arcs, n_cell_arcs, n_levels, max_level;
 * level may be NULL, else [n_pins] level per pin (timing_graph.hpp:33). */
int tdpg_graph_info(tdpg_session* s, int32_t counts[4], int32_t* level);
/* arcs in reference id order: from/to/kind(0 net, 1 cell)/owner, each [n_arcs] (any may be NULL) */
int tdpg_graph_arcs(tdpg_session* s, int32_t* from, int32_t* to, int32_t* kind, int32_t* owner);

/* ---- positions ------------------------------------------------------ */
int tdpg_set_positions(tdpg_session* s, const double* cell_xy);   /* [2*n_cells] host */
int tdpg_get_positions(tdpg_session* s, double* cell_xy);
int tdpg_pin_positions(tdpg_session* s, double* pin_xy);          /* [2*n_pins] out    */
/* Pin::terminal_pos of the terminal pins ([2*n_pins], entries of cell pins ignored): lets one session
 * serve repeated per-net calls (wa_wirelength / hpwl_net on terminal pins, wirelength.hpp:21-23). */
int tdpg_set_terminal_positions(tdpg_session* s, const double* pin_xy);

/* ---- binary design file ------------------------------------------------ */
/* A scalable SoA file holding what the reference's design JSON holds (design_io.cpp:63-193 reads and
 * writes that JSON): netlist, constraints, positions and pos_explicit (layout: design.py save_bin).
 * info: counts = cells, pins, nets, net pins, sources, endpoints; has_pin_names may be NULL.
 * read: the caller allocates d's arrays from the counts (n_* fields set); the scalars are filled in;
 * pin names (optional) come back as one NUL-separated blob of at most blob_cap bytes. */
int tdpg_design_bin_info(const char* path, int64_t counts[6], int32_t* has_pin_names);
int tdpg_design_bin_read(const char* path, tdpg_netlist* d, double* positions, uint8_t* pos_explicit,
                         char* pin_name_blob, int64_t blob_cap);
int tdpg_design_bin_write(const char* path, const tdpg_netlist* d, const double* positions,
                          const uint8_t* pos_explicit, double default_cell_delay);

/* ---- objective terms (at the session's current positions) ----------- */
/* wl = sum_e w_e * WA_e, hpwl exact; pin_grad [2*n_pins] (w_e-scaled) may be NULL. */
int tdpg_wirelength(tdpg_session* s, double gamma, const double* net_w, double* wl, double* hpwl,
                    double* pin_grad);
/* hpwl_total on caller-provided pin positions ([2*n_pins], wirelength.cpp:74-85). */
int tdpg_hpwl_pins(tdpg_session* s, const double* pin_xy, double* hpwl);
/* DesignConstraints::core (the density grid follows it). */
int tdpg_set_core(tdpg_session* s, const double core[4]);
/* DesignConstraints timing fields (clock_period, r_unit, c_unit) used by the STA. */
int tdpg_set_constraints(tdpg_session* s, double clock_period, double r_unit, double c_unit);
/* DensityGrid(nx, ny, target_density) then evaluate; d_cell [2*n_cells] may be NULL. */
int tdpg_set_grid(tdpg_session* s, int32_t nx, int32_t ny, double target_density);
int tdpg_density(tdpg_session* s, double* value, double* overflow, double* d_cell);
/* Density model of one-off evaluations (tdpg_density / tdpg_objective); the placement loop takes
 * tdpg_config.density_model.  Electrostatic: value = 1/2 sum rho psi with L psi = rho - mean(rho). */
int tdpg_set_density_model(tdpg_session* s, int32_t model);
/* Last electrostatic evaluation's charge map rho and potential psi ([nx*ny], bin bx*ny + by). */
int tdpg_density_fields(tdpg_session* s, double* rho, double* psi);
/* Measurement aid (no reference counterpart): shared-memory atomics the density scatter issues at the
   session's positions: lo_hi[0] = low-limb atomics (one per non-zero footprint entry), lo_hi[1] = upper-limb
   atomics (Grid limbs - 1 per such entry). */
int tdpg_density_atomics(tdpg_session* s, int64_t lo_hi[2]);

/* ---- pin-pair ledger (PinPairWeights) ------------------------------- */
int tdpg_pp_set(tdpg_session* s, int64_t q, const int32_t* a, const int32_t* b, const double* w);
int tdpg_pp_size(tdpg_session* s, int64_t* q);
int tdpg_pp_get(tdpg_session* s, int32_t* a, int32_t* b, double* w);
/* update_pair_weights: hits in order; a <= b canonical. */
int tdpg_pp_update(tdpg_session* s, int64_t n_hits, const int32_t* a, const int32_t* b,
                   const double* path_slack, double wns, double w0, double w1);
int tdpg_pp_loss(tdpg_session* s, int32_t kind, double* value, double* d_pin /* [2*n_pins] or NULL */);

/* ---- full objective: objective_and_gradient ------------------------- */
/* terms[6] = value, wl_term, density_term, pp_term, hpwl, overflow. */
int tdpg_objective(tdpg_session* s, double gamma, double lambda, double beta, int32_t pp_kind,
                   const double* net_w, double terms[6], double* d_cell /* [2*n_cells] or NULL */);

/* AdamState::step on a host flat vector (exposed for the reference-shaped API/tests). */
int tdpg_adam_step(int64_t n, double* x, const double* grad, double* m, double* v, int32_t* t, double lr,
                   double beta1, double beta2, double eps);

/* ---- timing ----------------------------------------------------------- */
/* run_sta at current positions.  Any output pointer may be NULL. */
int tdpg_sta(tdpg_session* s, double* arr, double* req, double* slack, uint8_t* arr_known, uint8_t* req_known,
             double* tns, double* wns);
/* report_timing_endpoint(n, k=1) on the last STA; counts[0..3] = n_paths, total_pins,
 * unique_endpoints, unique_pin_pairs; candidates_generated = n_paths. */
int tdpg_extract_endpoint(tdpg_session* s, int32_t n, int32_t k, int64_t counts[4]);
/* report_timing_endpoint(n, k) (policy 0, paths.cpp:167-189) or report_timing(n) ("topn", policy 1,
 * paths.cpp:136-165) on the last STA; n <= 0 = every violated endpoint.  counts[0..4] = n_paths,
 * total_pins, unique_endpoints, unique_pin_pairs, candidates_generated. */
int tdpg_extract(tdpg_session* s, int32_t policy, int32_t n, int32_t k, int64_t counts[5]);
int tdpg_paths_candidates(tdpg_session* s, int64_t* candidates);
/* k_worst_paths_to(endpoint, k) (paths.cpp:57-72); TDPG_ERR_ENDPOINT for a non-endpoint.
 * start [k+1], pins [cap], slack [k]. */
int tdpg_k_worst(tdpg_session* s, int32_t endpoint, int32_t k, int32_t* n_paths, int32_t* start, int32_t* pins,
                 int32_t cap, double* slack);
int tdpg_paths_get(tdpg_session* s, int32_t* path_start /* [n_paths+1] */, int32_t* pins, double* slack);
/* Counts of the last extraction (same layout as tdpg_extract_endpoint's counts). */
int tdpg_paths_counts(tdpg_session* s, int64_t counts[4]);
/* collect_pin_pairs of the last extraction: number of hits, then fetch */
int tdpg_paths_hits(tdpg_session* s, int64_t* n_hits, int32_t* a, int32_t* b, double* slack);
/* STA on caller-provided pin positions ([2*n_pins], e.g. tdp::PinPositions) instead of the
 * cells' positions; cleared by tdpg_set_positions.  (run_sta takes PinPositions, sta.hpp:50) */
int tdpg_set_pin_positions(tdpg_session* s, const double* pin_xy);
/* Download the last STA without recomputing it. */
int tdpg_sta_fetch(tdpg_session* s, double* arr, double* req, double* slack, uint8_t* arr_known,
                   uint8_t* req_known, double* tns, double* wns);
/* PathEnumerator::path_to(pin, rank) (paths.hpp:54): *n_pins = 0 when the pin has no rank-th path. */
int tdpg_path_to(tdpg_session* s, int32_t pin, int32_t rank, int32_t* pins, int32_t cap, int32_t* n_pins,
                 double* delay);
/* Device-timed duration (ms) of the last STA / extraction call, CUDA events. */
int tdpg_last_timing_ms(tdpg_session* s, double* sta_ms, double* extract_ms);

/* ---- the placement loop: run_placement ------------------------------ */
/* TimingRoundObserver (placer.hpp:134): called after every timing round with the iteration;
 * tdpg_sta_fetch / tdpg_paths_get / tdpg_paths_hits read that round's annotation and report. */
typedef void (*tdpg_round_cb)(void* user, int32_t iter);
int tdpg_set_round_callback(tdpg_session* s, tdpg_round_cb cb, void* user);
/* pos_explicit [n_cells] (bool) marks cells whose coordinates came from the file;
 * positions are the session's current positions on entry and the result on exit.
 * trace may be NULL; else capacity max_iters rows.  final[3] = tns, wns, hpwl. */
int tdpg_place(tdpg_session* s, const tdpg_config* cfg, const uint8_t* pos_explicit, tdpg_trace_row* trace,
               int32_t* n_rows, int32_t* stop_overflow, double final_[3]);

/* ---- bench/driver hooks (device-resident, no host copies) ------------ */
/* Prepare an iteration engine (grid, gamma, lambda schedule) for tdpg_iterate_dev. */
int tdpg_engine_init(tdpg_session* s, const tdpg_config* cfg, const uint8_t* pos_explicit);
/* Run n GP iterations (timing refresh per schedule) fully on device; optional device time. */
int tdpg_iterate_dev(tdpg_session* s, int32_t n_iters, double* device_ms);
int tdpg_engine_stats(tdpg_session* s, int32_t* iter, int32_t* refreshes, int64_t* launches);
/* Device time spent in timing refreshes so far (CUDA events), the last one, and the ledger size. */
int tdpg_engine_times(tdpg_session* s, double* refresh_ms_total, double* last_refresh_ms, int64_t* ledger_pairs);
/* Paths (and their pins) extracted by the engine's timing refreshes since tdpg_engine_init. */
int tdpg_engine_paths(tdpg_session* s, int64_t* paths, int64_t* path_pins);
/* One iteration through host buffers (positions in, positions + trace row out) — the e2e path. */
int tdpg_step_host(tdpg_session* s, const double* xy_in, double* xy_out, tdpg_trace_row* row);
/* Per-kernel device time (ms) of one iteration of each kind, measured with events. */
int tdpg_profile_iteration(tdpg_session* s, int32_t reps, double* out_ms, int32_t n_out, char* names, int32_t name_len);

/* ---- single-design multi-GPU: partitioned gradient + NCCL all-reduces ------------
 * Nets (WA entries and the net-arc pin pairs fused into WA) are split into contiguous WA-block ranges
 * balanced by net-pin entries, and the movable cells into contiguous slices of the spatial order.  Each
 * rank rasterises its cells into the int64 fixed-point grid, which is sum-all-reduced (exact: every rank
 * holds bitwise the single-GPU grid); bins are replicated; each rank folds its entries plus lambda x the
 * density gradient of its cells into a partial cell gradient, and one NCCL sum all-reduce over
 * [partial d_cell | WA, HPWL, PP block partials] completes gradient and objective terms on every rank;
 * Adam and timing refreshes are replicated (run_placement semantics kept).
 * tdpg_partition_plan: bounds [world+1] = per-rank WA block ranges, rank_entries [world] (host only).   */
int tdpg_partition_plan(int32_t n_nets, const int32_t* net_start, int32_t world, int32_t* bounds,
                        int64_t* rank_entries);
int tdpg_set_partition(tdpg_session* s, int32_t rank, int32_t world); /* no communicator: split-phase API */
int tdpg_comm_unique_id(uint8_t id[128]);                            /* ncclGetUniqueId (rank 0)        */
int tdpg_comm_init(tdpg_session* s, int32_t rank, int32_t world, const uint8_t id[128]);
/* Split-phase partitioned iteration (the caller reduces, e.g. tests on one GPU): tdpg_part_density runs
 * the scheduled refresh / re-sort and this rank's scatter and returns its grid (n_bins int64); phase A takes
 * the grid summed over ranks and returns this rank's all-reduce buffer (n_red doubles); phase B takes the
 * element-wise sum of those over ranks. */
int tdpg_part_density(tdpg_session* s, int64_t* acc, int64_t* n_bins);
int tdpg_part_step_a(tdpg_session* s, const int64_t* acc, double* red, int64_t* n_red);
int tdpg_part_step_b(tdpg_session* s, const double* red);
/* Device time (ms, averaged over iters) of the two collectives of a partitioned iteration run alone:
 * ms[0] the int64 density grid, ms[1] the gradient buffer of n_red doubles.  Collective: every rank calls. */
int tdpg_comm_bench(tdpg_session* s, int32_t iters, int64_t n_red, double ms[2]);

/* ---- synthetic designs (generate_synthetic semantics) ---------------- */
typedef struct tdpg_design tdpg_design;
/* Builds the netlist exactly as the reference generator (same mt19937_64 stream);
 * calibrate != 0 runs the 300-iteration coarse placement on the GPU to set the clock. */
int tdpg_generate(uint64_t seed, int32_t n_cells, int32_t n_registers, double avg_fanout, double fail_frac,
                  double r_unit, double c_unit, int32_t calibrate, tdpg_design** out);
int tdpg_design_view(tdpg_design* d, tdpg_netlist* view, const double** positions);
int tdpg_design_set_clock(tdpg_design* d, double clock_period);
int tdpg_design_destroy(tdpg_design* d);

#ifdef __cplusplus
}
#endif

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#endif /* TDPG_H */
