/*
 * tdp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's timing-driven GP hot path
 * (/root/reference/proj/src/*.cpp), used by tests/ as the parity checker and by
 * bench.py's cpu_baseline leg.  The product (paper_2503_11674_b200/) never
 * links, loads or calls it.  Every function cites the reference lines it
 * restates.  Pinned against the reference's own known-answer tests
 * (tests/test_oracle_golden.py) and against the reference compiled from its
 * sources (oracle/_ref, tests/test_oracle_vs_ref.py).
 */
#ifndef TDP_ORACLE_H
#define TDP_ORACLE_H

#include <stdint.h>

#include "tdpg.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
int orc_last_error_kind(void);

/* Stateless kernels ---------------------------------------------------- */
void orc_pin_positions(const tdpg_netlist* nl, const double* cell_xy, double* pin_xy);
double orc_wa(int32_t n, const double* xy, double gamma, double* grad);
double orc_hpwl_total(const tdpg_netlist* nl, const double* pin_xy);
int orc_density(const tdpg_netlist* nl, const double* cell_xy, int32_t nx, int32_t ny, double target_density,
                double* value, double* overflow, double* d_cell);
double orc_pp_loss(int64_t q, const int32_t* a, const int32_t* b, const double* w, int64_t n_pins,
                   const double* pin_xy, int32_t kind, double* d_pin);
void orc_adam_step(int64_t n, double* x, const double* g, double* m, double* v, int32_t* t, double lr, double b1,
                   double b2, double eps);
/* objective_and_gradient with an explicit ledger (sorted by (a, b)). */
int orc_objective(const tdpg_netlist* nl, const double* cell_xy, int32_t nx, int32_t ny, double td, double gamma,
                  double lambda, double beta, int32_t kind, const double* net_w, int64_t q, const int32_t* a,
                  const int32_t* b, const double* w, double terms[6], double* d_cell);

/* Session: timing graph + ledger + last extraction -------------------- */
void* orc_create(const tdpg_netlist* nl); /* NULL on error (orc_last_error) */
void orc_destroy(void* h);
int orc_graph_info(void* h, int32_t counts[4], int32_t* level, int32_t* arc_from, int32_t* arc_to,
                   int32_t* arc_kind, int32_t* arc_owner);
int orc_sta(void* h, const double* cell_xy, double* arr, double* req, double* slack, uint8_t* ak, uint8_t* rk,
            double* tns, double* wns);
/* report_timing_endpoint(n, k = 1) after run_sta at cell_xy; n <= 0 = all violated.
 * counts = n_paths, total_pins, unique_endpoints, unique_pin_pairs */
int orc_extract(void* h, const double* cell_xy, int32_t n, int64_t counts[4]);
/* same, counts[4] = candidates_generated */
int orc_extract5(void* h, const double* cell_xy, int32_t n, int64_t counts[5]);
/* report_timing_endpoint(n, k) (policy 0) or report_timing(n) (policy 1, "topn") through the
 * lazy PathEnumerator; n <= 0 is NOT special here (the reference's n). counts[4] = candidates. */
int orc_extract_policy(void* h, const double* cell_xy, int32_t policy, int32_t n, int32_t k, int64_t counts[5]);
/* k_worst_paths_to(endpoint, k); results via orc_paths_get. */
int orc_k_worst(void* h, const double* cell_xy, int32_t endpoint, int32_t k, int32_t* n_paths);
int orc_paths_get(void* h, int32_t* start, int32_t* pins, double* slack, int64_t* n_hits);
int orc_hits_get(void* h, int32_t* a, int32_t* b, double* slack);
int orc_pp_set(void* h, int64_t q, const int32_t* a, const int32_t* b, const double* w);
int orc_pp_update(void* h, int64_t n, const int32_t* a, const int32_t* b, const double* s, double wns, double w0,
                  double w1, int64_t* q_out);
int orc_pp_get(void* h, int32_t* a, int32_t* b, double* w);
/* run_placement; extraction must be endpoint/k = 1. final = tns, wns, hpwl. */
int orc_jitter(void* h, const double* init_xy, const uint8_t* pos_explicit, const tdpg_config* cfg, double* out_xy);
int orc_place(void* h, const double* init_xy, const uint8_t* pos_explicit, const tdpg_config* cfg, double* out_xy,
              tdpg_trace_row* trace, int32_t* n_rows, int32_t* stop_overflow, double final_[3]);

void orc_config_default(tdpg_config* cfg);

/* generate_synthetic's netlist (generator.cpp:60-244) without the clock calibration (clock 1.0);
 * tdp_oracle_gen.c.  orc_design_view points into the handle's arrays. */
int orc_generate(uint64_t seed, int32_t n_cells, int32_t n_registers, double avg_fanout, double fail_frac,
                 double r_unit, double c_unit, void** out);
int orc_design_view(void* d, tdpg_netlist* view, const double** positions);
void orc_design_destroy(void* d);

/* mt19937_64 (the C++ standard's engine), exposed for tests. */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;
void orc_mt64_seed(orc_mt64* r, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* r);

#ifdef __cplusplus
}
#endif
#endif
