/*
 * tdp_oracle_gen.c — TEST INFRASTRUCTURE ONLY (see tdp_oracle.h).
 *
 * Plain-C restatement of the reference's synthetic netlist generator,
 * generate_synthetic (/root/reference/proj/src/generator.cpp:60-244), without
 * the clock calibration (generator.cpp:246-260 runs run_placement; callers set
 * the clock themselves).  Same mt19937_64 stream and draw order
 * (include/tdp/rng.hpp:13-28), so the netlist is the reference's byte for byte
 * (tests/test_oracle_gen.py pins it against oracle/_ref).  Two deliberate
 * differences, both invisible in the output:
 *   - the reference's quadratic scans (idle-driver list per primary output,
 *     generator.cpp:198-201; connection rescan per driver, :209-217) are a
 *     Fenwick tree over idle drivers and a per-driver bucket of connections;
 *   - the register slot index (r + 1) * total_slots / (n_regs + 1)
 *     (generator.cpp:90) is computed in 64 bits: the reference's int product
 *     overflows above ~1.4e5 cells.
 * It exists so that the CPU reference arm of bench.py builds the 1M-cell
 * design without loading the product library.
 */
#include "tdp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { kLocalityWindow = 30, kMaxDepth = 20 };
static const double kLocalityProb = 0.7;

typedef struct {
    int32_t n_cells, n_pins, n_nets, n_sources, n_endpoints;
    double *cell_w, *cell_h, *cell_delay, *pin_term, *pin_off, *pin_cap, *positions;
    uint8_t *cell_fixed, *pin_dir;
    int32_t *pin_cell, *net_start, *net_pins, *sources, *endpoints;
    double clock, r_unit, c_unit, core[4];
} orc_design;

/* rng.hpp:13-28 */
static double g_unit(orc_mt64* r) { return (double)(orc_mt64_next(r) >> 11) * 0x1.0p-53; }
static double g_uniform(orc_mt64* r, double lo, double hi) { return lo + (hi - lo) * g_unit(r); }
static int64_t g_int(orc_mt64* r, int64_t lo, int64_t hi)
{
    const uint64_t range = (uint64_t)(hi - lo) + 1;
    return lo + (int64_t)(orc_mt64_next(r) % range);
}

/* generator.cpp:22-27 */
static int pick_driver_index(orc_mt64* r, int n)
{
    if (n > kLocalityWindow && g_unit(r) < kLocalityProb) return (int)g_int(r, n - kLocalityWindow, n - 1);
    return (int)g_int(r, 0, n - 1);
}

typedef struct {
    orc_design* D;
    int64_t cap_pins;
    int32_t *drv, *sink_cnt, *depth, *shallow; /* drivers (pin ids), per-driver sink count / depth */
    int n_drv, n_shallow;
    int32_t *conn_sink, *conn_drv; /* connections in creation order (sink pin, driver index) */
    int64_t n_conn;
} gen_state;

static int add_pin(gen_state* g, int32_t cell, double tx, double ty, double ox, double oy, uint8_t dir, double cap)
{
    orc_design* D = g->D;
    const int p = D->n_pins++;
    D->pin_cell[p] = cell;
    D->pin_term[2 * p] = tx, D->pin_term[2 * p + 1] = ty;
    D->pin_off[2 * p] = ox, D->pin_off[2 * p + 1] = oy;
    D->pin_dir[p] = dir;
    D->pin_cap[p] = cap;
    return p;
}

static void new_driver(gen_state* g, int pin, int depth)
{
    if (depth < kMaxDepth) g->shallow[g->n_shallow++] = g->n_drv; /* drivers below the bound, in order */
    g->drv[g->n_drv] = pin, g->sink_cnt[g->n_drv] = 0, g->depth[g->n_drv] = depth;
    ++g->n_drv;
}

static void add_conn(gen_state* g, int sink, int idx)
{
    g->conn_sink[g->n_conn] = sink, g->conn_drv[g->n_conn] = idx;
    ++g->n_conn;
    ++g->sink_cnt[idx];
}

/* generator.cpp:32-43: 16 biased tries, then a uniform pick among drivers below the depth bound
 * (the reference rebuilds that list each time; it only grows, in driver order, so it is kept). */
static int pick_shallow(gen_state* g, orc_mt64* r)
{
    for (int a = 0; a < 16; ++a) {
        const int idx = pick_driver_index(r, g->n_drv);
        if (g->depth[idx] < kMaxDepth) return idx;
    }
    return g->shallow[g_int(r, 0, g->n_shallow - 1)];
}

/* Fenwick tree over driver indices: k-th idle driver in O(log n). */
typedef struct { int32_t* t; int n, top; } fenwick;
static void fw_add(fenwick* f, int i, int d)
{
    for (++i; i <= f->n; i += i & -i) f->t[i] += d;
}
static int fw_kth(const fenwick* f, int k) /* 0-based */
{
    int pos = 0;
    for (int step = f->top; step; step >>= 1)
        if (pos + step <= f->n && f->t[pos + step] <= k) pos += step, k -= f->t[pos];
    return pos;
}

void orc_design_destroy(void* h)
{
    orc_design* D = (orc_design*)h;
    if (!D) return;
    free(D->cell_w), free(D->cell_h), free(D->cell_delay), free(D->pin_term), free(D->pin_off);
    free(D->pin_cap), free(D->positions), free(D->cell_fixed), free(D->pin_dir), free(D->pin_cell);
    free(D->net_start), free(D->net_pins), free(D->sources), free(D->endpoints);
    free(D);
}

int orc_generate(uint64_t seed, int32_t n_cells, int32_t n_registers, double avg_fanout, double fail_frac,
                 double r_unit, double c_unit, void** out)
{
    *out = NULL;
    /* generator.cpp:62-67 */
    if (n_cells < 1) return TDPG_ERR_VALIDATION;
    if (!(avg_fanout > 0.0) || avg_fanout > n_cells) return TDPG_ERR_VALIDATION;
    if (!(fail_frac >= 0.0 && fail_frac <= 1.0)) return TDPG_ERR_VALIDATION;
    if (!(r_unit > 0.0 && c_unit > 0.0)) return TDPG_ERR_VALIDATION;

    /* generator.cpp:69-79 */
    const int n_regs = n_registers >= 0 ? n_registers : n_cells / 10;
    const int n_pi = n_cells / 20 > 2 ? n_cells / 20 : 2;
    const int n_po = n_pi;
    const int n_drivers_total = n_pi + n_cells + n_regs;
    double mean_in = (avg_fanout * n_drivers_total - n_regs - n_po) / n_cells;
    mean_in = mean_in < 1.0 ? 1.0 : (mean_in > 8.0 ? 8.0 : mean_in);
    const int total_slots = n_cells + n_regs;
    const int max_in = (int)mean_in + 1;

    orc_design* D = (orc_design*)calloc(1, sizeof *D);
    gen_state g = {0};
    g.D = D;
    g.cap_pins = (int64_t)n_pi + n_po + (int64_t)total_slots * (max_in + 1);
    const size_t P = (size_t)g.cap_pins, S = (size_t)total_slots;
    D->cell_w = malloc(S * sizeof(double)), D->cell_h = malloc(S * sizeof(double));
    D->cell_delay = malloc(S * sizeof(double)), D->cell_fixed = calloc(S, 1);
    D->positions = malloc(2 * S * sizeof(double));
    D->pin_cell = malloc(P * sizeof(int32_t)), D->pin_term = malloc(2 * P * sizeof(double));
    D->pin_off = malloc(2 * P * sizeof(double)), D->pin_dir = malloc(P), D->pin_cap = malloc(P * sizeof(double));
    D->sources = malloc(((size_t)n_pi + n_regs) * sizeof(int32_t));
    D->endpoints = malloc(((size_t)n_po + n_regs) * sizeof(int32_t));
    const size_t ND = (size_t)n_drivers_total;
    g.drv = malloc(ND * sizeof(int32_t)), g.sink_cnt = malloc(ND * sizeof(int32_t));
    g.depth = malloc(ND * sizeof(int32_t)), g.shallow = malloc(ND * sizeof(int32_t));
    g.conn_sink = malloc(P * sizeof(int32_t)), g.conn_drv = malloc(P * sizeof(int32_t));
    uint8_t* slot_is_reg = calloc(S, 1);

    orc_mt64 rng;
    orc_mt64_seed(&rng, seed);
    for (int r = 0; r < n_regs; ++r) slot_is_reg[((int64_t)r + 1) * total_slots / (n_regs + 1)] = 1; /* :88-90 */

    /* primary inputs: terminals on the left edge, unit-square coordinates rescaled below (:107-121) */
    for (int i = 0; i < n_pi; ++i) {
        const int p = add_pin(&g, -1, 0.0, (i + 0.5) / n_pi, 0.0, 0.0, 1, 0.0);
        D->sources[D->n_sources++] = p;
        new_driver(&g, p, 0);
    }
    /* slots (:124-183); each draw in the reference's statement order */
    for (int slot = 0; slot < total_slots; ++slot) {
        const double w = g_uniform(&rng, 400.0, 800.0);
        const double h = g_uniform(&rng, 400.0, 800.0);
        const double delay = g_uniform(&rng, 0.5, 1.5);
        const int cell = D->n_cells;
        if (slot_is_reg[slot]) {
            const double dx = g_uniform(&rng, 0.0, w);
            const double dy = g_uniform(&rng, 0.0, h);
            const double cap = g_uniform(&rng, 0.5, 2.0);
            const int d_pin = add_pin(&g, cell, 0.0, 0.0, dx, dy, 0, cap);
            D->endpoints[D->n_endpoints++] = d_pin;
            add_conn(&g, d_pin, pick_driver_index(&rng, g.n_drv));
            const double qx = g_uniform(&rng, 0.0, w);
            const double qy = g_uniform(&rng, 0.0, h);
            const int q_pin = add_pin(&g, cell, 0.0, 0.0, qx, qy, 1, 0.0);
            D->sources[D->n_sources++] = q_pin;
            new_driver(&g, q_pin, 0);
        } else {
            const int n_in = (int)mean_in + (g_unit(&rng) < mean_in - floor(mean_in) ? 1 : 0);
            int depth_in = 0;
            for (int i = 0; i < (n_in > 1 ? n_in : 1); ++i) {
                const double dx = g_uniform(&rng, 0.0, w);
                const double dy = g_uniform(&rng, 0.0, h);
                const double cap = g_uniform(&rng, 0.5, 2.0);
                const int pin = add_pin(&g, cell, 0.0, 0.0, dx, dy, 0, cap);
                const int idx = pick_shallow(&g, &rng);
                if (g.depth[idx] > depth_in) depth_in = g.depth[idx];
                add_conn(&g, pin, idx);
            }
            const double ox = g_uniform(&rng, 0.0, w);
            const double oy = g_uniform(&rng, 0.0, h);
            const int o = add_pin(&g, cell, 0.0, 0.0, ox, oy, 1, 0.0);
            new_driver(&g, o, depth_in + 1);
        }
        D->cell_w[cell] = w, D->cell_h[cell] = h, D->cell_delay[cell] = delay;
        ++D->n_cells;
    }
    /* primary outputs (:187-206): a uniformly drawn idle, non-terminal driver when any exists */
    fenwick fw = {calloc((size_t)g.n_drv + 1, sizeof(int32_t)), g.n_drv, 1};
    while (fw.top * 2 <= fw.n) fw.top *= 2;
    int n_idle = 0;
    for (int d = 0; d < g.n_drv; ++d)
        if (g.sink_cnt[d] == 0 && D->pin_cell[g.drv[d]] >= 0) fw_add(&fw, d, 1), ++n_idle;
    for (int i = 0; i < n_po; ++i) {
        const double cap = g_uniform(&rng, 0.5, 2.0);
        const int p = add_pin(&g, -1, 1.0, (i + 0.5) / n_po, 0.0, 0.0, 0, cap);
        D->endpoints[D->n_endpoints++] = p;
        int idx;
        if (n_idle > 0) idx = fw_kth(&fw, (int)g_int(&rng, 0, n_idle - 1));
        else idx = (int)g_int(&rng, 0, g.n_drv - 1);
        if (g.sink_cnt[idx] == 0 && D->pin_cell[g.drv[idx]] >= 0) fw_add(&fw, idx, -1), --n_idle;
        add_conn(&g, p, idx);
    }
    free(fw.t);
    /* one net per driver with a sink, in driver order, sinks in connection order (:209-217) */
    int32_t* head = calloc((size_t)g.n_drv + 1, sizeof(int32_t));
    for (int64_t c = 0; c < g.n_conn; ++c) ++head[g.conn_drv[c] + 1];
    for (int d = 0; d < g.n_drv; ++d) head[d + 1] += head[d];
    int32_t* bucket = malloc((size_t)(g.n_conn > 0 ? g.n_conn : 1) * sizeof(int32_t));
    int32_t* fill = malloc((size_t)g.n_drv * sizeof(int32_t) + 1);
    memcpy(fill, head, (size_t)g.n_drv * sizeof(int32_t));
    for (int64_t c = 0; c < g.n_conn; ++c) bucket[fill[g.conn_drv[c]]++] = g.conn_sink[c];
    D->net_start = malloc(((size_t)g.n_drv + 1) * sizeof(int32_t));
    D->net_pins = malloc(((size_t)g.n_conn + g.n_drv + 1) * sizeof(int32_t));
    int64_t e = 0;
    D->net_start[0] = 0;
    for (int d = 0; d < g.n_drv; ++d) {
        if (g.sink_cnt[d] == 0) continue;
        D->net_pins[e++] = g.drv[d];
        for (int32_t j = head[d]; j < head[d + 1]; ++j) D->net_pins[e++] = bucket[j];
        D->net_start[++D->n_nets] = (int32_t)e;
    }
    free(head), free(bucket), free(fill);
    /* core: square at 75% utilisation (:220-225); terminals rescaled (:226-231) */
    double area = 0.0;
    for (int c = 0; c < D->n_cells; ++c) area += D->cell_w[c] * D->cell_h[c];
    const double side = ceil(sqrt(area / 0.75));
    D->core[0] = 0.0, D->core[1] = 0.0, D->core[2] = side, D->core[3] = side;
    for (int p = 0; p < D->n_pins; ++p) {
        if (D->pin_cell[p] >= 0) continue;
        D->pin_term[2 * p] = D->core[0] + D->pin_term[2 * p] * (D->core[2] - D->core[0]);
        D->pin_term[2 * p + 1] = D->core[1] + D->pin_term[2 * p + 1] * (D->core[3] - D->core[1]);
    }
    D->clock = 1.0, D->r_unit = r_unit, D->c_unit = c_unit; /* :233-236 (clock until calibrated) */
    for (int c = 0; c < D->n_cells; ++c) { /* centred starts (:240-242) */
        D->positions[2 * c] = D->core[0] + (D->core[2] - D->core[0] - D->cell_w[c]) / 2.0;
        D->positions[2 * c + 1] = D->core[1] + (D->core[3] - D->core[1] - D->cell_h[c]) / 2.0;
    }
    free(slot_is_reg), free(g.drv), free(g.sink_cnt), free(g.depth), free(g.shallow);
    free(g.conn_sink), free(g.conn_drv);
    *out = D;
    return TDPG_OK;
}

int orc_design_view(void* h, tdpg_netlist* v, const double** positions)
{
    const orc_design* D = (const orc_design*)h;
    memset(v, 0, sizeof *v);
    v->n_cells = D->n_cells, v->n_pins = D->n_pins, v->n_nets = D->n_nets;
    v->n_sources = D->n_sources, v->n_endpoints = D->n_endpoints;
    v->cell_w = D->cell_w, v->cell_h = D->cell_h, v->cell_delay = D->cell_delay, v->cell_fixed = D->cell_fixed;
    v->pin_cell = D->pin_cell, v->pin_term = D->pin_term, v->pin_off = D->pin_off, v->pin_dir = D->pin_dir;
    v->pin_cap = D->pin_cap, v->net_start = D->net_start, v->net_pins = D->net_pins, v->sources = D->sources;
    v->endpoints = D->endpoints, v->clock_period = D->clock, v->r_unit = D->r_unit, v->c_unit = D->c_unit;
    memcpy(v->core, D->core, sizeof D->core);
    v->pin_names = NULL;
    if (positions) *positions = D->positions;
    return TDPG_OK;
}
