/*
 * tdp_oracle.c — TEST INFRASTRUCTURE ONLY (see tdp_oracle.h).
 *
 * Plain-C restatement of the reference hot path, one function per reference
 * function, same floating-point operation order (compiled with
 * -ffp-contract=off, like the reference's x86-64 build which contains no FMA).
 * Citations are relative to /root/reference/proj.
 */
#include "tdp_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[512];
static _Thread_local int g_kind;

static int fail(int kind, const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    g_kind = kind;
    return kind;
}

const char* orc_last_error(void) { return g_err; }
int orc_last_error_kind(void) { return g_kind; }

/* std::min / std::max semantics (first argument wins unless strictly beaten). */
static inline double dmin(double a, double b) { return (b < a) ? b : a; }
static inline double dmax(double a, double b) { return (a < b) ? b : a; }
static inline int imin(int a, int b) { return (b < a) ? b : a; }
static inline int imax(int a, int b) { return (a < b) ? b : a; }

/* ---- mt19937_64 (C++ [rand.eng.mers] parameters) + include/tdp/rng.hpp:13-28 */
void orc_mt64_seed(orc_mt64* r, uint64_t seed)
{
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* r)
{
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

static double rng_unit(orc_mt64* r) { return (double)(orc_mt64_next(r) >> 11) * 0x1.0p-53; }
static double rng_uniform(orc_mt64* r, double lo, double hi) { return lo + (hi - lo) * rng_unit(r); }

/* ---- pin_positions: src/netlist.cpp:23-32 -------------------------------- */
void orc_pin_positions(const tdpg_netlist* nl, const double* cell_xy, double* pin_xy)
{
    for (int32_t p = 0; p < nl->n_pins; ++p) {
        const int32_t c = nl->pin_cell[p];
        const double ax = c < 0 ? nl->pin_term[2 * p] : cell_xy[2 * c];
        const double ay = c < 0 ? nl->pin_term[2 * p + 1] : cell_xy[2 * c + 1];
        pin_xy[2 * p] = ax + nl->pin_off[2 * p];
        pin_xy[2 * p + 1] = ay + nl->pin_off[2 * p + 1];
    }
}

/* ---- wa_dimension / wa_wirelength: src/wirelength.cpp:12-58 -------------- */
static double wa_dim(int32_t n, const double* xy, int axis, double gamma, double* grad)
{
    double hi = xy[axis], lo = hi;
    for (int32_t i = 0; i < n; ++i) {
        hi = dmax(hi, xy[2 * i + axis]);
        lo = dmin(lo, xy[2 * i + axis]);
    }
    double s_max = 0.0, t_max = 0.0, s_min = 0.0, t_min = 0.0;
    for (int32_t i = 0; i < n; ++i) {
        const double x = xy[2 * i + axis];
        const double eu = exp((x - hi) / gamma);
        s_max += eu;
        t_max += (x - hi) * eu;
        const double el = exp(-(x - lo) / gamma);
        s_min += el;
        t_min += (x - lo) * el;
    }
    const double max_term = t_max / s_max;
    const double min_term = t_min / s_min;
    for (int32_t i = 0; i < n; ++i) {
        const double xi = xy[2 * i + axis];
        const double eu = exp((xi - hi) / gamma);
        const double el = exp(-(xi - lo) / gamma);
        const double d_max = (eu / s_max) * (1.0 + ((xi - hi) - max_term) / gamma);
        const double d_min = (el / s_min) * (1.0 - ((xi - lo) - min_term) / gamma);
        grad[2 * i + axis] += d_max - d_min;
    }
    return (hi - lo) + (max_term - min_term);
}

double orc_wa(int32_t n, const double* xy, double gamma, double* grad)
{
    for (int32_t i = 0; i < 2 * n; ++i) grad[i] = 0.0;
    if (n < 2) return 0.0;
    const double vx = wa_dim(n, xy, 0, gamma, grad);
    const double vy = wa_dim(n, xy, 1, gamma, grad);
    return vx + vy;
}

/* ---- hpwl_net / hpwl_total: src/wirelength.cpp:60-85 --------------------- */
double orc_hpwl_total(const tdpg_netlist* nl, const double* pin_xy)
{
    double total = 0.0;
    for (int32_t e = 0; e < nl->n_nets; ++e) {
        const int32_t b = nl->net_start[e], n = nl->net_start[e + 1] - b;
        if (n < 2) continue; /* hpwl_net returns 0.0, and total += 0.0 is exact */
        const int32_t p0 = nl->net_pins[b];
        double xl = pin_xy[2 * p0], xh = xl, yl = pin_xy[2 * p0 + 1], yh = yl;
        for (int32_t i = 0; i < n; ++i) {
            const int32_t p = nl->net_pins[b + i];
            xl = dmin(xl, pin_xy[2 * p]);
            xh = dmax(xh, pin_xy[2 * p]);
            yl = dmin(yl, pin_xy[2 * p + 1]);
            yh = dmax(yh, pin_xy[2 * p + 1]);
        }
        total += (xh - xl) + (yh - yl);
    }
    return total;
}

/* ---- DensityGrid: src/density.cpp:13-158 ---------------------------------- */
static double bspline2(double u)
{
    const double a = fabs(u);
    if (a >= 1.5) return 0.0;
    if (a <= 0.5) return 0.75 - a * a;
    const double t = 1.5 - a;
    return 0.5 * t * t;
}

static double bspline2_integral(double u)
{
    if (u <= -1.5) return 0.0;
    if (u >= 1.5) return 1.0;
    if (u <= -0.5) {
        const double t = u + 1.5;
        return t * t * t / 6.0;
    }
    if (u <= 0.5) return 0.5 + 0.75 * u - u * u * u / 3.0;
    const double t = 1.5 - u;
    return 1.0 - t * t * t / 6.0;
}

static double extent_weight(double lo, double hi, double c, double h)
{
    return (bspline2_integral((hi - c) / h) - bspline2_integral((lo - c) / h)) * h / (hi - lo);
}

static double extent_weight_grad(double lo, double hi, double c, double h)
{
    return (bspline2((hi - c) / h) - bspline2((lo - c) / h)) / (hi - lo);
}

typedef struct {
    int32_t bin;
    double w, dwx, dwy;
} fp_entry;

int orc_density(const tdpg_netlist* nl, const double* cell_xy, int32_t nx, int32_t ny, double target_density,
                double* value, double* overflow, double* d_cell)
{
    if (nx < 1 || ny < 1) return fail(TDPG_ERR_VALIDATION, "validation error: density grid must be at least 1x1");
    const double x0 = nl->core[0], y0 = nl->core[1];
    const double bw = (nl->core[2] - nl->core[0]) / nx; /* density.cpp:57-59 */
    const double bh = (nl->core[3] - nl->core[1]) / ny;
    const double cap = target_density * bw * bh;
    double total_movable = 0.0;
    for (int32_t c = 0; c < nl->n_cells; ++c)
        if (!nl->cell_fixed[c]) total_movable += nl->cell_w[c] * nl->cell_h[c];

    const size_t n_bins = (size_t)nx * (size_t)ny;
    double* occ = calloc(n_bins, sizeof(double));
    /* fixed cells: exact overlap (density.cpp:75-93) */
    for (int32_t c = 0; c < nl->n_cells; ++c) {
        if (!nl->cell_fixed[c]) continue;
        const double xl = cell_xy[2 * c], xh = xl + nl->cell_w[c];
        const double yl = cell_xy[2 * c + 1], yh = yl + nl->cell_h[c];
        const int bx0 = imax(0, (int)floor((xl - x0) / bw));
        const int bx1 = imin(nx - 1, (int)floor((xh - x0) / bw));
        const int by0 = imax(0, (int)floor((yl - y0) / bh));
        const int by1 = imin(ny - 1, (int)floor((yh - y0) / bh));
        for (int bx = bx0; bx <= bx1; ++bx)
            for (int by = by0; by <= by1; ++by) {
                const double ox = dmin(xh, x0 + (bx + 1) * bw) - dmax(xl, x0 + bx * bw);
                const double oy = dmin(yh, y0 + (by + 1) * bh) - dmax(yl, y0 + by * bh);
                if (ox > 0.0 && oy > 0.0) occ[(size_t)bx * (size_t)ny + (size_t)by] += ox * oy;
            }
    }
    /* movable footprints (density.cpp:102-135), kept per cell for the gradient */
    int64_t* fp_start = malloc(((size_t)nl->n_cells + 1) * sizeof(int64_t));
    size_t cap_e = 1024, n_e = 0;
    fp_entry* ent = malloc(cap_e * sizeof(fp_entry));
    for (int32_t c = 0; c < nl->n_cells; ++c) {
        fp_start[c] = (int64_t)n_e;
        if (nl->cell_fixed[c]) continue;
        const double xl = cell_xy[2 * c], xh = xl + nl->cell_w[c];
        const double yl = cell_xy[2 * c + 1], yh = yl + nl->cell_h[c];
        const int bx0 = imax(0, (int)floor((xl - 1.5 * bw - x0) / bw - 0.5));
        const int bx1 = imin(nx - 1, (int)ceil((xh + 1.5 * bw - x0) / bw - 0.5));
        const int by0 = imax(0, (int)floor((yl - 1.5 * bh - y0) / bh - 0.5));
        const int by1 = imin(ny - 1, (int)ceil((yh + 1.5 * bh - y0) / bh - 0.5));
        const double area = nl->cell_w[c] * nl->cell_h[c];
        for (int bx = bx0; bx <= bx1; ++bx) {
            const double cx = x0 + (bx + 0.5) * bw;
            const double wx = extent_weight(xl, xh, cx, bw);
            const double dwx = extent_weight_grad(xl, xh, cx, bw);
            if (wx == 0.0 && dwx == 0.0) continue;
            for (int by = by0; by <= by1; ++by) {
                const double cy = y0 + (by + 0.5) * bh;
                const double wy = extent_weight(yl, yh, cy, bh);
                const double dwy = extent_weight_grad(yl, yh, cy, bh);
                if (wy == 0.0 && dwy == 0.0) continue;
                if (n_e == cap_e) ent = realloc(ent, (cap_e *= 2) * sizeof(fp_entry));
                ent[n_e].bin = bx * ny + by;
                ent[n_e].w = area * wx * wy;
                ent[n_e].dwx = area * dwx * wy;
                ent[n_e].dwy = area * wx * dwy;
                ++n_e;
            }
        }
    }
    fp_start[nl->n_cells] = (int64_t)n_e;
    for (size_t i = 0; i < n_e; ++i) occ[ent[i].bin] += ent[i].w;
    double val = 0.0, over = 0.0;
    for (size_t b = 0; b < n_bins; ++b) {
        const double ex = dmax(0.0, occ[b] - cap);
        occ[b] = ex; /* reuse as excess */
        val += ex * ex;
        over += ex;
    }
    *value = val;
    *overflow = total_movable > 0.0 ? over / total_movable : 0.0;
    if (d_cell)
        for (int32_t c = 0; c < nl->n_cells; ++c) {
            double gx = 0.0, gy = 0.0;
            for (int64_t i = fp_start[c]; i < fp_start[c + 1]; ++i) {
                const double f = 2.0 * occ[ent[i].bin];
                gx += f * ent[i].dwx;
                gy += f * ent[i].dwy;
            }
            d_cell[2 * c] = gx;
            d_cell[2 * c + 1] = gy;
        }
    free(ent);
    free(fp_start);
    free(occ);
    return 0;
}

/* ---- pin_pair_loss: src/pin_pairs.cpp:17-49 (ledger iterated in key order) */
double orc_pp_loss(int64_t q, const int32_t* a, const int32_t* b, const double* w, int64_t n_pins,
                   const double* pin_xy, int32_t kind, double* d_pin)
{
    double value = 0.0;
    if (d_pin)
        for (int64_t i = 0; i < 2 * n_pins; ++i) d_pin[i] = 0.0;
    for (int64_t i = 0; i < q; ++i) {
        const double dx = pin_xy[2 * a[i]] - pin_xy[2 * b[i]];
        const double dy = pin_xy[2 * a[i] + 1] - pin_xy[2 * b[i] + 1];
        double gx, gy;
        if (kind == 0) {
            value += w[i] * (dx * dx + dy * dy);
            gx = 2.0 * w[i] * dx;
            gy = 2.0 * w[i] * dy;
        } else {
            const double dist = sqrt(dx * dx + dy * dy);
            value += w[i] * dist;
            if (!(dist > 0.0)) continue;
            gx = w[i] * dx / dist;
            gy = w[i] * dy / dist;
        }
        if (d_pin) {
            d_pin[2 * a[i]] += gx;
            d_pin[2 * a[i] + 1] += gy;
            d_pin[2 * b[i]] -= gx;
            d_pin[2 * b[i] + 1] -= gy;
        }
    }
    return value;
}

/* ---- AdamState::step: src/placer.cpp:345-356 ----------------------------- */
void orc_adam_step(int64_t n, double* x, const double* g, double* m, double* v, int32_t* t, double lr, double b1,
                   double b2, double eps)
{
    ++*t;
    const double c1 = 1.0 - pow(b1, *t);
    const double c2 = 1.0 - pow(b2, *t);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        x[i] -= lr * (m[i] / c1) / (sqrt(v[i] / c2) + eps);
    }
}

/* ---- objective_and_gradient: src/placer.cpp:275-343 ---------------------- */
int orc_objective(const tdpg_netlist* nl, const double* cell_xy, int32_t nx, int32_t ny, double td, double gamma,
                  double lambda, double beta, int32_t kind, const double* net_w, int64_t q, const int32_t* a,
                  const int32_t* b, const double* w, double terms[6], double* d_cell)
{
    const int32_t P = nl->n_pins, C = nl->n_cells;
    double* pos = malloc((size_t)P * 2 * sizeof(double));
    double* pin_grad = calloc((size_t)P * 2, sizeof(double));
    orc_pin_positions(nl, cell_xy, pos);
    int32_t max_deg = 1;
    for (int32_t e = 0; e < nl->n_nets; ++e) max_deg = imax(max_deg, nl->net_start[e + 1] - nl->net_start[e]);
    double* nxy = malloc((size_t)max_deg * 2 * sizeof(double));
    double* ng = malloc((size_t)max_deg * 2 * sizeof(double));
    double wl = 0.0;
    for (int32_t e = 0; e < nl->n_nets; ++e) {
        const int32_t s0 = nl->net_start[e], n = nl->net_start[e + 1] - s0;
        for (int32_t i = 0; i < n; ++i) {
            nxy[2 * i] = pos[2 * nl->net_pins[s0 + i]];
            nxy[2 * i + 1] = pos[2 * nl->net_pins[s0 + i] + 1];
        }
        const double v = orc_wa(n, nxy, gamma, ng);
        const double we = net_w ? net_w[e] : 1.0;
        wl += we * v;
        for (int32_t i = 0; i < n; ++i) {
            const int32_t p = nl->net_pins[s0 + i];
            pin_grad[2 * p] += we * ng[2 * i];
            pin_grad[2 * p + 1] += we * ng[2 * i + 1];
        }
    }
    double dval, dover;
    double* dd = malloc((size_t)C * 2 * sizeof(double));
    const int rc = orc_density(nl, cell_xy, nx, ny, td, &dval, &dover, dd);
    if (rc) {
        free(pos), free(pin_grad), free(nxy), free(ng), free(dd);
        return rc;
    }
    double* ppd = malloc((size_t)P * 2 * sizeof(double));
    const double ppv = orc_pp_loss(q, a, b, w, P, pos, kind, ppd);
    double* g = d_cell ? d_cell : malloc((size_t)C * 2 * sizeof(double));
    for (int32_t i = 0; i < 2 * C; ++i) g[i] = 0.0;
    for (int32_t p = 0; p < P; ++p) {
        const int32_t c = nl->pin_cell[p];
        if (c < 0) continue;
        g[2 * c] += pin_grad[2 * p] + beta * ppd[2 * p];
        g[2 * c + 1] += pin_grad[2 * p + 1] + beta * ppd[2 * p + 1];
    }
    for (int32_t c = 0; c < C; ++c) {
        if (nl->cell_fixed[c]) {
            g[2 * c] = 0.0, g[2 * c + 1] = 0.0;
            continue;
        }
        g[2 * c] += lambda * dd[2 * c];
        g[2 * c + 1] += lambda * dd[2 * c + 1];
    }
    const double hpwl = orc_hpwl_total(nl, pos);
    const double value = wl + lambda * dval + beta * ppv;
    int finite = isfinite(value) && isfinite(wl) && isfinite(dval) && isfinite(ppv);
    for (int32_t i = 0; i < 2 * C && finite; ++i) finite = isfinite(g[i]);
    terms[0] = value, terms[1] = wl, terms[2] = dval, terms[3] = ppv, terms[4] = hpwl, terms[5] = dover;
    if (!d_cell) free(g);
    free(pos), free(pin_grad), free(nxy), free(ng), free(dd), free(ppd);
    if (!finite) return fail(TDPG_ERR_NONFINITE, "non-finite value: non-finite objective or gradient");
    return 0;
}

/* ---- session ---------------------------------------------------------------- */
typedef struct {
    tdpg_netlist nl;
    /* timing graph (src/timing_graph.cpp:49-138) */
    int32_t n_arcs, n_net_arcs, n_cell_arcs, n_levels;
    int32_t *from, *to, *kind, *owner;
    int32_t *in_start, *in_arcs, *out_start, *out_arcs;
    int32_t *level, *lvl_start, *lvl_pins;
    uint8_t *is_source, *is_endpoint;
    /* last STA */
    double *arr, *req, *slack;
    uint8_t *ak, *rk;
    double tns, wns;
    /* last extraction */
    int32_t n_paths;
    int32_t *p_start, *p_pins;
    double* p_slack;
    int64_t n_hits;
    int32_t *h_a, *h_b;
    double* h_s;
    /* ledger, sorted by (a, b) */
    int64_t q, q_cap;
    int32_t *la, *lb;
    double* lw;
} orc_session;

static const char* pin_name(const tdpg_netlist* nl, int32_t p, char* buf)
{
    if (nl->pin_names && nl->pin_names[p]) return nl->pin_names[p];
    snprintf(buf, 32, "p%d", p);
    return buf;
}

static void free_session(orc_session* s)
{
    void* ptrs[] = {s->from, s->to, s->kind, s->owner, s->in_start, s->in_arcs, s->out_start, s->out_arcs,
                    s->level, s->lvl_start, s->lvl_pins, s->is_source, s->is_endpoint, s->arr, s->req, s->slack,
                    s->ak, s->rk, s->p_start, s->p_pins, s->p_slack, s->h_a, s->h_b, s->h_s, s->la, s->lb, s->lw};
    for (size_t i = 0; i < sizeof ptrs / sizeof ptrs[0]; ++i) free(ptrs[i]);
    free(s);
}

void orc_destroy(void* h)
{
    if (h) free_session((orc_session*)h);
}

/* build_timing_graph: src/timing_graph.cpp:49-138 (+ report_cycle :12-45) */
static int build_graph(orc_session* s)
{
    const tdpg_netlist* nl = &s->nl;
    const int32_t P = nl->n_pins, C = nl->n_cells;
    s->is_source = calloc((size_t)P, 1);
    s->is_endpoint = calloc((size_t)P, 1);
    for (int32_t i = 0; i < nl->n_sources; ++i) s->is_source[nl->sources[i]] = 1;
    for (int32_t i = 0; i < nl->n_endpoints; ++i) s->is_endpoint[nl->endpoints[i]] = 1;
    /* cell_pins: ascending pin ids per cell (netlist.cpp:12-14) */
    int32_t* cp_start = calloc((size_t)C + 1, sizeof(int32_t));
    for (int32_t p = 0; p < P; ++p)
        if (nl->pin_cell[p] >= 0) cp_start[nl->pin_cell[p] + 1]++;
    for (int32_t c = 0; c < C; ++c) cp_start[c + 1] += cp_start[c];
    int32_t* cp = malloc(((size_t)cp_start[C] + 1) * sizeof(int32_t));
    int32_t* fill = malloc(((size_t)C + 1) * sizeof(int32_t));
    memcpy(fill, cp_start, (size_t)C * sizeof(int32_t));
    for (int32_t p = 0; p < P; ++p)
        if (nl->pin_cell[p] >= 0) cp[fill[nl->pin_cell[p]]++] = p;
    /* count arcs */
    int64_t na = nl->net_start[nl->n_nets] - nl->n_nets;
    int64_t nc = 0;
    for (int32_t c = 0; c < C; ++c) {
        int64_t ni = 0, no = 0;
        for (int32_t i = cp_start[c]; i < cp_start[c + 1]; ++i) {
            const int32_t p = cp[i];
            if (nl->pin_dir[p] == 0 && !s->is_endpoint[p]) ++ni;
            if (nl->pin_dir[p] == 1 && !s->is_source[p]) ++no;
        }
        nc += ni * no;
    }
    s->n_net_arcs = (int32_t)na;
    s->n_cell_arcs = (int32_t)nc;
    s->n_arcs = (int32_t)(na + nc);
    const size_t A = (size_t)s->n_arcs;
    s->from = malloc((A + 1) * sizeof(int32_t));
    s->to = malloc((A + 1) * sizeof(int32_t));
    s->kind = malloc((A + 1) * sizeof(int32_t));
    s->owner = malloc((A + 1) * sizeof(int32_t));
    int32_t k = 0;
    for (int32_t e = 0; e < nl->n_nets; ++e)
        for (int32_t i = nl->net_start[e] + 1; i < nl->net_start[e + 1]; ++i) {
            s->from[k] = nl->net_pins[nl->net_start[e]], s->to[k] = nl->net_pins[i], s->kind[k] = 0, s->owner[k] = e;
            ++k;
        }
    for (int32_t c = 0; c < C; ++c)
        for (int32_t i = cp_start[c]; i < cp_start[c + 1]; ++i) {
            const int32_t in = cp[i];
            if (nl->pin_dir[in] != 0 || s->is_endpoint[in]) continue;
            for (int32_t j = cp_start[c]; j < cp_start[c + 1]; ++j) {
                const int32_t out = cp[j];
                if (nl->pin_dir[out] != 1 || s->is_source[out]) continue;
                s->from[k] = in, s->to[k] = out, s->kind[k] = 1, s->owner[k] = c;
                ++k;
            }
        }
    free(cp_start), free(cp), free(fill);
    /* in/out arc lists, ascending arc id */
    s->in_start = calloc((size_t)P + 1, sizeof(int32_t));
    s->out_start = calloc((size_t)P + 1, sizeof(int32_t));
    for (size_t a = 0; a < A; ++a) s->in_start[s->to[a] + 1]++, s->out_start[s->from[a] + 1]++;
    for (int32_t p = 0; p < P; ++p) s->in_start[p + 1] += s->in_start[p], s->out_start[p + 1] += s->out_start[p];
    s->in_arcs = malloc((A + 1) * sizeof(int32_t));
    s->out_arcs = malloc((A + 1) * sizeof(int32_t));
    int32_t* fi = malloc(((size_t)P + 1) * sizeof(int32_t));
    int32_t* fo = malloc(((size_t)P + 1) * sizeof(int32_t));
    memcpy(fi, s->in_start, (size_t)P * sizeof(int32_t));
    memcpy(fo, s->out_start, (size_t)P * sizeof(int32_t));
    for (size_t a = 0; a < A; ++a) s->in_arcs[fi[s->to[a]]++] = (int32_t)a, s->out_arcs[fo[s->from[a]]++] = (int32_t)a;
    free(fi), free(fo);
    /* Kahn levelization (timing_graph.cpp:87-104) */
    int32_t* indeg = malloc(((size_t)P + 1) * sizeof(int32_t));
    int32_t* order = malloc(((size_t)P + 1) * sizeof(int32_t));
    s->level = calloc((size_t)P + 1, sizeof(int32_t));
    int32_t n_order = 0;
    for (int32_t p = 0; p < P; ++p) {
        indeg[p] = s->in_start[p + 1] - s->in_start[p];
        if (indeg[p] == 0) order[n_order++] = p;
    }
    for (int32_t head = 0; head < n_order; ++head) {
        const int32_t u = order[head];
        for (int32_t i = s->out_start[u]; i < s->out_start[u + 1]; ++i) {
            const int32_t v = s->to[s->out_arcs[i]];
            s->level[v] = imax(s->level[v], s->level[u] + 1);
            if (--indeg[v] == 0) order[n_order++] = v;
        }
    }
    if (n_order != P) { /* report_cycle, timing_graph.cpp:12-45 */
        uint8_t* remaining = calloc((size_t)P, 1);
        int32_t start = -1;
        for (int32_t p = 0; p < P; ++p)
            if (indeg[p] > 0) remaining[p] = 1, start = p;
        int32_t* seen_at = malloc((size_t)P * sizeof(int32_t));
        int32_t* walk = malloc((size_t)P * sizeof(int32_t));
        for (int32_t p = 0; p < P; ++p) seen_at[p] = -1;
        int32_t n_walk = 0, cur = start;
        while (seen_at[cur] < 0) {
            seen_at[cur] = n_walk;
            walk[n_walk++] = cur;
            for (int32_t i = s->in_start[cur]; i < s->in_start[cur + 1]; ++i) {
                const int32_t u = s->from[s->in_arcs[i]];
                if (remaining[u]) {
                    cur = u;
                    break;
                }
            }
        }
        char msg[400] = "", nb[32];
        for (int32_t i = seen_at[cur]; i < n_walk; ++i) {
            if (msg[0]) strncat(msg, " <- ", sizeof msg - strlen(msg) - 1);
            strncat(msg, pin_name(nl, walk[i], nb), sizeof msg - strlen(msg) - 1);
        }
        free(remaining), free(seen_at), free(walk), free(indeg), free(order);
        return fail(TDPG_ERR_CYCLE, "validation error: combinational cycle: %s", msg);
    }
    free(indeg), free(order);
    int32_t max_level = 0;
    for (int32_t p = 0; p < P; ++p) max_level = imax(max_level, s->level[p]);
    s->n_levels = P > 0 ? max_level + 1 : 1;
    s->lvl_start = calloc((size_t)s->n_levels + 1, sizeof(int32_t));
    for (int32_t p = 0; p < P; ++p) s->lvl_start[s->level[p] + 1]++;
    for (int32_t l = 0; l < s->n_levels; ++l) s->lvl_start[l + 1] += s->lvl_start[l];
    s->lvl_pins = malloc(((size_t)P + 1) * sizeof(int32_t));
    int32_t* fl = malloc(((size_t)s->n_levels + 1) * sizeof(int32_t));
    memcpy(fl, s->lvl_start, (size_t)s->n_levels * sizeof(int32_t));
    for (int32_t p = 0; p < P; ++p) s->lvl_pins[fl[s->level[p]]++] = p;
    free(fl);
    /* endpoint reachability (timing_graph.cpp:112-135) */
    uint8_t* reach = calloc((size_t)P + 1, 1);
    int32_t* stack = malloc(((size_t)P + 1) * sizeof(int32_t));
    int32_t sp = 0;
    for (int32_t i = 0; i < nl->n_sources; ++i)
        if (!reach[nl->sources[i]]) reach[nl->sources[i]] = 1, stack[sp++] = nl->sources[i];
    while (sp > 0) {
        const int32_t u = stack[--sp];
        for (int32_t i = s->out_start[u]; i < s->out_start[u + 1]; ++i) {
            const int32_t v = s->to[s->out_arcs[i]];
            if (!reach[v]) reach[v] = 1, stack[sp++] = v;
        }
    }
    int rc = 0;
    for (int32_t i = 0; i < nl->n_endpoints && !rc; ++i)
        if (!reach[nl->endpoints[i]]) {
            char nb[32];
            rc = fail(TDPG_ERR_VALIDATION, "validation error: endpoint \"%s\" unreachable from every source",
                      pin_name(nl, nl->endpoints[i], nb));
        }
    free(reach), free(stack);
    return rc;
}

void* orc_create(const tdpg_netlist* nl)
{
    orc_session* s = calloc(1, sizeof(orc_session));
    s->nl = *nl;
    if (build_graph(s)) {
        free_session(s);
        return NULL;
    }
    const size_t P = (size_t)nl->n_pins + 1;
    s->arr = malloc(P * sizeof(double));
    s->req = malloc(P * sizeof(double));
    s->slack = malloc(P * sizeof(double));
    s->ak = malloc(P);
    s->rk = malloc(P);
    return s;
}

int orc_graph_info(void* h, int32_t counts[4], int32_t* level, int32_t* arc_from, int32_t* arc_to,
                   int32_t* arc_kind, int32_t* arc_owner)
{
    orc_session* s = h;
    counts[0] = s->n_net_arcs, counts[1] = s->n_cell_arcs, counts[2] = s->n_levels, counts[3] = s->n_levels - 1;
    if (level) memcpy(level, s->level, (size_t)s->nl.n_pins * sizeof(int32_t));
    if (arc_from) memcpy(arc_from, s->from, (size_t)s->n_arcs * sizeof(int32_t));
    if (arc_to) memcpy(arc_to, s->to, (size_t)s->n_arcs * sizeof(int32_t));
    if (arc_kind) memcpy(arc_kind, s->kind, (size_t)s->n_arcs * sizeof(int32_t));
    if (arc_owner) memcpy(arc_owner, s->owner, (size_t)s->n_arcs * sizeof(int32_t));
    return 0;
}

/* net_delay / arc_delay: src/sta.cpp:10-21 */
static double arc_delay(const orc_session* s, int32_t a, const double* pos)
{
    if (s->kind[a] == 1) return s->nl.cell_delay[s->owner[a]];
    const int32_t f = s->from[a], t = s->to[a];
    const double len = fabs(pos[2 * f] - pos[2 * t]) + fabs(pos[2 * f + 1] - pos[2 * t + 1]);
    return (s->nl.r_unit * len) * (s->nl.c_unit * len + s->nl.pin_cap[t]);
}

/* propagate_arrival / propagate_required / compute_slacks / tns_wns: src/sta.cpp:33-133 */
static void sta_at(orc_session* s, const double* pos)
{
    const tdpg_netlist* nl = &s->nl;
    const int32_t P = nl->n_pins;
    for (int32_t l = 0; l < s->n_levels; ++l)
        for (int32_t i = s->lvl_start[l]; i < s->lvl_start[l + 1]; ++i) {
            const int32_t v = s->lvl_pins[i];
            if (s->is_source[v]) {
                s->arr[v] = 0.0, s->ak[v] = 1;
                continue;
            }
            double best = -INFINITY;
            int found = 0;
            for (int32_t j = s->in_start[v]; j < s->in_start[v + 1]; ++j) {
                const int32_t a = s->in_arcs[j];
                if (!s->ak[s->from[a]]) continue;
                const double cand = s->arr[s->from[a]] + arc_delay(s, a, pos);
                if (!found || cand > best) best = cand, found = 1;
            }
            s->arr[v] = found ? best : 0.0;
            s->ak[v] = (uint8_t)found;
        }
    for (int32_t l = s->n_levels - 1; l >= 0; --l)
        for (int32_t i = s->lvl_start[l]; i < s->lvl_start[l + 1]; ++i) {
            const int32_t u = s->lvl_pins[i];
            double best = INFINITY;
            int found = 0;
            if (s->is_endpoint[u]) best = nl->clock_period, found = 1;
            for (int32_t j = s->out_start[u]; j < s->out_start[u + 1]; ++j) {
                const int32_t a = s->out_arcs[j];
                if (!s->rk[s->to[a]]) continue;
                const double cand = s->req[s->to[a]] - arc_delay(s, a, pos);
                if (!found || cand < best) best = cand, found = 1;
            }
            s->req[u] = found ? best : nl->clock_period;
            s->rk[u] = (uint8_t)found;
        }
    for (int32_t p = 0; p < P; ++p) s->slack[p] = s->req[p] - s->arr[p];
    double tns = 0.0, wns = 0.0;
    for (int32_t i = 0; i < nl->n_endpoints; ++i) {
        const double sl = s->slack[nl->endpoints[i]];
        if (sl < 0.0) {
            tns += sl;
            if (sl < wns) wns = sl;
        }
    }
    s->tns = tns, s->wns = wns;
}

int orc_sta(void* h, const double* cell_xy, double* arr, double* req, double* slack, uint8_t* ak, uint8_t* rk,
            double* tns, double* wns)
{
    orc_session* s = h;
    const size_t P = (size_t)s->nl.n_pins;
    double* pos = malloc((P + 1) * 2 * sizeof(double));
    orc_pin_positions(&s->nl, cell_xy, pos);
    sta_at(s, pos);
    free(pos);
    if (arr) memcpy(arr, s->arr, P * sizeof(double));
    if (req) memcpy(req, s->req, P * sizeof(double));
    if (slack) memcpy(slack, s->slack, P * sizeof(double));
    if (ak) memcpy(ak, s->ak, P);
    if (rk) memcpy(rk, s->rk, P);
    if (tns) *tns = s->tns;
    if (wns) *wns = s->wns;
    return 0;
}

/* Rank-0 path of every pin under the PathEnumerator order (src/paths.cpp:19-55,
 * include/tdp/paths.hpp:63-69): worst delay, ties broken by the
 * lexicographically smallest full pin sequence.  Restated as a level-order DP
 * over rank-0 predecessor paths (rank-0 at v extends rank-0 at one of its
 * fan-in pins, paths.cpp:33-42). */
static int32_t materialize(const int32_t* pred, int32_t v, int32_t* buf, int32_t cap)
{
    int32_t n = 0;
    for (int32_t u = v; u >= 0 && n < cap; u = pred[u]) buf[n++] = u;
    for (int32_t i = 0; i < n / 2; ++i) {
        const int32_t t = buf[i];
        buf[i] = buf[n - 1 - i], buf[n - 1 - i] = t;
    }
    return n;
}

static int lex_less(const int32_t* a, int32_t na, const int32_t* b, int32_t nb)
{
    const int32_t n = na < nb ? na : nb;
    for (int32_t i = 0; i < n; ++i)
        if (a[i] != b[i]) return a[i] < b[i];
    return na < nb;
}

typedef struct {
    int32_t pin;
    double slack;
} ep_rank;

static int cmp_ep(const void* x, const void* y)
{
    const ep_rank* a = x;
    const ep_rank* b = y;
    if (a->slack != b->slack) return a->slack < b->slack ? -1 : 1;
    return (a->pin > b->pin) - (a->pin < b->pin);
}

int cmp_u64(const void* x, const void* y);
int cmp_i32(const void* x, const void* y);

/* collect_pin_pairs (paths.cpp:191-203) and finish_report counters (:89-102) over the session's
 * p_start / p_pins / p_slack.  counts[0..3] = n_paths, total_pins, unique_endpoints, unique_pin_pairs. */
static void finish_report(orc_session* s, int64_t* counts)
{
    const tdpg_netlist* nl = &s->nl;
    const int32_t nv = s->n_paths, off = s->p_start[nv];
    free(s->h_a), free(s->h_b), free(s->h_s);
    s->h_a = malloc(((size_t)off + 1) * sizeof(int32_t));
    s->h_b = malloc(((size_t)off + 1) * sizeof(int32_t));
    s->h_s = malloc(((size_t)off + 1) * sizeof(double));
    int64_t nh = 0;
    for (int32_t i = 0; i < nv; ++i)
        for (int32_t j = s->p_start[i]; j + 1 < s->p_start[i + 1]; ++j) {
            const int32_t p0 = s->p_pins[j], p1 = s->p_pins[j + 1];
            if (nl->pin_dir[p0] != 1) continue;
            s->h_a[nh] = p0 < p1 ? p0 : p1, s->h_b[nh] = p0 < p1 ? p1 : p0, s->h_s[nh] = s->p_slack[i];
            ++nh;
        }
    s->n_hits = nh;
    uint64_t* keys = malloc(((size_t)nh + 1) * sizeof(uint64_t));
    for (int64_t i = 0; i < nh; ++i) keys[i] = ((uint64_t)(uint32_t)s->h_a[i] << 32) | (uint32_t)s->h_b[i];
    qsort(keys, (size_t)nh, sizeof(uint64_t), cmp_u64);
    int64_t uniq = 0;
    for (int64_t i = 0; i < nh; ++i) uniq += (i == 0 || keys[i] != keys[i - 1]);
    free(keys);
    /* unique endpoints: distinct last pins */
    int32_t* last = malloc(((size_t)nv + 1) * sizeof(int32_t));
    for (int32_t i = 0; i < nv; ++i) last[i] = s->p_pins[s->p_start[i + 1] - 1];
    qsort(last, (size_t)nv, sizeof(int32_t), cmp_i32);
    int64_t ue = 0;
    for (int32_t i = 0; i < nv; ++i) ue += (i == 0 || last[i] != last[i - 1]);
    free(last);
    counts[0] = nv, counts[1] = off, counts[2] = ue, counts[3] = uniq;
}

int orc_extract(void* h, const double* cell_xy, int32_t n, int64_t counts[4])
{
    int64_t c5[5];
    const int rc = orc_extract5(h, cell_xy, n, c5);
    memcpy(counts, c5, 4 * sizeof(int64_t));
    return rc;
}

int orc_extract5(void* h, const double* cell_xy, int32_t n, int64_t counts[5])
{
    orc_session* s = h;
    const tdpg_netlist* nl = &s->nl;
    const int32_t P = nl->n_pins;
    double* pos = malloc(((size_t)P + 1) * 2 * sizeof(double));
    orc_pin_positions(nl, cell_xy, pos);
    sta_at(s, pos);
    /* violated endpoints, (slack, pin) ascending, clipped to n (paths.cpp:77-87, :177-178) */
    ep_rank* v = malloc(((size_t)nl->n_endpoints + 1) * sizeof(ep_rank));
    int32_t nv = 0;
    for (int32_t i = 0; i < nl->n_endpoints; ++i) {
        const int32_t e = nl->endpoints[i];
        if (s->slack[e] < 0.0) v[nv].pin = e, v[nv].slack = s->slack[e], ++nv;
    }
    qsort(v, (size_t)nv, sizeof(ep_rank), cmp_ep);
    if (n <= 0) n = nv;
    if (nv > n) nv = n;
    /* rank-0 DP */
    double* delay = malloc(((size_t)P + 1) * sizeof(double));
    int32_t* pred = malloc(((size_t)P + 1) * sizeof(int32_t));
    uint8_t* ok = calloc((size_t)P + 1, 1);
    const int32_t cap = s->n_levels + 2;
    int32_t* b1 = malloc((size_t)cap * sizeof(int32_t));
    int32_t* b2 = malloc((size_t)cap * sizeof(int32_t));
    for (int32_t l = 0; l < s->n_levels; ++l)
        for (int32_t i = s->lvl_start[l]; i < s->lvl_start[l + 1]; ++i) {
            const int32_t x = s->lvl_pins[i];
            pred[x] = -1;
            if (s->is_source[x]) {
                delay[x] = 0.0, ok[x] = 1;
                continue;
            }
            int found = 0;
            double best = 0.0;
            int32_t bu = -1;
            for (int32_t j = s->in_start[x]; j < s->in_start[x + 1]; ++j) {
                const int32_t a = s->in_arcs[j], u = s->from[a];
                if (!ok[u]) continue;
                const double cand = delay[u] + arc_delay(s, a, pos);
                int take = !found || cand > best;
                if (found && cand == best) {
                    const int32_t n1 = materialize(pred, u, b1, cap);
                    const int32_t n2 = materialize(pred, bu, b2, cap);
                    b1[n1] = x, b2[n2] = x;
                    take = lex_less(b1, n1 + 1, b2, n2 + 1);
                }
                if (take) best = cand, bu = u, found = 1;
            }
            if (found) delay[x] = best, pred[x] = bu, ok[x] = 1;
        }
    free(s->p_start), free(s->p_pins), free(s->p_slack);
    s->n_paths = nv;
    s->p_start = malloc(((size_t)nv + 1) * sizeof(int32_t));
    s->p_pins = malloc(((size_t)nv * (size_t)cap + 1) * sizeof(int32_t));
    s->p_slack = malloc(((size_t)nv + 1) * sizeof(double));
    int32_t off = 0;
    for (int32_t i = 0; i < nv; ++i) {
        s->p_start[i] = off;
        off += materialize(pred, v[i].pin, s->p_pins + off, cap);
        s->p_slack[i] = nl->clock_period - delay[v[i].pin]; /* paths.cpp:123 */
    }
    s->p_start[nv] = off;
    finish_report(s, counts);
    counts[4] = nv;
    free(v), free(delay), free(pred), free(ok), free(b1), free(b2), free(pos);
    return 0;
}

int cmp_u64(const void* x, const void* y)
{
    const uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
    return (a > b) - (a < b);
}

int cmp_i32(const void* x, const void* y)
{
    const int32_t a = *(const int32_t*)x, b = *(const int32_t*)y;
    return (a > b) - (a < b);
}

int orc_paths_get(void* h, int32_t* start, int32_t* pins, double* slack, int64_t* n_hits)
{
    orc_session* s = h;
    if (start) memcpy(start, s->p_start, ((size_t)s->n_paths + 1) * sizeof(int32_t));
    if (pins) memcpy(pins, s->p_pins, (size_t)s->p_start[s->n_paths] * sizeof(int32_t));
    if (slack) memcpy(slack, s->p_slack, (size_t)s->n_paths * sizeof(double));
    if (n_hits) *n_hits = s->n_hits;
    return 0;
}

int orc_hits_get(void* h, int32_t* a, int32_t* b, double* slack)
{
    orc_session* s = h;
    memcpy(a, s->h_a, (size_t)s->n_hits * sizeof(int32_t));
    memcpy(b, s->h_b, (size_t)s->n_hits * sizeof(int32_t));
    memcpy(slack, s->h_s, (size_t)s->n_hits * sizeof(double));
    return 0;
}

/* ---- PathEnumerator (src/paths.cpp:12-55, include/tdp/paths.hpp:43-93) ----------
 * Lazy k-best enumeration exactly as the reference: per pin a list of found records and a
 * candidate heap holding at most one candidate per in-arc (the next unconsumed predecessor
 * rank, paths.cpp:48-53).  The heap order is a strict total order (delay descending, then the
 * lexicographically smallest full pin sequence, paths.hpp:63-69), so a linear max search over the
 * at most fan-in candidates pops the same candidate as std::priority_queue.  Records link to
 * their predecessor (pin, rank) instead of copying pin vectors. */
typedef struct { double delay; int32_t pp, pr, len; } rea_rec;  /* pred pin / rank (-1: source) */
typedef struct { double delay; int32_t arc, pr; } rea_cand;
typedef struct {
    orc_session* s;
    const double* pos;
    uint8_t* init;
    rea_rec** found;
    int32_t *nf, *cf;
    rea_cand** heap;
    int32_t *nh, *ch;
    int32_t *b1, *b2, cap;
} rea_t;

static void rea_open(rea_t* r, orc_session* s, const double* pos)
{
    const size_t P = (size_t)s->nl.n_pins + 1;
    r->s = s, r->pos = pos;
    r->init = calloc(P, 1);
    r->found = calloc(P, sizeof(rea_rec*));
    r->nf = calloc(P, sizeof(int32_t)), r->cf = calloc(P, sizeof(int32_t));
    r->heap = calloc(P, sizeof(rea_cand*));
    r->nh = calloc(P, sizeof(int32_t)), r->ch = calloc(P, sizeof(int32_t));
    r->cap = s->n_levels + 2;
    r->b1 = malloc((size_t)r->cap * sizeof(int32_t)), r->b2 = malloc((size_t)r->cap * sizeof(int32_t));
}

static void rea_close(rea_t* r)
{
    const size_t P = (size_t)r->s->nl.n_pins + 1;
    for (size_t i = 0; i < P; ++i) free(r->found[i]), free(r->heap[i]);
    free(r->init), free(r->found), free(r->nf), free(r->cf), free(r->heap), free(r->nh), free(r->ch);
    free(r->b1), free(r->b2);
}

/* pin sequence of record (v, k), source first; returns its length */
static int32_t rea_seq(const rea_t* r, int32_t v, int32_t k, int32_t* buf)
{
    const int32_t n = r->found[v][k].len;
    for (int32_t i = n - 1; i >= 0; --i) {
        buf[i] = v;
        const rea_rec* e = &r->found[v][k];
        v = e->pp, k = e->pr;
    }
    return n;
}

/* CandidateOrder (paths.hpp:63-69): does candidate a come out of the heap before b? */
static int rea_before(rea_t* r, int32_t v, const rea_cand* a, const rea_cand* b)
{
    if (a->delay != b->delay) return a->delay > b->delay;
    const orc_session* s = r->s;
    const int32_t na = rea_seq(r, s->from[a->arc], a->pr, r->b1);
    const int32_t nb = rea_seq(r, s->from[b->arc], b->pr, r->b2);
    r->b1[na] = v, r->b2[nb] = v;
    return lex_less(r->b1, na + 1, r->b2, nb + 1);
}

static const rea_rec* rea_path_to(rea_t* r, int32_t v, int32_t rank);

/* push_candidate (paths.cpp:19-31) */
static void rea_push(rea_t* r, int32_t v, int32_t arc, int32_t pred_rank)
{
    const int32_t u = r->s->from[arc];
    const rea_rec* pred = rea_path_to(r, u, pred_rank);
    if (!pred) return;
    rea_cand c;
    c.delay = pred->delay + arc_delay(r->s, arc, r->pos);
    c.arc = arc, c.pr = pred_rank;
    if (r->nh[v] == r->ch[v]) {
        r->ch[v] = r->ch[v] ? 2 * r->ch[v] : 4;
        r->heap[v] = realloc(r->heap[v], (size_t)r->ch[v] * sizeof(rea_cand));
    }
    r->heap[v][r->nh[v]++] = c;
}

static void rea_append(rea_t* r, int32_t v, rea_rec e)
{
    if (r->nf[v] == r->cf[v]) {
        r->cf[v] = r->cf[v] ? 2 * r->cf[v] : 2;
        r->found[v] = realloc(r->found[v], (size_t)r->cf[v] * sizeof(rea_rec));
    }
    r->found[v][r->nf[v]++] = e;
}

/* initialize (paths.cpp:33-42) + path_to (paths.cpp:44-55) */
static const rea_rec* rea_path_to(rea_t* r, int32_t v, int32_t rank)
{
    const orc_session* s = r->s;
    if (!r->init[v]) {
        r->init[v] = 1;
        if (s->is_source[v]) {
            const rea_rec e = {0.0, -1, -1, 1};
            rea_append(r, v, e);
        } else {
            for (int32_t j = s->in_start[v]; j < s->in_start[v + 1]; ++j) rea_push(r, v, s->in_arcs[j], 0);
        }
    }
    while (r->nf[v] <= rank && r->nh[v] > 0) {
        int32_t best = 0;
        for (int32_t i = 1; i < r->nh[v]; ++i)
            if (rea_before(r, v, &r->heap[v][i], &r->heap[v][best])) best = i;
        const rea_cand top = r->heap[v][best];
        r->heap[v][best] = r->heap[v][--r->nh[v]];
        const int32_t u = s->from[top.arc];
        const rea_rec e = {top.delay, u, top.pr, r->found[u][top.pr].len + 1};
        rea_append(r, v, e);
        rea_push(r, v, top.arc, top.pr + 1);
    }
    return rank < r->nf[v] ? &r->found[v][rank] : NULL;
}

typedef struct {
    double slack;
    int32_t off, len;
    const int32_t* pool;
} path_ref;

static int cmp_path(const void* x, const void* y)
{   /* report_timing's order (paths.cpp:155-158): slack ascending, then pin sequence */
    const path_ref* a = x;
    const path_ref* b = y;
    if (a->slack != b->slack) return a->slack < b->slack ? -1 : 1;
    const int32_t* pa = a->pool + a->off;
    const int32_t* pb = b->pool + b->off;
    const int32_t n = a->len < b->len ? a->len : b->len;
    for (int32_t i = 0; i < n; ++i)
        if (pa[i] != pb[i]) return pa[i] < pb[i] ? -1 : 1;
    return (a->len > b->len) - (a->len < b->len);
}

/* report_timing_endpoint (policy 0, paths.cpp:167-189) / report_timing (policy 1, :136-165) at
 * cell_xy (run_sta first).  counts[4] = candidates_generated. */
int orc_extract_policy(void* h, const double* cell_xy, int32_t policy, int32_t n, int32_t k, int64_t counts[5])
{
    orc_session* s = h;
    const tdpg_netlist* nl = &s->nl;
    const int32_t P = nl->n_pins;
    double* pos = malloc(((size_t)P + 1) * 2 * sizeof(double));
    orc_pin_positions(nl, cell_xy, pos);
    sta_at(s, pos);
    ep_rank* v = malloc(((size_t)nl->n_endpoints + 1) * sizeof(ep_rank));
    int32_t nv = 0;
    for (int32_t i = 0; i < nl->n_endpoints; ++i) {
        const int32_t e = nl->endpoints[i];
        if (s->slack[e] < 0.0) v[nv].pin = e, v[nv].slack = s->slack[e], ++nv;
    }
    qsort(v, (size_t)nv, sizeof(ep_rank), cmp_ep);
    if (n <= 0) n = nv; /* the callers' convention: n <= 0 = every violated endpoint (placer.cpp:424-429) */
    if (nv > n) nv = n;
    const int32_t per = policy == 1 ? n : k; /* topn: n paths per endpoint (paths.cpp:148-151) */
    rea_t r;
    rea_open(&r, s, pos);
    /* enumerate_per_endpoint (paths.cpp:108-132), single shared enumerator */
    int64_t np = 0, cap_paths = 16, cap_pins = 1024, used = 0;
    path_ref* refs = malloc((size_t)cap_paths * sizeof(path_ref));
    int32_t* pool = malloc((size_t)cap_pins * sizeof(int32_t));
    for (int32_t i = 0; i < nv; ++i)
        for (int32_t j = 0; j < per; ++j) {
            const rea_rec* rec = rea_path_to(&r, v[i].pin, j);
            if (!rec) break;
            const int32_t len = rec->len;
            const double sl = nl->clock_period - rec->delay; /* paths.cpp:123 */
            if (np == cap_paths) cap_paths *= 2, refs = realloc(refs, (size_t)cap_paths * sizeof(path_ref));
            while (used + len > cap_pins) cap_pins *= 2, pool = realloc(pool, (size_t)cap_pins * sizeof(int32_t));
            rea_seq(&r, v[i].pin, j, pool + used);
            refs[np].slack = sl, refs[np].off = (int32_t)used, refs[np].len = len;
            used += len, ++np;
        }
    rea_close(&r);
    int64_t cand = np;
    if (policy == 1) {
        cand = (int64_t)nv * n; /* paths.cpp:149 */
        for (int64_t i = 0; i < np; ++i) refs[i].pool = pool;
        qsort(refs, (size_t)np, sizeof(path_ref), cmp_path);
        if (np > n) np = n;
    }
    free(s->p_start), free(s->p_pins), free(s->p_slack);
    s->n_paths = (int32_t)np;
    s->p_start = malloc(((size_t)np + 1) * sizeof(int32_t));
    s->p_pins = malloc(((size_t)used + 1) * sizeof(int32_t));
    s->p_slack = malloc(((size_t)np + 1) * sizeof(double));
    int32_t off = 0;
    for (int64_t i = 0; i < np; ++i) {
        s->p_start[i] = off;
        memcpy(s->p_pins + off, pool + refs[i].off, (size_t)refs[i].len * sizeof(int32_t));
        s->p_slack[i] = refs[i].slack;
        off += refs[i].len;
    }
    s->p_start[np] = off;
    finish_report(s, counts);
    counts[4] = cand;
    free(refs), free(pool), free(v), free(pos);
    return 0;
}

/* k_worst_paths_to (paths.cpp:57-72): EndpointError for a non-endpoint; results into the session's
 * path buffers (orc_paths_get). */
int orc_k_worst(void* h, const double* cell_xy, int32_t endpoint, int32_t k, int32_t* n_paths)
{
    orc_session* s = h;
    const tdpg_netlist* nl = &s->nl;
    if (endpoint < 0 || endpoint >= nl->n_pins || !s->is_endpoint[endpoint])
        return fail(TDPG_ERR_ENDPOINT, "validation error: pin %d is not an endpoint", endpoint);
    double* pos = malloc(((size_t)nl->n_pins + 1) * 2 * sizeof(double));
    orc_pin_positions(nl, cell_xy, pos);
    rea_t r;
    rea_open(&r, s, pos);
    free(s->p_start), free(s->p_pins), free(s->p_slack);
    s->p_start = malloc(((size_t)k + 1) * sizeof(int32_t));
    s->p_pins = malloc(((size_t)k * (size_t)r.cap + 1) * sizeof(int32_t));
    s->p_slack = malloc(((size_t)k + 1) * sizeof(double));
    int32_t np = 0, off = 0;
    for (; np < k; ++np) {
        const rea_rec* rec = rea_path_to(&r, endpoint, np);
        if (!rec) break;
        s->p_start[np] = off;
        off += rea_seq(&r, endpoint, np, s->p_pins + off);
        s->p_slack[np] = nl->clock_period - rec->delay;
    }
    s->p_start[np] = off;
    s->n_paths = np;
    s->n_hits = 0;
    rea_close(&r);
    free(pos);
    *n_paths = np;
    return 0;
}

/* ---- ledger: PinPairWeights + update_pair_weights (src/pin_pairs.cpp:7-15) */
static void ledger_reserve(orc_session* s, int64_t n)
{
    if (n <= s->q_cap) return;
    s->q_cap = n * 2 + 16;
    s->la = realloc(s->la, (size_t)s->q_cap * sizeof(int32_t));
    s->lb = realloc(s->lb, (size_t)s->q_cap * sizeof(int32_t));
    s->lw = realloc(s->lw, (size_t)s->q_cap * sizeof(double));
}

int orc_pp_set(void* h, int64_t q, const int32_t* a, const int32_t* b, const double* w)
{
    orc_session* s = h;
    ledger_reserve(s, q);
    memcpy(s->la, a, (size_t)q * sizeof(int32_t));
    memcpy(s->lb, b, (size_t)q * sizeof(int32_t));
    memcpy(s->lw, w, (size_t)q * sizeof(double));
    s->q = q;
    return 0;
}

int orc_pp_get(void* h, int32_t* a, int32_t* b, double* w)
{
    orc_session* s = h;
    memcpy(a, s->la, (size_t)s->q * sizeof(int32_t));
    memcpy(b, s->lb, (size_t)s->q * sizeof(int32_t));
    memcpy(w, s->lw, (size_t)s->q * sizeof(double));
    return 0;
}

typedef struct {
    uint64_t key;
    int64_t idx;
} hit_ref;

static int cmp_hit(const void* x, const void* y)
{
    const hit_ref* a = x;
    const hit_ref* b = y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    return (a->idx > b->idx) - (a->idx < b->idx);
}

static int64_t ledger_find(const orc_session* s, uint64_t key)
{
    int64_t lo = 0, hi = s->q;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        const uint64_t k = ((uint64_t)(uint32_t)s->la[mid] << 32) | (uint32_t)s->lb[mid];
        if (k < key) lo = mid + 1;
        else hi = mid;
    }
    if (lo < s->q && (((uint64_t)(uint32_t)s->la[lo] << 32) | (uint32_t)s->lb[lo]) == key) return lo;
    return -1;
}

/* Sequential semantics: hits in order; first encounter inserts w0, every later one
 * (this round or earlier) adds w1 * (slack / wns).  Grouping the hits by pair with
 * a stable order keeps each pair's additions in hit order, i.e. bitwise equal. */
int orc_pp_update(void* h, int64_t n, const int32_t* a, const int32_t* b, const double* sl, double wns, double w0,
                  double w1, int64_t* q_out)
{
    orc_session* s = h;
    if (wns >= 0.0) {
        if (q_out) *q_out = s->q;
        return 0;
    }
    hit_ref* r = malloc(((size_t)n + 1) * sizeof(hit_ref));
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
        if (sl[i] < 0.0) r[m].key = ((uint64_t)(uint32_t)a[i] << 32) | (uint32_t)b[i], r[m].idx = i, ++m;
    qsort(r, (size_t)m, sizeof(hit_ref), cmp_hit);
    int32_t* na = malloc(((size_t)m + 1) * sizeof(int32_t));
    int32_t* nb = malloc(((size_t)m + 1) * sizeof(int32_t));
    double* nw = malloc(((size_t)m + 1) * sizeof(double));
    int64_t n_new = 0;
    for (int64_t g = 0; g < m;) {
        int64_t e = g;
        while (e < m && r[e].key == r[g].key) ++e;
        const int64_t at = ledger_find(s, r[g].key);
        double w;
        int64_t i = g;
        if (at >= 0) w = s->lw[at];
        else w = w0, ++i;
        for (; i < e; ++i) w += w1 * (sl[r[i].idx] / wns);
        if (at >= 0) s->lw[at] = w;
        else na[n_new] = (int32_t)(r[g].key >> 32), nb[n_new] = (int32_t)(r[g].key & 0xFFFFFFFFu), nw[n_new] = w, ++n_new;
        g = e;
    }
    /* merge the new (sorted) pairs into the ledger */
    if (n_new) {
        const int64_t q0 = s->q;
        ledger_reserve(s, q0 + n_new);
        int64_t i = q0 - 1, j = n_new - 1, k = q0 + n_new - 1;
        while (j >= 0) {
            const uint64_t ki = i >= 0 ? (((uint64_t)(uint32_t)s->la[i] << 32) | (uint32_t)s->lb[i]) : 0;
            const uint64_t kj = ((uint64_t)(uint32_t)na[j] << 32) | (uint32_t)nb[j];
            if (i >= 0 && ki > kj) s->la[k] = s->la[i], s->lb[k] = s->lb[i], s->lw[k] = s->lw[i], --i;
            else s->la[k] = na[j], s->lb[k] = nb[j], s->lw[k] = nw[j], --j;
            --k;
        }
        s->q = q0 + n_new;
    }
    free(r), free(na), free(nb), free(nw);
    if (q_out) *q_out = s->q;
    return 0;
}

/* ---- run_placement: src/placer.cpp:358-484 ------------------------------- */
void orc_config_default(tdpg_config* c)
{
    memset(c, 0, sizeof *c); /* include/tdp/placer.hpp:22-57 */
    c->gamma_frac = 0.01, c->grid_nx = 16, c->grid_ny = 16, c->target_density = 0.6, c->beta = 2.5e-5;
    c->pp_loss = 0, c->net_weighting = 0, c->m = 15, c->w0 = 10.0, c->w1 = 0.2, c->timing_start_iter = 500;
    c->extraction = 0, c->k = 1, c->max_iters = 1500, c->stop_overflow = 0.0, c->mu = 1.05, c->lambda0 = 0.0;
    c->lambda_max = 1e8, c->step0_frac = 0.01, c->step_decay = 0.999, c->adam_beta1 = 0.9, c->adam_beta2 = 0.999;
    c->adam_eps = 1e-8, c->seed = 1, c->init_jitter_frac = 0.02, c->threads = 1;
}

static void clamp_to_core(double* x, double* y, double w, double h, const double* core)
{ /* placer.cpp:99-103, std::clamp */
    const double xh = core[2] - w, yh = core[3] - h;
    *x = *x < core[0] ? core[0] : (xh < *x ? xh : *x);
    *y = *y < core[1] ? core[1] : (yh < *y ? yh : *y);
}

/* placer.cpp:375-382: seeded jitter of every cell that is neither fixed nor explicitly placed */
int orc_jitter(void* h, const double* init_xy, const uint8_t* pos_explicit, const tdpg_config* cfg, double* out_xy)
{
    orc_session* s = h;
    const tdpg_netlist* nl = &s->nl;
    const int32_t C = nl->n_cells;
    const double* core = nl->core;
    const double cw = core[2] - core[0], ch = core[3] - core[1];
    memcpy(out_xy, init_xy, (size_t)C * 2 * sizeof(double));
    orc_mt64 rng;
    orc_mt64_seed(&rng, cfg->seed);
    for (int32_t c = 0; c < C; ++c) {
        if (nl->cell_fixed[c] || (pos_explicit && pos_explicit[c])) continue;
        out_xy[2 * c] += rng_uniform(&rng, -1.0, 1.0) * cfg->init_jitter_frac * cw;
        out_xy[2 * c + 1] += rng_uniform(&rng, -1.0, 1.0) * cfg->init_jitter_frac * ch;
        clamp_to_core(&out_xy[2 * c], &out_xy[2 * c + 1], nl->cell_w[c], nl->cell_h[c], core);
    }
    return 0;
}

int orc_place(void* h, const double* init_xy, const uint8_t* pos_explicit, const tdpg_config* cfg, double* out_xy,
              tdpg_trace_row* trace, int32_t* n_rows, int32_t* stop_overflow, double final_[3])
{
    orc_session* s = h;
    const tdpg_netlist* nl = &s->nl;
    const int32_t C = nl->n_cells, P = nl->n_pins;
    const double* core = nl->core;
    const double cw = core[2] - core[0], ch = core[3] - core[1];
    const double span = cw > ch ? cw : ch;
    const double gamma = cfg->gamma_frac * span;
    orc_jitter(h, init_xy, pos_explicit, cfg, out_xy);
    s->q = 0; /* fresh PinPairWeights */
    double* net_w = NULL;
    double terms[6];
    double* g = malloc((size_t)C * 2 * sizeof(double));
    double lambda = cfg->lambda0;
    if (lambda <= 0.0) {
        int rc = orc_objective(nl, out_xy, cfg->grid_nx, cfg->grid_ny, cfg->target_density, gamma, 0.0, 0.0,
                               cfg->pp_loss, NULL, 0, NULL, NULL, NULL, terms, g);
        double* d0 = malloc((size_t)C * 2 * sizeof(double));
        double dv, dov;
        if (!rc) rc = orc_density(nl, out_xy, cfg->grid_nx, cfg->grid_ny, cfg->target_density, &dv, &dov, d0);
        if (rc) {
            free(g), free(d0);
            return rc;
        }
        double wl1 = 0.0, d1 = 0.0;
        for (int32_t c = 0; c < C; ++c) {
            if (nl->cell_fixed[c]) continue;
            wl1 += fabs(g[2 * c]) + fabs(g[2 * c + 1]);
            d1 += fabs(d0[2 * c]) + fabs(d0[2 * c + 1]);
        }
        lambda = (wl1 > 0.0 && d1 > 0.0) ? wl1 / d1 : 1.0;
        free(d0);
    }
    const double lambda_cap = lambda * cfg->lambda_max;
    double* m = calloc((size_t)C * 2, sizeof(double));
    double* v = calloc((size_t)C * 2, sizeof(double));
    double* flat = malloc((size_t)C * 2 * sizeof(double));
    int32_t t = 0, rows = 0;
    int engaged = 0, rc = 0;
    *stop_overflow = 0;
    double* pos = malloc(((size_t)P + 1) * 2 * sizeof(double));
    for (int32_t iter = 0; iter < cfg->max_iters; ++iter) {
        int sta_row = 0;
        double row_tns = 0.0, row_wns = 0.0;
        if (iter >= cfg->timing_start_iter && (iter - cfg->timing_start_iter) % cfg->m == 0) {
            engaged = 1;
            int64_t cnt[5];
            if (cfg->extraction == 0 && cfg->k == 1) orc_extract(s, out_xy, 0, cnt); /* runs STA; n = n_fail */
            else orc_extract_policy(s, out_xy, cfg->extraction, 0, cfg->k, cnt);    /* placer.cpp:424-429 */
            sta_row = 1, row_tns = s->tns, row_wns = s->wns;
            if (s->wns < 0.0) orc_pp_update(s, s->n_hits, s->h_a, s->h_b, s->h_s, s->wns, cfg->w0, cfg->w1, NULL);
            if (cfg->net_weighting) { /* apply_net_weights, placer.cpp:262-273 */
                if (!net_w) net_w = malloc(((size_t)nl->n_nets + 1) * sizeof(double));
                for (int32_t e = 0; e < nl->n_nets; ++e) {
                    net_w[e] = 1.0;
                    if (s->wns >= 0.0) continue;
                    double worst = s->slack[nl->net_pins[nl->net_start[e]]];
                    for (int32_t i = nl->net_start[e] + 1; i < nl->net_start[e + 1]; ++i)
                        worst = dmin(worst, s->slack[nl->net_pins[i]]);
                    if (worst < 0.0) net_w[e] = 1.0 + (-worst) / (-s->wns);
                }
            }
        }
        rc = orc_objective(nl, out_xy, cfg->grid_nx, cfg->grid_ny, cfg->target_density, gamma, lambda, cfg->beta,
                           cfg->pp_loss, net_w, s->q, s->la, s->lb, s->lw, terms, g);
        if (rc) {
            if (rc == TDPG_ERR_NONFINITE) {
                char tmp[640];
                snprintf(tmp, sizeof tmp, "%s at iteration %d", g_err, iter);
                fail(rc, "%s", tmp);
            }
            break;
        }
        if (trace) {
            tdpg_trace_row* r = &trace[rows];
            r->iter = iter, r->has_timing = sta_row, r->tns = row_tns, r->wns = row_wns;
            r->hpwl = terms[4], r->overflow = terms[5], r->wl_term = terms[1], r->density_term = terms[2];
            r->pp_term = terms[3], r->lambda = lambda, r->beta_pp = cfg->beta * terms[3];
        }
        ++rows;
        if (engaged && terms[5] <= cfg->stop_overflow) {
            *stop_overflow = 1;
            break;
        }
        memcpy(flat, out_xy, (size_t)C * 2 * sizeof(double));
        const double lr = cfg->step0_frac * span * pow(cfg->step_decay, iter);
        orc_adam_step((int64_t)C * 2, flat, g, m, v, &t, lr, cfg->adam_beta1, cfg->adam_beta2, cfg->adam_eps);
        for (int32_t c = 0; c < C; ++c) {
            if (nl->cell_fixed[c]) continue;
            out_xy[2 * c] = flat[2 * c], out_xy[2 * c + 1] = flat[2 * c + 1];
            clamp_to_core(&out_xy[2 * c], &out_xy[2 * c + 1], nl->cell_w[c], nl->cell_h[c], core);
        }
        lambda = dmin(lambda * cfg->mu, lambda_cap);
    }
    if (!rc) {
        orc_pin_positions(nl, out_xy, pos);
        sta_at(s, pos);
        final_[0] = s->tns, final_[1] = s->wns, final_[2] = orc_hpwl_total(nl, pos);
    }
    *n_rows = rows;
    free(pos), free(m), free(v), free(flat), free(g), free(net_w);
    return rc;
}
