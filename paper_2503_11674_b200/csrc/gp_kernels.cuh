// gp_kernels.cuh — per-iteration GP kernels (WA wirelength, pin-pair attraction,
// bin density, fused gradient fold + Adam).  fp64, compiled with -fmad=false so
// every expression rounds exactly like the reference's x86-64 build.
#pragma once

#include "engine.cuh"

namespace tdpg {

constexpr int kBlock = 256;

__device__ __forceinline__ double2 entry_pos(int ec, double2 off, const double2* __restrict__ cell_xy,
                                             const double2* __restrict__ anchor)
{
    const double2 a = ec >= 0 ? cell_xy[ec] : anchor[-1 - ec];
    return make_double2(a.x + off.x, a.y + off.y); // netlist.cpp:28-29
}

__device__ __forceinline__ double2 pin_pos(int p, const int* __restrict__ pin_cell, const double2* __restrict__ off,
                                           const double2* __restrict__ cell_xy, const double2* __restrict__ anchor)
{
    const int c = pin_cell[p];
    const double2 a = c >= 0 ? cell_xy[c] : anchor[p];
    const double2 o = off[p];
    return make_double2(a.x + o.x, a.y + o.y);
}

struct GridDev {
    int nx, ny;
    double x0, y0, bw, bh, cap, scale, inv_scale, total_movable, inv_bw, inv_bh;
    double wide_w, wide_h; // cells wider / taller than this may span more than five bins (Grid::wide)
};

// Footprint of one cell along one axis (extent_weight / extent_weight_grad, density.cpp:41-49, and the
// bin range, :109-112) in three-point form.  Bin centres step by one pitch, so u = (edge - c_j) / pitch
// drops by exactly 1 from bin to bin: each edge meets one right, one middle and one left spline piece,
// at bins a, a+1, a+2 (t = u(a) in [0.5, 1.5)); below a the integral is 1 and the spline 0, above a+2
// both are 0.  So an axis costs six piece evaluations (the reference's formulas, bspline2 :15-22 and
// bspline2_integral :25-36) instead of two full piecewise evaluations per bin.  u differs from the
// reference's (edge - c_j) / pitch by rounding only (well inside the 1e-9 density tolerance).
struct Axis {
    int a_lo, a_hi;          // first piece bin of the lo / hi edge
    int b0, b1;              // bins with possibly non-zero weight, clipped to the grid
    double Flo[3], Fhi[3];   // integral pieces at a, a+1, a+2
    double Blo[3], Bhi[3];   // spline pieces at a, a+1, a+2
    double wscale, inv_len;  // pitch / (hi - lo), 1 / (hi - lo)
};

// U is clamped to [-4, nbins + 4] first: that moves only pieces lying outside the grid (so in-grid
// weights are unchanged) and keeps the bin arithmetic in int range for far-away or infinite edges.
__device__ __forceinline__ void edge_pieces(double U, int nbins, int& a, double (&F)[3], double (&B)[3])
{
    constexpr double kSixth = 1.0 / 6.0, kThird = 1.0 / 3.0;
    U = fmin(fmax(U, -4.0), static_cast<double>(nbins) + 4.0);
    const double af = floor(U - 0.5);
    a = static_cast<int>(af);
    const double t = U - af;    // u at bin a, in [0.5, 1.5)
    const double r = 1.5 - t;   // right piece, u = t
    F[0] = 1.0 - r * r * r * kSixth;
    B[0] = 0.5 * r * r;
    const double m = t - 1.0;   // middle piece, u = t - 1
    F[1] = 0.5 + 0.75 * m - m * m * m * kThird;
    B[1] = 0.75 - m * m;
    const double l = t - 0.5;   // left piece, u = t - 2: (u + 1.5)
    F[2] = l * l * l * kSixth;
    B[2] = 0.5 * l * l;
}

__device__ __forceinline__ Axis make_axis(double lo, double hi, double origin, double pitch, double inv_pitch,
                                          int nbins)
{
    Axis x;
    edge_pieces((lo - origin) * inv_pitch - 0.5, nbins, x.a_lo, x.Flo, x.Blo);
    edge_pieces((hi - origin) * inv_pitch - 0.5, nbins, x.a_hi, x.Fhi, x.Bhi);
    x.b0 = max(0, x.a_lo);
    x.b1 = min(nbins - 1, x.a_hi + 2);
    x.inv_len = 1.0 / (hi - lo);
    x.wscale = pitch * x.inv_len;
    return x;
}

__device__ __forceinline__ double piece_at(const double (&P)[3], int d, double below)
{
    return d < 0 ? below : (d == 0 ? P[0] : (d == 1 ? P[1] : (d == 2 ? P[2] : 0.0)));
}

// Weight and its derivative at bin j: (F(u_hi) - F(u_lo)) * pitch / len, (B(u_hi) - B(u_lo)) / len.
__device__ __forceinline__ void axis_at(const Axis& x, int j, double& w, double& dw)
{
    const int dl = j - x.a_lo, dh = j - x.a_hi;
    w = (piece_at(x.Fhi, dh, 1.0) - piece_at(x.Flo, dl, 1.0)) * x.wscale;
    dw = (piece_at(x.Bhi, dh, 0.0) - piece_at(x.Blo, dl, 0.0)) * x.inv_len;
}

__device__ __forceinline__ double axis_w(const Axis& x, int j)
{
    return (piece_at(x.Fhi, j - x.a_hi, 1.0) - piece_at(x.Flo, j - x.a_lo, 1.0)) * x.wscale;
}

// Fast path: an axis whose edges are at most two piece-bins apart (D = a_hi - a_lo <= 2, i.e. a cell up
// to ~2 bins wide — every movable cell at the configs' grid pitch) has all its weights in the five
// bins a_lo .. a_lo + 4.  The hi edge's pieces are shifted by D with selects; bins outside the grid get
// weight 0 (the reference clips its range, density.cpp:109-112).  Returns false for wider cells.
constexpr int kF5 = 5;
__device__ __forceinline__ bool axis5(double lo, double hi, double origin, double pitch, double inv_pitch, int nbins,
                                      int& b, double (&w)[kF5], double (&dw)[kF5], int* span = nullptr)
{
    double Fl[3], Bl[3], Fh[3], Bh[3];
    int al, ah;
    edge_pieces((lo - origin) * inv_pitch - 0.5, nbins, al, Fl, Bl);
    edge_pieces((hi - origin) * inv_pitch - 0.5, nbins, ah, Fh, Bh);
    const int D = ah - al;
    if (D > 2) return false;
    const bool d0 = D == 0, d1 = D == 1;
    const double fh[kF5] = {d0 ? Fh[0] : 1.0, d0 ? Fh[1] : (d1 ? Fh[0] : 1.0), d0 ? Fh[2] : (d1 ? Fh[1] : Fh[0]),
                            d0 ? 0.0 : (d1 ? Fh[2] : Fh[1]), (d0 || d1) ? 0.0 : Fh[2]};
    const double bh[kF5] = {d0 ? Bh[0] : 0.0, d0 ? Bh[1] : (d1 ? Bh[0] : 0.0), d0 ? Bh[2] : (d1 ? Bh[1] : Bh[0]),
                            d0 ? 0.0 : (d1 ? Bh[2] : Bh[1]), (d0 || d1) ? 0.0 : Bh[2]};
    const double fl[kF5] = {Fl[0], Fl[1], Fl[2], 0.0, 0.0};
    const double bl[kF5] = {Bl[0], Bl[1], Bl[2], 0.0, 0.0};
    const double inv_len = 1.0 / (hi - lo), ws = pitch * inv_len;
#pragma unroll
    for (int j = 0; j < kF5; ++j) {
        const bool in = al + j >= 0 && al + j < nbins;
        w[j] = in ? (fh[j] - fl[j]) * ws : 0.0;
        dw[j] = in ? (bh[j] - bl[j]) * inv_len : 0.0;
    }
    b = al;
    if (span) *span = D + 3; // bins a_lo .. a_lo + D + 2 carry the footprint (the rest are 0)
    return true;
}

struct IterCur { // schedule values of the iteration being executed
    double lr, c1, c2, lambda;
    int iter, do_adam, live, stop; // live: the iteration ran (the engine was not already stopped);
                                   // stop: it met the stop condition (k_fin_terms raises ctrl->stopped)
    double density, overflow;      // the density terms (k_fin_density -> k_fin_terms)
};

struct FinArgs {
    const double *part_wl, *part_hp, *part_pp, *part_d;
    int nb_wa, nb_pp, nb_d;
    double total_movable, beta;
    const Sched* sched;      // per-iteration schedule, or null (single evaluation)
    double lambda_single;    // lambda when sched == null
    double stop_overflow;
    Terms* terms;
    TraceRowDev* trace;      // may be null
    const double* timing_row; // [has_timing, tns, wns] written by the timing refresh
    double* timing_row_clear;
};

// launchers shared by gp.cu / place.cu
void launch_wirelength_ctrl(tdpg_session* s, double gamma, bool use_net_w, double* pw, double* ph, int nb,
                            const Ctrl* ctrl);
void launch_pp_ctrl(tdpg_session* s, int kind, double beta, double* pp, int nb, const Ctrl* ctrl);
void launch_wirelength_pp(tdpg_session* s, double gamma, bool use_net_w, double* part_wl, double* part_hp,
                          bool pp_fused, int kind, double beta, double* part_pp, const Ctrl* ctrl,
                          const cudaStream_t* branch, int n_branch);
void launch_dens_grad(tdpg_session* s, const Ctrl* ctrl, cudaStream_t st);
void launch_density_ctrl(tdpg_session* s, double* pd, int nb, const Ctrl* ctrl);
void launch_density_scatter_ctrl(tdpg_session* s, const Ctrl* ctrl);
void launch_density_bins_ctrl(tdpg_session* s, double* part_d, int nblk, const Ctrl* ctrl);
void launch_finalize(tdpg_session* s, const FinArgs& fa, Ctrl* ctrl, IterCur* cur);
// the finalize split in two (engine iteration graph): the density terms + stop decision + schedule values
// the cell kernel needs, on the density branch; the wirelength / pair terms, trace row and finiteness check
// beside the cell kernel
void launch_fin_density(tdpg_session* s, const FinArgs& fa, Ctrl* ctrl, IterCur* cur, cudaStream_t st);
void launch_fin_terms(tdpg_session* s, const FinArgs& fa, Ctrl* ctrl, const IterCur* cur, cudaStream_t st);
void launch_cells(tdpg_session* s, double2* d_cell, double2* m, double2* v, double b1, double b2, double eps,
                  const IterCur* cur, Ctrl* ctrl, bool dens_grad = true, const double2* folded = nullptr,
                  bool dgrad_folded = false);
void launch_fold(tdpg_session* s, double2* out, const Ctrl* ctrl);
void run_sta_async(tdpg_session* s, double* out3, bool pin_space = true);
void ledger_apply_sorted(tdpg_session* s, long long H, double wns, double w0, double w1);
int api_fail(int kind, const std::string& msg);

} // namespace tdpg
