// place.cu — run_placement (placer.cpp:358-484) as a device-resident loop.
//
// One GP iteration = WA -> pin pairs -> density scatter -> density bins -> finalize ->
// cells (fold + density gradient + Adam + clamp), captured once as a CUDA graph and
// replayed; per-iteration scalars (lr, Adam bias corrections, lambda) come from a
// schedule table computed on the host with the reference's own std::pow sequence, so the
// graph is identical every iteration.  The timing refresh (STA + extraction + ledger
// update, placer.cpp:415-435) runs on the same stream before the scheduled iterations.
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <random>

#include <cub/cub.cuh>

#include "gp_kernels.cuh"

namespace tdpg {

GridDev grid_dev(const tdpg_session* s);

struct Engine {
    tdpg_config cfg{};
    double span = 0, gamma = 0, lambda = 0, lambda_cap = 0;
    DBuf<Sched> sched;
    DBuf<Ctrl> ctrl;
    DBuf<TraceRowDev> trace;
    DBuf<double> timing_row; // has_timing, tns, wns
    DBuf<IterCur> cur;
    DBuf<Terms> terms;
    DBuf<double2> m, v;
    DBuf<double> part;
    DBuf<unsigned long long> obs_count; // observer rounds: unique pin pairs of the refresh
    int nb_wa = 0, nb_pp = 0, nb_d = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    int launched = 0, refreshes = 0, recaptures = 0;
    long long kernel_launches = 0;
    long long paths_host = 0, path_pins_host = 0; // paths extracted by host-sized refreshes (k > 1 / topn)
    int kernels_per_iter = 8; // 2 WA class groups + generic + scatter + bins + dens_grad + finalize + cells
    cudaGraphExec_t refresh_gexec = nullptr; // the whole timing refresh, captured once
    cudaGraphExec_t sort_gexec = nullptr;    // spatial re-sort of the cells
    cudaGraphExec_t gexec_sorted = nullptr;  // re-sort + iteration (non-partitioned engine)
    cudaGraphExec_t old_gexec = nullptr, old_gexec_sorted = nullptr, old_refresh = nullptr, old_sort = nullptr;
    bool old_lonly = false;
    unsigned long long old_epoch = 0;
    tdpg_config old_cfg{};
    int old_sort_every = 0;
    double consts[3] = {0, 0, 0}, old_consts[3] = {0, 0, 0}; // clock, r_unit, c_unit baked into the graphs
    unsigned long long epoch = 0;            // dbuf_epoch() when the graphs were captured
    bool refresh_lonly = false;              // the refresh graph leaves the STA results in L-space only
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> refresh_ev;
    int sort_every = 2; // iterations between spatial re-sorts of the cells (engine_init: 2 from 500K movable cells,
                        // else 4; bench iters/s at 200K: 2: 9,397, 3: 9,852, 4: 10,095; 1M ms/step over iterations
                        // 20-220: 1: 0.317, 2: 0.299, 3: 0.301, 4: 0.305; 4M: 2 vs 4 = 904 vs ~790 iters/s)
    double last_refresh_ms = 0, total_refresh_ms = 0;
    // branch streams + fork/join events of the captured iteration graph (density chain and the WA
    // size classes run as parallel graph branches)
    static constexpr int kBranches = 8;
    // partitioned mode: all-reduce buffer [partial d_cell (2C) | WA, HPWL, PP block partials (3 nb_wa)];
    // with a communicator the all-reduce sits inside gexec, otherwise (tests: reduction done by the
    // caller) the iteration is two graphs around it
    bool partitioned = false;
    DBuf<double> red;
    cudaGraphExec_t gexec_a0 = nullptr, gexec_a = nullptr, gexec_b = nullptr; // split phase: scatter | rest | cells
    int mov_lo = 0, mov_hi = 0; // this rank's slice of the spatial cell order (sharded density)
    cudaStream_t br[kBranches] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[kBranches] = {}, ev_bins = nullptr;
    ~Engine()
    {
        for (auto& b : br)
            if (b) cudaStreamDestroy(b);
        for (auto& e : ev_join)
            if (e) cudaEventDestroy(e);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_bins) cudaEventDestroy(ev_bins);
        if (gexec) cudaGraphExecDestroy(gexec);
        if (gexec_a0) cudaGraphExecDestroy(gexec_a0);
        if (gexec_a) cudaGraphExecDestroy(gexec_a);
        if (gexec_b) cudaGraphExecDestroy(gexec_b);
        if (graph) cudaGraphDestroy(graph);
        if (refresh_gexec) cudaGraphExecDestroy(refresh_gexec);
        if (sort_gexec) cudaGraphExecDestroy(sort_gexec);
        if (gexec_sorted) cudaGraphExecDestroy(gexec_sorted);
        for (cudaGraphExec_t g : {old_gexec, old_gexec_sorted, old_refresh, old_sort})
            if (g) cudaGraphExecDestroy(g);
        for (auto& e : refresh_ev) cudaEventDestroy(e.first), cudaEventDestroy(e.second);
    }
    // a previous engine of the session (engine_init again): its buffers, branch streams and events are
    // taken over instead of freed and re-allocated (cudaFree synchronises the device)
    void recycle(Engine& o)
    {
        sched = std::move(o.sched), ctrl = std::move(o.ctrl), trace = std::move(o.trace);
        timing_row = std::move(o.timing_row), cur = std::move(o.cur), terms = std::move(o.terms);
        m = std::move(o.m), v = std::move(o.v), part = std::move(o.part), red = std::move(o.red);
        obs_count = std::move(o.obs_count);
        std::swap(br, o.br), std::swap(ev_fork, o.ev_fork), std::swap(ev_join, o.ev_join);
        std::swap(ev_bins, o.ev_bins);
        if (!o.partitioned && o.gexec && !o.gexec_a) { // its graphs, for adopt_graphs
            std::swap(old_gexec, o.gexec), std::swap(old_gexec_sorted, o.gexec_sorted);
            std::swap(old_refresh, o.refresh_gexec), std::swap(old_sort, o.sort_gexec);
            old_lonly = o.refresh_lonly, old_epoch = o.epoch, old_cfg = o.cfg, old_sort_every = o.sort_every;
            std::memcpy(old_consts, o.consts, sizeof consts);
        }
    }
    // the configuration fields the captured graphs depend on (kernel arguments, schedule layout); the
    // ignored `threads` and the iteration count are not among them, nor are padding bytes
    static bool graph_cfg_equal(const tdpg_config& a, const tdpg_config& b)
    {
        auto same = [](double x, double y) { return std::memcmp(&x, &y, sizeof x) == 0; };
        return same(a.gamma_frac, b.gamma_frac) && a.grid_nx == b.grid_nx && a.grid_ny == b.grid_ny &&
               same(a.target_density, b.target_density) && same(a.beta, b.beta) && a.pp_loss == b.pp_loss &&
               a.net_weighting == b.net_weighting && a.m == b.m && same(a.w0, b.w0) && same(a.w1, b.w1) &&
               a.timing_start_iter == b.timing_start_iter && a.extraction == b.extraction && a.k == b.k &&
               same(a.stop_overflow, b.stop_overflow) && same(a.mu, b.mu) && same(a.lambda0, b.lambda0) &&
               same(a.lambda_max, b.lambda_max) && same(a.step0_frac, b.step0_frac) &&
               same(a.step_decay, b.step_decay) && same(a.adam_beta1, b.adam_beta1) &&
               same(a.adam_beta2, b.adam_beta2) && same(a.adam_eps, b.adam_eps) && a.seed == b.seed &&
               same(a.init_jitter_frac, b.init_jitter_frac) && a.density_model == b.density_model;
    }
    static void session_consts(const tdpg_session* s, double (&c)[3]) { c[0] = s->clock, c[1] = s->r_unit, c[2] = s->c_unit; }
    bool consts_match(const tdpg_session* s) const
    {
        double c[3];
        session_consts(s, c);
        return std::memcmp(c, consts, sizeof c) == 0;
    }
    // The previous engine's graphs point into exactly this engine's (recycled) buffers when no device
    // buffer moved since they were captured and the configuration (baked into kernel arguments) matches.
    bool adopt_graphs(const tdpg_session* s)
    {
        double c[3];
        session_consts(s, c);
        if (!old_gexec || old_epoch != dbuf_epoch() || partitioned || old_sort_every != sort_every ||
            !graph_cfg_equal(old_cfg, cfg) || std::memcmp(c, old_consts, sizeof c) != 0) {
            if (const char* e = std::getenv("TDPG_TRACE_INIT"); e && std::atoi(e) != 0)
                std::fprintf(stderr, "engine_init graphs not adopted: old %d epoch %llu/%llu part %d sort %d/%d cfg %d consts %d\n",
                             old_gexec != nullptr, (unsigned long long)old_epoch, dbuf_epoch().load(), partitioned, old_sort_every, sort_every,
                             graph_cfg_equal(old_cfg, cfg), std::memcmp(c, old_consts, sizeof c) == 0);
            // never adoptable now (this engine captures its own): freed here, in the call that re-captures
            // anyway, rather than by this engine's destructor inside the next engine_init
            for (cudaGraphExec_t* g : {&old_gexec, &old_gexec_sorted, &old_refresh, &old_sort})
                if (*g) cudaGraphExecDestroy(*g), *g = nullptr;
            return false;
        }
        std::swap(gexec, old_gexec), std::swap(gexec_sorted, old_gexec_sorted);
        std::swap(refresh_gexec, old_refresh), std::swap(sort_gexec, old_sort);
        refresh_lonly = old_lonly, epoch = old_epoch;
        std::memcpy(consts, old_consts, sizeof consts);
        return true;
    }
    double refresh_ms()
    {
        double t = 0.0;
        for (auto& e : refresh_ev) {
            float ms = 0.f;
            if (cudaEventSynchronize(e.second) == cudaSuccess && cudaEventElapsedTime(&ms, e.first, e.second) == cudaSuccess)
                t += ms;
        }
        return t;
    }
};

namespace {

void validate_config(const tdpg_config& c)
{ // placer.cpp:68-90, same messages
    auto bad = [](const char* m) { throw Error(TDPG_ERR_VALIDATION, std::string("validation error: config: ") + m); };
    if (c.grid_nx < 1 || c.grid_ny < 1) bad("density grid must be at least 1x1");
    if (!(c.target_density > 0.0)) bad("target_density must be > 0");
    if (!(c.gamma_frac > 0.0)) bad("gamma_frac must be > 0");
    if (c.beta < 0.0) bad("beta must be >= 0");
    if (c.m < 1) bad("m must be >= 1");
    if (!(c.w0 > 0.0)) bad("w0 must be > 0");
    if (c.w1 < 0.0) bad("w1 must be >= 0");
    if (c.timing_start_iter < 0) bad("timing_start_iter must be >= 0");
    if (c.k < 1) bad("k must be >= 1");
    if (c.max_iters < 0) bad("max_iters must be >= 0");
    if (c.stop_overflow < 0.0) bad("stop_overflow must be >= 0");
    if (!(c.mu > 0.0)) bad("mu must be > 0");
    if (!(c.lambda_max > 0.0)) bad("lambda_max must be > 0");
    if (!(c.step0_frac > 0.0)) bad("step0_frac must be > 0");
    if (!(c.step_decay > 0.0 && c.step_decay <= 1.0)) bad("step_decay must be in (0, 1]");
    if (!(c.adam_beta1 >= 0.0 && c.adam_beta1 < 1.0) || !(c.adam_beta2 >= 0.0 && c.adam_beta2 < 1.0))
        bad("adam betas must be in [0, 1)");
    if (!(c.adam_eps > 0.0)) bad("adam_eps must be > 0");
    if (c.init_jitter_frac < 0.0) bad("init_jitter_frac must be >= 0");
    if (c.threads < 1) bad("threads must be >= 1");
    if (c.extraction != 0 && c.extraction != 1) bad("extraction must be \"endpoint\" or \"topn\"");
    if (c.density_model != 0 && c.density_model != 1) bad("density_model must be \"overflow\" or \"electrostatic\"");
}

__global__ void k_l1_pair(int C, const double2* __restrict__ a, const double2* __restrict__ b,
                          const uint8_t* __restrict__ fixed, double* __restrict__ part)
{
    __shared__ double sh[kBlock / 32];
    double sa = 0.0, sb = 0.0;
    for (int c = blockIdx.x * kBlock + threadIdx.x; c < C; c += gridDim.x * kBlock) {
        if (fixed[c]) continue;
        sa += fabs(a[c].x) + fabs(a[c].y);
        sb += fabs(b[c].x) + fabs(b[c].y);
    }
    sa = block_sum<kBlock>(sa, sh);
    sb = block_sum<kBlock>(sb, sh);
    if (threadIdx.x == 0) part[2 * blockIdx.x] = sa, part[2 * blockIdx.x + 1] = sb;
}

// lambda0 "auto": |grad WL|_1 / |grad D|_1 over movable cells (placer.cpp:388-402).  One evaluation at
// lambda = 0 leaves both: d_cell = fold + 0 * density gradient is the wirelength gradient, and the raw
// density gradient in dgrad is what a lambda = 1 cell pass over zero entry gradients returns (0 + 1 * g),
// so the two norms are bitwise those of two separate passes.
double lambda_auto(tdpg_session* s, double gamma, int kind)
{
    evaluate_objective(s, gamma, 0.0, 0.0, kind, false, nullptr);
    const int nb_d = bins_blocks(s), nb = 148 * 2;
    s->lam_scratch.reserve(2 * static_cast<size_t>(s->C) + 2 * nb_d + 64 + 2 * nb);
    double* p2 = s->lam_scratch.p;
    k_l1_pair<<<nb, kBlock, 0, s->st>>>(s->C, s->d_cell, s->dgrad, s->cell_fixed, p2);
    CK_LAUNCH();
    // the loop expects zero entry gradients where its own kernels do not write (off-net pin slots; in a
    // partitioned engine, the other ranks' nets)
    s->grad_e.zero(s->st, s->E_tot);
    std::vector<double> h(2 * nb);
    CK(cudaMemcpyAsync(h.data(), p2, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    double wl1 = 0.0, d1 = 0.0;
    for (int i = 0; i < nb; ++i) wl1 += h[2 * i], d1 += h[2 * i + 1];
    return (wl1 > 0.0 && d1 > 0.0) ? wl1 / d1 : 1.0;
}

template <typename F>
cudaGraphExec_t capture(tdpg_session* s, F&& record)
{
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
    CK(cudaStreamBeginCapture(s->st, cudaStreamCaptureModeThreadLocal));
    record();
    CK(cudaStreamEndCapture(s->st, &g));
    CK(cudaGraphInstantiate(&x, g, 0));
    cudaGraphDestroy(g);
    return x;
}

// TDPG_GP_PDL=0: record the iteration graph without programmatic dependent launch edges
bool pdl_gp()
{
    static const bool on = [] {
        const char* e = std::getenv("TDPG_GP_PDL");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

// TDPG_FIN_SPLIT=0: one finalize kernel at the join (A/B switch).
bool fin_split()
{
    static const bool on = [] {
        const char* e = std::getenv("TDPG_FIN_SPLIT");
        return !(e && std::atoi(e) == 0);
    }();
    return on;
}

void capture_iteration(tdpg_session* s, Engine& E)
{
    const bool split = fin_split(); // (the finalize in two halves, both graph forms)
    if (E.gexec) cudaGraphExecDestroy(E.gexec), E.gexec = nullptr;
    double* part_wl = E.part.p;
    double* part_hp = part_wl + E.nb_wa;
    double* part_pp = part_hp + E.nb_wa;
    double* part_d = part_pp + E.nb_pp;
    FinArgs fa{};
    fa.part_wl = part_wl, fa.part_hp = part_hp, fa.part_pp = part_pp, fa.part_d = part_d;
    fa.nb_wa = E.nb_wa, fa.nb_pp = E.nb_pp, fa.nb_d = E.nb_d;
    fa.total_movable = s->grid.total_movable, fa.beta = E.cfg.beta;
    fa.sched = E.sched, fa.stop_overflow = E.cfg.stop_overflow, fa.terms = E.terms, fa.trace = E.trace;
    fa.timing_row = E.timing_row, fa.timing_row_clear = E.timing_row;
    if (!E.ev_bins) CK(cudaEventCreateWithFlags(&E.ev_bins, cudaEventDisableTiming));
    if (!E.ev_fork) {
        CK(cudaEventCreateWithFlags(&E.ev_fork, cudaEventDisableTiming));
        for (int k = 0; k < Engine::kBranches; ++k) {
            CK(cudaStreamCreateWithFlags(&E.br[k], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&E.ev_join[k], cudaEventDisableTiming));
        }
    }
    if (E.partitioned) {
        const long long C2 = 2LL * s->C;
        double* r_wl = E.red.p + C2;
        double* r_hp = r_wl + E.nb_wa;
        double* r_pp = r_hp + E.nb_wa;
        FinArgs fp = fa;
        fp.part_wl = r_wl, fp.part_hp = r_hp, fp.part_pp = r_pp;
        double2* folded = reinterpret_cast<double2*>(E.red.p);
        // Sharded iteration: fork; density branch: scatter of this rank's cell slice -> [int64 grid sum over
        // ranks] -> bins (replicated) -> density gradient of the slice; WA branches over this rank's nets;
        // join, fold this rank's entries + lambda * its cells' density gradient -> [sum over ranks] ->
        // finalize -> cells (replicated Adam).
        const int lo = E.mov_lo, hi = E.mov_hi;
        auto scatter = [&] { launch_density_scatter_part(s, E.ctrl, lo, hi, s->part_rank == 0); };
        auto record_a = [&](bool comm) {
            cudaStream_t main = s->st;
            CK(cudaEventRecord(E.ev_fork, main));
            for (int k = 0; k < Engine::kBranches; ++k) CK(cudaStreamWaitEvent(E.br[k], E.ev_fork, 0));
            s->st = E.br[0];
            if (comm) {
                scatter();
                comm_allreduce_i64(s, s->grid.acc.p, static_cast<size_t>(s->grid.bins()), E.br[0]);
            }
            launch_density_bins_ctrl(s, part_d, E.nb_d, E.ctrl);
            if (split) { // the density half of the finalize beside the slice's density gradient (see below)
                CK(cudaEventRecord(E.ev_bins, E.br[0]));
                CK(cudaStreamWaitEvent(E.br[3], E.ev_bins, 0));
                launch_fin_density(s, fa, E.ctrl, E.cur, E.br[3]);
            }
            launch_dens_grad_part(s, E.ctrl, E.br[0], lo, hi);
            s->st = main;
            cudaStream_t wa_st[Engine::kBranches] = {main};
            for (int k = 1; k < Engine::kBranches; ++k) wa_st[k] = E.br[k];
            launch_wirelength_pp(s, E.gamma, E.cfg.net_weighting != 0, r_wl, r_hp, true, E.cfg.pp_loss, E.cfg.beta,
                                 r_pp, E.ctrl, wa_st, Engine::kBranches);
            for (int k = 1; k < Engine::kBranches; ++k) {
                CK(cudaEventRecord(E.ev_join[k], E.br[k]));
                CK(cudaStreamWaitEvent(main, E.ev_join[k], 0));
            }
            launch_fold(s, folded, E.ctrl);
            CK(cudaEventRecord(E.ev_join[0], E.br[0]));
            CK(cudaStreamWaitEvent(main, E.ev_join[0], 0));
            launch_add_dgrad(s, E.sched, E.ctrl, folded, lo, hi);
        };
        // B: terms from the reduced partials, cells from the reduced fold (density gradient included)
        auto record_b = [&] {
            if (split) { // the terms half (reduced partials) beside the cell kernel
                cudaStream_t main = s->st;
                CK(cudaEventRecord(E.ev_fork, main));
                CK(cudaStreamWaitEvent(E.br[4], E.ev_fork, 0));
                launch_fin_terms(s, fp, E.ctrl, E.cur, E.br[4]);
                CK(cudaEventRecord(E.ev_join[4], E.br[4]));
                launch_cells(s, nullptr, E.m, E.v, E.cfg.adam_beta1, E.cfg.adam_beta2, E.cfg.adam_eps, E.cur, E.ctrl,
                             false, folded, true);
                CK(cudaStreamWaitEvent(main, E.ev_join[4], 0));
                return;
            }
            launch_finalize(s, fp, E.ctrl, E.cur);
            launch_cells(s, nullptr, E.m, E.v, E.cfg.adam_beta1, E.cfg.adam_beta2, E.cfg.adam_eps, E.cur, E.ctrl,
                         false, folded, true);
        };
        const size_t n_red = static_cast<size_t>(C2) + 3 * static_cast<size_t>(E.nb_wa);
        s->part_active = true;
        if (s->comm) {
            E.gexec = capture(s, [&] {
                record_a(true);
                comm_allreduce(s, E.red.p, n_red);
                record_b();
            });
        } else {
            E.gexec_a0 = capture(s, scatter);
            E.gexec_a = capture(s, [&] { record_a(false); });
            E.gexec_b = capture(s, record_b);
        }
        s->part_active = false;
        return;
    }
    s->pdl_graph = pdl_gp();
    auto record = [&](bool sort) {
        // fork: density chain (scatter -> bins -> density gradient) on branch 0, the WA size classes
        // (+ fused pin pairs, dense ledger) on the main stream and branches 1..7; join -> finalize -> cells
        cudaStream_t main = s->st;
        CK(cudaEventRecord(E.ev_fork, main));
        for (int k = 0; k < Engine::kBranches; ++k) CK(cudaStreamWaitEvent(E.br[k], E.ev_fork, 0));
        s->st = E.br[0];
        if (sort) sort_cells_spatial(s); // (only the density kernels read the spatial order)
        launch_density_ctrl(s, part_d, E.nb_d, E.ctrl);
        CK(cudaEventRecord(E.ev_bins, E.br[0])); // the density value partials are ready
        // split finalize: the density half (stop decision, schedule values for the cell kernel) on its own
        // branch beside the density gradient, so the cell kernel waits for the WA kernels, the density
        // gradient and it; the terms half (wirelength / pair terms, trace row) runs beside the cell kernel
        if (split) {
            CK(cudaStreamWaitEvent(E.br[3], E.ev_bins, 0));
            launch_fin_density(s, fa, E.ctrl, E.cur, E.br[3]);
            CK(cudaEventRecord(E.ev_join[3], E.br[3]));
        }
        launch_dens_grad(s, E.ctrl, E.br[0]);
        s->st = main;
        cudaStream_t wa_st[Engine::kBranches] = {main};
        for (int k = 1; k < Engine::kBranches; ++k) wa_st[k] = E.br[k];
        launch_wirelength_pp(s, E.gamma, E.cfg.net_weighting != 0, part_wl, part_hp, true, E.cfg.pp_loss,
                             E.cfg.beta, part_pp, E.ctrl, wa_st, Engine::kBranches);
        // finalize needs the WA partials and the density value, not the density gradient: it runs
        // beside the gradient kernel, and the cell kernel joins both
        for (int k = 1; k < Engine::kBranches; ++k) {
            CK(cudaEventRecord(E.ev_join[k], E.br[k]));
            CK(cudaStreamWaitEvent(main, E.ev_join[k], 0));
        }
        if (split) {
            CK(cudaEventRecord(E.ev_fork, main)); // (reused: every WA kernel is done)
            CK(cudaStreamWaitEvent(E.br[4], E.ev_fork, 0));
            CK(cudaStreamWaitEvent(E.br[4], E.ev_join[3], 0));
            launch_fin_terms(s, fa, E.ctrl, E.cur, E.br[4]);
            CK(cudaEventRecord(E.ev_join[4], E.br[4]));
            CK(cudaStreamWaitEvent(main, E.ev_join[3], 0));
        } else {
            CK(cudaStreamWaitEvent(main, E.ev_bins, 0));
            launch_finalize(s, fa, E.ctrl, E.cur);
        }
        CK(cudaEventRecord(E.ev_join[0], E.br[0]));
        CK(cudaStreamWaitEvent(main, E.ev_join[0], 0));
        launch_cells(s, nullptr, E.m, E.v, E.cfg.adam_beta1, E.cfg.adam_beta2, E.cfg.adam_eps, E.cur, E.ctrl,
                     false);
        if (split) CK(cudaStreamWaitEvent(main, E.ev_join[4], 0));
    };
    E.gexec = capture(s, [&] { record(false); });
    // the iterations that re-sort the cells: the sort heads the density branch, beside the WA kernels
    if (E.gexec_sorted) cudaGraphExecDestroy(E.gexec_sorted);
    E.gexec_sorted = capture(s, [&] { record(true); });
    s->pdl_graph = false;
}

} // namespace

void record_refresh(tdpg_session* s, Engine& E);

// TDPG_TRACE_INIT=1: engine_init phase times on stderr (host clock, stream synchronised)
struct InitTrace {
    bool on = false;
    std::chrono::steady_clock::time_point t;
    tdpg_session* s;
    explicit InitTrace(tdpg_session* ss) : s(ss)
    {
        const char* e = std::getenv("TDPG_TRACE_INIT");
        on = e && std::atoi(e) != 0;
        t = std::chrono::steady_clock::now();
    }
    void mark(const char* what)
    {
        if (!on) return;
        cudaStreamSynchronize(s->st);
        const auto n = std::chrono::steady_clock::now();
        std::fprintf(stderr, "engine_init %-22s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
        t = n;
    }
};

// ---- initial jitter (placer.cpp:375-382): every cell that is neither fixed nor explicitly placed, in
// cell order, takes two draws of a std::mt19937_64 seeded with cfg.seed (x then y), each mapped to
// rng_uniform(-1, 1) = -1 + 2 (draw >> 11) 2^-53, scaled by init_jitter_frac * core extent, then clamped
// into the core.  The raw engine stream is generated on the device, bitwise the libstdc++ sequence.
// With x[0..311] the seeded state and x[312 + k] the word tempered into draw k, the engine's
// regeneration is the lag-156 recurrence  x[j] = x[j - 156] ^ mix(x[j - 312], x[j - 311]),  so 156
// consecutive words are independent: thread t of one block computes word 312 + 156 k + t in step k,
// keeping x[j - 156] and x[j - 312] (its own last two words) in registers; x[j - 311] is thread t + 1's
// word of step k - 2 (thread 0's of step k - 1 for t = 155), read from a ring of steps in shared memory.
// Two steps per barrier: step k + 1 reads step k - 1 words only, except thread 155, which recomputes thread
// 0's step-k word from the ring.  The untempered words are stored; k_jit_apply tempers them.
constexpr int kMtN = 312, kMtM = 156;

__device__ __forceinline__ unsigned long long mt_mix(unsigned long long a, unsigned long long b)
{
    const unsigned long long y = (a & 0xFFFFFFFF80000000ull) | (b & 0x7FFFFFFFull);
    return (y >> 1) ^ ((0ull - (y & 1ull)) & 0xB5026F5AA96619E9ull);
}

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long y)
{
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    return y ^ (y >> 43);
}

__global__ void __launch_bounds__(160) k_mt19937_64(unsigned long long seed, const int* __restrict__ count,
                                                    int count_host, unsigned long long* __restrict__ out)
{
    __shared__ unsigned long long ring[4][kMtM];
    const int t = threadIdx.x;
    if (t == 0) { // the seeded state x[0..311] into ring slots 2 (x[0..155]) and 3 (x[156..311])
        unsigned long long x = seed;
        ring[2][0] = x;
        for (int i = 1; i < kMtN; ++i) {
            x = 6364136223846793005ull * (x ^ (x >> 62)) + i;
            ring[2 + i / kMtM][i % kMtM] = x;
        }
    }
    __syncthreads();
    unsigned long long r2 = 0, r1 = 0; // this thread's words of steps k - 2 and k - 1
    if (t < kMtM) r2 = ring[2][t], r1 = ring[3][t];
    const long long need = 2LL * (count ? *count : count_host);
    int s0 = 0; // ring slot of step k (steps k - 2, k - 1 in s0 + 2, s0 + 3 mod 4)
    for (long long base = 0; base < need; base += 2 * kMtM) {
        const int sm2 = (s0 + 2) & 3, sm1 = (s0 + 3) & 3, s1 = (s0 + 1) & 3;
        if (t < kMtM) {
            const unsigned long long b0 = t + 1 < kMtM ? ring[sm2][t + 1] : ring[sm1][0];
            unsigned long long b1;
            if (t + 1 < kMtM) b1 = ring[sm1][t + 1];
            else b1 = ring[sm1][0] ^ mt_mix(ring[sm2][0], ring[sm2][1]); // thread 0's step-k word
            const unsigned long long m1 = mt_mix(r1, b1);
            const unsigned long long x0 = r1 ^ mt_mix(r2, b0);
            const unsigned long long x1 = x0 ^ m1;
            ring[s0][t] = x0, ring[s1][t] = x1;
            r2 = x0, r1 = x1;
            if (base + t < need) out[base + t] = x0;
            if (base + kMtM + t < need) out[base + kMtM + t] = x1;
        }
        __syncthreads();
        s0 = (s0 + 2) & 3;
    }
}

__global__ void k_fill_f64(int n, double* __restrict__ p, double v)
{
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i < n) p[i] = v;
}

__global__ void k_jit_flags(int C, const uint8_t* __restrict__ fixed, const uint8_t* __restrict__ expl,
                            int* __restrict__ flag)
{
    const int c = blockIdx.x * kBlock + threadIdx.x;
    if (c < C) flag[c] = !fixed[c] && !(expl && expl[c]);
    else if (c == C) flag[c] = 0;
}

__global__ void k_jit_apply(int C, const int* __restrict__ flag, const int* __restrict__ rank,
                            const unsigned long long* __restrict__ raw, const double2* __restrict__ wh,
                            double2* __restrict__ xy, double frac, double cw, double ch, double4 core)
{
    const int c = blockIdx.x * kBlock + threadIdx.x;
    if (c >= C || !flag[c]) return;
    const long long r = 2LL * rank[c];
    const double ux = __ull2double_rn(mt_temper(raw[r]) >> 11) * 0x1.0p-53;
    const double uy = __ull2double_rn(mt_temper(raw[r + 1]) >> 11) * 0x1.0p-53;
    double2 p = xy[c];
    p.x = p.x + (-1.0 + (1.0 - -1.0) * ux) * frac * cw;
    p.y = p.y + (-1.0 + (1.0 - -1.0) * uy) * frac * ch;
    const double xh = core.z - wh[c].x, yh = core.w - wh[c].y;
    p.x = p.x < core.x ? core.x : (xh < p.x ? xh : p.x); // std::clamp
    p.y = p.y < core.y ? core.y : (yh < p.y ? yh : p.y);
    xy[c] = p;
}

void jitter_positions(tdpg_session* s, const tdpg_config* cfg, const uint8_t* pos_explicit, double cw, double ch,
                      InitTrace* tr = nullptr)
{
    const int C = s->C;
    s->jit_flag.reserve(C + 1), s->jit_rank.reserve(C + 1), s->jit_raw.reserve(2 * static_cast<size_t>(C) + 1);
    // which cells take a draw and their rank among them: recomputed only when pos_explicit changed
    const bool same = s->jit_flags_ok && s->jit_flags_at[0] == s->jit_flag.p && s->jit_flags_at[1] == s->jit_rank.p &&
                      (pos_explicit ? !s->jit_expl_null && s->h_jit_expl.size() == static_cast<size_t>(C) &&
                                          std::memcmp(s->h_jit_expl.data(), pos_explicit, C) == 0
                                    : s->jit_expl_null);
    if (!same) {
        const uint8_t* ex = nullptr;
        if (pos_explicit) s->jit_expl.upload(pos_explicit, C, s->st), ex = s->jit_expl.p;
        k_jit_flags<<<blocks_for(C + 1, kBlock), kBlock, 0, s->st>>>(C, s->cell_fixed, ex, s->jit_flag);
        CK_LAUNCH();
        size_t bytes = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, bytes, s->jit_flag.p, s->jit_rank.p, C + 1, s->st);
        void* tmp = cub_scratch(s, bytes);
        CK(cub::DeviceScan::ExclusiveSum(tmp, bytes, s->jit_flag.p, s->jit_rank.p, C + 1, s->st));
        s->jit_expl_null = pos_explicit == nullptr;
        if (pos_explicit) s->h_jit_expl.assign(pos_explicit, pos_explicit + C);
        else s->h_jit_expl.clear();
        s->jit_flags_at[0] = s->jit_flag.p, s->jit_flags_at[1] = s->jit_rank.p, s->jit_flags_ok = true;
    }
    // the raw stream depends on the seed only: every free cell's two draws are generated once per seed
    // (explicitly placed cells only shorten the prefix used) and kept for the next run with that seed
    if (s->n_free < 0) {
        int nf = 0;
        for (int c = 0; c < C; ++c) nf += s->h_cell_fixed[c] ? 0 : 1;
        s->n_free = nf;
    }
    const unsigned long long seed = static_cast<unsigned long long>(cfg->seed);
    const long long need = 2LL * s->n_free;
    if (!(s->jit_count >= need && s->jit_seed == seed && s->jit_ptr == s->jit_raw.p)) {
        s->jit_rank.reserve(C + 2);
        k_mt19937_64<<<1, 160, 0, s->st>>>(seed, nullptr, static_cast<int>(s->n_free), s->jit_raw);
        CK_LAUNCH();
        s->jit_seed = seed, s->jit_count = need, s->jit_ptr = s->jit_raw.p;
    }
    if (tr) tr->mark("jitter: flags + scan + mt19937_64");
    k_jit_apply<<<blocks_for(C, kBlock), kBlock, 0, s->st>>>(
        C, s->jit_flag, s->jit_rank, s->jit_raw, s->cell_wh, s->cell_xy, cfg->init_jitter_frac, cw, ch,
        make_double4(s->core[0], s->core[1], s->core[2], s->core[3]));
    CK_LAUNCH();
    s->sta_valid = false;
    s->pin_xy_external = false;
    refresh_fixed_baseline(s);
}

void engine_init(tdpg_session* s, const tdpg_config* cfg, const uint8_t* pos_explicit)
{
    InitTrace tr(s);
    validate_config(*cfg);
    auto E = std::make_unique<Engine>();
    E->cfg = *cfg;
    const double cw = s->core[2] - s->core[0], ch = s->core[3] - s->core[1];
    E->span = cw > ch ? cw : ch; // Rect::span (geometry.hpp:34)
    E->gamma = cfg->gamma_frac * E->span;

    // implicit starts get a seeded jitter (placer.cpp:375-382), on the device; the host work below
    // (old engine, graph captures) overlaps it
    jitter_positions(s, cfg, pos_explicit, cw, ch, &tr);
    tr.mark("jitter");
    {
        std::unique_ptr<Engine> old(s->eng);
        s->eng = nullptr;
        if (old) E->recycle(*old);
    }
    tr.mark("old engine recycled");
    ensure_grid(s, cfg->grid_nx, cfg->grid_ny, cfg->target_density);
    set_density_model(s, cfg->density_model);

    // fresh PinPairWeights: the engine keeps it dense (weight per sink pin, fused into WA)
    s->Q = 0;
    s->pp_dirty = true;
    s->dl_w.zero(s->st), s->ppw_e.zero(s->st), s->pp_mask.zero(s->st);
    s->q_count.reserve(2);
    s->q_count.zero(s->st);
    s->net_w.reserve(std::max(s->N, 1));
    if (cfg->net_weighting) {
        k_fill_f64<<<blocks_for(std::max(s->N, 1), kBlock), kBlock, 0, s->st>>>(s->N, s->net_w, 1.0);
        CK_LAUNCH();
    }

    tr.mark("upload + grid + ledger");
    const int T = std::max(cfg->max_iters, 1);
    E->sched.reserve(T); // (filled after lambda_auto, below)
    Ctrl c0{};
    c0.nonfinite_at = INT_MAX;
    E->ctrl.reserve(1);
    CK(cudaMemcpyAsync(E->ctrl.p, &c0, sizeof c0, cudaMemcpyHostToDevice, s->st));
    E->trace.reserve(T);
    E->timing_row.reserve(3);
    E->timing_row.zero(s->st);
    E->cur.reserve(1);
    E->terms.reserve(1);
    E->obs_count.reserve(1);
    E->m.reserve(s->C), E->v.reserve(s->C);
    E->m.zero(s->st), E->v.zero(s->st);
    E->nb_wa = wa_blocks(s), E->nb_pp = wa_blocks(s), E->nb_d = bins_blocks(s); // PP partials per WA block
    E->part.reserve(2 * E->nb_wa + E->nb_pp + 2 * E->nb_d + 8);
    E->part.zero(s->st);
    E->kernels_per_iter = 8 + (s->grid.n_wide > 0 ? 2 : 0); // (+ wide-cell scatter and density gradient)
    E->partitioned = s->part_world > 1 || s->part_comm1;
    if (fin_split()) E->kernels_per_iter += 1; // (finalize in two halves)
    if (E->partitioned) { // this rank's slice of the spatial order (the density scatter / gradient share)
        const long long nm = s->grid.n_movable;
        E->mov_lo = static_cast<int>(nm * s->part_rank / s->part_world);
        E->mov_hi = static_cast<int>(nm * (s->part_rank + 1) / s->part_world);
        E->kernels_per_iter += 1; // (the lambda * density gradient fold)
    }
    if (E->partitioned) { // entries of other ranks' nets must read as 0 in this rank's fold
        E->red.reserve(2 * static_cast<size_t>(s->C) + 3 * static_cast<size_t>(E->nb_wa) + 8);
        E->red.zero(s->st);
        s->grad_e.zero(s->st);
    }
    // the order goes stale as the cells spread; the re-sort's fixed cost weighs more on small designs
    E->sort_every = s->grid.n_movable >= 500000 ? 2 : 4;
    if (const char* se = std::getenv("TDPG_SORT_EVERY")) E->sort_every = std::max(1, std::atoi(se));
    // every buffer the graphs touch is sized before capture, so their pointers never move
    tr.mark("schedule + buffers");
    refresh_reserve(s);
    if (E->cfg.extraction == 0 && E->cfg.k > 1) kbest_refresh_reserve(s, E->cfg.k); // (the k-best refresh graph)
    s->ex_counts.zero(s->st); // (the refresh graph accumulates the run's path totals in [3], [4])
    place_tail_reserve(s); // (so a later run of the session finds every buffer where its graphs point)
    if (cfg->lambda0 <= 0.0) { // lambda_auto's scratch (an allocation after the capture would re-capture)
        const int nb_d = bins_blocks(s), nb = 148 * 2;
        s->lam_scratch.reserve(2 * static_cast<size_t>(s->C) + 2 * nb_d + 64 + 2 * nb);
        s->part.reserve(2 * wa_blocks(s) + pp_blocks(s) + 2 * nb_d + 64);
    }
    s->pin_xy_external = false;
    sort_cells_spatial(s);
    tr.mark("reserve + sort");
    s->eng = E.release();
    Engine& G = *s->eng;
    if (!G.adopt_graphs(s)) {
        Engine::session_consts(s, G.consts);
        capture_iteration(s, G);
        tr.mark("iteration graph");
        G.refresh_gexec = capture(s, [&] { record_refresh(s, G); });
        G.refresh_lonly = s->pins_stale, s->pins_stale = false; // (recorded, not run)
        tr.mark("refresh graph");
        G.sort_gexec = capture(s, [&] { sort_cells_spatial(s); });
        G.epoch = dbuf_epoch();
        tr.mark("sort graph");
    } else {
        tr.mark("graphs adopted");
    }

    G.lambda = cfg->lambda0 > 0.0 ? cfg->lambda0 : lambda_auto(s, G.gamma, cfg->pp_loss);
    tr.mark("lambda auto");
    G.lambda_cap = G.lambda * cfg->lambda_max;
    // per-iteration schedule (placer.cpp:470-471, :349-350, :477)
    std::vector<Sched> sch(T);
    double lam = G.lambda;
    for (int it = 0; it < T; ++it) {
        sch[it].lr = cfg->step0_frac * G.span * std::pow(cfg->step_decay, it);
        sch[it].c1 = 1.0 - std::pow(cfg->adam_beta1, it + 1);
        sch[it].c2 = 1.0 - std::pow(cfg->adam_beta2, it + 1);
        sch[it].lambda = lam;
        lam = std::min(lam * cfg->mu, G.lambda_cap);
    }
    G.sched.upload(sch, s->st);
    CK(cudaStreamSynchronize(s->st));
}

Ctrl read_ctrl(tdpg_session* s)
{
    Ctrl c;
    CK(cudaMemcpyAsync(&c, s->eng->ctrl.p, sizeof c, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    return c;
}

__global__ void k_count_heads32(long long cap, const long long* __restrict__ n_hits, const unsigned* __restrict__ k,
                                unsigned long long* __restrict__ out)
{
    const long long n = min(cap, *n_hits); // (the refresh sorts only the first size class >= the hit count)
    int c = 0;
    for (long long i = blockIdx.x * static_cast<long long>(kBlock) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * kBlock)
        c += (k[i] != 0xFFFFFFFFu) && (i == 0 || k[i - 1] != k[i]);
    c = warp_sum(c);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, static_cast<unsigned long long>(c));
}

__global__ void k_refresh_begin_gen(const double* sta_out, Ctrl* ctrl, double* timing_row)
{
    if (ctrl->stopped) return;
    timing_row[0] = 1.0, timing_row[1] = sta_out[0], timing_row[2] = sta_out[1];
    ctrl->engaged = 1;
}

void net_weights_engine(tdpg_session* s, const Ctrl* ctrl);

// The engine's timing refresh as recorded into its graph: k = 1 (one backtrace per violated endpoint,
// timing.cu refresh_record) or k > 1 (the k-best lists, kpaths.cu refresh_record_kbest).  The topn policy
// grows its list length until the report is complete, a host-driven loop: timing_refresh_general.
void record_refresh(tdpg_session* s, Engine& E)
{
    if (E.cfg.extraction == 0 && E.cfg.k > 1)
        refresh_record_kbest(s, E.ctrl, E.timing_row, E.cfg.w0, E.cfg.w1, E.cfg.net_weighting != 0, E.cfg.k);
    else
        refresh_record(s, E.ctrl, E.timing_row, E.cfg.w0, E.cfg.w1, E.cfg.net_weighting != 0);
}

// Timing round with k > 1 or the topn policy (placer.cpp:415-435): STA graph, then the k-best
// extraction (host-sized: the path count is data dependent), then the dense-ledger update and net
// weights, all on the session stream.
void timing_refresh_general(tdpg_session* s)
{
    Engine& E = *s->eng;
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    CK(cudaEventCreate(&ev.first));
    CK(cudaEventCreate(&ev.second));
    CK(cudaEventRecord(ev.first, s->st));
    run_sta_async(s, s->sta_out);
    k_refresh_begin_gen<<<1, 1, 0, s->st>>>(s->sta_out, E.ctrl, E.timing_row);
    CK_LAUNCH();
    double h[3];
    Ctrl c;
    CK(cudaMemcpyAsync(h, s->sta_out.p, sizeof h, cudaMemcpyDeviceToHost, s->st));
    CK(cudaMemcpyAsync(&c, E.ctrl.p, sizeof c, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    s->tns = h[0], s->wns = h[1];
    s->sta_valid = true, s->ties_resolved = false;
    s->n_paths = 0, s->n_path_pins = 0, s->n_hits = 0, s->uniq_pairs = 0, s->uniq_endpoints = 0, s->candidates = 0;
    E.kernel_launches += 2LL * s->L + 4;
    if (!c.stopped && h[1] < 0.0) {
        extract_policy_dev(s, E.cfg.extraction, static_cast<int>(h[2]), E.cfg.k, true);
        E.kernel_launches += s->L + 16;
        E.paths_host += s->n_paths, E.path_pins_host += s->n_path_pins;
        const long long H = s->n_hits;
        if (H > 0) {
            LedgerArgs la{};
            la.n_hits = nullptr, la.H = H, la.sta_out = s->sta_out, la.ctrl = E.ctrl, la.gen = true;
            la.hk = s->kh_key_s, la.hidx = s->kh_idx_s, la.hslack = s->hit_slack, la.w0 = E.cfg.w0;
            la.w1 = E.cfg.w1, la.dl_w = s->dl_w, la.ppw_e = s->ppw_e, la.pin_entry = s->pin_entry;
            la.pin_loc = s->pin_loc, la.pp_mask = s->pp_mask, la.q_count = s->q_count;
            launch_ledger_update(s, H, la);
            E.kernel_launches += 2;
        }
    }
    if (E.cfg.net_weighting) {
        net_weights_engine(s, E.ctrl);
        ++E.kernel_launches;
    }
    CK(cudaEventRecord(ev.second, s->st));
    E.refresh_ev.push_back(ev);
    ++E.refreshes;
    if (s->round_cb) {
        CK(cudaStreamSynchronize(s->st));
        s->round_cb(s->round_user, E.launched);
    }
}

// Timing round (placer.cpp:415-435) as one graph launch: STA, extraction of every violated endpoint,
// ledger update, net weights; nothing comes back to the host unless an observer is registered.
void timing_refresh(tdpg_session* s)
{
    Engine& E = *s->eng;
    if (E.cfg.extraction != 0) {
        timing_refresh_general(s);
        return;
    }
    const bool kbest = E.cfg.k > 1;
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    CK(cudaEventCreate(&ev.first));
    CK(cudaEventCreate(&ev.second));
    CK(cudaEventRecord(ev.first, s->st));
    CK(cudaGraphLaunch(E.refresh_gexec, s->st));
    s->pins_stale = E.refresh_lonly; // the sweep's per-pin arrays are left in L-space
    CK(cudaEventRecord(ev.second, s->st));
    E.refresh_ev.push_back(ev);
    // our kernels: pin_xy, 2 per level, slack keys, sta final, begin, ties, bt count, fill, bt write,
    // counts, violated count + two size-class picks, ledger short + long runs (+ net weights); k > 1:
    // the STA, begin, violated count + pick, one k-best merge per level, count, write, totals, hops, hit
    // total, hits, key pad, pick, ledger short + long runs (+ net weights)
    E.kernel_launches += (kbest ? 3LL * s->L + 17 : 2LL * s->L + 14) + (E.cfg.net_weighting ? 1 : 0);
    ++E.refreshes;
    if (s->round_cb) { // TimingRoundObserver (placer.cpp:434): this round's annotation and report
        sta_materialize_pins(s); // the observer may read per-pin timing
        double h[3];
        long long c[3];
        CK(cudaMemcpyAsync(h, s->sta_out.p, sizeof h, cudaMemcpyDeviceToHost, s->st));
        CK(cudaMemcpyAsync(c, s->ex_counts.p, sizeof c, cudaMemcpyDeviceToHost, s->st));
        unsigned long long* u = E.obs_count;
        CK(cudaMemsetAsync(u, 0, sizeof *u, s->st));
        if (kbest) kbest_refresh_publish(s);
        k_count_heads32<<<148 * 4, kBlock, 0, s->st>>>(kbest ? s->kb_hcap : s->hcap, s->ex_counts.p + 2,
                                                        kbest ? s->kh_key_s.p : s->eh_key_s.p, u);
        CK_LAUNCH();
        unsigned long long uq = 0;
        CK(cudaMemcpyAsync(&uq, u, sizeof uq, cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
        s->tns = h[0], s->wns = h[1];
        s->sta_valid = true, s->ties_resolved = true;
        s->n_paths = static_cast<int>(c[0]), s->n_path_pins = c[1], s->n_hits = 0;
        if (kbest) s->ties_resolved = false, s->candidates = c[0]; // (k-best paths need no tie resolution)
        s->uniq_pairs = s->n_paths ? static_cast<long long>(uq) : 0;
        s->round_cb(s->round_user, E.launched);
    }
}

// Run up to n iterations of the loop (refreshes per schedule), all enqueued without host syncs;
// after a stop (stop_overflow) the kernels see the device flag and do nothing.
void engine_release(tdpg_session* s)
{
    delete s->eng;
    s->eng = nullptr;
}

// Re-capture the engine's graphs when a device buffer they point into was (re)allocated since, or when
// the clock / RC units baked into their kernel arguments changed (tdpg_set_constraints).
void ensure_graphs(tdpg_session* s, Engine& E)
{
    if (E.epoch == dbuf_epoch() && E.consts_match(s)) return; // (tdpg_set_constraints may have moved them)
    Engine::session_consts(s, E.consts);
    if (E.gexec_a) cudaGraphExecDestroy(E.gexec_a), E.gexec_a = nullptr;
    if (E.gexec_b) cudaGraphExecDestroy(E.gexec_b), E.gexec_b = nullptr;
    capture_iteration(s, E);
    if (E.refresh_gexec) cudaGraphExecDestroy(E.refresh_gexec);
    E.refresh_gexec = capture(s, [&] { record_refresh(s, E); });
    E.refresh_lonly = s->pins_stale, s->pins_stale = false;
    if (E.sort_gexec) cudaGraphExecDestroy(E.sort_gexec);
    E.sort_gexec = capture(s, [&] { sort_cells_spatial(s); });
    E.epoch = dbuf_epoch();
    ++E.recaptures;
}

int engine_run(tdpg_session* s, int n)
{
    Engine& E = *s->eng;
    int done = 0;
    for (; done < n && E.launched < E.cfg.max_iters; ++done) {
        ensure_graphs(s, E);
        const int it = E.launched;
        if (it >= E.cfg.timing_start_iter && (it - E.cfg.timing_start_iter) % E.cfg.m == 0) timing_refresh(s);
        if (!E.gexec) throw Error(TDPG_ERR_INTERNAL, "partitioned engine without a communicator: use "
                                                      "tdpg_comm_init or the split-phase API");
        if (it % E.sort_every == 0) { // refresh the scatter's spatial cell order first
            if (E.gexec_sorted) {
                CK(cudaGraphLaunch(E.gexec_sorted, s->st));
            } else {
                CK(cudaGraphLaunch(E.sort_gexec, s->st));
                CK(cudaGraphLaunch(E.gexec, s->st));
            }
            E.kernel_launches += 1;
        } else {
            CK(cudaGraphLaunch(E.gexec, s->st));
        }
        E.kernel_launches += E.kernels_per_iter + (E.partitioned ? 1 : 0);
        ++E.launched;
    }
    return done;
}

// Split-phase iteration for a partitioned engine without a communicator (the caller reduces twice):
// phase 0 runs the scheduled refresh / re-sort and this rank's density scatter and returns its int64 grid;
// phase A takes the summed grid, runs the rest of the pre-reduction graph and returns this rank's
// all-reduce buffer; phase B takes the reduced buffer and finishes the iteration.
size_t part_phase_density(tdpg_session* s, long long* acc_host)
{
    Engine& E = *s->eng;
    if (!E.partitioned || !E.gexec_a0) throw Error(TDPG_ERR_INTERNAL, "engine is not in split-phase partitioned mode");
    ensure_graphs(s, E);
    const int it = E.launched;
    if (it >= E.cfg.timing_start_iter && (it - E.cfg.timing_start_iter) % E.cfg.m == 0) timing_refresh(s);
    if (it % E.sort_every == 0) CK(cudaGraphLaunch(E.sort_gexec, s->st));
    CK(cudaGraphLaunch(E.gexec_a0, s->st));
    const size_t B = static_cast<size_t>(s->grid.bins());
    if (acc_host) s->grid.acc.download(acc_host, B, s->st);
    CK(cudaStreamSynchronize(s->st));
    return B;
}

size_t part_phase_a(tdpg_session* s, const long long* acc_host, double* red_host)
{
    Engine& E = *s->eng;
    if (!E.partitioned || !E.gexec_a) throw Error(TDPG_ERR_INTERNAL, "engine is not in split-phase partitioned mode");
    const size_t B = static_cast<size_t>(s->grid.bins());
    CK(cudaMemcpyAsync(s->grid.acc.p, acc_host, B * sizeof(long long), cudaMemcpyHostToDevice, s->st));
    CK(cudaGraphLaunch(E.gexec_a, s->st));
    const size_t n = 2 * static_cast<size_t>(s->C) + 3 * static_cast<size_t>(E.nb_wa);
    if (red_host) E.red.download(red_host, n, s->st);
    CK(cudaStreamSynchronize(s->st));
    return n;
}

void part_phase_b(tdpg_session* s, const double* red_host)
{
    Engine& E = *s->eng;
    if (!E.partitioned || !E.gexec_b) throw Error(TDPG_ERR_INTERNAL, "engine is not in split-phase partitioned mode");
    const size_t n = 2 * static_cast<size_t>(s->C) + 3 * static_cast<size_t>(E.nb_wa);
    CK(cudaMemcpyAsync(E.red.p, red_host, n * sizeof(double), cudaMemcpyHostToDevice, s->st));
    CK(cudaGraphLaunch(E.gexec_b, s->st));
    ++E.launched;
    CK(cudaStreamSynchronize(s->st));
}

} // namespace tdpg

tdpg_session::~tdpg_session()
{
    delete eng; // Engine is complete here
    tdpg::comm_destroy(this);
    if (sta_gexec) cudaGraphExecDestroy(sta_gexec);
    if (sta_gexec_L) cudaGraphExecDestroy(sta_gexec_L);
    if (ex_gexec) cudaGraphExecDestroy(ex_gexec);
    if (st_req) cudaStreamSynchronize(st_req), cudaStreamDestroy(st_req);
    if (st_cond) cudaStreamDestroy(st_cond);
    if (ev_sta_fork) cudaEventDestroy(ev_sta_fork);
    if (ev_sta_join) cudaEventDestroy(ev_sta_join);
    if (st) {
        cudaStreamSynchronize(st);
        cudaCtxResetPersistingL2Cache(); // release the L2 lines this session pinned
        cudaStreamDestroy(st);
    }
}

using namespace tdpg;

#define API_BEGIN try {
#define API_END                                                                   \
    return TDPG_OK;                                                               \
    }                                                                             \
    catch (const ::tdpg::Error& e) { return ::tdpg::api_fail(e.kind, e.what()); } \
    catch (const std::exception& e) { return ::tdpg::api_fail(TDPG_ERR_INTERNAL, e.what()); }

extern "C" {

int tdpg_set_round_callback(tdpg_session* s, tdpg_round_cb cb, void* user)
{
    API_BEGIN
    s->round_cb = cb;
    s->round_user = user;
    API_END
}

int tdpg_engine_init(tdpg_session* s, const tdpg_config* cfg, const uint8_t* pos_explicit)
{
    API_BEGIN
    engine_init(s, cfg, pos_explicit);
    API_END
}

int tdpg_iterate_dev(tdpg_session* s, int32_t n, double* device_ms)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised (tdpg_engine_init)");
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, s->st));
    engine_run(s, n);
    CK(cudaEventRecord(e1, s->st));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (device_ms) *device_ms = ms;
    cudaEventDestroy(e0), cudaEventDestroy(e1);
    const Ctrl c = read_ctrl(s);
    if (c.nonfinite_at != INT_MAX)
        throw Error(TDPG_ERR_NONFINITE, "non-finite value: non-finite objective or gradient at iteration " +
                                            std::to_string(c.nonfinite_at));
    API_END
}

// Per-kernel device time of `reps` loop iterations (no refresh), CUDA events between launches.
int tdpg_profile_iteration(tdpg_session* s, int32_t reps, double* out_ms, int32_t n_out, char* names, int32_t name_len)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised (tdpg_engine_init)");
    Engine& E = *s->eng;
    static const char* kNames[7] = {"wirelength_pp", "spatial_sort", "density_scatter", "density_bins", "finalize",
                                    "dens_grad", "cells"};
    double* part_wl = E.part.p;
    double* part_hp = part_wl + E.nb_wa;
    double* part_pp = part_hp + E.nb_wa;
    double* part_d = part_pp + E.nb_pp;
    FinArgs fa{};
    fa.part_wl = part_wl, fa.part_hp = part_hp, fa.part_pp = part_pp, fa.part_d = part_d;
    fa.nb_wa = E.nb_wa, fa.nb_pp = E.nb_pp, fa.nb_d = E.nb_d;
    fa.total_movable = s->grid.total_movable, fa.beta = E.cfg.beta;
    fa.sched = E.sched, fa.stop_overflow = E.cfg.stop_overflow, fa.terms = E.terms, fa.trace = E.trace;
    fa.timing_row = E.timing_row, fa.timing_row_clear = E.timing_row;
    cudaEvent_t ev[8];
    for (auto& e : ev) CK(cudaEventCreate(&e));
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int r = 0; r < reps && E.launched < E.cfg.max_iters; ++r) {
        CK(cudaEventRecord(ev[0], s->st));
        launch_wirelength_pp(s, E.gamma, E.cfg.net_weighting != 0, part_wl, part_hp, true, E.cfg.pp_loss,
                             E.cfg.beta, part_pp, E.ctrl, nullptr, 0);
        CK(cudaEventRecord(ev[1], s->st));
        if (r % E.sort_every == 0) CK(cudaGraphLaunch(E.sort_gexec, s->st));
        CK(cudaEventRecord(ev[2], s->st));
        launch_density_scatter_ctrl(s, E.ctrl);
        CK(cudaEventRecord(ev[3], s->st));
        launch_density_bins_ctrl(s, part_d, E.nb_d, E.ctrl);
        CK(cudaEventRecord(ev[4], s->st));
        launch_finalize(s, fa, E.ctrl, E.cur);
        CK(cudaEventRecord(ev[5], s->st));
        launch_dens_grad(s, E.ctrl, s->st);
        CK(cudaEventRecord(ev[6], s->st));
        launch_cells(s, nullptr, E.m, E.v, E.cfg.adam_beta1, E.cfg.adam_beta2, E.cfg.adam_eps, E.cur, E.ctrl,
                     false);
        CK(cudaEventRecord(ev[7], s->st));
        CK(cudaEventSynchronize(ev[7]));
        for (int k = 0; k < 7; ++k) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ev[k], ev[k + 1]);
            acc[k] += ms;
        }
        ++E.launched;
        E.kernel_launches += E.kernels_per_iter;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    for (int k = 0; k < 7 && k < n_out; ++k) {
        out_ms[k] = acc[k] / std::max(reps, 1);
        if (names && name_len > 0) {
            std::strncpy(names + static_cast<size_t>(k) * name_len, kNames[k], name_len - 1);
            names[static_cast<size_t>(k) * name_len + name_len - 1] = 0;
        }
    }
    API_END
}

// One loop iteration through host buffers: positions in (pinned host -> device), the
// iteration (with its scheduled timing refresh), positions + trace row out.  This is the
// reference-shaped objective_and_gradient + AdamState::step call with host vectors.
int tdpg_step_host(tdpg_session* s, const double* xy_in, double* xy_out, tdpg_trace_row* row)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised (tdpg_engine_init)");
    Engine& E = *s->eng;
    if (xy_in) {
        CK(cudaMemcpyAsync(s->cell_xy.p, xy_in, sizeof(double2) * s->C, cudaMemcpyHostToDevice, s->st));
        s->sta_valid = false;
    }
    const int it = E.launched;
    engine_run(s, 1);
    if (xy_out) CK(cudaMemcpyAsync(xy_out, s->cell_xy.p, sizeof(double2) * s->C, cudaMemcpyDeviceToHost, s->st));
    TraceRowDev r{};
    if (row && it < E.cfg.max_iters)
        CK(cudaMemcpyAsync(&r, E.trace.p + it, sizeof r, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    if (row) {
        row->iter = r.iter, row->has_timing = r.has_timing, row->hpwl = r.hpwl, row->overflow = r.overflow;
        row->tns = r.tns, row->wns = r.wns, row->wl_term = r.wl_term, row->density_term = r.density_term;
        row->pp_term = r.pp_term, row->lambda = r.lambda, row->beta_pp = r.beta_pp;
    }
    API_END
}

int tdpg_part_density(tdpg_session* s, int64_t* acc, int64_t* n_bins)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised (tdpg_engine_init)");
    const size_t n = part_phase_density(s, reinterpret_cast<long long*>(acc));
    if (n_bins) *n_bins = static_cast<int64_t>(n);
    API_END
}

int tdpg_part_step_a(tdpg_session* s, const int64_t* acc, double* red, int64_t* n_red)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised (tdpg_engine_init)");
    if (!acc) throw Error(TDPG_ERR_VALIDATION, "validation error: tdpg_part_step_a needs the summed density grid");
    const size_t n = part_phase_a(s, reinterpret_cast<const long long*>(acc), red);
    if (n_red) *n_red = static_cast<int64_t>(n);
    API_END
}

int tdpg_part_step_b(tdpg_session* s, const double* red)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised (tdpg_engine_init)");
    part_phase_b(s, red);
    API_END
}

int tdpg_engine_stats(tdpg_session* s, int32_t* iter, int32_t* refreshes, int64_t* launches)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised");
    if (iter) *iter = s->eng->launched;
    if (refreshes) *refreshes = s->eng->refreshes;
    if (launches) *launches = s->eng->kernel_launches;
    API_END
}

int tdpg_engine_paths(tdpg_session* s, int64_t* paths, int64_t* path_pins)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised");
    long long c[5] = {0, 0, 0, 0, 0};
    CK(cudaMemcpyAsync(c, s->ex_counts.p, sizeof c, cudaMemcpyDeviceToHost, s->st));
    CK(cudaStreamSynchronize(s->st));
    if (paths) *paths = c[3] + s->eng->paths_host;
    if (path_pins) *path_pins = c[4] + s->eng->path_pins_host;
    API_END
}

int tdpg_engine_times(tdpg_session* s, double* refresh_ms_total, double* last_refresh_ms, int64_t* ledger_pairs)
{
    API_BEGIN
    if (!s->eng) throw Error(TDPG_ERR_INTERNAL, "engine not initialised");
    const double tot = s->eng->refresh_ms();
    if (refresh_ms_total) *refresh_ms_total = tot;
    if (last_refresh_ms) {
        *last_refresh_ms = 0.0;
        if (!s->eng->refresh_ev.empty()) {
            float ms = 0.f;
            const auto& e = s->eng->refresh_ev.back();
            if (cudaEventElapsedTime(&ms, e.first, e.second) == cudaSuccess) *last_refresh_ms = ms;
        }
    }
    if (ledger_pairs) {
        unsigned long long q = 0;
        CK(cudaMemcpyAsync(&q, s->q_count.p, sizeof q, cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
        *ledger_pairs = static_cast<int64_t>(q);
    }
    API_END
}

int tdpg_place(tdpg_session* s, const tdpg_config* cfg, const uint8_t* pos_explicit, tdpg_trace_row* trace,
               int32_t* n_rows, int32_t* stop_overflow, double final_[3])
{
    API_BEGIN
    engine_init(s, cfg, pos_explicit);
    InitTrace tr(s);
    engine_run(s, cfg->max_iters);
    if (cfg->extraction == 0 && cfg->k > 1) kbest_check(s); // (the captured k-best merge's in-arc flag)
    tr.mark("place: device loop");
    const Ctrl c = read_ctrl(s);
    if (c.nonfinite_at != INT_MAX)
        throw Error(TDPG_ERR_NONFINITE, "non-finite value: non-finite objective or gradient at iteration " +
                                            std::to_string(c.nonfinite_at));
    const int rows = c.rows;
    if (trace && rows > 0) {
        std::vector<TraceRowDev> tr(rows);
        s->eng->trace.download(tr.data(), rows, s->st);
        CK(cudaStreamSynchronize(s->st));
        for (int i = 0; i < rows; ++i) {
            tdpg_trace_row& r = trace[i];
            r.iter = tr[i].iter, r.has_timing = tr[i].has_timing, r.hpwl = tr[i].hpwl, r.overflow = tr[i].overflow;
            r.tns = tr[i].tns, r.wns = tr[i].wns, r.wl_term = tr[i].wl_term, r.density_term = tr[i].density_term;
            r.pp_term = tr[i].pp_term, r.lambda = tr[i].lambda, r.beta_pp = tr[i].beta_pp;
        }
    }
    if (n_rows) *n_rows = rows;
    if (stop_overflow) *stop_overflow = c.stopped;
    tr.mark("place: trace rows");
    dense_ledger_to_sorted(s); // PlacementOutcome::pair_weights as the sorted ledger (tdpg_pp_get)
    tr.mark("place: sorted ledger");
    // final STA + exact HPWL at the returned positions (placer.cpp:482, bindings.cpp:381-382); TNS / WNS
    // only, the per-pin arrays stay in L-space until a caller reads them
    run_sta_dev(s, false);
    tr.mark("place: final STA");
    double hp = 0.0;
    {
        const int nb = wa_blocks(s);
        s->part.reserve(2 * nb + 8);
        launch_wirelength(s, s->eng->gamma, false, s->part.p, s->part.p + nb, nb);
        std::vector<double> hh(nb);
        CK(cudaMemcpyAsync(hh.data(), s->part.p + nb, nb * sizeof(double), cudaMemcpyDeviceToHost, s->st));
        CK(cudaStreamSynchronize(s->st));
        for (double x : hh) hp += x;
    }
    if (final_) final_[0] = s->tns, final_[1] = s->wns, final_[2] = hp;
    API_END
}

} // extern "C"
