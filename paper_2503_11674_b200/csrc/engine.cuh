// engine.cuh — the device-resident session behind the tdpg C-ABI.
//
// HBM layout (all structure-of-arrays, fp64 like the reference):
//   cells     : xy double2[C] (lower-left origin), wh double2[C], delay[C], fixed u8[C]
//   pins      : cell int[P] (-1 terminal), off double2[P], anchor double2[P]
//               (terminal_pos), dir u8[P], cap[P]
//   net CSR   : net_start[N+1]; per net-pin entry e (driver first, then sinks):
//               e_cell int[E] (owner cell, or -1-pin for terminals), e_off double2[E]
//   fold CSR  : per cell, the entry ids of its pins in ascending pin id
//               (reference fold order, placer.cpp:318-325)
//   timing    : pins grouped by level (ascending id inside a level), per-pin in-arc
//               CSR (from-pin, ascending arc id) and out-arc CSR (to-pin)
//   grid      : int64 fixed-point occupancy accumulators (deterministic scatter),
//               excess double[B]
//   ledger    : sorted 64-bit pair keys (a<<32|b) + weights; per-pin incidence CSR
#pragma once

#include <functional>

#include <array>
#include <memory>
#include <string>
#include <vector>


#include "common.cuh"

struct tdpg_session;

namespace tdpg {

// Electrostatic density (electro.cu): twiddle / cosine tables and work rows of the grid's Poisson solve
// (hand-written shared-memory DCTs, no FFT library).
struct ElectroPlan {
    int nx = 0, ny = 0;
    struct Axis {
        int L = 0;
        DBuf<double2> tw, qt; // FFT twiddles (power-of-two lengths), quarter-wave twiddles
        DBuf<double> c4;      // cos(pi j / 2L), j < 4L (direct path for other lengths)
        DBuf<double> lam;     // 2 - 2 cos(pi u / L): the axis' Laplacian eigenvalues (times pitch^2)
        void make(int len, cudaStream_t st);
    } ax, ay;
    DBuf<double> rho, psi, r1, r2;
    void ensure(int gx, int gy);
    void release();
    ~ElectroPlan();
};

struct Grid {
    int model = 0; // 0: bin overflow penalty (density.cpp, the reference); 1: electrostatic (electro.cu)
    ElectroPlan electro;
    int nx = 0, ny = 0;
    double td = 0.0;
    double x0 = 0, y0 = 0, bw = 0, bh = 0, cap = 0, total_movable = 0;
    double scale = 1.0, inv_scale = 1.0; // fixed-point occupancy: q = rint(w * scale)
    // limbs of the windowed scatter's shared accumulators, so that 256 footprint entries per block fit each
    // 32-bit limb: 2 when every entry is below 2^45 (designs from ~30K cells up), 3 otherwise (session.cu)
    int limbs = 3;
    bool has_fixed = false;
    DBuf<long long> acc;
    DBuf<double> excess;
    DBuf<double> base; // fixed-cell exact overlap (density.cpp:75-93), when any fixed cell
    DBuf<int> perm, perm_tmp;  // movable cells in spatial (tile) order, for the windowed scatter
    // positions and sizes of the cells in that order, written by the scatter (coalesced) so the density
    // gradient streams them instead of repeating the perm -> cell gather chain
    DBuf<double2> xy_sp, wh_sp;
    DBuf<unsigned> perm_keys;
    int n_movable = 0;
    // movable cells that may span more than five bins on an axis (width > 1.99 pitch): their density
    // gradient runs in a separate pass, so the five-bin kernel carries no general-footprint code
    DBuf<int> wide;
    int n_wide = 0;
    double wide_w = 0, wide_h = 0;
    bool valid() const { return nx > 0; }
    long long bins() const { return static_cast<long long>(nx) * ny; }
};

// Per-iteration schedule entry (host-computed with the reference's std::pow).
struct Sched {
    double lr, c1, c2, lambda;
};

// Device scalars of one objective evaluation.
struct Terms {
    double value, wl, density, pp, hpwl, overflow;
};

// Device-side control block for the iteration loop.
struct Ctrl {
    int iter;          // next iteration index
    int stopped;       // stop_overflow reached (placer.cpp:459-462)
    int nonfinite_at;  // first iteration with a non-finite term/gradient, INT_MAX if none
    int engaged;       // timing rounds have started
    int rows;          // trace rows written
    int pad[3];
};

struct TraceRowDev {
    int iter, has_timing;
    double hpwl, overflow, tns, wns, wl_term, density_term, pp_term, lambda, beta_pp;
};

struct Engine; // placement loop state (place.cu)
void engine_release(tdpg_session* s); // deletes s->eng (place.cu, where Engine is complete)

// k-best extraction scratch (kpaths.cu), grow-only
struct KbScratch {
    DBuf<int> npath, npins, poff, pinoff, cstart, clen, cpins, order, idx0, flag;
    DBuf<double> cslack;
    DBuf<unsigned long long> key0, key1;
};

} // namespace tdpg

struct tdpg_session {
    // sizes
    // E: net-pin entries; E_tot: WA-layout slots (E_lay >= E) + off-net pins
    int C = 0, P = 0, N = 0, E = 0, E_tot = 0, S = 0, EP = 0, A = 0, A_net = 0, A_cell = 0, L = 0;
    double clock = 0, r_unit = 0, c_unit = 0, core[4] = {0, 0, 0, 0};
    cudaStream_t st = nullptr;
    cudaStream_t st_req = nullptr;                    // the STA's required-time sweep (beside arrival)
    cudaStream_t st_cond = nullptr;                   // captures conditional-node bodies (size-class sorts)
    cudaEvent_t ev_sta_fork = nullptr, ev_sta_join = nullptr;
    int device = 0;

    // host copies
    // (only what host-side work needs after creation: pin offsets, terminals, caps, directions, delays and
    // the net pin lists live on the device alone)
    std::vector<double> h_cell_w, h_cell_h;
    std::vector<uint8_t> h_cell_fixed, h_is_source, h_is_endpoint;
    std::vector<int> h_pin_cell, h_net_start, h_sources, h_endpoints, h_pin_net, h_pin_entry;
    std::vector<std::string> pin_names;
    bool pin_names_blank = false; // names were given and all empty (error text prints them empty)
    std::vector<int> h_level, h_lvl_start, h_arc_from, h_arc_to, h_arc_kind, h_arc_owner; // (level / arcs: lazy)
    bool h_level_valid = false, h_arcs_valid = false;
    tdpg::DBuf<int> arc_from, arc_to, arc_kind, arc_owner; // arcs by id (timing_graph.cpp:60-77)
    tdpg::HBuf<int> h_graph_small;

    // device netlist
    tdpg::DBuf<double2> cell_xy, cell_wh, anchor, pin_off, e_off;
    tdpg::DBuf<double> cell_delay, pin_cap;
    tdpg::DBuf<uint8_t> cell_fixed, pin_dir, is_source, is_endpoint;
    tdpg::DBuf<int> pin_cell, net_start, net_pins, e_cell, pin_entry, cell_ent_start, cell_ent;
    tdpg::DBuf<int> pin_net;        // pin -> net (-1: on no net)
    bool h_pin_maps_valid = false;  // h_pin_entry / h_pin_net downloaded (host_pin_maps)
    // WA layout: nets sorted by pin count; per block (pin count N or 0, first, count, entry base);
    // entries of N-pin nets slot-major per block, class-0 nets contiguous (wa_gen_start)
    tdpg::DBuf<int> net_by_size, wa_gen_start;
    tdpg::DBuf<int4> wa_blk;
    int n_wa_blocks = 0, E_lay = 0;
    int wa_cls_blk0[9] = {0}, wa_cls_nblk[9] = {0};
    int wa_cls_net0[9] = {0}, wa_cls_net1[9] = {0}, wa_cls_pos0[9] = {0}; // (WaAxisArgs)
    int wa_gen_nets = 0; // generic (class 0) nets: order positions [0, wa_gen_nets)
    // engine-mode pin pairs (dense ledger indexed by sink pin; fused into WA)
    tdpg::DBuf<uint32_t> pp_mask, pp_ord;   // per class-ordered net
    tdpg::DBuf<int> wa_gen_ord, pin_loc, pin_driver;
    tdpg::DBuf<double> ppw_e, dl_w;        // pair weight per WA slot / per sink pin (0 = none)

    // device timing graph
    tdpg::DBuf<int> lvl_pins, lvl_start, in_start, in_from, out_start, out_to, ep_sorted;
    // STA sweep over driver levels only: Output pins grouped by level, all Input pins (timing.cu)
    tdpg::DBuf<int> sta_out_pins, sta_in_pins;           // Output pins / Input pins, each grouped by level
    std::vector<int> h_sta_out_start, h_sta_in_start;    // [L + 1]
    tdpg::DBuf<unsigned long long> sta_akey, sta_rkey;   // push sweep: Output pins' arrival / required keys
    // Level-major copy of the timing graph for the push sweep (L-space index i <-> pin L_pin[i]; per
    // level its Input pins then its Output pins): every per-pin access of a level is coalesced.
    tdpg::DBuf<int> L_pin, L_in_start, L_in_from, L_out_start, L_out_to, L_cell, L_pred;
    tdpg::DBuf<int> L_of; // pin -> L-space index
    bool pins_stale = false; // the last STA left its results in L-space only (sta_materialize_pins)
    tdpg::DBuf<uint8_t> L_flags, L_ak, L_rk, L_tie; // flags: 1 source, 2 endpoint, 4 output
    tdpg::DBuf<double> L_cap, L_arr, L_req;
    tdpg::DBuf<double2> L_off, L_anchor, L_xy;
    std::vector<int> h_L_in_lo, h_L_in_hi; // per level: its Input pins' L range
    tdpg::DBuf<unsigned> grid_bar;   // persistent STA: grid barrier (arrival count, generation)
    int sta_grid = 0;                // co-resident blocks of the persistent STA kernel (0: per-level launches)

    // STA state
    tdpg::DBuf<double2> pin_xy;
    tdpg::DBuf<double> arr, req, slack;
    tdpg::DBuf<uint8_t> ak, rk, tie;
    tdpg::DBuf<int> pred, tie_list, counters; // counters: [0] tie count
    tdpg::DBuf<int> d_level, tie_scratch;
    tdpg::DBuf<double> sta_out;  // tns, wns, n_violated
    tdpg::DBuf<double> sta_part; // STA reduction partials
    cudaGraphExec_t sta_gexec = nullptr; // the per-level STA sweep, captured once
    std::array<uint64_t, 9> sta_graph_key{};
    cudaGraphExec_t ex_gexec = nullptr;    // endpoint extraction up to the host count read (timing.cu)
    std::array<long long, 4> ex_key{};
    cudaGraphExec_t sta_gexec_L = nullptr; // the same sweep leaving its results in L-space
    std::array<uint64_t, 9> sta_graph_key_L{};
    // ledger-update scratch
    tdpg::DBuf<uint8_t> lg_flag;
    tdpg::DBuf<double> lg_w, lg_new_w;
    tdpg::DBuf<unsigned long long> lg_new_k;
    tdpg::DBuf<int> lg_nsel;
    double tns = 0, wns = 0;
    bool sta_valid = false, ties_resolved = false;
    bool pin_xy_external = false; // STA uses caller-provided pin positions (tdpg_set_pin_positions)

    // GP scratch
    tdpg::DBuf<double2> grad_e, d_cell, dgrad; // per-entry WA(+PP) gradient, cell gradient, density gradient
    tdpg::DBuf<double> part; // per-block partial sums
    tdpg::Grid grid;
    tdpg::DBuf<double> net_w;
    bool has_net_w = false;

    // ledger + PP incidence
    tdpg::DBuf<unsigned long long> led_key, led_key2;
    tdpg::DBuf<double> led_w, led_w2;
    long long Q = 0;
    tdpg::DBuf<int> pp_pins, pp_start, pp_entry, pp_inc;
    int n_pp_pins = 0;
    bool pp_dirty = true;

    // extraction results
    tdpg::DBuf<int> ex_ep, ex_len, ex_hops, ex_off, ex_hoff, ex_pins;
    tdpg::DBuf<double> ex_slack;
    tdpg::DBuf<unsigned long long> hit_key, hit_key_s;
    tdpg::DBuf<unsigned> pair_bits; // unique-pair bits over sink pins (endpoint extraction)
    tdpg::DBuf<int> ex_tmp_pins;                // fixed-stride path slots (endpoint extraction)
    tdpg::DBuf<unsigned long long> ex_tmp_keys;
    tdpg::DBuf<int> hit_idx, hit_idx_s;
    tdpg::DBuf<double> hit_slack;
    int n_paths = 0;
    long long n_path_pins = 0, n_hits = 0, uniq_pairs = 0, uniq_endpoints = 0, candidates = 0;
    // k-best path lists (kpaths.cu): per pin K records (delay, pred pin / pred rank), record counts
    tdpg::DBuf<double> kb_delay;
    tdpg::DBuf<int2> kb_pred;
    tdpg::DBuf<int> kb_cnt;
    int kb_K = 0;
    tdpg::DBuf<int> kb_dn;        // k-best engine refresh: device path / path-pin counts
    tdpg::DBuf<long long> kb_H;   // ... and hit count
    long long kb_hcap = 0;
    tdpg::KbScratch kbx;
    tdpg::DBuf<unsigned> kh_key, kh_key_s; // engine refresh with k > 1 / topn: hits keyed by sink pin
    tdpg::DBuf<int> kh_idx_s;
    bool hits_sorted = false;
    double last_sta_ms = 0, last_extract_ms = 0;

    // engine-mode refresh buffers (capacity-sized; hits keyed by sink pin)
    tdpg::DBuf<unsigned> eh_key, eh_key_s;
    tdpg::DBuf<int> eh_idx, eh_idx_s;
    tdpg::DBuf<double> eh_slack;
    tdpg::DBuf<long long> ex_counts;                 // n_paths, path pins, hits of the last refresh
    tdpg::DBuf<unsigned long long> q_count;          // pairs in the dense ledger
    long long hcap = 0;

    // sort / scan scratch
    tdpg::DBuf<unsigned char> cub_tmp;
    tdpg::DBuf<unsigned long long> sort_k0, sort_k1;
    tdpg::DBuf<unsigned long long> ep_kc;             // the refresh's violated endpoints, compacted
    tdpg::DBuf<int> ep_vc;
    tdpg::DBuf<uint8_t> ep_flag;
    tdpg::DBuf<long long> ep_nv;                     // [0] violated count, [1..2] compaction counts
    tdpg::DBuf<int> sort_v0, sort_v1;
    tdpg::HBuf<long long> h_small;
    // initial jitter (place.cu): per-cell jitter flag / rank, the raw mt19937_64 stream, explicit flags
    tdpg::DBuf<int> jit_flag, jit_rank;
    // dense ledger -> sorted ledger (timing.cu dense_ledger_to_sorted): keys and weights, grow-only
    tdpg::DBuf<unsigned long long> dl_k0, dl_k1;
    tdpg::DBuf<double> dl_w0, dl_w1;
    tdpg::DBuf<unsigned long long> jit_raw;
    unsigned long long jit_seed = 0;   // jit_raw holds the first jit_count draws of mt19937_64(jit_seed)
    long long jit_count = -1;
    const unsigned long long* jit_ptr = nullptr;
    int n_free = -1;                   // cells that are not fixed (host count, lazily)
    tdpg::DBuf<double> lam_scratch;    // lambda_auto scratch
    tdpg::DBuf<uint8_t> jit_expl;
    // jit_flag / jit_rank are a function of pos_explicit (cell_fixed is fixed per session): the host copy
    // of the last pos_explicit (empty = none given) and the buffers it was computed into
    std::vector<uint8_t> h_jit_expl;
    bool jit_flags_ok = false, jit_expl_null = false;
    const void* jit_flags_at[2] = {nullptr, nullptr};

    // partitioned multi-GPU mode (partition.cu): this rank's WA block range, NCCL communicator
    int part_rank = 0, part_world = 1, part_b0 = 0, part_b1 = 0;
    bool part_comm1 = false; // a one-rank NCCL communicator drives the partitioned engine (TDPG_COMM_WORLD1 test)
    bool part_active = false; // WA launches honour the range only while the partitioned graph is recorded
    void* comm = nullptr; // ncclComm_t

    // placement engine
    tdpg::Engine* eng = nullptr;
    bool pdl_graph = false; // recording the iteration graph: GP kernels chained by programmatic dependent launch
    tdpg_round_cb round_cb = nullptr; // called after every timing round of tdpg_place
    void* round_user = nullptr; // owned; deleted in ~tdpg_session (place.cu)

    ~tdpg_session();
};

namespace tdpg {

// session.cu
void upload_positions(tdpg_session* s, const double* xy);
// host <-> device copies of netlist-sized arrays through the process-wide pinned staging buffers (session.cu)
void upload_bytes_staged(void* dst, const void* src, size_t bytes, cudaStream_t st);
void download_bytes(void* dst, const void* src, size_t bytes, cudaStream_t st);
void host_pin_maps(tdpg_session* s);
void refresh_fixed_baseline(tdpg_session* s);
void build_graph_device(tdpg_session* s); // graph.cu
void graph_host_level(tdpg_session* s);
void graph_host_arcs(tdpg_session* s);
void sta_setup(tdpg_session* s);
bool capturing(tdpg_session* s);
void pad_hit_keys(tdpg_session* s, long long cap, const long long* n_dev, unsigned* keys);
int bits_for_pins(int P);
void switch_hits_by_count(tdpg_session* s, const long long* d_n, long long cap,
                          const std::function<void(cudaStream_t, long long)>& body);
void refresh_begin(tdpg_session* s, Ctrl* ctrl, double* timing_row);
void net_weights_record(tdpg_session* s, const Ctrl* ctrl);
void sort_violated_endpoints(tdpg_session* s, const Ctrl* ctrl);
void sta_record(tdpg_session* s, double* out3, bool pin_space);
void kbest_refresh_reserve(tdpg_session* s, int K);
void refresh_record_kbest(tdpg_session* s, Ctrl* ctrl, double* timing_row, double w0, double w1, bool net_weighting,
                          int K);
void kbest_refresh_publish(tdpg_session* s);
void kbest_check(tdpg_session* s);
void sta_materialize_pins(tdpg_session* s); // per-pin STA arrays of an L-space-only sweep (timing.cu)
void place_tail_reserve(tdpg_session* s); // (timing.cu)
void ensure_grid(tdpg_session* s, int nx, int ny, double td);
void set_density_model(tdpg_session* s, int model);
void* cub_scratch(tdpg_session* s, size_t bytes);
void sort_cells_spatial(tdpg_session* s);

// gp.cu
void launch_wirelength(tdpg_session* s, double gamma, bool use_net_w, double* part_wl, double* part_hp, int nblk);
int wa_blocks(const tdpg_session* s);
void rebuild_pp_incidence(tdpg_session* s);
void launch_pp(tdpg_session* s, int kind, double beta, double* part_pp, int nblk);
int pp_blocks(const tdpg_session* s);
void launch_density(tdpg_session* s, double* part_d, int nblk);
int bins_blocks(const tdpg_session* s);
Terms evaluate_objective(tdpg_session* s, double gamma, double lambda, double beta, int kind, bool use_net_w,
                         double* d_cell_host);

// timing.cu
void run_sta_dev(tdpg_session* s, bool pin_space = true); // pin_space = false: results left in L-space
void sta_setup(tdpg_session* s);
bool capturing(tdpg_session* s);
void pad_hit_keys(tdpg_session* s, long long cap, const long long* n_dev, unsigned* keys);
int bits_for_pins(int P);
void switch_hits_by_count(tdpg_session* s, const long long* d_n, long long cap,
                          const std::function<void(cudaStream_t, long long)>& body);
void refresh_begin(tdpg_session* s, Ctrl* ctrl, double* timing_row);
void net_weights_record(tdpg_session* s, const Ctrl* ctrl);
void sort_violated_endpoints(tdpg_session* s, const Ctrl* ctrl);
void sta_record(tdpg_session* s, double* out3, bool pin_space);
void kbest_refresh_reserve(tdpg_session* s, int K);
void refresh_record_kbest(tdpg_session* s, Ctrl* ctrl, double* timing_row, double w0, double w1, bool net_weighting,
                          int K);
void kbest_refresh_publish(tdpg_session* s);
void kbest_check(tdpg_session* s);
void refresh_reserve(tdpg_session* s);
void refresh_record(tdpg_session* s, Ctrl* ctrl, double* timing_row, double w0, double w1, bool net_weighting);
void dense_ledger_to_sorted(tdpg_session* s);
void extract_endpoint_dev(tdpg_session* s, int n);
void resolve_ties_dev(tdpg_session* s);
void ledger_update_dev(tdpg_session* s, double wns, double w0, double w1, bool hits_all_violated);
// dense-ledger update (update_pair_weights) over hits sorted stably by sink pin (timing.cu)
struct LedgerArgs {
    const long long* n_hits; // device hit count (engine refresh) or nullptr: H
    long long H;
    const double* sta_out;
    const Ctrl* ctrl;
    bool gen;                // k > 1 / topn refresh (active while not stopped and wns < 0)
    const unsigned* hk;
    const int* hidx;
    const double* hslack;
    double w0, w1;
    double* dl_w;
    double* ppw_e;
    const int* pin_entry;
    const int* pin_loc;
    uint32_t* pp_mask;
    unsigned long long* q_count;
};
void launch_ledger_update(tdpg_session* s, long long cap, const LedgerArgs& a);
void net_weights_dev(tdpg_session* s);
int sorted_violated(tdpg_session* s);

// partition.cu
void comm_allreduce(tdpg_session* s, double* buf, size_t n);
void comm_allreduce_i64(tdpg_session* s, long long* buf, size_t n, cudaStream_t st);
void launch_density_scatter_part(tdpg_session* s, const Ctrl* ctrl, int lo, int hi, bool wide);
void launch_dens_grad_part(tdpg_session* s, const Ctrl* ctrl, cudaStream_t st, int lo, int hi);
void launch_add_dgrad(tdpg_session* s, const Sched* sched, const Ctrl* ctrl, double2* fold, int lo, int hi);
void comm_destroy(tdpg_session* s);

// electro.cu
void electro_solve(tdpg_session* s, cudaStream_t st);
void electro_energy(tdpg_session* s, double* part_d, int nblk, const Ctrl* ctrl, cudaStream_t st);

// kpaths.cu
void kbest_build(tdpg_session* s, int K);
void extract_policy_dev(tdpg_session* s, int policy, int n, int k, bool sink_keys);
void kbest_paths_of(tdpg_session* s, int pin, int K, std::vector<std::vector<int>>& paths, std::vector<double>& delay);

} // namespace tdpg
