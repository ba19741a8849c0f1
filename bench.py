"""bench.py — timing-driven GP on a 1M-cell synthetic netlist (BASELINE.json configs[2]).

One step = one GP iteration of run_placement (placer.cpp:412-478): WA wirelength +
pin-pair attraction + bin density, value and gradient, Adam step, clamp; a timing
refresh (STA + endpoint-policy extraction of every violated endpoint + ledger
update, placer.cpp:415-435) runs every m=15 steps and is included in the timed
region.  fp64 throughout, like the reference.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`value` = GP iterations/s over the whole job (N independent replicas when N > 1,
"replicas only").  `e2e` = run_placement through the C-ABI (tdpg_place) with pinned
host buffers (positions in, positions + trace rows out).  Extra keys
report the STA + top-k extraction sweep on the same 1M timing graph, the dominant
kernel's roofline and the reference CPU baseline.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
METRIC = "GP iters/s & top-k path-extraction ms at 1M cells; TNS/WNS/HPWL parity"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cells", type=int, default=1_000_000, help="generator spec n_cells (1.1x cells)")
    ap.add_argument("--grid", type=int, default=1024)
    ap.add_argument("--m", type=int, default=15)
    ap.add_argument("--fail-frac", type=float, default=0.8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-evals", type=int, default=2)
    ap.add_argument("--mode", default=None, choices=["replicas", "partition"],
                    help="N > 1: independent designs per GPU (weak scaling) or one design with nets partitioned "
                         "across GPUs and the cell gradient all-reduced by NCCL inside the iteration graph "
                         "(strong scaling, SURVEY §8e); default: partition when N > 1")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index, period_ms=None):
        self.index, self.rows, self.proc = index, [], None
        self.period_ms = period_ms or int(os.environ.get("TDPG_CLOCK_MS", "100"))

    def __enter__(self):
        if self.period_ms <= 0:
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, stdin=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 2 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 2 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def bench_config(args, iters):
    """The run_placement config of the timed workload (both arms).  Timing engages at the first timed
    iteration (timing_start_iter = W), so whatever --steps / --warmup are, the timed window opens with a
    timing refresh and holds one every m iterations."""
    return {"grid_nx": args.grid, "grid_ny": args.grid, "m": args.m, "timing_start_iter": args.warmup,
            "max_iters": iters, "seed": 1}


def lround(x):
    return int(np.floor(x + 0.5)) if x >= 0 else -int(np.floor(-x + 0.5))


def calibrate_clock(arr_ep, fail_frac):
    """generate_synthetic's clock rule (generator.cpp:249-260) applied at the run's start snapshot:
    the period at the (1 - fail_frac) quantile of the sorted endpoint arrivals."""
    a = np.sort(np.asarray(arr_ep, np.float64))
    n = a.size
    n_pass = min(max(lround((1.0 - fail_frac) * n), 0), n)
    if n_pass == 0:
        return max(a[0] * 0.95, 1e-9)
    if n_pass == n:
        return a[-1] * 1.05
    return 0.5 * (a[n_pass - 1] + a[n_pass])


def workload_config(args, d, world):
    """The `config` object both arms print (identical by construction)."""
    return {"workload": f"configs[2]: synthetic {d.n_cells}-cell / {d.n_nets}-net netlist (generator spec "
                        f"{args.cells}, seed 1), run_placement from its seeded jittered start (placer.cpp:375-382), "
                        f"clock calibrated there so {args.fail_frac:g} of the endpoints fail (generator.cpp:249-260); "
                        f"full timing-driven GP iteration (WA + pin-pair attraction + bin density + Adam), grid "
                        f"{args.grid}^2; timing engages at the first timed iteration and refreshes every {args.m} "
                        f"(STA + endpoint extraction of every violated endpoint + ledger update) inside the timed region",
            "cells": d.n_cells, "pins": d.n_pins, "nets": d.n_nets, "net_pins": d.n_net_pins,
            "endpoints": int(d.endpoints.size), "grid": args.grid, "m": args.m, "timing_start_iter": args.warmup,
            "fail_frac": args.fail_frac, "clock_period": float(d.clock_period),
            "l2": "working set per iteration > L2 (positions+netlist+gradients+grid ~ 2x 126 MB)",
            "parallelism": "single GPU" if world == 1 else f"{world} GPUs"}


def peaks():
    try:
        return json.load(open(PEAKS))
    except Exception:
        return {"hbm_gbs": 6650.0, "fallback": True}


def kernel_bytes(d, grid, E_tot):
    """Algorithmic (compulsory) bytes per launch of each GP kernel, fp64.  DESIGN.md §4."""
    C, P, N, E = d.n_cells, d.n_pins, d.n_nets, d.n_net_pins
    B = grid * grid
    return {
        # WA + the fused pin pairs (3 size-class kernels): net CSR + entry record (cell id, offset) + cell
        # positions once + per-entry gradient write
        "wirelength_pp": 4 * (N + 1) + E * (4 + 16) + 16 * C + 16 * E,
        # positions + sizes + fixed flags once, grid accumulators written once
        "density_scatter": C * (16 + 16 + 1) + 8 * B,
        # accumulators read + reset, excess written
        "density_bins": 3 * 8 * B,
        # perm + positions + sizes once, excess grid once, density gradient written
        "dens_grad": C * (4 + 16 + 16 + 16) + 8 * B,
        # fold CSR + entry gradients + fixed/positions/sizes/density gradient + Adam m,v r/w + positions written
        "cells": 4 * (C + 1) + 4 * E_tot + 16 * E_tot + C * (1 + 16 + 16 + 16) + C * (32 + 32) + 16 * C,
    }


def footprint_entries(d, xy, grid):
    """Non-zero density footprint entries (bins a cell's B-spline weights touch, five-bin form) at the
    given positions: (a_hi - a_lo + 3) bins per axis, clipped to the grid (gp_kernels.cuh axis5)."""
    x0, y0, x1, y1 = d.core
    tot = 0
    for lo, w, o, span in ((xy[:, 0], d.cell_w, x0, x1 - x0), (xy[:, 1], d.cell_h, y0, y1 - y0)):
        pitch = span / grid
        al = np.floor((lo - o) / pitch - 1.0)
        ah = np.floor((lo + w - o) / pitch - 1.0)
        b0, b1 = np.maximum(al, 0), np.minimum(ah + 2, grid - 1)
        n = np.maximum(b1 - b0 + 1, 0)
        tot = n if isinstance(tot, int) else tot * n
    return int(np.sum(tot[d.cell_fixed == 0]))


def iteration_bytes(d, grid, Q=0):
    """SURVEY.md §8(d) bytes_iter with p = 8 (fp64), plus the Adam step 2C*p*7."""
    C, N, E = d.n_cells, d.n_nets, d.n_net_pins
    p = 8
    B = grid * grid
    return 2 * C * p + 2 * C * p + E * (4 + 2 * p) + 4 * (N + 1) + 4 * E + Q * (8 + p) + 2 * C * p + 2 * B * p + 2 * C * p * 7


def design_file(args, seed=1):
    """The timed workload's design as a binary design file (design.py save_bin / load_bin; C-ABI
    tdpg_design_bin_*), shared by both arms: whichever arm runs first builds it (the product generator
    or the oracle's restatement — netlist-identical, tests/test_bench_workload.py) and the other reads it."""
    d = os.path.join(ROOT, "build", "designs")
    os.makedirs(d, exist_ok=True)
    return os.path.join(d, f"bench_c{args.cells}_s{seed}_f{args.fail_frac:g}.tdpb")


def load_or_make(args, maker, seed=1):
    from paper_2503_11674_b200.design import load_bin, save_bin
    path = design_file(args, seed)
    t0 = time.time()
    if os.path.exists(path):
        return load_bin(path), time.time() - t0, "file"
    d = maker(args, seed)
    if isinstance(d, tuple):
        d = d[0]
    tmp = f"{path}.{os.getpid()}"
    save_bin(d, tmp)
    os.replace(tmp, path)
    return d, time.time() - t0, "generated"


def make_design(args, seed=1):
    """The timed workload's design, built by the product: the generator's netlist, the run's jittered start
    (on the device, bitwise the reference's mt19937_64 draws) made explicit, the clock calibrated at that
    start with a device STA (bit-exact).  Returns (design, seconds)."""
    from paper_2503_11674_b200.engine import Session, generate
    t0 = time.time()
    d = generate(seed=seed, cells=args.cells, fail_frac=args.fail_frac, calibrate=False)
    s = Session(d)
    s.engine_init(bench_config(args, 1))
    xy0 = s.positions()
    arr = s.sta(xy0)["arr"]
    s.close()
    d.positions = xy0
    d.pos_explicit = np.ones(d.n_cells, np.uint8)
    d.clock_period = calibrate_clock(arr[d.endpoints], args.fail_frac)
    return d, time.time() - t0


def make_design_reference(args, seed=1):
    """The same design built without the product library: the oracle's generator restatement
    (tdp_oracle_gen.c, netlist-identical to the reference's and to the product's), its jitter
    restatement (placer.cpp:375-382) and the reference's own run_sta for the clock."""
    from oracle.oracle import Oracle, RefOracle
    d = Oracle.generate(seed=seed, cells=args.cells, fail_frac=args.fail_frac)
    xy0 = Oracle(d).jitter(bench_config(args, 1))
    arr = RefOracle(d).sta(xy0, threads=os.cpu_count() or 1)["arr"]
    d.positions = xy0
    d.pos_explicit = np.ones(d.n_cells, np.uint8)
    d.clock_period = calibrate_clock(arr[d.endpoints], args.fail_frac)
    return d


def extraction_sweep(d, ns=(1000, 3000, 10000, 30000, 100000)):
    """STA + report_timing_endpoint(n, 1) on a spread snapshot of the 1M graph, clock set so
    80% of endpoints fail (configs[3]); device time per n (CUDA events)."""
    from paper_2503_11674_b200.engine import Session
    rng = np.random.default_rng(1)
    xy = d.positions.copy()
    x0, y0, x1, y1 = d.core
    xy[:, 0] = x0 + rng.random(d.n_cells) * (x1 - x0 - d.cell_w)
    xy[:, 1] = y0 + rng.random(d.n_cells) * (y1 - y0 - d.cell_h)
    s = Session(d)
    t = s.sta(xy)
    clock0 = d.clock_period
    arr = t["arr"][d.endpoints]
    d.clock_period = float(np.quantile(arr, 0.2))
    s2 = Session(d)
    out = {}
    s2.set_positions(xy)
    for n in ns:
        best = None
        for _ in range(3):
            r = s2.extract(None, n=n, run_sta=True)
            tot = r["sta_ms"] + r["extract_ms"]
            if best is None or tot < best[0]:
                best = (tot, r["sta_ms"], r["extract_ms"], r["n_paths"])
        out[str(n)] = {"total_ms": round(best[0], 3), "sta_ms": round(best[1], 3), "extract_ms": round(best[2], 3),
                       "paths": best[3]}
    d.clock_period = clock0
    return out, xy


def cpu_baseline(d, args, xy_snapshot):
    """Reference CPU implementation (oracle/_ref: the reference's own sources) on a bounded
    sample of the same workload: objective_and_gradient on the 1M design (1 and nproc threads,
    the better quoted) + one STA / top-10K extraction."""
    from oracle.oracle import Oracle, RefOracle
    kind = "reference" if RefOracle.available() else "port"
    B = RefOracle if kind == "reference" else Oracle
    t0 = time.time()
    o = B(d)
    setup_s = time.time() - t0
    nproc = os.cpu_count() or 1
    gamma = 0.01 * d.span
    res = {}
    for th in sorted({1, nproc}):
        ts = []
        for _ in range(max(1, args.cpu_sample_evals)):
            t1 = time.perf_counter()
            if kind == "reference":
                o.objective(d.positions, args.grid, args.grid, 0.6, gamma, 1e-4, 2.5e-5, threads=th)
            else:
                o.objective(d.positions, args.grid, args.grid, 0.6, gamma, 1e-4, 2.5e-5)
            ts.append(time.perf_counter() - t1)
        res[th] = min(ts)
        if kind != "reference":
            break
    best_th = min(res, key=res.get)
    ex = {}
    if kind == "reference":
        r = o.extract(xy_snapshot, n=10000, threads=1)
        ex = {"sta_ms": round(r["sta_ms"], 1), "extract_top10k_ms": round(r["extract_ms"], 1)}
    return {"value": round(1.0 / res[best_th], 4), "unit": "iters/s", "cores": best_th, "kind": kind,
            "cpu_model": lscpu_model(), "nproc": nproc,
            "sample": f"objective_and_gradient on the {d.n_cells}-cell design, grid {args.grid}^2, "
                      f"{args.cpu_sample_evals} evals per thread count, best of threads {sorted(res)} "
                      f"(s/eval: {', '.join(f'{k}T {v:.2f}' for k, v in res.items())}); Adam + refresh excluded",
            "threads_tried": {str(k): round(v, 3) for k, v in res.items()}, "setup_s": round(setup_s, 1), **ex}


def lscpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    """--impl reference: the reference's own CPU implementation (its sources compiled by oracle/Makefile
    into oracle/_ref/libtdpref.so) on the same workload and schedule.  The design comes from the oracle's
    restatements, so this process never maps a product library.  Objective and STA use every host
    thread, extraction one (the enumerator memoises prefixes only single-threaded)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import RefOracle
    if not RefOracle.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libtdpref.so was not built"}), flush=True)
        return
    nproc = os.cpu_count() or 1
    t0 = time.time()
    d, _, source = load_or_make(args, make_design_reference)
    setup_s = time.time() - t0
    r = RefOracle(d)
    W, K = args.warmup, args.steps
    res = r.place_bench(bench_config(args, W + K), threads_obj=nproc, threads_sta=nproc, threads_ex=1)
    it_ms = res["iter_ms"][W:W + K]
    if it_ms.size < K:
        raise SystemExit(f"reference run stopped after {res['rows']} rows (stop_overflow)")
    tot_s = float(np.sum(it_ms)) / 1000.0
    val = K / tot_s
    paths_timed = int(np.sum(res["paths"][W:W + K]))
    rf = res["refresh_ms"][W:W + K]
    print(json.dumps({"impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": "iters/s",
                      "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": round(1000 * tot_s / K, 2),
                      "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                      "data": "synthetic", "config": workload_config(args, d, world),
                      "timed_window": {"refreshes": int(np.count_nonzero(rf)), "refresh_ms_each": round(
                          float(np.sum(rf)) / max(1, np.count_nonzero(rf)), 1), "paths_extracted": paths_timed,
                          "ledger_pairs_end": res["ledger_pairs"], "gp_iteration_ms": round(
                              float(np.sum(it_ms) - np.sum(rf)) / K, 2)},
                      "cpu_baseline": {"value": round(val, 4), "unit": "iters/s", "cores": nproc, "kind": "reference",
                                       "cpu_model": lscpu_model(),
                                       "sample": f"the whole workload: {W} warm-up + {K} timed iterations of the "
                                                 f"reference's run_placement loop (ref_harness.cpp ref_place_bench: "
                                                 f"objective_and_gradient + Adam every step, run_sta + "
                                                 f"report_timing_endpoint + collect_pin_pairs + update_pair_weights "
                                                 f"every {args.m}); objective/STA at {nproc} threads, extraction at 1"},
                      "e2e": {"value": round(val, 4), "unit": "iters/s", "h2d_bytes_per_step": 0,
                              "d2h_bytes_per_step": 0},
                      "setup_s": round(setup_s, 1), "design_source": source, "final": {"tns": res["tns"], "wns": res["wns"], "hpwl": res["hpwl"]}}),
          flush=True)


def traffic_for(d, grid, kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture of THIS configuration (cells and
    grid), or None when no capture of it exists."""
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tfile):
        return None
    return json.load(open(tfile)).get(f"{d.n_cells}x{grid}", {}).get(kernel)


def maxr_dev(x, torch):
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def red_len(s):
    from paper_2503_11674_b200.engine import red_size
    return red_size(s)


def run_ours(args):
    rank, world, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # (NCCL's init lines name the ranks and the transport)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2503_11674_b200.engine import Session

    mode = args.mode or ("partition" if world > 1 else "replicas")
    # (--mode partition at one GPU: the partitioned engine over a one-rank NCCL communicator, its all-reduces
    # captured in the iteration graph as at N > 1 — the N = 1 point of the partitioned scaling curve)
    partition = mode == "partition" and (world > 1 or args.mode == "partition")
    if partition and world == 1:
        os.environ["TDPG_COMM_WORLD1"] = "1"
    d, gen_s, source = load_or_make(args, make_design, 1 if partition else 1 + rank)  # partition: one design
    W, K = args.warmup, args.steps
    total_iters = W + K + 64
    cfg = bench_config(args, total_iters)
    t0 = time.time()
    s = Session(d)
    create_s = time.time() - t0
    if partition:
        from paper_2503_11674_b200 import distributed as D
        D.init_partitioned(s, rank, world)
    t0 = time.time()
    s.engine_init(cfg)
    init_s = time.time() - t0

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # the sampler runs from before the warm-up until after the timed region
    with Clocks(local) as clk:
        time.sleep(0.5)
        s.iterate(W)
        barrier()
        st0 = s.engine_stats()
        torch.cuda.profiler.start()  # (ncu --profile-from-start off captures exactly the timed region)
        dev_ms = s.iterate(K)
        torch.cuda.profiler.stop()
        st1 = s.engine_stats()
        barrier()
        time.sleep(0.3)
    ms = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    dev_ms_max = float(ms.item())
    value = (1 if partition else world) * K / (dev_ms_max / 1000.0)
    launches = st1["kernel_launches"] - st0["kernel_launches"]
    refreshes = st1["refreshes"] - st0["refreshes"]
    refresh_ms = st1["refresh_ms"] - st0["refresh_ms"]
    paths_timed = st1["paths"] - st0["paths"]
    if paths_timed <= 0:
        raise SystemExit(f"bench: the timed window extracted no path ({refreshes} refreshes): the workload "
                         "would not exercise the timing-driven path")

    # partitioned: the two collectives of an iteration timed alone (device, max over ranks), beside the
    # iteration they sit in
    comm = None
    if partition:
        ms_grid, ms_red = s.comm_bench(20)
        comm = {"allreduce_grid_ms": round(maxr_dev(ms_grid, torch), 4), "allreduce_grad_ms": round(maxr_dev(ms_red, torch), 4),
                "grid_bytes": 8 * args.grid * args.grid, "grad_bytes": 8 * red_len(s),
                "iteration_ms": round(dev_ms_max / K, 4),
                "what": "NCCL sum all-reduces of the int64 density grid and of [partial cell gradient | WA/HPWL/PP "
                        "partials], each timed alone (CUDA events, 20 reps); the iteration overlaps the second "
                        "with nothing (it ends the pre-reduction phase) and the first with the WA branch"}
    # per-kernel profile of loop iterations (roofline of the dominant kernel); a partitioned engine
    # is profiled through its replica twin on rank 0 below
    if partition and rank != 0:
        prof = {}
    elif partition:
        s_prof = Session(d)
        s_prof.engine_init(cfg)
        s_prof.iterate(W + K)
        prof = s_prof.profile_iteration(5)
    else:
        prof = s.profile_iteration(5)

    # e2e: the call a user makes — run_placement through the C-ABI (tdpg_place) on the same design and
    # schedule (timing from the first iteration, a refresh every m), K iterations from pinned host
    # positions to pinned host positions + the per-iteration trace rows; wall clock over the whole call
    # (its engine set-up, device loop, final STA), max over ranks.  Warm: on the session above after one
    # untimed call; cold: a fresh session (netlist upload + timing-graph levelization) + the call.
    C = d.n_cells
    hin = torch.empty(2 * C, dtype=torch.float64, pin_memory=True)
    hout = torch.empty(2 * C, dtype=torch.float64, pin_memory=True)
    hin.numpy()[:] = d.positions.reshape(-1)
    e2e_cfg = dict(bench_config(args, K), timing_start_iter=0)

    def maxr(x):
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([x], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    cold_s, cold_rows = None, 0
    if not partition:
        barrier()
        t0 = time.perf_counter()
        s_cold = Session(d)
        cold_rows, _ = s_cold.place_host(e2e_cfg, hin.data_ptr(), hout.data_ptr())
        cold_s = time.perf_counter() - t0
        s_cold.close()
        cold_s = maxr(cold_s)
    s.place_host(e2e_cfg, hin.data_ptr(), hout.data_ptr())  # warm-up call (lazy module loads, first captures)
    barrier()
    t0 = time.perf_counter()
    e2e_rows, _ = s.place_host(e2e_cfg, hin.data_ptr(), hout.data_ptr())
    e2e_s = maxr(time.perf_counter() - t0)
    e2e_val = (1 if partition else world) * e2e_rows / e2e_s
    sweep, xy_snap = (extraction_sweep(d) if rank == 0 else ({}, None))

    if rank != 0:
        return
    pk = peaks()
    E_tot = d.n_net_pins + int(np.sum(np.isin(np.arange(d.n_pins), d.net_pins, invert=True) & (d.pin_cell >= 0)))
    kb = kernel_bytes(d, args.grid, E_tot)
    dom = max((k for k in prof if k in kb), key=lambda k: prof[k])
    dom_ms = prof[dom]
    achieved = kb[dom] / (dom_ms / 1000.0) / 1e9
    iter_ms = sum(prof.values())
    # the scatter's other candidate bound: shared-memory atomics (two or three 32-bit limb adds per non-zero
    # footprint entry, counted on the device at the profiled positions) against the B200 rate measured by
    # tools/atom_peak.cu (random addresses in a 32 KB window; profiles/atom_peak_r02.json).  The B300 guide's
    # "2 cyc/lane" model (582 G/s) understated it 4.5x: the scatter is latency-bound, not atomics-bound.
    n_ent = footprint_entries(d, s.positions(), args.grid)
    from paper_2503_11674_b200.design import CONFIG_DEFAULTS
    at_lo, at_hi = s.density_atomics(args.grid, args.grid, CONFIG_DEFAULTS["target_density"], xy=s.positions())
    clk_summary = clk.summary()
    sm_ghz = (clk_summary.get("sm_mhz") or 1965.0) / 1000.0
    atom_peak, atom_src = 148 * 4 * sm_ghz * 1e9 / 2 / 1e9, "modelled: 2 cyc/lane x 4 SMSP x 148 SM"
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "atom_peak_r02.json")) as f:
            atom_peak = json.load(f)["random_g_lane_atomics_s"]
        atom_src = "measured on B200: tools/atom_peak.cu, random addresses in a 32 KB window (profiles/atom_peak_r02.json)"
    except (OSError, KeyError, ValueError):
        pass
    atom_ach = (at_lo + at_hi) / (prof.get("density_scatter", 1e9) / 1000.0) / 1e9 if "density_scatter" in prof else None
    ib = iteration_bytes(d, args.grid)
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(d, args, xy_snap)
        except Exception as e:  # reported, never fatal
            cpu = {"error": str(e)[:200]}
    gp_ms = (dev_ms_max - refresh_ms) / K
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "iters/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(dev_ms_max / K, 4), "higher_is_better": True,
        "scaling": "strong" if partition else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, d, world),
        "mode": ("nets and cells partitioned: NCCL all-reduces of the density grid and of the cell gradient inside "
                 "the iteration graph" if partition else "replicas") if world > 1 or partition else "single GPU",
        "partition": comm,
        "timed_window": {"refreshes": refreshes, "refresh_ms_each": round(refresh_ms / max(refreshes, 1), 3),
                         "paths_extracted": paths_timed, "path_pins_extracted": st1["path_pins"] - st0["path_pins"],
                         "ledger_pairs_end": st1["ledger_pairs"], "gp_iteration_ms": round(gp_ms, 4)},
        "e2e": {"value": round(e2e_val, 3), "unit": "iters/s",
                "h2d_bytes_per_step": round(16 * C / max(e2e_rows, 1), 1),
                "d2h_bytes_per_step": round((16 * C + 88 * e2e_rows) / max(e2e_rows, 1), 1),
                "steps": e2e_rows, "wall_s": round(e2e_s, 4),
                "cold": None if cold_s is None else {
                    "value": round(cold_rows / cold_s, 3), "wall_s": round(cold_s, 4),
                    "what": "fresh session (netlist upload + timing-graph levelization) + the same tdpg_place call"},
                "path": "tdpg_place (run_placement through the C-ABI): pinned positions in, device loop with "
                        "timing refresh every m from the first iteration, positions + trace rows out"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": pk.get("hbm_gbs"),
                     "unit": "GB/s", "frac": round(achieved / pk.get("hbm_gbs", 6650.0), 4),
                     "traffic": traffic_for(d, args.grid, dom), "algorithmic_bytes": kb[dom],
                     "kernel_ms": round(dom_ms, 4),
                     "peak_source": "measured" if "fallback" not in pk else "fallback",
                     "limiter": None if atom_ach is None else {
                         "kernel": "density_scatter", "bound": "smem_atomics", "unit": "G lane-atomics/s",
                         "achieved": round(atom_ach, 1), "peak": round(atom_peak, 1),
                         "frac": round(atom_ach / atom_peak, 3), "footprint_entries": n_ent,
                         "lane_atomics": at_lo + at_hi,
                         "peak_source": atom_src}},
        "iteration": {"gp_iteration_ms": round(gp_ms, 4),
                      "kernels_ms_serialised": {k: round(v, 4) for k, v in prof.items()}, "sum_ms": round(iter_ms, 4),
                      "bytes_iter_survey": ib,
                      "frac_of_hbm_serialised": round(ib / (iter_ms / 1000.0) / 1e9 / pk.get("hbm_gbs", 6650.0), 4),
                      "frac_of_hbm_graph": round(ib / (gp_ms / 1000.0) / 1e9 / pk.get("hbm_gbs", 6650.0), 4)},
        "extraction_sweep_ms": sweep,
        "clocks": clk_summary,
        "cpu_baseline": cpu,
        "setup_s": {"design": round(gen_s, 2), "design_source": source, "session_create": round(create_s, 3),
                    "engine_init": round(init_s, 3)},
    }
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
