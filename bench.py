"""Benchmark: one step = the whole hot path of the method on config c4 (BASELINE
configs[3]: blobby surface, N = 1M surface points -> 3M centres, sigma 0.01,
cutoff 6 sigma, GMRES(50) + shifted block-Jacobi local solves (F4,
reading R17), 256^3 grid).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

Step (all on the GPU, inputs resident in HBM when the timed region starts):
  a0 extend X -> X_ext, labels b      rbf_extend_points
  a1/a2 cell build + tile plan        rbf_build_cells
  a4 RAS/BJ setup (blocks, on-chip fp32 inverses W)   inside rbf_gmres_solve
  a5-a7 FGMRES fp32 tier -> fp64 tier  rbf_gmres_solve (true residual <= 1e-6)
  a8 grid evaluation                  rbf_eval_grid
value = useful kernel-pair evaluations of the step (matvecs x useful pairs per
matvec + grid pairs) / step seconds (max over ranks), summed over ranks.  N > 1:
one problem split by z slabs over the ranks (strong scaling, DESIGN.md §7;
--parallel replicas runs an independent seeded problem per rank instead).
e2e = the same metric through rbf_reconstruct_host with HOST buffers (H2D of
centres + b and D2H of weights + field inside the timed region).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RBF kernel-pair evals/s and fit+eval seconds at N=1M, 1/2/4/8 B200"
MUFU_PER_CLK_PER_SM = 16          # MUFU.EX2 lanes per SM per clock (B200_PROFILING / SURVEY §6.4)
SMS = 148
SM_MAX_MHZ = 1965.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-rows", type=int, default=0)
    ap.add_argument("--fit-iters", type=int, default=50)
    ap.add_argument("--weak", action="store_true",
                    help="c5 weak scaling (configs[4]): 1.25M points per GPU, sigma scaled to keep sigma/spacing")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="N>1 slab mode: the library's data plane over CUDA-IPC peer memory (default; the transport "
                         "the multi-process GPU tests run) or over NCCL send/recv + allreduce")
    ap.add_argument("--parallel", default="slab", choices=["slab", "replicas"],
                    help="N>1: one problem split by slabs over the ranks (strong scaling, SURVEY §8(e)) "
                         "or one independent seeded problem per rank (weak scaling)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook (tests/test_gpu_bench_slab.py): every rank on cuda:0 over a gloo
    # group, to run the N>1 plumbing on a one-GPU box -- never a measurement
    if os.environ.get("RBF_BENCH_SHARED_GPU") == "1":
        local = 0
    return rank, world, local


class Clocks:
    """nvidia-smi sampling during the timed region (the recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.p = None

    def start(self):
        """Start the sampler and wait for its first (pre-timing, discarded) sample:
        nvidia-smi's start-up (NVML init, driver queries) stays out of the timed
        region, the samples read at stop() are all taken during it."""
        try:
            if os.environ.get("RBF_BENCH_NO_CLOCKS"):   # diagnostics only: is the sampler perturbing the run?
                return
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms",
                                       os.environ.get("RBF_BENCH_CLOCKS_MS", "200")],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.p.stdout.readline()
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for k, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(k)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def precond_name(cfg) -> str:
    kind = {0: "no preconditioner", 1: "block-Jacobi", 2: "RAS"}[cfg.precond_kind]
    if cfg.precond_kind == 0:
        return kind
    ov = f", overlap {cfg.overlap_sigmas} sigma" if cfg.precond_kind == 2 else ""
    return (f"{kind}(core {cfg.core_target}{ov}, shift {cfg.shift} a, "
            f"{'fp32 on-chip' if cfg.local_fp32 else 'fp64'} local inverses)")


def zero_set_quality(R, ctx, d, field, lo, hi, gn):
    import torch
    data = torch.as_tensor(d["x"], dtype=torch.float64, device=field.device)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    e0.record(s)
    pts = R.zero_set(ctx, field.reshape(-1), lo, hi, gn, data, 2 * d["sigma"])
    e1.record(s)
    torch.cuda.synchronize()
    P = pts.cpu().numpy()
    out = {"points": int(P.shape[0]), "ms": e0.elapsed_time(e1), "eps": 2 * d["sigma"]}
    cfg = d["cfg"]
    if cfg.kind == "blobby" and P.shape[0]:
        from synth.surfaces import _blobby_params, blobby_field
        K = cfg.kw.get("K", 16)
        _, c, sk = _blobby_params(K, d.get("seed", 0), 0.25 if K <= 16 else 0.15)
        sel = P[np.random.default_rng(0).choice(P.shape[0], min(P.shape[0], 200000), replace=False)]
        g, grad = blobby_field(sel, c, sk)
        dist = np.abs(g) / np.linalg.norm(grad, axis=1)
        out.update(dist_to_true_surface={"mean": float(dist.mean()), "p99": float(np.quantile(dist, 0.99)),
                                         "max": float(dist.max()), "sampled_points": int(sel.shape[0]),
                                         "grid_step": float((hi[0] - lo[0]) / (gn[0] - 1))})
    return out


def isosurface_report(R, ctx, d, cells, kern, w, lo, hi, gn):
    """Alg.1 steps 3-4 on the eps-surrounding (rbf_isosurface, eps = 2 sigma):
    the grid evaluated on M_ext^eps only + the marching-tetrahedra mesh of its
    zero set (reading R24), timed with CUDA events (one warm call, then 3)."""
    import torch
    data = torch.as_tensor(d["x"], dtype=torch.float64, device="cuda")
    eps = 2 * d["sigma"]
    fm = torch.empty(gn[0] * gn[1] * gn[2], dtype=torch.float32, device="cuda")
    R.isosurface(ctx, cells, kern, w, lo, hi, gn, data, eps, field=fm)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(3):
        V, T = R.isosurface(ctx, cells, kern, w, lo, hi, gn, data, eps, field=fm)
    e1.record(s)
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(s)
    for _ in range(3):
        Fm = R.eval_grid_masked(ctx, cells, kern, w, lo, hi, gn, data, eps, out=fm)
    e3.record(s)
    torch.cuda.synchronize()
    masked = int((~torch.isnan(fm)).sum().item())
    return {"eps": eps, "ms": e0.elapsed_time(e1) / 3, "masked_eval_ms": e2.elapsed_time(e3) / 3,
            "masked_nodes": masked, "grid_nodes": int(fm.numel()), "vertices": int(V.shape[0]),
            "triangles": int(T.shape[0]),
            "note": "rbf_isosurface = eps mask (fp64 distances) + grid on the masked node blocks + marching "
                    "tetrahedra; outside the timed step (the step evaluates the full grid, Alg.1 step 3)"}


def density_report(R, ctx, d):
    """Density measures of the surface points on the GPU (Eq.7-11, rbf_density):
    q_X, h_max and the sigma heuristics next to the configured sigma."""
    import torch
    x = torch.as_tensor(d["x"], dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    e0.record(s)
    out = R.density(ctx, x)
    e1.record(s)
    torch.cuda.synchronize()
    out = {k: float(v) for k, v in out.items()}
    out.update(ms=e0.elapsed_time(e1), sigma_used=d["sigma"], points=int(x.shape[0]))
    return out


def measured_traffic(cfg_name: str):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    capture (profiles/), or None when there is none for this config."""
    for rnd in ("r02", "r01"):
        path = os.path.join(ROOT, "profiles", rnd, f"traffic_sum_f32_{cfg_name}.json")
        try:
            with open(path) as fh:
                return json.load(fh)["dram_bytes_per_launch"]
        except (OSError, KeyError, ValueError):
            continue
    return None


def measured_ex2(cfg_name: str):
    """MUFU.EX2 thread-instructions per launch of the symmetric fp32 kernel from the
    committed ncu capture (profiles/r02), or None."""
    path = os.path.join(ROOT, "profiles", "r02", f"ex2_sum_f32_{cfg_name}.json")
    try:
        with open(path) as fh:
            return json.load(fh)["mufu_ex2_thread_inst_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def gate_note(cfg_name: str):
    """What the north star's 1e-6 residual gate means for this config (F1)."""
    path = os.path.join(ROOT, "profiles", "r02", f"gate_1e-6_{cfg_name}.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return None


def make_problem(cfg_name: str, seed: int, weak_world: int = 0):
    """weak_world = G > 0 (c5 only, BASELINE configs[4] "weak scaling from 1.25M
    points per GPU at 8 B200"; SURVEY §8(c) reading 15): N = 1.25M G points,
    sigma = 0.004 sqrt(8/G) (constant sigma/spacing: constant work per GPU),
    grid n = round(512 (G/8)^(1/3)), delta = 0.1 sigma."""
    from synth import make_inputs
    t = time.time()
    if weak_world:
        if cfg_name != "c5":
            raise SystemExit("--weak applies to c5 (BASELINE configs[4])")
        g = weak_world
        sig = 0.004 * (8.0 / g) ** 0.5
        d = make_inputs(cfg_name, seed=seed, n=1250000 * g, sigma=sig, delta=0.1 * sig,
                        grid_n=int(round(512 * (g / 8.0) ** (1.0 / 3.0))))
    else:
        d = make_inputs(cfg_name, seed=seed)
    d["gen_s"] = time.time() - t
    return d


# ------------------------------------------------------------------ ours ----
def run_ours(args, rank, world, local):
    import torch
    import paper_1305_5179_b200 as R
    from paper_1305_5179_b200.dist import throughput

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    shared = os.environ.get("RBF_BENCH_SHARED_GPU") == "1"
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = None if shared else dev   # device of the max/sum reductions of the timings
    slab = world > 1 and args.parallel == "slab"
    d = make_problem(args.config, args.seed if slab else args.seed + rank, world if args.weak else 0)
    cfg = d["cfg"]
    ctx = R.Context(local, distributed=slab, transport=args.transport)
    kern = R.Kernel(d["sigma"], d["cutoff_sigmas"])
    x = torch.as_tensor(d["x"], device=dev)
    nrm = torch.as_tensor(d["normals"], device=dev)
    lo, hi, gn = d["grid_lo"], d["grid_hi"], d["grid_n"]
    # fit budget: the paper's Table II protocol, a fixed 50 GMRES iterations;
    # the 1e-6 gate is unattainable at c4's sigma/spacing (DESIGN.md finding F1)
    solve_kw = dict(restart=cfg.restart, rtol=1e-6, phase1_rtol=1e-4, kind=cfg.precond_kind,
                    core_target=cfg.core_target, overlap_sigmas=cfg.overlap_sigmas, shift=cfg.shift,
                    local_fp32=cfg.local_fp32, cgs_passes=cfg.cgs_passes, max_iters=args.fit_iters)

    # cell edge of the config (RBF_BENCH_CELL_DIV overrides, for sweeps)
    cell_edge = kern.sigma * kern.cutoff_sigmas / float(os.environ.get("RBF_BENCH_CELL_DIV", cfg.cell_div))
    solve_kw["cell_edge"] = cell_edge

    if slab:
        # the slab path over NCCL has only run on one GPU through the loopback
        # transport: before timing it, every rank checks the
        # distributed one-sided product against its own single-GPU product of the
        # same replicated input (bit-identical by construction) and fails loudly
        centres, _ = R.extend_points(ctx, x, nrm, d["delta"])
        wchk = torch.as_tensor(np.random.default_rng(5).normal(size=centres.shape[0]), device=dev)
        fd = R.matvec(ctx, R.Cells(ctx, centres, kern, cell_edge=cell_edge), kern, wchk)
        solo = R.Context(local)
        fs = R.matvec(solo, R.Cells(solo, centres, kern, cell_edge=cell_edge), kern, wchk)
        torch.cuda.synchronize()
        if not torch.equal(fd, fs):
            raise RuntimeError(f"rank {rank}: distributed product differs from the single-GPU product "
                               f"(max |diff| {float((fd - fs).abs().max()):.3e}); slab path not trusted")
        del solo, fd, fs, centres

    def step():
        centres, b = R.extend_points(ctx, x, nrm, d["delta"])
        cells = R.Cells(ctx, centres, kern, cell_edge=cell_edge)
        w, rep = R.gmres_solve(ctx, cells, kern, b, **{k: v for k, v in solve_kw.items() if k != "cell_edge"})
        field = R.eval_grid(ctx, cells, kern, w, lo, hi, gn)
        return cells, w, field, rep

    # pair accounting (outside the timed region): useful pairs per matvec and per grid pass
    centres, b = R.extend_points(ctx, x, nrm, d["delta"])
    cells = R.Cells(ctx, centres, kern, cell_edge=cell_edge)
    useful_mv, visited_mv = R.matvec_pairs(ctx, cells, kern)
    useful_grid, visited_grid = R.eval_grid_pairs(ctx, cells, kern, lo, hi, gn, visited=True)
    info = cells.info()
    del cells

    # warm-up holds the same references as the timed loop (the previous step's
    # cells, weights and field stay alive while the next step allocates), so
    # the device memory pools reach their steady size before timing
    # (the SAME names as the timed loop binds: with another name for the cells, the
    # last warm-up's cells stayed alive next to the first timed step's, the pool
    # grew by one more cell structure inside timed step 2 -- 3 ms normally, once
    # 188 ms on a box whose driver had just released 80 GB from the test suite)
    # Head-room in the library's memory pool (rbf_pool_reserve), taken after the
    # first warm-up step (which shows the footprint) so that the remaining
    # warm-up steps are the first users of the new memory: the stream-ordered
    # allocator occasionally has to grow the pool in a later step (its free
    # blocks do not always fit the repeating requests), and a driver allocation
    # inside the timed region costs 3 ms on an idle box but took 75-200 ms right
    # after the test suite's process had released tens of GB; the first step that
    # touches freshly reserved memory is 12-90 ms slower, so it must not be a
    # timed one either.
    for k in range(max(args.warmup, 2)):
        cells_last, w, field, rep = step()
        if k == 0:
            torch.cuda.synchronize()
            held, used = ctx.pool_stats()
            ctx.pool_reserve(max(held, 1 << 30))
    torch.cuda.synchronize()
    clocks = Clocks(local)
    # no cyclic-GC pause inside the timed regions (the solver's host steps are on
    # the critical path; a full collection costs ~20 ms): collect now, re-enable after
    gc.collect()
    gc.disable()
    ctx.profile(True)
    ctx.profile_query()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    launches0 = R.launch_count()
    trace = os.environ.get("RBF_BENCH_TRACE") is not None
    evs = []
    e0.record(s)
    for _ in range(args.steps):
        cells_last, w, field, rep = step()
        reps.append(rep)
        if trace:
            evs.append((torch.cuda.Event(enable_timing=True), time.perf_counter(), ctx.pool_stats()))
            evs[-1][0].record(s)
    e1.record(s)
    torch.cuda.synchronize()
    if trace:   # per-step device / host times (diagnostics, stderr)
        prev_e, prev_h = e0, None
        for ev, th, ps in evs:
            print(f"[bench trace] step {prev_e.elapsed_time(ev):.1f} ms (device)"
                  + (f", {1e3 * (th - prev_h):.1f} ms (host)" if prev_h else "")
                  + f", pool {ps[0] / 1e9:.2f} GB held / {ps[1] / 1e9:.2f} GB used", file=sys.stderr)
            prev_e, prev_h = ev, th
    launches = R.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    gc.enable()
    prof = ctx.profile_query()
    ctx.profile(False)
    mv32 = sum(r["matvecs_f32"] for r in reps)
    mv64 = sum(r["matvecs_f64"] for r in reps)
    pairs_rank = useful_mv * (mv32 + mv64) + useful_grid * args.steps
    ms_max, pairs_all, value = throughput(ms, pairs_rank, red_dev)

    # e2e through the C-ABI with HOST buffers (rank-local problem)
    e2e = None
    if not args.no_e2e:
        centres, b = R.extend_points(ctx, x, nrm, d["delta"])
        xyz_h = centres.cpu().pin_memory()
        b_h = b.cpu().pin_memory()
        n = xyz_h.shape[0]
        w_h = torch.empty(n, dtype=torch.float64).pin_memory()
        f_h = torch.empty((gn[2], gn[1], gn[0]), dtype=torch.float32).pin_memory()
        rkw = dict(solve_kw)
        for _ in range(max(1, min(args.warmup, 3))):   # warm
            R.reconstruct_host(ctx, xyz_h, b_h, kern, lo, hi, gn, w_out=w_h, field_out=f_h, **rkw)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        gc.collect()
        gc.disable()
        t0 = time.perf_counter()
        mv_e2e = 0
        for _ in range(args.steps):
            _, _, rep_e = R.reconstruct_host(ctx, xyz_h, b_h, kern, lo, hi, gn, w_out=w_h, field_out=f_h, **rkw)
            mv_e2e += rep_e["matvecs_f32"] + rep_e["matvecs_f64"]
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) * 1e3
        gc.enable()
        pe = useful_mv * mv_e2e + useful_grid * args.steps
        te, pe, ve = throughput(te, pe, red_dev)
        e2e = {"value": ve, "unit": "pairs/s", "ms_per_step": te / args.steps,
               "h2d_bytes_per_step": int(xyz_h.numel() * 4 + b_h.numel() * 4),
               "d2h_bytes_per_step": int(w_h.numel() * 8 + f_h.numel() * 4)}

    # Alg.1 step 3 output (outside the timed step): the eps-masked zero set of the
    # last field (rbf_zero_set, eps = 2 sigma, reading R11) and its distance to
    # the generator's exact surface g = 0 (first-order |g| / |grad g|)
    zs = dens = iso = None
    if rank == 0:
        zs = zero_set_quality(R, ctx, d, field, lo, hi, gn)
        dens = density_report(R, ctx, d)
    # collective in slab mode (the masked grid gathers the ranks' layers): every rank calls it
    iso = isosurface_report(R, ctx, d, cells_last, kern, w, lo, hi, gn)

    # roofline of the dominant kernel (fp32 summation), live CUDA-event timing
    t_mv, n_mv = prof["matvec_f32"]
    avg_mv_ms = t_mv / max(n_mv, 1)
    achieved = useful_mv / (avg_mv_ms * 1e-3) / 1e12
    peak_max = SMS * MUFU_PER_CLK_PER_SM * SM_MAX_MHZ * 1e6 / 1e12
    # the solver's operator under OP_AUTO (rbf_op_variant; sym_mode in summation.cu)
    sym = 2 if 3 * cfg.n // max(world if slab else 1, 1) >= (1 << 18) else 0
    kname = {0: "sum_f32_kernel (one-sided)", 1: "sum_f32_kernel (symmetric, 64-target tiles)",
             2: "sum_f32_symb_kernel (symmetric, 128-target tiles)"}[sym]
    roofline = {"bound": "alu", "kernel": kname + ", MUFU.EX2", "achieved": achieved, "peak": peak_max,
                "unit": "Tpairs/s", "frac": achieved / peak_max,
                "peak_basis": "148 SMs x 16 MUFU.EX2/clk x 1965 MHz (max clock; 16.00 ex2/clk/SM measured, "
                              "profiles/r01/peaks_mufu_ffma2.json); roofline of the one-sided algorithm, 1 ex2 per "
                              "useful pair (the symmetric kernel spends 1 ex2 per 2 pair contributions, reading R19)",
                "frac_at_measured_clock": (achieved / (SMS * MUFU_PER_CLK_PER_SM * clk["sm_mhz"] * 1e6 / 1e12)
                                           if clk.get("sm_mhz") else None),
                "avg_launch_ms": avg_mv_ms, "launches": n_mv, "useful_pairs_per_launch": useful_mv,
                "visited_pairs_per_launch": visited_mv, "traffic": measured_traffic(args.config)}
    # the same kernel against the MUFU.EX2 pipe it actually drives: the symmetric
    # kernel issues ex2_per_useful exponentials per useful ordered pair (ncu count,
    # profiles/r02; tools/plan_sim.py models it from the tile plan)
    ex2 = measured_ex2(args.config)
    if ex2 and sym == 2:
        roofline["ex2_per_launch"] = ex2
        roofline["ex2_per_useful_pair"] = ex2 / useful_mv
        roofline["mufu_busy_frac"] = ex2 / (avg_mv_ms * 1e-3) / (peak_max * 1e12)
    stage_ms = {k: round(v[0] / args.steps, 3) for k, v in prof.items()}

    cpu = None
    if rank == 0 and world == 1:
        cpu = cpu_baseline(d, args)
    last = reps[-1]
    out = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "fit_eval_s": ms_max / args.steps / 1e3,
        "higher_is_better": True, "scaling": "strong" if slab and not args.weak else "weak", "vs_baseline": None, "dtype": "f32+f64",
        "data": "synthetic (seeded blobby surface, SURVEY §8(c) reading 14)",
        "config": {"workload": f"{args.config}: {cfg.kind} K={cfg.kw.get('K')} N={cfg.n} surface points "
                               f"({3 * cfg.n} centres), sigma={cfg.sigma}, cutoff 6 sigma, GMRES({cfg.restart}) "
                               f"+ {precond_name(cfg)}, {args.fit_iters} iterations "
                               f"(Table II protocol) or true residual 1e-6, "
                               f"grid {gn[0]}^3",
                   "centres_per_gpu": 3 * cfg.n // world if slab else 3 * cfg.n,
                   "global_centres": 3 * cfg.n if slab else 3 * cfg.n * world,
                   "parallelism": (f"slab x{world} (z cell planes; halo exchange, reverse halo reduction and "
                                   f"Krylov all-reduces over the {args.transport} transport; the multi-rank path "
                                   "is verified on one GPU -- threads over the loopback transport and separate "
                                   "processes over the IPC transport -- not yet on a multi-GPU box)" if slab
                                   else f"replicas x{world} (independent seeded instances)"),
                   "l2": (f"working set >> 126 MB L2 (block inverses {last['precond_bytes'] / 1e9:.2f} GB, fp32 Krylov "
                          f"basis {4 * 3 * cfg.n * (2 * cfg.restart + 1) / 1e9:.2f} GB, cells + vectors + neighbour lists "
                          f"{(0.07 + 0.11) * 3 * cfg.n / 1e6:.2f} GB); no explicit flush")},
        "e2e": e2e, "gpu_launches": None, "clocks": clk, "roofline": roofline, "cpu_baseline": cpu,
        "detail": {"useful_pairs_per_matvec": useful_mv, "visited_pairs_per_matvec": visited_mv,
                   "useful_pairs_grid": useful_grid, "visited_pairs_grid": visited_grid,
                   "grid_useful_pairs_per_s": useful_grid / (prof["grid"][0] / max(prof["grid"][1], 1) * 1e-3)
                   if prof["grid"][1] else None,
                   "matvecs_f32_per_step": mv32 / args.steps,
                   "matvecs_f64_per_step": mv64 / args.steps, "stage_ms_per_step": stage_ms,
                   "iters_phase1": last["iters_phase1"], "iters_phase2": last["iters_phase2"],
                   "rel_residual_true": last["rel_residual_true"], "converged": last["converged"],
                   "ras_blocks": last["nblocks"], "precond_bytes": last["precond_bytes"], "zero_set": zs, "isosurface": iso,
                   "gate_1e-6": gate_note(args.config),
                   "density": dens,
                   "cells": info,
                   "gen_s": round(d["gen_s"], 1)},
    }
    out["gpu_launches"] = launches
    if rank == 0:
        print(json.dumps(out), flush=True)
    del cells_last, w, field
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()


# ------------------------------------------------------------- cpu oracle ---
def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(d, args, rows: int | None = None, extras: bool = True):
    """The oracle (oracle/, as it stands, never tuned for this) on the host cores:
    the headline is a bounded row sample of the same workload's brute-force fp64
    matvec (useful pairs/s); `steps` adds the two steps the paper times (Table II
    solve, Table III grid evaluation) on the small configs: c1 dense LU, c1 fp64
    GMRES + RAS, c1 full brute-force grid, c2 sampled grid."""
    from oracle import extend as OE
    from oracle import kernel as OK
    X = OE.extend(d["x"], d["normals"], d["delta"])
    n = X.shape[0]
    rows = rows or args.cpu_sample_rows or 400
    sel = np.sort(np.random.default_rng(1).choice(n, rows, replace=False))
    w = np.random.default_rng(2).normal(size=n)
    procs = os.cpu_count() or 1
    t = time.perf_counter()
    OK.matvec_parallel(X, w, d["sigma"], rows=sel, procs=procs)
    dt = time.perf_counter() - t
    useful = OK.pair_count(X, d["sigma"], rows=sel)
    out = {"value": useful / dt, "unit": "pairs/s", "cores": procs, "cpu_model": cpu_model(), "kind": "oracle",
           "dense_pairs_per_s": rows * n / dt,
           "sample": f"brute-force fp64 matvec rows ({rows} of {n} sampled targets x all {n} centres) of the "
                     f"same config; useful pairs counted on the same rows", "seconds": dt}
    if extras:
        out["steps"] = cpu_steps(procs)
    return out


def cpu_steps(procs: int) -> dict:
    """Oracle timings of the paper's timed steps on configs small enough to run."""
    from oracle import cells as OC
    from oracle import extend as OE
    from oracle import grid as OG
    from oracle import kernel as OK
    from oracle import solve as OS
    from synth import make_inputs
    res = {}
    d = make_inputs("c1")
    X = OE.extend(d["x"], d["normals"], d["delta"]).astype(np.float64)
    b = OE.labels(len(d["x"]), d["delta"]).astype(np.float32).astype(np.float64)
    sigma = d["sigma"]
    t = time.perf_counter()
    OS.lu_solve(X, b, sigma)
    res["c1_dense_lu_s"] = time.perf_counter() - t
    t = time.perf_counter()
    A = OK.dense_matrix(X, sigma)
    oc = OC.build(X.astype(np.float32), 6 * sigma, cell_edge=6 * sigma / 3.999)
    blocks = OS.ras_blocks(oc, sigma, 512, 3.0)
    perm, factors = oc["perm"], {}

    def M(v):
        z = np.empty_like(v)
        z[perm] = OS.ras_apply(blocks, oc["sorted"], v[perm], sigma, factors=factors)
        return z

    _, info = OS.gmres(lambda v: A @ v, b, restart=30, rtol=1e-6, maxit=200, apply_M=M)
    res["c1_gmres_ras_to_1e-6_s"] = time.perf_counter() - t
    res["c1_gmres_ras_iters"] = info["iters"]
    w = np.random.default_rng(3).normal(size=len(X))
    lo, hi, gn = d["grid_lo"], d["grid_hi"], d["grid_n"]
    t = time.perf_counter()
    OK.matvec_parallel(X, w, sigma, targets=OG.nodes(lo, hi, gn), procs=procs)
    res["c1_grid_full_s"] = time.perf_counter() - t
    res["c1_grid_nodes"] = int(np.prod(gn))
    d2 = make_inputs("c2")
    X2 = OE.extend(d2["x"], d2["normals"], d2["delta"]).astype(np.float64)
    w2 = np.random.default_rng(4).normal(size=len(X2))
    lo, hi, gn = d2["grid_lo"], d2["grid_hi"], d2["grid_n"]
    flat = np.sort(np.random.default_rng(5).choice(int(np.prod(gn)), 2000, replace=False))
    t = time.perf_counter()
    OK.matvec_parallel(X2, w2, d2["sigma"], targets=OG.nodes(lo, hi, gn, flat=flat), procs=procs)
    dt = time.perf_counter() - t
    res["c2_grid_sampled"] = {"nodes": len(flat), "seconds": dt,
                              "extrapolated_full_grid_s": dt * np.prod(gn) / len(flat)}
    return res


def run_reference(args, rank, world, local):
    if rank != 0:
        return
    d = make_problem(args.config, args.seed)
    rows = max(50, args.cpu_sample_rows or 200)
    for _ in range(max(args.warmup, 0) and 1):
        cpu_baseline(d, args, rows=50, extras=False)
    times, vals = [], []
    for _ in range(args.steps):
        cb = cpu_baseline(d, args, rows=rows, extras=False)
        times.append(cb["seconds"])
        vals.append(cb["value"])
    cfg = d["cfg"]
    v = float(np.median(vals))
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(times)) * 1e3,
           "higher_is_better": True, "scaling": "strong" if world > 1 and args.parallel == "slab" and not args.weak else "weak",
           "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": {"workload": f"{args.config}: N={cfg.n} ({3 * cfg.n} centres) "
                                                      f"sampled-row brute-force matvec"},
           "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": os.cpu_count(), "cpu_model": cpu_model(),
                            "kind": "oracle",
                            "sample": f"{rows} sampled target rows x all centres per step"},
           "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
