"""Benchmark: NLL+gradient evaluations per second of the Vecchia/VIF likelihood at
n = 1.1M, m = 30 (BASELINE.json metric), on synthetic NOAA-shaped station x day data.

One "step" = one optimizer evaluation: rebuild the structure at theta and
compute the NLL and its 7-component gradient (estimation.cpp:277-325), over all
n observations.  Neighbour search and inducing-point seeding are setup (their
wall time is reported separately as nn_search_s / seeding_s).

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
        [--workload vecchia|vif] [--stations S] [--days D]
For N > 1 launch under torch.distributed.run (one process per GPU); observations
are sharded by contiguous index ranges and partial sums all-reduced with NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "VIF/Vecchia NLL+grad evals/sec at n=1.1M, m=30 (1/2/4/8 B200); NN-search s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="vif", choices=["vecchia", "vif", "fitc"],
                    help="vif: cfg4 (headline); vecchia: cfg4 data, d_c neighbours; fitc: cfg5 (FITC, 2000 "
                         "inducing points, plus 1-day-ahead prediction at every station)")
    ap.add_argument("--m", type=int, default=None, help="sts kMeans++ inducing request (VIF 1000, FITC 2000)")
    ap.add_argument("--stations", type=int, default=10000)
    ap.add_argument("--days", type=int, default=110)
    ap.add_argument("--m_v", type=int, default=30)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.m is None:
        args.m = 2000 if args.workload == "fitc" else 1000
    return args


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([v.strip() for v in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if len(r) > 3 + k and r[3 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _synth():
    """synth.py loaded by path: the reference arm must not import the engine package (no libstgp_b200)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("_stgp_synth", os.path.join(ROOT, "paper_2602_03609_b200", "synth.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def make_data(stations, days, seed=20260203, reference=False):
    """Synthetic station x day data in order_observations order (dataset.cpp:81-114): the engine's
    ordering on the GPU arm, the oracle's (identical permutation, tests/test_ordering.py) on the
    reference arm."""
    synth = _synth()
    theta = synth.THETA_T3 if stations >= 2000 else synth.THETA_SEC4
    box = (4.6e6, 2.9e6) if stations >= 2000 else (1.0, 1.0)
    x, y, t, resp = synth.station_day(stations, days, box=box, theta=theta, seed=seed)
    if reference:
        from oracle import oracle as O
        perm = O.order_observations(t, seed)
    else:
        import paper_2602_03609_b200 as S
        perm = S.order_observations_perm(t, seed)
    return x[perm], y[perm], t[perm], resp[perm], theta


def bench_config(args, n, world):
    """The `config` object both arms print (same keys and values: the driver compares them)."""
    return {"workload": workload_name(args), "n": n, "m_v": args.m_v, "stations": args.stations,
            "days": args.days, "theta": "PAPER.md Table 3 (NOAA temperature)" if args.stations >= 2000
            else "PAPER.md section 4",
            "neighbors": {"vif": "d_r exact kNN (residual_neighbors)", "fitc": "none (FITC)",
                          "vecchia": "d_c exact kNN (correlation_neighbors)"}[args.workload],
            "inducing_request": args.m if args.workload in ("vif", "fitc") else None,
            "parallelism": f"index-shard x{world}",
            "l2": "inputs larger than L2 (nbr 132 MB + A 264 MB)" if args.workload == "vecchia"
            else "inputs larger than L2 (n x M f64 work arrays, 8-19 GB each)"}


# canonical algorithmic FP64 work per row: FMA = k^3/6 + 3 k^2 (Cholesky,
# two triangular solves per RHS, products), plus c_k kernel evaluations and c_k kernel
# gradients; KE = 30 flop, KG = 50 flop (device instruction counts of gneiting_eval /
# gneiting_grad incl. the exp port).
KE_FLOP, KG_FLOP = 30.0, 50.0
VIFGRAD_DRAM = 5.407542e9 + 0.379444e9  # vif_grad_stored_kernel, ncu at cfg4 (profiles/r02/v5)


def vecchia_flops(nbr_counts):
    k = nbr_counts.astype(np.float64)
    ck = (k + 1) * (k + 2) / 2
    return float(np.sum(2 * (k ** 3 / 6 + 3 * k ** 2) + ck * (KE_FLOP + KG_FLOP)))


def vif_flops(nbr_counts, M):
    """canonical FP64 work of one VIF NLL+grad:
    FMA = n [3.5 M^2 + (c_k + (k+1)^2 + k + 2) M + k^3/6 + k^2] + 2/3 M^3, plus n (M + c_k) KE and KG."""
    k = nbr_counts.astype(np.float64)
    ck = (k + 1) * (k + 2) / 2
    fma = np.sum(3.5 * M * M + (ck + (k + 1) ** 2 + k + 2) * M + k ** 3 / 6 + k ** 2) + 2.0 / 3.0 * M ** 3
    return float(2 * fma + np.sum((M + ck) * (KE_FLOP + KG_FLOP)))


def vif_rows_flops(nbr_counts, M):
    """canonical work of the fused VIF-gradient row kernel: closure Gram c_k M, Ga (k+1) M and
    aGa M FMAs, Cholesky k^3/6 and two solves 2 k^2, c_k KE + KG."""
    k = nbr_counts.astype(np.float64)
    ck = (k + 1) * (k + 2) / 2
    return float(np.sum(2 * ((ck + k + 2) * M + k ** 3 / 6 + 2 * k ** 2) + ck * (KE_FLOP + KG_FLOP)))


def vif_build_rows_flops(nbr_counts, M):
    """canonical work of the VIF build row kernel (vecchia_rows_kernel<build>): closure Gram c_k M FMA,
    Cholesky k^3/6 and one solve k^2 FMA, and c_k covariance evaluations (KE)."""
    k = nbr_counts.astype(np.float64)
    ck = (k + 1) * (k + 2) / 2
    return float(np.sum(2 * (ck * M + k ** 3 / 6 + k ** 2) + ck * KE_FLOP))


def fitc_flops(n, M):
    """canonical FP64 work of one FITC NLL+grad: W = L_m^{-1} U, K = I + W Lambda^{-1} W^T (symmetric),
    K^{-1} W, W diag(phi) W^T (symmetric), omega = L_m^{-T} omega' -> 3 n M^2 FMA, plus n M KE and KG."""
    return float(2 * 3.0 * n * M * M + n * M * (KE_FLOP + KG_FLOP))


def _oracle_sample(kind, x, y, t, theta, m_v, ns, Z=None):
    """Oracle model on the first ns ordered rows (a prefix with its predecessor neighbour sets is a
    self-contained model); the neighbour search is setup, not timed."""
    from oracle import oracle as O
    nbr = None
    if kind == "vif":
        nbr = O.dr_neighbors_rows(x[:ns], y[:ns], t[:ns], theta, Z, m_v)
    elif kind == "vecchia":
        nbr = O.dc_neighbors(x[:ns], y[:ns], t[:ns], theta, m_v)
    return O.OracleModel(kind, x[:ns], y[:ns], t[:ns], theta, nbr=nbr, Z=Z)


def _time_eval(om, resp, ns):
    """Objective::value + Objective::gradient as the reference runs them: build + nll, build + nll_grad
    (estimation.cpp:277-325; the oracle rebuilds the structure inside each call)."""
    t0 = time.perf_counter()
    om.nll(resp[:ns])
    om.nll_grad(resp[:ns])
    return time.perf_counter() - t0


SAMPLE_ROWS = {"vif": 30000, "fitc": 20000, "vecchia": 200000}


def cpu_sample(kind, x, y, t, resp, theta, m_v, Z=None):
    """cpu_baseline: the reference algorithm (oracle restatement, dense n x M^2 parts on OpenBLAS with
    all host threads, per-row work on OpenMP) on a prefix of >= 2 days of the ordered rows, scaled
    linearly to n (every term of one evaluation is linear in n at fixed M and m_v)."""
    from oracle import oracle as O
    cores = O.set_threads(os.cpu_count() or 1)
    blas = O.set_blas(True, cores)
    n = len(x)
    ns = min(n, SAMPLE_ROWS[kind])
    om = _oracle_sample(kind, x, y, t, theta, m_v, ns, Z)
    dt = _time_eval(om, resp, ns)
    O.set_blas(False)
    per_eval_full = dt * n / ns
    days = len(np.unique(t[:ns]))
    return {"value": 1.0 / per_eval_full, "unit": "evals/s", "cores": cores, "kind": "port",
            "sample": f"oracle {kind.upper()} build+nll+build+nll_grad on the first {ns} of {n} ordered rows "
                      f"({days} days{'' if Z is None else f', all {len(Z)} inducing points'}; {dt:.2f} s; dense "
                      f"parts on {'OpenBLAS' if blas else 'sequential loops'}), scaled linearly to n"}


def run_reference(args):
    """--impl reference: the reference algorithm's CPU path (the oracle restatement -- the reference itself
    cannot be built here, DESIGN.md §2 -- with its dense n x M^2 contractions on OpenBLAS) on all host
    cores, one bounded prefix sample of the workload per step, scaled to n.  Neither the engine package
    nor libstgp_b200.so is loaded on this arm."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle import oracle as O
    x, y, t, resp, theta = make_data(args.stations, args.days, reference=True)
    n = len(x)
    cores = O.set_threads(os.cpu_count() or 1)
    kind = args.workload
    Z = None
    if kind in ("vif", "fitc"):
        Z, _, _ = O.sts_kmeanspp(x, y, t, args.m, 20260203)
    ns = min(n, SAMPLE_ROWS[kind])
    om = _oracle_sample(kind, x, y, t, theta, args.m_v, ns, Z)
    blas = O.set_blas(True, cores)
    times = []
    for step in range(args.warmup + args.steps):
        dt = _time_eval(om, resp, ns)
        if step >= args.warmup:
            times.append(dt * n / ns)
    O.set_blas(False)
    per = statistics.median(times)
    val = 1.0 / per
    days = len(np.unique(t[:ns]))
    desc = (f"oracle {kind.upper()} build+nll+build+nll_grad on the first {ns} of {n} ordered rows ({days} days"
            f"{'' if Z is None else f', all {len(Z)} inducing points'}; dense parts on "
            f"{'OpenBLAS' if blas else 'sequential loops'}) per step, scaled linearly to n")
    line = {"metric": METRIC, "value": val, "unit": "evals/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (station x day layout of simulate.cpp, random-feature field + nugget)",
            "config": bench_config(args, n, world),
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": "evals/s", "cores": cores, "kind": "port", "sample": desc},
            "e2e": {"value": val, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_name(args):
    shape = (args.stations, args.days)
    if shape == (10000, 110):
        return {"vif": "cfg4-vif-dr-sts", "vecchia": "cfg4-vecchia-dc", "fitc": "cfg5-fitc-sts-predict"}[args.workload]
    if shape == (1000, 100) and args.m_v == 20:
        return {"vif": "cfg3-vif-dr-sts", "vecchia": "cfg2-vecchia-dc", "fitc": "fitc-1000x100"}[args.workload]
    return f"{args.workload}-{args.stations}x{args.days}-m{args.m}-mv{args.m_v}"


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import paper_2602_03609_b200 as S

    from paper_2602_03609_b200 import dist as D
    world, rank, local = D.env_ranks()
    dist = world > 1
    if dist:
        import torch.distributed as tdist
        torch.cuda.set_device(local)
        tdist.init_process_group("gloo")
    ctx = S.Context(local)
    if dist:
        D.setup_engine_comm(ctx, rank, world)

    x, y, t, resp, theta = make_data(args.stations, args.days)
    n = len(x)
    ds = S.SpaceTimeDataset(x, y, t, resp, ctx=ctx)
    # FP64 roofline denominators, measured first: the microbenchmarks also bring the GPU out of its
    # idle clock state before the (single-shot) searches are timed
    dfma_peak, dmma_peak = ctx.fp64_peak_tflops(), ctx.dmma_peak_tflops()
    ctx.profile(True)
    extra = {}
    if args.workload == "vif":
        t0 = time.perf_counter()
        ind = S.sts_kmeanspp(ds, args.m, 20260203)
        extra["seeding_s"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        nb = S.residual_neighbors(ds, theta, ind, args.m_v)
        nn_s = time.perf_counter() - t0
        knn_ms = ctx.profile_get("knn_dr")[0] + ctx.profile_get("dr_whiten")[0]
        warm = []
        for _ in range(5):  # warm repeats (identical sets); the median is reported
            t0 = time.perf_counter()
            nb = S.residual_neighbors(ds, theta, ind, args.m_v)
            warm.append(time.perf_counter() - t0)
        extra["nn_search_warm_s"] = statistics.median(warm)
        extra["nn_search_warm_all_s"] = warm
        s = S.build_vif(ds, theta, ind, nb, S.OBSERVATION)
        M = ind.M
        extra["inducing"] = {"m": args.m, "M": M, "m_s": ind.m_s, "m_t": ind.m_t}
    elif args.workload == "fitc":
        t0 = time.perf_counter()
        ind = S.sts_kmeanspp(ds, args.m, 20260203)
        extra["seeding_s"] = time.perf_counter() - t0
        nb, nn_s, knn_ms = None, None, None
        s = S.build_fitc(ds, theta, ind)
        M = ind.M
        extra["inducing"] = {"m": args.m, "M": M, "m_s": ind.m_s, "m_t": ind.m_t}
    else:
        t0 = time.perf_counter()
        nb = S.correlation_neighbors(ds, theta, args.m_v)
        nn_s = time.perf_counter() - t0
        knn_ms = ctx.profile_get("knn_dc")[0] + ctx.profile_get("knn_dr")[0] + ctx.profile_get("dr_whiten")[0]
        warm = []
        for _ in range(5):  # warm repeats (identical sets); the median is reported
            t0 = time.perf_counter()
            nb = S.correlation_neighbors(ds, theta, args.m_v)
            warm.append(time.perf_counter() - t0)
        extra["nn_search_warm_s"] = statistics.median(warm)
        extra["nn_search_warm_all_s"] = warm
        s = S.build_vecchia(ds, theta, nb, S.OBSERVATION)
        M = 0
    nbr = nb.indices() if nb is not None else None
    counts = (nbr >= 0).sum(axis=1) if nbr is not None else np.zeros(n, dtype=np.int64)

    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", local))
    thetas = [tuple(v * (1.0 + 0.01 * ((i % 5) - 2)) if j in (1, 2, 3) else v for j, v in enumerate(theta))
              for i in range(args.warmup + args.steps)]
    for i in range(args.warmup):
        S.evaluate(s, thetas[i])
    ctx.profile_reset()
    launches0 = ctx.kernel_launches()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for i in range(args.steps):
            v, g = S.evaluate(s, thetas[args.warmup + i])
        e1.record(stream)
        torch.cuda.synchronize()
    ms_total = e0.elapsed_time(e1)
    launches = ctx.kernel_launches() - launches0
    ms_step = ms_total / args.steps
    ms_step = D.max_over_ranks(ms_step)

    # e2e: the public API with host buffers (pinned y uploaded each step, nll+grad read back)
    pinned = torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
    pinned[:] = resp
    S.evaluate(s, thetas[0], pinned)
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.steps):
        S.evaluate(s, thetas[args.warmup + i], pinned)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    e2e_s = D.max_over_ranks(e2e_s)

    # roofline of the dominant kernel of this step, timed live with events on the context stream
    lo, hi = D.shard_range(n, rank, world)
    fp64_peak = max(dfma_peak, dmma_peak)
    prof = ctx.profile_all()

    def region_avg(name):
        ms_, cnt_ = prof.get(name, (0.0, 0))
        return ms_ / max(cnt_, 1)

    if args.workload == "vif":
        # the dominant kernel of the step (15% of it): the closure rows of the build
        kname = ("vecchia_rows_kernel<build>: closure Gram W_cl^T W_cl on DMMA, closure covariances, register "
                 "Cholesky, A and D per row")
        k_avg = region_avg("rows")
        flops_launch = vif_build_rows_flops(counts[lo:hi], M)
        step_flops = vif_flops(counts, M)
    elif args.workload == "fitc":
        # FITC is n M^2 products throughout, all on the int8 tensor cores (the int8_tensor object below
        # becomes the line's roofline); W = L_m^{-1} U is kept here as its FP64-equivalent rate
        kname = "W = L_m^{-1} U (triangle-cut Ozaki rows form on ozaki_tc_kernel), FP64-equivalent"
        k_avg = region_avg("W_trmm")
        flops_launch = float(M) * (M + 1) * (hi - lo)
        step_flops = fitc_flops(n, M)
    else:
        kname = "vecchia_rows_kernel<grad>"
        k_avg = region_avg("rows")
        flops_launch = vecchia_flops(counts[lo:hi])
        step_flops = vecchia_flops(counts)
    achieved = flops_launch / (k_avg * 1e-3) / 1e12
    # DRAM bytes of the row pass from one ncu --set full capture per kernel (cfg4, N = 1):
    # dram__bytes_read.sum + dram__bytes_write.sum, profiles/r01/rows_{build,grad}_full_ncu.txt
    cfg4_1 = args.workload == "vif" and (args.stations, args.days) == (10000, 110) and world == 1
    traffic = (14.260330e9 + 5.761680e9) if cfg4_1 else None
    breakdown = {k: round(ms_ / max(c_, 1), 3) for k, (ms_, c_) in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    roof = {"bound": "fp64", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": achieved / fp64_peak, "traffic": traffic,
            "traffic_source": ("ncu --set full dram__bytes_read+write of vecchia_rows_kernel<build> at cfg4 "
                               "(profiles/r02/v5/full_vecchia_rows_kernel.txt)") if traffic else None,
            "kernel": kname, "kernel_ms": k_avg,
            "kernel_share": k_avg / ms_step, "flop_per_launch": flops_launch,
            "peak_source": (f"measured in-run: max of DMMA m8n8k4 ({dmma_peak:.1f}) and DFMA ({dfma_peak:.1f}) "
                            "throughput microbenchmarks (MEASURED_PEAKS.json has no FP64 entry)"),
            # whole step in canonical FP64 flops, counting the products that run as int8 Ozaki emulation
            # as FP64 FMAs: an FP64-equivalent rate, which can exceed the FP64 peak (FITC does)
            "step_canonical_flop": step_flops, "step_fp64_equiv_tflops": step_flops / (ms_step * 1e-3) / 1e12,
            "step_fp64_equiv_frac": step_flops / (ms_step * 1e-3) / 1e12 / fp64_peak,
            "phase_ms": breakdown}
    if args.workload == "vif":
        # the whole closure-row pass of an evaluation: build rows + Ga (tile SDDMM) + gradient rows
        rp_ms = region_avg("rows") + region_avg("g_ga") + region_avg("rows_vifgrad")
        rp_flops = vif_rows_flops(counts[lo:hi], M)
        roof["row_pass"] = {
            "kernels": "vecchia_rows_kernel<build> + tile_ga_kernel + vif_grad_stored_kernel", "kernel_ms": rp_ms,
            "achieved": rp_flops / (rp_ms * 1e-3) / 1e12, "frac": rp_flops / (rp_ms * 1e-3) / 1e12 / fp64_peak,
            "traffic": (14.260330e9 + 5.761680e9 + 24.167864e9 + 0.286370e9 + VIFGRAD_DRAM) if cfg4_1 else None}
    # the FP64 products that run on the int8 tensor cores (Ozaki slicing, csrc/ozaki.cu): X = K^-1 V'
    # (FITC: K^-1 W), K = S S^T and V'F^T (FITC: W diag(phi) W^T), and the triangular W = L_m^-1 U and
    # omega = L_m^-T omega', each S(S+1)/2 int8 MACs per FP64 FMA (S = 6 slices for the row form, 7 for
    # the long reductions and the triangular products)
    # per evaluation: the region total over the evaluations profiled (timed steps and e2e steps alike)
    oz_ms = prof.get("oz_imma", (0.0, 0))[0] / max(prof.get("K_gemm_chol", (0.0, 1))[1], 1)
    if args.workload in ("vif", "fitc") and oz_ms > 0:
        s_all = os.environ.get("STGP_OZAKI_S")
        s_rows = int(os.environ.get("STGP_OZAKI_S_ROWS", s_all or 6))
        s_cols = int(os.environ.get("STGP_OZAKI_S_COLS", s_all or 7))
        ldm = (M + 15) // 16 * 16
        # X (rows form, full) and V'F^T (full), K = S S^T symmetric: its lower half (the kernel computes only
        # the tiles that reach the lower triangle and mirrors)
        s_tri = int(os.environ.get("STGP_OZAKI_S_TRMM", s_all or 7))
        pr_, pc_, pt_ = s_rows * (s_rows + 1) / 2, s_cols * (s_cols + 1) / 2, s_tri * (s_tri + 1) / 2
        if args.workload == "fitc" and os.environ.get("STGP_FITC_SYM_S", "1") != "0":
            # W diag(phi) W^T is symmetric and computed on one triangle of tiles, like K
            int8_ops = 2.0 * pr_ * ldm * ldm * (hi - lo) + 2 * pc_ * ldm * (ldm + 1) * (hi - lo)
        else:
            int8_ops = 2.0 * (pr_ + pc_) * ldm * ldm * (hi - lo) + pc_ * ldm * (ldm + 1) * (hi - lo)
        if os.environ.get("STGP_OZAKI_TRMM", "1") != "0":
            # two triangular products, M (M + 1) / 2 FMA per column each (algorithmic: the triangle)
            int8_ops += 2 * 2.0 * pt_ * ldm * (ldm + 1) / 2 * (hi - lo)
        int8_peak = 2.0 * peaks().get("bf16_tflops", 1669.7)
        roof["int8_tensor"] = {
            "bound": "tensor", "achieved": int8_ops / (oz_ms * 1e-3) / 1e12, "peak": int8_peak, "unit": "TOPS",
            "frac": int8_ops / (oz_ms * 1e-3) / 1e12 / int8_peak, "kernel_ms": oz_ms, "ops_per_step": int8_ops,
            "kernel": "ozaki_tc_kernel: hand-written tcgen05.mma kind::i8 (TMA, per-diagonal TMEM accumulators, "
                      "FP64 epilogue) over the Ozaki slices",
            "peak_source": "2 x measured dense bf16 (MEASURED_PEAKS.json burst; B200 int8:bf16 dense = 2:1)"}
        # the step's dominant kernel is the tcgen05 product kernel (VIF: its 16 launches take 32% of the
        # evaluation's kernel time against 18% for the closure-row build, profiles/r02/v12/launches_vif_summary.txt;
        # FITC: 70%): it becomes the line's roofline object, the FP64 view of the largest FP64 kernel kept beside it
        fp64_view = {k_: roof.pop(k_) for k_ in ("bound", "achieved", "peak", "unit", "frac", "traffic",
                                                  "traffic_source", "kernel", "kernel_ms", "kernel_share",
                                                  "flop_per_launch", "peak_source")}
        roof.update(roof.pop("int8_tensor"))
        roof["kernel_share"] = oz_ms / ms_step
        # DRAM bytes of the tcgen05 launches of one cfg4 evaluation (ncu launch list, N = 1)
        roof["traffic"] = 82.97e9 if cfg4_1 else None
        roof["traffic_source"] = ("ncu launch list of one cfg4 evaluation: dram__bytes_read+write summed over the "
                                  "ozaki_tc_kernel launches (profiles/r02/v12/launches_vif_summary.txt)") if cfg4_1 else None
        roof["rows_build" if args.workload == "vif" else "W_trmm_fp64_equiv"] = fp64_view
    line = {"metric": METRIC, "value": 1e3 / ms_step, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (station x day layout of simulate.cpp, random-feature field + nugget)",
            "config": bench_config(args, n, world),
            "nn_search_s": nn_s, "nn_search_kernel_ms": knn_ms, "nll": v, "grad": list(g),
            "e2e": {"value": 1.0 / e2e_s, "unit": "evals/s", "h2d_bytes_per_step": n * 8 + 64,
                    "d2h_bytes_per_step": 64},
            "gpu_launches": launches, "roofline": roof, "clocks": clk.summary()}
    line.update(extra)
    if args.workload == "vif":
        # the metric's Vecchia half on the same data: d_c neighbours (m_v), NLL+grad evaluations
        t0 = time.perf_counter()
        nbc = S.correlation_neighbors(ds, theta, args.m_v)
        vc_nn = time.perf_counter() - t0
        sv = S.build_vecchia(ds, theta, nbc, S.OBSERVATION)
        for i in range(args.warmup):
            S.evaluate(sv, thetas[i])
        D.barrier() if dist else None
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for i in range(args.steps):
            vv, _ = S.evaluate(sv, thetas[args.warmup + i])
        f1.record(stream)
        torch.cuda.synchronize()
        vms = D.max_over_ranks(f0.elapsed_time(f1) / args.steps)
        line["vecchia"] = {"workload": "cfg4-vecchia-dc (same data)", "evals_per_s": 1e3 / vms, "ms_per_step": vms,
                           "nn_search_s": vc_nn, "nll": vv}
        del sv, nbc
    if args.workload == "fitc" and world == 1:
        # cfg5's second half: 1-day-ahead predictive mean / variance at every station
        last = t == t.max()
        targets = np.column_stack([x[last], y[last], np.full(int(last.sum()), t.max() + 1.0)])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        S.predict(s, resp, None, None, targets)
        line["predict_first_s"] = time.perf_counter() - t0  # includes first-use module loads / pools
        t0 = time.perf_counter()
        pr = S.predict(s, resp, None, None, targets)
        line["predict_s"] = time.perf_counter() - t0
        line["predict_targets"] = int(len(targets))
        line["predict_var_range"] = [float(pr.var.min()), float(pr.var.max())]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_sample(args.workload, x, y, t, resp, theta, args.m_v,
                                          None if args.workload == "vecchia" else ind.points)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        tdist.barrier()
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
