#!/usr/bin/env python3
"""Benchmark of the batched AM iteration (arXiv 2109.13030) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

A step is one whole batch solve: BASELINE configuration C3 per GPU (batch 1000,
horizon 100, 3 circles, 30 dynamic obstacles, 100 AM iterations, seeded
synthetic scene), i.e. every row of the hot path (xi1, xi2, xi3, xi4, lambda,
residual, cost, argmin) plus, for N > 1, the best-of-batch exchange over NCCL.
Weak scaling: every rank solves its own 1000-instance shard of an N*1000 batch.

`value` = trajectories*iterations per second over all ranks, from CUDA events
around each step on the launching stream (max over ranks); L2 is flushed
(256 MiB memset) between steps, outside the events.  `e2e` measures the same
through the host-buffer C-ABI call (bmc_solve_host: pinned H2D of the inputs,
kernel, D2H of every output, synchronise).  `roofline` reports the fused
kernel against the FP32 issue peak; `cpu_baseline` is
the fp64 oracle timed on a bounded sample on this host.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CONFIGS, make_problem  # noqa: E402


def algorithmic_fp32_ops(q: int, m: int, n: int) -> float:
    """FP32 lane-instructions per (instance, iteration) of the method as formulated
    (DESIGN.md "Roofline"): per sample t, evaluation of x, y, psi, c, s and the
    first/second derivatives (9 x 11 FMA), the F^T(F xi - g) and P^T theta
    contractions (9 x 11 FMA), the velocity/acceleration projections and
    per-sample bookkeeping (20 + 6 m), and per (circle, obstacle) the
    branch-free closed-form projection with its two accumulations (8)."""
    return float(q) * (99 + 99 + 20 + 6 * m + 8 * m * n)


def fp32_peak(sm_mhz: float, sms: int = 148) -> float:
    return sms * 128 * sm_mhz * 1e6   # lane-instructions per second


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML polled every
    0.5 ms from a thread (a C3 region is ~10 ms), and nvidia-smi (100 ms period) as
    the fallback when NVML is unavailable or saw fewer than 3 samples."""

    NVML_PERIOD_S = 5e-4

    def __init__(self, gpus):
        self.gpus = gpus
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        self.nv = []            # (sm_mhz, reasons bitmask) from NVML
        self.nv_max = None
        self._stop = None
        self._thread = None

    def _nvml_start(self):
        import threading
        import pynvml
        import torch
        pynvml.nvmlInit()
        h = None
        try:   # the CUDA device's own NVML handle (CUDA_VISIBLE_DEVICES may renumber)
            uuid = str(torch.cuda.get_device_properties(self.gpus[0]).uuid)
            h = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpus[0])
        self.nv_max = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    self.nv.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)), int(reasons_fn(h))))
                except Exception:
                    return
                time.sleep(self.NVML_PERIOD_S)

        self._thread = threading.Thread(target=run, daemon=True)
        self._thread.start()

    def __enter__(self):
        try:
            self._nvml_start()
        except Exception:
            self._thread = None
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", ",".join(str(g) for g in self.gpus),
                 "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=5)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if len(self.nv) >= 3:
            import pynvml
            bits = {"hw_slowdown": pynvml.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksThrottleReasonSwPowerCap}
            reasons = sorted(nm for nm, b in bits.items() if any(r & b for _, r in self.nv))
            return {"sm_mhz": statistics.median(v for v, _ in self.nv), "sm_max_mhz": self.nv_max,
                    "reasons": reasons, "samples": len(self.nv), "sampler": "nvml, 0.5 ms"}
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(cfg, pr, sample: int, iters: int, sample_1t: int = 0):
    """The fp64 oracle, as it stands, on this host's cores (bounded sample), and
    with sample_1t > 0 also on one core (all cores and 1 core)."""
    from oracle import Oracle, OracleParams
    o = Oracle(OracleParams(q=cfg.q, T=cfg.T, degree=cfg.degree, r=cfg.offsets, v_max=cfg.v_max,
                            a_max=cfg.a_max, rho=cfg.rho, rho_psi=cfg.rho_psi, res_tol=cfg.res_tol), cfg.n)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"][:sample], iters, nthreads=cores)
    dt = time.perf_counter() - t0
    cb = dict(value=sample * iters / dt, unit="trajectories*iterations/s", cores=cores, kind="oracle",
              sample=f"{sample} instances x {iters} iterations of the {cfg.name} scene "
                     f"(fp64 C oracle, OpenMP over instances), {dt:.2f} s wall")
    if sample_1t > 0:
        t0 = time.perf_counter()
        o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"][:sample_1t], iters, nthreads=1)
        dt1 = time.perf_counter() - t0
        cb["one_core"] = dict(value=sample_1t * iters / dt1, unit="trajectories*iterations/s", cores=1,
                              sample=f"{sample_1t} instances x {iters} iterations, {dt1:.2f} s wall")
    return cb


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on the host cores."""
    if rank != 0:
        return
    pr = make_problem(cfg, 0)
    sample = args.ref_sample
    for _ in range(args.warmup):
        cpu_baseline(cfg, pr, max(1, sample // 4), cfg.K)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cb = cpu_baseline(cfg, pr, sample, cfg.K)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = args.steps * sample * cfg.K / tot
    line = dict(impl="reference", metric=metric_name(cfg), value=value, unit="trajectories*iterations/s",
                n_gpus=world, steps=args.steps, warmup=args.warmup,
                ms_per_step=1e3 * tot / args.steps, higher_is_better=True, scaling="weak", vs_baseline=None,
                dtype="f64", data="synthetic",
                config=workload(cfg, world) | {"reference_sample_instances": sample},
                cpu_baseline=dict(kind="oracle", cores=cb["cores"], sample=cb["sample"], value=value,
                                  unit="trajectories*iterations/s"),
                e2e=dict(value=value, unit="trajectories*iterations/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


def metric_name(cfg) -> str:
    return f"trajectories*iterations/s (batch solve: {cfg.B} instances/GPU x {cfg.K} AM iterations)"


def run_mpc(args, cfg):
    """NEXT-1: MPC ticks (fresh STOMP samples drawn on the device (NEXT-2), receding obstacles,
    warm-started lambda on the device, one K = 10 solve, D2H of the best trajectory, host state
    update) per second."""
    import torch
    from paper_2109_13030_b200.mpc import MPC, GpuBackend, MPCConfig
    from synth import make_tracks
    torch.cuda.set_device(0)
    mc = MPCConfig(cfg, horizon=10.0, dt=0.1, K=10, seed=0)
    m = MPC(mc, make_tracks(cfg, 0), GpuBackend(mc), B=cfg.B)
    for _ in range(args.warmup):
        m.tick()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        m.tick()
    wall = time.perf_counter() - t0
    solve_ms = [r.solve_ms for r in m.log[args.warmup:]]
    line = dict(metric=f"MPC control ticks/s (batch {cfg.B}, K = {mc.K} AM iterations per tick, horizon "
                       f"{mc.horizon:g} s)", value=args.steps / wall, unit="ticks/s", n_gpus=1, steps=args.steps,
                warmup=args.warmup, ms_per_step=1e3 * wall / args.steps, higher_is_better=True, scaling="weak",
                vs_baseline=None, dtype="f32 (fp64 KKT steps)", data="synthetic",
                config={"workload": f"NEXT-1 MPC on the {cfg.name} scene: {cfg.n} dynamic obstacles, {cfg.m} circles, "
                                    f"q = {cfg.q}, tick {mc.dt} s",
                        "paper_budget_s_per_tick": 0.04},
                solve_ms_per_tick={"mean": float(np.mean(solve_ms)), "max": float(np.max(solve_ms))},
                gpu_launches=2 * args.steps,   # bmc_sample_init + bmc_solve per tick
                e2e={"value": args.steps / wall, "unit": "ticks/s",
                     "h2d_bytes_per_step": int(cfg.n * 2 * cfg.q * 4 + cfg.n * 8),   # samples drawn on the device
                     "d2h_bytes_per_step": int(55 * 4 + 8 + 4 + 8)},
                robot={"t": m.t, "x": float(m.state[0, 0]), "y": float(m.state[1, 0])})
    print(json.dumps(line), flush=True)


def workload(cfg, world, global_batch=None):
    gb = cfg.B * world if global_batch is None else global_batch
    per = cfg.B if global_batch is None else -(-global_batch // world)
    kind = "batch {}/GPU".format(per) if global_batch is None else "batch {} split over {} GPU(s)".format(gb, world)
    return {"workload": f"{cfg.name}: {kind}, horizon {cfg.q}, {cfg.m} circles, {cfg.n} "
                        f"{'dynamic' if cfg.dynamic else 'static'} obstacles, {cfg.K} AM iterations",
            "batch_per_gpu": per, "global_batch": gb, "q": cfg.q, "m": cfg.m, "n_obs": cfg.n,
            "iters": cfg.K, "l2": "flushed between steps (256 MiB memset, outside the timed events)"}


def required_work(cfg):
    """Required-work accounting from the PROFILE build's count of the (round, obstacle)
    pairs the culled collision loop actually evaluates (profiles/required_work.json,
    tools/required_work.py): the fixed per-sample work plus 32 lanes x m circles x 8 FP32
    instructions per evaluated pair, per instance-iteration."""
    path = os.path.join(ROOT, "profiles", "required_work.json")
    try:
        rw = json.load(open(path)).get(cfg.name)
    except Exception:
        return None
    if not rw or rw.get("q") != cfg.q or rw.get("m") != cfg.m or rw.get("n") != cfg.n:
        return None
    return float(cfg.q) * (99 + 99 + 20 + 6 * cfg.m) + rw["evaluated_pairs_per_instance_iter"] * 32 * 8 * cfg.m, rw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--batch", type=int, default=None, help="override instances per GPU")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=16)
    ap.add_argument("--cpu-sample", type=int, default=960,
                    help="oracle instances for cpu_baseline (about 10-30 s on a 16-core host)")
    ap.add_argument("--cpu-sample-1t", type=int, default=32,
                    help="oracle instances for the one-core cpu_baseline column (about 5-10 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mpc", action="store_true",
                    help="NEXT-1: time the receding-horizon MPC tick (P:585) instead of the C3 batch solve")
    ap.add_argument("--ellipse", type=int, default=None, choices=[0, 1],
                    help="NEXT-4: the same scene with elliptical obstacles under alpha rule 0 (literal) or 1 (scaled)")
    ap.add_argument("--team-of-batch", action="store_true",
                    help="run every shard with the team size of the whole batch (bitwise the one-GPU solve)")
    ap.add_argument("--strong", type=int, default=0, metavar="B",
                    help="strong scaling: one global batch of B instances split over the GPUs (e.g. 16384, C5)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus == 1 else 1)))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    if args.batch:
        cfg = cfg.with_(B=args.batch)
    global_batch = None
    if args.strong:   # total work fixed: rank r solves instances [r per, (r+1) per) of args.strong
        global_batch = args.strong
        cfg = cfg.with_(B=-(-args.strong // world))

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    if args.mpc:
        run_mpc(args, cfg)
        return

    import torch
    from paper_2109_13030_b200 import solver_for
    from paper_2109_13030_b200.distributed import BestExchange, solve_sharded, solve_sharded_host

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    # every rank builds the same scene from the seed; rank r owns instances [r B, (r+1) B)
    n_glob = cfg.B * world if global_batch is None else global_batch
    glob = make_problem(cfg, 0, B=n_glob)
    skw = {}
    if args.ellipse is not None:   # NEXT-4: seeded semi-axes, the chosen alpha rule
        rng = np.random.default_rng(1000)
        glob["obs_ab"] = np.stack([rng.uniform(0.5, 0.9, cfg.n), rng.uniform(0.35, 0.7, cfg.n)], 1).astype(np.float32)
        skw["alpha_rule"] = args.ellipse
    shard = slice(min(rank * cfg.B, n_glob), min((rank + 1) * cfg.B, n_glob))
    init_h = np.ascontiguousarray(glob["init"][shard])
    B_rank = init_h.shape[0]
    assert B_rank > 0, "every rank needs a non-empty shard to time"
    init = torch.from_numpy(init_h).to(dev)
    obs = torch.from_numpy(glob["obs_xy"]).to(dev)
    ab = torch.from_numpy(glob["obs_ab"]).to(dev)
    solver = solver_for(cfg, device=local, **skw)
    # team size (warps per instance): the one this shard's size selects, as each GPU
    # would run it alone (`--team-of-batch`: the whole batch's, which makes every
    # instance bitwise the one-GPU solve's at the cost of a smaller team per shard)
    team = solver.team_for(n_glob) if args.team_of_batch else solver.team_for(B_rank)
    xchg = BestExchange(pg, dev) if world > 1 else None
    out = solver.solve(init, obs, ab, glob["bnd"], cfg.K, index_base=rank * cfg.B, team=team)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        solve_sharded(solver, xchg, init, obs, ab, glob["bnd"], cfg.K, rank * cfg.B, out=out, team=team)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    if pg is not None:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler([local]) as clk:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.zero_()
            ev[i][0].record(stream)
            kev[i][0].record(stream)
            solver.solve(init, obs, ab, glob["bnd"], cfg.K, index_base=rank * cfg.B, out=out, team=team)
            launches += solver.last_launches
            kev[i][1].record(stream)
            if xchg is not None:
                xchg.exchange(out["best"], out["coeffs"], rank * cfg.B)
                launches += 2   # bmc_pack_best + bmc_select_best (the all-gather is NCCL's)
            ev[i][1].record(stream)   # solve + exchange = solve_sharded (kernel timed separately by kev)
        torch.cuda.synchronize(dev)
        if pg is not None:
            torch.distributed.barrier()
        wall = time.perf_counter() - wall0
    clocks = clk.summary()
    if not clocks.get("sm_mhz") or clocks.get("samples", 0) < 3:
        # the timed region was shorter than the sampling period: sample the same
        # step in a 1.5 s soak right after it (reported as clock_window "soak")
        with ClockSampler([local]) as clk2:
            t_end = time.perf_counter() + 1.5
            while time.perf_counter() < t_end:   # kernel only: no collective in the soak
                for _ in range(20):
                    solver.solve(init, obs, ab, glob["bnd"], cfg.K, index_base=rank * cfg.B, out=out, team=team)
                torch.cuda.synchronize(dev)
        clocks = clk2.summary()
        clocks["clock_window"] = "soak (same step, 1.5 s, right after the timed region)"
    else:
        clocks["clock_window"] = "timed region"
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    t_dev = sum(step_ms) / 1e3
    if pg is not None:
        tt = torch.tensor([t_dev, sum(kern_ms) / 1e3], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_dev, t_kern = float(tt[0]), float(tt[1])
    else:
        t_kern = sum(kern_ms) / 1e3
    value = n_glob * cfg.K * args.steps / t_dev

    # ---- end to end through the host-buffer C-ABI (bmc_solve_host) ------------
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
    h_init, h_obs, h_ab = pin(init_h), pin(glob["obs_xy"]), pin(glob["obs_ab"])
    B = B_rank
    h_out = dict(coeffs=pin(np.empty((B, 5, 11), np.float32)), lambda_out=pin(np.empty((B, 5, 11), np.float32)),
                 residual=pin(np.empty((B, 2), np.float32)), cost=pin(np.empty((B,), np.float32)),
                 best=pin(np.empty((2,), np.int64)))
    # the user's call: the shard's solve from host buffers plus, for N > 1, the
    # best-of-batch exchange and the read-back of the global best (16 B + 220 B)
    g_best, g_coeffs = pin(np.empty(2, np.int64)), pin(np.empty(55, np.float32))

    def e2e_step():
        solve_sharded_host(solver, xchg, h_init, h_obs, h_ab, glob["bnd"], cfg.K, rank * cfg.B, out=h_out,
                           best_host=g_best, coeffs_host=g_coeffs, team=team)

    for _ in range(args.warmup):
        e2e_step()
    if pg is not None:
        torch.distributed.barrier()
    e2e_t = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        e2e_step()
        e2e_t.append(time.perf_counter() - t0)
    t_e2e = sum(e2e_t)
    if pg is not None:
        tt = torch.tensor([t_e2e], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(tt[0])
    e2e_value = n_glob * cfg.K * args.steps / t_e2e
    h2d = h_init.nbytes + h_obs.nbytes + h_ab.nbytes
    d2h = sum(v.nbytes for v in h_out.values()) + (g_best.nbytes + g_coeffs.nbytes if world > 1 else 0)

    if rank != 0:
        if pg is not None:
            torch.distributed.destroy_process_group()
        return
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    ops = algorithmic_fp32_ops(cfg.q, cfg.m, cfg.n) * B_rank * cfg.K      # per launch (rank 0's shard)
    kern_avg = t_kern / args.steps
    achieved = ops / kern_avg
    peak = fp32_peak(sm_max)
    roof = dict(bound="alu", achieved=achieved / 1e12, peak=peak / 1e12,
                unit="T FP32 lane-instr/s", frac=achieved / peak, traffic=None,
                kernel=f"bmc_am_kernel<{cfg.m}>", algorithmic_ops_per_launch=ops,
                kernel_ms=1e3 * kern_avg,
                peak_basis=f"148 SM x 128 FP32 lanes x {sm_max:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json)")
    if clocks.get("sm_mhz"):
        roof["frac_at_observed_clock"] = achieved / fp32_peak(clocks["sm_mhz"])
    # DRAM bytes per launch and issue activity of the current kernel: one ncu --set full
    # capture of this bench's launch (profiles/dram_traffic.json, written by tools/ncu_summary.py)
    traffic_file = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(traffic_file) and global_batch is None:
        try:
            tj = json.load(open(traffic_file))
            roof["traffic"] = tj.get(f"{cfg.name}_bytes_per_launch")
            roof["traffic_source"] = tj.get("source")
            if tj.get(f"{cfg.name}_issue_active_pct") is not None:
                roof["issue_active_pct"] = tj[f"{cfg.name}_issue_active_pct"]
        except Exception:
            pass
    rw = required_work(cfg)
    if rw is not None:   # the work the culled kernel must do, next to the method's algorithmic count
        req_ops = rw[0] * B_rank * cfg.K
        roof["required_ops_per_launch"] = req_ops
        roof["required_frac"] = req_ops / kern_avg / peak
        roof["required_basis"] = rw[1].get("source")
    line = dict(metric=metric_name(cfg), value=value, unit="trajectories*iterations/s", n_gpus=world, steps=args.steps,
                warmup=args.warmup, ms_per_step=1e3 * t_dev / args.steps, higher_is_better=True,
                scaling="weak" if global_batch is None else "strong", vs_baseline=None,
                dtype="f32 (fp64 KKT steps)", data="synthetic",
                config=workload(cfg, world, global_batch) | {"team": team} |
                ({"obstacles": f"ellipses a~U(0.5,0.9) b~U(0.35,0.7), alpha rule {args.ellipse}"}
                 if args.ellipse is not None else {}), clocks=clocks, gpu_launches=launches,
                e2e=dict(value=e2e_value, unit="trajectories*iterations/s", h2d_bytes_per_step=int(h2d),
                         d2h_bytes_per_step=int(d2h), ms_per_step=1e3 * t_e2e / args.steps),
                roofline=roof, wall_s=wall)
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(cfg, glob, min(args.cpu_sample, n_glob), cfg.K,
                                            sample_1t=min(args.cpu_sample_1t, n_glob))
    print(json.dumps(line), flush=True)
    if pg is not None:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
