"""Timing sweeps shaped like the paper's Tables V and VI.

  Table V: ms per AM iteration at B = 1000, obstacles
           n in {1, 5, 10, 15, 20, 25, 30} x circles m in {1, 2, 4}.
  Table VI: ms per iteration vs batch {5, 200, ..., 1000}
           (obstacles / circles unstated in the paper: C3's 3 x 30 here).
  C5       (BASELINE.json configs[4]): batch 100 ... 16384 at m = 3, n = 30.
  Ellipses (NEXT-4): the C3 scene with elliptical obstacles
           (a ~ U(0.5, 0.9), b ~ U(0.35, 0.7) m) under the literal rule (plain
           loop) and the scaled rule (culled, and with BMC_NOCULL=1 unculled).

Every point is one bmc_solve of K = 100 iterations on seeded C3-shaped dynamic
scenes (synth.make_problem), timed with CUDA events on the launching stream
(median of 10 after 3 warm-ups).  Usage (GPU box):
    python tools/sweeps.py [out.json]   -> JSON + a markdown table on stdout
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2109_13030_b200 import solver_for
from synth import CONFIGS, make_problem

# Table V of the paper (RTX 3080 Laptop, JAX), ms per iteration at B = 1000
PAPER_T5 = {1: [0.46, 0.5, 0.58, 0.76, 0.88, 1.02, 1.12],
            2: [0.8, 0.94, 1.18, 1.48, 1.8, 2.0, 2.4],
            4: [0.74, 1.22, 1.82, 2.4, 2.8, 3.6, 4.0]}
T5_N = [1, 5, 10, 15, 20, 25, 30]
# Table VI GPU column, s per iteration
PAPER_T6 = {5: 0.0016, 200: 0.0017, 400: 0.0026, 600: 0.0033, 800: 0.0039, 1000: 0.0045}


def ellipse_axes(n, seed=1000):
    rng = np.random.default_rng(seed)
    return np.stack([rng.uniform(0.5, 0.9, n), rng.uniform(0.35, 0.7, n)], 1).astype(np.float32)


def time_solve(cfg, reps=10, warm=3, alpha_rule=None):
    pr = make_problem(cfg, 0)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    kw = {}
    if alpha_rule is not None:   # ellipse scene
        pr["obs_ab"] = ellipse_axes(cfg.n)
        kw["alpha_rule"] = alpha_rule
    s = solver_for(cfg, device=0, **kw)
    args = (d(pr["init"]), d(pr["obs_xy"]), d(pr["obs_ab"]), pr["bnd"], cfg.K)
    out = s.solve(*args)
    for _ in range(warm):
        s.solve(*args, out=out)
    torch.cuda.synchronize()
    ts = []
    stream = torch.cuda.current_stream()
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.solve(*args, out=out)
        e1.record(stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    torch.cuda.set_device(0)
    base = CONFIGS["C3"]
    res = {"device": torch.cuda.get_device_name(0), "K": base.K, "table5": [], "table6": [], "c5": [],
           "ellipses": []}
    for m in (1, 2, 4):
        for idx, n in enumerate(T5_N):
            ms = time_solve(base.with_(m=m, n=n, B=1000))
            res["table5"].append({"m": m, "n": n, "ms_per_solve": ms, "ms_per_iter": ms / base.K,
                                  "paper_ms_per_iter": PAPER_T5[m][idx]})
    for B in (5, 200, 400, 600, 800, 1000):
        ms = time_solve(base.with_(B=B))
        res["table6"].append({"B": B, "ms_per_solve": ms, "s_per_iter": ms / base.K / 1e3,
                              "paper_s_per_iter": PAPER_T6[B]})
    for B in (100, 256, 1000, 2048, 4096, 8192, 16384):
        ms = time_solve(base.with_(B=B))
        res["c5"].append({"B": B, "ms_per_solve": ms, "traj_iter_per_s": B * base.K / (ms * 1e-3)})
    res["ellipses"].append({"scene": "C3 circles (reference)", "ms_per_solve": time_solve(base)})
    for rule, nocull in ((0, False), (1, False), (1, True)):
        if nocull:
            os.environ["BMC_NOCULL"] = "1"
        ms = time_solve(base, alpha_rule=rule)
        os.environ.pop("BMC_NOCULL", None)
        res["ellipses"].append({"scene": f"C3 ellipses, alpha rule {rule} ({'literal, plain loop' if rule == 0 else 'scaled'}"
                                         f"{', unculled' if nocull else (', culled' if rule else '')})",
                                "ms_per_solve": ms})
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(res, f, indent=1)
    print(f"# sweeps on {res['device']} (K = {base.K} iterations per solve, median of 10)\n")
    print("## Table V shape: ms per iteration, B = 1000 (paper: RTX 3080 Laptop, JAX)\n")
    print("| circles | " + " | ".join(f"n={n}" for n in T5_N) + " |")
    print("|---|" + "---|" * len(T5_N))
    for m in (1, 2, 4):
        row = [r for r in res["table5"] if r["m"] == m]
        print(f"| {m} (B200) | " + " | ".join(f"{r['ms_per_iter']:.4f}" for r in row) + " |")
        print(f"| {m} (paper) | " + " | ".join(f"{r['paper_ms_per_iter']:.2f}" for r in row) + " |")
    print("\n## Table VI shape: s per iteration vs batch (m = 3, n = 30)\n")
    print("| B | B200 | paper GPU |\n|---|---|---|")
    for r in res["table6"]:
        print(f"| {r['B']} | {r['s_per_iter']:.2e} | {r['paper_s_per_iter']:.1e} |")
    print("\n## C5 batch sweep (1 GPU)\n")
    print("| B | ms / solve | traj*iter/s |\n|---|---|---|")
    for r in res["c5"]:
        print(f"| {r['B']} | {r['ms_per_solve']:.3f} | {r['traj_iter_per_s']:.3e} |")
    print("\n## Ellipse scenes (NEXT-4), B = 1000, K = 100\n")
    print("| scene | ms / solve |\n|---|---|")
    for r in res["ellipses"]:
        print(f"| {r['scene']} | {r['ms_per_solve']:.3f} |")


if __name__ == "__main__":
    main()
