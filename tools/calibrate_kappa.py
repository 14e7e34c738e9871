"""Calibrate tests/parity.py KAPPA on the oracle alone (no GPU, no CUDA path).

For each calibration instance, the fp32 rounding model of the oracle is run
with the harness's N_MODEL seeds (the "spread" the harness measures) and with
N_PROBE further seeds, each probe standing in for another fp32 implementation.
Wherever a probe misses the parity bar against the fp64 oracle, the ratio
probe deviation / spread is recorded; KAPPA must cover every such ratio.

usage: python tools/calibrate_kappa.py [out.json]   (about 15 min on 8 cores)
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Oracle  # noqa: E402
from synth import CONFIGS, make_problem  # noqa: E402
from tests.helpers import bpoly_basis, oracle_params  # noqa: E402
from tests.parity import MODEL_SEED0, N_MODEL, bars, deviations, fp32_spread  # noqa: E402

N_PROBE = 4
CASES = [("C3", 0, 1000), ("C3", 1, 1000), ("C4", 0, 250), ("C2", 0, 100)]


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "profiles/kappa_calibration.json"
    rep = dict(n_model=N_MODEL, n_probe=N_PROBE, cases=[], ratios=[])
    for name, seed, B in CASES:
        t0 = time.time()
        cfg = CONFIGS[name]
        pr = make_problem(cfg, seed, B=B)
        o = Oracle(oracle_params(cfg), cfg.n)
        ref = o.solve(pr["bnd"], pr["obs_xy"], pr["obs_ab"], pr["init"], cfg.K)
        P, _, _ = bpoly_basis(cfg.q, cfg.T, cfg.degree)
        rows = np.arange(B)
        spread = fp32_spread(o, pr, rows, cfg.K, ref, P=P)
        bar = bars(cfg, ref, cfg.K)
        n_fail, worst = 0, 0.0
        for p in range(N_PROBE):
            s = MODEL_SEED0 + N_MODEL + p
            probe = fp32_spread(o, pr, rows, cfg.K, ref, P=P, seeds=[s])
            for k in probe:
                f = np.flatnonzero(probe[k] > bar[k])
                n_fail += len(f)
                for i in f:
                    r = float(probe[k][i] / max(spread[k][i], 1e-300))
                    worst = max(worst, r)
                    rep["ratios"].append(dict(case=f"{name} seed {seed}", inst=int(i), q=k, probe_seed=s,
                                              dev=float(probe[k][i]), spread=float(spread[k][i]), ratio=r))
        rep["cases"].append(dict(case=f"{name} seed {seed} B {B}", probe_bar_misses=n_fail, worst_ratio=worst,
                                 seconds=round(time.time() - t0, 1)))
        print(rep["cases"][-1], flush=True)
    rs = np.array([r["ratio"] for r in rep["ratios"]]) if rep["ratios"] else np.zeros(1)
    rep["summary"] = dict(n=len(rep["ratios"]), max=float(rs.max()), p99=float(np.quantile(rs, 0.99)),
                          p90=float(np.quantile(rs, 0.9)), median=float(np.median(rs)))
    print(rep["summary"])
    with open(out, "w") as f:
        json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
