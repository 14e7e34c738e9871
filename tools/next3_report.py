"""NEXT-3 report (dev aid, GPU): homotopy split around a blocker and the multi- vs
single-circle arc length at a 1.2 m gap, B = 1000, K = 100.  Writes profiles/<name>.md."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import CONFIGS, make_init, scene_blocker, scene_wall_gap  # noqa: E402
from tests.test_gpu_homotopy import geometry, solve, y_at_x  # noqa: E402

torch.cuda.set_device(0)
name = sys.argv[1] if len(sys.argv) > 1 else "r1_next3_homotopy"
lines = [f"# NEXT-3 quality checks ({name})", "", "B = 1000 STOMP samples (s_y = 5 m), K = 100, q = 100, T = 30 s, "
         "solved by libbmc.so on one B200.", ""]
sc = scene_blocker(100)
cfg = CONFIGS["C3"].with_(name="blocker", n=1)
g = solve(cfg, sc, make_init(cfg, seed=6, B=1000, sigma_y=5.0))
X, Y, arc = geometry(cfg, g["coeffs"])
feas = g["residual"][:, 0] <= cfg.res_tol
side = np.sign(y_at_x(X, Y, 15.0))
lines += ["## Blocker on the line (Fig. 1c)", "",
          f"feasible {int(feas.sum())} / 1000; above {int(np.sum(feas & (side > 0)))}, "
          f"below {int(np.sum(feas & (side < 0)))}; best index {int(g['best'][0])} "
          f"(arc {arc[int(g['best'][0])]:.2f} m)", ""]
lines += ["## Wall with a 1.2 m gap (Table II trend)", "", "| footprint | feasible | best arc [m] | y at the wall [m] | best cost |",
          "|---|---|---|---|---|"]
for m, inflate, lab in ((3, 0.3, "3 circles r 0.3"), (1, 0.8, "1 disk r 0.8")):
    sc = scene_wall_gap(100, inflate=inflate)
    cfg = CONFIGS["C3"].with_(name="wall", m=m, n=sc["obs_xy"].shape[0])
    g = solve(cfg, sc, make_init(cfg, seed=5, B=1000, sigma_y=5.0))
    X, Y, arc = geometry(cfg, g["coeffs"])
    feas = g["residual"][:, 0] <= cfg.res_tol
    b = int(g["best"][0])
    lines.append(f"| {lab} | {int(feas.sum())} | {arc[b]:.3f} | {y_at_x(X, Y, 15.0)[b]:+.2f} | {g['cost'][b]:.4f} |")
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", name + ".md")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
