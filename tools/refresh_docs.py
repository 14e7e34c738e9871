"""Refresh the measured numbers in profiles/README.md, DESIGN.md §10 and README.md from
the bench lines of one round session (dev aid): python tools/refresh_docs.py vNN"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
v = sys.argv[1]
J = lambda f: json.load(open(os.path.join(ROOT, "profiles", f)))
c3, c4 = J(f"r2_c3_{v}_bench.json"), J(f"r2_c4_{v}_bench.json")
c5, ell = J(f"r2_c5_strong16384_{v}_bench.json"), J(f"r2_c3_ellipses_rule1_{v}_bench.json")
dram = json.load(open(os.path.join(ROOT, "profiles", "dram_traffic.json")))
r3 = c3["roofline"]

p = os.path.join(ROOT, "profiles", "README.md")
s = open(p).read()
s = re.sub(r"r2_(c3|c4|c5_strong16384|c3_ellipses_rule1|sweeps)_v\d+", lambda m: f"r2_{m.group(1)}_{v}", s)
s = re.sub(r"\| `r2_c3_%s_bench.json` \|.*\n" % v,
           f"| `r2_c3_{v}_bench.json` | bench.py line (C3): {c3['ms_per_step']:.3f} ms/step (kernel {r3['kernel_ms']:.3f}), "
           f"{c3['value']:.3g} traj*iter/s, e2e {c3['e2e']['ms_per_step']:.3f} ms ({c3['e2e']['value']:.3g}), roofline frac "
           f"{r3['frac']:.3f}, required-work fraction {r3['required_frac']:.3f}, fp64 oracle {c3['cpu_baseline']['value']:.3g} "
           f"traj*iter/s on {c3['cpu_baseline']['cores']} cores and {c3['cpu_baseline']['one_core']['value']:.0f} on one |\n", s)
s = re.sub(r"\| `r2_c4_%s_bench.json` \|.*\n" % v,
           f"| `r2_c4_{v}_bench.json` | C4: {c4['ms_per_step']:.3f} ms ({c4['value']:.3g}), frac {c4['roofline']['frac']:.2f}, "
           f"required {c4['roofline']['required_frac']:.2f} |\n", s)
s = re.sub(r"\| `r2_c5_strong16384_%s_bench.json` \|.*\n" % v,
           f"| `r2_c5_strong16384_{v}_bench.json` | `--strong 16384` at N = 1 (C5's largest batch, one warp per instance): "
           f"{c5['ms_per_step']:.2f} ms, {c5['value']:.3g}, frac {c5['roofline']['frac']:.2f} |\n", s)
s = re.sub(r"\| `r2_c3_ellipses_rule1_%s_bench.json` \|.*\n" % v,
           f"| `r2_c3_ellipses_rule1_{v}_bench.json` | `--ellipse 1` (NEXT-4, scaled-rule ellipses, culled): "
           f"{ell['ms_per_step']:.3f} ms |\n", s)
s = re.sub(r"Round 2's kernel is \*\*v\d+\*\*", f"Round 2's kernel is **{v}**", s)
s = re.sub(r"from the v\d+ capture", f"from the {v} capture", s)
open(p, "w").write(s)

p = os.path.join(ROOT, "DESIGN.md")
s = open(p).read()
s = re.sub(r"r2_(c3|c4|c5_strong16384|c3_ellipses_rule1|sweeps)_v\d+", lambda m: f"r2_{m.group(1)}_{v}", s)
s = re.sub(r"\| C3 \(B 1000, m 3, n 30, K 100\) \|.*\n",
           f"| C3 (B 1000, m 3, n 30, K 100) | {c3['ms_per_step']:.3f} | {c3['value']:.3g} | {r3['frac']:.3f} | {r3['required_frac']:.3f} |\n", s)
s = re.sub(r"\| C4 \(B 1000, m 4, n 50, K 200\) \|.*\n",
           f"| C4 (B 1000, m 4, n 50, K 200) | {c4['ms_per_step']:.3f} | {c4['value']:.3g} | {c4['roofline']['frac']:.2f} | "
           f"{c4['roofline']['required_frac']:.2f} |\n", s)
s = re.sub(r"\| C5 B 16384 \(`--strong 16384`, N = 1\) \|.*\n",
           f"| C5 B 16384 (`--strong 16384`, N = 1) | {c5['ms_per_step']:.2f} | {c5['value']:.3g} | {c5['roofline']['frac']:.2f} | "
           f"{c5['roofline']['required_frac']:.2f} |\n", s)
s = re.sub(r"\| C3 scene, scaled-rule ellipses \(`--ellipse 1`\) \|.*\n",
           f"| C3 scene, scaled-rule ellipses (`--ellipse 1`) | {ell['ms_per_step']:.3f} | {ell['value']:.3g} | | |\n", s)
s = re.sub(r"Round 2 \(`profiles/r2_c3_v\d+_bench.json`\): value [^\n]*\n[^\n]*\n[^\n]*\n[^\n]*\n",
           f"Round 2 (`profiles/r2_c3_{v}_bench.json`): value {c3['value']:.3g} ({c3['ms_per_step']:.3f} ms per step,\n"
           f"kernel {r3['kernel_ms']:.3f} ms), e2e {c3['e2e']['value']:.3g} ({c3['e2e']['ms_per_step']:.3f} ms, pinned host buffers through\n"
           f"`bmc_solve_host`), roofline fraction {r3['frac']:.3f} (round 1: 0.446); the fp64 oracle\n"
           f"on the box's {c3['cpu_baseline']['cores']} host cores {c3['cpu_baseline']['value']:.2g} traj·iter/s, on one core "
           f"{c3['cpu_baseline']['one_core']['value']:.0f} (SURVEY §8d asks\n", s)
s = re.sub(r"C3 0\.\d+ ms \(fraction 0\.\d+ algorithmic, 0\.\d+ required; round 1 0\.446\)[^|]*\|",
           f"C3 {c3['ms_per_step']:.3f} ms (fraction {r3['frac']:.3f} algorithmic, {r3['required_frac']:.3f} required; round 1 0.446) |", s)
s = re.sub(r"\*\*0\.\d+ of the FP32 peak\*\* at 0\.\d+ ms", f"**{r3['required_frac']:.3f} of the FP32 peak** at {r3['kernel_ms']:.3f} ms", s)
s = re.sub(r"issue activity of the same launch \(`roofline.issue_active_pct`, \d+ %\)",
           f"issue activity of the same launch (`roofline.issue_active_pct`, {dram.get('C3_issue_active_pct', 0):.0f} %)", s)
open(p, "w").write(s)

p = os.path.join(ROOT, "README.md")
s = open(p).read()
s = re.sub(r"\| C3: B = 1000, q = 100, 3 circles, 30 dynamic obstacles, 100 iterations \|.*\n",
           f"| C3: B = 1000, q = 100, 3 circles, 30 dynamic obstacles, 100 iterations | {c3['ms_per_step']:.3f} ms per solve "
           f"({c3['e2e']['ms_per_step']:.3f} ms end to end from host buffers) | {c3['value']:.3g} trajectory-iterations/s "
           f"({c3['e2e']['value']:.3g} end to end) |\n", s)
s = re.sub(r"\| C4: B = 1000, 4 circles.*\n",
           f"| C4: B = 1000, 4 circles, 50 obstacles, tight bounds, 200 iterations | {c4['ms_per_step']:.2f} ms | {c4['value']:.3g} |\n", s)
s = re.sub(r"\| C5: B = 16384 \|.*\n", f"| C5: B = 16384 | {c5['ms_per_step']:.2f} ms | {c5['value']:.3g} |\n", s)
s = re.sub(r"\| C3 scene with elliptical obstacles.*\n",
           f"| C3 scene with elliptical obstacles, scaled alpha rule (culled) | {ell['ms_per_step']:.2f} ms | {ell['value']:.3g} |\n", s)
s = re.sub(r"The fp64 oracle on the same box does .*\n",
           f"The fp64 oracle on the same box does {c3['cpu_baseline']['value']:.2g} trajectory-iterations/s on "
           f"{c3['cpu_baseline']['cores']} host cores and {c3['cpu_baseline']['one_core']['value']:.0f} on one.\n", s)
s = re.sub(r"\(0\.\d+ of the FP32 peak as the method counts work, 0\.\d+ as the culled kernel must do it\)",
           f"({r3['frac']:.3f} of the FP32 peak as the method counts work, {r3['required_frac']:.3f} as the culled kernel must do it)", s)
open(p, "w").write(s)
print("C3", c3["ms_per_step"], r3["frac"])
