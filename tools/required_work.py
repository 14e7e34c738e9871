"""Required-work accounting for bench.py's roofline (run on a GPU box).

The culled collision loop (bmc_kernel.cuh coll_circ) evaluates only the
(round of 32 samples, obstacle) pairs whose clearance stamp no longer covers
the movement since it was stamped.  The PROFILE build counts them per warp
(slot "tested"); this script runs that build on a configuration and writes the
count per instance-iteration to profiles/required_work.json, which bench.py
turns into `roofline.required_frac`: the fixed per-sample work of the method
plus 32 lanes x m circles x 8 FP32 instructions per evaluated pair.

usage: python tools/required_work.py [C3 C4 ...]   (needs libbmc_prof.so:
       make -C paper_2109_13030_b200/csrc PROFILE=1)
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from synth import CONFIGS  # noqa: E402


def main():
    names = sys.argv[1:] or ["C3", "C4"]
    path = os.path.join(ROOT, "profiles", "required_work.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for name in names:
        env = dict(os.environ, BMC_PROF="1", BMC_LIB=os.path.join(ROOT, "paper_2109_13030_b200", "libbmc_prof.so"))
        p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "timecfg.py"), name], env=env,
                           capture_output=True, text=True, timeout=600)
        roles = {}
        for line in p.stderr.splitlines():
            m = re.search(r"warp-role (\d+) cycles/iter:.* tested=([0-9.]+)", line)
            if m:
                roles[int(m.group(1))] = float(m.group(2))   # the last solve's value wins
        if not roles:
            print(name, "no PROFILE output:", p.stderr[-500:])
            continue
        cfg = CONFIGS[name]
        pairs = sum(roles.values())
        out[name] = dict(q=cfg.q, m=cfg.m, n=cfg.n, evaluated_pairs_per_instance_iter=pairs,
                         pairs_total_per_instance_iter=((cfg.q + 31) // 32) * cfg.n,
                         source=f"PROFILE build (tools/required_work.py), {name} seed 0, per-warp 'tested' "
                                f"counts summed over the team's ranks")
        print(name, out[name])
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
