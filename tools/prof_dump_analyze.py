"""Per-team imbalance between the two ranks of a team (dev aid): PROFILE build,
BMC_PROF_DUMP=file tools/prof_c.sh; python tools/prof_dump_analyze.py file"""
import numpy as np, sys
a = np.loadtxt(sys.argv[1])
loop = a[:, 1]; d1a, ta, d1b, tb = a[:, 3], a[:, 4], a[:, 5], a[:, 6]
imb = np.abs(d1a - d1b)
o = np.argsort(loop)
print("teams", len(a), "loop mean %.0f p90 %.0f max %.0f" % (loop.mean(), np.percentile(loop, 90), loop.max()))
print("D1 rank0 mean %.0f rank1 mean %.0f; |imbalance| mean %.0f p90 %.0f" % (d1a.mean(), d1b.mean(), imb.mean(), np.percentile(imb, 90)))
top = o[-50:]
print("slowest 50 teams: loop %.0f, D1 r0 %.0f r1 %.0f, |imb| %.0f, tested r0 %.1f r1 %.1f" % (loop[top].mean(), d1a[top].mean(), d1b[top].mean(), imb[top].mean(), ta[top].mean()/101, tb[top].mean()/101))
print("corr(loop, max D1) %.2f" % np.corrcoef(loop, np.maximum(d1a, d1b))[0, 1])
