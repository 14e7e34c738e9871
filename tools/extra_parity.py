"""One-off full-batch parity beyond the suite (dev aid, GPU): C3 seeds 5-9 and C4 seeds
2-4 through the test functions of tests/test_gpu_parity.py."""
import sys, time
sys.path.insert(0, ".")
import torch
import __graft_entry__
__graft_entry__.build()
torch.cuda.set_device(0)
from tests import test_gpu_parity as T
for seed in range(5, 10):
    t = time.time()
    try:
        T.test_c3_full_batch_every_instance(seed); print("C3 seed", seed, "PASS", round(time.time() - t, 1), flush=True)
    except AssertionError as e:
        print("C3 seed", seed, "FAIL", str(e)[:400], flush=True)
for seed in range(2, 5):
    t = time.time()
    try:
        T.test_c4_full_batch_every_instance(seed); print("C4 seed", seed, "PASS", round(time.time() - t, 1), flush=True)
    except AssertionError as e:
        print("C4 seed", seed, "FAIL", str(e)[:400], flush=True)
