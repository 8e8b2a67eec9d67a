"""One-off randomized parity fuzz over 400 more seeds of tests/test_gpu_parity.py::test_randomized_configs (GPU box)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
os.chdir(ROOT)
import numpy as np, torch
import test_gpu_parity as T
from oracle import oracle as O
O.build()
cuda = torch.device('cuda', 0)
fails = 0
for seed in range(1000, 1400):
    try:
        T.test_randomized_configs.__wrapped__(seed, O, cuda) if hasattr(T.test_randomized_configs, '__wrapped__') else T.test_randomized_configs(seed, O, cuda)
    except Exception as e:
        fails += 1
        print('FAIL seed', seed, repr(e)[:300], flush=True)
print('fuzz done, failures:', fails)
