import sys
sys.path.insert(0, '/root/repo')
if sys.argv[1] == 'torch':
    import torch
    torch.zeros(1, device='cuda')
import numpy as np
import paper_2007_03576_b200 as hq
from hqr_inputs import random_case
hq.setup(0, flags=3)
H0, Z0, re, im = random_case(1, 256, 8)
try:
    hq.sweep(H0, Z0, 0, 255, re, im, 24)
    print('ok', sys.argv[1])
except Exception as e:
    print('fail', sys.argv[1], e)
