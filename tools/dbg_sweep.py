import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2007_03576_b200 as hq
from hqr_inputs import make, random_case
flags = int(sys.argv[1]); n=int(sys.argv[2]); ns=int(sys.argv[3]); win=int(sys.argv[4])
hq.setup(0, flags=flags)
H0, Z0, re, im = random_case(1, n, ns)
Hd, Zd = hq.to_device(H0), hq.to_device(Z0)
try:
    hq.sweep(Hd, Zd, 0, n-1, re, im, win)
    print('ok', flags, n, ns, win)
except Exception as e:
    print('fail', flags, n, ns, win, e)
