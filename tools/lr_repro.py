"""Repro of one LR fuzz case (debugging aid): python tools/lr_repro.py [t]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from tests.test_gpu_parity import fuzz_case
from paper_2111_02925_b200 import sz3g
t = int(sys.argv[1]) if len(sys.argv) > 1 else 0
xh, eb, mode, R = fuzz_case(t)
x = torch.from_numpy(np.ascontiguousarray(xh.reshape((1,) * (3 - xh.ndim) + xh.shape))).cuda()
res = sz3g.lr_compress(x, eb, mode, R, outlier_cap=x.numel())
torch.cuda.synchronize()
print("ok", x.shape, int(res.lr_flags.sum()), res.n_outliers)
