"""Dump a mid-size irradiance matrix (GPU-assembled) as .npy for CPU-side
solver experiments (development tool; tests never use it).

usage: python tools/dump_matrix.py out.npy [edge_m] [col_step]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_14137_b200 import uvd  # noqa: E402
from synth import configs, ward  # noqa: E402

out = sys.argv[1]
e = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
step = int(sys.argv[3]) if len(sys.argv) > 3 else 8
sc = uvd.Scene(ward.ward(0, 3, e))
lam, _ = sc.vantage(configs.FLOAT_OPTS)
cols = list(range(0, lam.shape[0], step))
A = sc.irradiance(lam, cols=cols)["A"][:, :sc.N].T.contiguous().cpu().numpy()  # (N, K)
np.savez_compressed(out, A=A.astype(np.float32))
print(out, A.shape, (A.sum(1) == 0).mean())
