#!/usr/bin/env python
"""One C5 construction (400^3 7-pt, SELL-32-256) -- for kernel launch lists of the build."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1507_08101_b200 import sellkit
sk = sellkit.load()
crs = sk.crs_stencil(7, 400)
torch.cuda.synchronize()
A = crs.build(32, 256)
