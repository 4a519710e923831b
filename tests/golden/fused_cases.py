"""Fused distributed golden cases (shared by make_golden.py and the GPU tests):
(name, flags, gamma); alpha 0.5, beta -1, delta 1, eta 0.3, block width 2."""
from paper_1507_08101_b200 import sellkit as sk

FUSED = [
    ("f1", sk.AXPBY | sk.SHIFT | sk.DOT_YY | sk.DOT_XY | sk.DOT_XX | sk.CHAIN_AXPBY, [0.25]),
    ("f2", sk.VSHIFT | sk.DOT_YY | sk.CHAIN_AXPBY, [0.25, -0.75]),
]
