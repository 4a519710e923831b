import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1507_08101_b200 import sellkit
sk = sellkit.load()
N = 20_000_000
m = k = int(sys.argv[1])
V, W, X = sk.densemat(N, m), sk.densemat(N, k), sk.densemat(m, k)
V.fill_hash(1); W.fill_hash(2); X.fill_hash(3)
one, zero = np.array([1.0]), np.array([0.0])
for _ in range(2):
    sk.call("sellkit_tsmm", W, V, X, one.ctypes.data, zero.ctypes.data)
    sk.call("sellkit_tsmttsm", X, V, W, one.ctypes.data, zero.ctypes.data, 0)
