#!/usr/bin/env python
"""Per-launch CUDA-event times of back-to-back C5 SpMMVs (400^3, w=8), with nvidia-smi
clock/power samples taken during the run: shows the burst-to-sustained transition."""
import json
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_08101_b200 import sellkit  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
sk = sellkit.load()
stream = torch.cuda.ExternalStream(sk.stream())
A = sk.crs_stencil(7, 400).build(32, 256)
N = 400 ** 3
x, y = sk.densemat(N, 8), sk.densemat(N, 8)
x.fill_hash(42)
lines = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active",
                         "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
th = threading.Thread(target=lambda: [lines.append((time.time(), l.strip())) for l in proc.stdout], daemon=True)
th.start()
time.sleep(0.5)
sk.set_sync(False)
evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
t0 = time.time()
evs[0].record(stream)
for i in range(reps):
    sk.spmv(y, A, x)
    evs[i + 1].record(stream)
sk.synchronize()
t1 = time.time()
time.sleep(0.3)
proc.terminate()
ts = [evs[i].elapsed_time(evs[i + 1]) for i in range(reps)]
print(json.dumps({"lib": os.environ.get("SELLKIT_B200_LIB", "default"), "ms": [round(t, 4) for t in ts]}))
print(json.dumps({"smi_during": [l for (t, l) in lines if t0 - 0.05 <= t <= t1 + 0.05]}))
