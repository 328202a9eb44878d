"""Device logistic-regression fit time (GPU box): n random Hadamard-like
rows of dimension d, E epochs of the reference's mini-batch descent
(evaluate.py:128-140) through train_logreg_device.

    N=2000000 D=128 EPOCHS=10 python scripts/bench_logreg.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2008_12336_b200 as gb  # noqa: E402
from paper_2008_12336_b200 import evaluate as ev  # noqa: E402

n = int(os.environ.get("N", "2000000"))
d = int(os.environ.get("D", "128"))
epochs = int(os.environ.get("EPOCHS", "10"))
g = torch.Generator(device="cuda").manual_seed(0)
X = (torch.rand(n, d, device="cuda", generator=g) - 0.5) * 0.02
y = (torch.rand(n, device="cuda", generator=g) < 0.5).to(torch.int8)
X[y == 1] += 0.001
f = ev.DeviceFeatureSet(rows=X.contiguous(), labels=y)
cfg = gb.LogRegConfig(epochs=epochs, seed=1)
gb.train_logreg_device(f, gb.LogRegConfig(epochs=1, seed=1))
torch.cuda.synchronize()
t0 = time.perf_counter()
m = gb.train_logreg_device(f, cfg)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
steps = epochs * -(-n // cfg.batch_size)
print(json.dumps({"n": n, "d": d, "epochs": epochs, "s": dt, "us_per_step": dt / steps * 1e6,
                  "w0": float(m.weights[0]), "b": m.bias}), flush=True)
