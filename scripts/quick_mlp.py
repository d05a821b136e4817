#!/usr/bin/env python3
"""Quick tf32x3 MLP parity probe (run under `timeout`): python scripts/quick_mlp.py [n ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2309_06619_b200 as rt  # noqa: E402
from oracle.mlp import mlp_abs_pass, mlp_predict  # noqa: E402
from rtgen import configs, mlp_weights  # noqa: E402

ctx = rt.Context(configs.read_lexicon(), 0)
ws, bs = mlp_weights(7)
ctx.set_mlp(ws, bs)
ctx.set_mlp_precision(os.environ.get("MODE", "tf32x3"))
for n in [int(a) for a in sys.argv[1:]] or [1, 129, 5000]:
    rng = np.random.default_rng(n)
    f = np.zeros((n, 8), np.uint16)
    f[:, :7] = rng.integers(0, 60, (n, 7))
    u = ctx.predict_mlp(torch.from_numpy(f.view(np.int16)).cuda()).cpu().numpy().astype(np.float64)
    want = mlp_predict(f, ws, bs)
    r = np.abs(u - want) / mlp_abs_pass(f, ws, bs)
    print(n, "max err / abs pass (units of 2^-24):", float(r.max() * 2 ** 24), "worst", int(r.argmax()), u[:3], want[:3],
          flush=True)
