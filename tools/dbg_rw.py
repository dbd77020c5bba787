"""Locate stencil addressing errors of a register-blocking variant (ADP_RW env):
delta image through a delta kernel must come back unchanged."""
import numpy as np
import paper_2502_09758_b200 as adp

for shape, k in [((24, 20, 3), 5), ((24, 20, 1), 5), ((64, 64, 1), 3)]:
    kern = np.zeros((k, k, shape[2])); kern[k // 2, k // 2, :] = 1.0
    op = adp.ConvOperator(adp.Kernel(kern, adp.DEPTHWISE2D), shape)
    bad = 0
    for (h, w, c) in [(0, 0, 0), (3, 5, shape[2] - 1), (10, 7, 0)]:
        x = np.zeros(shape); x[h, w, c] = 1.0
        y = op.apply(x)
        nz = np.argwhere(y != 0)
        if not np.array_equal(y, x):
            bad += 1
            print(shape, k, "delta at", (h, w, c), "-> nonzeros", nz[:6].tolist(), y[tuple(nz[0])] if len(nz) else None)
    x = np.random.default_rng(0).random(shape)
    y = op.apply(x)
    print(shape, k, "identity ok" if np.array_equal(y, x) else f"identity max err {np.abs(y - x).max()}", "bad deltas", bad)
