"""Decompress round trips on tiny shapes; prints the CUDA error on failure."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2309_09778_b200 as P
for shape in [tuple(int(v) for v in sys.argv[1].split("x"))]:
    x = (np.random.default_rng(sum(shape)).normal(0, 1, shape) * 10).astype(np.float32)
    try:
        buf = P.compress(x, rel_error=1e-2, repair_factor=1.0, device="cuda:0")
        y = P.decompress(buf, device="cuda:0")
        print(shape, "ok", np.abs(y - x).max())
    except Exception as e:
        print(shape, "FAIL", e)
        try:
            torch.cuda.synchronize()
        except Exception as e2:
            print("  cuda:", e2)
        break
