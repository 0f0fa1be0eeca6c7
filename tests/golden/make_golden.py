"""Generate tests/golden/transform_golden.npz by running the REFERENCE's own
transform.py (pkg/src/permez/transform.py) on seeded blocks.  Run in the
container that has /root/reference; the GPU box only reads the .npz.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from permez import transform as T  # noqa: E402  (the reference module)

rng = np.random.default_rng(20231009)
blocks = []
# 1) the SPEC example block
blocks.append(np.array([[-4.0, 0.5, 8.0, 0.0]], np.float32))
# 2) random blocks over several magnitude regimes, mixed sign, with zeros and sub-floor values
for i, (lo, hi) in enumerate([(-3, 3), (-30, 30), (-37, 38), (-1, 1), (0, 0.5)]):
    e = rng.uniform(lo, hi, (32, 32))
    x = (rng.choice([-1.0, 1.0], (32, 32)) * 10.0 ** e).astype(np.float32)
    x[rng.random((32, 32)) < 0.02] = 0.0
    if i == 2:
        x[0, :5] = np.float32(1e-40)  # subnormal -> reclassified as zero
    blocks.append(x)
# 3) a positive-only lognormal block
blocks.append(np.exp(rng.normal(0, 3, (32, 32))).astype(np.float32))

eps0 = T.float_floor(np.float32)
out = {"eps0": eps0}
b_rs = [1e-2, 1e-3, 1e-4]
for bi, blk in enumerate(blocks):
    z = T.zero_sub_floor_magnitudes(blk, eps0)
    st = T.compute_block_stats(z)
    for ri, b_r in enumerate(b_rs):
        p = T.make_transform_params(st, b_r)
        v = T.forward_map(z, p)
        inv = T.inverse_map(v, p)
        key = f"b{bi}_r{ri}"
        out[key + "_x"] = blk
        out[key + "_params"] = np.array([p.factor_pos, p.factor_neg, p.epsilon0, p.b_r, p.b_a, p.boundary,
                                         p.zero_code_value, p.zero_threshold, p.lg_pos, p.lg_neg])
        out[key + "_fwd"] = np.asarray(v, np.float64)
        out[key + "_inv32"] = np.asarray(inv, np.float64).astype(np.float32)
        out[key + "_b_r"] = np.float64(b_r)
# scalar KATs
p = T.make_transform_params(T.BlockStats(0.5, 8.0, True, True, 4), 0.01)
out["kat_params_0.5_8"] = np.array([p.factor_pos, p.factor_neg, p.b_a, p.boundary, p.zero_code_value])
out["kat_fwd_8"] = np.float64(T.forward_map(8.0, p))
out["kat_fwd_m0.5"] = np.float64(T.forward_map(-0.5, p))
out["kat_inv_2"] = np.float64(T.inverse_map(2.0, p))
p2 = T.make_transform_params(T.BlockStats(1.0, 1.0, False, False, 1), 0.001)
out["kat_factor_neg_1_1"] = np.float64(p2.factor_neg)
p3 = T.make_transform_params(T.BlockStats(1e-30, 1e30, False, False, 2), 0.01)
out["kat_factor_neg_big"] = np.float64(p3.factor_neg)
out["nblocks"] = np.int64(len(blocks))
out["numpy_version"] = np.array(np.__version__)
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "transform_golden.npz")
np.savez_compressed(path, **out)
print("wrote", path, os.path.getsize(path), "bytes")
