"""Rare-path reason counters of k_c_main (A/B build with -DPMZ_CSTATS).
Build here:  python tools/cstats.py build      (writes tools/micro/libpermez_cstats.so)
Run on GPU:  python tools/cstats.py run C5"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tools", "micro", "libpermez_cstats.so")
NAMES = ["rare lanes (c_rare)", "certain balance points"]
if sys.argv[1] == "build":
    sys.path.insert(0, ROOT)
    from paper_2309_09778_b200 import build as B
    cmd = ["/usr/local/cuda/bin/nvcc", *B.NVCC_FLAGS, "-DPMZ_CSTATS", "-o", SO, os.path.join(B.CSRC, "capi.cu")]
    subprocess.run(cmd, check=True)
else:
    os.environ["PMZ_LIB_PATH"] = SO
    sys.path.insert(0, ROOT)
    import torch
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import synthetic
    x = synthetic.generate(sys.argv[2], device="cuda").contiguous()
    codec = P.Codec("cuda:0")
    buf, info = codec.compress_device(x, P.CompressConfig(rel_error=1e-2, repair_factor=1.0))
    torch.cuda.synchronize()
    lib = ctypes.CDLL(SO)
    arr = (ctypes.c_uint64 * 16)()
    lib.pmz_cstats_read(arr)
    n = x.numel()
    print(f"{sys.argv[2]}: n={n} nbal={info.nbal} nrepair={info.nrepair}")
    for i, nm in enumerate(NAMES):
        print(f"  {nm:24s} {arr[i]:14d}  {arr[i] / n * 100:8.4f}% of elements")
