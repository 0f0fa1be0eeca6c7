"""Quick GPU-vs-oracle parity probe (development tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
import paper_2309_09778_b200 as P
from paper_2309_09778_b200 import synthetic as S

def diff_report(a: bytes, b: bytes):
    n = min(len(a), len(b))
    aa = np.frombuffer(a[:n], np.uint8); bb = np.frombuffer(b[:n], np.uint8)
    d = np.nonzero(aa != bb)[0]
    return f"len {len(a)} vs {len(b)}; first diff at {d[0] if d.size else None}; ndiff {d.size}"

cases = [("C1", None, 1e-2, 1.0), ("C2", (300, 520), 1e-2, 1.0), ("C2", None, 1e-2, 1.0), ("C2", None, 1e-3, 1.0),
         ("C2", None, 1e-2, 1.5), ("C4", (20, 100, 130), 1e-4, 1.0), ("C3", (64, 64, 96), 1e-2, 1.0)]
codec = P.Codec("cuda:0")
for name, shape, br, rf in cases:
    x = S.generate(name, shape=shape).numpy()
    cfg = P.CompressConfig(rel_error=br, repair_factor=rf)
    t = time.time()
    dbuf, info = codec.compress_device(torch.from_numpy(x).cuda(), cfg)
    torch.cuda.synchronize(); tg = time.time() - t
    g = dbuf.cpu().numpy().tobytes()
    t = time.time()
    r, rinfo = O.compress(x, O.OracleConfig(b_r=br, repair_factor=rf))
    to = time.time() - t
    ok = g == r
    print(f"{name} {x.shape} eps={br} rf={rf}: compress {'OK' if ok else 'MISMATCH'} m={info.m}/{rinfo['m']} "
          f"nbal={info.nbal}/{rinfo['nbal']} rep={info.nrepair}/{rinfo['nrepair']} CR={len(g)/x.nbytes:.4f} "
          f"gpu {tg*1e3:.1f}ms cpu {to*1e3:.1f}ms", flush=True)
    if not ok:
        print("   ", diff_report(g, r), flush=True)
    try:
        y = P.decompress(r, device="cuda:0")
        yo = O.decompress(r)
        same = np.array_equal(y.reshape(-1).view(np.uint32), yo.reshape(-1).view(np.uint32))
        print(f"    decompress {'OK' if same else 'MISMATCH'}", flush=True)
    except Exception as e:
        print("    decompress error", repr(e), flush=True)
