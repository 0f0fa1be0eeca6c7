"""Duplex PCIe ceiling of the slab pipeline: total bytes of the C5 e2e call
moved in slabs on two streams with no kernels (H2D a, D2H b concurrently)."""
import sys, time, torch
tot_h2d, tot_d2h = int(float(sys.argv[1]) * 1e9), int(float(sys.argv[2]) * 1e9)
for nsl in (8, 16, 32, 64):
    a, b = tot_h2d // nsl, tot_d2h // nsl
    hs = torch.empty(tot_h2d, dtype=torch.uint8, pin_memory=True); hd = torch.empty(tot_d2h, dtype=torch.uint8, pin_memory=True)
    da = [torch.empty(a, dtype=torch.uint8, device="cuda") for _ in range(3)]
    db = [torch.empty(b, dtype=torch.uint8, device="cuda") for _ in range(2)]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for mode in ("h2d", "d2h", "both"):
        for rep in range(2):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            for i in range(nsl):
                if mode != "d2h":
                    with torch.cuda.stream(s1): da[i % 3].copy_(hs[i * a:(i + 1) * a], non_blocking=True)
                if mode != "h2d":
                    with torch.cuda.stream(s2): hd[i * b:(i + 1) * b].copy_(db[i % 2], non_blocking=True)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"nslabs {nsl:3d} {mode:5s}: {1e3 * dt:7.1f} ms", flush=True)
    del hs, hd, da, db
