"""Benchmark of the B200 PW_REL block compression path (BASELINE.json metric:
"compress/decompress GB/s at PW_REL 1e-2 (1/2/4/8 B200); compression ratio").

Workload: config C5 of BASELINE.json (configs[4], the metric's 1/2/4/8-GPU
configuration, which fits one B200): float32 1024x1024x2048 (8 GiB, 2^31
points) Gaussian random field k^-3, mixed sign, seed 4, generated on the
device (synthetic stand-in: no public dataset), viewed as the 2-D grid
1048576 x 2048 (D18); PW_REL 1e-2, repair_factor 1.0 (every point
|x'-x| <= eps|x|), init_model (Lorenzo) perceptron, 256x256 blocks, 32-row
partitions.  A step = one compress of the field resident in HBM (one at a
time; the 8 GiB input is far larger than the 126 MB L2); decompress is timed
the same way and reported beside it.  N > 1 (torchrun): the SAME field is
sharded by whole block-rows (slowest axis) across the ranks -- strong scaling;
shards exchange only the select_m / codebook histograms (NCCL all-reduce) and
the per-shard sizes (NCCL all-gather).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C5]

Prints ONE JSON line on rank 0.  ``--impl reference`` times the reference
CPU path -- the C restatement in oracle/ (the reference ships no compress
code) -- on all host cores over a fixed block-row subset of
the same field.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0
METRIC = "compress GB/s at PW_REL 1e-2"
EPS0 = 1.1754943508222875e-38
# CPU sample: a contiguous slab of block-rows = 1/64 of C5
SAMPLE_FRACTION = 64


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self._stop, self._t = index, [], threading.Event(), None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and
                          s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def workload(name: str, eps: float):
    from paper_2309_09778_b200 import synthetic
    shape, _, seed, desc = synthetic.CONFIGS[name]
    return (f"{name}: f32 {'x'.join(map(str, shape))} ({np.prod(shape) * 4 / 2**30:.3g} GiB) {desc}, seed {seed}; "
            f"PW_REL {eps:g}, repair 1.0; 256x256 blocks, 32-row partitions, init_model")


def field_2d(name: str, dev):
    """The config's field generated on `dev`, as its 2-D grid view (D18)."""
    from paper_2309_09778_b200 import synthetic
    from paper_2309_09778_b200.pipeline import grid_view_shape
    x = synthetic.generate(name, device=dev)
    (r, c), _ = grid_view_shape(tuple(x.shape))
    return x.reshape(r, c)


def cpu_sample(x2d):
    """The fixed CPU sample: the first 1/64 of the block-rows (whole blocks)."""
    rows = x2d.shape[0]
    nbr = (rows + 255) // 256
    take = max(1, nbr // SAMPLE_FRACTION) * 256
    return x2d[: min(rows, take)]


def bench_config(args, world: int) -> dict:
    """`config` of the JSON line, identical in both arms (--impl ours / reference)."""
    return {"workload": workload(args.config, args.eps),
            "l2": "input 8 GiB >> 126 MB L2 (no flush needed), one field at a time",
            "parallelism": f"shard{world} (whole block-rows)" if world > 1 else "single"}


def oracle_compress_time(xs: np.ndarray, eps: float, reps: int, threads: int):
    from oracle import oracle as O
    cfg = O.OracleConfig(b_r=eps, repair_factor=1.0)
    O.compress(xs, cfg, nthreads=threads)  # warm
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        buf, info = O.compress(xs, cfg, nthreads=threads)
        ts.append(time.perf_counter() - t0)
    return ts, buf, info


def run_reference(args):
    """--impl reference: the reference CPU path (oracle/ restatement, all host
    threads) on the fixed 1/64 block-row sample of the same field."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import torch
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
    x = field_2d(args.config, dev)
    xs = np.ascontiguousarray(cpu_sample(x).cpu().numpy())
    del x
    threads = os.cpu_count() or 1
    ts, buf, _ = oracle_compress_time(xs, args.eps, args.warmup + args.steps, threads)
    ts = ts[args.warmup:] or ts
    t = sum(ts) / len(ts)
    gbs = xs.nbytes / t / 1e9
    sample = (f"first 1/{SAMPLE_FRACTION} of the block-rows of the {args.config} field "
              f"({xs.shape[0]}x{xs.shape[1]} f32, {xs.nbytes / 2**20:.0f} MiB) per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args, args.gpus),  # the same dict as the CUDA arm's line
        "reference_path": "oracle/permez_oracle.c (C restatement of the reference path: the reference ships "
                          "no compress code) + numpy split, OpenMP over blocks",
        "compression_ratio": len(buf) / xs.nbytes,
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5", help="BASELINE config (C5 = the metric's configuration)")
    ap.add_argument("--eps", type=float, default=1e-2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the FP32 perceptron perf-mode measurement")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run this many steps, no JSON timing claims")
    args = ap.parse_args()
    if args.profile_steps == 0:
        args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2309_09778_b200 as P
    from paper_2309_09778_b200 import _native as N
    from paper_2309_09778_b200.sharding import exchange_record_sizes, local_validation_blocks, plan_shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    sharded = world > 1 or bool(os.environ.get("PMZ_BENCH_SHARDED"))
    if sharded:
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)

    def allreduce(t):
        dist.all_reduce(t)

    cfg = P.CompressConfig(rel_error=args.eps, repair_factor=1.0)
    xg = field_2d(args.config, dev)  # every rank builds the same field (same seed), keeps its rows
    grows, C = xg.shape
    plan = plan_shard(grows, C, cfg.block_rows, cfg.block_cols, world, rank)
    x = xg[plan.row0: plan.row1]
    xs_host = np.ascontiguousarray(cpu_sample(xg).cpu().numpy()) if (rank == 0 and world == 1) else None
    d_val = torch.as_tensor(local_validation_blocks(plan, cfg.sample_rate, cfg.seed), dtype=torch.int64, device=dev)
    codec = P.Codec(dev)
    nblk = plan.nblocks
    offs = torch.empty(nblk + 1, dtype=torch.int64, device=dev)

    def compress_once(ev=None):
        buf, info = codec.compress_staged(x, cfg, block_row0=plan.block_row0, global_rows=grows,
                                          allreduce=allreduce if sharded else None, block_offsets=offs, events=ev,
                                          d_val=d_val)
        if sharded:  # the final NCCL gather of per-shard sizes -> container offsets
            exchange_record_sizes(info.nbytes - info.header_bytes, device=dev)
        return buf, info

    buf, info = compress_once()
    full_t = buf.cpu()
    full = full_t.numpy()
    hdr = P.Codec.parse_header(full)
    hdr.rows = x.shape[0]  # this shard's grid (the header carries the global rows)
    hdr.nblocks = nblk
    dbuf = buf.clone()
    doffs = offs.clone()
    y = torch.empty(x.shape, dtype=torch.float32, device=dev)

    def decompress_once(ev=None):
        return codec.decompress_device(dbuf, hdr, doffs, out=y, events=ev)

    # correctness guard on the benchmarked data: every point within the bound, zeros exact
    decompress_once()
    torch.cuda.synchronize()
    max_rel, zeros_ok = 0.0, True
    for r0 in range(0, x.shape[0], 65536):
        xa, ya = x[r0: r0 + 65536].double(), y[r0: r0 + 65536].double()
        xz = torch.where(xa.abs() <= EPS0, torch.zeros_like(xa), xa)
        nz = xz != 0
        if bool(nz.any()):
            max_rel = max(max_rel, float(((ya - xz).abs() / xz.abs())[nz].max()))
        zeros_ok &= bool((ya[~nz] == 0).all())
    assert max_rel <= args.eps and zeros_ok, (max_rel, zeros_ok)
    del xa, ya, xz, nz

    for _ in range(args.warmup):
        compress_once()
        decompress_once()
    torch.cuda.synchronize()
    if args.profile_steps:
        for _ in range(args.profile_steps):
            compress_once()
            decompress_once()
        torch.cuda.synchronize()
        return 0

    K = args.steps
    c_ms, d_ms, c_stage, d_stage = [], [], [], []
    launches = 0
    sampler = ClockSampler(local)
    with sampler:
        for _ in range(K):
            if sharded:
                dist.barrier()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(codec.stage_names_compress) + 1)]
            bufk, infok = compress_once(ev)  # synchronises (status read-back)
            torch.cuda.synchronize()
            c_ms.append(ev[0].elapsed_time(ev[-1]))
            c_stage.append([ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)])
            launches += infok.launches
            if sharded:
                dist.barrier()
            torch.cuda.synchronize()
            dev_ = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            decompress_once(dev_)
            torch.cuda.synchronize()
            d_ms.append(dev_[0].elapsed_time(dev_[2]))
            d_stage.append([dev_[0].elapsed_time(dev_[1]), dev_[1].elapsed_time(dev_[2])])
            launches += codec.last_decompress_launches
    assert infok.nbytes == info.nbytes

    # whole-job time = max over ranks of the per-step device time
    tot = torch.tensor([sum(c_ms), sum(d_ms)], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    c_step, d_step = float(tot[0]) / K, float(tot[1]) / K
    nb_t = torch.tensor([float(x.numel() * 4), float(info.nbytes - info.header_bytes)], dtype=torch.float64,
                        device=dev)
    if sharded:
        dist.all_reduce(nb_t)
    bytes_all = float(nb_t[0])
    cr = (float(nb_t[1]) + info.header_bytes) / bytes_all
    comp_gbs = bytes_all / (c_step / 1e3) / 1e9
    dec_gbs = bytes_all / (d_step / 1e3) / 1e9

    # FP32 perceptron perf mode (north star; container version 2): the same
    # field and timing, plus the perceptron-rounding mismatch counters against
    # the FP64 path (final codes and balance points compared position by
    # position through the code dumps) and the bound on every point
    fp32 = None
    if not args.no_fp32:
        from paper_2309_09778_b200.pipeline import code_mismatches
        cfg32 = P.CompressConfig(rel_error=args.eps, repair_factor=1.0, precision="fp32")
        offs32 = torch.empty(nblk + 1, dtype=torch.int64, device=dev)

        def compress32(ev=None, c=cfg32):
            b, i = codec.compress_staged(x, c, block_row0=plan.block_row0, global_rows=grows,
                                         allreduce=allreduce if sharded else None, block_offsets=offs32, events=ev,
                                         d_val=d_val)
            if sharded:
                exchange_record_sizes(i.nbytes - i.header_bytes, device=dev)
            return b, i

        b32, i32 = compress32()
        h32 = P.Codec.parse_header(b32[: min(int(i32.nbytes), 1 << 20)].cpu().numpy())
        h32.rows, h32.nblocks = x.shape[0], nblk
        db32, do32 = b32.clone(), offs32.clone()
        y32 = torch.empty(x.shape, dtype=torch.float32, device=dev)
        codec.decompress_device(db32, h32, do32, out=y32)
        torch.cuda.synchronize()
        mr32 = 0.0
        for r0 in range(0, x.shape[0], 65536):
            xa, ya = x[r0: r0 + 65536].double(), y32[r0: r0 + 65536].double()
            xz = torch.where(xa.abs() <= EPS0, torch.zeros_like(xa), xa)
            nz = xz != 0
            if bool(nz.any()):
                mr32 = max(mr32, float(((ya - xz).abs() / xz.abs())[nz].max()))
            assert bool((ya[~nz] == 0).all())
        assert mr32 <= args.eps, mr32
        del xa, ya, xz, nz
        c32_ms, d32_ms = [], []
        for it in range(1 + K):
            if sharded:
                dist.barrier()
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(codec.stage_names_compress) + 1)]
            compress32(ev)
            torch.cuda.synchronize()
            dv = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            codec.decompress_device(db32, h32, do32, out=y32, events=dv)
            torch.cuda.synchronize()
            if it:  # the first pass warms up
                c32_ms.append(ev[0].elapsed_time(ev[-1]))
                d32_ms.append(dv[0].elapsed_time(dv[2]))
        t32 = torch.tensor([sum(c32_ms) / K, sum(d32_ms) / K], dtype=torch.float64, device=dev)
        # mismatch counters: one compress of each precision into a code dump
        nd = codec.code_dump_numel(x.shape, cfg)
        dmp = {}
        for prec in ("fp64", "fp32"):
            dmp[prec] = torch.full((nd,), 0xFFFE, dtype=torch.int32, device=dev).to(torch.uint16)
            cd = P.CompressConfig(rel_error=args.eps, repair_factor=1.0, precision=prec, code_dump=dmp[prec])
            compress32(c=cd)
        cm = code_mismatches(dmp["fp64"], dmp["fp32"])
        del dmp
        cnt = torch.tensor([cm["codes"], cm["code_mismatches"], cm["balance_mismatches"],
                            int(i32.nbytes - i32.header_bytes), int(i32.nbal)], dtype=torch.float64, device=dev)
        if sharded:
            dist.all_reduce(t32, op=dist.ReduceOp.MAX)
            dist.all_reduce(cnt)
        cr32 = (float(cnt[3]) + i32.header_bytes) / bytes_all
        fp32 = {"value": bytes_all / (float(t32[0]) / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": float(t32[0]),
                "decompress": {"value": bytes_all / (float(t32[1]) / 1e3) / 1e9, "unit": "GB/s",
                               "ms_per_step": float(t32[1])},
                "container_version": int(h32.version), "compression_ratio": cr32,
                "cr_delta_vs_fp64": (cr32 - cr) / cr, "max_rel_err": mr32,
                "codes": int(cnt[0]), "code_mismatches_vs_fp64": int(cnt[1]),
                "code_mismatch_frac": float(cnt[1]) / max(1.0, float(cnt[0])),
                "balance_point_mismatches_vs_fp64": int(cnt[2]), "balance_count": int(cnt[4]),
                "note": "float32 surfaces, predictor, quantizer and recurrence; every point within the bound"}
        del y32, db32, b32

    # e2e through the public host-to-host API (hostpipe.HostPipeline) with
    # pinned host buffers, every step: the field goes host->device in slabs of
    # whole block-rows, each slab is compressed and its records go device->host
    # while the next slab uploads (validation blocks first, so m and the
    # codebook exist before the first slab is encoded); the reverse for
    # decompress (block index walk on the host inside the timed region).
    # Wall clock around the call with a device synchronise on both sides.
    e2e_c = e2e_d = None
    if not args.no_e2e:
        pipe = P.HostPipeline(codec)
        h_in = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        h_in.copy_(x)
        h_out = torch.empty(int(info.nbytes) + (1 << 20), dtype=torch.uint8, pin_memory=True)
        h_y = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
        e_ms, ed_ms = [], []
        for it in range(1 + max(2, min(K, 3))):
            if sharded:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            n2, i2 = pipe.compress(h_in, cfg, h_out, block_row0=plan.block_row0, global_rows=grows,
                                   allreduce=allreduce if sharded else None)
            if sharded:
                exchange_record_sizes(i2.nbytes - i2.header_bytes, device=dev)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            bi, bo = pipe.last_h2d_bytes, pipe.last_d2h_bytes
            if sharded:
                dist.barrier()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            pipe.decompress(h_out[:n2], h_y, shard_rows=x.shape[0] if sharded else None)
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            if it:  # the first pass allocates the slab buffers
                e_ms.append(1e3 * (t1 - t0))
                ed_ms.append(1e3 * (t3 - t2))
                di, do_ = pipe.last_h2d_bytes, pipe.last_d2h_bytes
        assert n2 == info.nbytes and torch.equal(h_out[:n2], full_t), "host pipeline container differs"
        assert torch.equal(h_y.view(torch.int32), y.cpu().view(torch.int32)), "host pipeline grid differs"
        et = torch.tensor([sum(e_ms) / len(e_ms), sum(ed_ms) / len(ed_ms)], dtype=torch.float64, device=dev)
        if sharded:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_c = {"value": bytes_all / (float(et[0]) / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": float(et[0]),
                 "ms_each": [round(v, 2) for v in e_ms], "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(bo),
                 "api": "HostPipeline.compress: pinned host field -> pinned host container, slabs of whole "
                        "block-rows, copies overlapped with the kernels; container identical to the device call"}
        e2e_d = {"value": bytes_all / (float(et[1]) / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": float(et[1]),
                 "ms_each": [round(v, 2) for v in ed_ms], "h2d_bytes_per_step": int(di), "d2h_bytes_per_step": int(do_),
                 "api": "HostPipeline.decompress: pinned host container -> pinned host grid (block index walk "
                        "on the host, slabs, copies overlapped); grid identical to the device call"}
        del h_in, h_out, h_y

    # roofline: algorithmic bytes per element 4 + 4 CR
    # (compress reads the f32 field and writes the container; decompress the
    # reverse) x elements processed, divided by the event-timed duration of
    # the dominant stage (and of the whole pipeline)
    hbm, peak_kind = peaks()
    n_local = x.numel()
    alg = 4.0 + 4.0 * cr
    cs = np.mean(np.array(c_stage), axis=0)
    ds = np.mean(np.array(d_stage), axis=0)
    names_c = codec.stage_names_compress
    names_d = codec.stage_names_decompress
    ic, id_ = int(np.argmax(cs)), int(np.argmax(ds))

    def roof(ms, what):
        ach = alg * n_local / (ms / 1e3) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "kernel": what, "ms": ms, "alg_bytes_per_elem": alg, "peak_kind": peak_kind}

    # DRAM bytes per launch of the dominant kernels from the committed ncu
    # capture of this configuration (tools/profile_round.sh -> profiles/)
    tr = {}
    tr_path = os.path.join(ROOT, "profiles", "traffic_latest.json")
    if os.path.exists(tr_path) and world == 1:
        try:
            tr = json.load(open(tr_path))
        except Exception:
            tr = {}
    roof_c = roof(float(cs[ic]), names_c[ic])
    roof_c["traffic"] = tr.get("compress_dominant_bytes_per_launch")
    roof_c["traffic_kernel"] = tr.get("compress_dominant_kernel")
    roof_c["pipeline"] = roof(c_step, "whole compress")
    roof_d = roof(float(ds[id_]), names_d[id_])
    roof_d["traffic"] = tr.get("decompress_dominant_bytes_per_launch")
    roof_d["traffic_kernel"] = tr.get("decompress_dominant_kernel")
    roof_d["pipeline"] = roof(d_step, "whole decompress")

    # what actually bounds the dominant kernels: instruction
    # issue.  Executed warp instructions per launch from the committed ncu
    # capture, divided by the live stage time, against SMs x 4 schedulers x
    # the SM clock sampled during the timed region.
    def issue(roofd, key, ms):
        wi = tr.get(key)
        mhz = sampler.summary().get("sm_mhz")
        if not wi or not mhz:
            return
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        peak = sms * 4 * mhz * 1e6
        roofd["issue"] = {"warp_inst_per_launch": wi, "achieved_warp_inst_per_s": wi / (ms / 1e3),
                          "peak_warp_inst_per_s": peak, "frac": wi / (ms / 1e3) / peak,
                          "note": "instruction-issue bound (ncu instruction count of the dominant kernel / live "
                                  "stage time); the HBM fraction above is the contract's figure"}
    issue(roof_c, "compress_dominant_warp_inst_per_launch", float(cs[ic]))
    issue(roof_d, "decompress_dominant_warp_inst_per_launch", float(ds[id_]))

    # CPU baseline + parity on the same sample (rank 0, N = 1): the oracle
    # restatement of the reference path on all host cores, and the CUDA path
    # on the identical sample -- containers must be byte-identical
    cpu_base, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and xs_host is not None:
        threads = os.cpu_count() or 1
        try:
            ts, ref, rinfo = oracle_compress_time(xs_host, args.eps, 2, threads)
            cpu_base = {"value": xs_host.nbytes / min(ts) / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
                        "sample": f"first 1/{SAMPLE_FRACTION} of the block-rows ({xs_host.shape[0]}x{xs_host.shape[1]}"
                                  f" f32, {xs_host.nbytes / 2**20:.0f} MiB), oracle restatement, OpenMP over blocks, "
                                  "best of 2"}
            gbuf, ginfo = codec.compress_device(torch.from_numpy(xs_host).to(dev), cfg)
            g = gbuf.cpu().numpy().tobytes()
            a, b = np.frombuffer(g, np.uint8), np.frombuffer(ref, np.uint8)
            n = min(a.size, b.size)
            parity = {"sample": "the CPU sample above", "container_identical": g == ref,
                      "differing_bytes": int((a[:n] != b[:n]).sum()) + abs(a.size - b.size),
                      "m": [ginfo.m, rinfo["m"]], "balance_count": [ginfo.nbal, rinfo["nbal"]],
                      "repairs": [ginfo.nrepair, rinfo["nrepair"]],
                      "cr_delta": (len(g) - len(ref)) / len(ref)}
        except Exception as ex:  # reported, never required
            cpu_base = {"value": None, "unit": "GB/s", "cores": threads, "kind": "port", "sample": f"failed: {ex!r}"}

    clocks = sampler.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": comp_gbs, "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": c_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, world),
            "compression_ratio": cr, "max_rel_err": max_rel, "m": info.m,
            "decompress": {"value": dec_gbs, "unit": "GB/s", "ms_per_step": d_step, "roofline": roof_d,
                           "e2e": e2e_d},
            "e2e": e2e_c,
            "roofline": roof_c,
            "stages_ms": {"compress": dict(zip(names_c, cs.tolist())), "decompress": dict(zip(names_d, ds.tolist()))},
            "parity": parity,
            "fp32_mode": fp32,
            "cpu_baseline": cpu_base,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
