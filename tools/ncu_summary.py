"""Summarise ncu --set full reports: duration, DRAM bytes, throughput, pipe
utilisation and stall reasons per kernel.  Optionally writes the DRAM traffic
of k_compress_ws to profiles/traffic_latest.json (read by bench.py for
roofline.traffic).

usage: python tools/ncu_summary.py OUT.txt REPORT.ncu-rep [REPORT ...]"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        yield {h: (v, u) for h, v, u in zip(hdr, r, units)}


def stalls(rep, kernel):
    sys.path.insert(0, os.path.dirname(__file__))
    out = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_hot.py"), rep, kernel, "0"],
                         capture_output=True, text=True).stdout
    return "\n".join(line for line in out.splitlines() if line.startswith(("samples", "stalls")))


def main():
    dst, reps = sys.argv[1], sys.argv[2:]
    lines, traffic, insts = [], {}, {}
    for rep in reps:
        for k in raw(rep):
            name = k.get("Kernel Name", ("?", ""))[0]
            short = name.split("(")[0]
            lines.append(f"== {short}  [{os.path.basename(rep)}]")
            for key in KEYS:
                if key in k:
                    v, u = k[key]
                    lines.append(f"   {key:62s} {v} {u}")
            st = stalls(rep, short.replace("void ", "").split("::")[-1].split("<")[0])
            lines.append("   " + st.replace("\n", "\n   "))
            for ln in st.splitlines():  # "samples N instructions M": executed warp instructions of the launch
                w = ln.split()
                if len(w) >= 4 and w[0] == "samples" and w[2] == "instructions":
                    insts[short] = int(w[3])
            try:
                rd = float(k["dram__bytes_read.sum"][0].replace(",", ""))
                wr = float(k["dram__bytes_write.sum"][0].replace(",", ""))
                unit = k["dram__bytes_read.sum"][1]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                traffic[short] = (rd + wr) * scale
            except (KeyError, ValueError):
                pass
    open(dst, "w").write("\n".join(lines) + "\n")
    tr = {}
    for name, b in traffic.items():
        if "k_c_main<3, 0, 1>" in name:  # the dominant compress kernel (bench roofline.traffic)
            tr["compress_dominant_bytes_per_launch"] = b
            tr["compress_dominant_kernel"] = name
            tr["compress_dominant_warp_inst_per_launch"] = insts.get(name)
        if "k_d_recon" in name:  # the dominant decompress kernel
            tr["decompress_dominant_bytes_per_launch"] = b
            tr["decompress_dominant_kernel"] = name
            # the bench's dominant decompress stage runs the decoder and the reconstruct kernel
            dec = sum(v for k2, v in insts.items() if "k_d_decode" in k2)
            tr["decompress_dominant_warp_inst_per_launch"] = (insts.get(name) or 0) + dec
    if tr:
        tr["source"] = os.path.basename(dst)
        path = os.path.join(os.path.dirname(__file__), "..", "profiles", "traffic_latest.json")
        json.dump(tr, open(path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
