#!/bin/bash
# Run on the GPU box (gpurun): GPU parity subset, then one ncu --set full
# capture of the kernel matching $1 at C5 (tools/scale_prof.py), then the
# event-timed C5 bench without the optional legs.
#   gpurun -- 'bash tools/kern_iter.sh k_d_decode name'
set -u
K=${1:-k_d_decode}; NAME=${2:-iter}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fp32_mode.py -x -q > gpurun_out/gputest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/gputest.log
python tools/scale_prof.py C5 > gpurun_out/plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:"$K" -c 1 \
  -o gpurun_out/$NAME python tools/scale_prof.py C5 > gpurun_out/ncu_$NAME.log 2>&1
echo "ncu rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 --no-fp32 --no-cpu-baseline --no-e2e > gpurun_out/bench_$NAME.log 2>&1
echo "bench rc=$?"
python - "$NAME" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print("compress", round(d["value"], 1), "GB/s", "decompress", round(d["decompress"]["value"], 1), "GB/s")
for k, v in d["stages_ms"].items():
    print(k, {a.split(" ")[0]: round(b, 3) for a, b in v.items()})
PY
